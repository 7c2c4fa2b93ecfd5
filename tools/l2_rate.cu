// l2_rate.cu -- per-SM read rate from an L2-resident buffer (tooling): G CTAs of 256 or
// 512 threads each stream their own 1 MB slice of an 8 MB buffer (resident in the
// 126 MB L2 after a warm pass) with U 16-byte loads in flight per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_rate tools/l2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U, int T>
__global__ void __launch_bounds__(T, 1) stream(const double2* __restrict__ a, size_t per_cta, int reps,
                                               double* out, long long* cyc) {
  const double2* p = a + (size_t)(blockIdx.x % 8) * per_cta;
  double s = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (size_t i = threadIdx.x; i < per_cta; i += (size_t)T * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = i + (size_t)u * T < per_cta ? __ldg(p + i + (size_t)u * T) : make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (s == 12345.0) out[0] = s;
}

template <int U, int T>
void run(int G) {
  const size_t per = (1 << 20) / 16;  // 1 MB per CTA slice (double2 elements)
  double2* a;
  double* o;
  long long* c;
  cudaMalloc(&a, per * 8 * 16);
  cudaMemset(a, 0, per * 8 * 16);
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8 * 1024);
  stream<U, T><<<G, T>>>(a, per, 1, o, c);
  cudaDeviceSynchronize();
  const int reps = 8;
  stream<U, T><<<G, T>>>(a, per, reps, o, c);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, c, 8 * G, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < G; ++i) avg += h[i];
  avg /= G;
  printf("G=%d T=%d U=%d: %.1f B/clk per SM (%s)\n", G, T, U, (double)per * 16 * reps / avg,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(a);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  for (int G : {8, 80, 148}) {
    run<4, 256>(G);
    run<8, 256>(G);
    run<16, 256>(G);
    run<8, 512>(G);
    run<16, 512>(G);
  }
  return 0;
}
