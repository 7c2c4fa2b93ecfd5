// sort_rate.cu -- micro-benchmark of the latency kernel's block bitonic sort (tooling)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kLT = 256;
constexpr int kLLive = 1024;
// bitonic sort of (key, val)[0, total) ascending by key, in place, one CTA; element
// e = r * kLT + tid lives in registers (r < 4: total <= 4 kLT); partners within a warp
// are exchanged by shuffles, across warps through shared memory (double-buffered with
// buf, 2 * 4 kLT words), across r inside the thread; padding keys are +inf
__device__ void lat_sort(uint64_t* key, double* val, uint64_t* buf, int total, int n2, int tid, int lane) {
  constexpr int NR = kLLive / kLT;
  static_assert(NR == 4, "four elements per thread");
  const int nr = (n2 + kLT - 1) / kLT;
  uint64_t K[NR];
  double V[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int e = r * kLT + tid;
    K[r] = e < total ? key[e] : ~0ull;
    V[r] = e < total ? val[e] : 0.0;
  }
  int pb = 0;
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= kLT) {  // partner in the same thread: j = kLT pairs (0,1), (2,3); 2 kLT (0,2), (1,3)
        auto cx = [&](uint64_t& k0, double& v0, uint64_t& k1, double& v1, int r) {
          const bool asc = ((r * kLT + tid) & k) == 0;
          const bool sw = (k0 > k1) == asc;
          const uint64_t tk = k0;
          const double tv = v0;
          k0 = sw ? k1 : k0;
          k1 = sw ? tk : k1;
          v0 = sw ? v1 : v0;
          v1 = sw ? tv : v1;
        };
        if (j == kLT) {
          cx(K[0], V[0], K[1], V[1], 0);
          if (nr > 2) cx(K[2], V[2], K[3], V[3], 2);
        } else {
          cx(K[0], V[0], K[2], V[2], 0);
          cx(K[1], V[1], K[3], V[3], 1);
        }
      } else if (j >= 32) {  // partner in another warp
        uint64_t* wk = pb ? key : buf;
        double* wv = pb ? val : reinterpret_cast<double*>(buf + kLLive);
        pb ^= 1;
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (r < nr) {
            wk[r * kLT + tid] = K[r];
            wv[r * kLT + tid] = V[r];
          }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (r < nr) {
            const int e = r * kLT + tid, f = e ^ j;
            const uint64_t pk = wk[f];
            const double pv = wv[f];
            const bool take_min = ((e & j) == 0) == ((e & k) == 0);
            const bool sw = take_min ? pk < K[r] : pk > K[r];  // selects, no branch
            K[r] = sw ? pk : K[r];
            V[r] = sw ? pv : V[r];
          }
      } else {  // partner in this warp
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (r < nr) {
            const int e = r * kLT + tid;
            const uint64_t pk = __shfl_xor_sync(0xffffffffu, K[r], j);
            const double pv = __shfl_xor_sync(0xffffffffu, V[r], j);
            const bool take_min = ((lane & j) == 0) == ((e & k) == 0);
            const bool sw = take_min ? pk < K[r] : pk > K[r];
            K[r] = sw ? pk : K[r];
            V[r] = sw ? pv : V[r];
          }
      }
    }
  }
  __syncthreads();  // every read of the exchange buffers is done
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int e = r * kLT + tid;
    if (e < total) {
      key[e] = K[r];
      val[e] = V[r];
    }
  }
  __syncthreads();
}

__device__ void warp_sort(uint64_t* key, double* val, int total, int n2, int tid, int lane) {
  uint64_t K = tid < total ? key[tid] : ~0ull;
  double V = tid < total ? val[tid] : 0.0;
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t pk = __shfl_xor_sync(0xffffffffu, K, j);
      const double pv = __shfl_xor_sync(0xffffffffu, V, j);
      const bool take_min = ((lane & j) == 0) == ((tid & k) == 0);
      const bool sw = take_min ? pk < K : pk > K;
      K = sw ? pk : K;
      V = sw ? pv : V;
    }
  if (tid < total) { key[tid] = K; val[tid] = V; }
  __syncthreads();
}
template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(int total, int reps, long long* cyc, int* ok) {
  __shared__ uint64_t key[kLLive], buf[2 * kLLive];
  __shared__ double val[kLLive];
  const int tid = threadIdx.x, lane = tid & 31;
  int n2 = 1;
  while (n2 < total) n2 <<= 1;
  long long acc = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < total; e += kLT) {
      key[e] = (uint64_t)((e * 2654435761u + rep * 97u) % 100003u) << 20;
      val[e] = (double)e;
    }
    __syncthreads();
    long long t0 = clock64();
    if (MODE == 0) lat_sort(key, val, buf, total, n2, tid, lane);
    else warp_sort(key, val, total, n2, tid, lane);
    long long t1 = clock64();
    acc += t1 - t0;
    for (int e = tid; e + 1 < total; e += kLT)
      if (key[e] > key[e + 1]) atomicAdd(ok, 1);
    __syncthreads();
  }
  if (tid == 0) *cyc = acc / reps;
}
int main() {
  long long* c; int* ok;
  cudaMalloc(&c, 8); cudaMalloc(&ok, 4);
  for (int total : {2, 4, 32}) {
    bench<1><<<1, 256>>>(total, 50, c, ok);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warp_sort total %d: %lld cycles\n", total, h);
  }
  for (int total : {1, 2, 4, 32, 100, 256, 372, 512, 1000}) {
    cudaMemset(ok, 0, 4);
    bench<0><<<1, 256>>>(total, 50, c, ok);
    long long h; int bad;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&bad, ok, 4, cudaMemcpyDeviceToHost);
    printf("total %d: %lld cycles, unsorted pairs %d (%s)\n", total, h, bad, cudaGetErrorString(cudaGetLastError()));
  }
}
