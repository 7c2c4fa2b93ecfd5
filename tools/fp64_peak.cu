// FP64 pipe micro-benchmarks for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = i; acc[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int l2 = 0, smemOptin = 0, clk = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"clock_khz\": %d",
         p.name, p.multiProcessorCount, l2, smemOptin, clk);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 4), block(32 * wpb);
    dmma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid.x * wpb;
    printf(", \"dmma_tflops_w%d\": %.2f", wpb, flops / ms / 1e9);
  }
  for (int tpb : {256, 512, 1024}) {
    int iters = 20000;
    dim3 grid(sms * 4), block(tpb);
    dfma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8.0 * iters * grid.x * tpb;
    printf(", \"dfma_tflops_t%d\": %.2f", tpb, flops / ms / 1e9);
  }
  printf("}\n");
  return 0;
}
