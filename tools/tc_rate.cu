// tc_rate.cu -- tcgen05.mma kind::i8 issue-rate micro-benchmark (tooling, not product).
// One CTA per SM issues R MMAs (M = 128, N = template, K = 32 bytes) on operands
// resident in shared memory (SS) or with A in TMEM (TS), into TMEM accumulators;
// reports cycles per MMA.  Answers: is an SS-mode M=128 N=64 int8 MMA bound by the
// tensor core (32 cycles) or by shared-memory operand reads (6 KB per MMA)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_rate tools/tc_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int N>
__host__ __device__ constexpr uint32_t idesc() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) rate(int R, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 16384; i += 128) sm[i] = (unsigned char)i;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) {
    const uint32_t sa = smem_u32(sm), sb = sa + 4096;
    const uint64_t da = desc(sa, 2048, 128), db = desc(sb, (N / 8) * 128, 128);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t dt = (uint32_t)((u % (TS ? 3 : (N >= 256 ? 2 : 4))) * N);  // rotate accumulators
        if (TS) {
          asm volatile(
              "{\n .reg .pred p, e;\n setp.ne.b32 p, 1, 0;\n elect.sync _|e, 0xffffffff;\n"
              " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt),
              "r"(448u), "l"(db), "n"(idesc<N>()));
        } else {
          asm volatile(
              "{\n .reg .pred p, e;\n setp.ne.b32 p, 1, 0;\n elect.sync _|e, 0xffffffff;\n"
              " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
              "l"(da), "l"(db), "n"(idesc<N>()));
        }
      }
    }
    if ((threadIdx.x & 31) == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n selp.u32 %0, 1, 0, P1;\n}\n"
          : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int N, bool TS>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int R = 2000;
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  rate<N, TS><<<148, 128, 32768>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("{\"mode\": \"%s\", \"M\": 128, \"N\": %d, \"K\": 32, \"cycles_per_mma\": %.2f, \"macs_per_cycle\": %.0f, \"err\": \"%s\"}\n",
         name, N, avg / (R * 8.0), 128.0 * N * 32 / (avg / (R * 8.0)), cudaGetErrorString(e));
  cudaFree(d);
}

// mode 1: 28 TS MMAs per round; 2: 7 cps (to slots 0-6) + 28 MMAs reading slot 7;
// 3: 7 cps + 28 MMAs reading slots 0-6 (dependent, the kernel's pattern); 4: 7 cps only
template <int MODE>
__global__ void __launch_bounds__(128, 1) cprate(int R, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 40960; i += 128) sm[i] = (unsigned char)i;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) {
    const uint32_t sa = smem_u32(sm), sb = sa + 7 * 4096;
    const uint64_t da = desc(sa, 2048, 128), db = desc(sb, 1024, 128);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      if (MODE >= 2) {
#pragma unroll
        for (int i = 0; i < 7; ++i)
          asm volatile(
              "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
              " @e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n}\n" ::"r"((uint32_t)(448 + 8 * i)),
              "l"(da + (uint64_t)((i * 4096) >> 4)));
      }
      if (MODE <= 3) {
#pragma unroll
        for (int i = 0; i < 7; ++i)
#pragma unroll
          for (int j = 0; j < 7 - i; ++j)
            asm volatile(
                "{\n .reg .pred p, e;\n setp.ne.b32 p, 1, 0;\n elect.sync _|e, 0xffffffff;\n"
                " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"((uint32_t)((i + j) * 64)),
                "r"((uint32_t)(MODE == 2 ? 448 + 56 : 448 + 8 * i)), "l"(db + (uint64_t)((j * 2048) >> 4)),
                "n"(idesc<64>()));
      }
    }
    if ((threadIdx.x & 31) == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n selp.u32 %0, 1, 0, P1;\n}\n"
          : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int MODE>
void run_cp() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int R = 500;
  cudaFuncSetAttribute(cprate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cprate<MODE><<<148, 128, 65536>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("{\"cp_mode\": %d, \"cycles_per_round\": %.1f, \"err\": \"%s\"}\n", MODE, avg / R, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run_cp<1>();
  run_cp<2>();
  run_cp<3>();
  run_cp<4>();
  run<32, false>("SS");
  run<64, false>("SS");
  run<128, false>("SS");
  run<256, false>("SS");
  run<32, true>("TS");
  run<64, true>("TS");
  run<128, true>("TS");
  return 0;
}
