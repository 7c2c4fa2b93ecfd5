// tc_i8_gemm.cu -- standalone validation of an int8 tcgen05.mma GEMM on sm_100a
// (the building block of the Ozaki-style FP64-accurate projection).
// C[M x N] (int32) = A[M x K] (s8) . B[N x K]^T (s8), K-major operands.
// CTA tile 128 x 256, K-block 128 bytes, 4-stage cp.async.bulk ring; warp 0 lane 0
// issues the bulk copies, warp 1 lane 0 issues tcgen05.mma (M=128, N=256, K=32),
// tcgen05.commit releases ring slots and signals the epilogue; 4 warps read the
// int32 accumulator from TMEM with tcgen05.ld.32x32b.
//
// Operands are pre-tiled (by the producer kernels in the library; here on the
// host) so that each (row block, K block) is one contiguous chunk in the UMMA
// canonical K-major SWIZZLE_NONE layout: [k-chunk c (16 B)][row group g][8 rows][16 B].
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_i8_gemm tc_i8_gemm.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 128;  // BK in bytes (= int8 elements)
constexpr int kStages = 4;
constexpr int kAChunk = BM * BK, kBChunk = BN * BK;  // bytes

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// bounded wait: traps (a clean launch error) instead of hanging if a phase never completes
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  for (long i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    if (ok) return;
    if (i > (1l << 24)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle: start, LBO (k-chunk stride), SBO (8-row group stride)
__device__ __forceinline__ uint64_t umma_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version 1 (Blackwell)
  return d;
}
// instruction descriptor: s8 x s8 -> s32, K-major A and B, M = 128, N = 256
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  uint32_t z = 0;
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate), "r"(z));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1)
    tc_i8_gemm(const int8_t* __restrict__ At, const int8_t* __restrict__ Bt, int32_t* __restrict__ C,
               int ldc, int n_tiles, int KB) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sA = smem;
  unsigned char* sB = smem + kStages * kAChunk;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBChunk);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = blockIdx.x / n_tiles, nb = blockIdx.x % n_tiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: 256 columns x 128 lanes of int32
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  const int8_t* gA = At + (size_t)mb * KB * kAChunk;
  const int8_t* gB = Bt + (size_t)nb * KB * kBChunk;
  if (warp == 0 && lane == 0) {  // producer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) mbar_wait(&empty[s], (uint32_t)(((kb / kStages) - 1) & 1));
      mbar_expect_tx(&full[s], kAChunk + kBChunk);
      bulk_g2s(sA + s * kAChunk, gA + (size_t)kb * kAChunk, kAChunk, &full[s]);
      bulk_g2s(sB + s * kBChunk, gB + (size_t)kb * kBChunk, kBChunk, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % kStages;
      mbar_wait(&full[s], (uint32_t)((kb / kStages) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int k = 0; k < BK / 32; ++k) {  // K = 32 bytes per MMA = 2 k-chunks of 16 B
        const uint64_t da = umma_desc(sA + s * kAChunk + k * 2 * (BM / 8) * 128, (BM / 8) * 128, 128);
        const uint64_t db = umma_desc(sB + s * kBChunk + k * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
        umma_i8(tmem, da, db, (kb | k) ? 1u : 0u);
      }
      umma_commit(&empty[s]);  // the slot is free once these MMAs have read it
    }
    umma_commit(done);
  }
  // epilogue: all 4 warps; warp w owns TMEM lanes (rows) 32w .. 32w+31
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = mb * BM + warp * 32 + lane;
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int32_t* dst = C + (size_t)row * ldc + nb * BN + c0;
#pragma unroll
    for (int j = 0; j < 32; j += 4) *reinterpret_cast<int4*>(dst + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// host: tile a row-major R x K int8 matrix into [row block][k block][k-chunk][row group][8][16]
static std::vector<int8_t> tile(const std::vector<int8_t>& M, int R, int K, int RB) {
  std::vector<int8_t> t((size_t)R * K);
  const int KB = K / BK;
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < K; ++k) {
      const int rb = r / RB, rr = r % RB, kb = k / BK, kk = k % BK;
      const size_t chunk = ((size_t)rb * KB + kb) * (size_t)RB * BK;
      const size_t off = chunk + ((size_t)(kk / 16) * (RB / 8) + rr / 8) * 128 + (rr % 8) * 16 + kk % 16;
      t[off] = M[(size_t)r * K + k];
    }
  return t;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 128, N = argc > 2 ? atoi(argv[2]) : 256,
            K = argc > 3 ? atoi(argv[3]) : 256;
  std::vector<int8_t> A((size_t)M * K), B((size_t)N * K);
  uint32_t st = 12345;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (int8_t)((int)(st >> 24) - 128); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  auto At = tile(A, M, K, BM), Bt = tile(B, N, K, BN);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, At.size()));
  CK(cudaMalloc(&dB, Bt.size()));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, At.data(), At.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, (size_t)M * N * 4));
  const size_t smem = kStages * (kAChunk + kBChunk) + 256;
  CK(cudaFuncSetAttribute(tc_i8_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int tiles = (M / BM) * (N / BN);
  tc_i8_gemm<<<tiles, 128, smem>>>(dA, dB, dC, N, N / BN, K / BK);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> Cg((size_t)M * N);
  CK(cudaMemcpy(Cg.data(), dC, Cg.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; i += (M > 512 ? 7 : 1))
    for (int j = 0; j < N; j += (N > 512 ? 5 : 1)) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[(size_t)i * K + k] * B[(size_t)j * K + k];
      if (s != Cg[(size_t)i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): %ld vs %d\n", i, j, s, Cg[(size_t)i * N + j]);
        ++bad;
      }
    }
  // timing
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) tc_i8_gemm<<<tiles, 128, smem>>>(dA, dB, dC, N, N / BN, K / BK);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * M * N * K;
  printf("{\"M\": %d, \"N\": %d, \"K\": %d, \"mismatches\": %ld, \"ms\": %.4f, \"tops\": %.1f}\n", M, N, K, bad,
         ms / 10, ops / (ms / 10 * 1e-3) / 1e12);
  return bad ? 2 : 0;
}
