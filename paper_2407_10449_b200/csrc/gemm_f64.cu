// gemm_f64.cu -- FP64 tensor-core GEMM for the projections of Alg. 1:
//   Q = N A^T  (q_{c,i} = a_i . nu_c)  and the periodic
//   refresh P = X A^T (Eq. 1 linearity, C13).
//
// sm_100a has no FP64 kind for tcgen05.mma, so the FP64 tensor path is DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).  Operands are stored in the
// fragment-tiled layout of common.cuh, so every 128 x 16 K-slice of an operand
// is one contiguous 16 KB chunk moved by a single cp.async.bulk (TMA bulk
// engine, SASS UBLKCP) into a 4-stage shared-memory ring guarded by mbarriers,
// and every fragment load is one conflict-free ld.shared.v2.f64.
// CTA tile 128 x 128, 8 warps of 64 x 32, no split-K (the reduction order of
// an output element does not depend on C, so results are bitwise invariant to
// how chains are sharded).
#include "common.cuh"
#include "internal.h"

namespace tmvn {
namespace {

constexpr int kStages = 4;
constexpr int kThreads = 256;
constexpr uint32_t kChunkBytes = kChunk * sizeof(double);  // 16 KB

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// out[R_pad x ldo] (row-major) = X[R_pad x K_pad] . W[S_pad x K_pad]^T, both tiled.
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_f64_kernel(const double* __restrict__ Xt, const double* __restrict__ Wt,
                       double* __restrict__ out, int64_t ldo, int s_tiles, int KB) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + kStages * kChunk;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kChunk);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb = blockIdx.x / s_tiles, sb = blockIdx.x % s_tiles;
  const double* gA = Xt + (int64_t)rb * KB * kChunk;
  const double* gB = Wt + (int64_t)sb * KB * kChunk;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto issue = [&](int kb) {
    int s = kb % kStages;
    mbar_expect_tx(&full[s], 2 * kChunkBytes);
    bulk_g2s(sA + s * kChunk, gA + (int64_t)kb * kChunk, kChunkBytes, &full[s]);
    bulk_g2s(sB + s * kChunk, gB + (int64_t)kb * kChunk, kChunkBytes, &full[s]);
  };
  if (tid == 0) {
    for (int kb = 0; kb < kStages - 1 && kb < KB; ++kb) issue(kb);
  }

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int wm = warp >> 2, wn = warp & 3;
  for (int kb = 0; kb < KB; ++kb) {
    __syncthreads();  // every warp is done with stage (kb - 1) % kStages
    if (tid == 0 && kb + kStages - 1 < KB) issue(kb + kStages - 1);
    const int s = kb % kStages;
    mbar_wait(&full[s], (uint32_t)((kb / kStages) & 1));
    const double* a = sA + s * kChunk;
    const double* b = sB + s * kChunk;
#pragma unroll
    for (int kh = 0; kh < 2; ++kh) {
      double2 fa[8], fb[4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        fa[i] = *reinterpret_cast<const double2*>(a + ((wm * 8 + i) * 2 + kh) * 64 + lane * 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        fb[j] = *reinterpret_cast<const double2*>(b + ((wn * 4 + j) * 2 + kh) * 64 + lane * 2);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[i].x, fb[j].x);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[i].y, fb[j].y);
    }
  }

  const int64_t row0 = (int64_t)rb * kTileR + wm * 64 + (lane >> 2);
  const int64_t col0 = (int64_t)sb * kTileR + wn * 32 + (lane & 3) * 2;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2 v;
      v.x = acc[i][j][0];
      v.y = acc[i][j][1];
      *reinterpret_cast<double2*>(out + (row0 + i * 8) * ldo + col0 + j * 8) = v;
    }
}

}  // namespace

size_t gemm_smem_bytes() { return (size_t)kStages * 2 * kChunkBytes + kStages * sizeof(uint64_t); }

cudaError_t launch_gemm_tn(const double* Xt, int64_t R_pad, const double* Wt, int64_t S_pad,
                           int64_t K_pad, double* out, int64_t ldo, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_f64_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)gemm_smem_bytes());
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int r_tiles = (int)(R_pad / kTileR), s_tiles = (int)(S_pad / kTileR), KB = (int)(K_pad / kTileK);
  if (r_tiles == 0 || s_tiles == 0) return cudaSuccess;
  gemm_tn_f64_kernel<<<r_tiles * s_tiles, kThreads, gemm_smem_bytes(), st>>>(Xt, Wt, out, ldo,
                                                                             s_tiles, KB);
  return cudaGetLastError();
}

}  // namespace tmvn
