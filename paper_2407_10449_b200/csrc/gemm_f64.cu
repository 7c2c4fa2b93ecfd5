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

// One output tile: 128 rows of X (chunk row block rb) x 32*NJ*4 columns of W
// starting at W row wrow0 (NJ = 4: a full 128-wide tile; 2: 64; 1: 32).  Warps:
// 2 (M) x 4 (N), warp tile 64 x 8 NJ.  kk = CTA-wide k-block counter (mbarrier
// phases).  Every output element is accumulated over the K blocks in the same
// order whatever NJ is, so the result does not depend on the tiling.
template <int NJ>
__device__ __forceinline__ void gemm_tile(double* sA, double* sB, uint64_t* full, const double* gA,
                                          const double* gB, double* __restrict__ out, int64_t ldo,
                                          int64_t row_base, int64_t col_base, int KB, int& kk) {
  constexpr uint32_t kBBytes = kChunkBytes * NJ / 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  auto issue = [&](int kb, int q) {
    const int s = q % kStages;
    mbar_expect_tx(&full[s], kChunkBytes + kBBytes);
    bulk_g2s(sA + s * kChunk, gA + (int64_t)kb * kChunk, kChunkBytes, &full[s]);
    bulk_g2s(sB + s * kChunk, gB + (int64_t)kb * kChunk, kBBytes, &full[s]);
  };
  __syncthreads();  // the previous tile's last stages are consumed
  if (tid == 0) {
    for (int kb = 0; kb < kStages - 1 && kb < KB; ++kb) issue(kb, kk + kb);
  }
  double acc[8][NJ][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kb = 0; kb < KB; ++kb) {
    const int q = kk + kb;
    __syncthreads();  // every warp is done with stage (q - 1) % kStages
    if (tid == 0 && kb + kStages - 1 < KB) issue(kb + kStages - 1, q + kStages - 1);
    const int s = q % kStages;
    mbar_wait(&full[s], (uint32_t)((q / kStages) & 1));
    const double* a = sA + s * kChunk;
    const double* b = sB + s * kChunk;
#pragma unroll
    for (int kh = 0; kh < 2; ++kh) {
      double2 fa[8], fb[NJ];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        fa[i] = *reinterpret_cast<const double2*>(a + ((wm * 8 + i) * 2 + kh) * 64 + lane * 2);
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        fb[j] = *reinterpret_cast<const double2*>(b + ((wn * NJ + j) * 2 + kh) * 64 + lane * 2);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], fa[i].x, fb[j].x);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], fa[i].y, fb[j].y);
    }
  }
  kk += KB;

  const int64_t row0 = row_base + wm * 64 + (lane >> 2);
  const int64_t col0 = col_base + wn * 8 * NJ + (lane & 3) * 2;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      double2 v;
      v.x = acc[i][j][0];
      v.y = acc[i][j][1];
      *reinterpret_cast<double2*>(out + (row0 + i * 8) * ldo + col0 + j * 8) = v;
    }
}

// out[R_pad x ldo] (row-major) = X[R_pad x K_pad] . W[S_pad x K_pad]^T, both tiled.
// Persistent: CTA b runs work items b, b + grid, ...; items < n_full are full
// 128 x 128 tiles, the remaining tiles are split into `split` column slices
// (128 x 128/split) so that the last wave is balanced.
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_f64_kernel(const double* __restrict__ Xt, const double* __restrict__ Wt,
                       double* __restrict__ out, int64_t ldo, int s_tiles, int KB, int n_full,
                       int n_items, int split) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + kStages * kChunk;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kChunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int kk = 0;
  for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
    int tile, part = 0;
    if (w < n_full) {
      tile = w;
    } else {
      tile = n_full + (w - n_full) / split;
      part = (w - n_full) % split;
    }
    const int rb = tile / s_tiles, sb = tile % s_tiles;
    const double* gA = Xt + (int64_t)rb * KB * kChunk;
    const int64_t row_base = (int64_t)rb * kTileR;
    if (w < n_full || split == 1) {
      gemm_tile<4>(sA, sB, full, gA, Wt + (int64_t)sb * KB * kChunk, out, ldo, row_base,
                   (int64_t)sb * kTileR, KB, kk);
    } else if (split == 2) {
      gemm_tile<2>(sA, sB, full, gA, Wt + (int64_t)sb * KB * kChunk + part * (kChunk / 2), out,
                   ldo, row_base, (int64_t)sb * kTileR + part * 64, KB, kk);
    } else {
      gemm_tile<1>(sA, sB, full, gA, Wt + (int64_t)sb * KB * kChunk + part * (kChunk / 4), out,
                   ldo, row_base, (int64_t)sb * kTileR + part * 32, KB, kk);
    }
  }
}

}  // namespace

size_t gemm_smem_bytes() { return (size_t)kStages * 2 * kChunkBytes + kStages * sizeof(uint64_t); }

static int g_gemm_sms = 0;

cudaError_t launch_gemm_tn(const double* Xt, int64_t R_pad, const double* Wt, int64_t S_pad,
                           int64_t K_pad, double* out, int64_t ldo, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_f64_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)gemm_smem_bytes());
    if (e != cudaSuccess) return e;
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_gemm_sms, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  const int r_tiles = (int)(R_pad / kTileR), s_tiles = (int)(S_pad / kTileR), KB = (int)(K_pad / kTileK);
  const int T = r_tiles * s_tiles;
  if (T == 0) return cudaSuccess;
  const int P = g_gemm_sms;
  // whole waves of full tiles; the rest (all tiles when there are fewer than SMs)
  // split into 1, 2 or 4 column slices, whichever finishes first (in units of a
  // full-tile time)
  const int rounds = T / P, rest = T - rounds * P;
  int best_split = 1;
  double best = 1e30;
  for (int f = 1; f <= 4; f *= 2) {
    const double t = rounds + (double)((rest * f + P - 1) / P) / f;
    if (t < best - 1e-9) {
      best = t;
      best_split = f;
    }
  }
  const int n_full = rounds * P;
  const int n_items = n_full + rest * best_split;
  const int G = n_items < P ? n_items : P;
  gemm_tn_f64_kernel<<<G, kThreads, gemm_smem_bytes(), st>>>(Xt, Wt, out, ldo, s_tiles, KB,
                                                              n_full, n_items, best_split);
  return cudaGetLastError();
}

}  // namespace tmvn
