// internal.h -- launchers shared by the runtime (runtime.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmvn {

// ---- GEMM (gemm_f64.cu) ----------------------------------------------------
size_t gemm_smem_bytes();
// out[R_pad x ldo] = X[R_pad x K_pad] . W[S_pad x K_pad]^T (X, W fragment-tiled).
cudaError_t launch_gemm_tn(const double* Xt, int64_t R_pad, const double* Wt, int64_t S_pad,
                           int64_t K_pad, double* out, int64_t ldo, cudaStream_t st);

// ---- fused per-chain ESS kernel (ess_chain.cu) -----------------------------
struct EssParams {
  // P (= A x_t, incremental), Q (= A nu): C_pad x ldp row-major.
  const double* P_cur;
  double* P_next;
  const double* Q;
  int64_t ldp;
  const double* b;
  int m;
  // X (iterates) and N (nu), fragment-tiled, C_pad x d_pad.
  double* X;
  double* N;
  int d;
  int64_t d_pad;
  int C;
  uint32_t chain_offset;
  uint64_t seed;
  uint32_t t;       // iteration index of this step
  int gen_next;     // 1: draw nu for t + 1 into N after the update
  double eps;       // S3.3 trim
  int record;       // accumulate S1 += x, S2 += x^2 into the tiled moments
  double* S1;
  double* S2;
  int64_t* rej;     // per chain rejection counter
  // test mode (intervals only): alpha/beta C x m, u C
  const double* g_alpha;
  const double* g_beta;
  const double* g_u;
  // scratch (per CTA)
  double2* gstash;  // gridDim.x * m   (arcs when m > kStashSmemMax)
  double2* ggaps;   // gridDim.x * (m + 2)
  int NB;           // buckets per level (power of two)
  // dumps (nullable)
  double* d_alpha;
  double* d_beta;
  uint8_t* d_active;
  double* d_seg_lo;
  double* d_seg_hi;
  int64_t seg_cap;
  int64_t* d_nseg;
  double* d_L;
  double* d_theta;
  double* d_slack;
  int32_t* d_accept;
};

constexpr int kEssThreads = 256;
constexpr int kLiveCap = 512;       // arcs sorted per batch in shared memory
constexpr int kGapSmem = 256;       // gaps kept in shared memory (rest in ggaps)
constexpr int kStashSmemMax = 4096; // arcs kept in shared memory when m <= this

int ess_buckets(int m);
size_t ess_smem_bytes(int m, int NB);
int ess_grid(int C, int m, int NB);  // persistent grid size
cudaError_t launch_ess_step(const EssParams& p, int grid, cudaStream_t st);
cudaError_t launch_ess_intervals(const EssParams& p, int grid, cudaStream_t st);

// ---- auxiliary kernels (aux_kernels.cu) -------------------------------------
// row-major [R x K] (leading dim ld) -> tiled [R_pad x K_pad]; padding is left untouched.
cudaError_t launch_pack(const double* src, int64_t R, int64_t K, int64_t ld, double* dst,
                        int64_t K_pad, cudaStream_t st);
cudaError_t launch_unpack(const double* src, int64_t R, int64_t K, int64_t K_pad, double* dst,
                          cudaStream_t st);
// nu for iteration t of chains [0, C) (global index chain_offset + c) into tiled N.
cudaError_t launch_normals(double* N, int C, int d, int64_t d_pad, uint64_t seed, uint32_t t,
                           uint32_t chain_offset, cudaStream_t st);
// first (c, i) with P[c, i] - b[i] >= 0 (strict start, C18); *flag = c * m + i or -1.
cudaError_t launch_start_check(const double* P, int64_t ldp, const double* b, int C, int m,
                               unsigned long long* flag, cudaStream_t st);
// sum over chains of a tiled C x d array -> out[d] (fixed order: deterministic)
cudaError_t launch_chain_sum(const double* S, int C, int d, int64_t d_pad, double* out,
                             cudaStream_t st);
// x-space moments with affine: X row-major (C_pad x ldx) = U L^T; S1 += X + mu, S2 += (X + mu)^2
cudaError_t launch_accum_affine(const double* Xrow, int64_t ldx, const double* mu, int C, int d,
                                double* S1row, double* S2row, cudaStream_t st);
cudaError_t launch_add_vec_rows(double* Xrow, int64_t ldx, const double* mu, int C, int d,
                                cudaStream_t st);
// u = L^{-1} (x - mu) per row, forward substitution (L row-major d x d).
cudaError_t launch_trsv_rows(const double* Xrow, const double* mu, const double* L, int C, int d,
                             double* Urow, cudaStream_t st);
cudaError_t launch_gather_rows_tiled(const double* Xt, int64_t d_pad, int d, const int64_t* rows,
                                     int n, double* out, cudaStream_t st);
cudaError_t launch_sum_i64(const int64_t* v, int n, int64_t* out, cudaStream_t st);
// b' = b - A mu (A row-major m x d), one warp per row
cudaError_t launch_gemv_shift(const double* A, const double* b, const double* mu, int m, int d,
                              double* out, cudaStream_t st);
// test kernels
cudaError_t launch_test_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out,
                               bool curand, cudaStream_t st);
cudaError_t launch_test_normals(uint64_t seed, uint32_t t, uint32_t c0, int C, int d, double* nu,
                                double* u, cudaStream_t st);
cudaError_t launch_test_arcs(const double* p, const double* q, const double* b, int64_t n,
                             double* alpha, double* beta, uint8_t* active, cudaStream_t st);

}  // namespace tmvn
