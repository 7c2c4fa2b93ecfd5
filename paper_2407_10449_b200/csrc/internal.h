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

// ---- int8 Ozaki-split projection on tcgen05 (gemm_i8.cu) -------------------
// Q[N_pad x ldq] (rows = nu rows, columns = A' rows) = Ns . As^T reconstructed in
// FP64: As = digits of A' (M_pad rows, blocks of 128), Ns = digits of nu (N_pad
// rows, blocks of 64), KB steps of 32 along d, S digits (6, 7 or 8);
// rowscale[i] = 2^(e_i + e_nu - 14).
size_t ozaki_smem_bytes(int S, int stages = 0);
// Fused arc construction in the projection's epilogue (options.fuse_arcs): for every
// chain c < C and constraint i < m, bit i % 32 of amask[c][i / 32] says whether
// hypot(P[c][i], Q[c][i]) > b[i] (C3), and then arcs[c][i] holds its arc (alpha, beta)
// of eq:roots (other entries are stale).  P: C_pad x ldp (= A x_t); arcs: C_pad x ald;
// amask: C_pad x mw (mw = ceil(m / 32)).
struct OzArcs {
  const double* P;
  int64_t ldp;
  const double* b;
  int m, C;
  double2* arcs;
  int64_t ald;
  uint32_t* amask;
  int mw;
};
// nu_{t_gen} for chains [0, C) (global index chain_offset + c), t_gen = (*t_dev or 0) +
// t + 1, drawn by the projection's epilogue warps between tiles into N (tiled C_pad x
// d_pad FP64) and its S int8 digits into Ns (options.rng_gemm).
struct OzRng {
  uint64_t seed;
  uint32_t t;
  const uint32_t* t_dev;
  uint32_t chain_offset;
  int C, d;
  int64_t d_pad;
  double* N;
  int8_t* Ns;
  int S;
  int64_t KB;
};
cudaError_t launch_ozaki_gemm(const int8_t* As, int64_t M_pad, const int8_t* Ns, int64_t N_pad,
                              int64_t KB, int S, const double* rowscale, double* Q, int64_t ldq,
                              cudaStream_t st, bool compact = false, const double* colscale = nullptr,
                              const OzArcs* arcs = nullptr, const OzRng* rng = nullptr);
// digits of the R rows of a fragment-tiled FP64 matrix into the oz layout with BR
// rows per block; per_row: exponent from each row's max |v| (rowscale[r] =
// 2^(e_r + e_other - 14)), else the fixed exponent e_fixed (|v| < 2^e_fixed).
cudaError_t launch_oz_slice(const double* src_tiled, int64_t R, int64_t d, int64_t d_pad, int S,
                            int64_t KB, int BR, int per_row, int e_fixed, int e_other, int8_t* dst,
                            double* rowscale, cudaStream_t st);

// ---- latency mode (latency.cu): one thread-block cluster per chain, all iterations ----
struct LatParams {
  const double* A;   // m x d_pad row-major, zero-padded (A' = A: no affine change of variable)
  const double* b;   // m
  int m, d;
  int64_t d_pad;
  double* X;         // tiled C_pad x d_pad: x_{t0} in, final iterates out
  int C;
  uint32_t chain_offset;
  uint64_t seed;
  uint32_t t0;
  int n_iter;
  int64_t K;         // refresh period of P = A x
  double eps;        // S3.3 trim
  int record;
  int64_t burn_in, thin;
  double* S1;        // tiled moments
  double* S2;
  int64_t* rej;      // per chain
  int* err;          // set when a chain's live arcs overflow CTA 0's buffer
  unsigned long long* startflag;  // non-null: check the start; lowest chain * m + i violating
  int cap;           // live arcs CTA 0 holds per iteration (latency_cap)
  int fp32;          // options.precision = 1: FP32 arithmetic (A32, b32), else FP64 (A, b)
  const float* A32;  // m x d_pad, zero-padded rows
  const float* b32;  // m
  // grid mode (gsz > 0: gsz CTAs of a cooperative grid per chain, no clusters): global
  // exchange scratch, zeroed by the host before the launch where noted
  int gsz;
  uint64_t *gtab_g, *gtab_a;  // C x gsz x 128 bucket tables
  int* gtab_c;
  uint64_t *gmrg_g, *gmrg_a;  // C x 128 merged tables
  int* gmrg_c;
  double2* glive;             // C x cap live arcs
  int* gcount;                // C x 2 (iteration parity; zeroed)
  double* gth;                // C x 2: theta, L
  int* gviol;                 // C x 2 (parity; zeroed)
  int* gstart;                // C (zeroed)
  double* gnu;                // C x d_pad: nu_{t+1} drawn by CTA 1 for CTA 0 (T-typed)
};
// constraint-parallel iterations (cp.cu)
constexpr int kCpBuckets = 128;
cudaError_t launch_cp_stats(const double* P0, const double* P1, const unsigned char* cur, const double* Q, int64_t ldp,
                            const double* b, int m, int C, uint64_t* gx, uint64_t* ma, int* cnt, double2* arcs,
                            cudaStream_t st);
cudaError_t launch_cp_live(const double2* arcs, int64_t ldp, int m, int C, const uint64_t* gx, const uint64_t* ma,
                           const int* cnt, int cap, double2* live, int* nlive, cudaStream_t st);
// dynamic shared memory of cp_theta for world * cap gathered arcs: 48 B per arc + 32
size_t cp_theta_smem(int world, int cap);
cudaError_t launch_cp_theta(const uint64_t* gx, const uint64_t* ma, const int* cnt, const double2* all_live,
                            const int* all_n, int world, int cap, uint64_t seed, uint32_t t, uint32_t chain_offset,
                            double eps, double* P0, double* P1, const unsigned char* cur, const double* Q,
                            int64_t ldp, const double* b, int m, int C, int* flags, double* theta, double* L,
                            cudaStream_t st);
cudaError_t launch_cp_commit(const int* flags, const double* theta, const double* L, double* X, const double* N,
                             int64_t d_pad, int d, unsigned char* cur, int C, int record, double* S1, double* S2,
                             int64_t* rej, cudaStream_t st);
size_t latency_smem_bytes(int64_t d_pad, int m, int cs, int cap);
int latency_cap(int64_t d_pad, int m, int cs, size_t smem_max);
int latency_cluster_size(int C, int64_t m, int64_t d_pad, size_t smem_max, bool fp32, int* cap_out);
cudaError_t launch_latency(const LatParams& p, int cs, cudaStream_t st);

// ---- warp mode (small.cu): one warp per chain, all iterations, A in shared memory ----
struct SmallParams {
  const double* A;   // m x d row-major (A' = A: no affine change of variable)
  const double* b;   // m
  int m, d;
  int64_t d_pad;
  double* X;         // tiled C_pad x d_pad: x_{t0} in, final iterates out
  int C;
  uint32_t chain_offset;
  uint64_t seed;
  uint32_t t0;
  int n_iter;
  int64_t K;         // refresh period of P = A x
  double eps;        // S3.3 trim
  int record;
  int64_t burn_in, thin;
  double* S1;        // tiled moment rows (one per chain group)
  double* S2;
  int64_t* rej;      // per chain
  unsigned long long* startflag;  // non-null: check the start; lowest chain * m + i violating
  int warp_bytes, n2;             // set by the launcher
};
// shared memory per warp; rows of A per lane (power of two, m <= 32 R)
size_t small_warp_bytes(int m, int64_t d_pad);
int small_rows(int m);
// warps per CTA the kernel allows (its register bound) with nw warps per chain
int small_max_warps(int m, int nw);
// groups_per_cta chain groups of nw warps (power of two, <= small_rows(m)) per CTA
cudaError_t launch_small(const SmallParams& p, int groups_per_cta, int nw, int grid, cudaStream_t st);

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
  uint32_t t;       // iteration index of this step (offset from *t_dev when t_dev is set)
  const uint32_t* t_dev;  // graph replay: iteration base in device memory (nullable)
  int rec_dev;      // 1: record flag computed from t (t >= burn_in, (t - burn_in) % thin == 0)
  int64_t burn_in, thin;
  int gen_next;     // 1: draw nu for t + 1 (into N after the update, or into N_next)
  double* N_next;   // non-null: nu_{t+1} goes to this buffer (options.rng_overlap: drawn while
                    // theta is computed; N keeps nu_t for the update)
  int64_t group_base;  // scratch index of this launch's first group (split launches)
  int* dyn_ctr;     // non-null: chains handed out dynamically by atomicAdd on dyn_ctr[t & 63]
                    // (the launch for t zeroes the slot of t + 32); null: round-robin
  int dyn_use;      // 0: round-robin even with dyn_ctr set (recorded iterations: the moment
                    // rows are per group, so the chain -> group map must be fixed)
  // fused arcs (options.fuse_arcs): per chain, the activity bitmask of the constraints
  // (amask, C_pad x mw words) and the arcs at their constraint index (arcs, C_pad x ald)
  // from the projection's epilogue; null: phase A computes the arcs from P and Q
  const double2* arcs;
  int64_t ald;
  const uint32_t* amask;
  int mw;
  int8_t* Ns;       // non-null: also write nu_{t+1}'s S digits (int8 projection, gemm_i8.cu)
  int ozS;
  int64_t ozKB;
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
  double2* gstash;  // groups * m   (arcs when not in shared memory)
  double2* ggaps;   // groups * (m + 2)
  int NB;           // buckets per level (power of two)
  int W;            // warps per chain (1, 2, 4, 8)
  int stash_smem;   // 1: arcs stashed in shared memory
  int CH;           // constraints per P/Q chunk streamed into shared memory (even)
  int grp_bytes, base_off, stash_off;  // per-group shared-memory layout (set by the launcher)
  int bucket_mode;  // level-1 buckets: 0 automatic (linear, octave after a general-path-heavy
                    // launch), 1 linear, 2 by octave
  int* gmode;       // automatic switch state: [0..2] general-path counters by t % 3, [3] sticky
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

constexpr int kEssThreads = 256;   // 8 warps per CTA = 8 / W chain groups
constexpr int kLiveCap = 256;      // arcs sorted per batch in shared memory (general path)
constexpr int kGapSmem = 128;      // gaps kept in shared memory (rest in ggaps)

// Shared memory of one chain group: [P/Q chunk ring: 2 slots x (P, Q) x CH
// doubles][2 mbarriers][buckets, live buffer, gaps][stash if stash_smem].
__host__ __device__ inline size_t ess_ring_bytes(int CH) { return CH > 0 ? (size_t)CH * 32 + 16 : 0; }
__host__ __device__ inline size_t ess_group_base_bytes(int NB) {
  size_t s = (size_t)NB * 3 * 8 + (size_t)kLiveCap * 16 + (size_t)kGapSmem * 16 + (size_t)NB * 8 +
             (size_t)kLiveCap * 16 + (size_t)NB * 3 * 4;
  return (s + 15) / 16 * 16;
}
// global-stash path (TMVN_ESS_AQUEUE): per warp, a queue of kAQueue active constraints
// (p, q doubles, index int) in shared memory where the stash would be
constexpr int kAQueue = 64;
constexpr int kAQueueBytes = kAQueue * 20;
__host__ __device__ inline size_t ess_group_smem_bytes(int m, int NB, int stash_smem, int CH, int W = 16) {
  size_t s = ess_ring_bytes(CH) + ess_group_base_bytes(NB);
  // stash: the arcs + constraint index (phase A compaction), or the chain's P and Q rows
  // (even length) + the compacted active indices; else (global stash) the warps' queues
  if (stash_smem) s += (size_t)((m + 1) & ~1) * 16 + (size_t)m * 4;
  else s += (size_t)W * kAQueueBytes;
  return (s + 15) / 16 * 16;
}

// per-group global stash: m arcs (double2) + m constraint indices (int), in double2 units
__host__ __device__ inline int64_t ess_gstash_stride(int64_t m) { return m + (m + 3) / 4; }

struct EssLaunch {
  int W, NB, stash_smem, grid, CH;
  int64_t groups;  // chain groups in the grid (scratch slots)
};
// launch configuration for C chains of m constraints (W_req 0 = automatic;
// ring_req: 1 = stream P/Q through shared memory, 0 = read them from global)
EssLaunch ess_plan(int C, int m, int W_req, int ring_req);
cudaError_t launch_ess_step(const EssParams& p, int grid, cudaStream_t st);
cudaError_t launch_ess_intervals(const EssParams& p, int grid, cudaStream_t st);
#ifdef TMVN_TIMELINE
void tl_access_gemm(unsigned long long* out, bool reset);
void tl_access_ess(unsigned long long* out, bool reset);
#endif
#ifdef TMVN_PHASE_TIMING
void lat_cycles(unsigned long long* out16, bool reset);
void phase_cycles(unsigned long long* out10, bool reset);
void oz_cycles(unsigned long long* out10, bool reset);
#endif

// ---- auxiliary kernels (aux_kernels.cu) -------------------------------------
// row-major [R x K] (leading dim ld) -> tiled [R_pad x K_pad]; padding is left untouched.
cudaError_t launch_to_f32(const double* src, int64_t R, int64_t K, int64_t ld, float* dst, int64_t K_pad,
                          cudaStream_t st);
cudaError_t launch_pack(const double* src, int64_t R, int64_t K, int64_t ld, double* dst,
                        int64_t K_pad, cudaStream_t st);
cudaError_t launch_unpack(const double* src, int64_t R, int64_t K, int64_t K_pad, double* dst,
                          cudaStream_t st);
// nu for iteration t of chains [0, C) (global index chain_offset + c) into tiled N.
cudaError_t launch_normals(double* N, int C, int d, int64_t d_pad, uint64_t seed, uint32_t t,
                           uint32_t chain_offset, cudaStream_t st);
// nu of iteration t (+ *t_dev when non-null) into tiled N and, when Ns != nullptr, its
// S int8 digits (KB K steps); ctas_per_sm 64-thread CTAs per SM (it runs beside other
// kernels: few CTAs so as not to crowd them off the SMs).
cudaError_t launch_nu(double* N, int8_t* Ns, int S, int64_t KB, int C, int d, int64_t d_pad,
                      uint64_t seed, uint32_t t, const uint32_t* t_dev, uint32_t chain_offset,
                      cudaStream_t st, int ctas_per_sm);
// max over rows of A' (tiled) of the int8 projection's stated bound over the FP64 DMMA
// bound at the expected |nu| (positive double bits in *out; 0 for an all-zero A').
cudaError_t launch_oz_guard(const double* At, int m, int d, int64_t d_pad, unsigned long long* out,
                            cudaStream_t st);
// first (c, i) with P[c, i] - b[i] >= 0 (strict start, C18); *flag = c * m + i or -1.
cudaError_t launch_start_check(const double* P, int64_t ldp, const double* b, int C, int m,
                               unsigned long long* flag, cudaStream_t st);
// sum over chains of a tiled C x d array -> out[d] (fixed order: deterministic);
// part: scratch of ceil(C / 64) * d doubles
cudaError_t launch_chain_sum(const double* S, int C, int d, int64_t d_pad, double* out,
                             double* part, cudaStream_t st);
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
cudaError_t launch_set_u32(uint32_t* dst, uint32_t value, cudaStream_t st);
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
