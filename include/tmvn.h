/*
 * tmvn.h -- C ABI of the B200-native batched linear elliptical slice sampler
 * for a standard normal truncated to a polytope {x : A x <= b}
 * (arXiv 2407.10449; "P:n" = /root/reference/PAPER.md line n).
 *
 * The library (paper_2407_10449_b200/libtmvn.so) runs C independent Markov
 * chains of Alg. 1 in FP64 on one sm_100a GPU.  Per chain and
 * iteration t it draws nu ~ N(0, I_d), forms the ellipse
 * x cos(theta) + nu sin(theta) (Eq. 1), computes the active
 * intervals I_act by the paper's sort + cumulative-max algorithm
 * (Alg. 3 / Prop. 1) from the per-constraint roots of Eq. 2
 * (eq:roots), samples theta uniformly on I_act, and applies
 * the S3.3 safeguard (reject an infeasible x_{t+1} and stay).
 *
 * Conventions shared by every entry point:
 *  - All functions return tmvn_status; nothing throws across the ABI.
 *  - "host or device" pointers: any pointer argument may point to host memory
 *    (pageable or pinned) or to device memory of the handle's GPU; the library
 *    copies with cudaMemcpyDefault (unified addressing).  The caller keeps
 *    ownership of every buffer it passes; the library never frees them.
 *  - Matrices are row-major, FP64, densely packed (leading dimension = #cols).
 *  - A handle is bound to the CUDA device that is current at tmvn_create.  It
 *    is not thread-safe: use one handle per thread / rank.
 *  - After an error the handle stays valid; tmvn_last_error() names the cause
 *    (for an infeasible start: the chain and constraint index).
 *  - tmvn_sample is synchronous with respect to the host.
 *  - Determinism: the output is a pure function of (A, b, mu, L, X0, seed,
 *    chain_offset, iter_offset, n_iter, options); it does not depend on how the
 *    chains are split across calls or GPUs (global chain index in the RNG
 *    counter, no split-K in the projection GEMM) provided every shard takes the
 *    same execution path: options.latency 0 or 1, or the automatic choice with
 *    options.total_chains set to the job's chain count (the latency mode sums
 *    its dot products in another order than the throughput path).  Moment sums
 *    agree across splits to rounding (different summation order), not bitwise.
 */
#ifndef TMVN_H_
#define TMVN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tmvn_ctx* tmvn_handle;

typedef enum {
  TMVN_OK = 0,
  TMVN_E_ARG = -1,              /* null pointer, bad size, non-finite input, C < 1 ...       */
  TMVN_E_EMPTY_POLYTOPE = -2,   /* a zero row of A with b_i < 0 ("invalid")          */
  TMVN_E_INFEASIBLE_START = -3, /* some a_i . x0 >= b_i: start must be strictly interior     */
  TMVN_E_FACTOR = -4,           /* L not lower-triangular with a positive diagonal (App. A)  */
  TMVN_E_CUDA = -5,             /* a CUDA runtime error                                      */
  TMVN_E_OOM = -6,              /* device allocation failed                                  */
  TMVN_E_STATE = -7             /* call out of order (e.g. moments before any sample)        */
} tmvn_status;

typedef struct {
  /* S3.3 trimming epsilon: every active interval [l, u] becomes
   * [l + eps, u - eps] except at the outer endpoints 0 and 2*pi; segments that
   * vanish are dropped; if all vanish the untrimmed set is used (C7).
   * Default 0.0 (FP64). */
  double trim_eps;
  /* P = A x_t is maintained incrementally (P <- P cos(theta) + Q sin(theta),
   * exact by Eq. 1) and recomputed as X A^T after every iteration t with
   * (t + 1) % recompute_every == 0.  Default 32; 1 = recompute every step. */
  int64_t recompute_every;
  /* Moment recording (S4.1 protocol): the iterate x_{t+1} produced by
   * iteration t is recorded iff record != 0, t >= burn_in and
   * (t - burn_in) % thin == 0.  Defaults: record 1, burn_in 0, thin 1. */
  int64_t burn_in, thin;
  int32_t record;
  /* Global index of the first chain of this handle (multi-GPU sharding) and
   * the iteration index of the first iteration of the next tmvn_sample (the
   * RNG counter base; resume).  Defaults 0, 0.  iter_offset advances by n_iter
   * after every successful tmvn_sample when auto_advance != 0 (default 1). */
  int64_t chain_offset;
  int64_t iter_offset;
  int32_t auto_advance;
  /* cudaStream_t to run on (e.g. torch.cuda.current_stream().cuda_stream);
   * NULL = the legacy default stream. */
  void* stream;
  /* 1: bracket every projection GEMM and every ESS launch of the hot loop with
   * CUDA events on `stream` and accumulate their durations (tmvn_get_profile).
   * Default 0. */
  int32_t profile;
  /* Warps of the fused per-chain kernel that own one chain: 1, 2, 4, 8 or 16
   * (16: one 512-thread CTA per chain); 0 (default) = chosen from C and m.
   * Results do not depend on it.  A small W whose chain groups' bucket tables
   * would not fit one CTA's shared memory (m in the thousands) is raised. */
  int32_t chain_warps;
  /* Chain shards run as independent GEMM -> ESS sequences on concurrent streams
   * (forked from / joined to `stream`), so the FP64 tensor GEMM of one shard
   * can overlap the ALU-bound per-chain kernel of another.  0 (default) =
   * automatic: 2 shards for >= 2048 chains, 4 for m >= 8192 and >= 1024 chains,
   * 1 when d > 2048 (the projection dominates and every shard would re-stream
   * its A' operand from HBM); measured on B200.  Results
   * do not depend on it (tested bitwise). */
  int32_t streams;
  /* 1: stream each chain's P and Q rows into shared memory with cp.async.bulk
   * through a 2-slot mbarrier ring (the next chain's rows prefetched); 0
   * (default): read them from global memory (measured faster on B200 at
   * config 3: the ring costs occupancy, profiles/r01/README.md). */
  int32_t ring;
  /* 1 (default): whole blocks of recompute_every iterations aligned to a
   * multiple of it are replayed as one CUDA graph (a single shard, no profiling,
   * no x-space moment recording); 0: one launch per kernel. */
  int32_t graphs;
  /* Projection GEMM Q = N A'^T (Alg. 1's A nu):
   *   0 (default): automatic = 1 when d <= 4096 and every row passes the dynamic-
   *      range guard (tmvn_profile.oz_guard_ratio <= 16: the int8 bound below is at
   *      most 16x the DMMA bound evaluated at the expected |nu|), else 2;
   *   1: int8 Ozaki split on the tcgen05 tensor cores (TMEM accumulators): A'
   *      row i scaled by 2^e_i > max_j |a_ij|, nu by 2^4 (Box-Muller |nu| < 8.58),
   *      both truncated to fixed point with 8S - 1 fraction bits and cut into S
   *      byte digits; the S(S+1)/2 exact int8 products of digit pairs with
   *      k + l <= S + 1 are summed in int32 per diagonal and recombined in FP64.
   *      Stated bound:
   *      |Q - a.nu| <= 2^(e_i + 4) d (S + 1) 2^(2 - 8S) + 2^-51 |Q|
   *      (truncation 2^(1-F) per product with F = 8S - 1, dropped diagonals
   *      <= (S - 1) 2^(2 - 8S) d, FP64 reconstruction; S = 7: 2^(e_i+4) d 2^-51).
   *      Requires d <= 4096 (int32 headroom); otherwise TMVN_E_ARG.
   *   2: FP64 on the DMMA tensor pipe (mma.sync f64; round-to-nearest FP64
   *      products, |Q - a.nu| <= 2 d 2^-53 sum_j |a_ij nu_j|).
   * The P refreshes (every recompute_every) and the start check use the same
   * product on X: with the int8 projection X is cut into digits with one
   * exponent per chain (max_j |x_cj| < 2^e_c; bound as above with 2^(e_i + e_c)
   * in place of 2^(e_i + 4)), with DMMA in FP64.  Results do not depend on C or
   * on the sharding. */
  int32_t projection;
  /* Digits S of the int8 projection: 6, 7 or 8 (0 = default 7: 55-bit fixed
   * point, 28 int8 MMAs per 32-wide K step). */
  int32_t ozaki_slices;
  /* 1: nu for iteration t + 1 is drawn by a small kernel on a second stream
   * while the projection GEMM of iteration t runs (on the CUDA cores the
   * tensor-core GEMM leaves idle), into the other of two nu buffers; the fused
   * per-chain kernel then only reads nu.  0 (default): the fused kernel draws nu
   * for t + 1 after its update (measured faster on B200 at config 3: 0.410 vs
   * 0.422 ms per iteration -- the co-running RNG slows the GEMM by ~20 us, the
   * per-chain kernel gains ~20 us).  Single shard only.  Results do not depend
   * on it (tested bitwise). */
  int32_t rng_ahead;
  /* Chain scheduling of the fused per-chain kernel: 2 dynamic (each group of
   * warps grabs its next chain with an atomic counter, one chain ahead), 1
   * round-robin, 0 (default) automatic: dynamic for long rows (8 warps per chain),
   * round-robin otherwise.  Results do not depend on it. */
  int32_t schedule;
  /* 1: pipelined schedule (one shard, no profiling): the projection GEMM of
   * iteration t + 1 runs concurrently with the fused per-chain kernel of
   * iteration t (Q double-buffered, nu triple-buffered and drawn two iterations
   * ahead on a third stream, the GEMM in a compact form on a high-priority
   * stream so that the two kernels share the SMs).  0 (default): serial.
   * Results do not depend on it. */
  int32_t pipeline;
  /* 1: latency mode -- one thread-block cluster (1-16 CTAs, distributed shared
   * memory) per chain runs all n_iter iterations in a single launch (the
   * regime of few chains, e.g. the paper's 1 or 10); with very
   * few chains and a large A, a cooperative grid of SMs / C CTAs per chain
   * instead (same results bitwise; chosen by the cost model).  Same RNG
   * counters and readings; the dot products sum in another order, so results
   * agree with the default path to rounding, not bitwise.  Not with the affine
   * change of variable (the default path runs then).  CTA 0 of a cluster holds
   * every live arc of an iteration (up to m, or what its shared memory allows);
   * if some iteration has more, the call is rerun on the default path from the
   * same start (tmvn_profile.latency_fallbacks).  2 (default): auto -- latency
   * mode when the job's chains (total_chains below) are at most half the SMs
   * (clusters of two or more CTAs) and a cost model fitted to B200 measurements
   * expects it to be faster (it re-reads A from L2 for every chain), else the
   * default path.  0: off (always the default path). */
  int32_t latency;
  /* 1: FP32-class arithmetic, the paper's precision (S3.3).
   * In the latency mode (options.latency, auto as in FP64): A . nu, A . x, the arcs, P' and the safeguard, x in single
   * precision; the interval comparisons and the inverse-CDF draw in FP64 on the
   * (exactly widened) FP32 endpoints; a live-arc overflow reruns the call on
   * the throughput path.  Otherwise (many chains, affine change of variable)
   * the throughput path with the int8 projection at 4 digits per operand
   * (bound below with S = 4: ~2^-26 relative, FP32-class) for Q, the refresh
   * and the start check; the rest stays FP64.  Use with trim_eps > 0 (S3.3
   * trimming); the safeguard rejects the rare infeasible proposal; iterates
   * are feasible to FP32 rounding.  Parity with the FP64 oracle is
   * statistical.  On the throughput path this is an "FP32-class projection,
   * FP64 elsewhere" mode: only Q, the refresh and the products feeding them are
   * FP32-class; arcs, I_act, theta, P' and x stay FP64.  The strict start check
   * (C18) always runs on an FP64-class product (FP64 DMMA) whatever this
   * setting.  0 (default): FP64. */
  int32_t precision;
  /* Chains of the whole job across every shard / rank (0 = this call's C).  The
   * automatic execution-path choice (latency = 2) is made from it, so that the
   * shards of one job (chain_offset) all take the same path and their chains
   * equal those of an unsharded run bitwise.  Set it whenever a job is split
   * (paper_2407_10449_b200.dist.shard does).  Default 0. */
  int64_t total_chains;
  /* 1: with the int8 projection (projection 0/1), the arcs of eq:roots
   * (readings C1-C5) are computed in the projection GEMM's epilogue
   * while the tensor cores run the next tile: each (chain, constraint) pair is
   * tested there against P = A x_t, and the active ones are appended to per-chain
   * arc lists, which the fused per-chain kernel reads instead of the P and Q rows
   * (same arc function, bit-identical arcs; list order is irrelevant to Alg. 3).
   * Not with options.pipeline (the projection of t + 1 would read P while the
   * per-chain kernel of t writes it).  0 (default): the per-chain kernel computes
   * them (measured faster on B200 at config 3: the epilogue's arc work, latency-
   * bound on 8 warps, doubles the projection's time, 0.177 -> 0.321 ms, while the
   * per-chain kernel gains 0.017-0.040 ms).  Results do not depend on it. */
  int32_t fuse_arcs;
  /* 1: with the int8 projection, nu for iteration t + 1 (Philox4x32-10 +
   * Box-Muller, C12, and its int8 digits) is drawn by the projection GEMM of
   * iteration t in its epilogue warps between tiles -- while the tensor cores run
   * -- instead of by the per-chain kernel after its update (nu double-buffered).
   * Same device function and counters: bitwise the same chains.  Ignored with
   * rng_ahead or pipeline.  0 (default): the per-chain kernel draws it (B200:
   * the per-chain kernel gains ~26 us at config 3, the projection loses ~21 us --
   * 0.384 vs 0.383 ms per iteration -- and config 5 loses 3 %). */
  int32_t rng_gemm;
  /* 1: the fused per-chain kernel draws nu for t + 1 while the last lane of
   * its highest warp computes theta (the other warps would idle at the
   * barrier), into the other of two nu buffers; 0 (default): after the update
   * (B200, config 3: 0.207 vs 0.211 ms per launch -- with four chain groups per
   * SM the kernel is throughput-bound, not idle at that barrier).  Results do
   * not depend on it (same counters, tested bitwise). */
  int32_t rng_overlap;
  /* Warp mode for small polytopes (small.cu): a group of 1-8 warps per chain
   * (options.small_warps) runs all n_iter iterations in one launch with A resident
   * in shared memory (column-major), Q = A nu one thread per row, the arcs
   * compacted by ballot, Alg. 3 as a bitonic sort + prefix max, the safeguard by a
   * group OR.  Needs FP64, no affine map, m <= 512 and A (d x 32 ceil(m / 32)
   * doubles) plus 4 groups' state in shared memory.  2 (default): whenever that
   * holds, options.latency is automatic (2) and the job is small --
   * total chains x (m d + 32 m) <= 3.2e7 -- decided from m, d and
   * options.total_chains (else this call's C), so every shard of a job takes the
   * same path (B200, per iteration: BASELINE config 2, 1024 chains, 11.4 us vs
   * 19.6 on the throughput path; config 1 3.9 vs 6.2 in the latency mode; the
   * S4.1 interval with 2000 chains 4.7 vs 14.5); 1: whenever it fits; 0: off.  Dot
   * products sum in index order: results agree with the other paths to rounding,
   * not bitwise. */
  int32_t warp_mode;
  /* Level-1 buckets of the per-chain kernel's Alg. 3 (bucketed sort, Prop. 1): 1
   * linear in alpha over [0, 2 pi]; 2 by octave of alpha (NB / 16 per octave over
   * [2^-12, 8)), for geometries whose arcs crowd just after theta = 0 (the paper's
   * S4.2 instances, unnormalised rows with b = A x0 + U[0, 1]); 0 (default):
   * linear, switching to octaves for the rest of the call once more than 1/8 of a
   * launch's chains went down the general (sorted) interval path or held more than
   * 4 m / NB + 32 arcs in one bucket (tmvn_profile.buckets_used).  Any monotone
   * bucketing gives the same I_act bit for bit: results do not depend on it. */
  int32_t buckets;
  /* Warp mode: warps per chain group (1, 2, 4 or 8, at most ceil(m / 32) rounded up to
   * a power of two).  0 (default): automatic -- one warp per chain when the job's
   * chains fill the SMs, else groups of up to 8 warps that split each chain's rows
   * of A, arcs, sort and coordinates (~32 resident warps per SM).  Trajectories do
   * not depend on it (every row's dot product sums in index order; the sorted arcs
   * give the same gaps); moment sums may differ in the last bits (their per-group
   * partial order follows the group layout). */
  int32_t small_warps;
} tmvn_options;

typedef struct {
  int64_t steps;       /* chain-iterations run (accepted or not) since the last reset        */
  int64_t rejections;  /* safeguard rejections + L = 0 stays (C9)       */
  int64_t recorded;    /* chain-iterations recorded into the moments                          */
} tmvn_stats;

typedef struct {
  int64_t launches;      /* kernels launched by the library (all kinds) since the last reset */
  int64_t gemm_launches; /* hot-loop projection GEMMs timed (Q = N A^T and P refreshes)     */
  double gemm_ms;        /* sum of their CUDA-event durations                                */
  double gemm_flops;     /* algorithmic flops of those GEMMs: 2 C m d each (no padding)      */
  int64_t ess_launches;  /* fused per-chain ESS launches timed                               */
  double ess_ms;
  double ess_bytes;      /* algorithmic HBM bytes of those launches:
                            24 B per constraint-eval + 32 B per chain-coordinate (+32 B
                            when the iteration is recorded into the moments)             */
  int64_t tc_launches;   /* hot-loop int8 tcgen05 projections timed (options.projection = 1) */
  double tc_ms;
  double tc_ops;         /* int8 tensor ops issued by those launches: S(S+1)/2 * 2 C m d     */
  double tc_flops;       /* FP64-equivalent algorithmic flops of those launches: 2 C m d     */
  int64_t latency_calls;      /* tmvn_sample calls run in latency mode (options.latency)      */
  int64_t latency_fallbacks;  /* of those, calls rerun on the default path (live-arc overflow) */
  int64_t latency_grid_calls; /* of those, calls run by the cooperative-grid variant          */
  /* dynamic-range guard of the automatic projection (options.projection = 0): max over
   * rows of A' of the int8 projection's stated bound at S = 7 over the FP64 DMMA bound
   * at the expected |nu|, 2^(e_i+4) d 8 2^-54 / (2 d 2^-53 sqrt(2/pi) ||a_i||_1); the
   * int8 projection is used only when it is <= 16 (else FP64 DMMA).  Set by
   * tmvn_create / tmvn_set_affine (kept by tmvn_reset_stats). */
  double oz_guard_ratio;
  int32_t projection_used;    /* projection of the last throughput-path call: 1 int8, 2 DMMA */
  int64_t warp_mode_calls;    /* tmvn_sample calls run in warp mode (options.warp_mode)        */
  /* level-1 bucket mapping the per-chain kernel ended the last call with: 1 linear,
   * 2 by octave (options.buckets = 2, or the automatic switch turned it on); 0 before
   * any throughput-path call.  Read from device memory by tmvn_get_profile (synchronises the device). */
  int32_t buckets_used;
} tmvn_profile;

/* Fills *opt with the defaults listed above. */
tmvn_status tmvn_default_options(tmvn_options* opt);

/* Creates a handle on the current CUDA device for the polytope {x : A x <= b}
 * (P:24).  A: m x d row-major FP64, b: m FP64 (host or device; both
 * copied).  Errors: TMVN_E_ARG (null, m < 1, d < 1, non-finite entries),
 * TMVN_E_EMPTY_POLYTOPE (a zero row with b_i < 0), TMVN_E_OOM,
 * TMVN_E_CUDA.  On error *out is NULL. */
tmvn_status tmvn_create(const double* A, const double* b, int64_t m, int64_t d, tmvn_handle* out);

/* Non-standard normal N(mu, L L^T) by the change of variable of App. A
 * (P:898-904): the chains run on u ~ N(0, I) truncated to
 * {u : (A L) u <= b - A mu} and report x = L u + mu.  mu: d (NULL = 0);
 * L: d x d row-major lower-triangular with a positive diagonal (NULL = I).
 * After this call X0 / out of tmvn_sample and the moments are in x-space.
 * Passing both NULL restores the standard normal.  Errors: TMVN_E_ARG,
 * TMVN_E_FACTOR (an entry above the diagonal is non-zero or a diagonal entry
 * is <= 0), TMVN_E_EMPTY_POLYTOPE (a zero row of A L with b - A mu < 0). */
tmvn_status tmvn_set_affine(tmvn_handle h, const double* mu, const double* L);

tmvn_status tmvn_set_options(tmvn_handle h, const tmvn_options* opt);
tmvn_status tmvn_get_options(tmvn_handle h, tmvn_options* opt);

/* Runs n_iter iterations of Alg. 1 for C chains.
 * X0: C x d row-major start points (host or device), strictly feasible
 * (a_i . x0 < b_i for all i, checked on the GPU: TMVN_E_INFEASIBLE_START names
 * the first offending chain / constraint).  out: C x d row-major final iterates
 * (host or device; out == X0 allowed).  Chain k of this call is global chain
 * chain_offset + k; its iteration t (t = iter_offset .. iter_offset+n_iter-1)
 * draws nu from Philox4x32-10 counters (j, t, chain, 0) and u from
 * (0, t, chain, 1) under key (seed & 0xffffffff, seed >> 32) (C12).
 * n_iter = 0 only checks and copies X0.  Requires t < 2^32 and
 * chain_offset + C <= 2^32.  Errors: TMVN_E_ARG, TMVN_E_INFEASIBLE_START,
 * TMVN_E_OOM, TMVN_E_CUDA. */
tmvn_status tmvn_sample(tmvn_handle h, const double* X0, int64_t C, int64_t n_iter, uint64_t seed,
                        double* out);

/* Counters since creation or the last tmvn_reset_stats. */
tmvn_status tmvn_get_stats(tmvn_handle h, tmvn_stats* st);

/* Sums over recorded iterates (x-space): sum[j] = sum x_j, sumsq[j] = sum x_j^2
 * (d each, host or device), *n = number of recorded chain-iterations (host).
 * The caller forms mean = sum / n and var = sumsq / n - mean^2 (S4.1).
 * Multi-GPU: all-reduce these three over ranks. */
tmvn_status tmvn_get_moments(tmvn_handle h, double* sum, double* sumsq, int64_t* n);
tmvn_status tmvn_reset_stats(tmvn_handle h);  /* also resets the profile */
/* Kernel timings collected while options.profile != 0 (launch counts always). */
tmvn_status tmvn_get_profile(tmvn_handle h, tmvn_profile* prof);

/* ------------------------------------------------------------------------ */
/* Constraint-parallel iterations (Prop. 1): for an A
 * too large for one GPU, rank r creates its handle with its own rows A_r, b_r
 * (tmvn_create) and every rank holds all C chains.  One iteration t is
 *   tmvn_cp_stats -> all-reduce (gx: max, ma: max, cnt: sum)
 *   tmvn_cp_live  -> all-gather (live, nlive) in rank order
 *   tmvn_cp_theta -> all-reduce (flags: max)
 *   tmvn_cp_commit
 * with the collectives run by the caller (torch.distributed / NCCL; the
 * Python class paper_2407_10449_b200.ConstraintParallel does it).  Every rank
 * draws the same nu and u (Philox counters), the merged bucket tables and the
 * gathered live arcs give every rank the same I_act and theta, and the
 * projection rows are computed per element in a fixed order, so the chains
 * are bitwise those of one GPU holding all rows.  All exchange buffers are
 * caller-owned device memory on the handle's stream:
 *   gx, ma: uint64 C x 128 (bucket max beta bits exact, max alpha high word),
 *   cnt: int32 C x 128, live: double C x cap x 2 (alpha, beta), nlive: int32 C
 *   (may exceed cap: arcs were dropped -- tmvn_cp_theta then sets that
 *   chain's flag to 2 and tmvn_cp_commit holds the chain; the caller must stop),
 *   all_live: world x C x cap x 2, all_n: world x C, flags: int32 C
 *   (0 accept, 1 safeguard violation, 2 live-arc overflow; all-reduced MAX).
 *   tmvn_cp_theta keeps world * cap arcs per chain in shared memory (48 B each):
 *   TMVN_E_ARG when that exceeds the device's opt-in limit (B200: world * cap
 *   <= 4842).
 * FP64 only (precision != 0: TMVN_E_ARG), no affine change of variable; stats / moments as for tmvn_sample
 * after tmvn_cp_end (per rank: identical on every rank).  Errors: TMVN_E_ARG,
 * TMVN_E_STATE (no tmvn_cp_begin), TMVN_E_INFEASIBLE_START (this rank's rows). */
tmvn_status tmvn_cp_begin(tmvn_handle h, const double* X0, int64_t C, int64_t n_iter, uint64_t seed);
tmvn_status tmvn_cp_stats(tmvn_handle h, int64_t t, uint64_t* gx, uint64_t* ma, int32_t* cnt);
tmvn_status tmvn_cp_live(tmvn_handle h, const uint64_t* gx, const uint64_t* ma, const int32_t* cnt, int32_t cap,
                         double* live, int32_t* nlive);
tmvn_status tmvn_cp_theta(tmvn_handle h, int64_t t, const uint64_t* gx, const uint64_t* ma, const int32_t* cnt,
                          const double* all_live, const int32_t* all_n, int32_t world, int32_t cap,
                          int32_t* flags);
tmvn_status tmvn_cp_commit(tmvn_handle h, int64_t t, const int32_t* flags);
tmvn_status tmvn_cp_end(tmvn_handle h, int64_t n_iter, double* out);

/* Last error message of this handle (or of the calling thread's last failed
 * tmvn_create when h is NULL).  Valid until the next call on the handle. */
const char* tmvn_last_error(tmvn_handle h);
const char* tmvn_version(void);
/* sizeof of the ABI structs, for bindings to check their layouts: out[0..3] =
 * tmvn_options, tmvn_stats, tmvn_profile, tmvn_step_dump.  Host-only (no device call). */
tmvn_status tmvn_struct_sizes(int64_t* out4);
void tmvn_destroy(tmvn_handle h);

/* ------------------------------------------------------------------------ */
/* Test hooks (same .so; not part of the public contract).  They run the     */
/* production device code on caller-given inputs so each stage can be        */
/* compared with the CPU oracle.  All pointers host or device.               */
/* ------------------------------------------------------------------------ */

/* Philox4x32-10 of the device path on n records: ctr 4n words, key 2n words -> out 4n. */
tmvn_status tmvn_test_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out);
/* cuRAND's curand_Philox4x32_10 on the device (library pin), same layout. */
tmvn_status tmvn_test_curand_philox(const uint32_t* ctr, const uint32_t* key, int64_t n,
                                    uint32_t* out);
/* nu (C x d) and u (C) for global chains c0 .. c0+C-1 at iteration t (C12). */
tmvn_status tmvn_test_normals(uint64_t seed, uint64_t t, int64_t c0, int64_t C, int64_t d,
                              double* nu, double* u);
/* Arcs of eq:roots (C1-C5) for n triples; active[i] = 1 iff hypot(p,q) > b. */
tmvn_status tmvn_test_arcs(const double* p, const double* q, const double* b, int64_t n,
                           double* alpha, double* beta, uint8_t* active);
/* I_act by the production kernel (Alg. 3) for C chains of m pairs each
 * (alpha, beta: C x m, every pair used; (0, 0) is a no-op padding pair),
 * then trimming by eps and theta = inverse CDF at u (C; NULL = no theta).
 * seg_lo/seg_hi: C x seg_cap canonical segments (untrimmed), nseg: C counts
 * (may exceed seg_cap), L: C total length after trimming, theta: C. */
tmvn_status tmvn_test_intervals(const double* alpha, const double* beta, int64_t m, int64_t C,
                                const double* u, double eps, double* seg_lo, double* seg_hi,
                                int64_t seg_cap, int64_t* nseg, double* L, double* theta);
/* The production int8 tcgen05 projection: out[R x S] = X[R x K] . W[S x K]^T with
 * W's rows scaled per row, X by the power of two above max |X|, `slices` digits
 * (4: the FP32-class projection of options.precision = 1; 6, 7, 8); K <= 4096. */
tmvn_status tmvn_test_ozaki_gemm(const double* X, int64_t R, const double* W, int64_t S, int64_t K,
                                 int32_t slices, double* out);
/* Latency mode's live-arc capacity per chain and iteration: cap > 0 lowers it
 * (to exercise the overflow fallback), 0 restores the automatic choice. */
tmvn_status tmvn_test_latency_cap(tmvn_handle h, int32_t cap);
/* Latency mode's grid variant (a cooperative grid of SMs / C CTAs per chain instead
 * of a cluster): mode 1 forces it whenever it fits, -1 never, 0 automatic. */
tmvn_status tmvn_test_latency_grid(tmvn_handle h, int32_t mode);
/* Launch configuration of tmvn_test_intervals: warps per chain (0 = automatic; 1, 2,
 * 4, 8, 16) and level-1 bucket mapping (1 linear, 2 by octave); process-wide. */
tmvn_status tmvn_test_interval_config(int32_t chain_warps, int32_t bucket_mode);
/* The production FP64 GEMM: out[R x S] = X[R x K] . W[S x K]^T (all row-major). */
tmvn_status tmvn_test_gemm(const double* X, int64_t R, const double* W, int64_t S, int64_t K,
                           double* out);

typedef struct {
  double* nu;        /* C x d  */
  double* u;         /* C      */
  double* p;         /* C x m  A x_t as used by the step            */
  double* q;         /* C x m  A nu                                 */
  double* alpha;     /* C x m  */
  double* beta;      /* C x m  */
  uint8_t* active;   /* C x m  */
  double* seg_lo;    /* C x seg_cap canonical untrimmed I_act      */
  double* seg_hi;    /* C x seg_cap */
  int64_t seg_cap;
  int64_t* nseg;     /* C */
  double* L;         /* C  total length after trimming               */
  double* theta;     /* C  */
  double* x_next;    /* C x d  x_{t+1} (= x_t when rejected)         */
  double* max_slack; /* C  max_i (P'_i - b_i) of the proposal        */
  int32_t* accept;   /* C  */
} tmvn_step_dump;

/* One iteration t of the production kernels from the given X_t (C x d, in the
 * handle's u-space; P recomputed from X_t by the production refresh product --
 * the int8 projection's digits of X when it is active, else FP64 DMMA), with every
 * intermediate dumped. */
tmvn_status tmvn_test_step(tmvn_handle h, const double* Xt, int64_t C, uint64_t seed, int64_t t,
                           tmvn_step_dump* dump);
/* tmvn_sample (production loop: incremental P, periodic refresh, fused RNG)
 * that also records, for the n_trace chains listed in chains[] (host), the
 * u-space iterate after every iteration: trace[(it * n_trace + k) * d + j],
 * it = 0 .. n_iter (row 0 = X0). */
tmvn_status tmvn_test_trace(tmvn_handle h, const double* X0, int64_t C, int64_t n_iter,
                            uint64_t seed, const int64_t* chains, int64_t n_trace, double* trace,
                            double* out);

#ifdef __cplusplus
}
#endif
#endif /* TMVN_H_ */
