// ess_chain.cu -- one fused kernel per ESS iteration for every chain (Alg. 1,
// P:169-181), everything after the projection GEMM:
//
//   A  arcs      per constraint i: r = |(p, q)|, the infeasible arc
//                (alpha_i, beta_i) of eq:roots (C1-C5); inactive
//                constraints (r <= b) are compacted away (rows in shared
//                memory: compacted indices, arcs over their (P, Q) entries; long
//                rows: per-warp queues of active constraints, arcs 32 at a time
//                into the global stash) while the level-1 bucket statistics of B
//                are gathered (linear or octave keys on alpha).
//   B  I_act     Alg. 3 / Prop. 1: sort the alphas, cumulative max
//                of the co-sorted betas, gaps [gamma_{k-1}, alpha_{i_k}] and
//                [gamma_m, 2 pi].  The sort is an MSD bucket sort on alpha whose
//                first level also yields, per bucket, max(alpha), max(beta):
//                the exclusive prefix max of max(beta) is gamma entering the
//                bucket, and a bucket whose max(alpha) does not exceed it can
//                hold no gap (Prop. 1), so only "live" buckets are gathered;
//                each live arc finds gamma before it within its own bucket
//                (group-parallel, no sort; par_intervals), or, when many arcs
//                are live, batches are bitonic-sorted and max-scanned.
//                Comparisons only: bit-identical to Alg. 2 on the same arcs
//                (P:400-402).  Oversized buckets are refined.
//   C  theta     canonical segments, S3.3 trim (C7), L = sum of lengths in
//                ascending order, theta = inverse CDF at u (C10).
//   D  update    P' = P cos(theta) + Q sin(theta) (Eq. 1), safeguard
//                accept iff max_i (P'_i - b_i) <= 0 (C8),
//                x <- x cos(theta) + nu sin(theta), moments, then nu for t+1.
//
// A chain is owned by a group of W warps (W in {1, 2, 4, 8, 16}); the 8 warps of a
// CTA (W <= 8; W = 16: one 512-thread CTA per chain) form 8/W independent groups
// that synchronise only among themselves
// (named barriers `bar.sync id, 32 W`, or __syncwarp for W = 1), each looping
// over chains (persistent grid).  Small W keeps many chains in flight per SM and
// turns most synchronisation into warp-level shuffles; large W suits few
// chains with many constraints.
#include <cfloat>
#include "common.cuh"
#include "internal.h"

namespace tmvn {
namespace {

constexpr uint64_t kTopBits = 0x7FF0000000000000ull;  // +inf: every alpha in [0, 2 pi] is below
#ifndef TMVN_ESS_BATCH
#define TMVN_ESS_BATCH 2
#endif
constexpr int kBatch = TMVN_ESS_BATCH;  // constraint pairs per thread with loads in flight
#ifndef TMVN_ESS_BATCH_A1
#define TMVN_ESS_BATCH_A1 1
#endif
constexpr int kBatchA1 = TMVN_ESS_BATCH_A1;  // the same in the active-test pass (fewer live registers)

__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(uint64_t b) { return __longlong_as_double((long long)b); }

struct Ctl {
  uint64_t rlo, rhi, klo;
  uint64_t pqbar;       // mbarrier: the chain's P and Q rows bulk-copied into shared memory
  int shift, mode;      // key: mode 0 linear on [0, 2 pi]; mode 1 (bits - klo) >> shift;
                        // mode 2 by octave (bucket_key)
  int oct_log2;         // mode 2: log2(buckets per octave)
  double G;             // running gamma: max beta over every arc already passed
  int n_act;
  int ngap;
  int total_live;
  int jo;
  int action;
  int nseg;
  double L, theta;
  int maxa_exact;       // max/min alpha per bucket exact (refinement levels)
  int fast;             // 1: I_act built by the parallel level-1 path
  int ncand;            // gaps found by the parallel path
  int crowd;            // a level-1 bucket held more than crowd_at arcs (par_intervals)
  int next;             // dynamic scheduling: the chain grabbed for the next round
  double u;             // u_{c,t} of "sample theta uniformly" (drawn at the chain's start)
};

enum { kAll = 0, kPrefix = 1, kSame = 2, kNarrow = 3 };

// Phase timing (tools/phase_timing.py builds with -DTMVN_PHASE_TIMING; never in
// the product build): thread 0 of every group accumulates clock64 deltas between
// the barriers that close each phase.
#ifdef TMVN_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[14];
#define PHASE(i)                      \
  do {                                \
    if (g.tid == 0) {                 \
      long long now_ = clock64();     \
      ph[i] += now_ - t_prev;         \
      t_prev = now_;                  \
    }                                 \
  } while (0)
#define PHASE_ADD(i, v)             \
  do {                              \
    if (g.tid == 0) ph[i] += (v);   \
  } while (0)
#else
#define PHASE(i) \
  do {           \
  } while (0)
#define PHASE_ADD(i, v) \
  do {                  \
  } while (0)
#endif

// --- a group of W warps owning one chain -------------------------------------
template <int W>
struct Grp {
  static constexpr int kThreads = W * 32;
  int gid;   // group index in the CTA (barrier id gid + 1)
  int tid;   // thread index in the group
  int warp;  // warp index in the group
  int lane;
  __device__ __forceinline__ void sync() const {
    if (W == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(kThreads) : "memory");
  }
  __device__ __forceinline__ int sync_or(int v) const {
    if (W == 1) return __any_sync(0xffffffffu, v);
    int r;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.s32 p, %1, 0;\n bar.red.or.pred q, %2, %3, p;\n"
        " selp.s32 %0, 1, 0, q;\n}\n"
        : "=r"(r)
        : "r"(v), "r"(gid + 1), "r"(kThreads)
        : "memory");
    return r;
  }
};

template <typename T>
__device__ __forceinline__ T warp_incl_max(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v = v > n ? v : n;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += n;
  }
  return v;
}
// exclusive max-scan of v over the group's threads (init `init`); *total = max(init, all v)
// tail_sync = false: the caller guarantees a group barrier before s_w is written again
template <int W>
__device__ uint64_t grp_excl_max(const Grp<W>& g, uint64_t v, uint64_t init, uint64_t* s_w,
                                 uint64_t* total, bool tail_sync = true) {
  const uint64_t inc = warp_incl_max(v);
  uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (g.lane == 0) exc = 0;
  if (W == 1) {
    const uint64_t t = __shfl_sync(0xffffffffu, inc, 31);
    *total = init > t ? init : t;
    return init > exc ? init : exc;
  }
  if (g.lane == 31) s_w[g.warp] = inc;
  g.sync();
  uint64_t pre = init, tot = init;
  for (int i = 0; i < W; ++i) {
    if (i < g.warp) pre = pre > s_w[i] ? pre : s_w[i];
    tot = tot > s_w[i] ? tot : s_w[i];
  }
  if (tail_sync) g.sync();
  *total = tot;
  return pre > exc ? pre : exc;
}
template <int W>
__device__ int grp_excl_sum(const Grp<W>& g, int v, int* s_w, int* total, bool tail_sync = true) {
  const int inc = warp_incl_sum(v);
  if (W == 1) {
    *total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - v;
  }
  if (g.lane == 31) s_w[g.warp] = inc;
  g.sync();
  int pre = 0, tot = 0;
  for (int i = 0; i < W; ++i) {
    if (i < g.warp) pre += s_w[i];
    tot += s_w[i];
  }
  if (tail_sync) g.sync();
  *total = tot;
  return pre + inc - v;
}

struct Smem {
  uint64_t* maxA;
  uint64_t* Gx;    // max beta per bucket; after the scan, in place, the exclusive prefix max
  uint64_t* minA;  // exact only on refinement levels
  uint64_t* keys;  // kLiveCap
  double* vals;    // kLiveCap
  double2* gaps;   // kGapSmem
  int* cnt;
  int* off;
  int* fill;       // NB: live arcs gathered into each level-1 bucket's range so far
  uint64_t* gin;   // NB: gamma entering each level-1 bucket (parallel path)
  uint64_t* cand;  // 2 kLiveCap: gaps (alpha, gamma) found by the parallel path, unordered
};

// Level-1 keys: mode 0 linear on [0, 2 pi]; mode 2 by octave (NB / 16 buckets per octave
// over [2^-12, 8) from the bit pattern, bucket 0 below -- for geometries whose arcs
// crowd just after theta = 0, options.buckets / the automatic switch); mode 1: the
// refinement levels' (bits - klo) >> shift.  All monotone in alpha, which is all that
// Alg. 3's bucketed form needs (Prop. 1): I_act is bit-identical for any of them.
__device__ __forceinline__ int bucket_key(double a, const Ctl& c, int NB, double scale) {
  if (c.mode == 0) {
    int k = (int)__dmul_rn(a, scale);
    return k < NB - 1 ? k : NB - 1;
  }
  const uint64_t bits = dbits(a);
  if (c.mode == 2) {
    if (bits < 0x3F30000000000000ull) return 0;  // alpha < 2^-12
    const int e = (int)(bits >> 52) - 1011;      // 0 .. 14 for alpha < 8
    const int k = 1 + (e << c.oct_log2) + (int)((bits >> c.shift) & c.klo);
    return k < NB - 1 ? k : NB - 1;
  }
  uint64_t k = (bits - c.klo) >> c.shift;
  return k < (uint64_t)(NB - 1) ? (int)k : NB - 1;
}

__device__ __forceinline__ void set_bits_mode(Ctl& c, int log2NB) {
  c.mode = 1;
  c.klo = c.rlo;
  uint64_t top = c.rhi < dbits(kTwoPi) ? c.rhi : dbits(kTwoPi);
  uint64_t span = top > c.rlo ? top - c.rlo : 0;
  int bl = span ? 64 - __clzll((long long)span) : 0;
  c.shift = bl > log2NB ? bl - log2NB : 0;
}

__device__ __forceinline__ void gap_store(const Smem& S, double2* gg, int k, double lo, double hi) {
  double2 v;
  v.x = lo;
  v.y = hi;
  if (k < kGapSmem) S.gaps[k] = v;
  else gg[k - kGapSmem] = v;
}
__device__ __forceinline__ double2 gap_load(const Smem& S, const double2* gg, int k) {
  return k < kGapSmem ? S.gaps[k] : gg[k - kGapSmem];
}

template <int W>
__device__ void clear_buckets(const Grp<W>& g, const Smem& S, int NB) {
  for (int j = g.tid; j < NB; j += Grp<W>::kThreads) {
    S.maxA[j] = 0;
    S.Gx[j] = 0;
    S.minA[j] = ~0ull;
    S.cnt[j] = 0;
    S.fill[j] = 0;
  }
}

// Bucket statistics without 64-bit shared atomics (those compile to CAS spin
// loops): non-negative doubles order like their bit patterns, so the max (min)
// of a bucket is found on the high 32-bit word with a native 32-bit atomic, and
// then on the low word among the values whose high word matched (bucket_add_lo).
__device__ __forceinline__ uint32_t* hi_word(uint64_t* a) { return reinterpret_cast<uint32_t*>(a) + 1; }
__device__ __forceinline__ uint32_t* lo_word(uint64_t* a) { return reinterpret_cast<uint32_t*>(a); }
__device__ __forceinline__ uint32_t hi32(double x) { return (uint32_t)(dbits(x) >> 32); }
__device__ __forceinline__ uint32_t lo32(double x) { return (uint32_t)dbits(x); }

// kCas: max beta exact in this pass by a 64-bit compare-and-swap, taken only while the
// value beats the bucket's current max (a plain 64-bit load first: about ln n swaps per
// bucket of n arcs), so that no low-word pass over the stash is needed (global stash)
__device__ __forceinline__ void max_u64_cas(uint64_t* a, uint64_t v) {
  uint64_t cur = *reinterpret_cast<volatile uint64_t*>(a);
  while (v > cur) {
    const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(a), cur, v);
    if (prev == cur) break;
    cur = prev;
  }
}
template <bool kExact, bool kCas = false>
__device__ __forceinline__ void bucket_add(const Smem& S, int k, double a, double b) {
  if (kCas) max_u64_cas(&S.Gx[k], dbits(b));
  else atomicMax(hi_word(&S.Gx[k]), hi32(b));
  atomicMax(hi_word(&S.maxA[k]), hi32(a));
  if (kExact) atomicMin(hi_word(&S.minA[k]), hi32(a));
  atomicAdd(&S.cnt[k], 1);
}
template <bool kExact>
__device__ __forceinline__ void bucket_add_lo(const Smem& S, int k, double a, double b) {
  if (hi32(b) == *hi_word(&S.Gx[k])) atomicMax(lo_word(&S.Gx[k]), lo32(b));
  if (kExact) {
    if (hi32(a) == *hi_word(&S.maxA[k])) atomicMax(lo_word(&S.maxA[k]), lo32(a));
    if (hi32(a) == *hi_word(&S.minA[k])) atomicMin(lo_word(&S.minA[k]), lo32(a));
  }
}

// A bucket that may hold a gap (Prop. 1: max alpha > gamma entering it).  On
// level 1 only the high word of max alpha is known (low word 0), so the test uses
// the largest value with that high word: conservative -- a dead bucket may be
// gathered and then emits no gap.  The same predicate counts and gathers.
__device__ __forceinline__ bool bucket_live(const Smem& S, const Ctl& c, int k) {
  const uint64_t ma = c.maxa_exact ? S.maxA[k] : (S.maxA[k] | 0xFFFFFFFFull);
  return S.cnt[k] > 0 && ma > S.Gx[k];
}

// Bitonic sort of keys/vals[0, n) (n <= kLiveCap) ascending by key (group-wide).
template <int W>
__device__ void grp_sort(const Grp<W>& g, const Smem& S, int n) {
  int n2 = 2;
  while (n2 < n) n2 <<= 1;
  for (int i = n + g.tid; i < n2; i += Grp<W>::kThreads) S.keys[i] = ~0ull;
  g.sync();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = g.tid; i < n2; i += Grp<W>::kThreads) {
        int l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          uint64_t ki = S.keys[i], kl = S.keys[l];
          if ((ki > kl) == up) {
            S.keys[i] = kl;
            S.keys[l] = ki;
            double t = S.vals[i];
            S.vals[i] = S.vals[l];
            S.vals[l] = t;
          }
        }
      }
      g.sync();
    }
  }
}

// Where the arcs of the active constraints live, by slot (compaction order):
//   kRows = false: stash[slot] = (alpha, beta) (shared or global memory);
//   kRows = true:  the chain's P and Q rows in shared memory (bulk-copied ahead of the
//                  chain), the arc of constraint i written over (Ps[i], Qs[i]), and
//                  idx[slot] = i (packed with the bucket, below).
// kRows: idx[slot] = constraint index | level-1 bucket << kIdxBits (set with the arc in
// phase A), so the live gather skips dead buckets' arcs without reading them
constexpr int kIdxBits = 21;
constexpr int kIdxMask = (1 << kIdxBits) - 1;
// TMVN_ESS_KEEPPQ (kRows): the arcs are not written over the rows; the rows stay in shared
// memory through phase D1 (P' read from there, no global re-read of P and Q), the buckets'
// max beta is exact by CAS in phase A (no low-word pass), and a reader of an arc
// recomputes it from (Ps[i], Qs[i], b[i]) by the same arc_of (bit-identical): only the live
// buckets' arcs on the parallel path, every pass of the (rare) general path
// Measured on B200 at config 3 (one shard, ncu): DRAM per launch 372 -> 331 MB, but the
// launch 205 -> 212 us (the next chain's rows are issued only after D1, and the live
// arcs are recomputed behind an extra barrier): off by default.
// L2 bulk prefetch of the next chain's P and Q rows on the global-stash path (long rows):
// off -- measured on B200 at config 4 (one launch over 1024 chains, ncu): DRAM reads 3.58 ->
// 3.39 GB, 1.68 -> 1.66 ms (the rows of every group's next chain, ~300 x 1.6 MB, do not
// stay in the 126 MB L2 until they are read); config 5 +0.5 %; config 3 takes the
// shared-memory path (its rows are bulk-copied into shared memory instead)
// constraints per level-1 bucket (ess_plan); B200, config 3 (NB = 128 at 16): 8 -> 0.216 ms,
// 32 -> 0.208 ms, 16 -> 0.204 ms per launch; config 4 (1024 buckets either way) unchanged
#ifndef TMVN_ESS_NB_DIV
#define TMVN_ESS_NB_DIV 16
#endif
// Global-stash path (long rows): each thread prefetches into L2 (prefetch.global.L2: no
// registers, no spills) the P and Q pairs it will load TMVN_ESS_PF_DIST passes later in the
// active-test loop of phase A and in the P' loop of phase D1, so that more of the row is
// in flight than the one pair per thread the register budget allows.  B200 (one launch over
// all chains, W = 8): config 4 1.647 -> 1.410 ms per launch at distance 2 (1: 1.420; 3: 1.421,
// 4: 1.425, 6: 1.436, 12: 1.552; with W = 16 for long rows, 2 stays best: 1 and 3 lose
// 1-2 % at config 4), config 5 -4 %.  TMVN_ESS_PF_ROWS: the same in D1 on the
// shared-memory path (config 3): 0.205 -> 0.207-0.209 ms, off.
#ifndef TMVN_ESS_PF_DIST
#define TMVN_ESS_PF_DIST 2
#endif
// the same for the live gather's stream of stored bucket keys (par_intervals B2, global
// stash): config 4 1.413 -> 1.364 ms per launch at distance 2 (4: 1.365), config 5 -2 %
#ifndef TMVN_ESS_PF_AKEY
#define TMVN_ESS_PF_AKEY 2
#endif
#ifndef TMVN_ESS_PF_ROWS
#define TMVN_ESS_PF_ROWS 0
#endif
#ifndef TMVN_ESS_NEXT_PREFETCH
#define TMVN_ESS_NEXT_PREFETCH 0
#endif
#ifndef TMVN_ESS_KEEPPQ
#define TMVN_ESS_KEEPPQ 0
#endif
constexpr bool kKeepPQ = TMVN_ESS_KEEPPQ != 0;
template <bool kRows>
struct ArcStore {
  double2* st;
  double* Ps;
  double* Qs;
  int* idx;
  const double* b;
  __device__ __forceinline__ double2 get(int slot) const {
    if (kRows) {
      const int i = idx[slot] & kIdxMask;
      if (kKeepPQ) {
        double al, be;
        arc_of(Ps[i], Qs[i], __ldg(b + i), al, be);  // active by phase A: same predicate
        return make_double2(al, be);
      }
      return make_double2(Ps[i], Qs[i]);
    }
    return st[slot];
  }
};

// Gather the arcs of live buckets with key < jo into keys/vals, sort, emit gaps.
template <int W, bool kRows>
__device__ void process_batch(const Grp<W>& g, const Smem& S, Ctl& ctl, const ArcStore<kRows>& stash,
                              int n_act, int jo, int n_live, int NB, double scale, double2* gg,
                              uint64_t* s_w64, int* s_w32) {
  for (int idx = g.tid; idx < n_act; idx += Grp<W>::kThreads) {
    double2 ab = stash.get(idx);
    uint64_t bits = dbits(ab.x);
    if (bits < ctl.rlo || bits > ctl.rhi) continue;
    int k = bucket_key(ab.x, ctl, NB, scale);
    if (k >= jo) continue;
    if (!bucket_live(S, ctl, k)) continue;  // dead bucket: no gap (Prop. 1)
    int pos = atomicAdd(&S.off[k], 1);
    S.keys[pos] = bits;
    S.vals[pos] = ab.y;
  }
  g.sync();
  grp_sort(g, S, n_live);
  // gamma before element e: max(Gx[bucket], max beta of earlier elements of the batch)
  const int per = (n_live + Grp<W>::kThreads - 1) / Grp<W>::kThreads;
  const int e0 = g.tid * per, e1 = min(n_live, e0 + per);
  uint64_t lmax = 0;
  for (int e = e0; e < e1; ++e) lmax = lmax > dbits(S.vals[e]) ? lmax : dbits(S.vals[e]);
  uint64_t tot64;
  const uint64_t run = grp_excl_max(g, lmax, 0, s_w64, &tot64);
  int mine = 0;
  {
    uint64_t r = run;
    for (int e = e0; e < e1; ++e) {
      uint64_t gb = S.Gx[bucket_key(bitsd(S.keys[e]), ctl, NB, scale)];
      gb = gb > r ? gb : r;
      if (S.keys[e] > gb) ++mine;
      uint64_t vb = dbits(S.vals[e]);
      r = r > vb ? r : vb;
    }
  }
  int total;
  int pos = grp_excl_sum(g, mine, s_w32, &total) + ctl.ngap;
  {
    uint64_t r = run;
    for (int e = e0; e < e1; ++e) {
      const double a = bitsd(S.keys[e]);
      uint64_t gb = S.Gx[bucket_key(a, ctl, NB, scale)];
      gb = gb > r ? gb : r;
      if (S.keys[e] > gb) gap_store(S, gg, pos++, bitsd(gb), a);
      uint64_t vb = dbits(S.vals[e]);
      r = r > vb ? r : vb;
    }
  }
  g.sync();
  if (g.tid == 0) ctl.ngap += total;
  g.sync();
}

// Group-wide Alg. 3 over the stashed arcs -> gaps (ascending); the general path,
// used when more than 32 arcs are live.  On entry the level-1 bucket statistics
// (linear keys on [0, 2 pi]; count, max beta exact, max alpha high word) are
// filled and untouched.
template <int W, bool kRows>
__device__ void build_intervals(const Grp<W>& g, const Smem& S, Ctl& ctl, const ArcStore<kRows>& stash,
                                int NB, int log2NB, double scale, double2* gg, uint64_t* s_w64,
                                int* s_w32) {
  constexpr int T = Grp<W>::kThreads;
  const int n_act = ctl.n_act;
  bool have_stats = true, have_min = false;
  for (;;) {
    if (!have_stats) {
      clear_buckets(g, S, NB);
      g.sync();
      for (int idx = g.tid; idx < n_act; idx += T) {
        double2 ab = stash.get(idx);
        uint64_t bits = dbits(ab.x);
        if (bits < ctl.rlo || bits > ctl.rhi) continue;
        bucket_add<true>(S, bucket_key(ab.x, ctl, NB, scale), ab.x, ab.y);
      }
      g.sync();
      for (int idx = g.tid; idx < n_act; idx += T) {
        double2 ab = stash.get(idx);
        uint64_t bits = dbits(ab.x);
        if (bits < ctl.rlo || bits > ctl.rhi) continue;
        bucket_add_lo<true>(S, bucket_key(ab.x, ctl, NB, scale), ab.x, ab.y);
      }
      if (g.tid == 0) ctl.maxa_exact = 1;
      g.sync();
      have_min = true;
    }
    have_stats = false;
    // scan buckets: Gx = exclusive prefix max of max beta (init G), in place; live counts, offsets
    const int per = (NB + T - 1) / T;
    const int j0 = g.tid * per, j1 = min(NB, j0 + per);
    uint64_t lmax = 0;
    for (int j = j0; j < j1; ++j) lmax = lmax > S.Gx[j] ? lmax : S.Gx[j];
    uint64_t Gtot;
    uint64_t run = grp_excl_max(g, lmax, dbits(ctl.G), s_w64, &Gtot);
    int lcount = 0;
    for (int j = j0; j < j1; ++j) {
      uint64_t mb = S.Gx[j];
      S.Gx[j] = run;
      run = run > mb ? run : mb;
      if (bucket_live(S, ctl, j)) lcount += S.cnt[j];
    }
    int total_live;
    int o = grp_excl_sum(g, lcount, s_w32, &total_live);
    if (total_live > kLiveCap && !have_min) continue;  // rare: redo the level with exact min/max alpha
    for (int j = j0; j < j1; ++j) {
      S.off[j] = o;
      if (bucket_live(S, ctl, j)) o += S.cnt[j];
    }
    if (g.tid == 0) {
      ctl.total_live = total_live;
      ctl.jo = NB;
    }
    g.sync();
    if (total_live > kLiveCap) {
      for (int j = j0; j < j1; ++j) {
        int lc = bucket_live(S, ctl, j) ? S.cnt[j] : 0;
        if (lc > 0 && S.off[j] + lc > kLiveCap) atomicMin(&ctl.jo, j);
      }
    }
    g.sync();
    if (g.tid == 0) {
      if (ctl.total_live <= kLiveCap) ctl.action = kAll;
      else if (S.off[ctl.jo] > 0) ctl.action = kPrefix;
      else if (S.minA[ctl.jo] == S.maxA[ctl.jo]) ctl.action = kSame;
      else ctl.action = kNarrow;
    }
    g.sync();
    const int action = ctl.action, jo = ctl.jo;
    if (action == kAll || action == kPrefix) {
      int n_live = action == kAll ? total_live : S.off[jo];
      if (n_live > 0) process_batch(g, S, ctl, stash, n_act, jo, n_live, NB, scale, gg, s_w64, s_w32);
    }
    if (g.tid == 0) {
      if (action == kAll) {
        ctl.G = bitsd(Gtot);
        if (ctl.rhi == kTopBits) {
          ctl.action = -1;  // done
        } else {
          ctl.rlo = ctl.rhi + 1;
          ctl.rhi = kTopBits;
          set_bits_mode(ctl, log2NB);
        }
      } else if (action == kPrefix) {
        ctl.G = bitsd(S.Gx[jo]);
        ctl.rlo = S.minA[jo];
        set_bits_mode(ctl, log2NB);
      } else if (action == kSame) {
        // every arc of the bucket has the same alpha: one gap at most (ties)
        double G = bitsd(S.Gx[jo]);
        double a = bitsd(S.minA[jo]);
        if (a > G) {
          gap_store(S, gg, ctl.ngap, G, a);
          ctl.ngap += 1;
        }
        ctl.G = bitsd(jo + 1 < NB ? S.Gx[jo + 1] : Gtot);  // max(G, max beta of bucket jo)
        ctl.rlo = S.maxA[jo] + 1;
        set_bits_mode(ctl, log2NB);
      } else {
        ctl.G = bitsd(S.Gx[jo]);
        ctl.rlo = S.minA[jo];
        ctl.rhi = S.maxA[jo];
        set_bits_mode(ctl, log2NB);
      }
    }
    g.sync();
    if (ctl.action == -1) break;
  }
  if (g.tid == 0) {
    if (ctl.G < kTwoPi) {  // the last segment [gamma_m, 2 pi]
      gap_store(S, gg, ctl.ngap, ctl.G, kTwoPi);
      ctl.ngap += 1;
    }
  }
  g.sync();
}

// ---------------------------------------------------------------------------
// Group-parallel Alg. 3 on the level-1 buckets (the common case).  By Prop. 1 a
// gap [gamma_{k-1}, alpha_{i_k}] needs alpha_{i_k} > gamma_{k-1}, where gamma
// before an arc = max(gamma entering its bucket, max beta of the arcs of the same
// bucket with a smaller alpha): gamma entering bucket j is the exclusive prefix
// max of the buckets' max beta (every arc, live or not), so only the arcs of
// "live" buckets (max alpha > gamma entering) are gathered, and each live arc
// finds its gamma by comparing with the arcs of its own bucket -- no sort, a
// handful of barriers, every thread of the group busy.  Equal alphas: the arc
// gathered first counts as the earlier one (any order is valid).
// The gaps (distinct alphas) are ordered by rank.  Comparisons only, so the
// segments are bit-identical to Alg. 2 on the same arcs.  Returns
// false, touching only gin / cand / fill, when more than kLiveCap arcs are live:
// the general path (build_intervals) then runs on the untouched statistics.
// ---------------------------------------------------------------------------

template <int W, bool kRows>
__device__ bool par_intervals(const Grp<W>& g, const Smem& S, Ctl& ctl, const ArcStore<kRows>& stash,
                              int NB, double scale, double2* gg, uint64_t* s_w64, int* s_w32,
                              int crowd_at, const int* akey) {
  constexpr int T = Grp<W>::kThreads;
  const int per = (NB + T - 1) / T;
  const int j0 = g.tid * per, j1 = min(NB, j0 + per);
  // B1: gamma entering each bucket; live counts and their offsets
  uint64_t lmax = 0;
  for (int j = j0; j < j1; ++j) lmax = lmax > S.Gx[j] ? lmax : S.Gx[j];
  uint64_t Gtot;
  // no trailing barriers in the two scans: s_w64 / s_w32 are next written after the
  // barriers below (grp_excl_sum's, and the one after the offsets)
  uint64_t run = grp_excl_max(g, lmax, dbits(ctl.G), s_w64, &Gtot, false);
  int lcount = 0;
  for (int j = j0; j < j1; ++j) {
    S.gin[j] = run;
    const int cj = S.cnt[j];
    if (cj > crowd_at) ctl.crowd = 1;  // read after the closing barrier
    // level 1: only the high word of max alpha is exact -> conservative test
    if (cj > 0 && (S.maxA[j] | 0xFFFFFFFFull) > run) lcount += cj;
    run = run > S.Gx[j] ? run : S.Gx[j];
  }
  int total;
  int o = grp_excl_sum(g, lcount, s_w32, &total, false);
  if (total > kLiveCap) {  // uniform: the general path runs (its first scan writes s_w64 / s_w32)
    g.sync();
    return false;
  }
  for (int j = j0; j < j1; ++j) {
    const int cj = S.cnt[j];
    const bool live = cj > 0 && (S.maxA[j] | 0xFFFFFFFFull) > S.gin[j];
    S.off[j] = live ? o : -1;
    if (live) o += cj;
  }
  if (g.tid == 0) ctl.ncand = 0;
  g.sync();
  // B2: gather the live buckets' arcs, grouped by bucket
  const int n_act = ctl.n_act;
  for (int idx = g.tid; idx < n_act; idx += T) {
    // akey (global stash): each arc's level-1 bucket, stored by phase A, so that only the
    // arcs of live buckets are read back from global memory
    int k;
    double2 ab;
    if (kRows && kKeepPQ) {  // the live arcs' constraint indices, their arcs below
      const int ik = stash.idx[idx];
      k = ik >> kIdxBits;
      const int ok = S.off[k];
      if (ok < 0) continue;
      S.keys[ok + atomicAdd(&S.fill[k], 1)] = (uint64_t)(ik & kIdxMask);
      continue;
    } else if (kRows) {
      const int ik = stash.idx[idx];
      k = ik >> kIdxBits;
      if (S.off[k] < 0) continue;
      ab = make_double2(stash.Ps[ik & kIdxMask], stash.Qs[ik & kIdxMask]);
    } else if (akey) {
      if (TMVN_ESS_PF_AKEY && idx + TMVN_ESS_PF_AKEY * T < n_act)  // the stream of bucket keys ahead
        asm volatile("prefetch.global.L2 [%0];" ::"l"(akey + idx + TMVN_ESS_PF_AKEY * T));
      k = akey[idx];
      if (S.off[k] < 0) continue;
      ab = stash.get(idx);
    } else {
      ab = stash.get(idx);
      k = bucket_key(ab.x, ctl, NB, scale);
    }
    const int ok = S.off[k];
    if (ok >= 0) {
      const int pos = ok + atomicAdd(&S.fill[k], 1);
      S.keys[pos] = dbits(ab.x);
      S.vals[pos] = ab.y;
    }
  }
  g.sync();
  if (kRows && kKeepPQ) {  // the gathered arcs recomputed densely (at most one per thread)
    for (int e = g.tid; e < total; e += T) {
      const int i = (int)S.keys[e];
      double al, be;
      arc_of(stash.Ps[i], stash.Qs[i], __ldg(stash.b + i), al, be);
      S.keys[e] = dbits(al);
      S.vals[e] = be;
    }
    g.sync();
  }
  // B3: gamma before every live arc from its own bucket; gaps to cand (unordered)
  for (int e = g.tid; e < total; e += T) {
    const uint64_t key = S.keys[e];
    const int k = bucket_key(bitsd(key), ctl, NB, scale);
    const int lo = S.off[k], hi = lo + S.cnt[k];
    uint64_t gm = S.gin[k];
    for (int f = lo; f < hi; ++f) {
      const uint64_t kf = S.keys[f];
      if (kf < key || (kf == key && f < e)) {
        const uint64_t vf = dbits(S.vals[f]);
        gm = gm > vf ? gm : vf;
      }
    }
    if (key > gm) {
      const int c = atomicAdd(&ctl.ncand, 1);
      S.cand[2 * c] = key;
      S.cand[2 * c + 1] = gm;
    }
  }
  g.sync();
  // B4: order the gaps by alpha (distinct among gaps), then [gamma_m, 2 pi]
  const int nc = ctl.ncand, ng = ctl.ngap;
  for (int c = g.tid; c < nc; c += T) {
    const uint64_t a = S.cand[2 * c];
    int rank = 0;
    for (int c2 = 0; c2 < nc; ++c2) rank += S.cand[2 * c2] < a ? 1 : 0;
    gap_store(S, gg, ng + rank, bitsd(S.cand[2 * c + 1]), bitsd(a));
  }
  g.sync();
  if (g.tid == 0) {
    int n = ng + nc;
    const double G = bitsd(Gtot);
    if (G < kTwoPi) gap_store(S, gg, n++, G, kTwoPi);  // the last segment [gamma_m, 2 pi]
    ctl.ngap = n;
    ctl.G = G;
  }
  g.sync();
  return true;
}

// Canonical segments (merge touching), trim, L and theta.  One thread.
__device__ void theta_from_gaps(const Smem& S, Ctl& ctl, double2* gg, double u, double eps) {
  int w = 0;
  for (int k = 0; k < ctl.ngap; ++k) {
    double2 g = gap_load(S, gg, k);
    if (w > 0) {
      double2 last = gap_load(S, gg, w - 1);
      if (last.y == g.x) {
        gap_store(S, gg, w - 1, last.x, g.y);
        continue;
      }
    }
    gap_store(S, gg, w++, g.x, g.y);
  }
  ctl.nseg = w;
  // S3.3 trim (C7): interior endpoints only; fall back to untrimmed if all vanish
  bool trim = eps > 0.0;
  int last_kept = -1;
  if (trim) {
    for (int k = 0; k < w; ++k) {
      double2 g = gap_load(S, gg, k);
      double lo = g.x == 0.0 ? 0.0 : __dadd_rn(g.x, eps);
      double hi = g.y == kTwoPi ? kTwoPi : __dsub_rn(g.y, eps);
      if (hi > lo) last_kept = k;
    }
    if (last_kept < 0) trim = false;
  }
  if (!trim) last_kept = w - 1;
  double total = 0.0;
  for (int k = 0; k < w; ++k) {
    double2 g = gap_load(S, gg, k);
    double lo = g.x, hi = g.y;
    if (trim) {
      lo = g.x == 0.0 ? 0.0 : __dadd_rn(g.x, eps);
      hi = g.y == kTwoPi ? kTwoPi : __dsub_rn(g.y, eps);
      if (!(hi > lo)) continue;
    }
    total = __dadd_rn(total, __dsub_rn(hi, lo));
  }
  ctl.L = total;
  ctl.theta = 0.0;
  if (!(total > 0.0)) return;
  double target = __dmul_rn(u, total);
  double before = 0.0;
  for (int k = 0; k < w; ++k) {
    double2 g = gap_load(S, gg, k);
    double lo = g.x, hi = g.y;
    if (trim) {
      lo = g.x == 0.0 ? 0.0 : __dadd_rn(g.x, eps);
      hi = g.y == kTwoPi ? kTwoPi : __dsub_rn(g.y, eps);
      if (!(hi > lo)) continue;
    }
    double after = __dadd_rn(before, __dsub_rn(hi, lo));
    if (after > target || k == last_kept) {
      ctl.theta = __dadd_rn(lo, __dsub_rn(target, before));
      return;
    }
    before = after;
  }
}

// Per-group shared memory: bucket arrays, live buffer, gaps (stash after them).
// The fixed-size arrays first (constant offsets from the group's base, folded into the
// shared-memory instructions), then the NB-sized ones.
__device__ __forceinline__ Smem carve(unsigned char* base, int NB) {
  Smem S;
  S.keys = reinterpret_cast<uint64_t*>(base);
  S.vals = reinterpret_cast<double*>(S.keys + kLiveCap);
  S.gaps = reinterpret_cast<double2*>(S.vals + kLiveCap);
  S.cand = reinterpret_cast<uint64_t*>(S.gaps + kGapSmem);
  S.maxA = S.cand + 2 * kLiveCap;
  S.Gx = S.maxA + NB;
  S.minA = S.Gx + NB;
  S.gin = S.minA + NB;
  S.cnt = reinterpret_cast<int*>(S.gin + NB);
  S.off = S.cnt + NB;
  S.fill = S.off + NB;
  return S;
}

// Append (al, be) to the stash and the level-1 bucket statistics; warp-aggregated
// slot allocation.  Must be reached by all 32 lanes of the warp.
__device__ __forceinline__ void stash_arc(const Smem& S, Ctl& ctl, double2* stash, bool act,
                                          double al, double be, int NB, double scale) {
  const unsigned mask = __ballot_sync(0xffffffffu, act);
  if (mask == 0) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&ctl.n_act, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (act) {
    const int slot = base + __popc(mask & ((1u << lane) - 1u));
    const int k = bucket_key(al, ctl, NB, scale);
    stash[slot] = make_double2(al, be);
    bucket_add<false>(S, k, al, be);
  }
}

// CTAs per SM the register allocation must allow: 4 (64 registers) for the config-3
// path (W = 8, arcs stashed in shared memory: 4 x 56 KB fit, no spills), 3 (80
// registers) elsewhere (at 64 those variants spill 100-200 bytes)
// global-stash path: per-warp queues of active constraints in shared memory (phase A),
// and the buckets' max beta by CAS (no low-word pass)
#ifndef TMVN_ESS_AQUEUE
#define TMVN_ESS_AQUEUE 1
#endif
#ifndef TMVN_ESS_CASMAX
#define TMVN_ESS_CASMAX 1
#endif
#ifndef TMVN_ESS_MIN_BLOCKS
#define TMVN_ESS_MIN_BLOCKS 3
#endif
#ifndef TMVN_ESS_W8_BLOCKS
#define TMVN_ESS_W8_BLOCKS 4
#endif
// automatic level-1 bucket switch (options.buckets = 0): octave mapping once more than
// C / 2^TMVN_GMODE_SHIFT chains of a launch took the general interval path
#ifndef TMVN_GMODE_SHIFT
#define TMVN_GMODE_SHIFT 3
#endif
// threads per CTA: 256 (8 / W chain groups), or one 32 W-thread group when W = 16
__host__ __device__ constexpr int ess_threads(int W) { return W > 8 ? 32 * W : kEssThreads; }
__host__ __device__ constexpr int ess_groups(int W) { return W >= 8 ? 1 : 8 / W; }
template <int W, bool kRing, bool kSmemStash>
constexpr int ess_min_blocks() {
  return W > 8 ? 2
               : (W == 8 && kSmemStash && !kRing) ? TMVN_ESS_W8_BLOCKS
                                                  : TMVN_ESS_MIN_BLOCKS;
}
// kSrc: where phase A's arcs come from -- 0: P and Q rows read from global memory (the
// active test and eq:roots here), 1: the same through a shared-memory bulk-copy ring,
// 2: the projection GEMM's epilogue (options.fuse_arcs: compacted arc lists per chain)
template <int W, bool kGiven, int kSrc, bool kSmemStash>
__global__ void __launch_bounds__(ess_threads(W), (ess_min_blocks<W, kSrc == 1, kSmemStash>())) ess_kernel(
    const EssParams p) {
  constexpr bool kRing = kSrc == 1;
  constexpr bool kArcsIn = kSrc == 2;
  constexpr int kGroups = ess_groups(W);
  constexpr int T = Grp<W>::kThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Ctl ctl_all[kGroups];
  __shared__ uint64_t s_w64_all[kGroups][W];
  __shared__ int s_w32_all[kGroups][W];
  Grp<W> g;
  g.gid = threadIdx.x / T;
  g.tid = threadIdx.x % T;
  g.warp = g.tid >> 5;
  g.lane = threadIdx.x & 31;
  Ctl& ctl = ctl_all[g.gid];
  uint64_t* s_w64 = s_w64_all[g.gid];
  int* s_w32 = s_w32_all[g.gid];
  const int NB = p.NB;
  const int log2NB = 31 - __clz(NB);
  const int m = p.m;
  const int CH = p.CH;
  // per-group layout offsets precomputed on the host (EssParams): no size arithmetic here
  unsigned char* gbase = smem_raw + g.gid * p.grp_bytes;
  double* ring = reinterpret_cast<double*>(gbase);  // slot s: P at ring + 2 s CH, Q after it
  uint64_t* rbar = reinterpret_cast<uint64_t*>(gbase + (size_t)CH * 32);
  Smem S = carve(gbase + p.base_off, NB);
  const int64_t gglobal = (int64_t)blockIdx.x * kGroups + g.gid;  // group id in the grid
  // the stash's address space is a template parameter, so that every access
  // compiles to LDS/STS (shared) or LDG/STG (global) -- a run-time choice would
  // make them generic loads, ~2K cycles per dependent list hop
  double2* stash;   // arcs in production order
  if (kSmemStash) {
    stash = reinterpret_cast<double2*>(gbase + p.stash_off);
  } else {
    stash = p.gstash + (gglobal + p.group_base) * ess_gstash_stride(m);
  }
  // production path with the arcs in shared memory: the chain's P and Q rows are
  // bulk-copied (cp.async.bulk, TMA engine: no registers, no load latency exposed)
  // into the stash region while the previous chain runs phases D; phase A tests and
  // computes the arcs from there
  constexpr bool kRows = !kGiven && kSrc == 0 && kSmemStash;
  // the queue path of phase A (global stash) takes the exact max beta by CAS: no
  // low-word pass re-reading the stash from global memory
  constexpr bool kCasPath = !kGiven && kSrc == 0 && !kSmemStash && TMVN_ESS_AQUEUE && TMVN_ESS_CASMAX;
  const int mm = (m + 1) & ~1;
  // the queue path's level-1 bucket of every stashed arc (the stash's m ints after its arcs)
  int* akey = kCasPath ? reinterpret_cast<int*>(stash + m) : nullptr;
  ArcStore<kRows> AS;
  AS.st = stash;
  AS.Ps = reinterpret_cast<double*>(stash);
  AS.Qs = AS.Ps + mm;
  AS.idx = reinterpret_cast<int*>(AS.Qs + mm);
  AS.b = p.b;
  uint32_t pqphase = 0;
  auto pq_issue = [&](int64_t cn) {  // one thread
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&ctl.pqbar, (uint32_t)mm * 16u);
    bulk_g2s(AS.Ps, p.P_cur + cn * p.ldp, (uint32_t)mm * 8u, &ctl.pqbar);
    bulk_g2s(AS.Qs, p.Q + cn * p.ldp, (uint32_t)mm * 8u, &ctl.pqbar);
  };
  double2* gg = p.ggaps + (gglobal + p.group_base) * (m + 2);
  const double scale = __ddiv_rn((double)NB, kTwoPi);
  const int64_t ngroups = (int64_t)gridDim.x * kGroups;
#ifdef TMVN_PHASE_TIMING
  long long ph[14] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long t_prev = clock64();
#endif

  // P/Q chunk stream (options.ring): the group's chains are gglobal + k ngroups;
  // chain k uses chunk sequence numbers k spc .. k spc + spc - 1 (A pass, then a D1
  // pass when the row spans several chunks); sequence q lives in ring slot q & 1.
  // Consuming q issues q + 1, so the next chunk -- the next chain's rows at the end
  // of a chain -- is in flight while this one is processed.
  const int nch = (mm + CH - 1) / CH;
  const int spc = nch == 1 ? 1 : 2 * nch;
  const int64_t nmy = gglobal < p.C ? (p.C - gglobal + ngroups - 1) / ngroups : 0;
  const int64_t total_seq = (kGiven || !kRing) ? 0 : nmy * spc;
  auto ring_issue = [&](int64_t q) {  // one thread
    if (q >= total_seq) return;
    const int64_t k = q / spc;
    const int j = (int)(q % spc) % nch;
    const int64_t cq = gglobal + k * ngroups;
    const int i0 = j * CH;
    const int n = min(CH, mm - i0);
    const int s = (int)(q & 1);
    mbar_expect_tx(&rbar[s], (uint32_t)n * 16u);
    bulk_g2s(ring + (size_t)s * 2 * CH, p.P_cur + cq * p.ldp + i0, (uint32_t)n * 8u, &rbar[s]);
    bulk_g2s(ring + (size_t)s * 2 * CH + CH, p.Q + cq * p.ldp + i0, (uint32_t)n * 8u, &rbar[s]);
  };
  auto ring_wait = [&](int64_t q) { mbar_wait(&rbar[q & 1], (uint32_t)((q >> 1) & 1)); };
  int64_t qseq = 0;  // next chunk sequence number to consume
  if (!kGiven && kRing) {
    if (g.tid == 0) {
      mbar_init(&rbar[0], 1);
      mbar_init(&rbar[1], 1);
      mbar_fence_init();
    }
    g.sync();
    if (g.tid == 0) ring_issue(0);
  }

#ifdef TMVN_EXP_STAGGER  // experiment: de-phase the CTAs of an SM (4 per SM at config 3)
  if (!kGiven) __nanosleep((unsigned)((blockIdx.x / gridDim.x * 0 + (blockIdx.x * 4 / gridDim.x)) * TMVN_EXP_STAGGER));
#endif
  // iteration index and record flag (from device memory under CUDA-graph replay)
  const uint32_t t_it = p.t_dev ? *p.t_dev + p.t : p.t;
#ifdef TMVN_TIMELINE
  if (!kGiven && threadIdx.x == 0) atomicMin(&g_tl[t_it & 255][2], tl_now());
#endif
  int record = p.record;
  if (p.rec_dev) {
    const int64_t tt = (int64_t)t_it;
    record = tt >= p.burn_in && ((tt - p.burn_in) % (p.thin < 1 ? 1 : p.thin)) == 0;
  }

  // dynamic scheduling: a group grabs its next chain one round ahead (so its rows can
  // be prefetched); groups that finish early take more chains
  // Recorded iterations run round-robin (the host clears dyn_use; group g owns chains g,
  // g + G, ...): each group adds its chains' iterates into its own moment row (row g of
  // S1 / S2) in chain order, so the sums are deterministic without per-chain accumulators
  const bool dyn = !kGiven && !kRing && p.dyn_ctr != nullptr && p.dyn_use;
  int* ctr = dyn ? p.dyn_ctr + (t_it & 63) : nullptr;
  if (!kGiven && p.dyn_ctr != nullptr && blockIdx.x == 0 && threadIdx.x == 0) p.dyn_ctr[(t_it + 32) & 63] = 0;
  if (dyn) {
    if (g.tid == T - 1) ctl.next = atomicAdd(ctr, 1);
    g.sync();
  }
  if (kRows) {  // the first chain's rows
    if (g.tid == T - 1) {
      mbar_init(&ctl.pqbar, 1);
      mbar_fence_init();
      const int64_t c0 = dyn ? (int64_t)ctl.next : gglobal;
      if (c0 < p.C) pq_issue(c0);
    }
    g.sync();
  }
  // level-1 bucket mapping of this launch: linear, or by octave when chosen (options.buckets
  // = 2) or when the automatic switch saw more than 1/8 of the previous launch's chains go
  // down the general interval path or crowd a level-1 bucket (counters: launch t counts into
  // slot t % 3, reads slot (t - 1) % 3, zeroes slot (t + 1) % 3; slot 3: sticky switch)
  int l1_mode = p.bucket_mode == 2 ? 2 : 0;
  if (!kGiven && p.bucket_mode == 0 && p.gmode != nullptr && NB >= 64) {
    // one thread per chain group reads the counters (a single L2 line every CTA would
    // otherwise hammer with 512 loads); the decision reaches the group through ctl.mode
    if (g.tid == 0) {
      const uint32_t tm3 = t_it % 3u;
      if (blockIdx.x == 0 && g.gid == 0) p.gmode[(tm3 + 1) % 3] = 0;
      const int prev = *(volatile int*)(p.gmode + (tm3 + 2) % 3);
      const bool sticky = *(volatile int*)(p.gmode + 3) != 0;
      const bool oct = sticky || ((int64_t)prev << TMVN_GMODE_SHIFT) > p.C;
      if (oct && !sticky) p.gmode[3] = 1;  // written once: stores to the line every CTA reads cost
      ctl.mode = oct ? 2 : 0;
    }
    g.sync();
    l1_mode = ctl.mode;
  }
  // per-chain state (bucket tables, control words), reset before the first chain and at
  // the end of every chain, so that the loop-top barrier orders it before phase A
  auto reset_chain_state = [&]() {
    clear_buckets(g, S, NB);
    if (g.tid == 0) {
      ctl.n_act = 0;
      ctl.ngap = 0;
      ctl.G = 0.0;  // gamma_0 = 0: the first segment is [0, alpha_{i_1}]
      ctl.rlo = 0;
      ctl.rhi = kTopBits;
      ctl.mode = l1_mode;
      if (l1_mode == 2) {  // NB / 16 buckets per octave
        ctl.oct_log2 = log2NB - 4;
        ctl.shift = 52 - (log2NB - 4);
        ctl.klo = (uint64_t)((NB >> 4) - 1);
      }
      ctl.maxa_exact = 0;
      ctl.crowd = 0;
    }
  };
  reset_chain_state();
  for (int64_t cc = dyn ? (int64_t)ctl.next : gglobal; cc < p.C;
       cc = dyn ? (int64_t)ctl.next : cc + ngroups) {
    const int c = (int)cc;
    const uint32_t gchain = p.chain_offset + (uint32_t)c;
    g.sync();
    PHASE(6);  // D2 of the previous chain (x, moments, next nu) + loop overhead
    if (!kGiven && g.tid == T - 1) {
      // u for this chain (Philox latency hidden behind phase A); the next chain's
      // P and Q rows are pulled into L2 now, so its phase A loads hit L2
      ctl.u = theta_uniform(p.seed, t_it, gchain);
      if (dyn) ctl.next = atomicAdd(ctr, 1);
      const int64_t cn = dyn ? (int64_t)ctl.next : cc + ngroups;
      if (kArcsIn && cn < p.C) {  // the next chain's activity masks and arcs into L2
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.amask + cn * p.mw),
                     "r"((uint32_t)((p.mw * 4 + 15) & ~15)) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.arcs + cn * p.ald),
                     "r"((uint32_t)m * 16u) : "memory");
      }
      if (TMVN_ESS_NEXT_PREFETCH && !kRing && !kArcsIn && !kRows && cn < p.C) {
        const uint32_t bytes = (uint32_t)(((int64_t)m * 8 + 15) & ~15ll);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.P_cur + cn * p.ldp), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.Q + cn * p.ldp), "r"(bytes)
                     : "memory");
      }
    }
    if (!kGiven) {  // phase D's x and nu rows of this chain into L2 early (64-byte runs)
      const int nruns = (int)(p.d_pad / 8);
      const int64_t xrow = tiled_row(c, p.d_pad);
      for (int ru = g.tid; ru < nruns; ru += T) {
        const int64_t o = xrow + tiled_col(8 * ru);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.X + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.N + o));
      }
    }
    PHASE(0);  // init

    // ---------------- A: arcs -> stash + level-1 bucket statistics ----------------
    const double* Prow = p.P_cur + (int64_t)c * p.ldp;
    const double* Qrow = p.Q + (int64_t)c * p.ldp;
    if (kArcsIn) {
      // this chain's P and Q rows (read by phase D) into L2 while the arcs are processed
      if (g.tid == T - 1) {
        const uint32_t bytes = (uint32_t)(((int64_t)m * 8 + 15) & ~15ll);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Prow), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Qrow), "r"(bytes) : "memory");
      }
      // the arcs of the active constraints from the projection's epilogue (eq:roots with
      // C1-C5 by the same arc_of): warp w takes the 32-constraint blocks w, w + W, ..., its
      // lanes load the activity masks, then four blocks' arcs at a time are in flight;
      // stash (compacted) + level-1 bucket statistics
      const uint32_t* am = p.amask + (int64_t)c * p.mw;
      const double2* arow = p.arcs + (int64_t)c * p.ald;
      const int nbw = (p.mw - g.warp + W - 1) / W;
      for (int k0 = 0; k0 < nbw; k0 += 32) {
        const uint32_t mine = k0 + g.lane < nbw ? am[g.warp + W * (k0 + g.lane)] : 0u;
        const int kn = min(32, nbw - k0);
        for (int k = 0; k < kn; k += 4) {
          uint32_t mk[4];
          double2 ab[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            mk[u] = __shfl_sync(0xffffffffu, mine, (k + u) & 31);
            if (k + u >= kn) mk[u] = 0u;
            ab[u] = make_double2(0.0, 0.0);
            if ((mk[u] >> g.lane) & 1u) ab[u] = arow[32 * (g.warp + W * (k0 + k + u)) + g.lane];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (mk[u] == 0u) continue;  // warp-uniform
            const bool act = (mk[u] >> g.lane) & 1u;
            int sb = 0;
            if (g.lane == 0) sb = atomicAdd(&ctl.n_act, __popc(mk[u]));
            sb = __shfl_sync(0xffffffffu, sb, 0);
            if (act) {
              stash[sb + __popc(mk[u] & ((1u << g.lane) - 1u))] = ab[u];
              bucket_add<false>(S, bucket_key(ab[u].x, ctl, NB, scale), ab[u].x, ab[u].y);
              if (p.d_alpha) {
                const int i = 32 * (g.warp + W * (k0 + k + u)) + g.lane;
                p.d_alpha[(int64_t)c * m + i] = ab[u].x;
                p.d_beta[(int64_t)c * m + i] = ab[u].y;
                p.d_active[(int64_t)c * m + i] = 1;
              }
            }
          }
        }
      }
    } else if (kGiven) {
      for (int i0 = 0; i0 < m; i0 += T) {
        const int i = i0 + g.tid;
        double al = 0.0, be = 0.0;
        if (i < m) {
          al = p.g_alpha[(int64_t)c * m + i];
          be = p.g_beta[(int64_t)c * m + i];
        }
        stash_arc(S, ctl, stash, i < m, al, be, NB, scale);
      }
    } else {
      if (kRing) {
      // constraint pairs (2i, 2i+1) of each chunk: P, Q from the shared-memory ring,
      // b (shared by all chains, L1/L2-resident) from global; kBatch pairs per thread,
      // their arcs computed before the stash appends (ILP)
      const double2* B2 = reinterpret_cast<const double2*>(p.b);
      for (int j = 0; j < nch; ++j) {
        ring_wait(qseq);
        if (g.tid == 0) ring_issue(qseq + 1);
        const double2* sP2 = reinterpret_cast<const double2*>(ring + (size_t)(qseq & 1) * 2 * CH);
        const double2* sQ2 = sP2 + CH / 2;
        const int i0 = j * CH;
        const int npairs = (min(CH, m - i0) + 1) / 2;
        for (int base = 0; base < npairs; base += kBatch * T) {
          double2 pp[kBatch], qq[kBatch], bb[kBatch];
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int pi = base + u * T + g.tid;
            if (pi < npairs) {
              pp[u] = sP2[pi];
              qq[u] = sQ2[pi];
              bb[u] = __ldg(B2 + i0 / 2 + pi);
            }
          }
          double al[2 * kBatch], be[2 * kBatch];
          bool act[2 * kBatch];
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int pi = base + u * T + g.tid;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int e = 2 * u + h;
              al[e] = 0.0;
              be[e] = 0.0;
              act[e] = false;
              if (pi < npairs && i0 + 2 * pi + h < m)
                act[e] = arc_of(h ? pp[u].y : pp[u].x, h ? qq[u].y : qq[u].x, h ? bb[u].y : bb[u].x,
                                al[e], be[e]);
            }
          }
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            if (base + u * T >= npairs) break;  // uniform
            const int pi = base + u * T + g.tid;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int e = 2 * u + h, i = i0 + 2 * pi + h;
              if (p.d_alpha && pi < npairs && i < m) {
                p.d_alpha[(int64_t)c * m + i] = act[e] ? al[e] : 0.0;
                p.d_beta[(int64_t)c * m + i] = act[e] ? be[e] : 0.0;
                p.d_active[(int64_t)c * m + i] = act[e] ? 1 : 0;
              }
              stash_arc(S, ctl, stash, act[e], al[e], be[e], NB, scale);
            }
          }
        }
        ++qseq;
        g.sync();  // the slot may be refilled from now on
      }
          } else if (kRows) {
      // (1) the active test (C3/C25) on every constraint pair from the rows in shared
      // memory, the active indices compacted; (2) the arcs of the active constraints,
      // every lane busy, each written over its own (P, Q) entry
      mbar_wait(&ctl.pqbar, pqphase);
      pqphase ^= 1u;
      const double2* P2 = reinterpret_cast<const double2*>(AS.Ps);
      const double2* Q2 = reinterpret_cast<const double2*>(AS.Qs);
      const double2* B2 = reinterpret_cast<const double2*>(p.b);
      int* sidx = AS.idx;
      const int npairs = (m + 1) / 2;
      const int npr = (npairs + T - 1) / T * T;  // whole warps stay in the loop (ballots)
      for (int pi = g.tid; pi < npr; pi += T) {
        const bool in = pi < npairs;
        double2 pp = make_double2(0.0, 0.0), qq = pp, bb = pp;
        if (in) {
          pp = P2[pi];
          qq = Q2[pi];
          bb = __ldg(B2 + pi);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * pi + h;
          const bool act = in && i < m && arc_active(h ? pp.y : pp.x, h ? qq.y : qq.x, h ? bb.y : bb.x);
          if (p.d_alpha && in && i < m && !act) {
            p.d_alpha[(int64_t)c * m + i] = 0.0;
            p.d_beta[(int64_t)c * m + i] = 0.0;
            p.d_active[(int64_t)c * m + i] = 0;
          }
          const unsigned mask = __ballot_sync(0xffffffffu, act);
          if (mask) {
            const int leader = __ffs(mask) - 1;
            int sb = 0;
            if (g.lane == leader) sb = atomicAdd(&ctl.n_act, __popc(mask));
            sb = __shfl_sync(0xffffffffu, sb, leader);
            if (act) sidx[sb + __popc(mask & ((1u << g.lane) - 1u))] = i;
          }
        }
      }
      g.sync();
      PHASE(10);  // A1: active test + compaction (the rest of phase A goes to slot 1)
      if (!kKeepPQ && g.tid == T - 1) {  // phase D's P and Q rows (global) back into L2 before it reads them
        const uint32_t bytes = (uint32_t)mm * 8u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Prow), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Qrow), "r"(bytes) : "memory");
      }
      const int n_act = ctl.n_act;
      for (int slot = g.tid; slot < n_act; slot += T) {
        const int i = sidx[slot];
        double al, be;
        arc_of(AS.Ps[i], AS.Qs[i], __ldg(p.b + i), al, be);  // active by pass 1: same predicate
        if (!kKeepPQ) {
          AS.Ps[i] = al;
          AS.Qs[i] = be;
        }
        const int k = bucket_key(al, ctl, NB, scale);
        sidx[slot] = i | (k << kIdxBits);
        bucket_add<false, kKeepPQ>(S, k, al, be);
        if (p.d_alpha) {
          p.d_alpha[(int64_t)c * m + i] = al;
          p.d_beta[(int64_t)c * m + i] = be;
          p.d_active[(int64_t)c * m + i] = 1;
        }
      }
          } else if (TMVN_ESS_AQUEUE) {
      // global stash (long rows): one pass -- the active test (C3/C25) on every constraint
      // pair; each warp queues its active constraints (p, q, index) in shared memory and
      // computes their arcs 32 at a time with every lane busy, straight into the stash
      // (no (p, q) round trip through global memory; ~40-75 % of the constraints are
      // inactive and would otherwise idle their lanes through two atan2)
      const double2* P2 = reinterpret_cast<const double2*>(Prow);
      const double2* Q2 = reinterpret_cast<const double2*>(Qrow);
      const double2* B2 = reinterpret_cast<const double2*>(p.b);
      unsigned char* qbase = gbase + p.stash_off + (size_t)g.warp * kAQueueBytes;
      double* qP = reinterpret_cast<double*>(qbase);
      double* qQ = qP + kAQueue;
      int* qI = reinterpret_cast<int*>(qQ + kAQueue);
      int qn = 0;  // warp-uniform
      auto drain = [&](int n) {  // the arcs of the queue's first n <= 32 entries
        __syncwarp();
        const bool mine = g.lane < n;
        double al = 0.0, be = 0.0;
        int i = 0;
        if (mine) {
          i = qI[g.lane];
          arc_of(qP[g.lane], qQ[g.lane], __ldg(p.b + i), al, be);  // active by the test: same predicate
        }
        int sb = 0;
        if (g.lane == 0) sb = atomicAdd(&ctl.n_act, n);
        sb = __shfl_sync(0xffffffffu, sb, 0);
        if (mine) {
          stash[sb + g.lane] = make_double2(al, be);
          const int k = bucket_key(al, ctl, NB, scale);
          if (kCasPath) akey[sb + g.lane] = k;
          bucket_add<false, kCasPath>(S, k, al, be);
          if (p.d_alpha) {
            p.d_alpha[(int64_t)c * m + i] = al;
            p.d_beta[(int64_t)c * m + i] = be;
            p.d_active[(int64_t)c * m + i] = 1;
          }
        }
        __syncwarp();
      };
      const int npairs = (m + 1) / 2;
      const int npr = (npairs + T - 1) / T * T;  // whole warps stay in the loop (ballots)
      for (int base = 0; base < npr; base += kBatchA1 * T) {
        if (TMVN_ESS_PF_DIST > 0) {  // the rows TMVN_ESS_PF_DIST passes ahead into L2 (no registers)
          const int pf = base + g.tid + TMVN_ESS_PF_DIST * kBatchA1 * T;
          if (pf < npairs) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(P2 + pf));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(Q2 + pf));
          }
        }
        double2 pp[kBatchA1], qq[kBatchA1], bb[kBatchA1];
#pragma unroll
        for (int u = 0; u < kBatchA1; ++u) {
          const int pi = base + u * T + g.tid;
          if (pi < npairs) {
            pp[u] = P2[pi];
            qq[u] = Q2[pi];
            bb[u] = __ldg(B2 + pi);
          }
        }
#pragma unroll
        for (int u = 0; u < kBatchA1; ++u) {
          if (base + u * T >= npr) break;  // uniform
          const int pi = base + u * T + g.tid;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = 2 * pi + h;
            const double pv = h ? pp[u].y : pp[u].x, qv = h ? qq[u].y : qq[u].x, bv = h ? bb[u].y : bb[u].x;
            const bool act = pi < npairs && i < m && arc_active(pv, qv, bv);
            if (p.d_alpha && pi < npairs && i < m && !act) {
              p.d_alpha[(int64_t)c * m + i] = 0.0;
              p.d_beta[(int64_t)c * m + i] = 0.0;
              p.d_active[(int64_t)c * m + i] = 0;
            }
            const unsigned mask = __ballot_sync(0xffffffffu, act);
            if (act) {
              const int pos = qn + __popc(mask & ((1u << g.lane) - 1u));
              qP[pos] = pv;
              qQ[pos] = qv;
              qI[pos] = i;
            }
            qn += __popc(mask);
            if (qn >= 32) {  // a full warp of arcs; the rest (< 32) moves to the front
              drain(32);
              const int rest = qn - 32;
              if (g.lane < rest) {
                qP[g.lane] = qP[32 + g.lane];
                qQ[g.lane] = qQ[32 + g.lane];
                qI[g.lane] = qI[32 + g.lane];
              }
              __syncwarp();
              qn = rest;
            }
          }
        }
      }
      if (qn > 0) drain(qn);
      PHASE(10);  // A1: active test + arcs (one pass here; slot 1 gets the barrier)
          } else {
      // (TMVN_ESS_AQUEUE = 0) two passes: (1) the active test (C3/C25) on every constraint pair, active
      // (p, q) and the index compacted into the stash; (2) the arcs of the active
      // constraints only, every lane busy (about 40 % of the constraints are
      // inactive at config 3 and would idle their lanes through two atan2)
      const double2* P2 = reinterpret_cast<const double2*>(Prow);
      const double2* Q2 = reinterpret_cast<const double2*>(Qrow);
      const double2* B2 = reinterpret_cast<const double2*>(p.b);
      int* sidx = reinterpret_cast<int*>(stash + m);  // m ints after the group's stash (shared or global)
      const int npairs = (m + 1) / 2;
      for (int base = 0; base < npairs; base += kBatchA1 * T) {
        double2 pp[kBatchA1], qq[kBatchA1], bb[kBatchA1];
#pragma unroll
        for (int u = 0; u < kBatchA1; ++u) {
          const int pi = base + u * T + g.tid;
          if (pi < npairs) {
            pp[u] = P2[pi];
            qq[u] = Q2[pi];
            bb[u] = __ldg(B2 + pi);
          }
        }
#pragma unroll
        for (int u = 0; u < kBatchA1; ++u) {
          if (base + u * T >= npairs) break;  // uniform
          const int pi = base + u * T + g.tid;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = 2 * pi + h;
            const double pv = h ? pp[u].y : pp[u].x, qv = h ? qq[u].y : qq[u].x, bv = h ? bb[u].y : bb[u].x;
            const bool act = pi < npairs && i < m && arc_active(pv, qv, bv);
            if (p.d_alpha && pi < npairs && i < m && !act) {
              p.d_alpha[(int64_t)c * m + i] = 0.0;
              p.d_beta[(int64_t)c * m + i] = 0.0;
              p.d_active[(int64_t)c * m + i] = 0;
            }
            const unsigned mask = __ballot_sync(0xffffffffu, act);
            if (mask) {
              const int leader = __ffs(mask) - 1;
              int sb = 0;
              if (g.lane == leader) sb = atomicAdd(&ctl.n_act, __popc(mask));
              sb = __shfl_sync(0xffffffffu, sb, leader);
              if (act) {
                const int slot = sb + __popc(mask & ((1u << g.lane) - 1u));
                stash[slot] = make_double2(pv, qv);
                sidx[slot] = i;
              }
            }
          }
        }
      }
      g.sync();
      PHASE(10);  // A1: active test + compaction (the rest of phase A goes to slot 1)
      const int n_act = ctl.n_act;
      for (int slot = g.tid; slot < n_act; slot += T) {
        const double2 pq = stash[slot];
        const int i = sidx[slot];
        double al, be;
        arc_of(pq.x, pq.y, __ldg(p.b + i), al, be);  // active by pass 1: same predicate
        stash[slot] = make_double2(al, be);
        bucket_add<false>(S, bucket_key(al, ctl, NB, scale), al, be);
        if (p.d_alpha) {
          p.d_alpha[(int64_t)c * m + i] = al;
          p.d_beta[(int64_t)c * m + i] = be;
          p.d_active[(int64_t)c * m + i] = 1;
        }
      }
          }
    }
    g.sync();
    PHASE(1);  // A: arcs, stash, level-1 statistics
    PHASE_ADD(8, ctl.n_act);

    // level-1 bucket ranges (exclusive scan of the counts), then one pass over the
    // stash: resolve the low words of max beta (see bucket_add) and scatter every arc
    // into its bucket's range (counting sort by bucket)
    if (!kCasPath && !(kRows && kKeepPQ)) {
      const int n_act = ctl.n_act;
      for (int idx = g.tid; idx < n_act; idx += T) {
        const double2 ab = AS.get(idx);
        bucket_add_lo<false>(S, bucket_key(ab.x, ctl, NB, scale), ab.x, ab.y);
      }
      g.sync();
    }
    PHASE(2);  // low-word pass

    // ---------------- B + C: I_act by Alg. 3, then theta ----------------
    // a chain is crowded when one level-1 bucket holds 4 x the mean constraints per
    // bucket + 32 arcs (phase A's bucket atomics and B3's scan serialise on it)
    const bool fast = par_intervals(g, S, ctl, AS, NB, scale, gg, s_w64, s_w32, 4 * (m / NB) + 32, akey);
    // nu_{t+1} drawn while the highest warp's last lane computes theta (options.rng_overlap:
    // the other W - 1 warps would wait at the barrier); into the other nu buffer (N_next),
    // since phase D still reads nu_t
    const bool rng_here = !kGiven && W > 1 && fast && p.gen_next && p.N_next != nullptr;
    if (fast && g.tid == T - 1) {  // theta on the highest warp (arbiter: highest warp id first)
      const double u = kGiven ? (p.g_u ? p.g_u[c] : 0.0) : ctl.u;
      theta_from_gaps(S, ctl, gg, u, p.eps);
    } else if (rng_here && g.warp < W - 1) {
      const int kpairs = (int)(p.d_pad / 2);
      const int64_t xr = tiled_row(c, p.d_pad);
      const int64_t zr = p.Ns ? oz_row(c, p.ozS, p.ozKB, kOzNuRows) : 0;
      for (int pk = g.tid; pk < kpairs; pk += 32 * (W - 1)) {
        const int k = 2 * pk;
        const double2 nv = normal_pair_at(p.seed, t_it + 1, gchain, k, p.d);
        *reinterpret_cast<double2*>(p.N_next + (xr + tiled_col(k))) = nv;
        if (p.Ns) oz_put_nu_pair_s(p.Ns + (zr + oz_col(k, p.ozS, kOzNuRows)), nv.x, nv.y, p.ozS);
      }
    }
    g.sync();
    PHASE(3);  // B (+C) on the parallel path
    PHASE_ADD(7, fast ? 0 : 1);
    // automatic level-1 mapping: count the chains that went down the general path or
    // crowded a level-1 bucket (arcs bunched in a few linear buckets); none once octave
    if (!kGiven && l1_mode == 0 && p.gmode != nullptr && g.tid == 0 && (!fast || ctl.crowd)) {
      atomicAdd(p.gmode + (t_it % 3u), 1);
      ctl.crowd = 0;
    }
    if (!fast) {
      build_intervals(g, S, ctl, AS, NB, log2NB, scale, gg, s_w64, s_w32);
      if (g.tid == 0) {
        const double u = kGiven ? (p.g_u ? p.g_u[c] : 0.0) : ctl.u;
        theta_from_gaps(S, ctl, gg, u, p.eps);
      }
      g.sync();
    }
    PHASE(4);  // B + C on the general path (rare)
    PHASE_ADD(9, ctl.ngap);
    if (kRows && !kKeepPQ && g.tid == T - 1) {  // stash free: the next chain's P and Q rows, beside phase D
      const int64_t cn = dyn ? (int64_t)ctl.next : cc + ngroups;
      if (cn < p.C) pq_issue(cn);
    }
    if (g.tid == 0) {
      if (p.d_nseg) p.d_nseg[c] = ctl.nseg;
      if (p.d_L) p.d_L[c] = ctl.L;
      if (p.d_theta) p.d_theta[c] = ctl.theta;
    }
    if (p.d_seg_lo) {
      const int ns = ctl.nseg;
      for (int k = g.tid; k < ns && k < p.seg_cap; k += T) {
        double2 gv = gap_load(S, gg, k);
        p.d_seg_lo[(int64_t)c * p.seg_cap + k] = gv.x;
        p.d_seg_hi[(int64_t)c * p.seg_cap + k] = gv.y;
      }
    }
    if (kGiven) {
      g.sync();  // the dumps above read ctl and the gaps
      reset_chain_state();
      continue;
    }

    // ---------------- D: safeguard, P', x update, moments, next nu ----------------
    const double L = ctl.L;
    // sin / cos by every thread: on the critical path in parallel, not behind a barrier
    double st = 0.0, ct = 1.0;
    if (L > 0.0) sincos(ctl.theta, &st, &ct);
    const int npairs = (m + 1) / 2;
    const double2* P2 = reinterpret_cast<const double2*>(Prow);
    const double2* B2 = reinterpret_cast<const double2*>(p.b);
    double2* Pn2 = reinterpret_cast<double2*>(p.P_next + (int64_t)c * p.ldp);
    int viol = 0;
    double smax = -DBL_MAX;
    // P' = P cos(theta) + Q sin(theta) from the ring: the chunk still resident when the
    // row is one chunk, else a second pass over the chunks
    for (int j = 0; kRing && j < nch; ++j) {
      int64_t qc = qseq - 1;  // single chunk: the one consumed in phase A
      if (nch > 1) {
        qc = qseq;
        ring_wait(qseq);
        if (g.tid == 0) ring_issue(qseq + 1);
      }
      const double2* sP2 = reinterpret_cast<const double2*>(ring + (size_t)(qc & 1) * 2 * CH);
      const double2* sQ2 = sP2 + CH / 2;
      const int i0 = j * CH;
      const int np = (min(CH, m - i0) + 1) / 2;
      if (L > 0.0) {
        for (int pi = g.tid; pi < np; pi += T) {
          const double2 pv = sP2[pi], qv = sQ2[pi], bv = __ldg(B2 + i0 / 2 + pi);
          double2 pn;
          pn.x = pv.x * ct + qv.x * st;
          pn.y = pv.y * ct + qv.y * st;
          const double s0 = pn.x - bv.x, s1 = pn.y - bv.y;  // b is +inf beyond m
          viol |= (s0 > 0.0) | (s1 > 0.0);
          smax = fmax(smax, fmax(s0, s1));
          Pn2[i0 / 2 + pi] = pn;
        }
      }
      if (nch > 1) {
        ++qseq;
        g.sync();
      }
    }
    if (!kRing && L > 0.0) {
      // the rows still in shared memory (TMVN_ESS_KEEPPQ), else from global memory
      const double2* Ps2 = (kRows && kKeepPQ) ? reinterpret_cast<const double2*>(AS.Ps) : P2;
      const double2* Q2 = (kRows && kKeepPQ) ? reinterpret_cast<const double2*>(AS.Qs)
                                             : reinterpret_cast<const double2*>(Qrow);
      for (int pi = g.tid; pi < npairs; pi += T) {
        if (TMVN_ESS_PF_DIST > 0 && (!kRows || TMVN_ESS_PF_ROWS)) {
          const int pf = pi + TMVN_ESS_PF_DIST * T;
          if (pf < npairs) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(Ps2 + pf));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(Q2 + pf));
          }
        }
        const double2 pv = Ps2[pi], qv = Q2[pi], bv = __ldg(B2 + pi);
        double2 pn;
        pn.x = pv.x * ct + qv.x * st;
        pn.y = pv.y * ct + qv.y * st;
        const double s0 = pn.x - bv.x, s1 = pn.y - bv.y;  // b is +inf beyond m
        viol |= (s0 > 0.0) | (s1 > 0.0);
        smax = fmax(smax, fmax(s0, s1));
        Pn2[pi] = pn;
      }
    }
    const int any_viol = g.sync_or(viol);
    const bool accept = (L > 0.0) && !any_viol;
    if (kRows && kKeepPQ && g.tid == T - 1) {  // rows read (barrier above): the next chain's, beside D2
      const int64_t cn = dyn ? (int64_t)ctl.next : cc + ngroups;
      if (cn < p.C) pq_issue(cn);
    }
    PHASE(5);  // D1: P' and the safeguard
    if (p.d_slack) {
      // group max of the slack (dump only)
      uint64_t key = dbits(smax) ^ ((dbits(smax) >> 63) ? ~0ull : 0x8000000000000000ull);
      uint64_t tot;
      grp_excl_max(g, key, 0, s_w64, &tot);
      if (g.tid == 0) {
        uint64_t bits = (tot >> 63) ? (tot ^ 0x8000000000000000ull) : ~tot;
        p.d_slack[c] = L > 0.0 ? bitsd(bits) : 0.0;
      }
    }
    if (!accept) {
      for (int pi = g.tid; pi < npairs; pi += T) Pn2[pi] = P2[pi];  // stay at x_t
    }
    // x (and moments, next nu) by coordinate pairs: one double2 of the tiled X / N each;
    // offsets = row part (per chain) + column part (stepped by 32-bit adds)
    const int kpairs = (int)(p.d_pad / 2);
    const int64_t xrow = tiled_row(c, p.d_pad);
    const int64_t mrow = tiled_row(gglobal + p.group_base, p.d_pad) - xrow;  // this group's moment row
    const int64_t zrow = p.Ns ? oz_row(c, p.ozS, p.ozKB, kOzNuRows) : 0;
    for (int pk = g.tid; pk < kpairs; pk += T) {
      const int k = 2 * pk;
      const int64_t o = xrow + tiled_col(k);
      double2* xr = reinterpret_cast<double2*>(p.X + o);
      double2* nr = reinterpret_cast<double2*>(p.N + o);
      double2 xv = *xr;
      if (accept) {
        const double2 nv = *nr;
        xv.x = xv.x * ct + nv.x * st;
        xv.y = xv.y * ct + nv.y * st;
        *xr = xv;
      }
      if (record) {  // the group's moment row (L2-resident): deterministic chain order
        double2* s1 = reinterpret_cast<double2*>(p.S1 + (o + mrow));
        double2* s2 = reinterpret_cast<double2*>(p.S2 + (o + mrow));
        double2 a1 = *s1, a2 = *s2;
        a1.x += xv.x;
        a1.y += xv.y;
        a2.x += xv.x * xv.x;
        a2.y += xv.y * xv.y;
        *s1 = a1;
        *s2 = a2;
      }
      if (p.gen_next && !rng_here) {
#ifdef TMVN_EXP_NO_RNG  // timing experiment only (wrong results): the kernel without drawing nu
        const double2 nv = make_double2(xv.y * 1e-3, xv.x * 1e-3);
#else
        const double2 nv = normal_pair_at(p.seed, t_it + 1, gchain, k, p.d);
#endif
        if (p.N_next) *reinterpret_cast<double2*>(p.N_next + o) = nv;
        else *nr = nv;
        if (p.Ns) oz_put_nu_pair_s(p.Ns + (zrow + oz_col(k, p.ozS, kOzNuRows)), nv.x, nv.y, p.ozS);
      }
    }
    if (g.tid == 0) {
      if (!accept) p.rej[c] += 1;
      if (p.d_accept) p.d_accept[c] = accept ? 1 : 0;
    }
    reset_chain_state();  // phase D reads neither the bucket tables nor ctl's interval words
  }
#ifdef TMVN_TIMELINE
  if (!kGiven && threadIdx.x == 0) atomicMax(&g_tl[t_it & 255][3], tl_now());
#endif
#ifdef TMVN_PHASE_TIMING
  g.sync();
  PHASE(6);
  if (g.tid == 0)
    for (int i = 0; i < 14; ++i) atomicAdd(&g_phase_cycles[i], (unsigned long long)ph[i]);
#endif
}

template <int W, bool kGiven, int kSrc, bool kSmemStash>
cudaError_t launch_k(const EssParams& p, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(ess_kernel<W, kGiven, kSrc, kSmemStash>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ess_kernel<W, kGiven, kSrc, kSmemStash><<<grid, ess_threads(W), smem, st>>>(p);
  return cudaGetLastError();
}

template <int W, bool kGiven>
cudaError_t launch_w(const EssParams& p, int grid, size_t smem, cudaStream_t st) {
  if (!kGiven && p.arcs) {
    return p.stash_smem ? launch_k<W, kGiven, 2, true>(p, grid, smem, st)
                        : launch_k<W, kGiven, 2, false>(p, grid, smem, st);
  }
  const bool ring = !kGiven && p.CH > 0;
  if (ring) {
    return p.stash_smem ? launch_k<W, kGiven, 1, true>(p, grid, smem, st)
                        : launch_k<W, kGiven, 1, false>(p, grid, smem, st);
  }
  return p.stash_smem ? launch_k<W, kGiven, 0, true>(p, grid, smem, st)
                      : launch_k<W, kGiven, 0, false>(p, grid, smem, st);
}

template <bool kGiven>
cudaError_t launch_any(const EssParams& p0, int grid, cudaStream_t st) {
  if (grid < 1) return cudaSuccess;
  EssParams p = p0;
  p.grp_bytes = (int)ess_group_smem_bytes(p.m, p.NB, p.stash_smem, p.CH, p.W);
  p.base_off = (int)ess_ring_bytes(p.CH);
  p.stash_off = p.base_off + (int)ess_group_base_bytes(p.NB);
  const size_t smem = (size_t)ess_groups(p.W) * (size_t)p.grp_bytes;
  switch (p.W) {
    case 1: return launch_w<1, kGiven>(p, grid, smem, st);
    case 2: return launch_w<2, kGiven>(p, grid, smem, st);
    case 4: return launch_w<4, kGiven>(p, grid, smem, st);
    case 8: return launch_w<8, kGiven>(p, grid, smem, st);
    case 16: return launch_w<16, kGiven>(p, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int W, int kSrc, bool kSmemStash>
int occupancy_k(size_t smem) {
  int per_sm = 0;
  cudaFuncSetAttribute(ess_kernel<W, false, kSrc, kSmemStash>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ess_kernel<W, false, kSrc, kSmemStash>,
                                                ess_threads(W), smem);
  return per_sm;
}

template <int W>
int occupancy_w(size_t smem, bool ring, bool smem_stash) {
  if (ring) return smem_stash ? occupancy_k<W, 1, true>(smem) : occupancy_k<W, 1, false>(smem);
  return smem_stash ? occupancy_k<W, 0, true>(smem) : occupancy_k<W, 0, false>(smem);
}

}  // namespace

#ifdef TMVN_PHASE_TIMING
void phase_cycles(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 14);
  if (reset) {
    unsigned long long z[14] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
}
#endif

static int g_sms = 0;

EssLaunch ess_plan(int C, int m, int W_req, int ring_req) {
  if (g_sms == 0) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  EssLaunch L;
  // warps per chain: as few as still give every SM several chains in flight;
  // more warps per chain when chains are few or constraints many
  int W = W_req;
  if (W != 1 && W != 2 && W != 4 && W != 8 && W != 16) {
    // measured on B200 (tools/ab_time.py): a full CTA per chain once rows are long;
    // fewer warps per chain (more chains in flight) for short rows
    W = m >= 1024 ? 8 : m >= 256 ? 4 : m >= 48 ? 2 : 1;
    // fewer chains than SMs: a whole CTA per chain (latency-bound regime; the paper's
    // S4.2 workload, 10 chains at d = m = 1000: 47 -> 34 us per launch)
    if (C <= g_sms && m >= 48) W = 8;
    // up to two chains per SM with long rows: a 512-thread CTA per chain (C = 80..256,
    // d = m = 1000: 5-9 % per iteration; beyond 2 x SMs chains, 16 warps lose)
    if (C <= 2 * g_sms && m >= 512) W = 16;
    // very long rows (the global-stash path with the streaming L2 prefetch): a 512-thread
    // CTA per chain whatever the chain count (B200, one launch over all chains: config 4
    // 1.364 -> 1.096 ms, config 5 25.3 -> 24.0 ms per launch)
    if (m >= 8192) W = 16;
  }
  // buckets: about 16 constraints (~8 arcs) per level-1 bucket, 64 .. 1024
  int NB = 64;
  while (NB < m / TMVN_ESS_NB_DIV && NB < 1024) NB <<= 1;
  // a requested W whose per-CTA chain groups' bucket tables would not fit in shared
  // memory (e.g. W = 1, 8 groups, with 1024 level-1 buckets): more warps, fewer groups
  auto min_bytes = [&](int w) {
    return (size_t)ess_groups(w) *
           ess_group_smem_bytes(m, NB, 0, ring_req ? std::min(256 * w, (m + 1) & ~1) : 0, w);
  };
  while (W < 8 && min_bytes(W) > 200 * 1024) W <<= 1;
  const int groups = ess_groups(W);
  // P/Q chunk: 256 W constraints (64 KB ring for a full CTA), never beyond the row;
  // CH = 0: no ring, P and Q are read from global memory
  const int mm = (m + 1) & ~1;
  int CH = 256 * W;
  if (CH > mm) CH = mm;
  if (ring_req == 0) CH = 0;
  // stash in shared memory when 2 CTAs per SM still fit
  int stash_smem = 0;
  if ((size_t)groups * ess_group_smem_bytes(m, NB, 1, CH) <= 112 * 1024) stash_smem = 1;
  const size_t smem = (size_t)groups * ess_group_smem_bytes(m, NB, stash_smem, CH, W);
  int per_sm = 0;
  switch (W) {
    case 1: per_sm = occupancy_w<1>(smem, CH > 0, stash_smem); break;
    case 2: per_sm = occupancy_w<2>(smem, CH > 0, stash_smem); break;
    case 4: per_sm = occupancy_w<4>(smem, CH > 0, stash_smem); break;
    case 16: per_sm = occupancy_w<16>(smem, CH > 0, stash_smem); break;
    default: per_sm = occupancy_w<8>(smem, CH > 0, stash_smem); break;
  }
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)g_sms * per_sm;
  const int64_t need = ((int64_t)C + groups - 1) / groups;
  L.W = W;
  L.NB = NB;
  L.CH = CH;
  L.stash_smem = stash_smem;
  L.grid = (int)(grid < need ? grid : need);
  L.groups = (int64_t)L.grid * groups;
  return L;
}

cudaError_t launch_ess_step(const EssParams& p, int grid, cudaStream_t st) {
  return launch_any<false>(p, grid, st);
}

cudaError_t launch_ess_intervals(const EssParams& p, int grid, cudaStream_t st) {
  return launch_any<true>(p, grid, st);
}


#ifdef TMVN_TIMELINE
void tl_access_ess(unsigned long long* out, bool reset) {
  cudaDeviceSynchronize();
  if (reset) {
    static unsigned long long z[256][4];
    for (int i = 0; i < 256; ++i) { z[i][0] = z[i][2] = ~0ull; z[i][1] = z[i][3] = 0; }
    cudaMemcpyToSymbol(g_tl, z, sizeof(z));
    unsigned int zs[2] = {0, 0};
    cudaMemcpyToSymbol(g_tl_seq, zs, sizeof(zs));
  } else {
    cudaMemcpyFromSymbol(out, g_tl, 256 * 4 * 8);
  }
}
#endif
}  // namespace tmvn
