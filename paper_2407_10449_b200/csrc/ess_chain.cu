// ess_chain.cu -- one fused kernel per ESS iteration for every chain (Alg. 1,
// P:169-181), everything after the projection GEMM:
//
//   A  arcs      per constraint i: r = hypot(p, q), the infeasible arc
//                (alpha_i, beta_i) of eq:roots (C1-C5); inactive
//                constraints (r <= b) are compacted away.
//   B  I_act     Alg. 3 / Prop. 1: sort the alphas, cumulative max
//                of the co-sorted betas, gaps [gamma_{k-1}, alpha_{i_k}] and
//                [gamma_m, 2 pi].  The sort is an MSD bucket sort on alpha whose
//                first level also yields, per bucket, max(alpha), max(beta):
//                the exclusive prefix max of max(beta) is gamma entering the
//                bucket, and a bucket whose max(alpha) does not exceed it can
//                hold no gap (Prop. 1), so only "live" buckets are gathered and
//                sorted in shared memory (bitonic) and scanned (max-scan).
//                Comparisons only: bit-identical to Alg. 2 on the same arcs
//                (P:400-402).  Oversized buckets are refined level by level.
//   C  theta     canonical segments, S3.3 trim (C7), L = sum of lengths in
//                ascending order, theta = inverse CDF at u (C10).
//   D  update    P' = P cos(theta) + Q sin(theta) (Eq. 1), safeguard
//                accept iff max_i (P'_i - b_i) <= 0 (C8),
//                x <- x cos(theta) + nu sin(theta), moments, then nu for t+1.
//
// One CTA (256 threads) per chain, persistent grid-stride over chains.
#include <cfloat>
#include "common.cuh"
#include "internal.h"

namespace tmvn {
namespace {

constexpr int kWarps = kEssThreads / 32;
constexpr uint64_t kTopBits = 0x7FF0000000000000ull;  // +inf: every alpha in [0, 2 pi] is below

__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(uint64_t b) { return __longlong_as_double((long long)b); }

struct Ctl {
  uint64_t rlo, rhi, klo;
  int shift, mode;      // key: mode 0 linear on [0, 2 pi]; mode 1 (bits - klo) >> shift
  double G;             // running gamma: max beta over every arc already passed
  int n_act;
  int ngap;
  int total_live;
  int jo;
  int action;
  int nseg;
  double L, theta;
  int viol;
  double slack;
};

enum { kAll = 0, kPrefix = 1, kSame = 2, kNarrow = 3 };

// --- block scans (blockDim == kEssThreads) -----------------------------------
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
// exclusive max-scan of v over threads (init `init`); *total = max(init, all v)
__device__ uint64_t block_excl_max(uint64_t v, uint64_t init, uint64_t* s_w, uint64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t inc = warp_incl_max(v);
  uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) exc = 0;
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  uint64_t pre = init;
  for (int i = 0; i < w; ++i) pre = pre > s_w[i] ? pre : s_w[i];
  uint64_t tot = init;
  for (int i = 0; i < kWarps; ++i) tot = tot > s_w[i] ? tot : s_w[i];
  __syncthreads();
  *total = tot;
  return pre > exc ? pre : exc;
}
__device__ int block_excl_sum(int v, int* s_w, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = warp_incl_sum(v);
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  int pre = 0, tot = 0;
  for (int i = 0; i < kWarps; ++i) {
    if (i < w) pre += s_w[i];
    tot += s_w[i];
  }
  __syncthreads();
  *total = tot;
  return pre + inc - v;
}

struct Smem {
  uint64_t* maxA;
  uint64_t* maxB;
  uint64_t* minA;
  uint64_t* Gx;
  int* cnt;
  int* off;
  uint64_t* keys;  // kLiveCap
  double* vals;    // kLiveCap
  double2* gaps;   // kGapSmem
  double2* stash;  // m (if in smem)
};

__device__ __forceinline__ int bucket_key(double a, const Ctl& c, int NB, double scale) {
  if (c.mode == 0) {
    int k = (int)__dmul_rn(a, scale);
    return k < NB - 1 ? k : NB - 1;
  }
  uint64_t k = (dbits(a) - c.klo) >> c.shift;
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

__device__ void clear_buckets(const Smem& S, int NB) {
  for (int j = threadIdx.x; j < NB; j += blockDim.x) {
    S.maxA[j] = 0;
    S.maxB[j] = 0;
    S.minA[j] = ~0ull;
    S.cnt[j] = 0;
  }
}

__device__ __forceinline__ void bucket_add(const Smem& S, int k, double a, double b) {
  atomicMax((unsigned long long*)&S.maxA[k], (unsigned long long)dbits(a));
  atomicMax((unsigned long long*)&S.maxB[k], (unsigned long long)dbits(b));
  atomicMin((unsigned long long*)&S.minA[k], (unsigned long long)dbits(a));
  atomicAdd(&S.cnt[k], 1);
}

// Bitonic sort of keys/vals[0, n) (n <= kLiveCap) ascending by key.
__device__ void block_sort(const Smem& S, int n) {
  int n2 = 2;
  while (n2 < n) n2 <<= 1;
  for (int i = n + threadIdx.x; i < n2; i += blockDim.x) S.keys[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
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
      __syncthreads();
    }
  }
}

// Gather the arcs of live buckets with key < jo into keys/vals, sort, emit gaps.
__device__ void process_batch(const Smem& S, Ctl& ctl, const double2* stash, int n_act, int jo,
                              int n_live, int NB, double scale, double2* gg, uint64_t* s_w64,
                              int* s_w32) {
  for (int idx = threadIdx.x; idx < n_act; idx += blockDim.x) {
    double2 ab = stash[idx];
    uint64_t bits = dbits(ab.x);
    if (bits < ctl.rlo || bits > ctl.rhi) continue;
    int k = bucket_key(ab.x, ctl, NB, scale);
    if (k >= jo) continue;
    if (!(S.cnt[k] > 0 && S.maxA[k] > S.Gx[k])) continue;  // dead bucket: no gap (Prop. 1)
    int pos = atomicAdd(&S.off[k], 1);
    S.keys[pos] = bits;
    S.vals[pos] = ab.y;
  }
  __syncthreads();
  block_sort(S, n_live);
  // gamma before element e: max(Gx[bucket], max beta of earlier elements of the batch)
  const int per = (n_live + blockDim.x - 1) / blockDim.x;
  const int e0 = threadIdx.x * per, e1 = min(n_live, e0 + per);
  uint64_t lmax = 0;
  for (int e = e0; e < e1; ++e) lmax = lmax > dbits(S.vals[e]) ? lmax : dbits(S.vals[e]);
  uint64_t tot64;
  uint64_t run = block_excl_max(lmax, 0, s_w64, &tot64);
  // first pass: count gaps of my elements
  int mine = 0;
  {
    uint64_t r = run;
    for (int e = e0; e < e1; ++e) {
      double a = bitsd(S.keys[e]);
      uint64_t g = S.Gx[bucket_key(a, ctl, NB, scale)];
      g = g > r ? g : r;
      if (S.keys[e] > g) ++mine;
      uint64_t vb = dbits(S.vals[e]);
      r = r > vb ? r : vb;
    }
  }
  int total;
  int pos = block_excl_sum(mine, s_w32, &total) + ctl.ngap;
  {
    uint64_t r = run;
    for (int e = e0; e < e1; ++e) {
      double a = bitsd(S.keys[e]);
      uint64_t g = S.Gx[bucket_key(a, ctl, NB, scale)];
      g = g > r ? g : r;
      if (S.keys[e] > g) gap_store(S, gg, pos++, bitsd(g), a);
      uint64_t vb = dbits(S.vals[e]);
      r = r > vb ? r : vb;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ctl.ngap += total;
  __syncthreads();
}

// Alg. 3 over the stashed arcs -> gaps (ascending) in S.gaps / gg; ctl.ngap set.
// On entry the level-1 bucket statistics (linear keys on [0, 2 pi]) are filled.
__device__ void build_intervals(const Smem& S, Ctl& ctl, const double2* stash, int NB, int log2NB,
                                double scale, double2* gg, uint64_t* s_w64, int* s_w32) {
  const int n_act = ctl.n_act;
  bool first = true;
  for (;;) {
    if (!first) {
      clear_buckets(S, NB);
      __syncthreads();
      for (int idx = threadIdx.x; idx < n_act; idx += blockDim.x) {
        double2 ab = stash[idx];
        uint64_t bits = dbits(ab.x);
        if (bits < ctl.rlo || bits > ctl.rhi) continue;
        bucket_add(S, bucket_key(ab.x, ctl, NB, scale), ab.x, ab.y);
      }
      __syncthreads();
    }
    first = false;
    // scan buckets: Gx = exclusive prefix max of maxB (init G); live counts and offsets
    const int per = (NB + blockDim.x - 1) / blockDim.x;
    const int j0 = threadIdx.x * per, j1 = min(NB, j0 + per);
    uint64_t lmax = 0;
    for (int j = j0; j < j1; ++j) lmax = lmax > S.maxB[j] ? lmax : S.maxB[j];
    uint64_t Gtot;
    uint64_t run = block_excl_max(lmax, dbits(ctl.G), s_w64, &Gtot);
    int lcount = 0;
    for (int j = j0; j < j1; ++j) {
      S.Gx[j] = run;
      run = run > S.maxB[j] ? run : S.maxB[j];
      if (S.cnt[j] > 0 && S.maxA[j] > S.Gx[j]) lcount += S.cnt[j];
    }
    int total_live;
    int o = block_excl_sum(lcount, s_w32, &total_live);
    for (int j = j0; j < j1; ++j) {
      S.off[j] = o;
      if (S.cnt[j] > 0 && S.maxA[j] > S.Gx[j]) o += S.cnt[j];
    }
    if (threadIdx.x == 0) {
      ctl.total_live = total_live;
      ctl.jo = NB;
    }
    __syncthreads();
    if (total_live > kLiveCap) {
      for (int j = j0; j < j1; ++j) {
        int lc = (S.cnt[j] > 0 && S.maxA[j] > S.Gx[j]) ? S.cnt[j] : 0;
        if (lc > 0 && S.off[j] + lc > kLiveCap) atomicMin(&ctl.jo, j);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (ctl.total_live <= kLiveCap) ctl.action = kAll;
      else if (S.off[ctl.jo] > 0) ctl.action = kPrefix;
      else if (S.minA[ctl.jo] == S.maxA[ctl.jo]) ctl.action = kSame;
      else ctl.action = kNarrow;
    }
    __syncthreads();
    const int action = ctl.action, jo = ctl.jo;
    if (action == kAll || action == kPrefix) {
      int n_live = action == kAll ? total_live : S.off[jo];
      if (n_live > 0) process_batch(S, ctl, stash, n_act, jo, n_live, NB, scale, gg, s_w64, s_w32);
    }
    if (threadIdx.x == 0) {
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
        uint64_t gb = S.Gx[jo] > S.maxB[jo] ? S.Gx[jo] : S.maxB[jo];
        ctl.G = bitsd(gb);
        ctl.rlo = S.maxA[jo] + 1;
        set_bits_mode(ctl, log2NB);
      } else {
        ctl.G = bitsd(S.Gx[jo]);
        ctl.rlo = S.minA[jo];
        ctl.rhi = S.maxA[jo];
        set_bits_mode(ctl, log2NB);
      }
    }
    __syncthreads();
    if (ctl.action == -1) break;
  }
  if (threadIdx.x == 0) {
    if (ctl.G < kTwoPi) {  // the last segment [gamma_m, 2 pi]
      gap_store(S, gg, ctl.ngap, ctl.G, kTwoPi);
      ctl.ngap += 1;
    }
  }
  __syncthreads();
}

// Canonical segments (merge touching), trim, L and theta.  Thread 0 only.
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

__device__ Smem carve(unsigned char* base, int NB, int m, bool stash_smem) {
  Smem S;
  S.maxA = reinterpret_cast<uint64_t*>(base);
  S.maxB = S.maxA + NB;
  S.minA = S.maxB + NB;
  S.Gx = S.minA + NB;
  S.keys = S.Gx + NB;
  S.vals = reinterpret_cast<double*>(S.keys + kLiveCap);
  S.gaps = reinterpret_cast<double2*>(S.vals + kLiveCap);
  S.stash = S.gaps + kGapSmem;
  S.cnt = reinterpret_cast<int*>(S.stash + (stash_smem ? m : 0));
  S.off = S.cnt + NB;
  return S;
}

template <bool kGiven>
__global__ void __launch_bounds__(kEssThreads) ess_kernel(const EssParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Ctl ctl;
  __shared__ uint64_t s_w64[kWarps];
  __shared__ int s_w32[kWarps];
  const int NB = p.NB;
  const int log2NB = 31 - __clz(NB);
  const int m = p.m;
  const bool stash_smem = m <= kStashSmemMax;
  Smem S = carve(smem_raw, NB, m, stash_smem);
  double2* stash = stash_smem ? S.stash : p.gstash + (int64_t)blockIdx.x * m;
  double2* gg = p.ggaps + (int64_t)blockIdx.x * (m + 2);
  const double scale = __ddiv_rn((double)NB, kTwoPi);
  const int tid = threadIdx.x;

  for (int c = blockIdx.x; c < p.C; c += gridDim.x) {
    const uint32_t gchain = p.chain_offset + (uint32_t)c;
    __syncthreads();
    if (tid == 0) {
      ctl.n_act = 0;
      ctl.ngap = 0;
      ctl.G = 0.0;  // gamma_0 = 0: the first segment is [0, alpha_{i_1}]
      ctl.rlo = 0;
      ctl.rhi = kTopBits;
      ctl.mode = 0;
      ctl.viol = 0;
      ctl.slack = -DBL_MAX;
    }
    clear_buckets(S, NB);
    __syncthreads();

    // ---------------- A: arcs -> stash + level-1 bucket statistics ----------------
    const double* Prow = p.P_cur + (int64_t)c * p.ldp;
    const double* Qrow = p.Q + (int64_t)c * p.ldp;
    for (int i = tid; i < m; i += blockDim.x) {
      double al, be;
      bool act;
      if (kGiven) {
        al = p.g_alpha[(int64_t)c * m + i];
        be = p.g_beta[(int64_t)c * m + i];
        act = true;
      } else {
        act = arc_of(Prow[i], Qrow[i], p.b[i], al, be);
        if (p.d_alpha) {
          p.d_alpha[(int64_t)c * m + i] = act ? al : 0.0;
          p.d_beta[(int64_t)c * m + i] = act ? be : 0.0;
          p.d_active[(int64_t)c * m + i] = act ? 1 : 0;
        }
      }
      if (act) {
        int slot = atomicAdd(&ctl.n_act, 1);
        stash[slot] = make_double2(al, be);
        bucket_add(S, bucket_key(al, ctl, NB, scale), al, be);
      }
    }
    __syncthreads();

    // ---------------- B: I_act by Alg. 3 ----------------
    build_intervals(S, ctl, stash, NB, log2NB, scale, gg, s_w64, s_w32);

    // ---------------- C: canonical segments, L, theta ----------------
    if (tid == 0) {
      double u = kGiven ? (p.g_u ? p.g_u[c] : 0.0) : theta_uniform(p.seed, p.t, gchain);
      theta_from_gaps(S, ctl, gg, u, p.eps);
      if (p.d_nseg) p.d_nseg[c] = ctl.nseg;
      if (p.d_L) p.d_L[c] = ctl.L;
      if (p.d_theta) p.d_theta[c] = ctl.theta;
    }
    __syncthreads();
    if (p.d_seg_lo) {
      int ns = ctl.nseg;
      for (int k = tid; k < ns && k < p.seg_cap; k += blockDim.x) {
        double2 g = gap_load(S, gg, k);
        p.d_seg_lo[(int64_t)c * p.seg_cap + k] = g.x;
        p.d_seg_hi[(int64_t)c * p.seg_cap + k] = g.y;
      }
    }
    if (kGiven) continue;

    // ---------------- D: safeguard, P', x update, moments, next nu ----------------
    const double L = ctl.L;
    double st = 0.0, ct = 1.0;
    if (L > 0.0) sincos(ctl.theta, &st, &ct);
    double* Pn = p.P_next + (int64_t)c * p.ldp;
    int viol = 0;
    double smax = -DBL_MAX;
    if (L > 0.0) {
      for (int i = tid; i < m; i += blockDim.x) {
        double pn = Prow[i] * ct + Qrow[i] * st;
        double s = pn - p.b[i];
        viol |= s > 0.0;
        smax = fmax(smax, s);
        Pn[i] = pn;
      }
    }
    const int any_viol = __syncthreads_or(viol);
    const bool accept = (L > 0.0) && !any_viol;
    if (p.d_slack) {
      // block max of the slack (dump only)
      uint64_t key = dbits(smax) ^ ((dbits(smax) >> 63) ? ~0ull : 0x8000000000000000ull);
      uint64_t tot;
      block_excl_max(key, 0, s_w64, &tot);
      if (tid == 0) {
        uint64_t bits = (tot >> 63) ? (tot ^ 0x8000000000000000ull) : ~tot;
        p.d_slack[c] = L > 0.0 ? bitsd(bits) : 0.0;
      }
    }
    if (!accept) {
      for (int i = tid; i < m; i += blockDim.x) Pn[i] = Prow[i];  // stay at x_t
    }
    const int runs = (int)(p.d_pad / 8);
    for (int a = tid; a < runs; a += blockDim.x) {
      int64_t o = run_offset(c, a, p.d_pad);
      double2* xr = reinterpret_cast<double2*>(p.X + o);
      double2* nr = reinterpret_cast<double2*>(p.N + o);
      double2 xv[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) xv[h] = xr[h];
      if (accept) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double2 nv = nr[h];
          xv[h].x = xv[h].x * ct + nv.x * st;
          xv[h].y = xv[h].y * ct + nv.y * st;
          xr[h] = xv[h];
        }
      }
      if (p.record) {
        double2* s1 = reinterpret_cast<double2*>(p.S1 + o);
        double2* s2 = reinterpret_cast<double2*>(p.S2 + o);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double2 a1 = s1[h], a2 = s2[h];
          a1.x += xv[h].x;
          a1.y += xv[h].y;
          a2.x += xv[h].x * xv[h].x;
          a2.y += xv[h].y * xv[h].y;
          s1[h] = a1;
          s2[h] = a2;
        }
      }
      if (p.gen_next) {
        double nn[8];
        normal_run(p.seed, p.t + 1, gchain, a, p.d, nn);
#pragma unroll
        for (int h = 0; h < 4; ++h) nr[h] = make_double2(nn[2 * h], nn[2 * h + 1]);
      }
    }
    if (tid == 0) {
      if (!accept) p.rej[c] += 1;
      if (p.d_accept) p.d_accept[c] = accept ? 1 : 0;
    }
  }
}

}  // namespace

int ess_buckets(int m) {
  int nb = 64;
  while (nb < m / 4 && nb < 1024) nb <<= 1;
  return nb;
}

size_t ess_smem_bytes(int m, int NB) {
  size_t s = (size_t)NB * 4 * sizeof(uint64_t) + (size_t)kLiveCap * 16 + (size_t)kGapSmem * 16;
  if (m <= kStashSmemMax) s += (size_t)m * 16;
  s += (size_t)NB * 2 * sizeof(int);
  return s;
}

static int g_sms = 0;

int ess_grid(int C, int m, int NB) {
  if (g_sms == 0) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  size_t smem = ess_smem_bytes(m, NB);
  int per_sm = 0;
  cudaFuncSetAttribute(ess_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ess_kernel<false>, kEssThreads, smem);
  if (per_sm < 1) per_sm = 1;
  int g = g_sms * per_sm;
  return C < g ? C : g;
}

cudaError_t launch_ess_step(const EssParams& p, int grid, cudaStream_t st) {
  size_t smem = ess_smem_bytes(p.m, p.NB);
  cudaError_t e = cudaFuncSetAttribute(ess_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (grid < 1) return cudaSuccess;
  ess_kernel<false><<<grid, kEssThreads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ess_intervals(const EssParams& p, int grid, cudaStream_t st) {
  size_t smem = ess_smem_bytes(p.m, p.NB);
  cudaError_t e = cudaFuncSetAttribute(ess_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (grid < 1) return cudaSuccess;
  ess_kernel<true><<<grid, kEssThreads, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace tmvn
