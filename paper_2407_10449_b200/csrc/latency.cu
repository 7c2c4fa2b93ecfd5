// latency.cu -- the latency mode (options.latency = 1): one thread-block cluster per
// chain runs every iteration of Alg. 1 in a single launch.
//
// The throughput path (GEMM over all chains, then one fused per-chain kernel per
// iteration) is launch- and latency-bound when there are fewer chains than SMs --
// the paper's own timing regime, 1 or 10 chains (S4.2).  Here the m
// constraints of a chain are split over the CS CTAs of a cluster (CS = 1..16, as many
// as the SMs allow), each CTA keeps x and nu (all d) and its slice of P = A x and
// Q = A nu in shared memory, and per iteration:
//   (a) nu_t (Philox + Box-Muller, C12; every CTA draws the whole vector),
//   (b) Q_i = a_i . nu for its rows (one warp per row, A' streamed from L2),
//   (c) the arcs of its rows (eq:roots, C1-C5) + level-1 bucket statistics
//       (count, max alpha high word, exact max beta),
//   -- cluster barrier: every CTA merges the CS bucket tables through distributed
//      shared memory, gamma entering each bucket = exclusive prefix max (Prop. 1),
//   (d) the arcs of live buckets are appended to CTA 0's buffer (DSMEM atomics),
//   -- barrier: CTA 0 builds I_act (gamma before an arc = max(gamma entering its
//      bucket, beta of the arcs of its bucket with a smaller alpha), Alg. 3 without
//      the sort), trims (C7) and samples theta (C10),
//   -- barrier: P' = P cos + Q sin for its rows, the safeguard (C8),
//   -- barrier: accept iff no CTA saw a violation; x <- x cos + nu sin (every CTA,
//      identically), moments of its coordinate slice, refresh P every K.
// Four cluster barriers per iteration, no kernel launches, no host round trips.
// Results follow the same RNG counters and readings as the throughput path; the
// dot products sum in a different order, so trajectories agree with it (and with
// the oracle) to rounding, not bitwise.
#include <cfloat>
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace tmvn {
namespace {

#ifndef TMVN_LAT_THREADS
#define TMVN_LAT_THREADS 256
#endif
constexpr int kLT = TMVN_LAT_THREADS;  // threads per CTA
constexpr int kLNB = 128;     // level-1 buckets over [0, 2 pi]
#ifndef TMVN_LAT_PIPE
#define TMVN_LAT_PIPE 1
#endif
// live arcs CTA 0 can hold per iteration: p.cap, sized on the host from the shared
// memory left (up to m); more in some iteration -> the call reruns on the default path
constexpr int kLNF = 1024;    // level-2 slots CTA 0 splits the live level-1 buckets into
constexpr int kLSmall = 64;   // up to this many live arcs CTA 0 skips level 2
constexpr int kLMinCap = 64;  // live-arc buffers hold at least this many (p.cap may be lower: test hook)

__device__ __forceinline__ uint64_t lbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double lbitsd(uint64_t b) { return __longlong_as_double((long long)b); }

struct LatShared {
  double* x;       // d_pad
  double* nu;      // d_pad
  double* nu2;     // d_pad: nu of the next iteration, drawn by CTAs 1.. while CTA 0 samples theta
  double* P0;      // mr each: current / proposal, swapped on accept
  double* P1;
  double* Q;       // mr
  double2* st;     // mr: arcs of this CTA's active constraints
  uint64_t* Gx;    // kLNB: max beta (exact after the low-word pass)
  uint64_t* mA;    // kLNB: max alpha (high word)
  int* cnt;        // kLNB
  uint64_t* gin;   // kLNB: merged gamma entering each bucket
  int* live;       // kLNB: merged live flag
  uint64_t* lkey;  // cap + 2 (CTA 0): live arcs' alpha bits
  double* lval;    // cap + 2: their beta
  double2* gaps;   // cap + 2: the gaps, over lkey / lval once those are consumed
  uint64_t* fb;    // kLNF (CTA 0): level-2 max beta, then gamma entering the slot
  uint64_t* fa;    // kLNF: level-2 max alpha
  int* fc;         // kLNF: level-2 count, then live flag
  int* fid;        // cap: level-2 slot of each live arc
  int* cl;         // cap: live arcs in live level-2 slots
  int* lrk;        // kLNB: rank of a live level-1 bucket among the live ones
  int* lb;         // kLNB: live level-1 bucket of each rank
  uint64_t* scr;   // 8 + kLT / 32 words of scan scratch
  uint64_t* cand;  // 2 cap
  double* M1;      // nk x kLT: this CTA's moment sums over the call (flushed at the end)
  double* M2;
  int* ints;       // [0] n_act, [1] live count, [2] viol, [3] ncand, [4] overflow
  double* dbl;     // [0] theta, [1] L, [2] u
};

__host__ __device__ __forceinline__ size_t lat_align(size_t v) { return (v + 15) / 16 * 16; }

// shared-memory layout (host: base = nullptr, only the size is used)
__host__ __device__ inline int lat_nk(int64_t d_pad, int cs) { return (int)((d_pad + (int64_t)cs * kLT - 1) / ((int64_t)cs * kLT)); }
__host__ __device__ inline size_t lat_carve(unsigned char* base, int64_t d_pad, int mr, int nk, int cap,
                                            LatShared& S) {
  size_t o = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = base + o;
    o += lat_align(bytes);
    return q;
  };
  S.x = reinterpret_cast<double*>(take(d_pad * 8));
  S.nu = reinterpret_cast<double*>(take(d_pad * 8));
  S.nu2 = reinterpret_cast<double*>(take(d_pad * 8));
  S.P0 = reinterpret_cast<double*>(take((size_t)mr * 8));
  S.P1 = reinterpret_cast<double*>(take((size_t)mr * 8));
  S.Q = reinterpret_cast<double*>(take((size_t)mr * 8));
  S.st = reinterpret_cast<double2*>(take((size_t)mr * 16));
  S.Gx = reinterpret_cast<uint64_t*>(take(kLNB * 8));
  S.mA = reinterpret_cast<uint64_t*>(take(kLNB * 8));
  S.cnt = reinterpret_cast<int*>(take(kLNB * 4));
  S.gin = reinterpret_cast<uint64_t*>(take(kLNB * 8));
  S.live = reinterpret_cast<int*>(take(kLNB * 4));
  S.lrk = reinterpret_cast<int*>(take(kLNB * 4));
  S.lb = reinterpret_cast<int*>(take(kLNB * 4));
  S.scr = reinterpret_cast<uint64_t*>(take((8 + kLT / 32) * 8));
  S.M1 = reinterpret_cast<double*>(take((size_t)nk * kLT * 8));
  S.M2 = reinterpret_cast<double*>(take((size_t)nk * kLT * 8));
  S.ints = reinterpret_cast<int*>(take(8 * 4));
  S.dbl = reinterpret_cast<double*>(take(4 * 8));
  S.lkey = reinterpret_cast<uint64_t*>(take((size_t)(cap + 2) * 8));
  S.lval = reinterpret_cast<double*>(take((size_t)(cap + 2) * 8));
  S.gaps = reinterpret_cast<double2*>(S.lkey);  // contiguous 16 (cap + 2) bytes
  S.cand = reinterpret_cast<uint64_t*>(take((size_t)2 * cap * 8));
  S.fb = reinterpret_cast<uint64_t*>(take(kLNF * 8));
  S.fa = reinterpret_cast<uint64_t*>(take(kLNF * 8));
  S.fc = reinterpret_cast<int*>(take(kLNF * 4));
  S.fid = reinterpret_cast<int*>(take((size_t)cap * 4));
  S.cl = reinterpret_cast<int*>(take((size_t)cap * 4));
  return o;
}

// Level-1 bucket of an angle in [0, 2 pi] from its FP64 bit pattern (monotone in the
// angle, which is all Alg. 3's bucketing needs): 8 buckets per octave over
// [2^-12, 8) -- buckets 1 .. 120 -- and everything below 2^-12 in bucket 0.  At
// S4.2 states the arcs start just past theta = 0 (alpha ~ slack / |q|), where a
// linear grid put every one of them into its first bucket; octaves spread them,
// and the buckets after the first arcs' ends are dead (max alpha <= gamma in).
constexpr int kLExpLo = 1023 - 12;
#ifndef TMVN_LAT_OCTAVE
#define TMVN_LAT_OCTAVE 1
#endif
__device__ __forceinline__ int lat_bucket(double a, double scale) {
#if !TMVN_LAT_OCTAVE
  const int kl = (int)__dmul_rn(a, scale);
  return kl < kLNB - 1 ? kl : kLNB - 1;
#endif
  const uint64_t bits = (uint64_t)__double_as_longlong(a);
  const int e = (int)(bits >> 52);  // a >= 0
  if (e < kLExpLo) return 0;
  const int k = 1 + ((e - kLExpLo) << 3) + (int)((bits >> 49) & 7);
  return k < kLNB - 1 ? k : kLNB - 1;
}
// position in [0, SUB) of an angle inside its level-1 bucket (level 2): the next 32
// mantissa bits, monotone within a bucket of one octave slice; bucket 0 spans many
// octaves and is one slot
__device__ __forceinline__ int lat_sub(double a, int k, int SUB, double scale) {
#if !TMVN_LAT_OCTAVE
  const double u = __dmul_rn(a, scale);
  return min(SUB - 1, (int)__dmul_rn(__dsub_rn(u, (double)k), (double)SUB));
#endif
  if (k == 0) return 0;
  const uint64_t bits = (uint64_t)__double_as_longlong(a);
  return (int)((((bits >> 17) & 0xFFFFFFFFull) * (uint64_t)SUB) >> 32);
}

// 16-byte vectors of the arithmetic type: FP64 (default) or FP32 (options.precision = 1)
template <typename T> struct LVec;
template <> struct LVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct LVec<float> { using V = float4; static constexpr int N = 4; };
__device__ __forceinline__ double vdot(const double2 a, const double2 w, double s) {
  return fma(a.y, w.y, fma(a.x, w.x, s));
}
__device__ __forceinline__ float vdot(const float4 a, const float4 w, float s) {
  return fmaf(a.w, w.w, fmaf(a.z, w.z, fmaf(a.y, w.y, fmaf(a.x, w.x, s))));
}

// dot products of up to four rows of A (row stride d_pad, zero-padded, 16-byte aligned)
// with v (shared, d_pad), one warp, fixed order: 16-byte loads, four partial sums per
// row, so that sixteen loads per lane are in flight (A is streamed from L2 every
// iteration: memory-level parallelism bounds this step)
template <typename T>
__device__ __forceinline__ void lat_dot4(const T* __restrict__ A, int nrow, int64_t d_pad, const T* v, int lane,
                                         T o[4]) {
  using V = typename LVec<T>::V;
  const V* __restrict__ R[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) R[q] = reinterpret_cast<const V*>(A + (q < nrow ? q : 0) * d_pad);
  const V* Vv = reinterpret_cast<const V*>(v);
  const int np = (int)(d_pad / LVec<T>::N);
  T s[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int u = 0; u < 4; ++u) s[q][u] = T(0);
#if TMVN_LAT_PIPE
  // blocks of 128 vectors in two halves, software-pipelined: the loads of the next
  // half are in flight while the current half is multiplied (same accumulation order
  // as the plain loop below); loads past the row are predicated off (zero)
  V a[4][2], bq[4][2];
  auto ld = [&](V (&dst)[4][2], int j0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < 2; ++u) dst[q][u] = j0 + 32 * u < np ? __ldg(R[q] + j0 + 32 * u) : V{};
  };
  auto mul = [&](const V (&src)[4][2], int j0, int u0) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const V w = j0 + 32 * u < np ? Vv[j0 + 32 * u] : V{};
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q][u0 + u] = vdot(src[q][u], w, s[q][u0 + u]);
    }
  };
  ld(a, lane);
  for (int j = lane; j < np; j += 128) {
    ld(bq, j + 64);
    mul(a, j, 0);
    if (j + 128 < np) ld(a, j + 128);
    mul(bq, j + 64, 2);
  }
#else
  // blocks of 128 vectors; the last block's loads past the row are predicated off
  // (zero), so every block is one round trip with sixteen loads per lane in flight
  for (int j = lane; j < np; j += 128) {
    V a[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[q][u] = j + 32 * u < np ? __ldg(R[q] + j + 32 * u) : V{};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const V w = j + 32 * u < np ? Vv[j + 32 * u] : V{};
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q][u] = vdot(a[q][u], w, s[q][u]);
    }
  }
#endif
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    T t = (s[q][0] + s[q][1]) + (s[q][2] + s[q][3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    o[q] = t;
  }
}
// rows [0, nr) of this CTA's slice (global rows i0 + r) . v -> out[r]; warps take row
// quads, in reverse order on alternate calls: when A exceeds L2, the rows streamed last
// (still in L2) are read first, instead of LRU evicting each just before its reuse.
// A row's sum has the same order either way.
template <typename T>
__device__ __forceinline__ void lat_rows(const T* __restrict__ A, int i0, int nr, int64_t d_pad, const T* v,
                                         T* out, int warp, int lane, bool reverse = false) {
  const int nq = (nr + 3) / 4;
  for (int k = warp; k < nq; k += kLT / 32) {
    const int r = 4 * (reverse ? nq - 1 - k : k);
    const int nrow = min(4, nr - r);
    T o[4];
    lat_dot4<T>(A + (int64_t)(i0 + r) * d_pad, nrow, d_pad, v, lane, o);
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < nrow) out[r + q] = o[q];
    }
  }
}

// the arc of one constraint in the arithmetic type, returned in FP64 (exact widening)
// for the interval machinery; FP32: the same construction (eq:roots, C1-C5) with
// single-precision atan2 / sqrt, 2 pi rounded to float, endpoints clamped to FP64 2 pi
__device__ __forceinline__ bool lat_arc(double p, double q, double b, double& al, double& be) {
  return arc_of(p, q, b, al, be);
}
__device__ __forceinline__ bool lat_arc(float p, float q, float b, double& al, double& be) {
  const float s2 = fmaf(p, p, fmaf(q, q, -b * b));
  if (!(b < 0.0f || s2 > 0.0f)) return false;
  const float s = sqrtf(fmaxf(s2, 0.0f));
  const float tau = atan2f(q, p), delta = atan2f(s, b);
  constexpr float kTwoPiF = 6.28318530717958647692f;
  float lo = tau - delta, hi = tau + delta;
  if (hi <= 0.0f) {
    lo += kTwoPiF;
    hi += kTwoPiF;
  } else if (lo >= 0.0f) {
  } else if (-lo <= hi) {
    lo = 0.0f;  // straddle (rounding only): snap the shorter side (C1)
  } else {
    lo += kTwoPiF;
    hi = kTwoPiF;
  }
  al = fmin((double)lo, kTwoPi);
  be = fmin((double)hi, kTwoPi);
  return true;
}

// canonical segments (merge touching), trim (C7), L and theta = inverse CDF at u (C10);
// one thread; the gaps are ascending
__device__ void lat_theta(double2* gaps, int ngap, double u, double eps, double* theta, double* Lout) {
  int w = 0;
  for (int k = 0; k < ngap; ++k) {
    const double2 g = gaps[k];
    if (w > 0 && gaps[w - 1].y == g.x) {
      gaps[w - 1].y = g.y;
      continue;
    }
    gaps[w++] = g;
  }
  bool trim = eps > 0.0;
  int last_kept = -1;
  if (trim) {
    for (int k = 0; k < w; ++k) {
      const double lo = gaps[k].x == 0.0 ? 0.0 : __dadd_rn(gaps[k].x, eps);
      const double hi = gaps[k].y == kTwoPi ? kTwoPi : __dsub_rn(gaps[k].y, eps);
      if (hi > lo) last_kept = k;
    }
    if (last_kept < 0) trim = false;
  }
  if (!trim) last_kept = w - 1;
  double total = 0.0;
  for (int k = 0; k < w; ++k) {
    double lo = gaps[k].x, hi = gaps[k].y;
    if (trim) {
      lo = gaps[k].x == 0.0 ? 0.0 : __dadd_rn(gaps[k].x, eps);
      hi = gaps[k].y == kTwoPi ? kTwoPi : __dsub_rn(gaps[k].y, eps);
      if (!(hi > lo)) continue;
    }
    total = __dadd_rn(total, __dsub_rn(hi, lo));
  }
  *Lout = total;
  *theta = 0.0;
  if (!(total > 0.0)) return;
  const double target = __dmul_rn(u, total);
  double before = 0.0;
  for (int k = 0; k < w; ++k) {
    double lo = gaps[k].x, hi = gaps[k].y;
    if (trim) {
      lo = gaps[k].x == 0.0 ? 0.0 : __dadd_rn(gaps[k].x, eps);
      hi = gaps[k].y == kTwoPi ? kTwoPi : __dsub_rn(gaps[k].y, eps);
      if (!(hi > lo)) continue;
    }
    const double after = __dadd_rn(before, __dsub_rn(hi, lo));
    if (after > target || k == last_kept) {
      *theta = __dadd_rn(lo, __dsub_rn(target, before));
      return;
    }
    before = after;
  }
}

#ifdef TMVN_PHASE_TIMING
__device__ unsigned long long g_lat_cycles[16];
#define LPH(i)                                                                          \
  do {                                                                                  \
    if (blockIdx.x == 0 && tid == 0) {                                                  \
      long long n_ = clock64();                                                         \
      lph[i] += n_ - lt_prev;                                                           \
      lt_prev = n_;                                                                     \
    }                                                                                   \
  } while (0)
#else
#define LPH(i) \
  do {         \
  } while (0)
#endif

// kGrid: the chain's CTAs are p.gsz CTAs of a cooperative grid instead of a thread-block
// cluster (more SMs per chain than a cluster's 16 when there are few chains and a large
// A): the exchanges go through global scratch instead of distributed shared memory and
// the barriers are grid barriers (one more, to merge the bucket tables bucket-parallel)
template <typename T, bool kGrid>
__global__ void __launch_bounds__(kLT, 1) latency_kernel(const LatParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  cg::grid_group grid = cg::this_grid();
  const int CS = kGrid ? p.gsz : (int)cluster.num_blocks();
  const int rank = kGrid ? (int)(blockIdx.x % p.gsz) : (int)cluster.block_rank();
  auto csync = [&]() {
    if constexpr (kGrid) grid.sync();
    else cluster.sync();
  };
  const int chain = (int)(blockIdx.x / CS);
  if (chain >= p.C) return;  // whole clusters only: uniform across the cluster
  const uint32_t gchain = p.chain_offset + (uint32_t)chain;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = p.m, d = p.d;
  const int mr = (m + CS - 1) / CS;
  const int i0 = rank * mr, i1 = min(m, i0 + mr), nr = i1 > i0 ? i1 - i0 : 0;
  extern __shared__ __align__(16) unsigned char lsm[];
  LatShared S;
  const int nk = lat_nk(p.d_pad, CS);
  lat_carve(lsm, p.d_pad, mr, nk, p.cap > kLMinCap ? p.cap : kLMinCap, S);  // buffers >= kLMinCap
  // CTA 0's buffers and flags, seen from every CTA of the cluster (grid: global scratch)
  int* r_ints0 = kGrid ? nullptr : cluster.map_shared_rank(S.ints, 0);
  uint64_t* r_lkey0 = kGrid ? nullptr : cluster.map_shared_rank(S.lkey, 0);
  double* r_lval0 = kGrid ? nullptr : cluster.map_shared_rank(S.lval, 0);
  double* r_dbl0 = kGrid ? p.gth + 2 * chain : cluster.map_shared_rank(S.dbl, 0);
  const double scale = __ddiv_rn((double)kLNB, kTwoPi);
  // the arithmetic type's views (x, nu, P, Q live in FP64-sized slots either way)
  const T* A = static_cast<const T*>(sizeof(T) == 8 ? (const void*)p.A : (const void*)p.A32);
  const T* bv = static_cast<const T*>(sizeof(T) == 8 ? (const void*)p.b : (const void*)p.b32);
  T* Sx = reinterpret_cast<T*>(S.x);
  T* Snu = reinterpret_cast<T*>(S.nu);    // nu_t
  T* SnuN = reinterpret_cast<T*>(S.nu2);  // nu_{t+1} (CTAs 1..CS-1 draw it during CTA 0's theta)

  T* SQ = reinterpret_cast<T*>(S.Q);

  // x_{t0} (all d) and P = A x for this CTA's rows
  for (int j = tid; j < p.d_pad; j += kLT) Sx[j] = j < d ? (T)p.X[tiled_offset(chain, j, p.d_pad)] : T(0);
  if (tid < 8) S.ints[tid] = 0;
  for (int k = 0; k < nk; ++k) {
    S.M1[k * kLT + tid] = 0.0;
    S.M2[k * kLT + tid] = 0.0;
  }
  __syncthreads();
  T* Pc = reinterpret_cast<T*>(S.P0);  // P = A x for this CTA's rows
  T* Pn = reinterpret_cast<T*>(S.P1);  // the proposal P'
  bool rev = false;  // alternate the row order of successive products (L2 reuse)
  auto gemv = [&](const T* v, T* out) {
    lat_rows<T>(A, i0, nr, p.d_pad, v, out, warp, lane, rev);
    rev = !rev;
  };
  gemv(Sx, Pc);
  __syncthreads();
  // strict start a_i . x0 < b_i (C18), checked here on the first P (FP64 mode; the
  // host checks FP32 starts in FP64 itself): lowest (chain, constraint) to the host,
  // and the cluster runs no iteration
  if (p.startflag) {
    int bad = 0;
    for (int r = tid; r < nr; r += kLT) {
      if (!((double)Pc[r] - (double)bv[i0 + r] < 0.0)) {  // NaN also fails
        atomicMin(p.startflag, (unsigned long long)chain * (unsigned long long)m + (unsigned long long)(i0 + r));
        bad = 1;
      }
    }
    bad = __syncthreads_or(bad);
    if (tid == 0) S.ints[6] = bad;
    if (kGrid && tid == 0 && bad) atomicOr(p.gstart + chain, 1);
  }
  int64_t rej = 0;
  csync();
  int start_bad = 0;
  if (p.startflag) {
    if constexpr (kGrid) start_bad = *(volatile int*)(p.gstart + chain);
    else start_bad = __syncthreads_or(tid < CS ? *cluster.map_shared_rank(S.ints + 6, tid) : 0);
  }
  const int n_iter = start_bad ? 0 : p.n_iter;
#ifdef TMVN_PHASE_TIMING
  long long lph[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long lt_prev = clock64();
#endif

  // (a) nu, u and cleared bucket tables for iteration tt, (b) Q = A nu for this CTA's
  // rows.  nu is drawn here, unless the CTAs 1.. drew it during the previous
  // iteration's theta phase, in which case CTA 0 copies CTA 1's (distributed shared
  // memory, or global scratch in the grid variant).  From the second iteration on this
  // runs between the two halves of the safeguard barrier: it does not depend on the
  // verdict, only x, P and the arcs do.
  auto prep = [&](uint32_t tt, T* nu_dst, bool drawn) {
    if (!drawn) {
      for (int pk = tid; pk < (int)(p.d_pad / 2); pk += kLT) {
        const double2 v = normal_pair_at(p.seed, tt, gchain, 2 * pk, d);
        nu_dst[2 * pk] = (T)v.x;
        nu_dst[2 * pk + 1] = (T)v.y;
      }
    } else if (rank == 0) {
      if constexpr (kGrid) {
        const T* src = reinterpret_cast<const T*>(p.gnu) + (int64_t)chain * p.d_pad;
        for (int j = tid; j < p.d_pad; j += kLT) nu_dst[j] = __ldcg(src + j);
      } else {
        const T* src = cluster.map_shared_rank(nu_dst, 1);
        for (int j = tid; j < p.d_pad; j += kLT) nu_dst[j] = src[j];
      }
    }
    if (rank == 0 && tid == 0) S.dbl[2] = theta_uniform(p.seed, tt, gchain);
    for (int j = tid; j < kLNB; j += kLT) {
      S.Gx[j] = 0;
      S.mA[j] = 0;
      S.cnt[j] = 0;
    }
    if (tid == 0) S.ints[0] = 0;
    __syncthreads();
    gemv(nu_dst, SQ);
    __syncthreads();
  };
  if (n_iter > 0) prep(p.t0, Snu, false);

  for (int it = 0; it < n_iter; ++it) {
    const uint32_t t = p.t0 + (uint32_t)it;
    LPH(0);
    LPH(1);
    // (c) arcs of the active rows + bucket statistics (high words, then low words)
    for (int r = tid; r < nr; r += kLT) {
      double al, be;
      if (lat_arc(Pc[r], SQ[r], __ldg(bv + i0 + r), al, be)) {
        const int slot = atomicAdd(&S.ints[0], 1);
        S.st[slot] = make_double2(al, be);
        const int k = lat_bucket(al, scale);
        atomicMax(reinterpret_cast<uint32_t*>(&S.Gx[k]) + 1, (uint32_t)(lbits(be) >> 32));
        atomicMax(reinterpret_cast<uint32_t*>(&S.mA[k]) + 1, (uint32_t)(lbits(al) >> 32));
        atomicAdd(&S.cnt[k], 1);
      }
    }
    __syncthreads();
    const int n_act = S.ints[0];
    for (int s = tid; s < n_act; s += kLT) {
      const double2 ab = S.st[s];
      const int k = lat_bucket(ab.x, scale);
      if ((uint32_t)(lbits(ab.y) >> 32) == (uint32_t)(S.Gx[k] >> 32))
        atomicMax(reinterpret_cast<uint32_t*>(&S.Gx[k]), (uint32_t)lbits(ab.y));
    }
    LPH(2);
    const int par = it & 1;
    if constexpr (kGrid) {  // this CTA's table to global scratch (after the low-word pass)
      __syncthreads();
      for (int k = tid; k < kLNB; k += kLT) {
        const int64_t o = ((int64_t)chain * CS + rank) * kLNB + k;
        p.gtab_g[o] = S.Gx[k];
        p.gtab_a[o] = S.mA[k];
        p.gtab_c[o] = S.cnt[k];
      }
    }
    csync();  // #1: every CTA's bucket table is complete
    if constexpr (kGrid) {
      // bucket-parallel merge: CTA r reduces buckets r, r + CS, ... over the CS tables
      uint64_t* red = reinterpret_cast<uint64_t*>(S.cand);  // scratch (16 words per warp)
      for (int k = rank; k < kLNB; k += CS) {
        uint64_t g = 0, a = 0;
        int c = 0;
        for (int r = tid; r < CS; r += kLT) {
          const int64_t o = ((int64_t)chain * CS + r) * kLNB + k;
          const uint64_t gv = __ldcg(p.gtab_g + o), av = __ldcg(p.gtab_a + o);  // other SMs' writes: L2
          g = g > gv ? g : gv;
          a = a > av ? a : av;
          c += __ldcg(p.gtab_c + o);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t g2 = __shfl_xor_sync(0xffffffffu, g, o), a2 = __shfl_xor_sync(0xffffffffu, a, o);
          g = g > g2 ? g : g2;
          a = a > a2 ? a : a2;
          c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
          red[3 * warp] = g;
          red[3 * warp + 1] = a;
          red[3 * warp + 2] = (uint64_t)c;
        }
        __syncthreads();
        if (tid == 0) {
          for (int w = 1; w < kLT / 32; ++w) {
            g = g > red[3 * w] ? g : red[3 * w];
            a = a > red[3 * w + 1] ? a : red[3 * w + 1];
            c += (int)red[3 * w + 2];
          }
          p.gmrg_g[(int64_t)chain * kLNB + k] = g;
          p.gmrg_a[(int64_t)chain * kLNB + k] = a;
          p.gmrg_c[(int64_t)chain * kLNB + k] = c;
        }
        __syncthreads();
      }
      if (rank == 0 && tid == 0) {  // the slots of iteration it + 1 (last read in it - 1)
        p.gcount[2 * chain + (par ^ 1)] = 0;
        p.gviol[2 * chain + (par ^ 1)] = 0;
      }
      csync();  // #1b: the merged table is complete
    }
    LPH(3);
    // merge the CS tables (every CTA, redundantly): thread j < kLNB owns bucket j and
    // reads it from every CTA (independent DSMEM loads, in flight together); gamma
    // entering each bucket = exclusive prefix max (warp scans + the 4 warp totals)
    {
      uint64_t g = 0, a = 0;
      int c = 0;
      if (tid < kLNB) {
        if constexpr (kGrid) {
          g = __ldcg(p.gmrg_g + (int64_t)chain * kLNB + tid);
          a = __ldcg(p.gmrg_a + (int64_t)chain * kLNB + tid);
          c = __ldcg(p.gmrg_c + (int64_t)chain * kLNB + tid);
        } else {
#pragma unroll 4
          for (int r = 0; r < CS; ++r) {
            const uint64_t gv = cluster.map_shared_rank(S.Gx, r)[tid];
            const uint64_t av = cluster.map_shared_rank(S.mA, r)[tid];
            const int cv = cluster.map_shared_rank(S.cnt, r)[tid];
            g = g > gv ? g : gv;
            a = a > av ? a : av;
            c += cv;
          }
        }
      }
      uint64_t inc = g;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = inc > n ? inc : n;
      }
      uint64_t* wtot = reinterpret_cast<uint64_t*>(S.cand);  // scratch: CTA 0 uses cand only after barrier #2
      if (lane == 31 && warp < kLNB / 32) wtot[warp] = inc;
      __syncthreads();
      if (tid < kLNB) {
        uint64_t pre = 0;  // gamma_0 = 0
        for (int w = 0; w < warp; ++w) pre = pre > wtot[w] ? pre : wtot[w];
        uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) exc = 0;
        const uint64_t gin = pre > exc ? pre : exc;
        S.gin[tid] = gin;
        // level 1: only the high word of max alpha is exact -> conservative test
        S.live[tid] = c > 0 && (a | 0xFFFFFFFFull) > gin;
        if (tid == kLNB - 1) {
          const uint64_t tot = gin > g ? gin : g;
          S.dbl[3] = lbitsd(tot);
        }
      }
    }
    __syncthreads();
    // (d) this CTA's arcs in live buckets -> CTA 0's buffer
    // an arc of a live bucket whose beta <= the gamma entering the bucket lies inside the
    // earlier arc that set that gamma (it starts before the bucket): it changes neither
    // the union nor any later gamma, so it is dropped here
    for (int s = tid; s < n_act; s += kLT) {
      const double2 ab = S.st[s];
      const int k = lat_bucket(ab.x, scale);
      if (S.live[k] && lbits(ab.y) > S.gin[k]) {
        if constexpr (kGrid) {
          const int pos = atomicAdd(p.gcount + 2 * chain + par, 1);
          if (pos < p.cap) p.glive[(int64_t)chain * p.cap + pos] = ab;
        } else {
          const int pos = atomicAdd(r_ints0 + 1, 1);
          if (pos < p.cap) {
            r_lkey0[pos] = lbits(ab.x);
            r_lval0[pos] = ab.y;
          }
        }
      }
    }
    LPH(4);
    csync();  // #2: the live arcs are in CTA 0 (grid: in global scratch)
    if constexpr (kGrid) {
      if (rank == 0) {
        const int total = *(volatile int*)(p.gcount + 2 * chain + par);
        if (tid == 0) S.ints[1] = total;
        for (int e = tid; e < total && e < p.cap; e += kLT) {
          const double2 ab = __ldcg(p.glive + (int64_t)chain * p.cap + e);
          S.lkey[e] = lbits(ab.x);
          S.lval[e] = ab.y;
        }
        __syncthreads();
      }
    }
    LPH(5);
    if (rank != 0 && it + 1 < n_iter) {  // nu_{t+1} while CTA 0 builds I_act and theta
      for (int pk = tid; pk < (int)(p.d_pad / 2); pk += kLT) {
        const double2 v = normal_pair_at(p.seed, t + 1, gchain, 2 * pk, d);
        SnuN[2 * pk] = (T)v.x;
        SnuN[2 * pk + 1] = (T)v.y;
        if (kGrid && rank == 1) {
          T* dst = reinterpret_cast<T*>(p.gnu) + (int64_t)chain * p.d_pad;
          dst[2 * pk] = (T)v.x;
          dst[2 * pk + 1] = (T)v.y;
        }
      }
    }
#ifdef TMVN_PHASE_TIMING
    if (blockIdx.x == 0 && tid == 0) lph[11] += S.ints[1];
#endif
    if (rank == 0) {
      const int total = S.ints[1];
      const uint64_t Gtot = lbits(S.dbl[3]);
      if (total > p.cap) {
        if (tid == 0) {
          S.ints[4] = 1;  // overflow: this iteration stays (L = 0); reported to the host
          S.dbl[0] = 0.0;
          S.dbl[1] = 0.0;
        }
      } else {
        // Level 2 (Alg. 3's bucketing applied once more, inside CTA 0): the live level-1
        // buckets, in order, are split into SUB equal slots each; slot index is monotone in
        // alpha, so gamma entering a slot = max(gamma entering its level-1 bucket, max beta
        // of the earlier slots), and only slots whose max alpha exceeds it can hold a gap
        // start. Arcs of such slots get gamma from the slot's earlier arcs (alpha order,
        // equal alphas by index: the same gap either way); the gaps are ranked by alpha.
        // (S4.2's arcs all start just past theta = 0: one live level-1 bucket holds them.)
        if (total <= kLSmall) {
          // few live arcs (small m, or the usual case far from the boundary): gamma before
          // each from the arcs of its own level-1 bucket directly, no level 2
          if (tid == 0) S.ints[3] = 0;
          __syncthreads();
          for (int e = tid; e < total; e += kLT) {
            const uint64_t key = S.lkey[e];
            const int k = lat_bucket(lbitsd(key), scale);
            uint64_t gm = S.gin[k];
            for (int f = 0; f < total; ++f) {
              const uint64_t kf = S.lkey[f];
              if ((kf < key || (kf == key && f < e)) && lat_bucket(lbitsd(kf), scale) == k) {
                const uint64_t vf = lbits(S.lval[f]);
                gm = gm > vf ? gm : vf;
              }
            }
            if (key > gm) {
              const int c3 = atomicAdd(&S.ints[3], 1);
              S.cand[2 * c3] = key;
              S.cand[2 * c3 + 1] = gm;
            }
          }
        } else {
          if (tid < kLNB) {
            const int lv = S.live[tid] ? 1 : 0;
            int ci = lv;
  #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int n = __shfl_up_sync(0xffffffffu, ci, o);
              if (lane >= o) ci += n;
            }
            if (lane == 31) S.scr[warp] = (uint64_t)ci;
          }
          for (int f = tid; f < kLNF; f += kLT) {
            S.fb[f] = 0;
            S.fa[f] = 0;
            S.fc[f] = 0;
          }
          if (tid == 0) {
            S.ints[3] = 0;
            S.ints[5] = 0;
          }
          __syncthreads();
          if (tid < kLNB) {
            int rk = 0;
            for (int w = 0; w < warp; ++w) rk += (int)S.scr[w];
            const int lv = S.live[tid] ? 1 : 0;
            int ci = lv;
  #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int n = __shfl_up_sync(0xffffffffu, ci, o);
              if (lane >= o) ci += n;
            }
            rk += ci - lv;
            S.lrk[tid] = rk;
            if (lv) S.lb[rk] = tid;
          }
          int nlb = 0;
          for (int w = 0; w < kLNB / 32; ++w) nlb += (int)S.scr[w];
          const int SUB = kLNF / (nlb > 0 ? nlb : 1);
          __syncthreads();
          LPH(12);
          for (int e = tid; e < total; e += kLT) {
            const uint64_t key = S.lkey[e];
            const int k = lat_bucket(lbitsd(key), scale);
            const int sub = lat_sub(lbitsd(key), k, SUB, scale);
            const int f = S.lrk[k] * SUB + sub;
            S.fid[e] = f;
            atomicMax(reinterpret_cast<unsigned long long*>(&S.fb[f]), (unsigned long long)lbits(S.lval[e]));
            atomicMax(reinterpret_cast<unsigned long long*>(&S.fa[f]), (unsigned long long)key);
            atomicAdd(&S.fc[f], 1);
          }
          __syncthreads();
          LPH(13);
          {  // exclusive prefix max of the slots' max beta (four slots per thread)
            constexpr int FP = kLNF / kLT;
            uint64_t mb[FP];
            uint64_t run = 0;
  #pragma unroll
            for (int q = 0; q < FP; ++q) {
              mb[q] = S.fb[tid * FP + q];
              run = run > mb[q] ? run : mb[q];
            }
            uint64_t inc = run;
  #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint64_t n = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= o) inc = inc > n ? inc : n;
            }
            if (lane == 31) S.scr[8 + warp] = inc;
            __syncthreads();
            uint64_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane == 0) ex = 0;
            for (int w = 0; w < warp; ++w) ex = ex > S.scr[8 + w] ? ex : S.scr[8 + w];
  #pragma unroll
            for (int q = 0; q < FP; ++q) {
              const int f = tid * FP + q;
              const int rk = f / SUB;
              if (rk < nlb) {
                const uint64_t gk = S.gin[S.lb[rk]];
                const uint64_t g = ex > gk ? ex : gk;
                const bool live = S.fc[f] > 0 && S.fa[f] > g;
                S.fb[f] = g;
                S.fc[f] = live ? 1 : 0;
              }
              ex = ex > mb[q] ? ex : mb[q];
            }
          }
          __syncthreads();
          LPH(15);
          for (int e = tid; e < total; e += kLT)
            if (S.fc[S.fid[e]]) S.cl[atomicAdd(&S.ints[5], 1)] = e;
          __syncthreads();
          const int nl2 = S.ints[5];
          for (int c = tid; c < nl2; c += kLT) {
            const int e = S.cl[c], f = S.fid[e];
            const uint64_t key = S.lkey[e];
            uint64_t gm = S.fb[f];
            for (int c2 = 0; c2 < nl2; ++c2) {
              const int e2 = S.cl[c2];
              if (S.fid[e2] != f) continue;
              const uint64_t k2 = S.lkey[e2];
              if (k2 < key || (k2 == key && e2 < e)) {
                const uint64_t v2 = lbits(S.lval[e2]);
                gm = gm > v2 ? gm : v2;
              }
            }
            if (key > gm) {
              const int c3 = atomicAdd(&S.ints[3], 1);
              S.cand[2 * c3] = key;
              S.cand[2 * c3 + 1] = gm;
            }
          }
        }
        __syncthreads();
        {
          const int nc = S.ints[3];
          for (int c = tid; c < nc; c += kLT) {
            const uint64_t a = S.cand[2 * c];
            int rnk = 0;
            for (int c2 = 0; c2 < nc; ++c2) rnk += S.cand[2 * c2] < a ? 1 : 0;
            S.gaps[rnk] = make_double2(lbitsd(S.cand[2 * c + 1]), lbitsd(a));
          }
        }
        __syncthreads();
        const int nc = S.ints[3];
        LPH(14);
        if (tid == 0) {
          int ng = nc;
          const double G = lbitsd(Gtot);
          if (G < kTwoPi) S.gaps[ng++] = make_double2(G, kTwoPi);  // [gamma_m, 2 pi]
          lat_theta(S.gaps, ng, S.dbl[2], p.eps, &S.dbl[0], &S.dbl[1]);
        }
      }
      if (tid == 0) S.ints[1] = 0;  // the live buffer is free for the next iteration
      if (kGrid && tid == 0) {
        p.gth[2 * chain] = S.dbl[0];
        p.gth[2 * chain + 1] = S.dbl[1];
      }
    }
    LPH(6);
    csync();  // #3: theta and L in CTA 0
    LPH(7);
    const double theta = kGrid ? *(volatile double*)(r_dbl0) : r_dbl0[0];
    const double L = kGrid ? *(volatile double*)(r_dbl0 + 1) : r_dbl0[1];
    T sn = T(0), cs = T(1);
    if (L > 0.0) sincos((T)theta, &sn, &cs);
    int viol = 0;
    if (L > 0.0) {
      for (int r = tid; r < nr; r += kLT) {
        const T pn = Pc[r] * cs + SQ[r] * sn;
        Pn[r] = pn;
        viol |= (pn - __ldg(bv + i0 + r)) > T(0) ? 1 : 0;
      }
    }
    viol = __syncthreads_or(viol);
    if (tid == 0) S.ints[2] = viol;
    if (kGrid && tid == 0 && viol) atomicOr(p.gviol + 2 * chain + par, 1);
    LPH(8);
    // #4: every CTA's safeguard verdict -- split: the next iteration's nu and Q in between
    if constexpr (kGrid) grid.sync();
    else asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if (it + 1 < n_iter) prep(t + 1, SnuN, CS > 1);
    if constexpr (!kGrid) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    LPH(9);
    int any;
    if constexpr (kGrid) any = *(volatile int*)(p.gviol + 2 * chain + par);
    else any = __syncthreads_or(tid < CS ? *cluster.map_shared_rank(S.ints + 2, tid) : 0);
    const bool accept = L > 0.0 && !any;
    if (accept) {
      T* tmp = Pc;
      Pc = Pn;
      Pn = tmp;
      for (int j = tid; j < p.d_pad; j += kLT) Sx[j] = Sx[j] * cs + Snu[j] * sn;
    } else {
      ++rej;
    }
    __syncthreads();
    const int64_t tt = (int64_t)t;
    if (p.record && tt >= p.burn_in && ((tt - p.burn_in) % (p.thin < 1 ? 1 : p.thin)) == 0) {
      for (int k = 0, j = rank * kLT + tid; j < d; ++k, j += CS * kLT) {  // this CTA's coordinates
        const double xv = (double)Sx[j];
        S.M1[k * kLT + tid] += xv;
        S.M2[k * kLT + tid] += xv * xv;
      }
    }
    if ((int64_t)(t + 1) % p.K == 0) {  // refresh P = A x (C13)
      gemv(Sx, Pc);
    }
    {  // nu_{t+1} is in SnuN
      T* tmp = Snu;
      Snu = SnuN;
      SnuN = tmp;
    }
    __syncthreads();
    LPH(10);
  }
#ifdef TMVN_PHASE_TIMING
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 16; ++i) atomicAdd(&g_lat_cycles[i], (unsigned long long)lph[i]);
#endif
  if (p.record) {
    for (int k = 0, j = rank * kLT + tid; j < d; ++k, j += CS * kLT) {
      const int64_t o = tiled_offset(chain, j, p.d_pad);
      p.S1[o] += S.M1[k * kLT + tid];
      p.S2[o] += S.M2[k * kLT + tid];
    }
  }
  if (rank == 0) {
    for (int j = tid; j < d; j += kLT) p.X[tiled_offset(chain, j, p.d_pad)] = (double)Sx[j];
    if (tid == 0) {
      p.rej[chain] += rej;
      if (S.ints[4]) atomicExch(p.err, 1);
    }
  }
  if constexpr (!kGrid) cluster.sync();  // no CTA leaves while another may still read its shared memory
}

}  // namespace

#ifdef TMVN_PHASE_TIMING
void lat_cycles(unsigned long long* out, bool reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_lat_cycles, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_lat_cycles, z, sizeof(z));
  }
}
#endif

size_t latency_smem_bytes(int64_t d_pad, int m, int cs, int cap) {
  LatShared S;
  return lat_carve(nullptr, d_pad, (m + cs - 1) / cs, lat_nk(d_pad, cs), cap > kLMinCap ? cap : kLMinCap, S);
}

// live-arc capacity: m if it fits, else as many as fit (0: the mode does not fit)
int latency_cap(int64_t d_pad, int m, int cs, size_t smem_max) {
  constexpr int kMinCap = kLMinCap;
  if (latency_smem_bytes(d_pad, m, cs, kMinCap) > smem_max) return 0;
  int lo = kMinCap, hi = m > kMinCap ? m : kMinCap;
  while (lo < hi) {
    const int mid = lo + (hi - lo + 1) / 2;
    if (latency_smem_bytes(d_pad, m, cs, mid) <= smem_max) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// clusters of cs CTAs (smem bytes each) that can be resident at once
template <typename T>
int latency_max_clusters_t(int cs, size_t smem) {
  if (cudaFuncSetAttribute(latency_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return 0;
  if (cs > 8 &&
      cudaFuncSetAttribute(latency_kernel<T, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cs);
  cfg.blockDim = dim3(kLT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, latency_kernel<T, false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// cluster size and live-arc capacity: the largest power of two cs <= 16 such that the
// shared memory fits, all C clusters are resident at once (clusters live inside one
// GPC: 16 chains x 8 CTAs do not all fit on 148 SMs), and each CTA keeps at least
// 32 K elements of A (smaller slices only add barrier and merge latency); if no cs
// keeps every cluster resident, the largest that fits (the clusters run in waves)
int latency_cluster_size(int C, int64_t m, int64_t d_pad, size_t smem_max, bool fp32, int* cap_out) {
  int cs_work = 1;
  while (cs_work < 16 && (int64_t)(2 * cs_work) * 32768 <= m * d_pad) cs_work <<= 1;
  int fallback = 0, fallback_cap = 0;
  for (int cs = 16; cs >= 1; cs >>= 1) {
    const int cap = latency_cap(d_pad, (int)m, cs, smem_max);
    if (cap == 0) continue;
    if (!fallback) {
      fallback = cs;
      fallback_cap = cap;
    }
    if (cs > cs_work) continue;
    const size_t smem = latency_smem_bytes(d_pad, (int)m, cs, cap);
    const int n = fp32 ? latency_max_clusters_t<float>(cs, smem) : latency_max_clusters_t<double>(cs, smem);
    if (n >= C) {
      *cap_out = cap;
      return cs;
    }
  }
  *cap_out = fallback_cap;
  return fallback;  // 0: does not fit
}

template <typename T>
cudaError_t launch_latency_t(const LatParams& p, int cs, cudaStream_t st) {
  const size_t smem = latency_smem_bytes(p.d_pad, p.m, cs, p.cap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.C * cs));
  cfg.blockDim = dim3(kLT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.gsz > 0) {  // cooperative grid of C x gsz CTAs (all resident: one per SM)
    cudaError_t e =
        cudaFuncSetAttribute(latency_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    return cudaLaunchKernelEx(&cfg, latency_kernel<T, true>, p);
  }
  cudaError_t e = cudaFuncSetAttribute(latency_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(latency_kernel<T, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  return cudaLaunchKernelEx(&cfg, latency_kernel<T, false>, p);
}

cudaError_t launch_latency(const LatParams& p, int cs, cudaStream_t st) {
  return p.fp32 ? launch_latency_t<float>(p, cs, st) : launch_latency_t<double>(p, cs, st);
}

}  // namespace tmvn
