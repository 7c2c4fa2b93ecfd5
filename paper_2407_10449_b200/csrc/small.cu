// small.cu -- the warp mode (options.warp_mode): a group of NW
// warps (NW = 1, 2, 4, 8; options.small_warps) per chain runs every iteration of Alg. 1
// for its chains in a single launch, with A resident in shared memory.  For
// small polytopes (m <= 512 and A small enough for shared memory: BASELINE configs 1
// and 2) the throughput path is bound by two launches per iteration and the latency
// mode by cluster barriers; here a group owns a chain for all n_iter iterations:
//   nu_t (Philox + Box-Muller, C12) into shared memory, u_t (with NW > 1 drawn by
//     warps 1..NW-1 while thread 0 computes theta of t - 1: nu double-buffered);
//   Q = A nu, one thread per row (A stored column-major: thread-contiguous, no bank
//     conflicts; nu broadcast), P = A x maintained incrementally (Eq. 1) and
//     recomputed every K (C13);
//   the arcs of eq:roots (C1-C5, the shared arc_of), compacted by ballot + a group
//     counter (any order);
//   Alg. 3 literally: a bitonic sort of (alpha, slot) by alpha -- one element per
//     thread in registers, shuffles below stride 32, shared memory across warps --,
//     the inclusive prefix max of beta (group scan), gaps [gamma_{k-1}, alpha_k] where
//     alpha_k > gamma_{k-1} (Prop. 1) and [gamma_n, 2 pi];
//   one thread: merge touching segments, trim (C7), L, theta = inverse CDF (C10),
//     sin / cos of theta;
//   P' = P cos + Q sin, the safeguard (C8) by a group OR, x update, moments.
// Named barriers per group (warp-synchronous when NW = 1), no cross-group state except
// A.  The dot products sum in index order (FMA, contraction fixed), so trajectories do
// not depend on NW and agree with the other paths and the oracle to rounding, not
// bitwise.
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace tmvn {
namespace {

__device__ __forceinline__ uint64_t sbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double sbitsd(uint64_t b) { return __longlong_as_double((long long)b); }

// canonical segments (merge touching), trim (C7), L and theta (C10); one lane
__device__ void small_theta(double2* gaps, int ngap, double u, double eps, double* theta, double* Lout) {
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

// A group of NW warps owning one chain (NW = 1: the warp mode proper; NW > 1 when the job
// has too few chains to fill the SMs one warp each): named barrier gid + 1 over its
// 32 NW threads, or warp-synchronous.
template <int NW>
struct SGrp {
  static constexpr int T = 32 * NW;
  int gid, tid, warp, lane;
  __device__ __forceinline__ void sync() const {
    if (NW == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(T) : "memory");
  }
  // group-wide OR of v (a barrier)
  __device__ __forceinline__ int sync_or(int v) const {
    if (NW == 1) return __any_sync(0xffffffffu, v);
    int r;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.s32 p, %1, 0;\n bar.red.or.pred q, %2, %3, p;\n"
        " selp.s32 %0, 1, 0, q;\n}\n"
        : "=r"(r)
        : "r"(v), "r"(gid + 1), "r"(T)
        : "memory");
    return r;
  }
};

// exclusive prefix (max of uint64 / sum of int) over the group's threads in thread order,
// the group total in *tot; scr: NW words, not rewritten before the group's next barrier
template <int NW>
__device__ __forceinline__ uint64_t sgrp_excl_max(const SGrp<NW>& g, uint64_t v, uint64_t* scr, uint64_t* tot) {
  uint64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t nb = __shfl_up_sync(0xffffffffu, inc, o);
    if (g.lane >= o) inc = inc > nb ? inc : nb;
  }
  uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (g.lane == 0) exc = 0;
  if (NW == 1) {
    *tot = __shfl_sync(0xffffffffu, inc, 31);
    return exc;
  }
  if (g.lane == 31) scr[g.warp] = inc;
  g.sync();
  uint64_t pre = 0, all = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint64_t sw = scr[w];
    if (w < g.warp) pre = pre > sw ? pre : sw;
    all = all > sw ? all : sw;
  }
  *tot = all;
  return pre > exc ? pre : exc;
}
template <int NW>
__device__ __forceinline__ int sgrp_excl_sum(const SGrp<NW>& g, int v, int* scr, int* tot) {
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int nb = __shfl_up_sync(0xffffffffu, inc, o);
    if (g.lane >= o) inc += nb;
  }
  if (NW == 1) {
    *tot = __shfl_sync(0xffffffffu, inc, 31);
    return inc - v;
  }
  if (g.lane == 31) scr[g.warp] = inc;
  g.sync();
  int pre = 0, all = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int sw = scr[w];
    if (w < g.warp) pre += sw;
    all += sw;
  }
  *tot = all;
  return pre + inc - v;
}

// v_out[i] = sum_j A[i][j] v[j] (in index order j = 0, 1, ...) for the RT rows
// i = tid + T r of this thread (A_T column-major with MS rows per column; rows >= m are
// zero in A_T).  Each row's sum is the same whichever thread computes it.
template <int RT, int T, int MS>
__device__ __forceinline__ void small_gemv(const double* __restrict__ AT, const double* v, int d, int tid,
                                           double (&out)[RT]) {
#pragma unroll
  for (int r = 0; r < RT; ++r) out[r] = 0.0;
  for (int j = 0; j < d; ++j) {
    const double vj = v[j];
    const double* col = AT + (size_t)j * MS + tid;
#pragma unroll
    for (int r = 0; r < RT; ++r) out[r] = fma(col[T * r], vj, out[r]);
  }
}

struct SmallWarp {
  double* x;     // d_pad
  double* nu;    // d_pad
  double* M1;    // d_pad (moments over this group's chains)
  double* M2;
  uint64_t* key; // n2: alpha bits (sort keys)
  double* val;   // n2: beta
  double2* gaps; // m + 2
  uint64_t* scr64;  // 8: group scan scratch
  int* scr32;       // 8
  double* ctl;      // [1] sin theta, [2] L, [3] cos theta, [4 + (t & 1)] u_t; n_act at ictl[0]
  int* ictl;
};

// Group control words after the per-warp state of small_warp_bytes
constexpr int kSmallCtlBytes = 8 * 8 + 8 * 4 + 6 * 8 + 16;

// threads per CTA: up to 1024 (64 registers) with at most 4 rows of A per thread, else
// up to 512 (small_max_warps)
template <int R, int NW>
__global__ void __launch_bounds__(R / NW >= 8 ? 512 : 1024, 1) small_kernel(const SmallParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = 32 * NW;
  constexpr int RT = R / NW;  // rows of A per thread
  constexpr int MS = 32 * R;
  SGrp<NW> g;
  g.gid = threadIdx.x / T;
  g.tid = threadIdx.x % T;
  g.warp = g.tid >> 5;
  g.lane = threadIdx.x & 31;
  const int ngr = blockDim.x / T;  // groups in the CTA
  const int m = p.m, d = p.d;
  double* AT = reinterpret_cast<double*>(smem);  // d x MS, column j = A[:, j] (zero rows >= m)
  // A' into shared memory, transposed (rows of the row-major input are strided reads)
  for (int e = threadIdx.x; e < d * MS; e += blockDim.x) {
    const int j = e / MS, i = e % MS;
    AT[e] = i < m ? p.A[(int64_t)i * d + j] : 0.0;
  }
  unsigned char* wbase = smem + (size_t)d * MS * 8 + (size_t)g.gid * p.warp_bytes;
  SmallWarp W;
  W.x = reinterpret_cast<double*>(wbase);
  W.nu = W.x + p.d_pad;
  W.M1 = W.nu + 2 * p.d_pad;  // nu double-buffered: nu_t at W.nu + (t & 1) d_pad
  W.M2 = W.M1 + p.d_pad;
  W.key = reinterpret_cast<uint64_t*>(W.M2 + p.d_pad);
  W.val = reinterpret_cast<double*>(W.key + p.n2);
  W.gaps = reinterpret_cast<double2*>(W.val + p.n2);
  W.scr64 = reinterpret_cast<uint64_t*>(wbase + p.warp_bytes - kSmallCtlBytes);
  W.scr32 = reinterpret_cast<int*>(W.scr64 + 8);
  W.ctl = reinterpret_cast<double*>(W.scr32 + 8);
  W.ictl = reinterpret_cast<int*>(W.ctl + 6);
  for (int j = g.tid; j < p.d_pad; j += T) {
    W.M1[j] = 0.0;
    W.M2[j] = 0.0;
  }
  __syncthreads();
  double bv[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) bv[r] = g.tid + T * r < m ? p.b[g.tid + T * r] : HUGE_VAL;
  const int64_t gw = (int64_t)blockIdx.x * ngr + g.gid;  // this group's global index (moment row)
  const int64_t ngroups = (int64_t)gridDim.x * ngr;
  const int kpairs = (int)(p.d_pad / 2);
  bool recorded_any = false;

  for (int64_t c = gw; c < p.C; c += ngroups) {
    const uint32_t gchain = p.chain_offset + (uint32_t)c;
    const int64_t xrow = tiled_row(c, p.d_pad);
    for (int j = g.tid; j < p.d_pad; j += T) W.x[j] = j < d ? p.X[xrow + tiled_col(j)] : 0.0;
    g.sync();
    double P[RT], Q[RT];
    small_gemv<RT, T, MS>(AT, W.x, d, g.tid, P);
    int n_iter = p.n_iter;
    if (p.startflag) {  // strict start a_i . x0 < b_i (C18): lowest (chain, constraint) to the host
      bool bad = false;
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int i = g.tid + T * r;
        if (i < m && !(P[r] - bv[r] < 0.0)) {
          atomicMin(p.startflag, (unsigned long long)c * (unsigned long long)m + (unsigned long long)i);
          bad = true;
        }
      }
      if (g.sync_or(bad)) n_iter = 0;
    }
    int64_t rej = 0;
    for (int it = 0; it < n_iter; ++it) {
      const uint32_t t = p.t0 + (uint32_t)it;
      // nu_t and u_t (C12); with NW > 1 drawn during theta of t - 1 (below) after the first
      double* nu = W.nu + (t & 1) * p.d_pad;
      if (NW == 1 || it == 0) {
        for (int pk = g.tid; pk < kpairs; pk += T) {
          const double2 v = normal_pair_at(p.seed, t, gchain, 2 * pk, d);
          nu[2 * pk] = v.x;
          nu[2 * pk + 1] = v.y;
        }
        if (g.tid == 0) W.ctl[4 + (t & 1)] = theta_uniform(p.seed, t, gchain);
      }
      if (g.tid == 0) W.ictl[0] = 0;
      g.sync();
      small_gemv<RT, T, MS>(AT, nu, d, g.tid, Q);
      // arcs of the active constraints (eq:roots, C1-C5), compacted (any order: sorted below)
      int n_w = 0;  // NW = 1: the running count in a register
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int i = g.tid + T * r;
        double al = 0.0, be = 0.0;
        const bool act = i < m && arc_of(P[r], Q[r], bv[r], al, be);
        const unsigned mask = __ballot_sync(0xffffffffu, act);
        if (mask) {
          int base = n_w;
          if (NW > 1) {
            if (g.lane == 0) base = atomicAdd(&W.ictl[0], __popc(mask));
            base = __shfl_sync(0xffffffffu, base, 0);
          }
          if (act) {
            const int slot = base + __popc(mask & ((1u << g.lane) - 1u));
            W.key[slot] = sbits(al);
            W.val[slot] = be;
          }
          n_w += __popc(mask);
        }
      }
      g.sync();
      const int n_act = NW == 1 ? n_w : W.ictl[0];
      // Alg. 3: sort by alpha (bitonic, padded with +inf keys), prefix max of beta, gaps
      int n2 = 1;
      while (n2 < n_act) n2 <<= 1;
      if (n2 < 32) n2 = 32;
      if (n2 <= T) {
        // one element per thread in registers, T of them (pads beyond n_act): strides below
        // 32 exchange by shuffles, strides >= 32 through W.key / W.val between barriers;
        // the pair's two threads take the same swap decision (ties may land in either
        // order -- the gaps do not depend on it, see the header)
        // (the network spans S = the power of two >= n_act only: the elements beyond are
        // +inf pads that stay in place, so the first S come out ascending)
        int S = 2;
        while (S < n_act) S <<= 1;
        n2 = T;
        // (key, slot) pairs: the slot (32 bits, one shuffle) indexes beta in W.val, which
        // the sort leaves in place; the cross-warp slot exchange goes through W.gaps
        // (free until the gaps are emitted; (m + 2) 16 >= 4 T whenever T > 32)
        int* xs = reinterpret_cast<int*>(W.gaps);
        uint64_t kk = g.tid < n_act ? W.key[g.tid] : 0x7FF0000000000000ull;
        int ii = g.tid < n_act ? g.tid : -1;
#pragma unroll 1
        for (int k = 2; k <= S; k <<= 1) {
#pragma unroll 1
          for (int jj = k >> 1; jj > 0; jj >>= 1) {
            uint64_t ok;
            int oi;
            if (jj >= 32) {
              g.sync();
              W.key[g.tid] = kk;
              xs[g.tid] = ii;
              g.sync();
              ok = W.key[g.tid ^ jj];
              oi = xs[g.tid ^ jj];
            } else {
              ok = __shfl_xor_sync(0xffffffffu, kk, jj);
              oi = __shfl_xor_sync(0xffffffffu, ii, jj);
            }
            const bool lower = (g.tid & jj) == 0, up = (g.tid & k) == 0;
            const uint64_t klo = lower ? kk : ok, khi = lower ? ok : kk;
            if ((klo > khi) == up) {
              kk = ok;
              ii = oi;
            }
          }
        }
        const double vv = ii >= 0 ? W.val[ii] : 0.0;
        g.sync();  // every beta read (and the last cross-warp exchange) before the write-back
        W.key[g.tid] = kk;  // each thread reads back only its own element below (E = 1)
        W.val[g.tid] = vv;
      } else {
        for (int e = n_act + g.tid; e < n2; e += T) {
          W.key[e] = 0x7FF0000000000000ull;
          W.val[e] = 0.0;
        }
        g.sync();
        // compare-exchange stages: a stride below 32 keeps both elements in the owning warp
        // (element e belongs to thread e mod T); a barrier around every stride >= 32
        for (int k = 2; k <= n2; k <<= 1) {
          for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int e = g.tid; e < n2; e += T) {
              const int l = e ^ jj;
              if (l > e) {
                const bool up = (e & k) == 0;
                const uint64_t ke = W.key[e], kl = W.key[l];
                if ((ke > kl) == up) {
                  W.key[e] = kl;
                  W.key[l] = ke;
                  const double tv = W.val[e];
                  W.val[e] = W.val[l];
                  W.val[l] = tv;
                }
              }
            }
            const int jn = jj > 1 ? jj >> 1 : k;  // the next stage's stride
            if (NW > 1 && (jj >= 32 || jn >= 32)) g.sync();
            else __syncwarp();
          }
        }
        if (NW > 1) g.sync();
      }
      // thread owns the sorted elements [tid E, tid E + E): gamma before each element is
      // max(0, prefix max of beta of the earlier ones) (gamma_0 = 0: [0, alpha_1] first)
      const int E = n2 >= T ? n2 / T : 1;
      const int e0 = g.tid * E;
      const int e1 = min(e0 + E, n_act);
      uint64_t lmax = 0;
      for (int e = e0; e < e1; ++e) lmax = lmax > sbits(W.val[e]) ? lmax : sbits(W.val[e]);
      uint64_t Gtot;
      const uint64_t run = sgrp_excl_max<NW>(g, lmax, W.scr64, &Gtot);
      int mine = 0;
      {
        uint64_t gm = run;
        for (int e = e0; e < e1; ++e) {
          if (W.key[e] > gm) ++mine;  // alpha_k > gamma_{k-1}: a gap (Prop. 1)
          const uint64_t vb = sbits(W.val[e]);
          gm = gm > vb ? gm : vb;
        }
      }
      int ngap0;
      const int before = sgrp_excl_sum<NW>(g, mine, W.scr32, &ngap0);
      {
        uint64_t gm = run;
        int pos = before;
        for (int e = e0; e < e1; ++e) {
          if (W.key[e] > gm) W.gaps[pos++] = make_double2(sbitsd(gm), sbitsd(W.key[e]));
          const uint64_t vb = sbits(W.val[e]);
          gm = gm > vb ? gm : vb;
        }
      }
      g.sync();
      if (g.tid == 0) {
        int ng = ngap0;
        const double G = sbitsd(Gtot);
        if (G < kTwoPi) W.gaps[ng++] = make_double2(G, kTwoPi);  // [gamma_n, 2 pi]
        double theta = 0.0, L = 0.0;
        small_theta(W.gaps, ng, W.ctl[4 + (t & 1)], p.eps, &theta, &L);
        double st0 = 0.0, ct0 = 1.0;
        if (L > 0.0) sincos(theta, &st0, &ct0);  // once per chain, not per thread
        W.ctl[1] = st0;
        W.ctl[2] = L;
        W.ctl[3] = ct0;
      } else if (NW > 1 && g.warp > 0 && it + 1 < n_iter) {
        // nu_{t+1}, u_{t+1} while one thread computes theta (the other buffer: nu_t is read
        // by the update below)
        double* nn = W.nu + ((t + 1) & 1) * p.d_pad;
        for (int pk = g.tid - 32; pk < kpairs; pk += T - 32) {
          const double2 v = normal_pair_at(p.seed, t + 1, gchain, 2 * pk, d);
          nn[2 * pk] = v.x;
          nn[2 * pk + 1] = v.y;
        }
        if (g.tid == 32) W.ctl[4 + ((t + 1) & 1)] = theta_uniform(p.seed, t + 1, gchain);
      }
      g.sync();
      const double st = W.ctl[1], L = W.ctl[2], ct = W.ctl[3];
      // P' = P cos + Q sin, the safeguard (C8), the update
      bool viol = false;
      double Pn[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        Pn[r] = fma(Q[r], st, __dmul_rn(P[r], ct));  // contraction fixed: the same in every instantiation
        viol |= (Pn[r] - bv[r]) > 0.0;  // b is +inf beyond m
      }
      const bool accept = (L > 0.0) && !g.sync_or(viol);
      if (accept) {
#pragma unroll
        for (int r = 0; r < RT; ++r) P[r] = Pn[r];
        for (int j = g.tid; j < d; j += T) W.x[j] = fma(nu[j], st, __dmul_rn(W.x[j], ct));
      } else {
        ++rej;
      }
      const int64_t tt = (int64_t)t;
      if (p.record && tt >= p.burn_in && ((tt - p.burn_in) % (p.thin < 1 ? 1 : p.thin)) == 0) {
        recorded_any = true;
        for (int j = g.tid; j < d; j += T) {
          const double xv = W.x[j];
          W.M1[j] += xv;
          W.M2[j] = fma(xv, xv, W.M2[j]);
        }
      }
      g.sync();
      if ((tt + 1) % p.K == 0) small_gemv<RT, T, MS>(AT, W.x, d, g.tid, P);  // refresh P = A x (C13)
    }
    for (int j = g.tid; j < d; j += T) p.X[xrow + tiled_col(j)] = W.x[j];
    if (g.tid == 0) p.rej[c] = rej;
    g.sync();
  }
  if (recorded_any) {  // this group's moment row (rows < C; zeroed by the host)
    const int64_t mrow = tiled_row(gw, p.d_pad);
    for (int j = g.tid; j < d; j += T) {
      p.S1[mrow + tiled_col(j)] = W.M1[j];
      p.S2[mrow + tiled_col(j)] = W.M2[j];
    }
  }
}

}  // namespace

size_t small_warp_bytes(int m, int64_t d_pad) {
  int n2 = 32;
  while (n2 < m) n2 <<= 1;
  return (size_t)(5 * d_pad * 8 + (size_t)n2 * 16 + (size_t)(m + 2) * 16 + kSmallCtlBytes + 15) / 16 * 16;
}

int small_rows(int m) {
  int R = 1;
  while (32 * R < m) R <<= 1;
  return R;
}

int small_max_warps(int m, int nw) { return small_rows(m) / nw >= 8 ? 16 : 32; }

cudaError_t launch_small(const SmallParams& p0, int groups_per_cta, int nw, int grid, cudaStream_t st) {
  SmallParams p = p0;
  const int R = small_rows(p.m);
  if (nw < 1 || nw > R || (nw & (nw - 1)) != 0 || groups_per_cta * nw > small_max_warps(p.m, nw))
    return cudaErrorInvalidValue;
  p.warp_bytes = (int)small_warp_bytes(p.m, p.d_pad);
  int n2 = 32;
  while (n2 < p.m) n2 <<= 1;
  p.n2 = n2;
  const size_t smem = (size_t)p.d * 32 * R * 8 + (size_t)groups_per_cta * p.warp_bytes;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 32 * nw * groups_per_cta, smem, st>>>(p);
    return cudaGetLastError();
  };
#define TMVN_SMALL_CASE(RR)                                  \
  case RR:                                                   \
    switch (nw) {                                            \
      case 1: return go(small_kernel<RR, 1>);                \
      case 2: if constexpr (RR >= 2) return go(small_kernel<RR, (RR >= 2 ? 2 : 1)>); break; \
      case 4: if constexpr (RR >= 4) return go(small_kernel<RR, (RR >= 4 ? 4 : 1)>); break; \
      case 8: if constexpr (RR >= 8) return go(small_kernel<RR, (RR >= 8 ? 8 : 1)>); break; \
    }                                                        \
    return cudaErrorInvalidValue;
  switch (R) {
    TMVN_SMALL_CASE(1)
    TMVN_SMALL_CASE(2)
    TMVN_SMALL_CASE(4)
    TMVN_SMALL_CASE(8)
    TMVN_SMALL_CASE(16)
    default: return cudaErrorInvalidValue;
  }
#undef TMVN_SMALL_CASE
}

}  // namespace tmvn
