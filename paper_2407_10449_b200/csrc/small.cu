// small.cu -- the warp mode (options.warp_mode): one warp per chain runs every
// iteration of Alg. 1 for its chains in a single launch, with A resident in
// shared memory.  For small polytopes (m <= 512 and A small enough for shared
// memory: BASELINE configs 1 and 2, m * d <= ~20K) the throughput path is bound by
// two launches per iteration and the latency mode by cluster barriers; here a warp
// owns a chain for all n_iter iterations:
//   nu_t (Philox + Box-Muller, C12) into shared memory, u_t;
//   Q = A nu, one lane per row (A stored column-major: lane-contiguous, no bank
//     conflicts; nu broadcast), P = A x maintained incrementally (Eq. 1) and
//     recomputed every K (C13);
//   the arcs of eq:roots (C1-C5, the shared arc_of), compacted by ballot;
//   Alg. 3 literally: a warp bitonic sort of the arcs by alpha, the inclusive
//     prefix max of beta (warp scan), gaps [gamma_{k-1}, alpha_k] where
//     alpha_k > gamma_{k-1} (Prop. 1) and [gamma_n, 2 pi];
//   one lane: merge touching segments, trim (C7), L, theta = inverse CDF (C10);
//   P' = P cos + Q sin, the safeguard (C8) by ballot, x update, moments.
// No block barriers (warp-synchronous), no cross-warp state except A.  The dot products
// sum in index order (with FMA), so trajectories agree with the other paths and the
// oracle to rounding, not bitwise.
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

// v_out[i] = sum_j A[i][j] v[j] for the R rows i = lane + 32 r of this lane (A_T column-
// major with ms = 32 R rows per column; rows >= m are zero in A_T)
template <int R>
__device__ __forceinline__ void small_gemv(const double* __restrict__ AT, const double* v, int d, int lane,
                                           double (&out)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = 0.0;
  for (int j = 0; j < d; ++j) {
    const double vj = v[j];
    const double* col = AT + (size_t)j * (32 * R) + lane;
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = fma(col[32 * r], vj, out[r]);
  }
}

struct SmallWarp {
  double* x;     // d_pad
  double* nu;    // d_pad
  double* M1;    // d_pad (moments over this warp's chains)
  double* M2;
  uint64_t* key; // n2: alpha bits (sort keys)
  double* val;   // n2: beta
  double2* gaps; // m + 2
};

template <int R>
__global__ void __launch_bounds__(512, 1) small_kernel(const SmallParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int m = p.m, d = p.d;
  constexpr int MS = 32 * R;
  double* AT = reinterpret_cast<double*>(smem);  // d x MS, column j = A[:, j] (zero rows >= m)
  // A' into shared memory, transposed (rows of the row-major input are strided reads)
  for (int e = threadIdx.x; e < d * MS; e += blockDim.x) {
    const int j = e / MS, i = e % MS;
    AT[e] = i < m ? p.A[(int64_t)i * d + j] : 0.0;
  }
  unsigned char* wbase = smem + (size_t)d * MS * 8 + (size_t)wib * p.warp_bytes;
  SmallWarp W;
  W.x = reinterpret_cast<double*>(wbase);
  W.nu = W.x + p.d_pad;
  W.M1 = W.nu + p.d_pad;
  W.M2 = W.M1 + p.d_pad;
  W.key = reinterpret_cast<uint64_t*>(W.M2 + p.d_pad);
  W.val = reinterpret_cast<double*>(W.key + p.n2);
  W.gaps = reinterpret_cast<double2*>(W.val + p.n2);
  for (int j = lane; j < p.d_pad; j += 32) {
    W.M1[j] = 0.0;
    W.M2[j] = 0.0;
  }
  __syncthreads();
  double bv[R];
#pragma unroll
  for (int r = 0; r < R; ++r) bv[r] = lane + 32 * r < m ? p.b[lane + 32 * r] : HUGE_VAL;
  const int64_t gw = (int64_t)blockIdx.x * nw + wib;  // this warp's global index (moment row)
  const int64_t nwarps = (int64_t)gridDim.x * nw;
  const int kpairs = (int)(p.d_pad / 2);
  bool recorded_any = false;

  for (int64_t c = gw; c < p.C; c += nwarps) {
    const uint32_t gchain = p.chain_offset + (uint32_t)c;
    const int64_t xrow = tiled_row(c, p.d_pad);
    for (int j = lane; j < p.d_pad; j += 32) W.x[j] = j < d ? p.X[xrow + tiled_col(j)] : 0.0;
    __syncwarp();
    double P[R], Q[R];
    small_gemv<R>(AT, W.x, d, lane, P);
    int n_iter = p.n_iter;
    if (p.startflag) {  // strict start a_i . x0 < b_i (C18): lowest (chain, constraint) to the host
      bool bad = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        if (i < m && !(P[r] - bv[r] < 0.0)) {
          atomicMin(p.startflag, (unsigned long long)c * (unsigned long long)m + (unsigned long long)i);
          bad = true;
        }
      }
      if (__any_sync(0xffffffffu, bad)) n_iter = 0;
    }
    int64_t rej = 0;
    for (int it = 0; it < n_iter; ++it) {
      const uint32_t t = p.t0 + (uint32_t)it;
      // nu_t and u_t (C12)
      for (int pk = lane; pk < kpairs; pk += 32) {
        const double2 v = normal_pair_at(p.seed, t, gchain, 2 * pk, d);
        W.nu[2 * pk] = v.x;
        W.nu[2 * pk + 1] = v.y;
      }
      const double u = __shfl_sync(0xffffffffu, lane == 0 ? theta_uniform(p.seed, t, gchain) : 0.0, 0);
      __syncwarp();
      small_gemv<R>(AT, W.nu, d, lane, Q);
      // arcs of the active constraints (eq:roots, C1-C5), compacted by ballot
      int n_act = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        double al = 0.0, be = 0.0;
        const bool act = i < m && arc_of(P[r], Q[r], bv[r], al, be);
        const unsigned mask = __ballot_sync(0xffffffffu, act);
        if (act) {
          const int slot = n_act + __popc(mask & ((1u << lane) - 1u));
          W.key[slot] = sbits(al);
          W.val[slot] = be;
        }
        n_act += __popc(mask);
      }
      // Alg. 3: sort by alpha (bitonic, padded with +inf keys), prefix max of beta, gaps
      int n2 = 1;
      while (n2 < n_act) n2 <<= 1;
      if (n2 < 32) n2 = 32;
      for (int e = n_act + lane; e < n2; e += 32) {
        W.key[e] = 0x7FF0000000000000ull;
        W.val[e] = 0.0;
      }
      __syncwarp();
      for (int k = 2; k <= n2; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          for (int e = lane; e < n2; e += 32) {
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
          __syncwarp();
        }
      }
      // lane owns the sorted elements [lane E, lane E + E): gamma before each element is
      // max(0, prefix max of beta of the earlier ones) (gamma_0 = 0: [0, alpha_1] first)
      const int E = n2 / 32;
      const int e0 = lane * E;
      uint64_t lmax = 0;
      for (int e = e0; e < e0 + E && e < n_act; ++e) lmax = lmax > sbits(W.val[e]) ? lmax : sbits(W.val[e]);
      uint64_t incl = lmax;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t nb = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = incl > nb ? incl : nb;
      }
      uint64_t run = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) run = 0;  // gamma_0 = 0 (bits of +0.0)
      const uint64_t Gtot = __shfl_sync(0xffffffffu, incl, 31);
      int mine = 0;
      {
        uint64_t g = run;
        for (int e = e0; e < e0 + E && e < n_act; ++e) {
          if (W.key[e] > g) ++mine;  // alpha_k > gamma_{k-1}: a gap (Prop. 1)
          const uint64_t vb = sbits(W.val[e]);
          g = g > vb ? g : vb;
        }
      }
      int before = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int nb = __shfl_up_sync(0xffffffffu, before, o);
        if (lane >= o) before += nb;
      }
      const int ngap0 = __shfl_sync(0xffffffffu, before, 31);
      before -= mine;
      {
        uint64_t g = run;
        int pos = before;
        for (int e = e0; e < e0 + E && e < n_act; ++e) {
          if (W.key[e] > g) W.gaps[pos++] = make_double2(sbitsd(g), sbitsd(W.key[e]));
          const uint64_t vb = sbits(W.val[e]);
          g = g > vb ? g : vb;
        }
      }
      __syncwarp();
      double theta = 0.0, L = 0.0;
      if (lane == 0) {
        int ng = ngap0;
        const double G = sbitsd(Gtot);
        if (G < kTwoPi) W.gaps[ng++] = make_double2(G, kTwoPi);  // [gamma_n, 2 pi]
        small_theta(W.gaps, ng, u, p.eps, &theta, &L);
      }
      theta = __shfl_sync(0xffffffffu, theta, 0);
      L = __shfl_sync(0xffffffffu, L, 0);
      // P' = P cos + Q sin, the safeguard (C8), the update
      double st = 0.0, ct = 1.0;
      if (L > 0.0) sincos(theta, &st, &ct);
      bool viol = false;
      double Pn[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Pn[r] = P[r] * ct + Q[r] * st;
        viol |= (Pn[r] - bv[r]) > 0.0;  // b is +inf beyond m
      }
      const bool accept = (L > 0.0) && !__any_sync(0xffffffffu, viol);
      if (accept) {
#pragma unroll
        for (int r = 0; r < R; ++r) P[r] = Pn[r];
        for (int j = lane; j < d; j += 32) W.x[j] = W.x[j] * ct + W.nu[j] * st;
      } else {
        ++rej;
      }
      const int64_t tt = (int64_t)t;
      if (p.record && tt >= p.burn_in && ((tt - p.burn_in) % (p.thin < 1 ? 1 : p.thin)) == 0) {
        recorded_any = true;
        for (int j = lane; j < d; j += 32) {
          const double xv = W.x[j];
          W.M1[j] += xv;
          W.M2[j] += xv * xv;
        }
      }
      __syncwarp();
      if ((tt + 1) % p.K == 0) small_gemv<R>(AT, W.x, d, lane, P);  // refresh P = A x (C13)
    }
    for (int j = lane; j < d; j += 32) p.X[xrow + tiled_col(j)] = W.x[j];
    if (lane == 0) p.rej[c] = rej;
    __syncwarp();
  }
  if (recorded_any) {  // this warp's moment row (rows < C; zeroed by the host)
    const int64_t mrow = tiled_row(gw, p.d_pad);
    for (int j = lane; j < d; j += 32) {
      p.S1[mrow + tiled_col(j)] = W.M1[j];
      p.S2[mrow + tiled_col(j)] = W.M2[j];
    }
  }
}

}  // namespace

size_t small_warp_bytes(int m, int64_t d_pad) {
  int n2 = 32;
  while (n2 < m) n2 <<= 1;
  return (size_t)(4 * d_pad * 8 + (size_t)n2 * 16 + (size_t)(m + 2) * 16 + 15) / 16 * 16;
}

int small_rows(int m) {
  int R = 1;
  while (32 * R < m) R <<= 1;
  return R;
}

cudaError_t launch_small(const SmallParams& p0, int warps_per_cta, int grid, cudaStream_t st) {
  SmallParams p = p0;
  const int R = small_rows(p.m);
  p.warp_bytes = (int)small_warp_bytes(p.m, p.d_pad);
  int n2 = 32;
  while (n2 < p.m) n2 <<= 1;
  p.n2 = n2;
  const size_t smem = (size_t)p.d * 32 * R * 8 + (size_t)warps_per_cta * p.warp_bytes;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 32 * warps_per_cta, smem, st>>>(p);
    return cudaGetLastError();
  };
  switch (R) {
    case 1: return go(small_kernel<1>);
    case 2: return go(small_kernel<2>);
    case 4: return go(small_kernel<4>);
    case 8: return go(small_kernel<8>);
    case 16: return go(small_kernel<16>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tmvn
