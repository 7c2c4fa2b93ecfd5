// cp.cu -- constraint-parallel iterations: the rows of A are split over
// ranks (GPUs); every rank holds all C chains' x (replicated) and the rows P_r = A_r x,
// Q_r = A_r nu of its own constraints.  One iteration of Alg. 1 becomes four
// launches around three collectives that the caller runs (torch.distributed / NCCL):
//
//   cp_stats   arcs of the rank's rows (eq:roots, C1-C5) -> per-chain level-1 bucket
//              tables over [0, 2 pi]: max beta (exact, two words), max alpha (high
//              word), count                         -> all-reduce (max, max, sum)
//   cp_live    gamma entering each bucket = exclusive prefix max of the merged max beta
//              (Prop. 1); the rank's arcs in live buckets (max alpha > gamma
//              in) with beta > gamma in         -> all-gather
//   cp_theta   every rank, identically: gamma before each gathered arc (its bucket's
//              gamma in and the beta of the bucket's arcs before it), the gaps, trim
//              (C7), theta by the inverse CDF (C10); P' = P cos + Q sin for the rank's
//              rows and the safeguard (C8)   -> all-reduce (max)
//   cp_commit  accept iff no rank saw a violation: x <- x cos + nu sin (every rank, the
//              same), P_r <- P'_r (a per-chain buffer flip, no copy), moments; else stay (C8)
//
// The union of the infeasible arcs is associative (Prop. 1), so the merged tables and
// the gathered live arcs give every rank the same I_act as one GPU holding all m rows;
// the projection rows are computed per element in a fixed order, so the trajectories
// are bitwise those of a single rank with the whole A.
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace tmvn {
namespace {

constexpr int kCT = 256;   // threads per chain (one CTA per chain)
constexpr int kCNB = kCpBuckets;

__device__ __forceinline__ uint64_t cbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double cbitsd(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ int cbucket(double a, double scale) {
  const int k = (int)__dmul_rn(a, scale);
  return k < kCNB - 1 ? k : kCNB - 1;
}

__global__ void __launch_bounds__(kCT) cp_stats_kernel(const double* __restrict__ P0, const double* __restrict__ P1,
                                                       const unsigned char* __restrict__ cur,
                                                       const double* __restrict__ Q, int64_t ldp,
                                                       const double* __restrict__ b, int m,
                                                       uint64_t* __restrict__ gx, uint64_t* __restrict__ ma,
                                                       int* __restrict__ cnt, double2* __restrict__ arcs) {
  __shared__ uint64_t sG[kCNB], sA[kCNB];
  __shared__ int sC[kCNB];
  const int c = blockIdx.x, tid = threadIdx.x;
  const double scale = __ddiv_rn((double)kCNB, kTwoPi);
  for (int k = tid; k < kCNB; k += kCT) {
    sG[k] = 0;
    sA[k] = 0;
    sC[k] = 0;
  }
  __syncthreads();
  const double* Pc = (cur[c] ? P1 : P0) + (int64_t)c * ldp;  // this chain's current P buffer
  const double* Qc = Q + (int64_t)c * ldp;
  double2* Ac = arcs + (int64_t)c * ldp;  // the row's arc, (-1, -1) when inactive: read by
                                          // the low-word pass and by cp_live (no recompute)
  for (int i = tid; i < m; i += kCT) {
    double al, be;
    if (arc_of(Pc[i], Qc[i], __ldg(b + i), al, be)) {
      const int k = cbucket(al, scale);
      atomicMax(reinterpret_cast<uint32_t*>(&sG[k]) + 1, (uint32_t)(cbits(be) >> 32));
      atomicMax(reinterpret_cast<uint32_t*>(&sA[k]) + 1, (uint32_t)(cbits(al) >> 32));
      atomicAdd(&sC[k], 1);
      Ac[i] = make_double2(al, be);
    } else {
      Ac[i] = make_double2(-1.0, -1.0);
    }
  }
  __syncthreads();
  for (int i = tid; i < m; i += kCT) {  // exact max beta: the low words
    const double2 ab = Ac[i];
    if (ab.x >= 0.0) {
      const int k = cbucket(ab.x, scale);
      if ((uint32_t)(cbits(ab.y) >> 32) == (uint32_t)(sG[k] >> 32))
        atomicMax(reinterpret_cast<uint32_t*>(&sG[k]), (uint32_t)cbits(ab.y));
    }
  }
  __syncthreads();
  for (int k = tid; k < kCNB; k += kCT) {
    gx[(int64_t)c * kCNB + k] = sG[k];
    ma[(int64_t)c * kCNB + k] = sA[k];
    cnt[(int64_t)c * kCNB + k] = sC[k];
  }
}

// gamma entering each bucket (exclusive prefix max of the merged max beta), the live
// flags (conservative on the high word of max alpha) and gamma after the last bucket
__device__ void cp_gamma(const uint64_t* gx, const uint64_t* ma, const int* cnt, uint64_t* gin, int* live,
                         uint64_t* gtot, uint64_t* wscr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t g = 0;
  if (tid < kCNB) g = gx[tid];
  uint64_t inc = g;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = inc > n ? inc : n;
  }
  if (lane == 31 && warp < kCNB / 32) wscr[warp] = inc;
  __syncthreads();
  if (tid < kCNB) {
    uint64_t pre = 0;
    for (int w = 0; w < warp; ++w) pre = pre > wscr[w] ? pre : wscr[w];
    uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) exc = 0;
    const uint64_t gi = pre > exc ? pre : exc;
    gin[tid] = gi;
    live[tid] = cnt[tid] > 0 && (ma[tid] | 0xFFFFFFFFull) > gi;
    if (tid == kCNB - 1) *gtot = gi > g ? gi : g;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kCT) cp_live_kernel(const double2* __restrict__ arcs, int64_t ldp, int m,
                                                      const uint64_t* __restrict__ gx, const uint64_t* __restrict__ ma,
                                                      const int* __restrict__ cnt, int cap,
                                                      double2* __restrict__ live_out, int* __restrict__ nlive) {
  __shared__ uint64_t gin[kCNB], wscr[8], gtot;
  __shared__ int live[kCNB], count;
  const int c = blockIdx.x, tid = threadIdx.x;
  const double scale = __ddiv_rn((double)kCNB, kTwoPi);
  if (tid == 0) count = 0;
  cp_gamma(gx + (int64_t)c * kCNB, ma + (int64_t)c * kCNB, cnt + (int64_t)c * kCNB, gin, live, &gtot, wscr);
  const double2* Ac = arcs + (int64_t)c * ldp;
  for (int i = tid; i < m; i += kCT) {
    const double2 ab = Ac[i];
    const double al = ab.x, be = ab.y;
    if (al >= 0.0) {
      const int k = cbucket(al, scale);
      // beta <= gamma in: inside the earlier arc that set gamma in (it starts before the
      // bucket): changes neither the union nor any later gamma
      if (live[k] && cbits(be) > gin[k]) {
        const int pos = atomicAdd(&count, 1);
        if (pos < cap) live_out[(int64_t)c * cap + pos] = make_double2(al, be);
      }
    }
  }
  __syncthreads();
  if (tid == 0) nlive[c] = count;
}

// canonical gaps (merge touching), trim (C7), L, theta = inverse CDF at u (C10); one thread
__device__ void cp_sample(double2* gaps, int ngap, double u, double eps, double* theta, double* Lout) {
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

__global__ void __launch_bounds__(kCT) cp_theta_kernel(
    const uint64_t* __restrict__ gx, const uint64_t* __restrict__ ma, const int* __restrict__ cnt,
    const double2* __restrict__ all_live, const int* __restrict__ all_n, int world, int cap, uint64_t seed,
    uint32_t t, uint32_t chain_offset, double eps, double* __restrict__ P0, double* __restrict__ P1,
    const unsigned char* __restrict__ cur, const double* __restrict__ Q, int64_t ldp, const double* __restrict__ b,
    int m, int* __restrict__ flags, double* __restrict__ theta_out, double* __restrict__ L_out) {
  extern __shared__ __align__(16) unsigned char csm[];
  __shared__ uint64_t gin[kCNB], wscr[8], gtot;
  __shared__ int live[kCNB], ncand, total_s, viol_s;
  __shared__ double th_s, L_s;
  const int c = blockIdx.x, tid = threadIdx.x;
  const double scale = __ddiv_rn((double)kCNB, kTwoPi);
  // the gathered arcs of every rank, then the gap candidates (key, gamma) after them
  int total = 0, overflow = 0;
  for (int r = 0; r < world; ++r) {
    const int n = all_n[(int64_t)r * gridDim.x + c];
    total += min(n, cap);
    overflow |= n > cap;  // some rank dropped live arcs of this chain: I_act would be wrong
  }
  uint64_t* key = reinterpret_cast<uint64_t*>(csm);
  double* val = reinterpret_cast<double*>(key + total);
  uint64_t* cand = reinterpret_cast<uint64_t*>(val + total);
  double2* gaps = reinterpret_cast<double2*>(cand + 2 * (size_t)total);
  if (tid == 0) {
    ncand = 0;
    total_s = total;
    viol_s = 0;
  }
  cp_gamma(gx + (int64_t)c * kCNB, ma + (int64_t)c * kCNB, cnt + (int64_t)c * kCNB, gin, live, &gtot, wscr);
  {
    int base = 0;
    for (int r = 0; r < world; ++r) {
      const int n = min(all_n[(int64_t)r * gridDim.x + c], cap);
      const double2* src = all_live + ((int64_t)r * gridDim.x + c) * cap;
      for (int e = tid; e < n; e += kCT) {
        const double2 ab = src[e];
        key[base + e] = cbits(ab.x);
        val[base + e] = ab.y;
      }
      base += n;
    }
  }
  __syncthreads();
  // gamma before arc e: gamma entering its bucket and the beta of the bucket's arcs
  // before it (alpha order; equal alphas by position: the same gap either way)
  for (int e = tid; e < total; e += kCT) {
    const uint64_t ke = key[e];
    const int k = cbucket(cbitsd(ke), scale);
    uint64_t gm = gin[k];
    for (int f = 0; f < total; ++f) {
      const uint64_t kf = key[f];
      if ((kf < ke || (kf == ke && f < e)) && cbucket(cbitsd(kf), scale) == k) {
        const uint64_t vf = cbits(val[f]);
        gm = gm > vf ? gm : vf;
      }
    }
    if (ke > gm) {
      const int q = atomicAdd(&ncand, 1);
      cand[2 * q] = ke;
      cand[2 * q + 1] = gm;
    }
  }
  __syncthreads();
  const int nc = ncand;
  for (int q = tid; q < nc; q += kCT) {  // gaps in alpha order
    const uint64_t a = cand[2 * q];
    int rnk = 0;
    for (int q2 = 0; q2 < nc; ++q2) rnk += cand[2 * q2] < a ? 1 : 0;
    gaps[rnk] = make_double2(cbitsd(cand[2 * q + 1]), cbitsd(a));
  }
  __syncthreads();
  if (tid == 0) {
    int ng = nc;
    const double G = cbitsd(gtot);
    if (G < kTwoPi) gaps[ng++] = make_double2(G, kTwoPi);  // [gamma_m, 2 pi]
    double th, L;
    cp_sample(gaps, ng, theta_uniform(seed, t, chain_offset + (uint32_t)c), eps, &th, &L);
    th_s = th;
    L_s = L;
    theta_out[c] = th;
    L_out[c] = L;
  }
  __syncthreads();
  const double L = L_s;
  double sn = 0.0, cs = 1.0;
  if (L > 0.0) sincos(th_s, &sn, &cs);
  int viol = 0;
  const double* Pc = (cur[c] ? P1 : P0) + (int64_t)c * ldp;  // this chain's P, and P' in the other
  const double* Qc = Q + (int64_t)c * ldp;
  double* Pnc = (cur[c] ? P0 : P1) + (int64_t)c * ldp;
  if (L > 0.0) {
    for (int i = tid; i < m; i += kCT) {
      const double pn = Pc[i] * cs + Qc[i] * sn;
      Pnc[i] = pn;
      viol |= (pn - __ldg(b + i)) > 0.0 ? 1 : 0;
    }
  }
  viol = __syncthreads_or(viol);
  // 2: live-arc overflow -- the chain stays (no commit of a wrong I_act) and the caller
  // aborts at the next check (ConstraintParallel: every recompute_every iterations)
  if (tid == 0) flags[c] = overflow ? 2 : viol;
}

__global__ void __launch_bounds__(kCT) cp_commit_kernel(const int* __restrict__ flags, const double* __restrict__ theta,
                                                        const double* __restrict__ Lv, double* __restrict__ X,
                                                        const double* __restrict__ N, int64_t d_pad, int d,
                                                        unsigned char* __restrict__ cur, int record,
                                                        double* __restrict__ S1, double* __restrict__ S2,
                                                        int64_t* __restrict__ rej) {
  const int c = blockIdx.x, tid = threadIdx.x;
  const double L = Lv[c];
  const bool accept = L > 0.0 && flags[c] == 0;
  double sn = 0.0, cs = 1.0;
  if (accept) sincos(theta[c], &sn, &cs);
  for (int j = tid; j < d; j += kCT) {
    const int64_t o = tiled_offset(c, j, d_pad);
    double xv = X[o];
    if (accept) {
      xv = xv * cs + N[o] * sn;
      X[o] = xv;
    }
    if (record) {
      S1[o] += xv;
      S2[o] += xv * xv;
    }
  }
  if (tid == 0) {
    if (accept) cur[c] ^= 1;  // P' becomes P: no copy
    else rej[c] += 1;
  }
}

}  // namespace

cudaError_t launch_cp_stats(const double* P0, const double* P1, const unsigned char* cur, const double* Q, int64_t ldp,
                            const double* b, int m, int C, uint64_t* gx, uint64_t* ma, int* cnt, double2* arcs,
                            cudaStream_t st) {
  cp_stats_kernel<<<C, kCT, 0, st>>>(P0, P1, cur, Q, ldp, b, m, gx, ma, cnt, arcs);
  return cudaGetLastError();
}
cudaError_t launch_cp_live(const double2* arcs, int64_t ldp, int m, int C, const uint64_t* gx, const uint64_t* ma,
                           const int* cnt, int cap, double2* live, int* nlive, cudaStream_t st) {
  cp_live_kernel<<<C, kCT, 0, st>>>(arcs, ldp, m, gx, ma, cnt, cap, live, nlive);
  return cudaGetLastError();
}
size_t cp_theta_smem(int world, int cap) {
  const size_t n = (size_t)world * cap;
  return n * 8 + n * 8 + 2 * n * 8 + (n + 2) * 16;
}
cudaError_t launch_cp_theta(const uint64_t* gx, const uint64_t* ma, const int* cnt, const double2* all_live,
                            const int* all_n, int world, int cap, uint64_t seed, uint32_t t, uint32_t chain_offset,
                            double eps, double* P0, double* P1, const unsigned char* cur, const double* Q,
                            int64_t ldp, const double* b, int m, int C, int* flags, double* theta, double* L,
                            cudaStream_t st) {
  const size_t smem = cp_theta_smem(world, cap);
  cudaError_t e = cudaFuncSetAttribute(cp_theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cp_theta_kernel<<<C, kCT, smem, st>>>(gx, ma, cnt, all_live, all_n, world, cap, seed, t, chain_offset, eps, P0, P1,
                                        cur, Q, ldp, b, m, flags, theta, L);
  return cudaGetLastError();
}
cudaError_t launch_cp_commit(const int* flags, const double* theta, const double* L, double* X, const double* N,
                             int64_t d_pad, int d, unsigned char* cur, int C, int record, double* S1, double* S2,
                             int64_t* rej, cudaStream_t st) {
  cp_commit_kernel<<<C, kCT, 0, st>>>(flags, theta, L, X, N, d_pad, d, cur, record, S1, S2, rej);
  return cudaGetLastError();
}

}  // namespace tmvn
