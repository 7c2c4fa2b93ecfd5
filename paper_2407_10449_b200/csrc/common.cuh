// common.cuh -- device-side building blocks of the sm_100a path (no oracle code).
//
//  * Fragment-tiled operand layout shared by the DMMA GEMM, the RNG and the
//    per-chain kernel.
//  * Philox4x32-10 + Box-Muller (the RNG contract, C12).
//  * The per-constraint arc of eq:roots with the C1-C5 readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmvn {

// ----------------------------------------------------------------------------
// Fragment-tiled layout of an R x K operand (R = chains or constraints,
// K = dimension d).  R is padded to a multiple of 128 and K to a multiple of 16.
// A 128 x 16 block is one contiguous 16 KB chunk (one cp.async.bulk); blocks of
// the same 128 rows are consecutive in K.  Inside a chunk, 8-row group g and
// k-half kh (k%16 / 8) own 64 doubles, ordered by mma.m8n8k4 lane:
//   lane = (r % 8) * 4 + (k % 4),  slot = lane * 2 + ((k % 8) / 4)
// so one ld.shared.v2.f64 per lane yields the A (row-major) or B (col-major)
// fragments of two consecutive k4 steps, with no bank conflicts.  A row's 8
// consecutive k (k = 8a .. 8a+7) form one contiguous 64-byte run.
// ----------------------------------------------------------------------------
constexpr int kTileR = 128;
constexpr int kTileK = 16;
constexpr int kChunk = kTileR * kTileK;  // doubles per chunk

__host__ __device__ inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

__host__ __device__ inline int64_t tiled_offset(int64_t r, int64_t k, int64_t K_pad) {
  int64_t chunk = (r / kTileR) * (K_pad / kTileK) + k / kTileK;
  int64_t g = (r % kTileR) / 8, kh = (k % kTileK) / 8;
  int64_t lane = (r % 8) * 4 + (k % 4);
  return chunk * kChunk + (g * 2 + kh) * 64 + lane * 2 + ((k % 8) / 4);
}

// Start of the 64-byte run holding k = 8a .. 8a+7 of row r.
__host__ __device__ inline int64_t run_offset(int64_t r, int64_t a, int64_t K_pad) {
  int64_t k = a * 8;
  int64_t chunk = (r / kTileR) * (K_pad / kTileK) + k / kTileK;
  int64_t g = (r % kTileR) / 8, kh = (k % kTileK) / 8;
  return chunk * kChunk + (g * 2 + kh) * 64 + (r % 8) * 8;
}
// Position inside a run of k (0..7 = k % 8).
__host__ __device__ inline int run_slot(int kk) { return (kk % 4) * 2 + kk / 4; }

// ----------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).
// ----------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    U4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 53-bit uniform on [0, 1) from (lo, hi) words.
__device__ __forceinline__ double u53(uint32_t lo, uint32_t hi) {
  uint64_t bits = ((uint64_t)hi << 32) | lo;
  return __dmul_rn((double)(bits >> 11), 1.1102230246251565e-16);  // 2^-53
}

constexpr double kTwoPi = 6.283185307179586;

// Two normals nu_{2j}, nu_{2j+1} of chain `chain` at iteration t (C12).
__device__ __forceinline__ void normal_pair(uint64_t seed, uint32_t j, uint32_t t, uint32_t chain,
                                            double& n0, double& n1) {
  U4 w = philox10(U4{j, t, chain, 0u}, (uint32_t)seed, (uint32_t)(seed >> 32));
  double ua = u53(w.x, w.y), ub = u53(w.z, w.w);
  double radius = sqrt(__dmul_rn(-2.0, log(__dsub_rn(1.0, ua))));
  double s, c;
  sincos(__dmul_rn(kTwoPi, ub), &s, &c);
  n0 = __dmul_rn(radius, c);
  n1 = __dmul_rn(radius, s);
}

// u_{c,t} for "sample uniformly theta ~ I_act": U_a of block (0, t, c, 1).
__device__ __forceinline__ double theta_uniform(uint64_t seed, uint32_t t, uint32_t chain) {
  U4 w = philox10(U4{0u, t, chain, 1u}, (uint32_t)seed, (uint32_t)(seed >> 32));
  return u53(w.x, w.y);
}

// Fill one 64-byte run (k = 8a .. 8a+7) of nu with normals; zeros for k >= d.
__device__ __forceinline__ void normal_run(uint64_t seed, uint32_t t, uint32_t chain, int a, int d,
                                           double out[8]) {
#pragma unroll
  for (int pr = 0; pr < 4; ++pr) {
    int k0 = a * 8 + pr * 2;
    double n0 = 0.0, n1 = 0.0;
    if (k0 < d) {
      normal_pair(seed, (uint32_t)(k0 / 2), t, chain, n0, n1);
      if (k0 + 1 >= d) n1 = 0.0;
    }
    out[run_slot(pr * 2)] = n0;
    out[run_slot(pr * 2 + 1)] = n1;
  }
}

// ----------------------------------------------------------------------------
// Infeasible arc of constraint (p, q, b) on the ellipse (Eq. 2, eq:roots):
// r = hypot(p, q); active iff r > b (C3); rho = clamp(b / r) (C5);
// tau = atan2(q, p); delta = acos(rho); (alpha, beta) = (tau - delta, tau + delta)
// shifted into [0, 2 pi] by C1.  Returns false for an inactive constraint.
// ----------------------------------------------------------------------------
__device__ __forceinline__ bool arc_of(double p, double q, double b, double& alpha, double& beta) {
  double r = hypot(p, q);
  if (!(r > b)) return false;
  double rho = __ddiv_rn(b, r);
  rho = fmin(fmax(rho, -1.0), 1.0);
  double tau = atan2(q, p);
  double delta = acos(rho);
  double lo = __dsub_rn(tau, delta);
  double hi = __dadd_rn(tau, delta);
  if (hi <= 0.0) {
    lo = __dadd_rn(lo, kTwoPi);
    hi = __dadd_rn(hi, kTwoPi);
  } else if (lo >= 0.0) {
    // inside [0, 2 pi]
  } else if (-lo <= hi) {
    lo = 0.0;                       // straddle (rounding only): snap the shorter side (C1)
  } else {
    lo = __dadd_rn(lo, kTwoPi);
    hi = kTwoPi;
  }
  alpha = lo;
  beta = hi;
  return true;
}

}  // namespace tmvn
