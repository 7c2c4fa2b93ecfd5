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
// k-half kh (k%16 / 8) own 64 doubles = eight 64-byte runs, one per row
// (r % 8), each run holding k = 8a .. 8a+7 in order.  Lane l of an
// mma.m8n8k4 reads doubles 2l, 2l+1 with one ld.shared.v2.f64: row l/4 and
// k = 2(l%4) + {0, 1}, i.e. the fragments of two k4-steps under the k
// permutation (j, v) -> 2j + v, which is the same for both operands, so the
// product is unchanged; the 32 lanes read 512 contiguous bytes (no bank
// conflicts).  A normal pair (nu_{2j}, nu_{2j+1}) is one aligned double2.
// ----------------------------------------------------------------------------
constexpr int kTileR = 128;
constexpr int kTileK = 16;
constexpr int kChunk = kTileR * kTileK;  // doubles per chunk

__host__ __device__ inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

// Start of the 64-byte run holding k = 8a .. 8a+7 of row r.
__host__ __device__ inline int64_t run_offset(int64_t r, int64_t a, int64_t K_pad) {
  int64_t chunk = (r / kTileR) * (K_pad / kTileK) + a / 2;
  int64_t g = (r % kTileR) / 8, kh = a % 2;
  return chunk * kChunk + (g * 2 + kh) * 64 + (r % 8) * 8;
}

__host__ __device__ inline int64_t tiled_offset(int64_t r, int64_t k, int64_t K_pad) {
  return run_offset(r, k / 8, K_pad) + (k % 8);
}

// The tiled offset separates into a row part and a column part:
// tiled_offset(r, k) = tiled_row(r) + tiled_col(k) (hot loops step k with 32-bit adds).
__host__ __device__ inline int64_t tiled_row(int64_t r, int64_t K_pad) {
  return (r / kTileR) * (K_pad / kTileK) * kChunk + ((r % kTileR) / 8) * 128 + (r % 8) * 8;
}
__host__ __device__ inline int tiled_col(int k) { return (k >> 4) * kChunk + ((k >> 3) & 1) * 64 + (k & 7); }

// ----------------------------------------------------------------------------
// mbarrier + cp.async.bulk (TMA bulk engine, SASS UBLKCP) helpers.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

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

// nu_{2j}, nu_{2j+1} for k0 = 2j < d as a double2 (zero beyond d).
__device__ __forceinline__ double2 normal_pair_at(uint64_t seed, uint32_t t, uint32_t chain, int k0,
                                                  int d) {
  double n0 = 0.0, n1 = 0.0;
  if (k0 < d) {
    normal_pair(seed, (uint32_t)(k0 / 2), t, chain, n0, n1);
    if (k0 + 1 >= d) n1 = 0.0;
  }
  return make_double2(n0, n1);
}

// Timeline instrumentation (variant build -DTMVN_TIMELINE only; tools/timeline.py):
// per launch sequence number, the first CTA start and last CTA end (globaltimer ns)
// of the projection GEMM (slots 0, 1) and of the per-chain kernel (slots 2, 3).
#ifdef TMVN_TIMELINE
// each translation unit has its own copy (no relocatable device code); the host
// helpers tl_access_* of gemm_i8.cu and ess_chain.cu reset / read them
static __device__ unsigned long long g_tl[256][4];
static __device__ unsigned int g_tl_seq[2];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// ----------------------------------------------------------------------------
// Digit layout of the int8 (Ozaki-split) projection operands (gemm_i8.cu).
// A value v with |v| < 2^e becomes the fixed-point integer
// X = trunc(v 2^(8S-1-e)), |X| < 2^(8S-1), cut into S two's-complement byte
// digits (digit 0 signed, the rest unsigned).  Operand rows are grouped in
// blocks of BR (128 for A', 64 for nu) and K in steps of 32 bytes; digit s of a
// (row block, K step) is one BR x 32 slice in the UMMA canonical K-major
// SWIZZLE_NONE layout: [k / 16 within the step][8-row group][row % 8][k % 16].
// ----------------------------------------------------------------------------
constexpr int kOzStepK = 32;   // K bytes per step (one tcgen05.mma kind::i8)
constexpr int kOzNuRows = 64;  // nu rows (chains) per block = MMA N
constexpr int kOzNuExp = 4;    // |nu| <= sqrt(-2 ln 2^-53) < 8.58 < 2^4

__host__ __device__ inline int64_t oz_offset(int64_t r, int64_t k, int s, int S, int64_t KB, int BR) {
  const int64_t blk = ((r / BR) * KB + k / kOzStepK) * S + s;
  return blk * (int64_t)(BR * kOzStepK) + ((k % kOzStepK) / 16) * (BR / 8) * 128 +
         ((r % BR) / 8) * 128 + (r % 8) * 16 + (k % 16);
}

// oz_offset(r, k, s, S, KB, BR) = oz_row(r) + oz_col(k) + s BR 32 (row / column parts)
__host__ __device__ inline int64_t oz_row(int64_t r, int S, int64_t KB, int BR) {
  return (r / BR) * KB * S * (int64_t)(BR * kOzStepK) + ((r % BR) / 8) * 128 + (r % 8) * 16;
}
__host__ __device__ inline int oz_col(int k, int S, int BR) {
  return (k / kOzStepK) * S * (BR * kOzStepK) + ((k % kOzStepK) / 16) * (BR / 8) * 128 + (k % 16);
}

__device__ __forceinline__ int64_t oz_fixed(double v, int S, int e) {
  return __double2ll_rz(scalbn(v, 8 * S - 1 - e));  // any e (A' rows may be tiny)
}
// nu (e = kOzNuExp): v 2^(8S-1-e) is an exact product with a normal power of two
__device__ __forceinline__ int64_t oz_fixed_nu(double v, int S) {
  return __double2ll_rz(v * __longlong_as_double((long long)(1023 + 8 * S - 1 - kOzNuExp) << 52));
}

__device__ __forceinline__ uint32_t oz_digit(int64_t X, int s, int S) {
  const int64_t sh = X >> (8 * (S - 1 - s));  // arithmetic shift
  return (uint32_t)(sh & 0xFF);               // digit 0: two's-complement byte of a value in [-128, 127]
}

// The S digits of the nu pair (v0, v1) at coordinates k, k + 1 (k even) of chain r:
// digit s of X is byte S-1-s of its 64-bit two's complement (|X| < 2^(8S-1)), so
// each 16-bit store is one byte permute of the two values' words; the S slices of
// one (row block, K step) are BR x 32 bytes apart.
__device__ __forceinline__ void oz_store_nu_pair(int8_t* Ns, int64_t r, int k, double v0, double v1,
                                                 int S, int64_t KB) {
  const int64_t X0 = oz_fixed_nu(v0, S), X1 = oz_fixed_nu(v1, S);
  const uint32_t lo0 = (uint32_t)X0, hi0 = (uint32_t)((uint64_t)X0 >> 32);
  const uint32_t lo1 = (uint32_t)X1, hi1 = (uint32_t)((uint64_t)X1 >> 32);
  int8_t* base = Ns + oz_offset(r, k, 0, S, KB, kOzNuRows);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    if (s < S) {
      const int b = S - 1 - s;  // byte of X
      const uint32_t w = b < 4 ? __byte_perm(lo0, lo1, (uint32_t)(b | ((b + 4) << 4)))
                               : __byte_perm(hi0, hi1, (uint32_t)((b - 4) | (b << 4)));
      *reinterpret_cast<uint16_t*>(base + s * (kOzNuRows * kOzStepK)) = (uint16_t)w;
    }
  }
}

// The same S digits at a precomputed address (digit 0 of the pair); S a compile-time
// constant: the byte selectors fold into the permutes.
template <int S>
__device__ __forceinline__ void oz_put_nu_pair(int8_t* base, double v0, double v1) {
  const int64_t X0 = oz_fixed_nu(v0, S), X1 = oz_fixed_nu(v1, S);
  const uint32_t lo0 = (uint32_t)X0, hi0 = (uint32_t)((uint64_t)X0 >> 32);
  const uint32_t lo1 = (uint32_t)X1, hi1 = (uint32_t)((uint64_t)X1 >> 32);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int b = S - 1 - s;
    const uint32_t w = b < 4 ? __byte_perm(lo0, lo1, (uint32_t)(b | ((b + 4) << 4)))
                             : __byte_perm(hi0, hi1, (uint32_t)((b - 4) | (b << 4)));
    *reinterpret_cast<uint16_t*>(base + s * (kOzNuRows * kOzStepK)) = (uint16_t)w;
  }
}
__device__ __forceinline__ void oz_put_nu_pair_s(int8_t* base, double v0, double v1, int S) {
  switch (S) {  // uniform
    case 4: oz_put_nu_pair<4>(base, v0, v1); break;
    case 6: oz_put_nu_pair<6>(base, v0, v1); break;
    case 8: oz_put_nu_pair<8>(base, v0, v1); break;
    default: oz_put_nu_pair<7>(base, v0, v1); break;
  }
}

// ----------------------------------------------------------------------------
// Branch-free FP64 atan2 (the libm one branches per octant and diverges inside a
// warp).  t = min(|x|,|y|) / max(|x|,|y|) in [0, 1]; for t > tan(pi/8) the
// identity atan(t) = pi/4 + atan((t-1)/(t+1)) folds the argument to
// |t'| <= tan(pi/8) with the same single quotient ((mn-mx)/(mn+mx)); then
// atan(t') = t' P(t'^2), P of degree 10 fitted by Chebyshev interpolation
// (tools/fit_atan.py: 2.2e-16 max relative error in FP64 Horner/FMA).  The
// octant is undone in one step, atan2 = base[code] +/- atan(t'), with the 8
// bases (sums of multiples of pi/4 and pi, rounded once) in constant memory.
// The quotient uses a hardware reciprocal estimate refined by two Newton steps
// (relative error ~1e-16).  Signed zeros follow atan2: y = -0 gives -0 / -pi.
// ----------------------------------------------------------------------------
__constant__ double kAtanP[11] = {1.0, -0.3333333333332844, 0.1999999999885511,
                                  -0.14285714180976467, 0.11111106180455946,
                                  -0.09090773074808414, 0.07689953496306857,
                                  -0.06640233930429408, 0.056883492268090106,
                                  -0.04348052215716462, 0.021135373157693246};
// code = big | swap << 1 | xneg << 2: result magnitude = base + sgn * atan(t')
__constant__ double kAtanBase[8] = {
    0.0,                    // t' = t
    0.7853981633974483,     // pi/4 + t'
    1.5707963267948966,     // pi/2 - t'
    0.7853981633974483,     // pi/2 - (pi/4 + t') = pi/4 - t'
    3.141592653589793,      // pi - t'
    2.356194490192345,      // pi - (pi/4 + t') = 3pi/4 - t'
    1.5707963267948966,     // pi - (pi/2 - t') = pi/2 + t'
    2.356194490192345};     // pi - (pi/4 - t') = 3pi/4 + t'
// sign of t' per code: + for codes 0, 1, 6, 7
__device__ __forceinline__ double fast_recip(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double fast_atan2(double y, double x) {
  const double ax = fabs(x), ay = fabs(y);
  const double mx = ay > ax ? ay : ax, mn = ay > ax ? ax : ay;  // |x|, |y|: no NaN handling needed
  const bool big = mn > 0.41421356237309503 * mx;
  const double num = big ? mn - mx : mn;
  const double den = big ? mn + mx : mx;
  const double t = den > 0.0 ? num * fast_recip(den) : 0.0;
  const double z = t * t;
  double pz = kAtanP[10];
#pragma unroll
  for (int i = 9; i >= 1; --i) pz = fma(pz, z, kAtanP[i]);
  const double at = fma(t * z, pz, t);  // atan(t') = t (1 + z P1(z))
  const int code = (big ? 1 : 0) | (ay > ax ? 2 : 0) | ((__double_as_longlong(x) < 0) ? 4 : 0);
  const double sat = ((0xC3u >> code) & 1u) ? at : -at;  // + for codes 0, 1, 6, 7
  const double r = kAtanBase[code] + sat;
  return (__double_as_longlong(y) < 0) ? -r : r;
}

// Two independent atan2 with the operations of fast_atan2 (bit-identical results):
// the polynomial coefficients are loaded once for both, and the two dependency
// chains interleave.
__device__ __forceinline__ void fast_atan2_2(double y1, double x1, double y2, double x2, double& r1,
                                             double& r2) {
  const double ax1 = fabs(x1), ay1 = fabs(y1), ax2 = fabs(x2), ay2 = fabs(y2);
  const double mx1 = ay1 > ax1 ? ay1 : ax1, mn1 = ay1 > ax1 ? ax1 : ay1;  // non-negative, no NaN
  const double mx2 = ay2 > ax2 ? ay2 : ax2, mn2 = ay2 > ax2 ? ax2 : ay2;
  const bool big1 = mn1 > 0.41421356237309503 * mx1, big2 = mn2 > 0.41421356237309503 * mx2;
  const double num1 = big1 ? mn1 - mx1 : mn1, den1 = big1 ? mn1 + mx1 : mx1;
  const double num2 = big2 ? mn2 - mx2 : mn2, den2 = big2 ? mn2 + mx2 : mx2;
  const double t1 = den1 > 0.0 ? num1 * fast_recip(den1) : 0.0;
  const double t2 = den2 > 0.0 ? num2 * fast_recip(den2) : 0.0;
  const double z1 = t1 * t1, z2 = t2 * t2;
  double p1 = kAtanP[10], p2 = kAtanP[10];
#pragma unroll
  for (int i = 9; i >= 1; --i) {
    const double c = kAtanP[i];
    p1 = fma(p1, z1, c);
    p2 = fma(p2, z2, c);
  }
  const double at1 = fma(t1 * z1, p1, t1), at2 = fma(t2 * z2, p2, t2);
  const int code1 = (big1 ? 1 : 0) | (ay1 > ax1 ? 2 : 0) | ((__double_as_longlong(x1) < 0) ? 4 : 0);
  const int code2 = (big2 ? 1 : 0) | (ay2 > ax2 ? 2 : 0) | ((__double_as_longlong(x2) < 0) ? 4 : 0);
  const double s1 = ((0xC3u >> code1) & 1u) ? at1 : -at1, s2 = ((0xC3u >> code2) & 1u) ? at2 : -at2;
  const double q1 = kAtanBase[code1] + s1, q2 = kAtanBase[code2] + s2;
  r1 = (__double_as_longlong(y1) < 0) ? -q1 : q1;
  r2 = (__double_as_longlong(y2) < 0) ? -q2 : q2;
}

// ----------------------------------------------------------------------------
// Infeasible arc of constraint (p, q, b) on the ellipse (Eq. 2, eq:roots):
// r = |(p, q)|; active iff r > b (C3); tau = atan2(q, p);
// delta = arccos(b / r) computed as atan2(s, b) with s = sqrt(r^2 - b^2) (the
// same angle in [0, pi]; the clamp of C5 becomes max(s^2, 0)); active iff
// b < 0 or s^2 > 0; (alpha, beta) = (tau - delta, tau + delta) shifted into
// [0, 2 pi] by C1.  Returns false for an inactive constraint.
// ----------------------------------------------------------------------------
__device__ __forceinline__ bool arc_active(double p, double q, double b) {
  const double s2 = fma(p, p, fma(q, q, -b * b));  // p^2 + q^2 - b^2
  return b < 0.0 || s2 > 0.0;
}
// sqrt(x) for x >= 0 within ~1 ulp (not correctly rounded; the arcs' parity bar is 1e-10):
// the MUFU reciprocal-square-root estimate, two Newton steps on it and one on the root --
// ~13 instructions instead of the IEEE sqrt's ~35 with its slow-path call; tiny or zero
// x (rare: near-tangent arcs) take the IEEE sqrt.
__device__ __forceinline__ double arc_sqrt(double x) {
  if (!(x >= 0x1p-1000)) return sqrt(x > 0.0 ? x : 0.0);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  const double r = x * y;
  return fma(0.5 * y, fma(-r, r, x), r);
}

__device__ __forceinline__ bool arc_of(double p, double q, double b, double& alpha, double& beta) {
  const double s2 = fma(p, p, fma(q, q, -b * b));  // p^2 + q^2 - b^2 (as in arc_active)
  if (!(b < 0.0 || s2 > 0.0)) return false;
  const double s = arc_sqrt(s2);
  double tau, delta;
  fast_atan2_2(q, p, s, b, tau, delta);
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
