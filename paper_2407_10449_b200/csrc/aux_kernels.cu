// aux_kernels.cu -- data movement and small kernels around the hot loop:
// layout conversion, the first nu draw, the strict start check (C18), moment
// reduction, App. A helpers, and the test-hook kernels.
#define QUALIFIERS static __forceinline__ __device__
#include <curand_philox4x32_x.h>
#include "common.cuh"
#include "internal.h"

namespace tmvn {
namespace {

__global__ void pack_kernel(const double* __restrict__ src, int64_t R, int64_t K, int64_t ld,
                            double* __restrict__ dst, int64_t K_pad) {
  int64_t n = R * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / K, k = e % K;
    dst[tiled_offset(r, k, K_pad)] = src[r * ld + k];
  }
}

__global__ void unpack_kernel(const double* __restrict__ src, int64_t R, int64_t K, int64_t K_pad,
                              double* __restrict__ dst) {
  int64_t n = R * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / K, k = e % K;
    dst[e] = src[tiled_offset(r, k, K_pad)];
  }
}

// one thread per normal pair (one double2 of the tiled N)
__global__ void normals_kernel(double* __restrict__ N, int C, int d, int64_t d_pad, uint64_t seed,
                               uint32_t t, uint32_t chain_offset) {
  const int pairs = (int)(d_pad / 2);
  int64_t n = (int64_t)C * pairs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(e / pairs), k0 = 2 * (int)(e % pairs);
    *reinterpret_cast<double2*>(N + tiled_offset(c, k0, d_pad)) =
        normal_pair_at(seed, t, chain_offset + (uint32_t)c, k0, d);
  }
}

// nu of iteration t (t_dev: graph replay, t offset from device memory) into the tiled
// FP64 N and, for the int8 projection, its digits Ns.  Launched on a second stream
// beside the projection GEMM of the previous iteration or the per-chain kernel
// (small 64-thread CTAs of < 40 registers: one fits in the 4 K registers that three
// per-chain CTAs leave free on an SM, several next to the GEMM's CTA).
__global__ void __launch_bounds__(64) nu_kernel(double* __restrict__ N, int8_t* __restrict__ Ns, int S,
                                                    int64_t KB, int C, int d, int64_t d_pad, uint64_t seed,
                                                    uint32_t t, const uint32_t* __restrict__ t_dev,
                                                    uint32_t chain_offset) {
  const uint32_t tt = t_dev ? *t_dev + t : t;
  // a warp = 4 consecutive chains x 8 consecutive pairs (16 coordinates): its nu stores
  // are 4 adjacent 64-byte runs of the tiled layout, its digit stores 64 contiguous
  // bytes per digit slice (4 rows x 16 bytes of one core matrix): whole sectors
  const int pblocks = (int)(d_pad / 16);
  const int64_t cblocks = (C + 3) / 4;
  const int64_t nw = cblocks * pblocks;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int c = (int)((w / pblocks) * 4 + (lane >> 3));
    const int k0 = (int)(w % pblocks) * 16 + 2 * (lane & 7);
    if (c >= C) continue;
    const double2 v = normal_pair_at(seed, tt, chain_offset + (uint32_t)c, k0, d);
    *reinterpret_cast<double2*>(N + tiled_offset(c, k0, d_pad)) = v;
    if (Ns) oz_store_nu_pair(Ns, c, k0, v.x, v.y, S, KB);
  }
}

__global__ void start_check_kernel(const double* __restrict__ P, int64_t ldp,
                                   const double* __restrict__ b, int C, int m,
                                   unsigned long long* flag) {
  int64_t n = (int64_t)C * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = e / m, i = e % m;
    double s = P[c * ldp + i] - b[i];
    if (!(s < 0.0)) atomicMin(flag, (unsigned long long)e);  // NaN also fails
  }
}

// Deterministic two-level sum over chains: block (x, y) sums chains
// [64y, 64y + 64) in index order for coordinates 128x .. 128x+127 into
// part[y][j]; chain_sum_final adds the parts in index order.
constexpr int kSumChunk = 64;
__global__ void chain_sum_part_kernel(const double* __restrict__ S, int C, int d, int64_t d_pad,
                                      double* __restrict__ part) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int c0 = blockIdx.y * kSumChunk;
  if (j >= d) return;
  double s = 0.0;
  int c1 = min(C, c0 + kSumChunk);
  for (int c = c0; c < c1; ++c) s += S[tiled_offset(c, j, d_pad)];
  part[(int64_t)blockIdx.y * d + j] = s;
}
__global__ void chain_sum_final_kernel(const double* __restrict__ part, int nparts, int d,
                                       double* __restrict__ out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double s = 0.0;
  for (int y = 0; y < nparts; ++y) s += part[(int64_t)y * d + j];
  out[j] = s;
}

__global__ void accum_affine_kernel(const double* __restrict__ X, int64_t ldx,
                                    const double* __restrict__ mu, int C, int d,
                                    double* __restrict__ S1, double* __restrict__ S2) {
  int64_t n = (int64_t)C * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = e / d, j = e % d;
    double x = X[c * ldx + j] + (mu ? mu[j] : 0.0);
    S1[e] += x;
    S2[e] += x * x;
  }
}

__global__ void add_vec_rows_kernel(double* __restrict__ X, int64_t ldx,
                                    const double* __restrict__ mu, int C, int d) {
  int64_t n = (int64_t)C * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = e / d, j = e % d;
    X[c * ldx + j] += mu[j];
  }
}

// Forward substitution u = L^{-1} (x - mu), one CTA per row, the dot products
// over the solved prefix reduced across the block.
__global__ void trsv_rows_kernel(const double* __restrict__ X, const double* __restrict__ mu,
                                 const double* __restrict__ L, int C, int d,
                                 double* __restrict__ U) {
  __shared__ double red[32];
  for (int c = blockIdx.x; c < C; c += gridDim.x) {
    const double* x = X + (int64_t)c * d;
    double* u = U + (int64_t)c * d;
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int k = threadIdx.x; k < j; k += blockDim.x) s += L[(int64_t)j * d + k] * u[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        u[j] = (x[j] - (mu ? mu[j] : 0.0) - t) / L[(int64_t)j * d + j];
      }
      __syncthreads();
    }
  }
}

__global__ void gather_rows_kernel(const double* __restrict__ Xt, int64_t d_pad, int d,
                                   const int64_t* __restrict__ rows, int n,
                                   double* __restrict__ out) {
  int64_t tot = (int64_t)n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = e / d, j = e % d;
    out[e] = Xt[tiled_offset(rows[k], j, d_pad)];
  }
}

__global__ void sum_i64_kernel(const int64_t* __restrict__ v, int n, int64_t* out) {
  __shared__ long long red[32];
  long long s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

__global__ void gemv_shift_kernel(const double* __restrict__ A, const double* __restrict__ b,
                                  const double* __restrict__ mu, int m, int d,
                                  double* __restrict__ out) {
  int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (row >= m) return;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s += A[(int64_t)row * d + j] * mu[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[row] = b[row] - s;
}

__global__ void test_philox_kernel(const uint32_t* __restrict__ ctr, const uint32_t* __restrict__ key,
                                   int64_t n, uint32_t* __restrict__ out, int use_curand) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t k0 = key[2 * i], k1 = key[2 * i + 1];
  if (use_curand) {
    uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
    uint4 r = curand_Philox4x32_10(c, make_uint2(k0, k1));
    out[4 * i] = r.x;
    out[4 * i + 1] = r.y;
    out[4 * i + 2] = r.z;
    out[4 * i + 3] = r.w;
  } else {
    U4 r = philox10(U4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, k0, k1);
    out[4 * i] = r.x;
    out[4 * i + 1] = r.y;
    out[4 * i + 2] = r.z;
    out[4 * i + 3] = r.w;
  }
}

__global__ void test_normals_kernel(uint64_t seed, uint32_t t, uint32_t c0, int C, int d,
                                    double* __restrict__ nu, double* __restrict__ u) {
  const int pairs = (d + 1) / 2;
  int64_t n = (int64_t)C * pairs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(e / pairs), k0 = 2 * (int)(e % pairs);
    double2 v = normal_pair_at(seed, t, c0 + (uint32_t)c, k0, d);
    nu[(int64_t)c * d + k0] = v.x;
    if (k0 + 1 < d) nu[(int64_t)c * d + k0 + 1] = v.y;
    if (k0 == 0 && u) u[c] = theta_uniform(seed, t, c0 + (uint32_t)c);
  }
}

__global__ void test_arcs_kernel(const double* __restrict__ p, const double* __restrict__ q,
                                 const double* __restrict__ b, int64_t n, double* alpha,
                                 double* beta, uint8_t* active) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double al = 0.0, be = 0.0;
  bool act = arc_of(p[i], q[i], b[i], al, be);
  alpha[i] = act ? al : 0.0;
  beta[i] = act ? be : 0.0;
  active[i] = act ? 1 : 0;
}

__global__ void set_u32_kernel(uint32_t* dst, uint32_t value) { *dst = value; }

// FP32 copy of a row-major R x K matrix into rows of K_pad (zero padding): FP32 mode
__global__ void to_f32_kernel(const double* __restrict__ src, int64_t R, int64_t K, int64_t ld,
                              float* __restrict__ dst, int64_t K_pad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R * K_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / K_pad, k = i - r * K_pad;
    dst[i] = k < K ? (float)src[r * ld + k] : 0.0f;
  }
}

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_to_f32(const double* src, int64_t R, int64_t K, int64_t ld, float* dst, int64_t K_pad,
                          cudaStream_t st) {
  if (R * K_pad == 0) return cudaSuccess;
  to_f32_kernel<<<grid_for(R * K_pad), 256, 0, st>>>(src, R, K, ld, dst, K_pad);
  return cudaGetLastError();
}

cudaError_t launch_pack(const double* src, int64_t R, int64_t K, int64_t ld, double* dst,
                        int64_t K_pad, cudaStream_t st) {
  if (R * K == 0) return cudaSuccess;
  pack_kernel<<<grid_for(R * K), 256, 0, st>>>(src, R, K, ld, dst, K_pad);
  return cudaGetLastError();
}
cudaError_t launch_unpack(const double* src, int64_t R, int64_t K, int64_t K_pad, double* dst,
                          cudaStream_t st) {
  if (R * K == 0) return cudaSuccess;
  unpack_kernel<<<grid_for(R * K), 256, 0, st>>>(src, R, K, K_pad, dst);
  return cudaGetLastError();
}
cudaError_t launch_normals(double* N, int C, int d, int64_t d_pad, uint64_t seed, uint32_t t,
                           uint32_t chain_offset, cudaStream_t st) {
  int64_t n = (int64_t)C * (d_pad / 2);
  if (n == 0) return cudaSuccess;
  normals_kernel<<<grid_for(n), 256, 0, st>>>(N, C, d, d_pad, seed, t, chain_offset);
  return cudaGetLastError();
}
cudaError_t launch_nu(double* N, int8_t* Ns, int S, int64_t KB, int C, int d, int64_t d_pad,
                      uint64_t seed, uint32_t t, const uint32_t* t_dev, uint32_t chain_offset,
                      cudaStream_t st, int ctas_per_sm) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if ((int64_t)C * (d_pad / 2) == 0) return cudaSuccess;
  nu_kernel<<<sms * ctas_per_sm, 64, 0, st>>>(N, Ns, S, KB, C, d, d_pad, seed, t, t_dev, chain_offset);
  return cudaGetLastError();
}
cudaError_t launch_start_check(const double* P, int64_t ldp, const double* b, int C, int m,
                               unsigned long long* flag, cudaStream_t st) {
  start_check_kernel<<<grid_for((int64_t)C * m), 256, 0, st>>>(P, ldp, b, C, m, flag);
  return cudaGetLastError();
}
// Dynamic-range guard of the int8 projection (options.projection = 0): per row of A',
// ratio_i = (stated int8 bound at S = 7) / (FP64 DMMA bound at the expected |nu|)
//         = 2^(e_i + 4) d 8 2^-54 / (2 d 2^-53 sqrt(2 / pi) ||a_i||_1),
// max_j |a_ij| < 2^e_i; the maximum over rows lands in *out (as ordered bits).
__global__ void oz_guard_kernel(const double* __restrict__ At, int m, int d, int64_t d_pad,
                                unsigned long long* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= m) return;
  double mx = 0.0, l1 = 0.0;
  for (int k = lane; k < d; k += 32) {
    const double v = fabs(At[tiled_offset(warp, k, d_pad)]);
    mx = fmax(mx, v);
    l1 += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  if (lane == 0 && mx > 0.0) {
    int e = 0;
    frexp(mx, &e);
    const double ratio = scalbn(1.0, e + 4) * 8.0 * 0.5 / (0.7978845608028654 * l1);  // 2^-54 / 2^-53 = 1/2
    atomicMax(out, (unsigned long long)__double_as_longlong(ratio));
  }
}

cudaError_t launch_oz_guard(const double* At, int m, int d, int64_t d_pad, unsigned long long* out,
                            cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  oz_guard_kernel<<<(unsigned)(((int64_t)m * 32 + 255) / 256), 256, 0, st>>>(At, m, d, d_pad, out);
  return cudaGetLastError();
}

cudaError_t launch_chain_sum(const double* S, int C, int d, int64_t d_pad, double* out,
                             double* part, cudaStream_t st) {
  int nparts = (C + kSumChunk - 1) / kSumChunk;
  chain_sum_part_kernel<<<dim3((d + 127) / 128, nparts), 128, 0, st>>>(S, C, d, d_pad, part);
  chain_sum_final_kernel<<<(d + 127) / 128, 128, 0, st>>>(part, nparts, d, out);
  return cudaGetLastError();
}
cudaError_t launch_accum_affine(const double* Xrow, int64_t ldx, const double* mu, int C, int d,
                                double* S1row, double* S2row, cudaStream_t st) {
  accum_affine_kernel<<<grid_for((int64_t)C * d), 256, 0, st>>>(Xrow, ldx, mu, C, d, S1row, S2row);
  return cudaGetLastError();
}
cudaError_t launch_add_vec_rows(double* Xrow, int64_t ldx, const double* mu, int C, int d,
                                cudaStream_t st) {
  add_vec_rows_kernel<<<grid_for((int64_t)C * d), 256, 0, st>>>(Xrow, ldx, mu, C, d);
  return cudaGetLastError();
}
cudaError_t launch_trsv_rows(const double* Xrow, const double* mu, const double* L, int C, int d,
                             double* Urow, cudaStream_t st) {
  int g = C < 148 * 8 ? C : 148 * 8;
  trsv_rows_kernel<<<g, 128, 0, st>>>(Xrow, mu, L, C, d, Urow);
  return cudaGetLastError();
}
cudaError_t launch_gather_rows_tiled(const double* Xt, int64_t d_pad, int d, const int64_t* rows,
                                     int n, double* out, cudaStream_t st) {
  if ((int64_t)n * d == 0) return cudaSuccess;
  gather_rows_kernel<<<grid_for((int64_t)n * d), 256, 0, st>>>(Xt, d_pad, d, rows, n, out);
  return cudaGetLastError();
}
cudaError_t launch_sum_i64(const int64_t* v, int n, int64_t* out, cudaStream_t st) {
  sum_i64_kernel<<<1, 1024, 0, st>>>(v, n, out);
  return cudaGetLastError();
}
cudaError_t launch_set_u32(uint32_t* dst, uint32_t value, cudaStream_t st) {
  set_u32_kernel<<<1, 1, 0, st>>>(dst, value);
  return cudaGetLastError();
}
cudaError_t launch_gemv_shift(const double* A, const double* b, const double* mu, int m, int d,
                              double* out, cudaStream_t st) {
  gemv_shift_kernel<<<(m + 7) / 8, 256, 0, st>>>(A, b, mu, m, d, out);
  return cudaGetLastError();
}
cudaError_t launch_test_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out,
                               bool curand, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  test_philox_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(ctr, key, n, out, curand ? 1 : 0);
  return cudaGetLastError();
}
cudaError_t launch_test_normals(uint64_t seed, uint32_t t, uint32_t c0, int C, int d, double* nu,
                                double* u, cudaStream_t st) {
  int64_t n = (int64_t)C * ((d + 1) / 2);
  if (n == 0) return cudaSuccess;
  test_normals_kernel<<<grid_for(n), 256, 0, st>>>(seed, t, c0, C, d, nu, u);
  return cudaGetLastError();
}
cudaError_t launch_test_arcs(const double* p, const double* q, const double* b, int64_t n,
                             double* alpha, double* beta, uint8_t* active, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  test_arcs_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(p, q, b, n, alpha, beta, active);
  return cudaGetLastError();
}

}  // namespace tmvn
