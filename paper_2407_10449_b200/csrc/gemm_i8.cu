// gemm_i8.cu -- FP64-accurate projection Q = N A'^T on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM), by an Ozaki-style integer
// split (the "stated mixed-precision scheme"
// of north_star for the O(md) matvec of P:292-293).
//
// Scheme.  Every operand value v is scaled by a power of two 2^e into (-1, 1)
// (A': one exponent per constraint row, from the row's max |a|; nu: the fixed
// 2^4, since Box-Muller output satisfies |nu| <= sqrt(-2 ln 2^-53) < 8.58) and
// truncated to the two's-complement fixed-point integer X = trunc(v 2^(8S-1))
// (|X| < 2^(8S-1), error < 2^-(8S-1)).  X is cut into S byte digits
// X = d_1 2^(8(S-1)) + sum_{k>=2} d_k 2^(8(S-k)): d_1 signed (s8), d_k unsigned
// (u8).  Then
//     sum_j X^a_j X^nu_j = sum_{k,l} (sum_j d^a_{k,j} d^nu_{l,j}) 2^(8(2S-k-l)),
// and the products are grouped by diagonal D = k + l: one int32 TMEM accumulator
// per D = 2 .. S+1 collects every pair (k, l) on it (exact: |acc| < 2^31 for
// d <= 4096).  The S(S+1)/2 int8 MMAs per K step are exact; the pairs with
// k + l > S + 1 are dropped (weight <= 2^(-8S)).  The epilogue forms
//     q_i = 2^(e_i + e_nu - 14) * sum_{D} acc_D 2^(-8(D-2))
// by summing the diagonals exactly in two 64-bit integers (the low one < 2^47: its
// conversion is exact; the high one is exact below 2^53) and one FP64 FMA.  Error
// bound (stated in
// include/tmvn.h, tested in tests/test_gpu_ozaki.py):
//     |q - a.nu| <= 2^(e_i + e_nu) d (S + 1) 2^(2 - 8S) + 2^-51 |q|
// (per product: truncation of both operands < 2^(1 - (8S-1)); dropped diagonals
// D >= S + 2: < (S - 1) 2^(2 - 8S) per unit of d; the reconstruction's two
// roundings, <= 2^-52 |q|), i.e.
// FP64-class accuracy relative to max_j |a_ij| * 2^e_nu * d, independent
// of C; the result is a deterministic function of (A', nu) (no split-K, fixed
// reconstruction order), so chains are bitwise independent of the sharding.
//
// Kernel.  Persistent, one 448-thread CTA per SM (TMEM: all 512 columns).
// Output tile: 128 constraints (MMA M, TMEM lanes) x 64 chains (MMA N); the
// S accumulators take S x 64 TMEM columns.  K steps of 32 bytes: one stage =
// S A' digit slices (S x 4 KB) + S nu digit slices (S x 2 KB), each a single
// contiguous cp.async.bulk (the operands are stored pre-tiled in the UMMA
// canonical K-major SWIZZLE_NONE layout by the slicing kernels below and by the
// fused per-chain kernel, which writes nu's digits as it draws nu).
//   warp 0 lane 0: producer (bulk copies into a kStages ring, mbarrier tx)
//   warp 1:        MMA issuer (elect.sync; S(S+1)/2 tcgen05.mma per stage,
//                  tcgen05.commit frees the ring slot; after the tile, commits
//                  to tmem_full)
//   warps 2-5:     A loaders (digit slices 0-3 of each stage into TMEM,
//                  tcgen05.st, double-buffered)
//   warps 6-13:    epilogue (tcgen05.ld 32x32b, integer + FP64 reconstruction, coalesced stores
//                  of Q[chain][constraint]), then arrive on tmem_empty;
//                  with options.fuse_arcs also the arcs of eq:roots.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace tmvn {

namespace {

constexpr int kOzBM = 128;        // constraints per tile (MMA M, TMEM lanes)
constexpr int kOzBN = kOzNuRows;  // chains per tile (MMA N)
constexpr int kOzBK = kOzStepK;   // K bytes per stage (one MMA K step for kind::i8)
constexpr int kASlice = kOzBM * kOzBK;  // 4096 bytes
constexpr int kNSlice = kOzBN * kOzBK;  // 2048 bytes
// 8 epilogue warps (two per TMEM lane quadrant, 32 columns each): the MMA warp waits
// less for the accumulators to drain (measured +1 % per iteration at config 3 over 4
// warps, which had left registers for the RNG kernel of options.rng_ahead beside it)
#ifndef TMVN_OZ_EPI
#define TMVN_OZ_EPI 8
#endif
constexpr int kOzEpiWarps = TMVN_OZ_EPI;
#ifndef TMVN_OZ_LOADERS
#define TMVN_OZ_LOADERS 4
#endif
constexpr int kOzLoadWarps = TMVN_OZ_LOADERS;  // 4, or 8 (a second set after the epilogue warps)
constexpr int kOzThreads = 32 * (2 + kOzLoadWarps + kOzEpiWarps);  // producer, MMA, loaders, epilogue
__host__ __device__ constexpr int oz_stage_bytes(int S) { return S * (kASlice + kNSlice); }
int g_oz_launch_seq = 0;  // host-side launch counter (timeline builds label launches with it)
// ring depth: as many stages as fit in 226 KB of shared memory (S = 6: 6, 7: 5, 8: 4)
#ifndef TMVN_OZ_MAX_STAGES
#define TMVN_OZ_MAX_STAGES 6
#endif
__host__ __device__ constexpr int oz_stages(int S) {
  return (226 * 1024) / oz_stage_bytes(S) > TMVN_OZ_MAX_STAGES ? TMVN_OZ_MAX_STAGES
                                                                 : (226 * 1024) / oz_stage_bytes(S);
}

// 2^(-8 k), k = 0 .. 4 (epilogue reconstruction)
__device__ constexpr double kOzInvPow2[5] = {1.0, 0.00390625, 1.52587890625e-05, 5.9604644775390625e-08,
                                             2.3283064365386962890625e-10};

// ---- tcgen05 / mbarrier wrappers -------------------------------------------
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// shared-memory matrix descriptor: K-major, no swizzle; lbo = byte stride between
// the two 16-byte K chunks, sbo = byte stride between 8-row core-matrix groups
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  return d;
}
// instruction descriptor of kind::i8: D = s32, A/B signedness, K-major, N, M
__host__ __device__ constexpr uint32_t idesc_i8(bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         ((uint32_t)(kOzBN >> 3) << 17) | ((uint32_t)(kOzBM >> 4) << 24);
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// All S(S+1)/2 digit-pair MMAs of one K step: A' digit i x nu digit j into the
// accumulator of diagonal i + j (TMEM columns (i + j) * 64; the allocation of all
// 512 columns starts at column 0).  Every operand is a compile-time constant or a
// warp-uniform value, so the issue is a plain sequence of UTCIMMA (elect.sync, no
// waterfall loop).  FIRST: the first K step of a tile, where pair (0, j)
// initialises accumulator j.
//
// A from TMEM (TS) or shared memory (SS).  tools/tc_rate.cu on the B200: an
// M=128 N=64 int8 MMA takes 48 cycles with both operands in shared memory (6 KB
// of operand reads at 128 B/cycle) and 32 cycles with A in TMEM (the tensor-core
// floor); tcgen05.cp into TMEM runs on the MMA pipe (7 copies of 4 KB: 448
// cycles, mostly serialised with the MMAs).  So the first NTS digit slices of a
// K step are written into TMEM by four loader warps (ld.shared + tcgen05.st, off
// the MMA pipe) into one of two buffers, and their MMAs read A there; the last
// slices, which feed only 1-3 MMAs, stay SS.  TMEM: S x 64 accumulator columns +
// 2 x NTS x 8 A columns <= 512 (S = 7: NTS = 4, all 512 columns).
template <int S>
__host__ __device__ constexpr int oz_nts() {
  return (512 - S * 64) / 16 < S - 2 ? (512 - S * 64) / 16 : S - 2;
}
template <int S>
__host__ __device__ constexpr uint32_t oz_acol(int buf, int i) {
  return (uint32_t)(S * 64 + buf * oz_nts<S>() * 8 + 8 * i);
}

template <int I, int J, int S, bool FIRST>
struct PairMma {
  static __device__ __forceinline__ void run(uint64_t da, uint64_t dn, uint32_t abuf) {
    constexpr uint32_t idesc = idesc_i8(I == 0, J == 0);
    constexpr uint32_t acc = (FIRST && I == 0) ? 0u : 1u;
    if constexpr (I < oz_nts<S>()) {
      asm volatile(
          "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
          " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"((uint32_t)((I + J) * kOzBN)),
          "r"(abuf + 8 * I), "l"(dn + (uint64_t)((J * kNSlice) >> 4)), "n"(idesc), "n"(acc));
    } else {
      asm volatile(
          "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
          " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"((uint32_t)((I + J) * kOzBN)),
          "l"(da + (uint64_t)((I * kASlice) >> 4)), "l"(dn + (uint64_t)((J * kNSlice) >> 4)), "n"(idesc),
          "n"(acc));
    }
    if constexpr (J + 1 < S - I) PairMma<I, J + 1, S, FIRST>::run(da, dn, abuf);
    else if constexpr (I + 1 < S) PairMma<I + 1, 0, S, FIRST>::run(da, dn, abuf);
  }
};
template <int S, bool FIRST>
__device__ __forceinline__ void issue_stage(uint64_t da, uint64_t dn, uint32_t abuf) {
  PairMma<0, 0, S, FIRST>::run(da, dn, abuf);
}

// Tile order: bands of kOzBand chain blocks; inside a band the chain block varies
// fastest, so each A' digit block is read once per band (from L2 for the band's
// other chain blocks) and the band's nu blocks stay in L2 across the constraint
// blocks.  With A' digits larger than L2 (config 5: 470 MB) the plain
// constraint-fastest order streamed them once per chain block.  Results do not
// depend on the order (every tile sums its whole K range).
// band of 16 chain blocks (1024 chains): B200, config 5 136.4 vs 137.7 ms per
// iteration with 8 (32: 137.6); config 3 unchanged
#ifndef TMVN_OZ_BAND
#define TMVN_OZ_BAND 16
#endif
__device__ __forceinline__ void oz_tile(int tile, int MB, int NBt, int& mb, int& nb) {
  constexpr int GN = TMVN_OZ_BAND;
  const int band = tile / (MB * GN);
  const int nb0 = band * GN;
  const int gn = NBt - nb0 < GN ? NBt - nb0 : GN;
  const int r = tile - band * MB * GN;
  mb = r / gn;
  nb = nb0 + r % gn;
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint4& a, const uint4& b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

// Role timing (timing build -DTMVN_PHASE_TIMING only; tools/oz_timing.py):
// [0] MMA wait full, [1] MMA wait tmem_empty, [2] MMA issue, [3] epilogue wait
// tmem_full, [4] epilogue work, [5] producer wait empty, [6] tiles, [7] CTA cycles,
// [8] MMA wait for the A loaders (included in [0]), [9] A loaders wait for the MMAs
// to release a TMEM A buffer
#ifdef TMVN_PHASE_TIMING
__device__ unsigned long long g_oz_cycles[10];
#define OZT(var) const long long var = clock64()
#define OZADD(i, v) atomicAdd(&g_oz_cycles[i], (unsigned long long)(v))
#else
#define OZT(var)
#define OZADD(i, v)
#endif

// warps: 0 producer, 1 MMA issuer, 2-5 A loaders, 6.. epilogue (warp w may access
// TMEM lanes 32 (w % 4) .. 32 (w % 4) + 31 only: each role covers the 4 quadrants)
// STAGES: ring depth (0 = as many as fit; 3 = the compact variant that leaves room
// on the SM for a CTA of the per-chain kernel when the two run concurrently)
// nu_{t+1} drawn by the epilogue warps between tiles (options.rng_gemm): blocks of 256
// coordinate pairs of the chains b, b + grid, ... of this CTA, a share after each tile
// (the warps are otherwise waiting for the next tile's accumulators) and the rest at
// the end.  Same device function and counters as everywhere (C12): bitwise the same nu.
__device__ __forceinline__ void oz_rng_blocks(const OzRng& r, uint32_t t_gen, int et, int64_t& chain, int& pk0,
                                              int nblk) {
  const int kpairs = (int)(r.d_pad / 2);
  for (int i = 0; i < nblk && chain < r.C; ++i) {
    const int pk = pk0 + et;
    if (pk < kpairs) {
      const int k = 2 * pk;
      const double2 nv = normal_pair_at(r.seed, t_gen, r.chain_offset + (uint32_t)chain, k, r.d);
      *reinterpret_cast<double2*>(r.N + tiled_row(chain, r.d_pad) + tiled_col(k)) = nv;
      oz_put_nu_pair_s(r.Ns + oz_row(chain, r.S, r.KB, kOzNuRows) + oz_col(k, r.S, kOzNuRows), nv.x, nv.y, r.S);
    }
    pk0 += 32 * kOzEpiWarps;
    if (pk0 >= kpairs) {
      pk0 = 0;
      chain += gridDim.x;
    }
  }
}

template <int S, int STAGES, bool CS, bool ARCS, bool RNG>
__global__ void __launch_bounds__(kOzThreads, 1)
    ozaki_gemm_kernel(const int8_t* __restrict__ As, const int8_t* __restrict__ Ns,
                      const double* __restrict__ rowscale, const double* __restrict__ colscale,
                      double* __restrict__ Q, int64_t ldq, int MB, int NBt, int KB, int dbg_seq,
                      const OzArcs arc, const OzRng rng) {
  constexpr int kStage = oz_stage_bytes(S);
  constexpr int kOzStages = STAGES ? STAGES : oz_stages(S);
  constexpr int NTS = oz_nts<S>();
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzStages * kStage);
  uint64_t* empty = full + kOzStages;
  uint64_t* tfull = empty + kOzStages;
  uint64_t* tempty = tfull + 1;
  uint64_t* afull = tempty + 1;   // [2]: A buffer written (4 loader warps)
  uint64_t* aempty = afull + 2;   // [2]: the MMAs reading an A buffer completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kOzEpiWarps);  // one arrive per epilogue warp
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], kOzLoadWarps);
      mbar_init(&aempty[b], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0) __trap();  // all 512 columns: the allocation starts at lane 0, column 0
  const int tiles = MB * NBt;
#ifdef TMVN_TIMELINE
  const unsigned int tl_slot = (unsigned)dbg_seq & 255;  // host launch sequence number
  if (threadIdx.x == 0) atomicMin(&g_tl[tl_slot][0], tl_now());
#else
  (void)dbg_seq;
#endif
  OZT(t_start);
#ifdef TMVN_PHASE_TIMING
  long long acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#endif

  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int mb, nb;
        oz_tile(tile, MB, NBt, mb, nb);
        const int8_t* ga = As + (size_t)mb * KB * S * kASlice;
        const int8_t* gn = Ns + (size_t)nb * KB * S * kNSlice;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kOzStages;
          OZT(w0);
          if (it >= kOzStages) mbar_wait(&empty[s], ((it / kOzStages) - 1) & 1);
          OZT(w1);
#ifdef TMVN_PHASE_TIMING
          acc0 += w1 - w0;
#endif
          unsigned char* st = ring + s * kStage;
          mbar_expect_tx(&full[s], kStage);
          bulk_g2s(st, ga + (size_t)kb * S * kASlice, S * kASlice, &full[s]);
          bulk_g2s(st + S * kASlice, gn + (size_t)kb * S * kNSlice, S * kNSlice, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer: the whole warp runs the loop, one elected lane issues
      // descriptors of stage 0; a stage / slice offset is a constant add to the
      // 14-bit address field (ring < 256 KB: no carry)
      const uint64_t dA0 = umma_desc(smem_u32(ring), (kOzBM / 8) * 128, 128);
      const uint64_t dN0 = umma_desc(smem_u32(ring) + S * kASlice, (kOzBN / 8) * 128, 128);
      uint32_t it = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
        OZT(e0);
        if (tcount > 0) {
          mbar_wait(tempty, (tcount - 1) & 1);
          tc_fence_after();
        }
        OZT(e1);
#ifdef TMVN_PHASE_TIMING
        acc1 += e1 - e0;
#endif
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kOzStages;
          const int b = it & 1;
          OZT(f0);
          mbar_wait(&full[s], (it / kOzStages) & 1);
          OZT(fa);
          if (NTS > 0) mbar_wait(&afull[b], (it >> 1) & 1);
          tc_fence_after();
          OZT(f1);
#ifdef TMVN_PHASE_TIMING
          acc0 += f1 - f0;
          acc3 += f1 - fa;
#endif
          const uint64_t so = (uint64_t)((s * kStage) >> 4);
          const uint32_t abuf = b ? oz_acol<S>(1, 0) : oz_acol<S>(0, 0);
          if (kb == 0) issue_stage<S, true>(dA0 + so, dN0 + so, abuf);
          else issue_stage<S, false>(dA0 + so, dN0 + so, abuf);
          if (lane == 0) {
            umma_commit(&empty[s]);  // ring slot free once these MMAs have read it
            if (NTS > 0) umma_commit(&aempty[b]);
          }
          __syncwarp();
#ifdef TMVN_PHASE_TIMING
          acc2 += clock64() - f1;
#endif
        }
        if (lane == 0) umma_commit(tfull);  // accumulators of this tile complete
        __syncwarp();
      }
    }
  } else if (warp < 6 || warp >= 6 + kOzEpiWarps) {  // ---- A loaders: row 32 (warp % 4) + lane
    if (NTS > 0) {                                    // of each TS slice into TMEM
      const int quad = warp & 3;
      const int li = warp < 6 ? warp - 2 : 4 + warp - (6 + kOzEpiWarps);
      const int i0 = kOzLoadWarps == 8 ? (li >> 2) : 0, istep = kOzLoadWarps == 8 ? 2 : 1;
      const int row = quad * 32 + lane;
      const uint32_t roff = (uint32_t)((row / 8) * 128 + (row % 8) * 16);
      const uint32_t lanebase = (uint32_t)(quad * 32) << 16;
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kOzStages;
          const int b = it & 1;
          mbar_wait(&full[s], (it / kOzStages) & 1);
          OZT(la);
          if (it >= 2) mbar_wait(&aempty[b], ((it >> 1) - 1) & 1);
#ifdef TMVN_PHASE_TIMING
          acc3 += clock64() - la;
#endif
          tc_fence_after();
          const unsigned char* st = ring + s * kStage + roff;
#pragma unroll
          for (int i = i0; i < NTS; i += istep) {
            const uint4 lo = *reinterpret_cast<const uint4*>(st + i * kASlice);
            const uint4 hi = *reinterpret_cast<const uint4*>(st + i * kASlice + (kOzBM / 8) * 128);
            tmem_st8(tmem + lanebase + (b ? oz_acol<S>(1, i) : oz_acol<S>(0, i)), lo, hi);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&afull[b]);
        }
      }
    }
  } else {  // ---- epilogue: warps 6.. (with 8 warps: 6-9 columns 0-31, 10-13 columns 32-63)
    const int quad = warp & 3;
    const int c0 = ((warp - 6) / 4) * (kOzBN * 4 / kOzEpiWarps);
    const int row_in_tile = quad * 32 + lane;
    uint32_t tcount = 0;
    // RNG share per tile: this CTA's blocks of pairs spread over its tiles
    const int et = threadIdx.x - 32 * 6;
    int64_t rchain = blockIdx.x;
    int rpk0 = 0;
    int rshare = 0;
    uint32_t t_gen = 0;
    if (RNG) {
      t_gen = (rng.t_dev ? *rng.t_dev : 0u) + rng.t + 1u;
      const int nblk_chain = (int)((rng.d_pad / 2 + 32 * kOzEpiWarps - 1) / (32 * kOzEpiWarps));
      const int64_t nch = blockIdx.x < rng.C ? (rng.C - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
      const int ntiles = (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
      rshare = (int)((nch * nblk_chain + ntiles - 1) / (ntiles > 0 ? ntiles : 1));
    }
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
      int mb, nb;
      oz_tile(tile, MB, NBt, mb, nb);
      const int64_t row = (int64_t)mb * kOzBM + row_in_tile;
      const double scale = __ldg(rowscale + row);
      OZT(g0);
      mbar_wait(tfull, tcount & 1);
      tc_fence_after();
      OZT(g1);
#ifdef TMVN_PHASE_TIMING
      acc0 += g1 - g0;
#endif
      double* qcol = Q + (int64_t)nb * kOzBN * ldq + row;
#pragma unroll 1
      for (int cc = c0; cc < c0 + kOzBN * 4 / kOzEpiWarps; cc += 8) {
        int32_t acc[S][8];
#pragma unroll
        for (int D = 0; D < S; ++D)
          tmem_ld8(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(D * kOzBN + cc), acc[D]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          // the diagonals combined exactly in two 64-bit integers (IMAD.WIDE), then two
          // conversions and one FMA (S int32 -> FP64 conversions per output cost 26 % more
          // epilogue cycles, tools/oz_timing.py): hi = sum_{D < H} acc_D 2^(8(H-1-D))
          // (|hi| < 2^55), lo = sum_{D >= H} acc_D 2^(8(S-1-D)),
          // h = (hi + lo 2^(-8(S-H))) 2^(-8(H-1))
          constexpr int H = (S + 1) / 2;
          long long hi = (long long)acc[H - 1][j], lo = (long long)acc[S - 1][j];
#pragma unroll
          for (int D = H - 2; D >= 0; --D) hi += (long long)acc[D][j] * (1ll << (8 * (H - 1 - D)));
#pragma unroll
          for (int D = S - 2; D >= H; --D) lo += (long long)acc[D][j] * (1ll << (8 * (S - 1 - D)));
          const double h = __fma_rn(__ll2double_rn(lo), kOzInvPow2[S - H], __ll2double_rn(hi));
          const double sc0 = scale * kOzInvPow2[H - 1];  // exact: powers of two
          // per-column power of two (refresh of P = X A'^T: 2^(e_c - 4) per chain), exact
          const double sc = CS ? __dmul_rn(sc0, __ldg(colscale + (int64_t)nb * kOzBN + cc + j)) : sc0;
          qcol[(int64_t)(cc + j) * ldq] = __dmul_rn(h, sc);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      // Fused arc construction (options.fuse_arcs; eq:roots P:922-934 with C1-C5): with the
      // accumulators released, while the MMAs of the next tile run, this thread's
      // constraint `row` is tested against each of its chains -- p from P = A x_t, q the
      // value just stored (re-read from L2, program order) -- and an active constraint's
      // arc is stored at its own index in the chain's row of `arcs`, the warp's ballot as
      // the activity mask of the 32 constraints (no atomics, no ordering: fire-and-forget)
      if (ARCS) {
        const bool rv = row < arc.m;
        const double bi = rv ? __ldg(arc.b + row) : 0.0;
#pragma unroll 1
        for (int cc = c0; cc < c0 + kOzBN * 4 / kOzEpiWarps; cc += 8) {
          double pv[8], qv[8];
          const int64_t ch0 = (int64_t)nb * kOzBN + cc;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            pv[j] = 0.0;
            qv[j] = 0.0;
            if (rv && ch0 + j < arc.C) {
              pv[j] = arc.P[(ch0 + j) * arc.ldp + row];
              qv[j] = qcol[(int64_t)(cc + j) * ldq];
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (ch0 + j >= arc.C) break;  // uniform: padded chains
            double al = 0.0, be = 0.0;
            const bool act = rv && arc_of(pv[j], qv[j], bi, al, be);
            const unsigned mask = __ballot_sync(0xffffffffu, act);
            if (act) arc.arcs[(ch0 + j) * arc.ald + row] = make_double2(al, be);
            if (lane == 0 && (row >> 5) < arc.mw) arc.amask[(ch0 + j) * arc.mw + (row >> 5)] = mask;
          }
        }
      }
      if (RNG) oz_rng_blocks(rng, t_gen, et, rchain, rpk0, rshare);
#ifdef TMVN_PHASE_TIMING
      acc1 += clock64() - g1;
#endif
    }
    if (RNG) oz_rng_blocks(rng, t_gen, et, rchain, rpk0, 1 << 30);  // the rest
  }
#ifdef TMVN_PHASE_TIMING
  if (lane == 0) {
    if (warp == 0) OZADD(5, acc0);
    if (warp == 1) { OZADD(0, acc0); OZADD(1, acc1); OZADD(2, acc2); OZADD(8, acc3); }
    if (warp == 2) OZADD(9, acc3);
    if (warp == 6) { OZADD(3, acc0); OZADD(4, acc1); }
    if (threadIdx.x == 0) OZADD(7, clock64() - t_start);
  }
  if (threadIdx.x == 64) {
    int nt = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) ++nt;
    OZADD(6, nt);
  }
#endif
  __syncthreads();
#ifdef TMVN_TIMELINE
  if (threadIdx.x == 0) atomicMax(&g_tl[tl_slot][1], tl_now());
#endif
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}


// ---- digit slicing ----------------------------------------------------------
// One warp per row of a fragment-tiled FP64 matrix (R rows, d columns):
// per_row != 0: e_r = exponent of the row's max |v| (v_max < 2^e_r), rowscale[r] =
// 2^(e_r + e_other - 14); else e_r = e_fixed for every row.  Writes all S digits
// of every (r, k < KB*32) (zeros beyond d).
__global__ void oz_slice_kernel(const double* __restrict__ src, int R, int d, int64_t d_pad, int S,
                                int KB, int BR, int per_row, int e_fixed, int e_other,
                                int8_t* __restrict__ dst, double* __restrict__ rowscale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const int64_t r = warp;
  int e = e_fixed;
  if (per_row) {
    double mx = 0.0;
    for (int k = lane; k < d; k += 32) mx = fmax(mx, fabs(src[tiled_offset(r, k, d_pad)]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): mx < 2^e
    if (lane == 0) rowscale[r] = scalbn(1.0, e + e_other - 14);
  }
  const int K = KB * kOzBK;
  for (int k = lane; k < K; k += 32) {
    const int64_t X = k < d ? oz_fixed(src[tiled_offset(r, k, d_pad)], S, e) : 0;
    for (int s = 0; s < S; ++s) dst[oz_offset(r, k, s, S, KB, BR)] = (int8_t)(uint8_t)oz_digit(X, s, S);
  }
}

}  // namespace

#ifdef TMVN_PHASE_TIMING
void oz_cycles(unsigned long long* out10, bool reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out10, g_oz_cycles, sizeof(unsigned long long) * 10);
  if (reset) {
    unsigned long long z[10] = {0};
    cudaMemcpyToSymbol(g_oz_cycles, z, sizeof(z));
  }
}
#endif

size_t ozaki_smem_bytes(int S, int stages) {
  return (size_t)(stages ? stages : oz_stages(S)) * oz_stage_bytes(S) + 256;
}

cudaError_t launch_oz_slice(const double* src_tiled, int64_t R, int64_t d, int64_t d_pad, int S,
                            int64_t KB, int BR, int per_row, int e_fixed, int e_other, int8_t* dst,
                            double* rowscale, cudaStream_t st) {
  if (R <= 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (R * 32 + threads - 1) / threads;
  oz_slice_kernel<<<(unsigned)blocks, threads, 0, st>>>(src_tiled, (int)R, (int)d, d_pad, S, (int)KB,
                                                         BR, per_row, e_fixed, e_other, dst, rowscale);
  return cudaGetLastError();
}

template <int S, int STAGES, bool CS, bool ARCS, bool RNG = false>
static cudaError_t launch_oz_t(const int8_t* As, int64_t M_pad, const int8_t* Ns, int64_t N_pad,
                               int64_t KB, const double* rowscale, const double* colscale, double* Q,
                               int64_t ldq, cudaStream_t st, const OzArcs& arc, const OzRng& rng = OzRng{}) {
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = ozaki_smem_bytes(S, STAGES);
  cudaError_t e = cudaFuncSetAttribute(ozaki_gemm_kernel<S, STAGES, CS, ARCS, RNG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int MB = (int)(M_pad / kOzBM), NBt = (int)(N_pad / kOzBN);
  const int tiles = MB * NBt;
  const int grid = tiles < num_sms ? tiles : num_sms;
  ozaki_gemm_kernel<S, STAGES, CS, ARCS, RNG><<<grid, kOzThreads, smem, st>>>(
      As, Ns, rowscale, colscale, Q, ldq, MB, NBt, (int)KB, g_oz_launch_seq++, arc, rng);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_gemm(const int8_t* As, int64_t M_pad, const int8_t* Ns, int64_t N_pad,
                              int64_t KB, int S, const double* rowscale, double* Q, int64_t ldq,
                              cudaStream_t st, bool compact, const double* colscale, const OzArcs* arcs,
                              const OzRng* rng) {
  if (M_pad % kOzBM || N_pad % kOzBN || KB < 1) return cudaErrorInvalidValue;
  if ((arcs || rng) && (colscale || compact)) return cudaErrorInvalidValue;
  if (arcs && rng) return cudaErrorInvalidValue;
  const OzArcs none{};
  if (rng) {
    switch (S) {
      case 4: return launch_oz_t<4, 0, false, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, none, *rng);
      case 6: return launch_oz_t<6, 0, false, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, none, *rng);
      case 7: return launch_oz_t<7, 0, false, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, none, *rng);
      case 8: return launch_oz_t<8, 0, false, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, none, *rng);
      default: return cudaErrorInvalidValue;
    }
  }
  if (arcs) {
    switch (S) {
      case 4: return launch_oz_t<4, 0, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, *arcs);
      case 6: return launch_oz_t<6, 0, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, *arcs);
      case 7: return launch_oz_t<7, 0, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, *arcs);
      case 8: return launch_oz_t<8, 0, false, true>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, *arcs);
      default: return cudaErrorInvalidValue;
    }
  }
#define TMVN_OZ_CASE(SS, ST)                                                                  \
  case SS:                                                                                    \
    return colscale ? launch_oz_t<SS, ST, true, false>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, none) \
                    : launch_oz_t<SS, ST, false, false>(As, M_pad, Ns, N_pad, KB, rowscale, colscale, Q, ldq, st, none);
  if (compact) {
    switch (S) {
      TMVN_OZ_CASE(4, 3)
      TMVN_OZ_CASE(6, 3)
      TMVN_OZ_CASE(7, 3)
      TMVN_OZ_CASE(8, 3)
      default: return cudaErrorInvalidValue;
    }
  }
  switch (S) {
    TMVN_OZ_CASE(4, 0)
    TMVN_OZ_CASE(6, 0)
    TMVN_OZ_CASE(7, 0)
    TMVN_OZ_CASE(8, 0)
    default: return cudaErrorInvalidValue;
  }
#undef TMVN_OZ_CASE
}


#ifdef TMVN_TIMELINE
void tl_access_gemm(unsigned long long* out, bool reset) {
  cudaDeviceSynchronize();
  if (reset) {
    g_oz_launch_seq = 0;
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
