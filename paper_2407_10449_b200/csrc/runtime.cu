// runtime.cu -- host runtime behind the C ABI of include/tmvn.h: the handle,
// device buffers, the per-iteration launch sequence of Alg. 1 and the test hooks.
//
// Per iteration t (all on one stream, two launches in steady state):
//   GEMM  Q = N A^T                                    (gemm_f64.cu)
//   ESS   arcs -> I_act -> theta -> P', x, moments, nu_{t+1}   (ess_chain.cu)
//   every recompute_every iterations: GEMM P = X A^T  (C13)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include <nvtx3/nvToolsExt.h>

#include "../../include/tmvn.h"
#include "common.cuh"
#include "internal.h"

using namespace tmvn;

namespace {

thread_local std::string g_create_error;

// NVTX range (header-only NVTX v3: a no-op unless a tool such as nsys / ncu is attached)
// around each host-side stage of the call and each hot-loop launch, named by SURVEY 8(a) row
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct tmvn_ctx {
  int device = 0;
  int64_t m = 0, d = 0, m_pad = 0, d_pad = 0, d_r128 = 0;
  // constraints
  double* A_row = nullptr;  // m x d (original)
  double* A_pad = nullptr;  // m x d_pad, zero-padded rows (latency mode; made on first use)
  float* A32 = nullptr;     // FP32 copies for options.precision = 1 (made on first use)
  float* b32 = nullptr;
  double* b_orig = nullptr; // m
  double* A_tiled = nullptr;  // tiled m_pad x d_pad of the ORIGINAL A (for A L)
  double* At = nullptr;     // tiled m_pad x d_pad of A' (= A L if affine)
  double* b_eff = nullptr;  // m, b' = b - A mu
  // affine (App. A)
  bool affine = false;
  double* mu = nullptr;      // d
  double* L = nullptr;       // d x d row-major
  double* L_tiled = nullptr; // rows j = L[j, :], tiled d_r128 x d_pad  (x = U L^T)
  // chains
  int64_t C_cap = 0, C_pad = 0;
  double *X = nullptr, *N = nullptr, *P0 = nullptr, *P1 = nullptr, *Q = nullptr;
  double* N2 = nullptr;  // second nu buffer: nu_t lives in buffer t & 1 when the RNG runs ahead
  // pipelined schedule (options.pipeline): nu_t in buffer t % 3, Q_t in buffer t & 1
  double* N3 = nullptr;
  int8_t* Ns3 = nullptr;
  double* Q2 = nullptr;
  // int8 refresh of P = X A'^T: digits of X (C_pad rows) and 2^(e_c - 4) per chain
  int8_t* Xs = nullptr;
  double* xscale = nullptr;
  // fused arcs (options.fuse_arcs): per-chain arc lists written by the projection's epilogue
  double2* arcs = nullptr;  // C_pad x m_pad
  uint32_t* amask = nullptr;  // C_pad x mw activity bits
  int64_t arcs_rows = 0;
  cudaStream_t gemm_stream = nullptr;
  cudaEvent_t ev_q[2] = {nullptr, nullptr}, ev_nu[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_ess = nullptr, ev_join[2] = {nullptr, nullptr}, ev_essb = nullptr;
  cudaStream_t essb_stream = nullptr;  // the second part of a split per-chain launch
  // the RNG stream: nu_{t+1} is drawn beside the projection GEMM of iteration t
  cudaStream_t rng_stream = nullptr;
  int* dyn = nullptr;  // dynamic chain scheduling counters: 64 slots per shard
  int* gmode = nullptr;  // level-1 bucket switch state: 4 ints per shard (EssParams.gmode)
  cudaEvent_t ev_pre = nullptr, ev_rng = nullptr;
  double *S1 = nullptr, *S2 = nullptr;       // tiled moments (u-space == x-space w/o affine)
  double *S1x = nullptr, *S2x = nullptr;     // row-major x-space moments (affine)
  double *stage = nullptr, *stage2 = nullptr;  // row-major C_pad x max(d_pad, d_r128)
  int64_t* rej = nullptr;
  double* Xsnap = nullptr;  // X before a latency-mode call (its overflow fallback)
  size_t Xsnap_n = 0;
  int lat_cap_max = 0;  // test hook: latency-mode live-arc capacity cap (0 = automatic)
  int lat_grid_mode = 0;  // test hook: 0 automatic, 1 grid mode whenever it fits, -1 never
  unsigned char* lat_gscratch = nullptr;  // grid-mode exchange scratch
  size_t lat_gscratch_n = 0;
  // constraint-parallel iterations (tmvn_cp_*): chains, seed, first iteration, scratch
  int64_t cp_C = 0, cp_t0 = 0;
  uint64_t cp_seed = 0;
  int64_t cp_nrec = 0;
  double* cp_tl = nullptr;  // 2 C_pad: theta, L per chain
  double2* cp_arcs = nullptr;  // C_pad x m_pad: this iteration's arcs ((-1, -1): inactive)
  unsigned char* cp_cur = nullptr;  // C_pad: which of P0 / P1 holds each chain's P
  int64_t cp_rows = 0;              // chains the scratch above is sized for
  int64_t lat_memo_C = -1;  // latency_cluster_size's answer for this C (m, d fixed per handle)
  int lat_memo_fp32 = -1, lat_memo_cs = 0, lat_memo_cap = 0;
  int64_t* dsum = nullptr;
  double* msum = nullptr;  // 2 d (device) moment reduction targets (sum, sum of squares)
  // pinned host landing area for the small per-call reads (flags, counters, the two
  // moment vectors): async copies to pageable memory would stage through the driver
  double* pin = nullptr;    // 8 + 2 d doubles
  unsigned long long* dflag = nullptr;
  double2 *gstash = nullptr, *ggaps = nullptr;
  int64_t scratch_groups = 0;  // chain groups the scratch is sized for
  bool scratch_stash = false;  // gstash / gnext allocated
  // int8 Ozaki projection (options.projection = 1, gemm_i8.cu)
  int8_t* As = nullptr;       // digits of A' (m_pad rows), valid for ozS_A digits (0 = stale)
  double* rowscale = nullptr; // m_pad
  int ozS_A = 0;
  double oz_ratio = 0.0;  // dynamic-range guard: max_i int8 bound / FP64 bound (use_oz)
  int8_t* Ns = nullptr;       // digits of nu (C_pad rows)
  int8_t* Ns2 = nullptr;      // second buffer (nu of odd iterations when the RNG runs ahead)
  int ozS_N = 0;
  int64_t Ns_rows = 0;
  int64_t ozKB = 0;
  EssLaunch plan{};
  int nshards = 1;                      // concurrent chain shards (streams)
  std::vector<cudaStream_t> shard_streams;
  cudaEvent_t fork_event = nullptr;
  std::vector<cudaEvent_t> join_events;
  // CUDA-graph replay of aligned blocks of recompute_every iterations
  cudaStream_t capture_stream = nullptr;
  uint32_t* d_tbase = nullptr;
  cudaGraphExec_t graph_exec[2] = {nullptr, nullptr};  // by P parity at block start
  std::vector<unsigned char> graph_sig[2];
  // state
  tmvn_options opt{};
  tmvn_stats stats{};
  std::vector<double> mom_sum, mom_sq;
  std::string err;
  // profiling (tmvn_get_profile)
  tmvn_profile prof{};
  std::vector<cudaEvent_t> events;
  // trace hook
  const int64_t* trace_rows = nullptr;
  int trace_n = 0;
  double* trace_dev = nullptr;
};

namespace {

tmvn_status fail(tmvn_ctx* h, tmvn_status s, const std::string& msg) {
  if (h) h->err = msg;
  else g_create_error = msg;
  return s;
}

tmvn_status cuda_fail(tmvn_ctx* h, cudaError_t e, const char* where) {
  std::string msg = std::string(where) + ": " + cudaGetErrorString(e);
  return fail(h, e == cudaErrorMemoryAllocation ? TMVN_E_OOM : TMVN_E_CUDA, msg);
}

#define CK(h, expr)                                          \
  do {                                                       \
    cudaError_t e_ = (expr);                                 \
    if (e_ != cudaSuccess) return cuda_fail((h), e_, #expr); \
  } while (0)

// a kernel launch of the library: checked and counted
#define KL(h, expr)          \
  do {                       \
    CK(h, expr);             \
    (h)->prof.launches += 1; \
  } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemset(*p, 0, count * sizeof(T));
}

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

std::vector<double> to_host(const double* p, size_t n) {
  std::vector<double> v(n);
  if (n) cudaMemcpy(v.data(), p, n * sizeof(double), cudaMemcpyDefault);
  return v;
}

cudaStream_t stream_of(const tmvn_ctx* h) { return (cudaStream_t)h->opt.stream; }

void free_arcs(tmvn_ctx* h) {
  dfree(h->arcs); dfree(h->amask);
  h->arcs_rows = 0;
}

void free_chain_buffers(tmvn_ctx* h) {
  free_arcs(h);
  dfree(h->X); dfree(h->N); dfree(h->N2); dfree(h->N3); dfree(h->P0); dfree(h->P1); dfree(h->Q);
  dfree(h->Q2); dfree(h->Ns3); dfree(h->Xs); dfree(h->xscale);
  dfree(h->S1); dfree(h->S2); dfree(h->S1x); dfree(h->S2x);
  dfree(h->stage); dfree(h->stage2); dfree(h->rej);
  dfree(h->gstash); dfree(h->ggaps);
  dfree(h->Ns); dfree(h->Ns2);
  h->Ns_rows = 0;
  h->ozS_N = 0;
  h->C_cap = h->C_pad = 0;
}

tmvn_status ensure_chains(tmvn_ctx* h, int64_t C) {
  if (C <= h->C_cap) return TMVN_OK;
  free_chain_buffers(h);
  const int64_t C_pad = round_up(C, kTileR);
  const size_t cd = (size_t)C_pad * h->d_pad, cm = (size_t)C_pad * h->m_pad;
  const size_t wide = (size_t)C_pad * std::max(h->d_pad, h->d_r128);
  CK(h, dalloc(&h->X, cd));
  CK(h, dalloc(&h->N, cd));
  CK(h, dalloc(&h->N2, cd));
  CK(h, dalloc(&h->P0, cm));
  CK(h, dalloc(&h->P1, cm));
  CK(h, dalloc(&h->Q, cm));
  CK(h, dalloc(&h->S1, cd));
  CK(h, dalloc(&h->S2, cd));
  CK(h, dalloc(&h->stage, wide));
  CK(h, dalloc(&h->stage2, wide));
  CK(h, dalloc(&h->rej, (size_t)C_pad));
  h->scratch_groups = 0;
  h->scratch_stash = false;
  h->C_cap = C;
  h->C_pad = C_pad;
  return TMVN_OK;
}

// Shards, launch plan of the fused kernel (per shard) and its per-group scratch.
tmvn_status plan_ess(tmvn_ctx* h, int64_t C) {
  int S = h->opt.streams;
  if (S <= 0) {
    // auto (measured on B200): chain shards as independent GEMM ->
    // per-chain sequences on concurrent streams fill each other's tails (the persistent
    // per-chain kernel's last round, the GEMM's last tiles) -- config 3 (4096 chains,
    // d = 1000) 0.381 -> 0.359 ms per iteration with 2 shards, config 4 (1024 chains,
    // m = 100000) 2.44 -> 1.98 ms with 4 -- unless the projection dominates and its A'
    // operand exceeds L2 (config 5, d = 4096: every shard re-streams 470 MB of digits,
    // 125 -> 145 ms with 2 shards)
    // (with 512-thread CTAs per chain for m >= 8192 and the streaming L2 prefetch, config 4
    // measured best at 2 shards: 1.396 ms per iteration vs 1.446 at 4, 1.578 at 1)
    S = 1;
    if (h->d <= 2048) {
      if (h->m >= 8192 && C >= 2 * 256) S = 2;
      else if (C >= 2 * 1024) S = 2;
    }
  }
  if (h->trace_dev) S = 1;
  const int64_t per = round_up((C + S - 1) / S, kTileR);
  S = (int)((C + per - 1) / per);
  h->nshards = S;
  while ((int)h->shard_streams.size() < S) {
    cudaStream_t s_;
    CK(h, cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    h->shard_streams.push_back(s_);
    cudaEvent_t e;
    CK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->join_events.push_back(e);
  }
  if (!h->fork_event) CK(h, cudaEventCreateWithFlags(&h->fork_event, cudaEventDisableTiming));
  h->plan = ess_plan((int)std::min(per, C), (int)h->m, h->opt.chain_warps, h->opt.ring);
  const bool need_stash = !h->plan.stash_smem;
  const int64_t G = h->plan.groups * S;
  if (G > h->scratch_groups || (need_stash && !h->scratch_stash)) {
    dfree(h->gstash); dfree(h->ggaps);
    const int64_t Gn = std::max(G, h->scratch_groups);
    if (need_stash || h->scratch_stash) {
      CK(h, dalloc(&h->gstash, (size_t)Gn * ess_gstash_stride(h->m)));
      h->scratch_stash = true;
    }
    CK(h, dalloc(&h->ggaps, (size_t)Gn * (h->m + 2)));
    h->scratch_groups = Gn;
  }
  return TMVN_OK;
}

tmvn_status ensure_affine_moments(tmvn_ctx* h) {
  if (h->S1x) return TMVN_OK;
  CK(h, dalloc(&h->S1x, (size_t)h->C_pad * h->d));
  CK(h, dalloc(&h->S2x, (size_t)h->C_pad * h->d));
  return TMVN_OK;
}

// Automatic projection (options.projection = 0): the int8 Ozaki split when d <= 4096 and
// its stated bound is within kOzGuard times the FP64 DMMA bound (at the expected |nu|) on
// every row of A' (rows with a wide dynamic range, where a row's
// max |a_ij| sets the int8 grid but its L1 norm sets the DMMA bound, take DMMA).
constexpr double kOzGuard = 16.0;
bool use_oz(const tmvn_ctx* h) {
  return h->opt.projection == 1 || (h->opt.projection == 0 && h->d <= 4096 && h->oz_ratio <= kOzGuard);
}
// digits per operand: 7 (FP64-class, default), 6 or 8 by option; options.precision = 1
// (FP32) takes 4 (31 fraction bits: FP32-class, 10 digit-pair MMAs instead of 28)
int oz_slices(const tmvn_ctx* h) {
  if (h->opt.precision == 1) return 4;
  return h->opt.ozaki_slices ? h->opt.ozaki_slices : 7;
}

tmvn_status update_oz_guard(tmvn_ctx* h, cudaStream_t st) {
  CK(h, launch_oz_guard(h->At, (int)h->m, (int)h->d, h->d_pad, h->dflag, st));
  unsigned long long bits = 0;
  CK(h, cudaMemcpyAsync(&bits, h->dflag, sizeof(bits), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  std::memcpy(&h->oz_ratio, &bits, sizeof(double));
  h->prof.oz_guard_ratio = h->oz_ratio;
  return TMVN_OK;
}

// Arc construction fused into the int8 projection's epilogue (options.fuse_arcs): the
// per-chain kernel then starts from compacted arc lists instead of the P and Q rows.
bool fuse_arcs(const tmvn_ctx* h) { return use_oz(h) && h->opt.fuse_arcs != 0; }
// activity-mask words per chain: ceil(m / 32), padded to 16 bytes (bulk-prefetched rows)
int amask_words(const tmvn_ctx* h) { return (int)round_up((h->m + 31) / 32, 4); }

tmvn_status ensure_arcs(tmvn_ctx* h) {
  if (!fuse_arcs(h) || h->arcs_rows >= h->C_pad) return TMVN_OK;
  free_arcs(h);
  CK(h, dalloc(&h->arcs, (size_t)h->C_pad * h->m_pad));
  CK(h, dalloc(&h->amask, (size_t)h->C_pad * amask_words(h)));
  h->arcs_rows = h->C_pad;
  return TMVN_OK;
}

OzArcs arcs_for(const tmvn_ctx* h, int64_t c0, int64_t C, const double* Pb) {
  OzArcs a;
  a.P = Pb;
  a.ldp = h->m_pad;
  a.b = h->b_eff;
  a.m = (int)h->m;
  a.C = (int)C;
  a.arcs = h->arcs + c0 * h->m_pad;
  a.ald = h->m_pad;
  a.mw = amask_words(h);
  a.amask = h->amask + c0 * a.mw;
  return a;
}

// Digits of A' (once per A' and digit count) and the nu digit buffer (per C_pad).
tmvn_status ensure_ozaki(tmvn_ctx* h) {
  if (!use_oz(h)) return TMVN_OK;
  const int S = oz_slices(h);
  const int64_t KB = (h->d + kOzStepK - 1) / kOzStepK;
  cudaStream_t st = stream_of(h);
  if (h->ozS_A != S || h->ozKB != KB) {
    dfree(h->As);
    if (!h->rowscale) CK(h, dalloc(&h->rowscale, (size_t)h->m_pad));
    CK(h, dalloc(&h->As, (size_t)h->m_pad * KB * kOzStepK * S));
    KL(h, launch_oz_slice(h->At, h->m_pad, h->d, h->d_pad, S, KB, 128, 1, 0, kOzNuExp, h->As,
                          h->rowscale, st));
    h->ozS_A = S;
    h->ozKB = KB;
  }
  if (fuse_arcs(h)) {
    tmvn_status as = ensure_arcs(h);
    if (as != TMVN_OK) return as;
  }
  if (h->ozS_N != S || h->Ns_rows < h->C_pad || !h->Xs) {
    dfree(h->Ns); dfree(h->Ns2); dfree(h->Ns3); dfree(h->Xs); dfree(h->xscale);
    CK(h, dalloc(&h->Ns, (size_t)h->C_pad * KB * kOzStepK * S));
    CK(h, dalloc(&h->Ns2, (size_t)h->C_pad * KB * kOzStepK * S));
    CK(h, dalloc(&h->Xs, (size_t)h->C_pad * KB * kOzStepK * S));
    CK(h, dalloc(&h->xscale, (size_t)h->C_pad));
    h->ozS_N = S;
    h->Ns_rows = h->C_pad;
  }
  return TMVN_OK;
}

// nu buffers: buffer b holds nu of the iterations t with t & 1 == b when the RNG runs
// ahead on its own stream; buffer 0 otherwise
double* nu_f64(const tmvn_ctx* h, int b) { return b == 0 ? h->N : b == 1 ? h->N2 : h->N3; }
int8_t* nu_dig(const tmvn_ctx* h, int b) { return b == 0 ? h->Ns : b == 1 ? h->Ns2 : h->Ns3; }

int8_t* oz_rows(const tmvn_ctx* h, int64_t c0, int b = 0) {
  return nu_dig(h, b) + (c0 / kOzNuRows) * h->ozKB * kOzStepK * oz_slices(h) * kOzNuRows;
}

// nu_{t+1} drawn by the int8 projection of iteration t in its epilogue warps (between
// tiles, while the tensor cores run) instead of by the per-chain kernel after its update
// (options.rng_gemm): nu_t then lives in buffer t & 1.  Not with rng_ahead / pipeline.
bool rng_in_gemm(const tmvn_ctx* h) { return use_oz(h) && h->opt.rng_gemm != 0 && h->opt.rng_ahead == 0; }

OzRng rng_for(const tmvn_ctx* h, int64_t c0, int64_t C, uint64_t seed, uint32_t t, const uint32_t* t_dev,
              int b_out) {
  OzRng r;
  r.seed = seed;
  r.t = t;
  r.t_dev = t_dev;
  r.chain_offset = (uint32_t)(h->opt.chain_offset + c0);
  r.C = (int)C;
  r.d = (int)h->d;
  r.d_pad = h->d_pad;
  r.N = nu_f64(h, b_out) + c0 * h->d_pad;
  r.Ns = oz_rows(h, c0, b_out);
  r.S = oz_slices(h);
  r.KB = h->ozKB;
  return r;
}

// Q rows [c0, c0 + Rp) = nu A'^T by the configured projection (nu from buffer b).
// arcs (nullable, int8 projection only): fuse the arc construction into its epilogue
// rng (nullable, int8 projection only): also draw nu_{t+1} in its epilogue warps
cudaError_t launch_projection(const tmvn_ctx* h, int64_t c0, int64_t Rp, cudaStream_t st, int b = 0,
                              double* Qout = nullptr, bool compact = false, const OzArcs* arcs = nullptr,
                              const OzRng* rng = nullptr) {
  double* Qb = (Qout ? Qout : h->Q) + c0 * h->m_pad;
  if (use_oz(h))
    return launch_ozaki_gemm(h->As, h->m_pad, oz_rows(h, c0, b), Rp, h->ozKB, oz_slices(h), h->rowscale,
                             Qb, h->m_pad, st, compact, nullptr, arcs, rng);
  return launch_gemm_tn(nu_f64(h, b) + c0 * h->d_pad, Rp, h->At, h->m_pad, h->d_pad, Qb, h->m_pad, st);
}

// The refresh P[c0, c0 + C) = X A'^T (C13): with the int8 projection, X is cut into
// digits with one exponent per chain (max_j |x_cj| < 2^e_c) and the same tcgen05
// kernel computes it (stated bound of include/tmvn.h with 2^(e_i + e_c)); else FP64 DMMA.
// Pb: the shard's P rows (already offset by c0)
cudaError_t launch_refresh(tmvn_ctx* h, int64_t c0, int64_t C, double* Pb, cudaStream_t st) {
  const int64_t Rp = round_up(C, kTileR);
  if (!use_oz(h) || !h->Xs)
    return launch_gemm_tn(h->X + c0 * h->d_pad, Rp, h->At, h->m_pad, h->d_pad, Pb, h->m_pad, st);
  const int S = oz_slices(h);
  int8_t* xs = h->Xs + (c0 / kOzNuRows) * h->ozKB * kOzStepK * S * kOzNuRows;
  cudaError_t e = launch_oz_slice(h->X + c0 * h->d_pad, C, h->d, h->d_pad, S, h->ozKB, kOzNuRows, 1, 0,
                                  14 - kOzNuExp, xs, h->xscale + c0, st);  // xscale = 2^(e_c - 4)
  if (e != cudaSuccess) return e;
  return launch_ozaki_gemm(h->As, h->m_pad, xs, Rp, h->ozKB, S, h->rowscale, Pb, h->m_pad, st, false,
                           h->xscale + c0);
}

// nu of iteration t for chains [0, C) (and its digits for the int8 projection).
cudaError_t launch_first_nu(tmvn_ctx* h, int64_t C, uint64_t seed, uint32_t t, cudaStream_t st, int b = 0) {
  cudaError_t e = launch_normals(nu_f64(h, b), (int)C, (int)h->d, h->d_pad, seed, t,
                                 (uint32_t)h->opt.chain_offset, st);
  h->prof.launches += 1;
  if (e != cudaSuccess || !use_oz(h)) return e;
  h->prof.launches += 1;
  return launch_oz_slice(nu_f64(h, b), C, h->d, h->d_pad, oz_slices(h), h->ozKB, kOzNuRows, 0, kOzNuExp,
                         0, nu_dig(h, b), nullptr, st);
}

// nu of iteration t (+ *t_dev) into buffer b, on the RNG stream
cudaError_t launch_nu_ahead(tmvn_ctx* h, int64_t C, uint64_t seed, uint32_t t, const uint32_t* t_dev,
                            int b, cudaStream_t st, int ctas_per_sm = 10) {
  return launch_nu(nu_f64(h, b), use_oz(h) ? nu_dig(h, b) : nullptr, oz_slices(h), h->ozKB, (int)C,
                   (int)h->d, h->d_pad, seed, t, t_dev, (uint32_t)h->opt.chain_offset, st, ctas_per_sm);
}

tmvn_status ensure_rng_stream(tmvn_ctx* h) {
  if (!h->rng_stream) CK(h, cudaStreamCreateWithFlags(&h->rng_stream, cudaStreamNonBlocking));
  if (!h->ev_pre) CK(h, cudaEventCreateWithFlags(&h->ev_pre, cudaEventDisableTiming));
  if (!h->ev_rng) CK(h, cudaEventCreateWithFlags(&h->ev_rng, cudaEventDisableTiming));
  return TMVN_OK;
}

bool finite_all(const std::vector<double>& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

EssParams base_params(tmvn_ctx* h, int C) {
  EssParams p;
  std::memset(&p, 0, sizeof(p));
  p.ldp = h->m_pad;
  p.b = h->b_eff;
  p.m = (int)h->m;
  p.X = h->X;
  p.N = h->N;
  p.d = (int)h->d;
  p.d_pad = h->d_pad;
  p.C = C;
  p.chain_offset = (uint32_t)h->opt.chain_offset;
  p.eps = h->opt.trim_eps;
  p.burn_in = h->opt.record ? h->opt.burn_in : ((int64_t)1 << 62);  // no record: never
  p.thin = h->opt.thin;
  p.S1 = h->S1;
  p.S2 = h->S2;
  p.rej = h->rej;
  p.gstash = h->gstash;
  p.ggaps = h->ggaps;
  p.NB = h->plan.NB;
  p.W = h->plan.W;
  p.CH = h->plan.CH;
  p.stash_smem = h->plan.stash_smem;
  p.Ns = use_oz(h) ? h->Ns : nullptr;
  p.ozS = oz_slices(h);
  p.ozKB = h->ozKB;
  p.bucket_mode = h->opt.buckets;
  p.gmode = h->gmode;
  if (fuse_arcs(h) && h->arcs) {
    p.arcs = h->arcs;
    p.ald = h->m_pad;
    p.amask = h->amask;
    p.mw = amask_words(h);
  }
  return p;
}

// X0 (C x d, host/device, x-space) -> tiled X (u-space).
tmvn_status load_X(tmvn_ctx* h, const double* X0, int64_t C) {
  cudaStream_t st = stream_of(h);
  const int64_t d = h->d;
  CK(h, cudaMemcpyAsync(h->stage, X0, (size_t)C * d * sizeof(double), cudaMemcpyDefault, st));
  if (h->affine) {
    KL(h, launch_trsv_rows(h->stage, h->mu, h->L, (int)C, (int)d, h->stage2, st));
    KL(h, launch_pack(h->stage2, C, d, d, h->X, h->d_pad, st));
  } else {
    KL(h, launch_pack(h->stage, C, d, d, h->X, h->d_pad, st));
  }
  return TMVN_OK;
}

// tiled X (u-space) -> out (C x d, x-space).
tmvn_status store_X(tmvn_ctx* h, int64_t C, double* out) {
  cudaStream_t st = stream_of(h);
  const int64_t d = h->d;
  if (h->affine) {
    KL(h, launch_gemm_tn(h->X, h->C_pad, h->L_tiled, h->d_r128, h->d_pad, h->stage, h->d_r128, st));
    KL(h, launch_add_vec_rows(h->stage, h->d_r128, h->mu, (int)C, (int)d, st));
    CK(h, cudaMemcpy2DAsync(out, d * sizeof(double), h->stage, h->d_r128 * sizeof(double),
                            d * sizeof(double), C, cudaMemcpyDefault, st));
  } else {
    KL(h, launch_unpack(h->X, C, d, h->d_pad, h->stage, st));
    CK(h, cudaMemcpyAsync(out, h->stage, (size_t)C * d * sizeof(double), cudaMemcpyDefault, st));
  }
  return TMVN_OK;
}

// P = X A'^T, then the strict start check (C18).
tmvn_status start_check(tmvn_ctx* h, int64_t C, double* P) {
  Nvtx nv("a0 start check (P = X A'^T, strict a_i.x0 < b_i)");
  cudaStream_t st = stream_of(h);
  // the same product as the periodic refresh, so that a call resumed at a multiple of
  // recompute_every continues bitwise like an uninterrupted one
  KL(h, launch_refresh(h, 0, C, P, st));
  // the strict check itself always on an FP64-class product: with the FP32-class
  // projection (precision = 1, 4 digits) a start within ~1e-6 relative of a face could be
  // misjudged, so there it is checked on an FP64 DMMA product in the other P buffer
  const double* Pchk = P;
  if (use_oz(h) && oz_slices(h) < 7) {
    double* Po = (P == h->P0) ? h->P1 : h->P0;
    KL(h, launch_gemm_tn(h->X, h->C_pad, h->At, h->m_pad, h->d_pad, Po, h->m_pad, st));
    Pchk = Po;
  }
  CK(h, cudaMemsetAsync(h->dflag, 0xff, sizeof(unsigned long long), st));
  KL(h, launch_start_check(Pchk, h->m_pad, h->b_eff, (int)C, (int)h->m, h->dflag, st));
  unsigned long long* fp = reinterpret_cast<unsigned long long*>(h->pin);
  CK(h, cudaMemcpyAsync(fp, h->dflag, sizeof(*fp), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  const unsigned long long flag = *fp;
  if (flag != ~0ull) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "infeasible start: chain %lld violates constraint %lld (a_i . x0 >= b_i; the start "
             "must be strictly interior)",
             (long long)(flag / h->m), (long long)(flag % h->m));
    return fail(h, TMVN_E_INFEASIBLE_START, buf);
  }
  return TMVN_OK;
}

bool recorded_iter(const tmvn_options& o, int64_t t) {
  if (!o.record || t < o.burn_in) return false;
  int64_t thin = o.thin < 1 ? 1 : o.thin;
  return ((t - o.burn_in) % thin) == 0;
}

// One captured block of K iterations starting at an iteration t with t % K == 0:
// (GEMM Q = N A'^T, ESS) x K, then the refresh GEMM P = X A'^T.  The ESS launches
// read t from h->d_tbase (set by a one-thread kernel before each replay) and
// compute their record flag from t, so one graph serves every aligned block.
tmvn_status block_graph(tmvn_ctx* h, const EssParams& base, int64_t C, int64_t K, double* Pc,
                        double* Pn, bool ahead, bool gem, bool ovl, uint64_t seed, cudaGraphExec_t* out) {
  const int parity = Pc == h->P0 ? 0 : 1;
  const bool twobuf = ahead || gem || ovl;  // nu_t in buffer t & 1
  EssParams p = base;
  p.t_dev = h->d_tbase;
  p.rec_dev = 1;
  // one graph serves blocks with and without recorded iterations: round-robin chains
  // whenever recording is on (the per-group moment rows need a fixed chain -> group map)
  p.dyn_use = h->opt.record ? 0 : 1;
  p.gen_next = (twobuf && !ovl) ? 0 : 1;
  if (twobuf) p.Ns = nullptr;
  p.t = 0;
  p.P_cur = Pc;
  p.P_next = Pn;
  std::vector<unsigned char> sig(sizeof(EssParams) + 2 * sizeof(int64_t) + 2 * sizeof(void*) + 16);
  std::memcpy(sig.data() + sizeof(EssParams) + 16 + 2 * sizeof(void*), &seed, 8);
  const int64_t ah = (ahead ? 1 : 0) | (gem ? 2 : 0) | (ovl ? 4 : 0);
  std::memcpy(sig.data() + sizeof(EssParams) + 24 + 2 * sizeof(void*), &ah, 8);
  std::memcpy(sig.data(), &p, sizeof(EssParams));
  std::memcpy(sig.data() + sizeof(EssParams), &C, sizeof(int64_t));
  std::memcpy(sig.data() + sizeof(EssParams) + 8, &K, sizeof(int64_t));
  const void* ptrs[2] = {use_oz(h) ? (const void*)h->As : (const void*)h->At, h->Q};
  std::memcpy(sig.data() + sizeof(EssParams) + 16, ptrs, sizeof(ptrs));
  if (h->graph_exec[parity] && h->graph_sig[parity] == sig) {
    *out = h->graph_exec[parity];
    return TMVN_OK;
  }
  if (h->graph_exec[parity]) {
    cudaGraphExecDestroy(h->graph_exec[parity]);
    h->graph_exec[parity] = nullptr;
  }
  if (!h->capture_stream) CK(h, cudaStreamCreateWithFlags(&h->capture_stream, cudaStreamNonBlocking));
  cudaStream_t cs = h->capture_stream;
  const int64_t Rp = round_up(C, kTileR);
  CK(h, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  cudaError_t err = cudaSuccess;
  double *pc = Pc, *pn = Pn;
  // block start t is a multiple of K (even): nu_{t+i} in buffer i & 1
  for (int64_t i = 0; i < K && err == cudaSuccess; ++i) {
    if (ahead) {  // nu_{t+i+1} on the RNG stream, beside this projection
      if ((err = cudaEventRecord(h->ev_pre, cs)) != cudaSuccess) break;
      if ((err = cudaStreamWaitEvent(h->rng_stream, h->ev_pre, 0)) != cudaSuccess) break;
      if ((err = launch_nu_ahead(h, C, seed, (uint32_t)(i + 1), h->d_tbase, (int)((i + 1) & 1),
                                 h->rng_stream)) != cudaSuccess)
        break;
      if ((err = cudaEventRecord(h->ev_rng, h->rng_stream)) != cudaSuccess) break;
    }
    const OzArcs ga = arcs_for(h, 0, C, pc);
    const OzRng gr = rng_for(h, 0, C, seed, (uint32_t)i, h->d_tbase, (int)((i + 1) & 1));
    err = launch_projection(h, 0, Rp, cs, twobuf ? (int)(i & 1) : 0, nullptr, false, p.arcs ? &ga : nullptr,
                            gem ? &gr : nullptr);
    if (err != cudaSuccess) break;
    p.t = (uint32_t)i;
    p.P_cur = pc;
    p.P_next = pn;
    p.N = nu_f64(h, twobuf ? (int)(i & 1) : 0);
    if (ovl) {
      p.N_next = nu_f64(h, (int)((i + 1) & 1));
      p.Ns = use_oz(h) ? oz_rows(h, 0, (int)((i + 1) & 1)) : nullptr;
    }
    err = launch_ess_step(p, h->plan.grid, cs);
    if (err == cudaSuccess && ahead) err = cudaStreamWaitEvent(cs, h->ev_rng, 0);  // join: nu_{t+i+1} ready
    std::swap(pc, pn);
  }
  if (err == cudaSuccess) err = launch_refresh(h, 0, C, pc, cs);
  cudaGraph_t graph = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(cs, &graph);
  if (err != cudaSuccess) return cuda_fail(h, err, "graph capture");
  if (e2 != cudaSuccess) return cuda_fail(h, e2, "cudaStreamEndCapture");
  cudaError_t e3 = cudaGraphInstantiate(&h->graph_exec[parity], graph, 0);
  cudaGraphDestroy(graph);
  if (e3 != cudaSuccess) return cuda_fail(h, e3, "cudaGraphInstantiate");
  h->graph_sig[parity] = sig;
  *out = h->graph_exec[parity];
  return TMVN_OK;
}

// Pipelined schedule (options.pipeline, one shard): the projection of iteration
// t + 1 runs concurrently with the per-chain kernel of iteration t (Q double-
// buffered; the GEMM on a high-priority stream in its compact 3-stage form, so that a
// CTA of the per-chain kernel fits beside it on every SM, and the per-chain kernel
// schedules its chains dynamically), and nu_{t+2} is drawn on a third stream (nu
// triple-buffered: nu_t in buffer t % 3).  Per iteration t the order is
//   RNG(t+2)  after ESS(t-1)            (nu buffer (t+2)%3 last read by ESS(t-1))
//   GEMM(t+1) after ESS(t-1), RNG(t+1)  (Q buffer (t+1)&1 last read by ESS(t-1))
//   ESS(t)    after GEMM(t)
// Results are bitwise those of the serial schedule.
tmvn_status ensure_pipeline(tmvn_ctx* h) {
  const size_t cd = (size_t)h->C_pad * h->d_pad, cm = (size_t)h->C_pad * h->m_pad;
  if (!h->N3) CK(h, dalloc(&h->N3, cd));
  if (!h->Q2) CK(h, dalloc(&h->Q2, cm));
  if (use_oz(h) && !h->Ns3) CK(h, dalloc(&h->Ns3, (size_t)h->C_pad * h->ozKB * kOzStepK * oz_slices(h)));
  if (!h->gemm_stream) {
    int lo = 0, hi = 0;
    CK(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(h, cudaStreamCreateWithPriority(&h->gemm_stream, cudaStreamNonBlocking, hi));
  }
  tmvn_status rs = ensure_rng_stream(h);
  if (rs != TMVN_OK) return rs;
  for (auto* e : {&h->ev_q[0], &h->ev_q[1], &h->ev_nu[0], &h->ev_nu[1], &h->ev_nu[2], &h->ev_ess,
                  &h->ev_join[0], &h->ev_join[1], &h->ev_essb})
    if (!*e) CK(h, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  if (!h->essb_stream) CK(h, cudaStreamCreateWithFlags(&h->essb_stream, cudaStreamNonBlocking));
  return TMVN_OK;
}

tmvn_status run_loop_pipe(tmvn_ctx* h, int64_t C, int64_t n_iter, uint64_t seed, double* P_cur,
                          int64_t* n_recorded) {
  tmvn_status ps = ensure_pipeline(h);
  if (ps != TMVN_OK) return ps;
  cudaStream_t A = stream_of(h), B = h->gemm_stream, R = h->rng_stream;
  const int64_t t0 = h->opt.iter_offset;
  const int64_t K = h->opt.recompute_every < 1 ? 1 : h->opt.recompute_every;
  const int64_t Rp = round_up(C, kTileR);
  const bool oz = use_oz(h);
  double* P_next = (P_cur == h->P0) ? h->P1 : h->P0;
  double* Qb[2] = {h->Q, h->Q2};
  EssParams p = base_params(h, (int)C);
  p.seed = seed;
  p.gen_next = 0;
  p.Ns = nullptr;
  p.arcs = nullptr;  // GEMM(t + 1) runs beside ESS(t), which is still writing P: no fused arcs
  p.amask = nullptr;
  if (!h->dyn) CK(h, dalloc(&h->dyn, (size_t)64 * 16));
  CK(h, cudaMemsetAsync(h->dyn, 0, sizeof(int) * 64 * 16, A));
  p.dyn_ctr = h->dyn;
  if (!h->gmode) CK(h, dalloc(&h->gmode, (size_t)4 * 16));
  CK(h, cudaMemsetAsync(h->gmode, 0, sizeof(int) * 4 * 16, A));
  p.gmode = h->gmode;
  auto proj = [&](int64_t t) -> cudaError_t {
    return launch_projection(h, 0, Rp, B, (int)(t % 3), Qb[t & 1], oz);
  };
  // prologue: nu_{t0} (A), nu_{t0+1} (R), Q_{t0} (B)
  CK(h, cudaEventRecord(h->ev_ess, A));  // orders B and R after all earlier work on A
  CK(h, launch_first_nu(h, C, seed, (uint32_t)t0, A, (int)(t0 % 3)));
  CK(h, cudaEventRecord(h->ev_nu[t0 % 3], A));
  if (n_iter > 1) {
    CK(h, cudaStreamWaitEvent(R, h->ev_ess, 0));
    KL(h, launch_nu_ahead(h, C, seed, (uint32_t)(t0 + 1), nullptr, (int)((t0 + 1) % 3), R));
    CK(h, cudaEventRecord(h->ev_nu[(t0 + 1) % 3], R));
  }
  CK(h, cudaStreamWaitEvent(B, h->ev_nu[t0 % 3], 0));
  KL(h, proj(t0));
  CK(h, cudaEventRecord(h->ev_q[t0 & 1], B));
  int64_t nrec = 0;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t t = t0 + it;
    if (it + 2 < n_iter) {  // nu_{t+2}
      CK(h, cudaStreamWaitEvent(R, h->ev_ess, 0));
      KL(h, launch_nu_ahead(h, C, seed, (uint32_t)(t + 2), nullptr, (int)((t + 2) % 3), R));
      CK(h, cudaEventRecord(h->ev_nu[(t + 2) % 3], R));
    }
    if (it + 1 < n_iter) {  // Q_{t+1}, beside ESS(t)
      CK(h, cudaStreamWaitEvent(B, h->ev_ess, 0));
      CK(h, cudaStreamWaitEvent(B, h->ev_nu[(t + 1) % 3], 0));
      KL(h, proj(t + 1));
      CK(h, cudaEventRecord(h->ev_q[(t + 1) & 1], B));
    }
    const bool rec = recorded_iter(h->opt, t);
    CK(h, cudaStreamWaitEvent(A, h->ev_q[t & 1], 0));
    p.P_cur = P_cur;
    p.P_next = P_next;
    p.Q = Qb[t & 1];
    p.N = nu_f64(h, (int)(t % 3));
    p.t = (uint32_t)t;
    p.record = (rec && !h->affine) ? 1 : 0;
    p.dyn_use = p.record ? 0 : 1;
    KL(h, launch_ess_step(p, h->plan.grid, A));
    std::swap(P_cur, P_next);
    if (rec && h->affine) {
      KL(h, launch_gemm_tn(h->X, Rp, h->L_tiled, h->d_r128, h->d_pad, h->stage, h->d_r128, A));
      KL(h, launch_accum_affine(h->stage, h->d_r128, h->mu, (int)C, (int)h->d, h->S1x, h->S2x, A));
    }
    if ((t + 1) % K == 0 && it + 1 < n_iter)
      KL(h, launch_refresh(h, 0, C, P_cur, A));
    CK(h, cudaEventRecord(h->ev_ess, A));
    if (rec) ++nrec;
  }
  // join the GEMM and RNG streams into the library stream (part b joined every iteration)
  CK(h, cudaEventRecord(h->ev_join[0], B));
  CK(h, cudaEventRecord(h->ev_join[1], R));
  CK(h, cudaStreamWaitEvent(A, h->ev_join[0], 0));
  CK(h, cudaStreamWaitEvent(A, h->ev_join[1], 0));
  *n_recorded = nrec;
  return TMVN_OK;
}

// The hot loop.  On entry X holds x_{t0} (tiled) and P_cur = X A'^T.
// The chains are split into `shards` row blocks (multiples of 128 chains), each an
// independent GEMM -> ESS sequence on its own stream: the DMMA GEMM of one shard
// co-runs with the FP64/ALU-bound ESS kernel of another.  Per-chain results do not
// depend on the split (no split-K; global chain index in the RNG counters).
tmvn_status run_loop(tmvn_ctx* h, int64_t C, int64_t n_iter, uint64_t seed, double* P_cur,
                     int64_t* n_recorded) {
  h->prof.projection_used = use_oz(h) ? 1 : 2;
  if (h->opt.pipeline == 1 && h->nshards == 1 && !h->trace_dev && h->opt.profile == 0 && n_iter > 0)
    return run_loop_pipe(h, C, n_iter, seed, P_cur, n_recorded);
  cudaStream_t st = stream_of(h);
  const int64_t t0 = h->opt.iter_offset;
  const int64_t K = h->opt.recompute_every < 1 ? 1 : h->opt.recompute_every;
  double* P_next = (P_cur == h->P0) ? h->P1 : h->P0;
  // nu_{t+1} drawn on the RNG stream beside the projection GEMM of iteration t (one
  // shard, options.rng_ahead): nu_t lives in buffer t & 1
  const bool ahead = h->opt.rng_ahead != 0 && h->nshards == 1 && !h->trace_dev;
  if (ahead) {
    tmvn_status rs = ensure_rng_stream(h);
    if (rs != TMVN_OK) return rs;
  }
  // nu_{t+1} drawn by the projection of iteration t (options.rng_gemm): nu_t in buffer t & 1
  const bool gem = !ahead && rng_in_gemm(h);
  // nu_{t+1} drawn by the per-chain kernel while theta is computed (options.rng_overlap)
  const bool ovl = !ahead && !gem && h->opt.rng_overlap != 0 && h->plan.W > 1;
  const bool twobuf = ahead || gem || ovl;
  CK(h, launch_first_nu(h, C, seed, (uint32_t)t0, st, twobuf ? (int)(t0 & 1) : 0));
  if (!h->dyn) CK(h, dalloc(&h->dyn, (size_t)64 * 16));
  if (!h->gmode) CK(h, dalloc(&h->gmode, (size_t)4 * 16));
  CK(h, cudaMemsetAsync(h->gmode, 0, sizeof(int) * 4 * 16, st));
  // dynamic hand-out pays for long rows (W = 8); for short ones the atomic's latency
  // is comparable to a chain's work (config 2: 17 -> 22 us per launch), so auto = W == 8
  const bool dyn = (h->opt.schedule == 2 || (h->opt.schedule == 0 && h->plan.W == 8)) && h->nshards <= 16;
  if (dyn) CK(h, cudaMemsetAsync(h->dyn, 0, sizeof(int) * 64 * 16, st));
  // ---- shards
  int S = h->nshards;
  const int64_t per = round_up((C + S - 1) / S, kTileR);
  S = (int)((C + per - 1) / per);
  struct Shard {
    int64_t c0, C;
    cudaStream_t st;
    EssParams p;
    double *Pc, *Pn;
  };
  std::vector<Shard> sh(S);
  for (int s = 0; s < S; ++s) {
    Shard& x = sh[s];
    x.c0 = s * per;
    x.C = std::min(per, C - x.c0);
    x.st = S == 1 ? st : h->shard_streams[s];
    x.p = base_params(h, (int)x.C);
    x.p.X = h->X + x.c0 * h->d_pad;
    x.p.N = h->N + x.c0 * h->d_pad;
    if (x.p.Ns) x.p.Ns = oz_rows(h, x.c0);
    x.p.S1 = h->S1 + x.c0 * h->d_pad;
    x.p.S2 = h->S2 + x.c0 * h->d_pad;
    x.p.rej = h->rej + x.c0;
    x.p.dyn_ctr = dyn ? h->dyn + 64 * s : nullptr;
    x.p.gmode = h->gmode + 4 * (s % 16);
    x.p.chain_offset = (uint32_t)(h->opt.chain_offset + x.c0);
    x.p.gstash = h->gstash ? h->gstash + (size_t)s * h->plan.groups * ess_gstash_stride(h->m) : nullptr;
    x.p.ggaps = h->ggaps + (size_t)s * h->plan.groups * (h->m + 2);
    x.p.Q = h->Q + x.c0 * h->m_pad;
    if (x.p.arcs) {
      x.p.arcs = h->arcs + x.c0 * h->m_pad;
      x.p.amask = h->amask + x.c0 * x.p.mw;
    }
    x.p.seed = seed;
    x.Pc = P_cur + x.c0 * h->m_pad;
    x.Pn = P_next + x.c0 * h->m_pad;
  }
  if (S > 1) {  // fork
    CK(h, cudaEventRecord(h->fork_event, st));
    for (int s = 0; s < S; ++s) CK(h, cudaStreamWaitEvent(sh[s].st, h->fork_event, 0));
  }
  int64_t nrec = 0;
  // profiling: event pairs around the hot-loop GEMMs (kind 0) and ESS launches (kind 1)
  const bool prof = h->opt.profile != 0;
  std::vector<int> kinds;
  std::vector<int64_t> kind_C;
  auto ev_mark = [&](size_t idx, cudaStream_t s_) -> cudaError_t {
    while (h->events.size() <= idx) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      h->events.push_back(e);
    }
    return cudaEventRecord(h->events[idx], s_);
  };
#define TIMED(kind, nC, s_, expr)                           \
  do {                                                      \
    if (prof) CK(h, ev_mark(2 * kinds.size(), s_));         \
    KL(h, expr);                                            \
    if (prof) {                                             \
      CK(h, ev_mark(2 * kinds.size() + 1, s_));             \
      kinds.push_back(kind);                                \
      kind_C.push_back(nC);                                 \
    }                                                       \
  } while (0)
  const bool graphs = h->opt.graphs != 0 && S == 1 && !prof && !h->trace_dev &&
                      !(h->affine && h->opt.record) && (K % 2 == 0);
  if (graphs && !h->d_tbase) CK(h, dalloc(&h->d_tbase, 1));
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t t = t0 + it;
    if (graphs && t % K == 0 && n_iter - it >= K) {  // a whole aligned block: replay
      Shard& x = sh[0];
      cudaGraphExec_t ge;
      tmvn_status gs = block_graph(h, x.p, C, K, x.Pc, x.Pn, ahead, gem, ovl, seed, &ge);
      if (gs != TMVN_OK) return gs;
      Nvtx nv("graph block: (a2 projection, ess_kernel) x K, a3 refresh");
      KL(h, launch_set_u32(h->d_tbase, (uint32_t)t, st));
      CK(h, cudaGraphLaunch(ge, st));
      h->prof.launches += (ahead ? 3 : 2) * K + 1;
      for (int64_t i = 0; i < K; ++i) nrec += recorded_iter(h->opt, t + i) ? 1 : 0;
      it += K - 1;  // K even: P parity unchanged, the block ends with the refresh
      continue;
    }
    const bool rec = recorded_iter(h->opt, t);
    for (int s = 0; s < S; ++s) {
      Shard& x = sh[s];
      const int64_t Rp = round_up(x.C, kTileR);
      const int b = twobuf ? (int)(t & 1) : 0;
      if (ahead && it + 1 < n_iter) {  // nu_{t+1} into the other buffer, beside this projection
        CK(h, cudaEventRecord(h->ev_pre, x.st));
        CK(h, cudaStreamWaitEvent(h->rng_stream, h->ev_pre, 0));
        KL(h, launch_nu_ahead(h, C, seed, (uint32_t)(t + 1), nullptr, b ^ 1, h->rng_stream));
        CK(h, cudaEventRecord(h->ev_rng, h->rng_stream));
      }
      const OzArcs xa = arcs_for(h, x.c0, x.C, x.Pc);
      const OzRng xr = rng_for(h, x.c0, x.C, seed, (uint32_t)t, nullptr, b ^ 1);
      {
        Nvtx nv(gem ? "a2 projection Q = N A'^T (+ a1 nu_{t+1} in the epilogue)" : "a2 projection Q = N A'^T");
        TIMED(use_oz(h) ? 2 : 0, x.C, x.st,
              launch_projection(h, x.c0, Rp, x.st, b, nullptr, false, x.p.arcs ? &xa : nullptr,
                                (gem && it + 1 < n_iter) ? &xr : nullptr));
      }
      x.p.P_cur = x.Pc;
      x.p.P_next = x.Pn;
      x.p.t = (uint32_t)t;
      x.p.gen_next = ((!twobuf || ovl) && it + 1 < n_iter) ? 1 : 0;
      if (twobuf) {
        x.p.N = nu_f64(h, b) + x.c0 * h->d_pad;
        x.p.Ns = nullptr;
      }
      if (ovl) {  // nu_{t+1} (and its digits) into the other buffer
        x.p.N_next = nu_f64(h, b ^ 1) + x.c0 * h->d_pad;
        x.p.Ns = use_oz(h) ? oz_rows(h, x.c0, b ^ 1) : nullptr;
      }
      x.p.record = (rec && !h->affine) ? 1 : 0;
      x.p.dyn_use = x.p.record ? 0 : 1;  // recorded: round-robin (per-group moment rows)
      {
        Nvtx nv("a1,a3-a9 ess_kernel (arcs, Alg. 3, theta, P', safeguard, x, moments, nu_{t+1})");
        TIMED(x.p.record ? 3 : 1, x.C, x.st, launch_ess_step(x.p, h->plan.grid, x.st));
      }
      if (ahead && it + 1 < n_iter) CK(h, cudaStreamWaitEvent(x.st, h->ev_rng, 0));  // nu_{t+1} ready
      std::swap(x.Pc, x.Pn);
      if (rec && h->affine) {
        double* stg = h->stage + x.c0 * h->d_r128;
        KL(h, launch_gemm_tn(x.p.X, Rp, h->L_tiled, h->d_r128, h->d_pad, stg, h->d_r128, x.st));
        KL(h, launch_accum_affine(stg, h->d_r128, h->mu, (int)x.C, (int)h->d, h->S1x + x.c0 * h->d,
                                  h->S2x + x.c0 * h->d, x.st));
      }
      if ((t + 1) % K == 0 && it + 1 < n_iter) {
        Nvtx nv("a3 refresh P = X A'^T");
        TIMED(0, x.C, x.st, launch_refresh(h, x.c0, x.C, x.Pc, x.st));
      }
    }
    if (rec) ++nrec;
    if (h->trace_dev) {  // S == 1 when tracing
      KL(h, launch_gather_rows_tiled(h->X, h->d_pad, (int)h->d, h->trace_rows, h->trace_n,
                                     h->trace_dev + (size_t)(it + 1) * h->trace_n * h->d, st));
    }
  }
#undef TIMED
  if (S > 1) {  // join
    for (int s = 0; s < S; ++s) {
      CK(h, cudaEventRecord(h->join_events[s], sh[s].st));
      CK(h, cudaStreamWaitEvent(st, h->join_events[s], 0));
    }
  }
  *n_recorded = nrec;
  if (prof && !kinds.empty()) {
    CK(h, cudaStreamSynchronize(st));
    for (size_t k = 0; k < kinds.size(); ++k) {
      float ms = 0.f;
      CK(h, cudaEventElapsedTime(&ms, h->events[2 * k], h->events[2 * k + 1]));
      const double nC = (double)kind_C[k];
      if (kinds[k] == 2) {
        const double S = oz_slices(h);
        h->prof.tc_launches += 1;
        h->prof.tc_ms += ms;
        h->prof.tc_flops += 2.0 * nC * (double)h->m * (double)h->d;
        h->prof.tc_ops += S * (S + 1) / 2 * 2.0 * nC * (double)h->m * (double)h->d;
      } else if (kinds[k] == 0) {
        h->prof.gemm_launches += 1;
        h->prof.gemm_ms += ms;
        h->prof.gemm_flops += 2.0 * nC * (double)h->m * (double)h->d;
      } else {
        // P, Q read + P' write (24 B per constraint-eval); X r/w, nu read + next nu write
        // and its int8 digits (32 + S B per chain-coordinate); when recorded, the moment
        // rows of the groups (S1, S2 r/w, 32 B per group-coordinate, L2-resident)
        const double S = use_oz(h) ? (double)oz_slices(h) : 0.0;
        h->prof.ess_launches += 1;
        h->prof.ess_ms += ms;
        h->prof.ess_bytes += 24.0 * nC * (double)h->m + (32.0 + S) * nC * (double)h->d +
                             (kinds[k] == 3 ? 32.0 * (double)h->plan.groups * (double)h->d : 0.0);
      }
    }
  }
  return TMVN_OK;
}

// Reduce per-chain moments / rejections into the handle's counters.
tmvn_status finish_stats(tmvn_ctx* h, int64_t C, int64_t n_iter, int64_t nrec) {
  Nvtx nv("a9 moment / counter reduction");
  cudaStream_t st = stream_of(h);
  const int64_t d = h->d;
  int64_t* rp = reinterpret_cast<int64_t*>(h->pin);
  double* s = h->pin + 8;
  double* q = s + d;
  KL(h, launch_sum_i64(h->rej, (int)C, h->dsum, st));
  CK(h, cudaMemcpyAsync(rp, h->dsum, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (nrec > 0) {
    // the two sums land in separate halves of msum: one host sync for both
    double* m2 = h->msum + d;
    if (h->affine) {
      // row-major C x d accumulators: reuse the tiled reducer through a pack
      KL(h, launch_pack(h->S1x, C, d, d, h->stage2, h->d_pad, st));
      KL(h, launch_chain_sum(h->stage2, (int)C, (int)d, h->d_pad, h->msum, h->stage, st));
      h->prof.launches += 1;  // two kernels
      KL(h, launch_pack(h->S2x, C, d, d, h->stage2, h->d_pad, st));
      KL(h, launch_chain_sum(h->stage2, (int)C, (int)d, h->d_pad, m2, h->stage, st));
      h->prof.launches += 1;  // two kernels
    } else {
      KL(h, launch_chain_sum(h->S1, (int)C, (int)d, h->d_pad, h->msum, h->stage, st));
      h->prof.launches += 1;  // two kernels
      KL(h, launch_chain_sum(h->S2, (int)C, (int)d, h->d_pad, m2, h->stage, st));
      h->prof.launches += 1;  // two kernels
    }
    CK(h, cudaMemcpyAsync(s, h->msum, 2 * d * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  CK(h, cudaStreamSynchronize(st));
  const int64_t rej = *rp;
  if (nrec > 0) {
    for (int64_t j = 0; j < d; ++j) {
      h->mom_sum[j] += s[j];
      h->mom_sq[j] += q[j];
    }
  }
  h->stats.steps += C * n_iter;
  h->stats.rejections += rej;
  h->stats.recorded += C * nrec;
  return TMVN_OK;
}

tmvn_status clear_accumulators(tmvn_ctx* h, int64_t n_iter) {
  cudaStream_t st = stream_of(h);
  bool any = false;
  for (int64_t it = 0; it < n_iter && !any; ++it) any = recorded_iter(h->opt, h->opt.iter_offset + it);
  if (any) {
    size_t cd = (size_t)h->C_pad * h->d_pad;
    if (h->affine) {
      if (ensure_affine_moments(h) != TMVN_OK) return TMVN_E_OOM;
      CK(h, cudaMemsetAsync(h->S1x, 0, (size_t)h->C_pad * h->d * sizeof(double), st));
      CK(h, cudaMemsetAsync(h->S2x, 0, (size_t)h->C_pad * h->d * sizeof(double), st));
    } else {
      CK(h, cudaMemsetAsync(h->S1, 0, cd * sizeof(double), st));
      CK(h, cudaMemsetAsync(h->S2, 0, cd * sizeof(double), st));
    }
  }
  CK(h, cudaMemsetAsync(h->rej, 0, (size_t)h->C_pad * sizeof(int64_t), st));
  return TMVN_OK;
}

tmvn_status check_sample_args(tmvn_ctx* h, const double* X0, int64_t C, int64_t n_iter,
                              const double* out) {
  if (!h) return fail(nullptr, TMVN_E_ARG, "null handle");
  if (!X0 || !out) return fail(h, TMVN_E_ARG, "X0 and out must be non-null");
  if (C < 1 || n_iter < 0) return fail(h, TMVN_E_ARG, "need C >= 1 and n_iter >= 0");
  if (h->opt.chain_offset < 0 || h->opt.chain_offset + C > (int64_t)1 << 32)
    return fail(h, TMVN_E_ARG, "global chain index must fit in 32 bits");
  if (h->opt.iter_offset < 0 || h->opt.iter_offset + n_iter >= (int64_t)1 << 32)
    return fail(h, TMVN_E_ARG, "iteration index must fit in 32 bits");
  if (C > (int64_t)1 << 30) return fail(h, TMVN_E_ARG, "C too large");
  return TMVN_OK;
}

tmvn_status set_device(tmvn_ctx* h) {
  CK(h, cudaSetDevice(h->device));
  return TMVN_OK;
}

}  // namespace

// =============================================================================
extern "C" {

tmvn_status tmvn_default_options(tmvn_options* o) {
  if (!o) return TMVN_E_ARG;
  std::memset(o, 0, sizeof(*o));
  o->trim_eps = 0.0;
  o->recompute_every = 32;
  o->burn_in = 0;
  o->thin = 1;
  o->record = 1;
  o->chain_offset = 0;
  o->iter_offset = 0;
  o->auto_advance = 1;
  o->stream = nullptr;
  o->profile = 0;
  o->chain_warps = 0;
  o->streams = 0;
  o->ring = 0;
  o->graphs = 1;
  o->projection = 0;
  o->ozaki_slices = 0;
  o->rng_ahead = 0;  // measured slower on B200 (the GEMM loses more than the ESS kernel gains)
  o->schedule = 0;
  o->pipeline = 0;
  o->latency = 2;
  o->precision = 0;
  o->total_chains = 0;
  o->fuse_arcs = 0;
  o->rng_gemm = 0;
  o->rng_overlap = 0;
  o->buckets = 0;
  o->small_warps = 0;
  o->warp_mode = 2;  // auto (small polytopes, few chains: small_fits)
  return TMVN_OK;
}

tmvn_status tmvn_struct_sizes(int64_t* out4) {
  if (!out4) return fail(nullptr, TMVN_E_ARG, "null argument");
  out4[0] = (int64_t)sizeof(tmvn_options);
  out4[1] = (int64_t)sizeof(tmvn_stats);
  out4[2] = (int64_t)sizeof(tmvn_profile);
  out4[3] = (int64_t)sizeof(tmvn_step_dump);
  return TMVN_OK;
}

const char* tmvn_version(void) { return "tmvn-b200 0.2 (sm_100a, FP64 DMMA + int8 tcgen05 Ozaki)"; }

const char* tmvn_last_error(tmvn_handle h) { return h ? h->err.c_str() : g_create_error.c_str(); }

tmvn_status tmvn_create(const double* A, const double* b, int64_t m, int64_t d, tmvn_handle* out) {
  if (!out) return fail(nullptr, TMVN_E_ARG, "out is null");
  *out = nullptr;
  if (!A || !b) return fail(nullptr, TMVN_E_ARG, "A and b must be non-null");
  if (m < 1 || d < 1) return fail(nullptr, TMVN_E_ARG, "need m >= 1 and d >= 1");
  if (d > (1 << 24) || m > (1 << 30)) return fail(nullptr, TMVN_E_ARG, "need d <= 2^24 and m <= 2^30");
  if (m > (1 << 30) || d > (1 << 24)) return fail(nullptr, TMVN_E_ARG, "m or d too large");
  std::vector<double> hA = to_host(A, (size_t)m * d), hb = to_host(b, (size_t)m);
  if (!finite_all(hA) || !finite_all(hb)) return fail(nullptr, TMVN_E_ARG, "A and b must be finite");
  for (int64_t i = 0; i < m; ++i) {
    bool zero = true;
    for (int64_t j = 0; j < d && zero; ++j) zero = hA[(size_t)i * d + j] == 0.0;
    if (zero && hb[i] < 0.0) {
      char buf[160];
      snprintf(buf, sizeof(buf), "empty polytope: row %lld of A is zero and b < 0 (P:914)", (long long)i);
      return fail(nullptr, TMVN_E_EMPTY_POLYTOPE, buf);
    }
  }
  tmvn_ctx* h = new tmvn_ctx();
  cudaGetDevice(&h->device);
  h->m = m;
  h->d = d;
  h->m_pad = round_up(m, kTileR);
  h->d_pad = round_up(d, kTileK);
  h->d_r128 = round_up(d, kTileR);
  tmvn_default_options(&h->opt);
  h->mom_sum.assign(d, 0.0);
  h->mom_sq.assign(d, 0.0);
  auto bad = [&](cudaError_t e, const char* w) {
    std::string msg = std::string(w) + ": " + cudaGetErrorString(e);
    tmvn_destroy(h);
    return fail(nullptr, e == cudaErrorMemoryAllocation ? TMVN_E_OOM : TMVN_E_CUDA, msg);
  };
  cudaError_t e;
  if ((e = dalloc(&h->A_row, (size_t)m * d)) != cudaSuccess) return bad(e, "alloc A");
  if ((e = dalloc(&h->b_orig, (size_t)h->m_pad)) != cudaSuccess) return bad(e, "alloc b");
  if ((e = dalloc(&h->b_eff, (size_t)h->m_pad)) != cudaSuccess) return bad(e, "alloc b'");
  if ((e = dalloc(&h->A_tiled, (size_t)h->m_pad * h->d_pad)) != cudaSuccess) return bad(e, "alloc At");
  h->At = h->A_tiled;
  if ((e = dalloc(&h->dflag, 1)) != cudaSuccess) return bad(e, "alloc flag");
  if ((e = dalloc(&h->dsum, 1)) != cudaSuccess) return bad(e, "alloc sum");
  if ((e = dalloc(&h->msum, (size_t)2 * d)) != cudaSuccess) return bad(e, "alloc msum");
  if ((e = cudaMallocHost(&h->pin, (size_t)(8 + 2 * d) * sizeof(double))) != cudaSuccess) {
    h->pin = nullptr;
    return bad(e, "alloc pinned scratch");
  }
  cudaMemcpy(h->A_row, hA.data(), hA.size() * sizeof(double), cudaMemcpyHostToDevice);
  // b padded to m_pad with +inf: padded constraints (zero rows of A) are never active
  std::vector<double> hb_pad(hb);
  hb_pad.resize((size_t)h->m_pad, HUGE_VAL);
  cudaMemcpy(h->b_orig, hb_pad.data(), hb_pad.size() * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(h->b_eff, hb_pad.data(), hb_pad.size() * sizeof(double), cudaMemcpyHostToDevice);
  if ((e = launch_pack(h->A_row, m, d, d, h->A_tiled, h->d_pad, 0)) != cudaSuccess) return bad(e, "pack A");
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bad(e, "create");
  if (update_oz_guard(h, 0) != TMVN_OK) {
    std::string msg = h->err;
    tmvn_destroy(h);
    return fail(nullptr, TMVN_E_CUDA, msg);
  }
  *out = h;
  return TMVN_OK;
}

tmvn_status tmvn_set_affine(tmvn_handle h, const double* mu, const double* L) {
  if (!h) return fail(nullptr, TMVN_E_ARG, "null handle");
  if (set_device(h) != TMVN_OK) return TMVN_E_CUDA;
  const int64_t d = h->d, m = h->m;
  cudaStream_t st = stream_of(h);
  if (!mu && !L) {
    if (h->At != h->A_tiled) dfree(h->At);
    h->At = h->A_tiled;
    CK(h, cudaMemcpy(h->b_eff, h->b_orig, m * sizeof(double), cudaMemcpyDeviceToDevice));
    dfree(h->mu); dfree(h->L); dfree(h->L_tiled);
    h->affine = false;
    h->ozS_A = 0;
    return update_oz_guard(h, st);
  }
  std::vector<double> hmu = mu ? to_host(mu, d) : std::vector<double>(d, 0.0);
  std::vector<double> hL(d * d, 0.0);
  if (L) hL = to_host(L, (size_t)d * d);
  else for (int64_t j = 0; j < d; ++j) hL[j * d + j] = 1.0;
  if (!finite_all(hmu) || !finite_all(hL)) return fail(h, TMVN_E_ARG, "mu and L must be finite");
  for (int64_t j = 0; j < d; ++j) {
    if (!(hL[j * d + j] > 0.0)) return fail(h, TMVN_E_FACTOR, "L must have a positive diagonal");
    for (int64_t k = j + 1; k < d; ++k)
      if (hL[j * d + k] != 0.0) return fail(h, TMVN_E_FACTOR, "L must be lower-triangular");
  }
  if (!h->mu) CK(h, dalloc(&h->mu, (size_t)d));
  if (!h->L) CK(h, dalloc(&h->L, (size_t)d * d));
  if (!h->L_tiled) CK(h, dalloc(&h->L_tiled, (size_t)h->d_r128 * h->d_pad));
  CK(h, cudaMemcpy(h->mu, hmu.data(), d * sizeof(double), cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(h->L, hL.data(), (size_t)d * d * sizeof(double), cudaMemcpyHostToDevice));
  KL(h, launch_pack(h->L, d, d, d, h->L_tiled, h->d_pad, st));
  // A' = A L = A (L^T)^T : W operand = L^T (rows j = column j of L)
  std::vector<double> hLT((size_t)d * d);
  for (int64_t j = 0; j < d; ++j)
    for (int64_t k = 0; k < d; ++k) hLT[j * d + k] = hL[k * d + j];
  double *LT = nullptr, *LTt = nullptr, *Aprime = nullptr;
  CK(h, dalloc(&LT, (size_t)d * d));
  CK(h, dalloc(&LTt, (size_t)h->d_r128 * h->d_pad));
  CK(h, dalloc(&Aprime, (size_t)h->m_pad * h->d_r128));
  CK(h, cudaMemcpy(LT, hLT.data(), (size_t)d * d * sizeof(double), cudaMemcpyHostToDevice));
  KL(h, launch_pack(LT, d, d, d, LTt, h->d_pad, st));
  KL(h, launch_gemm_tn(h->A_tiled, h->m_pad, LTt, h->d_r128, h->d_pad, Aprime, h->d_r128, st));
  if (h->At == h->A_tiled) CK(h, dalloc(&h->At, (size_t)h->m_pad * h->d_pad));
  KL(h, launch_pack(Aprime, m, d, h->d_r128, h->At, h->d_pad, st));
  KL(h, launch_gemv_shift(h->A_row, h->b_orig, h->mu, (int)m, (int)d, h->b_eff, st));
  CK(h, cudaStreamSynchronize(st));
  dfree(LT); dfree(LTt); dfree(Aprime);
  h->affine = true;
  h->ozS_A = 0;  // A' changed: digits stale
  {
    tmvn_status gs = update_oz_guard(h, st);
    if (gs != TMVN_OK) return gs;
  }
  dfree(h->S1x); dfree(h->S2x);
  return TMVN_OK;
}

tmvn_status tmvn_set_options(tmvn_handle h, const tmvn_options* o) {
  if (!h || !o) return fail(h, TMVN_E_ARG, "null argument");
  if (!(o->trim_eps >= 0.0) || !(o->trim_eps < 3.14159)) return fail(h, TMVN_E_ARG, "need 0 <= trim_eps < pi");
  if (o->recompute_every < 1 || o->thin < 1 || o->burn_in < 0) return fail(h, TMVN_E_ARG, "bad recompute_every / thin / burn_in");
  if (o->chain_offset < 0 || o->iter_offset < 0) return fail(h, TMVN_E_ARG, "offsets must be >= 0");
  if (o->chain_warps != 0 && o->chain_warps != 1 && o->chain_warps != 2 && o->chain_warps != 4 &&
      o->chain_warps != 8 && o->chain_warps != 16)
    return fail(h, TMVN_E_ARG, "chain_warps must be 0, 1, 2, 4, 8 or 16");
  if (o->projection < 0 || o->projection > 2) return fail(h, TMVN_E_ARG, "projection must be 0, 1 or 2");
  if (o->latency < 0 || o->latency > 2) return fail(h, TMVN_E_ARG, "latency must be 0, 1 or 2");
  if (o->precision < 0 || o->precision > 1) return fail(h, TMVN_E_ARG, "precision must be 0 (FP64) or 1 (FP32)");
  if (o->ozaki_slices != 0 && (o->ozaki_slices < 6 || o->ozaki_slices > 8))
    return fail(h, TMVN_E_ARG, "ozaki_slices must be 0, 6, 7 or 8");
  if (o->small_warps != 0 && o->small_warps != 1 && o->small_warps != 2 && o->small_warps != 4 &&
      o->small_warps != 8)
    return fail(h, TMVN_E_ARG, "small_warps must be 0, 1, 2, 4 or 8");
  if (o->projection == 1 && h->d > 4096)
    return fail(h, TMVN_E_ARG, "projection = 1 (int8 tcgen05) needs d <= 4096 (int32 accumulator headroom)");
  h->opt = *o;
  return TMVN_OK;
}

tmvn_status tmvn_get_options(tmvn_handle h, tmvn_options* o) {
  if (!h || !o) return fail(h, TMVN_E_ARG, "null argument");
  *o = h->opt;
  return TMVN_OK;
}

// The latency mode (options.latency = 1): one cluster of CTAs per chain runs every
// iteration in one launch (latency.cu).  Taken when the problem fits its limits (no
// affine change of variable, shared memory), else the throughput loop runs.
// options.latency = 2 (auto) takes it when there are at most SMs / 2 chains (clusters of
// two or more CTAs) and the cost model below expects it to be faster.
// Latency-mode configuration for C chains: cluster size (or cooperative-grid CTAs per
// chain), live-arc capacity and the cost model's time per iteration.  False when the
// mode cannot run.
bool latency_config(tmvn_ctx* h, int64_t C, int sms, int smem_max, int* cs_out, int* cap_out,
                    int* gsz_out, double* t_out) {
  const bool fp32 = h->opt.precision == 1;
  int cap = 0, cs = 0;
  if (h->lat_memo_C == C && h->lat_memo_fp32 == (int)fp32) {  // occupancy queries cost ~10 us each
    cs = h->lat_memo_cs;
    cap = h->lat_memo_cap;
  } else {
    cs = latency_cluster_size((int)C, h->m, h->d_pad, (size_t)smem_max, fp32, &cap);
    h->lat_memo_C = C;
    h->lat_memo_fp32 = (int)fp32;
    h->lat_memo_cs = cs;
    h->lat_memo_cap = cap;
  }
  if (cs == 0 || cap == 0) return false;
  // Cost model (S12, fitted to B200 measurements, tools/grid_probe.py): a CTA
  // streams its rows of A (eb bytes per element) each iteration at ~100 GB/s when A is
  // L2-resident, ~57 GB/s when it is not; besides, a cluster iteration costs ~12.8 us,
  // a cooperative-grid one (SMs / C CTAs per chain, six grid barriers) ~20 + 0.9 C us.
  const double eb = fp32 ? 4.0 : 8.0;
  const double abytes = eb * (double)h->m * (double)h->d_pad;
  const double r_sm = abytes <= 80e6 ? 100e9 : 57e9;
  auto q_time = [&](int n) { return (double)((h->m + n - 1) / n) * (double)h->d_pad * eb / r_sm; };
  double t_lat = 12.8e-6 + q_time(cs);
  int gsz = 0;
  {
    const int G = sms / (int)C;
    const double t_grid = (20.0 + 0.9 * (double)C) * 1e-6 + q_time(G > 0 ? G : 1);
    const bool better = t_grid < 0.9 * t_lat;
    const bool want = h->lat_grid_mode == 1 || (h->lat_grid_mode == 0 && better);
    if (want && G > cs && G >= 2) {
      const int capg = latency_cap(h->d_pad, (int)h->m, G, (size_t)smem_max);
      if (capg > 0) {
        gsz = G;
        cs = G;
        cap = capg;
        t_lat = t_grid;
      }
    }
  }
  *cs_out = cs;
  *cap_out = cap;
  *gsz_out = gsz;
  *t_out = t_lat;
  return true;
}

bool latency_fits(tmvn_ctx* h, int64_t C, int* cs_out, int* cap_out, int* gsz_out) {
  if (h->opt.latency == 0 || h->affine) return false;
  int dev = 0, sms = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int cs = 0, cap = 0, gsz = 0;
  double t_lat = 0.0;
  if (h->opt.latency == 2) {
    // auto: decided from the JOB's chain count (options.total_chains; 0 = this call's C),
    // so that every shard of a job takes the same path (the two paths sum in different
    // orders: results agree to rounding, not bitwise)
    const int64_t Cj = h->opt.total_chains > 0 ? h->opt.total_chains : C;
    if (2 * Cj > sms) return false;
    if (!latency_config(h, Cj, sms, smem_max, &cs, &cap, &gsz, &t_lat)) return false;
    // the default path: ~50 us + 7.8 ps per element of A at few chains
    const double t_def = 50e-6 + 7.8e-12 * (double)h->m * (double)h->d;
    if (t_lat >= t_def) return false;
  }
  if (!latency_config(h, C, sms, smem_max, &cs, &cap, &gsz, &t_lat)) return false;
  if (h->lat_cap_max > 0 && cap > h->lat_cap_max) cap = h->lat_cap_max;
  *cs_out = cs;
  *cap_out = cap;
  *gsz_out = gsz;
  return true;
}

// Warp mode (options.warp_mode, small.cu): FP64, no affine map, m <= 512 and A (d x
// 32 R doubles, column-major) in shared memory beside >= 1 warp's state.  Decided from
// (m, d) only, so every shard of a job takes the same path.  Warps per CTA: as few as
// spread the job's chains over the SMs (up to 16).
constexpr double kWarpAutoWork = 3.2e7;
bool small_fits(tmvn_ctx* h, int64_t C, int* wpc_out, int* nw_out, int* grid_out) {
  if (h->opt.warp_mode == 0 || h->affine || h->opt.precision != 0 || h->m > 512) return false;
  // auto only under the automatic path choice: latency = 0 / 1 ask for a specific path
  if (h->opt.warp_mode == 2 && h->opt.latency != 2) return false;
  int dev = 0, sms = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t a_bytes = (size_t)h->d * 32 * small_rows((int)h->m) * 8;
  const size_t wb = small_warp_bytes((int)h->m, h->d_pad);
  if (a_bytes + wb > (size_t)smem_max) return false;
  int wmax = (int)std::min<size_t>(16, ((size_t)smem_max - a_bytes) / wb);
  if (h->opt.warp_mode == 2 && wmax < 4) return false;  // auto: a few chains per CTA at least
  // auto: only while the job's GEMV + sort work per iteration is small (B200, warp mode vs
  // the throughput path, tools/warp_vs_default.py, BASELINE config 2 shapes: 1024 chains --
  // 1.35e7 below -- 11.4 vs 19.6 us per iteration, 2048 chains (2.7e7) 22.8 vs 28.9 us,
  // 4096 chains (5.4e7) 64.8 vs 39.0 us); from the job's total chains, so that every
  // shard takes the same path
  const int64_t Ctot = h->opt.total_chains > 0 ? h->opt.total_chains : C;
  if (h->opt.warp_mode == 2 && (double)Ctot * ((double)h->m * (double)h->d + 32.0 * (double)h->m) > kWarpAutoWork)
    return false;
  int wpc = (int)std::min<int64_t>(wmax, std::max<int64_t>(1, (C + sms - 1) / sms));
  // warps per chain: a group of nw warps when the chains alone leave the SMs short of
  // ~32 resident warps (each chain's rows, arcs, sort and coordinates split nw ways; the
  // trajectories do not depend on nw), at most one row of A per thread
  int nw = 1;
  const int mi = (int)h->m;
  while (nw < 8 && 2 * nw <= small_rows(mi) && wpc * 2 * nw <= small_max_warps(mi, 2 * nw) && wpc <= 15) nw *= 2;
  if (h->opt.small_warps > 0 && h->opt.small_warps <= small_rows(mi)) {  // requested (run_small checks the rest)
    nw = h->opt.small_warps;
    wpc = std::min(wpc, std::max(1, small_max_warps(mi, nw) / nw));
    if (nw > 1) wpc = std::min(wpc, 15);
  }
  int64_t grid = (C + wpc - 1) / wpc;
  if (grid > sms) grid = sms;  // one CTA per SM (A per CTA); groups loop over their chains
  *wpc_out = wpc;
  *nw_out = nw;
  *grid_out = (int)grid;
  return true;
}

tmvn_status run_small(tmvn_ctx* h, int64_t C, int64_t n_iter, uint64_t seed, int wpc, int nw, int grid,
                      int64_t* n_recorded) {
  cudaStream_t st = stream_of(h);
  SmallParams p;
  std::memset(&p, 0, sizeof(p));
  p.A = h->A_row;
  p.b = h->b_eff;
  p.m = (int)h->m;
  p.d = (int)h->d;
  p.d_pad = h->d_pad;
  p.X = h->X;
  p.C = (int)C;
  p.chain_offset = (uint32_t)h->opt.chain_offset;
  p.seed = seed;
  p.t0 = (uint32_t)h->opt.iter_offset;
  p.n_iter = (int)n_iter;
  p.K = h->opt.recompute_every < 1 ? 1 : h->opt.recompute_every;
  p.eps = h->opt.trim_eps;
  p.record = h->opt.record;
  p.burn_in = h->opt.burn_in;
  p.thin = h->opt.thin;
  p.S1 = h->S1;
  p.S2 = h->S2;
  p.rej = h->rej;
  p.startflag = h->dflag;
  CK(h, cudaMemsetAsync(h->dflag, 0xff, sizeof(unsigned long long), st));
  if (h->opt.small_warps > small_rows((int)h->m))
    return fail(h, TMVN_E_ARG, "options.small_warps exceeds the rows of A per warp (ceil(m / 32) rounded up to a power of two)");
  KL(h, launch_small(p, wpc, nw, grid, st));
  unsigned long long* fp = reinterpret_cast<unsigned long long*>(h->pin);
  CK(h, cudaMemcpyAsync(fp, h->dflag, sizeof(*fp), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  const unsigned long long flag = *fp;
  if (flag != ~0ull) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "infeasible start: chain %lld violates constraint %lld (a_i . x0 >= b_i; the start "
             "must be strictly interior)",
             (long long)(flag / h->m), (long long)(flag % h->m));
    return fail(h, TMVN_E_INFEASIBLE_START, buf);
  }
  int64_t nrec = 0;
  for (int64_t it = 0; it < n_iter; ++it) nrec += recorded_iter(h->opt, h->opt.iter_offset + it) ? 1 : 0;
  *n_recorded = nrec;
  h->prof.warp_mode_calls += 1;
  return TMVN_OK;
}

// returns TMVN_OK with *overflow = true (nothing usable written) when some iteration had
// more live arcs than the capacity: the caller restores X and runs the default path
tmvn_status run_latency(tmvn_ctx* h, int64_t C, int64_t n_iter, uint64_t seed, int cs, int cap, int gsz,
                        bool check_start, int64_t* n_recorded, bool* overflow) {
  cudaStream_t st = stream_of(h);
  if (!h->A_pad) {
    CK(h, dalloc(&h->A_pad, (size_t)(h->m * h->d_pad)));
    CK(h, cudaMemsetAsync(h->A_pad, 0, (size_t)(h->m * h->d_pad) * sizeof(double), st));
    CK(h, cudaMemcpy2DAsync(h->A_pad, (size_t)h->d_pad * sizeof(double), h->A_row, (size_t)h->d * sizeof(double),
                            (size_t)h->d * sizeof(double), (size_t)h->m, cudaMemcpyDeviceToDevice, st));
  }
  LatParams p;
  std::memset(&p, 0, sizeof(p));
  if (h->opt.precision == 1) {
    if (!h->A32) {
      CK(h, dalloc(&h->A32, (size_t)(h->m * h->d_pad)));
      KL(h, launch_to_f32(h->A_row, h->m, h->d, h->d, h->A32, h->d_pad, st));
    }
    if (!h->b32) CK(h, dalloc(&h->b32, (size_t)h->m));
    KL(h, launch_to_f32(h->b_eff, 1, h->m, h->m, h->b32, h->m, st));  // b' may change (set_affine)
    p.fp32 = 1;
    p.A32 = h->A32;
    p.b32 = h->b32;
  }
  p.A = h->A_pad;
  p.b = h->b_eff;
  p.m = (int)h->m;
  p.d = (int)h->d;
  p.d_pad = h->d_pad;
  p.X = h->X;
  p.C = (int)C;
  p.chain_offset = (uint32_t)h->opt.chain_offset;
  p.seed = seed;
  p.t0 = (uint32_t)h->opt.iter_offset;
  p.n_iter = (int)n_iter;
  p.K = h->opt.recompute_every < 1 ? 1 : h->opt.recompute_every;
  p.eps = h->opt.trim_eps;
  p.record = h->opt.record;
  p.burn_in = h->opt.burn_in;
  p.thin = h->opt.thin;
  p.S1 = h->S1;
  p.S2 = h->S2;
  p.rej = h->rej;
  p.cap = cap;
  p.gsz = gsz;
  if (gsz > 0) {  // grid-mode exchange scratch (zeroed: counters, flags)
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t n_tab = (size_t)C * gsz * 128, n_mrg = (size_t)C * 128;
    const size_t b_tg = al(n_tab * 8), b_tc = al(n_tab * 4), b_mg = al(n_mrg * 8), b_mc = al(n_mrg * 4);
    const size_t b_live = al((size_t)C * cap * 16), b_small = al((size_t)C * 2 * 8);
    const size_t b_nu = al((size_t)C * h->d_pad * 8);
    const size_t total = 2 * b_tg + b_tc + 2 * b_mg + b_mc + b_live + 4 * b_small + b_nu;
    if (h->lat_gscratch_n < total) {
      dfree(h->lat_gscratch);
      h->lat_gscratch = nullptr;
      h->lat_gscratch_n = 0;
      CK(h, dalloc(&h->lat_gscratch, total));
      h->lat_gscratch_n = total;
    }
    unsigned char* q = h->lat_gscratch;
    p.gtab_g = reinterpret_cast<uint64_t*>(q); q += b_tg;
    p.gtab_a = reinterpret_cast<uint64_t*>(q); q += b_tg;
    p.gtab_c = reinterpret_cast<int*>(q); q += b_tc;
    p.gmrg_g = reinterpret_cast<uint64_t*>(q); q += b_mg;
    p.gmrg_a = reinterpret_cast<uint64_t*>(q); q += b_mg;
    p.gmrg_c = reinterpret_cast<int*>(q); q += b_mc;
    p.glive = reinterpret_cast<double2*>(q); q += b_live;
    unsigned char* zero0 = q;
    p.gcount = reinterpret_cast<int*>(q); q += b_small;
    p.gviol = reinterpret_cast<int*>(q); q += b_small;
    p.gstart = reinterpret_cast<int*>(q); q += b_small;
    CK(h, cudaMemsetAsync(zero0, 0, (size_t)(q - zero0), stream_of(h)));
    p.gth = reinterpret_cast<double*>(q); q += b_small;
    p.gnu = reinterpret_cast<double*>(q); q += b_nu;
  }
  if (!h->dyn) CK(h, dalloc(&h->dyn, (size_t)64 * 16));
  p.err = h->dyn + 64 * 16 - 1;
  CK(h, cudaMemsetAsync(p.err, 0, sizeof(int), st));
  if (check_start) {
    p.startflag = h->dflag;
    CK(h, cudaMemsetAsync(h->dflag, 0xff, sizeof(unsigned long long), st));
  }
  KL(h, launch_latency(p, cs, st));
  int* ep = reinterpret_cast<int*>(h->pin);
  unsigned long long* fp = reinterpret_cast<unsigned long long*>(h->pin + 1);
  *fp = ~0ull;
  CK(h, cudaMemcpyAsync(ep, p.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (check_start) CK(h, cudaMemcpyAsync(fp, h->dflag, sizeof(*fp), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  const int err = *ep;
  const unsigned long long flag = *fp;
  if (flag != ~0ull) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "infeasible start: chain %lld violates constraint %lld (a_i . x0 >= b_i; the start "
             "must be strictly interior)",
             (long long)(flag / h->m), (long long)(flag % h->m));
    return fail(h, TMVN_E_INFEASIBLE_START, buf);
  }
  *overflow = err != 0;
  if (err) return TMVN_OK;
  int64_t nrec = 0;
  for (int64_t it = 0; it < n_iter; ++it) nrec += recorded_iter(h->opt, h->opt.iter_offset + it) ? 1 : 0;
  *n_recorded = nrec;
  return TMVN_OK;
}

tmvn_status tmvn_sample(tmvn_handle h, const double* X0, int64_t C, int64_t n_iter, uint64_t seed,
                        double* out) {
  Nvtx nv("tmvn_sample");
  tmvn_status s = check_sample_args(h, X0, C, n_iter, out);
  if (s != TMVN_OK) return s;
  if ((s = set_device(h)) != TMVN_OK) return s;
  if ((s = ensure_chains(h, C)) != TMVN_OK) return s;
  if ((s = plan_ess(h, C)) != TMVN_OK) return s;
  if ((s = ensure_ozaki(h)) != TMVN_OK) return s;
  if ((s = load_X(h, X0, C)) != TMVN_OK) return s;
  int swpc = 0, snw = 1, sgrid = 0;
  if (n_iter > 0 && small_fits(h, C, &swpc, &snw, &sgrid)) {  // warp mode: the kernel checks the start
    Nvtx nw("warp mode (one warp per chain, all iterations, A in shared memory)");
    if ((s = clear_accumulators(h, n_iter)) != TMVN_OK) return s;
    int64_t nrec = 0;
    if ((s = run_small(h, C, n_iter, seed, swpc, snw, sgrid, &nrec)) != TMVN_OK) return s;
    if ((s = store_X(h, C, out)) != TMVN_OK) return s;
    if ((s = finish_stats(h, C, n_iter, nrec)) != TMVN_OK) return s;
    if (h->opt.auto_advance) h->opt.iter_offset += n_iter;
    return TMVN_OK;
  }
  int lcs = 0, lcap = 0;
  int lgsz = 0;
  const bool lat = n_iter > 0 && latency_fits(h, C, &lcs, &lcap, &lgsz);
  // the FP64 latency kernel checks the start on its own first P = A x0 (no GEMM here)
  const bool kernel_checks = lat && h->opt.precision == 0;
  if (!kernel_checks && (s = start_check(h, C, h->P0)) != TMVN_OK) return s;
  if ((s = clear_accumulators(h, n_iter)) != TMVN_OK) return s;
  int64_t nrec = 0;
  bool done = false;
  if (lat) {
    // X is kept so that an overflowing call can rerun on the default path
    const size_t cd = (size_t)h->C_pad * h->d_pad;
    if (h->Xsnap_n < cd) {
      dfree(h->Xsnap);
      h->Xsnap = nullptr;
      h->Xsnap_n = 0;
      CK(h, dalloc(&h->Xsnap, cd));
      h->Xsnap_n = cd;
    }
    cudaStream_t st = stream_of(h);
    CK(h, cudaMemcpyAsync(h->Xsnap, h->X, cd * sizeof(double), cudaMemcpyDeviceToDevice, st));
    bool overflow = false;
    Nvtx nl("latency mode (all iterations, one launch)");
    if ((s = run_latency(h, C, n_iter, seed, lcs, lcap, lgsz, kernel_checks, &nrec, &overflow)) != TMVN_OK)
      return s;
    done = !overflow;
    h->prof.latency_calls += 1;
    h->prof.latency_grid_calls += lgsz > 0 ? 1 : 0;
    h->prof.latency_fallbacks += overflow ? 1 : 0;
    if (overflow) {
      CK(h, cudaMemcpyAsync(h->X, h->Xsnap, cd * sizeof(double), cudaMemcpyDeviceToDevice, st));
      if (kernel_checks && (s = start_check(h, C, h->P0)) != TMVN_OK) return s;  // P0 for run_loop
      if ((s = clear_accumulators(h, n_iter)) != TMVN_OK) return s;
    }
  }
  if (!done && (s = run_loop(h, C, n_iter, seed, h->P0, &nrec)) != TMVN_OK) return s;
  if ((s = store_X(h, C, out)) != TMVN_OK) return s;
  if ((s = finish_stats(h, C, n_iter, nrec)) != TMVN_OK) return s;
  if (h->opt.auto_advance) h->opt.iter_offset += n_iter;
  return TMVN_OK;
}

tmvn_status tmvn_get_stats(tmvn_handle h, tmvn_stats* st) {
  if (!h || !st) return fail(h, TMVN_E_ARG, "null argument");
  *st = h->stats;
  return TMVN_OK;
}

tmvn_status tmvn_get_moments(tmvn_handle h, double* sum, double* sumsq, int64_t* n) {
  if (!h || !sum || !sumsq || !n) return fail(h, TMVN_E_ARG, "null argument");
  if (set_device(h) != TMVN_OK) return TMVN_E_CUDA;
  CK(h, cudaMemcpy(sum, h->mom_sum.data(), h->d * sizeof(double), cudaMemcpyDefault));
  CK(h, cudaMemcpy(sumsq, h->mom_sq.data(), h->d * sizeof(double), cudaMemcpyDefault));
  *n = h->stats.recorded;
  return TMVN_OK;
}

tmvn_status tmvn_get_profile(tmvn_handle h, tmvn_profile* prof) {
  if (!h || !prof) return fail(h, TMVN_E_ARG, "null argument");
  *prof = h->prof;
  prof->buckets_used = 0;
  if (h->gmode) {  // slot 3 of every shard: the automatic switch's sticky flag
    int g[4 * 16];
    CK(h, cudaMemcpy(g, h->gmode, sizeof(g), cudaMemcpyDeviceToHost));
    int oct = h->opt.buckets == 2 ? 1 : 0;
    for (int s = 0; s < 16; ++s) oct |= g[4 * s + 3];
    prof->buckets_used = oct ? 2 : 1;
  }
  return TMVN_OK;
}

tmvn_status tmvn_reset_stats(tmvn_handle h) {
  if (!h) return fail(nullptr, TMVN_E_ARG, "null handle");
  h->stats = tmvn_stats{};
  h->prof = tmvn_profile{};
  h->prof.oz_guard_ratio = h->oz_ratio;
  std::fill(h->mom_sum.begin(), h->mom_sum.end(), 0.0);
  std::fill(h->mom_sq.begin(), h->mom_sq.end(), 0.0);
  return TMVN_OK;
}

void tmvn_destroy(tmvn_handle h) {
  if (!h) return;
  cudaSetDevice(h->device);
  for (cudaEvent_t e : h->events) cudaEventDestroy(e);
  for (cudaEvent_t e : h->join_events) cudaEventDestroy(e);
  for (cudaStream_t s_ : h->shard_streams) cudaStreamDestroy(s_);
  if (h->fork_event) cudaEventDestroy(h->fork_event);
  for (int i = 0; i < 2; ++i)
    if (h->graph_exec[i]) cudaGraphExecDestroy(h->graph_exec[i]);
  if (h->capture_stream) cudaStreamDestroy(h->capture_stream);
  if (h->rng_stream) cudaStreamDestroy(h->rng_stream);
  if (h->gemm_stream) cudaStreamDestroy(h->gemm_stream);
  if (h->essb_stream) cudaStreamDestroy(h->essb_stream);
  if (h->ev_essb) cudaEventDestroy(h->ev_essb);
  for (cudaEvent_t e : {h->ev_q[0], h->ev_q[1], h->ev_nu[0], h->ev_nu[1], h->ev_nu[2], h->ev_ess,
                        h->ev_join[0], h->ev_join[1]})
    if (e) cudaEventDestroy(e);
  if (h->ev_pre) cudaEventDestroy(h->ev_pre);
  if (h->ev_rng) cudaEventDestroy(h->ev_rng);
  dfree(h->d_tbase);
  dfree(h->dyn);
  free_chain_buffers(h);
  if (h->At != h->A_tiled) dfree(h->At);
  dfree(h->A_tiled); dfree(h->A_row); dfree(h->A_pad); dfree(h->Xsnap); dfree(h->lat_gscratch); dfree(h->cp_tl); dfree(h->cp_arcs); dfree(h->cp_cur); dfree(h->A32); dfree(h->b32); dfree(h->b_orig); dfree(h->b_eff);
  dfree(h->mu); dfree(h->L); dfree(h->L_tiled);
  dfree(h->dflag); dfree(h->dsum); dfree(h->msum); dfree(h->gmode);
  if (h->pin) cudaFreeHost(h->pin);
  dfree(h->As); dfree(h->rowscale);
  delete h;
}

// ---------------------------------------------------------------- test hooks
#define TCK(expr)                                                       \
  do {                                                                  \
    cudaError_t e_ = (expr);                                            \
    if (e_ != cudaSuccess) return cuda_fail(nullptr, e_, #expr);        \
  } while (0)

}  // extern "C"

namespace {
template <typename T>
struct Tmp {
  T* p = nullptr;
  ~Tmp() { if (p) cudaFree(p); }
};
template <typename T>
cudaError_t tmp_in(Tmp<T>& t, const T* src, size_t n) {
  cudaError_t e = cudaMalloc((void**)&t.p, (n ? n : 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  if (src && n) return cudaMemcpy(t.p, src, n * sizeof(T), cudaMemcpyDefault);
  return cudaMemset(t.p, 0, (n ? n : 1) * sizeof(T));
}
template <typename T>
cudaError_t tmp_out(T* dst, const Tmp<T>& t, size_t n) {
  if (!dst || !n) return cudaSuccess;
  return cudaMemcpy(dst, t.p, n * sizeof(T), cudaMemcpyDefault);
}
}  // namespace

extern "C" {

tmvn_status tmvn_test_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
  if (!ctr || !key || !out || n < 0) return fail(nullptr, TMVN_E_ARG, "bad args");
  Tmp<uint32_t> c, k, o;
  TCK(tmp_in(c, ctr, 4 * n)); TCK(tmp_in(k, key, 2 * n)); TCK(tmp_in(o, (const uint32_t*)nullptr, 4 * n));
  TCK(launch_test_philox(c.p, k.p, n, o.p, false, 0));
  TCK(cudaDeviceSynchronize());
  TCK(tmp_out(out, o, 4 * n));
  return TMVN_OK;
}

tmvn_status tmvn_test_curand_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
  if (!ctr || !key || !out || n < 0) return fail(nullptr, TMVN_E_ARG, "bad args");
  Tmp<uint32_t> c, k, o;
  TCK(tmp_in(c, ctr, 4 * n)); TCK(tmp_in(k, key, 2 * n)); TCK(tmp_in(o, (const uint32_t*)nullptr, 4 * n));
  TCK(launch_test_philox(c.p, k.p, n, o.p, true, 0));
  TCK(cudaDeviceSynchronize());
  TCK(tmp_out(out, o, 4 * n));
  return TMVN_OK;
}

tmvn_status tmvn_test_normals(uint64_t seed, uint64_t t, int64_t c0, int64_t C, int64_t d, double* nu,
                              double* u) {
  if (C < 0 || d < 1 || !nu) return fail(nullptr, TMVN_E_ARG, "bad args");
  Tmp<double> dn, du;
  TCK(tmp_in(dn, (const double*)nullptr, (size_t)C * d)); TCK(tmp_in(du, (const double*)nullptr, (size_t)C));
  TCK(launch_test_normals(seed, (uint32_t)t, (uint32_t)c0, (int)C, (int)d, dn.p, du.p, 0));
  TCK(cudaDeviceSynchronize());
  TCK(tmp_out(nu, dn, (size_t)C * d));
  if (u) TCK(tmp_out(u, du, (size_t)C));
  return TMVN_OK;
}

tmvn_status tmvn_test_arcs(const double* p, const double* q, const double* b, int64_t n, double* alpha,
                           double* beta, uint8_t* active) {
  if (!p || !q || !b || !alpha || !beta || !active || n < 0) return fail(nullptr, TMVN_E_ARG, "bad args");
  Tmp<double> dp, dq, db, da, dbe;
  Tmp<uint8_t> dact;
  TCK(tmp_in(dp, p, n)); TCK(tmp_in(dq, q, n)); TCK(tmp_in(db, b, n));
  TCK(tmp_in(da, (const double*)nullptr, n)); TCK(tmp_in(dbe, (const double*)nullptr, n));
  TCK(tmp_in(dact, (const uint8_t*)nullptr, n));
  TCK(launch_test_arcs(dp.p, dq.p, db.p, n, da.p, dbe.p, dact.p, 0));
  TCK(cudaDeviceSynchronize());
  TCK(tmp_out(alpha, da, n)); TCK(tmp_out(beta, dbe, n)); TCK(tmp_out(active, dact, n));
  return TMVN_OK;
}

static int g_test_chain_warps = 0;
static int g_test_bucket_mode = 1;  // the intervals hook: 1 linear level-1 buckets, 2 by octave

tmvn_status tmvn_test_interval_config(int32_t chain_warps, int32_t bucket_mode) {
  if (chain_warps != 0 && chain_warps != 1 && chain_warps != 2 && chain_warps != 4 && chain_warps != 8 &&
      chain_warps != 16)
    return fail(nullptr, TMVN_E_ARG, "chain_warps must be 0, 1, 2, 4, 8 or 16");
  if (bucket_mode != 1 && bucket_mode != 2) return fail(nullptr, TMVN_E_ARG, "bucket_mode must be 1 or 2");
  g_test_chain_warps = chain_warps;
  g_test_bucket_mode = bucket_mode;
  return TMVN_OK;
}

tmvn_status tmvn_test_intervals(const double* alpha, const double* beta, int64_t m, int64_t C,
                                const double* u, double eps, double* seg_lo, double* seg_hi,
                                int64_t seg_cap, int64_t* nseg, double* L, double* theta) {
  if (!alpha || !beta || m < 1 || C < 1 || seg_cap < 0) return fail(nullptr, TMVN_E_ARG, "bad args");
  const size_t cm = (size_t)C * m;
  Tmp<double> da, db, du, dlo, dhi, dL, dth;
  Tmp<int64_t> dns;
  Tmp<double2> gstash, ggaps;
  TCK(tmp_in(da, alpha, cm)); TCK(tmp_in(db, beta, cm));
  TCK(tmp_in(du, u, u ? (size_t)C : 0));
  TCK(tmp_in(dlo, (const double*)nullptr, (size_t)C * seg_cap)); TCK(tmp_in(dhi, (const double*)nullptr, (size_t)C * seg_cap));
  TCK(tmp_in(dL, (const double*)nullptr, (size_t)C)); TCK(tmp_in(dth, (const double*)nullptr, (size_t)C));
  TCK(tmp_in(dns, (const int64_t*)nullptr, (size_t)C));
  const EssLaunch plan = ess_plan((int)C, (int)m, g_test_chain_warps, 0);
  const int grid = plan.grid;
  if (!plan.stash_smem) {
    TCK(tmp_in(gstash, (const double2*)nullptr, (size_t)plan.groups * ess_gstash_stride(m)));
  }
  TCK(tmp_in(ggaps, (const double2*)nullptr, (size_t)plan.groups * (m + 2)));
  EssParams p;
  std::memset(&p, 0, sizeof(p));
  p.m = (int)m;
  p.C = (int)C;
  p.eps = eps;
  p.g_alpha = da.p;
  p.g_beta = db.p;
  p.g_u = u ? du.p : nullptr;
  p.gstash = gstash.p;
  p.ggaps = ggaps.p;
  p.NB = plan.NB;
  p.W = plan.W;
  p.CH = plan.CH;
  p.stash_smem = plan.stash_smem;
  p.bucket_mode = g_test_bucket_mode;
  p.d_seg_lo = seg_cap ? dlo.p : nullptr;
  p.d_seg_hi = dhi.p;
  p.seg_cap = seg_cap;
  p.d_nseg = dns.p;
  p.d_L = dL.p;
  p.d_theta = dth.p;
  TCK(launch_ess_intervals(p, grid, 0));
  TCK(cudaDeviceSynchronize());
  TCK(tmp_out(seg_lo, dlo, (size_t)C * seg_cap)); TCK(tmp_out(seg_hi, dhi, (size_t)C * seg_cap));
  TCK(tmp_out(nseg, dns, (size_t)C)); TCK(tmp_out(L, dL, (size_t)C)); TCK(tmp_out(theta, dth, (size_t)C));
  return TMVN_OK;
}

tmvn_status tmvn_test_gemm(const double* X, int64_t R, const double* W, int64_t S, int64_t K, double* out) {
  if (!X || !W || !out || R < 1 || S < 1 || K < 1) return fail(nullptr, TMVN_E_ARG, "bad args");
  const int64_t Rp = round_up(R, kTileR), Sp = round_up(S, kTileR), Kp = round_up(K, kTileK);
  Tmp<double> dx, dw, xt, wt, o;
  TCK(tmp_in(dx, X, (size_t)R * K)); TCK(tmp_in(dw, W, (size_t)S * K));
  TCK(tmp_in(xt, (const double*)nullptr, (size_t)Rp * Kp)); TCK(tmp_in(wt, (const double*)nullptr, (size_t)Sp * Kp));
  TCK(tmp_in(o, (const double*)nullptr, (size_t)Rp * Sp));
  TCK(launch_pack(dx.p, R, K, K, xt.p, Kp, 0));
  TCK(launch_pack(dw.p, S, K, K, wt.p, Kp, 0));
  TCK(launch_gemm_tn(xt.p, Rp, wt.p, Sp, Kp, o.p, Sp, 0));
  TCK(cudaDeviceSynchronize());
  TCK(cudaMemcpy2D(out, S * sizeof(double), o.p, Sp * sizeof(double), S * sizeof(double), R, cudaMemcpyDefault));
  return TMVN_OK;
}

tmvn_status tmvn_test_ozaki_gemm(const double* X, int64_t R, const double* W, int64_t S, int64_t K,
                                 int32_t slices, double* out) {
  if (!X || !W || !out || R < 1 || S < 1 || K < 1 || K > 4096 || !(slices == 4 || (slices >= 6 && slices <= 8)))
    return fail(nullptr, TMVN_E_ARG, "bad args");
  const int64_t Rp = round_up(R, kTileR), Sp = round_up(S, kTileR), Kp = round_up(K, kTileK);
  const int64_t KB = (K + kOzStepK - 1) / kOzStepK;
  std::vector<double> hx = to_host(X, (size_t)R * K);
  double mx = 0.0;
  for (double v : hx) mx = std::max(mx, std::fabs(v));
  int ex = 0;
  if (mx > 0.0) std::frexp(mx, &ex);  // max |X| < 2^ex
  Tmp<double> dx, dw, xt, wt, o, rs;
  Tmp<int8_t> xs, ws;
  TCK(tmp_in(dx, hx.data(), (size_t)R * K)); TCK(tmp_in(dw, W, (size_t)S * K));
  TCK(tmp_in(xt, (const double*)nullptr, (size_t)Rp * Kp)); TCK(tmp_in(wt, (const double*)nullptr, (size_t)Sp * Kp));
  TCK(tmp_in(o, (const double*)nullptr, (size_t)Rp * Sp)); TCK(tmp_in(rs, (const double*)nullptr, (size_t)Sp));
  TCK(tmp_in(xs, (const int8_t*)nullptr, (size_t)Rp * KB * kOzStepK * slices));
  TCK(tmp_in(ws, (const int8_t*)nullptr, (size_t)Sp * KB * kOzStepK * slices));
  TCK(launch_pack(dx.p, R, K, K, xt.p, Kp, 0));
  TCK(launch_pack(dw.p, S, K, K, wt.p, Kp, 0));
  TCK(launch_oz_slice(wt.p, Sp, K, Kp, slices, KB, 128, 1, 0, ex, ws.p, rs.p, 0));
  TCK(launch_oz_slice(xt.p, Rp, K, Kp, slices, KB, kOzNuRows, 0, ex, 0, xs.p, nullptr, 0));
  TCK(launch_ozaki_gemm(ws.p, Sp, xs.p, Rp, KB, slices, rs.p, o.p, Sp, 0));
  TCK(cudaDeviceSynchronize());
  TCK(cudaMemcpy2D(out, S * sizeof(double), o.p, Sp * sizeof(double), S * sizeof(double), R, cudaMemcpyDefault));
  return TMVN_OK;
}

tmvn_status tmvn_test_step(tmvn_handle h, const double* Xt, int64_t C, uint64_t seed, int64_t t,
                           tmvn_step_dump* dump) {
  if (!h || !Xt || C < 1 || t < 0 || t >= ((int64_t)1 << 32) || !dump) return fail(h, TMVN_E_ARG, "bad args");
  tmvn_status s;
  if ((s = set_device(h)) != TMVN_OK) return s;
  if ((s = ensure_chains(h, C)) != TMVN_OK) return s;
  if ((s = plan_ess(h, C)) != TMVN_OK) return s;
  if ((s = ensure_ozaki(h)) != TMVN_OK) return s;
  cudaStream_t st = stream_of(h);
  const int64_t m = h->m, d = h->d;
  const int grid = h->plan.grid;
  // X_t is given in u-space
  CK(h, cudaMemcpyAsync(h->stage, Xt, (size_t)C * d * sizeof(double), cudaMemcpyDefault, st));
  CK(h, launch_pack(h->stage, C, d, d, h->X, h->d_pad, st));
  // P = X_t A'^T by the production refresh product (int8 digits of X per chain with the
  // int8 projection, FP64 DMMA otherwise), as at the start check and every K iterations
  CK(h, launch_refresh(h, 0, C, h->P0, st));
  CK(h, launch_first_nu(h, C, seed, (uint32_t)t, st));
  {
    const OzArcs ta = arcs_for(h, 0, C, h->P0);
    const bool fa = fuse_arcs(h) && h->arcs;
    CK(h, launch_projection(h, 0, h->C_pad, st, 0, nullptr, false, fa ? &ta : nullptr));
  }
  CK(h, cudaMemsetAsync(h->rej, 0, (size_t)h->C_pad * sizeof(int64_t), st));
  const size_t cm = (size_t)C * m;
  const int64_t cap = dump->seg_cap > 0 ? dump->seg_cap : 0;
  Tmp<double> da, db, dlo, dhi, dL, dth, dsl;
  Tmp<uint8_t> dact;
  Tmp<int64_t> dns;
  Tmp<int32_t> dacc;
  CK(h, tmp_in(da, (const double*)nullptr, cm)); CK(h, tmp_in(db, (const double*)nullptr, cm));
  CK(h, tmp_in(dact, (const uint8_t*)nullptr, cm));
  CK(h, tmp_in(dlo, (const double*)nullptr, (size_t)C * cap)); CK(h, tmp_in(dhi, (const double*)nullptr, (size_t)C * cap));
  CK(h, tmp_in(dL, (const double*)nullptr, (size_t)C)); CK(h, tmp_in(dth, (const double*)nullptr, (size_t)C));
  CK(h, tmp_in(dsl, (const double*)nullptr, (size_t)C));
  CK(h, tmp_in(dns, (const int64_t*)nullptr, (size_t)C)); CK(h, tmp_in(dacc, (const int32_t*)nullptr, (size_t)C));
  // nu, p, q before the step mutates them
  if (dump->nu) {
    CK(h, launch_unpack(h->N, C, d, h->d_pad, h->stage2, st));
    CK(h, cudaMemcpyAsync(dump->nu, h->stage2, (size_t)C * d * sizeof(double), cudaMemcpyDefault, st));
  }
  if (dump->p) CK(h, cudaMemcpy2DAsync(dump->p, m * sizeof(double), h->P0, h->m_pad * sizeof(double), m * sizeof(double), C, cudaMemcpyDefault, st));
  if (dump->q) CK(h, cudaMemcpy2DAsync(dump->q, m * sizeof(double), h->Q, h->m_pad * sizeof(double), m * sizeof(double), C, cudaMemcpyDefault, st));
  if (dump->u) {  // u of block (0, t, c, 1), drawn by the same device function as the step
    Tmp<double> dn, du;
    CK(h, tmp_in(dn, (const double*)nullptr, (size_t)C * d));
    CK(h, tmp_in(du, (const double*)nullptr, (size_t)C));
    CK(h, cudaStreamSynchronize(st));
    CK(h, launch_test_normals(seed, (uint32_t)t, (uint32_t)h->opt.chain_offset, (int)C, (int)d, dn.p, du.p, st));
    CK(h, cudaStreamSynchronize(st));
    CK(h, tmp_out(dump->u, du, (size_t)C));
  }
  EssParams p = base_params(h, (int)C);
  p.P_cur = h->P0;
  p.P_next = h->P1;
  p.Q = h->Q;
  p.seed = seed;
  p.t = (uint32_t)t;
  p.gen_next = 0;
  p.record = 0;
  p.d_alpha = da.p;
  p.d_beta = db.p;
  p.d_active = dact.p;
  p.d_seg_lo = cap ? dlo.p : nullptr;
  p.d_seg_hi = dhi.p;
  p.seg_cap = cap;
  p.d_nseg = dns.p;
  p.d_L = dL.p;
  p.d_theta = dth.p;
  p.d_slack = dsl.p;
  p.d_accept = dacc.p;
  CK(h, launch_ess_step(p, grid, st));
  CK(h, cudaStreamSynchronize(st));
  if (dump->x_next) {
    CK(h, launch_unpack(h->X, C, d, h->d_pad, h->stage2, st));
    CK(h, cudaMemcpyAsync(dump->x_next, h->stage2, (size_t)C * d * sizeof(double), cudaMemcpyDefault, st));
  }
  CK(h, cudaStreamSynchronize(st));
  CK(h, tmp_out(dump->alpha, da, cm)); CK(h, tmp_out(dump->beta, db, cm)); CK(h, tmp_out(dump->active, dact, cm));
  CK(h, tmp_out(dump->seg_lo, dlo, (size_t)C * cap)); CK(h, tmp_out(dump->seg_hi, dhi, (size_t)C * cap));
  CK(h, tmp_out(dump->nseg, dns, (size_t)C)); CK(h, tmp_out(dump->L, dL, (size_t)C));
  CK(h, tmp_out(dump->theta, dth, (size_t)C)); CK(h, tmp_out(dump->max_slack, dsl, (size_t)C));
  CK(h, tmp_out(dump->accept, dacc, (size_t)C));
  return TMVN_OK;
}

tmvn_status tmvn_test_trace(tmvn_handle h, const double* X0, int64_t C, int64_t n_iter, uint64_t seed,
                            const int64_t* chains, int64_t n_trace, double* trace, double* out) {
  if (!h || !chains || n_trace < 1 || !trace) return fail(h, TMVN_E_ARG, "bad args");
  for (int64_t k = 0; k < n_trace; ++k)
    if (chains[k] < 0 || chains[k] >= C) return fail(h, TMVN_E_ARG, "trace chain out of range");
  if (h->affine) return fail(h, TMVN_E_STATE, "trace hook records u-space; unset affine first");
  tmvn_status s = check_sample_args(h, X0, C, n_iter, out);
  if (s != TMVN_OK) return s;
  if ((s = set_device(h)) != TMVN_OK) return s;
  if ((s = ensure_chains(h, C)) != TMVN_OK) return s;
  h->trace_dev = reinterpret_cast<double*>(1);  // plan a single shard
  s = plan_ess(h, C);
  h->trace_dev = nullptr;
  if (s != TMVN_OK) return s;
  if ((s = ensure_ozaki(h)) != TMVN_OK) return s;
  Tmp<int64_t> rows;
  Tmp<double> tr;
  CK(h, tmp_in(rows, chains, (size_t)n_trace));
  CK(h, tmp_in(tr, (const double*)nullptr, (size_t)(n_iter + 1) * n_trace * h->d));
  if ((s = load_X(h, X0, C)) != TMVN_OK) return s;
  CK(h, launch_gather_rows_tiled(h->X, h->d_pad, (int)h->d, rows.p, (int)n_trace, tr.p, stream_of(h)));
  if ((s = start_check(h, C, h->P0)) != TMVN_OK) return s;
  if ((s = clear_accumulators(h, n_iter)) != TMVN_OK) return s;
  h->trace_rows = rows.p;
  h->trace_n = (int)n_trace;
  h->trace_dev = tr.p;
  int64_t nrec = 0;
  s = run_loop(h, C, n_iter, seed, h->P0, &nrec);
  h->trace_dev = nullptr;
  h->trace_rows = nullptr;
  if (s != TMVN_OK) return s;
  if ((s = store_X(h, C, out)) != TMVN_OK) return s;
  if ((s = finish_stats(h, C, n_iter, nrec)) != TMVN_OK) return s;
  CK(h, tmp_out(trace, tr, (size_t)(n_iter + 1) * n_trace * h->d));
  if (h->opt.auto_advance) h->opt.iter_offset += n_iter;
  return TMVN_OK;
}

// ---- constraint-parallel iterations (cp.cu) ---------------------------
tmvn_status tmvn_cp_begin(tmvn_handle h, const double* X0, int64_t C, int64_t n_iter, uint64_t seed) {
  tmvn_status s = check_sample_args(h, X0, C, n_iter, X0);
  if (s != TMVN_OK) return s;
  if (h->affine) return fail(h, TMVN_E_ARG, "constraint-parallel iterations: no affine change of variable");
  if (h->opt.precision != 0) return fail(h, TMVN_E_ARG, "constraint-parallel iterations are FP64 only (precision 0)");
  if ((s = set_device(h)) != TMVN_OK) return s;
  if ((s = ensure_chains(h, C)) != TMVN_OK) return s;
  if ((s = ensure_ozaki(h)) != TMVN_OK) return s;
  if ((s = load_X(h, X0, C)) != TMVN_OK) return s;
  if ((s = start_check(h, C, h->P0)) != TMVN_OK) return s;  // this rank's rows
  if ((s = clear_accumulators(h, n_iter)) != TMVN_OK) return s;
  if (h->cp_rows < h->C_pad) {  // scratch kept across calls (re-allocated only to grow)
    dfree(h->cp_tl);
    dfree(h->cp_arcs);
    dfree(h->cp_cur);
    h->cp_tl = nullptr;
    h->cp_arcs = nullptr;
    h->cp_cur = nullptr;
    h->cp_rows = 0;
    CK(h, dalloc(&h->cp_tl, (size_t)2 * h->C_pad));
    CK(h, dalloc(&h->cp_arcs, (size_t)h->C_pad * h->m_pad));
    CK(h, dalloc(&h->cp_cur, (size_t)h->C_pad));
    h->cp_rows = h->C_pad;
  }
  CK(h, cudaMemsetAsync(h->cp_cur, 0, (size_t)h->C_pad, stream_of(h)));  // P in P0 (start check)
  h->cp_C = C;
  h->cp_seed = seed;
  h->cp_t0 = h->opt.iter_offset;
  h->cp_nrec = 0;
  return TMVN_OK;
}

tmvn_status tmvn_cp_stats(tmvn_handle h, int64_t t, uint64_t* gx, uint64_t* ma, int32_t* cnt) {
  if (!h || !h->cp_C || !gx || !ma || !cnt) return fail(h, TMVN_E_STATE, "tmvn_cp_stats: call tmvn_cp_begin first");
  cudaStream_t st = stream_of(h);
  const int64_t C = h->cp_C;
  KL(h, launch_first_nu(h, C, h->cp_seed, (uint32_t)t, st));  // nu_t (+ digits), every rank alike
  KL(h, launch_projection(h, 0, round_up(C, kTileR), st));    // Q_r = nu A_r^T
  KL(h, launch_cp_stats(h->P0, h->P1, h->cp_cur, h->Q, h->m_pad, h->b_eff, (int)h->m, (int)C, gx, ma, cnt,
                        h->cp_arcs, st));
  return TMVN_OK;
}

tmvn_status tmvn_cp_live(tmvn_handle h, const uint64_t* gx, const uint64_t* ma, const int32_t* cnt, int32_t cap,
                         double* live, int32_t* nlive) {
  if (!h || !h->cp_C || !live || !nlive || cap < 1) return fail(h, TMVN_E_ARG, "tmvn_cp_live: bad arguments");
  KL(h, launch_cp_live(h->cp_arcs, h->m_pad, (int)h->m, (int)h->cp_C, gx, ma, cnt, cap,
                       reinterpret_cast<double2*>(live), nlive, stream_of(h)));
  return TMVN_OK;
}

tmvn_status tmvn_cp_theta(tmvn_handle h, int64_t t, const uint64_t* gx, const uint64_t* ma, const int32_t* cnt,
                          const double* all_live, const int32_t* all_n, int32_t world, int32_t cap, int32_t* flags) {
  if (!h || !h->cp_C || !all_live || !all_n || !flags || world < 1 || cap < 1)
    return fail(h, TMVN_E_ARG, "tmvn_cp_theta: bad arguments");
  {
    int smem_max = 0;
    CK(h, cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    if (cp_theta_smem(world, cap) > (size_t)smem_max) {
      char buf[200];
      snprintf(buf, sizeof(buf), "tmvn_cp_theta: world * cap = %lld live arcs per chain need %zu B of shared "
               "memory (> %d): lower cap to at most %lld", (long long)world * cap, cp_theta_smem(world, cap),
               smem_max, (long long)(((size_t)smem_max - 32) / 48 / (size_t)world));
      return fail(h, TMVN_E_ARG, buf);
    }
  }
  KL(h, launch_cp_theta(gx, ma, cnt, reinterpret_cast<const double2*>(all_live), all_n, world, cap, h->cp_seed,
                        (uint32_t)t, (uint32_t)h->opt.chain_offset, h->opt.trim_eps, h->P0, h->P1, h->cp_cur,
                        h->Q, h->m_pad, h->b_eff, (int)h->m, (int)h->cp_C, flags, h->cp_tl, h->cp_tl + h->C_pad,
                        stream_of(h)));
  return TMVN_OK;
}

tmvn_status tmvn_cp_commit(tmvn_handle h, int64_t t, const int32_t* flags) {
  if (!h || !h->cp_C || !flags) return fail(h, TMVN_E_ARG, "tmvn_cp_commit: bad arguments");
  cudaStream_t st = stream_of(h);
  const bool rec = recorded_iter(h->opt, t);
  h->cp_nrec += rec ? 1 : 0;
  KL(h, launch_cp_commit(flags, h->cp_tl, h->cp_tl + h->C_pad, h->X, h->N, h->d_pad, (int)h->d, h->cp_cur,
                         (int)h->cp_C, rec ? 1 : 0, h->S1, h->S2, h->rej, st));
  const int64_t K = h->opt.recompute_every < 1 ? 1 : h->opt.recompute_every;
  if ((t + 1) % K == 0) {  // C13: fresh P = X A_r^T into P0 for every chain
    KL(h, launch_refresh(h, 0, h->cp_C, h->P0, st));
    CK(h, cudaMemsetAsync(h->cp_cur, 0, (size_t)h->C_pad, st));
  }
  return TMVN_OK;
}

tmvn_status tmvn_cp_end(tmvn_handle h, int64_t n_iter, double* out) {
  if (!h || !h->cp_C || !out) return fail(h, TMVN_E_ARG, "tmvn_cp_end: bad arguments");
  tmvn_status s;
  const int64_t C = h->cp_C;
  if ((s = store_X(h, C, out)) != TMVN_OK) return s;
  if ((s = finish_stats(h, C, n_iter, h->cp_nrec)) != TMVN_OK) return s;
  if (h->opt.auto_advance) h->opt.iter_offset = h->cp_t0 + n_iter;
  h->cp_C = 0;
  return TMVN_OK;
}

tmvn_status tmvn_test_latency_grid(tmvn_handle h, int32_t mode) {
  if (!h || mode < -1 || mode > 1) return fail(h, TMVN_E_ARG, "latency grid mode must be -1, 0 or 1");
  h->lat_grid_mode = mode;
  h->lat_memo_C = -1;
  return TMVN_OK;
}
tmvn_status tmvn_test_latency_cap(tmvn_handle h, int32_t cap) {
  if (!h || cap < 0) return fail(h, TMVN_E_ARG, "latency cap must be >= 0");
  h->lat_cap_max = cap;
  return TMVN_OK;
}

#ifdef TMVN_PHASE_TIMING
// timing build only (tools/phase_timing.py): per-phase CTA cycles of ess_kernel
tmvn_status tmvn_test_phase_cycles(uint64_t* out10, int reset) {
  tmvn::phase_cycles(reinterpret_cast<unsigned long long*>(out10), reset != 0);
  return TMVN_OK;
}
tmvn_status tmvn_test_lat_cycles(uint64_t* out16, int reset) {
  tmvn::lat_cycles(reinterpret_cast<unsigned long long*>(out16), reset != 0);
  return TMVN_OK;
}
tmvn_status tmvn_test_oz_cycles(uint64_t* out10, int reset) {
  tmvn::oz_cycles(reinterpret_cast<unsigned long long*>(out10), reset != 0);
  return TMVN_OK;
}
#endif

#ifdef TMVN_TIMELINE
// timeline build only (tools/timeline.py): reset / read the per-launch timestamps
tmvn_status tmvn_test_timeline(uint64_t* out, int reset) {
  std::vector<unsigned long long> g(256 * 4), e(256 * 4);
  tmvn::tl_access_gemm(g.data(), reset != 0);
  tmvn::tl_access_ess(e.data(), reset != 0);
  if (!reset)
    for (int i = 0; i < 256; ++i) {
      out[i * 4 + 0] = g[i * 4 + 0];
      out[i * 4 + 1] = g[i * 4 + 1];
      out[i * 4 + 2] = e[i * 4 + 2];
      out[i * 4 + 3] = e[i * 4 + 3];
    }
  return TMVN_OK;
}
#endif
}  // extern "C"
