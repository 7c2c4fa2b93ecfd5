// =============================================================================
// oracle/oracle.cpp -- CPU ORACLE FOR arXiv 2407.10449 (linear elliptical slice
// sampling of a polytope-truncated standard normal).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// The product path (paper_2407_10449_b200/) never links, loads or calls it,
// and this file shares no code, header, table or helper with the CUDA path.
//
// It is a plain, slow, obviously-correct implementation in FP64:
//   * no blocking, no fusion, no reordering beyond the paper's definitions;
//   * dot products are sequential loops in index order (no BLAS);
//   * I_act is computed BY DEFINITION with the brute-force Alg. 2, never with
//     the sort + cumulative-max of Alg. 3 (Prop. 1 says both give the same set);
//   * built with -O2 -ffp-contract=off, never -ffast-math.
//
// Citations: "P:n" = /root/reference/PAPER.md line n; "C<k>" = the reading
// numbered k in DESIGN.md section "Readings" (same numbering as SURVEY 8(c)).
//
// Pins (tests/test_oracle_*.py, run with -m "not gpu"):
//   philox       -> Random123 known-answer vectors + cuRAND's own host Philox
//   normals      -> distribution tests (mean, variance, KS) -- textbook
//   arc          -> Fig. 1 / Fig. 2 printed data, Eq. 2 residual, sign scan
//   intervals    -> Fig. 1 caption, App. "Brute Force" closed form, sorting
//                   reduction (S3.1), dense-theta-grid membership
//   sample_theta -> closed forms + chi-square uniformity
//   step / run   -> 1-D truncated-normal closed-form moments (S4.1 table),
//                   orthant half-normal moments, 2-D rejection sampling,
//                   unconstrained N(0,I), Ax <= b at every iterate
//   whitening    -> App. A closed-form example + round trip
// No function here is "parity unpinned".
// =============================================================================
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// 2*pi rounded to double (C12; also the right end of [0, 2*pi]).
const double kTwoPi = 6.283185307179586;

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written out round by
// round.  Counter (x, y, z, w), key (k0, k1).  C12.
// ---------------------------------------------------------------------------
const uint32_t kPhiloxM0 = 0xD2511F53u;
const uint32_t kPhiloxM1 = 0xCD9E8D57u;
const uint32_t kPhiloxW0 = 0x9E3779B9u;
const uint32_t kPhiloxW1 = 0xBB67AE85u;

void philox_round(uint32_t c[4], const uint32_t k[2]) {
  uint64_t prod0 = (uint64_t)kPhiloxM0 * (uint64_t)c[0];
  uint64_t prod1 = (uint64_t)kPhiloxM1 * (uint64_t)c[2];
  uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
  uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
  uint32_t n0 = hi1 ^ c[1] ^ k[0];
  uint32_t n1 = lo1;
  uint32_t n2 = hi0 ^ c[3] ^ k[1];
  uint32_t n3 = lo0;
  c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int round = 0; round < 10; ++round) {
    philox_round(c, k);
    k[0] += kPhiloxW0;
    k[1] += kPhiloxW1;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// The Philox block for (j, t, c, s) under `seed` (C12).
void philox_block(uint64_t seed, uint32_t j, uint64_t t, uint64_t c, uint32_t s, uint32_t w[4]) {
  uint32_t ctr[4] = {j, (uint32_t)t, (uint32_t)c, s};
  uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  philox4x32_10(ctr, key, w);
}

// 53-bit uniform in [0, 1) from two 32-bit words (C12).
double uniform53(uint32_t lo, uint32_t hi) {
  uint64_t bits = ((uint64_t)hi << 32) | (uint64_t)lo;
  return (double)(bits >> 11) * (1.0 / 9007199254740992.0);  // 2^-53
}

// nu_{c,t} ~ N(0, I_d): Box-Muller on block (j, t, c, 0) for pair j (C12;
// Alg. 1 line "sample nu_t ~ N(0, I)").
void normals(uint64_t seed, uint64_t t, uint64_t c, int64_t d, double* nu) {
  for (int64_t j = 0; 2 * j < d; ++j) {
    uint32_t w[4];
    philox_block(seed, (uint32_t)j, t, c, 0u, w);
    double ua = uniform53(w[0], w[1]);
    double ub = uniform53(w[2], w[3]);
    double radius = std::sqrt(-2.0 * std::log(1.0 - ua));
    double phi = kTwoPi * ub;
    nu[2 * j] = radius * std::cos(phi);
    if (2 * j + 1 < d) nu[2 * j + 1] = radius * std::sin(phi);
  }
}

// u_{c,t} ~ U[0, 1) for "sample uniformly theta ~ I_act": U_a of block (0, t, c, 1).
double uniform_u(uint64_t seed, uint64_t t, uint64_t c) {
  uint32_t w[4];
  philox_block(seed, 0u, t, c, 1u, w);
  return uniform53(w[0], w[1]);
}

// ---------------------------------------------------------------------------
// Roots of Eq. 2 by the recommended formula eq:roots:
//   r = hypot(p, q); tau = atan2(q, p); delta = arccos(b / r);
//   roots tau -/+ delta; infeasible arc (alpha, beta) = (tau - delta, tau + delta)
// normalised into [0, 2*pi] by C1.  Inactive (padding) iff r <= b (C3).
// Returns 1 if active, 0 if inactive.
// ---------------------------------------------------------------------------
int arc(double p, double q, double b, double* alpha, double* beta) {
  double r = std::hypot(p, q);           // C25
  if (!(r > b)) {                        // C3 / C4: no root or tangent from inside
    *alpha = 0.0; *beta = 0.0;
    return 0;
  }
  double rho = b / r;
  if (rho < -1.0) rho = -1.0;            // C5 clamp
  if (rho > 1.0) rho = 1.0;
  double tau = std::atan2(q, p);         // tau in [-pi, pi]
  double delta = std::acos(rho);         // delta in [0, pi]
  double lo = tau - delta;
  double hi = tau + delta;
  // C1: add a multiple of 2*pi so the arc lies in [0, 2*pi].
  if (hi <= 0.0) {
    lo = lo + kTwoPi;
    hi = hi + kTwoPi;
  } else if (lo >= 0.0) {
    // already inside [0, 2*pi]
  } else {
    // straddles theta = 0: only possible through rounding for feasible x_t (C1)
    if (-lo <= hi) { lo = 0.0; }
    else { lo = lo + kTwoPi; hi = kTwoPi; }
  }
  *alpha = lo;
  *beta = hi;
  return 1;
}

// ---------------------------------------------------------------------------
// Alg. 2: I_act^(0) = [0, 2pi]; I_act^(i) = I_act^(i-1) cap
// ([0, alpha_i] cup [beta_i, 2pi]).  Output in canonical form: zero-length
// segments dropped, touching segments merged (C19/C20, P4).
// ---------------------------------------------------------------------------
struct Seg { double lo, hi; };

void intervals_alg2(const double* alpha, const double* beta, const uint8_t* active, int64_t m,
                    std::vector<Seg>& out) {
  std::vector<Seg> cur, nxt;
  cur.push_back(Seg{0.0, kTwoPi});
  for (int64_t i = 0; i < m; ++i) {
    if (active && !active[i]) continue;   // padding pairs are no-ops
    double a = alpha[i], b = beta[i];
    nxt.clear();
    for (const Seg& s : cur) {
      if (s.lo <= a) {
        Seg piece{s.lo, std::min(s.hi, a)};
        if (piece.hi > piece.lo) nxt.push_back(piece);
      }
      if (b <= s.hi) {
        Seg piece{std::max(s.lo, b), s.hi};
        if (piece.hi > piece.lo) nxt.push_back(piece);
      }
    }
    cur.swap(nxt);
  }
  // canonical form: drop zero-length (already done), merge touching segments
  out.clear();
  for (const Seg& s : cur) {
    if (!out.empty() && out.back().hi == s.lo) out.back().hi = s.hi;
    else out.push_back(s);
  }
}

// S3.3 trimming with reading C7.
void trim(const std::vector<Seg>& in, double eps, std::vector<Seg>& out) {
  out.clear();
  if (!(eps > 0.0)) { out = in; return; }
  for (const Seg& s : in) {
    double lo = (s.lo == 0.0) ? 0.0 : s.lo + eps;
    double hi = (s.hi == kTwoPi) ? kTwoPi : s.hi - eps;
    if (hi > lo) out.push_back(Seg{lo, hi});
  }
  if (out.empty()) out = in;
}

// "sample uniformly theta ~ I_act" by the inverse CDF over the
// segments in ascending order (C10).  Returns L; theta via *theta.
double sample_theta(const std::vector<Seg>& segs, double u, double* theta) {
  double total = 0.0;
  for (const Seg& s : segs) total = total + (s.hi - s.lo);
  if (!(total > 0.0)) { *theta = 0.0; return total; }
  double target = u * total;
  double before = 0.0;   // S_{k-1}
  for (size_t k = 0; k < segs.size(); ++k) {
    double after = before + (segs[k].hi - segs[k].lo);   // S_k
    // first k with S_k > u*L; the last segment if u*L rounded up to L (C10)
    if (after > target || k + 1 == segs.size()) {
      *theta = segs[k].lo + (target - before);
      return total;
    }
    before = after;
  }
  *theta = 0.0;
  return total;
}

double dot(const double* a, const double* x, int64_t d) {
  double s = 0.0;
  for (int64_t j = 0; j < d; ++j) s = s + a[j] * x[j];
  return s;
}

}  // namespace

extern "C" {

// Per-step dump (P6 parity, O10).  Any pointer may be NULL.
typedef struct {
  double* nu;        // d
  double* u;         // 1
  double* p;         // m   A x_t
  double* q;         // m   A nu
  double* alpha;     // m
  double* beta;      // m
  uint8_t* active;   // m
  double* seg_lo;    // seg_cap
  double* seg_hi;    // seg_cap
  int64_t seg_cap;
  int64_t* nseg;     // 1   (canonical, untrimmed count)
  double* L;         // 1   (after trimming)
  double* theta;     // 1
  double* x_prop;    // d   proposed x' (before the safeguard)
  double* max_slack; // 1   max_i (a_i x' - b_i), fresh
  int32_t* accept;   // 1
} orc_dump;

void orc_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  philox4x32_10(ctr, key, out);
}

void orc_philox_block(uint64_t seed, uint32_t j, uint64_t t, uint64_t c, uint32_t s, uint32_t* w) {
  philox_block(seed, j, t, c, s, w);
}

void orc_normals(uint64_t seed, uint64_t t, uint64_t c, int64_t d, double* nu) {
  normals(seed, t, c, d, nu);
}

double orc_uniform(uint64_t seed, uint64_t t, uint64_t c) { return uniform_u(seed, t, c); }

// Batched arcs: n triples (p, q, b) -> (alpha, beta, active).
void orc_arcs(const double* p, const double* q, const double* b, int64_t n,
              double* alpha, double* beta, uint8_t* active) {
  for (int64_t i = 0; i < n; ++i) active[i] = (uint8_t)arc(p[i], q[i], b[i], &alpha[i], &beta[i]);
}

// Alg. 2 on one chain's pairs.  Returns the number of canonical segments
// (may exceed cap; only min(cap, n) are written).
int64_t orc_intervals(const double* alpha, const double* beta, const uint8_t* active, int64_t m,
                      double* seg_lo, double* seg_hi, int64_t cap) {
  std::vector<Seg> segs;
  intervals_alg2(alpha, beta, active, m, segs);
  for (int64_t k = 0; k < (int64_t)segs.size() && k < cap; ++k) {
    seg_lo[k] = segs[k].lo;
    seg_hi[k] = segs[k].hi;
  }
  return (int64_t)segs.size();
}

// Segment count of the running set after each constraint (App. "Brute Force").
void orc_intervals_trace(const double* alpha, const double* beta, int64_t m, int64_t* counts) {
  std::vector<Seg> cur, nxt;
  cur.push_back(Seg{0.0, kTwoPi});
  for (int64_t i = 0; i < m; ++i) {
    nxt.clear();
    for (const Seg& s : cur) {
      if (s.lo <= alpha[i]) { Seg pc{s.lo, std::min(s.hi, alpha[i])}; if (pc.hi > pc.lo) nxt.push_back(pc); }
      if (beta[i] <= s.hi) { Seg pc{std::max(s.lo, beta[i]), s.hi}; if (pc.hi > pc.lo) nxt.push_back(pc); }
    }
    cur.swap(nxt);
    counts[i] = (int64_t)cur.size();
  }
}

int64_t orc_trim(const double* lo, const double* hi, int64_t n, double eps, double* out_lo,
                 double* out_hi) {
  std::vector<Seg> in, out;
  for (int64_t k = 0; k < n; ++k) in.push_back(Seg{lo[k], hi[k]});
  trim(in, eps, out);
  for (size_t k = 0; k < out.size(); ++k) { out_lo[k] = out[k].lo; out_hi[k] = out[k].hi; }
  return (int64_t)out.size();
}

double orc_sample_theta(const double* lo, const double* hi, int64_t n, double u, double* L) {
  std::vector<Seg> segs;
  for (int64_t k = 0; k < n; ++k) segs.push_back(Seg{lo[k], hi[k]});
  double theta = 0.0;
  *L = segs.empty() ? 0.0 : sample_theta(segs, u, &theta);
  return theta;
}

// One step of Alg. 1 for global chain c at iteration t, with the
// S3.3 safeguard (tol 0, C8) and C9 for L = 0.
// x is d; x_next receives x_{t+1} (= x_t if rejected).  Returns 1 accepted,
// 0 rejected (safeguard or L = 0).
int orc_step(const double* A, const double* b, int64_t m, int64_t d, const double* x,
             uint64_t seed, uint64_t t, uint64_t c, double eps, double* x_next, orc_dump* dump) {
  std::vector<double> nu(d), p(m), q(m), alpha(m), beta(m), xp(d);
  std::vector<uint8_t> active(m);
  normals(seed, t, c, d, nu.data());                                  // O1
  double u = uniform_u(seed, t, c);
  for (int64_t i = 0; i < m; ++i) {                                   // O2
    p[i] = dot(A + i * d, x, d);
    q[i] = dot(A + i * d, nu.data(), d);
  }
  for (int64_t i = 0; i < m; ++i)                                     // O3
    active[i] = (uint8_t)arc(p[i], q[i], b[i], &alpha[i], &beta[i]);
  std::vector<Seg> segs, tsegs;
  intervals_alg2(alpha.data(), beta.data(), active.data(), m, segs);  // O4
  trim(segs, eps, tsegs);                                             // O5
  double theta = 0.0;
  double L = tsegs.empty() ? 0.0 : sample_theta(tsegs, u, &theta);    // O6, O7
  int accept = 0;
  double max_slack = 0.0;
  if (L > 0.0) {
    double ct = std::cos(theta), st = std::sin(theta);
    for (int64_t j = 0; j < d; ++j) xp[j] = x[j] * ct + nu[j] * st;   // O8, Eq. 1
    max_slack = -INFINITY;
    for (int64_t i = 0; i < m; ++i) {                                 // O9
      double s = dot(A + i * d, xp.data(), d) - b[i];
      if (s > max_slack) max_slack = s;
    }
    accept = (m == 0 || max_slack <= 0.0) ? 1 : 0;
  } else {
    for (int64_t j = 0; j < d; ++j) xp[j] = x[j];
  }
  for (int64_t j = 0; j < d; ++j) x_next[j] = accept ? xp[j] : x[j];
  if (dump) {
    if (dump->nu) std::memcpy(dump->nu, nu.data(), sizeof(double) * d);
    if (dump->u) *dump->u = u;
    if (dump->p) std::memcpy(dump->p, p.data(), sizeof(double) * m);
    if (dump->q) std::memcpy(dump->q, q.data(), sizeof(double) * m);
    if (dump->alpha) std::memcpy(dump->alpha, alpha.data(), sizeof(double) * m);
    if (dump->beta) std::memcpy(dump->beta, beta.data(), sizeof(double) * m);
    if (dump->active) std::memcpy(dump->active, active.data(), m);
    if (dump->nseg) *dump->nseg = (int64_t)segs.size();
    for (int64_t k = 0; k < (int64_t)segs.size() && k < dump->seg_cap; ++k) {
      if (dump->seg_lo) dump->seg_lo[k] = segs[k].lo;
      if (dump->seg_hi) dump->seg_hi[k] = segs[k].hi;
    }
    if (dump->L) *dump->L = L;
    if (dump->theta) *dump->theta = theta;
    if (dump->x_prop) std::memcpy(dump->x_prop, xp.data(), sizeof(double) * d);
    if (dump->max_slack) *dump->max_slack = max_slack;
    if (dump->accept) *dump->accept = accept;
  }
  return accept;
}

// App. A: A' = A L, b' = b - A mu.  L is d x d lower-triangular
// row-major (may be NULL = I); mu is d (may be NULL = 0).
void orc_whiten(const double* A, const double* b, int64_t m, int64_t d, const double* mu,
                const double* L, double* A_out, double* b_out) {
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < d; ++j) {
      double s = 0.0;
      if (L) { for (int64_t k = 0; k < d; ++k) s = s + A[i * d + k] * L[k * d + j]; }
      else s = A[i * d + j];
      A_out[i * d + j] = s;
    }
    b_out[i] = b[i] - (mu ? dot(A + i * d, mu, d) : 0.0);
  }
}

// u = L^{-1} (x - mu) by forward substitution.
void orc_whiten_point(const double* x, int64_t d, const double* mu, const double* L, double* u) {
  for (int64_t j = 0; j < d; ++j) {
    double s = x[j] - (mu ? mu[j] : 0.0);
    if (L) {
      for (int64_t k = 0; k < j; ++k) s = s - L[j * d + k] * u[k];
      s = s / L[j * d + j];
    }
    u[j] = s;
  }
}

// x = L u + mu.
void orc_unwhiten_point(const double* u, int64_t d, const double* mu, const double* L, double* x) {
  for (int64_t j = 0; j < d; ++j) {
    double s = 0.0;
    if (L) { for (int64_t k = 0; k <= j; ++k) s = s + L[j * d + k] * u[k]; }
    else s = u[j];
    x[j] = s + (mu ? mu[j] : 0.0);
  }
}

// Many chains: chain k (0-based, local) has global index
// chain_offset + k and runs iterations t = iter_offset .. iter_offset+n_iter-1.
// (A, b) are the (already whitened, if any) constraints in u-space; X0/X_out
// are u-space C x d row-major.  If mu/L are given, moments are accumulated in
// x-space (x = L u + mu).  An iterate x_{t+1} is recorded iff
// t >= burn_in and (t - burn_in) % thin == 0 (S4.1 protocol).
// sum/sumsq (d) and n_rec/rejections (1) are written if non-NULL; per_chain_rej
// (C) if non-NULL.  nthreads <= 0 = OpenMP default.
void orc_run(const double* A, const double* b, int64_t m, int64_t d, const double* X0, int64_t C,
             int64_t n_iter, uint64_t seed, int64_t chain_offset, int64_t iter_offset, double eps,
             int64_t burn_in, int64_t thin, const double* mu, const double* L, double* X_out,
             double* sum, double* sumsq, int64_t* n_rec, int64_t* rejections,
             int64_t* per_chain_rej, int nthreads) {
  std::vector<double> csum((size_t)C * d, 0.0), csq((size_t)C * d, 0.0);
  std::vector<int64_t> crec(C, 0), crej(C, 0);
  if (thin < 1) thin = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t k = 0; k < C; ++k) {
    std::vector<double> x(X0 + k * d, X0 + (k + 1) * d), xn(d), xo(d);
    for (int64_t it = 0; it < n_iter; ++it) {
      uint64_t t = (uint64_t)(iter_offset + it);
      int acc = orc_step(A, b, m, d, x.data(), seed, t, (uint64_t)(chain_offset + k), eps,
                         xn.data(), nullptr);
      if (!acc) crej[k] += 1;
      x.swap(xn);
      int64_t tt = (int64_t)t;
      if (tt >= burn_in && ((tt - burn_in) % thin) == 0) {
        if (mu || L) orc_unwhiten_point(x.data(), d, mu, L, xo.data());
        else xo = x;
        for (int64_t j = 0; j < d; ++j) {
          csum[k * d + j] = csum[k * d + j] + xo[j];
          csq[k * d + j] = csq[k * d + j] + xo[j] * xo[j];
        }
        crec[k] += 1;
      }
    }
    std::memcpy(X_out + k * d, x.data(), sizeof(double) * d);
  }
  // deterministic reduction in chain order
  if (sum) for (int64_t j = 0; j < d; ++j) { double s = 0.0; for (int64_t k = 0; k < C; ++k) s = s + csum[k * d + j]; sum[j] = s; }
  if (sumsq) for (int64_t j = 0; j < d; ++j) { double s = 0.0; for (int64_t k = 0; k < C; ++k) s = s + csq[k * d + j]; sumsq[j] = s; }
  int64_t nr = 0, nj = 0;
  for (int64_t k = 0; k < C; ++k) { nr += crec[k]; nj += crej[k]; }
  if (n_rec) *n_rec = nr;
  if (rejections) *rejections = nj;
  if (per_chain_rej) for (int64_t k = 0; k < C; ++k) per_chain_rej[k] = crej[k];
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
