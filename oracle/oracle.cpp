// oracle.cpp -- CPU ORACLE (TEST INFRASTRUCTURE ONLY; see oracle.h header).
//
// Plain restatement of the reference's hot path. Every function cites the
// reference line(s) it follows. Built with -ffp-contract=off so that no FMA
// contraction changes the op order.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;
thread_local long g_div_iter = -1;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// ---------------------------------------------------------------- rng
// rng.cpp:11 kGolden, rng.cpp:14-18 mix64, rng.cpp:20-22 absorb
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t absorb(uint64_t s, uint64_t v) { return mix64((s + kGolden) ^ v); }
// rng.cpp:26-33 StreamRng constructor
inline uint64_t stream_state(uint64_t seed, uint32_t purpose, uint64_t worker,
                             uint64_t iteration) {
  uint64_t s = mix64(seed + kGolden);
  s = absorb(s, purpose);
  s = absorb(s, worker);
  s = absorb(s, iteration);
  return s;
}
// rng.cpp:35-38: next_u64 does state += kGolden; return mix64(state).
// Draw k (0-based) is therefore mix64(state0 + (k+1)*kGolden).
inline uint64_t draw(uint64_t state0, uint64_t k) { return mix64(state0 + (k + 1) * kGolden); }
// rng.cpp:40-42 next_unit
inline double unit_of(uint64_t u) { return static_cast<double>(u >> 11) * 0x1.0p-53; }
inline float bucket_value(uint64_t u) { return static_cast<float>(2.0 * unit_of(u) - 1.0); }

// ---------------------------------------------------------------- dense matrix
// Eigen-free stand-in for MixingMatrix = Eigen::MatrixXd (topology.hpp:14).
struct Mat {
  int n = 0;
  std::vector<double> a;  // row-major
  explicit Mat(int n_ = 0) : n(n_), a(size_t(n_) * n_, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) * n + j]; }
  double operator()(int i, int j) const { return a[size_t(i) * n + j]; }
};

Mat matmul(const Mat& x, const Mat& y) {
  Mat r(x.n);
  for (int i = 0; i < x.n; ++i)
    for (int k = 0; k < x.n; ++k) {
      const double xik = x(i, k);
      for (int j = 0; j < x.n; ++j) r(i, j) += xik * y(k, j);
    }
  return r;
}

// Cyclic Jacobi eigenvalues of a symmetric matrix (validation only; replaces
// Eigen's SelfAdjointEigenSolver, "symmetric eigendecomposition").
std::vector<double> sym_eigenvalues(Mat a) {
  const int n = a.n;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += a(i, j) * a(i, j);
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (std::fabs(a(p, q)) < 1e-300) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) /
                         (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = a(i, i);
  std::sort(ev.begin(), ev.end(), std::greater<double>());
  return ev;
}

// ---------------------------------------------------------------- validate
// topology.hpp:16-34: each check within 1e-12, eigenvalues in (-1, 1].
or_validation validate_mat(const Mat& w) {
  or_validation r{};
  const int n = w.n;
  const double tol = 1e-12;
  r.min_entry = n ? w(0, 0) : 0.0;
  for (int i = 0; i < n; ++i) {
    double rs = 0.0, cs = 0.0;
    for (int j = 0; j < n; ++j) {
      r.max_asymmetry = std::max(r.max_asymmetry, std::fabs(w(i, j) - w(j, i)));
      r.min_entry = std::min(r.min_entry, w(i, j));
      rs += w(i, j);
      cs += w(j, i);
    }
    r.max_row_error = std::max(r.max_row_error, std::fabs(rs - 1.0));
    r.max_col_error = std::max(r.max_col_error, std::fabs(cs - 1.0));
  }
  r.symmetric = r.max_asymmetry <= tol;
  r.nonnegative = r.min_entry >= -tol;
  r.rows_stochastic = r.max_row_error <= tol;
  r.cols_stochastic = r.max_col_error <= tol;
  // Spectrum of the symmetric part; only meaningful (and only reported as in
  // range) when the input is symmetric.
  Mat sp(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) sp(i, j) = 0.5 * (w(i, j) + w(j, i));
  const auto ev = n ? sym_eigenvalues(sp) : std::vector<double>{};
  r.max_eigenvalue = n ? ev.front() : 0.0;
  r.min_eigenvalue = n ? ev.back() : 0.0;
  r.eigenvalues_in_range =
      r.symmetric && n > 0 && r.min_eigenvalue > -1.0 + 1e-10 && r.max_eigenvalue <= 1.0 + 1e-10;
  return r;
}
bool passes(const or_validation& v) {
  return v.symmetric && v.nonnegative && v.rows_stochastic && v.cols_stochastic &&
         v.eigenvalues_in_range;
}

}  // namespace

// ---------------------------------------------------------------- schedule
// MixingSchedule (topology.hpp:40-63): immutable periodic list of matrices plus
// the derived neighbour lists (w_ij > 0, self included, ascending; :54).
struct or_sched {
  int workers = 0, wpn = 1;
  std::vector<Mat> rounds;
  std::vector<std::vector<std::vector<int>>> nbrs;
};

namespace {

bool is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }
int ilog2(int n) {
  int r = 0;
  while ((1 << r) < n) ++r;
  return r;
}

// from_matrices (topology.hpp:36-45): validate every round and the
// connectivity of the period's union graph.
int build(int n, int wpn, std::vector<Mat> rounds, or_sched** out) {
  if (n < 1) return fail(OR_CONFIG_ERROR, "schedule: workers must be >= 1");
  if (rounds.empty()) return fail(OR_CONFIG_ERROR, "schedule: empty");
  for (size_t r = 0; r < rounds.size(); ++r) {
    if (rounds[r].n != n) return fail(OR_CONFIG_ERROR, "schedule: size mismatch");
    if (!passes(validate_mat(rounds[r])))
      return fail(OR_CONFIG_ERROR, "schedule: round " + std::to_string(r + 1) + " invalid");
  }
  // union-graph connectivity (BFS)
  std::vector<int> seen(n, 0), q{0};
  seen[0] = 1;
  for (size_t h = 0; h < q.size(); ++h)
    for (const Mat& w : rounds)
      for (int j = 0; j < n; ++j)
        if (w(q[h], j) > 0.0 && !seen[j]) seen[j] = 1, q.push_back(j);
  if (int(q.size()) != n) return fail(OR_CONFIG_ERROR, "schedule: union graph disconnected");
  auto* s = new or_sched;
  s->workers = n;
  s->wpn = wpn;
  s->rounds = std::move(rounds);
  for (const Mat& w : s->rounds) {
    std::vector<std::vector<int>> nb(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if (w(i, j) > 0.0) nb[i].push_back(j);
    s->nbrs.push_back(std::move(nb));
  }
  *out = s;
  return OR_OK;
}

// pairwise matching: matched pairs 1/2 each, unmatched keep 1
Mat matching(int n, const std::vector<std::pair<int, int>>& pairs) {
  Mat w(n);
  std::vector<int> matched(n, 0);
  for (auto [a, b] : pairs) {
    w(a, a) = w(b, b) = w(a, b) = w(b, a) = 0.5;
    matched[a] = matched[b] = 1;
  }
  for (int i = 0; i < n; ++i)
    if (!matched[i]) w(i, i) = 1.0;
  return w;
}

// exact group averaging (AER): 1/|G| inside each group
Mat groups(int n, const std::vector<std::vector<int>>& gs) {
  Mat w(n);
  for (const auto& g : gs)
    for (int a : g)
      for (int b : g) w(a, b) = 1.0 / double(g.size());
  return w;
}

// AER merged-pair sequence over M nodes (topology.hpp:73-78; Fig. 9
// PAPER.md:882-1021): M=2 -> (0,1); M=4 -> (2,3),(0,1),(0,2),(1,3);
// M>=8 -> h = 1,2,4..M/2, pairs (j, j+h) with (j & h) == 0, ascending j.
std::vector<std::pair<int, int>> aer_pairs(int M) {
  if (M == 2) return {{0, 1}};
  if (M == 4) return {{2, 3}, {0, 1}, {0, 2}, {1, 3}};
  std::vector<std::pair<int, int>> p;
  for (int h = 1; h < M; h <<= 1)
    for (int j = 0; j < M; ++j)
      if ((j & h) == 0) p.push_back({j, j + h});
  return p;
}

const Mat* round_mat(const or_sched* s, long round) {
  if (!s || s->rounds.empty() || round < 1) return nullptr;
  return &s->rounds[size_t((round - 1) % long(s->rounds.size()))];
}
const std::vector<std::vector<int>>* round_nbrs(const or_sched* s, long round) {
  if (!s || s->rounds.empty() || round < 1) return nullptr;
  return &s->nbrs[size_t((round - 1) % long(s->rounds.size()))];
}

// ---------------------------------------------------------------- optimizer
struct Scalars {  // derived once per step in double
  double b1, omb1, b2, omb2, c1, c2, neg_alpha, eps, inv_s, bv, ombv;
};

int check_cfg(const or_adam_cfg* c) {
  if (!c) return fail(OR_CONFIG_ERROR, "optimizer: null config");
  if (!(c->alpha > 0.0)) return fail(OR_CONFIG_ERROR, "optimizer: alpha must be > 0");
  if (!(c->beta1 >= 0.0 && c->beta1 < c->beta2 && c->beta2 < 1.0))
    return fail(OR_CONFIG_ERROR, "optimizer: need 0 <= beta1 < beta2 < 1");
  if (!(c->eps > 0.0)) return fail(OR_CONFIG_ERROR, "optimizer: eps must be > 0");
  return OR_OK;
}

// SPEC.md:276 (t = 0 -> ConfigError); SPEC.md:292-294 (T mod s, t > T).
// f32: the fp32 mirror first rounds alpha, beta1, beta2, eps to float (the
// bucket precision) and derives everything else in double from those, so
// that e.g. beta2 + (1 - beta2) == 1 holds for the values the kernel uses
// (SURVEY.md Appendix A).  The fp64 path uses the configuration as given.
int scalars(const or_adam_cfg* cin, int algo, long t, long T, Scalars* o, bool f32 = false) {
  or_adam_cfg rounded;
  const or_adam_cfg* c = cin;
  if (f32 && cin) {
    rounded = *cin;
    rounded.alpha = double(float(cin->alpha));
    rounded.beta1 = double(float(cin->beta1));
    rounded.beta2 = double(float(cin->beta2));
    rounded.eps = double(float(cin->eps));
    c = &rounded;
  }
  if (int rc = check_cfg(c)) return rc;
  if (t < 1) return fail(OR_CONFIG_ERROR, "step: t must be >= 1");
  long tau = t;
  if (algo == OR_ACCUM) {
    if (c->s < 1) return fail(OR_CONFIG_ERROR, "accum_adam_step: s must be >= 1");
    if (T < 1 || T % c->s != 0) return fail(OR_CONFIG_ERROR, "accum_adam_step: T mod s != 0");
    if (t > T) return fail(OR_CONFIG_ERROR, "accum_adam_step: t exceeds T");
    tau = (t + c->s - 1) / c->s;  // t_hat = ceil(t/s), Alg. 3 line 4
  }
  o->b1 = c->beta1;
  o->omb1 = 1.0 - c->beta1;
  o->b2 = c->beta2;
  o->omb2 = 1.0 - c->beta2;
  o->c1 = 1.0 / (1.0 - std::pow(c->beta1, double(tau)));
  o->c2 = 1.0 / (1.0 - std::pow(c->beta2, double(tau)));
  o->neg_alpha = -c->alpha;
  o->eps = c->eps;
  o->inv_s = 1.0 / double(algo == OR_ACCUM ? c->s : 1);
  // Alg. 3 line 12: beta2 by default, beta1 as printed when paper_literal
  o->bv = c->paper_literal ? c->beta1 : c->beta2;
  o->ombv = c->paper_literal ? 1.0 - c->beta1 : 1.0 - c->beta2;
  return OR_OK;
}

template <class T>
struct TS {  // scalars in the working precision
  T b1, omb1, b2, omb2, c1, c2, neg_alpha, eps, inv_s, bv, ombv;
  explicit TS(const Scalars& s)
      : b1(T(s.b1)), omb1(T(s.omb1)), b2(T(s.b2)), omb2(T(s.omb2)), c1(T(s.c1)), c2(T(s.c2)),
        neg_alpha(T(s.neg_alpha)), eps(T(s.eps)), inv_s(T(s.inv_s)), bv(T(s.bv)),
        ombv(T(s.ombv)) {}
};

// dadam_step (Alg. 1 lines 4-6) in the op order of the
// reference primitives: scale = c*a (vec.cpp:34-38), add (vec.cpp:20-25),
// hadamard_square (vec.cpp:45-49), div_by_sqrt_plus_eps = m/(sqrt(v)+eps)
// (vec.cpp:51-57), axpy y += c*x (vec.cpp:40-43).
template <class T>
void dadam_elems(T* x, const T* g, T* m, T* v, const T* mixed, size_t d, const TS<T>& s) {
  for (size_t e = 0; e < d; ++e) {
    const T gi = g[e];
    const T mn = s.b1 * m[e] + s.omb1 * gi;
    const T vn = s.b2 * v[e] + s.omb2 * (gi * gi);
    const T dir = (s.c1 * mn) / (std::sqrt(s.c2 * vn) + s.eps);
    x[e] = mixed[e] + s.neg_alpha * dir;
    m[e] = mn;
    v[e] = vn;
  }
}

// accum_adam_step (Alg. 3 lines 4-14). m_t, v_t transient.
template <class T>
void accum_elems(T* x, const T* g, T* mh, T* vh, T* b, const T* mixed, size_t d,
                 const TS<T>& s, bool fold) {
  for (size_t e = 0; e < d; ++e) {
    const T gi = g[e];
    const T mt = s.b1 * mh[e] + s.omb1 * gi;
    const T vt = s.b2 * vh[e] + s.omb2 * (gi * gi);
    const T dir = (s.c1 * mt) / (std::sqrt(s.c2 * vt) + s.eps);
    x[e] = mixed[e] + s.neg_alpha * dir;
    const T bn = b[e] + s.inv_s * gi;
    if (fold) {
      mh[e] = s.b1 * mh[e] + s.omb1 * bn;
      vh[e] = s.bv * vh[e] + s.ombv * (bn * bn);
      b[e] = T(0);
    } else {
      b[e] = bn;
    }
  }
}

template <class T>
bool all_finite(const T* a, size_t d) {
  for (size_t e = 0; e < d; ++e)
    if (!std::isfinite(a[e])) return false;
  return true;
}

// Mixed neighbour sum: mixed = 0; for j ascending: mixed += w_ij * x_j (axpy,
// vec.cpp:40-43).  The accumulation is always in double with the double
// weights; the fp32 mirror rounds the finished sum to float once (the CUDA
// kernel does the same in fp64 registers).  Rounding each w_ij to float
// instead would bias sum_j w_ij away from 1 (e.g. 6*(float)(1/6) = 1+3e-8) and
// drift the models by ~3e-6 over 100 steps.
template <class T>
void mix_into(T* mixed, const T* xprev, size_t d, const std::vector<int>& nb, const Mat& w,
              int i) {
  std::vector<double> acc(d, 0.0);
  for (int j : nb) {
    const double wij = w(i, j);
    const T* xj = xprev + size_t(j) * d;
    for (size_t e = 0; e < d; ++e) acc[e] = acc[e] + wij * double(xj[e]);
  }
  for (size_t e = 0; e < d; ++e) mixed[e] = T(acc[e]);
}

void set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);  // parallel.hpp:33-40
#else
  (void)threads;
#endif
}

// All-Reduce Adam step (Alg. 2): gbar =
// mean_of(g_1..g_N) (vec.cpp:59-69: ascending sum in double, then * 1/N),
// every worker applies Adam with gbar and no mixing (x + (-alpha) * dir).
// Workers must hold identical states (max |x_i - x_0| <= 1e-12) -> else InvariantError.
template <class T>
int allreduce_step(const or_sched* s, size_t d, long t, uint64_t seed, bool gen_grad, const T* gin, T* x,
                   T* m, T* v, const TS<T>& ts) {
  const int n = s->workers;
  for (int i = 1; i < n; ++i)
    for (size_t e = 0; e < d; ++e)
      if (std::fabs(double(x[size_t(i) * d + e]) - double(x[e])) > 1e-12)
        return fail(OR_INVARIANT, "allreduce_adam_step: worker states diverged");
  std::vector<double> acc(d, 0.0);
  std::vector<T> g(d), gbar(d);
  for (int i = 0; i < n; ++i) {
    const T* gi = gin ? gin + size_t(i) * d : nullptr;
    if (gen_grad) {
      const uint64_t st = stream_state(seed, 2u, uint64_t(i), uint64_t(t));
      for (size_t e = 0; e < d; ++e) g[e] = T(bucket_value(draw(st, e)));
      gi = g.data();
    }
    for (size_t e = 0; e < d; ++e) acc[e] = acc[e] + double(gi[e]);
  }
  const double inv = 1.0 / double(n);
  for (size_t e = 0; e < d; ++e) gbar[e] = T(acc[e] * inv);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int i = 0; i < n; ++i) {
    const size_t o = size_t(i) * d;
    std::vector<T> self(x + o, x + o + d);  // "mixing" with W = I: x_i itself
    dadam_elems(x + o, gbar.data(), m + o, v + o, self.data(), d, ts);
    if (!all_finite(x + o, d) || !all_finite(m + o, d) || !all_finite(v + o, d)) bad = 1;
  }
  if (bad) {
    g_div_iter = t;
    return fail(OR_DIVERGENCE, "non-finite state at iteration " + std::to_string(t));
  }
  return OR_OK;
}

// One Jacobi step for all nodes (parallel_for over workers, parallel.hpp:13-23;
// snapshot semantics SPEC.md:317). gen_grad: draw g_i^(t) from the Minibatch stream.
template <class T>
int step_all(const or_sched* s, int algo, const or_adam_cfg* cfg, size_t d, long t, long T_,
             uint64_t seed, bool gen_grad, const T* gin, T* x, T* xprev, T* m, T* v, T* b) {
  Scalars sc;
  if (int rc = scalars(cfg, algo, t, T_, &sc, sizeof(T) == 4)) return rc;
  const TS<T> ts(sc);
  const Mat* w = round_mat(s, t);
  const auto* nb = round_nbrs(s, t);
  if (!w) return fail(OR_CONFIG_ERROR, "step: empty schedule or round < 1");
  const int n = s->workers;
  std::memcpy(xprev, x, sizeof(T) * size_t(n) * d);
  const bool fold = algo == OR_ACCUM && (t % cfg->s == 0);
  int bad = 0;
  if (algo == OR_ALLREDUCE) return allreduce_step<T>(s, d, t, seed, gen_grad, gin, x, m, v, ts);
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int i = 0; i < n; ++i) {
    std::vector<T> mixed(d), gbuf;
    const T* g = gin ? gin + size_t(i) * d : nullptr;
    if (gen_grad) {
      gbuf.resize(d);
      const uint64_t st = stream_state(seed, 2u /*Minibatch*/, uint64_t(i), uint64_t(t));
      for (size_t e = 0; e < d; ++e) gbuf[e] = T(bucket_value(draw(st, e)));
      g = gbuf.data();
    }
    mix_into(mixed.data(), xprev, d, (*nb)[i], *w, i);
    const size_t o = size_t(i) * d;
    if (algo == OR_DADAM)
      dadam_elems(x + o, g, m + o, v + o, mixed.data(), d, ts);
    else
      accum_elems(x + o, g, m + o, v + o, b + o, mixed.data(), d, ts, fold);
    if (!all_finite(x + o, d) || !all_finite(m + o, d) || !all_finite(v + o, d)) bad = 1;
  }
  if (bad) {
    g_div_iter = t;
    return fail(OR_DIVERGENCE, "non-finite state at iteration " + std::to_string(t));
  }
  return OR_OK;
}

template <class T>
int run(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed, size_t d,
        long t0, long t1, long T_, int threads, T* x, T* m, T* v, T* b) {
  if (!s) return fail(OR_CONFIG_ERROR, "run: empty schedule");
  if (algo == OR_ACCUM && !b) return fail(OR_CONFIG_ERROR, "run: accumulator buffer missing");
  set_threads(threads);
  std::vector<T> xprev(size_t(s->workers) * d);
  for (long t = t0; t <= t1; ++t)
    if (int rc = step_all<T>(s, algo, cfg, d, t, T_, seed, true, nullptr, x, xprev.data(), m, v,
                             b))
      return rc;
  return OR_OK;
}

// Column-sampled run (see oracle.h): same per-element arithmetic as step_all.
template <class T>
int run_cols(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed,
             const uint64_t* cols, size_t nc, int dispersed, long t0, long t1, long T_, int threads,
             T* x, T* m, T* v, T* b) {
  if (!s) return fail(OR_CONFIG_ERROR, "run_cols: empty schedule");
  if (algo == OR_ACCUM && !b) return fail(OR_CONFIG_ERROR, "run_cols: accumulator buffer missing");
  set_threads(threads);
  const int n = s->workers;
  for (int i = 0; i < n; ++i) {  // x^(0)
    const uint64_t st = dispersed ? stream_state(seed, 6u, uint64_t(i), 0) : stream_state(seed, 4u, 0, 0);
    for (size_t c = 0; c < nc; ++c) x[size_t(i) * nc + c] = T(bucket_value(draw(st, cols[c])));
  }
  std::vector<T> xprev(size_t(n) * nc);
  for (long t = t0; t <= t1; ++t) {
    Scalars sc;
    if (int rc = scalars(cfg, algo, t, T_, &sc, sizeof(T) == 4)) return rc;
    const TS<T> ts(sc);
    const Mat& w = *round_mat(s, t);
    const auto& nb = *round_nbrs(s, t);
    std::memcpy(xprev.data(), x, sizeof(T) * xprev.size());
    const bool fold = algo == OR_ACCUM && (t % cfg->s == 0);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int i = 0; i < n; ++i) {
      std::vector<T> mixed(nc), g(nc);
      const uint64_t st = stream_state(seed, 2u, uint64_t(i), uint64_t(t));
      for (size_t c = 0; c < nc; ++c) g[c] = T(bucket_value(draw(st, cols[c])));
      mix_into(mixed.data(), xprev.data(), nc, nb[i], w, i);
      const size_t o = size_t(i) * nc;
      if (algo == OR_DADAM)
        dadam_elems(x + o, g.data(), m + o, v + o, mixed.data(), nc, ts);
      else
        accum_elems(x + o, g.data(), m + o, v + o, b + o, mixed.data(), nc, ts, fold);
      if (!all_finite(x + o, nc) || !all_finite(m + o, nc) || !all_finite(v + o, nc)) bad = 1;
    }
    if (bad) {
      g_div_iter = t;
      return fail(OR_DIVERGENCE, "non-finite state at iteration " + std::to_string(t));
    }
  }
  return OR_OK;
}

}  // namespace

// ================================================================= extern "C"
extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }
long or_last_divergence_iteration(void) { return g_div_iter; }

void or_rng_u64(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration,
                uint64_t first, size_t n, uint64_t* out) {
  const uint64_t st = stream_state(seed, purpose, worker, iteration);
  for (size_t k = 0; k < n; ++k) out[k] = draw(st, first + k);
}
void or_rng_unit(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration,
                 uint64_t first, size_t n, double* out) {
  const uint64_t st = stream_state(seed, purpose, worker, iteration);
  for (size_t k = 0; k < n; ++k) out[k] = unit_of(draw(st, first + k));
}
void or_fill_f32(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration, size_t n,
                 float* out) {
  const uint64_t st = stream_state(seed, purpose, worker, iteration);
  for (size_t k = 0; k < n; ++k) out[k] = bucket_value(draw(st, k));
}

// make_complete (topology.hpp:65-66)
// make_one_peer_ring (topology.hpp:67-69)
// make_one_peer_exponential (topology.hpp:70-72)
// make_aer (topology.hpp:73-78)
// static exponential: not in the reference: undirected
// circulant i +/- 2^k (2^k < n), uniform weight 1/(deg+1).
int or_make(int kind, int n, int wpn, or_sched** out) {
  if (!out) return fail(OR_CONFIG_ERROR, "make: null out");
  *out = nullptr;
  if (n < 1) return fail(OR_CONFIG_ERROR, "make: n must be >= 1");
  std::vector<Mat> rounds;
  switch (kind) {
    case OR_COMPLETE: {
      Mat w(n);
      for (double& e : w.a) e = 1.0 / double(n);
      rounds.push_back(w);
      return build(n, 1, rounds, out);
    }
    case OR_ONE_PEER_RING: {
      if (n < 2 || n % 2) return fail(OR_CONFIG_ERROR, "make_one_peer_ring: N must be even");
      std::vector<std::pair<int, int>> r1, r2;
      for (int k = 0; k < n / 2; ++k) {
        r1.push_back({2 * k, 2 * k + 1});
        r2.push_back({2 * k + 1, (2 * k + 2) % n});
      }
      rounds.push_back(matching(n, r1));
      rounds.push_back(matching(n, r2));
      return build(n, 1, rounds, out);
    }
    case OR_ONE_PEER_EXP: {
      if (n < 2 || !is_pow2(n))
        return fail(OR_CONFIG_ERROR, "make_one_peer_exponential: N must be a power of 2");
      for (int r = 1; r <= ilog2(n); ++r) {
        std::vector<std::pair<int, int>> pr;
        for (int i = 0; i < n; ++i) {
          const int j = i ^ (1 << (r - 1));
          if (i < j) pr.push_back({i, j});
        }
        rounds.push_back(matching(n, pr));
      }
      return build(n, 1, rounds, out);
    }
    case OR_AER: {
      if (wpn < 1 || n % wpn) return fail(OR_CONFIG_ERROR, "make_aer: wpn must divide N");
      const int M = n / wpn;
      if (M < 2 || !is_pow2(M))
        return fail(OR_CONFIG_ERROR, "make_aer: node count must be a power of 2 >= 2");
      for (auto [a, b] : aer_pairs(M)) {
        std::vector<std::vector<int>> gs;
        for (int k = 0; k < M; ++k) {
          if (k == b) continue;  // folded into a's group
          std::vector<int> g;
          for (int q = 0; q < wpn; ++q) g.push_back(k * wpn + q);
          if (k == a)
            for (int q = 0; q < wpn; ++q) g.push_back(b * wpn + q);
          std::sort(g.begin(), g.end());
          gs.push_back(g);
        }
        rounds.push_back(groups(n, gs));
      }
      return build(n, wpn, rounds, out);
    }
    case OR_STATIC_EXP: {
      if (n < 2) return fail(OR_CONFIG_ERROR, "static_exponential: N must be >= 2");
      std::vector<std::vector<int>> adj(n);
      for (int i = 0; i < n; ++i) {
        for (int h = 1; h < n; h <<= 1) {
          adj[i].push_back((i + h) % n);
          adj[i].push_back(((i - h) % n + n) % n);
        }
        adj[i].push_back(i);
        std::sort(adj[i].begin(), adj[i].end());
        adj[i].erase(std::unique(adj[i].begin(), adj[i].end()), adj[i].end());
      }
      Mat w(n);
      for (int i = 0; i < n; ++i)
        for (int j : adj[i]) w(i, j) = 1.0 / double(adj[i].size());
      rounds.push_back(w);
      return build(n, 1, rounds, out);
    }
    default:
      return fail(OR_CONFIG_ERROR, "make: unknown topology kind");
  }
}

int or_from_matrices(const double* w, int n, int period, int wpn, or_sched** out) {
  if (!w || !out || period < 1 || n < 1) return fail(OR_CONFIG_ERROR, "from_matrices: bad args");
  if (wpn < 1 || n % wpn) return fail(OR_CONFIG_ERROR, "from_matrices: wpn must divide N");
  std::vector<Mat> rounds;
  for (int r = 0; r < period; ++r) {
    Mat m(n);
    std::memcpy(m.a.data(), w + size_t(r) * n * n, sizeof(double) * n * n);
    rounds.push_back(m);
  }
  return build(n, wpn, rounds, out);
}

void or_free(or_sched* s) { delete s; }

int or_info(const or_sched* s, int* workers, int* period, int* wpn, int* is_static) {
  if (!s) return fail(OR_CONFIG_ERROR, "info: empty schedule");
  if (workers) *workers = s->workers;
  if (period) *period = int(s->rounds.size());
  if (wpn) *wpn = s->wpn;
  if (is_static) *is_static = s->rounds.size() == 1;
  return OR_OK;
}

// matrix_at (topology.hpp:53): 1-based, periodic
int or_matrix(const or_sched* s, long round, double* w) {
  const Mat* m = round_mat(s, round);
  if (!m) return fail(OR_CONFIG_ERROR, "matrix_at: empty schedule or round < 1");
  std::memcpy(w, m->a.data(), sizeof(double) * m->a.size());
  return OR_OK;
}

// neighbors_at (topology.hpp:54-55): ascending, self included
int or_neighbors(const or_sched* s, long round, int worker, int* idx, double* w, int cap,
                 int* count) {
  const Mat* m = round_mat(s, round);
  if (!m) return fail(OR_CONFIG_ERROR, "neighbors_at: empty schedule or round < 1");
  if (worker < 0 || worker >= s->workers) return fail(OR_CONFIG_ERROR, "neighbors_at: bad worker");
  const auto& nb = (*round_nbrs(s, round))[size_t(worker)];
  if (count) *count = int(nb.size());
  if (int(nb.size()) > cap) return fail(OR_CONFIG_ERROR, "neighbors_at: capacity too small");
  for (size_t k = 0; k < nb.size(); ++k) {
    if (idx) idx[k] = nb[k];
    if (w) w[k] = (*m)(worker, nb[k]);
  }
  return OR_OK;
}

int or_validate(const double* w, int n, or_validation* out) {
  if (!w || !out || n < 0) return fail(OR_CONFIG_ERROR, "validate: bad args");
  Mat m(n);
  std::memcpy(m.a.data(), w, sizeof(double) * size_t(n) * n);
  *out = validate_mat(m);
  return OR_OK;
}

// spectral_lambda (topology.hpp:82-84)
int or_spectral_lambda(const double* w, int n, double* out) {
  if (!w || !out || n < 1) return fail(OR_CONFIG_ERROR, "spectral_lambda: bad args");
  Mat m(n);
  std::memcpy(m.a.data(), w, sizeof(double) * size_t(n) * n);
  if (validate_mat(m).max_asymmetry > 1e-12)
    return fail(OR_CONFIG_ERROR, "spectral_lambda: matrix not symmetric");
  if (n == 1) return *out = 0.0, OR_OK;
  const auto ev = sym_eigenvalues(m);
  *out = std::max(std::fabs(ev[1]), std::fabs(ev[size_t(n) - 1]));
  return OR_OK;
}

// effective_lambda (topology.hpp:86-88): sigma_max(W^(P)..W^(1) - J/N)
int or_effective_lambda(const or_sched* s, double* out) {
  if (!s || s->rounds.empty() || !out) return fail(OR_CONFIG_ERROR, "effective_lambda: empty");
  const int n = s->workers;
  Mat p(n);
  for (int i = 0; i < n; ++i) p(i, i) = 1.0;
  for (const Mat& w : s->rounds) p = matmul(w, p);
  for (double& e : p.a) e -= 1.0 / double(n);
  Mat ata(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += p(k, i) * p(k, j);
      ata(i, j) = acc;
    }
  const auto ev = sym_eigenvalues(ata);
  *out = std::sqrt(std::max(0.0, ev.front()));
  return OR_OK;
}

// gossip_consensus (topology.hpp:90-100)
int or_gossip_consensus(const or_sched* s, const double* x0, int n, size_t d, int rounds,
                        int threads, double* err) {
  if (!s || s->rounds.empty()) return fail(OR_CONFIG_ERROR, "gossip_consensus: empty schedule");
  if (n != s->workers) return fail(OR_CONFIG_ERROR, "gossip_consensus: x0 size mismatch");
  if (rounds < 0) return fail(OR_CONFIG_ERROR, "gossip_consensus: rounds < 0");
  set_threads(threads);
  std::vector<double> x(x0, x0 + size_t(n) * d), y(size_t(n) * d), xbar(d, 0.0);
  for (int i = 0; i < n; ++i)  // mean_of (vec.cpp:59-69)
    for (size_t e = 0; e < d; ++e) xbar[e] += x[size_t(i) * d + e];
  const double inv = 1.0 / double(n);
  for (double& e : xbar) e *= inv;
  auto disp = [&](const std::vector<double>& a) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      double si = 0.0;
      for (size_t e = 0; e < d; ++e) {
        const double dlt = a[size_t(i) * d + e] - xbar[e];
        si += dlt * dlt;
      }
      acc += si;
    }
    return acc;
  };
  const double d0 = disp(x);
  if (d0 == 0.0) {
    for (int t = 0; t <= rounds; ++t) err[t] = 0.0;
    return OR_OK;
  }
  err[0] = 1.0;
  for (int t = 1; t <= rounds; ++t) {
    const Mat& w = *round_mat(s, t);
    const auto& nb = *round_nbrs(s, t);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) mix_into(y.data() + size_t(i) * d, x.data(), d, nb[i], w, i);
    std::swap(x, y);
    err[t] = disp(x) / d0;
  }
  return OR_OK;
}

#define STEP_GUARD(cond, msg) \
  if (!(cond)) return fail(OR_CONFIG_ERROR, msg)

int or_dadam_step_f64(double* x, const double* g, double* m, double* v, const double* mixed,
                      size_t d, const or_adam_cfg* cfg, long t) {
  Scalars sc;
  if (int rc = scalars(cfg, OR_DADAM, t, 0, &sc)) return rc;
  dadam_elems<double>(x, g, m, v, mixed, d, TS<double>(sc));
  return OR_OK;
}
int or_dadam_step_f32(float* x, const float* g, float* m, float* v, const float* mixed, size_t d,
                      const or_adam_cfg* cfg, long t) {
  Scalars sc;
  if (int rc = scalars(cfg, OR_DADAM, t, 0, &sc, true)) return rc;
  dadam_elems<float>(x, g, m, v, mixed, d, TS<float>(sc));
  return OR_OK;
}
int or_accum_adam_step_f64(double* x, const double* g, double* mh, double* vh, double* b,
                           const double* mixed, size_t d, const or_adam_cfg* cfg, long t, long T) {
  Scalars sc;
  if (int rc = scalars(cfg, OR_ACCUM, t, T, &sc)) return rc;
  accum_elems<double>(x, g, mh, vh, b, mixed, d, TS<double>(sc), t % cfg->s == 0);
  return OR_OK;
}
int or_accum_adam_step_f32(float* x, const float* g, float* mh, float* vh, float* b,
                           const float* mixed, size_t d, const or_adam_cfg* cfg, long t, long T) {
  Scalars sc;
  if (int rc = scalars(cfg, OR_ACCUM, t, T, &sc, true)) return rc;
  accum_elems<float>(x, g, mh, vh, b, mixed, d, TS<float>(sc), t % cfg->s == 0);
  return OR_OK;
}

int or_run_f64(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed, size_t d,
               long t0, long t1, long T, int threads, double* x, double* m, double* v,
               double* b) {
  return run<double>(s, algo, cfg, seed, d, t0, t1, T, threads, x, m, v, b);
}
int or_run_f32(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed, size_t d,
               long t0, long t1, long T, int threads, float* x, float* m, float* v, float* b) {
  return run<float>(s, algo, cfg, seed, d, t0, t1, T, threads, x, m, v, b);
}
int or_step_all_f64(const or_sched* s, int algo, const or_adam_cfg* cfg, size_t d, long t, long T,
                    int threads, const double* g, double* x, double* xprev, double* m, double* v,
                    double* b) {
  if (!s) return fail(OR_CONFIG_ERROR, "step_all: empty schedule");
  set_threads(threads);
  return step_all<double>(s, algo, cfg, d, t, T, 0, false, g, x, xprev, m, v, b);
}
int or_step_all_f32(const or_sched* s, int algo, const or_adam_cfg* cfg, size_t d, long t, long T,
                    int threads, const float* g, float* x, float* xprev, float* m, float* v, float* b) {
  if (!s) return fail(OR_CONFIG_ERROR, "step_all: empty schedule");
  set_threads(threads);
  return step_all<float>(s, algo, cfg, d, t, T, 0, false, g, x, xprev, m, v, b);
}
int or_run_cols_f32(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed,
                    const uint64_t* cols, size_t nc, int dispersed, long t0, long t1, long T,
                    int threads, float* x, float* m, float* v, float* b) {
  return run_cols<float>(s, algo, cfg, seed, cols, nc, dispersed, t0, t1, T, threads, x, m, v, b);
}
int or_run_cols_f64(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed,
                    const uint64_t* cols, size_t nc, int dispersed, long t0, long t1, long T,
                    int threads, double* x, double* m, double* v, double* b) {
  return run_cols<double>(s, algo, cfg, seed, cols, nc, dispersed, t0, t1, T, threads, x, m, v, b);
}
int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
