// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiled together with the reference's own proj/src/vec.cpp and
// proj/src/rng.cpp (straight from /root/reference, never copied) into
// oracle/_ref/libdeclab_ref.so by oracle/Makefile.  It exposes, over a C ABI:
//   * the reference StreamRng draws (rng.hpp:23-39), to pin the oracle RNG
//     and to generate the golden vectors in tests/golden/;
//   * DAdam / AccumAdam composed *only* from the reference's vec.cpp
//     primitives (scale, add, axpy, hadamard_square, div_by_sqrt_plus_eps,
//     all_finite) and the reference's parallel_for over workers
//     (parallel.hpp:13-23) -- i.e. the reference's CPU path for the step, as
//     SPEC.md:272-298 defines it on top of the shipped primitives.  The
//     reference ships no topology.cpp, so the neighbour lists
//     and weights are passed in by the caller.
// This is the "reference" CPU arm of bench.py and the pin for oracle.cpp.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "declab/errors.hpp"
#include "declab/parallel.hpp"
#include "declab/rng.hpp"
#include "declab/vec.hpp"

using namespace declab;

namespace {
thread_local std::string g_err;
thread_local long g_div = -1;
}  // namespace

extern "C" {

typedef struct {
  double alpha, beta1, beta2, eps;
  int s;
  int paper_literal;
} ref_adam_cfg;

const char* ref_last_error(void) { return g_err.c_str(); }
long ref_last_divergence_iteration(void) { return g_div; }

void ref_rng_u64(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration, size_t n,
                 uint64_t* out) {
  StreamRng r(seed, static_cast<Stream>(purpose), worker, iteration);
  for (size_t k = 0; k < n; ++k) out[k] = r.next_u64();
}
void ref_rng_unit(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration, size_t n,
                  double* out) {
  StreamRng r(seed, static_cast<Stream>(purpose), worker, iteration);
  for (size_t k = 0; k < n; ++k) out[k] = r.next_unit();
}
double ref_speed_multiplier(uint64_t seed, uint64_t worker, uint64_t iteration, double sigma2,
                            int k) {
  StreamRng r(seed, Stream::SpeedNoise, worker, iteration);
  double p = 1.0;
  for (int i = 0; i <= k; ++i) p = sample_speed_multiplier(r, sigma2);
  return p;
}
/* vec.cpp:51-57 exposed for op-order KATs */
void ref_div_by_sqrt_plus_eps(const double* m, const double* v, size_t n, double eps,
                              double* out) {
  Vec a(m, m + n), b(v, v + n);
  Vec r = div_by_sqrt_plus_eps(a, b, eps);
  std::memcpy(out, r.data(), n * sizeof(double));
}

/* Multi-worker run of DAdam (algo 0) / AccumAdam (algo 1), steps t0..t1.
 * nbr_idx / nbr_w: period x n x maxdeg, nbr_cnt: period x n (ascending, self incl.).
 * gen_grad: g_i^(t) = (float)(2u-1) from StreamRng(seed, Minibatch, i, t); otherwise
 * g_fixed (n x d) is used every step.  elapsed_s: wall time of the step loop. */
int ref_run(int algo, int n, size_t d, int period, int maxdeg, const int* nbr_idx,
            const double* nbr_w, const int* nbr_cnt, const ref_adam_cfg* cfg, uint64_t seed,
            long t0, long t1, long T, int threads, int gen_grad, const double* g_fixed,
            double* x, double* m, double* v, double* b, double* elapsed_s) {
  try {
    if (t0 < 1) throw ConfigError("step: t must be >= 1");
    if (algo == 1 && (cfg->s < 1 || T % cfg->s != 0 || t1 > T))
      throw ConfigError("accum_adam_step: bad s / T");
    set_threads(threads);
    std::vector<Vec> X(n), M(n), V(n), B(n), G(n);
    for (int i = 0; i < n; ++i) {
      X[i].assign(x + size_t(i) * d, x + size_t(i + 1) * d);
      M[i].assign(m + size_t(i) * d, m + size_t(i + 1) * d);
      V[i].assign(v + size_t(i) * d, v + size_t(i + 1) * d);
      B[i] = b ? Vec(b + size_t(i) * d, b + size_t(i + 1) * d) : zeros(d);
      if (!gen_grad) G[i].assign(g_fixed + size_t(i) * d, g_fixed + size_t(i + 1) * d);
    }
    const auto start = std::chrono::steady_clock::now();
    for (long t = t0; t <= t1; ++t) {
      const long tau = algo == 1 ? (t + cfg->s - 1) / cfg->s : t;
      const double c1 = 1.0 / (1.0 - std::pow(cfg->beta1, double(tau)));
      const double c2 = 1.0 / (1.0 - std::pow(cfg->beta2, double(tau)));
      const double bv = cfg->paper_literal ? cfg->beta1 : cfg->beta2;
      const bool fold = algo == 1 && t % cfg->s == 0;
      const int r = int((t - 1) % period);
      const std::vector<Vec> Xprev = X;  // Jacobi snapshot
      std::vector<int> bad(n, 0);
      if (algo == 2) {  // All-Reduce Adam: gbar = mean_of(g), no mixing
        std::vector<Vec> Gt(n);
        for (int i = 0; i < n; ++i) {
          if (gen_grad) {
            StreamRng rng(seed, Stream::Minibatch, uint64_t(i), uint64_t(t));
            Gt[i].resize(d);
            for (size_t e = 0; e < d; ++e) Gt[i][e] = double(static_cast<float>(2.0 * rng.next_unit() - 1.0));
          } else {
            Gt[i] = G[i];
          }
        }
        const Vec gbar = mean_of(Gt);
        for (int i = 1; i < n; ++i)
          if (linf_norm(sub(X[i], X[0])) > 1e-12) throw InvariantError("allreduce_adam_step: workers diverged");
        parallel_for(Exec::OpenMP, n, [&](int i) {
          M[i] = add(scale(M[i], cfg->beta1), scale(gbar, 1.0 - cfg->beta1));
          V[i] = add(scale(V[i], cfg->beta2), scale(hadamard_square(gbar), 1.0 - cfg->beta2));
          const Vec dir = div_by_sqrt_plus_eps(scale(M[i], c1), scale(V[i], c2), cfg->eps);
          Vec xn = Xprev[i];
          axpy(-cfg->alpha, dir, xn);
          X[i] = std::move(xn);
          bad[i] = !(all_finite(X[i]) && all_finite(M[i]) && all_finite(V[i]));
        });
        for (int i = 0; i < n; ++i)
          if (bad[i]) throw DivergenceError(t, "non-finite state at iteration " + std::to_string(t));
        continue;
      }
      parallel_for(Exec::OpenMP, n, [&](int i) {
        Vec g;
        if (gen_grad) {
          StreamRng rng(seed, Stream::Minibatch, uint64_t(i), uint64_t(t));
          g.resize(d);
          for (size_t e = 0; e < d; ++e)
            g[e] = double(static_cast<float>(2.0 * rng.next_unit() - 1.0));
        } else {
          g = G[i];
        }
        Vec mixed = zeros(d);
        const size_t o = (size_t(r) * n + i) * maxdeg;
        for (int k = 0; k < nbr_cnt[size_t(r) * n + i]; ++k)
          axpy(nbr_w[o + k], Xprev[size_t(nbr_idx[o + k])], mixed);
        if (algo == 0) {
          M[i] = add(scale(M[i], cfg->beta1), scale(g, 1.0 - cfg->beta1));
          V[i] = add(scale(V[i], cfg->beta2), scale(hadamard_square(g), 1.0 - cfg->beta2));
          const Vec dir = div_by_sqrt_plus_eps(scale(M[i], c1), scale(V[i], c2), cfg->eps);
          axpy(-cfg->alpha, dir, mixed);
          X[i] = std::move(mixed);
        } else {
          const Vec mt = add(scale(M[i], cfg->beta1), scale(g, 1.0 - cfg->beta1));
          const Vec vt = add(scale(V[i], cfg->beta2), scale(hadamard_square(g), 1.0 - cfg->beta2));
          const Vec dir = div_by_sqrt_plus_eps(scale(mt, c1), scale(vt, c2), cfg->eps);
          axpy(-cfg->alpha, dir, mixed);
          X[i] = std::move(mixed);
          B[i] = add(B[i], scale(g, 1.0 / double(cfg->s)));
          if (fold) {
            M[i] = add(scale(M[i], cfg->beta1), scale(B[i], 1.0 - cfg->beta1));
            V[i] = add(scale(V[i], bv), scale(hadamard_square(B[i]), 1.0 - bv));
            B[i] = zeros(d);
          }
        }
        bad[i] = !(all_finite(X[i]) && all_finite(M[i]) && all_finite(V[i]));
      });
      for (int i = 0; i < n; ++i)
        if (bad[i]) throw DivergenceError(t, "non-finite state at iteration " + std::to_string(t));
    }
    if (elapsed_s)
      *elapsed_s =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    for (int i = 0; i < n; ++i) {
      std::memcpy(x + size_t(i) * d, X[i].data(), d * sizeof(double));
      std::memcpy(m + size_t(i) * d, M[i].data(), d * sizeof(double));
      std::memcpy(v + size_t(i) * d, V[i].data(), d * sizeof(double));
      if (b) std::memcpy(b + size_t(i) * d, B[i].data(), d * sizeof(double));
    }
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    g_div = e.iteration;
    return 3;
  } catch (const InvariantError& e) {
    g_err = e.what();
    return 4;
  }
}

int ref_max_threads(void) { return max_threads(); }

}  // extern "C"
