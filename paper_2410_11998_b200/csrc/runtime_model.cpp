// runtime_model.cpp -- the paper's per-iteration runtime model.
//
// Discrete-event recurrences of PAPER.md Appendix A.5 (All-Reduce and
// decentralized training) and the SGP variant of A.8.1,
// evaluated verbatim; closed-form best speedup Eq. (3);
// speed multipliers p^(i,t) from the truncated normal of rng.cpp:54-73 drawn
// from StreamRng(seed, SpeedNoise, i, t) (common random numbers across modes).
// Contract: SPEC.md:415-507.  Host-only; single-threaded per replicate.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "dg_internal.hpp"

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// StreamRng (rng.cpp:26-62): keyed SplitMix64 state, next_unit, Box-Muller.
struct Rng {
  uint64_t state;
  Rng(uint64_t seed, uint64_t purpose, uint64_t worker, uint64_t iteration) {
    uint64_t s = mix64(seed + kGolden);
    s = mix64((s + kGolden) ^ purpose);
    s = mix64((s + kGolden) ^ worker);
    s = mix64((s + kGolden) ^ iteration);
    state = s;
  }
  double unit() {
    state += kGolden;
    return static_cast<double>(mix64(state) >> 11) * 0x1.0p-53;
  }
  double normal() {
    const double u1 = 1.0 - unit();
    const double u2 = unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925287 * u2);
  }
};

// sample_speed_multiplier (rng.cpp:64-73): parent N(1, sigma2) truncated to [0.5, 1.5]
double speed_multiplier(uint64_t seed, uint64_t worker, uint64_t iteration, double sigma2) {
  if (sigma2 < 0) dg::config_error("speed multiplier: sigma2 must be >= 0");
  if (sigma2 == 0.0) return 1.0;
  Rng r(seed, 3 /*SpeedNoise*/, worker, iteration);
  const double sd = std::sqrt(sigma2);
  for (;;) {
    const double p = 1.0 + sd * r.normal();
    if (p >= 0.5 && p <= 1.5) return p;
  }
}

void check(const dg_rm_params* p) {
  if (!p) dg::config_error("runtime model: null params");
  if (p->N < 1 || p->b < 1) dg::config_error("runtime model: N and b must be >= 1");
  if (!(p->theta >= 0) || !(p->gamma > 0)) dg::config_error("runtime model: need theta >= 0, gamma > 0");
  if (!(p->omega > 0) || (p->omega > 1 && !p->allow_omega_above_one))
    dg::config_error("runtime model: omega must be in (0, 1] (allow_omega_above_one to override)");
  if (!(p->sigma2 >= 0)) dg::config_error("runtime model: sigma2 must be >= 0");
  if (p->workers_per_node < 1 || p->N % p->workers_per_node)
    dg::config_error("runtime model: workers_per_node must divide N");
}

// Completion-time record layout per (t, i): F, B_1..B_b, U_1..U_b, C_1..C_b.
struct Trace {
  int N, b;
  std::vector<double> v;  // (T+1) x N x (1 + 3b); iteration 0 = all zeros
  Trace(long T, int N_, int b_) : N(N_), b(b_), v(size_t(T + 1) * N_ * (1 + 3 * b_), 0.0) {}
  double* at(long t, int i) { return &v[(size_t(t) * N + i) * (1 + 3 * b)]; }
  double& F(long t, int i) { return at(t, i)[0]; }
  double& B(long t, int i, int k) { return at(t, i)[k]; }              // k = 1..b
  double& U(long t, int i, int k) { return at(t, i)[b + k]; }          // k = 1..b (AR: U stored at k=1)
  double& C(long t, int i, int k) { return at(t, i)[2 * b + k]; }
};

void simulate(int mode, const dg_rm_params* prm, const dg_schedule* s, long T, uint64_t seed, Trace& tr,
              double* runtimes) {
  const int N = prm->N, b = prm->b;
  const double theta = prm->theta, gamma = prm->gamma, omega = prm->omega;
  const double fwd = (mode == DG_RM_ALLREDUCE && !prm->normalized) ? double(b) / N : 1.0 / N;
  double prev_max = 0.0;
  std::vector<double> p(N);
  for (long t = 1; t <= T; ++t) {
    for (int i = 0; i < N; ++i) p[i] = speed_multiplier(seed, uint64_t(i), uint64_t(t), prm->sigma2);
    if (mode == DG_RM_ALLREDUCE) {  // PAPER.md Appendix A.5, All-Reduce system
      for (int i = 0; i < N; ++i) {
        tr.F(t, i) = tr.U(t - 1, i, 1) + p[i] * fwd;
        tr.B(t, i, b) = p[i] * 2.0 / N + tr.F(t, i);
        for (int k = b - 1; k >= 1; --k) tr.B(t, i, k) = p[i] * 2.0 / N + tr.B(t, i, k + 1);
      }
      for (int k = b; k >= 1; --k) {
        double mx = 0.0;
        for (int j = 0; j < N; ++j) {
          mx = std::max(mx, tr.B(t, j, k));
          if (k < b) mx = std::max(mx, tr.C(t, j, k + 1));
        }
        for (int i = 0; i < N; ++i) tr.C(t, i, k) = gamma + mx;
      }
      for (int i = 0; i < N; ++i) tr.U(t, i, 1) = tr.C(t, i, 1) + theta * b;
    } else {  // decentralized system / SGP variant (A.8.1)
      const dg::Round* rd = s ? &s->at(t) : nullptr;
      const int wpn = prm->workers_per_node;
      for (int i = 0; i < N; ++i) tr.F(t, i) = tr.U(t - 1, i, 1) + p[i] / N;
      for (int k = b; k >= 1; --k) {
        for (int i = 0; i < N; ++i)
          tr.B(t, i, k) = p[i] * 2.0 / N + (k == b ? tr.F(t, i) : tr.U(t, i, k + 1));
        for (int i = 0; i < N; ++i) {
          double ready;
          if (mode == DG_RM_SGP) {  // U_k waits for the whole node L(i)
            ready = 0.0;
            const int g0 = (i / wpn) * wpn;
            for (int j = g0; j < g0 + wpn; ++j) ready = std::max({ready, tr.B(t, j, k), tr.C(t - 1, j, k)});
          } else {
            ready = std::max(tr.B(t, i, k), tr.C(t - 1, i, k));
          }
          tr.U(t, i, k) = ready + theta;
        }
        for (int i = 0; i < N; ++i) {
          double mx = 0.0;
          auto consider = [&](int j) {
            mx = std::max(mx, tr.U(t, j, k));
            mx = std::max(mx, k == b ? tr.C(t - 1, j, 1) : tr.C(t, j, k + 1));
          };
          if (rd)
            for (int j : rd->nbr[i]) consider(j);
          else
            for (int j = 0; j < N; ++j) consider(j);  // complete topology
          tr.C(t, i, k) = omega * gamma + mx;
        }
      }
    }
    double mx = 0.0;
    for (int i = 0; i < N; ++i) mx = std::max(mx, tr.U(t, i, 1));
    runtimes[t - 1] = mx - prev_max;  // increment of the global max finish time
    prev_max = mx;
  }
}

}  // namespace

extern "C" {

int dg_rm_simulate(int mode, const dg_rm_params* prm, const dg_schedule* s, long T, uint64_t seed,
                   double* runtimes, double* timeline) {
  return dg::guarded([&] {
    check(prm);
    if (mode < DG_RM_ALLREDUCE || mode > DG_RM_SGP) dg::config_error("runtime model: unknown mode");
    if (T < 1 || !runtimes) dg::config_error("runtime model: T must be >= 1");
    if (s && s->n != prm->N) dg::config_error("runtime model: schedule size != N");
    Trace tr(T, prm->N, prm->b);
    simulate(mode, prm, s, T, seed, tr, runtimes);
    if (timeline) std::memcpy(timeline, tr.v.data() + size_t(prm->N) * (1 + 3 * prm->b),
                              sizeof(double) * size_t(T) * prm->N * (1 + 3 * prm->b));
  });
}

// Eq. (3): piecewise with breakpoint gamma = 2/N.
int dg_rm_closed_form_speedup(double gamma, int N, int b, double theta, double* out) {
  return dg::guarded([&] {
    if (!out || !(gamma > 0) || N < 1 || b < 1 || !(theta >= 0)) dg::config_error("speedup: bad arguments");
    const double den = 3.0 + theta * N;
    *out = gamma <= 2.0 / N ? 1.0 + (1.0 / b) * (N * gamma) / den : 1.0 + (N * gamma - 2.0 + 2.0 / b) / den;
  });
}

int dg_rm_speed_multiplier(uint64_t seed, uint64_t worker, uint64_t iteration, double sigma2, double* out) {
  return dg::guarded([&] {
    if (!out) dg::config_error("speed_multiplier: null output");
    *out = speed_multiplier(seed, worker, iteration, sigma2);
  });
}

}  // extern "C"
