// schedule.cpp -- host side of libdg: topology / peer-schedule generator,
// mixing-matrix validation, lambda helpers, per-rank round plans.
//
// Replaces declab's topology module (proj/include/declab/topology.hpp:12-100,
// contract SPEC.md:77-188; the reference ships only the header).  The builders
// are closed-form peer tables (XOR / ring / AER group formulas) rather than the
// dense-matrix construction the reference's Eigen types imply; dense matrices
// are materialised only for validation and for dg_schedule_matrix.
#include <algorithm>
#include <cmath>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <numeric>

#include "dg_internal.hpp"

namespace {
thread_local std::string t_err;
thread_local long t_div = -1;

bool pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }
int log2i(int n) { return 31 - __builtin_clz(unsigned(n)); }

using dg::Round;

// Pairwise-matching round: partner(i) == i keeps weight 1, matched pairs 1/2
// each.
template <class Partner>
Round matching_round(int n, Partner partner) {
  Round r;
  r.nbr.resize(n);
  r.w.resize(n);
  for (int i = 0; i < n; ++i) {
    const int p = partner(i);
    if (p == i) {
      r.nbr[i] = {i};
      r.w[i] = {1.0};
    } else {
      r.nbr[i] = {std::min(i, p), std::max(i, p)};
      r.w[i] = {0.5, 0.5};
    }
  }
  return r;
}

// Group-averaging round: every worker's group gets 1/|G| (AER).
Round group_round(int n, const std::vector<int>& group_of) {
  std::vector<std::vector<int>> members(n);
  for (int i = 0; i < n; ++i) members[group_of[i]].push_back(i);  // ascending by construction
  Round r;
  r.nbr.resize(n);
  r.w.resize(n);
  for (int i = 0; i < n; ++i) {
    const auto& g = members[group_of[i]];
    r.nbr[i] = g;
    r.w[i].assign(g.size(), 1.0 / double(g.size()));
  }
  return r;
}

// Symmetric eigenvalues (validation only), cyclic Jacobi rotations, descending.
std::vector<double> eig_sym(std::vector<double> a, int n) {
  auto A = [&](int i, int j) -> double& { return a[size_t(i) * n + j]; };
  for (int it = 0; it < 64; ++it) {
    double off = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if (i != j) off += A(i, j) * A(i, j);
    if (off < 1e-30) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double tau = (A(q, q) - A(p, p)) / (2 * apq);
        const double t = std::copysign(1.0, tau) / (std::fabs(tau) + std::hypot(1.0, tau));
        const double c = 1 / std::hypot(1.0, t), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- A J
          const double x = A(k, p), y = A(k, q);
          A(k, p) = c * x - s * y;
          A(k, q) = s * x + c * y;
        }
        for (int k = 0; k < n; ++k) {  // A <- J^T A
          const double x = A(p, k), y = A(q, k);
          A(p, k) = c * x - s * y;
          A(q, k) = s * x + c * y;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = A(i, i);
  std::sort(ev.rbegin(), ev.rend());
  return ev;
}

// MixingSchedule::from_matrices contract (topology.hpp:36-39): every round
// passes validate() and the period's union graph is connected.
dg_schedule* finish(int n, int wpn, std::vector<Round> rounds, const char* name = "custom") {
  if (rounds.empty()) dg::config_error("schedule: empty");
  for (size_t r = 0; r < rounds.size(); ++r) {
    const auto v = dg::validate_dense(
        [&] {
          std::vector<double> w(size_t(n) * n, 0.0);
          for (int i = 0; i < n; ++i)
            for (size_t k = 0; k < rounds[r].nbr[i].size(); ++k)
              w[size_t(i) * n + rounds[r].nbr[i][k]] = rounds[r].w[i][k];
          return w;
        }(),
        n);
    if (!(v.symmetric && v.nonnegative && v.rows_stochastic && v.cols_stochastic &&
          v.eigenvalues_in_range))
      dg::config_error("schedule: round " + std::to_string(r + 1) + " fails validate()");
  }
  std::vector<int> parent(n);
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  };
  for (const Round& rd : rounds)
    for (int i = 0; i < n; ++i)
      for (int j : rd.nbr[i]) parent[find(i)] = find(j);
  for (int i = 0; i < n; ++i)
    if (find(i) != find(0)) dg::config_error("schedule: union graph is disconnected");
  auto* s = new dg_schedule;
  s->n = n;
  s->wpn = wpn;
  s->name = name ? name : "";
  s->rounds = std::move(rounds);
  return s;
}

template <class Build>
int make(dg_schedule** out, Build&& b) {
  return dg::guarded([&] {
    if (!out) dg::config_error("null output handle");
    *out = nullptr;
    *out = b();
  });
}
}  // namespace

// ---------------------------------------------------------------- internals
void dg::set_error(int code, const std::string& msg, long iteration) {
  (void)code;
  t_err = msg;
  if (iteration >= 0) t_div = iteration;
}

const dg::Round& dg_schedule::at(long round) const {
  if (rounds.empty()) dg::config_error("schedule: empty (rejected by consumers, topology.hpp:42)");
  if (round < 1) dg::config_error("schedule: rounds are 1-based");
  return rounds[size_t((round - 1) % long(rounds.size()))];
}

std::vector<double> dg::dense(const dg_schedule& s, long round) {
  const Round& r = s.at(round);
  std::vector<double> w(size_t(s.n) * s.n, 0.0);
  for (int i = 0; i < s.n; ++i)
    for (size_t k = 0; k < r.nbr[i].size(); ++k) w[size_t(i) * s.n + r.nbr[i][k]] = r.w[i][k];
  return w;
}

// validate(W): topology.hpp:16-34,80; SPEC.md:130-136 (1e-12 tolerances,
// eigenvalues in (-1, 1]).
dg_validation dg::validate_dense(const std::vector<double>& w, int n) {
  dg_validation v{};
  constexpr double tol = 1e-12;
  v.min_entry = n ? w[0] : 0.0;
  std::vector<double> sym(size_t(n) * n);
  for (int i = 0; i < n; ++i) {
    double row = 0, col = 0;
    for (int j = 0; j < n; ++j) {
      const double a = w[size_t(i) * n + j], b = w[size_t(j) * n + i];
      v.max_asymmetry = std::max(v.max_asymmetry, std::fabs(a - b));
      v.min_entry = std::min(v.min_entry, a);
      row += a;
      col += b;
      sym[size_t(i) * n + j] = 0.5 * (a + b);
    }
    v.max_row_error = std::max(v.max_row_error, std::fabs(row - 1));
    v.max_col_error = std::max(v.max_col_error, std::fabs(col - 1));
  }
  v.symmetric = v.max_asymmetry <= tol;
  v.nonnegative = v.min_entry >= -tol;
  v.rows_stochastic = v.max_row_error <= tol;
  v.cols_stochastic = v.max_col_error <= tol;
  if (n > 0) {
    const auto ev = eig_sym(sym, n);
    v.max_eigenvalue = ev.front();
    v.min_eigenvalue = ev.back();
  }
  v.eigenvalues_in_range = v.symmetric && n > 0 && v.min_eigenvalue > -1 + 1e-10 &&
                           v.max_eigenvalue <= 1 + 1e-10;
  return v;
}

// Round plan for one rank: which sources each resident node mixes (in
// ascending global-id order) and which buckets cross NVLink.
dg::RoundPlan dg::build_round_plan(const dg_schedule& s, int world, int rank, long round) {
  const Round& rd = s.at(round);
  const int N = s.n;
  if (world < 1 || rank < 0 || rank >= world) config_error("plan: bad rank / world size");
  if (world > N) config_error("plan: more GPUs than nodes");
  RoundPlan p;
  const int first = first_node_of(rank, N, world), last = first_node_of(rank + 1, N, world);
  p.n_local = last - first;
  if (p.n_local > kMaxLocal) config_error("plan: more than 64 resident nodes per GPU");
  // distinct remote buckets needed here, ordered by (owner, node)
  std::vector<std::pair<int, int>> need;
  for (int i = first; i < last; ++i)
    for (int j : rd.nbr[i])
      if (j < first || j >= last) need.push_back({owner_of(j, N, world), j});
  std::sort(need.begin(), need.end());
  need.erase(std::unique(need.begin(), need.end()), need.end());
  if (int(need.size()) > kMaxRemote) config_error("plan: too many remote buckets per round");
  for (auto [peer, j] : need) {
    p.recv_peer.push_back(peer);
    p.recv_node.push_back(j);
  }
  auto slot_of = [&](int j) {
    return int(std::lower_bound(need.begin(), need.end(), std::make_pair(owner_of(j, N, world), j)) -
               need.begin());
  };
  for (int li = 0; li < p.n_local; ++li) {
    const int i = first + li;
    const auto& nb = rd.nbr[i];
    if (int(nb.size()) > kMaxDeg) config_error("plan: node degree above 16");
    p.deg[li] = int(nb.size());
    p.max_deg = std::max(p.max_deg, p.deg[li]);
    for (size_t k = 0; k < nb.size(); ++k) {
      const int j = nb[k];
      p.src[li][k] = (j >= first && j < last) ? j - first : p.n_local + slot_of(j);
      p.w[li][k] = rd.w[i][k];
    }
  }
  // mixing components: union-find over resident-resident edges of the round
  {
    std::vector<int> par(p.n_local);
    std::iota(par.begin(), par.end(), 0);
    auto find = [&](int x) {
      while (par[x] != x) x = par[x] = par[par[x]];
      return x;
    };
    for (int li = 0; li < p.n_local; ++li)
      for (int k = 0; k < p.deg[li]; ++k)
        if (p.src[li][k] < p.n_local) par[find(li)] = find(p.src[li][k]);
    std::vector<std::vector<int>> comps;
    std::vector<int> comp_of(p.n_local, -1);
    for (int li = 0; li < p.n_local; ++li) {  // ascending => components ordered by first node
      const int r = find(li);
      if (comp_of[r] < 0) {
        comp_of[r] = int(comps.size());
        comps.emplace_back();
      }
      comps[comp_of[r]].push_back(li);
    }
    size_t biggest = 0;
    for (const auto& c : comps) biggest = std::max(biggest, c.size());
    int cs = 1;
    while (cs < int(biggest)) cs <<= 1;
    if (int(comps.size()) * cs > kMaxLocal) {  // too much padding: one component of everything
      std::vector<int> all(p.n_local);
      std::iota(all.begin(), all.end(), 0);
      comps = {all};
      cs = 1;
      while (cs < p.n_local) cs <<= 1;
    }
    p.comp_size = cs;
    int nsb = 2;
    for (const auto& members : comps) {
      RoundPlan::Component c;
      c.members = members;
      std::vector<std::pair<int, int>> src;  // (global id, source code)
      for (int li : members)
        for (int k = 0; k < p.deg[li]; ++k) {
          const int sidx = p.src[li][k];
          const int code = sidx < p.n_local ? sidx : -(sidx - p.n_local + 1);
          const int gid = sidx < p.n_local ? first + sidx : p.recv_node[sidx - p.n_local];
          src.push_back({gid, code});
        }
      std::sort(src.begin(), src.end());
      src.erase(std::unique(src.begin(), src.end()), src.end());
      for (auto [gid, code] : src) c.srcs.push_back(code);
      c.w.assign(members.size(), std::vector<double>(src.size(), 0.0));
      for (size_t jm = 0; jm < members.size(); ++jm) {
        const int li = members[jm];
        for (int k = 0; k < p.deg[li]; ++k) {
          const int sidx = p.src[li][k];
          const int gid = sidx < p.n_local ? first + sidx : p.recv_node[sidx - p.n_local];
          const size_t pos =
              std::lower_bound(src.begin(), src.end(), std::make_pair(gid, INT32_MIN)) - src.begin();
          c.w[jm][pos] = p.w[li][k];
        }
      }
      while (nsb < int(src.size())) nsb <<= 1;
      p.comps.push_back(std::move(c));
    }
    p.src_bound = std::max(nsb, cs);
    // > 32 distinct sources (e.g. static exponential over many GPUs): the round
    // can only run x double-buffered, one gather per node (make_pingpong)
    p.oversize = p.src_bound > 32;
  }
  // sends: resident node j goes to every other rank hosting a node that mixes j
  std::vector<std::pair<int, int>> sends;
  for (int i = 0; i < N; ++i) {
    const int h = owner_of(i, N, world);
    if (h == rank) continue;
    for (int j : rd.nbr[i])
      if (j >= first && j < last) sends.push_back({h, j});
  }
  std::sort(sends.begin(), sends.end());
  sends.erase(std::unique(sends.begin(), sends.end()), sends.end());
  for (auto [h, j] : sends) {
    p.send_peer.push_back(h);
    p.send_node.push_back(j);
  }
  return p;
}

void dg::make_pingpong(RoundPlan& p, int first) {
  p.comps.clear();
  p.comp_size = 1;
  int nsb = 2;
  for (int li = 0; li < p.n_local; ++li) {
    RoundPlan::Component c;
    c.members = {li};
    std::vector<std::pair<int, int>> src;  // (global id, k)
    for (int k = 0; k < p.deg[li]; ++k) {
      const int sidx = p.src[li][k];
      src.push_back({sidx < p.n_local ? first + sidx : p.recv_node[sidx - p.n_local], k});
    }
    std::sort(src.begin(), src.end());
    c.w.assign(1, std::vector<double>());
    for (auto [gid, k] : src) {
      const int sidx = p.src[li][k];
      c.srcs.push_back(sidx < p.n_local ? sidx : -(sidx - p.n_local + 1));
      c.w[0].push_back(p.w[li][k]);
    }
    while (nsb < int(c.srcs.size())) nsb <<= 1;
    p.comps.push_back(std::move(c));
  }
  p.src_bound = nsb;
  p.pingpong = true;
}

// ================================================================== C ABI
extern "C" {

const char* dg_last_error(void) { return t_err.c_str(); }
long dg_last_divergence_iteration(void) { return t_div; }
int dg_version(void) { return 100; }

int dg_make_complete(int n, dg_schedule** out) {  // topology.hpp:65-66
  return make(out, [&] {
    if (n < 1) dg::config_error("make_complete: N must be >= 1");
    Round r;
    r.nbr.resize(n);
    r.w.resize(n);
    for (int i = 0; i < n; ++i) {
      r.nbr[i].resize(n);
      std::iota(r.nbr[i].begin(), r.nbr[i].end(), 0);
      r.w[i].assign(n, 1.0 / double(n));
    }
    return finish(n, 1, {r}, "complete");
  });
}

int dg_make_one_peer_ring(int n, dg_schedule** out) {  // topology.hpp:67-69
  return make(out, [&] {
    if (n < 2 || n % 2) dg::config_error("make_one_peer_ring: N must be even and >= 2");
    // round 1: (2k, 2k+1); round 2: (2k+1, 2k+2 mod N)
    Round r1 = matching_round(n, [](int i) { return i ^ 1; });
    Round r2 = matching_round(n, [n](int i) { return (i & 1) ? (i + 1) % n : (i + n - 1) % n; });
    return finish(n, 1, {r1, r2}, "one_peer_ring");
  });
}

int dg_make_one_peer_exponential(int n, dg_schedule** out) {  // topology.hpp:70-72
  return make(out, [&] {
    if (n < 2 || !pow2(n)) dg::config_error("make_one_peer_exponential: N must be a power of 2");
    std::vector<Round> rs;
    for (int r = 0; r < log2i(n); ++r) rs.push_back(matching_round(n, [r](int i) { return i ^ (1 << r); }));
    return finish(n, 1, rs, "one_peer_exponential");
  });
}

int dg_make_aer(int n, int wpn, dg_schedule** out) {  // topology.hpp:73-78
  return make(out, [&] {
    if (wpn < 1 || n < 1 || n % wpn) dg::config_error("make_aer: workers_per_node must divide N");
    const int M = n / wpn;
    if (M < 2 || !pow2(M)) dg::config_error("make_aer: node count must be a power of 2 >= 2");
    // merged node pair per round: Fig. 9 order for M=4;
    // hop distances 1,2,4..M/2 with (j, j+h), j & h == 0, ascending otherwise
    std::vector<std::pair<int, int>> merges;
    if (M == 2) {
      merges = {{0, 1}};
    } else if (M == 4) {
      merges = {{2, 3}, {0, 1}, {0, 2}, {1, 3}};
    } else {
      for (int h = 1; h < M; h <<= 1)
        for (int j = 0; j < M; ++j)
          if (!(j & h)) merges.push_back({j, j + h});
    }
    std::vector<Round> rs;
    for (auto [a, b] : merges) {
      std::vector<int> group(n);
      for (int i = 0; i < n; ++i) {
        const int node = i / wpn;
        group[i] = node == b ? a : node;
      }
      rs.push_back(group_round(n, group));
    }
    return finish(n, wpn, rs, "aer");
  });
}

int dg_make_static_exponential(int n, dg_schedule** out) {
  return make(out, [&] {
    if (n < 2) dg::config_error("static_exponential: N must be >= 2");
    Round r;
    r.nbr.resize(n);
    r.w.resize(n);
    for (int i = 0; i < n; ++i) {
      auto& nb = r.nbr[i];
      nb.push_back(i);
      for (int h = 1; h < n; h <<= 1) {
        nb.push_back((i + h) % n);
        nb.push_back((i - h % n + n) % n);
      }
      std::sort(nb.begin(), nb.end());
      nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
      r.w[i].assign(nb.size(), 1.0 / double(nb.size()));
    }
    return finish(n, 1, {r}, "static_exponential");
  });
}

int dg_schedule_from_matrices(const double* w, int n, int period, int wpn, dg_schedule** out) {
  return dg_schedule_from_matrices_named("custom", w, n, period, wpn, out);
}

int dg_schedule_from_matrices_named(const char* name, const double* w, int n, int period, int wpn,
                                    dg_schedule** out) {
  return make(out, [&] {  // topology.hpp:44-45
    if (!w || n < 1 || period < 1) dg::config_error("from_matrices: bad arguments");
    if (wpn < 1 || n % wpn) dg::config_error("from_matrices: workers_per_node must divide N");
    std::vector<Round> rs(period);
    for (int r = 0; r < period; ++r) {
      rs[r].nbr.resize(n);
      rs[r].w.resize(n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const double x = w[(size_t(r) * n + i) * n + j];
          if (x > 0.0) {
            rs[r].nbr[i].push_back(j);
            rs[r].w[i].push_back(x);
          }
        }
    }
    if (!name) dg::config_error("from_matrices: null name");
    dg_schedule* s = finish(n, wpn, rs, name);
    // finish() validated the positive part; negative entries must also fail
    for (int r = 0; r < period; ++r)
      for (size_t k = 0; k < size_t(n) * n; ++k)
        if (w[size_t(r) * n * n + k] < -1e-12) {
          delete s;
          dg::config_error("from_matrices: negative weight");
        }
    return s;
  });
}

int dg_schedule_info(const dg_schedule* s, int* workers, int* period, int* wpn, int* is_static) {
  return dg::guarded([&] {
    if (!s || s->rounds.empty()) dg::config_error("schedule: empty");
    if (workers) *workers = s->n;
    if (period) *period = int(s->rounds.size());
    if (wpn) *wpn = s->wpn;
    if (is_static) *is_static = s->rounds.size() == 1;
  });
}

int dg_schedule_neighbors(const dg_schedule* s, long round, int worker, int* idx, double* w,
                          int cap, int* count) {
  return dg::guarded([&] {
    if (!s) dg::config_error("schedule: null");
    const Round& r = s->at(round);
    if (worker < 0 || worker >= s->n) dg::config_error("neighbors_at: worker out of range");
    const auto& nb = r.nbr[worker];
    if (count) *count = int(nb.size());
    if (int(nb.size()) > cap) dg::config_error("neighbors_at: capacity too small");
    for (size_t k = 0; k < nb.size(); ++k) {
      if (idx) idx[k] = nb[k];
      if (w) w[k] = r.w[worker][k];
    }
  });
}

int dg_schedule_matrix(const dg_schedule* s, long round, double* w) {
  return dg::guarded([&] {
    if (!s || !w) dg::config_error("matrix_at: null argument");
    const auto d = dg::dense(*s, round);
    std::memcpy(w, d.data(), d.size() * sizeof(double));
  });
}

void dg_schedule_free(dg_schedule* s) { delete s; }

namespace {
void copy_out(const std::string& v, char* buf, size_t cap, size_t* len) {
  if (len) *len = v.size();
  if (buf && cap) {
    const size_t k = std::min(cap - 1, v.size());
    std::memcpy(buf, v.data(), k);
    buf[k] = '\0';
  }
  if (buf && cap <= v.size()) dg::config_error("string: capacity too small");
}
}  // namespace

int dg_schedule_name(const dg_schedule* s, char* buf, size_t cap, size_t* len) {  // topology.hpp:50
  return dg::guarded([&] {
    if (!s) dg::config_error("schedule: null");
    copy_out(s->name, buf, cap, len);
  });
}

int dg_validation_pass(const dg_validation* v) {  // MixingValidation::pass(), topology.hpp:29-32
  return v && v->symmetric && v->nonnegative && v->rows_stochastic && v->cols_stochastic &&
         v->eigenvalues_in_range;
}

int dg_validation_describe(const dg_validation* v, char* buf, size_t cap, size_t* len) {
  return dg::guarded([&] {  // MixingValidation::describe(), topology.hpp:33
    if (!v) dg::config_error("validation: null");
    auto yn = [](int b) { return b ? "yes" : "NO"; };
    char tmp[512];
    std::snprintf(tmp, sizeof(tmp),
                  "%s: symmetric=%s (max |w_ij - w_ji| %.3g), nonnegative=%s (min entry %.3g), "
                  "rows_stochastic=%s (max |row sum - 1| %.3g), cols_stochastic=%s (max |col sum - 1| %.3g), "
                  "eigenvalues_in_range=%s ([%.6g, %.6g] in (-1, 1])",
                  dg_validation_pass(v) ? "valid" : "INVALID", yn(v->symmetric), v->max_asymmetry,
                  yn(v->nonnegative), v->min_entry, yn(v->rows_stochastic), v->max_row_error,
                  yn(v->cols_stochastic), v->max_col_error, yn(v->eigenvalues_in_range), v->min_eigenvalue,
                  v->max_eigenvalue);
    copy_out(tmp, buf, cap, len);
  });
}

int dg_validate(const double* w, int n, dg_validation* out) {
  return dg::guarded([&] {
    if (!w || !out || n < 0) dg::config_error("validate: bad arguments");
    *out = dg::validate_dense(std::vector<double>(w, w + size_t(n) * n), n);
  });
}

int dg_spectral_lambda(const double* w, int n, double* out) {  // topology.hpp:82-84
  return dg::guarded([&] {
    if (!w || !out || n < 1) dg::config_error("spectral_lambda: bad arguments");
    std::vector<double> a(w, w + size_t(n) * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if (std::fabs(a[size_t(i) * n + j] - a[size_t(j) * n + i]) > 1e-12)
          dg::config_error("spectral_lambda: matrix is not symmetric");
    if (n == 1) {
      *out = 0.0;
      return;
    }
    const auto ev = eig_sym(a, n);
    *out = std::max(std::fabs(ev[1]), std::fabs(ev[n - 1]));
  });
}

int dg_effective_lambda(const dg_schedule* s, double* out) {  // topology.hpp:86-88
  return dg::guarded([&] {
    if (!s || !out || s->rounds.empty()) dg::config_error("effective_lambda: empty schedule");
    const int n = s->n;
    std::vector<double> p(size_t(n) * n, 0.0), q(size_t(n) * n);
    for (int i = 0; i < n; ++i) p[size_t(i) * n + i] = 1.0;
    for (size_t r = 0; r < s->rounds.size(); ++r) {  // P <- W^(r) P, sparse rows
      const Round& rd = s->rounds[r];
      std::fill(q.begin(), q.end(), 0.0);
      for (int i = 0; i < n; ++i)
        for (size_t k = 0; k < rd.nbr[i].size(); ++k)
          for (int j = 0; j < n; ++j)
            q[size_t(i) * n + j] += rd.w[i][k] * p[size_t(rd.nbr[i][k]) * n + j];
      std::swap(p, q);
    }
    for (double& x : p) x -= 1.0 / double(n);
    std::vector<double> ata(size_t(n) * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) ata[size_t(i) * n + j] += p[size_t(k) * n + i] * p[size_t(k) * n + j];
    *out = std::sqrt(std::max(0.0, eig_sym(ata, n).front()));
  });
}

int dg_plan_exchange(const dg_schedule* s, int world, int rank, long round, int* send_peer,
                     int* send_node, int* nsend, int* recv_peer, int* recv_node, int* nrecv,
                     int cap) {
  return dg::guarded([&] {
    if (!s) dg::config_error("plan: null schedule");
    const auto p = dg::build_round_plan(*s, world, rank, round);
    if (nsend) *nsend = int(p.send_node.size());
    if (nrecv) *nrecv = int(p.recv_node.size());
    if (int(p.send_node.size()) > cap || int(p.recv_node.size()) > cap)
      dg::config_error("plan: capacity too small");
    for (size_t k = 0; k < p.send_node.size(); ++k) {
      if (send_peer) send_peer[k] = p.send_peer[k];
      if (send_node) send_node[k] = p.send_node[k];
    }
    for (size_t k = 0; k < p.recv_node.size(); ++k) {
      if (recv_peer) recv_peer[k] = p.recv_peer[k];
      if (recv_node) recv_node[k] = p.recv_node[k];
    }
  });
}

}  // extern "C"
