// The INTEGRATION.md section-2 adapter pattern as a compiled C++20 consumer of
// include/dg.h: a declab-shaped MixingSchedule / validate() / error taxonomy
// (topology.hpp:14-100, errors.hpp:8-26) implemented over the C ABI, with
// std::vector row-major matrices standing in for Eigen (absent in this image).
// tests/test_c_abi.py compiles it with g++ and checks its output against the
// oracle.  Prints one line per schedule round and per worker.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "dg.h"

namespace declab_b200 {

// errors.hpp taxonomy <- dg_status
struct ConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DivergenceError : std::runtime_error {
  long iteration;
  DivergenceError(long it, const std::string& m) : std::runtime_error(m), iteration(it) {}
};
struct InvariantError : std::logic_error {
  using std::logic_error::logic_error;
};

inline void check(int rc) {
  if (rc == DG_OK) return;
  const std::string m = dg_last_error();
  if (rc == DG_CONFIG_ERROR) throw ConfigError(m);
  if (rc == DG_DIVERGENCE) throw DivergenceError(dg_last_divergence_iteration(), m);
  throw InvariantError(m);
}

using Matrix = std::vector<double>;  // n x n row-major

// MixingSchedule (topology.hpp:40-63): immutable, owns the C handle
class MixingSchedule {
 public:
  explicit MixingSchedule(dg_schedule* s) : s_(s) {
    int st = 0;
    check(dg_schedule_info(s_, &n_, &p_, &wpn_, &st));
    static_ = st != 0;
  }
  MixingSchedule(const MixingSchedule&) = delete;
  MixingSchedule& operator=(const MixingSchedule&) = delete;
  ~MixingSchedule() { dg_schedule_free(s_); }
  int workers() const { return n_; }
  int period() const { return p_; }
  int workers_per_node() const { return wpn_; }
  bool is_static() const { return static_; }
  std::string name() const {
    char buf[64];
    size_t len = 0;
    check(dg_schedule_name(s_, buf, sizeof buf, &len));
    return std::string(buf, len);
  }
  Matrix matrix_at(long round) const {
    Matrix w(static_cast<size_t>(n_) * static_cast<size_t>(n_));
    check(dg_schedule_matrix(s_, round, w.data()));
    return w;
  }
  // neighbors_at(t)[i]: ascending, self included (topology.hpp:54)
  std::vector<std::vector<int>> neighbors_at(long round) const {
    std::vector<std::vector<int>> out(static_cast<size_t>(n_));
    std::vector<int> idx(static_cast<size_t>(n_));
    std::vector<double> w(static_cast<size_t>(n_));
    for (int i = 0; i < n_; ++i) {
      int cnt = 0;
      check(dg_schedule_neighbors(s_, round, i, idx.data(), w.data(), n_, &cnt));
      out[size_t(i)].assign(idx.begin(), idx.begin() + cnt);
    }
    return out;
  }

 private:
  dg_schedule* s_;
  int n_ = 0, p_ = 0, wpn_ = 1;
  bool static_ = false;
};

inline MixingSchedule make_one_peer_exponential(int n) {
  dg_schedule* s = nullptr;
  check(dg_make_one_peer_exponential(n, &s));
  return MixingSchedule(s);
}
inline MixingSchedule make_aer(int n, int wpn) {
  dg_schedule* s = nullptr;
  check(dg_make_aer(n, wpn, &s));
  return MixingSchedule(s);
}
inline MixingSchedule make_static_exponential(int n) {
  dg_schedule* s = nullptr;
  check(dg_make_static_exponential(n, &s));
  return MixingSchedule(s);
}

inline dg_validation validate(const Matrix& w, int n) {
  dg_validation v;
  check(dg_validate(w.data(), n, &v));
  return v;
}

}  // namespace declab_b200

int main() {
  using namespace declab_b200;
  auto dump = [](const char* label, const MixingSchedule& s) {
    std::printf("schedule %s name=%s n=%d period=%d wpn=%d static=%d\n", label, s.name().c_str(), s.workers(),
                s.period(), s.workers_per_node(), int(s.is_static()));
    for (long r = 1; r <= s.period(); ++r) {
      const auto nb = s.neighbors_at(r);
      for (int i = 0; i < s.workers(); ++i) {
        std::printf("round %ld worker %d:", r, i);
        for (int j : nb[size_t(i)]) std::printf(" %d", j);
        std::printf("\n");
      }
      const dg_validation v = validate(s.matrix_at(r), s.workers());
      std::printf("validate %s round %ld pass=%d\n", label, r, dg_validation_pass(&v));
    }
  };
  dump("one_peer_exponential8", make_one_peer_exponential(8));
  dump("aer8_2", make_aer(8, 2));
  dump("static_exponential8", make_static_exponential(8));
  try {
    make_one_peer_exponential(6);  // not a power of two -> ConfigError (errors.hpp:10-12)
    std::printf("error none\n");
  } catch (const ConfigError& e) {
    std::printf("error ConfigError\n");
  }
  return 0;
}
