// dg_internal.hpp -- shared host-side declarations of libdg (not part of the ABI).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "dg.h"

namespace dg {

// ------------------------------------------------------------------ errors
// C++ exceptions inside the library, mapped to dg_status at the C boundary
// (mirrors errors.hpp:8-26).
struct Error : std::runtime_error {
  int code;
  long iteration;
  Error(int c, const std::string& m, long it = -1) : std::runtime_error(m), code(c), iteration(it) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(DG_CONFIG_ERROR, m); }

void set_error(int code, const std::string& msg, long iteration = -1);

template <class F>
int guarded(F&& f) {
  try {
    f();
    return DG_OK;
  } catch (const Error& e) {
    set_error(e.code, e.what(), e.iteration);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error(DG_CONFIG_ERROR, "host allocation failed");
    return DG_CONFIG_ERROR;
  } catch (const std::exception& e) {
    set_error(DG_INVARIANT, e.what());
    return DG_INVARIANT;
  }
}

// ------------------------------------------------------------------ schedule
// Immutable periodic schedule (topology.hpp:40-63) stored as closed-form
// neighbour tables: per round, per worker, ascending neighbour ids (self
// included) and weights.  Dense matrices are materialised on demand.
struct Round {
  std::vector<std::vector<int>> nbr;     // [worker] ascending
  std::vector<std::vector<double>> w;    // [worker] aligned with nbr
};

}  // namespace dg

struct dg_schedule {
  int n = 0;
  int wpn = 1;
  std::string name;  // MixingSchedule::name() (topology.hpp:50)
  std::vector<dg::Round> rounds;
  const dg::Round& at(long round) const;  // 1-based periodic; throws ConfigError
};

namespace dg {

std::vector<double> dense(const dg_schedule& s, long round);
dg_validation validate_dense(const std::vector<double>& w, int n);

// ------------------------------------------------------------------ plans
constexpr int kMaxLocal = 64;   // resident nodes per GPU (64 x 125M x 16 B = 128 GB fits one B200)
constexpr int kMaxDeg = 16;     // neighbours per node (self included)
constexpr int kMaxRemote = kMaxLocal * kMaxDeg;  // distinct remote buckets per round per GPU (implied bound)

// Placement: node i lives on rank floor(i*G/N) (SURVEY.md 8 common notation).
inline int owner_of(int node, int nodes, int world) {
  return int((long long)node * world / nodes);
}
inline int first_node_of(int rank, int nodes, int world) {
  return int(((long long)rank * nodes + world - 1) / world);
}

// One round's execution plan for one rank.
struct RoundPlan {
  int n_local = 0;
  // mixing plan, sources: [0, n_local) = resident node buckets, n_local + r = recv slot r
  int deg[kMaxLocal] = {};
  int src[kMaxLocal][kMaxDeg] = {};
  double w[kMaxLocal][kMaxDeg] = {};  // w_ij (the kernel mixes in fp64, rounds once)
  int max_deg = 0;
  // mixing components: connected pieces of the round's mixing graph restricted
  // to this GPU (one kernel grid row each)
  struct Component {
    std::vector<int> members;            // resident node indices, ascending
    std::vector<int> srcs;               // distinct sources, ascending global id:
                                         //   >= 0 resident node index, < 0 recv slot -(r+1)
    std::vector<std::vector<double>> w;  // [member][source] weight, 0 = not a neighbour
  };
  std::vector<Component> comps;
  int comp_size = 1;  // NC: power of two >= largest member count (comps * NC <= 16)
  int src_bound = 2;  // NS: power of two >= largest source count, >= NC
  // x double-buffered for this round: every resident node is its own
  // component reading x^(t-1) from the current x buffer and writing x^(t) to
  // the other one (large mixing components; see make_pingpong)
  bool pingpong = false;
  // some component has > 32 distinct sources: the round must run ping-pong
  bool oversize = false;
  // P2P transport: pull each distinct remote bucket once into local slots with
  // the copy engines (set when resident nodes read the same remote buckets
  // >= 1.75x on average: in-kernel peer loads bypass the local L2 and cross
  // NVLink once per reader, but run ~1.8x faster than copy-engine pulls)
  bool pull = false;
  // run on the x-sharing kernel (xshare.cuh); otherwise the legacy.cu kernels
  bool xshare = false;
  // exchange (ordered by (peer, node))
  std::vector<int> send_peer, send_node;  // send_node: global id of a resident node
  std::vector<int> recv_peer, recv_node;  // recv slot r holds recv_node[r]
};

RoundPlan build_round_plan(const dg_schedule& s, int world, int rank, long round);
// Re-express a round plan as one single-member component per resident node
// (sources = that node's neighbours, ascending global id) for the
// double-buffered x path.
void make_pingpong(RoundPlan& p, int first_node);

}  // namespace dg
