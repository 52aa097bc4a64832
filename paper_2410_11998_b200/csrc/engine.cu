// engine.cu -- device side of libdg: semantic per-node steps and the fused
// gossip + Adam engine (one per GPU) with the chunked, double-buffered NCCL
// exchange over NVLink.
//
// Replaces the hot loop of the reference's trainsim (Jacobi
// snapshot, mixed sum, per-worker dadam_step / accum_adam_step) and the
// paper's bucketed overlap (Fig. 1).
#include <cuda.h>  // CUstream / CUdeviceptr types for the stream memory operations (entry points)
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>

#include "dg_internal.hpp"
#include "kernels.cuh"
#include "launch.hpp"
#include "xshare.cuh"

namespace dg {
namespace {

constexpr size_t kDefaultChunk = 6553600;  // 25 MiB of fp32 (PAPER.md:328 DDP bucket)
constexpr size_t kAlign = 64;              // floats: 256-byte aligned node buckets / chunks


void check_cfg(const dg_adam_cfg* c) {  // OptimizerConfig invariants
  if (!c) config_error("optimizer: null config");
  if (!(c->alpha > 0.0)) config_error("optimizer: alpha must be > 0");
  if (!(c->beta1 >= 0.0 && c->beta1 < c->beta2 && c->beta2 < 1.0))
    config_error("optimizer: need 0 <= beta1 < beta2 < 1");
  if (!(c->eps > 0.0)) config_error("optimizer: eps must be > 0");
}

// Per-step scalars: alpha, beta1, beta2, eps are first
// rounded to fp32 (the bucket precision); every derived scalar (1 - beta,
// bias corrections) is computed in double from those and cast once, so e.g.
// beta2 + (1 - beta2) == 1 for the values the kernel multiplies with.
// t = 0 -> ConfigError; AccumAdam: T mod s == 0, t <= T
// (SPEC.md:292-294), bias-correction exponent ceil(t/s) (Alg. 3 line 4).
DevScalars scalars(const dg_adam_cfg* cin, int algo, long t, long T, bool* fold) {
  check_cfg(cin);
  dg_adam_cfg rounded = *cin;
  rounded.alpha = double(float(cin->alpha));
  rounded.beta1 = double(float(cin->beta1));
  rounded.beta2 = double(float(cin->beta2));
  rounded.eps = double(float(cin->eps));
  const dg_adam_cfg* c = &rounded;
  if (t < 1) config_error("step: t must be >= 1");
  long tau = t;
  if (algo == DG_ALGO_ACCUM) {
    if (c->s < 1) config_error("accum_adam_step: s must be >= 1");
    if (T < 1 || T % c->s) config_error("accum_adam_step: T mod s != 0");
    if (t > T) config_error("accum_adam_step: t exceeds T");
    tau = (t + c->s - 1) / c->s;
  } else if (algo != DG_ALGO_DADAM && algo != DG_ALGO_ALLREDUCE) {
    config_error("unknown algorithm");
  }
  if (fold) *fold = algo == DG_ALGO_ACCUM && t % c->s == 0;
  const double bv = c->paper_literal ? c->beta1 : c->beta2;
  DevScalars s;
  s.b1 = float(c->beta1);
  s.omb1 = float(1.0 - c->beta1);
  s.b2 = float(c->beta2);
  s.omb2 = float(1.0 - c->beta2);
  s.c1 = float(1.0 / (1.0 - std::pow(c->beta1, double(tau))));
  s.c2 = float(1.0 / (1.0 - std::pow(c->beta2, double(tau))));
  s.neg_alpha = float(-c->alpha);
  s.eps = float(c->eps);
  s.inv_s = float(1.0 / double(algo == DG_ALGO_ACCUM ? c->s : 1));
  s.bv = float(bv);
  s.ombv = float(1.0 - bv);
  return s;
}

// StreamRng state for (seed, purpose, worker, iteration) (rng.cpp:26-33).
uint64_t host_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t stream_state(uint64_t seed, uint64_t purpose, uint64_t worker, uint64_t iteration) {
  constexpr uint64_t g = 0x9e3779b97f4a7c15ull;
  uint64_t s = host_mix64(seed + g);
  s = host_mix64((s + g) ^ purpose);
  s = host_mix64((s + g) ^ worker);
  s = host_mix64((s + g) ^ iteration);
  return s;
}

unsigned grid_for(long long work_items, int blocks_per_sm) {
  const long long want = (work_items + 255) / 256;
  const long long cap = (long long)current_sms() * blocks_per_sm;
  return unsigned(std::max(1LL, std::min(want, cap)));
}

// Semantic-step divergence flag (one per device; the module global).
__device__ int g_semantic_flag = INT_MAX;
int* semantic_flag() {
  void* p = nullptr;
  CU(cudaGetSymbolAddress(&p, g_semantic_flag));
  return static_cast<int*>(p);
}

// ------------------------------------------------------------------ stream memory operations
// In-place P2P transport (DDP buckets): per-range cross-GPU ordering with
// stream-ordered 64-bit flags -- cuStreamWaitValue64 on this GPU's own flag
// array (the front end waits, no SM spins) and cuStreamWriteValue64 into the
// peers' flag arrays (IPC-mapped), resolved through the runtime's driver
// entry points so libdg does not link libcuda.
struct MemOps {
  CUresult (*wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
  CUresult (*write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
};
const MemOps& memops() {
  static const MemOps m = [] {
    MemOps r;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", reinterpret_cast<void**>(&r.wait64), cudaEnableDefault,
                                &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      r.wait64 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&r.write64), cudaEnableDefault,
                                &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      r.write64 = nullptr;
    cudaGetLastError();
    return r;
  }();
  return m;
}
void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw Error(DG_CUDA_ERROR, std::string(what) + ": CUresult " + std::to_string(int(r)));
}
// DG_SIGNAL_KERNEL=1: peers' flags written by a 1-warp kernel (release stores
// over NVLink) instead of cuStreamWriteValue64
constexpr int kMaxSignal = 8;
struct SignalArgs {
  unsigned long long* dst[kMaxSignal];
  int n;
  unsigned long long value;
};
__global__ void signal_peers(const __grid_constant__ SignalArgs a) {
  if (threadIdx.x < a.n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.dst[threadIdx.x]), "l"(a.value) : "memory");
  }
}

// ------------------------------------------------------------------ x-sharing launch (default K1)
// DG_XSHARE: 1 (default) the x-sharing kernel (xshare.cuh) wherever every
// round fits it, 0 the register-streaming kernels of legacy.cu (round-1
// paths, kept for sweeps and for rounds with > 8 members, sources or
// neighbours per mixing component).
bool xshare_enabled() {
  static const bool v = env_int("DG_XSHARE", 1) != 0;
  return v;
}
// DG_PREFETCH: column blocks (32 float4 columns, 512 B per stream) the
// x-sharing kernel prefetches into L2 ahead of use (default 1, 0 = off)
int xshare_prefetch() {
  static const int v = std::max(0, std::min(64, env_int("DG_PREFETCH", 1)));
  return v;
}

// Host image of one round's groups: whole mixing components packed first-fit
// into groups of <= 8 members and <= 8 source rows (rows of different
// components are never shared, so a member's sum only sees its own
// component's rows, ascending global id).
struct GroupPlan {
  struct Group {
    std::vector<int> members;           // resident node indices
    std::vector<int> srcs;              // rows: >= 0 resident node index, < 0 recv slot -(r+1)
    std::vector<std::vector<double>> w; // [member][row]
  };
  bool ok = false;
  bool colw = true;  // every source row is read with one weight by all its readers
  int max_deg = 0;
  std::vector<Group> groups;
};

GroupPlan build_group_plan(const RoundPlan& p) {
  GroupPlan gp;
  for (const auto& c : p.comps) {
    const int cm = int(c.members.size()), cs = int(c.srcs.size());
    if (cm > kShNodes || cs > kShRows) return gp;  // ok = false
    if (gp.groups.empty() || int(gp.groups.back().members.size()) + cm > kShNodes ||
        int(gp.groups.back().srcs.size()) + cs > kShRows)
      gp.groups.emplace_back();
    auto& g = gp.groups.back();
    const int r0 = int(g.srcs.size());
    for (auto& row : g.w) row.resize(r0 + cs, 0.0);
    g.srcs.insert(g.srcs.end(), c.srcs.begin(), c.srcs.end());
    for (int jm = 0; jm < cm; ++jm) {
      g.members.push_back(c.members[jm]);
      std::vector<double> row(r0 + cs, 0.0);
      int deg = 0;
      for (int k = 0; k < cs; ++k) {
        row[r0 + k] = c.w[jm][k];
        deg += c.w[jm][k] != 0.0;
      }
      if (deg > kShDeg) return gp;
      gp.max_deg = std::max(gp.max_deg, deg);
      g.w.push_back(row);
    }
    for (int k = 0; k < cs; ++k) {  // column-uniform weights?
      double wk = 0.0;
      for (int jm = 0; jm < cm; ++jm) {
        const double x = c.w[jm][k];
        if (x == 0.0) continue;
        if (wk == 0.0) wk = x;
        else if (x != wk) gp.colw = false;
      }
    }
  }
  gp.ok = !gp.groups.empty();
  return gp;
}

template <int DEG, int ALGO, bool FOLD, bool COLW, bool XP>
void launch_xshare_t(const ShArgs& a, int ngroups, int warps, int sms, cudaStream_t st) {
  auto kern = gossip_adam_xshare<DEG, ALGO, FOLD, COLW, XP>;
  static std::map<int, int> occ_of;  // resident CTAs per SM by CTA size
  int& occ = occ_of[warps];
  if (!occ) {
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * warps, 0), "xshare occupancy");
    occ = std::max(1, occ);
  }
  const long long blocks = std::max(1LL, ((a.n >> 2) + 31) / 32);
  const long long resident = std::max(1LL, (long long)(grid_waves() * occ * sms) / ngroups);
  dim3 grid(unsigned(std::min(blocks, resident)), unsigned(ngroups));
  kern<<<grid, 32 * warps, 0, st>>>(a);
}

void launch_xshare(const ShArgs& a, int ngroups, int warps, int max_deg, bool colw, int algo, bool fold,
                   int sms, cudaStream_t st, bool xp) {
#define DG_XS_X(D, A, F, C)                                            \
  if (xp) {                                                            \
    return launch_xshare_t<D, A, F, C, true>(a, ngroups, warps, sms, st);  \
  } else {                                                             \
    return launch_xshare_t<D, A, F, C, false>(a, ngroups, warps, sms, st); \
  }
#define DG_XS_C(D, A, F) \
  if (colw) {            \
    DG_XS_X(D, A, F, true)  \
  } else {               \
    DG_XS_X(D, A, F, false) \
  }
#define DG_XS_D(A, F)   \
  if (max_deg <= 2) {   \
    DG_XS_C(2, A, F)    \
  } else if (max_deg <= 4) { \
    DG_XS_C(4, A, F)    \
  } else if (max_deg <= 6) { \
    DG_XS_C(6, A, F)    \
  } else {              \
    DG_XS_C(8, A, F)    \
  }
  if (algo == DG_ALGO_DADAM) {
    DG_XS_D(0, false)
  } else if (fold) {
    DG_XS_D(1, true)
  } else {
    DG_XS_D(1, false)
  }
#undef DG_XS_D
#undef DG_XS_C
#undef DG_XS_X
}

}  // namespace
}  // namespace dg

// ===================================================================== engine
struct dg_engine {
  // configuration
  int N = 0, G = 1, rank = 0, device = 0, algo = 0, first = 0, NL = 0, P = 0;
  size_t d = 0, d_pad = 0, chunk = 0, n_chunks = 0;
  long T = 0;
  dg_adam_cfg adam{};
  std::vector<dg::RoundPlan> plans;
  int max_recv = 0;
  // device memory
  float* arena[5] = {};  // X, G, M, V, ACC: [NL][d_pad]
  float* slots = nullptr;  // [2][max_recv][chunk]
  int* flag = nullptr;     // first divergent iteration (INT_MAX = none)
  // streams / events
  cudaStream_t comp = nullptr, comm = nullptr;
  cudaEvent_t ev_begin = nullptr, ev_slot_free[2] = {};
  std::vector<cudaEvent_t> ev_recv;
  ncclComm_t nccl = nullptr;
  // stats
  long launches = 0, steps = 0;
  double sent = 0, received = 0, hbm = 0;
  std::vector<unsigned char> argbuf;
  bool xshare = false;  // x-sharing kernel for every round (decided globally)
  std::vector<dg::GroupPlan> gplans;  // per round
  dg::ShArgs sargs;
  void launch_groups(const dg::GroupPlan& tp, float* const* x, float* const* xo, const float* const* g,
                          float* const* m, float* const* v, float* const* b, const float* const* slot_ptr,
                          size_t off, size_t len, const dg::DevScalars& s, bool fold, long t, int sms,
                          float* const* xp = nullptr);
  // optional per-launch CUDA-event timing (bench roofline)
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
  std::vector<double> tev_bytes;
  size_t tev_used = 0;
  double kernel_ms = 0, timed_bytes = 0;
  long timed_launches = 0;
  void harvest_timing();
  // times (optionally) and counts one launch of ours on the compute stream
  template <class F>
  void timed(double bytes, double nvl_bytes, F&& launch, int kernels = 1);
  std::vector<double> tev_remote;  // NVLink bytes read in-kernel per timed launch
  double remote_ms = 0, remote_bytes = 0;
  // bucketed steps (f1)
  bool in_place = false;
  float* rbuf = nullptr;                     // [max_recv][d_pad] recv buffers for step_range
  std::map<size_t, cudaEvent_t> range_ev;   // exchange-complete event per range offset
  std::map<size_t, long> range_posted;      // iteration whose exchange is posted per range
  cudaEvent_t ev_user = nullptr;
  void post_range_exchange(const dg::RoundPlan& q, size_t off, size_t len);
  void step_range(long t, size_t off, size_t len);
  // All-Reduce Adam (f3)
  double* gsum = nullptr;  // [d_pad] fp64 gradient column sums
  double* xbar_ref = nullptr;  // fixed fp64 column sums for the consensus error (f2)
  int* inv_flag = nullptr; // first iteration with drifting workers (INT_MAX = none)
  void step_allreduce(long t, const dg::DevScalars& s);

  float* x_alt = nullptr;  // second x buffer (ping-pong rounds)
  int xcur = 0;            // which x buffer holds the current x (identical on every rank)
  // P2P transport: every rank's two x buffers mapped into this process (CUDA IPC)
  int transport = DG_TRANSPORT_P2P;
  std::vector<float*> peer_base[2];  // [buffer][rank]; own rank = own pointers
  std::vector<char> round_remote;    // per round: any rank mixes a remote bucket
  float* bar_buf = nullptr;          // 1-element all-reduce = cross-GPU step barrier
  std::vector<cudaStream_t> pull;    // copy-engine pull streams (pull rounds)
  std::vector<cudaEvent_t> pull_ev;
  long barriers = 0;
  // DG_NCCL_REGISTER=1: NCCL user-buffer registration of the exchanged
  // buffers (x, x_alt, recv slots, range buffers) for zero-copy p2p
  std::vector<void*> nccl_regs;
  void nccl_register(void* p, size_t bytes) {
    static const bool on = dg::env_int("DG_NCCL_REGISTER", 0) != 0;
    if (!on || !nccl || !p) return;
    void* h = nullptr;
    NC(ncclCommRegister(nccl, p, bytes, &h));
    nccl_regs.push_back(h);
  }
  const float* peer_x(int node) const {
    const int owner = dg::owner_of(node, N, G);
    return peer_base[xcur][owner] + size_t(node - dg::first_node_of(owner, N, G)) * d_pad;
  }
  float* buf(int which, int local) const {
    const float* base = (which == DG_BUF_X && xcur) ? x_alt : arena[which];
    return const_cast<float*>(base) + size_t(local) * d_pad;
  }
  float* x_other(int local) const { return (xcur ? arena[DG_BUF_X] : x_alt) + size_t(local) * d_pad; }
  // SMs the fused kernel may fill: all of them in intra-GPU rounds; in exchange
  // rounds DG_RESERVE_SMS (default 0) are left to NCCL's kernels
  int sm_total = 0, reserve_sms = 0;
  bool diag_skip_kernel = false;  // DG_DIAG_SKIP_KERNEL: exchange only (diagnostics; wrong results)
  int sms_for(const dg::RoundPlan& p) const {
    const bool comm = !(p.send_node.empty() && p.recv_node.empty());
    return std::max(1, comm ? sm_total - reserve_sms : sm_total);
  }
  // Fault injection for the exchange-protocol tests (DG_FAULT_*, read at
  // create time; INTEGRATION.md "Environment"): delay this rank's streams,
  // and overwrite every consumed buffer with NaN as soon as the protocol
  // declares it free, so a missing wait shows up as a divergence or a
  // mismatch instead of passing on benign timing.
  long long fault_ns = 0;  // spin per step on this rank (DG_FAULT_DELAY_US, DG_FAULT_RANK)
  bool poison = false;     // DG_FAULT_POISON=1
  void fault_delay(cudaStream_t st) {
    if (fault_ns > 0) {
      dg::fault_spin<<<1, 1, 0, st>>>(fault_ns);
      CU(cudaGetLastError());
    }
  }
  void poison_range(float* p, size_t n, cudaStream_t st) {
    if (poison && p && n) CU(cudaMemsetAsync(p, 0xFF, n * sizeof(float), st));  // 0xFFFFFFFF = NaN
  }
  void enqueue_fused(const dg::RoundPlan& p, size_t off, size_t len, int slot_set,
                     const dg::DevScalars& s, bool fold, long t, const float* const* slot_override = nullptr,
                     float* const* xpub_out = nullptr);
  void step(long t);
  // In-place P2P transport (DG_ENGINE_IN_PLACE + P2P; the f1 DDP wrapper):
  // x never moves, so each update also publishes x^(t) into xpub[t % 2],
  // which peers read in-kernel over NVLink at t + 1.  Per range and rank, a
  // 64-bit flag "finished iteration v - 1" orders it: before updating range
  // k at t a rank waits until every peer signalled t (its x^(t-1) is
  // published and it has finished reading our x^(t-2) in xpub[t % 2]), then
  // signals t + 1 to every peer.
  bool inplace_p2p = false;
  float* xpub[2] = {};                      // [NL][d_pad] each
  unsigned long long* sig = nullptr;        // [kMaxRanges][G], written by the peers
  std::vector<unsigned long long*> peer_sig;  // every rank's sig (own = sig)
  std::map<size_t, int> range_slot;         // range offset -> flag row (first-use order)
  std::map<size_t, long> range_last;        // last iteration stepped per range
  bool signal_kernel = false;
  // push variant (DG_INPLACE_PUSH, default on when every resident node has at
  // most one remote reader rank per round): the update kernel STORES x^(t)
  // straight into the reader's receive slot over NVLink (posted writes) and
  // reads its own neighbours' x^(t-1) from local slots; xpub[] are then the
  // receive buffers [parity][recv slot][d_pad].  Same flags, same waits.
  bool push = false;
  std::vector<std::vector<std::pair<int, int>>> push_dst;  // [round][local node] -> (reader rank, its slot) or (-1,-1)
  static constexpr int kMaxRanges = 4096;
  // P2P push exchange (DG_P2P_PUSH=1, engines that are not in place): every
  // step's kernel also stores x^(t) of each resident node into the receive
  // slots of its remote readers of round t+1 (posted NVLink writes), so every
  // round reads only local memory and x is updated in place; a stream-ordered
  // barrier before every step orders the slot parities.  x^(t-1) is seeded
  // with peer copies before a step when x changed outside the engine.
  bool p2p_push = false;
  float* pbuf[2] = {};  // receive slots [parity][max_recv][d_pad], written by the peers
  std::vector<std::vector<std::array<std::pair<int, int>, dg::kPushMax>>> pdst;  // [round][local] -> (rank, slot)
  long seeded_for = -1;  // step whose x^(t-1) is in the readers' slots
  void push_seed(long t);
  void step_range_p2p(long t, size_t off, size_t len);
  void signal_range(int slot, unsigned long long value);
  // CUDA graphs of whole step ranges (dg_engine_run_steps): small buckets are
  // launch-bound (BASELINE config 1: 8 x 2^20 params, ~36 us of HBM per step),
  // so t_first..t_last are captured once from the compute stream (and the
  // streams it forks to) and replayed as one graph launch.  A graph bakes in
  // the x buffer it starts from, so it replays only from the same xcur.
  struct GraphRec {
    long t0 = 0, t1 = 0;
    int x0 = 0, x1 = 0;
    cudaGraphExec_t exec = nullptr;
    long launches = 0, steps = 0, barriers = 0;
    double hbm = 0, sent = 0, received = 0, remote = 0;
  };
  std::vector<GraphRec> graphs;
  bool capturing = false;
  double cap_hbm = 0, cap_remote = 0;
  long cap_launches = 0;
  std::vector<long> tev_n;  // kernels covered by each timed record
  GraphRec& capture(long t0, long t1);
  void run_steps(long t0, long t1, int flags);
  ~dg_engine();
};

dg_engine::~dg_engine() {
  if (device >= 0) cudaSetDevice(device);
  if (comp) cudaStreamSynchronize(comp);
  if (comm) cudaStreamSynchronize(comm);
  // P2P: peers may still be reading this rank's exported x buffers over NVLink
  // (their last exchange-round kernel); one more stream-ordered barrier before
  // anything exported is unmapped or freed (destroy is collective)
  if (transport == DG_TRANSPORT_P2P && G > 1 && nccl && bar_buf && comp) {
    if (ncclAllReduce(bar_buf, bar_buf, 1, ncclFloat, ncclSum, nccl, comp) == ncclSuccess)
      cudaStreamSynchronize(comp);
  }
  for (void* h : nccl_regs) ncclCommDeregister(nccl, h);
  if (nccl) ncclCommDestroy(nccl);
  for (float* a : arena)
    if (a) cudaFree(a);
  if (slots) cudaFree(slots);
  if (x_alt) cudaFree(x_alt);
  if (bar_buf) cudaFree(bar_buf);
  for (int r = 0; r < int(peer_sig.size()); ++r)
    if (r != rank && peer_sig[r]) cudaIpcCloseMemHandle(peer_sig[r]);
  for (float* p : xpub)
    if (p) cudaFree(p);
  for (float* p : pbuf)
    if (p) cudaFree(p);
  if (sig) cudaFree(sig);
  for (int b = 0; b < 2; ++b)
    for (int r = 0; r < int(peer_base[b].size()); ++r)
      if (r != rank && peer_base[b][r]) cudaIpcCloseMemHandle(peer_base[b][r]);
  if (flag) cudaFree(flag);
  if (inv_flag) cudaFree(inv_flag);
  if (gsum) cudaFree(gsum);
  if (xbar_ref) cudaFree(xbar_ref);
  if (rbuf) cudaFree(rbuf);
  for (auto& kv : range_ev)
    if (kv.second) cudaEventDestroy(kv.second);
  if (ev_user) cudaEventDestroy(ev_user);
  if (ev_begin) cudaEventDestroy(ev_begin);
  for (auto e : ev_slot_free)
    if (e) cudaEventDestroy(e);
  for (auto e : ev_recv) cudaEventDestroy(e);
  for (auto& pr : tev) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  for (auto& gr : graphs)
    if (gr.exec) cudaGraphExecDestroy(gr.exec);
  if (comp) cudaStreamDestroy(comp);
  if (comm) cudaStreamDestroy(comm);
  for (auto st : pull) cudaStreamDestroy(st);
  for (auto ev : pull_ev) cudaEventDestroy(ev);
}

void dg_engine::enqueue_fused(const dg::RoundPlan& p, size_t off, size_t len, int slot_set,
                              const dg::DevScalars& s, bool fold, long t, const float* const* slot_override,
                              float* const* xpub_out) {
  float *x[dg::kMaxLocal], *xo[dg::kMaxLocal], *m[dg::kMaxLocal], *v[dg::kMaxLocal], *b[dg::kMaxLocal];
  const float* g[dg::kMaxLocal];
  for (int i = 0; i < NL; ++i) {
    x[i] = buf(DG_BUF_X, i);
    xo[i] = p.pingpong ? x_other(i) : x[i];
    g[i] = buf(DG_BUF_G, i);
    m[i] = buf(DG_BUF_M, i);
    v[i] = buf(DG_BUF_V, i);
    b[i] = algo == DG_ALGO_ACCUM ? buf(DG_BUF_ACC, i) : nullptr;
  }
  const float* slot_ptr[dg::kMaxRemote];
  for (int r = 0; r < int(p.recv_node.size()); ++r)
    slot_ptr[r] = slot_override                  ? slot_override[r]
                  : transport == DG_TRANSPORT_P2P ? peer_x(p.recv_node[r]) + off
                                                  : slots + (size_t(slot_set) * max_recv + r) * chunk;
  const dg::Buffers bf{slot_ptr, x, xo, g, m, v, algo == DG_ALGO_ACCUM ? b : nullptr, xpub_out};
  const bool st_k = p.xshare;
  const bool tma = !st_k && dg::use_tma(p) && p.n_local <= dg::kSlots;  // TmaArgs holds <= 16 member rows
  dg::LaunchFn fn = nullptr;
  const dg::GroupPlan* tp = nullptr;
  if (st_k) {
    const size_t ri = size_t(&p - plans.data());
    if (ri >= gplans.size() || !gplans[ri].ok) throw dg::Error(DG_INVARIANT, "xshare: plan not owned by the engine");
    tp = &gplans[ri];
  }
  // legacy kernels take <= kSlots members per launch (FusedArgs): rounds with
  // more components than that (> 16 resident nodes) run in batches
  std::vector<dg::RoundPlan> batches;
  if (!st_k && !tma) {
    const size_t cmax = size_t(dg::kSlots / std::max(1, p.comp_size));
    if (p.comps.size() > cmax) {
      for (size_t c0 = 0; c0 < p.comps.size(); c0 += cmax) {
        batches.push_back(p);
        auto& q = batches.back();
        q.comps.assign(p.comps.begin() + long(c0), p.comps.begin() + long(std::min(p.comps.size(), c0 + cmax)));
      }
    } else {
      dg::fill_args(argbuf, p, bf, off, len, s, int(t), flag);
      fn = dg::pick(p.comp_size, dg::launch_ns(p), algo, fold);
    }
  }
  // algorithmic LOCAL HBM bytes of this launch (remote buckets: recv-slot reads
  // for NCCL; for P2P they come over NVLink and are counted in `received`)
  const double per = algo == DG_ALGO_DADAM ? 28.0 : (fold ? 36.0 : 28.0);
  const bool pushed = push || p2p_push;  // x^(t) copies stored into peers' slots, remote rows local
  const double remote_hbm = ((transport == DG_TRANSPORT_P2P && !slot_override) || (xpub_out && !pushed))
                                ? 0.0
                                : 4.0 * double(p.recv_node.size());
  // (+4 B per param for the in-place P2P publish copy of x^(t); pushed copies land in peer HBM)
  const double bytes = double(len) * ((per + (xpub_out && !pushed ? 4.0 : 0.0)) * p.n_local + remote_hbm);
  // NVLink bytes the launch reads in-kernel (P2P exchange rounds, in-place P2P ranges)
  const double nvl = ((transport == DG_TRANSPORT_P2P && !slot_override) || xpub_out)
                         ? 4.0 * double(len) * double(p.recv_node.size())
                         : 0.0;
#if DG_XS_IDX32
  const size_t pieces = (len + (size_t(1) << 30) - 1) >> 30;  // launch_groups splits at 2^30 elements
#else
  const size_t pieces = 1;
#endif
  const int nk = st_k ? int(pieces) * ((int(tp->groups.size()) + dg::kShGroups - 1) / dg::kShGroups)
                      : std::max<int>(1, int(batches.size()));
  timed(bytes, nvl, [&] {
    if (st_k) {
      launch_groups(*tp, x, xo, g, m, v, b, slot_ptr, off, len, s, fold, t, sms_for(p), xpub_out);
    } else if (tma) {
      dg::launch_tma(p, bf, algo, fold, off, len, s, int(t), flag, comp);
    } else if (batches.empty()) {
      fn(argbuf.data(), (long long)(len / 4), int(p.comps.size()), sms_for(p), comp);
    } else {
      for (const auto& q : batches) {  // kernel parameters are copied at launch: argbuf is reusable
        dg::fill_args(argbuf, q, bf, off, len, s, int(t), flag);
        dg::pick(q.comp_size, dg::launch_ns(q), algo, fold)(argbuf.data(), (long long)(len / 4),
                                                             int(q.comps.size()), sms_for(p), comp);
      }
    }
  }, nk);
}

// One launch per (up to) kShGroups groups of the round; pointers at offset off.
void dg_engine::launch_groups(const dg::GroupPlan& tp, float* const* x, float* const* xo,
                                   const float* const* g, float* const* m, float* const* v, float* const* b,
                                   const float* const* slot_ptr, size_t off, size_t len,
                                   const dg::DevScalars& s, bool fold, long t, int sms, float* const* xp) {
  const int ng = int(tp.groups.size());
#if DG_XS_IDX32
  const size_t piece = size_t(1) << 30;  // the kernel indexes columns in 32 bits
#else
  const size_t piece = len;
#endif
  const size_t len_all = len, off_all = off;
  for (size_t o2 = 0; o2 < len_all; o2 += piece) {
  off = off_all + o2;
  len = std::min(piece, len_all - o2);
  for (int g0 = 0; g0 < ng; g0 += dg::kShGroups) {
    auto& a = sargs;
    std::memset(&a, 0, sizeof(a));
    const int cnt = std::min(dg::kShGroups, ng - g0);
    int warps = 1;
    for (int k = 0; k < cnt; ++k) {
      const auto& G = tp.groups[size_t(g0 + k)];
      auto& d = a.grp[k];
      d.nl = int(G.members.size());
      d.nx = int(G.srcs.size());
      warps = std::max(warps, std::max(d.nl, d.nx));  // a warp per member and per source row
      for (int j = 0; j < d.nx; ++j) {
        const int c = G.srcs[size_t(j)];
        d.row[j] = c >= 0 ? x[c] + off : slot_ptr[-c - 1] + o2;
        if (c >= 0 || (transport != DG_TRANSPORT_P2P && !xp)) d.local_rows |= 1u << j;
        d.wrow[j] = 0.0;
        for (int q = 0; q < d.nl; ++q)
          if (G.w[size_t(q)][size_t(j)] != 0.0) d.wrow[j] = G.w[size_t(q)][size_t(j)];
      }
      for (int q = 0; q < d.nl; ++q) {
        const int li = G.members[size_t(q)];
        d.xo[q] = xo[li] + off;
        for (int k = 0; k < dg::kPushMax; ++k) {
          float* dst = xp ? xp[li * dg::kPushMax + k] : nullptr;
          d.xp[q][k] = dst ? dst + off : nullptr;
        }
        d.g[q] = g[li] + off;
        d.m[q] = m[li] + off;
        d.v[q] = v[li] + off;
        d.b[q] = algo == DG_ALGO_ACCUM ? b[li] + off : nullptr;
        int k = 0;
        for (int j = 0; j < d.nx; ++j) {
          const double wq = G.w[size_t(q)][size_t(j)];
          if (wq == 0.0) continue;
          d.src[q][k] = (unsigned char)j;
          d.w[q][k] = wq;
          ++k;
        }
        d.deg[q] = k;
        for (; k < dg::kShDeg; ++k) {
          d.src[q][k] = (unsigned char)dg::kShRows;
          d.w[q][k] = 0.0;
        }
      }
    }
    a.s = s;
    a.n = (long long)len;
    a.t = int(t);
    a.prefetch = dg::xshare_prefetch();
    a.contiguous = dg::env_int("DG_XS_CONTIG", 0) != 0;
    a.div_flag = flag;
    bool has_xp = false;
    for (int k = 0; k < cnt; ++k)
      for (int q = 0; q < a.grp[k].nl; ++q)
        for (int j = 0; j < dg::kPushMax; ++j) has_xp |= a.grp[k].xp[q][j] != nullptr;
    dg::launch_xshare(a, cnt, warps, tp.max_deg, tp.colw, algo, fold, sms, comp, has_xp);
  }
  }
}

template <class F>
void dg_engine::timed(double bytes, double nvl_bytes, F&& launch, int kernels) {
  if (capturing) {  // recorded into a graph: no per-launch events, bytes kept for the replays
    launch();
    dg::cuda_check(cudaGetLastError(), "kernel launch (capture)");
    cap_launches += kernels;
    cap_hbm += bytes;
    cap_remote += nvl_bytes;
    launches += kernels;
    hbm += bytes;
    return;
  }
  if (timing) {
    if (tev_used == tev.size()) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      tev.push_back({a, b});
      tev_bytes.push_back(0);
      tev_remote.push_back(0);
      tev_n.push_back(1);
    }
    CU(cudaEventRecord(tev[tev_used].first, comp));
  }
  launch();
  dg::cuda_check(cudaGetLastError(), "kernel launch");
  if (timing) {
    CU(cudaEventRecord(tev[tev_used].second, comp));
    tev_remote[tev_used] = nvl_bytes;
    tev_n[tev_used] = kernels;
    tev_bytes[tev_used++] = bytes;
  }
  launches += kernels;
  hbm += bytes;
}

void dg_engine::step_allreduce(long t, const dg::DevScalars& s) {
  dg::NodePtrs g{};
  dg::NodeMutPtrs x{}, m{}, v{};
  for (int i = 0; i < NL; ++i) {
    g.p[i] = buf(DG_BUF_G, i);
    x.p[i] = buf(DG_BUF_X, i);
    m.p[i] = buf(DG_BUF_M, i);
    v.p[i] = buf(DG_BUF_V, i);
  }
  const unsigned grid = dg::grid_for((long long)d, 8);
  // column sums of the resident gradients: read NL x 4 B, write 8 B per element
  timed(double(d) * (4.0 * NL + 8.0), 0.0, [&] {
    dg::column_sum<<<grid, 256, 0, comp>>>(gsum, g, NL, (long long)d);
  });
  if (G > 1) NC(ncclAllReduce(gsum, gsum, d, ncclDouble, ncclSum, nccl, comp));  // the All-Reduce
  // update: read gsum 8 B + x, m, v; write x, m, v
  timed(double(d) * (24.0 * NL + 8.0), 0.0, [&] {
    dg::allreduce_adam<<<grid, 256, 0, comp>>>(x, m, v, NL, gsum, 1.0 / double(N), (long long)d, s, int(t), flag,
                                               inv_flag);
  });
}

void dg_engine::harvest_timing() {
  for (size_t k = 0; k < tev_used; ++k) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, tev[k].first, tev[k].second));
    kernel_ms += ms;
    timed_bytes += tev_bytes[k];
    timed_launches += tev_n[k];
    if (tev_remote[k] > 0) {
      remote_ms += ms;
      remote_bytes += tev_remote[k];
    }
  }
  tev_used = 0;
}

void dg_engine::post_range_exchange(const dg::RoundPlan& q, size_t off, size_t len) {
  NC(ncclGroupStart());
  for (size_t k = 0; k < q.send_node.size(); ++k)
    NC(ncclSend(buf(DG_BUF_X, q.send_node[k] - first) + off, len, ncclFloat, q.send_peer[k], nccl, comm));
  for (size_t r = 0; r < q.recv_node.size(); ++r)
    NC(ncclRecv(rbuf + r * d_pad + off, len, ncclFloat, q.recv_peer[r], nccl, comm));
  NC(ncclGroupEnd());
  cudaEvent_t& ev = range_ev[off];
  if (!ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CU(cudaEventRecord(ev, comm));
  sent += 4.0 * double(len) * double(q.send_node.size());
  received += 4.0 * double(len) * double(q.recv_node.size());
}

void dg_engine::signal_range(int slot, unsigned long long value) {
  // every peer learns "this rank finished iteration value - 1 on the range"
  if (signal_kernel) {
    dg::SignalArgs a{};
    for (int r = 0; r < G; ++r)
      if (r != rank) a.dst[a.n++] = peer_sig[r] + size_t(slot) * G + rank;
    a.value = value;
    dg::signal_peers<<<1, 32, 0, comp>>>(a);
    CU(cudaGetLastError());
    return;
  }
  for (int r = 0; r < G; ++r)
    if (r != rank)
      dg::cu_check(dg::memops().write64(reinterpret_cast<CUstream>(comp),
                                        reinterpret_cast<CUdeviceptr>(peer_sig[r] + size_t(slot) * G + rank), value,
                                        CU_STREAM_WRITE_VALUE_DEFAULT),
                   "cuStreamWriteValue64");
}

// In-place P2P range update (see the inplace_p2p fields): no copies, no NCCL;
// the peers' x^(t-1) of the range is read in-kernel over NVLink from their
// publish buffers.
void dg_engine::step_range_p2p(long t, size_t off, size_t len) {
  bool fold = false;
  const dg::DevScalars s = dg::scalars(&adam, algo, t, T, &fold);
  CU(cudaSetDevice(device));
  auto it = range_slot.find(off);
  if (it == range_slot.end()) {
    if (int(range_slot.size()) >= kMaxRanges) dg::config_error("step_range: more than 4096 distinct ranges");
    it = range_slot.emplace(off, int(range_slot.size())).first;
  }
  const int slot = it->second;
  ++steps;
  const long last = range_last.count(off) ? range_last[off] : -1;
  const size_t ri = size_t((t - 1) % P), ni = size_t(t % P);
  if (last != t - 1) {  // first step of this range (or a restart): publish x^(t-1)
    for (int i = 0; i < NL; ++i) {
      if (push) {  // into the round-t readers' receive slots (peer copies)
        const auto [q, sl] = push_dst[ri][size_t(i)];
        if (q >= 0)
          CU(cudaMemcpyAsync(peer_base[(t - 1) & 1][q] + size_t(sl) * d_pad + off, buf(DG_BUF_X, i) + off,
                             len * sizeof(float), cudaMemcpyDeviceToDevice, comp));
      } else {
        CU(cudaMemcpyAsync(xpub[(t - 1) & 1] + size_t(i) * d_pad + off, buf(DG_BUF_X, i) + off,
                           len * sizeof(float), cudaMemcpyDeviceToDevice, comp));
      }
    }
    signal_range(slot, (unsigned long long)t);
  }
  fault_delay(comp);
  // every peer finished iteration t-1 on this range
  for (int r = 0; r < G; ++r)
    if (r != rank)
      dg::cu_check(dg::memops().wait64(reinterpret_cast<CUstream>(comp),
                                       reinterpret_cast<CUdeviceptr>(sig + size_t(slot) * G + r),
                                       (cuuint64_t)t, CU_STREAM_WAIT_VALUE_GEQ),
                   "cuStreamWaitValue64");
  const dg::RoundPlan& p = plans[ri];
  std::vector<const float*> slot_ptr(std::max<size_t>(1, p.recv_node.size()));
  for (size_t r = 0; r < p.recv_node.size(); ++r) {
    if (push) {  // pushed here by the owner at t-1
      slot_ptr[r] = xpub[(t - 1) & 1] + r * d_pad + off;
    } else {
      const int node = p.recv_node[r], owner = dg::owner_of(node, N, G);
      slot_ptr[r] = peer_base[(t - 1) & 1][owner] + size_t(node - dg::first_node_of(owner, N, G)) * d_pad + off;
    }
  }
  // [node][kPushMax] bases (the launch adds the range offset; null = no copy)
  float* pub[dg::kMaxLocal * dg::kPushMax] = {};
  for (int i = 0; i < NL; ++i) {
    if (push) {
      const auto [q, sl] = push_dst[ni][size_t(i)];
      pub[i * dg::kPushMax] = q >= 0 ? peer_base[t & 1][q] + size_t(sl) * d_pad : nullptr;
    } else {
      pub[i * dg::kPushMax] = xpub[t & 1] + size_t(i) * d_pad;
    }
  }
  sent += 4.0 * double(len) * double(p.send_node.size());
  received += 4.0 * double(len) * double(p.recv_node.size());
  if (!diag_skip_kernel) enqueue_fused(p, off, len, 0, s, fold, t, slot_ptr.data(), pub);
  if (push)  // consumed receive slots: the owners refill this parity only after our t+1 signal
    for (size_t r = 0; r < p.recv_node.size(); ++r) poison_range(xpub[(t - 1) & 1] + r * d_pad + off, len, comp);
  signal_range(slot, (unsigned long long)(t + 1));
  range_last[off] = t;
}

// U_k of the paper: wait for this range's round-t exchange (posted at t-1 or
// now), update the range, post its round-(t+1) exchange.
void dg_engine::step_range(long t, size_t off, size_t len) {
  if (!in_place) dg::config_error("step_range: engine was not created with DG_ENGINE_IN_PLACE");
  if (algo == DG_ALGO_ALLREDUCE) dg::config_error("step_range: not available for All-Reduce Adam");
  if (off % dg::kAlign || off >= d || len == 0 || len > d - off)
    dg::config_error("step_range: range must start at a multiple of 64 and lie inside [0, d)");
  if (inplace_p2p) return step_range_p2p(t, off, len);
  bool fold = false;
  const dg::DevScalars s = dg::scalars(&adam, algo, t, T, &fold);
  CU(cudaSetDevice(device));
  const dg::RoundPlan& p = plans[size_t((t - 1) % P)];
  const bool comm_now = G > 1 && !(p.send_node.empty() && p.recv_node.empty());
  if (comm_now && !rbuf) {
    CU(cudaMalloc(&rbuf, sizeof(float) * std::max(1, max_recv) * d_pad));
    nccl_register(rbuf, sizeof(float) * std::max(1, max_recv) * d_pad);
  }
  std::vector<const float*> slot_ptr(std::max<size_t>(1, p.recv_node.size()));
  fault_delay(t & 1 ? comp : comm);
  if (comm_now) {
    auto it = range_posted.find(off);
    if (it == range_posted.end() || it->second != t) {  // not pre-posted: exchange x^(t-1) now
      CU(cudaEventRecord(ev_begin, comp));
      CU(cudaStreamWaitEvent(comm, ev_begin, 0));
      post_range_exchange(p, off, len);
    }
    CU(cudaStreamWaitEvent(comp, range_ev[off], 0));
    for (size_t r = 0; r < p.recv_node.size(); ++r) slot_ptr[r] = rbuf + r * d_pad + off;
  }
  if (!diag_skip_kernel) enqueue_fused(p, off, len, 0, s, fold, t, comm_now ? slot_ptr.data() : nullptr);
  if (comm_now)  // the range's recv buffers are consumed; the next exchange into them waits on comp
    for (size_t r = 0; r < p.recv_node.size(); ++r) poison_range(rbuf + r * d_pad + off, len, comp);
  range_posted.erase(off);
  const dg::RoundPlan& q = plans[size_t(t % P)];
  if (G > 1 && !(q.send_node.empty() && q.recv_node.empty())) {
    if (!rbuf) {
      CU(cudaMalloc(&rbuf, sizeof(float) * std::max(1, max_recv) * d_pad));
      nccl_register(rbuf, sizeof(float) * std::max(1, max_recv) * d_pad);
    }
    CU(cudaEventRecord(ev_begin, comp));  // x^(t)[off, off+len) final
    CU(cudaStreamWaitEvent(comm, ev_begin, 0));
    post_range_exchange(q, off, len);     // C_k for iteration t+1, overlaps the caller's next work
    range_posted[off] = t + 1;
  }
}

// Peer copies of every resident node's current x (= x^(t-1)) into the slots
// of its round-t remote readers (parity (t-1)&1), before step t's barrier.
void dg_engine::push_seed(long t) {
  const size_t ri = size_t((t - 1) % P);
  for (int i = 0; i < NL; ++i)
    for (int k = 0; k < dg::kPushMax; ++k) {
      const auto [q, sl] = pdst[ri][size_t(i)][size_t(k)];
      if (q < 0) continue;
      CU(cudaMemcpyAsync(peer_base[(t - 1) & 1][q] + size_t(sl) * d_pad, buf(DG_BUF_X, i), d * sizeof(float),
                         cudaMemcpyDeviceToDevice, comp));
    }
  seeded_for = t;
}

void dg_engine::step(long t) {
  if (!range_posted.empty())
    dg::config_error("step: bucketed exchanges are in flight (use dg_engine_step_range consistently)");
  bool fold = false;
  const dg::DevScalars s = dg::scalars(&adam, algo, t, T, &fold);
  CU(cudaSetDevice(device));
  const size_t ri = size_t((t - 1) % P);
  const dg::RoundPlan& p = plans[ri];
  if (inplace_p2p) return step_range_p2p(t, 0, d);
  ++steps;
  if (algo == DG_ALGO_ALLREDUCE) return step_allreduce(t, s);
  if (transport == DG_TRANSPORT_P2P && G > 1 && p2p_push) {
    if (seeded_for != t) push_seed(t);  // x^(t-1) into the round-t readers' slots
    fault_delay(comp);
    // Barrier (every peer finished step t-1) before a step that reads its
    // receive slots (round t remote: the peers' pushes of x^(t-1) have landed)
    // or pushes (round t+1 remote: no peer still reads the parity t&1 slots
    // this kernel refills -- their last reader ran before this barrier).
    const size_t ni = size_t(t % P);
    if (round_remote[ri] || round_remote[ni]) {
      NC(ncclAllReduce(bar_buf, bar_buf, 1, ncclFloat, ncclSum, nccl, comp));
      ++barriers;
    }
    std::vector<const float*> slot_ptr(std::max<size_t>(1, p.recv_node.size()));
    for (size_t r = 0; r < p.recv_node.size(); ++r) slot_ptr[r] = pbuf[(t - 1) & 1] + r * d_pad;
    float* dst[dg::kMaxLocal * dg::kPushMax] = {};
    size_t npush = 0;
    for (int i = 0; i < NL; ++i)
      for (int k = 0; k < dg::kPushMax; ++k) {
        const auto [q, sl] = pdst[ni][size_t(i)][size_t(k)];
        if (q < 0) continue;
        dst[i * dg::kPushMax + k] = peer_base[t & 1][q] + size_t(sl) * d_pad;
        ++npush;
      }
    sent += 4.0 * double(d) * double(npush);
    received += 4.0 * double(d) * double(p.recv_node.size());
    enqueue_fused(p, 0, d, 0, s, fold, t, slot_ptr.data(), npush ? dst : nullptr);
    for (size_t r = 0; r < p.recv_node.size(); ++r) poison_range(pbuf[(t - 1) & 1] + r * d_pad, d, comp);
    if (p.pingpong) xcur ^= 1;
    seeded_for = t + 1;
    return;
  }
  if (transport == DG_TRANSPORT_P2P && G > 1) {
    // Cross-GPU step barrier, stream-ordered on the compute stream, before any
    // step that reads peers' x^(t-1) (their step t-1 must be complete) and
    // before the step after one (peers must have finished reading the buffer
    // this step may overwrite).  Every rank takes the same decision.
    const size_t prev = size_t((t - 2 + P) % P);
    if (!(t & 1)) fault_delay(comp);  // late writer: peers wait for this rank at the barrier
    if (round_remote[ri] || (t > 1 && round_remote[prev])) {
      NC(ncclAllReduce(bar_buf, bar_buf, 1, ncclFloat, ncclSum, nccl, comp));
      ++barriers;
    }
    if (t & 1) fault_delay(comp);  // late reader: this rank reads peers' x^(t-1) after they moved on
    // no peer reads the stale x buffer past the barrier (it held x^(t-2) or older)
    if (x_alt) poison_range(xcur ? arena[DG_BUF_X] : x_alt, NL * d_pad, comp);
    sent += 4.0 * double(d) * double(p.send_node.size());
    received += 4.0 * double(d) * double(p.recv_node.size());
    if (!p.pull) {
      enqueue_fused(p, 0, d, 0, s, fold, t);  // remote sources read over NVLink inside the kernel
    } else {
      // copy-engine pulls of each distinct remote bucket, chunk by chunk into
      // double-buffered local slots, overlapped with the kernel on the previous chunk
      CU(cudaEventRecord(ev_begin, comp));  // after the barrier: peers' x^(t-1) final
      const int np = std::min<int>(int(pull.size()), int(p.recv_node.size()));
      for (int q = 0; q < np; ++q) CU(cudaStreamWaitEvent(pull[q], ev_begin, 0));
      const float* slot_ptr[dg::kMaxRemote];
      for (size_t k = 0; k < n_chunks; ++k) {
        const size_t off = k * chunk, len = std::min(chunk, d - off);
        const int set = int(k & 1);
        for (int q = 0; q < np; ++q)
          if (k >= 2) CU(cudaStreamWaitEvent(pull[q], ev_slot_free[set], 0));
        // one copy stream per remote bucket (round robin): concurrent copy engines
        for (size_t r = 0; r < p.recv_node.size(); ++r) {
          float* dst = slots + (size_t(set) * max_recv + r) * chunk;
          CU(cudaMemcpyAsync(dst, peer_x(p.recv_node[r]) + off, len * sizeof(float), cudaMemcpyDeviceToDevice,
                             pull[r % np]));
          slot_ptr[r] = dst;
        }
        for (int q = 0; q < np; ++q) {
          CU(cudaEventRecord(pull_ev[q], pull[q]));
          CU(cudaStreamWaitEvent(comp, pull_ev[q], 0));
        }
        enqueue_fused(p, off, len, set, s, fold, t, slot_ptr);
        poison_range(slots + size_t(set) * max_recv * chunk, size_t(max_recv) * chunk, comp);
        CU(cudaEventRecord(ev_slot_free[set], comp));
      }
    }
    if (p.pingpong) xcur ^= 1;
    return;
  }
  fault_delay(t & 1 ? comp : comm);
  // stale x buffer (x^(t-2) or older): its last readers -- step t-1's kernels and
  // the sends they waited for -- are all ordered before this point on comp
  if (x_alt) poison_range(xcur ? arena[DG_BUF_X] : x_alt, NL * d_pad, comp);
  if (p.send_node.empty() && p.recv_node.empty()) {  // intra-GPU round: one launch
    enqueue_fused(p, 0, d, 0, s, fold, t);
    if (p.pingpong) xcur ^= 1;
    return;
  }
  // comm stream starts after everything already queued on the compute stream
  // (x^(t-1) final, previous step's slots consumed)
  CU(cudaEventRecord(ev_begin, comp));
  CU(cudaStreamWaitEvent(comm, ev_begin, 0));
  for (size_t k = 0; k < n_chunks; ++k) {
    const size_t off = k * chunk, len = std::min(chunk, d - off);
    const int set = int(k & 1);
    if (k >= 2) CU(cudaStreamWaitEvent(comm, ev_slot_free[set], 0));  // chunk k-2 consumed slot set
    NC(ncclGroupStart());
    for (size_t q = 0; q < p.send_node.size(); ++q)
      NC(ncclSend(buf(DG_BUF_X, p.send_node[q] - first) + off, len, ncclFloat, p.send_peer[q], nccl,
                  comm));
    for (size_t r = 0; r < p.recv_node.size(); ++r)
      NC(ncclRecv(slots + (size_t(set) * max_recv + r) * chunk, len, ncclFloat, p.recv_peer[r], nccl,
                  comm));
    NC(ncclGroupEnd());
    CU(cudaEventRecord(ev_recv[k], comm));
    sent += 4.0 * double(len) * double(p.send_node.size());
    received += 4.0 * double(len) * double(p.recv_node.size());
    // fused kernel on chunk k once its neighbour buckets have landed (and the
    // sends of the in-place x chunk have drained)
    CU(cudaStreamWaitEvent(comp, ev_recv[k], 0));
    if (!diag_skip_kernel) enqueue_fused(p, off, len, set, s, fold, t);
    poison_range(slots + size_t(set) * max_recv * chunk, size_t(max_recv) * chunk, comp);
    CU(cudaEventRecord(ev_slot_free[set], comp));
  }
  if (p.pingpong) xcur ^= 1;
}

dg_engine::GraphRec& dg_engine::capture(long t0, long t1) {
  for (auto& gr : graphs)
    if (gr.t0 == t0 && gr.t1 == t1 && gr.x0 == xcur) return gr;
  if (graphs.size() >= 8) {  // small cache: oldest out
    CU(cudaGraphExecDestroy(graphs.front().exec));
    graphs.erase(graphs.begin());
  }
  GraphRec gr;
  gr.t0 = t0;
  gr.t1 = t1;
  gr.x0 = xcur;
  // host-side bookkeeping that step() advances while capturing; restored
  // after, and re-applied on every replay
  const long l0 = launches, s0 = steps, b0 = barriers;
  const long seed0 = seeded_for;
  seeded_for = t0;  // P2P push: the seed copies stay outside the graph (run_steps issues them)
  const double h0 = hbm, se0 = sent, r0 = received;
  cap_hbm = cap_remote = 0;
  cap_launches = 0;
  cudaGraph_t g = nullptr;
  CU(cudaStreamBeginCapture(comp, cudaStreamCaptureModeThreadLocal));
  capturing = true;
  try {
    for (long t = t0; t <= t1; ++t) step(t);
  } catch (...) {
    capturing = false;
    cudaStreamEndCapture(comp, &g);
    if (g) cudaGraphDestroy(g);
    xcur = gr.x0;
    seeded_for = seed0;
    launches = l0, steps = s0, barriers = b0, hbm = h0, sent = se0, received = r0;
    throw;
  }
  capturing = false;
  CU(cudaStreamEndCapture(comp, &g));
  gr.x1 = xcur;
  xcur = gr.x0;
  seeded_for = seed0;
  gr.launches = launches - l0, gr.steps = steps - s0, gr.barriers = barriers - b0;
  gr.hbm = hbm - h0, gr.sent = sent - se0, gr.received = received - r0, gr.remote = cap_remote;
  launches = l0, steps = s0, barriers = b0, hbm = h0, sent = se0, received = r0;
  const cudaError_t ie = cudaGraphInstantiate(&gr.exec, g, 0);
  cudaGraphDestroy(g);
  CU(ie);
  graphs.push_back(gr);
  return graphs.back();
}

void dg_engine::run_steps(long t0, long t1, int flags) {
  if (t0 < 1 || t1 < t0) dg::config_error("run_steps: need 1 <= t_first <= t_last");
  if (!range_posted.empty())
    dg::config_error("run_steps: bucketed exchanges are in flight (use dg_engine_step_range consistently)");
  CU(cudaSetDevice(device));
  if (!(flags & DG_RUN_GRAPH)) {
    for (long t = t0; t <= t1; ++t) step(t);
    return;
  }
  GraphRec& gr = capture(t0, t1);
  if (flags & DG_RUN_CAPTURE_ONLY) return;
  if (p2p_push && seeded_for != t0) push_seed(t0);
  if (timing) {
    if (tev_used == tev.size()) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      tev.push_back({a, b});
      tev_bytes.push_back(0);
      tev_remote.push_back(0);
      tev_n.push_back(1);
    }
    CU(cudaEventRecord(tev[tev_used].first, comp));
  }
  CU(cudaGraphLaunch(gr.exec, comp));
  if (timing) {
    CU(cudaEventRecord(tev[tev_used].second, comp));
    tev_bytes[tev_used] = gr.hbm;
    tev_remote[tev_used] = gr.remote;
    tev_n[tev_used++] = gr.launches;
  }
  xcur = gr.x1;
  if (p2p_push) seeded_for = t1 + 1;
  launches += gr.launches, steps += gr.steps, barriers += gr.barriers;
  hbm += gr.hbm, sent += gr.sent, received += gr.received;
}

// ===================================================================== C ABI
using dg::guarded;

extern "C" {

int dg_nccl_unique_id(void* out128) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    if (!out128) dg::config_error("nccl_unique_id: null output");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
  });
}

int dg_engine_create(const dg_engine_config* c, dg_engine** out) {
  return guarded([&] {
    if (!c || !out) dg::config_error("engine_create: null argument");
    *out = nullptr;
    if (!c->schedule || c->schedule->rounds.empty()) dg::config_error("engine_create: empty schedule");
    if (c->d < 1) dg::config_error("engine_create: d must be >= 1");
    if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size)
      dg::config_error("engine_create: bad rank / world_size");
    if (c->world_size > 1 && !c->nccl_id) dg::config_error("engine_create: nccl_id required");
    bool fold;
    dg::scalars(&c->adam, c->algo, 1, c->algo == DG_ALGO_ACCUM ? c->total_steps : 1, &fold);
    auto e = std::make_unique<dg_engine>();
    e->device = c->device;
    e->N = c->schedule->n;
    e->G = c->world_size;
    e->rank = c->rank;
    e->algo = c->algo;
    e->adam = c->adam;
    e->T = c->total_steps;
    e->d = c->d;
    e->d_pad = (c->d + dg::kAlign - 1) / dg::kAlign * dg::kAlign;
    size_t ch = c->chunk ? c->chunk : dg::kDefaultChunk;
    ch = (std::min(ch, c->d) + dg::kAlign - 1) / dg::kAlign * dg::kAlign;
    e->chunk = ch;
    e->n_chunks = (c->d + ch - 1) / ch;
    e->P = int(c->schedule->rounds.size());
    e->first = dg::first_node_of(c->rank, e->N, e->G);
    for (int r = 1; r <= e->P; ++r) {
      e->plans.push_back(dg::build_round_plan(*c->schedule, e->G, e->rank, r));
      e->max_recv = std::max(e->max_recv, int(e->plans.back().recv_node.size()));
    }
    e->NL = e->plans[0].n_local;
    e->in_place = (c->flags & DG_ENGINE_IN_PLACE) != 0;
    e->transport = c->transport == DG_TRANSPORT_NCCL ? DG_TRANSPORT_NCCL : DG_TRANSPORT_P2P;
    bool auto_transport = c->transport == DG_TRANSPORT_AUTO;
    if (const char* tr = std::getenv("DG_TRANSPORT")) {
      e->transport = std::string(tr) == "nccl" ? DG_TRANSPORT_NCCL : DG_TRANSPORT_P2P;
      auto_transport = false;
    }
    bool p2p = e->transport == DG_TRANSPORT_P2P && e->G > 1 && c->algo != DG_ALGO_ALLREDUCE;
    // x double-buffered ("ping-pong") rounds: mixing components of >=
    // DG_PINGPONG_MIN_NC members (default 4) anywhere, and with the P2P transport
    // every round in which any rank reads a remote bucket.  Decided from the
    // global schedule so that every rank flips its x buffer identically.
    const char* ppenv = std::getenv("DG_PINGPONG_MIN_NC");
    const int pp_min = e->in_place ? 0 : (ppenv ? std::atoi(ppenv) : 4);
    bool any_pp = false;
    e->round_remote.assign(e->P, 0);
    // every rank's plan of every round: the x-sharing kernel is used only if it
    // fits every round on every rank, so all ranks take identical x-buffer decisions
    std::vector<std::vector<dg::RoundPlan>> all(e->P);
    e->xshare = dg::xshare_enabled();
    for (int r = 0; r < e->P; ++r)
      for (int g = 0; g < e->G; ++g) {
        all[r].push_back(g == e->rank ? e->plans[r] : dg::build_round_plan(*c->schedule, e->G, g, r + 1));
        e->xshare = e->xshare && dg::build_group_plan(all[r].back()).ok;
      }
    // P2P exchange rounds (remote x^(t-1) read in-kernel over NVLink) run the
    // legacy kernels unless DG_XSHARE_REMOTE=1: the x-sharing kernel loads
    // each row one column block ahead only, which does not cover NVLink
    // latency (config 3 at 2 GPUs: 19.9 ms vs 9.2 ms, measured)
    const bool xs_remote = dg::env_int("DG_XSHARE_REMOTE", 0) != 0;
    // Rounds whose mixing components are all pairs (one-peer topologies) with
    // buckets of <= 2^24 params or fewer than 8 resident nodes run the legacy pair kernel unless
    // DG_XSHARE_PAIRS=1: a pair's two rows are read by one thread anyway, and
    // without the per-column CTA barrier small buckets run faster (config 1,
    // 8 x 2^20: 44.3 vs 49.6 us per step), large ones do not (config 2 at
    // 125M: 0.921 vs 0.932).  In-place engines run pair rounds on the legacy
    // pair kernel at every size (it writes the P2P publish copy and hides
    // NVLink latency better), other rounds on the x-sharing kernel.
    const bool xs_pairs = dg::env_int("DG_XSHARE_PAIRS", 0) != 0;
    e->gplans.resize(size_t(e->P));
    // P2P push feasibility (every rank decides identically from the global plans):
    // <= kPushMax reader ranks per node and round, and every round runs a
    // kernel that stores the copies (x-sharing, or the plain legacy pair kernel)
    bool want_push = p2p && !e->in_place && dg::env_int("DG_P2P_PUSH", 0) != 0;
    if (want_push) {
      e->pdst.assign(size_t(e->P), std::vector<std::array<std::pair<int, int>, dg::kPushMax>>(size_t(e->NL)));
      for (auto& rr : e->pdst)
        for (auto& a : rr) a.fill({-1, -1});
      for (int r = 0; r < e->P && want_push; ++r) {
        bool pairs = true;
        for (int g = 0; g < e->G; ++g)
          for (const auto& cp : all[r][g].comps) pairs = pairs && cp.members.size() <= 2 && cp.srcs.size() <= 2;
        std::vector<int> readers(size_t(e->N), 0);  // remote reader ranks per node
        for (int g = 0; g < e->G && want_push; ++g) {  // every rank's kernel must store the copies
          const int nl_g = dg::first_node_of(g + 1, e->N, e->G) - dg::first_node_of(g, e->N, e->G);
          const bool small = e->d <= (size_t(1) << 24) || nl_g < 8;
          const bool xs = e->xshare && (!pairs || !small || xs_pairs);
          const auto& q = all[r][g];
          if (!xs && !(q.comp_size <= 2 && !dg::use_tma(q) &&
                       (q.comp_size == 2 || int(q.comps.size()) < dg::warps_min_nc())))
            want_push = false;
          for (size_t sl = 0; sl < q.recv_node.size(); ++sl) {
            const int node = q.recv_node[sl];
            if (++readers[size_t(node)] > dg::kPushMax) want_push = false;
            const int li = node - e->first;
            if (li < 0 || li >= e->NL) continue;
            auto& a = e->pdst[size_t(r)][size_t(li)];
            int k = 0;
            while (k < dg::kPushMax && a[size_t(k)].first >= 0) ++k;
            if (k < dg::kPushMax) a[size_t(k)] = {g, int(sl)};
          }
        }
      }
      // (identical on every rank: every input above is global)
    }
    e->p2p_push = want_push;
    for (int r = 0; r < e->P; ++r) {
      bool pp = false, pairs = true;
      for (int g = 0; g < e->G; ++g) {
        if (!all[r][g].recv_node.empty()) e->round_remote[r] = 1;
        for (const auto& cp : all[r][g].comps) pairs = pairs && cp.members.size() <= 2 && cp.srcs.size() <= 2;
      }
      // in place, pair rounds may also run the legacy pair kernel (it writes the
      // publish copy too) as long as the plain per-thread kernel is the one picked
      const bool plain_pairs = pairs && !xs_pairs && !dg::use_tma(e->plans[r]) &&
                               (e->plans[r].comp_size == 2 || int(e->plans[r].comps.size()) < dg::warps_min_nc());
      // launch/latency-bound buckets, or too few resident nodes to fill the
      // x-sharing CTAs (a group of one pair is a 2-warp CTA: config 2 at 4 GPUs,
      // 2 nodes per GPU, ran 2.02 ms/step vs 1.43 ms on the legacy kernel)
      const bool small = e->d <= (size_t(1) << 24) || e->NL < 8;
      const bool xs = e->xshare && (e->in_place ? !plain_pairs
                                                : ((!p2p || want_push || !e->round_remote[r] || xs_remote) &&
                                                   (!pairs || !small || xs_pairs)));
      e->plans[r].xshare = xs;
      for (int g = 0; g < e->G; ++g) {
        const auto& q = all[r][g];
        // the legacy kernels take components of <= 16 members (FusedArgs / TmaArgs)
        if (!xs && ((pp_min > 0 && q.comp_size >= pp_min) || q.oversize || q.comp_size > dg::kSlots)) pp = true;
      }
      // in place: peers read xpub; push: remote rows are local receive slots
      if (p2p && !e->in_place && !want_push && e->round_remote[r]) pp = true;
      if (pp && xs) {
        // x-sharing kernel: in place on this GPU; only peers' readers (P2P
        // exchange rounds) need x^(t) in the other buffer
        e->plans[r].pingpong = true;
        any_pp = true;
      } else if (pp) {
        // pair components in P2P exchange rounds keep their structure (each
        // remote source is loaded once per column, in registers) and only
        // redirect x^(t) to the other buffer; otherwise one gather per node
        // (4-8 nodes: one warp per node in a CTA, so remote lines are shared
        // through L1 -- config 3 at 2 GPUs: 9.2 ms vs 10.8 ms kept whole)
        const char* kenv = std::getenv("DG_P2P_KEEP_NC");  // largest component kept whole (default 2)
        const int keep_nc = kenv ? std::atoi(kenv) : 2;
        if (e->in_place) dg::config_error("engine: a mixing component has > 32 sources; in-place mode cannot double-buffer x");
        const bool keep = p2p && e->round_remote[r] && e->plans[r].comp_size <= keep_nc && !e->plans[r].oversize;
        if (keep)
          e->plans[r].pingpong = true;
        else
          dg::make_pingpong(e->plans[r], e->first);
        any_pp = true;
      }
      // P2P pull decision: NVLink reads per column = remote sources summed over the
      // components (a component's thread loads each of its sources once; repeats
      // across member rows hit L1), vs the distinct remote buckets.  With one warp
      // per node (gossip_adam_warps) the CTA shares every remote line: distinct.
      auto& pr = e->plans[r];
      long remote_reads = 0;
      for (const auto& cp : pr.comps)
        for (size_t k = 0; k < cp.srcs.size(); ++k)
          if (cp.srcs[k] < 0) ++remote_reads;
      const int ncomp = int(pr.comps.size());
      if (pr.comp_size == 1 && ncomp >= dg::warps_min_nc() && ncomp <= 8) remote_reads = long(pr.recv_node.size());
      if (xs) {  // each group row is loaded once per column
        e->gplans[size_t(r)] = dg::build_group_plan(pr);
        remote_reads = 0;
        for (const auto& gr : e->gplans[size_t(r)].groups)
          for (int c : gr.srcs) remote_reads += c < 0;
      }
      const char* pv = std::getenv("DG_P2P_PULL");  // 0 never, 1 auto (default), 2 always
      const int pull_mode = pv ? std::atoi(pv) : 1;
      // in-kernel peer loads reach ~770 GB/s, copy-engine pulls ~420 GB/s (measured):
      // pull only when a remote bucket is read >= 1.75x on average
      pr.pull = p2p && !e->in_place && !want_push && !pr.recv_node.empty() &&
                (pull_mode == 2 || (pull_mode == 1 && 4 * remote_reads >= 7 * long(pr.recv_node.size())));
    }
    if (e->NL < 1) dg::config_error("engine_create: no resident nodes on this rank");
    if (p2p && e->in_place && (!e->xshare || !dg::memops().wait64 || !dg::memops().write64)) {
      // the publish copy of x^(t) is written by the x-sharing kernel only
      if (!auto_transport)
        dg::config_error("engine_create: in-place P2P needs the x-sharing kernel and stream memory operations");
      e->transport = DG_TRANSPORT_NCCL;
      p2p = false;
    }
    e->inplace_p2p = p2p && e->in_place;
    e->signal_kernel = dg::env_int("DG_SIGNAL_KERNEL", 0) != 0;
    if (e->inplace_p2p && dg::env_int("DG_INPLACE_PUSH", 1) != 0) {
      // reader rank and receive slot of every resident node, per round (from
      // every rank's plan); push only if each node has <= 1 remote reader rank
      bool ok = true;
      e->push_dst.assign(size_t(e->P), std::vector<std::pair<int, int>>(size_t(e->NL), {-1, -1}));
      for (int r = 0; r < e->P && ok; ++r)
        for (int g = 0; g < e->G && ok; ++g) {
          if (g == e->rank) continue;
          const auto& rn = all[r][g].recv_node;
          for (size_t sl = 0; sl < rn.size(); ++sl) {
            const int li = rn[sl] - e->first;
            if (li < 0 || li >= e->NL) continue;
            auto& dst = e->push_dst[size_t(r)][size_t(li)];
            if (dst.first >= 0) ok = false;
            dst = {g, int(sl)};
          }
        }
      e->push = ok;
    }
    CU(cudaSetDevice(c->device));
    e->sm_total = dg::sm_count(c->device);
    if (const char* rs = std::getenv("DG_RESERVE_SMS")) e->reserve_sms = std::max(0, std::atoi(rs));
    e->diag_skip_kernel = std::getenv("DG_DIAG_SKIP_KERNEL") != nullptr;
    if (dg::env_int("DG_FAULT_RANK", e->G > 1 ? 1 : 0) == e->rank)
      e->fault_ns = 1000LL * std::max(0, dg::env_int("DG_FAULT_DELAY_US", 0));
    e->poison = dg::env_int("DG_FAULT_POISON", 0) != 0;
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithFlags(&e->comp, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithPriority(&e->comm, cudaStreamNonBlocking, hi));  // comm first
    CU(cudaEventCreateWithFlags(&e->ev_begin, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&e->ev_user, cudaEventDisableTiming));
    for (auto& ev : e->ev_slot_free) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->ev_recv.resize(e->n_chunks);
    for (auto& ev : e->ev_recv) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const int kinds = c->algo == DG_ALGO_ACCUM ? 5 : 4;
    for (int k = 0; k < kinds; ++k) {
      CU(cudaMalloc(&e->arena[k], sizeof(float) * e->d_pad * e->NL));
      CU(cudaMemsetAsync(e->arena[k], 0, sizeof(float) * e->d_pad * e->NL, e->comp));
    }
    if ((any_pp || (p2p && !e->p2p_push)) && !e->in_place) {
      CU(cudaMalloc(&e->x_alt, sizeof(float) * e->d_pad * e->NL));
      CU(cudaMemsetAsync(e->x_alt, 0, sizeof(float) * e->d_pad * e->NL, e->comp));
    }
    if (e->p2p_push)
      for (auto& pb : e->pbuf) {
        CU(cudaMalloc(&pb, sizeof(float) * e->d_pad * size_t(std::max(1, e->max_recv))));
        CU(cudaMemsetAsync(pb, 0, sizeof(float) * e->d_pad * size_t(std::max(1, e->max_recv)), e->comp));
      }
    if (e->inplace_p2p) {
      // pull: publish copies [node]; push: receive slots [slot] (written by the peers)
      const size_t rows = e->push ? size_t(std::max(1, e->max_recv)) : size_t(e->NL);
      for (auto& pb : e->xpub) {
        CU(cudaMalloc(&pb, sizeof(float) * e->d_pad * rows));
        CU(cudaMemsetAsync(pb, 0, sizeof(float) * e->d_pad * rows, e->comp));
      }
      const size_t nsig = size_t(dg_engine::kMaxRanges) * e->G;
      CU(cudaMalloc(&e->sig, sizeof(unsigned long long) * nsig));
      CU(cudaMemsetAsync(e->sig, 0, sizeof(unsigned long long) * nsig, e->comp));
    }
    bool any_pull = false;
    for (const auto& pr : e->plans) any_pull |= pr.pull;
    if (any_pull) {
      const char* ps = std::getenv("DG_PULL_STREAMS");  // measured: 1 and 8 streams perform alike
      const int nps = std::max(1, std::min(e->max_recv, ps ? std::atoi(ps) : 2));
      e->pull.resize(nps);
      e->pull_ev.resize(nps);
      for (int q = 0; q < nps; ++q) {
        CU(cudaStreamCreateWithPriority(&e->pull[q], cudaStreamNonBlocking, hi));
        CU(cudaEventCreateWithFlags(&e->pull_ev[q], cudaEventDisableTiming));
      }
    }
    if (e->max_recv && (!p2p || any_pull))
      CU(cudaMalloc(&e->slots, sizeof(float) * 2 * e->max_recv * e->chunk));
    CU(cudaMalloc(&e->flag, sizeof(int)));
    CU(cudaMalloc(&e->inv_flag, sizeof(int)));
    const int none = INT_MAX;
    CU(cudaMemcpyAsync(e->flag, &none, sizeof(int), cudaMemcpyHostToDevice, e->comp));
    CU(cudaMemcpyAsync(e->inv_flag, &none, sizeof(int), cudaMemcpyHostToDevice, e->comp));
    if (c->algo == DG_ALGO_ALLREDUCE) CU(cudaMalloc(&e->gsum, sizeof(double) * e->d_pad));
    CU(cudaStreamSynchronize(e->comp));
    if (e->G > 1) {
      ncclUniqueId id;
      std::memcpy(&id, c->nccl_id, sizeof(id));
      NC(ncclCommInitRank(&e->nccl, e->G, id, e->rank));
    }
    for (int b = 0; b < 2; ++b) e->peer_base[b].assign(e->G, nullptr);
    // exported buffers: x and x_alt, or (in place) the two publish buffers + the flags
    float* exp0 = e->inplace_p2p ? e->xpub[0] : e->p2p_push ? e->pbuf[0] : e->arena[DG_BUF_X];
    float* exp1 = e->inplace_p2p ? e->xpub[1] : e->p2p_push ? e->pbuf[1] : e->x_alt;
    e->peer_base[0][e->rank] = exp0;
    e->peer_base[1][e->rank] = exp1;
    e->peer_sig.assign(e->G, nullptr);
    e->peer_sig[e->rank] = e->sig;
    if (p2p) {
      // Exchange CUDA IPC handles of both x buffers (one 128-byte record per
      // rank), open the peers', then AGREE on the outcome (all-reduce min of a
      // per-rank success flag) so every rank commits to the same transport.
      // Only CUDA (IPC) failures are tolerated locally; NCCL errors propagate.
      static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
      constexpr size_t kRec = 192;  // three handles per rank: exp0, exp1, flags (in place)
      std::vector<char> mine(kRec, 0), all(kRec * size_t(e->G));
      int ok = 1;
      std::string why;
      auto attempt = [&](auto&& f) {
        if (!ok) return;
        try {
          f();
        } catch (const dg::Error& err) {
          if (err.code != DG_CUDA_ERROR) throw;
          ok = 0;
          why = err.what();
          cudaGetLastError();
        }
      };
      attempt([&] {
        CU(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data()), exp0));
        CU(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data() + 64), exp1));
        if (e->sig) CU(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data() + 128), e->sig));
      });
      char* dbuf = nullptr;
      int* dok = nullptr;
      CU(cudaMalloc(&dbuf, all.size()));
      CU(cudaMalloc(&dok, sizeof(int)));
      CU(cudaMemcpy(dbuf + kRec * size_t(e->rank), mine.data(), kRec, cudaMemcpyHostToDevice));
      NC(ncclAllGather(dbuf + kRec * size_t(e->rank), dbuf, kRec, ncclChar, e->nccl, e->comp));
      CU(cudaStreamSynchronize(e->comp));
      CU(cudaMemcpy(all.data(), dbuf, all.size(), cudaMemcpyDeviceToHost));
      attempt([&] {
        for (int g = 0; g < e->G; ++g) {
          if (g == e->rank) continue;
          for (int b = 0; b < 2; ++b) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, all.data() + kRec * size_t(g) + 64 * b, 64);
            void* ptr = nullptr;
            CU(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            e->peer_base[b][g] = static_cast<float*>(ptr);
          }
          if (e->sig) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, all.data() + kRec * size_t(g) + 128, 64);
            void* ptr = nullptr;
            CU(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            e->peer_sig[g] = static_cast<unsigned long long*>(ptr);
          }
        }
      });
      CU(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
      NC(ncclAllReduce(dok, dok, 1, ncclInt, ncclMin, e->nccl, e->comp));
      CU(cudaStreamSynchronize(e->comp));
      CU(cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost));
      CU(cudaFree(dbuf));
      CU(cudaFree(dok));
      if (ok) {
        CU(cudaMalloc(&e->bar_buf, sizeof(float)));
        CU(cudaMemset(e->bar_buf, 0, sizeof(float)));
      } else {
        for (int g = 0; g < e->G; ++g) {
          for (int b = 0; b < 2; ++b)
            if (g != e->rank && e->peer_base[b][g]) {
              cudaIpcCloseMemHandle(e->peer_base[b][g]);
              e->peer_base[b][g] = nullptr;
            }
          if (g != e->rank && e->peer_sig[g]) {
            cudaIpcCloseMemHandle(e->peer_sig[g]);
            e->peer_sig[g] = nullptr;
          }
        }
        e->inplace_p2p = false;
        e->p2p_push = false;
        // every rank reaches this branch together (agreed flag)
        if (!auto_transport)
          dg::config_error("engine_create: P2P transport unavailable (CUDA IPC failed on some rank" +
                           (why.empty() ? std::string(")") : std::string(": ") + why + ")"));
        e->transport = DG_TRANSPORT_NCCL;
        p2p = false;
        if (e->max_recv && !e->slots) CU(cudaMalloc(&e->slots, sizeof(float) * 2 * e->max_recv * e->chunk));
      }
    }
    if (e->G > 1 && e->transport == DG_TRANSPORT_NCCL) {
      e->nccl_register(e->arena[DG_BUF_X], sizeof(float) * e->d_pad * e->NL);
      e->nccl_register(e->x_alt, sizeof(float) * e->d_pad * e->NL);
      e->nccl_register(e->slots, sizeof(float) * 2 * e->max_recv * e->chunk);
    }
    *out = e.release();
  });
}

int dg_engine_buffer(dg_engine* e, int local, int which, float** p) {
  return guarded([&] {
    if (!e || !p) dg::config_error("engine_buffer: null argument");
    if (local < 0 || local >= e->NL) dg::config_error("engine_buffer: local node out of range");
    if (which < 0 || which > 4 || !e->arena[which]) dg::config_error("engine_buffer: no such buffer");
    *p = e->buf(which, local);
    if (which == DG_BUF_X) e->seeded_for = -1;  // the caller may write x: re-seed pushed copies
  });
}

static void check_slice(dg_engine* e, int local, int which, size_t off, size_t cnt) {
  if (!e) dg::config_error("engine: null handle");
  if (local < 0 || local >= e->NL) dg::config_error("engine: local node out of range");
  if (which < 0 || which > 4 || !e->arena[which]) dg::config_error("engine: no such buffer");
  if (off > e->d || cnt > e->d - off) dg::config_error("engine: slice out of range");
}

int dg_engine_upload(dg_engine* e, int local, int which, const float* host, size_t off, size_t cnt) {
  return guarded([&] {
    check_slice(e, local, which, off, cnt);
    CU(cudaSetDevice(e->device));
    if (which == DG_BUF_X) e->seeded_for = -1;
    CU(cudaMemcpyAsync(e->buf(which, local) + off, host, cnt * sizeof(float), cudaMemcpyHostToDevice,
                       e->comp));
  });
}

int dg_engine_download(dg_engine* e, int local, int which, float* host, size_t off, size_t cnt) {
  return guarded([&] {
    check_slice(e, local, which, off, cnt);
    CU(cudaSetDevice(e->device));
    CU(cudaMemcpyAsync(host, e->buf(which, local) + off, cnt * sizeof(float), cudaMemcpyDeviceToHost,
                       e->comp));
    CU(cudaStreamSynchronize(e->comp));
  });
}

int dg_engine_gather(dg_engine* e, int local, int which, const uint64_t* idx, size_t n, float* out) {
  return guarded([&] {
    check_slice(e, local, which, 0, 0);
    if (n && (!idx || !out)) dg::config_error("engine_gather: null argument");
    for (size_t k = 0; k < n; ++k)
      if (idx[k] >= e->d) dg::config_error("engine_gather: index out of range");
    if (!n) return;
    CU(cudaSetDevice(e->device));
    uint64_t* didx = nullptr;
    float* dout = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&didx), n * sizeof(uint64_t), e->comp));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&dout), n * sizeof(float), e->comp));
    CU(cudaMemcpyAsync(didx, idx, n * sizeof(uint64_t), cudaMemcpyHostToDevice, e->comp));
    dg::gather_kernel<<<unsigned((n + 255) / 256), 256, 0, e->comp>>>(dout, e->buf(which, local), didx,
                                                                       (long long)n);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, dout, n * sizeof(float), cudaMemcpyDeviceToHost, e->comp));
    CU(cudaFreeAsync(didx, e->comp));
    CU(cudaFreeAsync(dout, e->comp));
    CU(cudaStreamSynchronize(e->comp));
  });
}

int dg_engine_fill_synthetic(dg_engine* e, int which, uint64_t seed, uint32_t purpose, int per_node,
                             uint64_t iteration) {
  return guarded([&] {
    check_slice(e, 0, which, 0, 0);
    CU(cudaSetDevice(e->device));
    if (which == DG_BUF_X) e->seeded_for = -1;
    for (int i = 0; i < e->NL; ++i) {
      const uint64_t st =
          dg::stream_state(seed, purpose, per_node ? uint64_t(e->first + i) : 0, iteration);
      dg::synth_fill<<<dg::grid_for((long long)e->d, 8), 256, 0, e->comp>>>(e->buf(which, i),
                                                                           (long long)e->d, st);
      CU(cudaGetLastError());
    }
  });
}

// fp64 column sums of the current x over all N nodes (collective), into `colsum`
static void consensus_colsum(dg_engine* e, double* colsum, const dg::NodePtrs& xp) {
  const unsigned grid = dg::grid_for((long long)e->d, 8);
  dg::column_sum<<<grid, 256, 0, e->comp>>>(colsum, xp, e->NL, (long long)e->d);
  CU(cudaGetLastError());
  if (e->G > 1) NC(ncclAllReduce(colsum, colsum, e->d, ncclDouble, ncclSum, e->nccl, e->comp));
}

int dg_engine_consensus_fix_mean(dg_engine* e) {
  return guarded([&] {
    if (!e) dg::config_error("engine_consensus_fix_mean: null handle");
    CU(cudaSetDevice(e->device));
    dg::NodePtrs xp{};
    for (int i = 0; i < e->NL; ++i) xp.p[i] = e->buf(DG_BUF_X, i);
    if (!e->xbar_ref) CU(cudaMalloc(&e->xbar_ref, e->d * sizeof(double)));
    consensus_colsum(e, e->xbar_ref, xp);
    CU(cudaStreamSynchronize(e->comp));
  });
}

int dg_engine_consensus(dg_engine* e, double* dispersion, double* mean_sq) {
  return guarded([&] {
    if (!e) dg::config_error("engine_consensus: null handle");
    CU(cudaSetDevice(e->device));
    dg::NodePtrs xp{};
    for (int i = 0; i < e->NL; ++i) xp.p[i] = e->buf(DG_BUF_X, i);
    double* colsum = e->xbar_ref;
    double* out = nullptr;
    if (!colsum) CU(cudaMallocAsync(reinterpret_cast<void**>(&colsum), e->d * sizeof(double), e->comp));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&out), 2 * sizeof(double), e->comp));
    CU(cudaMemsetAsync(out, 0, 2 * sizeof(double), e->comp));
    const unsigned grid = dg::grid_for((long long)e->d, 8);
    if (!e->xbar_ref) consensus_colsum(e, colsum, xp);
    // mean term counted once (rank 0); dispersion of the resident nodes on every rank
    dg::dispersion<<<grid, 256, 0, e->comp>>>(out, colsum, 1.0 / double(e->N), xp, e->NL, (long long)e->d,
                                              e->rank == 0);
    CU(cudaGetLastError());
    if (e->G > 1) NC(ncclAllReduce(out, out, 2, ncclDouble, ncclSum, e->nccl, e->comp));
    double h[2];
    CU(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, e->comp));
    if (colsum != e->xbar_ref) CU(cudaFreeAsync(colsum, e->comp));
    CU(cudaFreeAsync(out, e->comp));
    CU(cudaStreamSynchronize(e->comp));
    if (dispersion) *dispersion = h[0];
    if (mean_sq) *mean_sq = h[1];
  });
}

int dg_engine_step_range(dg_engine* e, long t, size_t off, size_t len) {
  return guarded([&] {
    if (!e) dg::config_error("engine_step_range: null handle");
    e->step_range(t, off, len);
  });
}

int dg_engine_wait_stream(dg_engine* e, void* stream) {
  return guarded([&] {
    if (!e) dg::config_error("engine_wait_stream: null handle");
    CU(cudaSetDevice(e->device));
    CU(cudaEventRecord(e->ev_user, static_cast<cudaStream_t>(stream)));
    CU(cudaStreamWaitEvent(e->comp, e->ev_user, 0));
  });
}

int dg_engine_join(dg_engine* e, void* stream) {
  return guarded([&] {
    if (!e) dg::config_error("engine_join: null handle");
    CU(cudaSetDevice(e->device));
    CU(cudaEventRecord(e->ev_user, e->comp));
    CU(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e->ev_user, 0));
  });
}

int dg_engine_step(dg_engine* e, long t) {
  return guarded([&] {
    if (!e) dg::config_error("engine_step: null handle");
    e->step(t);
  });
}

int dg_engine_run_steps(dg_engine* e, long t_first, long t_last, int flags) {
  return guarded([&] {
    if (!e) dg::config_error("engine_run_steps: null handle");
    e->run_steps(t_first, t_last, flags);
  });
}

int dg_engine_sync(dg_engine* e) {
  return guarded([&] {
    if (!e) dg::config_error("engine_sync: null handle");
    CU(cudaSetDevice(e->device));
    CU(cudaStreamSynchronize(e->comm));
    for (auto st : e->pull) CU(cudaStreamSynchronize(st));
    CU(cudaStreamSynchronize(e->comp));
    if (e->nccl) {
      ncclResult_t ar;
      NC(ncclCommGetAsyncError(e->nccl, &ar));
      NC(ar);
    }
    e->harvest_timing();
    int f = INT_MAX;
    CU(cudaMemcpy(&f, e->flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (f != INT_MAX)
      throw dg::Error(DG_DIVERGENCE, "non-finite state at iteration " + std::to_string(f), f);
    int inv = INT_MAX;
    CU(cudaMemcpy(&inv, e->inv_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (inv != INT_MAX)
      throw dg::Error(DG_INVARIANT, "allreduce_adam_step: worker states diverged at iteration " + std::to_string(inv));
  });
}

int dg_engine_streams(dg_engine* e, void** compute, void** comm) {
  return guarded([&] {
    if (!e) dg::config_error("engine_streams: null handle");
    if (compute) *compute = e->comp;
    if (comm) *comm = e->comm;
  });
}

int dg_engine_get_stats(const dg_engine* e, dg_engine_stats* o) {
  return guarded([&] {
    if (!e || !o) dg::config_error("engine_stats: null argument");
    o->local_nodes = e->NL;
    o->first_node = e->first;
    o->nodes = e->N;
    o->world_size = e->G;
    o->rank = e->rank;
    o->d = e->d;
    o->chunk = e->chunk;
    o->kernel_launches = e->launches;
    o->steps = e->steps;
    o->bytes_sent = e->sent;
    o->bytes_received = e->received;
    o->hbm_bytes = e->hbm;
    int v = 0;
    ncclGetVersion(&v);
    o->nccl_version = v;
    o->kernel_ms = e->kernel_ms;
    o->timed_launches = e->timed_launches;
    o->timed_hbm_bytes = e->timed_bytes;
    o->transport = e->transport;
    o->barriers = e->barriers;
    o->remote_kernel_ms = e->remote_ms;
    o->remote_bytes = e->remote_bytes;
  });
}

int dg_engine_set_timing(dg_engine* e, int on) {
  return guarded([&] {
    if (!e) dg::config_error("engine_set_timing: null handle");
    CU(cudaSetDevice(e->device));
    if (!on) {
      CU(cudaStreamSynchronize(e->comp));
      e->tev_used = 0;
      e->kernel_ms = e->timed_bytes = e->remote_ms = e->remote_bytes = 0;
      e->timed_launches = 0;
    }
    e->timing = on != 0;
  });
}

void dg_engine_destroy(dg_engine* e) { delete e; }

// ------------------------------------------------------------------ semantic API
int dg_gossip_mix_f32(float* mixed, const float* const* xs, const double* w, int count, size_t d,
                      void* stream) {
  return guarded([&] {
    if (!mixed || (count > 0 && (!xs || !w)) || count < 0) dg::config_error("gossip_mix: bad arguments");
    auto st = static_cast<cudaStream_t>(stream);
    double* scratch = nullptr;  // fp64 partial sums when more than 16 sources
    if (count > dg::kMixPtrs) CU(cudaMallocAsync(reinterpret_cast<void**>(&scratch), d * sizeof(double), st));
    int done = 0;
    do {
      dg::MixArgs a{};
      a.count = std::min(count - done, dg::kMixPtrs);
      a.accumulate = done > 0;
      for (int k = 0; k < a.count; ++k) {
        a.xs[k] = xs[done + k];
        a.w[k] = w[done + k];
      }
      done += a.count;
      dg::mix_kernel<<<dg::grid_for((long long)d, 8), 256, 0, st>>>(mixed, scratch, a, (long long)d,
                                                                   done >= count);
      CU(cudaGetLastError());
    } while (done < count);
    if (scratch) CU(cudaFreeAsync(scratch, st));
  });
}

static void node_step_launch(int algo, float* x, const float* g, float* m, float* v, float* b,
                             const float* mixed, size_t d, const dg_adam_cfg* cfg, long t, long T,
                             void* stream) {
  if (!x || !g || !m || !v || !mixed || (algo == DG_ALGO_ACCUM && !b))
    dg::config_error("step: null buffer");
  bool fold = false;
  const dg::DevScalars s = dg::scalars(cfg, algo, t, T, &fold);
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec4 = al(x) && al(g) && al(m) && al(v) && al(mixed) && (!b || al(b));
  auto st = static_cast<cudaStream_t>(stream);
  const unsigned grid = dg::grid_for((long long)(vec4 ? (d + 3) / 4 : d), 8);
  int* f = dg::semantic_flag();
  if (algo == DG_ALGO_DADAM)
    dg::node_step<0, false><<<grid, 256, 0, st>>>(x, g, m, v, b, mixed, (long long)d, s, int(t), f, vec4);
  else if (fold)
    dg::node_step<1, true><<<grid, 256, 0, st>>>(x, g, m, v, b, mixed, (long long)d, s, int(t), f, vec4);
  else
    dg::node_step<1, false><<<grid, 256, 0, st>>>(x, g, m, v, b, mixed, (long long)d, s, int(t), f, vec4);
  CU(cudaGetLastError());
}

int dg_dadam_step_f32(float* x, const float* g, float* m, float* v, const float* mixed, size_t d,
                      const dg_adam_cfg* cfg, long t, void* stream) {
  return guarded([&] { node_step_launch(DG_ALGO_DADAM, x, g, m, v, nullptr, mixed, d, cfg, t, 0, stream); });
}

int dg_accum_adam_step_f32(float* x, const float* g, float* mh, float* vh, float* acc,
                           const float* mixed, size_t d, const dg_adam_cfg* cfg, long t, long T,
                           void* stream) {
  return guarded([&] { node_step_launch(DG_ALGO_ACCUM, x, g, mh, vh, acc, mixed, d, cfg, t, T, stream); });
}

int dg_step_check_divergence(void* stream) {
  return guarded([&] {
    CU(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    int f = INT_MAX;
    CU(cudaMemcpyFromSymbol(&f, dg::g_semantic_flag, sizeof(int)));
    const int none = INT_MAX;
    CU(cudaMemcpyToSymbol(dg::g_semantic_flag, &none, sizeof(int)));
    if (f != INT_MAX)
      throw dg::Error(DG_DIVERGENCE, "non-finite state at iteration " + std::to_string(f), f);
  });
}

int dg_fill_synthetic_f32(float* out, size_t n, uint64_t seed, uint32_t purpose, uint64_t worker,
                          uint64_t iteration, void* stream) {
  return guarded([&] {
    if (!out && n) dg::config_error("fill_synthetic: null output");
    const uint64_t st = dg::stream_state(seed, purpose, worker, iteration);
    dg::synth_fill<<<dg::grid_for((long long)n, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        out, (long long)n, st);
    CU(cudaGetLastError());
  });
}

}  // extern "C"
