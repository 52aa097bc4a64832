// engine.cu -- device side of libdg: semantic per-node steps and the fused
// gossip + Adam engine (one per GPU) with the chunked, double-buffered NCCL
// exchange over NVLink.
//
// Replaces the hot loop of the reference's trainsim (Jacobi
// snapshot, mixed sum, per-worker dadam_step / accum_adam_step) and the
// paper's bucketed overlap (Fig. 1).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>

#include "dg_internal.hpp"
#include "kernels.cuh"

namespace dg {
namespace {

constexpr size_t kDefaultChunk = 6553600;  // 25 MiB of fp32 (PAPER.md:328 DDP bucket)
constexpr size_t kAlign = 64;              // floats: 256-byte aligned node buckets / chunks

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(DG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(DG_NCCL_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
}
#define CU(x) ::dg::cuda_check((x), #x)
#define NC(x) ::dg::nccl_check((x), #x)

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
  } else if (algo != DG_ALGO_DADAM) {
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

int sm_count(int dev) {
  int n = 0;
  CU(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}
int current_sms() {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  return sm_count(dev);
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

// ------------------------------------------------------------------ fused launch table
using LaunchFn = void (*)(const void* args, unsigned grid, cudaStream_t st);

template <int NL, int DEG, int ALGO, bool FOLD>
void launch_fused(const void* args, unsigned grid, cudaStream_t st) {
  gossip_adam_fused<NL, DEG, ALGO, FOLD>
      <<<grid, 256, 0, st>>>(*static_cast<const FusedArgs<NL, DEG>*>(args));
}

template <int NL, int DEG>
LaunchFn pick_algo(int algo, bool fold) {
  if (algo == DG_ALGO_DADAM) return launch_fused<NL, DEG, 0, false>;
  return fold ? launch_fused<NL, DEG, 1, true> : launch_fused<NL, DEG, 1, false>;
}
template <int NL>
LaunchFn pick_deg(int deg, int algo, bool fold) {
  if (deg <= 2) return pick_algo<NL, 2>(algo, fold);
  if (deg <= 4) return pick_algo<NL, 4>(algo, fold);
  if (deg <= 8) return pick_algo<NL, 8>(algo, fold);
  return pick_algo<NL, 16>(algo, fold);
}
int round_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
int round_deg(int d) { return d <= 2 ? 2 : d <= 4 ? 4 : d <= 8 ? 8 : 16; }
LaunchFn pick(int nl, int deg, int algo, bool fold) {
  switch (round_pow2(nl)) {
    case 1: return pick_deg<1>(deg, algo, fold);
    case 2: return pick_deg<2>(deg, algo, fold);
    case 4: return pick_deg<4>(deg, algo, fold);
    case 8: return pick_deg<8>(deg, algo, fold);
    default: return pick_deg<16>(deg, algo, fold);
  }
}

// Fills a FusedArgs<NL,DEG> image in a byte buffer (layout computed by the template).
template <int NL, int DEG>
void fill_args_t(std::vector<unsigned char>& buf, const RoundPlan& p, const float* const* local_x,
                 const float* const* slot, float* const* x, const float* const* g, float* const* m,
                 float* const* v, float* const* b, size_t off, size_t len, const DevScalars& s,
                 int t, int* flag) {
  buf.assign(sizeof(FusedArgs<NL, DEG>), 0);
  auto* a = reinterpret_cast<FusedArgs<NL, DEG>*>(buf.data());
  for (int i = 0; i < NL; ++i) {
    a->deg[i] = i < p.n_local ? p.deg[i] : 0;
    for (int k = 0; k < DEG; ++k) {
      if (i < p.n_local && k < p.deg[i]) {
        const int sidx = p.src[i][k];
        a->src[i][k] = sidx < p.n_local ? local_x[sidx] + off : slot[sidx - p.n_local];
        a->w[i][k] = p.w[i][k];
      }
    }
    if (i < p.n_local) {
      a->x[i] = x[i] + off;
      a->g[i] = g[i] + off;
      a->m[i] = m[i] + off;
      a->v[i] = v[i] + off;
      a->b[i] = b ? b[i] + off : nullptr;
    }
  }
  a->s = s;
  a->n = (long long)len;
  a->t = t;
  a->div_flag = flag;
}
template <int NL>
void fill_deg(int deg, std::vector<unsigned char>& buf, const RoundPlan& p, const float* const* lx,
              const float* const* slot, float* const* x, const float* const* g, float* const* m,
              float* const* v, float* const* b, size_t off, size_t len, const DevScalars& s, int t,
              int* flag) {
  switch (round_deg(deg)) {
    case 2: return fill_args_t<NL, 2>(buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    case 4: return fill_args_t<NL, 4>(buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    case 8: return fill_args_t<NL, 8>(buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    default: return fill_args_t<NL, 16>(buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
  }
}
void fill_args(std::vector<unsigned char>& buf, const RoundPlan& p, const float* const* lx,
               const float* const* slot, float* const* x, const float* const* g, float* const* m,
               float* const* v, float* const* b, size_t off, size_t len, const DevScalars& s,
               int t, int* flag) {
  switch (round_pow2(p.n_local)) {
    case 1: return fill_deg<1>(p.max_deg, buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    case 2: return fill_deg<2>(p.max_deg, buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    case 4: return fill_deg<4>(p.max_deg, buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    case 8: return fill_deg<8>(p.max_deg, buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
    default: return fill_deg<16>(p.max_deg, buf, p, lx, slot, x, g, m, v, b, off, len, s, t, flag);
  }
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
  int blocks_per_sm = 4;
  std::vector<unsigned char> argbuf;
  // optional per-launch CUDA-event timing (bench roofline)
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
  std::vector<double> tev_bytes;
  size_t tev_used = 0;
  double kernel_ms = 0, timed_bytes = 0;
  long timed_launches = 0;
  void harvest_timing();

  float* buf(int which, int local) const { return arena[which] + size_t(local) * d_pad; }
  void enqueue_fused(const dg::RoundPlan& p, size_t off, size_t len, int slot_set,
                     const dg::DevScalars& s, bool fold, long t);
  void step(long t);
  ~dg_engine();
};

dg_engine::~dg_engine() {
  if (device >= 0) cudaSetDevice(device);
  if (comp) cudaStreamSynchronize(comp);
  if (comm) cudaStreamSynchronize(comm);
  if (nccl) ncclCommDestroy(nccl);
  for (float* a : arena)
    if (a) cudaFree(a);
  if (slots) cudaFree(slots);
  if (flag) cudaFree(flag);
  if (ev_begin) cudaEventDestroy(ev_begin);
  for (auto e : ev_slot_free)
    if (e) cudaEventDestroy(e);
  for (auto e : ev_recv) cudaEventDestroy(e);
  for (auto& pr : tev) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (comp) cudaStreamDestroy(comp);
  if (comm) cudaStreamDestroy(comm);
}

void dg_engine::enqueue_fused(const dg::RoundPlan& p, size_t off, size_t len, int slot_set,
                              const dg::DevScalars& s, bool fold, long t) {
  const float* lx[dg::kMaxLocal];
  float *x[dg::kMaxLocal], *m[dg::kMaxLocal], *v[dg::kMaxLocal], *b[dg::kMaxLocal];
  const float* g[dg::kMaxLocal];
  for (int i = 0; i < NL; ++i) {
    lx[i] = x[i] = buf(DG_BUF_X, i);
    g[i] = buf(DG_BUF_G, i);
    m[i] = buf(DG_BUF_M, i);
    v[i] = buf(DG_BUF_V, i);
    b[i] = algo == DG_ALGO_ACCUM ? buf(DG_BUF_ACC, i) : nullptr;
  }
  const float* slot_ptr[dg::kMaxRemote];
  for (int r = 0; r < int(p.recv_node.size()); ++r)
    slot_ptr[r] = slots + (size_t(slot_set) * max_recv + r) * chunk;
  dg::fill_args(argbuf, p, lx, slot_ptr, x, g, m, v, b, off, len, s, int(t), flag);
  const auto fn = dg::pick(p.n_local, p.max_deg, algo, fold);
  const unsigned grid = dg::grid_for((long long)(len + 3) / 4, blocks_per_sm);
  const double per = algo == DG_ALGO_DADAM ? 28.0 : (fold ? 36.0 : 28.0);
  const double bytes = double(len) * (per * p.n_local + 4.0 * double(p.recv_node.size()));
  if (timing) {
    if (tev_used == tev.size()) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      tev.push_back({a, b});
      tev_bytes.push_back(0);
    }
    CU(cudaEventRecord(tev[tev_used].first, comp));
  }
  fn(argbuf.data(), grid, comp);
  dg::cuda_check(cudaGetLastError(), "fused kernel launch");
  if (timing) {
    CU(cudaEventRecord(tev[tev_used].second, comp));
    tev_bytes[tev_used++] = bytes;
  }
  ++launches;
  hbm += bytes;
}

void dg_engine::harvest_timing() {
  for (size_t k = 0; k < tev_used; ++k) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, tev[k].first, tev[k].second));
    kernel_ms += ms;
    timed_bytes += tev_bytes[k];
    ++timed_launches;
  }
  tev_used = 0;
}

void dg_engine::step(long t) {
  bool fold = false;
  const dg::DevScalars s = dg::scalars(&adam, algo, t, T, &fold);
  CU(cudaSetDevice(device));
  const dg::RoundPlan& p = plans[size_t((t - 1) % P)];
  ++steps;
  if (p.send_node.empty() && p.recv_node.empty()) {  // intra-GPU round: one launch
    enqueue_fused(p, 0, d, 0, s, fold, t);
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
    enqueue_fused(p, off, len, set, s, fold, t);
    CU(cudaEventRecord(ev_slot_free[set], comp));
  }
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
    if (e->NL < 1) dg::config_error("engine_create: no resident nodes on this rank");
    CU(cudaSetDevice(c->device));
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithFlags(&e->comp, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithPriority(&e->comm, cudaStreamNonBlocking, hi));  // comm first
    CU(cudaEventCreateWithFlags(&e->ev_begin, cudaEventDisableTiming));
    for (auto& ev : e->ev_slot_free) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->ev_recv.resize(e->n_chunks);
    for (auto& ev : e->ev_recv) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const int kinds = c->algo == DG_ALGO_ACCUM ? 5 : 4;
    for (int k = 0; k < kinds; ++k) {
      CU(cudaMalloc(&e->arena[k], sizeof(float) * e->d_pad * e->NL));
      CU(cudaMemsetAsync(e->arena[k], 0, sizeof(float) * e->d_pad * e->NL, e->comp));
    }
    if (e->max_recv) CU(cudaMalloc(&e->slots, sizeof(float) * 2 * e->max_recv * e->chunk));
    CU(cudaMalloc(&e->flag, sizeof(int)));
    const int none = INT_MAX;
    CU(cudaMemcpyAsync(e->flag, &none, sizeof(int), cudaMemcpyHostToDevice, e->comp));
    CU(cudaStreamSynchronize(e->comp));
    if (e->G > 1) {
      ncclUniqueId id;
      std::memcpy(&id, c->nccl_id, sizeof(id));
      NC(ncclCommInitRank(&e->nccl, e->G, id, e->rank));
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

int dg_engine_fill_synthetic(dg_engine* e, int which, uint64_t seed, uint32_t purpose, int per_node,
                             uint64_t iteration) {
  return guarded([&] {
    check_slice(e, 0, which, 0, 0);
    CU(cudaSetDevice(e->device));
    for (int i = 0; i < e->NL; ++i) {
      const uint64_t st =
          dg::stream_state(seed, purpose, per_node ? uint64_t(e->first + i) : 0, iteration);
      dg::synth_fill<<<dg::grid_for((long long)e->d, 8), 256, 0, e->comp>>>(e->buf(which, i),
                                                                           (long long)e->d, st);
      CU(cudaGetLastError());
    }
  });
}

int dg_engine_step(dg_engine* e, long t) {
  return guarded([&] {
    if (!e) dg::config_error("engine_step: null handle");
    e->step(t);
  });
}

int dg_engine_sync(dg_engine* e) {
  return guarded([&] {
    if (!e) dg::config_error("engine_sync: null handle");
    CU(cudaSetDevice(e->device));
    CU(cudaStreamSynchronize(e->comm));
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
  });
}

int dg_engine_set_timing(dg_engine* e, int on) {
  return guarded([&] {
    if (!e) dg::config_error("engine_set_timing: null handle");
    CU(cudaSetDevice(e->device));
    if (!on) {
      CU(cudaStreamSynchronize(e->comp));
      e->tev_used = 0;
      e->kernel_ms = e->timed_bytes = 0;
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
