// legacy.cu -- the round-1 fused-kernel variants (register-streaming per-thread,
// warp-per-node, cooperative and TMA producer/consumer kernels) and their
// launch tables.  Not the default: the engine runs gossip_adam_staged unless
// DG_STAGED=0 or a round does not fit it.  A separate
// translation unit so the many template instantiations build in parallel.
#define DG_KERNELS_TEMPLATES_ONLY 1
#include <algorithm>
#include <cstring>
#include <map>

#include "launch.hpp"

namespace dg {

// ------------------------------------------------------------------ fused launch table
// One entry per (component size NC, degree bound DEG, algorithm, fold).  Each
// entry sizes its grid from the occupancy API so that exactly one wave of
// CTAs is resident (grid-stride loop inside), split across the components.

int coop_min_nc() {  // DG_COOP_MIN_NC: smallest component size using the cooperative kernel
  static const int v = [] {
    const char* e = std::getenv("DG_COOP_MIN_NC");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}

template <int NC, int NS, int ALGO, bool FOLD>
void launch_coop(const void* args, long long cols, int n_comp, int sms, cudaStream_t st) {
  auto kern = gossip_adam_coop<NC, NS, ALGO, FOLD>;
  constexpr int threads = CoopShape<NC, NS>::threads;
  static const int occ = [&] {
    int o = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, 0), "occupancy");
    return std::max(1, o);
  }();
  const long long resident = std::max(1LL, (long long)(grid_waves() * occ * sms));
  const long long per_comp = std::max(1LL, resident / n_comp);
  const long long need = (cols * NC + threads - 1) / threads;
  const dim3 grid(unsigned(std::max(1LL, std::min(per_comp, need))), unsigned(n_comp));
  kern<<<grid, threads, 0, st>>>(*static_cast<const FusedArgs<NC, NS>*>(args));
}

// DG_WARPS_MIN_NC: launches of >= this many (and <= 8) single-member components
// run one warp per node (default 4; measured static exponential 0.80 -> 0.84,
// AER AccumAdam 0.91 -> 0.96 of HBM: neighbour re-reads stop missing L2)
int warps_min_nc() {
  static const int v = [] {
    const char* e = std::getenv("DG_WARPS_MIN_NC");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}
template <int NS, int ALGO, bool FOLD>
void launch_warps(const void* args, long long cols, int n_comp, int sms, cudaStream_t st) {
  auto kern = gossip_adam_warps<NS, ALGO, FOLD>;
  const int threads = 32 * n_comp;
  static int occ_by_nc[9] = {};
  int& occ = occ_by_nc[n_comp];
  if (!occ) {
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0), "occupancy");
    occ = std::max(1, occ);
  }
  const long long resident = std::max(1LL, (long long)(grid_waves() * occ * sms));
  const long long need = (cols + 31) / 32;
  kern<<<unsigned(std::max(1LL, std::min(resident, need))), threads, 0, st>>>(
      *static_cast<const FusedArgs<1, NS>*>(args));
}

template <int NC, int NS, int ALGO, bool FOLD>
void launch_fused(const void* args, long long cols, int n_comp, int sms, cudaStream_t st) {
  if constexpr (NC >= 2) {
    if (NC >= coop_min_nc()) return launch_coop<NC, NS, ALGO, FOLD>(args, cols, n_comp, sms, st);
  } else {
    if (n_comp >= warps_min_nc() && n_comp <= 8) return launch_warps<NS, ALGO, FOLD>(args, cols, n_comp, sms, st);
  }
  auto kern = gossip_adam_fused<NC, NS, ALGO, FOLD>;
  constexpr int threads = LaunchShape<NC, NS>::threads;
  static const int occ = [&] {
    int o = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, 0), "occupancy");
    return std::max(1, o);
  }();
  const long long resident = std::max(1LL, (long long)(grid_waves() * occ * sms));
  const long long per_comp = std::max(1LL, resident / n_comp);
  const long long need = (cols + threads - 1) / threads;
  const dim3 grid(unsigned(std::max(1LL, std::min(per_comp, need))), unsigned(n_comp));
  kern<<<grid, threads, 0, st>>>(*static_cast<const FusedArgs<NC, NS>*>(args));
}

template <int NC, int NS>
LaunchFn pick_algo(int algo, bool fold) {
  if (algo == DG_ALGO_DADAM) return launch_fused<NC, NS, 0, false>;
  return fold ? launch_fused<NC, NS, 1, true> : launch_fused<NC, NS, 1, false>;
}
template <int NC>
LaunchFn pick_ns(int ns, int algo, bool fold) {
  // instantiated only for NS >= NC
  if (ns <= 2 && NC <= 2) return pick_algo<NC, (NC <= 2 ? 2 : NC)>(algo, fold);
  if (ns <= 4 && NC <= 4) return pick_algo<NC, (NC <= 4 ? 4 : NC)>(algo, fold);
  if (ns <= 6 && NC == 1) return pick_algo<1, 6>(algo, fold);  // static-exponential nodes (84 -> 80 regs)
  if (ns <= 8 && NC <= 8) return pick_algo<NC, (NC <= 8 ? 8 : NC)>(algo, fold);
  if (ns <= 16) return pick_algo<NC, 16>(algo, fold);
  return pick_algo<NC, 32>(algo, fold);
}
LaunchFn pick(int nc, int ns, int algo, bool fold) {
  switch (nc) {
    case 1: return pick_ns<1>(ns, algo, fold);
    case 2: return pick_ns<2>(ns, algo, fold);
    case 4: return pick_ns<4>(ns, algo, fold);
    case 8: return pick_ns<8>(ns, algo, fold);
    default: return pick_ns<16>(ns, algo, fold);
  }
}

// Builds the FusedArgs<NC,NS> image of one launch in a byte buffer.
template <int NC, int NS>
void fill_args_t(std::vector<unsigned char>& buf, const RoundPlan& p, const Buffers& bf, size_t off,
                 size_t len, const DevScalars& s, int t, int* flag) {
  using A = FusedArgs<NC, NS>;
  buf.assign(sizeof(A), 0);
  auto* a = reinterpret_cast<A*>(buf.data());
  if (int(p.comps.size()) > A::CMAX) config_error("plan: too many mixing components");
  for (size_t c = 0; c < p.comps.size(); ++c) {
    const auto& cp = p.comps[c];
    if (int(cp.members.size()) > NC || int(cp.srcs.size()) > NS) config_error("plan: component too large");
    a->nm[c] = int(cp.members.size());
    a->ns[c] = int(cp.srcs.size());
    for (size_t k = 0; k < cp.srcs.size(); ++k) {
      const int code = cp.srcs[k];
      a->src[c][k] = code >= 0 ? bf.x[code] + off : bf.slot[-code - 1];
    }
    for (size_t j = 0; j < cp.members.size(); ++j) {
      const int li = cp.members[j];
      for (size_t k = 0; k < cp.srcs.size(); ++k) a->w[c][j][k] = cp.w[j][k];
      a->x[c][j] = bf.xout[li] + off;
      for (int k = 0; k < kPushMax; ++k) {
        float* dst = bf.xpub ? bf.xpub[li * kPushMax + k] : nullptr;
        a->xp[c][j][k] = dst ? dst + off : nullptr;
      }
      a->g[c][j] = bf.g[li] + off;
      a->m[c][j] = bf.m[li] + off;
      a->v[c][j] = bf.v[li] + off;
      a->b[c][j] = bf.b ? bf.b[li] + off : nullptr;
    }
  }
  a->s = s;
  a->n = (long long)len;
  a->t = t;
  a->div_flag = flag;
}
// source count that selects the NS instantiation: the largest actual source
// count of the plan's components (src_bound is rounded up to a power of two).
// pick() and fill_args() must agree on it (same FusedArgs<NC, NS> layout).
int launch_ns(const RoundPlan& p) {
  size_t ns = 1;
  for (const auto& c : p.comps) ns = std::max(ns, c.srcs.size());
  return int(ns);
}
template <int NC>
void fill_ns(std::vector<unsigned char>& buf, const RoundPlan& p, const Buffers& bf, size_t off,
             size_t len, const DevScalars& s, int t, int* flag) {
  const int ns = launch_ns(p);
  if (ns <= 2 && NC <= 2) return fill_args_t<NC, (NC <= 2 ? 2 : NC)>(buf, p, bf, off, len, s, t, flag);
  if (ns <= 4 && NC <= 4) return fill_args_t<NC, (NC <= 4 ? 4 : NC)>(buf, p, bf, off, len, s, t, flag);
  if (ns <= 6 && NC == 1) return fill_args_t<1, 6>(buf, p, bf, off, len, s, t, flag);
  if (ns <= 8 && NC <= 8) return fill_args_t<NC, (NC <= 8 ? 8 : NC)>(buf, p, bf, off, len, s, t, flag);
  if (ns <= 16) return fill_args_t<NC, 16>(buf, p, bf, off, len, s, t, flag);
  return fill_args_t<NC, 32>(buf, p, bf, off, len, s, t, flag);
}
void fill_args(std::vector<unsigned char>& buf, const RoundPlan& p, const Buffers& bf, size_t off,
               size_t len, const DevScalars& s, int t, int* flag) {
  switch (p.comp_size) {
    case 1: return fill_ns<1>(buf, p, bf, off, len, s, t, flag);
    case 2: return fill_ns<2>(buf, p, bf, off, len, s, t, flag);
    case 4: return fill_ns<4>(buf, p, bf, off, len, s, t, flag);
    case 8: return fill_ns<8>(buf, p, bf, off, len, s, t, flag);
    default: return fill_ns<16>(buf, p, bf, off, len, s, t, flag);
  }
}

// ------------------------------------------------------------------ TMA-staged launch
int tma_mode() {  // DG_TMA: 0 never (default), 1 components of >= 4 members, 2 always
  static const int v = [] {
    const char* e = std::getenv("DG_TMA");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
bool use_tma(const RoundPlan& p) {
  const int m = tma_mode();
  return m == 2 || (m == 1 && p.comp_size >= 4);
}

template <int ALGO, bool FOLD, int NS>
void launch_tma_n(const TmaArgs& a, size_t smem, long long units, cudaStream_t st) {
  auto kern = gossip_adam_tma<ALGO, FOLD, NS>;
  static bool configured = false;
  if (!configured) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
               "tma smem attribute");
    configured = true;
  }
  int occ = 0;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTmaThreads, smem), "tma occupancy");
  const long long resident = std::max(1LL, (long long)std::max(1, occ) * current_sms());
  const unsigned grid = unsigned(std::max(1LL, std::min(units, resident)));
  kern<<<grid, kTmaThreads, smem, st>>>(a);
}
template <int ALGO, bool FOLD>
void launch_tma_t(const TmaArgs& a, int ns_max, size_t smem, long long units, cudaStream_t st) {
  if (ns_max <= 2) return launch_tma_n<ALGO, FOLD, 2>(a, smem, units, st);
  if (ns_max <= 4) return launch_tma_n<ALGO, FOLD, 4>(a, smem, units, st);
  if (ns_max <= 8) return launch_tma_n<ALGO, FOLD, 8>(a, smem, units, st);
  if (ns_max <= 16) return launch_tma_n<ALGO, FOLD, 16>(a, smem, units, st);
  return launch_tma_n<ALGO, FOLD, 32>(a, smem, units, st);
}

void launch_tma(const RoundPlan& p, const Buffers& bf, int algo, bool fold, size_t off, size_t len,
                const DevScalars& s, int t, int* flag, cudaStream_t st) {
  thread_local TmaArgs a;  // large POD (~9 KB), reused per host thread
  std::memset(&a, 0, sizeof(a));
  const int K = algo == DG_ALGO_ACCUM ? 4 : 3;
  a.n_comp = int(p.comps.size());
  int row = 0, rows_max = 0, srow = 0;
  for (size_t c = 0; c < p.comps.size(); ++c) {
    const auto& cp = p.comps[c];
    if (int(cp.srcs.size()) > kTmaMaxSrc) config_error("tma: too many sources in a component");
    a.nm[c] = int(cp.members.size());
    a.ns[c] = int(cp.srcs.size());
    a.row0[c] = row;
    a.srow0[c] = srow;
    const int rows = a.ns[c] + a.nm[c] * K;
    if (srow + rows > kTmaMaxRows) config_error("tma: too many staged rows");
    for (size_t k = 0; k < cp.srcs.size(); ++k) {
      const int code = cp.srcs[k];
      a.row_ptr[srow++] = code >= 0 ? bf.x[code] + off : bf.slot[-code - 1];
    }
    for (size_t j = 0; j < cp.members.size(); ++j, ++row) {
      const int li = cp.members[j];
      a.row_node[row] = li;
      for (size_t k = 0; k < cp.srcs.size(); ++k) a.w[row][k] = cp.w[j][k];
      a.row_ptr[srow++] = bf.g[li] + off;
      a.row_ptr[srow++] = bf.m[li] + off;
      a.row_ptr[srow++] = bf.v[li] + off;
      if (K == 4) a.row_ptr[srow++] = bf.b[li] + off;
    }
    rows_max = std::max(rows_max, rows);
  }
  for (int i = 0; i < p.n_local; ++i) {
    a.xb[i] = bf.xout[i] + off;
    a.mb[i] = bf.m[i] + off;
    a.vb[i] = bf.v[i] + off;
    a.bb[i] = bf.b ? bf.b[i] + off : nullptr;
  }
  a.s = s;
  a.n = (long long)len;
  // tile: as large as the stage budget allows, with members x float4 columns a
  // multiple of the CTA size so every thread gets the same number of items
  int nm_max = 1, ns_max = 2;
  for (int c = 0; c < a.n_comp; ++c) {
    nm_max = std::max(nm_max, a.nm[c]);
    ns_max = std::max(ns_max, a.ns[c]);
  }
  const int ct = kTmaConsumerWarps * 32;
  int cols = ct / std::min(nm_max, ct) / 32 * 32;  // float4 columns per consumer-thread round
  cols = std::max(32, cols);
  const int max_cols = DG_TMA_STAGE_BYTES / (16 * rows_max);
  const int tile4 = max_cols >= cols ? max_cols / cols * cols : std::max(32, max_cols / 32 * 32);
  a.tile = tile4 * 4;
  a.rows_max = rows_max;
  a.t = t;
  a.div_flag = flag;
  const size_t stage_bytes = size_t(rows_max) * a.tile * sizeof(float);
  a.stages = int(std::min<size_t>(DG_TMA_STAGES, (227 * 1024 - 256) / stage_bytes));
  if (a.stages < 2) config_error("tma: component too large for a 2-stage shared-memory ring");
  const size_t smem = 256 + size_t(a.stages) * stage_bytes;
  const long long units = ((long long)len + a.tile - 1) / a.tile * a.n_comp;
  if (algo == DG_ALGO_DADAM)
    launch_tma_t<0, false>(a, ns_max, smem, units, st);
  else if (fold)
    launch_tma_t<1, true>(a, ns_max, smem, units, st);
  else
    launch_tma_t<1, false>(a, ns_max, smem, units, st);
}


}  // namespace dg
