// launch.hpp -- host-side launch interface shared by engine.cu (engine, staged
// kernel) and legacy.cu (the round-1 register-streaming / TMA kernel variants,
// kept behind DG_STAGED=0 for sweeps).  Internal, not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "dg_internal.hpp"
#include "kernels.cuh"

namespace dg {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(DG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(DG_NCCL_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
}
#define CU(x) ::dg::cuda_check((x), #x)
#define NC(x) ::dg::nccl_check((x), #x)

inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
inline int sm_count(int dev) {
  int n = 0;
  CU(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}
inline int current_sms() {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  return sm_count(dev);
}
inline double grid_waves() {  // DG_WAVES: resident-wave multiplier (tuning knob, default 1)
  static const double w = [] {
    const char* e = std::getenv("DG_WAVES");
    return e ? std::max(0.05, std::atof(e)) : 1.0;
  }();
  return w;
}

using LaunchFn = void (*)(const void* args, long long cols, int n_comp, int sms, cudaStream_t st);
// Builds the FusedArgs<NC,NS> image of one launch in a byte buffer.
struct Buffers {
  const float* const* slot;  // recv slot base per remote source (already at chunk start)
  float* const* x;           // x^(t-1) (mixing sources)
  float* const* xout;        // where x^(t) goes (== x in place, the other buffer when ping-pong)
  const float* const* g;
  float* const* m;
  float* const* v;
  float* const* b;  // null for DAdam
  float* const* xpub = nullptr;  // [node][kPushMax] extra copies of x^(t) (gossip_adam_fused only)
};

// legacy.cu
LaunchFn pick(int nc, int ns, int algo, bool fold);
int launch_ns(const RoundPlan& p);
void fill_args(std::vector<unsigned char>& buf, const RoundPlan& p, const Buffers& bf, size_t off, size_t len,
               const DevScalars& s, int t, int* flag);
int warps_min_nc();
bool use_tma(const RoundPlan& p);
void launch_tma(const RoundPlan& p, const Buffers& bf, int algo, bool fold, size_t off, size_t len,
                const DevScalars& s, int t, int* flag, cudaStream_t st);

}  // namespace dg
