// nvl_probe.cu -- single-process, two-GPU harness for NVLink evidence of the
// exchange-round fused kernels (ncu may not wrap a multi-rank command, so the
// rank-0 side of an exchange round is reproduced here in one process).
//
// GPU 0 holds 4 resident nodes (x, g, m, v and the second x buffer); GPU 1
// holds the 4 remote neighbours' x^(t-1).  Round = one-peer exponential hop 4
// over 8 nodes on 2 GPUs (BASELINE config 2 at 2 GPUs): node i mixes with
// node i + 4, weights 1/2, every source pair crosses NVLink.  The kernels are
// the engine's own templates, launched as the engine launches them for a P2P
// exchange round (x^(t) to the other buffer):
//   legacy   gossip_adam_fused<1,2,DAdam>: 4 single-member components,
//            sources {local i, peer i+4}   (default for P2P exchange rounds)
//   xshare   gossip_adam_xshare<2,DAdam,COLW>: one group, 4 members, 8 rows
//            (DG_XSHARE_REMOTE=1, and the in-place P2P transport)
// plus the same launches with the peer rows replaced by local copies, which
// isolates the NVLink cost.  Prints GB/s per kernel (CUDA events); under
//   ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
// the NVLink counters come from hardware.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr \
//        -I include -I paper_2410_11998_b200/csrc -o build/nvl_probe scripts/nvl_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "xshare.cuh"

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                     \
    }                                                                                   \
  } while (0)

using namespace dg;

// plain float4 copy (one grid-stride pass): the NVLink read vs write probe
__global__ void __launch_bounds__(256) copy4(float4* __restrict__ dst, const float4* __restrict__ src, long long n4) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += (long long)gridDim.x * 256) dst[i] = src[i];
}

int main(int argc, char** argv) {
  const long long d = argc > 1 ? atoll(argv[1]) : 125000000LL;  // params per node
  const int iters = argc > 2 ? atoi(argv[2]) : 5;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::fprintf(stderr, "needs 2 GPUs\n");
    return 2;
  }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  if (!can) {
    std::fprintf(stderr, "no peer access 0 -> 1\n");
    return 2;
  }
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  const size_t bytes = size_t(d) * sizeof(float);
  float *xr[4], *xl[4], *xrl[4], *g[4], *m[4], *v[4], *xo[4];
  CK(cudaSetDevice(1));
  for (int i = 0; i < 4; ++i) {
    CK(cudaMalloc(&xr[i], bytes));  // remote neighbours i + 4 on GPU 1
    CK(cudaMemset(xr[i], 0, bytes));
  }
  CK(cudaSetDevice(0));
  for (int i = 0; i < 4; ++i) {
    for (float** p : {&xl[i], &xrl[i], &g[i], &m[i], &v[i], &xo[i]}) {
      CK(cudaMalloc(p, bytes));
      CK(cudaMemset(*p, 0, bytes));
    }
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  DevScalars s{0.974f, 0.026f, 0.999f, 0.001f, 1.0f, 1.0f, -2e-3f, 1e-8f, 1.0f, 0.999f, 0.001f};
  int* flag = nullptr;
  CK(cudaMalloc(&flag, sizeof(int)));
  CK(cudaMemset(flag, 0x7f, sizeof(int)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  for (int remote = 1; remote >= 0; --remote) {
    float* const* other = remote ? xr : xrl;
    // ---- legacy: 4 components of one member, sources {i, i+4}
    {
      FusedArgs<1, 2> a{};
      for (int c = 0; c < 4; ++c) {
        a.src[c][0] = xl[c];
        a.src[c][1] = other[c];
        a.w[c][0][0] = a.w[c][0][1] = 0.5;
        a.ns[c] = 2;
        a.nm[c] = 1;
        a.x[c][0] = xo[c];
        a.g[c][0] = g[c];
        a.m[c][0] = m[c];
        a.v[c][0] = v[c];
      }
      a.s = s;
      a.n = d;
      a.t = 1;
      a.div_flag = flag;
      auto k = gossip_adam_fused<1, 2, 0, false>;
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, LaunchShape<1, 2>::threads, 0));
      dim3 grid(unsigned(occ * sms / 4), 4);
      k<<<grid, LaunchShape<1, 2>::threads>>>(a);  // warm-up
      CK(cudaEventRecord(e0));
      for (int it = 0; it < iters; ++it) k<<<grid, LaunchShape<1, 2>::threads>>>(a);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= iters;
      const double hbm = 4.0 * d * (28.0 + (remote ? 0.0 : 4.0)), nvl = remote ? 4.0 * d * 4.0 : 0.0;
      std::printf("legacy gossip_adam_fused<1,2> %s: %.3f ms  local HBM %.0f GB/s  NVLink %.0f GB/s\n",
                  remote ? "peer rows (NVLink)" : "local rows       ", ms, hbm / ms / 1e6, nvl / ms / 1e6);
    }
    // ---- x-sharing: one group, 4 members, rows {0,1,2,3 local, 4..7 peer}
    {
      ShArgs a{};
      ShGroup& G = a.grp[0];
      G.nl = 4;
      G.nx = 8;
      for (int r = 0; r < 4; ++r) {
        G.row[r] = xl[r];
        G.row[4 + r] = other[r];
        G.wrow[r] = G.wrow[4 + r] = 0.5;
      }
      G.local_rows = remote ? 0x0fu : 0xffu;
      for (int q = 0; q < 4; ++q) {
        G.xo[q] = xo[q];
        G.g[q] = g[q];
        G.m[q] = m[q];
        G.v[q] = v[q];
        G.deg[q] = 2;
        G.src[q][0] = (unsigned char)q;
        G.src[q][1] = (unsigned char)(4 + q);
        for (int k2 = 2; k2 < kShDeg; ++k2) G.src[q][k2] = (unsigned char)kShRows;
      }
      a.s = s;
      a.n = d;
      a.t = 1;
      a.prefetch = 1;
      a.div_flag = flag;
      auto k = gossip_adam_xshare<2, 0, false, true>;
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0));
      dim3 grid(unsigned(occ * sms), 1);
      k<<<grid, 256>>>(a);
      CK(cudaEventRecord(e0));
      for (int it = 0; it < iters; ++it) k<<<grid, 256>>>(a);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= iters;
      const double hbm = 4.0 * d * (28.0 + (remote ? 0.0 : 4.0)), nvl = remote ? 4.0 * d * 4.0 : 0.0;
      std::printf("xshare gossip_adam_xshare<2>  %s: %.3f ms  local HBM %.0f GB/s  NVLink %.0f GB/s\n",
                  remote ? "peer rows (NVLink)" : "local rows       ", ms, hbm / ms / 1e6, nvl / ms / 1e6);
    }
  }
  CK(cudaDeviceSynchronize());

  // ---- the f1 (DDP) in-place P2P range step, one node per GPU: each GPU's
  // legacy pair kernel reads its own x and the peer's publish buffer over
  // NVLink and writes x in place + its own publish copy.  Both GPUs at once
  // (bidirectional NVLink traffic, as in training) and GPU 0 alone.
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  float *ix[2], *ig[2], *im[2], *iv[2], *ipub[2][2];
  cudaStream_t st[2];
  cudaEvent_t b0[2], b1[2];
  for (int dv = 0; dv < 2; ++dv) {
    CK(cudaSetDevice(dv));
    for (float** p : {&ix[dv], &ig[dv], &im[dv], &iv[dv], &ipub[dv][0], &ipub[dv][1]}) {
      CK(cudaMalloc(p, bytes));
      CK(cudaMemset(*p, 0, bytes));
    }
    CK(cudaStreamCreateWithFlags(&st[dv], cudaStreamNonBlocking));
    CK(cudaEventCreate(&b0[dv]));
    CK(cudaEventCreate(&b1[dv]));
  }
  auto args_for = [&](int dv) {
    FusedArgs<1, 2> a{};
    const int peer = 1 - dv;
    a.src[0][dv] = ix[dv];            // ascending global id: node 0 then node 1
    a.src[0][peer] = ipub[peer][0];   // peer's x^(t-1) publish buffer (over NVLink)
    a.w[0][0][0] = a.w[0][0][1] = 0.5;
    a.ns[0] = 2;
    a.nm[0] = 1;
    a.x[0][0] = ix[dv];
    a.xp[0][0] = ipub[dv][1];
    a.g[0][0] = ig[dv];
    a.m[0][0] = im[dv];
    a.v[0][0] = iv[dv];
    a.s = s;
    a.n = d;
    a.t = 1;
    a.div_flag = flag;
    return a;
  };
  for (int both = 1; both >= 0; --both) {
    float ms[2] = {0, 0};
    for (int dv = 0; dv <= both; ++dv) {
      CK(cudaSetDevice(dv));
      auto k = gossip_adam_fused<1, 2, 0, false>;
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, LaunchShape<1, 2>::threads, 0));
      const FusedArgs<1, 2> a = args_for(dv);
      k<<<dim3(unsigned(occ * sms), 1), LaunchShape<1, 2>::threads, 0, st[dv]>>>(a);  // warm-up
    }
    for (int dv = 0; dv <= both; ++dv) {
      CK(cudaSetDevice(dv));
      CK(cudaStreamSynchronize(st[dv]));
    }
    for (int dv = 0; dv <= both; ++dv) {
      CK(cudaSetDevice(dv));
      auto k = gossip_adam_fused<1, 2, 0, false>;
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, LaunchShape<1, 2>::threads, 0));
      const FusedArgs<1, 2> a = args_for(dv);
      CK(cudaEventRecord(b0[dv], st[dv]));
      for (int it = 0; it < iters; ++it) k<<<dim3(unsigned(occ * sms), 1), LaunchShape<1, 2>::threads, 0, st[dv]>>>(a);
      CK(cudaEventRecord(b1[dv], st[dv]));
    }
    for (int dv = 0; dv <= both; ++dv) {
      CK(cudaSetDevice(dv));
      CK(cudaEventSynchronize(b1[dv]));
      CK(cudaEventElapsedTime(&ms[dv], b0[dv], b1[dv]));
      ms[dv] /= iters;
      std::printf("in-place pair kernel (+publish), %s: GPU %d %.3f ms  local HBM %.0f GB/s  NVLink %.0f GB/s\n",
                  both ? "both GPUs at once" : "GPU 0 alone      ", dv, ms[dv], 32.0 * d / ms[dv] / 1e6,
                  4.0 * d / ms[dv] / 1e6);
    }
  }
  for (int dv = 0; dv < 2; ++dv) {
    CK(cudaSetDevice(dv));
    CK(cudaDeviceSynchronize());
  }
  // ---- NVLink pull (remote reads) vs push (remote posted writes) of 0.5 GB,
  // one GPU and both GPUs at once
  for (int push = 0; push < 2; ++push)
    for (int both = 0; both < 2; ++both) {
      float ms[2] = {0, 0};
      for (int rep = 0; rep < 2; ++rep) {  // rep 0 = warm-up
        for (int dv = 0; dv <= both; ++dv) {
          CK(cudaSetDevice(dv));
          const int peer = 1 - dv;
          float4* dst = reinterpret_cast<float4*>(push ? ipub[peer][1] : ipub[dv][1]);
          const float4* src = reinterpret_cast<const float4*>(push ? ix[dv] : ipub[peer][0]);
          CK(cudaEventRecord(b0[dv], st[dv]));
          for (int it = 0; it < iters; ++it) copy4<<<unsigned(sms * 8), 256, 0, st[dv]>>>(dst, src, d / 4);
          CK(cudaEventRecord(b1[dv], st[dv]));
        }
        for (int dv = 0; dv <= both; ++dv) {
          CK(cudaSetDevice(dv));
          CK(cudaEventSynchronize(b1[dv]));
          CK(cudaEventElapsedTime(&ms[dv], b0[dv], b1[dv]));
        }
      }
      for (int dv = 0; dv <= both; ++dv)
        std::printf("NVLink %s, %s: GPU %d %.3f ms per 0.5 GB = %.0f GB/s\n", push ? "push (remote writes)" : "pull (remote reads) ",
                    both ? "both GPUs" : "one GPU  ", dv, ms[dv] / iters, 4.0 * d / (ms[dv] / iters) / 1e6);
    }
  return 0;
}
