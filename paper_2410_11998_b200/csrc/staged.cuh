// staged.cuh -- the default fused gossip + Adam kernel of libdg (sm_100a):
// TMA bulk-copy staging of every mixed x^(t-1) bucket and each node's g, m, v
// rows into a shared-memory ring, one warp per resident node.  Included by
// engine.cu only (legacy.cu holds the round-1 variants).
#pragma once
#include "kernels.cuh"

namespace dg {

// ------------------------------------------------------------------ shared-memory staged kernel
// The default fused kernel (DESIGN.md §3 K1).  One CTA = one warp per resident
// node; the CTA walks column tiles of TW float4 columns.  Every x^(t-1) bucket
// the round mixes (resident rows and remote rows: NVLink peer buckets or recv
// slots) is staged ONCE per tile in shared memory, together with each node's
// g, m, v[, acc] rows, by 1-D bulk async copies (TMA, cp.async.bulk, completion
// counted on the stage's mbarrier), S-1 tiles ahead of the tile being computed.
// Lane 0 of warp w issues the copies of node w's own rows and of x rows
// w, w + nl, ...; no thread spends instructions or registers on addresses or
// in-flight data, so the issue slots go to the arithmetic (fp64 mixing, IEEE
// div/sqrt).  Warp w forms node w's mixed sum from the staged rows (ascending
// global source id, fp64, one rounding), applies the Adam update and stores
// x^(t), m, v[, acc] straight to HBM.  Every neighbour line crosses DRAM (or
// NVLink) once per tile however many resident nodes mix it.
//
// Jacobi snapshot: a tile's columns of every resident node are
// handled by one CTA and all of its x rows have landed in shared memory (the
// stage's mbarrier phase completed) before any warp stores x^(t) of that tile,
// so x is updated in place.  Remote readers (P2P exchange rounds) need x^(t)
// in the other buffer: xo[] then points there (the host decides).
constexpr int kStMaxRows = 48;   // staged x rows per tile (resident + remote sources)
constexpr int kStMaxNodes = 16;  // resident nodes (warps per CTA)
constexpr int kMaxDegDev = 16;   // neighbours per node, self included (dg_internal.hpp kMaxDeg)
constexpr int kStMaxStages = 4;
struct StagedArgs {
  const float* xsrc[kStMaxRows];       // x^(t-1) rows at this launch's offset: [0,nl) resident, then remote
  float* xo[kStMaxNodes];              // where node w's x^(t) goes
  const float* g[kStMaxNodes];
  float* m[kStMaxNodes];
  float* v[kStMaxNodes];
  float* b[kStMaxNodes];               // AccumAdam accumulator (null for DAdam)
  double w[kStMaxNodes][kMaxDegDev];   // node w's weights, ascending global neighbour id
  unsigned char src[kStMaxNodes][kMaxDegDev];  // staged row of each neighbour
  int deg[kStMaxNodes];
  int nl, nx;                          // resident nodes, staged x rows
  int tw_shift;                        // float4 columns per tile = 32 << tw_shift
  DevScalars s;
  long long n;                         // elements in this launch
  int t;
  int* div_flag;
};

template <int ALGO, bool FOLD, int S>
__global__ void __launch_bounds__(512, 2) gossip_adam_staged(const __grid_constant__ StagedArgs a) {
  constexpr int K = ALGO == 1 ? 4 : 3;  // own rows per node: g, m, v[, acc]
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);       // one mbarrier per stage
  float4* sm = reinterpret_cast<float4*>(smraw + 128);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nl = a.nl, nx = a.nx, TWS = 5 + a.tw_shift, TW = 1 << TWS;
  const long long n4 = a.n >> 2;
  const long long tiles = (n4 + TW - 1) / TW;
  const long long mine = blockIdx.x < tiles ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int stage_f4 = (nx + K * nl) * TW;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], nl);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // lane 0 of warp w: node w's own rows and x rows w, w + nl, ... of local tile i
  auto issue = [&](long long i) {
    const long long c0 = (blockIdx.x + i * gridDim.x) * TW;
    const uint32_t bytes = uint32_t(min((long long)TW, n4 - c0)) * 16u;
    const int s = int(i % S);
    float4* st = sm + s * stage_f4;
    int rows = K;
    for (int r = w; r < nx; r += nl) ++rows;
    mbar_expect_tx(&full[s], bytes * rows);
    for (int r = w; r < nx; r += nl) tma_load_1d(st + r * TW, a.xsrc[r] + (c0 << 2), bytes, &full[s]);
    float4* ow = st + (nx + w * K) * TW;
    tma_load_1d(ow, a.g[w] + (c0 << 2), bytes, &full[s]);
    tma_load_1d(ow + TW, a.m[w] + (c0 << 2), bytes, &full[s]);
    tma_load_1d(ow + 2 * TW, a.v[w] + (c0 << 2), bytes, &full[s]);
    if constexpr (K == 4) tma_load_1d(ow + 3 * TW, a.b[w] + (c0 << 2), bytes, &full[s]);
  };

  const int deg = a.deg[w];
  bool bad = false;
  if (lane == 0)
    for (int i = 0; i < S - 1 && i < mine; ++i) issue(i);
  for (long long i = 0; i < mine; ++i) {
    const int s = int(i % S);
    mbar_wait(&full[s], uint32_t((i / S) & 1));  // every row of tile i has landed
    const long long c0 = (blockIdx.x + i * gridDim.x) * TW;
    const float4* st = sm + s * stage_f4;
    for (int c = lane; c < TW; c += 32) {
      const long long q = c0 + c;
      if (q >= n4) break;
      double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
      for (int k = 0; k < deg; ++k) {
        const double wt = a.w[w][k];
        const float4 xv = st[a.src[w][k] * TW + c];
        ax = mix_acc(ax, wt, xv.x);
        ay = mix_acc(ay, wt, xv.y);
        az = mix_acc(az, wt, xv.z);
        aw = mix_acc(aw, wt, xv.w);
      }
      const float4 mx = make_float4(__double2float_rn(ax), __double2float_rn(ay), __double2float_rn(az),
                                    __double2float_rn(aw));
      const float4* ow = st + (nx + w * K) * TW + c;
      const float4 g = ow[0];
      float4 m = ow[TW], v = ow[2 * TW], x;
      const long long e = q << 2;
      if (ALGO == 0) {
        bool ok = dadam_elem(mx.x, g.x, x.x, m.x, v.x, a.s);
        ok &= dadam_elem(mx.y, g.y, x.y, m.y, v.y, a.s);
        ok &= dadam_elem(mx.z, g.z, x.z, m.z, v.z, a.s);
        ok &= dadam_elem(mx.w, g.w, x.w, m.w, v.w, a.s);
        bad |= !ok;
        st4(a.xo[w] + e, x);
        st4_mv(a.m[w] + e, m);
        st4_mv(a.v[w] + e, v);
      } else {
        float4 b = ow[3 * TW];
        bool ok = accum_elem<FOLD>(mx.x, g.x, x.x, m.x, v.x, b.x, a.s);
        ok &= accum_elem<FOLD>(mx.y, g.y, x.y, m.y, v.y, b.y, a.s);
        ok &= accum_elem<FOLD>(mx.z, g.z, x.z, m.z, v.z, b.z, a.s);
        ok &= accum_elem<FOLD>(mx.w, g.w, x.w, m.w, v.w, b.w, a.s);
        bad |= !ok;
        st4(a.xo[w] + e, x);
        st4_mv(a.b[w] + e, b);
        if (FOLD) {
          st4_mv(a.m[w] + e, m);
          st4_mv(a.v[w] + e, v);
        }
      }
    }
    __syncthreads();  // every warp is done with stage s: refill it with tile i + S
    if (lane == 0 && i + S < mine) issue(i + S);
  }
  // scalar tail (n % 4 elements) in CTA 0: every read of the tail columns
  // precedes the barrier, every write follows it (in-place Jacobi snapshot)
  const long long tail0 = n4 << 2;
  if (blockIdx.x == 0 && tail0 < a.n) {
    const long long e = tail0 + lane;
    const bool live = lane < a.n - tail0;
    float x = 0.f, m = 0.f, v = 0.f, b = 0.f;
    bool ok = true;
    if (live) {
      double acc = 0.0;
      for (int k = 0; k < deg; ++k) acc = mix_acc(acc, a.w[w][k], a.xsrc[a.src[w][k]][e]);
      m = a.m[w][e];
      v = a.v[w][e];
      if (ALGO == 0) {
        ok = dadam_elem(__double2float_rn(acc), a.g[w][e], x, m, v, a.s);
      } else {
        b = a.b[w][e];
        ok = accum_elem<FOLD>(__double2float_rn(acc), a.g[w][e], x, m, v, b, a.s);
      }
    }
    __syncthreads();
    if (live) {
      bad |= !ok;
      a.xo[w][e] = x;
      if (ALGO == 0 || FOLD) {
        a.m[w][e] = m;
        a.v[w][e] = v;
      }
      if (ALGO == 1) a.b[w][e] = b;
    }
  }
  report_divergence(bad, a.t, a.div_flag);
}

}  // namespace dg
