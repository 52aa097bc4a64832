// xshare.cuh -- the default fused gossip + Adam kernel of libdg (sm_100a).
// Included by engine.cu only (legacy.cu holds the round-1 register-streaming
// and warp-specialised TMA variants, used when a round does not fit this one).
//
// DESIGN.md §3 K1.  A CTA owns a GROUP of whole mixing components (<= 8
// resident member nodes, <= 8 distinct x^(t-1) source rows); warp w is member
// w and converter of source row w (a CTA has max(members, rows) warps), and
// all warps walk the same float4 columns (lane l of every warp on column
// blockIdx.x*32 + l, grid-stride).  Per column:
//
//   1. warp w loads source row w (one 128-bit load per lane), converts the
//      4 elements to fp64 and, when every reader of the
//      row uses the same weight w_r (all built-in topologies), multiplies by
//      w_r ONCE; the 4 doubles go to a double-buffered shared-memory table
//      P[r][lane].  It also issues its own g, m, v[, acc] loads.
//   2. __syncthreads (the table is complete; the previous use of the other
//      buffer ended one barrier ago).
//   3. warp w sums P[src][lane] over its member's neighbours in ascending
//      global id (fp64, one rounding -- the oracle's op order, bit-exact),
//      applies the DAdam / AccumAdam update and stores x^(t), m, v[, acc].
//
// So every x element is loaded from HBM (or NVLink) once and converted once
// however many members mix it; the round-1 warp-per-node kernel converted it
// once per reader (6x for static exponential), which kept its XU pipe ~45 %
// busy at the HBM roofline.  Here a thread holds one member's 4-5 float4
// streams: 3 CTAs of 8 warps per SM.  Every lane prefetches its streams into
// L2 (prefetch.global.L2) DG_PREFETCH column blocks ahead, so the demand loads
// mostly hit L2: the DRAM latency is covered without registers.  Non-finite
// results are detected by an FFMA-by-zero accumulator (nan_acc), one vote per
// launch.  Measured (config 3, kernel fraction of the HBM copy): lane-0 bulk
// prefetch 0.84 -> per-lane prefetch 0.87; loading x one column block ahead
// (DG_XS_XPIPE=1) 0.78.
//
// Jacobi snapshot: every read of a column's x rows (step 1)
// precedes the barrier, every x^(t) store of that column (step 3) follows it,
// and only this CTA touches the column of the group's members (components
// are closed), so x is updated in place.  Remote readers (P2P exchange
// rounds) need x^(t) in the other buffer: xo[] then points there.
#pragma once
#include "kernels.cuh"

namespace dg {

constexpr int kShRows = 8;    // source rows per group
constexpr int kShNodes = 8;   // member nodes per group (= warps per CTA)
constexpr int kShDeg = 8;     // neighbours per member (self included)
constexpr int kShGroups = 8;  // groups per launch (blockIdx.y)

struct ShGroup {
  const float* row[kShRows];          // x^(t-1) source rows (resident, peer or recv slot)
  double wrow[kShRows];               // COLW: the weight every reader of row r uses
  float* xo[kShNodes];                // where member q's x^(t) goes
#if !DG_XS_XP_LAST
  float* xp[kShNodes][kPushMax];      // extra copies of x^(t) (publish buffer / peers' receive slots)
#endif
  const float* g[kShNodes];
  float* m[kShNodes];
  float* v[kShNodes];
  float* b[kShNodes];                 // AccumAdam accumulator (null for DAdam)
  double w[kShNodes][kShDeg];         // !COLW: member q's weight on its k-th neighbour
  unsigned char src[kShNodes][kShDeg];  // member q's k-th neighbour (ascending global id) as a row;
                                        // kShRows (the zero row) past its degree
  int deg[kShNodes];
  int nl, nx;
  unsigned local_rows;                // bit r: row r is a resident bucket (L2-prefetchable)
#if DG_XS_XP_LAST
  float* xp[kShNodes][kPushMax];      // extra copies of x^(t) (publish buffer / peers' receive slots)
#endif
};
struct ShArgs {
  ShGroup grp[kShGroups];
  DevScalars s;
  long long n;  // elements in this launch
  int t;
  int prefetch;    // column blocks prefetched into L2 ahead of use (DG_PREFETCH)
  int contiguous;  // 1: one contiguous range of column blocks per CTA (DG_XS_CONTIG)
  int* div_flag;
};

// P table: [2 buffers][kShRows + 1][2 component pairs][32 lanes] double2 (a
// warp's 128-bit accesses touch 512 consecutive bytes: conflict-free).  Row
// kShRows is all zeros: members with fewer than DEG neighbours pad their list
// with it (acc + 0.0 == acc exactly, acc starting at +0 can never be -0).
constexpr int kShRowD2 = 2 * 32;                    // double2 per row
constexpr int kShBufD2 = (kShRows + 1) * kShRowD2;  // double2 per buffer

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

#ifndef DG_XS_PF
#define DG_XS_PF 1      // per-lane prefetch.global.L2 (0: lane-0 bulk prefetch)
#endif
#ifndef DG_XS_NANACC
#define DG_XS_NANACC 1  // non-finite detection by FFMA-by-zero accumulation (0: isfinite)
#endif
#ifndef DG_XS_XPIPE
#define DG_XS_XPIPE 0   // 1: x^(t-1) rows loaded one column block ahead (measured slower: 0.78 vs 0.87)
#endif

// Measured (bench.py kernel fraction of the HBM copy, B200; sweep in
// profiles/r2_xshare_sweep.md):            config 3  config 2  static accum  AER accum
//   64-bit indices, IEEE div/sqrt calls      0.873     0.932     0.914         0.953
//   + 32-bit indices                         0.897     0.934     0.923         0.963
//   + branch-free Adam direction             0.908     0.920     0.933         0.959
// so the branch-free direction is used from 4 neighbours up (DG_XS_FASTDIV=2).
#ifndef DG_XS_FASTDIV
#define DG_XS_FASTDIV 2  // 1: branch-free 4-wide Adam direction (adam_dir4); 2: when DEG >= 4; 0: never
#endif
// x rows staged 2 column blocks ahead measured 0.908 -> 0.923 on config 3 in one sweep
// (sweep 3) but 0.905 -> 0.880 in the final build (sweep 6, same box class), so staging is
// off by default; 4 blocks 0.834; x one block ahead in registers (DG_XS_XPIPE) 0.816.
#ifndef DG_XS_STAGE
#define DG_XS_STAGE 0    // > 0: x rows staged that many column blocks ahead (cp.async ring)
#endif
#ifndef DG_XS_IDX32
#define DG_XS_IDX32 1    // 1: 32-bit column indices (the host splits launches at 2^30 elements)
#endif

#ifndef DG_XS_MINB
#define DG_XS_MINB 3  // resident CTAs per SM the register budget is sized for
#endif
// XP: members may store extra copies of x^(t) (ShGroup::xp: in-place P2P
// publish buffer or push receive slots).  A separate instantiation, so the
// plain kernel carries none of it.
template <int DEG, int ALGO, bool FOLD, bool COLW, bool XP = false>
__global__ void __launch_bounds__(32 * kShNodes, DG_XS_MINB) gossip_adam_xshare(const __grid_constant__ ShArgs a) {
  __shared__ double2 P[2 * kShBufD2];
  constexpr bool kFastDir = DG_XS_FASTDIV == 1 || (DG_XS_FASTDIV == 2 && DEG >= 4);
  const ShGroup& gp = a.grp[blockIdx.y];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nl = gp.nl, nx = gp.nx;
  const bool member = w < nl;  // warp w updates member w ...
  const bool conv = w < nx;    // ... and converts source row w
#if DG_XS_IDX32
  using idx_t = unsigned;  // a.n < 2^31 (launch_groups splits longer ranges)
#else
  using idx_t = long long;
#endif
  const idx_t nn = idx_t(a.n);
  const idx_t n4 = nn >> 2;
  // column blocks of this CTA: blk = first + i * step, i < count -- grid-stride
  // (default: at any moment the CTAs sweep one compact window of every
  // stream, so DRAM rows are used whole) or one contiguous range per CTA
  const idx_t nblk = (n4 + 31) >> 5;
  idx_t first, step, count;
  if (a.contiguous) {
    const idx_t per = (nblk + gridDim.x - 1) / gridDim.x;
    first = idx_t(blockIdx.x) * per;
    step = 1;
    count = first < nblk ? min(nblk, first + per) - first : idx_t(0);
  } else {
    first = blockIdx.x;
    step = gridDim.x;
    count = blockIdx.x < nblk ? (nblk - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  }
  const float* xr = conv ? gp.row[w] : nullptr;
  const double wr = conv && COLW ? gp.wrow[w] : 1.0;
  const bool pf_x = conv && (gp.local_rows >> w & 1);  // resident row: prefetchable into L2
  const float* gq = member ? gp.g[w] : nullptr;
  float* xq = member ? gp.xo[w] : nullptr;
  // extra x^(t) copies: pointers stay in the constant bank (read at the store)
  const bool any_xp = XP && member && (gp.xp[w][0] || gp.xp[w][1] || gp.xp[w][2] || gp.xp[w][3]);
  auto store_xp = [&](idx_t e, const float4& x) {
#pragma unroll
    for (int k = 0; k < kPushMax; ++k)
      if (gp.xp[w][k]) st4(gp.xp[w][k] + e, x);
  };
  float* mq = member ? gp.m[w] : nullptr;
  float* vq = member ? gp.v[w] : nullptr;
  float* bq = member ? gp.b[w] : nullptr;
  // member w's neighbour rows (ascending global id, zero row padded) as
  // double2 offsets into a buffer, and (!COLW) the weights
  int soff[DEG];
  double wk[COLW ? 1 : DEG];
#pragma unroll
  for (int k = 0; k < DEG; ++k) {
    soff[k] = (member ? gp.src[w][k] : kShRows) * kShRowD2 + lane;
    if (!COLW) wk[k] = member ? gp.w[w][k] : 0.0;
  }
  if (threadIdx.x < 2 * kShRowD2) {  // the zero rows of both buffers
    const int b = threadIdx.x / kShRowD2, i = threadIdx.x % kShRowD2;
    P[b * kShBufD2 + kShRows * kShRowD2 + i] = make_double2(0.0, 0.0);
  }
  // L2 prefetch of this warp's streams DG_PREFETCH column blocks ahead.
  // DG_XS_PF=1 (default): every lane prefetches its own 16 B with
  // prefetch.global.L2 (one warp instruction per stream, 4 lines).
  // DG_XS_PF=0: lane 0 issues one cp.async.bulk.prefetch.L2 per stream (the
  // operand must be uniform, so the compiler wraps each in a waterfall loop:
  // ~90 instructions per column block, measured).
  const int pd = a.prefetch;
  auto prefetch = [&](idx_t i) {
    if (i >= count) return;
#if DG_XS_PF
    const idx_t pe = (((first + i * step) << 5) + lane) << 2;
    if (pe >= nn) return;
    if (member) {
      prefetch_l2_line(gq + pe);
      prefetch_l2_line(mq + pe);
      prefetch_l2_line(vq + pe);
      if (ALGO == 1) prefetch_l2_line(bq + pe);
    }
    if (pf_x) prefetch_l2_line(xr + pe);
#else
    if (lane != 0) return;
    const idx_t e = (first + i * step) << 7;  // first element of the block
    const uint32_t bytes = uint32_t(min(idx_t(128), ((nn - e) + 3) & ~idx_t(3))) * 4u;
    if (member) {
      prefetch_l2(gq + e, bytes);
      prefetch_l2(mq + e, bytes);
      prefetch_l2(vq + e, bytes);
      if (ALGO == 1) prefetch_l2(bq + e, bytes);
    }
    if (pf_x) prefetch_l2(xr + e, bytes);
#endif
  };
  for (int i = 0; i < pd; ++i) prefetch(i);
#if DG_XS_NANACC
  float z = 0.0f;  // non-finite accumulator (nan_acc)
#endif
  bool bad = false;
  int buf = 0;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  // x^(t-1) rows staged kStage column blocks ahead with cp.async into a
  // per-lane shared-memory ring (no registers held; peer rows over NVLink
  // have microseconds to arrive).  Each lane reads back only the 16 B it
  // copied itself, so cp.async.wait_group is the only synchronisation.
  // Staging pays from 4 neighbours up (pairs measured 0.932 -> 0.89 with it).
  constexpr int kStage = DEG >= 4 ? DG_XS_STAGE : 0;
  constexpr int kSlots = kStage > 0 ? kStage + 2 : 1;
  __shared__ __align__(16) float4 XR[kShRows * kSlots * 32];
  const uint32_t xr_base = uint32_t(__cvta_generic_to_shared(&XR[(w * kSlots) * 32 + lane]));
  auto stage = [&](idx_t i) {  // issue block i of this warp's row (one commit group per block)
    if (conv && i < count) {
      const idx_t qi = ((first + i * step) << 5) + lane;
      const uint32_t dst = xr_base + uint32_t(i % kSlots) * 32u * 16u;
      const float* src = qi < n4 ? xr + (qi << 2) : xr;
      const int bytes = qi < n4 ? 16 : 0;  // zero-fill past the end
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if constexpr (kStage > 0) {
#pragma unroll
    for (int j = 0; j < kStage; ++j) stage(idx_t(j));
  }
#if DG_XS_XPIPE
  // x^(t-1) row loaded one column block ahead: the conversion below never
  // waits on DRAM, so the warps reach the barrier together
  // (addresses clamped to the last column instead of selecting zeros: a
  // select on the loaded value would wait for the load right away)
  float4 xnext = zero4;
  if (conv && count > 0) xnext = ld4(xr + (min((first << 5) + lane, n4 - 1) << 2));
#endif
  for (idx_t i = 0; i < count; ++i, buf ^= 1) {
    prefetch(i + pd);
    const idx_t q = ((first + i * step) << 5) + lane;
    const bool live = q < n4;  // false only for lanes of the last column block
    const idx_t e = q << 2;
    float4 g, m, v, bb;
    if (member && live) {
      g = ld_stream(gq + e);
      m = ld4(mq + e);
      v = ld4(vq + e);
      if (ALGO == 1) bb = ld4(bq + e);
    }
    double2* Pb = P + buf * kShBufD2;
    if constexpr (kStage > 0) {
      stage(i + kStage);
      asm volatile("cp.async.wait_group %0;" ::"n"(kStage) : "memory");  // block i has landed
    }
    if (conv) {
      float4 x;
      if constexpr (kStage > 0) {
        x = XR[(w * kSlots + int(i % kSlots)) * 32 + lane];
      } else {
#if DG_XS_XPIPE
        x = xnext;
        if (i + 1 < count) xnext = ld4(xr + (min(((first + (i + 1) * step) << 5) + lane, n4 - 1) << 2));
#else
        x = live ? ld4(xr + e) : zero4;
#endif
      }
      double2 lo, hi;
      if (COLW) {
        lo = make_double2(__dmul_rn(wr, double(x.x)), __dmul_rn(wr, double(x.y)));
        hi = make_double2(__dmul_rn(wr, double(x.z)), __dmul_rn(wr, double(x.w)));
      } else {
        lo = make_double2(double(x.x), double(x.y));
        hi = make_double2(double(x.z), double(x.w));
      }
      Pb[w * kShRowD2 + lane] = lo;
      Pb[w * kShRowD2 + 32 + lane] = hi;
    }
    __syncthreads();  // table complete; the other buffer's readers are one barrier back
    if (member && live) {
      double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
#pragma unroll
      for (int k = 0; k < DEG; ++k) {
        const double2 lo = Pb[soff[k]], hi = Pb[soff[k] + 32];
        if (COLW) {
          ax = __dadd_rn(ax, lo.x);
          ay = __dadd_rn(ay, lo.y);
          az = __dadd_rn(az, hi.x);
          aw = __dadd_rn(aw, hi.y);
        } else {
          ax = __dadd_rn(ax, __dmul_rn(wk[k], lo.x));
          ay = __dadd_rn(ay, __dmul_rn(wk[k], lo.y));
          az = __dadd_rn(az, __dmul_rn(wk[k], hi.x));
          aw = __dadd_rn(aw, __dmul_rn(wk[k], hi.y));
        }
      }
      const float4 mx = make_float4(__double2float_rn(ax), __double2float_rn(ay), __double2float_rn(az),
                                    __double2float_rn(aw));
      float4 x;
      if (ALGO == 0) {
#if DG_XS_NANACC
        if (kFastDir) {
          dadam4(mx, g, x, m, v, a.s);
        } else {
        dadam_core(mx.x, g.x, x.x, m.x, v.x, a.s);
        dadam_core(mx.y, g.y, x.y, m.y, v.y, a.s);
        dadam_core(mx.z, g.z, x.z, m.z, v.z, a.s);
        dadam_core(mx.w, g.w, x.w, m.w, v.w, a.s);
        }
        nan_acc(z, x.x, m.x, v.x);
        nan_acc(z, x.y, m.y, v.y);
        nan_acc(z, x.z, m.z, v.z);
        nan_acc(z, x.w, m.w, v.w);
#else
        bool ok = dadam_elem(mx.x, g.x, x.x, m.x, v.x, a.s);
        ok &= dadam_elem(mx.y, g.y, x.y, m.y, v.y, a.s);
        ok &= dadam_elem(mx.z, g.z, x.z, m.z, v.z, a.s);
        ok &= dadam_elem(mx.w, g.w, x.w, m.w, v.w, a.s);
        bad |= !ok;
#endif
        st4(xq + e, x);
        if constexpr (XP) {
          if (any_xp) store_xp(e, x);
        }
        st4_mv(mq + e, m);
        st4_mv(vq + e, v);
      } else {
#if DG_XS_NANACC
        if (kFastDir) {
          accum4<FOLD>(mx, g, x, m, v, bb, a.s);
        } else {
        accum_core<FOLD>(mx.x, g.x, x.x, m.x, v.x, bb.x, a.s);
        accum_core<FOLD>(mx.y, g.y, x.y, m.y, v.y, bb.y, a.s);
        accum_core<FOLD>(mx.z, g.z, x.z, m.z, v.z, bb.z, a.s);
        accum_core<FOLD>(mx.w, g.w, x.w, m.w, v.w, bb.w, a.s);
        }
        nan_acc(z, x.x, m.x, v.x);
        nan_acc(z, x.y, m.y, v.y);
        nan_acc(z, x.z, m.z, v.z);
        nan_acc(z, x.w, m.w, v.w);
#else
        bool ok = accum_elem<FOLD>(mx.x, g.x, x.x, m.x, v.x, bb.x, a.s);
        ok &= accum_elem<FOLD>(mx.y, g.y, x.y, m.y, v.y, bb.y, a.s);
        ok &= accum_elem<FOLD>(mx.z, g.z, x.z, m.z, v.z, bb.z, a.s);
        ok &= accum_elem<FOLD>(mx.w, g.w, x.w, m.w, v.w, bb.w, a.s);
        bad |= !ok;
#endif
        st4(xq + e, x);
        if constexpr (XP) {
          if (any_xp) store_xp(e, x);
        }
        st4_mv(bq + e, bb);
        if (FOLD) {
          st4_mv(mq + e, m);
          st4_mv(vq + e, v);
        }
      }
    }
  }
#if DG_XS_NANACC
  bad = z != z;
#endif
  if constexpr (kStage > 0) asm volatile("cp.async.wait_all;" ::: "memory");
  // scalar tail (n % 4 elements): CTA 0, lane l of member warp w takes element
  // n4*4 + l; all x reads precede the barrier, all writes follow it
  const idx_t tail0 = n4 << 2;
  if (blockIdx.x == 0 && tail0 < nn) {
    __syncthreads();  // the last column block's table reads are done
    const idx_t e = tail0 + lane;
    const bool t_live = idx_t(lane) < nn - tail0;
    if (conv) {
      const double xe = t_live ? double(xr[e]) : 0.0;
      P[w * kShRowD2 + lane] = make_double2(COLW ? __dmul_rn(wr, xe) : xe, 0.0);
    }
    __syncthreads();
    if (member && t_live) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < DEG; ++k) {
        const double p = P[soff[k]].x;
        acc = COLW ? __dadd_rn(acc, p) : __dadd_rn(acc, __dmul_rn(wk[k], p));
      }
      const float mx = __double2float_rn(acc);
      float x, m = mq[e], v = vq[e];
      if (ALGO == 0) {
        bad |= !dadam_elem(mx, gq[e], x, m, v, a.s);
        mq[e] = m;
        vq[e] = v;
      } else {
        float b = bq[e];
        bad |= !accum_elem<FOLD>(mx, gq[e], x, m, v, b, a.s);
        bq[e] = b;
        if (FOLD) {
          mq[e] = m;
          vq[e] = v;
        }
      }
      xq[e] = x;
      if constexpr (XP) {
        if (any_xp)
#pragma unroll
          for (int k = 0; k < kPushMax; ++k)
            if (gp.xp[w][k]) gp.xp[w][k][e] = x;
      }
    }
  }
  report_divergence(bad, a.t, a.div_flag);
}

}  // namespace dg
