// scan2d_fwd.cuh -- forward 2D selective scan kernel (sm_100a).
//
// Replaces scan2d::tiled_scan_2d_forward (proj/src/engine.cpp:154-243).  Same
// recurrences (reference.cpp:85-112, engine.cpp:103-121, :196-216):
//   hh(i,j) = fma(Abar, hh(i,j-1), Bbar x)      horizontal, left to right
//   h(i,j)  = fma(Abar, h(i-1,j), hh(i,j))      vertical, top to bottom
//   y(i,j)  = D x + sum_d C h
//
// Work decomposition (B200-first, not the reference's T x T tile loop):
//  * A warp owns a column group of one scan (or `seg` whole scans when the grid
//    is narrow) and walks ALL rows top to bottom, so the vertical state h of
//    its columns never leaves registers: no vertical carries, no look-back.
//  * Lanes = (chunk, state): lane l of a chunk owns state d = l for J
//    consecutive columns.  Per row a lane discretises its J cells
//    (softplus once per cell, spread over the chunk's lanes and shuffled),
//    folds them into one (a, b) pair, and a shuffle scan over the chunks of
//    the warp gives each chunk its horizontal carry-in (the SegmentedBlockScan
//    of PAPER.md:137; segment boundaries = shuffle width when scans are packed).
//  * The horizontal carry between the column groups of a wide scan flows warp
//    to warp through a shared-memory ring guarded by mbarriers, and CTA to CTA
//    through global memory (release/acquire progress counters; CTAs take
//    tickets so a producer is always resident before its consumer).  Only one
//    FMA per state sits on that chain per row; everything else overlaps.
//  * y = D x + sum_d C h is a reduce-scatter over the chunk's state lanes.
//  * Optional emissions: the reference CarryState (ph, pv) for any tile T,
//    and the training residual (h checkpoints every K rows + the CTA-boundary
//    horizontal carries) consumed by the backward kernel.
#pragma once

#include "scan2d_common.cuh"

namespace s2d {

template <typename T>
struct Ring {
  T data[kRing][32];
  uint64_t full[kRing];
  uint64_t empty[kRing];
};

template <typename T, int LPC, int J>
struct RowIn {
  static constexpr int DPL = (J + LPC - 1) / LPC;  // cells whose softplus this lane computes
  T x[J];
  T b[J];
  T c[J];
  T zz[DPL];
};

// Per-lane geometry shared by the forward and backward kernels.
struct LaneGeo {
  int64_t s;     // scan index
  int wpos;      // warp position within the scan's width
  int col0;      // first column of this lane's chunk
  int l;         // state lane
  int chunk;     // chunk within the warp
  int lane_in_seg;
  int segw;      // lanes per segment (shuffle width)
  bool scan_ok;  // s < S
  bool st_ok;    // scan_ok && l < N
};

template <int LPC, int J>
__device__ __forceinline__ bool lane_geometry(const Plan& pl, int64_t S, int64_t unit, int lane,
                                              LaneGeo& g) {
  g.l = lane & (LPC - 1);
  g.chunk = lane / LPC;
  g.segw = 32 / pl.seg;
  g.lane_in_seg = lane & (g.segw - 1);
  int cis;
  if (pl.seg > 1) {
    const int segi = g.chunk / pl.cps;
    g.s = unit * pl.seg + segi;
    g.wpos = 0;
    cis = g.chunk % pl.cps;
  } else {
    g.s = unit / pl.wps;
    g.wpos = static_cast<int>(unit % pl.wps);
    cis = g.chunk;
  }
  g.col0 = g.wpos * pl.colsw + cis * J;
  g.scan_ok = g.s < S;
  return g.wpos < pl.wreal;  // false: padding warp without real columns
}

template <typename T, int LPC, int J>
__device__ __forceinline__ void load_row(RowIn<T, LPC, J>& r, const T* __restrict__ xs,
                                         const T* __restrict__ zs, const T* __restrict__ Bs,
                                         const T* __restrict__ Cs, int i, int W, int N,
                                         const LaneGeo& g) {
  const size_t base = static_cast<size_t>(i) * W;
#pragma unroll
  for (int k = 0; k < J; ++k) {
    const int j = g.col0 + k;
    const bool ok = g.scan_ok && j < W;
    r.x[k] = ok ? __ldg(xs + base + j) : T(0);
    const bool okd = ok && g.l < N;
    const size_t e = (base + j) * N + g.l;
    r.b[k] = okd ? __ldg(Bs + e) : T(0);
    r.c[k] = okd ? __ldg(Cs + e) : T(0);
  }
#pragma unroll
  for (int m = 0; m < RowIn<T, LPC, J>::DPL; ++m) {
    const int kk = g.l + m * LPC;
    const int j = g.col0 + kk;
    const bool ok = g.scan_ok && kk < J && j < W;
    r.zz[m] = ok ? __ldg(zs + base + j) : T(0);
  }
}

// delta for the J cells of the lane's chunk: each softplus is evaluated once
// per cell (spread over the chunk's lanes) and broadcast with shuffles.
template <typename T, int LPC, int J>
__device__ __forceinline__ void chunk_delta(const RowIn<T, LPC, J>& r, T bias, int lane,
                                            T (&delta)[J]) {
  constexpr int DPL = RowIn<T, LPC, J>::DPL;
  T dl[DPL];
#pragma unroll
  for (int m = 0; m < DPL; ++m) dl[m] = Num<T>::softplus(r.zz[m] + bias);
  const int base_lane = lane & ~(LPC - 1);
#pragma unroll
  for (int k = 0; k < J; ++k) delta[k] = __shfl_sync(kFull, dl[k / LPC], base_lane + (k % LPC));
}

// Inclusive scan of (P, L) affine pairs over the chunks of a segment, left to
// right: compose(first, second) = (P2 P1, fma(P2, L1, L2)) (types.hpp:121-124).
template <typename T, int LPC>
__device__ __forceinline__ void chunk_scan_fwd(T& P, T& L, int lane_in_seg, int span, int segw) {
#pragma unroll
  for (int off = LPC; off < 32; off <<= 1) {
    if (off >= span) break;
    const T Pu = __shfl_up_sync(kFull, P, off, segw);
    const T Lu = __shfl_up_sync(kFull, L, off, segw);
    if (lane_in_seg >= off) {
      L = fma(P, Lu, L);
      P = P * Pu;
    }
  }
}

template <typename T, int LPC, int J>
__global__ void __launch_bounds__(512) scan2d_fwd_kernel(const Args<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Ring<T>* rings = reinterpret_cast<Ring<T>*>(smem);
  const Plan& pl = a.plan;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  __shared__ int s_cta;
  if (threadIdx.x == 0) s_cta = pl.ncb > 1 ? atomicAdd(a.flags, 1) : static_cast<int>(blockIdx.x);
  for (int q = threadIdx.x; q < pl.nw * kRing; q += blockDim.x) {
    mbar_init(&rings[q / kRing].full[q % kRing], 32);
    mbar_init(&rings[q / kRing].empty[q % kRing], 32);
  }
  __syncthreads();
  const int64_t cta = s_cta;
  const int64_t unit = cta * pl.nw + warp;
  if (unit >= pl.units) return;
  LaneGeo g;
  if (!lane_geometry<LPC, J>(pl, a.S, unit, lane, g)) return;

  const int H = a.H, W = a.W, N = a.N;
  const int cb = g.wpos / pl.nw;  // CTA index across the scan's width
  const bool has_pred = g.wpos > 0;
  const bool has_succ = g.wpos + 1 < pl.wreal;
  const bool pred_global = has_pred && warp == 0;
  const bool succ_global = has_succ && warp == pl.nw - 1;
  g.st_ok = g.scan_ok && g.l < N;

  const int64_t s = g.scan_ok ? g.s : 0;
  const int64_t p = s % a.P, grp = s / a.G;
  const size_t HW = static_cast<size_t>(H) * W;
  const T Ad = g.st_ok ? a.A[p * N + g.l] : T(0);
  const T A2 = Num<T>::a_scale(Ad);
  const T Dsk = a.Dskip[p], bias = a.bias[p];
  const T* xs = a.x + s * HW;
  const T* zs = a.z + s * HW;
  const T* Bs = a.B + grp * HW * N;
  const T* Cs = a.C + grp * HW * N;
  T* ys = a.y + s * HW;

  // optional emission geometry
  const int Tt = a.T_tile;
  const int kh = (H + Tt - 1) / Tt, kw = (W + Tt - 1) / Tt;
  const int nbm1 = pl.nb - 1;
  const int ncbm1 = pl.ncb - 1;
  int* prog_in = pred_global ? a.flags + 1 + s * ncbm1 + (cb - 1) : nullptr;
  int* prog_out = succ_global ? a.flags + 1 + s * ncbm1 + cb : nullptr;
  const T* hc_in = pred_global ? a.hcarry + ((s * ncbm1 + (cb - 1)) * H) * N : nullptr;
  T* hc_out = succ_global ? a.hcarry + ((s * ncbm1 + cb) * H) * N : nullptr;
  int seen = 0;  // last observed progress of the global predecessor

  using RS_ = RS<LPC, J>;
  T hv[J];
#pragma unroll
  for (int k = 0; k < J; ++k) hv[k] = T(0);

  RowIn<T, LPC, J> cur, nxt;
  load_row<T, LPC, J>(cur, xs, zs, Bs, Cs, 0, W, N, g);

  for (int i = 0; i < H; ++i) {
    if (i + 1 < H) load_row<T, LPC, J>(nxt, xs, zs, Bs, Cs, i + 1, W, N, g);

    // ---- discretise (math.hpp:76-89) and fold the chunk into one affine pair
    T delta[J], av[J], uv[J];
    chunk_delta<T, LPC, J>(cur, bias, lane, delta);
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const bool ok = g.scan_ok && (g.col0 + k) < W;
      av[k] = ok ? Num<T>::exp_scaled(delta[k] * A2) : T(1);
      uv[k] = (delta[k] * cur.b[k]) * cur.x[k];
    }
    T Pc = av[0], Lc = uv[0];
#pragma unroll
    for (int k = 1; k < J; ++k) {
      Lc = fma(av[k], Lc, uv[k]);
      Pc = Pc * av[k];
    }
    // ---- shuffle scan over the chunks of the segment
    T Pi = Pc, Li = Lc;
    chunk_scan_fwd<T, LPC>(Pi, Li, g.lane_in_seg, pl.cps * LPC, g.segw);
    T Pe = __shfl_up_sync(kFull, Pi, LPC, g.segw);
    T Le = __shfl_up_sync(kFull, Li, LPC, g.segw);
    if (g.lane_in_seg < LPC) {
      Pe = T(1);
      Le = T(0);
    }

    // ---- carry from the column group on the left
    T ew = T(0);
    const int slot = i % kRing;
    const uint32_t par = static_cast<uint32_t>(i / kRing) & 1u;
    if (has_pred) {
      if (!pred_global) {
        Ring<T>& r = rings[warp];
        mbar_wait(&r.full[slot], par);
        ew = r.data[slot][g.l];
        mbar_arrive(&r.empty[slot]);
      } else {
        if (seen <= i) seen = wait_flag_gt(prog_in, i);
        ew = g.l < N ? ld_relaxed_gpu(hc_in + static_cast<size_t>(i) * N + g.l) : T(0);
      }
    }
    if (has_succ) {
      // warp aggregate lives in the last chunk's lanes; one FMA on the chain
      const T Pt = __shfl_sync(kFull, Pi, (pl.cpw - 1) * LPC + g.l);
      const T Lt = __shfl_sync(kFull, Li, (pl.cpw - 1) * LPC + g.l);
      const T out = fma(Pt, ew, Lt);
      if (!succ_global) {
        Ring<T>& r = rings[warp + 1];
        mbar_wait(&r.empty[slot], par ^ 1u);
        if (g.chunk == 0) r.data[slot][g.l] = out;
        mbar_arrive(&r.full[slot]);
      } else {
        if (g.chunk == 0 && g.l < N) {
          hc_out[static_cast<size_t>(i) * N + g.l] = out;
          __threadfence();
        }
        __syncwarp();
        if (lane == 0) st_release_gpu(prog_out, i + 1);
      }
    }
    T hh = fma(Pe, ew, Le);

    // ---- horizontal then vertical recurrence, C readout
    const bool pv_row = (a.pv != nullptr) && ((i % Tt) == Tt - 1 || i == H - 1);
    const bool ck_row = (a.ckpt != nullptr) && ((i % pl.K) == pl.K - 1) && (i < H - 1);
    T prod[J];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      hh = fma(av[k], hh, uv[k]);
      const T h = fma(av[k], hv[k], hh);
      hv[k] = h;
      prod[k] = cur.c[k] * h;
      const int j = g.col0 + k;
      if (g.st_ok && j < W) {
        if (a.ph != nullptr && ((j % Tt) == Tt - 1 || j == W - 1)) {
          const size_t slotp = (static_cast<size_t>(s * kh + i / Tt) * kw + j / Tt) * Tt;
          a.ph[(slotp + i % Tt) * N + g.l] = hh;
        }
        if (pv_row) {
          const size_t slotp = (static_cast<size_t>(s * kh + i / Tt) * kw + j / Tt) * Tt;
          a.pv[(slotp + j % Tt) * N + g.l] = h;
        }
        if (ck_row) a.ckpt[((static_cast<size_t>(s) * nbm1 + i / pl.K) * W + j) * N + g.l] = h;
      }
    }
    const int cbase = reduce_scatter<LPC, J>(prod, g.l);
    if ((g.l & (RS_::kReplica - 1)) == 0 && g.scan_ok) {
#pragma unroll
      for (int m = 0; m < RS_::kKeep; ++m) {
        const int k = cbase + m;
        const int j = g.col0 + k;
        if (j < W) ys[static_cast<size_t>(i) * W + j] = fma(Dsk, select_col<J>(cur.x, k), prod[m]);
      }
    }
    if (i + 1 < H) cur = nxt;
  }
}

}  // namespace s2d
