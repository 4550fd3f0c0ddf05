// scan2d_fwd.cuh -- forward 2D selective scan kernel (sm_100a).
//
// Replaces scan2d::tiled_scan_2d_forward (proj/src/engine.cpp:154-243).  Same
// recurrences (reference.cpp:85-112, engine.cpp:103-121, :196-216):
//   hh(i,j) = fma(Abar, hh(i,j-1), Bbar x)      horizontal, left to right
//   h(i,j)  = fma(Abar, h(i-1,j), hh(i,j))      vertical, top to bottom
//   y(i,j)  = D x + sum_d C h
//
// Work decomposition (B200-first, not the reference's T x T tile loop):
//  * One warp (= one CTA) owns `colsw` columns of one scan -- or `seg` whole
//    narrow scans -- and walks ALL rows top to bottom, so the vertical state h
//    of its columns lives in registers for the whole scan: no vertical
//    carries, no look-back, no state ever written to HBM.
//  * Row data (x, z, B, C slices) streams through a per-warp shared-memory
//    ring of `stages` rows filled with cp.async (LDGSTS), so several rows are
//    in flight per warp without holding registers.
//  * Lanes = (chunk, state group): a lane owns SPL states (float4 loads) of J
//    consecutive columns.  Per row it discretises its cells (softplus once per
//    cell, spread over the chunk's lanes and shuffled), folds the J cells into
//    one affine pair per state, and a shuffle scan over the chunks gives each
//    chunk its horizontal carry-in (the SegmentedBlockScan of PAPER.md:137;
//    segment boundaries = shuffle width when narrow scans are packed).
//  * The carry between the column groups of a wide scan goes warp to warp
//    through global memory as tagged 8-byte words (value + row tag in one
//    store: no fences on the chain).  Warps take tickets so a producer is
//    always resident before its consumer.  Only one FMA per state per row sits
//    on the chain.
//  * y = D x + sum_d C h: in-lane sum over the lane's states, then a
//    reduce-scatter over the chunk's lanes.
//  * Optional emissions: the reference CarryState (ph, pv) for any tile T,
//    and the training residual (h every K rows + the horizontal carries at
//    every Q-column boundary) consumed by the backward kernel.
#pragma once

#include "scan2d_common.cuh"

namespace s2d {

// element offsets of one pipeline stage (per segment): X | Z | [DY] | B | C
template <typename T>
struct StageLayout {
  int xo, zo, dyo, bo, co, seg_stride;
  __host__ __device__ static int pad(int n) {
    const int e = 16 / static_cast<int>(sizeof(T));
    return (n + e - 1) / e * e;
  }
  __host__ __device__ StageLayout(int colsw, int N, bool with_dy) {
    const int pc = pad(colsw), pb = pad(colsw * N);
    xo = 0;
    zo = pc;
    dyo = 2 * pc;
    bo = (with_dy ? 3 : 2) * pc;
    co = bo + pb;
    seg_stride = co + pb;
  }
  // elements per stage incl. a tail pad for over-reading vector loads
  __host__ __device__ static int stage_elems(int colsw, int N, int seg, bool with_dy) {
    StageLayout L(colsw, N, with_dy);
    return L.seg_stride * seg + pad(8);
  }
};

template <typename T, int SPL, int LPC, int J>
__global__ void __launch_bounds__(32, 16) scan2d_fwd_kernel(const Args<T> a) {
  constexpr int CPW = 32 / LPC;
  constexpr int DPL = (J + LPC - 1) / LPC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const Geo& ge = a.plan.f;
  const int lane = threadIdx.x;
  const int H = a.H, W = a.W, N = a.N;

  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    unit = __shfl_sync(kFull, t, 0);
  }
  const int q = lane % LPC;
  const int c = lane / LPC;
  const int segw = 32 / ge.seg;
  const int lane_in_seg = lane & (segw - 1);
  const int gseg = c / ge.cps;
  const int cis = c % ge.cps;
  int64_t s;
  int wpos;
  if (ge.seg > 1) {
    s = unit * ge.seg + gseg;
    wpos = 0;
  } else {
    s = unit / ge.wreal;
    wpos = static_cast<int>(unit % ge.wreal);
  }
  const bool scan_ok = s < a.S;
  const int64_t sc = scan_ok ? s : 0;
  const int c0 = wpos * ge.colsw;
  const int colc = c0 + cis * J;  // first column of this lane's chunk
  const int p = static_cast<int>(sc % a.P);
  const int64_t grp = sc / a.G;
  const size_t HW = static_cast<size_t>(H) * W;
  const bool vec = (N % SPL) == 0;

  T A2[SPL];
  bool dok[SPL];
#pragma unroll
  for (int e = 0; e < SPL; ++e) {
    const int d = q * SPL + e;
    dok[e] = scan_ok && d < N;
    A2[e] = dok[e] ? Num<T>::a_scale(a.A[static_cast<int64_t>(p) * N + d]) : T(0);
  }
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  // zero the ring once (no NaN garbage in never-written padding)
  for (int e = lane; e < ge.stages * ge.stage_elems; e += 32) smem[e] = T(0);
  __syncwarp();

  const StageLayout<T> Ls(ge.colsw, N, false);
  const int nstage = ge.stages;

  auto issue = [&](int r, int st) {
    T* dst0 = smem + static_cast<size_t>(st) * ge.stage_elems;
    for (int g = 0; g < ge.seg; ++g) {
      const int64_t sg = ge.seg > 1 ? unit * ge.seg + g : s;
      if (sg >= a.S) break;
      const int ncols = min(ge.colsw, W - c0);
      if (ncols <= 0) break;
      T* dst = dst0 + g * Ls.seg_stride;
      const size_t ro = (static_cast<size_t>(sg) * H + r) * W + c0;
      copy_span(dst + Ls.xo, a.x + ro, ncols, lane);
      copy_span(dst + Ls.zo, a.z + ro, ncols, lane);
      const size_t bo = ((static_cast<size_t>(sg / a.G) * H + r) * W + c0) * N;
      copy_span(dst + Ls.bo, a.B + bo, ncols * N, lane);
      copy_span(dst + Ls.co, a.C + bo, ncols * N, lane);
    }
  };

  // optional emissions (per-column tile geometry computed once)
  const bool save = a.ckpt != nullptr;
  const bool emit_ref = a.ph != nullptr;
  const int Tt = a.T_tile;
  const int kh = (H + Tt - 1) / Tt, kw = (W + Tt - 1) / Tt;
  const int nbm1 = a.plan.nb - 1, K = a.plan.K, Q = a.plan.Q, nq = a.plan.nq;
  unsigned last_col_mask = 0;
  int iwk[J], cck[J];
#pragma unroll
  for (int k = 0; k < J; ++k) {
    const int j = colc + k;
    iwk[k] = j / Tt;
    cck[k] = j % Tt;
    if (j < W && (cck[k] == Tt - 1 || j == W - 1)) last_col_mask |= 1u << k;
  }
  // horizontal carry plumbing (tagged words, [S][nq][H][N])
  const bool has_pred = wpos > 0;
  const bool has_succ = wpos + 1 < ge.wreal;
  CarrySlot<T>* hc_in = has_pred ? a.hcarry + ((sc * nq + (c0 / Q - 1)) * H) * N : nullptr;
  CarrySlot<T>* hc_out = has_succ ? a.hcarry + ((sc * nq + ((c0 + ge.colsw) / Q - 1)) * H) * N : nullptr;
  // chunk starts on an interior Q boundary: saved for the backward
  const bool chunk_q = save && cis > 0 && (colc % Q) == 0 && colc < W;
  CarrySlot<T>* hc_mid = chunk_q ? a.hcarry + ((sc * nq + (colc / Q - 1)) * H) * N : nullptr;

  T hv[J][SPL];
#pragma unroll
  for (int k = 0; k < J; ++k)
#pragma unroll
    for (int e = 0; e < SPL; ++e) hv[k][e] = T(0);

  for (int r = 0; r < nstage - 1; ++r) {
    if (r < H) issue(r, r);
    cp_async_commit();
  }
  int st = 0;
  int ti = 0, ih = 0;   // row within tile / tile row (reference CarryState)
  int kb = 0, bi = 0;   // row within band / band index (residual checkpoints)
  for (int i = 0; i < H; ++i) {
    {
      const int r = i + nstage - 1;
      int sn = st + nstage - 1;
      if (sn >= nstage) sn -= nstage;
      if (r < H) issue(r, sn);
      cp_async_commit();
    }
    cp_async_wait_dyn(nstage - 1);
    __syncwarp();
    const T* stg = smem + static_cast<size_t>(st) * ge.stage_elems + gseg * Ls.seg_stride;

    // ---- discretise (math.hpp:76-89)
    T dl[DPL];
#pragma unroll
    for (int m = 0; m < DPL; ++m) {
      const int kk = q + m * LPC;
      dl[m] = kk < J ? Num<T>::softplus(stg[Ls.zo + cis * J + kk] + bias) : T(0);
    }
    T delta[J];
    const int base_lane = lane & ~(LPC - 1);
#pragma unroll
    for (int k = 0; k < J; ++k) delta[k] = __shfl_sync(kFull, dl[k / LPC], base_lane + (k % LPC));

    T av[J][SPL], uv[J][SPL];
    T Pc[SPL], Lc[SPL];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const int col = cis * J + k;
      const bool okc = scan_ok && (c0 + col) < W;
      const T xk = stg[Ls.xo + col];
      T bq[SPL];
      lds_states<T, SPL>(bq, stg + Ls.bo + col * N + q * SPL, vec);
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        const bool ok = okc && dok[e];
        av[k][e] = ok ? Num<T>::exp_scaled(delta[k] * A2[e]) : T(1);
        uv[k][e] = ok ? (delta[k] * bq[e]) * xk : T(0);
        if (k == 0) {
          Pc[e] = av[k][e];
          Lc[e] = uv[k][e];
        } else {
          Lc[e] = fma(av[k][e], Lc[e], uv[k][e]);
          Pc[e] = Pc[e] * av[k][e];
        }
      }
    }
    // ---- shuffle scan over the chunks of the segment (types.hpp:121-124 compose)
#pragma unroll
    for (int off = LPC; off < 32; off <<= 1) {
      if (off >= segw) break;
      T Pu[SPL], Lu[SPL];
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        Pu[e] = __shfl_up_sync(kFull, Pc[e], off, segw);
        Lu[e] = __shfl_up_sync(kFull, Lc[e], off, segw);
      }
      if (lane_in_seg >= off) {
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          Lc[e] = fma(Pc[e], Lu[e], Lc[e]);
          Pc[e] = Pc[e] * Pu[e];
        }
      }
    }
    T hh[SPL];
    {
      T Pe[SPL], Le[SPL], ew[SPL];
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        Pe[e] = __shfl_up_sync(kFull, Pc[e], LPC, segw);
        Le[e] = __shfl_up_sync(kFull, Lc[e], LPC, segw);
        if (lane_in_seg < LPC) {
          Pe[e] = T(1);
          Le[e] = T(0);
        }
        ew[e] = T(0);
      }
      // ---- carry from the column group on the left
      if (has_pred) {
#pragma unroll
        for (int e = 0; e < SPL; ++e)
          if (dok[e]) ew[e] = CarrySlot<T>::get_wait(hc_in + static_cast<size_t>(i) * N + q * SPL + e, row_tag(a.epoch, i));
      }
      if (has_succ) {
        T out[SPL];
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          const T Pt = __shfl_sync(kFull, Pc[e], (CPW - 1) * LPC + q);
          const T Lt = __shfl_sync(kFull, Lc[e], (CPW - 1) * LPC + q);
          out[e] = fma(Pt, ew[e], Lt);
        }
        if (c == CPW - 1) {
#pragma unroll
          for (int e = 0; e < SPL; ++e)
            if (dok[e]) CarrySlot<T>::put(hc_out + static_cast<size_t>(i) * N + q * SPL + e, out[e], row_tag(a.epoch, i));
        }
      }
#pragma unroll
      for (int e = 0; e < SPL; ++e) hh[e] = fma(Pe[e], ew[e], Le[e]);
      if (chunk_q) {
#pragma unroll
        for (int e = 0; e < SPL; ++e)
          if (dok[e]) CarrySlot<T>::put(hc_mid + static_cast<size_t>(i) * N + q * SPL + e, hh[e], row_tag(a.epoch, i));
      }
    }

    // ---- horizontal then vertical recurrence, C readout
    const bool pv_row = emit_ref && (ti == Tt - 1 || i == H - 1);
    const bool ck_row = save && kb == K - 1 && i < H - 1;
    T yk[J];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const int col = cis * J + k;
      T cq[SPL];
      lds_states<T, SPL>(cq, stg + Ls.co + col * N + q * SPL, vec);
      T acc = T(0);
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        hh[e] = fma(av[k][e], hh[e], uv[k][e]);
        const T h = fma(av[k][e], hv[k][e], hh[e]);
        hv[k][e] = h;
        acc = fma(dok[e] ? cq[e] : T(0), h, acc);
      }
      yk[k] = acc;
      const int j = colc + k;
      if (emit_ref && scan_ok && j < W) {
        const size_t tile0 = (static_cast<size_t>(sc) * kh + ih) * kw + iwk[k];
        if ((last_col_mask >> k) & 1u) {
#pragma unroll
          for (int e = 0; e < SPL; ++e)
            if (dok[e]) a.ph[(tile0 * Tt + ti) * N + q * SPL + e] = hh[e];
        }
        if (pv_row) {
#pragma unroll
          for (int e = 0; e < SPL; ++e)
            if (dok[e]) a.pv[(tile0 * Tt + cck[k]) * N + q * SPL + e] = hv[k][e];
        }
      }
      if (ck_row && scan_ok && j < W && q * SPL < N)
        stg_states<T, SPL>(a.ckpt + ((static_cast<size_t>(sc) * nbm1 + bi) * W + j) * N + q * SPL, hv[k],
                           N - q * SPL, vec);
    }
    using RS_ = RS<LPC, J>;
    const int cbase = reduce_scatter<LPC, J>(yk, q);
    if ((q & (RS_::kReplica - 1)) == 0 && scan_ok) {
      T* yrow = a.y + sc * HW + static_cast<size_t>(i) * W;
#pragma unroll
      for (int m = 0; m < RS_::kKeep; ++m) {
        const int k = cbase + m;
        const int j = colc + k;
        if (j < W) yrow[j] = fma(Dsk, stg[Ls.xo + cis * J + k], yk[m]);
      }
    }
    __syncwarp();
    if (++st == nstage) st = 0;
    if (++ti == Tt) {
      ti = 0;
      ++ih;
    }
    if (++kb == K) {
      kb = 0;
      ++bi;
    }
  }
}

}  // namespace s2d
