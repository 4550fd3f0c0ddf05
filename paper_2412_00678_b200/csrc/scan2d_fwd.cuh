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
//    ring of `stages` rows filled with cp.async (scan2d_stage.cuh), so several
//    rows are in flight per warp without holding registers.
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

#include "scan2d_stage.cuh"

namespace s2d {

// Lane geometry shared by the forward and backward kernels.
struct LaneMap {
  int q, c, segw, lane_in_seg, gseg, cis;
  int64_t s;    // scan of this lane
  int64_t s0;   // first scan of the warp
  int wpos, c0, colc, seg_scans, ncols;
  bool scan_ok;
};

template <int LPC, int J>
__device__ __forceinline__ LaneMap lane_map(const Geo& ge, int64_t unit, int lane, int64_t S, int W) {
  LaneMap m;
  m.q = lane % LPC;
  m.c = lane / LPC;
  m.segw = 32 / ge.seg;
  m.lane_in_seg = lane & (m.segw - 1);
  m.gseg = m.c / ge.cps;
  m.cis = m.c % ge.cps;
  if (ge.seg > 1) {
    m.s0 = unit * ge.seg;
    m.s = m.s0 + m.gseg;
    m.wpos = 0;
  } else {
    m.s0 = unit / ge.wreal;
    m.s = m.s0;
    m.wpos = static_cast<int>(unit % ge.wreal);
  }
  m.scan_ok = m.s < S;
  m.c0 = m.wpos * ge.colsw;
  m.colc = m.c0 + m.cis * J;
  const int64_t left = S - m.s0;
  m.seg_scans = static_cast<int>(left < ge.seg ? left : ge.seg);
  m.ncols = min(ge.colsw, W - m.c0);
  return m;
}

template <typename T, int SPL, int LPC, int J>
__global__ void __launch_bounds__(32, 16) scan2d_fwd_kernel(const Args<T> a) {
  constexpr int CPW = 32 / LPC;
  constexpr int DPL = (J + LPC - 1) / LPC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const Geo& ge = a.plan.f;
  const int lane = threadIdx.x;
  const int H = a.H, W = a.W, N = a.N, Np = ge.Np;

  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) griddep_wait();  // the begin kernel's header writes are visible
  const uint32_t epoch = ge.wreal > 1 ? load_epoch(a.hdr) : 0u;
  if (ge.wreal > 1) {
    int t = 0;
    if (lane == 0) {
      t = atomicAdd(a.ticket, 1);
      if (t == 0) a.hdr->magic = a.magic;  // the carry region now follows this layout
    }
    unit = __shfl_sync(kFull, t, 0);
  }
  const LaneMap lm = lane_map<LPC, J>(ge, unit, lane, a.S, W);
  const int q = lm.q, cis = lm.cis, segw = lm.segw, lane_in_seg = lm.lane_in_seg;
  const int64_t sc = lm.scan_ok ? lm.s : 0;
  const int p = param_row(sc, a.S, a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const int nvalid = N - q * SPL;  // valid states of this lane's group (may be <= 0)

  T A2[SPL];
#pragma unroll
  for (int e = 0; e < SPL; ++e) {
    const int d = q * SPL + e;
    A2[e] = (lm.scan_ok && d < N) ? a.A[static_cast<int64_t>(p) * N + d] : T(0);  // natural units (exp_nat)
  }
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  // ring + copy table
  for (int e = lane; e < ge.stages * ge.stage_elems; e += 32) smem[e] = T(0);
  const StageLayout<T> Ls(ge.colsw, Np, false);
  Stager<T> stg;
  stg.xvec = a.xvec != 0;
  stg.bvec = a.bvec != 0;
  stg.zoff = Ls.zo - Ls.xo;
  stg.dyoff = 0;
  stg.coff = Ls.co - Ls.bo;
  stg.x0 = a.x + lm.s0 * HW;
  stg.z0 = a.z + lm.s0 * HW;
  stg.dy0 = nullptr;
  stg.B0 = a.B + bc_row(lm.s0, a.G) * HW * N;
  stg.C0 = a.C + bc_row(lm.s0, a.G) * HW * N;
  stg.xstride = W;
  stg.bstride = static_cast<size_t>(W) * N;
  stg.build(reinterpret_cast<CopyEntry*>(smem + ge.table_off), lane, lm.seg_scans, lm.c0, lm.ncols, N, Np,
            HW, Ls, lm.s0, a.G);
  const int nstage = ge.stages;
  // static staging: one unpacked scan per warp, 16-byte units legal
  constexpr int EPV = 16 / static_cast<int>(sizeof(T));
  constexpr int MX = (CPW * J + 32 * EPV - 1) / (32 * EPV);
  constexpr int MB = (J * SPL + EPV - 1) / EPV;
  const bool sstat = ge.seg == 1 && a.xvec && a.bvec;
  const int xunits = lm.ncols / EPV, bunits = lm.ncols * N / EPV;
  const uint32_t smem_addr = smem_u32(smem);
  auto issue_row = [&](int r, int st_) {
    if (sstat)
      stg.template issue_static<MX, MB>(smem_addr + st_ * ge.stage_elems * static_cast<int>(sizeof(T)), r, lane,
                                        xunits, bunits, Ls, false, true);
    else
      stg.issue(smem + st_ * ge.stage_elems, r, lane, false, true);
  };

  // optional emissions
  const bool save = a.ckpt != nullptr;
  const bool emit_ref = a.ph != nullptr;
  const int Tt = a.T_tile;
  const int nbm1 = a.plan.nb - 1, K = a.plan.K, Q = a.plan.Q, nq = a.plan.nq;
  // horizontal carry plumbing (tagged words, [S][nq][H][N])
  const bool has_pred = lm.wpos > 0;
  const bool has_succ = lm.wpos + 1 < ge.wreal;
  CarrySlot<T>* hc_in = has_pred ? a.hcarry + ((sc * nq + (lm.c0 / Q - 1)) * H) * N + q * SPL : nullptr;
  CarrySlot<T>* hc_out =
      has_succ ? a.hcarry + ((sc * nq + ((lm.c0 + ge.colsw) / Q - 1)) * H) * N + q * SPL : nullptr;
  // residual (plain values): the warp's outgoing carry, and the carry-in of a
  // chunk starting on an interior Q boundary
  T* hr_out = save && has_succ && lm.scan_ok ? a.hres + ((sc * nq + ((lm.c0 + ge.colsw) / Q - 1)) * H) * N + q * SPL : nullptr;
  // (segments past the last scan alias scan 0: they must not write)
  const bool chunk_q = save && lm.scan_ok && cis > 0 && (lm.colc % Q) == 0 && lm.colc < W;
  T* hr_mid = chunk_q ? a.hres + ((sc * nq + (lm.colc / Q - 1)) * H) * N + q * SPL : nullptr;
  T* yrow = a.y + sc * HW;

  T hv[J][SPL];
#pragma unroll
  for (int k = 0; k < J; ++k)
#pragma unroll
    for (int e = 0; e < SPL; ++e) hv[k][e] = T(0);

  __syncwarp();
  for (int r = 0; r < nstage - 1; ++r) {
    if (r < H) issue_row(r, r);
    cp_async_commit();
  }
  int st = 0;
  int ti = 0, ih = 0;  // row within tile / tile row (reference CarryState)
  int kb = 0, bi = 0;  // row within band / band index (residual checkpoints)
  for (int i = 0; i < H; ++i) {
    {
      const int r = i + nstage - 1;
      int sn = st + nstage - 1;
      if (sn >= nstage) sn -= nstage;
      if (r < H) issue_row(r, sn);
      cp_async_commit();
    }
    cp_async_wait_dyn(nstage - 1);
    __syncwarp();
    const T* sx = smem + st * ge.stage_elems + lm.gseg * Ls.seg_stride;
    // issue the carry-in load now; it is resolved after the row's local work
    CarryPre<T, SPL> cpre;
    const bool fast_carry = sizeof(T) == 4 && has_pred && nvalid >= SPL && (N % 2 == 0 || SPL == 1);
    if (fast_carry) carry_load<SPL>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i) * N),
                                    *reinterpret_cast<CarryPre<float, SPL>*>(&cpre));

    // ---- discretise (math.hpp:76-89): softplus once per cell, then shuffles
    T dl[DPL];
#pragma unroll
    for (int m = 0; m < DPL; ++m) {
      const int kk = q + m * LPC;
      dl[m] = kk < J ? Num<T>::softplus(sx[Ls.zo + cis * J + kk] + bias) : T(0);
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
      const T xk = sx[Ls.xo + col];
      T bq[SPL];
      lds_states<T, SPL>(bq, sx + Ls.bo + col * Np + q * SPL, true);
      const T dx = delta[k];
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        av[k][e] = Num<T>::exp_nat(dx * A2[e]);
        uv[k][e] = (dx * bq[e]) * xk;
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
      const bool act = lane_in_seg >= off;
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        Lc[e] = act ? fma(Pc[e], Lu[e], Lc[e]) : Lc[e];
        Pc[e] = act ? Pc[e] * Pu[e] : Pc[e];
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
      const int tag = row_tag(epoch, i);
      // ---- carry from the column group on the left
      if (fast_carry) {
        if constexpr (sizeof(T) == 4)
          carry_resolve<SPL>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i) * N), cpre,
                             tag, ew);
      } else if (has_pred) {
        carry_get_wait<T, SPL>(hc_in + static_cast<size_t>(i) * N, ew, tag, nvalid);
      }
      if (has_succ) {
        T out[SPL];
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          const T Pt = __shfl_sync(kFull, Pc[e], (CPW - 1) * LPC + q);
          const T Lt = __shfl_sync(kFull, Lc[e], (CPW - 1) * LPC + q);
          out[e] = fma(Pt, ew[e], Lt);
        }
        if (lm.c == CPW - 1) {
          carry_put<T, SPL>(hc_out + static_cast<size_t>(i) * N, out, tag, nvalid);
          if (hr_out != nullptr) store_states<T, SPL>(hr_out + static_cast<size_t>(i) * N, out, nvalid);
        }
      }
#pragma unroll
      for (int e = 0; e < SPL; ++e) hh[e] = fma(Pe[e], ew[e], Le[e]);
      if (chunk_q) store_states<T, SPL>(hr_mid + static_cast<size_t>(i) * N, hh, nvalid);
    }

    // ---- horizontal then vertical recurrence, C readout
    T yk[J];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const int col = cis * J + k;
      T cq[SPL];
      lds_states<T, SPL>(cq, sx + Ls.co + col * Np + q * SPL, true);
      T acc = T(0);
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        hh[e] = fma(av[k][e], hh[e], uv[k][e]);
        const T h = fma(av[k][e], hv[k][e], hh[e]);
        hv[k][e] = h;
        acc = fma(cq[e], h, acc);
      }
      yk[k] = acc;
      if (emit_ref) {  // reference CarryState (engine.cpp:188-194, :217-220)
        const int j = lm.colc + k;
        if (lm.scan_ok && j < W) {
          const int kh = (H + Tt - 1) / Tt, kw = (W + Tt - 1) / Tt;
          const size_t tile0 = (static_cast<size_t>(sc) * kh + ih) * kw + j / Tt;
          if (j % Tt == Tt - 1 || j == W - 1) {
#pragma unroll
            for (int e = 0; e < SPL; ++e)
              if (e < nvalid) a.ph[(tile0 * Tt + ti) * N + q * SPL + e] = hh[e];
          }
          if (ti == Tt - 1 || i == H - 1) {
#pragma unroll
            for (int e = 0; e < SPL; ++e)
              if (e < nvalid) a.pv[(tile0 * Tt + j % Tt) * N + q * SPL + e] = hv[k][e];
          }
        }
      }
    }
    if (save && kb == K - 1 && i < H - 1 && lm.scan_ok && nvalid > 0) {
      T* ck = a.ckpt + ((static_cast<size_t>(sc) * nbm1 + bi) * W) * N + q * SPL;
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const int j = lm.colc + k;
        if (j < W)
          stg_states<T, SPL>(ck + static_cast<size_t>(j) * N, hv[k], nvalid, nvalid >= SPL && (N % SPL) == 0);
      }
    }
    using RS_ = RS<LPC, J>;
    const int cbase = reduce_scatter<LPC, J>(yk, q);
    if ((q & (RS_::kReplica - 1)) == 0 && lm.scan_ok) {
      T* yr = yrow + static_cast<size_t>(i) * W + lm.colc + cbase;
      const T* xr = sx + Ls.xo + cis * J + cbase;
      if constexpr (RS_::kKeep >= 4 && sizeof(T) == 4) {
        if (a.yvec && lm.colc + cbase + RS_::kKeep <= W) {
#pragma unroll
          for (int m = 0; m < RS_::kKeep; m += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(xr + m);
            *reinterpret_cast<float4*>(yr + m) =
                make_float4(fmaf(Dsk, xv.x, yk[m]), fmaf(Dsk, xv.y, yk[m + 1]), fmaf(Dsk, xv.z, yk[m + 2]),
                            fmaf(Dsk, xv.w, yk[m + 3]));
          }
        } else {
#pragma unroll
          for (int m = 0; m < RS_::kKeep; ++m)
            if (lm.colc + cbase + m < W) yr[m] = fma(Dsk, xr[m], yk[m]);
        }
      } else {
#pragma unroll
        for (int m = 0; m < RS_::kKeep; ++m)
          if (lm.colc + cbase + m < W) yr[m] = fma(Dsk, xr[m], yk[m]);
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
