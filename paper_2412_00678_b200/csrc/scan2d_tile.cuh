// scan2d_tile.cuh -- "tile-transpose" forward kernel for N >= 4 (sm_100a).
//
// Same recurrences as scan2d_fwd.cuh (reference.cpp:85-112):
//   hh(i,j) = fma(Abar, hh(i,j-1), Bbar x)      h(i,j) = fma(Abar, h(i-1,j), hh(i,j))
//   y(i,j)  = D x + sum_d C h
// but organised so that neither scan needs shuffles:
//  * one warp owns a STRIP of CW columns of one scan and walks it in tiles of
//    R rows (R * N/4 = 32: R = 8 rows for N = 16);
//  * phase 1 (row lanes): lane (r, q) owns row r of the tile and states
//    4q..4q+3; it walks the CW columns left to right with the horizontal
//    carry in registers (4 independent FMA chains) and writes hh to shared
//    memory.  The strip's carry-in per row comes from the strip on the left
//    (tagged words in global memory, one hop per tile);
//  * phase 2 (column lanes): lane (j, s) owns column j and N/QV states; it
//    walks the R rows top to bottom with the vertical state h in registers
//    for the whole scan, reads hh back, and folds C h into y (one xor shuffle
//    when a column is split over QV = 32/CW lanes).
// Shared-memory rows are padded so that both the row-lane and the
// column-lane access patterns are bank-conflict free.  Tiles stream through a
// cp.async ring (2-3 tiles), copied with 16-byte units and immediate offsets.
#pragma once

#include "scan2d_fwd.cuh"

namespace s2d {

template <typename T, int N, int CW, int SH = 4>
struct TileShape {
  static constexpr int QH = N / SH;           // row lanes per row (SH states each)
  static constexpr int R = 32 / QH;           // rows per tile
  static constexpr int QV = 32 / CW;          // column lanes per column
  static constexpr int SV = N / QV;           // states per column lane
  static constexpr int PAD = N;               // row padding of the [R][CW][N] blocks (floats):
                                              // rows of one access group land on distinct banks
  static constexpr int BP = CW * N + PAD;     // padded row pitch of B / C / HH
  static constexpr int XP = CW;               // row pitch of X / Z / DL
  // stage: X[R][XP] Z[R][XP] B[R][BP] C[R][BP]
  static constexpr int XO = 0, ZO = R * XP, BO = 2 * R * XP, CO = BO + R * BP;
  static constexpr int STAGE = CO + R * BP;
  // hh is written in place over B (same lane reads B then writes hh), delta in
  // place over Z: no scratch beyond the stages
  static constexpr int SCRATCH = 0;
  static constexpr int EPV = 16 / sizeof(T);
  static constexpr int XU = R * CW / EPV;         // 16-byte units of one X (or Z) tile
  static constexpr int BU = R * CW * N / EPV;     // 16-byte units of one B (or C) tile
  static constexpr int XUL = (XU + 31) / 32;      // per lane
  static constexpr int BUL = (BU + 31) / 32;
  static constexpr int BUR = CW * N / EPV;        // units per row of B
  static_assert(QH >= 1 && R >= 1 && QV >= 1 && SV >= 1, "bad tile shape");
};

template <typename T, int N, int CW, int SH>
__global__ void __launch_bounds__(32, 8) scan2d_fwd_tile_kernel(const Args<T> a) {
  using TS = TileShape<T, N, CW, SH>;
  constexpr int R = TS::R, QH = TS::QH, QV = TS::QV, SV = TS::SV, EPV = TS::EPV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const Geo& ge = a.plan.f;
  const int lane = threadIdx.x;
  const int H = a.H, W = a.W;
  const int nstage = ge.stages;

  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    unit = __shfl_sync(kFull, t, 0);
  }
  const int64_t s = unit / ge.wreal;
  const int wpos = static_cast<int>(unit % ge.wreal);
  const int c0 = wpos * CW;
  const int ncols = min(CW, W - c0);
  const int p = static_cast<int>(s % a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  // phase-1 identity: row r1, states SH*q1 .. SH*q1+SH-1
  const int r1 = lane / QH, q1 = lane % QH;
  // phase-2 identity: column j2, states s2*SV .. s2*SV+SV-1
  const int j2 = lane / QV, s2 = lane % QV;
  T A1[SH], A2v[SV];
#pragma unroll
  for (int e = 0; e < SH; ++e) A1[e] = Num<T>::a_scale(a.A[static_cast<int64_t>(p) * N + q1 * SH + e]);
#pragma unroll
  for (int e = 0; e < SV; ++e) A2v[e] = Num<T>::a_scale(a.A[static_cast<int64_t>(p) * N + s2 * SV + e]);

  for (int e = lane; e < nstage * TS::STAGE; e += 32) smem[e] = T(0);
  __syncwarp();

  // ---- tile copies (rows r0 .. r0+R-1, columns c0 .. c0+ncols-1)
  const T* xg = a.x + s * HW + c0;
  const T* zg = a.z + s * HW + c0;
  const T* Bg = a.B + (s / a.G) * HW * N + static_cast<size_t>(c0) * N;
  const T* Cg = a.C + (s / a.G) * HW * N + static_cast<size_t>(c0) * N;
  const int xunits_row = ncols / EPV, bunits_row = ncols * N / EPV;
  const size_t WN = static_cast<size_t>(W) * N;
  const uint32_t sbase = smem_u32(smem);
  auto issue_tile = [&](int r0, int st) {
    const uint32_t sb = sbase + st * TS::STAGE * static_cast<int>(sizeof(T));
    constexpr int XR = CW / EPV;  // x units per row
#pragma unroll
    for (int m = 0; m < TS::XUL; ++m) {
      const int u = lane + 32 * m;
      const int rr = u / XR, cu = u % XR;
      if (u < TS::XU && cu < xunits_row && r0 + rr < H) {
        const size_t go = static_cast<size_t>(r0 + rr) * W + cu * EPV;
        const uint32_t so = (rr * TS::XP + cu * EPV) * sizeof(T);
        cp_async16_raw(sb + (TS::XO * sizeof(T)) + so, xg + go);
        cp_async16_raw(sb + (TS::ZO * sizeof(T)) + so, zg + go);
      }
    }
    const T* bt = Bg + static_cast<size_t>(r0) * WN;
    const T* ct = Cg + static_cast<size_t>(r0) * WN;
#pragma unroll
    for (int m = 0; m < TS::BUL; ++m) {
      int rr, cu;
      if constexpr (TS::BUR % 32 == 0) {
        rr = (32 * m) / TS::BUR;
        cu = (32 * m) % TS::BUR + lane;
      } else {
        const int u = lane + 32 * m;
        rr = u / TS::BUR;
        cu = u % TS::BUR;
      }
      if (cu < bunits_row && r0 + rr < H) {
        const size_t go = rr * WN + cu * EPV;
        const uint32_t so = (rr * TS::BP + cu * EPV) * sizeof(T);
        cp_async16_raw(sb + (TS::BO * sizeof(T)) + so, bt + go);
        cp_async16_raw(sb + (TS::CO * sizeof(T)) + so, ct + go);
      }
    }
  };

  // ---- carries (tagged words [S][nq][H][N]); strips are the Q grid (Q == CW)
  const bool save = a.ckpt != nullptr;
  const int nq = a.plan.nq, K = a.plan.K, nbm1 = a.plan.nb - 1;
  const bool has_pred = wpos > 0, has_succ = wpos + 1 < ge.wreal;
  const CarrySlot<T>* hc_in = has_pred ? a.hcarry + ((s * nq + (wpos - 1)) * H) * N + q1 * SH : nullptr;
  CarrySlot<T>* hc_out = has_succ ? a.hcarry + ((s * nq + wpos) * H) * N + q1 * SH : nullptr;
  const bool emit_ref = a.ph != nullptr;
  const int Tt = a.T_tile;
  const int kh = (H + Tt - 1) / Tt, kw = (W + Tt - 1) / Tt;

  T hv[SV];
#pragma unroll
  for (int e = 0; e < SV; ++e) hv[e] = T(0);

  const int ntiles = (H + R - 1) / R;
  int kb = 0, bi = 0;  // row within band / band index (residual checkpoints)
  for (int t = 0; t < nstage - 1; ++t) {
    if (t < ntiles) issue_tile(t * R, t);
    cp_async_commit();
  }
  int st = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int r0 = t * R;
    {
      const int tn = t + nstage - 1;
      int sn = st + nstage - 1;
      if (sn >= nstage) sn -= nstage;
      if (tn < ntiles) issue_tile(tn * R, sn);
      cp_async_commit();
    }
    // carry-in for this lane's row, issued before the wait so it overlaps
    const int i1 = r0 + r1;
    const bool row1_ok = i1 < H;
    CarryPre<T, SH> cpre;
    if constexpr (sizeof(T) == 4) {
      if (has_pred && row1_ok)
        carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i1) * N),
                       *reinterpret_cast<CarryPre<float, SH>*>(&cpre));
    }
    cp_async_wait_dyn(nstage - 1);
    __syncwarp();
    T* sg = smem + st * TS::STAGE;
    T* dls = sg + TS::ZO;  // delta, in place over z
    T* hhs = sg + TS::BO;  // hh, in place over B

    // ================= phase 1: horizontal scan, lane = (row r1, states 4 q1 ..)
    // delta for the row's cells: the QH lanes of a row split its CW cells
#pragma unroll
    for (int m = 0; m < CW / QH; ++m) {
      const int j = q1 + m * QH;
      dls[r1 * TS::XP + j] = Num<T>::softplus(dls[r1 * TS::XP + j] + bias);
    }
    __syncwarp();
    T hh[SH];
    if (has_pred && row1_ok) {
      if constexpr (sizeof(T) == 4) {
        carry_resolve<SH>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i1) * N), cpre,
                         row_tag(a.epoch, i1), hh);
      } else {
        carry_get_wait<T, SH>(hc_in + static_cast<size_t>(i1) * N, hh, row_tag(a.epoch, i1), SH);
      }
    } else {
#pragma unroll
      for (int e = 0; e < SH; ++e) hh[e] = T(0);
    }
    {
      const T* xr = sg + TS::XO + r1 * TS::XP;
      const T* dr = dls + r1 * TS::XP;
      T* hr = hhs + r1 * TS::BP + q1 * SH;  // reads B, then overwrites it with hh
#pragma unroll 4
      for (int j = 0; j < CW; ++j) {
        T b4[SH];
        lds_states<T, SH>(b4, hr + j * N, true);
        const T dj = dr[j], xj = xr[j];
#pragma unroll
        for (int e = 0; e < SH; ++e) {
          const T av = Num<T>::exp_scaled(dj * A1[e]);
          hh[e] = fma(av, hh[e], (dj * b4[e]) * xj);
        }
        if (j < ncols) sts_states<T, SH>(hr + j * N, hh);
        if (emit_ref && row1_ok && j < ncols) {  // reference P^h (engine.cpp:186-194)
          const int jg = c0 + j;
          if (jg % Tt == Tt - 1 || jg == W - 1) {
            const size_t tile0 = (static_cast<size_t>(s) * kh + i1 / Tt) * kw + jg / Tt;
#pragma unroll
            for (int e = 0; e < SH; ++e) a.ph[(tile0 * Tt + i1 % Tt) * N + q1 * SH + e] = hh[e];
          }
        }
        if (j == ncols - 1 && has_succ && row1_ok)
          carry_put<T, SH>(hc_out + static_cast<size_t>(i1) * N, hh, row_tag(a.epoch, i1), SH);
      }
    }
    __syncwarp();

    // ================= phase 2: vertical scan + readout, lane = (column j2, states s2 SV ..)
    {
      const int jg = c0 + j2;
      const bool col_ok = j2 < ncols;
      const T* hcol = hhs + j2 * N + s2 * SV;
      const T* ccol = sg + TS::CO + j2 * N + s2 * SV;
      T* yp = a.y + s * HW + static_cast<size_t>(r0) * W + jg;
      const int rows = min(R, H - r0);
      for (int r = 0; r < rows; ++r) {
        const int i = r0 + r;
        const T dj = dls[r * TS::XP + j2];
        T acc0 = T(0), acc1 = T(0);
        constexpr int V = SV < 4 ? SV : 4;  // states per shared-memory vector load
#pragma unroll
        for (int e0 = 0; e0 < SV; e0 += V) {
          T h4[V], c4[V];
          lds_states<T, V>(h4, hcol + r * TS::BP + e0, true);
          lds_states<T, V>(c4, ccol + r * TS::BP + e0, true);
#pragma unroll
          for (int e = 0; e < V; ++e) {
            const T av = Num<T>::exp_scaled(dj * A2v[e0 + e]);
            const T h = fma(av, hv[e0 + e], h4[e]);
            hv[e0 + e] = h;
            if (e & 1)
              acc1 = fma(c4[e], h, acc1);
            else
              acc0 = fma(c4[e], h, acc0);
          }
        }
        T acc = acc0 + acc1;
#pragma unroll
        for (int o = 1; o < QV; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (col_ok) {
          if (s2 == 0) yp[static_cast<size_t>(r) * W] = fma(Dsk, sg[TS::XO + r * TS::XP + j2], acc);
          if (save && kb == K - 1 && i < H - 1) {
            T* ck = a.ckpt + ((static_cast<size_t>(s) * nbm1 + bi) * W + jg) * N + s2 * SV;
            stg_states<T, SV>(ck, hv, SV, true);
          }
          if (emit_ref && ((i % Tt) == Tt - 1 || i == H - 1)) {  // reference P^v (:217-220)
            const size_t tile0 = (static_cast<size_t>(s) * kh + i / Tt) * kw + jg / Tt;
#pragma unroll
            for (int e = 0; e < SV; ++e) a.pv[(tile0 * Tt + jg % Tt) * N + s2 * SV + e] = hv[e];
          }
        }
        if (++kb == K) {
          kb = 0;
          ++bi;
        }
      }
    }
    __syncwarp();
    if (++st == nstage) st = 0;
  }
}

}  // namespace s2d
