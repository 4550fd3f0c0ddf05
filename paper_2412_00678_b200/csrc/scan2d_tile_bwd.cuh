// scan2d_tile_bwd.cuh -- "tile-transpose" backward kernel for N in {4,8,16,32}.
//
// Replaces scan2d::tiled_scan_2d_backward (proj/src/engine.cpp:245-410) with
// the same adjoints (engine.cpp:304-397):
//   G  = fma(C, dy, Abar(i+1,j) G(i+1,j))          Gh = G + Abar(i,j+1) Gh(i,j+1)
//   dAbar = fma(Gh, hh(i,j-1), G h(i-1,j));  dA += dAbar delta Abar
//   ddelta = sum_d dAbar Abar A + Gh B x;    dB = Gh delta x;   dC = dy h
//   dx = fma(D, dy, delta sum_d Gh B);  dz = ddelta sigmoid(z+bias);  dbias, dD
// Forward states are recomputed, never stored: the forward residual gives h at
// the last row of every tile (K = R rows) and the horizontal carry at every
// 16-column strip boundary.
//
// One warp owns a 16-column strip of one scan and visits its R-row tiles
// bottom to top.  Per tile (all operands staged in shared memory):
//   F1 row lanes    delta, sigmoid per cell; hh left->right from the saved carry
//   F2 column lanes h top->down from the checkpoint (rows kept in smem)
//   R1 column lanes G bottom->up (the reverse vertical state stays in registers
//                   across tiles), dC = dy h; G overwrites C in place
//   R2 row lanes    Gh right->left (carry from the right strip: tagged words,
//                   reverse tickets), chain rule, dB; per-cell sums over the
//                   row's lanes by reduce-scatter, then dx, dz
// dA / dbias / dD: per-lane accumulators, warp butterfly, fixed-order reduction
// (scan2d_reduce_params_kernel) -- bit-reproducible.
#pragma once

#include "scan2d_tile.cuh"

namespace s2d {

template <typename T, int N, int CW, int SH = 4>
struct TileShapeB {
  using F = TileShape<T, N, CW, SH>;
  static constexpr int QH = F::QH, R = F::R, QV = F::QV, SV = F::SV, BP = F::BP, XP = F::XP, EPV = F::EPV;
  // X | D (delta over z) | DY | SG (sigmoid) | B | G (C then G) | HH | HU[(R+1)]
  static constexpr int XO = 0, DO = R * XP, YO = 2 * R * XP, SO = 3 * R * XP;
  static constexpr int BO = 4 * R * XP, GO = BO + R * BP, HHO = GO + R * BP, HUO = HHO + R * BP;
  static constexpr int TOTAL = HUO + (R + 1) * BP;
  static constexpr int XU = R * CW / EPV, BU = R * CW * N / EPV, XUL = (XU + 31) / 32, BUL = (BU + 31) / 32;
  static constexpr int BUR = CW * N / EPV;
};

template <typename T, int N, int CW, int SH>
__global__ void __launch_bounds__(32, 8) scan2d_bwd_tile_kernel(const Args<T> a) {
  using TS = TileShapeB<T, N, CW, SH>;
  constexpr int R = TS::R, QH = TS::QH, QV = TS::QV, SV = TS::SV, EPV = TS::EPV, BP = TS::BP, XP = TS::XP;
  constexpr int V = SV < 4 ? SV : 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const Geo& ge = a.plan.b;
  const int lane = threadIdx.x;
  const int H = a.H, W = a.W;

  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(kFull, t, 0);
    const int64_t ss = t / ge.wreal;  // reverse order within a scan: rightmost strip first
    unit = ss * ge.wreal + (ge.wreal - 1 - t % ge.wreal);
  }
  const int64_t s = unit / ge.wreal;
  const int wpos = static_cast<int>(unit % ge.wreal);
  const int c0 = wpos * CW;
  const int ncols = min(CW, W - c0);
  const int p = static_cast<int>(s % a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  const int r1 = lane / QH, q1 = lane % QH;  // row lanes: row r1, states SH q1 ..
  const int j2 = lane / QV, s2 = lane % QV;  // column lanes: column j2, states s2 SV ..
  T A1[SH], Au1[SH], A2v[SV];
#pragma unroll
  for (int e = 0; e < SH; ++e) {
    Au1[e] = a.A[static_cast<int64_t>(p) * N + q1 * SH + e];
    A1[e] = Num<T>::a_scale(Au1[e]);
  }
#pragma unroll
  for (int e = 0; e < SV; ++e) A2v[e] = Num<T>::a_scale(a.A[static_cast<int64_t>(p) * N + s2 * SV + e]);

  for (int e = lane; e < TS::TOTAL; e += 32) sm[e] = T(0);
  __syncwarp();

  const T* xg = a.x + s * HW + c0;
  const T* zg = a.z + s * HW + c0;
  const T* yg = a.dy + s * HW + c0;
  const T* Bg = a.B + (s / a.G) * HW * N + static_cast<size_t>(c0) * N;
  const T* Cg = a.C + (s / a.G) * HW * N + static_cast<size_t>(c0) * N;
  const int xunits_row = ncols / EPV, bunits_row = ncols * N / EPV;
  const size_t WN = static_cast<size_t>(W) * N;
  const uint32_t sbase = smem_u32(sm);
  constexpr int ES = static_cast<int>(sizeof(T));
  auto issue_tile = [&](int r0) {
    constexpr int XR = CW / EPV;
#pragma unroll
    for (int m = 0; m < TS::XUL; ++m) {
      const int u = lane + 32 * m;
      const int rr = u / XR, cu = u % XR;
      if (u < TS::XU && cu < xunits_row && r0 + rr < H) {
        const size_t go = static_cast<size_t>(r0 + rr) * W + cu * EPV;
        const uint32_t so = (rr * XP + cu * EPV) * ES;
        cp_async16_raw(sbase + TS::XO * ES + so, xg + go);
        cp_async16_raw(sbase + TS::DO * ES + so, zg + go);
        cp_async16_raw(sbase + TS::YO * ES + so, yg + go);
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
        const uint32_t so = (rr * BP + cu * EPV) * ES;
        cp_async16_raw(sbase + TS::BO * ES + so, bt + go);
        cp_async16_raw(sbase + TS::GO * ES + so, ct + go);
      }
    }
    cp_async_commit();
  };

  const int nq = a.plan.nq, K = a.plan.K, nbm1 = a.plan.nb - 1;
  const bool has_pred = wpos > 0, has_succ = wpos + 1 < ge.wreal;
  const CarrySlot<T>* hc_in = has_pred ? a.hcarry + ((s * nq + (wpos - 1)) * H) * N + q1 * SH : nullptr;
  const int wb = ge.wreal - 1;
  const CarrySlot<T>* rc_in = has_succ ? a.rcarry + ((s * wb + wpos) * H) * N + q1 * SH : nullptr;
  CarrySlot<T>* rc_out = has_pred ? a.rcarry + ((s * wb + (wpos - 1)) * H) * N + q1 * SH : nullptr;
  T* dBg = a.dB + s * HW * N + static_cast<size_t>(c0) * N;
  T* dCg = a.dC + s * HW * N + static_cast<size_t>(c0) * N;
  T* dxg = a.dx + s * HW + c0;
  T* dzg = a.dz + s * HW + c0;

  T dn[SV];  // Abar(i+1) G(i+1), carried up across tiles (column lanes)
#pragma unroll
  for (int e = 0; e < SV; ++e) dn[e] = T(0);
  T dA_acc[SH];
#pragma unroll
  for (int e = 0; e < SH; ++e) dA_acc[e] = T(0);
  T dbias_acc = T(0), dD_acc = T(0);

  T* Xs = sm + TS::XO;
  T* Ds = sm + TS::DO;
  T* Ys = sm + TS::YO;
  T* Ss = sm + TS::SO;
  T* Bs = sm + TS::BO;
  T* Gs = sm + TS::GO;
  T* HHs = sm + TS::HHO;
  T* HUs = sm + TS::HUO;

  const int ntiles = (H + R - 1) / R;
  for (int t = ntiles - 1; t >= 0; --t) {
    const int r0 = t * R;
    const int rows = min(R, H - r0);
    issue_tile(r0);
    const int i1 = r0 + r1;
    const bool row_ok = r1 < rows;
    // saved forward carry (residual) and the reverse carry: loads issued early
    T hh0[SH];
#pragma unroll
    for (int e = 0; e < SH; ++e) hh0[e] = T(0);
    if (has_pred && row_ok) carry_get<T, SH>(hc_in + static_cast<size_t>(i1) * N, hh0, SH);
    CarryPre<T, SH> rpre;
    if constexpr (sizeof(T) == 4) {
      if (has_succ && row_ok)
        carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(rc_in + static_cast<size_t>(i1) * N),
                       *reinterpret_cast<CarryPre<float, SH>*>(&rpre));
    }
    // checkpoint row (h at row r0 - 1) for the column lanes
    T hprev[SV];
#pragma unroll
    for (int e = 0; e < SV; ++e) hprev[e] = T(0);
    if (t > 0 && j2 < ncols) {
      const T* ck = a.ckpt + ((static_cast<size_t>(s) * nbm1 + (t - 1)) * W + c0 + j2) * N + s2 * SV;
#pragma unroll
      for (int e = 0; e < SV; ++e) hprev[e] = ck[e];
    }
    cp_async_wait<0>();
    __syncwarp();

    // ============ F1 (row lanes): delta, sigmoid, hh left -> right
#pragma unroll
    for (int m = 0; m < CW / QH; ++m) {
      const int j = q1 + m * QH;
      const T v = Ds[r1 * XP + j] + bias;
      Ds[r1 * XP + j] = Num<T>::softplus(v);
      Ss[r1 * XP + j] = Num<T>::sigmoid(v);
    }
    __syncwarp();
    {
      T hh[SH];
#pragma unroll
      for (int e = 0; e < SH; ++e) hh[e] = hh0[e];
      const T* xr = Xs + r1 * XP;
      const T* dr = Ds + r1 * XP;
      const T* br = Bs + r1 * BP + q1 * SH;
      T* hr = HHs + r1 * BP + q1 * SH;
#pragma unroll 4
      for (int j = 0; j < CW; ++j) {
        T b4[SH];
        lds_states<T, SH>(b4, br + j * N, true);
        const T dj = dr[j], xj = xr[j];
#pragma unroll
        for (int e = 0; e < SH; ++e) hh[e] = fma(Num<T>::exp_scaled(dj * A1[e]), hh[e], (dj * b4[e]) * xj);
        sts_states<T, SH>(hr + j * N, hh);
      }
    }
    // ============ F2 (column lanes): h top -> down, rows -1 .. rows-1 into HU
    {
      T* hu = HUs + j2 * N + s2 * SV;
#pragma unroll
      for (int e0 = 0; e0 < SV; e0 += V) {
        T v[V];
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] = hprev[e0 + e];
        if constexpr (V == 4 && sizeof(T) == 4)
          *reinterpret_cast<float4*>(hu + e0) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int e = 0; e < V; ++e) hu[e0 + e] = v[e];
      }
      __syncwarp();
      const T* hhc = HHs + j2 * N + s2 * SV;
      for (int r = 0; r < rows; ++r) {
        const T dj = Ds[r * XP + j2];
#pragma unroll
        for (int e0 = 0; e0 < SV; e0 += V) {
          T h4[V];
          lds_states<T, V>(h4, hhc + r * BP + e0, true);
#pragma unroll
          for (int e = 0; e < V; ++e)
            hprev[e0 + e] = fma(Num<T>::exp_scaled(dj * A2v[e0 + e]), hprev[e0 + e], h4[e]);
          T* dst = hu + (r + 1) * BP + e0;
          if constexpr (V == 4 && sizeof(T) == 4)
            *reinterpret_cast<float4*>(dst) = make_float4(hprev[e0], hprev[e0 + 1], hprev[e0 + 2], hprev[e0 + 3]);
          else
#pragma unroll
            for (int e = 0; e < V; ++e) dst[e] = hprev[e0 + e];
        }
      }
    }
    __syncwarp();
    // ============ R1 (column lanes): G bottom -> up, dC = dy h; G over C
    {
      const bool col_ok = j2 < ncols;
      T* gc = Gs + j2 * N + s2 * SV;
      const T* hu = HUs + j2 * N + s2 * SV;
      for (int r = rows - 1; r >= 0; --r) {
        const T dj = Ds[r * XP + j2], dyv = Ys[r * XP + j2];
        T* dCrow = dCg + (static_cast<size_t>(r0 + r) * W + j2) * N + s2 * SV;
#pragma unroll
        for (int e0 = 0; e0 < SV; e0 += V) {
          T c4[V], h4[V], dc[V];
          lds_states<T, V>(c4, gc + r * BP + e0, true);
          lds_states<T, V>(h4, hu + (r + 1) * BP + e0, true);
#pragma unroll
          for (int e = 0; e < V; ++e) {
            const T g = fma(c4[e], dyv, dn[e0 + e]);  // engine.cpp:321
            c4[e] = g;
            dn[e0 + e] = Num<T>::exp_scaled(dj * A2v[e0 + e]) * g;
            dc[e] = dyv * h4[e];
          }
          T* gdst = gc + r * BP + e0;
          if constexpr (V == 4 && sizeof(T) == 4)
            *reinterpret_cast<float4*>(gdst) = make_float4(c4[0], c4[1], c4[2], c4[3]);
          else
#pragma unroll
            for (int e = 0; e < V; ++e) gdst[e] = c4[e];
          if (col_ok) stg_states<T, V>(dCrow + e0, dc, V, true);
        }
      }
    }
    __syncwarp();
    // ============ R2 (row lanes): Gh right -> left, chain rule
    {
      T rho[SH];
#pragma unroll
      for (int e = 0; e < SH; ++e) rho[e] = T(0);
      if (has_succ && row_ok) {
        if constexpr (sizeof(T) == 4)
          carry_resolve<SH>(reinterpret_cast<const CarrySlot<float>*>(rc_in + static_cast<size_t>(i1) * N), rpre,
                            row_tag(a.epoch, i1), rho);
        else
          carry_get_wait<T, SH>(rc_in + static_cast<size_t>(i1) * N, rho, row_tag(a.epoch, i1), SH);
      }
      const T* xr = Xs + r1 * XP;
      const T* dr = Ds + r1 * XP;
      const T* br = Bs + r1 * BP + q1 * SH;
      const T* gr = Gs + r1 * BP + q1 * SH;
      const T* hr = HHs + r1 * BP + q1 * SH;
      const T* ur = HUs + r1 * BP + q1 * SH;  // h(i-1): HU row r1 is tile row r1 - 1
      T* dBrow = dBg + static_cast<size_t>(i1) * WN + q1 * SH;
      // columns in groups of QH: per-cell sums over the row's QH lanes by
      // reduce-scatter, one finished cell per lane per group
#pragma unroll
      for (int gs = CW - QH; gs >= 0; gs -= QH) {
        T ddp[QH], sgb[QH];
#pragma unroll
        for (int jj = QH - 1; jj >= 0; --jj) {
          const int j = gs + jj;
          T g4[SH], b4[SH], hl[SH], hu4[SH];
          lds_states<T, SH>(g4, gr + j * N, true);
          lds_states<T, SH>(b4, br + j * N, true);
          lds_states<T, SH>(hu4, ur + j * N, true);
          if (j > 0) {
            lds_states<T, SH>(hl, hr + (j - 1) * N, true);
          } else {
#pragma unroll
            for (int e = 0; e < SH; ++e) hl[e] = hh0[e];
          }
          const T dj = dr[j], xj = xr[j];
          T dd = T(0), sg = T(0), dBv[SH];
#pragma unroll
          for (int e = 0; e < SH; ++e) {
            const T av = Num<T>::exp_scaled(dj * A1[e]);
            const T gh = g4[e] + rho[e];  // engine.cpp:346
            rho[e] = av * gh;
            const T dab = fma(gh, hl[e], g4[e] * hu4[e]);  // engine.cpp:383
            if (row_ok) dA_acc[e] = fma(dab, dj * av, dA_acc[e]);
            dd = fma(gh, b4[e] * xj, fma(dab, av * Au1[e], dd));
            sg = fma(gh, b4[e], sg);
            dBv[e] = gh * (dj * xj);
          }
          ddp[jj] = dd;
          sgb[jj] = sg;
          if (row_ok && j < ncols) stg_states<T, SH>(dBrow + static_cast<size_t>(j) * N, dBv, SH, true);
        }
        const int cb = reduce_scatter<QH, QH>(ddp, q1);
        reduce_scatter<QH, QH>(sgb, q1);
        const int j = gs + cb;
        if (row_ok && j < ncols) {
          const T dv = dr[j], xv = xr[j], dyv = Ys[r1 * XP + j], sv = Ss[r1 * XP + j];
          const T dzv = ddp[0] * sv;
          dxg[static_cast<size_t>(i1) * W + j] = fma(Dsk, dyv, dv * sgb[0]);
          dzg[static_cast<size_t>(i1) * W + j] = dzv;
          dbias_acc += dzv;
          dD_acc = fma(dyv, xv, dD_acc);
        }
      }
      if (has_pred && row_ok)
        carry_put<T, SH>(rc_out + static_cast<size_t>(i1) * N, rho, row_tag(a.epoch, i1), SH);
    }
    __syncwarp();
  }

  // ---- per-(scan, strip) partials, fixed order
#pragma unroll
  for (int e = 0; e < SH; ++e)
    for (int h = QH; h < 32; h <<= 1) dA_acc[e] += __shfl_xor_sync(kFull, dA_acc[e], h);
  for (int h = 1; h < 32; h <<= 1) {
    dbias_acc += __shfl_xor_sync(kFull, dbias_acc, h);
    dD_acc += __shfl_xor_sync(kFull, dD_acc, h);
  }
  T* part = a.part + (static_cast<size_t>(s) * ge.wreal + wpos) * (N + 2);
  if (lane < QH) {
#pragma unroll
    for (int e = 0; e < SH; ++e) part[q1 * SH + e] = dA_acc[e];
  }
  if (lane == 0) {
    part[N] = dbias_acc;
    part[N + 1] = dD_acc;
  }
}

}  // namespace s2d
