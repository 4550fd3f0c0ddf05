// scan2d_bwd.cuh -- backward 2D selective scan kernels (sm_100a).
//
// Replaces scan2d::tiled_scan_2d_backward (proj/src/engine.cpp:245-410): the
// same adjoint recurrences and chain rule (engine.cpp:304-397),
//   G(i,j)  = fma(C, dy, Abar(i+1,j) G(i+1,j))          reverse vertical
//   Gh(i,j) = G(i,j) + Abar(i,j+1) Gh(i,j+1)              reverse horizontal
//   dAbar   = fma(Gh, hh(i,j-1), G h(i-1,j))
//   dA += dAbar delta Abar;  ddelta = sum_d dAbar Abar A + Gh B x
//   dB = Gh delta x;  dC = dy h;  dx = fma(D, dy, delta sum_d Gh B)
//   dz = ddelta sigmoid(z + bias);  dbias = sum dz;  dD = sum dy x
// with forward states RECOMPUTED, not stored (north_star): the forward
// residual holds only h at the last row of every K-row band plus the
// horizontal carries at every Q-column boundary.
//
// Same warp/column-group decomposition as the forward (one warp per CTA).
// Bands of K rows are visited bottom to top.  Per band:
//   phase F  re-runs the forward over the band top to bottom from the
//            checkpoint, keeping h of the band's rows and each chunk's
//            horizontal carry-in in shared memory;
//   phase R  walks the band bottom to top: G in registers (vertical),
//            Gh by a right-to-left chunk scan + warp chain (tagged words,
//            reverse tickets), then the chain rule.
// Both phases stream their rows through one cp.async ring (the job sequence
// F rows, R rows, next band, ...), so prefetch never drains at band edges.
// dA / dbias / dD are kept per lane and reduced in a fixed order (warp
// butterfly, then scan2d_reduce_params_kernel in ascending scan order) -- no
// floating-point atomics, so results are bit-reproducible
// (test_backward.cpp:56-74).
#pragma once

#include "scan2d_fwd.cuh"

namespace s2d {

// job t in [0, 2H): bands bottom-up; per band K forward rows then K reverse rows
struct Job {
  int row, r0, isR;
};
__device__ __forceinline__ Job job_of(int t, int H, int K, int nb) {
  const int last0 = (nb - 1) * K;
  const int L = H - last0;  // rows of the bottom band
  Job j;
  if (t < 2 * L) {
    j.r0 = last0;
    j.isR = t >= L;
    j.row = j.isR ? last0 + (2 * L - 1 - t) : last0 + t;
  } else {
    const int u = t - 2 * L;
    const int b = nb - 2 - u / (2 * K);
    const int v = u % (2 * K);
    j.r0 = b * K;
    j.isR = v >= K;
    j.row = j.isR ? j.r0 + (2 * K - 1 - v) : j.r0 + v;
  }
  return j;
}

template <typename T>
__host__ __device__ inline int bwd_band_elems(int K, int J, int SPL) {
  // hb[(K+1)][J][32][SPL] + ec[K][32][SPL]
  return ((K + 1) * J + K) * 32 * SPL;
}

template <typename T, int SPL, int LPC, int J>
__global__ void __launch_bounds__(32, 16) scan2d_bwd_kernel(const Args<T> a) {
  constexpr int CPW = 32 / LPC;
  constexpr int DPL = (J + LPC - 1) / LPC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const Geo& ge = a.plan.b;
  const int lane = threadIdx.x;
  const int H = a.H, W = a.W, N = a.N;
  const int K = a.plan.K, nb = a.plan.nb;

  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(kFull, t, 0);
    // reverse order within a scan: the rightmost column group starts first
    const int64_t ss = t / ge.wreal;
    unit = ss * ge.wreal + (ge.wreal - 1 - t % ge.wreal);
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
  const int colc = c0 + cis * J;
  const int p = static_cast<int>(sc % a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const bool vec = (N % SPL) == 0;

  T A2[SPL], Ad[SPL];
  bool dok[SPL];
#pragma unroll
  for (int e = 0; e < SPL; ++e) {
    const int d = q * SPL + e;
    dok[e] = scan_ok && d < N;
    Ad[e] = dok[e] ? a.A[static_cast<int64_t>(p) * N + d] : T(0);
    A2[e] = Num<T>::a_scale(Ad[e]);
  }
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  const int nstage = ge.stages;
  T* hb = smem + static_cast<size_t>(nstage) * ge.stage_elems;  // [(K+1)][J][32][SPL]
  T* ec = hb + static_cast<size_t>(K + 1) * J * 32 * SPL;        // [K][32][SPL]
  for (int e = lane; e < nstage * ge.stage_elems; e += 32) smem[e] = T(0);
  __syncwarp();

  const StageLayout<T> Ls(ge.colsw, N, true);
  auto issue = [&](int t, int st) {
    const Job jb = job_of(t, H, K, nb);
    T* dst0 = smem + static_cast<size_t>(st) * ge.stage_elems;
    for (int g = 0; g < ge.seg; ++g) {
      const int64_t sg = ge.seg > 1 ? unit * ge.seg + g : s;
      if (sg >= a.S) break;
      const int ncols = min(ge.colsw, W - c0);
      if (ncols <= 0) break;
      T* dst = dst0 + g * Ls.seg_stride;
      const size_t ro = (static_cast<size_t>(sg) * H + jb.row) * W + c0;
      copy_span(dst + Ls.xo, a.x + ro, ncols, lane);
      copy_span(dst + Ls.zo, a.z + ro, ncols, lane);
      const size_t bo = ((static_cast<size_t>(sg / a.G) * H + jb.row) * W + c0) * N;
      copy_span(dst + Ls.bo, a.B + bo, ncols * N, lane);
      if (jb.isR) {
        copy_span(dst + Ls.dyo, a.dy + ro, ncols, lane);
        copy_span(dst + Ls.co, a.C + bo, ncols * N, lane);
      }
    }
  };

  const int nbm1 = nb - 1, Q = a.plan.Q, nq = a.plan.nq;
  const bool has_pred = wpos > 0;
  const bool has_succ = wpos + 1 < ge.wreal;
  // saved forward carry into this warp's first column (residual, no waiting)
  const CarrySlot<T>* hc_in = has_pred ? a.hcarry + ((sc * nq + (c0 / Q - 1)) * H) * N : nullptr;
  // reverse chain: receive from wpos+1, send to wpos-1 ([S][wreal-1][H][N])
  const int wb = ge.wreal - 1;
  const CarrySlot<T>* rc_in = has_succ ? a.rcarry + ((sc * wb + wpos) * H) * N : nullptr;
  CarrySlot<T>* rc_out = has_pred ? a.rcarry + ((sc * wb + (wpos - 1)) * H) * N : nullptr;
  T* dxs = a.dx + sc * HW;
  T* dzs = a.dz + sc * HW;
  T* dBs = a.dB + sc * HW * N;
  T* dCs = a.dC + sc * HW * N;

  T dn[J][SPL];  // Abar(i+1) G(i+1): the reverse vertical state (engine.cpp:323)
  T hv[J][SPL];  // forward vertical state during phase F
#pragma unroll
  for (int k = 0; k < J; ++k)
#pragma unroll
    for (int e = 0; e < SPL; ++e) {
      dn[k][e] = T(0);
      hv[k][e] = T(0);
    }
  T dA_acc[SPL];
#pragma unroll
  for (int e = 0; e < SPL; ++e) dA_acc[e] = T(0);
  T dbias_acc = T(0), dD_acc = T(0);

  const int njobs = 2 * H;
  for (int t = 0; t < nstage - 1; ++t) {
    if (t < njobs) issue(t, t);
    cp_async_commit();
  }
  int st = 0;
  for (int t = 0; t < njobs; ++t) {
    {
      const int tn = t + nstage - 1;
      int sn = st + nstage - 1;
      if (sn >= nstage) sn -= nstage;
      if (tn < njobs) issue(tn, sn);
      cp_async_commit();
    }
    cp_async_wait_dyn(nstage - 1);
    __syncwarp();
    const T* stg = smem + static_cast<size_t>(st) * ge.stage_elems + gseg * Ls.seg_stride;
    const Job jb = job_of(t, H, K, nb);
    const int i = jb.row;
    const int rb = i - jb.r0;  // row within the band

    // ---- discretise the row (shared by both phases)
    T dl[DPL], sl[DPL];
#pragma unroll
    for (int m = 0; m < DPL; ++m) {
      const int kk = q + m * LPC;
      const T v = kk < J ? stg[Ls.zo + cis * J + kk] + bias : T(0);
      dl[m] = Num<T>::softplus(v);
      sl[m] = jb.isR ? Num<T>::sigmoid(v) : T(0);
    }
    T delta[J], sig[J];
    const int base_lane = lane & ~(LPC - 1);
#pragma unroll
    for (int k = 0; k < J; ++k) {
      delta[k] = __shfl_sync(kFull, dl[k / LPC], base_lane + (k % LPC));
      sig[k] = __shfl_sync(kFull, sl[k / LPC], base_lane + (k % LPC));
    }
    T av[J][SPL], uv[J][SPL], bq[J][SPL];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const int col = cis * J + k;
      const bool okc = scan_ok && (c0 + col) < W;
      const T xk = stg[Ls.xo + col];
      lds_states<T, SPL>(bq[k], stg + Ls.bo + col * N + q * SPL, vec);
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        const bool ok = okc && dok[e];
        av[k][e] = ok ? Num<T>::exp_scaled(delta[k] * A2[e]) : T(1);
        uv[k][e] = ok ? (delta[k] * bq[k][e]) * xk : T(0);
        if (!ok) bq[k][e] = T(0);
      }
    }

    if (!jb.isR) {
      // ================================================= phase F (recompute)
      if (rb == 0) {
        T* h0 = hb;  // row -1 of the band: the checkpoint
#pragma unroll
        for (int k = 0; k < J; ++k) {
          const int j = colc + k;
          T v[SPL];
#pragma unroll
          for (int e = 0; e < SPL; ++e) v[e] = T(0);
          if (jb.r0 > 0 && scan_ok && j < W)
            lds_states<T, SPL>(v, a.ckpt + ((static_cast<size_t>(sc) * nbm1 + (jb.r0 / K - 1)) * W + j) * N + q * SPL,
                               false);
#pragma unroll
          for (int e = 0; e < SPL; ++e) {
            hv[k][e] = dok[e] ? v[e] : T(0);
            h0[(k * 32 + lane) * SPL + e] = hv[k][e];
          }
        }
      }
      T Pc[SPL], Lc[SPL];
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        Pc[e] = av[0][e];
        Lc[e] = uv[0][e];
      }
#pragma unroll
      for (int k = 1; k < J; ++k)
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          Lc[e] = fma(av[k][e], Lc[e], uv[k][e]);
          Pc[e] = Pc[e] * av[k][e];
        }
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
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        T Pe = __shfl_up_sync(kFull, Pc[e], LPC, segw);
        T Le = __shfl_up_sync(kFull, Lc[e], LPC, segw);
        if (lane_in_seg < LPC) {
          Pe = T(1);
          Le = T(0);
        }
        const T ew = (has_pred && dok[e]) ? CarrySlot<T>::get(hc_in + static_cast<size_t>(i) * N + q * SPL + e)
                                          : T(0);
        hh[e] = fma(Pe, ew, Le);
        ec[(rb * 32 + lane) * SPL + e] = hh[e];
      }
      T* hrow = hb + static_cast<size_t>(rb + 1) * J * 32 * SPL;
#pragma unroll
      for (int k = 0; k < J; ++k)
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          hh[e] = fma(av[k][e], hh[e], uv[k][e]);
          hv[k][e] = fma(av[k][e], hv[k][e], hh[e]);
          hrow[(k * 32 + lane) * SPL + e] = hv[k][e];
        }
    } else {
      // ================================================= phase R (adjoints)
      T G[J][SPL], dyk[J];
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const int col = cis * J + k;
        dyk[k] = stg[Ls.dyo + col];
        T cq[SPL];
        lds_states<T, SPL>(cq, stg + Ls.co + col * N + q * SPL, vec);
        const bool okc = scan_ok && (c0 + col) < W;
#pragma unroll
        for (int e = 0; e < SPL; ++e) G[k][e] = fma((okc && dok[e]) ? cq[e] : T(0), dyk[k], dn[k][e]);
      }
      // chunk reverse map rho_out = al rho_in + be (engine.cpp:343-350)
      T al[SPL], be[SPL];
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        T r = T(0);
        T prod = T(1);
#pragma unroll
        for (int k = J - 1; k >= 0; --k) {
          r = av[k][e] * (G[k][e] + r);
          prod = prod * av[k][e];
        }
        al[e] = prod;
        be[e] = r;
      }
      const int span = segw;
#pragma unroll
      for (int off = LPC; off < 32; off <<= 1) {
        if (off >= span) break;
        T ad[SPL], bd[SPL];
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          ad[e] = __shfl_down_sync(kFull, al[e], off, segw);
          bd[e] = __shfl_down_sync(kFull, be[e], off, segw);
        }
        if (lane_in_seg + off < span) {
#pragma unroll
          for (int e = 0; e < SPL; ++e) {
            be[e] = fma(al[e], bd[e], be[e]);
            al[e] = al[e] * ad[e];
          }
        }
      }
      T rho[SPL];
      {
        T rw[SPL];
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          rw[e] = (has_succ && dok[e])
                      ? CarrySlot<T>::get_wait(rc_in + static_cast<size_t>(i) * N + q * SPL + e, row_tag(a.epoch, i))
                      : T(0);
        }
        if (has_pred) {
          T out[SPL];
#pragma unroll
          for (int e = 0; e < SPL; ++e) {
            const T at = __shfl_sync(kFull, al[e], q);  // chunk 0 holds the warp aggregate
            const T bt = __shfl_sync(kFull, be[e], q);
            out[e] = fma(at, rw[e], bt);
          }
          if (c == 0) {
#pragma unroll
            for (int e = 0; e < SPL; ++e)
              if (dok[e])
                CarrySlot<T>::put(rc_out + static_cast<size_t>(i) * N + q * SPL + e, out[e], row_tag(a.epoch, i));
          }
        }
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          T ae = __shfl_down_sync(kFull, al[e], LPC, segw);
          T bx = __shfl_down_sync(kFull, be[e], LPC, segw);
          if (lane_in_seg + LPC >= span) {
            ae = T(1);
            bx = T(0);
          }
          rho[e] = fma(ae, rw[e], bx);
        }
      }
      // chain rule (engine.cpp:355-397)
      T Gh[J][SPL];
#pragma unroll
      for (int k = J - 1; k >= 0; --k)
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          Gh[k][e] = G[k][e] + rho[e];
          rho[e] = av[k][e] * Gh[k][e];
        }
      T hl[SPL];
#pragma unroll
      for (int e = 0; e < SPL; ++e) hl[e] = ec[(rb * 32 + lane) * SPL + e];
      const T* hup = hb + static_cast<size_t>(rb) * J * 32 * SPL;
      const T* hcur = hup + J * 32 * SPL;
      T ddp[J], sgb[J];
      const size_t rowb = static_cast<size_t>(i) * W;
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const int j = colc + k;
        const bool okc = scan_ok && j < W;
        const T xk = stg[Ls.xo + cis * J + k];
        T hu[SPL], hc[SPL], dBv[SPL], dCv[SPL];
        lds_states<T, SPL>(hu, hup + (k * 32 + lane) * SPL, true);
        lds_states<T, SPL>(hc, hcur + (k * 32 + lane) * SPL, true);
        T dd = T(0), sg = T(0);
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          const T dab = fma(Gh[k][e], hl[e], G[k][e] * hu[e]);
          hl[e] = fma(av[k][e], hl[e], uv[k][e]);
          if (okc && dok[e]) dA_acc[e] = fma(dab, delta[k] * av[k][e], dA_acc[e]);
          dd = fma(Gh[k][e], bq[k][e] * xk, fma(dab, av[k][e] * Ad[e], dd));
          sg = fma(Gh[k][e], bq[k][e], sg);
          dBv[e] = Gh[k][e] * (delta[k] * xk);
          dCv[e] = dyk[k] * hc[e];
          dn[k][e] = av[k][e] * G[k][e];
        }
        ddp[k] = dd;
        sgb[k] = sg;
        if (okc && q * SPL < N) {
          stg_states<T, SPL>(dBs + (rowb + j) * N + q * SPL, dBv, N - q * SPL, vec);
          stg_states<T, SPL>(dCs + (rowb + j) * N + q * SPL, dCv, N - q * SPL, vec);
        }
      }
      using RS_ = RS<LPC, J>;
      const int cbase = reduce_scatter<LPC, J>(ddp, q);
      reduce_scatter<LPC, J>(sgb, q);
      if ((q & (RS_::kReplica - 1)) == 0 && scan_ok) {
#pragma unroll
        for (int m = 0; m < RS_::kKeep; ++m) {
          const int k = cbase + m;
          const int j = colc + k;
          if (j < W) {
            const T dyv = stg[Ls.dyo + cis * J + k], xv = stg[Ls.xo + cis * J + k];
            const T dv = select_col<J>(delta, k), sv = select_col<J>(sig, k);
            const T dzv = ddp[m] * sv;
            dxs[rowb + j] = fma(Dsk, dyv, dv * sgb[m]);
            dzs[rowb + j] = dzv;
            dbias_acc += dzv;
            dD_acc = fma(dyv, xv, dD_acc);
          }
        }
      }
    }
    __syncwarp();
    if (++st == nstage) st = 0;
  }

  // ---- per-(scan, warp) partials, reduced in a fixed order
#pragma unroll
  for (int e = 0; e < SPL; ++e)
    for (int h = LPC; h < segw; h <<= 1) dA_acc[e] += __shfl_xor_sync(kFull, dA_acc[e], h);
  for (int h = 1; h < segw; h <<= 1) {
    dbias_acc += __shfl_xor_sync(kFull, dbias_acc, h);
    dD_acc += __shfl_xor_sync(kFull, dD_acc, h);
  }
  if (scan_ok) {
    T* part = a.part + (static_cast<size_t>(s) * ge.wreal + wpos) * (N + 2);
    if (lane_in_seg < LPC) {
#pragma unroll
      for (int e = 0; e < SPL; ++e)
        if (dok[e]) part[q * SPL + e] = dA_acc[e];
    }
    if (lane_in_seg == 0) {
      part[N] = dbias_acc;
      part[N + 1] = dD_acc;
    }
  }
}

// dA[p][d], dbias[p], dD[p]: sum over scans s = p, p + P, ... (ascending) and
// their warps (ascending) -- the fixed order of engine.cpp:404-408.
template <typename T>
__global__ void scan2d_reduce_params_kernel(const T* __restrict__ part, int64_t S, int wps, int P, int N,
                                            T* dA, T* dbias, T* dD) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(P) * (N + 2);
  if (t >= total) return;
  const int p = static_cast<int>(t / (N + 2)), q = static_cast<int>(t % (N + 2));
  T acc = T(0);
  for (int64_t s = p; s < S; s += P)
    for (int w = 0; w < wps; ++w) acc += part[(s * wps + w) * (N + 2) + q];
  if (q < N)
    dA[static_cast<int64_t>(p) * N + q] = acc;
  else if (q == N)
    dbias[p] = acc;
  else
    dD[p] = acc;
}

// dB / dC of shared-B/C layouts (G > 1): out[grp] = sum over the group's scans
// in ascending order.
template <typename T>
__global__ void scan2d_reduce_group_kernel(const T* __restrict__ per_scan, int64_t groups, int G,
                                           size_t hwn, T* __restrict__ out) {
  const size_t total = static_cast<size_t>(groups) * hwn;
  for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t grp = e / hwn, off = e % hwn;
    T acc = T(0);
    for (int m = 0; m < G; ++m) acc += per_scan[(grp * G + m) * hwn + off];
    out[e] = acc;
  }
}

}  // namespace s2d
