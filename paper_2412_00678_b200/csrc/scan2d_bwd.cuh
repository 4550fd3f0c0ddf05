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
  constexpr int DPL = (J + LPC - 1) / LPC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const Geo& ge = a.plan.b;
  const int lane = threadIdx.x;
  const int H = a.H, W = a.W, N = a.N, Np = ge.Np;
  const int K = a.plan.K, nb = a.plan.nb;

  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) griddep_wait();  // the begin kernel's header writes are visible
  const uint32_t epoch = ge.wreal > 1 ? load_epoch(a.hdr) : 0u;
  if (ge.wreal > 1) {
    int t = 0;
    if (lane == 0) {
      t = atomicAdd(a.ticket, 1);
      if (t == 0) a.hdr->magic = a.magic;  // the carry region now follows this layout
    }
    t = __shfl_sync(kFull, t, 0);
    // reverse order within a scan: the rightmost column group starts first
    const int64_t ss = t / ge.wreal;
    unit = ss * ge.wreal + (ge.wreal - 1 - t % ge.wreal);
  }
  const LaneMap lm = lane_map<LPC, J>(ge, unit, lane, a.S, W);
  const int q = lm.q, cis = lm.cis, segw = lm.segw, lane_in_seg = lm.lane_in_seg;
  const int64_t sc = lm.scan_ok ? lm.s : 0;
  const int p = param_row(sc, a.S, a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const int nvalid = N - q * SPL;
  const bool svec = a.ovec && nvalid >= SPL && (N % SPL) == 0;  // vector global stores of the lane's states

  T Ad[SPL];  // natural units: Abar = exp_nat(delta A)
#pragma unroll
  for (int e = 0; e < SPL; ++e) {
    const int d = q * SPL + e;
    Ad[e] = (lm.scan_ok && d < N) ? a.A[static_cast<int64_t>(p) * N + d] : T(0);
  }
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  const int nstage = ge.stages;
  T* hb = smem + static_cast<size_t>(nstage) * ge.stage_elems;  // [(K+1)][J][32][SPL]
  T* ec = hb + static_cast<size_t>(K + 1) * J * 32 * SPL;        // [K][32][SPL]
  for (int e = lane; e < nstage * ge.stage_elems; e += 32) smem[e] = T(0);

  const StageLayout<T> Ls(ge.colsw, Np, true);
  Stager<T> stg;
  stg.xvec = a.xvec != 0;
  stg.bvec = a.bvec != 0;
  stg.zoff = Ls.zo - Ls.xo;
  stg.dyoff = Ls.dyo - Ls.xo;
  stg.coff = Ls.co - Ls.bo;
  stg.x0 = a.x + lm.s0 * HW;
  stg.z0 = a.z + lm.s0 * HW;
  stg.dy0 = a.dy + lm.s0 * HW;
  stg.B0 = a.B + bc_row(lm.s0, a.G) * HW * N;
  stg.C0 = a.C + bc_row(lm.s0, a.G) * HW * N;
  stg.xstride = W;
  stg.bstride = static_cast<size_t>(W) * N;
  stg.build(reinterpret_cast<CopyEntry*>(smem + ge.table_off), lane, lm.seg_scans, lm.c0, lm.ncols, N, Np,
            HW, Ls, lm.s0, a.G);

  const int nbm1 = nb - 1, Q = a.plan.Q, nq = a.plan.nq;
  const bool has_pred = lm.wpos > 0;
  const bool has_succ = lm.wpos + 1 < ge.wreal;
  // saved forward carry into this warp's first column (residual, no waiting)
  const T* hc_in = has_pred ? a.hres + ((sc * nq + (lm.c0 / Q - 1)) * H) * N + q * SPL : nullptr;
  // reverse chain: receive from wpos+1, send to wpos-1 ([S][wreal-1][H][N])
  const int wb = ge.wreal - 1;
  const CarrySlot<T>* rc_in = has_succ ? a.rcarry + ((sc * wb + lm.wpos) * H) * N + q * SPL : nullptr;
  CarrySlot<T>* rc_out = has_pred ? a.rcarry + ((sc * wb + (lm.wpos - 1)) * H) * N + q * SPL : nullptr;
  T* dxs = a.dx + sc * HW;
  T* dzs = a.dz + sc * HW;
  T* dBs = a.dB + sc * HW * N + q * SPL;
  T* dCs = a.dC + sc * HW * N + q * SPL;

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
  // per-cell scalar sums run over the whole strip: accumulate in double
  double dbias_acc = 0.0, dD_acc = 0.0;

  __syncwarp();
  const int njobs = 2 * H;
  for (int t = 0; t < nstage - 1; ++t) {
    if (t < njobs) {
      const Job jb = job_of(t, H, K, nb);
      stg.issue(smem + t * ge.stage_elems, jb.row, lane, jb.isR, jb.isR);
    }
    cp_async_commit();
  }
  int st = 0;
  for (int t = 0; t < njobs; ++t) {
    {
      const int tn = t + nstage - 1;
      int sn = st + nstage - 1;
      if (sn >= nstage) sn -= nstage;
      if (tn < njobs) {
        const Job jn = job_of(tn, H, K, nb);
        stg.issue(smem + sn * ge.stage_elems, jn.row, lane, jn.isR, jn.isR);
      }
      cp_async_commit();
    }
    cp_async_wait_dyn(nstage - 1);
    __syncwarp();
    const T* sx = smem + st * ge.stage_elems + lm.gseg * Ls.seg_stride;
    const Job jb = job_of(t, H, K, nb);
    const int i = jb.row;
    const int rb = i - jb.r0;  // row within the band

    // ---- discretise the row (shared by both phases)
    T dl[DPL], sl[DPL];
#pragma unroll
    for (int m = 0; m < DPL; ++m) {
      const int kk = q + m * LPC;
      const T v = kk < J ? sx[Ls.zo + cis * J + kk] + bias : T(0);
      dl[m] = Num<T>::softplus(v);
      sl[m] = jb.isR ? Num<T>::sigmoid(v) : T(0);
    }
    T delta[J];
    const int base_lane = lane & ~(LPC - 1);
#pragma unroll
    for (int k = 0; k < J; ++k) delta[k] = __shfl_sync(kFull, dl[k / LPC], base_lane + (k % LPC));
    T av[J][SPL], uv[J][SPL];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const int col = cis * J + k;
      const T xk = sx[Ls.xo + col];
      T bq[SPL];
      lds_states<T, SPL>(bq, sx + Ls.bo + col * Np + q * SPL, true);
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        av[k][e] = Num<T>::exp_nat(delta[k] * Ad[e]);
        uv[k][e] = (delta[k] * bq[e]) * xk;
      }
    }

    if (!jb.isR) {
      // ================================================= phase F (recompute)
      if (rb == 0) {
        const T* ck = a.ckpt + ((static_cast<size_t>(sc) * nbm1 + (jb.r0 / K - 1)) * W) * N + q * SPL;
#pragma unroll
        for (int k = 0; k < J; ++k) {
          const int j = lm.colc + k;
#pragma unroll
          for (int e = 0; e < SPL; ++e) {
            hv[k][e] = (jb.r0 > 0 && lm.scan_ok && j < W && e < nvalid) ? ck[static_cast<size_t>(j) * N + e] : T(0);
            hb[(k * 32 + lane) * SPL + e] = hv[k][e];
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
      T ew[SPL];
      if (has_pred)
        load_states<T, SPL>(ew, hc_in + static_cast<size_t>(i) * N, nvalid);
      else {
#pragma unroll
        for (int e = 0; e < SPL; ++e) ew[e] = T(0);
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
        hh[e] = fma(Pe, ew[e], Le);
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
      T sig[J];
#pragma unroll
      for (int k = 0; k < J; ++k) sig[k] = __shfl_sync(kFull, sl[k / LPC], base_lane + (k % LPC));
      T G[J][SPL];
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const int col = cis * J + k;
        const T dyk = sx[Ls.dyo + col];
        T cq[SPL];
        lds_states<T, SPL>(cq, sx + Ls.co + col * Np + q * SPL, true);
#pragma unroll
        for (int e = 0; e < SPL; ++e) G[k][e] = fma(cq[e], dyk, dn[k][e]);  // engine.cpp:321
      }
      // chunk reverse map rho_out = al rho_in + be (engine.cpp:343-350)
      T al[SPL], be[SPL];
#pragma unroll
      for (int e = 0; e < SPL; ++e) {
        T r = T(0), pr = T(1);
#pragma unroll
        for (int k = J - 1; k >= 0; --k) {
          r = av[k][e] * (G[k][e] + r);
          pr = pr * av[k][e];
        }
        al[e] = pr;
        be[e] = r;
      }
#pragma unroll
      for (int off = LPC; off < 32; off <<= 1) {
        if (off >= segw) break;
        T ad[SPL], bd[SPL];
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          ad[e] = __shfl_down_sync(kFull, al[e], off, segw);
          bd[e] = __shfl_down_sync(kFull, be[e], off, segw);
        }
        if (lane_in_seg + off < segw) {
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
        for (int e = 0; e < SPL; ++e) rw[e] = T(0);
        const int tag = row_tag(epoch, i);
        if (has_succ) carry_get_wait<T, SPL>(rc_in + static_cast<size_t>(i) * N, rw, tag, nvalid);
        if (has_pred) {
          T out[SPL];
#pragma unroll
          for (int e = 0; e < SPL; ++e) {
            const T at = __shfl_sync(kFull, al[e], q);  // chunk 0 holds the warp aggregate
            const T bt = __shfl_sync(kFull, be[e], q);
            out[e] = fma(at, rw[e], bt);
          }
          if (lm.c == 0) carry_put<T, SPL>(rc_out + static_cast<size_t>(i) * N, out, tag, nvalid);
        }
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          T ae = __shfl_down_sync(kFull, al[e], LPC, segw);
          T bx = __shfl_down_sync(kFull, be[e], LPC, segw);
          if (lane_in_seg + LPC >= segw) {
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
        const int col = cis * J + k;
        const int j = lm.colc + k;
        const T xk = sx[Ls.xo + col], dyk = sx[Ls.dyo + col];
        T bq[SPL], hu[SPL], hc[SPL], dBv[SPL], dCv[SPL];
        lds_states<T, SPL>(bq, sx + Ls.bo + col * Np + q * SPL, true);
        lds_states<T, SPL>(hu, hup + (k * 32 + lane) * SPL, true);
        lds_states<T, SPL>(hc, hcur + (k * 32 + lane) * SPL, true);
        T dd = T(0), sg = T(0);
        const T dax = delta[k] * xk;
#pragma unroll
        for (int e = 0; e < SPL; ++e) {
          const T dab = fma(Gh[k][e], hl[e], G[k][e] * hu[e]);
          hl[e] = fma(av[k][e], hl[e], uv[k][e]);
          dA_acc[e] = fma(dab, delta[k] * av[k][e], dA_acc[e]);
          dd = fma(Gh[k][e], bq[e] * xk, fma(dab, av[k][e] * Ad[e], dd));
          sg = fma(Gh[k][e], bq[e], sg);
          dBv[e] = Gh[k][e] * dax;
          dCv[e] = dyk * hc[e];
          dn[k][e] = av[k][e] * G[k][e];
        }
        ddp[k] = dd;
        sgb[k] = sg;
        if (lm.scan_ok && j < W && nvalid > 0) {
          stg_states<T, SPL>(dBs + (rowb + j) * N, dBv, nvalid, svec);
          stg_states<T, SPL>(dCs + (rowb + j) * N, dCv, nvalid, svec);
        }
      }
      using RS_ = RS<LPC, J>;
      const int cbase = reduce_scatter<LPC, J>(ddp, q);
      reduce_scatter<LPC, J>(sgb, q);
      if ((q & (RS_::kReplica - 1)) == 0 && lm.scan_ok) {
#pragma unroll
        for (int m = 0; m < RS_::kKeep; ++m) {
          const int k = cbase + m;
          const int j = lm.colc + k;
          if (j < W) {
            const T dyv = sx[Ls.dyo + cis * J + k], xv = sx[Ls.xo + cis * J + k];
            const T dv = select_col<J>(delta, k), sv = select_col<J>(sig, k);
            const T dzv = ddp[m] * sv;
            dxs[rowb + j] = fma(Dsk, dyv, dv * sgb[m]);
            dzs[rowb + j] = dzv;
            dbias_acc += static_cast<double>(dzv);
            dD_acc = fma(static_cast<double>(dyv), static_cast<double>(xv), dD_acc);
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
  if (lm.scan_ok) {
    T* part = a.part + (static_cast<size_t>(lm.s) * ge.wreal + lm.wpos) * (N + 2);
    if (lane_in_seg < LPC) {
#pragma unroll
      for (int e = 0; e < SPL; ++e)
        if (e < nvalid) part[q * SPL + e] = dA_acc[e];
    }
    if (lane_in_seg == 0) {
      part[N] = static_cast<T>(dbias_acc);
      part[N + 1] = static_cast<T>(dD_acc);
    }
  }
}

// dA[p][d], dbias[p], dD[p]: sum over scans s = p, p + P, ... and their warps.
// One warp per output: lane l sums terms l, l + 32, ... in ascending order,
// then a fixed xor butterfly -- a fixed order (bit-reproducible) whose
// dependent chain is 32x shorter than a single-thread walk (P = 1 over 128
// scans x 13 strips took ~0.3 ms that way).
template <typename T>
__global__ void scan2d_reduce_params_kernel(const T* __restrict__ part, int64_t S, int wps, int P, int N,
                                            T* dA, T* dbias, T* dD) {
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = static_cast<int64_t>(P) * (N + 2);
  if (t >= total) return;  // warp-uniform
  const int p = static_cast<int>(t / (N + 2)), q = static_cast<int>(t % (N + 2));
  const int64_t terms = (S / P) * wps;
  T acc = T(0);
#pragma unroll 4
  for (int64_t k = lane; k < terms; k += 32) {
    const int64_t s = p + (k / wps) * P;
    const int w = static_cast<int>(k % wps);
    acc += part[(s * wps + w) * (N + 2) + q];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane != 0) return;
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
