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
// horizontal carries at CTA column-group boundaries.
//
// Same warp/column-group decomposition as the forward.  Bands of K rows are
// visited bottom to top.  Per band:
//   phase F  re-runs the forward over the band top to bottom from the
//            checkpoint, keeping h of the band's rows and each chunk's
//            horizontal carry-in in shared memory;
//   phase R  walks the band bottom to top: G in registers (vertical),
//            Gh by a right-to-left chunk scan + warp/CTA chain, then the
//            chain rule.  dA / dbias / dD are kept per lane and reduced in a
//            fixed order (warp butterfly, then scan_reduce_params_kernel in
//            ascending scan order) -- no floating-point atomics, so the
//            result is bit-reproducible (test_backward.cpp:56-74).
#pragma once

#include "scan2d_fwd.cuh"

namespace s2d {

template <typename T, int LPC, int J>
struct RowInB {
  static constexpr int DPL = (J + LPC - 1) / LPC;
  T x[J];
  T b[J];
  T c[J];
  T dy[J];
  T zz[DPL];
};

template <typename T, int LPC, int J>
__device__ __forceinline__ void load_row_b(RowInB<T, LPC, J>& r, const T* __restrict__ xs,
                                           const T* __restrict__ zs, const T* __restrict__ Bs,
                                           const T* __restrict__ Cs, const T* __restrict__ dys,
                                           int i, int W, int N, const LaneGeo& g, bool with_c) {
  const size_t base = static_cast<size_t>(i) * W;
#pragma unroll
  for (int k = 0; k < J; ++k) {
    const int j = g.col0 + k;
    const bool ok = g.scan_ok && j < W;
    r.x[k] = ok ? __ldg(xs + base + j) : T(0);
    const bool okd = ok && g.l < N;
    const size_t e = (base + j) * N + g.l;
    r.b[k] = okd ? __ldg(Bs + e) : T(0);
    if (with_c) {
      r.c[k] = okd ? __ldg(Cs + e) : T(0);
      r.dy[k] = ok ? __ldg(dys + base + j) : T(0);
    }
  }
#pragma unroll
  for (int m = 0; m < RowInB<T, LPC, J>::DPL; ++m) {
    const int kk = g.l + m * LPC;
    const int j = g.col0 + kk;
    const bool ok = g.scan_ok && kk < J && j < W;
    r.zz[m] = ok ? __ldg(zs + base + j) : T(0);
  }
}

template <typename T, int LPC, int J>
__device__ __forceinline__ void chunk_delta_sig(const T (&zz)[RowInB<T, LPC, J>::DPL], T bias,
                                                int lane, T (&delta)[J], T (&sig)[J],
                                                bool want_sig) {
  constexpr int DPL = RowInB<T, LPC, J>::DPL;
  T dl[DPL], sl[DPL];
#pragma unroll
  for (int m = 0; m < DPL; ++m) {
    const T v = zz[m] + bias;
    dl[m] = Num<T>::softplus(v);
    sl[m] = want_sig ? Num<T>::sigmoid(v) : T(0);
  }
  const int base_lane = lane & ~(LPC - 1);
#pragma unroll
  for (int k = 0; k < J; ++k) {
    delta[k] = __shfl_sync(kFull, dl[k / LPC], base_lane + (k % LPC));
    if (want_sig) sig[k] = __shfl_sync(kFull, sl[k / LPC], base_lane + (k % LPC));
  }
}

// Inclusive right-to-left scan of reverse affine maps rho_out = al rho_in + be
// over the chunks of a segment: chunk c absorbs everything to its right.
template <typename T, int LPC>
__device__ __forceinline__ void chunk_scan_rev(T& al, T& be, int lane_in_seg, int span, int segw) {
#pragma unroll
  for (int off = LPC; off < 32; off <<= 1) {
    if (off >= span) break;
    const T ad = __shfl_down_sync(kFull, al, off, segw);
    const T bd = __shfl_down_sync(kFull, be, off, segw);
    if (lane_in_seg + off < span) {
      be = fma(al, bd, be);
      al = al * ad;
    }
  }
}

template <typename T>
__host__ __device__ inline size_t bwd_warp_smem_bytes(int K, int J) {
  size_t b = 2 * sizeof(Ring<T>) + (static_cast<size_t>(K + 1) * J * 32 + static_cast<size_t>(K) * 32) * sizeof(T);
  return (b + 15) & ~static_cast<size_t>(15);
}

template <typename T, int LPC, int J>
__global__ void __launch_bounds__(512) scan2d_bwd_kernel(const Args<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Plan& pl = a.plan;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = pl.K;
  const size_t wstride = bwd_warp_smem_bytes<T>(K, J);

  __shared__ int s_cta;
  if (threadIdx.x == 0) {
    if (pl.ncb > 1) {
      const int t = atomicAdd(a.flags, 1);  // reverse ticket order: right CTA first
      s_cta = (t / pl.ncb) * pl.ncb + (pl.ncb - 1 - t % pl.ncb);
    } else {
      s_cta = static_cast<int>(blockIdx.x);
    }
  }
  for (int q = threadIdx.x; q < pl.nw * kRing; q += blockDim.x) {
    Ring<T>* rr = reinterpret_cast<Ring<T>*>(smem + (q / kRing) * wstride);
    mbar_init(&rr[0].full[q % kRing], 32);
    mbar_init(&rr[0].empty[q % kRing], 32);
    mbar_init(&rr[1].full[q % kRing], 32);
    mbar_init(&rr[1].empty[q % kRing], 32);
  }
  __syncthreads();
  const int64_t unit = static_cast<int64_t>(s_cta) * pl.nw + warp;
  if (unit >= pl.units) return;
  LaneGeo g;
  if (!lane_geometry<LPC, J>(pl, a.S, unit, lane, g)) return;

  unsigned char* my = smem + warp * wstride;
  Ring<T>& ring_f = reinterpret_cast<Ring<T>*>(my)[0];  // forward carries from warp-1
  Ring<T>& ring_r = reinterpret_cast<Ring<T>*>(my)[1];  // reverse carries from warp+1
  T* hb = reinterpret_cast<T*>(my + 2 * sizeof(Ring<T>));  // [(K+1)][J][32]
  T* ec = hb + static_cast<size_t>(K + 1) * J * 32;       // [K][32]
  Ring<T>* next_ring_f =
      warp + 1 < pl.nw ? &reinterpret_cast<Ring<T>*>(smem + (warp + 1) * wstride)[0] : nullptr;
  Ring<T>* prev_ring_r =
      warp > 0 ? &reinterpret_cast<Ring<T>*>(smem + (warp - 1) * wstride)[1] : nullptr;

  const int H = a.H, W = a.W, N = a.N;
  const int cb = g.wpos / pl.nw;
  const bool has_pred = g.wpos > 0;
  const bool has_succ = g.wpos + 1 < pl.wreal;
  const bool pred_global = has_pred && warp == 0;
  const bool succ_global = has_succ && warp == pl.nw - 1;
  g.st_ok = g.scan_ok && g.l < N;

  const int64_t s = g.scan_ok ? g.s : 0;
  const int64_t p = s % a.P;
  const int64_t grp = s / a.G;
  const size_t HW = static_cast<size_t>(H) * W;
  const T Ad = g.st_ok ? a.A[p * N + g.l] : T(0);
  const T A2 = Num<T>::a_scale(Ad);
  const T Dsk = a.Dskip[p], bias = a.bias[p];
  const T* xs = a.x + s * HW;
  const T* zs = a.z + s * HW;
  const T* Bs = a.B + grp * HW * N;
  const T* Cs = a.C + grp * HW * N;
  const T* dys = a.dy + s * HW;
  T* dxs = a.dx + s * HW;
  T* dzs = a.dz + s * HW;
  T* dBs = a.dB + s * HW * N;  // per-scan layout (group-reduced afterwards when G > 1)
  T* dCs = a.dC + s * HW * N;
  const int nbm1 = pl.nb - 1, ncbm1 = pl.ncb - 1;
  const T* hc_in = pred_global ? a.hcarry + ((s * ncbm1 + (cb - 1)) * H) * N : nullptr;
  int* rprog_in = succ_global ? a.flags + 1 + s * ncbm1 + cb : nullptr;
  int* rprog_out = pred_global ? a.flags + 1 + s * ncbm1 + (cb - 1) : nullptr;
  const T* rc_in = succ_global ? a.rcarry + ((s * ncbm1 + cb) * H) * N : nullptr;
  T* rc_out = pred_global ? a.rcarry + ((s * ncbm1 + (cb - 1)) * H) * N : nullptr;
  int rseen = 0;

  using RS_ = RS<LPC, J>;
  T dn[J];
#pragma unroll
  for (int k = 0; k < J; ++k) dn[k] = T(0);
  T dA_acc = T(0), dbias_acc = T(0), dD_acc = T(0);
  int fcount = 0;  // rows pushed through the forward ring (ring phase bookkeeping)
  int rcount = 0;  // rows pushed through the reverse ring

  for (int b = pl.nb - 1; b >= 0; --b) {
    const int r0 = b * K;
    const int r1 = min(H, r0 + K);
    // ================================================= phase F (recompute)
    T hv[J];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      const int j = g.col0 + k;
      hv[k] = (b > 0 && g.st_ok && j < W)
                  ? a.ckpt[((static_cast<size_t>(s) * nbm1 + (b - 1)) * W + j) * N + g.l]
                  : T(0);
      hb[k * 32 + lane] = hv[k];
    }
    RowInB<T, LPC, J> cur, nxt;
    load_row_b<T, LPC, J>(cur, xs, zs, Bs, Cs, dys, r0, W, N, g, false);
    for (int i = r0; i < r1; ++i) {
      if (i + 1 < r1) load_row_b<T, LPC, J>(nxt, xs, zs, Bs, Cs, dys, i + 1, W, N, g, false);
      T delta[J], sig[J], av[J], uv[J];
      chunk_delta_sig<T, LPC, J>(cur.zz, bias, lane, delta, sig, false);
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
      T Pi = Pc, Li = Lc;
      chunk_scan_fwd<T, LPC>(Pi, Li, g.lane_in_seg, pl.cps * LPC, g.segw);
      T Pe = __shfl_up_sync(kFull, Pi, LPC, g.segw);
      T Le = __shfl_up_sync(kFull, Li, LPC, g.segw);
      if (g.lane_in_seg < LPC) {
        Pe = T(1);
        Le = T(0);
      }
      const int slot = fcount % kRing;
      const uint32_t par = static_cast<uint32_t>(fcount / kRing) & 1u;
      ++fcount;
      T ew = T(0);
      if (has_pred) {
        if (!pred_global) {
          mbar_wait(&ring_f.full[slot], par);
          ew = ring_f.data[slot][g.l];
          mbar_arrive(&ring_f.empty[slot]);
        } else {
          ew = g.l < N ? hc_in[static_cast<size_t>(i) * N + g.l] : T(0);
        }
      }
      if (has_succ && !succ_global) {
        const T Pt = __shfl_sync(kFull, Pi, (pl.cpw - 1) * LPC + g.l);
        const T Lt = __shfl_sync(kFull, Li, (pl.cpw - 1) * LPC + g.l);
        const T out = fma(Pt, ew, Lt);
        mbar_wait(&next_ring_f->empty[slot], par ^ 1u);
        if (g.chunk == 0) next_ring_f->data[slot][g.l] = out;
        mbar_arrive(&next_ring_f->full[slot]);
      }
      T hh = fma(Pe, ew, Le);
      ec[(i - r0) * 32 + lane] = hh;
      T* hrow = hb + static_cast<size_t>(i - r0 + 1) * J * 32;
#pragma unroll
      for (int k = 0; k < J; ++k) {
        hh = fma(av[k], hh, uv[k]);
        hv[k] = fma(av[k], hv[k], hh);
        hrow[k * 32 + lane] = hv[k];
      }
      if (i + 1 < r1) cur = nxt;
    }
    __syncwarp();
    // ================================================= phase R (adjoints)
    load_row_b<T, LPC, J>(cur, xs, zs, Bs, Cs, dys, r1 - 1, W, N, g, true);
    for (int i = r1 - 1; i >= r0; --i) {
      if (i - 1 >= r0) load_row_b<T, LPC, J>(nxt, xs, zs, Bs, Cs, dys, i - 1, W, N, g, true);
      T delta[J], sig[J], av[J], uv[J], G[J], Gh[J];
      chunk_delta_sig<T, LPC, J>(cur.zz, bias, lane, delta, sig, true);
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const bool ok = g.scan_ok && (g.col0 + k) < W;
        av[k] = ok ? Num<T>::exp_scaled(delta[k] * A2) : T(1);
        uv[k] = (delta[k] * cur.b[k]) * cur.x[k];
        G[k] = fma(cur.c[k], cur.dy[k], dn[k]);  // engine.cpp:321
      }
      // chunk's reverse affine map rho_out = al rho_in + be (engine.cpp:343-350)
      T al = av[0], be;
      {
        T r = T(0);
#pragma unroll
        for (int k = J - 1; k >= 0; --k) {
          const T gh = G[k] + r;
          r = av[k] * gh;
        }
        be = r;
#pragma unroll
        for (int k = 1; k < J; ++k) al = al * av[k];
      }
      T ai = al, bi = be;
      chunk_scan_rev<T, LPC>(ai, bi, g.lane_in_seg, pl.cps * LPC, g.segw);
      T ae = __shfl_down_sync(kFull, ai, LPC, g.segw);
      T bx = __shfl_down_sync(kFull, bi, LPC, g.segw);
      if (g.lane_in_seg + LPC >= pl.cps * LPC) {
        ae = T(1);
        bx = T(0);
      }
      const int slot = rcount % kRing;
      const uint32_t par = static_cast<uint32_t>(rcount / kRing) & 1u;
      ++rcount;
      T rw = T(0);
      if (has_succ) {
        if (!succ_global) {
          mbar_wait(&ring_r.full[slot], par);
          rw = ring_r.data[slot][g.l];
          mbar_arrive(&ring_r.empty[slot]);
        } else {
          if (rseen <= H - 1 - i) rseen = wait_flag_gt(rprog_in, H - 1 - i);
          rw = g.l < N ? ld_relaxed_gpu(rc_in + static_cast<size_t>(i) * N + g.l) : T(0);
        }
      }
      if (has_pred) {
        const T at = __shfl_sync(kFull, ai, g.l);  // chunk 0 holds the warp aggregate
        const T bt = __shfl_sync(kFull, bi, g.l);
        const T out = fma(at, rw, bt);
        if (!pred_global) {
          mbar_wait(&prev_ring_r->empty[slot], par ^ 1u);
          if (g.chunk == 0) prev_ring_r->data[slot][g.l] = out;
          mbar_arrive(&prev_ring_r->full[slot]);
        } else {
          if (g.chunk == 0 && g.l < N) {
            rc_out[static_cast<size_t>(i) * N + g.l] = out;
            __threadfence();
          }
          __syncwarp();
          if (lane == 0) st_release_gpu(rprog_out, H - i);
        }
      }
      {
        T r = fma(ae, rw, bx);
#pragma unroll
        for (int k = J - 1; k >= 0; --k) {
          Gh[k] = G[k] + r;
          r = av[k] * Gh[k];
        }
      }
      // chain rule (engine.cpp:355-397)
      const T* hup = hb + static_cast<size_t>(i - r0) * J * 32;
      const T* hcur = hup + J * 32;
      T hl = ec[(i - r0) * 32 + lane];
      T ddp[J], sgb[J];
      const size_t rowb = static_cast<size_t>(i) * W;
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const int j = g.col0 + k;
        const bool ok = g.st_ok && j < W;
        const T dab = fma(Gh[k], hl, G[k] * hup[k * 32 + lane]);
        hl = fma(av[k], hl, uv[k]);
        if (ok) dA_acc = fma(dab, delta[k] * av[k], dA_acc);
        ddp[k] = fma(Gh[k], cur.b[k] * cur.x[k], dab * (av[k] * Ad));
        sgb[k] = Gh[k] * cur.b[k];
        if (ok) {
          dBs[(rowb + j) * N + g.l] = Gh[k] * (delta[k] * cur.x[k]);
          dCs[(rowb + j) * N + g.l] = cur.dy[k] * hcur[k * 32 + lane];
        }
        dn[k] = av[k] * G[k];
      }
      const int cbase = reduce_scatter<LPC, J>(ddp, g.l);
      reduce_scatter<LPC, J>(sgb, g.l);
      if ((g.l & (RS_::kReplica - 1)) == 0 && g.scan_ok) {
#pragma unroll
        for (int m = 0; m < RS_::kKeep; ++m) {
          const int k = cbase + m;
          const int j = g.col0 + k;
          if (j < W) {
            const T dyv = select_col<J>(cur.dy, k), xv = select_col<J>(cur.x, k);
            const T dv = select_col<J>(delta, k), sv = select_col<J>(sig, k);
            const T dzv = ddp[m] * sv;
            dxs[rowb + j] = fma(Dsk, dyv, dv * sgb[m]);
            dzs[rowb + j] = dzv;
            dbias_acc += dzv;
            dD_acc = fma(dyv, xv, dD_acc);
          }
        }
      }
      if (i - 1 >= r0) cur = nxt;
    }
    __syncwarp();
  }

  // ---- per-(scan, warp) partials, reduced in a fixed order
  for (int h = LPC; h < g.segw; h <<= 1) dA_acc += __shfl_xor_sync(kFull, dA_acc, h);
  for (int h = 1; h < g.segw; h <<= 1) {
    dbias_acc += __shfl_xor_sync(kFull, dbias_acc, h);
    dD_acc += __shfl_xor_sync(kFull, dD_acc, h);
  }
  if (g.scan_ok) {
    T* part = a.part + (static_cast<size_t>(g.s) * pl.wps + g.wpos) * (N + 2);
    if (g.lane_in_seg < LPC && g.l < N) part[g.l] = dA_acc;
    if (g.lane_in_seg == 0) {
      part[N] = dbias_acc;
      part[N + 1] = dD_acc;
    }
  }
}

// dA[p][d], dbias[p], dD[p]: sum over scans s = p, p + P, ... (ascending) and
// their warps (ascending) -- the fixed order of engine.cpp:404-408.
template <typename T>
__global__ void scan2d_reduce_params_kernel(const T* __restrict__ part, int64_t S, int wps,
                                            int wreal, int P, int N, T* dA, T* dbias, T* dD) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(P) * (N + 2);
  if (t >= total) return;
  const int p = static_cast<int>(t / (N + 2)), q = static_cast<int>(t % (N + 2));
  T acc = T(0);
  for (int64_t s = p; s < S; s += P)
    for (int w = 0; w < wreal; ++w) acc += part[(s * wps + w) * (N + 2) + q];
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
