// scan2d_rows1.cuh -- "row sweep" forward and backward kernels for N = 1
// (the VMamba-style configurations: 7x7 ... 56x56 grids, one state).
//
// Same recurrences as the reference (reference.cpp:85-112, engine.cpp:304-397)
// with a single state, so there is no state dimension to spread over lanes:
//  * one warp owns whole scans -- SPW = 32 / SEG of them side by side (2 x 56,
//    4 x 28, 4 x 14, 4 x 7 columns) -- and walks the rows top to bottom; lane
//    q of a segment owns J consecutive columns (16 / 8 / 4-byte loads), so a row
//    of x, z, B, C is one coalesced load per operand, straight into registers
//    several rows ahead.  No shared memory, no inter-warp carries;
//  * horizontal scan per row: the lane folds its J cells into one affine pair
//    (prod Abar, local hh), a shuffle scan over the segment's lanes (the
//    SegmentedBlockScan of PAPER.md:137, block_scan.cpp:14-51: segments are
//    shuffle widths) gives each lane its carry-in, then J FMAs finish hh;
//  * the vertical state h of the lane's columns stays in registers;
//  * the training forward checkpoints h every K = 4 rows; the backward walks
//    4-row bands bottom-up: re-runs the band forward from the checkpoint
//    (keeping hh and h of the band in registers), then walks it bottom-up with
//    G (vertical) in registers and Gh by a reverse shuffle scan, and applies
//    the chain rule.  Loads run one row-job ahead in ping-pong registers.
#pragma once

#include "scan2d_fwd.cuh"
#include "scan2d_tile2.cuh"

namespace s2d {

constexpr int kRows1K = 4;  // checkpoint interval (rows) of the N = 1 kernels

template <typename T, int J>
__device__ __forceinline__ void ldg_row(T (&v)[J], const T* p, bool ok) {
  if (ok) {
    ldg_states<T, J>(v, p);
  } else {
#pragma unroll
    for (int k = 0; k < J; ++k) v[k] = T(0);
  }
}

template <typename T, int J>
__device__ __forceinline__ void stg_row(T* p, const T (&v)[J]) {
  stg_stream<T, J>(p, v);
}

// Bulk L2 prefetch (TMA unit, SASS UBLKPF) of rows [r0, r1) of one scan's map:
// one contiguous span, widened to 16-byte boundaries.
template <typename T>
__device__ __forceinline__ void bulk_rows_l2(const T* map, int r0, int r1, int W) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(map + static_cast<size_t>(r0) * W) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(map + static_cast<size_t>(r1) * W) + 15) & ~uintptr_t(15);
  if (a1 > a0) bulk_prefetch_l2(reinterpret_cast<const void*>(a0), static_cast<uint32_t>(a1 - a0));
}

// inclusive segmented scan of affine pairs (a, b): element q composed after q-1
template <typename T, int SEG>
__device__ __forceinline__ void seg_scan_fwd(T& ap, T& b, int q) {
#pragma unroll
  for (int off = 1; off < SEG; off <<= 1) {
    const T a2 = __shfl_up_sync(kFull, ap, off, SEG);
    const T b2 = __shfl_up_sync(kFull, b, off, SEG);
    if (q >= off) {
      b = fma(ap, b2, b);
      ap *= a2;
    }
  }
}
// the same from the right (reverse horizontal recurrence of the backward)
template <typename T, int SEG>
__device__ __forceinline__ void seg_scan_rev(T& ap, T& b, int q) {
#pragma unroll
  for (int off = 1; off < SEG; off <<= 1) {
    const T a2 = __shfl_down_sync(kFull, ap, off, SEG);
    const T b2 = __shfl_down_sync(kFull, b, off, SEG);
    if (q + off < SEG) {
      b = fma(ap, b2, b);
      ap *= a2;
    }
  }
}

struct Rows1Id {
  int64_t s;
  int q, seg;
  bool ok;
};

template <int SEG>
__device__ __forceinline__ Rows1Id rows1_id(int64_t S, int WJ) {
  constexpr int SPW = 32 / SEG;
  Rows1Id id;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  id.seg = lane / SEG;
  id.q = lane % SEG;
  id.s = warp * SPW + id.seg;
  id.ok = id.s < S && id.q < WJ;
  return id;
}

// ================================================================== forward

template <typename T, int J, int SEG, bool ACC = false>
__global__ void __launch_bounds__(128) scan2d_fwd_rows1_kernel(const Args<T> a) {
  using F = Fn<T, ACC>;
  constexpr int K = kRows1K;
  const int H = a.H, W = a.W, WJ = W / J;
  const Rows1Id id = rows1_id<SEG>(a.S, WJ);
  const int q = id.q;
  const int64_t s = id.s < a.S ? id.s : a.S - 1;
  const bool ok = id.ok;
  const int p = param_row(s, a.S, a.P);
  const T A1 = F::a_scale(a.A[p]), Dsk = a.Dskip[p], bias = a.bias[p];
  const size_t HW = static_cast<size_t>(H) * W;
  const T* xg = a.x + s * HW + q * J;
  const T* zg = a.z + s * HW + q * J;
  const T* Bg = a.B + bc_row(s, a.G) * HW + q * J;
  const T* Cg = a.C + bc_row(s, a.G) * HW + q * J;
  T* yg = a.y + s * HW + q * J;
  T* ck = a.ckpt == nullptr ? nullptr : a.ckpt + static_cast<size_t>(s) * (a.plan.nb - 1) * W + q * J;
  T h[J];
#pragma unroll
  for (int k = 0; k < J; ++k) h[k] = T(0);
  if (a.vtop != nullptr && ok) ldg_states<T, J>(h, a.vtop + s * W + q * J);

  // K rows in flight: static register slots (loop unrolled by K)
  T xs[K][J], zs[K][J], bs[K][J], cs[K][J];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const bool rv = ok && r < H;
    const size_t o = static_cast<size_t>(r) * W;
    ldg_row<T, J>(xs[r], xg + o, rv);
    ldg_row<T, J>(zs[r], zg + o, rv);
    ldg_row<T, J>(bs[r], Bg + o, rv);
    ldg_row<T, J>(cs[r], Cg + o, rv);
  }
  for (int i0 = 0; i0 < H; i0 += K) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int i = i0 + r;
      if (i < H) {  // warp-uniform
        T d[J], av[J], u[J];
        T hl = T(0), ap = T(1);
#pragma unroll
        for (int k = 0; k < J; ++k) {
          d[k] = F::softplus(zs[r][k] + bias);
          av[k] = ok ? F::exp_scaled(d[k] * A1) : T(1);
          u[k] = (d[k] * bs[r][k]) * xs[r][k];  // math.hpp:86-89
          hl = fma(av[k], hl, u[k]);
          ap *= av[k];
        }
        seg_scan_fwd<T, SEG>(ap, hl, q);
        T hh = __shfl_up_sync(kFull, hl, 1, SEG);
        if (q == 0) hh = T(0);
        T y[J];
#pragma unroll
        for (int k = 0; k < J; ++k) {
          hh = fma(av[k], hh, u[k]);
          h[k] = fma(av[k], h[k], hh);
          y[k] = fma(Dsk, xs[r][k], cs[r][k] * h[k]);
        }
        if (ok) {
          stg_row<T, J>(yg + static_cast<size_t>(i) * W, y);
          if (ck != nullptr && r == K - 1 && i < H - 1) stg_row<T, J>(ck + static_cast<size_t>(i / K) * W, h);
          if (a.vbot != nullptr && i == H - 1) stg_row<T, J>(a.vbot + s * W + q * J, h);
        }
        // L2 prefetch: bulk spans of 2K rows, 2K..4K rows ahead (K..4K at the
        // start), by each scan's first lane (pf_mode 2); or row i + pfd line by line.  Then refill this
        // slot with row i + K.
        if (a.plan.pf_mode == 2) {
          if (r == 0 && (i0 % (2 * K)) == 0 && q == 0 && ok && i0 + K < H) {
            const int p0 = i0 == 0 ? K : i0 + 2 * K, p1 = min(H, i0 + 4 * K);
            const T* xm = xg - q * J;
            bulk_rows_l2(xm, p0, p1, W);
            bulk_rows_l2(zg - q * J, p0, p1, W);
            bulk_rows_l2(Bg - q * J, p0, p1, W);
            bulk_rows_l2(Cg - q * J, p0, p1, W);
          }
        } else if (ok && i + a.plan.pfd < H) {
          const size_t o2 = static_cast<size_t>(i + a.plan.pfd) * W;
          prefetch_l2(xg + o2);
          prefetch_l2(zg + o2);
          prefetch_l2(Bg + o2);
          prefetch_l2(Cg + o2);
        }
        const int in = i + K;
        const bool rv = ok && in < H;
        const size_t o = static_cast<size_t>(rv ? in : 0) * W;
        ldg_row<T, J>(xs[r], xg + o, rv);
        ldg_row<T, J>(zs[r], zg + o, rv);
        ldg_row<T, J>(bs[r], Bg + o, rv);
        ldg_row<T, J>(cs[r], Cg + o, rv);
      }
    }
  }
}

// ================================================================= backward

template <typename T, int J>
struct Rows1Job {
  T x[J], z[J], b[J], c[J], dy[J];
};

// one lane's J elements, global -> shared, zero-filled when !ok (cp.async .ca
// takes 4 / 8 / 16 bytes: the lane's own columns, no cross-lane traffic)
template <typename T, int J>
__device__ __forceinline__ void cp_lane(uint32_t sdst, const T* g, bool ok) {
  constexpr int BYTES = J * static_cast<int>(sizeof(T));
  constexpr int PIECE = BYTES < 16 ? BYTES : 16;
  static_assert(PIECE == 4 || PIECE == 8 || PIECE == 16, "cp.async size");
  const int src = ok ? PIECE : 0;
#pragma unroll
  for (int o = 0; o < BYTES; o += PIECE)
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(sdst + o),
                 "l"(reinterpret_cast<const char*>(g) + o), "n"(PIECE), "r"(src)
                 : "memory");
}

template <typename T, int J>
__device__ __forceinline__ void load_job(Rows1Job<T, J>& jb, const T* xg, const T* zg, const T* Bg, const T* Cg,
                                         const T* yg, int row, int H, int W, bool ok, bool rev) {
  const bool rv = ok && row >= 0 && row < H;
  const size_t o = static_cast<size_t>(rv ? row : 0) * W;
  ldg_row<T, J>(jb.x, xg + o, rv);
  ldg_row<T, J>(jb.z, zg + o, rv);
  ldg_row<T, J>(jb.b, Bg + o, rv);
  if (rev) {
    ldg_row<T, J>(jb.c, Cg + o, rv);
    ldg_row<T, J>(jb.dy, yg + o, rv);
  }
}

template <typename T, int J, int SEG, bool ACC = false>
__global__ void __launch_bounds__(128, 4) scan2d_bwd_rows1_kernel(const Args<T> a) {
  using F = Fn<T, ACC>;
  constexpr int K = kRows1K;
  const int H = a.H, W = a.W, WJ = W / J;
  const Rows1Id id = rows1_id<SEG>(a.S, WJ);
  const int q = id.q;
  const int64_t s = id.s < a.S ? id.s : a.S - 1;
  const bool ok = id.ok;
  const int p = param_row(s, a.S, a.P);
  const T A1 = F::a_scale(a.A[p]), Dsk = a.Dskip[p], bias = a.bias[p];
  const T Au = a.A[p];  // A itself (A1 = A log2 e feeds ex2)
  const size_t HW = static_cast<size_t>(H) * W;
  const size_t off = s * HW + q * J;
  const T* xg = a.x + off;
  const T* zg = a.z + off;
  const T* Bg = a.B + bc_row(s, a.G) * HW + q * J;
  const T* Cg = a.C + bc_row(s, a.G) * HW + q * J;
  const T* yg = a.dy + off;
  T* dxg = a.dx + off;
  T* dzg = a.dz + off;
  T* dBg = a.dB + off;
  T* dCg = a.dC + off;
  const int nb = (H + K - 1) / K;
  const T* ck = a.ckpt + static_cast<size_t>(s) * (a.plan.nb - 1) * W + q * J;

  T dn[J];  // Abar(i+1) G(i+1) per column, carried up
#pragma unroll
  for (int k = 0; k < J; ++k) dn[k] = T(0);
  if (a.gbot != nullptr && ok) ldg_states<T, J>(dn, a.gbot + s * W + q * J);
  // per-scan scalar sums over every cell: accumulate in double
  double dA_acc = 0.0, db_acc = 0.0, dD_acc = 0.0;

  // job order per band: F rows r0 .. r0+K-1, then R rows r0+K-1 .. r0.  Each
  // lane streams its own columns of the next NJ-1 row-jobs into a private
  // shared-memory ring with cp.async (no registers held for the prefetch).
  constexpr int NJ = J * sizeof(T) > 16 ? 2 : 4;  // static smem <= 48 KB (fp64 J = 4 never runs)
  static_assert((2 * K) % NJ == 0, "job slots must tile a band");
  __shared__ __align__(16) T ring[4][NJ][5][32][J];  // [warp in CTA][slot][operand][lane][J]
  T(*my)[5][32][J] = ring[(threadIdx.x >> 5) & 3];
  const int lane = threadIdx.x & 31;
  // job jj counted from band bb's first job (jj >= 2K: the band above)
  auto issue = [&](int bb, int jj) {
    const int band = bb - jj / (2 * K), loc = jj % (2 * K);
    const bool rev = loc >= K;
    const int row = band * K + (rev ? 2 * K - 1 - loc : loc);
    const bool rv = ok && band >= 0 && row >= 0 && row < H;
    const int o = rv ? row * W : 0;
    T(*sl)[32][J] = my[jj % NJ];
    cp_lane<T, J>(smem_u32(sl[0][lane]), xg + o, rv);
    cp_lane<T, J>(smem_u32(sl[1][lane]), zg + o, rv);
    cp_lane<T, J>(smem_u32(sl[2][lane]), Bg + o, rv);
    if (rev) {
      cp_lane<T, J>(smem_u32(sl[3][lane]), Cg + o, rv);
      cp_lane<T, J>(smem_u32(sl[4][lane]), yg + o, rv);
    }
    cp_async_commit();
  };
  auto fetch = [&](int jj, Rows1Job<T, J>& jb, bool rev) {
    cp_async_wait<NJ - 1>();
    T(*sl)[32][J] = my[jj % NJ];
    lds_vec<T, J>(jb.x, sl[0][lane]);
    lds_vec<T, J>(jb.z, sl[1][lane]);
    lds_vec<T, J>(jb.b, sl[2][lane]);
    if (rev) {
      lds_vec<T, J>(jb.c, sl[3][lane]);
      lds_vec<T, J>(jb.dy, sl[4][lane]);
    }
  };
#pragma unroll
  for (int jj = 0; jj < NJ - 1; ++jj) issue(nb - 1, jj);
  for (int b = nb - 1; b >= 0; --b) {
    const int r0 = b * K;
    T hp0[J];  // h of the row above the band (checkpoint / band carry / zeros)
#pragma unroll
    for (int k = 0; k < J; ++k) hp0[k] = T(0);
    if (ok) {
      if (b > 0)
        ldg_states<T, J>(hp0, ck + (b - 1) * W);
      else if (a.vtop != nullptr)
        ldg_states<T, J>(hp0, a.vtop + s * W + q * J);
    }
    T hhr[K][J], hr[K][J];
    // ---- F: re-run the band's forward
    {
      T hcur[J];
#pragma unroll
      for (int k = 0; k < J; ++k) hcur[k] = hp0[k];
#pragma unroll
      for (int r = 0; r < K; ++r) {
        issue(b, r + NJ - 1);
        Rows1Job<T, J> cur;
        fetch(r, cur, false);
        T av[J], u[J];
        T hl = T(0), ap = T(1);
#pragma unroll
        for (int k = 0; k < J; ++k) {
          const T d = F::softplus(cur.z[k] + bias);
          av[k] = ok ? F::exp_scaled(d * A1) : T(1);
          u[k] = (d * cur.b[k]) * cur.x[k];
          hl = fma(av[k], hl, u[k]);
          ap *= av[k];
        }
        seg_scan_fwd<T, SEG>(ap, hl, q);
        T hh = __shfl_up_sync(kFull, hl, 1, SEG);
        if (q == 0) hh = T(0);
#pragma unroll
        for (int k = 0; k < J; ++k) {
          hh = fma(av[k], hh, u[k]);
          hhr[r][k] = hh;
          hcur[k] = fma(av[k], hcur[k], hh);
          hr[r][k] = hcur[k];
        }
      }
    }
    // ---- R: bottom-up through the band; G vertical, Gh by a reverse scan
#pragma unroll
    for (int rr = K - 1; rr >= 0; --rr) {
      const int jidx = K + (K - 1 - rr);  // job index within the band: K .. 2K-1
      issue(b, jidx + NJ - 1);
      Rows1Job<T, J> cur;
      fetch(jidx, cur, true);
      const int i = r0 + rr;
      T d[J], av[J], sg[J], G[J];
      T rl = T(0), ap = T(1);  // lane aggregate of the reverse horizontal map
#pragma unroll
      for (int k = 0; k < J; ++k) {
        const T v = cur.z[k] + bias;
        d[k] = F::softplus(v);
        sg[k] = F::sigmoid(v);
        av[k] = ok ? F::exp_scaled(d[k] * A1) : T(1);
        if (i < H) {  // rows past the grid (bottom band) stay inert
          G[k] = fma(cur.c[k], cur.dy[k], dn[k]);  // engine.cpp:321
          dn[k] = av[k] * G[k];
        } else {
          G[k] = T(0);
        }
      }
#pragma unroll
      for (int k = J - 1; k >= 0; --k) {  // rho(j) = Abar(j) (G(j) + rho(j+1))
        rl = av[k] * (G[k] + rl);
        ap *= av[k];
      }
      seg_scan_rev<T, SEG>(ap, rl, q);
      T rho = __shfl_down_sync(kFull, rl, 1, SEG);  // carry from the lanes to the right
      if (q == SEG - 1) rho = T(0);
      T hl_prev = __shfl_up_sync(kFull, hhr[rr][J - 1], 1, SEG);  // hh(i, j-1) of column 0
      if (q == 0) hl_prev = T(0);
      T dx[J], dz[J], dB[J], dC[J];
#pragma unroll
      for (int k = J - 1; k >= 0; --k) {
        const T gh = G[k] + rho;  // engine.cpp:346
        rho = av[k] * gh;
        const T hl = k > 0 ? hhr[rr][k > 0 ? k - 1 : 0] : hl_prev;
        const T hu = rr > 0 ? hr[rr > 0 ? rr - 1 : 0][k] : hp0[k];
        const T dab = fma(gh, hl, G[k] * hu);  // engine.cpp:383
        const T t = dab * av[k];
        dA_acc = fma(static_cast<double>(t), static_cast<double>(d[k]), dA_acc);
        const T gb = gh * cur.b[k];
        const T dd = fma(t, Au, gb * cur.x[k]);
        dB[k] = gh * (d[k] * cur.x[k]);
        dC[k] = cur.dy[k] * hr[rr][k];
        dx[k] = fma(Dsk, cur.dy[k], d[k] * gb);
        dz[k] = dd * sg[k];
        if (ok && i < H) {
          db_acc += static_cast<double>(dz[k]);
          dD_acc = fma(static_cast<double>(cur.dy[k]), static_cast<double>(cur.x[k]), dD_acc);
        }
      }
      if (ok && i < H) {
        const int o = i * W;
        stg_row<T, J>(dxg + o, dx);
        stg_row<T, J>(dzg + o, dz);
        stg_row<T, J>(dBg + o, dB);
        stg_row<T, J>(dCg + o, dC);
      }
    }
  }
  if (a.gtop != nullptr && ok) stg_row<T, J>(a.gtop + s * W + q * J, dn);
  // per-scan partials: sum over the segment's lanes (fixed butterfly order)
#pragma unroll
  for (int o = 1; o < SEG; o <<= 1) {
    dA_acc += __shfl_xor_sync(kFull, dA_acc, o, SEG);
    db_acc += __shfl_xor_sync(kFull, db_acc, o, SEG);
    dD_acc += __shfl_xor_sync(kFull, dD_acc, o, SEG);
  }
  if (q == 0 && id.s < a.S) {
    if (a.fuse) {  // P == S: one warp segment owns the scan -- write the gradients directly
      a.dA_out[id.s] = static_cast<T>(dA_acc);
      a.dbias_out[id.s] = static_cast<T>(db_acc);
      a.dD_out[id.s] = static_cast<T>(dD_acc);
    } else {
      T* part = a.part + static_cast<size_t>(id.s) * 3;  // [S][1][N + 2], N = 1
      part[0] = static_cast<T>(dA_acc);
      part[1] = static_cast<T>(db_acc);
      part[2] = static_cast<T>(dD_acc);
    }
  }
}

}  // namespace s2d
