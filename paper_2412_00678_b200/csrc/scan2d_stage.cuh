// scan2d_stage.cuh -- per-warp row staging through shared memory (cp.async).
//
// A warp needs, per row, its column slice of the per-scan arrays (x, z, and dy
// in the backward) and of the per-state arrays (B, C): a handful of short
// contiguous spans (several when narrow scans are packed into one warp).  The
// spans are identical for every row up to a constant row stride, so each lane
// builds once a small table of its copy units (16-byte units when every span
// is 16-byte aligned, else element units) and replays it per row: one
// table load, one address add and one LDGSTS per unit.
//
// Stage layout (elements, per packed segment):  X | Z | DY | B | C, with the
// state dimension padded to Np = next_pow2(N) in B / C so that lanes owning
// padded states read zeros (no masks in the inner loops); the ring is zeroed
// once, and positions no span ever writes stay zero.
#pragma once

#include "scan2d_common.cuh"

namespace s2d {

struct CopyEntry {
  int dst;  // element offset within the stage (relative to the X or B region base)
  int src;  // element offset relative to the row base of the warp's first scan
};

template <typename T>
struct StageLayout {
  int xo, zo, dyo, bo, co, seg_stride;
  __host__ __device__ static int pad(int n) {
    const int e = 16 / static_cast<int>(sizeof(T));
    return (n + e - 1) / e * e;
  }
  __host__ __device__ StageLayout(int colsw, int Np, bool with_dy) {
    const int pc = pad(colsw), pb = pad(colsw * Np);
    xo = 0;
    zo = pc;
    dyo = 2 * pc;
    bo = (with_dy ? 3 : 2) * pc;
    co = bo + pb;
    seg_stride = co + pb;
  }
  __host__ __device__ static int stage_elems(int colsw, int Np, int seg, bool with_dy) {
    StageLayout L(colsw, Np, with_dy);
    return L.seg_stride * seg;
  }
};

// number of table entries per lane for the x-like / B-like spans of a warp
__host__ __device__ inline int stage_units_x(int seg, int ncols, bool vec, int epv) {
  const int per = vec ? ncols / epv : ncols;
  return (seg * per + 31) / 32;
}
__host__ __device__ inline int stage_units_b(int seg, int ncols, int N, bool vec, int epv) {
  const int per = vec ? ncols * N / epv : ncols * N;
  return (seg * per + 31) / 32;
}

template <typename T>
struct Stager {
  static constexpr int EPV = 16 / static_cast<int>(sizeof(T));
  const CopyEntry* xt;
  const CopyEntry* bt;
  int nx, nb;
  bool xvec, bvec;
  int zoff, dyoff, coff;  // Z, DY, C region offsets relative to X / B
  // row-0 bases of the warp's first scan
  const T* x0;
  const T* z0;
  const T* dy0;
  const T* B0;
  const T* C0;
  size_t xstride, bstride;
  int xc0, bc0;  // column offset of the warp's window in x-like / B-like rows (static path)

  // Build the lane's table (once).  seg_scans: scans present in this warp
  // (>= 1), c0 / ncols: column window, N / Np: states and padded states.
  __device__ void build(CopyEntry* table, int lane, int seg_scans, int c0, int ncols, int N, int Np,
                        size_t HW, const StageLayout<T>& L, int64_t s0, int G) {
    xt = table;
    xc0 = c0;
    bc0 = c0 * N;
    const int xper = xvec ? ncols / EPV : ncols;
    const int xtot = seg_scans * xper;
    nx = (xtot + 31) / 32;
    for (int m = 0; m < nx; ++m) {
      const int idx = m * 32 + lane;
      CopyEntry e{-1, 0};
      if (idx < xtot) {
        const int g = idx / xper, u = idx % xper;
        const int col = xvec ? u * EPV : u;
        e.dst = g * L.seg_stride + L.xo + col;
        e.src = static_cast<int>(g * HW) + c0 + col;
      }
      table[m * 32 + lane] = e;
    }
    CopyEntry* btw = table + nx * 32;
    bt = btw;
    const int bper = bvec ? ncols * N / EPV : ncols * N;
    const int btot = seg_scans * bper;
    nb = (btot + 31) / 32;
    const int64_t g0 = s0 / G;
    for (int m = 0; m < nb; ++m) {
      const int idx = m * 32 + lane;
      CopyEntry e{-1, 0};
      if (idx < btot) {
        const int g = idx / bper, u = idx % bper;
        const int el = bvec ? u * EPV : u;  // element within the (ncols x N) span
        const int col = el / N, d = el % N;
        const int64_t grp = (s0 + g) / G - g0;
        e.dst = g * L.seg_stride + L.bo + col * Np + d;
        e.src = static_cast<int>(grp * HW * N) + c0 * N + el;
      }
      btw[m * 32 + lane] = e;
    }
    __syncwarp();
  }

  // Static fast path (one unpacked scan per warp, 16-byte units legal): lane
  // copies x/z unit `lane` and B/C units lane + 32 m, m < MB = J*SPL/4, all
  // with immediate offsets; `stage_addr` is the shared address of the stage.
  template <int MX, int MB>
  __device__ __forceinline__ void issue_static(uint32_t stage_addr, int r, int lane, int xunits, int bunits,
                                               const StageLayout<T>& L, bool with_dy, bool with_c) const {
    constexpr int es = static_cast<int>(sizeof(T));
    const T* xs = x0 + r * xstride + xc0 + lane * EPV;
    const T* zs = z0 + r * xstride + xc0 + lane * EPV;
    const uint32_t xd = stage_addr + (L.xo + lane * EPV) * es;
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      if (lane + 32 * m < xunits) {
        cp_async16_raw(xd + m * 512, xs + m * 32 * EPV);
        cp_async16_raw(xd + zoff * es + m * 512, zs + m * 32 * EPV);
        if (with_dy)
          cp_async16_raw(xd + dyoff * es + m * 512, dy0 + r * xstride + xc0 + lane * EPV + m * 32 * EPV);
      }
    }
    const T* bs = B0 + r * bstride + bc0 + lane * EPV;
    const T* cs = C0 + r * bstride + bc0 + lane * EPV;
    const uint32_t bd = stage_addr + (L.bo + lane * EPV) * es;
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      if (lane + 32 * m < bunits) {
        cp_async16_raw(bd + m * 512, bs + m * 32 * EPV);
        if (with_c) cp_async16_raw(bd + coff * es + m * 512, cs + m * 32 * EPV);
      }
    }
  }

  // Issue the copies of row r into stage `stage` (x, z always; dy / C when
  // requested).
  __device__ __forceinline__ void issue(T* stage, int r, int lane, bool with_dy, bool with_c) const {
    const T* xr = x0 + r * xstride;
    const T* zr = z0 + r * xstride;
    const T* dyr = dy0 + r * xstride;
    for (int m = 0; m < nx; ++m) {
      const CopyEntry e = xt[m * 32 + lane];
      if (e.dst < 0) continue;
      if (xvec) {
        cp_async16(stage + e.dst, xr + e.src);
        cp_async16(stage + e.dst + zoff, zr + e.src);
        if (with_dy) cp_async16(stage + e.dst + dyoff, dyr + e.src);
      } else {
        cp_async_elem(stage + e.dst, xr + e.src);
        cp_async_elem(stage + e.dst + zoff, zr + e.src);
        if (with_dy) cp_async_elem(stage + e.dst + dyoff, dyr + e.src);
      }
    }
    const T* Br = B0 + r * bstride;
    const T* Cr = C0 + r * bstride;
    for (int m = 0; m < nb; ++m) {
      const CopyEntry e = bt[m * 32 + lane];
      if (e.dst < 0) continue;
      if (bvec) {
        cp_async16(stage + e.dst, Br + e.src);
        if (with_c) cp_async16(stage + e.dst + coff, Cr + e.src);
      } else {
        cp_async_elem(stage + e.dst, Br + e.src);
        if (with_c) cp_async_elem(stage + e.dst + coff, Cr + e.src);
      }
    }
  }
};

}  // namespace s2d
