// scan2d_tile2.cuh -- register-streamed "tile-transpose" forward and backward
// kernels for N in {4, 8, 16, 32} (sm_100a).
//
// Same recurrences as the reference engine (reference.cpp:85-112,
// engine.cpp:103-121 / :196-216 forward, engine.cpp:304-397 backward):
//   hh(i,j) = fma(Abar, hh(i,j-1), Bbar x)      h(i,j) = fma(Abar, h(i-1,j), hh(i,j))
//   y(i,j)  = D x + sum_d C h
//   G  = fma(C, dy, Abar(i+1,j) G(i+1,j))      Gh = G + Abar(i,j+1) Gh(i,j+1)
//   dAbar = Gh hh(i,j-1) + G h(i-1,j);  dA += dAbar delta Abar;  ddelta = sum_d dAbar Abar A + Gh B x
//   dB = Gh delta x;  dC = dy h;  dx = D dy + delta sum_d Gh B;  dz = ddelta sigmoid(z+bias)
//
// Decomposition (one warp = one 16-column STRIP of one scan, walking the strip
// in tiles of R rows; R * N / SH = 32):
//  * row lanes (r, q) own row r of the tile and SH consecutive states: they run
//    the horizontal recurrences (hh forward, Gh backward) with the carry in
//    registers.  Their B operands come straight from HBM into registers
//    (8/16-byte loads, 64 contiguous bytes per row), the next tile's loaded
//    column by column as each column is retired -- B never touches shared
//    memory;
//  * column lanes (j, s) own column j and SV = N/2 states: they run the
//    vertical recurrences (h forward, G backward) with the state in registers
//    across tiles.  Their C operands stream through shared memory with
//    cp.async, one tile ahead;
//  * the only transposes are hh (row -> column lanes) and G (column -> row
//    lanes), through three rotating [R][16 N + N] slots (C of this tile, hh of
//    this tile, C of the next tile); the row padding and a per-column rotation
//    of the column lanes' 16-byte units keep both access patterns
//    bank-conflict free;
//  * the backward splits dAbar = Gh hh(i,j-1) + G h(i-1,j): the column lanes
//    fold the G h(i-1,j) half into dA and ddelta themselves (they own h), so
//    h never has to be transposed back to the row lanes;
//  * a CTA holds up to 13 (forward) / 12 (backward) warps = consecutive strips
//    in scan-major order; neighbouring strips of one scan in one CTA pass the
//    horizontal carry through an mbarrier-guarded shared-memory ring, strips in
//    different CTAs through tagged 8-byte words in global memory (CTA tickets
//    keep producers resident).  A training forward also stores hh at every
//    strip boundary (plain values, residual `hres`) and h at the last row of
//    every tile (checkpoints), so the backward recomputes instead of storing
//    states.
// Shared memory per warp (fp32, N = 16): 14.3 KB forward, 16.5 KB backward.
#pragma once

#include "scan2d_fwd.cuh"

namespace s2d {

template <typename T>
struct LnScale;
template <>
struct LnScale<float> {
  // A1 = A log2(e) (exp_scaled takes base-2 exponents); A = A1 ln 2
  static constexpr float v = 0.6931471805599453f;
};
template <>
struct LnScale<double> {
  static constexpr double v = 1.0;  // fp64 keeps A unscaled (Num<double>::a_scale)
};

template <typename T, int N, int CW, int SH>
struct T2Shape {
  static constexpr int QH = N / SH;      // row lanes per row
  static constexpr int R = 32 / QH;      // rows per tile
  static constexpr int QV = 32 / CW;     // column lanes per column
  static constexpr int SV = N / QV;      // states per column lane
  static constexpr int BP = CW * N + N;  // padded slot row pitch (elements)
  static constexpr int SLOT = R * BP;
  static constexpr int CELLS = R * CW;
  static constexpr int EPV = 16 / static_cast<int>(sizeof(T));
  static constexpr int RG = QH < CW ? QH : CW;  // columns per reduce-scatter group (backward)
  static constexpr int BUR = CW * N / EPV;       // 16-byte units per slot row
  // forward:  slots[3] | X[2] | Z[2] (z, then delta in place) | DX (delta x)
  static constexpr int F_X = 3 * SLOT, F_Z = F_X + 2 * CELLS, F_DX = F_Z + 2 * CELLS;
  static constexpr int F_TOTAL_RAW = F_DX + CELLS;
  // two 8-byte mbarriers (the TMA stage barriers of tiles u and u+1) close the region
  static constexpr int F_BAR = (F_TOTAL_RAW + EPV - 1) / EPV * EPV;
  static constexpr int F_TOTAL = F_BAR + EPV;
  // backward: slots[3] | X[2] | Z[2] | DY[2] | DX | SG (sigmoid) | DV (column-lane ddelta) | SCR[N]
  static constexpr int B_X = 3 * SLOT, B_Z = B_X + 2 * CELLS, B_Y = B_Z + 2 * CELLS;
  static constexpr int B_DX = B_Y + 2 * CELLS, B_SG = B_DX + CELLS, B_DV = B_SG + CELLS;
  static constexpr int B_SCR = B_DV + CELLS, B_AS = B_SCR + N, B_DAC = B_AS + N;
  // per-warp regions are padded to 16 bytes (cp.async destinations)
  static constexpr int B_BAR = (B_DAC + 32 * SV + EPV - 1) / EPV * EPV;
  static constexpr int B_TOTAL = B_BAR + EPV;
  static_assert(QH >= 1 && QH <= 32 && R >= 1 && SV >= 1, "tile shape");
  static_assert(CW % EPV == 0 && (CELLS % EPV) == 0, "16-byte copy units");
};

// ----------------------------------------------------------------- helpers

// SH consecutive elements from global memory (streaming, no L1 allocation)
template <typename T, int SH>
__device__ __forceinline__ void ldg_states(T (&v)[SH], const T* p) {
  if constexpr (sizeof(T) == 4 && SH % 4 == 0) {
#pragma unroll
    for (int e = 0; e < SH; e += 4) {
      const float4 q = __ldcs(reinterpret_cast<const float4*>(p + e));
      v[e] = q.x, v[e + 1] = q.y, v[e + 2] = q.z, v[e + 3] = q.w;
    }
  } else if constexpr (sizeof(T) == 4 && SH == 2) {
    const float2 q = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = q.x, v[1] = q.y;
  } else if constexpr (sizeof(T) == 8 && SH % 2 == 0) {
#pragma unroll
    for (int e = 0; e < SH; e += 2) {
      const double2 q = __ldcs(reinterpret_cast<const double2*>(p + e));
      v[e] = q.x, v[e + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < SH; ++e) v[e] = __ldcs(p + e);
  }
}

template <typename T, int SH>
__device__ __forceinline__ void stg_stream(T* p, const T (&v)[SH]) {
  if constexpr (sizeof(T) == 4 && SH % 4 == 0) {
#pragma unroll
    for (int e = 0; e < SH; e += 4) __stcs(reinterpret_cast<float4*>(p + e), make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
  } else if constexpr (sizeof(T) == 4 && SH == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  } else if constexpr (sizeof(T) == 8 && SH % 2 == 0) {
#pragma unroll
    for (int e = 0; e < SH; e += 2) __stcs(reinterpret_cast<double2*>(p + e), make_double2(v[e], v[e + 1]));
  } else {
#pragma unroll
    for (int e = 0; e < SH; ++e) __stcs(p + e, v[e]);
  }
}

// SH consecutive elements added into global memory (L2 reductions, no return
// value): the shared-B/C backward's in-place dB / dC group sums.  fp32 vector
// reductions flush denormal addends to zero.
template <typename T, int SH>
__device__ __forceinline__ void red_states(T* p, const T (&v)[SH]) {
  if constexpr (sizeof(T) == 4 && SH % 4 == 0) {
#pragma unroll
    for (int e = 0; e < SH; e += 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + e), "f"(v[e]), "f"(v[e + 1]),
                   "f"(v[e + 2]), "f"(v[e + 3])
                   : "memory");
  } else if constexpr (sizeof(T) == 4 && SH == 2) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v[0]), "f"(v[1]) : "memory");
  } else {
#pragma unroll
    for (int e = 0; e < SH; ++e) atomicAdd(p + e, v[e]);
  }
}

// V consecutive elements from / to shared memory (V a power of two)
template <typename T, int V>
__device__ __forceinline__ void lds_vec(T (&v)[V], const T* p) {
  constexpr int E = 16 / static_cast<int>(sizeof(T));  // elements per 16-byte access
  if constexpr (V % E == 0 && sizeof(T) == 4) {
#pragma unroll
    for (int e = 0; e < V; e += 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + e);
      v[e] = q.x, v[e + 1] = q.y, v[e + 2] = q.z, v[e + 3] = q.w;
    }
  } else if constexpr (V % E == 0 && sizeof(T) == 8) {
#pragma unroll
    for (int e = 0; e < V; e += 2) {
      const double2 q = *reinterpret_cast<const double2*>(p + e);
      v[e] = q.x, v[e + 1] = q.y;
    }
  } else if constexpr (V == 2 && sizeof(T) == 4) {
    const float2 q = *reinterpret_cast<const float2*>(p);
    v[0] = q.x, v[1] = q.y;
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) v[e] = p[e];
  }
}

template <typename T, int V>
__device__ __forceinline__ void sts_vec(T* p, const T (&v)[V]) {
  constexpr int E = 16 / static_cast<int>(sizeof(T));
  if constexpr (V % E == 0 && sizeof(T) == 4) {
#pragma unroll
    for (int e = 0; e < V; e += 4) *reinterpret_cast<float4*>(p + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
  } else if constexpr (V % E == 0 && sizeof(T) == 8) {
#pragma unroll
    for (int e = 0; e < V; e += 2) *reinterpret_cast<double2*>(p + e) = make_double2(v[e], v[e + 1]);
  } else if constexpr (V == 2 && sizeof(T) == 4) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) p[e] = v[e];
  }
}

// Column-lane state vectors (SV states of one column, 16-byte units): lane
// (j, s) visits its units in an order rotated by `rot` so that the 8 lanes of a
// quarter-warp touch 8 distinct bank quads (fp32 N = 16: columns 2 apart alias
// otherwise -> 2-way conflicts; N = 32: 4-way).  Register v[h*UE + k] holds
// state s*SV + ((h + rot) % NU)*UE + k of the column.
template <typename T, int SV>
struct ColVec {
  static constexpr int UE = 16 / static_cast<int>(sizeof(T)) < SV ? 16 / static_cast<int>(sizeof(T)) : SV;
  static constexpr int NU = SV / UE;
  int rot;
  __device__ __forceinline__ int unit(int h) const { return NU == 1 ? 0 : (h + rot) & (NU - 1); }
  __device__ __forceinline__ int state(int e) const { return unit(e / UE) * UE + e % UE; }
  __device__ __forceinline__ void lds(T (&v)[SV], const T* p) const {
#pragma unroll
    for (int h = 0; h < NU; ++h) {
      T t[UE];
      lds_vec<T, UE>(t, p + unit(h) * UE);
#pragma unroll
      for (int k = 0; k < UE; ++k) v[h * UE + k] = t[k];
    }
  }
  __device__ __forceinline__ void sts(T* p, const T (&v)[SV]) const {
#pragma unroll
    for (int h = 0; h < NU; ++h) {
      T t[UE];
#pragma unroll
      for (int k = 0; k < UE; ++k) t[k] = v[h * UE + k];
      sts_vec<T, UE>(p + unit(h) * UE, t);
    }
  }
  __device__ __forceinline__ void ldg(T (&v)[SV], const T* p) const {
#pragma unroll
    for (int h = 0; h < NU; ++h) {
      T t[UE];
      ldg_states<T, UE>(t, p + unit(h) * UE);
#pragma unroll
      for (int k = 0; k < UE; ++k) v[h * UE + k] = t[k];
    }
  }
  __device__ __forceinline__ void stg(T* p, const T (&v)[SV]) const {
#pragma unroll
    for (int h = 0; h < NU; ++h) {
      T t[UE];
#pragma unroll
      for (int k = 0; k < UE; ++k) t[k] = v[h * UE + k];
      stg_stream<T, UE>(p + unit(h) * UE, t);
    }
  }
  __device__ __forceinline__ void red(T* p, const T (&v)[SV]) const {
#pragma unroll
    for (int h = 0; h < NU; ++h) {
      T t[UE];
#pragma unroll
      for (int k = 0; k < UE; ++k) t[k] = v[h * UE + k];
      red_states<T, UE>(p + unit(h) * UE, t);
    }
  }
};

template <typename T, int N, int SV>
__device__ __forceinline__ ColVec<T, SV> col_vec(int j2) {
  ColVec<T, SV> c;
  // word offset of column j2 modulo 32 banks, in units of the lane's SV-state span
  c.rot = sizeof(T) == 4 ? ((j2 * N) / 32) & (ColVec<T, SV>::NU - 1) : 0;
  return c;
}

// rows r0 .. r0+R-1, columns 0 .. ncols-1 of an [H][W] plane (g already offset
// by the strip's first column) -> [R][CW] in shared memory, 16-byte units
template <typename TS, typename T>
__device__ __forceinline__ void issue_cells(uint32_t sdst, const T* g, int r0, int H, int W, int ncols,
                                            int lane, bool vec) {
  constexpr int XR = TS::CELLS / TS::R / TS::EPV;  // units per row (CW / EPV)
  constexpr int XU = TS::R * XR;
  if (!vec) {  // rows not 16-byte aligned (W % (16 / sizeof(T)) != 0): one element per copy
    constexpr int CW = TS::CELLS / TS::R;
#pragma unroll
    for (int u0 = 0; u0 < TS::CELLS; u0 += 32) {
      const int u = u0 + lane;
      const int rr = u / CW, cc = u % CW;
      if (u < TS::CELLS && cc < ncols && r0 + rr < H)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sdst + u * static_cast<uint32_t>(sizeof(T))),
                     "l"(g + static_cast<size_t>(r0 + rr) * W + cc), "n"(sizeof(T)));
    }
    return;
  }
#pragma unroll
  for (int u0 = 0; u0 < XU; u0 += 32) {
    const int u = u0 + lane;
    const int rr = u / XR, cu = u % XR;
    if ((XU % 32 == 0 || u < XU) && cu * TS::EPV < ncols && r0 + rr < H)
      cp_async16_raw(sdst + (rr * (TS::CELLS / TS::R) + cu * TS::EPV) * static_cast<uint32_t>(sizeof(T)),
                     g + static_cast<size_t>(r0 + rr) * W + cu * TS::EPV);
  }
}

// rows r0 .. r0+R-1 of a [H][W][N] tensor, the strip's ncols columns (g offset
// by c0 * N) -> one [R][BP] slot
template <typename TS, int N, typename T>
__device__ __forceinline__ void issue_slot(uint32_t sdst, const T* g, int r0, int H, size_t WN, int ncols,
                                           int lane) {
  constexpr int BUR = TS::BUR;
  constexpr int BU = TS::R * BUR;
  const int bunits = ncols * N / TS::EPV;
#pragma unroll
  for (int u0 = 0; u0 < BU; u0 += 32) {
    int rr, cu;
    if constexpr (BUR % 32 == 0) {
      rr = u0 / BUR;
      cu = u0 % BUR + lane;
    } else {
      const int u = u0 + lane;
      rr = u / BUR;
      cu = u % BUR;
    }
    if ((BU % 32 == 0 || u0 + lane < BU) && cu < bunits && r0 + rr < H)
      cp_async16_raw(sdst + (rr * TS::BP + cu * TS::EPV) * static_cast<uint32_t>(sizeof(T)),
                     g + static_cast<size_t>(r0 + rr) * WN + cu * TS::EPV);
  }
}

// row lane's B operand for one tile: B[r0 + r1][c0 + j][q1 SH ..] for j < CW
template <typename T, int CW, int SH>
__device__ __forceinline__ void load_b_rows(T (&b)[CW][SH], const T* Bg, int i1, int H, size_t WN, int ncols,
                                            int N) {
  const bool ok = i1 < H;
  const T* p = Bg + static_cast<size_t>(ok ? i1 : 0) * WN;
#pragma unroll
  for (int j = 0; j < CW; ++j) {
    if (ok && j < ncols) {
      ldg_states<T, SH>(b[j], p + static_cast<size_t>(j) * N);
    } else {
#pragma unroll
      for (int e = 0; e < SH; ++e) b[j][e] = T(0);
    }
  }
}

__device__ __forceinline__ int slot_next(int s) { return s == 2 ? 0 : s + 1; }

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Bulk L2 prefetch by the TMA unit (UBLKPF): `bytes` (multiple of 16) from a
// 16-byte aligned address, no registers, no completion tracking.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// L2 prefetch of rows r0 .. r0+R-1 of the strip (B / C spans of ncols x N
// elements, and the x / z / dy cells), so the tile's register / cp.async loads
// hit L2.  Mode 1: per-lane prefetch.global.L2 of 128-byte lines (three
// instructions per lane per tile); mode 2: bulk prefetches by the TMA unit
// (cp.async.bulk.prefetch.L2), one per row span, issued by lane 0.  (A bulk
// prefetch takes its address in a uniform register: issued from many lanes
// with different addresses the compiler serialises them in a loop over lanes,
// measured as ~9 % of the backward's issue slots.)
template <typename T, int R>
__device__ __forceinline__ void prefetch_tile_l2(int mode, int lane, int r0, int H, int ncols, int N, size_t WN,
                                                 int W, const T* Bs, const T* Cs, const T* xs, const T* zs,
                                                 const T* ys, bool xvec) {
  const int rows = min(R, H - r0);
  if (rows <= 0) return;
  const uint32_t sb = static_cast<uint32_t>(ncols * N * sizeof(T));
  if (mode == 2) {
    if (lane == 0) {
      for (int r = 0; r < rows; ++r) {
        bulk_prefetch_l2(Bs + static_cast<size_t>(r0 + r) * WN, sb);
        bulk_prefetch_l2(Cs + static_cast<size_t>(r0 + r) * WN, sb);
      }
    }
    return;
  }
  // mode 1: lines of the B / C row spans (<= 2 * R * 8 lines of 128 B for a
  // 1 KB span), then one line per x / z / dy row
  const int lines = static_cast<int>((sb + 127) / 128);
  const int total = 2 * rows * lines;
  for (int u = lane; u < total; u += 32) {
    const int plane = u / (rows * lines), rem = u % (rows * lines), r = rem / lines, l = rem % lines;
    const char* base = reinterpret_cast<const char*>((plane == 0 ? Bs : Cs) + static_cast<size_t>(r0 + r) * WN);
    prefetch_l2(base + l * 128);
  }
  const int planes = ys != nullptr ? 3 : 2;
  if (lane < planes * rows) {
    const int k = lane / rows, r = lane % rows;
    const T* p = (k == 0 ? xs : k == 1 ? zs : ys) + static_cast<size_t>(r0 + r) * W;
    prefetch_l2(p);
  }
  (void)xvec;
}


// ------------------------------------------------------------ CTA = strips
//
// A CTA holds `nw` warps = `nw` adjacent strips of one scan (all 13 strips of a
// 200-wide grid).  Warps of one CTA are issued fairly by the SM, so the
// horizontal carry chain between them stays in lockstep; the carry moves
// through a shared-memory ring guarded by mbarriers (full: producer -> consumer,
// empty: consumer -> producer, RING tiles deep).  Only the boundaries between
// CTAs of one scan (grids wider than nw * 16 columns) use the tagged global
// words, and CTAs take tickets so a producer CTA is always resident first.

constexpr int kRing = 4;  // carry ring depth (tiles)
// cross-CTA horizontal carries loaded one tile ahead: forward (measured: cfg2
// with scans straddling CTAs 176.7 -> 158.2 us, 64 x 1024^2 1918 -> 1809 us)
// and backward (S2D_CARRY_PF_B)
#ifndef S2D_CARRY_PF
#define S2D_CARRY_PF 1
#endif
#ifndef S2D_CARRY_PF_B
#define S2D_CARRY_PF_B 0
#endif
// warps (strips) per CTA at most.  Forward: 13 (128 registers, 13 strips = a
// 200-column scan per CTA).  Backward: 12 = 3 per SM sub-partition, so up to
// 168 registers per thread (no spills).
constexpr int kTileMaxWarps = 15;
constexpr int kTileMaxWarpsBwd = 12;

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
// shared-window addresses (uint32) versions: the ring computes them with
// integer arithmetic instead of a generic->shared conversion per call
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
#ifndef S2D_MBAR_HINT
#define S2D_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
#if S2D_MBAR_HINT > 0
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra W%=;\n\t}" ::"r"(bar),
      "r"(parity), "n"(S2D_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) { mbar_wait_s(smem_u32(bar), parity); }

// ---- TMA staging of a tile (cp.async.bulk, SASS UBLKCP): lane 0 arms the
// stage's mbarrier with the tile's byte count and issues one bulk copy per row
// span -- the C rows (ncols x N elements, contiguous) and, when the rows are
// 16-byte aligned, the x / z (/ dy) rows; the warp waits on the barrier's phase
// instead of cp.async groups.  The destination slot was last read by generic
// loads (the previous use ended with __syncwarp), hence the proxy fence.
__device__ __forceinline__ void mbar_init_tma(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <typename TS, int N, typename T>
__device__ __forceinline__ void tma_tile(uint32_t bar, uint32_t cdst, const T* Cg, int r0, int H, size_t WN, int W,
                                         int ncols, bool cells, uint32_t xd, const T* xg, uint32_t zd, const T* zg,
                                         uint32_t yd, const T* yg) {
  constexpr uint32_t ES = sizeof(T);
  const int rows = max(0, min(TS::R, H - r0));
  const uint32_t cb = static_cast<uint32_t>(ncols * N) * ES, xb = static_cast<uint32_t>(ncols) * ES;
  const int planes = !cells ? 0 : (yg != nullptr ? 3 : 2);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, static_cast<uint32_t>(rows) * (cb + planes * xb));
  for (int r = 0; r < rows; ++r) {
    const size_t gr = static_cast<size_t>(r0 + r);
    bulk_g2s(cdst + static_cast<uint32_t>(r * TS::BP) * ES, Cg + gr * WN, cb, bar);
    if (planes > 0) {
      const uint32_t co = static_cast<uint32_t>(r * (TS::CELLS / TS::R)) * ES;
      bulk_g2s(xd + co, xg + gr * W, xb, bar);
      bulk_g2s(zd + co, zg + gr * W, xb, bar);
      if (planes > 2) bulk_g2s(yd + co, yg + gr * W, xb, bar);
    }
  }
}

// Carry ring of one CTA: data [nw-1][kRing][32 lanes][SH], barriers full / empty
// [nw-1][kRing].  Boundary b sits between warps b and b+1.
template <typename T, int SH>
struct CarryRing {
  T* data;
  uint64_t* full;
  uint64_t* empty;
  uint32_t full_s, empty_s;  // shared-window addresses of full / empty
  static __host__ __device__ size_t bytes(int nw) {
    const size_t nb = nw > 1 ? nw - 1 : 0;
    return nb * kRing * 32 * SH * sizeof(T) + 2 * nb * kRing * sizeof(uint64_t);
  }
  __device__ void setup(unsigned char* base, int nw) {
    const int nb = nw > 1 ? nw - 1 : 0;
    data = reinterpret_cast<T*>(base);
    full = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(nb) * kRing * 32 * SH * sizeof(T));
    empty = full + nb * kRing;
    full_s = smem_u32(full);
    empty_s = smem_u32(empty);
  }
  // producer side: tile index u (0, 1, 2, ... in the warp's own visiting order)
  __device__ __forceinline__ void put(int b, int u, int lane, const T (&v)[SH]) {
    const int k = u % kRing;
    const uint32_t bo = static_cast<uint32_t>(b * kRing + k) * 8u;
    mbar_wait_s(empty_s + bo, ((u / kRing) & 1) ^ 1);
    T* d = data + ((b * kRing + k) * 32 + lane) * SH;
#pragma unroll
    for (int e = 0; e < SH; ++e) d[e] = v[e];
    mbar_arrive_s(full_s + bo);
  }
  __device__ __forceinline__ void get(int b, int u, int lane, T (&v)[SH]) {
    const int k = u % kRing;
    const uint32_t bo = static_cast<uint32_t>(b * kRing + k) * 8u;
    mbar_wait_s(full_s + bo, (u / kRing) & 1);
    const T* d = data + ((b * kRing + k) * 32 + lane) * SH;
#pragma unroll
    for (int e = 0; e < SH; ++e) v[e] = d[e];
    mbar_arrive_s(empty_s + bo);
  }
};

// CTA ticket + strip identity.  The S x wreal strips are numbered scan-major
// and dealt to CTAs in contiguous runs of nw (one warp each), so a CTA may end
// one scan and start the next: every SM gets an equal share of strips (139 of
// the 148 SMs busy for 128 scans x 13 strips instead of 128).  Consecutive
// warps of one scan pass the carry through the shared-memory ring; the first /
// last warp of a run uses the tagged global words.  CTAs take tickets so the
// CTA holding a strip's producer is always resident first.  rev (backward):
// strips are dealt right to left, so warp wi+1 holds the LEFT neighbour.
struct StripId {
  int64_t s;
  int strip, wi, nw;
  bool valid;
};

template <typename T>
__device__ __forceinline__ StripId strip_id(const Geo& ge, const Args<T>& a, bool rev) {
  __shared__ int tk;
  const int64_t S = a.S;
  StripId id;
  id.nw = blockDim.x / 32;
  id.wi = threadIdx.x / 32;
  int64_t unit = blockIdx.x;
  if (ge.wreal > 1) {
    griddep_wait();  // the begin kernel has reset the ticket and advanced the epoch
    if (threadIdx.x == 0) {
      tk = atomicAdd(a.ticket, 1);
      if (tk == 0) a.hdr->magic = a.magic;  // the carry region now follows this layout
    }
    __syncthreads();
    unit = tk;
  }
  const int64_t total = S * ge.wreal;
  int64_t g = unit * id.nw + id.wi;
  id.valid = g < total;
  if (rev) g = total - 1 - g;
  if (!id.valid) g = 0;
  id.s = g / ge.wreal;
  id.strip = static_cast<int>(g % ge.wreal);
  return id;
}

// ================================================================== forward

template <typename T, int N, int CW, int SH, bool EMIT = false, bool ACC = false>
__global__ void __launch_bounds__(32 * kTileMaxWarps, 1) scan2d_fwd_tile2_kernel(const Args<T> a) {
  using F = Fn<T, ACC>;
  using TS = T2Shape<T, N, CW, SH>;
  constexpr int R = TS::R, QH = TS::QH, QV = TS::QV, SV = TS::SV, BP = TS::BP, CELLS = TS::CELLS;
  constexpr uint32_t ES = sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& ge = a.plan.f;
  const StripId id = strip_id(ge, a, false);
  const uint32_t epoch = ge.wreal > 1 ? load_epoch(a.hdr) : 0u;
  const int lane = threadIdx.x & 31;
  CarryRing<T, SH> ring;
  ring.setup(smem_raw + static_cast<size_t>(id.nw) * TS::F_TOTAL * ES, id.nw);
  if (threadIdx.x < (id.nw - 1) * kRing) {
    mbar_init(ring.full + threadIdx.x, 32);
    mbar_init(ring.empty + threadIdx.x, 32);
  }
  __syncthreads();
  if (!id.valid) return;
  T* sm = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(id.wi) * TS::F_TOTAL;
  const int H = a.H, W = a.W;
  const int64_t s = id.s;
  const int wpos = id.strip;
  const int c0 = wpos * CW;
  const int ncols = min(CW, W - c0);
  const int p = param_row(s, a.S, a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const size_t WN = static_cast<size_t>(W) * N;
  const T Dsk = a.Dskip[p], bias = a.bias[p];

  const int r1 = lane / QH, q1 = lane % QH;  // row lanes
  const int j2 = lane / QV, s2 = lane % QV;  // column lanes
  const ColVec<T, SV> cv = col_vec<T, N, SV>(j2);
  T A1[SH], A2[SV];
#pragma unroll
  for (int e = 0; e < SH; ++e) A1[e] = F::a_scale(a.A[static_cast<int64_t>(p) * N + q1 * SH + e]);
#pragma unroll
  for (int e = 0; e < SV; ++e) A2[e] = F::a_scale(a.A[static_cast<int64_t>(p) * N + s2 * SV + cv.state(e)]);

  for (int e = lane; e < TS::F_TOTAL; e += 32) sm[e] = T(0);
  __syncwarp();

  const T* xg = a.x + s * HW + c0;
  const T* zg = a.z + s * HW + c0;
  const T* Bg = a.B + bc_row(s, a.G) * HW * N + static_cast<size_t>(c0) * N + q1 * SH;
  const T* Cg = a.C + bc_row(s, a.G) * HW * N + static_cast<size_t>(c0) * N;
  const uint32_t sbase = smem_u32(sm);
  const bool xrow16 = a.xvec != 0;  // x / z rows 16-byte aligned

  const bool save = a.ckpt != nullptr;
  const int nq = a.plan.nq, nbm1 = a.plan.nb - 1;  // checkpoints every R rows (plan.K == R)
  const bool has_pred = wpos > 0, has_succ = wpos + 1 < ge.wreal;
  // carry-in: ring from the warp on the left, or the global word across a CTA boundary
  const bool pred_ring = has_pred && id.wi > 0;
  const bool succ_ring = has_succ && id.wi + 1 < id.nw;
  const CarrySlot<T>* hc_in = has_pred ? a.hcarry + ((s * nq + (wpos - 1)) * H) * N + q1 * SH : nullptr;
  CarrySlot<T>* hc_out = has_succ && !succ_ring ? a.hcarry + ((s * nq + wpos) * H) * N + q1 * SH : nullptr;
  // residual copy of every boundary carry (plain values, read by the backward)
  T* hr_out = save && has_succ ? a.hres + ((s * nq + wpos) * H) * N + q1 * SH : nullptr;
  const int jg2 = c0 + j2;
  const bool col_ok = j2 < ncols;
  // reference CarryState emission (the C++ engine shim asks for it)
  constexpr bool emit = EMIT;  // (a separate instantiation: no registers spent when off)
  const int Tt = EMIT ? a.T_tile : 1;
  const int kht = EMIT ? (H + Tt - 1) / Tt : 1, kwt = EMIT ? (W + Tt - 1) / Tt : 1;

  T hv[SV];  // vertical state: zeros, or the row above the band (row-band shard)
#pragma unroll
  for (int e = 0; e < SV; ++e) hv[e] = T(0);
  if (a.link_in != nullptr) link_wait(a.link_in + s * ge.wreal + wpos, a.link_seq, lane);
  if (a.vtop != nullptr && col_ok) cv.ldg(hv, a.vtop + (s * W + jg2) * N + s2 * SV);

  const int ntiles = (H + R - 1) / R;
  int sc = 0;  // slot holding this tile's C; sc+1: hh of this tile; sc+2: C of the next tile
  // TMA staging (stage barriers at the end of the warp's region) or cp.async
  const bool tma = a.plan.tma != 0;
  const bool tcells = a.plan.tma == 2 && xrow16;  // x / z / dy rows by TMA too
  uint64_t* tbar = reinterpret_cast<uint64_t*>(sm + TS::F_BAR);
  if (tma) {
    if (lane == 0) {
      mbar_init_tma(tbar);
      mbar_init_tma(tbar + 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0)
      tma_tile<TS, N>(smem_u32(tbar), sbase + sc * TS::SLOT * ES, Cg, 0, H, WN, W, ncols, tcells,
                      sbase + TS::F_X * ES, xg, sbase + TS::F_Z * ES, zg, 0u, static_cast<const T*>(nullptr));
    if (!tcells) {
      issue_cells<TS>(sbase + TS::F_X * ES, xg, 0, H, W, ncols, lane, xrow16);
      issue_cells<TS>(sbase + TS::F_Z * ES, zg, 0, H, W, ncols, lane, xrow16);
    }
  } else {
    issue_slot<TS, N>(sbase + sc * TS::SLOT * ES, Cg, 0, H, WN, ncols, lane);
    issue_cells<TS>(sbase + TS::F_X * ES, xg, 0, H, W, ncols, lane, xrow16);
    issue_cells<TS>(sbase + TS::F_Z * ES, zg, 0, H, W, ncols, lane, xrow16);
  }
  cp_async_commit();
  T bc[CW][SH];
  load_b_rows<T, CW, SH>(bc, Bg, r1, H, WN, ncols, N);

  // horizontal carry from a strip in another CTA: loaded one tile ahead (the
  // tag tells a stale word; the resolve then re-polls)
  CarryPre<T, SH> cpre;
#if S2D_CARRY_PF
  if constexpr (sizeof(T) == 4) {
    if (has_pred && !pred_ring && r1 < H)
      carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(r1) * N),
                     *reinterpret_cast<CarryPre<float, SH>*>(&cpre));
  }
#endif
  const int pft = a.plan.pf_all ? 0 : a.plan.pft_f;
  const int pfmode = a.plan.pf_mode;
  if (a.plan.pf_all)
    for (int t2 = 1; t2 < ntiles; ++t2)
      prefetch_tile_l2<T, R>(pfmode, lane, t2 * R, H, ncols, N, WN, W, Bg - q1 * SH, Cg, xg, zg, nullptr, xrow16);
  for (int t = 0; t < ntiles; ++t) {
    const int r0 = t * R;
    const int par = t & 1;
    const int sh = slot_next(sc), sn = slot_next(sh);
#ifndef S2D_NO_PF
    if (pft > 0 && t + pft < ntiles)
      prefetch_tile_l2<T, R>(pfmode, lane, r0 + pft * R, H, ncols, N, WN, W, Bg - q1 * SH, Cg, xg, zg, nullptr, xrow16);
#endif
    // ---- prefetch tile t+1: C into the free slot, x / z into the other parity
    //      (its B operand is loaded into the same registers right after phase 1)
    if (t + 1 < ntiles) {
      if (tma) {
        if (lane == 0)
          tma_tile<TS, N>(smem_u32(tbar + ((t + 1) & 1)), sbase + sn * TS::SLOT * ES, Cg, r0 + R, H, WN, W, ncols,
                          tcells, sbase + (TS::F_X + (par ^ 1) * CELLS) * ES, xg,
                          sbase + (TS::F_Z + (par ^ 1) * CELLS) * ES, zg, 0u, static_cast<const T*>(nullptr));
        if (!tcells) {
          issue_cells<TS>(sbase + (TS::F_X + (par ^ 1) * CELLS) * ES, xg, r0 + R, H, W, ncols, lane, xrow16);
          issue_cells<TS>(sbase + (TS::F_Z + (par ^ 1) * CELLS) * ES, zg, r0 + R, H, W, ncols, lane, xrow16);
        }
      } else {
        issue_slot<TS, N>(sbase + sn * TS::SLOT * ES, Cg, r0 + R, H, WN, ncols, lane);
        issue_cells<TS>(sbase + (TS::F_X + (par ^ 1) * CELLS) * ES, xg, r0 + R, H, W, ncols, lane, xrow16);
        issue_cells<TS>(sbase + (TS::F_Z + (par ^ 1) * CELLS) * ES, zg, r0 + R, H, W, ncols, lane, xrow16);
      }
    }
    cp_async_commit();
    const int i1 = r0 + r1;
    const bool row_ok = i1 < H;
#if !S2D_CARRY_PF
    if constexpr (sizeof(T) == 4) {
      if (has_pred && !pred_ring && row_ok)
        carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i1) * N),
                       *reinterpret_cast<CarryPre<float, SH>*>(&cpre));
    }
#endif
    cp_async_wait<1>();
    if (tma) mbar_wait(tbar + (t & 1), (t >> 1) & 1);
    __syncwarp();
    T* Xs = sm + TS::F_X + par * CELLS;
    T* Ds = sm + TS::F_Z + par * CELLS;  // z, then delta in place
    T* DXs = sm + TS::F_DX;
    T* Cs = sm + sc * TS::SLOT;
    T* HHs = sm + sh * TS::SLOT;

    // ---- delta = softplus(z + bias) and delta x, once per cell
#pragma unroll
    for (int c = lane; c < CELLS; c += 32) {
      const T d = F::softplus(Ds[c] + bias);
      Ds[c] = d;
      DXs[c] = d * Xs[c];
    }
    __syncwarp();

    // ---- phase 1 (row lanes): hh left -> right
    T hh[SH];
#pragma unroll
    for (int e = 0; e < SH; ++e) hh[e] = T(0);
    if (pred_ring) {
      ring.get(id.wi - 1, t, lane, hh);
      if (!row_ok) {
#pragma unroll
        for (int e = 0; e < SH; ++e) hh[e] = T(0);
      }
    } else if (has_pred && row_ok) {
      if constexpr (sizeof(T) == 4) {
        carry_resolve<SH>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i1) * N),
                          *reinterpret_cast<CarryPre<float, SH>*>(&cpre), row_tag(epoch, i1),
                          *reinterpret_cast<float(*)[SH]>(hh));
#if S2D_CARRY_PF
        if (i1 + R < H)
          carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(hc_in + static_cast<size_t>(i1 + R) * N),
                         *reinterpret_cast<CarryPre<float, SH>*>(&cpre));
#endif
      } else {
        carry_get_wait<T, SH>(hc_in + static_cast<size_t>(i1) * N, hh, row_tag(epoch, i1), SH);
      }
    }
    {
      const T* dr = Ds + r1 * CW;
      const T* ur = DXs + r1 * CW;
      T* hr = HHs + r1 * BP + q1 * SH;
#pragma unroll
      for (int j0 = 0; j0 < CW; j0 += 4) {
        T d4[4], u4[4];
        lds_vec<T, 4>(d4, dr + j0);
        lds_vec<T, 4>(u4, ur + j0);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = j0 + jj;
#pragma unroll
          for (int e = 0; e < SH; ++e) hh[e] = fma(F::exp_scaled(d4[jj] * A1[e]), hh[e], bc[j][e] * u4[jj]);
          if (j < ncols) sts_vec<T, SH>(hr + j * N, hh);
          // reference CarryState P^h (engine.cpp:188-194): hh at the last column of
          // every reference tile (edge slots stay zero, the reference's pass-through)
          if (emit && row_ok && j < ncols && ((c0 + j) % Tt == Tt - 1 || c0 + j == W - 1)) {
            const size_t tl = (static_cast<size_t>(s) * kht + i1 / Tt) * kwt + (c0 + j) / Tt;
#pragma unroll
            for (int e = 0; e < SH; ++e) a.ph[(tl * Tt + i1 % Tt) * N + q1 * SH + e] = hh[e];
          }
          // column j is done with B: load the next tile's in place
          if (t + 1 < ntiles && j < ncols && i1 + R < H)
            ldg_states<T, SH>(bc[j], Bg + static_cast<size_t>(i1 + R) * WN + static_cast<size_t>(j) * N);
        }
      }
      // strips other than the last are full (ncols == CW): hh is the boundary carry
      if (succ_ring) ring.put(id.wi, t, lane, hh);
      if (has_succ && row_ok && !succ_ring)
        carry_put<T, SH>(hc_out + static_cast<size_t>(i1) * N, hh, row_tag(epoch, i1), SH);
      if (save && has_succ && row_ok) stg_stream<T, SH>(hr_out + static_cast<size_t>(i1) * N, hh);
    }
    __syncwarp();

    // ---- phase 2 (column lanes): h top -> down, y = D x + sum_d C h
    {
      const T* hcol = HHs + j2 * N + s2 * SV;
      const T* ccol = Cs + j2 * N + s2 * SV;
      T* yp = a.y + s * HW + static_cast<size_t>(r0) * W + jg2;
      const int rows = min(R, H - r0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const T dj = Ds[r * CW + j2];
        T h4[SV], c4[SV];
        cv.lds(h4, hcol + r * BP);
        cv.lds(c4, ccol + r * BP);
        T acc0 = T(0), acc1 = T(0);
#pragma unroll
        for (int e = 0; e < SV; ++e) {
          hv[e] = fma(F::exp_scaled(dj * A2[e]), hv[e], h4[e]);
          if (e & 1)
            acc1 = fma(c4[e], hv[e], acc1);
          else
            acc0 = fma(c4[e], hv[e], acc0);
        }
        T acc = acc0 + acc1;
#pragma unroll
        for (int o = 1; o < QV; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
        const int i = r0 + r;
        if (r < rows && col_ok) {
          if (s2 == 0) __stcs(yp + static_cast<size_t>(r) * W, fma(Dsk, Xs[r * CW + j2], acc));
          if (save && r == R - 1 && i < H - 1) {  // checkpoint: h at the last row of every tile
            T* ck = a.ckpt + ((static_cast<size_t>(s) * nbm1 + t) * W + jg2) * N + s2 * SV;
            cv.stg(ck, hv);
          }
          if (i == H - 1 && a.vbot != nullptr)  // row-band shard: the next band's vtop
            cv.stg(a.vbot + (s * W + jg2) * N + s2 * SV, hv);
          if (emit && (i % Tt == Tt - 1 || i == H - 1)) {  // reference CarryState P^v (engine.cpp:217-220)
            const size_t tl = (static_cast<size_t>(s) * kht + i / Tt) * kwt + jg2 / Tt;
#pragma unroll
            for (int e = 0; e < SV; ++e) a.pv[(tl * Tt + jg2 % Tt) * N + s2 * SV + cv.state(e)] = hv[e];
          }
        }
      }
    }
    __syncwarp();
    sc = sn;
  }
  if (a.link_out != nullptr) link_post(a.link_out + s * ge.wreal + wpos, a.link_seq, lane);
}

// ================================================================= backward

// CW = 16: up to 13 warps (128 registers); CW = 32 (fp32, N <= 16): up to 8
// warps with the register room for 32-column strips (7 strips cover 200 columns)
// RED: dB / dC summed over the B/C group in place (a.red; a compile-time
// variant -- a runtime branch around the stores cost the default kernel 16 %)
template <typename T, int N, int CW, int SH, bool ACC = false, bool RED = false>
__global__ void __launch_bounds__(CW == 16 ? 32 * kTileMaxWarpsBwd : 256, 1) scan2d_bwd_tile2_kernel(const Args<T> a) {
  using F = Fn<T, ACC>;
  using TS = T2Shape<T, N, CW, SH>;
  constexpr int R = TS::R, QH = TS::QH, QV = TS::QV, SV = TS::SV, BP = TS::BP, CELLS = TS::CELLS;
  constexpr int RG = TS::RG;
  constexpr uint32_t ES = sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& ge = a.plan.b;
  const StripId id = strip_id(ge, a, true);
  const uint32_t epoch = ge.wreal > 1 ? load_epoch(a.hdr) : 0u;
  const int lane = threadIdx.x & 31;
  CarryRing<T, SH> ring;
  ring.setup(smem_raw + static_cast<size_t>(id.nw) * TS::B_TOTAL * ES, id.nw);
  if (threadIdx.x < (id.nw - 1) * kRing) {
    mbar_init(ring.full + threadIdx.x, 32);
    mbar_init(ring.empty + threadIdx.x, 32);
  }
  __syncthreads();
  if (!id.valid) return;
  T* sm = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(id.wi) * TS::B_TOTAL;
  const int H = a.H, W = a.W;
  const int64_t s = id.s;
  const int wpos = id.strip;
  const int c0 = wpos * CW;
  const int ncols = min(CW, W - c0);
  const int p = param_row(s, a.S, a.P);
  const size_t HW = static_cast<size_t>(H) * W;
  const size_t WN = static_cast<size_t>(W) * N;
  const T Dsk = a.Dskip[p], bias = a.bias[p];
  const T LN = LnScale<T>::v;

  const int r1 = lane / QH, q1 = lane % QH;
  const int j2 = lane / QV, s2 = lane % QV;
  const ColVec<T, SV> cv = col_vec<T, N, SV>(j2);
  T A1[SH];
#pragma unroll
  for (int e = 0; e < SH; ++e) A1[e] = F::a_scale(a.A[static_cast<int64_t>(p) * N + q1 * SH + e]);

  for (int e = lane; e < TS::B_TOTAL; e += 32) sm[e] = T(0);
  __syncwarp();
  // column lanes re-read their scaled A from shared memory in each phase (registers)
  T* As = sm + TS::B_AS;
  for (int e = lane; e < N; e += 32) As[e] = F::a_scale(a.A[static_cast<int64_t>(p) * N + e]);
  T* DAs = sm + TS::B_DAC + lane * SV;  // this lane's column-lane dA accumulators
  __syncwarp();

  const T* xg = a.x + s * HW + c0;
  const T* zg = a.z + s * HW + c0;
  const T* yg = a.dy + s * HW + c0;
  const T* Bg = a.B + bc_row(s, a.G) * HW * N + static_cast<size_t>(c0) * N + q1 * SH;
  const T* Cg = a.C + bc_row(s, a.G) * HW * N + static_cast<size_t>(c0) * N;
  const uint32_t sbase = smem_u32(sm);
  const bool xrow16 = a.xvec != 0;  // x / z / dy rows 16-byte aligned

  const int nq = a.plan.nq, nbm1 = a.plan.nb - 1;
  const bool has_pred = wpos > 0, has_succ = wpos + 1 < ge.wreal;
  // reverse carry: from the warp on the right (warp wi-1, ring) or across the
  // CTA boundary (global); to the warp on the left (warp wi+1)
  const bool succ_ring = has_succ && id.wi > 0;
  const bool pred_ring = has_pred && id.wi + 1 < id.nw;
  // saved forward carries sit on the forward's 16-column grid (plan.Q)
  const T* hc_in = has_pred ? a.hres + ((s * nq + (c0 / a.plan.Q - 1)) * H) * N + q1 * SH : nullptr;
  const int wb = ge.wreal - 1;
  const CarrySlot<T>* rc_in = has_succ ? a.rcarry + ((s * wb + wpos) * H) * N + q1 * SH : nullptr;
  CarrySlot<T>* rc_out = has_pred ? a.rcarry + ((s * wb + (wpos - 1)) * H) * N + q1 * SH : nullptr;
  // a.red: dB / dC of the scan's B/C group, summed in place by L2 reductions
  const int64_t sbc = RED ? bc_row(s, a.G) : s;
  T* dBg = a.dB + sbc * HW * N + static_cast<size_t>(c0) * N + q1 * SH;
  T* dCg = a.dC + sbc * HW * N + static_cast<size_t>(c0) * N + s2 * SV;
  T* dxg = a.dx + s * HW + c0;
  T* dzg = a.dz + s * HW + c0;
  const int jg2 = c0 + j2;
  const bool col_ok = j2 < ncols;

  T dn[SV];  // Abar(i+1,j) G(i+1,j), carried up across tiles (column lanes)
#pragma unroll
  for (int e = 0; e < SV; ++e) dn[e] = T(0);
  if (a.link_in != nullptr) link_wait(a.link_in + s * ge.wreal + wpos, a.link_seq, lane);
  if (a.gbot != nullptr && col_ok) cv.ldg(dn, a.gbot + (s * W + jg2) * N + s2 * SV);
  T dAr[SH];
#pragma unroll
  for (int e = 0; e < SH; ++e) dAr[e] = T(0);
  // per-cell scalar sums run over the whole strip: accumulate in double
  double dbias_acc = 0.0, dD_acc = 0.0;

  const int ntiles = (H + R - 1) / R;
  int sc = 0;  // slot with C (then G) of this tile; sc+1: hh; sc+2: C of the next tile up
  const bool tma = a.plan.tma != 0;
  const bool tcells = a.plan.tma == 2 && xrow16;  // x / z / dy rows by TMA too
  uint64_t* tbar = reinterpret_cast<uint64_t*>(sm + TS::B_BAR);
  {
    const int rl = (ntiles - 1) * R;
    const int par = (ntiles - 1) & 1;
    if (tma) {
      if (lane == 0) {
        mbar_init_tma(tbar);
        mbar_init_tma(tbar + 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0)
        tma_tile<TS, N>(smem_u32(tbar), sbase + sc * TS::SLOT * ES, Cg, rl, H, WN, W, ncols, tcells,
                        sbase + (TS::B_X + par * CELLS) * ES, xg, sbase + (TS::B_Z + par * CELLS) * ES, zg,
                        sbase + (TS::B_Y + par * CELLS) * ES, yg);
      if (!tcells) {
        issue_cells<TS>(sbase + (TS::B_X + par * CELLS) * ES, xg, rl, H, W, ncols, lane, xrow16);
        issue_cells<TS>(sbase + (TS::B_Z + par * CELLS) * ES, zg, rl, H, W, ncols, lane, xrow16);
        issue_cells<TS>(sbase + (TS::B_Y + par * CELLS) * ES, yg, rl, H, W, ncols, lane, xrow16);
      }
    } else {
      issue_slot<TS, N>(sbase + sc * TS::SLOT * ES, Cg, rl, H, WN, ncols, lane);
      issue_cells<TS>(sbase + (TS::B_X + par * CELLS) * ES, xg, rl, H, W, ncols, lane, xrow16);
      issue_cells<TS>(sbase + (TS::B_Z + par * CELLS) * ES, zg, rl, H, W, ncols, lane, xrow16);
      issue_cells<TS>(sbase + (TS::B_Y + par * CELLS) * ES, yg, rl, H, W, ncols, lane, xrow16);
    }
    cp_async_commit();
  }
  T bc[CW][SH];
  load_b_rows<T, CW, SH>(bc, Bg, (ntiles - 1) * R + r1, H, WN, ncols, N);
  T hh0n[SH];  // saved forward carry of the next tile up
#pragma unroll
  for (int e = 0; e < SH; ++e) hh0n[e] = T(0);
  {
    const int ib = (ntiles - 1) * R + r1;
    if (has_pred && ib < H) ldg_states<T, SH>(hh0n, hc_in + static_cast<size_t>(ib) * N);
  }

  const int pft = a.plan.pf_all ? 0 : a.plan.pft_b;
  const int pfmode = a.plan.pf_mode;
  if (a.plan.pf_all)
    for (int t2 = ntiles - 2; t2 >= 0; --t2)
      prefetch_tile_l2<T, R>(pfmode, lane, t2 * R, H, ncols, N, WN, W, Bg - q1 * SH, Cg, xg, zg, yg, xrow16);
#if S2D_CARRY_PF_B
  CarryPre<T, SH> rpre;  // reverse carry from a strip in another CTA, one tile ahead
  if constexpr (sizeof(T) == 4) {
    const int ib = (ntiles - 1) * R + r1;
    if (has_succ && !succ_ring && ib < H)
      carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(rc_in + static_cast<size_t>(ib) * N),
                     *reinterpret_cast<CarryPre<float, SH>*>(&rpre));
  }
#endif
  for (int t = ntiles - 1; t >= 0; --t) {
    const int u = ntiles - 1 - t;  // visiting index (ring phase)
    const int r0 = t * R;
#ifndef S2D_NO_PF
    if (pft > 0 && t - pft >= 0)
      prefetch_tile_l2<T, R>(pfmode, lane, r0 - pft * R, H, ncols, N, WN, W, Bg - q1 * SH, Cg, xg, zg, yg, xrow16);
#endif
    const int rows = min(R, H - r0);
    const int par = t & 1;
    const int sh = slot_next(sc), sn = slot_next(sh);
    // this tile's B operand (row lanes) was loaded column by column as the
    // previous tile's R2 finished with each column (one register set only)
    if (t > 0) {
      const int ru = r0 - R;
      if (tma) {
        if (lane == 0)
          tma_tile<TS, N>(smem_u32(tbar + ((u + 1) & 1)), sbase + sn * TS::SLOT * ES, Cg, ru, H, WN, W, ncols,
                          tcells, sbase + (TS::B_X + (par ^ 1) * CELLS) * ES, xg,
                          sbase + (TS::B_Z + (par ^ 1) * CELLS) * ES, zg, sbase + (TS::B_Y + (par ^ 1) * CELLS) * ES,
                          yg);
        if (!tcells) {
          issue_cells<TS>(sbase + (TS::B_X + (par ^ 1) * CELLS) * ES, xg, ru, H, W, ncols, lane, xrow16);
          issue_cells<TS>(sbase + (TS::B_Z + (par ^ 1) * CELLS) * ES, zg, ru, H, W, ncols, lane, xrow16);
          issue_cells<TS>(sbase + (TS::B_Y + (par ^ 1) * CELLS) * ES, yg, ru, H, W, ncols, lane, xrow16);
        }
      } else {
        issue_slot<TS, N>(sbase + sn * TS::SLOT * ES, Cg, ru, H, WN, ncols, lane);
        issue_cells<TS>(sbase + (TS::B_X + (par ^ 1) * CELLS) * ES, xg, ru, H, W, ncols, lane, xrow16);
        issue_cells<TS>(sbase + (TS::B_Z + (par ^ 1) * CELLS) * ES, zg, ru, H, W, ncols, lane, xrow16);
        issue_cells<TS>(sbase + (TS::B_Y + (par ^ 1) * CELLS) * ES, yg, ru, H, W, ncols, lane, xrow16);
      }
    }
    cp_async_commit();
    const int i1 = r0 + r1;
    const bool row_ok = r1 < rows;
    // saved forward carry (residual; loaded one tile ahead), reverse carry
    // prefetch, checkpoint row
    T hh0[SH];
#pragma unroll
    for (int e = 0; e < SH; ++e) hh0[e] = hh0n[e], hh0n[e] = T(0);
    if (has_pred && t > 0) ldg_states<T, SH>(hh0n, hc_in + static_cast<size_t>(i1 - R) * N);
#if !S2D_CARRY_PF_B
    CarryPre<T, SH> rpre;
    if constexpr (sizeof(T) == 4) {
      if (has_succ && !succ_ring && row_ok)
        carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(rc_in + static_cast<size_t>(i1) * N),
                       *reinterpret_cast<CarryPre<float, SH>*>(&rpre));
    }
#endif
    T hp0[SV];  // h(r0 - 1, j): the forward checkpoint
#pragma unroll
    for (int e = 0; e < SV; ++e) hp0[e] = T(0);
    if (t > 0 && col_ok) {
      const T* ck = a.ckpt + ((static_cast<size_t>(s) * nbm1 + (t - 1)) * W + jg2) * N + s2 * SV;
      cv.ldg(hp0, ck);
    } else if (a.vtop != nullptr && col_ok) {  // row-band shard: h of the row above the band
      cv.ldg(hp0, a.vtop + (s * W + jg2) * N + s2 * SV);
    }
    cp_async_wait<1>();
    if (tma) mbar_wait(tbar + (u & 1), (u >> 1) & 1);
    __syncwarp();
    T* Xs = sm + TS::B_X + par * CELLS;
    T* Ds = sm + TS::B_Z + par * CELLS;  // z, then delta in place
    T* Ys = sm + TS::B_Y + par * CELLS;
    T* DXs = sm + TS::B_DX;
    T* SGs = sm + TS::B_SG;
    T* DVs = sm + TS::B_DV;
    T* Cs = sm + sc * TS::SLOT;   // C, then G in place
    T* HHs = sm + sh * TS::SLOT;  // hh

    // ---- per cell: delta, sigmoid, delta x
#pragma unroll
    for (int c = lane; c < CELLS; c += 32) {
      const T v = Ds[c] + bias;
      const T d = F::softplus(v);
      Ds[c] = d;
      SGs[c] = F::sigmoid(v);
      DXs[c] = d * Xs[c];
    }
    __syncwarp();

    // ---- CA (column lanes): G bottom -> up, over C in place (engine.cpp:321)
    {
      T* gcol = Cs + j2 * N + s2 * SV;
      T A2[SV];
      cv.lds(A2, As + s2 * SV);
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const T dj = Ds[r * CW + j2], dyv = Ys[r * CW + j2];
        T g4[SV];
        cv.lds(g4, gcol + r * BP);
#pragma unroll
        for (int e = 0; e < SV; ++e) {
          const T g = fma(g4[e], dyv, dn[e]);
          dn[e] = F::exp_scaled(dj * A2[e]) * g;
          g4[e] = g;
        }
        if (col_ok) cv.sts(gcol + r * BP, g4);
      }
    }
    // ---- F1 (row lanes): hh left -> right from the saved carry
    {
      T hh[SH];
#pragma unroll
      for (int e = 0; e < SH; ++e) hh[e] = hh0[e];
      const T* dr = Ds + r1 * CW;
      const T* ur = DXs + r1 * CW;
      T* hr = HHs + r1 * BP + q1 * SH;
#pragma unroll
      for (int j0 = 0; j0 < CW; j0 += 4) {
        T d4[4], u4[4];
        lds_vec<T, 4>(d4, dr + j0);
        lds_vec<T, 4>(u4, ur + j0);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = j0 + jj;
#pragma unroll
          for (int e = 0; e < SH; ++e) hh[e] = fma(F::exp_scaled(d4[jj] * A1[e]), hh[e], bc[j][e] * u4[jj]);
          if (j < ncols) sts_vec<T, SH>(hr + j * N, hh);
        }
      }
    }
    __syncwarp();

    // ---- CB (column lanes): h top -> down from the checkpoint, dC = dy h, and
    //      the G h(i-1,j) half of dAbar into dA and ddelta
    {
      const T* hcol = HHs + j2 * N + s2 * SV;
      const T* gcol = Cs + j2 * N + s2 * SV;
      T hcur[SV], A2[SV], dAc[SV];
      cv.lds(A2, As + s2 * SV);
#pragma unroll
      for (int e = 0; e < SV; ++e) hcur[e] = hp0[e], dAc[e] = T(0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const T dj = Ds[r * CW + j2], dyv = Ys[r * CW + j2];
        T h4[SV], g4[SV];
        cv.lds(h4, hcol + r * BP);
        cv.lds(g4, gcol + r * BP);
        T ddv = T(0);
#pragma unroll
        for (int e = 0; e < SV; ++e) {
          const T av = F::exp_scaled(dj * A2[e]);
          const T tv = g4[e] * hcur[e] * av;  // G h(i-1,j) Abar
          dAc[e] = fma(tv, dj, dAc[e]);
          ddv = fma(tv, A2[e], ddv);
          hcur[e] = fma(av, hcur[e], h4[e]);
        }
#pragma unroll
        for (int o = 1; o < QV; o <<= 1) ddv += __shfl_xor_sync(kFull, ddv, o);
        if (col_ok && r < rows) {
          if (s2 == 0) DVs[r * CW + j2] = ddv;
          T dc[SV];
#pragma unroll
          for (int e = 0; e < SV; ++e) dc[e] = dyv * hcur[e];
          if constexpr (RED)
            cv.red(dCg + (static_cast<size_t>(r0 + r) * W + j2) * N, dc);
          else
            cv.stg(dCg + (static_cast<size_t>(r0 + r) * W + j2) * N, dc);
        }
      }
      T acc[SV];  // DAs holds the lane's dA partials in natural state order
      cv.lds(acc, DAs);
#pragma unroll
      for (int e = 0; e < SV; ++e) acc[e] += dAc[e];
      cv.sts(DAs, acc);
    }
    __syncwarp();

    // ---- R2 (row lanes): Gh right -> left, the Gh hh(i,j-1) half, dB, per-cell sums
    {
      T rho[SH];
#pragma unroll
      for (int e = 0; e < SH; ++e) rho[e] = T(0);
      if (succ_ring) {
        ring.get(id.wi - 1, u, lane, rho);
        if (!row_ok) {
#pragma unroll
          for (int e = 0; e < SH; ++e) rho[e] = T(0);
        }
      } else if (has_succ && row_ok) {
        if constexpr (sizeof(T) == 4) {
          carry_resolve<SH>(reinterpret_cast<const CarrySlot<float>*>(rc_in + static_cast<size_t>(i1) * N),
                            *reinterpret_cast<CarryPre<float, SH>*>(&rpre), row_tag(epoch, i1),
                            *reinterpret_cast<float(*)[SH]>(rho));
#if S2D_CARRY_PF_B
          if (t > 0)  // the next tile up
            carry_load<SH>(reinterpret_cast<const CarrySlot<float>*>(rc_in + static_cast<size_t>(i1 - R) * N),
                           *reinterpret_cast<CarryPre<float, SH>*>(&rpre));
#endif
        } else
          carry_get_wait<T, SH>(rc_in + static_cast<size_t>(i1) * N, rho, row_tag(epoch, i1), SH);
      }
      const T* dr = Ds + r1 * CW;
      const T* ur = DXs + r1 * CW;
      const T* gr = Cs + r1 * BP + q1 * SH;
      const T* hr = HHs + r1 * BP + q1 * SH;
      T* dBrow = dBg + static_cast<size_t>(i1) * WN;
#pragma unroll
      for (int gs = CW - RG; gs >= 0; gs -= RG) {
        T ddp[RG], sgb[RG];
#pragma unroll
        for (int jj = RG - 1; jj >= 0; --jj) {
          const int j = gs + jj;
          T g4[SH], hl[SH];
          lds_vec<T, SH>(g4, gr + j * N);
          if (j > 0) {
            lds_vec<T, SH>(hl, hr + (j - 1) * N);
          } else {
#pragma unroll
            for (int e = 0; e < SH; ++e) hl[e] = hh0[e];
          }
          const T dj = dr[j], uj = ur[j];
          T dd = T(0), sg = T(0), dBv[SH];
#pragma unroll
          for (int e = 0; e < SH; ++e) {
            const T av = F::exp_scaled(dj * A1[e]);
            const T gh = g4[e] + rho[e];  // engine.cpp:346
            rho[e] = av * gh;
            const T th = rho[e] * hl[e];  // Gh hh(i,j-1) Abar
            dAr[e] = fma(th, dj, dAr[e]);
            dd = fma(th, A1[e], dd);
            sg = fma(gh, bc[j][e], sg);
            dBv[e] = gh * uj;
          }
          ddp[jj] = dd;
          sgb[jj] = sg;
          if (row_ok && j < ncols) {
            if constexpr (RED)
              red_states<T, SH>(dBrow + static_cast<size_t>(j) * N, dBv);
            else
              stg_stream<T, SH>(dBrow + static_cast<size_t>(j) * N, dBv);
          }
        }
        // columns gs .. gs+RG-1 are done with B: load the next tile's (one up) in place
        if (t > 0) {
#pragma unroll
          for (int jj = 0; jj < RG; ++jj) {
            const int j = gs + jj;
            if (j < ncols)
              ldg_states<T, SH>(bc[j], Bg + static_cast<size_t>(i1 - R) * WN + static_cast<size_t>(j) * N);
          }
        }
        const int cb = reduce_scatter<QH, RG>(ddp, q1);
        reduce_scatter<QH, RG>(sgb, q1);
        constexpr int REP = RS<QH, RG>::kReplica;
        const int j = gs + cb;
        if (row_ok && j < ncols && (q1 & (REP - 1)) == 0) {
          const int c = r1 * CW + j;
          const T dv = Ds[c], xv = Xs[c], dyv = Ys[c];
          const T dd = fma(ddp[0] + DVs[c], LN, xv * sgb[0]);  // ddelta = sum_d dAbar Abar A + x sum_d Gh B
          const T dzv = dd * SGs[c];
          dxg[static_cast<size_t>(i1) * W + j] = fma(Dsk, dyv, dv * sgb[0]);
          dzg[static_cast<size_t>(i1) * W + j] = dzv;
          dbias_acc += static_cast<double>(dzv);
          dD_acc = fma(static_cast<double>(dyv), static_cast<double>(xv), dD_acc);
        }
      }
      if (pred_ring)
        ring.put(id.wi, u, lane, rho);
      else if (has_pred && row_ok)
        carry_put<T, SH>(rc_out + static_cast<size_t>(i1) * N, rho, row_tag(epoch, i1), SH);
    }
    __syncwarp();
    sc = sn;
  }

  if (a.gtop != nullptr && col_ok)  // row-band shard: the band above continues from here
    cv.stg(a.gtop + (s * W + jg2) * N + s2 * SV, dn);
  if (a.link_out != nullptr) link_post(a.link_out + s * ge.wreal + wpos, a.link_seq, lane);

  // ---- per-(scan, strip) partials, fixed order: dA = row-lane part + column-lane part
#pragma unroll
  for (int e = 0; e < SH; ++e)
    for (int h = QH; h < 32; h <<= 1) dAr[e] += __shfl_xor_sync(kFull, dAr[e], h);
  T dAc[SV];
  lds_vec<T, SV>(dAc, DAs);
#pragma unroll
  for (int e = 0; e < SV; ++e)
    for (int h = QV; h < 32; h <<= 1) dAc[e] += __shfl_xor_sync(kFull, dAc[e], h);
  for (int h = 1; h < 32; h <<= 1) {
    dbias_acc += __shfl_xor_sync(kFull, dbias_acc, h);
    dD_acc += __shfl_xor_sync(kFull, dD_acc, h);
  }
  T* scr = sm + TS::B_SCR;
  if (lane < QH) {
#pragma unroll
    for (int e = 0; e < SH; ++e) scr[q1 * SH + e] = dAr[e];
  }
  __syncwarp();
  T* part = a.part + (static_cast<size_t>(s) * ge.wreal + wpos) * (N + 2);
  if (lane < QV) {
#pragma unroll
    for (int e = 0; e < SV; ++e) part[s2 * SV + e] = scr[s2 * SV + e] + dAc[e];
  }
  if (lane == 0) {
    part[N] = static_cast<T>(dbias_acc);
    part[N + 1] = static_cast<T>(dD_acc);
  }
  if (a.fuse) {  // P == S: the scan's last strip adds the partials, strip order fixed
    bool last = ge.wreal == 1;
    if (!last) {
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(a.scan_cnt + s, 1);
      last = __shfl_sync(kFull, old, 0) == ge.wreal - 1;
      if (last) __threadfence();
    }
    if (last) {
      const T* ps = a.part + static_cast<size_t>(s) * ge.wreal * (N + 2);
      for (int k = lane; k < N + 2; k += 32) {
        T acc = T(0);
        for (int w = 0; w < ge.wreal; ++w) acc += __ldcg(ps + static_cast<size_t>(w) * (N + 2) + k);
        if (k < N)
          a.dA_out[static_cast<size_t>(s) * N + k] = acc;
        else if (k == N)
          a.dbias_out[s] = acc;
        else
          a.dD_out[s] = acc;
      }
    }
  }
}

}  // namespace s2d
