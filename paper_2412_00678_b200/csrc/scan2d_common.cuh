// scan2d_common.cuh -- device building blocks shared by the forward and backward
// 2D selective-scan kernels (sm_100a).
//
// Numerics follow the reference helpers (proj/include/scan2d/math.hpp):
//   softplus with the cutoff 20 (:14-21), sigmoid (:23-28),
//   Abar = exp(delta * A)       (:81-84; fp32 via ex2.approx, fp64 via exp),
//   Bbar x = (delta * B) * x    (:86-89), ssm_step = fma(a, h, b) (:92-95).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace s2d {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRing = 4;  // depth of the intra-CTA carry rings (rows in flight per hop)

// ------------------------------------------------------------------ numerics

template <typename T>
struct Num;

template <>
struct Num<float> {
  // exp(x) as 2^(x log2 e) on the MUFU.EX2 pipe; the caller pre-scales A by log2 e
  static __device__ __forceinline__ float exp_scaled(float x_log2e) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x_log2e));
    return r;
  }
  static __device__ __forceinline__ float a_scale(float a) { return a * 1.4426950408889634f; }
  static __device__ __forceinline__ float softplus(float v) {
    return v > 20.0f ? v : log1pf(__expf(v));
  }
  static __device__ __forceinline__ float sigmoid(float v) {
    if (v >= 0.0f) return __frcp_rn(1.0f + __expf(-v));
    const float e = __expf(v);
    return e / (1.0f + e);
  }
};

template <>
struct Num<double> {
  static __device__ __forceinline__ double exp_scaled(double x) { return exp(x); }
  static __device__ __forceinline__ double a_scale(double a) { return a; }
  static __device__ __forceinline__ double softplus(double v) {
    return v > 20.0 ? v : log1p(exp(v));
  }
  static __device__ __forceinline__ double sigmoid(double v) {
    if (v >= 0.0) return 1.0 / (1.0 + exp(-v));
    const double e = exp(v);
    return e / (1.0 + e);
  }
};

// ------------------------------------------------------------ shared memory

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mbarrier wrappers (CTA scope).  arrive has release semantics, try_wait acquire.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------ gpu-scope signalling

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float ld_relaxed_gpu(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_gpu(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Spin (all lanes) until *flag > target; returns the observed value.
__device__ __forceinline__ int wait_flag_gt(const int* flag, int target) {
  int v = ld_acquire_gpu(flag);
  while (v <= target) {
    __nanosleep(32);
    v = ld_acquire_gpu(flag);
  }
  return v;
}

// ------------------------------------------------------- warp collectives

// Reduce-scatter of v[J] over the LPC lanes of a chunk (lane bits below LPC).
// On return lane l holds max(J/LPC, 1) consecutive columns starting at the
// returned offset; lanes that only differ in the low "replica" bits hold
// identical bits (the final butterfly adds are commutative pairs).
template <int LPC, int J, typename T>
__device__ __forceinline__ int reduce_scatter(T (&v)[J], int l) {
  int colbase = 0;
#pragma unroll
  for (int s = 0; (LPC >> (s + 1)) >= 1; ++s) {
    const int h = LPC >> (s + 1);
    const int V = (J >> s) > 1 ? (J >> s) : 1;
    const bool up = (l & h) != 0;
    if (V > 1) {
      const int half = V / 2;
#pragma unroll
      for (int m = 0; m < half; ++m) {
        const T send = up ? v[m] : v[m + half];
        const T keep = up ? v[m + half] : v[m];
        v[m] = keep + __shfl_xor_sync(kFull, send, h);
      }
      if (up) colbase += half;
    } else {
      v[0] += __shfl_xor_sync(kFull, v[0], h);
    }
  }
  return colbase;
}

// columns each lane keeps after reduce_scatter, and the replica span
template <int LPC, int J>
struct RS {
  static constexpr int kKeep = (J / LPC) > 1 ? (J / LPC) : 1;
  static constexpr int kDistinct = J / kKeep;        // distinct column groups per chunk
  static constexpr int kReplica = LPC / kDistinct;   // lanes holding the same columns
};

template <int J, typename T>
__device__ __forceinline__ T select_col(const T (&v)[J], int k) {
  T r = v[0];
#pragma unroll
  for (int m = 1; m < J; ++m)
    if (m == k) r = v[m];
  return r;
}

// butterfly sum over the lane bits in [lo_bit_mask .. 32) selected by `mask_bits`
template <typename T>
__device__ __forceinline__ T xor_sum(T v, int first, int last_exclusive) {
  for (int h = first; h < last_exclusive; h <<= 1) v += __shfl_xor_sync(kFull, v, h);
  return v;
}

// ---------------------------------------------------------------- planning

// Launch geometry shared by host and device (see scan2d_capi.cu: make_plan).
struct Plan {
  int lpc;      // lanes per chunk = state lanes (power of two <= 32)
  int J;        // columns per chunk (per lane)
  int cpw;      // chunks per warp = 32 / lpc
  int seg;      // scans packed per warp (power of two; 1 when a scan spans >= 1 warp)
  int cps;      // chunks per segment = cpw / seg
  int wps;      // warps per scan (padded: nw * ncb) -- 1 when seg > 1
  int wreal;    // warps per scan that own at least one real column
  int nw;       // warps per CTA
  int ncb;      // CTAs across one scan's width (cross-CTA carry chain when > 1)
  int K;        // backward band rows (= checkpoint interval of the residual)
  int nb;       // ceil(H / K)
  int64_t units;  // logical warps = ceil(S / seg) * wps
  int64_t ctas;
  int colsw;    // columns per warp (per segment)
};

template <typename T>
struct Args {
  // inputs
  const T* x;
  const T* z;
  const T* B;
  const T* C;
  const T* A;
  const T* Dskip;
  const T* bias;
  const T* dy;
  // forward outputs
  T* y;
  T* ph;
  T* pv;
  T* ckpt;     // residual: h at the last row of each band but the last, [S][nb-1][W][N]
  T* hcarry;   // horizontal carry at CTA boundaries, [S][ncb-1][H][N]
  // backward outputs
  T* dx;
  T* dz;
  T* dB;       // [S][H][W][N] (per scan; reduced over the B/C group afterwards when G > 1)
  T* dC;
  T* part;     // per (scan, warp) partials: [S][wps][N + 2] = dA[N], dbias, dD
  T* rcarry;   // reverse carry at CTA boundaries, [S][ncb-1][H][N]
  int* flags;  // [0] ticket, [1 + s*(ncb-1) + cb] progress of boundary cb of scan s
  // shape
  int64_t S;
  int H, W, N, T_tile, P, G;
  Plan plan;
};

}  // namespace s2d
