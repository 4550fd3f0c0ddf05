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

// ------------------------------------------------------------------ numerics

template <typename T>
struct Num;

template <>
struct Num<float> {
  // exp(x) as 2^(x log2 e) on the MUFU.EX2 pipe; the caller pre-scales A by log2 e
#ifdef S2D_POLY_EXP  // diagnostics: 2^t by range reduction + degree-7 polynomial (< 1 ulp)
  static __device__ __forceinline__ float exp_scaled(float t) {
    t = fmaxf(t, -126.0f);
    const float k = rintf(t);
    const float f = t - k;  // exact, |f| <= 0.5
    float p = 1.5252733804059841e-05f;
    p = fmaf(p, f, 1.5403530393381608e-04f);
    p = fmaf(p, f, 1.3333558146428443e-03f);
    p = fmaf(p, f, 9.6181291076284772e-03f);
    p = fmaf(p, f, 5.5504108664821580e-02f);
    p = fmaf(p, f, 2.4022650695910071e-01f);
    p = fmaf(p, f, 6.9314718055994531e-01f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (static_cast<int>(k) << 23));
  }
#else
  static __device__ __forceinline__ float exp_scaled(float x_log2e) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x_log2e));
    return r;
  }
#endif
  static __device__ __forceinline__ float a_scale(float a) { return a * 1.4426950408889634f; }
  // exp(x) for natural x with the rounding of x log2 e and the low part of
  // log2 e folded back: no per-state systematic bias from a pre-rounded
  // A log2 e (the general warp kernels, where N can reach 128 states and
  // that bias adds up coherently in the per-scan dbias sum)
  static __device__ __forceinline__ float exp_nat(float x) {
    const float t = x * 1.44269502162933349609375f;
    const float e = fmaf(x, 1.44269502162933349609375f, -t) + x * 1.925963033500011079e-8f;
    const float r = exp_scaled(t);
    return fmaf(r, e * 0.6931471805599453f, r);
  }
  static __device__ __forceinline__ float rcp(float v) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
  }
  // softplus(v) = max(v, 0) + log1p(exp(-|v|)), log1p(t) = 2 atanh(t / (2 + t)).
  // With s = t/(2+t) in [0, 1/3], the odd atanh series to s^13 leaves a
  // relative error < 2e-8; two MUFU ops (ex2, rcp) and ~14 FMA-pipe ops.
#ifdef S2D_ACCURATE_SCALARS  // diagnostics: IEEE-accurate scalar functions
  static __device__ __forceinline__ float softplus(float v) { return v > 20.0f ? v : log1pf(expf(v)); }
  static __device__ __forceinline__ float sigmoid(float v) {
    if (v >= 0.0f) return 1.0f / (1.0f + expf(-v));
    const float e = expf(v);
    return e / (1.0f + e);
  }
#else
  static __device__ __forceinline__ float softplus(float v) {
    const float t = exp_scaled(-fabsf(v) * 1.4426950408889634f);
    const float s = t * rcp(2.0f + t);
    const float s2 = s * s;
    float p = 1.0f / 13.0f;
    p = fmaf(p, s2, 1.0f / 11.0f);
    p = fmaf(p, s2, 1.0f / 9.0f);
    p = fmaf(p, s2, 1.0f / 7.0f);
    p = fmaf(p, s2, 1.0f / 5.0f);
    p = fmaf(p, s2, 1.0f / 3.0f);
    p = fmaf(p, s2, 1.0f);
    const float l1p = 2.0f * s * p;
    const float r = fmaxf(v, 0.0f) + l1p;
    return v > 20.0f ? v : r;
  }
  static __device__ __forceinline__ float sigmoid(float v) {
    const float e = exp_scaled(-fabsf(v) * 1.4426950408889634f);  // exp(-|v|)
    const float r = rcp(1.0f + e);
    return v >= 0.0f ? r : e * r;
  }
#endif
};

template <>
struct Num<double> {
  static __device__ __forceinline__ double exp_scaled(double x) { return exp(x); }
  static __device__ __forceinline__ double a_scale(double a) { return a; }
  static __device__ __forceinline__ double exp_nat(double x) { return exp(x); }
  static __device__ __forceinline__ double softplus(double v) {
    return v > 20.0 ? v : log1p(exp(v));
  }
  static __device__ __forceinline__ double sigmoid(double v) {
    if (v >= 0.0) return 1.0 / (1.0 + exp(-v));
    const double e = exp(v);
    return e / (1.0 + e);
  }
};

// Accurate-exponential policy (desc flag SCAN2D_FLAG_ACCURATE): MUFU.EX2
// (ex2.approx) carries up to ~2 ulp of relative error with a consistent sign,
// which the 2D recurrences accumulate along every path -- the measured cause of
// the fast path's fp32 error being ~2-3x the reference fp32 engine's.  The
// accurate policy evaluates 2^t by range reduction (t = k + f, |f| <= 1/2) and a
// degree-7 polynomial in f (truncation < 6e-9 relative, i.e. < 0.1 ulp before
// rounding), the scaling by 2^k exact; softplus / sigmoid use it and IEEE
// division.  Kernels take it as a template parameter (no cost when off).
template <typename T, bool ACC>
struct Fn : Num<T> {};

template <>
struct Fn<float, true> {
  static __device__ __forceinline__ float exp_scaled(float t) {
    t = fminf(fmaxf(t, -125.0f), 126.0f);
    const float k = rintf(t);
    const float f = t - k;  // exact
    float p = 1.5252733804059841e-05f;
    p = fmaf(p, f, 1.5403530393381608e-04f);
    p = fmaf(p, f, 1.3333558146428443e-03f);
    p = fmaf(p, f, 9.6181291076284772e-03f);
    p = fmaf(p, f, 5.5504108664821580e-02f);
    p = fmaf(p, f, 2.4022650695910071e-01f);
    p = fmaf(p, f, 6.9314718055994531e-01f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (static_cast<int>(k) << 23));
  }
  static __device__ __forceinline__ float a_scale(float a) { return Num<float>::a_scale(a); }
  static __device__ __forceinline__ float softplus(float v) {
    const float t = exp_scaled(-fabsf(v) * 1.4426950408889634f);
    const float s = __fdiv_rn(t, 2.0f + t);
    const float s2 = s * s;
    float p = 1.0f / 13.0f;
    p = fmaf(p, s2, 1.0f / 11.0f);
    p = fmaf(p, s2, 1.0f / 9.0f);
    p = fmaf(p, s2, 1.0f / 7.0f);
    p = fmaf(p, s2, 1.0f / 5.0f);
    p = fmaf(p, s2, 1.0f / 3.0f);
    p = fmaf(p, s2, 1.0f);
    const float r = fmaxf(v, 0.0f) + 2.0f * s * p;
    return v > 20.0f ? v : r;
  }
  static __device__ __forceinline__ float sigmoid(float v) {
    const float e = exp_scaled(-fabsf(v) * 1.4426950408889634f);
    const float r = __fdiv_rn(1.0f, 1.0f + e);
    return v >= 0.0f ? r : e * r;
  }
};

// ------------------------------------------------------------ shared memory

// Parameter row p = s mod P and B/C group s / G of scan s, without a 64-bit
// integer division in the common cases (per-scan parameters P == S, G == 1,
// or S < 2^31: a 32-bit division) -- the 64-bit ones are software routines
// that were a visible share of the short row kernels' instructions.
__device__ __forceinline__ int param_row(int64_t s, int64_t S, int P) {
  if (P == S) return static_cast<int>(s);
  if (s < 0x7fffffff) return static_cast<int>(static_cast<uint32_t>(s) % static_cast<uint32_t>(P));
  return static_cast<int>(s % P);
}
__device__ __forceinline__ int64_t bc_row(int64_t s, int G) {
  if (G == 1) return s;
  if (s < 0x7fffffff) return static_cast<int64_t>(static_cast<uint32_t>(s) / static_cast<uint32_t>(G));
  return s / G;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async (LDGSTS): global -> shared without staging through registers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
// No "memory" clobber: the destination slot is fenced by the __syncwarp that
// ends its previous use and by cp_async_wait (which has one) before its next
// read, so the compiler may schedule the issue among surrounding work.
__device__ __forceinline__ void cp_async16_raw(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_elem(float* smem, const float* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_elem(double* smem, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int NPending>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(NPending) : "memory");
}
// wait until at most n committed groups are pending (n is warp-uniform)
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    default: cp_async_wait<7>(); break;
  }
}

// Band hand-off flags at system scope (the producer may be another GPU).
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Wait (lane 0 polls, the warp follows) until *flag == seq.  A producer that
// never arrives (a misconfigured link) must neither hang the GPU nor let the
// strip continue on a stale carry: after 10 s the kernel traps, so the launch
// fails loudly (cudaErrorLaunchFailure on the next synchronisation).
__device__ __forceinline__ void link_wait(const int* flag, int seq, int lane) {
  if (lane == 0) {
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flag) != seq) {
      __nanosleep(200);
      if (global_ns() - t0 > 10000000000ull) __trap();
    }
  }
  __syncwarp();
}
// Publish: every lane's carry stores are made visible system-wide first.
__device__ __forceinline__ void link_post(int* flag, int seq, int lane) {
  __threadfence_system();
  __syncwarp();
  if (lane == 0) st_release_sys(flag, seq);
}

// Pause between polls of a carry word.  __nanosleep deschedules the warp for
// far longer than asked on sm_100 when the word is not ready yet (one global
// hop between two CTAs measured 2.2x slower with it); a short clock spin keeps
// the re-poll latency near the L2 round trip.
#ifdef S2D_NO_POLL_PAUSE
__device__ __forceinline__ void poll_pause() {}
#else
__device__ __forceinline__ void poll_pause() {
  const long long t0 = clock64();
  while (clock64() - t0 < 64) {
  }
}
#endif

// ------------------------------------------------------ gpu-scope carries
//
// Workspace header (first bytes of every chained launch's workspace).  The
// epoch lives in device memory and is advanced by scan2d_begin_kernel, which
// runs in stream order before every chained launch (so a captured CUDA graph
// advances it on every replay).  `magic` identifies the workspace layout the
// carry region was last used with: on a mismatch (fresh memory, or a workspace
// last used for another descriptor / op) the begin kernel clears the carry
// region before any tag is trusted; the main kernel then records the magic.
struct WsHdr {
  int ticket;      // CTA / warp ticket counter (reset by the begin kernel)
  uint32_t epoch;  // tag base of the current launch, in [0, kTagSpan)
  uint32_t magic;  // layout hash of the last launch that used the carry region
  uint32_t pad;
};
//
// Tags are quiet-NaN bit patterns 0x7fc00001 .. 0x7ffffffd, unique per (launch,
// row) modulo kTagSpan: no finite float can be mistaken for a tag, and neither
// can the canonical NaNs 0x7fffffff (GPU) / 0x7fc00000 (CPU) or zeroed memory.
// Every consumed slot is rewritten by every launch with the same layout, so a
// stale slot only ever holds the previous launch's tag, and the epoch step
// (H + 1, or H + 2 when that is a multiple of kTagSpan) makes that tag differ.
constexpr uint32_t kTagSpan = 0x3ffffdu;
#ifdef S2D_MASK_TAG
__device__ __forceinline__ int row_tag(uint32_t epoch, int row) {
  return static_cast<int>(0x7fc00001u + ((epoch + static_cast<uint32_t>(row)) & 0x1fffffu));
}
#else
__device__ __forceinline__ int row_tag(uint32_t epoch, int row) {
  return static_cast<int>(0x7fc00001u + (epoch + static_cast<uint32_t>(row)) % kTagSpan);
}
#endif
// Programmatic dependent launch: a chained kernel is launched while its begin
// kernel may still run; it waits here (before touching the header or any
// carry slot) until the begin kernel's writes are visible.  A no-op when the
// kernel was launched without the PDL attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint32_t load_epoch(const WsHdr* h) {
  return *reinterpret_cast<const volatile uint32_t*>(&h->epoch) % kTagSpan;
}
//
// Column-group carries travel between warps (one warp per CTA) through global
// memory.  fp32: the value and its row tag share one naturally aligned 8-byte
// word, so a single relaxed store publishes both (no fence on the chain).
// fp64: value, fence, then tag.

template <typename T>
struct CarrySlot;

template <>
struct CarrySlot<float> {
  uint64_t w;
  static __device__ __forceinline__ void put(CarrySlot* p, float v, int tag) {
    const uint64_t w = (static_cast<uint64_t>(static_cast<uint32_t>(tag)) << 32) |
                       static_cast<uint64_t>(__float_as_uint(v));
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(&p->w), "l"(w) : "memory");
  }
  static __device__ __forceinline__ float get_wait(const CarrySlot* p, int tag) {
    uint64_t w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(&p->w) : "memory");
    while (static_cast<int>(w >> 32) != tag) {
      poll_pause();
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(&p->w) : "memory");
    }
    return __uint_as_float(static_cast<uint32_t>(w));
  }
  static __device__ __forceinline__ float get(const CarrySlot* p) {
    return __uint_as_float(static_cast<uint32_t>(p->w));
  }
};

template <>
struct CarrySlot<double> {
  double v;
  long long tag;
  static __device__ __forceinline__ void put(CarrySlot* p, double v, int tag) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(&p->v), "d"(v) : "memory");
    __threadfence();
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(&p->tag), "l"(static_cast<long long>(tag))
                 : "memory");
  }
  static __device__ __forceinline__ double get_wait(const CarrySlot* p, int tag) {
    long long t;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(t) : "l"(&p->tag) : "memory");
    while (static_cast<int>(t) != tag) {
      poll_pause();
      asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(t) : "l"(&p->tag) : "memory");
    }
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(&p->v) : "memory");
    return v;
  }
  static __device__ __forceinline__ double get(const CarrySlot* p) { return p->v; }
};

// SPL consecutive carry slots (states q*SPL .. q*SPL+SPL-1 of one row).
template <typename T, int SPL>
__device__ __forceinline__ void carry_put(CarrySlot<T>* p, const T (&v)[SPL], int tag, int nvalid) {
  if constexpr (sizeof(T) == 4 && SPL >= 2) {
    if (nvalid >= SPL && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int e = 0; e < SPL; e += 2) {
        const uint64_t w0 = (static_cast<uint64_t>(static_cast<uint32_t>(tag)) << 32) | __float_as_uint(v[e]);
        const uint64_t w1 = (static_cast<uint64_t>(static_cast<uint32_t>(tag)) << 32) | __float_as_uint(v[e + 1]);
        asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(&p[e].w), "l"(w0), "l"(w1)
                     : "memory");
      }
      return;
    }
  }
#pragma unroll
  for (int e = 0; e < SPL; ++e)
    if (e < nvalid) CarrySlot<T>::put(p + e, v[e], tag);
}

template <typename T, int SPL>
__device__ __forceinline__ void carry_get_wait(const CarrySlot<T>* p, T (&v)[SPL], int tag, int nvalid) {
  if constexpr (sizeof(T) == 4 && SPL >= 2) {
    if (nvalid >= SPL && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      uint64_t w[SPL];
      bool ok;
      int spins = 0;
      do {
        if (spins++) poll_pause();
#pragma unroll
        for (int e = 0; e < SPL; e += 2)
          asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                       : "=l"(w[e]), "=l"(w[e + 1])
                       : "l"(&p[e].w)
                       : "memory");
        ok = true;
#pragma unroll
        for (int e = 0; e < SPL; ++e) ok = ok && static_cast<int>(w[e] >> 32) == tag;
      } while (!ok);
#pragma unroll
      for (int e = 0; e < SPL; ++e) v[e] = __uint_as_float(static_cast<uint32_t>(w[e]));
      return;
    }
  }
#pragma unroll
  for (int e = 0; e < SPL; ++e) v[e] = e < nvalid ? CarrySlot<T>::get_wait(p + e, tag) : T(0);
}

// Prefetchable carry read: `carry_load` issues the loads (no waiting) and
// `carry_resolve` checks the tags, re-polling only if the producer was late.
template <typename T, int SPL>
struct CarryPre {
  uint64_t w[SPL];
};

template <int SPL>
__device__ __forceinline__ void carry_load(const CarrySlot<float>* p, CarryPre<float, SPL>& c) {
  if constexpr (SPL >= 2) {
#pragma unroll
    for (int e = 0; e < SPL; e += 2)
      asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                   : "=l"(c.w[e]), "=l"(c.w[e + 1])
                   : "l"(&p[e].w)
                   : "memory");
  } else {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(c.w[0]) : "l"(&p[0].w) : "memory");
  }
}

template <int SPL>
__device__ __forceinline__ void carry_resolve(const CarrySlot<float>* p, CarryPre<float, SPL>& c, int tag,
                                              float (&v)[SPL]) {
  bool ok = true;
#pragma unroll
  for (int e = 0; e < SPL; ++e) ok = ok && static_cast<int>(c.w[e] >> 32) == tag;
  while (!ok) {
    poll_pause();
    carry_load<SPL>(p, c);
    ok = true;
#pragma unroll
    for (int e = 0; e < SPL; ++e) ok = ok && static_cast<int>(c.w[e] >> 32) == tag;
  }
#pragma unroll
  for (int e = 0; e < SPL; ++e) v[e] = __uint_as_float(static_cast<uint32_t>(c.w[e]));
}

template <typename T, int SPL>
__device__ __forceinline__ void carry_get(const CarrySlot<T>* p, T (&v)[SPL], int nvalid) {
#pragma unroll
  for (int e = 0; e < SPL; ++e) v[e] = e < nvalid ? CarrySlot<T>::get(p + e) : T(0);
}

// plain (untagged) residual copies of carries: the first nvalid states
template <typename T, int SPL>
__device__ __forceinline__ void store_states(T* p, const T (&v)[SPL], int nvalid) {
#pragma unroll
  for (int e = 0; e < SPL; ++e)
    if (e < nvalid) p[e] = v[e];
}
template <typename T, int SPL>
__device__ __forceinline__ void load_states(T (&v)[SPL], const T* p, int nvalid) {
#pragma unroll
  for (int e = 0; e < SPL; ++e) v[e] = e < nvalid ? p[e] : T(0);
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

template <int LPC, int J>
struct RS {
  static constexpr int kKeep = (J / LPC) > 1 ? (J / LPC) : 1;
  static constexpr int kDistinct = J / kKeep;
  static constexpr int kReplica = LPC / kDistinct;
};

template <int J, typename T>
__device__ __forceinline__ T select_col(const T (&v)[J], int k) {
  T r = v[0];
#pragma unroll
  for (int m = 1; m < J; ++m)
    if (m == k) r = v[m];
  return r;
}

// SPL consecutive states of one cell from shared memory
template <typename T, int SPL>
__device__ __forceinline__ void lds_states(T (&out)[SPL], const T* p, bool vec) {
  if constexpr (SPL == 4 && sizeof(T) == 4) {
    if (vec) {
      const float4 v = *reinterpret_cast<const float4*>(p);
      out[0] = v.x;
      out[1] = v.y;
      out[2] = v.z;
      out[3] = v.w;
      return;
    }
  }
  if constexpr (SPL == 2 && sizeof(T) == 4) {
    if (vec) {
      const float2 v = *reinterpret_cast<const float2*>(p);
      out[0] = v.x;
      out[1] = v.y;
      return;
    }
  }
  if constexpr (SPL >= 2 && sizeof(T) == 8) {
    if (vec) {
#pragma unroll
      for (int s = 0; s < SPL; s += 2) {
        const double2 v = *reinterpret_cast<const double2*>(p + s);
        out[s] = v.x;
        out[s + 1] = v.y;
      }
      return;
    }
  }
#pragma unroll
  for (int s = 0; s < SPL; ++s) out[s] = p[s];
}

// SPL consecutive states to shared memory (vectorised)
template <typename T, int SPL>
__device__ __forceinline__ void sts_states(T* p, const T (&v)[SPL]) {
  if constexpr (sizeof(T) == 4 && SPL % 4 == 0) {
#pragma unroll
    for (int e = 0; e < SPL; e += 4) *reinterpret_cast<float4*>(p + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
  } else if constexpr (sizeof(T) == 4 && SPL == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else if constexpr (sizeof(T) == 8 && SPL % 2 == 0) {
#pragma unroll
    for (int e = 0; e < SPL; e += 2) *reinterpret_cast<double2*>(p + e) = make_double2(v[e], v[e + 1]);
  } else {
#pragma unroll
    for (int e = 0; e < SPL; ++e) p[e] = v[e];
  }
}

template <typename T, int SPL>
__device__ __forceinline__ void stg_states(T* p, const T (&v)[SPL], int nvalid, bool vec) {
  if constexpr (SPL > 4 && SPL % 4 == 0 && sizeof(T) == 4) {
    if (vec && nvalid >= SPL) {
#pragma unroll
      for (int e = 0; e < SPL; e += 4)
        *reinterpret_cast<float4*>(p + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      return;
    }
  }
  if constexpr (SPL == 4 && sizeof(T) == 4) {
    if (vec) {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
      return;
    }
  }
  if constexpr (SPL == 2 && sizeof(T) == 4) {
    if (vec) {
      *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
      return;
    }
  }
#pragma unroll
  for (int s = 0; s < SPL; ++s)
    if (s < nvalid) p[s] = v[s];
}

// ---------------------------------------------------------------- planning

// Geometry of one kernel direction.  A warp owns `colsw` columns of one scan
// (or `seg` whole narrow scans); lanes = (chunk, state group): SPL states of
// J consecutive columns per lane, LPC lanes per chunk, CPW = 32/LPC chunks.
struct Geo {
  int tile;     // 1: tile kernels (scan2d_tile2.cuh), CW = colsw
  int rows1;    // 1: N = 1 row-sweep kernels (scan2d_rows1.cuh): J columns per lane, `seg` lanes per scan
  int spl, lpc, cpw, J;
  int Np;       // states padded to spl * lpc (zero-filled in shared memory)
  int seg;      // scans packed per warp (power of two)
  int cps;      // chunks per segment = cpw / seg
  int colsw;    // columns per warp (per segment)
  int wreal;    // warps per scan with at least one real column
  int stages;   // depth of the cp.async row pipeline
  int64_t units;  // warps (= CTAs) in the launch
  int stage_elems;  // elements per pipeline stage
  int table_off;    // element offset of the copy table in shared memory
  int smem_bytes;   // dynamic shared memory per CTA (tile kernels: per warp)
  int cta_warps;    // tile kernels: warps (strips) per CTA, set at launch
  int ctas_per_scan;  // tile kernels: CTAs per scan, set at launch
};

struct Plan {
  Geo f;      // forward
  Geo b;      // backward
  int K;      // backward band rows (= residual checkpoint interval)
  int nb;     // ceil(H / K)
  int Q;      // column interval of the saved horizontal carries (= b.colsw)
  int nq;     // ceil(W / Q) - 1 carry boundaries per row
  int warp_ok;  // the warp kernels' geometry fits this residual layout (else tile / rows1 kernels only)
  int pfd;      // N = 1 forward: L2 prefetch distance in rows
  int pft_f, pft_b;  // tile kernels: bulk L2 prefetch distance in tiles (forward / backward; 0 = off)
  int pf_all;        // tile kernels: prefetch the whole strip into L2 at the start (small problems)
  int pf_mode;       // tile kernels: 1 = per-lane line prefetches, 2 = TMA bulk prefetches (lane 0)
  int tma;           // tile kernels: stage C (and aligned x / z / dy rows) by TMA bulk copies
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
  T* ckpt;              // residual: h at the last row of each band but the last, [S][nb-1][W][N]
  // row-band shard (one band of a taller grid): vertical carries across the band edges
  const T* vtop;        // h of the row above the band, [S][W][N] (NULL = zeros)
  T* vbot;              // forward: h of the band's last row, [S][W][N] (NULL = not wanted)
  const T* gbot;        // backward: Abar G of the row below the band, [S][W][N] (NULL = zeros)
  T* gtop;              // backward: Abar G of the band's first row, [S][W][N] (NULL = not wanted)
  // in-kernel hand-off between bands on different GPUs (scan2d_*_band_linked):
  // per (scan, 16-column strip) flags; a strip waits until link_in[s][strip]
  // == link_seq before reading its incoming carry (vtop forward, gbot
  // backward) and publishes link_out[s][strip] = link_seq after storing its
  // outgoing carry (vbot / gtop, typically peer memory over NVLink)
  const int* link_in;
  int* link_out;
  int link_seq;
  int acc;               // accurate exponential policy (Fn<T, true>)
  CarrySlot<T>* hcarry; // forward chain: tagged horizontal carries at Q-column boundaries, [S][nq][H][N]
  T* hres;              // residual: plain horizontal carries at every Q-column boundary, [S][nq][H][N]
  // backward outputs
  T* dx;
  T* dz;
  T* dB;       // [S][H][W][N] (per scan; reduced over the B/C group afterwards when G > 1)
  T* dC;
  T* part;     // per (scan, warp) partials: [S][wreal_b][N + 2] = dA[N], dbias, dD
  // fused parameter-gradient reduction (per-scan parameters, P == S): the last
  // strip of a scan to finish sums the scan's partials in strip order
  int fuse;
  int* scan_cnt;  // [S] strips finished per scan (zeroed before the launch)
  T* dA_out;
  T* dbias_out;
  T* dD_out;
  CarrySlot<T>* rcarry;  // reverse carry at backward warp boundaries, [S][wreal_b-1][H][N]
  int* ticket;           // warp ticket counter (= &hdr->ticket; reset by the begin kernel)
  WsHdr* hdr;            // workspace header (epoch, layout magic); NULL when nothing is chained
  uint32_t magic;        // layout hash this launch records in hdr->magic
  int pdl;               // launch with programmatic stream serialization (after a begin kernel)
  int xvec, bvec, yvec;  // 16-byte copy units legal for x-like / B-like spans; vector y stores
  int ovec;              // backward: dB / dC 16-byte aligned (vector state stores legal)
  int red;               // backward, G > 1: dB / dC accumulated in place over the group (L2 reductions)
  // shape
  int64_t S;
  int H, W, N, T_tile, P, G;
  Plan plan;
};

}  // namespace s2d
