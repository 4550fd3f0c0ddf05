// scan2d_comparators.cu -- the reference's two comparator operators on the GPU
// (SURVEY.md §8f row 1), behind the same C ABI:
//
//   scan2d_forward_naive   naive_scan_2d          (proj/src/engine.cpp:412-487)
//   scan2d_forward_flat1d  block_scan_1d_forward  (proj/src/engine.cpp:489-526)
//
// They exist to be compared against the tiled operator (Table 3 of the paper,
// PAPER.md:280-282) and follow the reference's strategies on purpose:
// naive materialises all N horizontal state maps in HBM and re-derives the
// discretisation in a second, column-wise pass; flat1d scans the row-major
// flattened grid as a 1D sequence (the Mamba baseline).  Association orders
// follow the reference (state sums in ascending d), so fp64 results match the
// sequential oracle to rounding.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/scan2d_cuda.h"
#include "scan2d_common.cuh"

namespace s2d {
namespace {

template <typename T>
__device__ __forceinline__ T abar_exact(T delta, T a) {
  return Num<T>::exp_scaled(delta * Num<T>::a_scale(a));
}

// pass 1: one thread per (scan, row, state) walks the row left to right and
// writes the horizontal state map  maps[s][d][i][j]  (engine.cpp:426-450)
template <typename T>
__global__ void naive_rows_kernel(const T* __restrict__ x, const T* __restrict__ z, const T* __restrict__ B,
                                  const T* __restrict__ A, const T* __restrict__ bias, int64_t S, int H,
                                  int W, int N, int P, int G, T* __restrict__ maps) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = S * H * N;
  if (t >= total) return;
  const int d = static_cast<int>(t % N);
  const int i = static_cast<int>((t / N) % H);
  const int64_t s = t / (static_cast<int64_t>(N) * H);
  const int64_t p = s % P, g = s / G;
  const size_t HW = static_cast<size_t>(H) * W;
  const T ad = A[p * N + d], bs = bias[p];
  T state = T(0);
  T* map = maps + (static_cast<size_t>(s) * N + d) * HW + static_cast<size_t>(i) * W;
  for (int j = 0; j < W; ++j) {
    const size_t cell = static_cast<size_t>(i) * W + j;
    const T dv = Num<T>::softplus(z[s * HW + cell] + bs);
    const T av = abar_exact(dv, ad);
    const T bx = (dv * B[(g * HW + cell) * N + d]) * x[s * HW + cell];
    state = fma(av, state, bx);
    map[j] = state;
  }
}

// pass 2: one thread per (scan, column) walks down the rows; per row the state
// sum runs over d ascending (engine.cpp:454-484); vertical states live in a
// global scratch vst[s][d][j]
template <typename T>
__global__ void naive_cols_kernel(const T* __restrict__ x, const T* __restrict__ z, const T* __restrict__ C,
                                  const T* __restrict__ A, const T* __restrict__ Dskip,
                                  const T* __restrict__ bias, const T* __restrict__ maps, int64_t S, int H,
                                  int W, int N, int P, int G, T* __restrict__ vst, T* __restrict__ y) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= S * W) return;
  const int j = static_cast<int>(t % W);
  const int64_t s = t / W;
  const int64_t p = s % P, g = s / G;
  const size_t HW = static_cast<size_t>(H) * W;
  const T bs = bias[p], dsk = Dskip[p];
  T* vs = vst + static_cast<size_t>(s) * N * W + j;
  for (int d = 0; d < N; ++d) vs[static_cast<size_t>(d) * W] = T(0);
  for (int i = 0; i < H; ++i) {
    const size_t cell = static_cast<size_t>(i) * W + j;
    const T dv = Num<T>::softplus(z[s * HW + cell] + bs);
    T acc = T(0);
    for (int d = 0; d < N; ++d) {
      const T av = abar_exact(dv, A[p * N + d]);
      T st = vs[static_cast<size_t>(d) * W];
      st = fma(av, st, maps[(static_cast<size_t>(s) * N + d) * HW + cell]);
      vs[static_cast<size_t>(d) * W] = st;
      acc = fma(C[(g * HW + cell) * N + d], st, acc);
    }
    y[s * HW + cell] = fma(dsk, x[s * HW + cell], acc);
  }
}

// flat1d: one thread per (scan, state) scans the flattened grid; states go to
// a scratch h[s][k][d]; then one thread per cell sums over d ascending
// (engine.cpp:506-518)
template <typename T>
__global__ void flat_scan_kernel(const T* __restrict__ x, const T* __restrict__ z, const T* __restrict__ B,
                                 const T* __restrict__ A, const T* __restrict__ bias, int64_t S, int64_t L,
                                 int N, int P, int G, T* __restrict__ hs) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= S * N) return;
  const int d = static_cast<int>(t % N);
  const int64_t s = t / N;
  const int64_t p = s % P, g = s / G;
  const T ad = A[p * N + d], bs = bias[p];
  T state = T(0);
  for (int64_t k = 0; k < L; ++k) {
    const T dv = Num<T>::softplus(z[s * L + k] + bs);
    const T av = abar_exact(dv, ad);
    const T bx = (dv * B[(g * L + k) * N + d]) * x[s * L + k];
    state = fma(av, state, bx);
    hs[(s * L + k) * N + d] = state;
  }
}

template <typename T>
__global__ void flat_readout_kernel(const T* __restrict__ x, const T* __restrict__ C, const T* __restrict__ Dskip,
                                    const T* __restrict__ hs, int64_t S, int64_t L, int N, int P, int G,
                                    T* __restrict__ y) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= S * L) return;
  const int64_t s = t / L, k = t % L;
  const int64_t p = s % P, g = s / G;
  T acc = T(0);
  for (int d = 0; d < N; ++d) acc = fma(C[(g * L + k) * N + d], hs[t * N + d], acc);
  y[t] = fma(Dskip[p], x[t], acc);
}

// flat1d, parallel (the "CUB 1D scan" of Table 3 / Mamba's selective scan;
// block_scan_1d_forward's segmented block scan, block_scan.cpp:28-88, on the
// GPU) with a decoupled look-back across CTAs.  The row-major flattening of
// every scan is cut into chunks of kFlatThreads x kFlatEpt elements; CTAs
// take chunk tickets in order (a chunk's predecessors were handed out first).
// Per chunk and state d: the affine pairs (Abar, Bbar x) of a thread's
// elements are folded in registers, combined by a warp shuffle scan and a
// scan over the warp totals; the CTA publishes the chunk AGGREGATE, then
// looks back over its predecessors -- composing aggregates until it meets a
// published INCLUSIVE state -- to get the state entering the chunk
// (block_scan.cpp:51: the carry folded into the head), publishes its own
// INCLUSIVE state and finishes y = sum_d C_d h_d (d ascending, engine.cpp:
// 506-518) in registers.  The N state sequences never touch HBM; only
// 3 N values per chunk do.
constexpr int kFlatThreads = 256;
constexpr int kFlatEpt = 2;
constexpr int kFlatMaxN = 16;  // larger N: the sequential flat kernels above
constexpr int kFlatChunk = kFlatThreads * kFlatEpt;

struct FlatWs {  // workspace: [ticket][status S*nch][aggA, aggB, inc: S*nch*N each]
  int* ticket;
  int* status;  // 0 none, 1 aggregate, 2 inclusive
  void* vals;
};

template <typename T, int N>
__global__ void __launch_bounds__(kFlatThreads) flat_lookback_kernel(
    const T* __restrict__ x, const T* __restrict__ z, const T* __restrict__ B, const T* __restrict__ C,
    const T* __restrict__ A, const T* __restrict__ Dskip, const T* __restrict__ bias, int64_t S, int64_t L,
    int nch, int P, int G, T* __restrict__ y, FlatWs ws) {
  constexpr int NW = kFlatThreads / 32;
  __shared__ T wa[NW][N], wb[NW][N], carry[N], aggA[N], aggB[N];
  __shared__ int64_t tile_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) tile_s = atomicAdd(ws.ticket, 1);
  __syncthreads();
  const int64_t tile = tile_s;
  const int64_t s = tile / nch;
  const int c = static_cast<int>(tile % nch);
  const int64_t p = s % P, g = s / G;
  const int64_t base = static_cast<int64_t>(c) * kFlatChunk;
  const int cnt = static_cast<int>(L - base < kFlatChunk ? L - base : kFlatChunk);
  const T bs = bias[p], dsk = Dskip[p];
  const size_t nv = static_cast<size_t>(S) * nch * N;
  T* vA = static_cast<T*>(ws.vals);
  T* vB = vA + nv;
  T* vI = vB + nv;
  const size_t slot = (static_cast<size_t>(s) * nch + c) * N;

  T dl[kFlatEpt], xv[kFlatEpt], yacc[kFlatEpt], bq[kFlatEpt][N], cq[kFlatEpt][N];
#pragma unroll
  for (int k = 0; k < kFlatEpt; ++k) {
    const int idx = tid * kFlatEpt + k;
    const bool ok = idx < cnt;
    const int64_t e = base + (ok ? idx : 0);
    xv[k] = ok ? x[s * L + e] : T(0);
    dl[k] = ok ? Num<T>::softplus(z[s * L + e] + bs) : T(0);
    yacc[k] = T(0);
#pragma unroll
    for (int d = 0; d < N; ++d) {
      bq[k][d] = ok ? B[(g * L + e) * N + d] : T(0);
      cq[k][d] = ok ? C[(g * L + e) * N + d] : T(0);
    }
  }
  T fa[N], fb[N];  // this thread's exclusive prefix within its warp
#pragma unroll
  for (int d = 0; d < N; ++d) {
    const T ad = Num<T>::a_scale(A[p * N + d]);
    T aa = T(1), bb = T(0);
#pragma unroll
    for (int k = 0; k < kFlatEpt; ++k) {
      const bool ok = tid * kFlatEpt + k < cnt;
      const T av = ok ? Num<T>::exp_scaled(dl[k] * ad) : T(1);
      bb = fma(av, bb, (dl[k] * bq[k][d]) * xv[k]);
      aa = av * aa;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T pa = __shfl_up_sync(kFull, aa, o), pb = __shfl_up_sync(kFull, bb, o);
      if (lane >= o) {
        bb = fma(aa, pb, bb);
        aa = aa * pa;
      }
    }
    if (lane == 31) wa[wid][d] = aa, wb[wid][d] = bb;
    const T ea = __shfl_up_sync(kFull, aa, 1), eb = __shfl_up_sync(kFull, bb, 1);
    fa[d] = lane == 0 ? T(1) : ea;
    fb[d] = lane == 0 ? T(0) : eb;
  }
  __syncthreads();
  // chunk aggregate per state, then publish it (AGGREGATE) or, for the first
  // chunk of a scan, the inclusive state directly
  if (tid < N) {
    T a2 = T(1), b2 = T(0);
    for (int w = 0; w < NW; ++w) {
      b2 = fma(wa[w][tid], b2, wb[w][tid]);
      a2 = wa[w][tid] * a2;
    }
    aggA[tid] = a2, aggB[tid] = b2;
    if (c == 0) {
      vI[slot + tid] = b2;
    } else {
      vA[slot + tid] = a2;
      vB[slot + tid] = b2;
    }
    __threadfence();
  }
  __syncthreads();
  if (tid == 0)
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ws.status + s * nch + c), "r"(c == 0 ? 2 : 1)
                 : "memory");
  // look back (one thread per state)
  if (tid < N) {
    T h = T(0);
    if (c > 0) {
      T accA = T(1), accB = T(0);
      int k = c - 1;
      while (true) {
        int st;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(st) : "l"(ws.status + s * nch + k) : "memory");
        if (st == 2) {
          h = fma(accA, __ldcg(vI + (static_cast<size_t>(s) * nch + k) * N + tid), accB);
          break;
        }
        if (st == 1) {
          const size_t o = (static_cast<size_t>(s) * nch + k) * N + tid;
          accB = fma(accA, __ldcg(vB + o), accB);
          accA = accA * __ldcg(vA + o);
          if (--k < 0) {
            h = accB;
            break;
          }
        }
      }
      vI[slot + tid] = fma(aggA[tid], h, aggB[tid]);
      __threadfence();
    }
    carry[tid] = h;
  }
  __syncthreads();
  if (tid == 0 && c > 0)
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ws.status + s * nch + c), "r"(2) : "memory");
#pragma unroll
  for (int d = 0; d < N; ++d) {
    T h = carry[d];
    for (int w = 0; w < wid; ++w) h = fma(wa[w][d], h, wb[w][d]);
    h = fma(fa[d], h, fb[d]);
    const T ad = Num<T>::a_scale(A[p * N + d]);
#pragma unroll
    for (int k = 0; k < kFlatEpt; ++k) {
      if (tid * kFlatEpt + k < cnt) {
        h = fma(Num<T>::exp_scaled(dl[k] * ad), h, (dl[k] * bq[k][d]) * xv[k]);
        yacc[k] = fma(cq[k][d], h, yacc[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kFlatEpt; ++k) {
    const int idx = tid * kFlatEpt + k;
    if (idx < cnt) y[s * L + base + idx] = fma(dsk, xv[k], yacc[k]);
  }
}

size_t flat_lookback_ws(int64_t S, int64_t L, int N, size_t es) {
  const int64_t nch = (L + kFlatChunk - 1) / kFlatChunk;
  return 256 + (static_cast<size_t>(S * nch) * sizeof(int) + 255) / 256 * 256 +
         3 * static_cast<size_t>(S * nch) * N * es;
}

unsigned blocks_for(int64_t n, int threads) { return static_cast<unsigned>((n + threads - 1) / threads); }

template <typename T>
int run_naive(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C, const void* A,
              const void* Dskip, const void* bias, void* y, void* ws, cudaStream_t st) {
  const int64_t S = d.num_scans;
  const size_t HW = static_cast<size_t>(d.height) * d.width;
  T* maps = static_cast<T*>(ws);
  T* vst = maps + static_cast<size_t>(S) * d.state_dim * HW;
  const int th = 128;
  naive_rows_kernel<T><<<blocks_for(S * d.height * d.state_dim, th), th, 0, st>>>(
      static_cast<const T*>(x), static_cast<const T*>(z), static_cast<const T*>(B), static_cast<const T*>(A),
      static_cast<const T*>(bias), S, d.height, d.width, d.state_dim, d.params_period, d.bc_group, maps);
  naive_cols_kernel<T><<<blocks_for(S * d.width, th), th, 0, st>>>(
      static_cast<const T*>(x), static_cast<const T*>(z), static_cast<const T*>(C), static_cast<const T*>(A),
      static_cast<const T*>(Dskip), static_cast<const T*>(bias), maps, S, d.height, d.width, d.state_dim,
      d.params_period, d.bc_group, vst, static_cast<T*>(y));
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}

template <typename T>
int run_flat(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C, const void* A,
             const void* Dskip, const void* bias, void* y, void* ws, cudaStream_t st) {
  const int64_t S = d.num_scans;
  const int64_t L = static_cast<int64_t>(d.height) * d.width;
  if (d.state_dim <= kFlatMaxN && (d.state_dim & (d.state_dim - 1)) == 0) {
    const int64_t nch = (L + kFlatChunk - 1) / kFlatChunk;
    unsigned char* w = static_cast<unsigned char*>(ws);
    FlatWs fw{reinterpret_cast<int*>(w), reinterpret_cast<int*>(w + 256),
              w + 256 + (static_cast<size_t>(S * nch) * sizeof(int) + 255) / 256 * 256};
    // ticket + chunk status flags start at zero on every call
    if (cudaMemsetAsync(w, 0, 256 + static_cast<size_t>(S * nch) * sizeof(int), st) != cudaSuccess)
      return SCAN2D_ECUDA;
    const unsigned grid = static_cast<unsigned>(S * nch);
    auto go = [&](auto kern) {
      kern<<<grid, kFlatThreads, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(z),
                                          static_cast<const T*>(B), static_cast<const T*>(C),
                                          static_cast<const T*>(A), static_cast<const T*>(Dskip),
                                          static_cast<const T*>(bias), S, L, static_cast<int>(nch),
                                          d.params_period, d.bc_group, static_cast<T*>(y), fw);
    };
    switch (d.state_dim) {
      case 1: go(flat_lookback_kernel<T, 1>); break;
      case 2: go(flat_lookback_kernel<T, 2>); break;
      case 4: go(flat_lookback_kernel<T, 4>); break;
      case 8: go(flat_lookback_kernel<T, 8>); break;
      default: go(flat_lookback_kernel<T, 16>); break;
    }
    return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
  }
  T* hs = static_cast<T*>(ws);
  const int th = 128;
  flat_scan_kernel<T><<<blocks_for(S * d.state_dim, th), th, 0, st>>>(
      static_cast<const T*>(x), static_cast<const T*>(z), static_cast<const T*>(B), static_cast<const T*>(A),
      static_cast<const T*>(bias), S, L, d.state_dim, d.params_period, d.bc_group, hs);
  flat_readout_kernel<T><<<blocks_for(S * L, th), th, 0, st>>>(
      static_cast<const T*>(x), static_cast<const T*>(C), static_cast<const T*>(Dskip), hs, S, L, d.state_dim,
      d.params_period, d.bc_group, static_cast<T*>(y));
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}

int basic_check(const scan2d_desc* d) {
  if (d == nullptr || d->num_scans < 1 || d->height < 1 || d->width < 1 || d->state_dim < 1 ||
      d->state_dim > SCAN2D_MAX_STATE_DIM || d->params_period < 1 || d->num_scans % d->params_period ||
      d->bc_group < 1 || d->num_scans % d->bc_group || (d->dtype != SCAN2D_F32 && d->dtype != SCAN2D_F64))
    return SCAN2D_EINVAL;
  return SCAN2D_OK;
}

}  // namespace
}  // namespace s2d

extern "C" {

size_t scan2d_comparator_workspace_bytes(const scan2d_desc* d, int variant) {
  if (s2d::basic_check(d) != SCAN2D_OK) return 0;
  const size_t es = d->dtype == SCAN2D_F64 ? 8 : 4;
  const size_t S = static_cast<size_t>(d->num_scans), HW = static_cast<size_t>(d->height) * d->width;
  if (variant == SCAN2D_VARIANT_NAIVE) return es * S * d->state_dim * (HW + d->width);
  if (d->state_dim <= s2d::kFlatMaxN && (d->state_dim & (d->state_dim - 1)) == 0)  // look-back kernel
    return s2d::flat_lookback_ws(d->num_scans, static_cast<int64_t>(d->height) * d->width, d->state_dim, es);
  return es * S * HW * d->state_dim;
}

int scan2d_forward_variant(const scan2d_desc* d, int variant, const void* x, const void* z, const void* B,
                           const void* C, const void* A, const void* Dskip, const void* bias, void* y, void* ws,
                           size_t ws_bytes, scan2d_stream_t stream) {
  int rc = s2d::basic_check(d);
  if (rc != SCAN2D_OK) return rc;
  if (!x || !z || !B || !C || !A || !Dskip || !bias || !y) return SCAN2D_EINVAL;
  if (variant != SCAN2D_VARIANT_NAIVE && variant != SCAN2D_VARIANT_FLAT1D) return SCAN2D_EINVAL;
  if (ws == nullptr || ws_bytes < scan2d_comparator_workspace_bytes(d, variant)) return SCAN2D_ENOMEM;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (variant == SCAN2D_VARIANT_NAIVE)
    return d->dtype == SCAN2D_F64 ? s2d::run_naive<double>(*d, x, z, B, C, A, Dskip, bias, y, ws, st)
                                  : s2d::run_naive<float>(*d, x, z, B, C, A, Dskip, bias, y, ws, st);
  return d->dtype == SCAN2D_F64 ? s2d::run_flat<double>(*d, x, z, B, C, A, Dskip, bias, y, ws, st)
                                : s2d::run_flat<float>(*d, x, z, B, C, A, Dskip, bias, y, ws, st);
}

}  // extern "C"
