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
// GPU): one CTA per scan walks the row-major flattened grid in chunks of
// kThreads x kEpt elements.  Per chunk and state d: the affine pairs
// (Abar, Bbar x) of a thread's kEpt elements are folded in registers, the
// kThreads folds are combined by a warp shuffle scan and a scan over the warp
// totals in shared memory, the running carry of the previous chunks enters as
// the head of the sequence (b <- fma(a, carry, b), block_scan.cpp:51), and
// y accumulates C_d h over d ascending in registers (engine.cpp:506-518) --
// the N state sequences never touch HBM.  B and C of the chunk are staged in
// shared memory with coalesced loads.
constexpr int kFlatThreads = 256;
constexpr int kFlatEpt = 2;
constexpr int kFlatMaxN = 16;  // larger N: the sequential flat kernels above

template <typename T, int N>
__global__ void __launch_bounds__(kFlatThreads) flat_block_kernel(
    const T* __restrict__ x, const T* __restrict__ z, const T* __restrict__ B, const T* __restrict__ C,
    const T* __restrict__ A, const T* __restrict__ Dskip, const T* __restrict__ bias, int64_t L, int P, int G,
    T* __restrict__ y) {
  constexpr int CH = kFlatThreads * kFlatEpt;
  constexpr int NW = kFlatThreads / 32;
  extern __shared__ __align__(16) unsigned char flat_smem[];
  T* sB = reinterpret_cast<T*>(flat_smem);          // [CH][N]
  T* sC = sB + CH * N;                              // [CH][N]
  T* wa = sC + CH * N;                              // [NW][N] warp totals (a)
  T* wb = wa + NW * kFlatMaxN;                      // [NW][N] warp totals (b)
  T* carry = wb + NW * kFlatMaxN;                   // [N] running h
  const int64_t s = blockIdx.x;
  const int64_t p = s % P, g = s / G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const T bs = bias[p], dsk = Dskip[p];
  for (int d = tid; d < N; d += kFlatThreads) carry[d] = T(0);
  const T* xs = x + s * L;
  const T* zs = z + s * L;
  const T* Bs = B + g * L * N;
  const T* Cs = C + g * L * N;
  for (int64_t base = 0; base < L; base += CH) {
    const int cnt = static_cast<int>(L - base < CH ? L - base : CH);
    __syncthreads();  // previous chunk done with sB / sC / carry reads
    for (int e = tid; e < cnt * N; e += kFlatThreads) {
      sB[e] = Bs[base * N + e];
      sC[e] = Cs[base * N + e];
    }
    T dl[kFlatEpt], xv[kFlatEpt], yacc[kFlatEpt];
#pragma unroll
    for (int k = 0; k < kFlatEpt; ++k) {
      const int idx = tid * kFlatEpt + k;
      const bool ok = idx < cnt;
      xv[k] = ok ? xs[base + idx] : T(0);
      dl[k] = ok ? Num<T>::softplus(zs[base + idx] + bs) : T(0);
      yacc[k] = T(0);
    }
    __syncthreads();
    T fa[N], fb[N];  // this thread's exclusive prefix within its warp
#pragma unroll
    for (int d = 0; d < N; ++d) {
      const T ad = Num<T>::a_scale(A[p * N + d]);
      T aa = T(1), bb = T(0);
#pragma unroll
      for (int k = 0; k < kFlatEpt; ++k) {
        const int idx = tid * kFlatEpt + k;
        const bool ok = idx < cnt;
        const T av = ok ? Num<T>::exp_scaled(dl[k] * ad) : T(1);
        const T bx = ok ? (dl[k] * sB[idx * N + d]) * xv[k] : T(0);
        bb = fma(av, bb, bx);
        aa = av * aa;
      }
      // inclusive warp scan of the folds (compose: earlier first)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T pa = __shfl_up_sync(kFull, aa, o), pb = __shfl_up_sync(kFull, bb, o);
        if (lane >= o) {
          bb = fma(aa, pb, bb);
          aa = aa * pa;
        }
      }
      if (lane == 31) {
        wa[wid * kFlatMaxN + d] = aa;
        wb[wid * kFlatMaxN + d] = bb;
      }
      // exclusive within the warp
      const T ea = __shfl_up_sync(kFull, aa, 1), eb = __shfl_up_sync(kFull, bb, 1);
      fa[d] = lane == 0 ? T(1) : ea;
      fb[d] = lane == 0 ? T(0) : eb;
    }
    __syncthreads();
#pragma unroll
    for (int d = 0; d < N; ++d) {
      // prefix = carry, then the totals of the warps before this one, then the lane prefix
      T h = carry[d];
      for (int w = 0; w < wid; ++w) h = fma(wa[w * kFlatMaxN + d], h, wb[w * kFlatMaxN + d]);
      h = fma(fa[d], h, fb[d]);
      const T ad = Num<T>::a_scale(A[p * N + d]);
#pragma unroll
      for (int k = 0; k < kFlatEpt; ++k) {
        const int idx = tid * kFlatEpt + k;
        if (idx < cnt) {
          const T av = Num<T>::exp_scaled(dl[k] * ad);
          h = fma(av, h, (dl[k] * sB[idx * N + d]) * xv[k]);
          yacc[k] = fma(sC[idx * N + d], h, yacc[k]);
        }
      }
      if (tid * kFlatEpt + kFlatEpt - 1 >= cnt - 1 && tid * kFlatEpt <= cnt - 1) fb[d] = h;  // chunk's last h
    }
#pragma unroll
    for (int k = 0; k < kFlatEpt; ++k) {
      const int idx = tid * kFlatEpt + k;
      if (idx < cnt) y[s * L + base + idx] = fma(dsk, xv[k], yacc[k]);
    }
    __syncthreads();  // every thread has read carry[]
    if (tid * kFlatEpt + kFlatEpt - 1 >= cnt - 1 && tid * kFlatEpt <= cnt - 1) {
#pragma unroll
      for (int d = 0; d < N; ++d) carry[d] = fb[d];
    }
  }
}

size_t flat_block_smem(int N, size_t es) {
  return es * (2 * static_cast<size_t>(kFlatThreads) * kFlatEpt * N + 2 * (kFlatThreads / 32) * kFlatMaxN +
               kFlatMaxN);
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
    const size_t smem = flat_block_smem(d.state_dim, sizeof(T));
    const unsigned grid = static_cast<unsigned>(S);
    cudaError_t e = cudaSuccess;
    auto go = [&](auto kern) {
      if (smem > 48 * 1024)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e == cudaSuccess)
        kern<<<grid, kFlatThreads, smem, st>>>(static_cast<const T*>(x), static_cast<const T*>(z),
                                               static_cast<const T*>(B), static_cast<const T*>(C),
                                               static_cast<const T*>(A), static_cast<const T*>(Dskip),
                                               static_cast<const T*>(bias), L, d.params_period, d.bc_group,
                                               static_cast<T*>(y));
    };
    switch (d.state_dim) {
      case 1: go(flat_block_kernel<T, 1>); break;
      case 2: go(flat_block_kernel<T, 2>); break;
      case 4: go(flat_block_kernel<T, 4>); break;
      case 8: go(flat_block_kernel<T, 8>); break;
      default: go(flat_block_kernel<T, 16>); break;
    }
    if (e != cudaSuccess) return SCAN2D_ECUDA;
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
  if (d->state_dim <= s2d::kFlatMaxN && (d->state_dim & (d->state_dim - 1)) == 0)
    return 16;  // block-scan kernel: no HBM state sequences
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
