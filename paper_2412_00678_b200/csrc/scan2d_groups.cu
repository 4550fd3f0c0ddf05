// scan2d_groups.cu -- state dimensions N > 128 (the reference allows up to
// 2048, engine.cpp:19 kMaxStateDim) as passes over state groups of <= 128.
//
// The recurrences of different states are independent (only delta, computed
// from z, is shared): h_d depends on state d alone, and every cross-state
// quantity is a sum over d -- y = D x + sum_d C h, and in the backward
// ddelta, the sum_d Gh B feeding dx, hence dz and dbias.  So the scan runs once
// per group g (states [128 g, 128 g + N_g)) on gathered B_g, C_g, A_g with the
// skip term D only in group 0, and the per-group results are added: y = sum y_g,
// dx = sum dx_g, dz = sum dz_g, dbias = sum dbias_g, dD = dD_0; dA, dB, dC (and
// the optional CarryState ph / pv) are scattered back per group.  Each group
// keeps its own residual (the caller's residual buffer holds all of them).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/scan2d_cuda.h"

namespace {

constexpr int kGroup = 128;
constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }
size_t es_of(int dtype) { return dtype == SCAN2D_F64 ? 8 : 4; }

template <typename T>
__global__ void strided_copy_kernel(T* __restrict__ dst, int64_t dst_pitch, const T* __restrict__ src,
                                    int64_t src_pitch, int64_t rows, int cols) {
  const int64_t n = rows * cols;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / cols;
    const int c = static_cast<int>(t % cols);
    dst[r * dst_pitch + c] = src[r * src_pitch + c];
  }
}

template <typename T>
__global__ void add_kernel(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[t] += src[t];
}

int blocks_for(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8)); }

// rows x cols block of a row-major matrix with `pitch` columns, starting at column c0
int copy_cols(int dtype, void* dst, int64_t dpitch, int64_t dc0, const void* src, int64_t spitch, int64_t sc0,
              int64_t rows, int cols, cudaStream_t st) {
  if (rows * cols == 0) return SCAN2D_OK;
  if (dtype == SCAN2D_F64)
    strided_copy_kernel<double><<<blocks_for(rows * cols), 256, 0, st>>>(
        static_cast<double*>(dst) + dc0, dpitch, static_cast<const double*>(src) + sc0, spitch, rows, cols);
  else
    strided_copy_kernel<float><<<blocks_for(rows * cols), 256, 0, st>>>(
        static_cast<float*>(dst) + dc0, dpitch, static_cast<const float*>(src) + sc0, spitch, rows, cols);
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}

int add_into(int dtype, void* dst, const void* src, int64_t n, cudaStream_t st) {
  if (n == 0) return SCAN2D_OK;
  if (dtype == SCAN2D_F64)
    add_kernel<double><<<blocks_for(n), 256, 0, st>>>(static_cast<double*>(dst), static_cast<const double*>(src), n);
  else
    add_kernel<float><<<blocks_for(n), 256, 0, st>>>(static_cast<float*>(dst), static_cast<const float*>(src), n);
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}

int ngroups(const scan2d_desc& d) { return (d.state_dim + kGroup - 1) / kGroup; }

scan2d_desc group_desc(const scan2d_desc& d, int g) {
  scan2d_desc gd = d;
  gd.state_dim = std::min(kGroup, d.state_dim - g * kGroup);
  return gd;
}

struct GLayout {
  size_t b = 0, c = 0, a = 0, t0 = 0, t1 = 0, dA = 0, dB = 0, dC = 0, dD = 0, dbias = 0, zero = 0, ph = 0,
         pv = 0, inner = 0, total = 0;
  size_t inner_bytes = 0;
};

GLayout glayout(const scan2d_desc& d, int op) {
  const size_t es = es_of(d.dtype);
  const size_t S = static_cast<size_t>(d.num_scans), HW = static_cast<size_t>(d.height) * d.width;
  const size_t SB = S / d.bc_group, P = static_cast<size_t>(d.params_period);
  const size_t cells_b = SB * HW;
  GLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes);
    return o;
  };
  L.b = take(es * cells_b * kGroup);
  L.c = take(es * cells_b * kGroup);
  L.a = take(es * P * kGroup);
  L.zero = take(es * P);
  L.t0 = take(es * S * HW);  // y_g, or dx_g
  if (op == SCAN2D_OP_BWD) {
    L.t1 = take(es * S * HW);  // dz_g
    L.dA = take(es * P * kGroup);
    L.dB = take(es * cells_b * kGroup);
    L.dC = take(es * cells_b * kGroup);
    L.dD = take(es * P);
    L.dbias = take(es * P);
  } else {
    const size_t kh = (d.height + d.tile - 1) / d.tile, kw = (d.width + d.tile - 1) / d.tile;
    const size_t carries = S * kh * kw * d.tile * kGroup;
    L.ph = take(es * carries);
    L.pv = take(es * carries);
  }
  size_t inner = 0;
  for (int g = 0; g < ngroups(d); ++g) {
    const scan2d_desc gd = group_desc(d, g);
    inner = std::max(inner, scan2d_workspace_bytes(&gd, op));
  }
  L.inner = take(inner);
  L.inner_bytes = inner;
  L.total = off;
  return L;
}

}  // namespace

// ---- entry points used by scan2d_capi.cu for N > 128

size_t scan2d_groups_workspace_bytes(const scan2d_desc& d, int op) { return glayout(d, op).total; }

size_t scan2d_groups_residual_bytes(const scan2d_desc& d) {
  size_t tot = 0;
  for (int g = 0; g < ngroups(d); ++g) {
    const scan2d_desc gd = group_desc(d, g);
    tot += align_up(scan2d_residual_bytes(&gd));
  }
  return tot;
}

static size_t residual_offset(const scan2d_desc& d, int g) {
  size_t off = 0;
  for (int k = 0; k < g; ++k) {
    const scan2d_desc gd = group_desc(d, k);
    off += align_up(scan2d_residual_bytes(&gd));
  }
  return off;
}

int scan2d_groups_forward(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C,
                          const void* A, const void* Dskip, const void* bias, void* y, void* ph, void* pv,
                          void* residual, void* ws, size_t ws_bytes, cudaStream_t st) {
  const GLayout L = glayout(d, SCAN2D_OP_FWD);
  if (ws == nullptr || ws_bytes < L.total) return SCAN2D_ENOMEM;
  unsigned char* w = static_cast<unsigned char*>(ws);
  const size_t es = es_of(d.dtype);
  const int64_t S = d.num_scans, HW = static_cast<int64_t>(d.height) * d.width;
  const int64_t cells_b = S / d.bc_group * HW, P = d.params_period, N = d.state_dim;
  const int64_t kh = (d.height + d.tile - 1) / d.tile, kw = (d.width + d.tile - 1) / d.tile;
  const int64_t crow = S * kh * kw * d.tile;  // CarryState rows of N states
  if (cudaMemsetAsync(w + L.zero, 0, es * P, st) != cudaSuccess) return SCAN2D_ECUDA;
  int rc;
  for (int g = 0; g < ngroups(d); ++g) {
    const scan2d_desc gd = group_desc(d, g);
    const int ng = gd.state_dim;
    if ((rc = copy_cols(d.dtype, w + L.b, ng, 0, B, N, g * kGroup, cells_b, ng, st)) != SCAN2D_OK) return rc;
    if ((rc = copy_cols(d.dtype, w + L.c, ng, 0, C, N, g * kGroup, cells_b, ng, st)) != SCAN2D_OK) return rc;
    if ((rc = copy_cols(d.dtype, w + L.a, ng, 0, A, N, g * kGroup, P, ng, st)) != SCAN2D_OK) return rc;
    void* yg = g == 0 ? y : static_cast<void*>(w + L.t0);
    void* res = residual == nullptr ? nullptr : static_cast<unsigned char*>(residual) + residual_offset(d, g);
    rc = scan2d_forward(&gd, x, z, w + L.b, w + L.c, w + L.a, g == 0 ? Dskip : w + L.zero, bias, yg,
                        ph ? w + L.ph : nullptr, pv ? w + L.pv : nullptr, res, w + L.inner, L.inner_bytes,
                        reinterpret_cast<scan2d_stream_t>(st));
    if (rc != SCAN2D_OK) return rc;
    if (g > 0 && (rc = add_into(d.dtype, y, yg, S * HW, st)) != SCAN2D_OK) return rc;
    if (ph != nullptr) {
      if ((rc = copy_cols(d.dtype, ph, N, g * kGroup, w + L.ph, ng, 0, crow, ng, st)) != SCAN2D_OK) return rc;
      if ((rc = copy_cols(d.dtype, pv, N, g * kGroup, w + L.pv, ng, 0, crow, ng, st)) != SCAN2D_OK) return rc;
    }
  }
  return SCAN2D_OK;
}

int scan2d_groups_backward(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C,
                           const void* A, const void* Dskip, const void* bias, const void* residual,
                           const void* dy, void* dx, void* dz, void* dA, void* dB, void* dC, void* dDskip,
                           void* dbias, void* ws, size_t ws_bytes, cudaStream_t st) {
  const GLayout L = glayout(d, SCAN2D_OP_BWD);
  if (ws == nullptr || ws_bytes < L.total) return SCAN2D_ENOMEM;
  unsigned char* w = static_cast<unsigned char*>(ws);
  const size_t es = es_of(d.dtype);
  const int64_t S = d.num_scans, HW = static_cast<int64_t>(d.height) * d.width;
  const int64_t cells_b = S / d.bc_group * HW, P = d.params_period, N = d.state_dim;
  if (cudaMemsetAsync(w + L.zero, 0, es * P, st) != cudaSuccess) return SCAN2D_ECUDA;
  int rc;
  for (int g = 0; g < ngroups(d); ++g) {
    const scan2d_desc gd = group_desc(d, g);
    const int ng = gd.state_dim;
    if ((rc = copy_cols(d.dtype, w + L.b, ng, 0, B, N, g * kGroup, cells_b, ng, st)) != SCAN2D_OK) return rc;
    if ((rc = copy_cols(d.dtype, w + L.c, ng, 0, C, N, g * kGroup, cells_b, ng, st)) != SCAN2D_OK) return rc;
    if ((rc = copy_cols(d.dtype, w + L.a, ng, 0, A, N, g * kGroup, P, ng, st)) != SCAN2D_OK) return rc;
    const void* res = static_cast<const unsigned char*>(residual) + residual_offset(d, g);
    const bool first = g == 0;
    rc = scan2d_backward(&gd, x, z, w + L.b, w + L.c, w + L.a, first ? Dskip : w + L.zero, bias, res, dy,
                         first ? dx : w + L.t0, first ? dz : w + L.t1, w + L.dA, w + L.dB, w + L.dC,
                         first ? dDskip : w + L.dD, first ? dbias : w + L.dbias, w + L.inner, L.inner_bytes,
                         reinterpret_cast<scan2d_stream_t>(st));
    if (rc != SCAN2D_OK) return rc;
    if (!first) {
      if ((rc = add_into(d.dtype, dx, w + L.t0, S * HW, st)) != SCAN2D_OK) return rc;
      if ((rc = add_into(d.dtype, dz, w + L.t1, S * HW, st)) != SCAN2D_OK) return rc;
      if ((rc = add_into(d.dtype, dbias, w + L.dbias, P, st)) != SCAN2D_OK) return rc;
    }
    if ((rc = copy_cols(d.dtype, dA, N, g * kGroup, w + L.dA, ng, 0, P, ng, st)) != SCAN2D_OK) return rc;
    if ((rc = copy_cols(d.dtype, dB, N, g * kGroup, w + L.dB, ng, 0, cells_b, ng, st)) != SCAN2D_OK) return rc;
    if ((rc = copy_cols(d.dtype, dC, N, g * kGroup, w + L.dC, ng, 0, cells_b, ng, st)) != SCAN2D_OK) return rc;
  }
  return SCAN2D_OK;
}
