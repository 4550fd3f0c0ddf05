// scan2d_capi.cu -- C-ABI entry points (include/scan2d_cuda.h): descriptor
// validation, launch planning, workspace / residual carving, kernel launches.
//
// Validation mirrors require_shapes (proj/src/engine.cpp:21-30) and the tile
// check (:163-164); the backward's stale-state check mirrors engine.cpp:248-249.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/scan2d_cuda.h"
#include "scan2d_launch.h"

using s2d::Args;
using s2d::Plan;

namespace {

thread_local int g_last_launches = 0;

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t dtype_size(int dtype) { return dtype == SCAN2D_F64 ? sizeof(double) : sizeof(float); }

int check_desc(const scan2d_desc* d) {
  if (d == nullptr) return SCAN2D_EINVAL;
  if (d->num_scans < 1 || d->height < 1 || d->width < 1) return SCAN2D_EINVAL;
  if (d->state_dim < 1 || d->state_dim > SCAN2D_MAX_STATE_DIM) return SCAN2D_EINVAL;
  if (d->tile < 1) return SCAN2D_EINVAL;
  if (d->params_period < 1 || d->num_scans % d->params_period != 0) return SCAN2D_EINVAL;
  if (d->bc_group < 1 || d->num_scans % d->bc_group != 0) return SCAN2D_EINVAL;
  if (d->dtype != SCAN2D_F32 && d->dtype != SCAN2D_F64) return SCAN2D_EINVAL;
  if (d->reserved != 0) return SCAN2D_EINVAL;
  if (d->state_dim > 32) return SCAN2D_EUNSUPPORTED;  // state groups > 32: not yet
  return SCAN2D_OK;
}

// Launch geometry.  One plan serves both directions: the backward consumes the
// forward's residual, whose layout depends on (ncb, nw, colsw, K).
Plan make_plan(const scan2d_desc& d) {
  Plan p{};
  const int N = d.state_dim, W = d.width, H = d.height;
  const bool dbl = d.dtype == SCAN2D_F64;
  p.lpc = std::min(32, next_pow2(N));
  p.cpw = 32 / p.lpc;
  // columns per lane: wide enough to amortise the per-row shuffle scan, small
  // enough to keep the vertical state and the prefetched row in registers
  if (p.lpc >= 4) {
    p.J = 4;
  } else {
    const int need = static_cast<int>(ceil_div(W, p.cpw));
    p.J = std::min(8, next_pow2(std::max(1, need)));
  }
  if (dbl) p.J = std::min(p.J, 4);
  const int chunks_per_scan = static_cast<int>(ceil_div(W, p.J));
  if (chunks_per_scan <= p.cpw / 2) {
    // narrow grids: pack several scans into one warp (segmented shuffles)
    p.cps = next_pow2(chunks_per_scan);
    p.seg = p.cpw / p.cps;
  } else {
    p.cps = p.cpw;
    p.seg = 1;
  }
  p.colsw = p.cps * p.J;
  p.wreal = static_cast<int>(ceil_div(W, p.colsw));
  if (p.seg > 1) p.wreal = 1;
  if (p.wreal <= 16) {
    p.ncb = 1;
    p.wps = p.wreal;
    p.nw = p.wps * std::max(1, 8 / p.wps);
  } else {
    p.ncb = static_cast<int>(ceil_div(p.wreal, 16));
    p.nw = static_cast<int>(ceil_div(p.wreal, p.ncb));
    p.wps = p.nw * p.ncb;
  }
  p.units = ceil_div(d.num_scans, p.seg) * p.wps;
  p.ctas = ceil_div(p.units, p.nw);
  p.K = std::min(8, H);
  p.nb = static_cast<int>(ceil_div(H, p.K));
  return p;
}

struct WsLayout {
  size_t flags = 0, hcarry = 0, rcarry = 0, part = 0, dbc = 0, total = 0;
};

// forward workspace: [flags][hcarry (when no residual is given)]
// backward workspace: [flags][rcarry][part][per-scan dB, dC (G > 1)]
WsLayout ws_layout(const scan2d_desc& d, const Plan& p, int op) {
  const size_t es = dtype_size(d.dtype);
  const size_t S = static_cast<size_t>(d.num_scans);
  const size_t bnd = S * static_cast<size_t>(p.ncb - 1);
  WsLayout L;
  size_t off = 0;
  L.flags = off;
  off += align_up(sizeof(int) * (1 + bnd));
  if (op == SCAN2D_OP_FWD) {
    L.hcarry = off;
    off += align_up(es * bnd * d.height * d.state_dim);
  } else {
    L.rcarry = off;
    off += align_up(es * bnd * d.height * d.state_dim);
    L.part = off;
    off += align_up(es * S * p.wps * (d.state_dim + 2));
    if (d.bc_group > 1) {
      L.dbc = off;
      off += align_up(2 * es * S * d.height * d.width * d.state_dim);
    }
  }
  L.total = off;
  return L;
}

struct ResLayout {
  size_t ckpt = 0, hcarry = 0, total = 0;
};

ResLayout res_layout(const scan2d_desc& d, const Plan& p) {
  const size_t es = dtype_size(d.dtype);
  const size_t S = static_cast<size_t>(d.num_scans);
  ResLayout R;
  R.ckpt = 0;
  size_t off = align_up(es * S * (p.nb - 1) * d.width * d.state_dim);
  R.hcarry = off;
  off += align_up(es * S * (p.ncb - 1) * d.height * d.state_dim);
  R.total = std::max<size_t>(off, kAlign);
  return R;
}

int device_check() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SCAN2D_ECUDA;
  static int cached[64] = {0};  // 0 unknown, 1 ok, 2 unsupported
  if (dev < 0 || dev >= 64) return SCAN2D_ECUDA;
  if (cached[dev] == 0) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return SCAN2D_ECUDA;
    cached[dev] = (major == 10 && minor == 0) ? 1 : 2;
  }
  return cached[dev] == 1 ? SCAN2D_OK : SCAN2D_EUNSUPPORTED;
}

template <typename T>
int forward_impl(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C,
                 const void* A, const void* Dskip, const void* bias, void* y, void* ph, void* pv,
                 void* residual, void* ws, size_t ws_bytes, cudaStream_t stream) {
  g_last_launches = 0;
  if (!x || !z || !B || !C || !A || !Dskip || !bias || !y) return SCAN2D_EINVAL;
  if ((ph == nullptr) != (pv == nullptr)) return SCAN2D_EINVAL;
  int rc = device_check();
  if (rc != SCAN2D_OK) return rc;
  const Plan p = make_plan(d);
  const WsLayout L = ws_layout(d, p, SCAN2D_OP_FWD);
  if (ws_bytes < L.total || (L.total > 0 && ws == nullptr)) return SCAN2D_ENOMEM;
  unsigned char* w = static_cast<unsigned char*>(ws);
  Args<T> a{};
  a.x = static_cast<const T*>(x);
  a.z = static_cast<const T*>(z);
  a.B = static_cast<const T*>(B);
  a.C = static_cast<const T*>(C);
  a.A = static_cast<const T*>(A);
  a.Dskip = static_cast<const T*>(Dskip);
  a.bias = static_cast<const T*>(bias);
  a.y = static_cast<T*>(y);
  a.ph = static_cast<T*>(ph);
  a.pv = static_cast<T*>(pv);
  a.flags = reinterpret_cast<int*>(w + L.flags);
  if (residual != nullptr) {
    const ResLayout R = res_layout(d, p);
    unsigned char* r = static_cast<unsigned char*>(residual);
    a.ckpt = reinterpret_cast<T*>(r + R.ckpt);
    a.hcarry = reinterpret_cast<T*>(r + R.hcarry);
  } else {
    a.ckpt = nullptr;
    a.hcarry = reinterpret_cast<T*>(w + L.hcarry);
  }
  a.S = d.num_scans;
  a.H = d.height;
  a.W = d.width;
  a.N = d.state_dim;
  a.T_tile = d.tile;
  a.P = d.params_period;
  a.G = d.bc_group;
  a.plan = p;
  if (p.ncb > 1) {
    const size_t fb = sizeof(int) * (1 + static_cast<size_t>(d.num_scans) * (p.ncb - 1));
    if (cudaMemsetAsync(a.flags, 0, fb, stream) != cudaSuccess) return SCAN2D_ECUDA;
  }
  if (ph != nullptr) {
    const size_t kh = ceil_div(d.height, d.tile), kw = ceil_div(d.width, d.tile);
    const size_t cb = sizeof(T) * static_cast<size_t>(d.num_scans) * kh * kw * d.tile * d.state_dim;
    if (cudaMemsetAsync(ph, 0, cb, stream) != cudaSuccess) return SCAN2D_ECUDA;
    if (cudaMemsetAsync(pv, 0, cb, stream) != cudaSuccess) return SCAN2D_ECUDA;
  }
  if (s2d::launch_fwd<T>(a, s2d::fwd_smem_bytes<T>(p), stream) != cudaSuccess) return SCAN2D_ECUDA;
  g_last_launches = 1;
  return SCAN2D_OK;
}

template <typename T>
int backward_impl(const scan2d_desc& d, const void* x, const void* z, const void* B,
                  const void* C, const void* A, const void* Dskip, const void* bias,
                  const void* residual, const void* dy, void* dx, void* dz, void* dA, void* dB,
                  void* dC, void* dDskip, void* dbias, void* ws, size_t ws_bytes,
                  cudaStream_t stream) {
  g_last_launches = 0;
  if (residual == nullptr) return SCAN2D_ESTALE;
  if (!x || !z || !B || !C || !A || !Dskip || !bias || !dy) return SCAN2D_EINVAL;
  if (!dx || !dz || !dA || !dB || !dC || !dDskip || !dbias) return SCAN2D_EINVAL;
  int rc = device_check();
  if (rc != SCAN2D_OK) return rc;
  const Plan p = make_plan(d);
  const WsLayout L = ws_layout(d, p, SCAN2D_OP_BWD);
  if (ws_bytes < L.total || ws == nullptr) return SCAN2D_ENOMEM;
  unsigned char* w = static_cast<unsigned char*>(ws);
  const ResLayout R = res_layout(d, p);
  const unsigned char* r = static_cast<const unsigned char*>(residual);
  Args<T> a{};
  a.x = static_cast<const T*>(x);
  a.z = static_cast<const T*>(z);
  a.B = static_cast<const T*>(B);
  a.C = static_cast<const T*>(C);
  a.A = static_cast<const T*>(A);
  a.Dskip = static_cast<const T*>(Dskip);
  a.bias = static_cast<const T*>(bias);
  a.dy = static_cast<const T*>(dy);
  a.ckpt = const_cast<T*>(reinterpret_cast<const T*>(r + R.ckpt));
  a.hcarry = const_cast<T*>(reinterpret_cast<const T*>(r + R.hcarry));
  a.dx = static_cast<T*>(dx);
  a.dz = static_cast<T*>(dz);
  T* dB_ps = static_cast<T*>(dB);
  T* dC_ps = static_cast<T*>(dC);
  const size_t hwn = static_cast<size_t>(d.height) * d.width * d.state_dim;
  if (d.bc_group > 1) {
    dB_ps = reinterpret_cast<T*>(w + L.dbc);
    dC_ps = dB_ps + static_cast<size_t>(d.num_scans) * hwn;
  }
  a.dB = dB_ps;
  a.dC = dC_ps;
  a.part = reinterpret_cast<T*>(w + L.part);
  a.rcarry = reinterpret_cast<T*>(w + L.rcarry);
  a.flags = reinterpret_cast<int*>(w + L.flags);
  a.S = d.num_scans;
  a.H = d.height;
  a.W = d.width;
  a.N = d.state_dim;
  a.T_tile = d.tile;
  a.P = d.params_period;
  a.G = d.bc_group;
  a.plan = p;
  if (p.ncb > 1) {
    const size_t fb = sizeof(int) * (1 + static_cast<size_t>(d.num_scans) * (p.ncb - 1));
    if (cudaMemsetAsync(a.flags, 0, fb, stream) != cudaSuccess) return SCAN2D_ECUDA;
  }
  int launches = 0;
  if (s2d::launch_bwd<T>(a, s2d::bwd_smem_bytes<T>(p), stream) != cudaSuccess) return SCAN2D_ECUDA;
  ++launches;
  if (s2d::launch_reduce_params<T>(a.part, d.num_scans, p.wps, p.wreal, d.params_period,
                                   d.state_dim, static_cast<T*>(dA), static_cast<T*>(dbias),
                                   static_cast<T*>(dDskip), stream) != cudaSuccess)
    return SCAN2D_ECUDA;
  ++launches;
  if (d.bc_group > 1) {
    const int64_t groups = d.num_scans / d.bc_group;
    if (s2d::launch_reduce_group<T>(dB_ps, groups, d.bc_group, hwn, static_cast<T*>(dB), stream) !=
            cudaSuccess ||
        s2d::launch_reduce_group<T>(dC_ps, groups, d.bc_group, hwn, static_cast<T*>(dC), stream) !=
            cudaSuccess)
      return SCAN2D_ECUDA;
    launches += 2;
  }
  g_last_launches = launches;
  return SCAN2D_OK;
}

}  // namespace

extern "C" {

int scan2d_check_desc(const scan2d_desc* desc) { return check_desc(desc); }

size_t scan2d_workspace_bytes(const scan2d_desc* desc, int op) {
  if (check_desc(desc) != SCAN2D_OK) return 0;
  const Plan p = make_plan(*desc);
  return ws_layout(*desc, p, op).total;
}

size_t scan2d_residual_bytes(const scan2d_desc* desc) {
  if (check_desc(desc) != SCAN2D_OK) return 0;
  const Plan p = make_plan(*desc);
  return res_layout(*desc, p).total;
}

int scan2d_forward(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                   const void* C, const void* A, const void* Dskip, const void* bias, void* y,
                   void* ph, void* pv, void* residual, void* workspace, size_t workspace_bytes,
                   scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->dtype == SCAN2D_F64)
    return forward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                                workspace_bytes, st);
  return forward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                             workspace_bytes, st);
}

int scan2d_backward(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                    const void* C, const void* A, const void* Dskip, const void* bias,
                    const void* residual, const void* dy, void* dx, void* dz, void* dA,
                    void* dB, void* dC, void* dDskip, void* dbias, void* workspace,
                    size_t workspace_bytes, scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->dtype == SCAN2D_F64)
    return backward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB,
                                 dC, dDskip, dbias, workspace, workspace_bytes, st);
  return backward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC,
                              dDskip, dbias, workspace, workspace_bytes, st);
}

int scan2d_fwd_f32(const scan2d_desc* desc, const float* x, const float* z, const float* B,
                   const float* C, const float* A, const float* Dskip, const float* bias,
                   float* y, float* ph, float* pv, void* residual, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F32;
  return scan2d_forward(&d, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                        workspace_bytes, stream);
}

int scan2d_fwd_f64(const scan2d_desc* desc, const double* x, const double* z, const double* B,
                   const double* C, const double* A, const double* Dskip, const double* bias,
                   double* y, double* ph, double* pv, void* residual, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F64;
  return scan2d_forward(&d, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                        workspace_bytes, stream);
}

int scan2d_bwd_f32(const scan2d_desc* desc, const float* x, const float* z, const float* B,
                   const float* C, const float* A, const float* Dskip, const float* bias,
                   const void* residual, const float* dy, float* dx, float* dz, float* dA,
                   float* dB, float* dC, float* dDskip, float* dbias, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F32;
  return scan2d_backward(&d, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                         dbias, workspace, workspace_bytes, stream);
}

int scan2d_bwd_f64(const scan2d_desc* desc, const double* x, const double* z, const double* B,
                   const double* C, const double* A, const double* Dskip, const double* bias,
                   const void* residual, const double* dy, double* dx, double* dz, double* dA,
                   double* dB, double* dC, double* dDskip, double* dbias, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F64;
  return scan2d_backward(&d, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                         dbias, workspace, workspace_bytes, stream);
}

int scan2d_plan_info(const scan2d_desc* desc, int op, int64_t* out8) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  if (out8 == nullptr) return SCAN2D_EINVAL;
  (void)op;
  const Plan p = make_plan(*desc);
  out8[0] = p.lpc;
  out8[1] = p.J;
  out8[2] = p.seg;
  out8[3] = p.wps;
  out8[4] = p.nw;
  out8[5] = p.ncb;
  out8[6] = p.ctas;
  out8[7] = p.K;
  return SCAN2D_OK;
}

int scan2d_last_launch_count(void) { return g_last_launches; }

const char* scan2d_status_string(int status) {
  switch (status) {
    case SCAN2D_OK: return "ok";
    case SCAN2D_EINVAL: return "invalid argument (shape / descriptor)";
    case SCAN2D_ESTALE: return "stale or missing saved forward state";
    case SCAN2D_ECUDA: return "CUDA runtime / launch error";
    case SCAN2D_ENOMEM: return "workspace too small";
    case SCAN2D_EUNSUPPORTED: return "unsupported device or configuration";
    default: return "unknown status";
  }
}

int scan2d_version(void) { return 1; }

}  // extern "C"
