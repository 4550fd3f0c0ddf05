// scan2d_host.cu -- host-operand entry point (include/scan2d_cuda.h,
// scan2d_train_host): the reference API takes and returns host data
// (engine.hpp:88-102, Grid<T> holds std::vector), so the drop-in path is
// host -> device -> scan -> host.  This runtime pipelines it: the S scans go in
// `chunks` groups through two device buffer sets; chunk k's host->device
// copies, chunk k-1's forward + backward kernels and chunk k-2's device->host
// copies run concurrently on three streams ordered by events, so the PCIe
// transfers in both directions overlap each other and the kernels.
//
// Three device buffer sets rotate, so chunk k+2's host->device copies never
// wait for chunk k's device->host copies to drain.  Device buffers, streams and
// events are cached per host thread and per (descriptor, chunk count).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/scan2d_cuda.h"

namespace {

size_t es_of(int dtype) { return dtype == SCAN2D_F64 ? 8 : 4; }

struct Slot {
  // inputs: x z B C A D bias dy | outputs: y dx dz dA dB dC dD dbias
  void* in[8] = {};
  void* out[8] = {};
  void* residual = nullptr;
  void* wsf = nullptr;
  void* wsb = nullptr;
  size_t wsf_bytes = 0, wsb_bytes = 0;
};

struct Ctx {
  scan2d_desc desc{};
  int chunks = 0, chunk_scans = 0;
  bool with_bwd = false;
  int device = -1;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  static constexpr int kSlots = 3;
  cudaEvent_t ev_in[kSlots] = {}, ev_out[kSlots] = {}, ev_free[kSlots] = {}, ev_start = nullptr;
  Slot slot[kSlots];
  ~Ctx() {
    for (Slot& s : slot) {
      for (void* p : s.in) cudaFree(p);
      for (void* p : s.out) cudaFree(p);
      cudaFree(s.residual);
      cudaFree(s.wsf);
      cudaFree(s.wsb);
    }
    for (int i = 0; i < kSlots; ++i) {
      cudaEventDestroy(ev_in[i]);
      cudaEventDestroy(ev_out[i]);
      cudaEventDestroy(ev_free[i]);
    }
    cudaEventDestroy(ev_start);
    cudaStreamDestroy(h2d);
    cudaStreamDestroy(comp);
    cudaStreamDestroy(d2h);
  }
};

thread_local std::unique_ptr<Ctx> g_ctx;

bool same(const scan2d_desc& a, const scan2d_desc& b) { return std::memcmp(&a, &b, sizeof(a)) == 0; }

// per-scan element counts of the eight inputs / outputs (P == S, G == 1 per chunk)
void counts(const scan2d_desc& d, int64_t s, size_t (&in)[8], size_t (&out)[8]) {
  const size_t hw = static_cast<size_t>(d.height) * d.width, n = d.state_dim;
  const size_t S = static_cast<size_t>(s);
  const size_t c[8] = {S * hw, S * hw, S * hw * n, S * hw * n, S * n, S, S, S * hw};
  const size_t o[8] = {S * hw, S * hw, S * hw, S * n, S * hw * n, S * hw * n, S, S};
  for (int i = 0; i < 8; ++i) in[i] = c[i], out[i] = o[i];
}

int setup(const scan2d_desc& d, int chunks, bool with_bwd) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SCAN2D_ECUDA;
  if (g_ctx && same(g_ctx->desc, d) && g_ctx->chunks == chunks && g_ctx->with_bwd == with_bwd &&
      g_ctx->device == dev)
    return SCAN2D_OK;
  g_ctx.reset();
  auto c = std::make_unique<Ctx>();
  c->desc = d;
  c->chunks = chunks;
  c->with_bwd = with_bwd;
  c->device = dev;
  c->chunk_scans = static_cast<int>((d.num_scans + chunks - 1) / chunks);
  if (cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->comp, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking) != cudaSuccess)
    return SCAN2D_ECUDA;
  for (int i = 0; i < Ctx::kSlots; ++i)
    if (cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming) != cudaSuccess)
      return SCAN2D_ECUDA;
  if (cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming) != cudaSuccess) return SCAN2D_ECUDA;
  scan2d_desc cd = d;
  cd.num_scans = c->chunk_scans;
  cd.params_period = c->chunk_scans;
  cd.bc_group = 1;
  const size_t es = es_of(d.dtype);
  size_t in[8], out[8];
  counts(d, c->chunk_scans, in, out);
  for (Slot& s : c->slot) {
    for (int i = 0; i < 8; ++i) {
      if (cudaMalloc(&s.in[i], in[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
      if ((with_bwd || i == 0) && cudaMalloc(&s.out[i], out[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
    }
    s.wsf_bytes = scan2d_workspace_bytes(&cd, SCAN2D_OP_FWD);
    if (cudaMalloc(&s.wsf, s.wsf_bytes) != cudaSuccess) return SCAN2D_ENOMEM;
    if (with_bwd) {
      s.wsb_bytes = scan2d_workspace_bytes(&cd, SCAN2D_OP_BWD);
      if (cudaMalloc(&s.wsb, s.wsb_bytes) != cudaSuccess) return SCAN2D_ENOMEM;
      if (cudaMalloc(&s.residual, scan2d_residual_bytes(&cd)) != cudaSuccess) return SCAN2D_ENOMEM;
    }
  }
  g_ctx = std::move(c);
  return SCAN2D_OK;
}

}  // namespace

extern "C" int scan2d_train_host(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                                 const void* C, const void* A, const void* Dskip, const void* bias,
                                 const void* dy, void* y, void* dx, void* dz, void* dA, void* dB, void* dC,
                                 void* dDskip, void* dbias, int chunks, scan2d_stream_t stream) {
  int rc = scan2d_check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  const scan2d_desc& d = *desc;
  if (!x || !z || !B || !C || !A || !Dskip || !bias || !y) return SCAN2D_EINVAL;
  const bool bwd = dy != nullptr;
  if (bwd && (!dx || !dz || !dA || !dB || !dC || !dDskip || !dbias)) return SCAN2D_EINVAL;
  if (chunks < 1) {  // auto: >= 32 MB of host->device traffic per chunk, at most 8 chunks
    size_t in[8], out[8];
    counts(d, d.num_scans, in, out);
    size_t bytes = 0;
    for (int i = 0; i < 8; ++i) bytes += in[i] * es_of(d.dtype);
    chunks = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, bytes / (32u << 20))));
  }
  if (chunks > d.num_scans) chunks = static_cast<int>(d.num_scans);
  // chunks split scans, so parameters and B/C must be per scan
  if (d.params_period != d.num_scans || d.bc_group != 1) return SCAN2D_EUNSUPPORTED;
  rc = setup(d, chunks, bwd);
  if (rc != SCAN2D_OK) return rc;
  Ctx& c = *g_ctx;
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = es_of(d.dtype);
  const void* hin[8] = {x, z, B, C, A, Dskip, bias, dy};
  void* hout[8] = {y, dx, dz, dA, dB, dC, dDskip, dbias};
  // everything starts after the work already on the caller's stream
  if (cudaEventRecord(c.ev_start, user) != cudaSuccess) return SCAN2D_ECUDA;
  cudaStreamWaitEvent(c.h2d, c.ev_start, 0);
  const int nchunk = static_cast<int>((d.num_scans + c.chunk_scans - 1) / c.chunk_scans);
  for (int k = 0; k < nchunk; ++k) {
    const int sl = k % Ctx::kSlots;
    Slot& s = c.slot[sl];
    const int64_t s0 = static_cast<int64_t>(k) * c.chunk_scans;
    const int64_t sk = std::min<int64_t>(c.chunk_scans, d.num_scans - s0);
    size_t in[8], out[8], in0[8], out0[8];
    counts(d, sk, in, out);
    counts(d, s0, in0, out0);  // element offsets of this chunk in the host arrays
    if (k >= Ctx::kSlots) cudaStreamWaitEvent(c.h2d, c.ev_free[sl], 0);
    for (int i = 0; i < (bwd ? 8 : 7); ++i)
      if (cudaMemcpyAsync(s.in[i], static_cast<const char*>(hin[i]) + in0[i] * es, in[i] * es,
                          cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
        return SCAN2D_ECUDA;
    cudaEventRecord(c.ev_in[sl], c.h2d);
    cudaStreamWaitEvent(c.comp, c.ev_in[sl], 0);
    scan2d_desc cd = d;
    cd.num_scans = sk;
    cd.params_period = static_cast<int32_t>(sk);
    rc = scan2d_forward(&cd, s.in[0], s.in[1], s.in[2], s.in[3], s.in[4], s.in[5], s.in[6], s.out[0], nullptr,
                        nullptr, bwd ? s.residual : nullptr, s.wsf, s.wsf_bytes,
                        reinterpret_cast<scan2d_stream_t>(c.comp));
    if (rc != SCAN2D_OK) return rc;
    if (bwd) {
      rc = scan2d_backward(&cd, s.in[0], s.in[1], s.in[2], s.in[3], s.in[4], s.in[5], s.in[6], s.residual,
                           s.in[7], s.out[1], s.out[2], s.out[3], s.out[4], s.out[5], s.out[6], s.out[7], s.wsb,
                           s.wsb_bytes, reinterpret_cast<scan2d_stream_t>(c.comp));
      if (rc != SCAN2D_OK) return rc;
    }
    cudaEventRecord(c.ev_out[sl], c.comp);
    cudaStreamWaitEvent(c.d2h, c.ev_out[sl], 0);
    for (int i = 0; i < (bwd ? 8 : 1); ++i)
      if (cudaMemcpyAsync(static_cast<char*>(hout[i]) + out0[i] * es, s.out[i], out[i] * es,
                          cudaMemcpyDeviceToHost, c.d2h) != cudaSuccess)
        return SCAN2D_ECUDA;
    cudaEventRecord(c.ev_free[sl], c.d2h);
  }
  // the caller's stream resumes after the last device -> host copy
  for (int k = std::max(0, nchunk - Ctx::kSlots); k < nchunk; ++k)
    cudaStreamWaitEvent(user, c.ev_free[k % Ctx::kSlots], 0);
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}
