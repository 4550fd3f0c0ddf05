// scan2d_host.cu -- host-operand entry point (include/scan2d_cuda.h,
// scan2d_train_host): the reference API takes and returns host data
// (engine.hpp:88-102, Grid<T> holds std::vector), so the drop-in path is
// host -> device -> scan -> host.  This runtime pipelines it: the S scans go
// through the device in chunks; chunk k's host->device copies, chunk k-1's
// forward + backward kernels and chunk k-2's device->host copies run
// concurrently on three streams ordered by events, so the PCIe transfers in
// both directions overlap each other and the kernels.
//
// Three device buffer sets rotate, so chunk k+2's host->device copies never
// wait for chunk k's device->host copies to drain.  The per-scan parameters
// (A, Dskip, bias) go over once before the first chunk and their gradients come
// back once after the last, so a chunk costs five copies each way.  The first
// and the last base chunk are split into 1/8, 1/8, 1/4, 1/2 pieces (ramp): the
// device->host direction starts, and the host->device direction finishes, after
// one small piece instead of one whole chunk.  Device buffers, streams and
// events are cached per host thread and per (descriptor, chunk count).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <memory>
#include <utility>
#include <vector>

#include "../../include/scan2d_cuda.h"

namespace {

size_t es_of(int dtype) { return dtype == SCAN2D_F64 ? 8 : 4; }

// per-chunk operands: inputs x z B C dy | outputs y dx dz dB dC
constexpr int kIn = 5, kOut = 5;

struct Slot {
  void* in[kIn] = {};
  void* out[kOut] = {};
  void* residual = nullptr;
  void* wsf = nullptr;
  void* wsb = nullptr;
  size_t wsf_bytes = 0, wsb_bytes = 0;
};

struct Ctx {
  scan2d_desc desc{};
  int chunks = 0, chunk_scans = 0;
  std::vector<std::pair<int64_t, int64_t>> sched;  // (first scan, scans) per chunk
  void* par[3] = {};   // A [S][N], Dskip [S], bias [S] (whole problem)
  void* dpar[3] = {};  // dA, dDskip, dbias
  bool with_bwd = false;
  int device = -1;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  static constexpr int kSlots = 3;
  cudaEvent_t ev_in[kSlots] = {}, ev_out[kSlots] = {}, ev_free[kSlots] = {}, ev_start = nullptr;
  Slot slot[kSlots];
  ~Ctx() {
    for (void* p : par) cudaFree(p);
    for (void* p : dpar) cudaFree(p);
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

// element counts of the per-chunk operands for s scans (P == S, G == 1)
void counts(const scan2d_desc& d, int64_t s, size_t (&in)[kIn], size_t (&out)[kOut]) {
  const size_t hw = static_cast<size_t>(d.height) * d.width, n = d.state_dim;
  const size_t S = static_cast<size_t>(s);
  const size_t c[kIn] = {S * hw, S * hw, S * hw * n, S * hw * n, S * hw};
  const size_t o[kOut] = {S * hw, S * hw, S * hw, S * hw * n, S * hw * n};
  for (int i = 0; i < kIn; ++i) in[i] = c[i];
  for (int i = 0; i < kOut; ++i) out[i] = o[i];
}

// chunk schedule: `chunks` base chunks of c0 scans; the first and the last are
// split into 1/8, 1/8, 1/4, 1/2 (resp. reversed) pieces when large enough
std::vector<std::pair<int64_t, int64_t>> schedule(int64_t S, int chunks, int64_t c0) {
  std::vector<int64_t> sizes;
  auto ramp = [&](int64_t n, bool up) {
    std::vector<int64_t> p;
    if (n >= 8)
      p = {n / 8, n / 8, n / 4, n - n / 8 - n / 8 - n / 4};
    else
      p = {n};
    if (!up) std::reverse(p.begin(), p.end());
    for (int64_t v : p) sizes.push_back(v);
  };
  int64_t left = S;
  for (int k = 0; k < chunks && left > 0; ++k) {
    const int64_t n = std::min(c0, left);
    left -= n;
    if (chunks > 1 && k == 0)
      ramp(n, true);
    else if (chunks > 1 && left == 0)
      ramp(n, false);
    else
      sizes.push_back(n);
  }
  std::vector<std::pair<int64_t, int64_t>> out;
  int64_t s0 = 0;
  for (int64_t v : sizes) {
    if (v <= 0) continue;
    out.emplace_back(s0, v);
    s0 += v;
  }
  return out;
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
  c->sched = schedule(d.num_scans, chunks, c->chunk_scans);
  scan2d_desc cd = d;
  cd.num_scans = c->chunk_scans;
  cd.params_period = c->chunk_scans;
  cd.bc_group = 1;
  const size_t es = es_of(d.dtype);
  const size_t S = static_cast<size_t>(d.num_scans), N = static_cast<size_t>(d.state_dim);
  const size_t pc[3] = {S * N, S, S};
  for (int i = 0; i < 3; ++i) {
    if (cudaMalloc(&c->par[i], pc[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
    if (with_bwd && cudaMalloc(&c->dpar[i], pc[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
  }
  size_t in[kIn], out[kOut];
  counts(d, c->chunk_scans, in, out);
  for (Slot& s : c->slot) {
    for (int i = 0; i < kIn; ++i)
      if ((with_bwd || i < 4) && cudaMalloc(&s.in[i], in[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
    for (int i = 0; i < kOut; ++i)
      if ((with_bwd || i == 0) && cudaMalloc(&s.out[i], out[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
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
  const size_t es = es_of(d.dtype);
  if (chunks < 1) {  // auto: >= 32 MB of host->device traffic per chunk, at most 8 chunks
    size_t in[kIn], out[kOut];
    counts(d, d.num_scans, in, out);
    size_t bytes = 0;
    for (int i = 0; i < kIn; ++i) bytes += in[i] * es;
    chunks = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, bytes / (32u << 20))));
  }
  if (chunks > d.num_scans) chunks = static_cast<int>(d.num_scans);
  // chunks split scans, so parameters and B/C must be per scan
  if (d.params_period != d.num_scans || d.bc_group != 1) return SCAN2D_EUNSUPPORTED;
  rc = setup(d, chunks, bwd);
  if (rc != SCAN2D_OK) return rc;
  Ctx& c = *g_ctx;
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  const size_t N = static_cast<size_t>(d.state_dim);
  const size_t pc[3] = {static_cast<size_t>(d.num_scans) * N, static_cast<size_t>(d.num_scans),
                        static_cast<size_t>(d.num_scans)};
  const void* hpar[3] = {A, Dskip, bias};
  void* hdpar[3] = {dA, dDskip, dbias};
  const void* hin[kIn] = {x, z, B, C, dy};
  void* hout[kOut] = {y, dx, dz, dB, dC};
  // everything starts after the work already on the caller's stream
  if (cudaEventRecord(c.ev_start, user) != cudaSuccess) return SCAN2D_ECUDA;
  cudaStreamWaitEvent(c.h2d, c.ev_start, 0);
  for (int i = 0; i < 3; ++i)
    if (cudaMemcpyAsync(c.par[i], hpar[i], pc[i] * es, cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
      return SCAN2D_ECUDA;
  const int nchunk = static_cast<int>(c.sched.size());
  for (int k = 0; k < nchunk; ++k) {
    const int sl = k % Ctx::kSlots;
    Slot& s = c.slot[sl];
    const int64_t s0 = c.sched[k].first, sk = c.sched[k].second;
    size_t in[kIn], out[kOut], in0[kIn], out0[kOut];
    counts(d, sk, in, out);
    counts(d, s0, in0, out0);  // element offsets of this chunk in the host arrays
    if (k >= Ctx::kSlots) cudaStreamWaitEvent(c.h2d, c.ev_free[sl], 0);
    for (int i = 0; i < (bwd ? kIn : 4); ++i)
      if (cudaMemcpyAsync(s.in[i], static_cast<const char*>(hin[i]) + in0[i] * es, in[i] * es,
                          cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
        return SCAN2D_ECUDA;
    cudaEventRecord(c.ev_in[sl], c.h2d);
    cudaStreamWaitEvent(c.comp, c.ev_in[sl], 0);
    scan2d_desc cd = d;
    cd.num_scans = sk;
    cd.params_period = static_cast<int32_t>(sk);
    const char* pA = static_cast<const char*>(c.par[0]) + s0 * N * es;
    const char* pD = static_cast<const char*>(c.par[1]) + s0 * es;
    const char* pb = static_cast<const char*>(c.par[2]) + s0 * es;
    rc = scan2d_forward(&cd, s.in[0], s.in[1], s.in[2], s.in[3], pA, pD, pb, s.out[0], nullptr, nullptr,
                        bwd ? s.residual : nullptr, s.wsf, s.wsf_bytes, reinterpret_cast<scan2d_stream_t>(c.comp));
    if (rc != SCAN2D_OK) return rc;
    if (bwd) {
      rc = scan2d_backward(&cd, s.in[0], s.in[1], s.in[2], s.in[3], pA, pD, pb, s.residual, s.in[4], s.out[1],
                           s.out[2], static_cast<char*>(c.dpar[0]) + s0 * N * es, s.out[3], s.out[4],
                           static_cast<char*>(c.dpar[1]) + s0 * es, static_cast<char*>(c.dpar[2]) + s0 * es,
                           s.wsb, s.wsb_bytes, reinterpret_cast<scan2d_stream_t>(c.comp));
      if (rc != SCAN2D_OK) return rc;
    }
    cudaEventRecord(c.ev_out[sl], c.comp);
    cudaStreamWaitEvent(c.d2h, c.ev_out[sl], 0);
    for (int i = 0; i < (bwd ? kOut : 1); ++i)
      if (cudaMemcpyAsync(static_cast<char*>(hout[i]) + out0[i] * es, s.out[i], out[i] * es,
                          cudaMemcpyDeviceToHost, c.d2h) != cudaSuccess)
        return SCAN2D_ECUDA;
    cudaEventRecord(c.ev_free[sl], c.d2h);
  }
  // parameter gradients: once, after the last chunk's kernels (d2h is ordered after them)
  if (bwd)
    for (int i = 0; i < 3; ++i)
      if (cudaMemcpyAsync(hdpar[i], c.dpar[i], pc[i] * es, cudaMemcpyDeviceToHost, c.d2h) != cudaSuccess)
        return SCAN2D_ECUDA;
  if (cudaEventRecord(c.ev_start, c.d2h) != cudaSuccess) return SCAN2D_ECUDA;
  // the caller's stream resumes after the last device -> host copy (d2h is in order)
  cudaStreamWaitEvent(user, c.ev_start, 0);
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}
