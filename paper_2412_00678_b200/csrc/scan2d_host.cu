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
// wait for chunk k's device->host copies to drain.  The parameters (A, Dskip,
// bias) go over once before the first chunk and their gradients come back once
// after the last, so a chunk costs five copies each way.  Shared B/C (G > 1)
// and shared parameters (P < S, the model layout) are served by cutting the
// scans at multiples of lcm(G, P): a chunk then owns whole B/C groups (its
// dB / dC slices are its own) and starts at parameter row 0, so it uses the
// whole parameter table and its parameter gradients are added into the
// totals on the compute stream, in chunk order (bit-reproducible).  The first
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
  void* dpar[3] = {};  // shared parameters (P < S): this chunk's dA, dDskip, dbias
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
      for (void* p : s.dpar) cudaFree(p);
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

template <typename T>
__global__ void accumulate_kernel(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[t] += src[t];
}

int accumulate(int dtype, void* dst, const void* src, int64_t n, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 4));
  if (n <= 0) return SCAN2D_OK;
  if (dtype == SCAN2D_F64)
    accumulate_kernel<double><<<blocks, 256, 0, st>>>(static_cast<double*>(dst), static_cast<const double*>(src), n);
  else
    accumulate_kernel<float><<<blocks, 256, 0, st>>>(static_cast<float*>(dst), static_cast<const float*>(src), n);
  return cudaGetLastError() == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}

int64_t gcd64(int64_t a, int64_t b) { return b == 0 ? a : gcd64(b, a % b); }

// scans per chunk quantum: whole B/C groups, and whole parameter periods when
// the parameters are shared (P < S)
int64_t quantum(const scan2d_desc& d) {
  const int64_t G = d.bc_group, P = d.params_period;
  if (P == d.num_scans) return G;
  return G / gcd64(G, P) * P;
}

// element counts of the per-chunk operands for s scans (s a multiple of G)
void counts(const scan2d_desc& d, int64_t s, size_t (&in)[kIn], size_t (&out)[kOut]) {
  const size_t hw = static_cast<size_t>(d.height) * d.width, n = d.state_dim;
  const size_t S = static_cast<size_t>(s), SB = static_cast<size_t>(s / d.bc_group);
  const size_t c[kIn] = {S * hw, S * hw, SB * hw * n, SB * hw * n, S * hw};
  const size_t o[kOut] = {S * hw, S * hw, S * hw, SB * hw * n, SB * hw * n};
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
  const int64_t q = quantum(d), units = d.num_scans / q;
  const int64_t cu = (units + chunks - 1) / chunks;  // quanta per base chunk
  c->chunk_scans = static_cast<int>(cu * q);
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
  c->sched = schedule(units, chunks, cu);  // in quanta
  for (auto& pc : c->sched) pc.first *= q, pc.second *= q;
  const bool shared_par = d.params_period != d.num_scans;
  scan2d_desc cd = d;
  cd.num_scans = c->chunk_scans;
  cd.params_period = shared_par ? d.params_period : c->chunk_scans;
  const size_t es = es_of(d.dtype);
  const size_t P = static_cast<size_t>(d.params_period), N = static_cast<size_t>(d.state_dim);
  const size_t pc[3] = {P * N, P, P};
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
      if (shared_par)
        for (int i = 0; i < 3; ++i)
          if (cudaMalloc(&s.dpar[i], pc[i] * es) != cudaSuccess) return SCAN2D_ENOMEM;
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
  // chunks are cut at whole quanta (B/C groups, parameter periods)
  const int64_t nunits = d.num_scans / quantum(d);
  if (chunks > nunits) chunks = static_cast<int>(nunits);
  rc = setup(d, chunks, bwd);
  if (rc != SCAN2D_OK) return rc;
  Ctx& c = *g_ctx;
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  const size_t N = static_cast<size_t>(d.state_dim);
  const bool shared_par = d.params_period != d.num_scans;
  const size_t P = static_cast<size_t>(d.params_period);
  const size_t pc[3] = {P * N, P, P};
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
  if (bwd && shared_par) {  // shared parameter gradients: summed over the chunks in order
    cudaStreamWaitEvent(c.comp, c.ev_start, 0);
    for (int i = 0; i < 3; ++i)
      if (cudaMemsetAsync(c.dpar[i], 0, pc[i] * es, c.comp) != cudaSuccess) return SCAN2D_ECUDA;
  }
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
    cd.params_period = shared_par ? d.params_period : static_cast<int32_t>(sk);
    const int64_t p0 = shared_par ? 0 : s0;  // first parameter row of the chunk
    const char* pA = static_cast<const char*>(c.par[0]) + p0 * N * es;
    const char* pD = static_cast<const char*>(c.par[1]) + p0 * es;
    const char* pb = static_cast<const char*>(c.par[2]) + p0 * es;
    rc = scan2d_forward(&cd, s.in[0], s.in[1], s.in[2], s.in[3], pA, pD, pb, s.out[0], nullptr, nullptr,
                        bwd ? s.residual : nullptr, s.wsf, s.wsf_bytes, reinterpret_cast<scan2d_stream_t>(c.comp));
    if (rc != SCAN2D_OK) return rc;
    if (bwd) {
      void* gA = shared_par ? s.dpar[0] : static_cast<char*>(c.dpar[0]) + s0 * N * es;
      void* gD = shared_par ? s.dpar[1] : static_cast<char*>(c.dpar[1]) + s0 * es;
      void* gb = shared_par ? s.dpar[2] : static_cast<char*>(c.dpar[2]) + s0 * es;
      rc = scan2d_backward(&cd, s.in[0], s.in[1], s.in[2], s.in[3], pA, pD, pb, s.residual, s.in[4], s.out[1],
                           s.out[2], gA, s.out[3], s.out[4], gD, gb, s.wsb, s.wsb_bytes,
                           reinterpret_cast<scan2d_stream_t>(c.comp));
      if (rc != SCAN2D_OK) return rc;
      if (shared_par) {
        const void* src[3] = {gA, gD, gb};
        for (int i = 0; i < 3; ++i)
          if ((rc = accumulate(d.dtype, c.dpar[i], src[i], static_cast<int64_t>(pc[i]), c.comp)) != SCAN2D_OK)
            return rc;
      }
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
