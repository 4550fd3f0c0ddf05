// ref_capi.cpp -- extern "C" wrapper over the REFERENCE library, compiled
// together with the reference's own sources (/root/reference/proj/src/*.cpp)
// into oracle/_ref/libscan2d_ref.so by oracle/Makefile.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the oracle restatement, by
// tests/golden/make_golden.py to produce golden vectors, and by bench.py's
// cpu_baseline / --impl reference legs to time the reference CPU engine.
// This file contains no reference code; it only calls the reference API
// declared in engine.hpp:88-102, reference.hpp:35-71, gradcheck.hpp:36,
// fixtures.hpp:20-37.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <sstream>
#include <thread>
#include <vector>

#include "scan2d/engine.hpp"
#include "scan2d/tensor_io.hpp"
#include "scan2d/fixtures.hpp"
#include "scan2d/gradcheck.hpp"
#include "scan2d/math.hpp"
#include "scan2d/reference.hpp"

using namespace scan2d;

namespace {

template <typename T>
Grid<T> grid_from(int h, int w, int d, const T* p) {
  return Grid<T>(h, w, d, std::vector<T>(p, p + static_cast<std::size_t>(h) * w * d));
}

template <typename T>
void random_instance_into(int h, int w, int n, std::uint64_t seed, T* x, T* z, T* b, T* c,
                          T* a, T* dskip, T* bias) {
  auto inst = random_instance<T>(h, w, n, seed);
  std::memcpy(x, inst.x.data.data(), sizeof(T) * inst.x.data.size());
  std::memcpy(z, inst.inputs.z_raw.data.data(), sizeof(T) * inst.inputs.z_raw.data.size());
  std::memcpy(b, inst.inputs.b.data.data(), sizeof(T) * inst.inputs.b.data.size());
  std::memcpy(c, inst.inputs.c.data.data(), sizeof(T) * inst.inputs.c.data.size());
  std::memcpy(a, inst.params.a.data(), sizeof(T) * inst.params.a.size());
  *dskip = inst.params.d_skip;
  *bias = inst.params.bias;
}

template <typename T>
int tiled_fwd(int h, int w, int n, int t, const T* x, const T* z, const T* b, const T* c,
              const T* a, T dskip, T bias, T* y, T* ph, T* pv) {
  try {
    Grid<T> gx = grid_from(h, w, 1, x);
    SelectiveInputs<T> in(grid_from(h, w, 1, z), grid_from(h, w, n, b), grid_from(h, w, n, c));
    ScanParams<T> params(std::vector<T>(a, a + n), dskip, bias);
    TileConfig tiles(h, w, t);
    auto res = tiled_scan_2d_forward(gx, in, params, tiles, 1, nullptr, false);
    std::memcpy(y, res.y.data.data(), sizeof(T) * res.y.data.size());
    if (ph) std::memcpy(ph, res.carries.ph.data(), sizeof(T) * res.carries.ph.size());
    if (pv) std::memcpy(pv, res.carries.pv.data(), sizeof(T) * res.carries.pv.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

template <typename T>
int tiled_bwd(int h, int w, int n, int t, const T* x, const T* z, const T* b, const T* c,
              const T* a, T dskip, T bias, const T* dy, T* dx, T* dz, T* da, T* db, T* dc,
              T* dd, T* dbias) {
  try {
    Grid<T> gx = grid_from(h, w, 1, x);
    SelectiveInputs<T> in(grid_from(h, w, 1, z), grid_from(h, w, n, b), grid_from(h, w, n, c));
    ScanParams<T> params(std::vector<T>(a, a + n), dskip, bias);
    TileConfig tiles(h, w, t);
    auto fwd = tiled_scan_2d_forward(gx, in, params, tiles);
    auto g = tiled_scan_2d_backward(fwd.saved, grid_from(h, w, 1, dy));
    std::memcpy(dx, g.dx.data.data(), sizeof(T) * g.dx.data.size());
    std::memcpy(dz, g.dz_raw.data.data(), sizeof(T) * g.dz_raw.data.size());
    std::memcpy(da, g.da.data(), sizeof(T) * g.da.size());
    std::memcpy(db, g.db.data.data(), sizeof(T) * g.db.data.size());
    std::memcpy(dc, g.dc.data.data(), sizeof(T) * g.dc.data.size());
    *dd = g.dd;
    *dbias = g.dbias;
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

template <typename T>
int oracle_fwd(int h, int w, int n, const T* x, const T* z, const T* b, const T* c, const T* a,
               T dskip, T bias, T* y, T* hh, T* hs) {
  try {
    Grid<T> gx = grid_from(h, w, 1, x);
    SelectiveInputs<T> in(grid_from(h, w, 1, z), grid_from(h, w, n, b), grid_from(h, w, n, c));
    ScanParams<T> params(std::vector<T>(a, a + n), dskip, bias);
    auto g = discretize(gx, in, params);
    auto s = scan_2d_sequential(g, in.c, params.d_skip, gx);
    std::memcpy(y, s.y.data.data(), sizeof(T) * s.y.data.size());
    if (hh) std::memcpy(hh, s.h_hor.data.data(), sizeof(T) * s.h_hor.data.size());
    if (hs) std::memcpy(hs, s.h.data.data(), sizeof(T) * s.h.data.size());
    return 0;
  } catch (...) {
    return 1;
  }
}

// S scans spread over a std::thread pool in contiguous blocks (the model.cpp:177
// pattern), one reference call per scan with threads = 1.  Params of scan s at
// s % P, B/C at s / G.  Returns wall seconds of the parallel region.
template <typename T>
double batch_run(std::int64_t S, int P, int G, int h, int w, int n, int t, int threads,
                 int do_bwd, const T* x, const T* z, const T* b, const T* c, const T* a,
                 const T* dskip, const T* bias, const T* dy, T* y, T* dx, T* dz = nullptr,
                 T* da = nullptr, T* db = nullptr, T* dc = nullptr, T* dd = nullptr, T* dbias = nullptr) {
  const std::size_t hw = static_cast<std::size_t>(h) * w, hwn = hw * n;
  if (threads < 1) threads = 1;
  if (threads > S) threads = static_cast<int>(S);
  const std::int64_t chunk = (S + threads - 1) / threads;
  auto body = [&](std::int64_t s0, std::int64_t s1) {
    for (std::int64_t s = s0; s < s1; ++s) {
      const std::int64_t p = s % P, g = s / G;
      Grid<T> gx = grid_from(h, w, 1, x + s * hw);
      SelectiveInputs<T> in(grid_from(h, w, 1, z + s * hw), grid_from(h, w, n, b + g * hwn),
                            grid_from(h, w, n, c + g * hwn));
      ScanParams<T> params(std::vector<T>(a + p * n, a + (p + 1) * n), dskip[p], bias[p]);
      TileConfig tiles(h, w, t);
      auto fwd = tiled_scan_2d_forward(gx, in, params, tiles, 1, nullptr, do_bwd != 0);
      if (y) std::memcpy(y + s * hw, fwd.y.data.data(), sizeof(T) * hw);
      if (do_bwd) {
        auto gr = tiled_scan_2d_backward(fwd.saved, grid_from(h, w, 1, dy + s * hw));
        if (dx) std::memcpy(dx + s * hw, gr.dx.data.data(), sizeof(T) * hw);
        // full gradient bundle (per-scan parameters and B/C only: P == S, G == 1)
        if (dz) std::memcpy(dz + s * hw, gr.dz_raw.data.data(), sizeof(T) * hw);
        if (da) std::memcpy(da + s * n, gr.da.data(), sizeof(T) * n);
        if (db) std::memcpy(db + s * hwn, gr.db.data.data(), sizeof(T) * hwn);
        if (dc) std::memcpy(dc + s * hwn, gr.dc.data.data(), sizeof(T) * hwn);
        if (dd) dd[s] = gr.dd;
        if (dbias) dbias[s] = gr.dbias;
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int k = 0; k < threads; ++k) {
    const std::int64_t s0 = k * chunk, s1 = std::min<std::int64_t>(S, s0 + chunk);
    if (s0 >= s1) break;
    pool.emplace_back(body, s0, s1);
  }
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // namespace

extern "C" {

void ref_random_instance_f64(int h, int w, int n, std::uint64_t seed, double* x, double* z,
                             double* b, double* c, double* a, double* d, double* bias) {
  random_instance_into<double>(h, w, n, seed, x, z, b, c, a, d, bias);
}
void ref_random_instance_f32(int h, int w, int n, std::uint64_t seed, float* x, float* z,
                             float* b, float* c, float* a, float* d, float* bias) {
  random_instance_into<float>(h, w, n, seed, x, z, b, c, a, d, bias);
}
void ref_fill_normal_f64(std::uint64_t seed, std::size_t count, double* out) {
  Rng rng(seed);
  for (std::size_t k = 0; k < count; ++k) out[k] = rng.normal();
}

int ref_tiled_fwd_f64(int h, int w, int n, int t, const double* x, const double* z,
                      const double* b, const double* c, const double* a, double d, double bias,
                      double* y, double* ph, double* pv) {
  return tiled_fwd<double>(h, w, n, t, x, z, b, c, a, d, bias, y, ph, pv);
}
int ref_tiled_fwd_f32(int h, int w, int n, int t, const float* x, const float* z,
                      const float* b, const float* c, const float* a, float d, float bias,
                      float* y, float* ph, float* pv) {
  return tiled_fwd<float>(h, w, n, t, x, z, b, c, a, d, bias, y, ph, pv);
}
int ref_tiled_bwd_f64(int h, int w, int n, int t, const double* x, const double* z,
                      const double* b, const double* c, const double* a, double d, double bias,
                      const double* dy, double* dx, double* dz, double* da, double* db,
                      double* dc, double* dd, double* dbias) {
  return tiled_bwd<double>(h, w, n, t, x, z, b, c, a, d, bias, dy, dx, dz, da, db, dc, dd,
                           dbias);
}
int ref_tiled_bwd_f32(int h, int w, int n, int t, const float* x, const float* z,
                      const float* b, const float* c, const float* a, float d, float bias,
                      const float* dy, float* dx, float* dz, float* da, float* db, float* dc,
                      float* dd, float* dbias) {
  return tiled_bwd<float>(h, w, n, t, x, z, b, c, a, d, bias, dy, dx, dz, da, db, dc, dd,
                          dbias);
}
int ref_oracle_fwd_f64(int h, int w, int n, const double* x, const double* z, const double* b,
                       const double* c, const double* a, double d, double bias, double* y,
                       double* hh, double* hs) {
  return oracle_fwd<double>(h, w, n, x, z, b, c, a, d, bias, y, hh, hs);
}
int ref_oracle_fwd_f32(int h, int w, int n, const float* x, const float* z, const float* b,
                       const float* c, const float* a, float d, float bias, float* y, float* hh,
                       float* hs) {
  return oracle_fwd<float>(h, w, n, x, z, b, c, a, d, bias, y, hh, hs);
}
float ref_fast_expf(float x) { return num::fast_expf(x); }

// groups: dx, dz_raw, da, db, dc, dd, dbias -> out[2*k] = max_rel, out[2*k+1] = max_abs_small
int ref_gradcheck(int h, int w, int n, std::uint64_t seed, double step, int tile, double* out) {
  auto r = gradcheck(h, w, n, seed, step, tile);
  for (std::size_t k = 0; k < r.groups.size(); ++k) {
    out[2 * k] = r.groups[k].max_rel;
    out[2 * k + 1] = r.groups[k].max_abs_small;
  }
  return static_cast<int>(r.groups.size());
}

double ref_batch_f32(std::int64_t S, int P, int G, int h, int w, int n, int t, int threads,
                     int do_bwd, const float* x, const float* z, const float* b, const float* c,
                     const float* a, const float* d, const float* bias, const float* dy,
                     float* y, float* dx) {
  return batch_run<float>(S, P, G, h, w, n, t, threads, do_bwd, x, z, b, c, a, d, bias, dy, y,
                          dx);
}
double ref_batch_f64(std::int64_t S, int P, int G, int h, int w, int n, int t, int threads,
                     int do_bwd, const double* x, const double* z, const double* b,
                     const double* c, const double* a, const double* d, const double* bias,
                     const double* dy, double* y, double* dx) {
  return batch_run<double>(S, P, G, h, w, n, t, threads, do_bwd, x, z, b, c, a, d, bias, dy, y,
                           dx);
}

// T2DM through the reference's own tensor I/O (tensor_io.cpp:78-151): the
// golden encoder / decoder the repository's format code is checked against.
std::size_t ref_t2dm_encode(int dtype, int ndim, const std::uint64_t* dims, const void* data, unsigned char* out,
                            std::size_t cap) {
  Tensor t;
  t.dtype = dtype == 1 ? Dtype::f64 : Dtype::f32;
  t.dims.assign(dims, dims + ndim);
  const std::size_t n = t.count();
  if (dtype == 1)
    t.f64.assign(static_cast<const double*>(data), static_cast<const double*>(data) + n);
  else
    t.f32.assign(static_cast<const float*>(data), static_cast<const float*>(data) + n);
  std::ostringstream os;
  try {
    write_tensor(t, os);
  } catch (...) {
    return 0;
  }
  const std::string b = os.str();
  if (b.size() > cap) return 0;
  std::memcpy(out, b.data(), b.size());
  return b.size();
}
// -1 = decoded (payload copied to out_data when given), else TensorIoError::Kind
int ref_t2dm_decode(const unsigned char* buf, std::size_t len, std::size_t* offset, void* out_data) {
  std::istringstream is(std::string(reinterpret_cast<const char*>(buf), len));
  try {
    Tensor t = read_tensor(is);
    if (out_data) {
      if (t.dtype == Dtype::f64)
        std::memcpy(out_data, t.f64.data(), 8 * t.f64.size());
      else
        std::memcpy(out_data, t.f32.data(), 4 * t.f32.size());
    }
    return -1;
  } catch (const TensorIoError& e) {
    *offset = e.offset;
    return static_cast<int>(e.kind);
  }
}

// Every gradient group per scan (P == S, G == 1; the bench's parity report).
double ref_batch_grads_f32(std::int64_t S, int h, int w, int n, int t, int threads, const float* x,
                           const float* z, const float* b, const float* c, const float* a,
                           const float* d, const float* bias, const float* dy, float* y, float* dx,
                           float* dz, float* da, float* db, float* dc, float* dd, float* dbias) {
  return batch_run<float>(S, static_cast<int>(S), 1, h, w, n, t, threads, 1, x, z, b, c, a, d, bias, dy, y,
                          dx, dz, da, db, dc, dd, dbias);
}
double ref_batch_grads_f64(std::int64_t S, int h, int w, int n, int t, int threads, const double* x,
                           const double* z, const double* b, const double* c, const double* a,
                           const double* d, const double* bias, const double* dy, double* y,
                           double* dx, double* dz, double* da, double* db, double* dc, double* dd,
                           double* dbias) {
  return batch_run<double>(S, static_cast<int>(S), 1, h, w, n, t, threads, 1, x, z, b, c, a, d, bias, dy,
                           y, dx, dz, da, db, dc, dd, dbias);
}

}  // extern "C"
