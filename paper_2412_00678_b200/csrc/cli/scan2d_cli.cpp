// scan2d_cli -- command-line entry point over the C ABI (include/scan2d_cuda.h,
// include/scan2d_t2dm.h): the reference artifact's CLI (SPEC.md:455-500,
// subcommands SPEC.md:471-477; the reference's tools/scan2d_cli.cpp is listed
// in proj/CMakeLists.txt:35 but not shipped) for the GPU operator.
//
//   scan      --input X.t2dm --output Y.t2dm [--variant tiled2d|naive2d|seq1d]
//             [--tile T] [--state-dim N] [--seed S] [--dtype f32|f64]
//             [--z F --b F --c F --a F --dskip F --bias F]
//             x is [H,W] (T2DM v1) or [S,H,W] (v2); missing operands are drawn
//             from --seed (x, z, B, C ~ N(0,1), A ~ -U(0.05,0.95), D ~ N(0,1),
//             bias ~ U(-0.5,0.5): the reference's random_instance distribution)
//   verify    --sizes 16x16,56x56 --seeds 0,1 [--dtype f32|f64] [--state-dim N]
//             tiled2d against the naive 2D operator computed in f64 (a different
//             algorithm: N horizontal state maps, then a column pass), tile
//             invariance (y identical for T in {1, 5, 16, 64}), and the
//             backward's fp64 finite-difference check on a sample of entries
//   gradcheck --height H --width W --state-dim N --seed S
//   bench     --variant V --height H --width W --state-dim N [--tile T]
//             [--reps R] [--warmup K] [--batch S] [--backward] [--dtype f32|f64]
//
// Output: one JSON object per line on stdout.  Exit codes: 0 ok, 1 a check
// failed, 2 usage error (SPEC.md: "exit codes 0/1/2").
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../../include/scan2d_cuda.h"
#include "../../../include/scan2d_t2dm.h"

namespace {

[[noreturn]] void usage(const char* msg) {
  std::fprintf(stderr,
               "scan2d_cli: %s\n"
               "usage: scan2d_cli {scan|verify|gradcheck|bench} [--flag value ...]\n"
               "  scan      --input X.t2dm --output Y.t2dm [--variant tiled2d|naive2d|seq1d] [--tile T]\n"
               "            [--state-dim N] [--seed S] [--dtype f32|f64] [--z|--b|--c|--a|--dskip|--bias FILE]\n"
               "  verify    --sizes HxW,... --seeds S,... [--dtype f32|f64] [--state-dim N]\n"
               "  gradcheck --height H --width W --state-dim N --seed S\n"
               "  bench     --variant V --height H --width W --state-dim N [--tile T] [--reps R] [--warmup K]\n"
               "            [--batch S] [--backward] [--dtype f32|f64]\n",
               msg);
  std::exit(2);
}

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  long num(const std::string& k, long d) const {
    auto it = kv.find(k);
    if (it == kv.end()) return d;
    char* end = nullptr;
    const long v = std::strtol(it->second.c_str(), &end, 10);
    if (end == it->second.c_str() || *end != 0) usage(("bad integer for --" + k).c_str());
    return v;
  }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& flags,
           const std::vector<std::string>& switches) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string f = argv[i];
    if (f.rfind("--", 0) != 0) usage(("unexpected argument " + f).c_str());
    f = f.substr(2);
    if (std::find(switches.begin(), switches.end(), f) != switches.end()) {
      a.kv[f] = "1";
      continue;
    }
    if (std::find(flags.begin(), flags.end(), f) == flags.end()) usage(("unknown flag --" + f).c_str());
    if (i + 1 >= argc) usage(("missing value for --" + f).c_str());
    a.kv[f] = argv[++i];
  }
  if (const char* t = std::getenv("SCAN2D_THREADS")) (void)t;  // accepted, results are thread-invariant
  return a;
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      std::fprintf(stderr, "scan2d_cli: CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                   __LINE__);                                                                  \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)

void check_rc(int rc, const char* where) {
  if (rc != SCAN2D_OK) {
    std::fprintf(stderr, "scan2d_cli: %s: %s\n", where, scan2d_status_string(rc));
    std::exit(1);
  }
}

// ---------------------------------------------------------------- host data

// splitmix64 stream + Box-Muller: the random_instance distribution
// (x, z, B, C ~ N(0,1); A ~ -U(0.05, 0.95); D ~ N(0,1); bias ~ U(-0.5, 0.5))
struct Gen {
  uint64_t s;
  explicit Gen(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  double normal() {
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * uniform());
  }
};

struct Problem {  // host operands, f64 (cast on upload)
  int64_t S = 1;
  int H = 1, W = 1, N = 1;
  std::vector<double> x, z, B, C, A, D, bias, dy;
};

Problem random_problem(int64_t S, int H, int W, int N, uint64_t seed) {
  Problem p;
  p.S = S, p.H = H, p.W = W, p.N = N;
  const size_t hw = static_cast<size_t>(H) * W;
  p.x.resize(S * hw), p.z.resize(S * hw), p.dy.resize(S * hw);
  p.B.resize(S * hw * N), p.C.resize(S * hw * N);
  p.A.resize(S * N), p.D.resize(S), p.bias.resize(S);
  for (int64_t s = 0; s < S; ++s) {
    Gen g(seed * 1000003ull + static_cast<uint64_t>(s));
    for (size_t k = 0; k < hw; ++k) p.x[s * hw + k] = g.normal();
    for (size_t k = 0; k < hw; ++k) p.z[s * hw + k] = g.normal();
    for (size_t k = 0; k < hw * N; ++k) p.B[s * hw * N + k] = g.normal();
    for (size_t k = 0; k < hw * N; ++k) p.C[s * hw * N + k] = g.normal();
    for (int d = 0; d < N; ++d) p.A[s * N + d] = -(0.05 + 0.9 * g.uniform());
    p.D[s] = g.normal();
    p.bias[s] = g.uniform() - 0.5;
    for (size_t k = 0; k < hw; ++k) p.dy[s * hw + k] = g.normal();
  }
  return p;
}

// -------------------------------------------------------------- device data

struct Dev {
  void* p = nullptr;
  size_t n = 0;
  Dev() = default;
  explicit Dev(size_t bytes) : n(bytes) { CK(cudaMalloc(&p, bytes ? bytes : 16)); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() {
    if (p) cudaFree(p);
  }
};

template <typename T>
void up(Dev& d, const std::vector<double>& h) {
  std::vector<T> t(h.begin(), h.end());
  CK(cudaMemcpy(d.p, t.data(), sizeof(T) * t.size(), cudaMemcpyHostToDevice));
}

template <typename T>
std::vector<double> down(const Dev& d, size_t n) {
  std::vector<T> t(n);
  CK(cudaMemcpy(t.data(), d.p, sizeof(T) * n, cudaMemcpyDeviceToHost));
  return std::vector<double>(t.begin(), t.end());
}

struct DevProblem {
  scan2d_desc desc{};
  size_t es;
  Dev x, z, B, C, A, D, bias, dy;
  template <typename T>
  void load(const Problem& p) {
    up<T>(x, p.x), up<T>(z, p.z), up<T>(B, p.B), up<T>(C, p.C), up<T>(A, p.A), up<T>(D, p.D);
    up<T>(bias, p.bias), up<T>(dy, p.dy);
  }
  DevProblem(const Problem& p, int dtype, int tile)
      : es(dtype == SCAN2D_F64 ? 8 : 4),
        x(es * p.x.size()), z(es * p.z.size()), B(es * p.B.size()), C(es * p.C.size()), A(es * p.A.size()),
        D(es * p.D.size()), bias(es * p.bias.size()), dy(es * p.dy.size()) {
    desc.num_scans = p.S, desc.height = p.H, desc.width = p.W, desc.state_dim = p.N, desc.tile = tile;
    desc.params_period = static_cast<int32_t>(p.S), desc.bc_group = 1, desc.dtype = dtype;
    if (dtype == SCAN2D_F64)
      load<double>(p);
    else
      load<float>(p);
  }
};

enum class Variant { Tiled, Naive, Flat };

Variant parse_variant(const std::string& v) {
  if (v == "tiled2d" || v == "seq2d") return Variant::Tiled;
  if (v == "naive2d") return Variant::Naive;
  if (v == "seq1d" || v == "flat1d" || v == "cub1d") return Variant::Flat;
  usage(("unknown variant " + v).c_str());
}

// forward of one variant; y must hold S*H*W elements
void forward(DevProblem& dp, Variant v, Dev& y, Dev* res = nullptr, Dev* ph = nullptr, Dev* pv = nullptr) {
  const scan2d_desc& d = dp.desc;
  if (v == Variant::Tiled) {
    Dev ws(scan2d_workspace_bytes(&d, SCAN2D_OP_FWD));
    check_rc(scan2d_forward(&d, dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, y.p,
                            ph ? ph->p : nullptr, pv ? pv->p : nullptr, res ? res->p : nullptr, ws.p, ws.n,
                            nullptr),
             "scan2d_forward");
  } else {
    const int var = v == Variant::Naive ? SCAN2D_VARIANT_NAIVE : SCAN2D_VARIANT_FLAT1D;
    Dev ws(scan2d_comparator_workspace_bytes(&d, var));
    check_rc(scan2d_forward_variant(&d, var, dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, y.p,
                                    ws.p, ws.n, nullptr),
             "scan2d_forward_variant");
  }
  CK(cudaDeviceSynchronize());
}

double rel_error(const std::vector<double>& got, const std::vector<double>& ref) {
  // normwise error of the reference tests (test_util.hpp:17-26)
  double num = 0.0, den = 1.0;
  for (size_t i = 0; i < ref.size(); ++i) {
    num = std::max(num, std::fabs(got[i] - ref[i]));
    den = std::max(den, std::fabs(ref[i]));
  }
  return num / den;
}

// ------------------------------------------------------------ T2DM helpers

std::vector<double> read_t2dm(const std::string& path, std::vector<uint64_t>& dims) {
  scan2d_tensor t{};
  size_t off = 0;
  const int rc = scan2d_t2dm_read(path.c_str(), &t, &off);
  if (rc != SCAN2D_T2DM_OK) {
    std::fprintf(stderr, "scan2d_cli: %s: %s at byte %zu\n", path.c_str(), scan2d_t2dm_status_string(rc), off);
    std::exit(1);
  }
  dims.assign(t.dims, t.dims + t.ndim);
  size_t n = 1;
  for (auto d : dims) n *= d;
  std::vector<double> v(n);
  for (size_t i = 0; i < n; ++i)
    v[i] = t.dtype == 1 ? static_cast<const double*>(t.data)[i] : static_cast<const float*>(t.data)[i];
  scan2d_t2dm_free(&t);
  return v;
}

void write_t2dm(const std::string& path, const std::vector<double>& v, const std::vector<uint64_t>& dims,
                int dtype) {
  scan2d_tensor t{};
  t.dtype = dtype;
  t.ndim = static_cast<int>(dims.size());
  for (size_t i = 0; i < dims.size(); ++i) t.dims[i] = dims[i];
  std::vector<float> f;
  if (dtype == 0) {
    f.assign(v.begin(), v.end());
    t.data = f.data();
  } else {
    t.data = const_cast<double*>(v.data());
  }
  size_t bytes = 0;
  const int rc = scan2d_t2dm_write(path.c_str(), &t, &bytes);
  if (rc != SCAN2D_T2DM_OK) {
    std::fprintf(stderr, "scan2d_cli: %s: %s\n", path.c_str(), scan2d_t2dm_status_string(rc));
    std::exit(1);
  }
}

int dtype_of(const Args& a) {
  const std::string d = a.str("dtype", "f32");
  if (d == "f32") return SCAN2D_F32;
  if (d == "f64") return SCAN2D_F64;
  usage("--dtype must be f32 or f64");
}

// ---------------------------------------------------------------- commands

int cmd_scan(const Args& a) {
  if (!a.has("input") || !a.has("output")) usage("scan needs --input and --output");
  std::vector<uint64_t> xd;
  std::vector<double> x = read_t2dm(a.str("input"), xd);
  if (xd.size() == 1) xd.push_back(1);
  if (xd.size() != 2 && xd.size() != 3) usage("--input must be [H,W] or [S,H,W]");
  const int64_t S = xd.size() == 3 ? static_cast<int64_t>(xd[0]) : 1;
  const int H = static_cast<int>(xd[xd.size() - 2]), W = static_cast<int>(xd[xd.size() - 1]);
  const int N = static_cast<int>(a.num("state-dim", 16));
  const int T = static_cast<int>(a.num("tile", 16));
  const int dtype = dtype_of(a);
  Problem p = random_problem(S, H, W, N, static_cast<uint64_t>(a.num("seed", 0)));
  p.x = x;
  const size_t hw = static_cast<size_t>(H) * W;
  auto load = [&](const char* flag, std::vector<double>& dst, size_t n) {
    if (!a.has(flag)) return;
    std::vector<uint64_t> dd;
    std::vector<double> v = read_t2dm(a.str(flag), dd);
    if (v.size() != n) usage((std::string("--") + flag + " has the wrong element count").c_str());
    dst = v;
  };
  load("z", p.z, S * hw), load("b", p.B, S * hw * N), load("c", p.C, S * hw * N);
  load("a", p.A, S * N), load("dskip", p.D, S), load("bias", p.bias, S);
  DevProblem dp(p, dtype, T);
  check_rc(scan2d_check_desc(&dp.desc), "descriptor");
  Dev y(dp.es * S * hw);
  const Variant v = parse_variant(a.str("variant", "tiled2d"));
  forward(dp, v, y);
  std::vector<double> yh = dtype == SCAN2D_F64 ? down<double>(y, S * hw) : down<float>(y, S * hw);
  std::vector<uint64_t> od = xd.size() == 3 ? xd : std::vector<uint64_t>{xd[0], xd[1]};
  write_t2dm(a.str("output"), yh, od, dtype);
  std::printf("{\"command\": \"scan\", \"variant\": \"%s\", \"scans\": %lld, \"height\": %d, \"width\": %d, "
              "\"state_dim\": %d, \"tile\": %d, \"dtype\": \"%s\", \"output\": \"%s\"}\n",
              a.str("variant", "tiled2d").c_str(), static_cast<long long>(S), H, W, N, T,
              dtype == SCAN2D_F64 ? "f64" : "f32", a.str("output").c_str());
  return 0;
}

std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  size_t b = 0;
  while (b <= s.size()) {
    size_t e = s.find(c, b);
    if (e == std::string::npos) e = s.size();
    if (e > b) out.push_back(s.substr(b, e - b));
    b = e + 1;
  }
  return out;
}

// analytic gradients (f64) and central differences of L = sum dy * y on a
// sample of entries of every group; returns the worst relative error per group
struct GradReport {
  const char* name;
  double max_rel = 0.0;
  double max_abs = 0.0;
};

std::vector<GradReport> gradcheck(const Problem& p0, int samples, double step) {
  const int64_t S = p0.S;
  const size_t hw = static_cast<size_t>(p0.H) * p0.W;
  auto loss = [&](const Problem& p) {
    DevProblem dp(p, SCAN2D_F64, 16);
    Dev y(8 * S * hw);
    forward(dp, Variant::Tiled, y);
    std::vector<double> yh = down<double>(y, S * hw);
    double l = 0.0;
    for (size_t i = 0; i < yh.size(); ++i) l += p.dy[i] * yh[i];
    return l;
  };
  DevProblem dp(p0, SCAN2D_F64, 16);
  const scan2d_desc& d = dp.desc;
  Dev y(8 * S * hw), res(scan2d_residual_bytes(&d)), wsf(scan2d_workspace_bytes(&d, SCAN2D_OP_FWD));
  Dev wsb(scan2d_workspace_bytes(&d, SCAN2D_OP_BWD));
  Dev dx(8 * S * hw), dz(8 * S * hw), dA(8 * p0.A.size()), dB(8 * p0.B.size()), dC(8 * p0.C.size()),
      dD(8 * S), db(8 * S);
  check_rc(scan2d_forward(&d, dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, y.p, nullptr, nullptr,
                          res.p, wsf.p, wsf.n, nullptr),
           "scan2d_forward");
  check_rc(scan2d_backward(&d, dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, res.p, dp.dy.p, dx.p,
                           dz.p, dA.p, dB.p, dC.p, dD.p, db.p, wsb.p, wsb.n, nullptr),
           "scan2d_backward");
  CK(cudaDeviceSynchronize());
  struct G {
    const char* name;
    std::vector<double> Problem::*field;
    Dev* grad;
  } groups[] = {{"dx", &Problem::x, &dx},   {"dz_raw", &Problem::z, &dz}, {"da", &Problem::A, &dA},
                {"db", &Problem::B, &dB},   {"dc", &Problem::C, &dC},     {"dd", &Problem::D, &dD},
                {"dbias", &Problem::bias, &db}};
  std::vector<GradReport> out;
  for (auto& g : groups) {
    const std::vector<double>& base = p0.*(g.field);
    std::vector<double> an = down<double>(*g.grad, base.size());
    GradReport r{g.name};
    const size_t n = base.size();
    for (int k = 0; k < samples && k < static_cast<int>(n); ++k) {
      const size_t i = n <= static_cast<size_t>(samples) ? k : (static_cast<size_t>(k) * 7919u) % n;
      Problem pp = p0, pm = p0;
      (pp.*(g.field))[i] += step;
      (pm.*(g.field))[i] -= step;
      const double fd = (loss(pp) - loss(pm)) / (2 * step);
      const double err = std::fabs(fd - an[i]);
      // gradcheck.cpp GroupAccum::take: relative error where |analytic| >= 1e-6
      // (small_cutoff, gradcheck.hpp:22), absolute error below it
      if (std::fabs(an[i]) < 1e-6)
        r.max_abs = std::max(r.max_abs, err);
      else
        r.max_rel = std::max(r.max_rel, err / std::fabs(an[i]));
    }
    out.push_back(r);
  }
  return out;
}

int cmd_gradcheck(const Args& a) {
  const int H = static_cast<int>(a.num("height", 6)), W = static_cast<int>(a.num("width", 7));
  const int N = static_cast<int>(a.num("state-dim", 4));
  Problem p = random_problem(1, H, W, N, static_cast<uint64_t>(a.num("seed", 0)));
  // every component of every group by default (as gradcheck.cpp); --samples caps it
  auto rep = gradcheck(p, static_cast<int>(a.num("samples", 1 << 20)), 1e-6);
  bool ok = true;
  std::printf("{\"command\": \"gradcheck\", \"height\": %d, \"width\": %d, \"state_dim\": %d, \"groups\": {", H, W, N);
  for (size_t k = 0; k < rep.size(); ++k) {
    // the reference's finite-difference gate (test_backward.cpp:40-45): rel <= 1e-6 and
    // abs <= 1e-9 on the small components
    const bool g_ok = rep[k].max_rel <= 1e-6 && rep[k].max_abs <= 1e-9;
    ok = ok && g_ok;
    std::printf("%s\"%s\": {\"max_rel\": %.3e, \"max_abs_small\": %.3e}", k ? ", " : "", rep[k].name, rep[k].max_rel,
                rep[k].max_abs);
  }
  std::printf("}, \"pass\": %s}\n", ok ? "true" : "false");
  return ok ? 0 : 1;
}

int cmd_verify(const Args& a) {
  if (!a.has("sizes")) usage("verify needs --sizes");
  const int dtype = dtype_of(a);
  const int N = static_cast<int>(a.num("state-dim", 16));
  std::vector<std::string> seeds = split(a.str("seeds", "0"), ',');
  bool ok = true;
  for (const std::string& sz : split(a.str("sizes"), ',')) {
    int H = 0, W = 0;
    if (std::sscanf(sz.c_str(), "%dx%d", &H, &W) != 2 || H < 1 || W < 1) usage(("bad size " + sz).c_str());
    for (const std::string& sd : seeds) {
      const uint64_t seed = std::strtoull(sd.c_str(), nullptr, 10);
      Problem p = random_problem(2, H, W, N, seed);
      const size_t n = 2 * static_cast<size_t>(H) * W;
      // reference: the naive 2D operator in f64 (an independent algorithm)
      DevProblem ref(p, SCAN2D_F64, 16);
      Dev yr(8 * n);
      forward(ref, Variant::Naive, yr);
      const std::vector<double> y_ref = down<double>(yr, n);
      // tiled in the requested dtype
      DevProblem dp(p, dtype, 16);
      Dev y(dp.es * n);
      forward(dp, Variant::Tiled, y);
      const std::vector<double> y0 = dtype == SCAN2D_F64 ? down<double>(y, n) : down<float>(y, n);
      const double err = rel_error(y0, y_ref);
      // tile invariance (test_engine.cpp): the reference tile T only shapes the
      // CarryState emission -- y must be the same bits for every T
      std::vector<double> yt0;
      bool tile_inv = true;
      for (int T : {1, 5, 16, 64}) {
        DevProblem dt(p, dtype, T);
        Dev yt(dt.es * n);
        const size_t kh = (H + T - 1) / T, kw = (W + T - 1) / T;
        Dev ph(dt.es * 2 * kh * kw * T * N), pv(dt.es * 2 * kh * kw * T * N);
        forward(dt, Variant::Tiled, yt, nullptr, &ph, &pv);
        std::vector<double> yh = dtype == SCAN2D_F64 ? down<double>(yt, n) : down<float>(yt, n);
        if (yt0.empty())
          yt0 = yh;
        else
          tile_inv = tile_inv && yh == yt0;
      }
      tile_inv = tile_inv && rel_error(yt0, y0) <= (dtype == SCAN2D_F64 ? 1e-12 : 1e-4);
      const double gate = dtype == SCAN2D_F64 ? 1e-12 : 1e-4;
      const bool c_ok = err <= gate && tile_inv;
      ok = ok && c_ok;
      std::printf("{\"command\": \"verify\", \"size\": \"%dx%d\", \"seed\": %llu, \"state_dim\": %d, "
                  "\"dtype\": \"%s\", \"max_rel_error\": %.3e, \"tolerance\": %.0e, \"tile_invariant\": %s, "
                  "\"pass\": %s}\n",
                  H, W, static_cast<unsigned long long>(seed), N, dtype == SCAN2D_F64 ? "f64" : "f32", err, gate,
                  tile_inv ? "true" : "false", c_ok ? "true" : "false");
      std::fflush(stdout);
      if (!c_ok) return 1;  // first failing case (SPEC.md: nonzero exit with the first failure)
    }
  }
  return ok ? 0 : 1;
}

int cmd_bench(const Args& a) {
  const Variant v = parse_variant(a.str("variant", "tiled2d"));
  const int H = static_cast<int>(a.num("height", 56)), W = static_cast<int>(a.num("width", 56));
  const int N = static_cast<int>(a.num("state-dim", 16)), T = static_cast<int>(a.num("tile", 16));
  const int reps = static_cast<int>(a.num("reps", 20)), warm = static_cast<int>(a.num("warmup", 3));
  const int64_t S = a.num("batch", 1);
  const bool bwd = a.has("backward");
  if (bwd && v != Variant::Tiled) usage("--backward: tiled2d only (the comparators have no backward)");
  const int dtype = dtype_of(a);
  Problem p = random_problem(S, H, W, N, 1234);
  DevProblem dp(p, dtype, T);
  check_rc(scan2d_check_desc(&dp.desc), "descriptor");
  const scan2d_desc& d = dp.desc;
  const size_t n = static_cast<size_t>(S) * H * W;
  Dev y(dp.es * n), res(bwd ? scan2d_residual_bytes(&d) : 16);
  Dev wsf(v == Variant::Tiled ? scan2d_workspace_bytes(&d, SCAN2D_OP_FWD)
                              : scan2d_comparator_workspace_bytes(
                                    &d, v == Variant::Naive ? SCAN2D_VARIANT_NAIVE : SCAN2D_VARIANT_FLAT1D));
  Dev wsb(bwd ? scan2d_workspace_bytes(&d, SCAN2D_OP_BWD) : 16);
  Dev dx(bwd ? dp.es * n : 16), dz(bwd ? dp.es * n : 16), dA(bwd ? dp.es * S * N : 16),
      dB(bwd ? dp.es * n * N : 16), dC(bwd ? dp.es * n * N : 16), dD(bwd ? dp.es * S : 16),
      db(bwd ? dp.es * S : 16);
  auto step = [&]() {
    if (v == Variant::Tiled) {
      check_rc(scan2d_forward(&d, dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, y.p, nullptr,
                              nullptr, bwd ? res.p : nullptr, wsf.p, wsf.n, nullptr),
               "scan2d_forward");
      if (bwd)
        check_rc(scan2d_backward(&d, dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, res.p, dp.dy.p,
                                 dx.p, dz.p, dA.p, dB.p, dC.p, dD.p, db.p, wsb.p, wsb.n, nullptr),
                 "scan2d_backward");
    } else {
      check_rc(scan2d_forward_variant(&d, v == Variant::Naive ? SCAN2D_VARIANT_NAIVE : SCAN2D_VARIANT_FLAT1D,
                                      dp.x.p, dp.z.p, dp.B.p, dp.C.p, dp.A.p, dp.D.p, dp.bias.p, y.p, wsf.p,
                                      wsf.n, nullptr),
               "scan2d_forward_variant");
    }
  };
  for (int i = 0; i < warm; ++i) step();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, nullptr));
  for (int i = 0; i < reps; ++i) step();
  CK(cudaEventRecord(e1, nullptr));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double per = ms * 1e-3 / reps;
  // reference counting model (memsim.cpp:45-46): fwd 2 HW + 2 HW N reads, HW writes;
  // bwd adds dy (read) and dx, dz, dB, dC (writes)
  const double hwS = static_cast<double>(n);
  const double reads = hwS * (2 + 2.0 * N) + (bwd ? hwS * (3 + 2.0 * N) : 0.0);
  const double writes = hwS + (bwd ? hwS * (2 + 2.0 * N) : 0.0);
  // flops per (cell, state): discretise 3, recurrences 4, readout 2 (forward); backward ~3x
  const double flops = hwS * N * 9.0 * (bwd ? 4.0 : 1.0);
  std::printf("{\"command\": \"bench\", \"variant\": \"%s\", \"height\": %d, \"width\": %d, \"state_dim\": %d, "
              "\"tile\": %d, \"dtype\": \"%s\", \"batch\": %lld, \"pass\": \"%s\", \"repetitions\": %d, "
              "\"warmup\": %d, \"wall_time_per_rep_s\": %.6e, \"throughput_maps_per_s\": %.6e, \"flops\": %.6e, "
              "\"mem_report\": {\"payload_reads\": %.0f, \"payload_writes\": %.0f, \"hbm_gbytes_per_s\": %.3f}}\n",
              a.str("variant", "tiled2d").c_str(), H, W, N, T, dtype == SCAN2D_F64 ? "f64" : "f32",
              static_cast<long long>(S), bwd ? "fwd+bwd" : "fwd", reps, warm, per, static_cast<double>(S) / per,
              flops, reads, writes, (reads + writes) * dp.es / per / 1e9);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage("missing subcommand");
  const std::string cmd = argv[1];
  if (cmd == "scan")
    return cmd_scan(parse(argc, argv, 2, {"input", "output", "variant", "tile", "state-dim", "seed", "dtype", "z",
                                          "b", "c", "a", "dskip", "bias", "threads"},
                          {}));
  if (cmd == "verify")
    return cmd_verify(parse(argc, argv, 2, {"sizes", "seeds", "dtype", "state-dim", "threads"}, {}));
  if (cmd == "gradcheck")
    return cmd_gradcheck(parse(argc, argv, 2, {"height", "width", "state-dim", "seed", "samples", "threads"}, {}));
  if (cmd == "bench")
    return cmd_bench(parse(argc, argv, 2, {"variant", "height", "width", "state-dim", "tile", "reps", "warmup",
                                           "batch", "dtype", "threads"},
                           {"backward"}));
  usage(("unknown subcommand " + cmd).c_str());
}
