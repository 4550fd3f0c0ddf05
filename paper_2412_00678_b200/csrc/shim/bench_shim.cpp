// bench_shim -- the drop-in path measured as a reference user sees it: S scans
// through the reference's own C++ API (scan2d::tiled_scan_2d_forward /
// tiled_scan_2d_backward, engine.hpp:88-102) with host Grid operands, served by
// libscan2d_engine_cuda.so (engine_shim.cpp) on the GPU.  The S scans are
// spread over P host threads in contiguous blocks, one call per scan -- the
// model.cpp:177 pattern the reference arm of bench.py times on the CPU.
// Compiled against the reference headers only (csrc/Makefile target `shim`).
//
// usage: bench_shim --scans S --height H --width W --state-dim N [--threads P]
//                   [--reps R] [--warmup K] [--forward-only]
// Prints one JSON line: seconds per pass (median), Gelem/s = S*H*W / pass.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <malloc.h>

#include "scan2d/engine.hpp"

using namespace scan2d;

namespace {

struct Gen {  // splitmix64 + Box-Muller (random_instance distribution)
  uint64_t s;
  explicit Gen(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  float normal() {
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * uniform()));
  }
};

struct Scan {
  Grid<float> x, dy;
  SelectiveInputs<float> in;
  ScanParams<float> pr;
};

Scan make_scan(int h, int w, int n, uint64_t seed) {
  Gen g(seed);
  auto grid = [&](int d) {
    std::vector<float> v(static_cast<size_t>(h) * w * d);
    for (auto& e : v) e = g.normal();
    return Grid<float>(h, w, d, std::move(v));
  };
  Scan s;
  s.x = grid(1);
  Grid<float> z = grid(1), b = grid(n), c = grid(n);
  s.in = SelectiveInputs<float>(std::move(z), std::move(b), std::move(c));
  std::vector<float> a(n);
  for (auto& e : a) e = static_cast<float>(-(0.05 + 0.9 * g.uniform()));
  const float dsk = g.normal();
  const float bias = static_cast<float>(g.uniform() - 0.5);
  s.pr = ScanParams<float>(std::move(a), dsk, bias);
  s.dy = grid(1);
  return s;
}

long arg(int argc, char** argv, const char* name, long dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return std::strtol(argv[i + 1], nullptr, 10);
  return dflt;
}
bool flag(int argc, char** argv, const char* name) {
  for (int i = 1; i < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return true;
  return false;
}

}  // namespace

int main(int argc, char** argv) {
  // The reference API returns fresh multi-megabyte vectors per call: keep freed
  // blocks in the heap instead of mmap / munmap per call (with many threads the
  // page faults serialise on the process's address-space lock).  Applied to
  // this driver only; --no-mallopt keeps glibc's defaults.
  if (!flag(argc, argv, "--no-mallopt")) {
    mallopt(M_MMAP_THRESHOLD, 1 << 30);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
  }
  const int S = static_cast<int>(arg(argc, argv, "--scans", 128));
  const int H = static_cast<int>(arg(argc, argv, "--height", 200));
  const int W = static_cast<int>(arg(argc, argv, "--width", 200));
  const int N = static_cast<int>(arg(argc, argv, "--state-dim", 16));
  const int T = static_cast<int>(arg(argc, argv, "--tile", 16));
  int P = static_cast<int>(arg(argc, argv, "--threads", std::thread::hardware_concurrency()));
  const int reps = static_cast<int>(arg(argc, argv, "--reps", 5));
  const int warm = static_cast<int>(arg(argc, argv, "--warmup", 2));
  const bool bwd = !flag(argc, argv, "--forward-only");
  P = std::max(1, std::min(P, S));
  std::vector<Scan> scans;
  scans.reserve(S);
  for (int s = 0; s < S; ++s) scans.push_back(make_scan(H, W, N, 1000 + s));
  const TileConfig tiles(H, W, T);
  double checksum = 0.0;
  auto pass = [&]() {
    std::vector<std::thread> pool;
    std::vector<double> part(P, 0.0);
    const int chunk = (S + P - 1) / P;
    for (int k = 0; k < P; ++k) {
      pool.emplace_back([&, k]() {
        for (int s = k * chunk; s < std::min(S, (k + 1) * chunk); ++s) {
          const Scan& sc = scans[s];
          auto f = tiled_scan_2d_forward(sc.x, sc.in, sc.pr, tiles, 1, nullptr, bwd);
          part[k] += f.y.data[0];
          if (bwd) {
            auto g = tiled_scan_2d_backward(f.saved, sc.dy, 1);
            part[k] += g.dbias;
          }
        }
      });
    }
    for (auto& t : pool) t.join();
    for (double v : part) checksum += v;
  };
  for (int i = 0; i < warm; ++i) pass();
  std::vector<double> secs;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    pass();
    secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(secs.begin(), secs.end());
  const double med = secs[secs.size() / 2];
  const double in_bytes = 4.0 * S * H * W * (3.0 + 2.0 * N + (bwd ? 1.0 : 0.0));
  const double out_bytes = 4.0 * S * H * W * (1.0 + (bwd ? 2.0 + 2.0 * N : 0.0));
  std::printf("{\"api\": \"reference C++ API (tiled_scan_2d_forward/backward) on libscan2d_engine_cuda.so\", "
              "\"scans\": %d, \"height\": %d, \"width\": %d, \"state_dim\": %d, \"tile\": %d, \"pass\": \"%s\", "
              "\"host_threads\": %d, \"reps\": %d, \"seconds_per_pass\": %.6f, \"gelem_per_s\": %.6f, "
              "\"h2d_bytes_per_pass\": %.0f, \"d2h_bytes_per_pass\": %.0f, \"checksum\": %.6e}\n",
              S, H, W, N, T, bwd ? "fwd+bwd" : "fwd", P, reps, med, S * double(H) * W / med / 1e9, in_bytes,
              out_bytes, checksum);
  return 0;
}
