// Test infrastructure: the reference's gradcheck (gradcheck.cpp) on the CUDA
// engine shim, per group, after a prefix of saved forwards of other shapes
// (the order the reference suites run in).
#include <cstdio>
#include <cstdlib>

#include "scan2d/engine.hpp"
#include "scan2d/fixtures.hpp"
#include "scan2d/gradcheck.hpp"

using namespace scan2d;

static void fwd(int h, int w, int n, int t, std::uint64_t seed, bool bwd) {
  auto inst = random_instance<double>(h, w, n, seed);
  auto f = tiled_scan_2d_forward(inst.x, inst.inputs, inst.params, TileConfig(h, w, t));
  if (bwd) tiled_scan_2d_backward(f.saved, Grid<double>::zeros(h, w));
}

int main() {
  const int skip = std::getenv("PREFIX") ? std::atoi(std::getenv("PREFIX")) : 99;
  const int pre[][5] = {{33, 29, 6, 8, 0}, {33, 29, 6, 8, 0}, {33, 29, 6, 8, 0}, {33, 29, 6, 8, 0},
                        {9, 9, 2, 4, 0},   {16, 12, 3, 4, 0}, {5, 6, 3, 2, 1},   {7, 4, 2, 3, 1}};
  int k = 0;
  for (auto& p : pre)
    if (k++ < skip) fwd(p[0], p[1], p[2], p[3], 11 + k, p[4]);
  const int cases[][5] = {{5, 4, 3, 0, 3}, {4, 5, 2, 7, 1}, {4, 5, 2, 7, 2}, {4, 5, 2, 7, 6}};
  for (auto& c : cases) {
    auto r = gradcheck(c[0], c[1], c[2], static_cast<std::uint64_t>(c[3]), 1e-6, c[4]);
    std::printf("H=%d W=%d N=%d seed=%d T=%d:", c[0], c[1], c[2], c[3], c[4]);
    for (auto& g : r.groups) std::printf(" %s %.2e/%.2e", g.name.c_str(), g.max_rel, g.max_abs_small);
    std::printf("\n");
  }
  return 0;
}
