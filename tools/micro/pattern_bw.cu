// Diagnostics (not part of the library): HBM bandwidth of the tile backward's
// ACCESS PATTERN with no arithmetic.  Geometry as scan2d_bwd_tile2_kernel at
// cfg2: S scans of H x W, N = 16, one warp per 16-column strip walking 4-row
// tiles bottom-up, 12-warp CTAs.  Per tile a warp reads B (8 B per lane per
// column, 4 rows x 1 KB), C (1 KB rows), x / z / dy (64 B rows) and writes
// dB, dC (1 KB rows) and dx, dz (64 B rows) -- 276 B per cell like the kernel.
// Variants (argv[1]): 0 = the kernel's instruction mix (LDG.64 B, LDG.128 C,
// STG.64 dB, STG.128 dC); 1 = every row moved with 16-byte accesses by all
// lanes (fully coalesced 512 B per instruction).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pattern_bw pattern_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int S = 128, H = 200, W = 200, N = 16, CW = 16, R = 4, NW = 12;

__global__ void __launch_bounds__(32 * NW, 1) pattern(const float* __restrict__ B, const float* __restrict__ C,
                                                     const float* __restrict__ x, const float* __restrict__ z,
                                                     const float* __restrict__ dy, float* __restrict__ dB,
                                                     float* __restrict__ dC, float* __restrict__ dx,
                                                     float* __restrict__ dz, int variant) {
  const int strips = (W + CW - 1) / CW;
  const int g = blockIdx.x * NW + threadIdx.x / 32;
  if (g >= S * strips) return;
  const int s = g / strips, c0 = (g % strips) * CW, ncols = min(CW, W - c0);
  const int lane = threadIdx.x & 31;
  const size_t HW = (size_t)H * W, WN = (size_t)W * N;
  float acc = 0.f;
  for (int r0 = (H / R - 1) * R; r0 >= 0; r0 -= R) {
    if (variant == 0) {
      // row lanes: r1 = lane / 8, q = lane % 8 (2 states each), 16 columns
      const int r1 = lane / 8, q = lane % 8;
      const size_t rb = (s * HW + (size_t)(r0 + r1) * W + c0) * N + q * 2;
      float2 bacc = make_float2(0.f, 0.f);
      for (int j = 0; j < ncols; ++j) {
        const float2 b = __ldcs(reinterpret_cast<const float2*>(B + rb + (size_t)j * N));
        bacc.x += b.x, bacc.y += b.y;
        __stcs(reinterpret_cast<float2*>(dB + rb + (size_t)j * N), make_float2(b.x * 2.f, bacc.y));
      }
      // column lanes: j = lane / 2, s2 = lane % 2 (8 states = 2 x 16 B)
      const int j2 = lane / 2, s2 = lane % 2;
      if (j2 < ncols)
        for (int r = 0; r < R; ++r) {
          const size_t cb = (s * HW + (size_t)(r0 + r) * W + c0 + j2) * N + s2 * 8;
          const float4 c_a = __ldcs(reinterpret_cast<const float4*>(C + cb));
          const float4 c_b = __ldcs(reinterpret_cast<const float4*>(C + cb + 4));
          __stcs(reinterpret_cast<float4*>(dC + cb), c_a);
          __stcs(reinterpret_cast<float4*>(dC + cb + 4), c_b);
          acc += c_a.x + c_b.w;
        }
      acc += bacc.x;
    } else {
      // every 1 KB row span of B / C / dB / dC: 64 units of 16 B over 32 lanes
      for (int r = 0; r < R; ++r) {
        const size_t base = (s * HW + (size_t)(r0 + r) * W + c0) * N;
        for (int u = lane; u < ncols * N / 4; u += 32) {
          const float4 b = __ldcs(reinterpret_cast<const float4*>(B + base) + u);
          const float4 c = __ldcs(reinterpret_cast<const float4*>(C + base) + u);
          __stcs(reinterpret_cast<float4*>(dB + base) + u, b);
          __stcs(reinterpret_cast<float4*>(dC + base) + u, c);
          acc += b.x + c.y;
        }
      }
    }
    // x / z / dy in, dx / dz out: 64 B rows
    if (lane < R * 4) {
      const int r = lane / 4, u = lane % 4;
      const size_t xb = s * HW + (size_t)(r0 + r) * W + c0;
      if (u * 4 < ncols) {
        const float4 a = __ldcs(reinterpret_cast<const float4*>(x + xb) + u);
        const float4 b = __ldcs(reinterpret_cast<const float4*>(z + xb) + u);
        const float4 c = __ldcs(reinterpret_cast<const float4*>(dy + xb) + u);
        __stcs(reinterpret_cast<float4*>(dx + xb) + u, make_float4(a.x + c.x, a.y, a.z, a.w));
        __stcs(reinterpret_cast<float4*>(dz + xb) + u, make_float4(b.x, b.y + acc, b.z, b.w));
      }
    }
  }
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const size_t HW = (size_t)H * W, big = (size_t)S * HW * N, small = (size_t)S * HW;
  float *B, *C, *dB, *dC, *x, *z, *dy, *dx, *dz;
  cudaMalloc(&B, big * 4); cudaMalloc(&C, big * 4); cudaMalloc(&dB, big * 4); cudaMalloc(&dC, big * 4);
  cudaMalloc(&x, small * 4); cudaMalloc(&z, small * 4); cudaMalloc(&dy, small * 4);
  cudaMalloc(&dx, small * 4); cudaMalloc(&dz, small * 4);
  cudaMemset(B, 0, big * 4); cudaMemset(C, 0, big * 4); cudaMemset(x, 0, small * 4);
  cudaMemset(z, 0, small * 4); cudaMemset(dy, 0, small * 4);
  const int strips = (W + CW - 1) / CW;
  const int ctas = (S * strips + NW - 1) / NW;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) pattern<<<ctas, 32 * NW>>>(B, C, x, z, dy, dB, dC, dx, dz, variant);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) pattern<<<ctas, 32 * NW>>>(B, C, x, z, dy, dB, dC, dx, dz, variant);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double bytes = 4.0 * S * HW * (5 + 4 * N);
  printf("variant %d: %.1f us, %.0f GB/s (algorithmic %.0f MB)  err=%s\n", variant, ms * 1e3, bytes / ms / 1e6,
         bytes / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
