/*
 * scan2d_oracle.h -- CPU parity oracle for the 2D selective scan.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the CUDA library,
 * the C-ABI, the C++ engine shim) may link or call this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it, and only as the checker.
 *
 * A plain-C restatement of the reference algorithm (arXiv 2412.00678 artifact
 * under /root/reference/proj).  Every function cites the reference lines it
 * follows.  Parity of this restatement is pinned in two ways:
 *   - against the reference library itself, built from its own sources into
 *     oracle/_ref/ by oracle/Makefile (tests/test_oracle.py), and
 *   - against golden vectors produced by that library and committed under
 *     tests/golden/ (tests/golden/make_golden.py).
 *
 * Layouts follow the reference Grid<T> (types.hpp:55-57): x, z, y, dy, dx, dz
 * are [H][W]; B, C, dB, dC are [H][W][N] with N fastest; A and dA are [N].
 */
#ifndef SCAN2D_ORACLE_H
#define SCAN2D_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* splitmix64 + Box-Muller generator, rng.hpp:11-61 */
typedef struct orc_rng {
  uint64_t state;
  double spare;
  int has_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
int orc_rng_uniform_int(orc_rng* r, int lo, int hi);

/* random_instance, fixtures.hpp:20-37.  Output buffers: x,z [h*w], B,C [h*w*n],
 * A [n], D, bias scalars. */
void orc_random_instance_f64(int h, int w, int n, uint64_t seed, double* x, double* z,
                             double* B, double* C, double* A, double* D, double* bias);
void orc_random_instance_f32(int h, int w, int n, uint64_t seed, float* x, float* z,
                             float* B, float* C, float* A, float* D, float* bias);
/* Rng(seed).fill_normal(v), rng.hpp:44-46 */
void orc_fill_normal_f64(uint64_t seed, size_t count, double* out);
void orc_fill_normal_f32(uint64_t seed, size_t count, float* out);

/* num::fast_expf, math.hpp:39-70 */
float orc_fast_expf(float x);

/* Sequential forward: discretize (reference.cpp:24-46) then scan_2d_sequential
 * (reference.cpp:70-114).  hh / hs (nullable) receive the horizontal and full
 * states [h][w][n]. */
void orc_fwd_f64(int h, int w, int n, const double* x, const double* z, const double* B,
                 const double* C, const double* A, double D, double bias, double* y,
                 double* hh, double* hs);
void orc_fwd_f32(int h, int w, int n, const float* x, const float* z, const float* B,
                 const float* C, const float* A, float D, float bias, float* y, float* hh,
                 float* hs);

/* CarryState (engine.hpp:29-46) rebuilt from sequential states with the edge
 * pass-through rule of engine.cpp:188-194, :217-220.  ph, pv: [kh][kw][t][n]. */
void orc_carries_f64(int h, int w, int n, int t, const double* hh, const double* hs,
                     double* ph, double* pv);
void orc_carries_f32(int h, int w, int n, int t, const float* hh, const float* hs,
                     float* ph, float* pv);

/* Backward: the chain rule of tiled_scan_2d_backward (engine.cpp:245-410) with
 * one tile covering the grid, i.e. full-grid reverse scans; scalar groups are
 * reduced row-major.  dA [n]; dD, dbias scalars. */
void orc_bwd_f64(int h, int w, int n, const double* x, const double* z, const double* B,
                 const double* C, const double* A, double D, double bias, const double* dy,
                 double* dx, double* dz, double* dA, double* dB, double* dC, double* dD,
                 double* dbias);
void orc_bwd_f32(int h, int w, int n, const float* x, const float* z, const float* B,
                 const float* C, const float* A, float D, float bias, const float* dy,
                 float* dx, float* dz, float* dA, float* dB, float* dC, float* dD,
                 float* dbias);

/* Batched layout of the C-ABI (include/scan2d_cuda.h): S scans, params of scan s
 * at index s % P, B/C of scan s at index s / G.  dA [P][n], dD/dbias [P],
 * dB/dC [S/G][h][w][n] accumulate in ascending scan order.  threads <= 1 runs
 * serially; otherwise scans are split over a std-thread-free pthread pool. */
void orc_fwd_batch_f64(int64_t S, int P, int G, int h, int w, int n, const double* x,
                       const double* z, const double* B, const double* C, const double* A,
                       const double* D, const double* bias, double* y, int threads);
void orc_fwd_batch_f32(int64_t S, int P, int G, int h, int w, int n, const float* x,
                       const float* z, const float* B, const float* C, const float* A,
                       const float* D, const float* bias, float* y, int threads);
void orc_bwd_batch_f64(int64_t S, int P, int G, int h, int w, int n, const double* x,
                       const double* z, const double* B, const double* C, const double* A,
                       const double* D, const double* bias, const double* dy, double* dx,
                       double* dz, double* dA, double* dB, double* dC, double* dD,
                       double* dbias);
void orc_bwd_batch_f32(int64_t S, int P, int G, int h, int w, int n, const float* x,
                       const float* z, const float* B, const float* C, const float* A,
                       const float* D, const float* bias, const float* dy, float* dx,
                       float* dz, float* dA, float* dB, float* dC, float* dD, float* dbias);

#ifdef __cplusplus
}
#endif

#endif /* SCAN2D_ORACLE_H */
