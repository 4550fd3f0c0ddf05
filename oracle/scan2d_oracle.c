/*
 * scan2d_oracle.c -- CPU parity oracle for the 2D selective scan.
 *
 * TEST INFRASTRUCTURE ONLY (see scan2d_oracle.h).  Never linked into the
 * product library.  Restates the reference algorithm from
 * /root/reference/proj (cited file:line per function); pinned against the
 * reference library built into oracle/_ref/ and against tests/golden/.
 *
 * Compiled with -ffp-contract=off: every fused multiply-add below is an
 * explicit fma()/fmaf() exactly where the reference calls std::fma.
 */
#include "scan2d_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->has_spare = 0;
}

/* rng.hpp:22-27 (splitmix64) */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:30 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:32.  The reference is built with GCC's default -ffp-contract=fast on
 * an FMA target (x86-64-v3), which contracts lo + (hi - lo) * u into one fma. */
static double orc_rng_uniform_lohi(orc_rng* r, double lo, double hi) {
  return fma(hi - lo, orc_rng_uniform(r), lo);
}

/* rng.hpp:35-37 */
int orc_rng_uniform_int(orc_rng* r, int lo, int hi) {
  return lo + (int)(orc_rng_next(r) % (uint64_t)(hi - lo + 1));
}

/* rng.hpp:39-52 (Box-Muller with one spare) */
double orc_rng_normal(orc_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  if (u1 < 1e-300) u1 = 1e-300;
  double rad = sqrt(-2.0 * log(u1));
  double t = 6.283185307179586 * u2;
  r->spare = rad * sin(t);
  r->has_spare = 1;
  return rad * cos(t);
}

void orc_fill_normal_f64(uint64_t seed, size_t count, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (size_t k = 0; k < count; ++k) out[k] = orc_rng_normal(&r);
}

void orc_fill_normal_f32(uint64_t seed, size_t count, float* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (size_t k = 0; k < count; ++k) out[k] = (float)orc_rng_normal(&r);
}

/* fixtures.hpp:20-37: x, z, B, C ~ N(0,1) in that order, then A ~ -U(0.05,0.95),
 * then D ~ N(0,1), bias ~ U(-0.5,0.5).  Drawn in double, cast per element. */
#define ORC_DEFINE_INSTANCE(T, SUF)                                                     \
  void orc_random_instance_##SUF(int h, int w, int n, uint64_t seed, T* x, T* z, T* B, \
                                 T* C, T* A, T* D, T* bias) {                           \
    orc_rng r;                                                                          \
    orc_rng_init(&r, seed);                                                             \
    const size_t hw = (size_t)h * (size_t)w;                                            \
    for (size_t k = 0; k < hw; ++k) x[k] = (T)orc_rng_normal(&r);                       \
    for (size_t k = 0; k < hw; ++k) z[k] = (T)orc_rng_normal(&r);                       \
    for (size_t k = 0; k < hw * (size_t)n; ++k) B[k] = (T)orc_rng_normal(&r);           \
    for (size_t k = 0; k < hw * (size_t)n; ++k) C[k] = (T)orc_rng_normal(&r);           \
    for (int d = 0; d < n; ++d) A[d] = (T)(-orc_rng_uniform_lohi(&r, 0.05, 0.95));      \
    *D = (T)orc_rng_normal(&r);                                                         \
    *bias = (T)orc_rng_uniform_lohi(&r, -0.5, 0.5);                                     \
  }

ORC_DEFINE_INSTANCE(double, f64)
ORC_DEFINE_INSTANCE(float, f32)

/* --------------------------------------------------------------- math.hpp */

static inline float bits_to_float(uint32_t u) {
  float f;
  memcpy(&f, &u, sizeof f);
  return f;
}

/* math.hpp:39-70: degree-5 minimax exp with two-step 2^k scaling, flush below
 * -87.33654 */
float orc_fast_expf(float x) {
  const float kMaxIn = 88.02f;
  const float kMinIn = -87.33654f;
  const int flush = x < kMinIn;
  float xc = fminf(fmaxf(x, kMinIn), kMaxIn);
  const float kLog2e = 1.44269504088896341f;
  const float kLn2Hi = 0.693359375f;
  const float kLn2Lo = -2.12194440e-4f;
  float kf = floorf(fmaf(xc, kLog2e, 0.5f));
  float r = fmaf(kf, -kLn2Hi, xc);
  r = fmaf(kf, -kLn2Lo, r);
  float p = 1.9875691500e-4f;
  p = fmaf(p, r, 1.3981999507e-3f);
  p = fmaf(p, r, 8.3334519073e-3f);
  p = fmaf(p, r, 4.1665795894e-2f);
  p = fmaf(p, r, 1.6666665459e-1f);
  p = fmaf(p, r, 5.0000001201e-1f);
  float y = fmaf(p, r * r, r) + 1.0f;
  int k = (int)kf;
  int k0 = k >> 1;
  int k1 = k - k0;
  float s0 = bits_to_float((uint32_t)(k0 + 127) << 23);
  float s1 = bits_to_float((uint32_t)(k1 + 127) << 23);
  y = y * s0 * s1;
  return flush ? 0.0f : y;
}

/* math.hpp:14-21 softplus with the cutoff 20; :23-28 sigmoid; :72-73 apply_exp */
static inline double softplus_f64(double v) { return v > 20.0 ? v : log1p(exp(v)); }
static inline float softplus_f32(float v) { return v > 20.0f ? v : log1pf(expf(v)); }
static inline double sigmoid_f64(double v) {
  if (v >= 0.0) return 1.0 / (1.0 + exp(-v));
  double e = exp(v);
  return e / (1.0 + e);
}
static inline float sigmoid_f32(float v) {
  if (v >= 0.0f) return 1.0f / (1.0f + expf(-v));
  float e = expf(v);
  return e / (1.0f + e);
}
static inline double abar_f64(double delta, double a) { return exp(delta * a); }
static inline float abar_f32(float delta, float a) { return orc_fast_expf(delta * a); }

/* ------------------------------------------------ forward / carries / backward */

#define ORC_DEFINE_SCAN(T, SUF, FMA)                                                     \
  /* reference.cpp:24-46 discretize + reference.cpp:70-114 scan_2d_sequential */         \
  void orc_fwd_##SUF(int h, int w, int n, const T* x, const T* z, const T* B, const T* C,  \
                     const T* A, T D, T bias, T* y, T* hh_out, T* hs_out) {              \
    const size_t hw = (size_t)h * (size_t)w, hwn = hw * (size_t)n;                      \
    T* abar = (T*)malloc(sizeof(T) * hwn);                                               \
    T* bx = (T*)malloc(sizeof(T) * hwn);                                                 \
    T* hh = hh_out ? hh_out : (T*)malloc(sizeof(T) * hwn);                               \
    T* hs = hs_out ? hs_out : (T*)malloc(sizeof(T) * hwn);                               \
    for (size_t c = 0; c < hw; ++c) {                                                    \
      const T delta = softplus_##SUF(z[c] + bias);                                       \
      for (int d = 0; d < n; ++d) {                                                      \
        abar[c * n + d] = abar_##SUF(delta, A[d]);                                       \
        bx[c * n + d] = (delta * B[c * n + d]) * x[c];                                   \
      }                                                                                  \
    }                                                                                    \
    for (int i = 0; i < h; ++i)                                                          \
      for (int j = 0; j < w; ++j) {                                                      \
        const size_t base = ((size_t)i * w + j) * n;                                     \
        for (int d = 0; d < n; ++d) {                                                    \
          const T left = j > 0 ? hh[base - n + d] : (T)0;                                \
          hh[base + d] = FMA(abar[base + d], left, bx[base + d]);                        \
        }                                                                                \
      }                                                                                  \
    for (int i = 0; i < h; ++i)                                                          \
      for (int j = 0; j < w; ++j) {                                                      \
        const size_t base = ((size_t)i * w + j) * n;                                     \
        T acc = 0;                                                                       \
        for (int d = 0; d < n; ++d) {                                                    \
          const T up = i > 0 ? hs[base - (size_t)w * n + d] : (T)0;                      \
          const T hv = FMA(abar[base + d], up, hh[base + d]);                            \
          hs[base + d] = hv;                                                             \
          acc = FMA(C[base + d], hv, acc);                                               \
        }                                                                                \
        y[(size_t)i * w + j] = FMA(D, x[(size_t)i * w + j], acc);                        \
      }                                                                                  \
    free(abar);                                                                          \
    free(bx);                                                                            \
    if (!hh_out) free(hh);                                                               \
    if (!hs_out) free(hs);                                                               \
  }                                                                                      \
                                                                                         \
  /* engine.hpp:29-46 slot layout; engine.cpp:188-194 / :217-220 pass-through */         \
  void orc_carries_##SUF(int h, int w, int n, int t, const T* hh, const T* hs, T* ph,     \
                         T* pv) {                                                        \
    const int kh = (h + t - 1) / t, kw = (w + t - 1) / t;                                \
    for (int ih = 0; ih < kh; ++ih)                                                      \
      for (int iw = 0; iw < kw; ++iw) {                                                  \
        const size_t slot = ((size_t)ih * kw + iw) * (size_t)t * n;                      \
        const int jl = (iw + 1) * t < w ? (iw + 1) * t - 1 : w - 1;                      \
        const int il = (ih + 1) * t < h ? (ih + 1) * t - 1 : h - 1;                      \
        for (int rr = 0; rr < t; ++rr) {                                                 \
          const int gi = ih * t + rr;                                                    \
          for (int d = 0; d < n; ++d)                                                    \
            ph[slot + (size_t)rr * n + d] =                                              \
                gi < h ? hh[((size_t)gi * w + jl) * n + d] : (T)0;                       \
        }                                                                                \
        for (int cc = 0; cc < t; ++cc) {                                                 \
          const int gj = iw * t + cc;                                                    \
          for (int d = 0; d < n; ++d)                                                    \
            pv[slot + (size_t)cc * n + d] =                                              \
                gj < w ? hs[((size_t)il * w + gj) * n + d] : (T)0;                       \
        }                                                                                \
      }                                                                                  \
  }                                                                                      \
                                                                                         \
  /* engine.cpp:276-400 with one tile covering the grid, reduction row-major */          \
  void orc_bwd_##SUF(int h, int w, int n, const T* x, const T* z, const T* B, const T* C,  \
                     const T* A, T D, T bias, const T* dy, T* dx, T* dz, T* dA, T* dB,     \
                     T* dC, T* dD, T* dbias) {                                           \
    const size_t hw = (size_t)h * (size_t)w, hwn = hw * (size_t)n;                      \
    T* delta = (T*)malloc(sizeof(T) * hw);                                               \
    T* abar = (T*)malloc(sizeof(T) * hwn);                                               \
    T* hh = (T*)malloc(sizeof(T) * hwn);                                                 \
    T* hs = (T*)malloc(sizeof(T) * hwn);                                                 \
    T* gs = (T*)malloc(sizeof(T) * hwn);                                                 \
    T* gh = (T*)malloc(sizeof(T) * hwn);                                                 \
    T* work = (T*)malloc(sizeof(T) * (size_t)w * n);                                     \
    T* right = (T*)malloc(sizeof(T) * (size_t)n);                                        \
    T* yscratch = (T*)malloc(sizeof(T) * hw);                                            \
    for (size_t c = 0; c < hw; ++c) {                                                    \
      delta[c] = softplus_##SUF(z[c] + bias);                                            \
      for (int d = 0; d < n; ++d) abar[c * n + d] = abar_##SUF(delta[c], A[d]);          \
    }                                                                                    \
    /* scans 1 + 2 (engine.cpp:294-302): the forward states */                           \
    orc_fwd_##SUF(h, w, n, x, z, B, C, A, D, bias, yscratch, hh, hs);                    \
    /* scan 3, reverse vertical (engine.cpp:304-327): G = fma(C, dy, a_below*G_below) */ \
    for (size_t k = 0; k < (size_t)w * n; ++k) work[k] = 0;                              \
    for (int i = h - 1; i >= 0; --i)                                                     \
      for (int j = 0; j < w; ++j) {                                                      \
        const size_t cell = (size_t)i * w + j, base = cell * n;                          \
        T* dn = work + (size_t)j * n;                                                    \
        for (int d = 0; d < n; ++d) {                                                    \
          const T gval = FMA(C[base + d], dy[cell], dn[d]);                              \
          gs[base + d] = gval;                                                           \
          dn[d] = abar[base + d] * gval;                                                 \
        }                                                                                \
      }                                                                                  \
    /* scan 4, reverse horizontal (engine.cpp:329-353): Gh = G + a_right*Gh_right */     \
    for (int i = 0; i < h; ++i) {                                                        \
      for (int d = 0; d < n; ++d) right[d] = 0;                                          \
      for (int j = w - 1; j >= 0; --j) {                                                 \
        const size_t base = ((size_t)i * w + j) * n;                                     \
        for (int d = 0; d < n; ++d) {                                                    \
          const T gval = gs[base + d] + right[d];                                        \
          gh[base + d] = gval;                                                           \
          right[d] = abar[base + d] * gval;                                              \
        }                                                                                \
      }                                                                                  \
    }                                                                                    \
    /* chain rule (engine.cpp:355-397) */                                                \
    for (int d = 0; d < n; ++d) dA[d] = 0;                                               \
    T dbias_t = 0, dd_t = 0;                                                             \
    for (int i = 0; i < h; ++i)                                                          \
      for (int j = 0; j < w; ++j) {                                                      \
        const size_t cell = (size_t)i * w + j, base = cell * n;                          \
        const T dyv = dy[cell], xv = x[cell], dv = delta[cell];                          \
        const T sig = sigmoid_##SUF(z[cell] + bias);                                     \
        T ddelta = 0, sum_ghor_b = 0;                                                    \
        for (int d = 0; d < n; ++d) {                                                    \
          const T hh_left = j > 0 ? hh[base - n + d] : (T)0;                             \
          const T h_up = i > 0 ? hs[base - (size_t)w * n + d] : (T)0;                    \
          const T gver = gs[base + d], ghr = gh[base + d];                               \
          const T dabar = FMA(ghr, hh_left, gver * h_up);                                \
          const T av = abar[base + d];                                                   \
          dA[d] = FMA(dabar, dv * av, dA[d]);                                            \
          ddelta = FMA(dabar, av * A[d], ddelta);                                        \
          ddelta = FMA(ghr, B[base + d] * xv, ddelta);                                   \
          dB[base + d] = ghr * (dv * xv);                                                \
          dC[base + d] = dyv * hs[base + d];                                             \
          sum_ghor_b = FMA(ghr, B[base + d], sum_ghor_b);                                \
        }                                                                                \
        dx[cell] = FMA(D, dyv, dv * sum_ghor_b);                                         \
        dz[cell] = ddelta * sig;                                                         \
        dbias_t += ddelta * sig; /* product shared with dz: not contracted (:393-394) */   \
        dd_t = FMA(dyv, xv, dd_t);           /* contracted += (engine.cpp:395) */        \
      }                                                                                  \
    *dD = dd_t;                                                                          \
    *dbias = dbias_t;                                                                    \
    free(delta);                                                                         \
    free(abar);                                                                          \
    free(hh);                                                                            \
    free(hs);                                                                            \
    free(gs);                                                                            \
    free(gh);                                                                            \
    free(work);                                                                          \
    free(right);                                                                         \
    free(yscratch);                                                                      \
  }

ORC_DEFINE_SCAN(double, f64, fma)
ORC_DEFINE_SCAN(float, f32, fmaf)

/* ------------------------------------------------------------ batched layout */

typedef struct {
  int64_t s0, s1;
  int P, G, h, w, n, dbl;
  const void *x, *z, *B, *C, *A, *D, *bias;
  void* y;
} orc_fwd_job;

static void* orc_fwd_worker(void* arg) {
  orc_fwd_job* j = (orc_fwd_job*)arg;
  const size_t hw = (size_t)j->h * (size_t)j->w, hwn = hw * (size_t)j->n;
  for (int64_t s = j->s0; s < j->s1; ++s) {
    const int64_t p = s % j->P, g = s / j->G;
    if (j->dbl) {
      orc_fwd_f64(j->h, j->w, j->n, (const double*)j->x + s * hw, (const double*)j->z + s * hw,
                  (const double*)j->B + g * hwn, (const double*)j->C + g * hwn,
                  (const double*)j->A + p * j->n, ((const double*)j->D)[p],
                  ((const double*)j->bias)[p], (double*)j->y + s * hw, NULL, NULL);
    } else {
      orc_fwd_f32(j->h, j->w, j->n, (const float*)j->x + s * hw, (const float*)j->z + s * hw,
                  (const float*)j->B + g * hwn, (const float*)j->C + g * hwn,
                  (const float*)j->A + p * j->n, ((const float*)j->D)[p],
                  ((const float*)j->bias)[p], (float*)j->y + s * hw, NULL, NULL);
    }
  }
  return NULL;
}

static void orc_fwd_batch(int64_t S, int P, int G, int h, int w, int n, int dbl, const void* x,
                          const void* z, const void* B, const void* C, const void* A,
                          const void* D, const void* bias, void* y, int threads) {
  if (threads < 1) threads = 1;
  if (threads > S) threads = (int)S;
  orc_fwd_job* jobs = (orc_fwd_job*)calloc((size_t)threads, sizeof(orc_fwd_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int64_t chunk = (S + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    orc_fwd_job* j = &jobs[t];
    j->s0 = t * chunk;
    j->s1 = (t + 1) * chunk < S ? (t + 1) * chunk : S;
    j->P = P; j->G = G; j->h = h; j->w = w; j->n = n; j->dbl = dbl;
    j->x = x; j->z = z; j->B = B; j->C = C; j->A = A; j->D = D; j->bias = bias; j->y = y;
  }
  if (threads == 1) {
    orc_fwd_worker(&jobs[0]);
  } else {
    for (int t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, orc_fwd_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  }
  free(jobs);
  free(tids);
}

void orc_fwd_batch_f64(int64_t S, int P, int G, int h, int w, int n, const double* x,
                       const double* z, const double* B, const double* C, const double* A,
                       const double* D, const double* bias, double* y, int threads) {
  orc_fwd_batch(S, P, G, h, w, n, 1, x, z, B, C, A, D, bias, y, threads);
}

void orc_fwd_batch_f32(int64_t S, int P, int G, int h, int w, int n, const float* x,
                       const float* z, const float* B, const float* C, const float* A,
                       const float* D, const float* bias, float* y, int threads) {
  orc_fwd_batch(S, P, G, h, w, n, 0, x, z, B, C, A, D, bias, y, threads);
}

#define ORC_DEFINE_BWD_BATCH(T, SUF)                                                      \
  void orc_bwd_batch_##SUF(int64_t S, int P, int G, int h, int w, int n, const T* x,      \
                           const T* z, const T* B, const T* C, const T* A, const T* D,    \
                           const T* bias, const T* dy, T* dx, T* dz, T* dA, T* dB, T* dC, \
                           T* dD, T* dbias) {                                             \
    const size_t hw = (size_t)h * (size_t)w, hwn = hw * (size_t)n;                       \
    const int64_t ngroups = S / G;                                                        \
    memset(dA, 0, sizeof(T) * (size_t)P * n);                                             \
    memset(dD, 0, sizeof(T) * (size_t)P);                                                 \
    memset(dbias, 0, sizeof(T) * (size_t)P);                                              \
    memset(dB, 0, sizeof(T) * (size_t)ngroups * hwn);                                     \
    memset(dC, 0, sizeof(T) * (size_t)ngroups * hwn);                                     \
    T* tA = (T*)malloc(sizeof(T) * (size_t)n);                                            \
    T* tB = (T*)malloc(sizeof(T) * hwn);                                                  \
    T* tC = (T*)malloc(sizeof(T) * hwn);                                                  \
    for (int64_t s = 0; s < S; ++s) {                                                     \
      const int64_t p = s % P, g = s / G;                                                 \
      T tD, tbias;                                                                        \
      orc_bwd_##SUF(h, w, n, x + s * hw, z + s * hw, B + g * hwn, C + g * hwn, A + p * n, \
                    D[p], bias[p], dy + s * hw, dx + s * hw, dz + s * hw, tA, tB, tC, &tD,  \
                    &tbias);                                                              \
      for (int d = 0; d < n; ++d) dA[p * n + d] += tA[d];                                 \
      dD[p] += tD;                                                                        \
      dbias[p] += tbias;                                                                  \
      for (size_t k = 0; k < hwn; ++k) {                                                  \
        dB[g * hwn + k] += tB[k];                                                         \
        dC[g * hwn + k] += tC[k];                                                         \
      }                                                                                   \
    }                                                                                     \
    free(tA);                                                                             \
    free(tB);                                                                             \
    free(tC);                                                                             \
  }

ORC_DEFINE_BWD_BATCH(double, f64)
ORC_DEFINE_BWD_BATCH(float, f32)
