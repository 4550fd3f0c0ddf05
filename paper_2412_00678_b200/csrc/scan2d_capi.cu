// scan2d_capi.cu -- C-ABI entry points (include/scan2d_cuda.h): descriptor
// validation, launch planning, workspace / residual carving, kernel launches.
//
// Validation mirrors require_shapes (proj/src/engine.cpp:21-30) and the tile
// check (:163-164); the backward's stale-state check mirrors engine.cpp:248-249.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <initializer_list>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <cstdint>
#include <cstring>

#include "../../include/scan2d_cuda.h"
#include "scan2d_launch.h"

using s2d::Args;
using s2d::Plan;

// scan2d_groups.cu: state dimensions above 128 as passes over state groups
size_t scan2d_groups_workspace_bytes(const scan2d_desc& d, int op);
size_t scan2d_groups_residual_bytes(const scan2d_desc& d);
int scan2d_groups_forward(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C,
                          const void* A, const void* Dskip, const void* bias, void* y, void* ph, void* pv,
                          void* residual, void* ws, size_t ws_bytes, cudaStream_t st);
int scan2d_groups_backward(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C,
                           const void* A, const void* Dskip, const void* bias, const void* residual,
                           const void* dy, void* dx, void* dz, void* dA, void* dB, void* dC, void* dDskip,
                           void* dbias, void* ws, size_t ws_bytes, cudaStream_t st);
constexpr int kMaxKernelN = 128;

namespace {

thread_local int g_last_launches = 0;

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t dtype_size(int dtype) { return dtype == SCAN2D_F64 ? sizeof(double) : sizeof(float); }

int check_desc(const scan2d_desc* d) {
  if (d == nullptr) return SCAN2D_EINVAL;
  if (d->num_scans < 1 || d->height < 1 || d->width < 1) return SCAN2D_EINVAL;
  if (d->state_dim < 1 || d->state_dim > SCAN2D_MAX_STATE_DIM) return SCAN2D_EINVAL;
  if (d->tile < 1) return SCAN2D_EINVAL;
  if (d->params_period < 1 || d->num_scans % d->params_period != 0) return SCAN2D_EINVAL;
  if (d->bc_group < 1 || d->num_scans % d->bc_group != 0) return SCAN2D_EINVAL;
  if (d->dtype != SCAN2D_F32 && d->dtype != SCAN2D_F64) return SCAN2D_EINVAL;
  if ((d->flags & ~(SCAN2D_FLAG_ACCURATE | SCAN2D_FLAG_GROUP_RED)) != 0) return SCAN2D_EINVAL;
  // N > 128 runs as passes over state groups of <= 128 (scan2d_groups.cu)
  return SCAN2D_OK;
}

// Geometry of one direction (see s2d::Geo).  N <= 128: SPL = 4 states per lane
// (float4), LPC = Np / 4 lanes per chunk; N <= 2 uses SPL = Np, LPC = 1.
// Tuning overrides (diagnostics / sweeps only): SCAN2D_FWD_J, SCAN2D_BWD_J,
// SCAN2D_FWD_STAGES, SCAN2D_BWD_STAGES, SCAN2D_BAND_ROWS.
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  if (v == nullptr || *v == 0) return dflt;
  const int x = std::atoi(v);
  return x > 0 ? x : dflt;
}

s2d::Geo make_geo(const scan2d_desc& d, bool bwd) {
  s2d::Geo g{};
  const int N = d.state_dim, W = d.width;
  const bool dbl = d.dtype == SCAN2D_F64;
  const int Np = next_pow2(N);
  g.spl = Np >= 4 ? 4 : Np;
  g.lpc = Np / g.spl;
  g.Np = Np;
  g.cpw = 32 / g.lpc;
  if (g.spl == 4)
    g.J = bwd ? 2 : 4;
  else
    g.J = bwd ? 4 : 8;
  if (dbl) g.J = std::min(g.J, 2);
  g.J = env_int(bwd ? "SCAN2D_BWD_J" : "SCAN2D_FWD_J", g.J);
  if (g.J != 1 && g.J != 2 && g.J != 4 && g.J != 8) g.J = 2;
  if (bwd && g.J > 4) g.J = 4;
  const int chunks = static_cast<int>(ceil_div(W, g.J));
  if (chunks <= g.cpw / 2) {
    g.cps = next_pow2(chunks);
    g.seg = g.cpw / g.cps;
  } else {
    g.cps = g.cpw;
    g.seg = 1;
  }
  g.colsw = g.cps * g.J;
  g.wreal = g.seg > 1 ? 1 : static_cast<int>(ceil_div(W, g.colsw));
  g.units = ceil_div(d.num_scans, g.seg) * g.wreal;
  g.stages = env_int(bwd ? "SCAN2D_BWD_STAGES" : "SCAN2D_FWD_STAGES", bwd ? 3 : 4);
  g.stages = std::max(2, std::min(8, g.stages));
  return g;
}

// Shared memory: pipeline stages, backward band storage, then the copy table.
// The table size depends on whether 16-byte copy units are legal (vec flags).
int finish_geo(s2d::Geo& g, const scan2d_desc& d, bool bwd, int K, bool xvec, bool bvec) {
  const bool dbl = d.dtype == SCAN2D_F64;
  const int es = static_cast<int>(dtype_size(d.dtype));
  g.stage_elems = dbl ? s2d::stage_elems<double>(g.colsw, g.Np, g.seg, bwd)
                      : s2d::stage_elems<float>(g.colsw, g.Np, g.seg, bwd);
  size_t elems = static_cast<size_t>(g.stages) * g.stage_elems;
  if (bwd) elems += dbl ? s2d::band_elems<double>(K, g.J, g.spl) : s2d::band_elems<float>(K, g.J, g.spl);
  g.table_off = static_cast<int>(elems);
  const int epv = 16 / es;
  const int ncols = std::min<int>(g.colsw, d.width);
  const int nx = s2d::stage_units_x(g.seg, ncols, xvec, epv);
  const int nbu = s2d::stage_units_b(g.seg, ncols, d.state_dim, bvec, epv);
  const size_t bytes = elems * es + static_cast<size_t>(nx + nbu) * 32 * sizeof(s2d::CopyEntry);
  if (bytes > 200 * 1024) return SCAN2D_EUNSUPPORTED;
  g.smem_bytes = static_cast<int>(bytes);
  return SCAN2D_OK;
}

// One plan serves both directions: the backward consumes the forward's
// residual (checkpoints every K rows, carries every Q columns).
// strip width of the tile-transpose forward = carry grid Q for N in {4,8,16,32}
int tile_cw() { return 16; }

// backward strip width: 16 columns (13-warp CTAs); 32-column strips (8-warp
// CTAs, fp32, SH = 2, N <= 16) measured slower on B200 -- SCAN2D_TILE_CWB=32
int tile_cw_bwd(const scan2d_desc& d, int sh) {
  const bool wide = d.dtype == SCAN2D_F32 && sh == 2 && d.state_dim <= 16;
  const int dflt = 16;
  const int v = env_int("SCAN2D_TILE_CWB", dflt);
  return (v == 16 || (v == 32 && wide)) ? v : dflt;
}

// states per row lane of the tile kernels (scan2d_tile2.cuh): SH = 2 for fp32
// (16 B operand registers per column), 1 for fp64.  It fixes the tile height
// R = 32 SH / N and so the checkpoint interval K: descriptor-level.
int tile_sh(const scan2d_desc& d) {
  const int dflt = d.dtype == SCAN2D_F64 ? 1 : 2;
  const int v = env_int("SCAN2D_TILE_SH", dflt);
  return (v == 1 || v == 2) && 32 * v / d.state_dim >= 1 ? v : dflt;
}

// N = 1 grids up to 128 columns run the row-sweep kernels (scan2d_rows1.cuh):
// a warp owns whole scans, so there are no horizontal carries; h is
// checkpointed every 4 rows.  The warp kernels (reference CarryState emission)
// accept the same residual layout.
bool rows1_shape(const scan2d_desc& d) {
  const int wmax = d.dtype == SCAN2D_F64 ? 64 : 128;  // 32 lanes x 16 bytes
  return d.state_dim == 1 && d.width <= wmax && env_int("SCAN2D_ROWS1", 1) == 1;
}

int make_plan(const scan2d_desc& d, Plan& p) {
  p = Plan{};
  p.b = make_geo(d, true);
  p.f = make_geo(d, false);
  p.pfd = env_int("SCAN2D_ROWS1_PFD", 6);  // measured: 6 rows ahead best on cfg3 / cfg4a (4..12, 1000 = off)
  // tile kernels: bulk L2 prefetch distance in tiles (1000 = off)
  p.pft_f = env_int("SCAN2D_TILE_PFF", 1000);
  p.pft_b = env_int("SCAN2D_TILE_PFB", 1);  // measured on cfg2: 1 tile ahead 0.308 vs 0.326 ms
  p.pf_mode = env_int("SCAN2D_TILE_PFMODE", 2);
  // tile staging: 3 (default) cp.async; 1: C rows by TMA bulk copies, 2: C + x / z / dy rows.  Measured on
  // cfg2 (fwd / bwd us): cp.async 160 / 304, TMA C 166 / 322, TMA all 177 / 319 -- one bulk copy per row
  // span issued by one lane serialises the issue; kept as an option (profiles/README.md).
  p.tma = env_int("SCAN2D_TILE_TMA", 3);
  if (p.tma > 2) p.tma = 0;
  if (p.pft_f >= 1000) p.pft_f = 0;
  if (p.pft_b >= 1000) p.pft_b = 0;
  // small problems (inputs well inside L2): the tile kernels prefetch every
  // tile of their strip into L2 at the start, so only the first tile waits on
  // DRAM (latency-bound launches: cfg1, Table 3's single maps)
  {
    const size_t es = dtype_size(d.dtype);
    const size_t in_bytes = es * static_cast<size_t>(d.num_scans) * d.height * d.width * (3 + 2 * d.state_dim);
    // (few tiles only: every row of every plane is one bulk prefetch, and a
    // long queue of them measured slower -- 56^2 / 200^2 single maps)
    p.pf_all = in_bytes <= (static_cast<size_t>(env_int("SCAN2D_PF_ALL_MB", 48)) << 20) &&
               d.height <= env_int("SCAN2D_PF_ALL_ROWS", 32);
  }
  if (rows1_shape(d)) {
    // row forward: 1 = line prefetches pfd rows ahead, 2 = bulk spans (SCAN2D_ROWS1_PFMODE)
    p.pf_mode = env_int("SCAN2D_ROWS1_PFMODE", 1);
    p.K = 4;
    p.nb = static_cast<int>(ceil_div(d.height, p.K));
    p.Q = d.width;
    p.nq = 0;
    p.warp_ok = p.f.wreal == 1 && p.b.wreal == 1;  // W <= 128 (fp32) / 64 (fp64): always
    return SCAN2D_OK;
  }
  p.K = std::min(env_int("SCAN2D_BAND_ROWS", 8), static_cast<int>(d.height));
  p.nb = static_cast<int>(ceil_div(d.height, p.K));
  const int N = d.state_dim;
  if (N == 4 || N == 8 || N == 16 || N == 32) {
    // Fixed 16-column carry grid, whatever forward kernel runs (the
    // tile-transpose kernel walks 16-column strips): the residual layout then
    // depends on the descriptor only, never on pointer alignment.
    p.Q = tile_cw();
    p.nq = static_cast<int>(ceil_div(d.width, p.Q)) - 1;
    // checkpoints every backward tile (R = 32 * SH / N rows)
    p.K = std::min(32 * tile_sh(d) / N, static_cast<int>(d.height));
    p.nb = static_cast<int>(ceil_div(d.height, p.K));
    // the warp kernels (fallback for unaligned operands, CarryState emission)
    // must put their column-group boundaries on the same 16-column grid
    auto widen = [&](s2d::Geo& g, int jmax) {
      while (g.wreal > 1 && (g.colsw % p.Q) != 0 && g.J < jmax) {
        g.J *= 2;
        g.colsw = g.cps * g.J;
        g.wreal = static_cast<int>(ceil_div(d.width, g.colsw));
        g.units = ceil_div(d.num_scans, g.seg) * g.wreal;
      }
    };
    widen(p.b, 4);
    widen(p.f, 8);
    p.warp_ok = !(p.b.wreal > 1 && (p.b.colsw % p.Q) != 0) &&
                !((p.Q % p.f.J) != 0 || (p.f.wreal > 1 && (p.f.colsw % p.Q) != 0));
    return SCAN2D_OK;
  }
  if (p.b.wreal > 1) {
    p.Q = p.b.colsw;
    p.nq = static_cast<int>(ceil_div(d.width, p.Q)) - 1;
    // forward warp boundaries and chunk starts must sit on the Q grid
    const bool ok = (p.Q % p.f.J) == 0 && (p.f.wreal == 1 || (p.f.colsw % p.Q) == 0);
    if (!ok) p.f = p.b, p.f.stages = 4;
  } else {
    p.Q = std::max(1, d.width);
    p.nq = 0;
  }
  if (p.f.wreal > 1 && p.nq == 0) {  // forward chains need carry slots too
    p.Q = p.f.colsw;
    p.nq = static_cast<int>(ceil_div(d.width, p.Q)) - 1;
  }
  p.warp_ok = 1;
  return SCAN2D_OK;
}

// 16-byte copy units are legal when every span of every row starts 16-byte
// aligned: base pointers aligned and all row / column offsets multiples of 16 B.
void vec_flags(const scan2d_desc& d, const Plan& p, const void* x, const void* z, const void* dy,
               const void* B, const void* C, const void* y, bool& xvec, bool& bvec, bool& yvec) {
  const int es = static_cast<int>(dtype_size(d.dtype));
  const int epv = 16 / es;
  auto al = [](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool cols_ok = (p.f.colsw % epv) == 0 && (p.b.colsw % epv) == 0;
  xvec = al(x) && al(z) && al(dy) && (d.width % epv) == 0 && cols_ok;
  bvec = al(B) && al(C) && next_pow2(d.state_dim) == d.state_dim &&
         (static_cast<int64_t>(d.width) * d.state_dim) % epv == 0 &&
         (static_cast<int64_t>(p.f.colsw) * d.state_dim) % epv == 0 &&
         (static_cast<int64_t>(p.b.colsw) * d.state_dim) % epv == 0;
  yvec = al(y) && (d.width % 4) == 0;
}

// Tile-transpose kernels (scan2d_tile2.cuh): N in {4, 8, 16, 32}, 16-byte
// aligned B / C rows, strips of 16 columns (the carry grid Q becomes 16); x / z
// / dy rows that are not 16-byte aligned are staged element by element.
// They also emit the reference CarryState (ph / pv) when asked.
bool use_tile_fwd(const scan2d_desc& d, bool xvec, bool bvec, bool emit) {
  (void)xvec;  // x / z / dy rows that are not 16-byte aligned take element copies (issue_cells)
  if (emit && env_int("SCAN2D_TILE_EMIT", 1) != 1) return false;  // (diagnostics: warp-kernel emission)
  const int N = d.state_dim;
  if (!(N == 4 || N == 8 || N == 16 || N == 32) || !bvec) return false;
  return env_int("SCAN2D_TILE_FWD", 1) == 1;
}

// J columns per lane: 16-byte loads when rows and pointers allow, else 8 / 4.
// Returns false when no J puts a row on <= 32 lanes (wide odd grids: warp kernels).
// The forward prefers J = 2 (more warps; measured faster at 56 and 28 columns),
// the backward J = 4 (more work per lane between its shuffle scans).
bool rows1_geo(s2d::Geo& g, const scan2d_desc& d, int align_bytes, bool bwd) {
  const int es = static_cast<int>(dtype_size(d.dtype));
  // preferred J first; wider / narrower ones when the width or alignment needs it
  const int pref = env_int(bwd ? "SCAN2D_ROWS1_JB" : "SCAN2D_ROWS1_JF", bwd ? 4 : 2);
  const int order[3] = {pref, pref == 4 ? 2 : 4, 1};
  int J = 0;
  for (int j : order) {
    if (d.width % j == 0 && j * es <= 16 && align_bytes % (j * es) == 0 && d.width / j <= 32) {
      J = j;
      break;
    }
  }
  if (J == 0) return false;
  g = s2d::Geo{};
  g.rows1 = 1;
  g.J = J;
  g.cps = std::max(8, next_pow2(d.width / J));  // lanes per scan (shuffle segment)
  g.seg = 32 / g.cps;                            // scans per warp
  g.wreal = 1;
  g.colsw = d.width;
  g.units = ceil_div(d.num_scans, g.seg);
  g.smem_bytes = 0;
  return true;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// largest power of two <= 16 dividing every address (x-like and B-like operands)
int ptr_align(std::initializer_list<const void*> ps) {
  int a = 16;
  for (const void* q : ps) {
    if (q == nullptr) continue;
    const uintptr_t v = reinterpret_cast<uintptr_t>(q);
    while (a > 1 && (v % a) != 0) a >>= 1;
  }
  return a;
}

int plan_with_flags(const scan2d_desc& d, Plan& p, bool xvec, bool bvec, bool emit = false,
                    int align_bytes = 16) {
  int rc = make_plan(d, p);
  if (rc != SCAN2D_OK) return rc;
  if (rows1_shape(d)) {
    s2d::Geo gb, gf;
    if (rows1_geo(gb, d, align_bytes, true) && rows1_geo(gf, d, align_bytes, false)) {
      p.b = gb;
      if (emit) return finish_geo(p.f, d, false, p.K, xvec, bvec);
      p.f = gf;
      return SCAN2D_OK;
    }
  }
  if (use_tile_fwd(d, xvec, bvec, emit)) {
    const bool dbl = d.dtype == SCAN2D_F64;
    s2d::Geo& g = p.f;
    g.tile = 1;
    g.spl = tile_sh(d);
    g.lpc = d.state_dim / g.spl;
    g.cpw = 32 / g.lpc;
    g.J = 1;
    g.Np = d.state_dim;
    g.seg = 1;
    g.cps = g.cpw;
    g.colsw = p.Q;
    g.wreal = static_cast<int>(ceil_div(d.width, p.Q));
    g.units = d.num_scans * g.wreal;
    g.stages = env_int("SCAN2D_TILE_STAGES", 1);
    const int el = dbl ? s2d::tile_elems<double>(d.state_dim, g.colsw, g.spl, g.stages, false)
                       : s2d::tile_elems<float>(d.state_dim, g.colsw, g.spl, g.stages, false);
    g.stage_elems = 0;
    g.table_off = 0;
    g.smem_bytes = static_cast<int>(static_cast<size_t>(el) * dtype_size(d.dtype));
    if (el < 0 || g.smem_bytes > 200 * 1024) return SCAN2D_EUNSUPPORTED;
    if (env_int("SCAN2D_TILE_BWD", 1) == 1) {
      s2d::Geo& b = p.b;
      b = g;
      b.stages = 1;
      b.spl = tile_sh(d);
      b.lpc = d.state_dim / b.spl;
      b.cpw = 32 / b.lpc;
      b.colsw = tile_cw_bwd(d, b.spl);
      b.wreal = static_cast<int>(ceil_div(d.width, b.colsw));
      b.units = d.num_scans * b.wreal;
      const int eb = dbl ? s2d::tile_elems<double>(d.state_dim, b.colsw, b.spl, 1, true)
                         : s2d::tile_elems<float>(d.state_dim, b.colsw, b.spl, 1, true);
      b.smem_bytes = static_cast<int>(static_cast<size_t>(eb) * dtype_size(d.dtype));
      if (eb < 0 || b.smem_bytes > 200 * 1024) return SCAN2D_EUNSUPPORTED;
      return SCAN2D_OK;
    }
    if (!p.warp_ok) return SCAN2D_EUNSUPPORTED;
    return finish_geo(p.b, d, true, p.K, xvec, bvec);
  }
  if (!p.warp_ok) return SCAN2D_EUNSUPPORTED;
  rc = finish_geo(p.f, d, false, p.K, xvec, bvec);
  if (rc != SCAN2D_OK) return rc;
  return finish_geo(p.b, d, true, p.K, xvec, bvec);
}

size_t slot_size(int dtype) { return dtype == SCAN2D_F64 ? 16 : 8; }

struct WsLayout {
  size_t ticket = 0, cnt = 0, hcarry = 0, rcarry = 0, part = 0, dbc = 0, total = 0;
};

// forward workspace: [ticket][hcarry (the forward's tagged carry chain)]
// backward workspace: [ticket][rcarry][part][per-scan dB, dC (G > 1)]
WsLayout ws_layout(const scan2d_desc& d, const Plan& p, int op) {
  const size_t es = dtype_size(d.dtype), ss = slot_size(d.dtype);
  const size_t S = static_cast<size_t>(d.num_scans);
  WsLayout L;
  size_t off = 0;
  L.ticket = off;
  off += kAlign;
  if (op == SCAN2D_OP_BWD) {  // per-scan finish counters, right after the ticket (one memset)
    L.cnt = off;
    off += align_up(sizeof(int) * S);
  }
  if (op == SCAN2D_OP_FWD) {
    L.hcarry = off;
    off += align_up(ss * S * p.nq * d.height * d.state_dim);
  } else {
    L.rcarry = off;
    off += align_up(ss * S * (p.b.wreal - 1) * d.height * d.state_dim);
    L.part = off;
    off += align_up(es * S * p.b.wreal * (d.state_dim + 2));
    if (d.bc_group > 1) {
      L.dbc = off;
      off += align_up(2 * es * S * d.height * d.width * d.state_dim);
    }
  }
  L.total = off;
  return L;
}

struct ResLayout {
  size_t ckpt = 0, hres = 0, total = 0;
};

ResLayout res_layout(const scan2d_desc& d, const Plan& p) {
  const size_t es = dtype_size(d.dtype);
  const size_t S = static_cast<size_t>(d.num_scans);
  ResLayout R;
  R.ckpt = 0;
  size_t off = align_up(es * S * (p.nb - 1) * d.width * d.state_dim);
  R.hres = off;
  off += align_up(es * S * p.nq * d.height * d.state_dim);
  R.total = std::max<size_t>(off, kAlign);
  return R;
}

// Runs before every chained launch, in stream order (captured CUDA graphs
// replay it too): resets the ticket and the per-scan finish counters, advances
// the device-side epoch, and -- when the header's magic does not match this
// launch's layout (fresh or re-purposed memory) -- clears the carry region so
// that no stale word can carry a valid tag.  Every CTA reads the magic before
// any writer exists (the main kernel records it), so all agree on `fresh`.
__global__ void scan2d_begin_kernel(s2d::WsHdr* h, uint32_t magic, uint32_t step, int* cnt, int64_t ncnt,
                                    uint4* clr, int64_t nclr) {
  const bool fresh = *reinterpret_cast<volatile uint32_t*>(&h->magic) != magic;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = tid; i < ncnt; i += nth) cnt[i] = 0;
  if (fresh)
    for (int64_t i = tid; i < nclr; i += nth) clr[i] = make_uint4(0u, 0u, 0u, 0u);
  s2d::griddep_launch_dependents();  // the chained kernel may launch now; it waits for our writes
  if (tid == 0) {
    h->ticket = 0;
    h->epoch = fresh ? 0u : (h->epoch % s2d::kTagSpan + step) % s2d::kTagSpan;
  }
}

uint32_t fnv(uint32_t hsh, uint64_t v) {
  for (int i = 0; i < 8; ++i) hsh = (hsh ^ static_cast<uint32_t>((v >> (8 * i)) & 0xff)) * 16777619u;
  return hsh;
}

// Layout hash of one chained launch: the descriptor, the op, and every plan
// field that decides where a carry slot lives.  Never 0 (cleared memory).
uint32_t layout_magic(const scan2d_desc& d, const Plan& p, int op, size_t carry_off, size_t carry_bytes) {
  uint32_t hsh = 2166136261u;
  for (uint64_t v : {static_cast<uint64_t>(d.num_scans), static_cast<uint64_t>(d.height),
                     static_cast<uint64_t>(d.width), static_cast<uint64_t>(d.state_dim),
                     static_cast<uint64_t>(d.tile), static_cast<uint64_t>(d.params_period),
                     static_cast<uint64_t>(d.bc_group), static_cast<uint64_t>(d.dtype),
                     static_cast<uint64_t>(op), static_cast<uint64_t>(p.f.wreal), static_cast<uint64_t>(p.b.wreal),
                     static_cast<uint64_t>(p.f.colsw), static_cast<uint64_t>(p.b.colsw),
                     static_cast<uint64_t>(p.f.tile), static_cast<uint64_t>(p.b.tile),
                     static_cast<uint64_t>(p.nq), static_cast<uint64_t>(p.Q),
                     static_cast<uint64_t>(carry_off), static_cast<uint64_t>(carry_bytes)})
    hsh = fnv(hsh, v);
  return hsh == 0 ? 1u : hsh;
}

// Host-side memory of the magic last enqueued per workspace address, so the
// common case (the same workspace reused with the same layout) launches a
// single-CTA begin kernel.  The device still checks the magic itself: a wrong
// guess (the caller overwrote the workspace) costs a slow single-CTA clear,
// never a wrong result.
struct MagicCache {
  static constexpr int kSlots = 64;
  std::mutex mu;
  const void* ws[kSlots] = {};
  uint32_t magic[kSlots] = {};
  int next = 0;
  bool seen_and_set(const void* w, uint32_t m) {
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < kSlots; ++i)
      if (ws[i] == w) {
        const bool hit = magic[i] == m;
        magic[i] = m;
        return hit;
      }
    ws[next] = w;
    magic[next] = m;
    next = (next + 1) % kSlots;
    return false;
  }
};
MagicCache g_magic_cache;

// Enqueue the begin kernel for a chained launch (see scan2d_begin_kernel).
cudaError_t launch_begin(s2d::WsHdr* h, uint32_t magic, int H, int* cnt, int64_t ncnt, void* clr,
                         size_t clr_bytes, cudaStream_t st) {
  uint32_t step = static_cast<uint32_t>(H) + 1u;
  if (step % s2d::kTagSpan == 0) ++step;
  step %= s2d::kTagSpan;
  const int64_t nclr = static_cast<int64_t>(clr_bytes / 16);
  const int threads = 256;
  int64_t blocks = 1;
  if (!g_magic_cache.seen_and_set(h, magic)) {
    const int64_t work = std::max<int64_t>(ncnt, nclr);
    blocks = std::max<int64_t>(1, std::min<int64_t>(2 * 148, (work + threads * 8 - 1) / (threads * 8)));
  }
  scan2d_begin_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(h, magic, step, cnt, ncnt,
                                                                          static_cast<uint4*>(clr), nclr);
  return cudaGetLastError();
}

int device_check() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SCAN2D_ECUDA;
  static int cached[64] = {0};  // 0 unknown, 1 ok, 2 unsupported
  if (dev < 0 || dev >= 64) return SCAN2D_ECUDA;
  if (cached[dev] == 0) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return SCAN2D_ECUDA;
    cached[dev] = (major == 10 && minor == 0) ? 1 : 2;
  }
  return cached[dev] == 1 ? SCAN2D_OK : SCAN2D_EUNSUPPORTED;
}

template <typename T>
void fill_common(Args<T>& a, const scan2d_desc& d, const Plan& p, const void* x, const void* z,
                 const void* B, const void* C, const void* A, const void* Dskip, const void* bias) {
  a.x = static_cast<const T*>(x);
  a.z = static_cast<const T*>(z);
  a.B = static_cast<const T*>(B);
  a.C = static_cast<const T*>(C);
  a.A = static_cast<const T*>(A);
  a.Dskip = static_cast<const T*>(Dskip);
  a.bias = static_cast<const T*>(bias);
  a.S = d.num_scans;
  a.H = d.height;
  a.W = d.width;
  a.N = d.state_dim;
  a.T_tile = d.tile;
  a.P = d.params_period;
  a.G = d.bc_group;
  a.acc = (d.flags & SCAN2D_FLAG_ACCURATE) != 0;
  a.plan = p;
}

template <typename T>
void set_flags(Args<T>& a, bool xvec, bool bvec, bool yvec) {
  a.xvec = xvec;
  a.bvec = bvec;
  a.yvec = yvec;
}

template <typename T>
int forward_impl(const scan2d_desc& d, const void* x, const void* z, const void* B, const void* C,
                 const void* A, const void* Dskip, const void* bias, void* y, void* ph, void* pv,
                 void* residual, void* ws, size_t ws_bytes, cudaStream_t stream,
                 const void* vtop = nullptr, void* vbot = nullptr, const int* lin = nullptr, int* lout = nullptr,
                 int lseq = 0) {
  g_last_launches = 0;
  if (!x || !z || !B || !C || !A || !Dskip || !bias || !y) return SCAN2D_EINVAL;
  if ((ph == nullptr) != (pv == nullptr)) return SCAN2D_EINVAL;
  int rc = device_check();
  if (rc != SCAN2D_OK) return rc;
  Plan p;
  rc = make_plan(d, p);
  if (rc != SCAN2D_OK) return rc;
  bool xvec, bvec, yvec;
  vec_flags(d, p, x, z, nullptr, B, C, y, xvec, bvec, yvec);
  rc = plan_with_flags(d, p, xvec, bvec, ph != nullptr, ptr_align({x, z, B, C, y}));
  if (rc != SCAN2D_OK) return rc;
  const WsLayout L = ws_layout(d, p, SCAN2D_OP_FWD);
  if (ws_bytes < L.total || ws == nullptr) return SCAN2D_ENOMEM;
  if (!al16(ws) || !al16(residual)) return SCAN2D_EINVAL;  // (header, carry slots, vector stores)
  unsigned char* w = static_cast<unsigned char*>(ws);
  Args<T> a{};
  fill_common(a, d, p, x, z, B, C, A, Dskip, bias);
  set_flags(a, xvec, bvec, yvec);
  a.y = static_cast<T*>(y);
  a.ph = static_cast<T*>(ph);
  a.pv = static_cast<T*>(pv);
  if ((vtop != nullptr || vbot != nullptr) && !p.f.tile) return SCAN2D_EUNSUPPORTED;
  a.vtop = static_cast<const T*>(vtop);
  a.vbot = static_cast<T*>(vbot);
  if ((lin != nullptr || lout != nullptr) && !p.f.tile) return SCAN2D_EUNSUPPORTED;
  a.link_in = lin;
  a.link_out = lout;
  a.link_seq = lseq;
  a.hdr = reinterpret_cast<s2d::WsHdr*>(w + L.ticket);
  a.ticket = &a.hdr->ticket;
  if (residual != nullptr) {
    const ResLayout R = res_layout(d, p);
    unsigned char* r = static_cast<unsigned char*>(residual);
    a.ckpt = reinterpret_cast<T*>(r + R.ckpt);
    a.hres = reinterpret_cast<T*>(r + R.hres);
  } else {
    a.ckpt = nullptr;
    a.hres = nullptr;
  }
  a.hcarry = reinterpret_cast<s2d::CarrySlot<T>*>(w + L.hcarry);
  int launches = 0;
  if (p.f.wreal > 1) {
    const size_t cb = L.total - L.hcarry;
    a.magic = layout_magic(d, p, SCAN2D_OP_FWD, L.hcarry, cb);
    if (launch_begin(a.hdr, a.magic, d.height, nullptr, 0, w + L.hcarry, cb, stream) != cudaSuccess)
      return SCAN2D_ECUDA;
    a.pdl = env_int("SCAN2D_PDL", 1) == 1;
    ++launches;
  }
  if (ph != nullptr) {
    const size_t kh = ceil_div(d.height, d.tile), kw = ceil_div(d.width, d.tile);
    const size_t cb = sizeof(T) * static_cast<size_t>(d.num_scans) * kh * kw * d.tile * d.state_dim;
    if (cudaMemsetAsync(ph, 0, cb, stream) != cudaSuccess) return SCAN2D_ECUDA;
    if (cudaMemsetAsync(pv, 0, cb, stream) != cudaSuccess) return SCAN2D_ECUDA;
  }
  if (s2d::launch_fwd<T>(a, stream) != cudaSuccess) return SCAN2D_ECUDA;
  g_last_launches = launches + 1;
  return SCAN2D_OK;
}

template <typename T>
int backward_impl(const scan2d_desc& d, const void* x, const void* z, const void* B,
                  const void* C, const void* A, const void* Dskip, const void* bias,
                  const void* residual, const void* dy, void* dx, void* dz, void* dA, void* dB,
                  void* dC, void* dDskip, void* dbias, void* ws, size_t ws_bytes,
                  cudaStream_t stream, const void* vtop = nullptr, const void* gbot = nullptr,
                  void* gtop = nullptr, const int* lin = nullptr, int* lout = nullptr, int lseq = 0) {
  g_last_launches = 0;
  if (residual == nullptr) return SCAN2D_ESTALE;
  if (!x || !z || !B || !C || !A || !Dskip || !bias || !dy) return SCAN2D_EINVAL;
  if (!dx || !dz || !dA || !dB || !dC || !dDskip || !dbias) return SCAN2D_EINVAL;
  int rc = device_check();
  if (rc != SCAN2D_OK) return rc;
  Plan p;
  rc = make_plan(d, p);
  if (rc != SCAN2D_OK) return rc;
  bool xvec, bvec, yvec;
  vec_flags(d, p, x, z, dy, B, C, nullptr, xvec, bvec, yvec);
  unsigned char* w = static_cast<unsigned char*>(ws);
  // the state-vector outputs take 16-byte stores (tile kernels: dB / dC, warp
  // kernels: the lane's 4 states); with G > 1 they go to the workspace first
  // (every workspace region starts at a multiple of 256 bytes from its base)
  const bool out_al = (reinterpret_cast<uintptr_t>(dB) & 15) == 0 && (reinterpret_cast<uintptr_t>(dC) & 15) == 0;
  const bool want_red = d.bc_group > 1 && (d.flags & SCAN2D_FLAG_GROUP_RED) != 0;
  // (G > 1: the per-scan gradients go to the workspace unless the tile kernel
  // reduces in place -- which kernel runs is known only after planning, so with
  // the reduction requested both destinations must allow 16-byte stores)
  const bool ws_al = (reinterpret_cast<uintptr_t>(w) & 15) == 0;
  const bool ovec = d.bc_group > 1 ? ws_al && (!want_red || out_al) : out_al;
  if (!ovec) bvec = false;  // no tile backward (it stores dB / dC with 8 / 16-byte vectors)
  rc = plan_with_flags(d, p, xvec, bvec, false, ptr_align({x, z, B, C, dy, dx, dz, dB, dC}));
  if (rc != SCAN2D_OK) return rc;
  // in-place group reductions: tile kernels only (the others keep the workspace path)
  const bool red = want_red && p.b.tile && p.b.colsw == 16;
  const WsLayout L = ws_layout(d, p, SCAN2D_OP_BWD);
  if (ws_bytes < L.total || ws == nullptr) return SCAN2D_ENOMEM;
  if (!al16(ws) || !al16(residual)) return SCAN2D_EINVAL;  // (header, carry slots, vector stores)
  const ResLayout R = res_layout(d, p);
  const unsigned char* r = static_cast<const unsigned char*>(residual);
  Args<T> a{};
  fill_common(a, d, p, x, z, B, C, A, Dskip, bias);
  set_flags(a, xvec, bvec, yvec);
  a.dy = static_cast<const T*>(dy);
  a.ovec = ovec;
  a.ckpt = const_cast<T*>(reinterpret_cast<const T*>(r + R.ckpt));
  a.hres = const_cast<T*>(reinterpret_cast<const T*>(r + R.hres));
  a.hcarry = nullptr;
  if ((vtop != nullptr || gbot != nullptr || gtop != nullptr) && !p.b.tile) return SCAN2D_EUNSUPPORTED;
  a.vtop = static_cast<const T*>(vtop);
  a.gbot = static_cast<const T*>(gbot);
  a.gtop = static_cast<T*>(gtop);
  if ((lin != nullptr || lout != nullptr) && !p.b.tile) return SCAN2D_EUNSUPPORTED;
  a.link_in = lin;
  a.link_out = lout;
  a.link_seq = lseq;
  a.dx = static_cast<T*>(dx);
  a.dz = static_cast<T*>(dz);
  T* dB_ps = static_cast<T*>(dB);
  T* dC_ps = static_cast<T*>(dC);
  const size_t hwn = static_cast<size_t>(d.height) * d.width * d.state_dim;
  const int64_t groups = d.num_scans / d.bc_group;
  if (red) {
    if (cudaMemsetAsync(dB, 0, groups * hwn * sizeof(T), stream) != cudaSuccess ||
        cudaMemsetAsync(dC, 0, groups * hwn * sizeof(T), stream) != cudaSuccess)
      return SCAN2D_ECUDA;
  } else if (d.bc_group > 1) {
    dB_ps = reinterpret_cast<T*>(w + L.dbc);
    dC_ps = dB_ps + static_cast<size_t>(d.num_scans) * hwn;
  }
  a.dB = dB_ps;
  a.dC = dC_ps;
  a.red = red;
  a.part = reinterpret_cast<T*>(w + L.part);
  a.rcarry = reinterpret_cast<s2d::CarrySlot<T>*>(w + L.rcarry);
  a.hdr = reinterpret_cast<s2d::WsHdr*>(w + L.ticket);
  a.ticket = &a.hdr->ticket;
  // per-scan parameters: the kernels finish dA / dbias / dD themselves (fixed
  // strip order, no extra launch); shared parameters need the reduction kernel
  const bool fuse = (p.b.tile || p.b.rows1) && d.params_period == d.num_scans;
  a.fuse = fuse;
  a.scan_cnt = reinterpret_cast<int*>(w + L.cnt);
  a.dA_out = static_cast<T*>(dA);
  a.dbias_out = static_cast<T*>(dbias);
  a.dD_out = static_cast<T*>(dDskip);
  int launches = 0;
  if (p.b.wreal > 1) {
    const size_t cb = L.part - L.rcarry;
    a.magic = layout_magic(d, p, SCAN2D_OP_BWD, L.rcarry, cb);
    if (launch_begin(a.hdr, a.magic, d.height, a.scan_cnt, d.num_scans, w + L.rcarry, cb, stream) !=
        cudaSuccess)
      return SCAN2D_ECUDA;
    a.pdl = env_int("SCAN2D_PDL", 1) == 1;
    ++launches;
  }
  if (s2d::launch_bwd<T>(a, stream) != cudaSuccess) return SCAN2D_ECUDA;
  ++launches;
  if (!fuse) {
    if (s2d::launch_reduce_params<T>(a.part, d.num_scans, p.b.wreal, d.params_period, d.state_dim,
                                     static_cast<T*>(dA), static_cast<T*>(dbias),
                                     static_cast<T*>(dDskip), stream) != cudaSuccess)
      return SCAN2D_ECUDA;
    ++launches;
  }
  if (d.bc_group > 1 && !red) {
    if (s2d::launch_reduce_group<T>(dB_ps, groups, d.bc_group, hwn, static_cast<T*>(dB), stream) !=
            cudaSuccess ||
        s2d::launch_reduce_group<T>(dC_ps, groups, d.bc_group, hwn, static_cast<T*>(dC), stream) !=
            cudaSuccess)
      return SCAN2D_ECUDA;
    launches += 2;
  }
  g_last_launches = launches;
  return SCAN2D_OK;
}

}  // namespace

extern "C" {

int scan2d_check_desc(const scan2d_desc* desc) { return check_desc(desc); }

// The kernel choice depends on pointer alignment (16-byte copy units), so the
// workspace covers every plan a call with this descriptor can take.
size_t scan2d_workspace_bytes(const scan2d_desc* desc, int op) {
  if (check_desc(desc) != SCAN2D_OK) return 0;
  if (desc->state_dim > kMaxKernelN) return scan2d_groups_workspace_bytes(*desc, op);
  size_t best = 0;
  bool any = false;
  for (int v = 0; v < 2; ++v) {
    Plan p;
    if (plan_with_flags(*desc, p, v == 1, v == 1) != SCAN2D_OK) continue;
    any = true;
    best = std::max(best, ws_layout(*desc, p, op).total);
  }
  return any ? best : 0;
}

size_t scan2d_residual_bytes(const scan2d_desc* desc) {
  if (check_desc(desc) != SCAN2D_OK) return 0;
  if (desc->state_dim > kMaxKernelN) return scan2d_groups_residual_bytes(*desc);
  Plan p;
  if (plan_with_flags(*desc, p, false, false) != SCAN2D_OK) return 0;
  return res_layout(*desc, p).total;
}

int scan2d_forward(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                   const void* C, const void* A, const void* Dskip, const void* bias, void* y,
                   void* ph, void* pv, void* residual, void* workspace, size_t workspace_bytes,
                   scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->state_dim > kMaxKernelN) {
    if (!x || !z || !B || !C || !A || !Dskip || !bias || !y || ((ph == nullptr) != (pv == nullptr)))
      return SCAN2D_EINVAL;
    return scan2d_groups_forward(*desc, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                                 workspace_bytes, st);
  }
  if (desc->dtype == SCAN2D_F64)
    return forward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                                workspace_bytes, st);
  return forward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                             workspace_bytes, st);
}

int scan2d_backward(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                    const void* C, const void* A, const void* Dskip, const void* bias,
                    const void* residual, const void* dy, void* dx, void* dz, void* dA,
                    void* dB, void* dC, void* dDskip, void* dbias, void* workspace,
                    size_t workspace_bytes, scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->state_dim > kMaxKernelN) {
    if (residual == nullptr) return SCAN2D_ESTALE;
    if (!x || !z || !B || !C || !A || !Dskip || !bias || !dy || !dx || !dz || !dA || !dB || !dC || !dDskip ||
        !dbias)
      return SCAN2D_EINVAL;
    return scan2d_groups_backward(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                                  dbias, workspace, workspace_bytes, st);
  }
  if (desc->dtype == SCAN2D_F64)
    return backward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB,
                                 dC, dDskip, dbias, workspace, workspace_bytes, st);
  return backward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC,
                              dDskip, dbias, workspace, workspace_bytes, st);
}

int scan2d_forward_band(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                        const void* C, const void* A, const void* Dskip, const void* bias,
                        const void* h_top, void* y, void* h_bottom, void* residual, void* workspace,
                        size_t workspace_bytes, scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  if (desc->state_dim > kMaxKernelN) return SCAN2D_EUNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->dtype == SCAN2D_F64)
    return forward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, y, nullptr, nullptr, residual, workspace,
                                workspace_bytes, st, h_top, h_bottom);
  return forward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, y, nullptr, nullptr, residual, workspace,
                             workspace_bytes, st, h_top, h_bottom);
}

int scan2d_backward_band(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                         const void* C, const void* A, const void* Dskip, const void* bias,
                         const void* h_top, const void* residual, const void* dy, const void* g_bottom,
                         void* dx, void* dz, void* dA, void* dB, void* dC, void* dDskip, void* dbias,
                         void* g_top, void* workspace, size_t workspace_bytes, scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  if (desc->state_dim > kMaxKernelN) return SCAN2D_EUNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->dtype == SCAN2D_F64)
    return backward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                                 dbias, workspace, workspace_bytes, st, h_top, g_bottom, g_top);
  return backward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                              dbias, workspace, workspace_bytes, st, h_top, g_bottom, g_top);
}

int scan2d_band_strips(const scan2d_desc* desc) {
  if (check_desc(desc) != SCAN2D_OK) return 0;
  return static_cast<int>(ceil_div(desc->width, tile_cw()));
}

int scan2d_forward_band_linked(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                               const void* C, const void* A, const void* Dskip, const void* bias,
                               const void* h_top, void* y, void* h_bottom, void* residual, const int* in_flags,
                               int* out_flags, int seq, void* workspace, size_t workspace_bytes,
                               scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  if (desc->state_dim > kMaxKernelN) return SCAN2D_EUNSUPPORTED;
  if (tile_cw_bwd(*desc, tile_sh(*desc)) != tile_cw()) return SCAN2D_EUNSUPPORTED;  // one strip grid both ways
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->dtype == SCAN2D_F64)
    return forward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, y, nullptr, nullptr, residual, workspace,
                                workspace_bytes, st, h_top, h_bottom, in_flags, out_flags, seq);
  return forward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, y, nullptr, nullptr, residual, workspace,
                             workspace_bytes, st, h_top, h_bottom, in_flags, out_flags, seq);
}

int scan2d_backward_band_linked(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                                const void* C, const void* A, const void* Dskip, const void* bias,
                                const void* h_top, const void* residual, const void* dy, const void* g_bottom,
                                void* dx, void* dz, void* dA, void* dB, void* dC, void* dDskip, void* dbias,
                                void* g_top, const int* in_flags, int* out_flags, int seq, void* workspace,
                                size_t workspace_bytes, scan2d_stream_t stream) {
  const int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  if (desc->state_dim > kMaxKernelN) return SCAN2D_EUNSUPPORTED;
  if (tile_cw_bwd(*desc, tile_sh(*desc)) != tile_cw()) return SCAN2D_EUNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (desc->dtype == SCAN2D_F64)
    return backward_impl<double>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                                 dbias, workspace, workspace_bytes, st, h_top, g_bottom, g_top, in_flags,
                                 out_flags, seq);
  return backward_impl<float>(*desc, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip, dbias,
                              workspace, workspace_bytes, st, h_top, g_bottom, g_top, in_flags, out_flags, seq);
}

int scan2d_ipc_export(const void* dev_ptr, unsigned char handle[64], uint64_t* offset) {
  if (dev_ptr == nullptr || handle == nullptr || offset == nullptr) return SCAN2D_EINVAL;
  // the driver's cuMemGetAddressRange through the runtime's entry-point query
  // (no link-time dependency on libcuda)
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (get_range == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      return SCAN2D_ECUDA;
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return SCAN2D_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return SCAN2D_ECUDA;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *offset = static_cast<uint64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return SCAN2D_OK;
}

int scan2d_ipc_open(const unsigned char handle[64], uint64_t offset, void** dev_ptr, void** base) {
  if (dev_ptr == nullptr || handle == nullptr || base == nullptr) return SCAN2D_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  if (cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return SCAN2D_ECUDA;
  *dev_ptr = static_cast<unsigned char*>(*base) + offset;
  return SCAN2D_OK;
}

int scan2d_ipc_close(void* base) {
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? SCAN2D_OK : SCAN2D_ECUDA;
}

int scan2d_fwd_f32(const scan2d_desc* desc, const float* x, const float* z, const float* B,
                   const float* C, const float* A, const float* Dskip, const float* bias,
                   float* y, float* ph, float* pv, void* residual, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F32;
  return scan2d_forward(&d, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                        workspace_bytes, stream);
}

int scan2d_fwd_f64(const scan2d_desc* desc, const double* x, const double* z, const double* B,
                   const double* C, const double* A, const double* Dskip, const double* bias,
                   double* y, double* ph, double* pv, void* residual, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F64;
  return scan2d_forward(&d, x, z, B, C, A, Dskip, bias, y, ph, pv, residual, workspace,
                        workspace_bytes, stream);
}

int scan2d_bwd_f32(const scan2d_desc* desc, const float* x, const float* z, const float* B,
                   const float* C, const float* A, const float* Dskip, const float* bias,
                   const void* residual, const float* dy, float* dx, float* dz, float* dA,
                   float* dB, float* dC, float* dDskip, float* dbias, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F32;
  return scan2d_backward(&d, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                         dbias, workspace, workspace_bytes, stream);
}

int scan2d_bwd_f64(const scan2d_desc* desc, const double* x, const double* z, const double* B,
                   const double* C, const double* A, const double* Dskip, const double* bias,
                   const void* residual, const double* dy, double* dx, double* dz, double* dA,
                   double* dB, double* dC, double* dDskip, double* dbias, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream) {
  if (desc == nullptr) return SCAN2D_EINVAL;
  scan2d_desc d = *desc;
  d.dtype = SCAN2D_F64;
  return scan2d_backward(&d, x, z, B, C, A, Dskip, bias, residual, dy, dx, dz, dA, dB, dC, dDskip,
                         dbias, workspace, workspace_bytes, stream);
}

int scan2d_plan_info(const scan2d_desc* desc, int op, int64_t* out8) {
  int rc = check_desc(desc);
  if (rc != SCAN2D_OK) return rc;
  if (desc->state_dim > kMaxKernelN) {  // per state group of 128
    scan2d_desc g = *desc;
    g.state_dim = kMaxKernelN;
    return scan2d_plan_info(&g, op, out8);
  }
  if (out8 == nullptr) return SCAN2D_EINVAL;
  Plan p;
  rc = make_plan(*desc, p);
  if (rc != SCAN2D_OK) return rc;
  bool xvec = true, bvec = true, yvec = true;
  vec_flags(*desc, p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, xvec, bvec, yvec);
  rc = plan_with_flags(*desc, p, xvec, bvec);
  if (rc != SCAN2D_OK) return rc;
  const s2d::Geo& g = op == SCAN2D_OP_BWD ? p.b : p.f;
  out8[0] = g.spl * 100 + g.lpc;  // states per lane * 100 + lanes per chunk
  out8[1] = g.J;
  out8[2] = g.seg;
  out8[3] = g.wreal;
  out8[4] = g.colsw;
  out8[5] = g.smem_bytes;
  out8[6] = g.units;
  out8[7] = p.K;
  return SCAN2D_OK;
}

int scan2d_last_launch_count(void) { return g_last_launches; }

const char* scan2d_status_string(int status) {
  switch (status) {
    case SCAN2D_OK: return "ok";
    case SCAN2D_EINVAL: return "invalid argument (shape / descriptor)";
    case SCAN2D_ESTALE: return "stale or missing saved forward state";
    case SCAN2D_ECUDA: return "CUDA runtime / launch error";
    case SCAN2D_ENOMEM: return "workspace too small";
    case SCAN2D_EUNSUPPORTED: return "unsupported device or configuration";
    default: return "unknown status";
  }
}

int scan2d_version(void) { return 1; }

}  // extern "C"
