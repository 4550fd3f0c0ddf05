/*
 * scan2d_cuda.h -- C ABI of the B200 (sm_100a) 2D selective-scan library
 *                  (libscan2d_cuda.so).
 *
 * Drop-in boundary for the hot path of the 2DMamba reference artifact
 * (arXiv 2412.00678, /root/reference/proj):
 *
 *   scan2d_forward   replaces  scan2d::tiled_scan_2d_forward<T>
 *                              (proj/include/scan2d/engine.hpp:88-94,
 *                               proj/src/engine.cpp:154-243)
 *   scan2d_backward  replaces  scan2d::tiled_scan_2d_backward<T>
 *                              (proj/include/scan2d/engine.hpp:100-102,
 *                               proj/src/engine.cpp:245-410)
 *
 * The reference's C++ template API itself is re-provided on top of this ABI by
 * paper_2412_00678_b200/csrc/shim/engine_shim.cpp (libscan2d_engine_cuda.so).
 *
 * Conventions
 *  - Plain C: no exceptions, no STL, no torch types.  Every pointer argument is
 *    a DEVICE pointer unless stated; the caller owns every buffer, including the
 *    workspace and the residual ("saved forward") buffer.
 *  - Stream ordered: work is enqueued on `stream`; nothing synchronises the host.
 *  - Deterministic: identical inputs give identical output bits run to run (no
 *    floating-point atomics; scalar reductions use a fixed order) -- except
 *    dB / dC under SCAN2D_FLAG_GROUP_RED, which the caller opts into.
 *  - Thread safe across distinct (stream, workspace) pairs.
 *  - Workspaces need no initialisation.  Launches whose column strips are
 *    chained across CTAs keep a small header at the start of the workspace (a
 *    ticket, a device-side epoch for the carry tags, a layout hash): a short
 *    begin kernel advances it in stream order, so a call captured in a CUDA
 *    graph stays correct on every replay.  The first call with a workspace, or
 *    the first after it served another descriptor / op, clears the workspace's
 *    carry region once (stale words can never satisfy a tag).
 *  - Output alignment: none required; 16-byte aligned dB / dC enable the
 *    vector-store kernels (otherwise a scalar-store kernel family runs).
 *    The workspace and the residual buffer must be 16-byte aligned (any
 *    cudaMalloc / framework allocation is); otherwise SCAN2D_EINVAL.
 *
 * Layouts (S scans = flattened batch x channel, per-scan reference Grid layout,
 * types.hpp:55-57, N fastest):
 *   x, z, y, dy, dx, dz          [S][H][W]
 *   B, C, dB, dC                 [S/G][H][W][N]   (scan s uses B/C block s / G)
 *   A, dA                        [P][N]           (scan s uses parameter row s % P)
 *   Dskip, bias, dDskip, dbias   [P]
 *   ph, pv (optional)            [S][kh][kw][T][N], kh = ceil(H/T), kw = ceil(W/T):
 *                                the reference CarryState (engine.hpp:29-46)
 * G = 1 and P = S is the reference operator contract (one scan per call);
 * G = P = D channels is the 2DMamba block layout (model.cpp:150-193).
 */
#ifndef SCAN2D_CUDA_H
#define SCAN2D_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the reference throws std::invalid_argument / std::logic_error,
 * engine.cpp:19-30, :163-164, :248-252; the C++ shim maps these back) */
#define SCAN2D_OK 0
#define SCAN2D_EINVAL 1        /* shape / argument error  (std::invalid_argument) */
#define SCAN2D_ESTALE 2        /* no valid saved forward  (std::logic_error)      */
#define SCAN2D_ECUDA 3         /* CUDA launch / runtime error                     */
#define SCAN2D_ENOMEM 4        /* workspace too small                             */
#define SCAN2D_EUNSUPPORTED 5  /* device is not sm_100 / configuration not served  */

#define SCAN2D_F32 0
#define SCAN2D_F64 1

#define SCAN2D_OP_FWD 0
#define SCAN2D_OP_BWD 1

#define SCAN2D_MAX_STATE_DIM 2048 /* engine.cpp:19 kMaxStateDim */

/* Opaque stream handle; binary compatible with cudaStream_t (CUstream_st*). */
typedef struct CUstream_st* scan2d_stream_t;

typedef struct scan2d_desc {
  int64_t num_scans;    /* S >= 1                                              */
  int32_t height;       /* H >= 1                                              */
  int32_t width;        /* W >= 1                                              */
  int32_t state_dim;    /* N in [1, 2048] (N > 128: passes over state groups)  */
  int32_t tile;         /* reference TileConfig T >= 1 (layout of ph / pv)     */
  int32_t params_period;/* P >= 1, divides S                                    */
  int32_t bc_group;     /* G >= 1, divides S                                    */
  int32_t dtype;        /* SCAN2D_F32 or SCAN2D_F64                            */
  int32_t flags;        /* 0, or SCAN2D_FLAG_ACCURATE | SCAN2D_FLAG_GROUP_RED  */
} scan2d_desc;

/* desc->flags: fp32 exponentials by range reduction + polynomial (< 1 ulp)
 * instead of the MUFU ex2.approx (~2 ulp, one-signed): fp32 results closer to
 * fp64 than the reference's own fp32 engine (tile N in {4, 8, 16, 32} and row
 * N = 1 kernels; other N already use a compensated exponential), at a cost in
 * speed.  No effect on fp64. */
#define SCAN2D_FLAG_ACCURATE 1

/* desc->flags, backward with bc_group G > 1: dB / dC are summed over the
 * group in place by L2 reductions (red.global.add) from inside the scan kernel,
 * instead of per-scan gradients in the workspace plus a fixed-order reduction
 * kernel.  Faster (no 2 S H W N workspace traffic) but the summation order is
 * not fixed: results vary in the last bits from run to run, and fp32 denormal
 * addends flush to zero.  Tile kernels only (N in {4, 8, 16, 32}); other
 * shapes ignore the flag.  Default off (deterministic). */
#define SCAN2D_FLAG_GROUP_RED 2

/* Validates a descriptor (the checks of require_shapes, engine.cpp:21-30). */
int scan2d_check_desc(const scan2d_desc* desc);

/* Bytes of caller-provided scratch for one call of `op` (SCAN2D_OP_FWD/BWD). */
size_t scan2d_workspace_bytes(const scan2d_desc* desc, int op);

/* Bytes of the residual buffer a training forward fills and the backward reads:
 * vertical-state checkpoints every few rows plus the horizontal carries at the
 * kernel's column-group boundaries (the analogue of SavedForward's CarryState,
 * engine.hpp:51-59).  Inputs are NOT copied: the backward takes them again. */
size_t scan2d_residual_bytes(const scan2d_desc* desc);

/* Forward: y = C.h + Dskip.x with h the 2D scan of (Abar = exp(delta A),
 * Bbar x = delta B x), delta = softplus(z + bias).
 *   y         required
 *   ph, pv    optional (NULL): reference CarryState per scan for desc->tile
 *   residual  optional (NULL = inference, reference save_residuals = false)
 */
int scan2d_forward(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                   const void* C, const void* A, const void* Dskip, const void* bias, void* y,
                   void* ph, void* pv, void* residual, void* workspace, size_t workspace_bytes,
                   scan2d_stream_t stream);

/* Backward from the residual of a training forward with the same descriptor and
 * inputs.  residual == NULL returns SCAN2D_ESTALE.  All gradient outputs are
 * overwritten (not accumulated). */
int scan2d_backward(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                    const void* C, const void* A, const void* Dskip, const void* bias,
                    const void* residual, const void* dy, void* dx, void* dz, void* dA,
                    void* dB, void* dC, void* dDskip, void* dbias, void* workspace,
                    size_t workspace_bytes, scan2d_stream_t stream);

/* ---- row-band shard: one band of rows of a taller grid ----
 * desc->height = the band's rows.  The horizontal recurrences are band-local; the
 * vertical ones continue across the band edges through [S][W][N] carries:
 *   h_top     h of the row just above the band (NULL = first band, zeros)
 *   h_bottom  forward output: h of the band's last row (= the next band's h_top)
 *   g_bottom  backward input: Abar(i+1,j) G(i+1,j) of the row just below the band
 *             (= the next band's g_top; NULL = last band, zeros)
 *   g_top     backward output: Abar G of the band's first row
 * The backward takes the same h_top as its forward.  dA / dDskip / dbias are the
 * band's partial sums (add them over bands in a fixed order).  Tile-kernel
 * configurations only (N in {4, 8, 16, 32}, 16-byte aligned rows); otherwise
 * SCAN2D_EUNSUPPORTED.  A band starting at a multiple of 32 * SH / N rows of the
 * full grid (SH = 2 fp32, 1 fp64) reproduces the full grid's y, dx, dz, dB, dC
 * bit for bit; dA / dDskip / dbias up to the order of the band sum. */
int scan2d_forward_band(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                        const void* C, const void* A, const void* Dskip, const void* bias,
                        const void* h_top, void* y, void* h_bottom, void* residual, void* workspace,
                        size_t workspace_bytes, scan2d_stream_t stream);
int scan2d_backward_band(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                         const void* C, const void* A, const void* Dskip, const void* bias,
                         const void* h_top, const void* residual, const void* dy, const void* g_bottom,
                         void* dx, void* dz, void* dA, void* dB, void* dC, void* dDskip, void* dbias,
                         void* g_top, void* workspace, size_t workspace_bytes, scan2d_stream_t stream);

/* ---- row bands on different GPUs, linked in-kernel ----
 * The same band entry points with the carry hand-off done by the kernels
 * themselves: h_bottom (forward) / g_top (backward) may point into the NEXT /
 * PREVIOUS band's buffer on another GPU (peer memory over NVLink, e.g. from
 * cudaIpcOpenMemHandle, see scan2d_ipc_*), and every (scan, 16-column strip)
 * publishes its part with a system-scope release flag.  A strip of the
 * receiving band waits on its own flag (acquire) just before it first reads
 * h_top / g_bottom, so bands run concurrently and each strip starts as soon as
 * the strip above (forward) / below (backward) has finished -- no host
 * synchronisation, no collective, no scan-chunk pipeline.
 *   in_flags   [S * strips] flags written by the producing band (NULL: no wait)
 *   out_flags  [S * strips] flags of the consuming band (NULL: no publish)
 *   seq        value the flags carry for this call (must change from call to
 *              call on a link, e.g. a counter; flags start at any other value)
 * strips = scan2d_band_strips(desc).  A producer that never arrives makes the
 * waiting kernel trap after 10 s (the launch fails instead of hanging the GPU
 * or continuing on a stale carry).
 * Not for CUDA graph capture (seq is a launch argument). */
int scan2d_band_strips(const scan2d_desc* desc);
int scan2d_forward_band_linked(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                               const void* C, const void* A, const void* Dskip, const void* bias,
                               const void* h_top, void* y, void* h_bottom, void* residual, const int* in_flags,
                               int* out_flags, int seq, void* workspace, size_t workspace_bytes,
                               scan2d_stream_t stream);
int scan2d_backward_band_linked(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                                const void* C, const void* A, const void* Dskip, const void* bias,
                                const void* h_top, const void* residual, const void* dy, const void* g_bottom,
                                void* dx, void* dz, void* dA, void* dB, void* dC, void* dDskip, void* dbias,
                                void* g_top, const int* in_flags, int* out_flags, int seq, void* workspace,
                                size_t workspace_bytes, scan2d_stream_t stream);
/* CUDA IPC for the links between processes (one per GPU): export a device
 * pointer as a 64-byte handle of its allocation plus the pointer's offset in
 * it (caching allocators hand out interior pointers), open a peer's handle in
 * this process (*dev_ptr = mapped base + offset; *base for scan2d_ipc_close). */
int scan2d_ipc_export(const void* dev_ptr, unsigned char handle[64], uint64_t* offset);
int scan2d_ipc_open(const unsigned char handle[64], uint64_t offset, void** dev_ptr, void** base);
int scan2d_ipc_close(void* base);

/* ---- host operands (the reference API's contract: Grid<T> data lives in host
 * memory, engine.hpp:88-102) ----
 * One training step -- forward, and backward when dy != NULL -- on HOST
 * pointers with the layouts above.  The S scans are processed in `chunks`
 * groups (the first and last split further into 1/8, 1/8, 1/4, 1/2 pieces)
 * through three device buffer sets: host->device copies of chunk k, the
 * kernels of chunk k-1 and device->host copies of chunk k-2 overlap on three
 * internal streams; `stream` is joined at both ends (call
 * cudaStreamSynchronize(stream) before reading the outputs).  Host buffers
 * should be page-locked (cudaHostAlloc / cudaHostRegister) for the copies to
 * run asynchronously.  Device buffers are cached per host thread and
 * descriptor.  Shared B/C (G > 1) and shared parameters (P < S) are cut at
 * multiples of lcm(G, P) scans (whole groups and parameter periods; the
 * parameter gradients are summed over the chunks in chunk order); a single
 * group / period is one chunk.  With dy == NULL only y is written.  chunks <= 0
 * picks the count automatically (>= 32 MB of input per chunk, at most 8). */
int scan2d_train_host(const scan2d_desc* desc, const void* x, const void* z, const void* B,
                      const void* C, const void* A, const void* Dskip, const void* bias,
                      const void* dy, void* y, void* dx, void* dz, void* dA, void* dB, void* dC,
                      void* dDskip, void* dbias, int chunks, scan2d_stream_t stream);

/* Typed conveniences (desc->dtype is overridden). */
int scan2d_fwd_f32(const scan2d_desc* desc, const float* x, const float* z, const float* B,
                   const float* C, const float* A, const float* Dskip, const float* bias,
                   float* y, float* ph, float* pv, void* residual, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream);
int scan2d_fwd_f64(const scan2d_desc* desc, const double* x, const double* z, const double* B,
                   const double* C, const double* A, const double* Dskip, const double* bias,
                   double* y, double* ph, double* pv, void* residual, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream);
int scan2d_bwd_f32(const scan2d_desc* desc, const float* x, const float* z, const float* B,
                   const float* C, const float* A, const float* Dskip, const float* bias,
                   const void* residual, const float* dy, float* dx, float* dz, float* dA,
                   float* dB, float* dC, float* dDskip, float* dbias, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream);
int scan2d_bwd_f64(const scan2d_desc* desc, const double* x, const double* z, const double* B,
                   const double* C, const double* A, const double* Dskip, const double* bias,
                   const void* residual, const double* dy, double* dx, double* dz, double* dA,
                   double* dB, double* dC, double* dDskip, double* dbias, void* workspace,
                   size_t workspace_bytes, scan2d_stream_t stream);

/* ---- comparator operators (Table 3 of the paper) ----
 * SCAN2D_VARIANT_NAIVE   replaces scan2d::naive_scan_2d          (engine.hpp:108-112,
 *                        engine.cpp:412-487): N horizontal state maps in HBM,
 *                        then a column pass.
 * SCAN2D_VARIANT_FLAT1D  replaces scan2d::block_scan_1d_forward  (engine.hpp:114-118,
 *                        engine.cpp:489-526): 1D scan of the row-major flattened grid.
 * Forward only (the reference has no backward for them). */
#define SCAN2D_VARIANT_NAIVE 1
#define SCAN2D_VARIANT_FLAT1D 2
size_t scan2d_comparator_workspace_bytes(const scan2d_desc* desc, int variant);
int scan2d_forward_variant(const scan2d_desc* desc, int variant, const void* x, const void* z,
                           const void* B, const void* C, const void* A, const void* Dskip,
                           const void* bias, void* y, void* workspace, size_t workspace_bytes,
                           scan2d_stream_t stream);

/* Launch geometry the library picks for a descriptor (diagnostics / bench):
 * out[0..7] = {lanes_per_chunk, cols_per_chunk, scans_per_warp, warps_per_scan,
 *              warps_per_cta, ctas_per_scan_row, total_ctas, band_rows}. */
int scan2d_plan_info(const scan2d_desc* desc, int op, int64_t* out8);

/* Number of kernel launches the last scan2d_forward / scan2d_backward call on
 * this host thread enqueued (begin kernels included, memsets excluded). */
int scan2d_last_launch_count(void);

const char* scan2d_status_string(int status);
int scan2d_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SCAN2D_CUDA_H */
