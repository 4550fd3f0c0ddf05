// scan2d_launch.h -- internal interface between the C-ABI host code
// (scan2d_capi.cu) and the per-dtype kernel instantiation units
// (scan2d_kern_f32.cu, scan2d_kern_f64.cu).
#pragma once

#include <cuda_runtime.h>

#include "scan2d_stage.cuh"

namespace s2d {

// Returns cudaSuccess or the launch error.  Kernels are picked by (spl, lpc, J).
template <typename T>
cudaError_t launch_fwd(const Args<T>& a, cudaStream_t stream);
template <typename T>
cudaError_t launch_bwd(const Args<T>& a, cudaStream_t stream);
template <typename T>
cudaError_t launch_reduce_params(const T* part, int64_t S, int wps, int P, int N, T* dA, T* dbias,
                                 T* dD, cudaStream_t stream);
template <typename T>
cudaError_t launch_reduce_group(const T* per_scan, int64_t groups, int G, size_t hwn, T* out,
                                cudaStream_t stream);
// shared-memory geometry (elements of T)
template <typename T>
int stage_elems(int colsw, int Np, int seg, bool bwd);
template <typename T>
int band_elems(int K, int J, int SPL);
// tile-transpose kernels: shared elements (row-lane states SH, strip width CW)
template <typename T>
int tile_elems(int N, int CW, int SH, int stages, bool bwd);

}  // namespace s2d
