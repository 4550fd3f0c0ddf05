// scan2d_launch.h -- internal interface between the C-ABI host code
// (scan2d_capi.cu) and the per-dtype kernel instantiation units
// (scan2d_kern_f32.cu, scan2d_kern_f64.cu).
#pragma once

#include <cuda_runtime.h>

#include "scan2d_common.cuh"

namespace s2d {

// Returns cudaSuccess or the launch error.  Kernels are picked by (lpc, J).
template <typename T>
cudaError_t launch_fwd(const Args<T>& a, size_t smem_bytes, cudaStream_t stream);
template <typename T>
cudaError_t launch_bwd(const Args<T>& a, size_t smem_bytes, cudaStream_t stream);
template <typename T>
cudaError_t launch_reduce_params(const T* part, int64_t S, int wps, int wreal, int P, int N, T* dA,
                                 T* dbias, T* dD, cudaStream_t stream);
template <typename T>
cudaError_t launch_reduce_group(const T* per_scan, int64_t groups, int G, size_t hwn, T* out,
                                cudaStream_t stream);
template <typename T>
size_t fwd_smem_bytes(const Plan& p);
template <typename T>
size_t bwd_smem_bytes(const Plan& p);

}  // namespace s2d
