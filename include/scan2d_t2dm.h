/*
 * scan2d_t2dm.h -- "T2DM" binary tensor files (host code, part of
 *                  libscan2d_cuda.so; no CUDA involved).
 *
 * Replaces the reference's tensor I/O (proj/include/scan2d/tensor_io.hpp:11-16,
 * proj/src/tensor_io.cpp:78-151) behind a C ABI:
 *
 *   magic "T2DM" | version u8 | dtype u8 (0 = f32, 1 = f64) | ndim u8 |
 *   reserved u8 = 0 | ndim x u64 dims (little endian) | row-major payload (LE)
 *
 * Version 1 is the reference format, byte for byte: 1 <= ndim <= 3
 * (tensor_io.cpp:17), so a single Grid [H][W][D].  Version 2 is the same
 * layout with 1 <= ndim <= 8, for the batched C-ABI tensors ([S][H][W],
 * [S][H][W][N]); the writer emits version 1 whenever ndim <= 3.
 *
 * Reader checks, in the reference's order and with its error kinds
 * (TensorIoError::Kind): magic (offset 0), version (4), dtype (5), ndim (6),
 * every dim in [1, 2^32] and the element count without overflow (the dim's
 * offset), truncation (the offset where the stream ended), non-finite payload
 * entries (the entry's offset).
 */
#ifndef SCAN2D_T2DM_H
#define SCAN2D_T2DM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCAN2D_T2DM_OK 0
#define SCAN2D_T2DM_BAD_MAGIC 1
#define SCAN2D_T2DM_BAD_VERSION 2
#define SCAN2D_T2DM_BAD_DTYPE 3
#define SCAN2D_T2DM_BAD_SHAPE 4
#define SCAN2D_T2DM_TRUNCATED 5
#define SCAN2D_T2DM_NON_FINITE 6
#define SCAN2D_T2DM_IO 7

#define SCAN2D_T2DM_MAX_NDIM 8

typedef struct scan2d_tensor {
  int32_t dtype;   /* 0 = f32, 1 = f64 (SCAN2D_F32 / SCAN2D_F64)           */
  int32_t ndim;    /* 1 .. 8                                                */
  uint64_t dims[SCAN2D_T2DM_MAX_NDIM];
  void* data;      /* row-major payload; owned by the caller, or by the
                      library after a read (release with scan2d_t2dm_free) */
} scan2d_tensor;

/* Bytes of the encoding of t (0 if t is invalid). */
size_t scan2d_t2dm_encoded_bytes(const scan2d_tensor* t);
/* Encode into buf (capacity cap); *len = bytes written. */
int scan2d_t2dm_encode(const scan2d_tensor* t, void* buf, size_t cap, size_t* len);
/* Decode a complete buffer; allocates out->data.  *err_offset (optional) =
 * byte offset of the failure. */
int scan2d_t2dm_decode(const void* buf, size_t len, scan2d_tensor* out, size_t* err_offset);
/* Files. */
int scan2d_t2dm_write(const char* path, const scan2d_tensor* t, size_t* bytes_written);
int scan2d_t2dm_read(const char* path, scan2d_tensor* out, size_t* err_offset);
void scan2d_t2dm_free(scan2d_tensor* t);
const char* scan2d_t2dm_status_string(int status);

#ifdef __cplusplus
}
#endif

#endif /* SCAN2D_T2DM_H */
