"""T2DM tensor files through the C ABI (include/scan2d_t2dm.h): the
reference's tensor I/O (proj/include/scan2d/tensor_io.hpp:11-16,
proj/src/tensor_io.cpp:78-151) -- version 1 byte-compatible with it (1 to 3
dims), version 2 for batched tensors (up to 8 dims).

    write(path, array)       numpy float32 / float64 array -> file
    read(path) -> array      numpy array of the file's dtype and dims
    encode(array) -> bytes / decode(bytes) -> array

Errors raise ``T2dmError`` whose ``kind`` mirrors the reference's
TensorIoError::Kind and whose ``offset`` is the failing byte position."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import lib

KINDS = {1: "BadMagic", 2: "BadVersion", 3: "BadDtype", 4: "BadShape", 5: "Truncated", 6: "NonFinite", 7: "Io"}
MAX_NDIM = 8


class Tensor(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("ndim", C.c_int32), ("dims", C.c_uint64 * MAX_NDIM), ("data", C.c_void_p)]


class T2dmError(ValueError):
    def __init__(self, status: int, offset: int, where: str):
        self.status, self.offset = status, offset
        self.kind = KINDS.get(status, "Unknown")
        super().__init__(f"{where}: {lib.scan2d_t2dm_status_string(status).decode()} at byte {offset}")


_T = C.POINTER(Tensor)
lib.scan2d_t2dm_encoded_bytes.argtypes = [_T]
lib.scan2d_t2dm_encoded_bytes.restype = C.c_size_t
lib.scan2d_t2dm_encode.argtypes = [_T, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
lib.scan2d_t2dm_encode.restype = C.c_int
lib.scan2d_t2dm_decode.argtypes = [C.c_void_p, C.c_size_t, _T, C.POINTER(C.c_size_t)]
lib.scan2d_t2dm_decode.restype = C.c_int
lib.scan2d_t2dm_write.argtypes = [C.c_char_p, _T, C.POINTER(C.c_size_t)]
lib.scan2d_t2dm_write.restype = C.c_int
lib.scan2d_t2dm_read.argtypes = [C.c_char_p, _T, C.POINTER(C.c_size_t)]
lib.scan2d_t2dm_read.restype = C.c_int
lib.scan2d_t2dm_free.argtypes = [_T]
lib.scan2d_t2dm_free.restype = None
lib.scan2d_t2dm_status_string.argtypes = [C.c_int]
lib.scan2d_t2dm_status_string.restype = C.c_char_p


def _tensor_of(a: np.ndarray):
    if a.dtype not in (np.float32, np.float64):
        raise TypeError("T2DM holds float32 or float64 tensors")
    if not 1 <= a.ndim <= MAX_NDIM:
        raise ValueError(f"T2DM holds 1 to {MAX_NDIM} dims")
    a = np.ascontiguousarray(a)
    t = Tensor()
    t.dtype = 1 if a.dtype == np.float64 else 0
    t.ndim = a.ndim
    for i, d in enumerate(a.shape):
        t.dims[i] = d
    t.data = a.ctypes.data
    return t, a


def _array_of(t: Tensor) -> np.ndarray:
    shape = tuple(int(t.dims[i]) for i in range(t.ndim))
    dt = np.float64 if t.dtype == 1 else np.float32
    n = int(np.prod(shape))
    buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(t.data)
    out = np.frombuffer(bytes(buf), dtype=dt).reshape(shape).copy()
    lib.scan2d_t2dm_free(C.byref(t))
    return out


def encode(a: np.ndarray) -> bytes:
    t, keep = _tensor_of(a)
    n = lib.scan2d_t2dm_encoded_bytes(C.byref(t))
    buf = C.create_string_buffer(max(n, 1))
    ln = C.c_size_t(0)
    rc = lib.scan2d_t2dm_encode(C.byref(t), buf, n, C.byref(ln))
    if rc:
        raise T2dmError(rc, 0, "encode")
    del keep
    return buf.raw[: ln.value]


def decode(b: bytes) -> np.ndarray:
    t = Tensor()
    off = C.c_size_t(0)
    raw = C.create_string_buffer(b, len(b)) if b else C.create_string_buffer(1)
    rc = lib.scan2d_t2dm_decode(raw, len(b), C.byref(t), C.byref(off))
    if rc:
        raise T2dmError(rc, off.value, "decode")
    return _array_of(t)


def write(path: str, a: np.ndarray) -> int:
    t, keep = _tensor_of(a)
    n = C.c_size_t(0)
    rc = lib.scan2d_t2dm_write(str(path).encode(), C.byref(t), C.byref(n))
    if rc:
        raise T2dmError(rc, 0, f"write {path}")
    del keep
    return n.value


def read(path: str) -> np.ndarray:
    t = Tensor()
    off = C.c_size_t(0)
    rc = lib.scan2d_t2dm_read(str(path).encode(), C.byref(t), C.byref(off))
    if rc:
        raise T2dmError(rc, off.value, f"read {path}")
    return _array_of(t)
