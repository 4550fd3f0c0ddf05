"""T2DM tensor files (include/scan2d_t2dm.h) against the
reference's own tensor I/O (tensor_io.cpp:78-151, compiled into
oracle/_ref/libscan2d_ref.so): identical bytes for every v1 tensor, the
reference decodes what we write and we decode what it writes, the same error
kinds and offsets on corrupted streams (test_tensor_io.cpp), and the v2
extension for batched tensors.  Host code only (CPU)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2412_00678_b200 import t2dm

REF_KINDS = ["BadMagic", "BadVersion", "BadDtype", "BadShape", "Truncated", "NonFinite", "Io"]  # enum order


@pytest.fixture(scope="module")
def ref():
    from oracle_lib import REF_SO

    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built")
    L = C.CDLL(REF_SO)
    L.ref_t2dm_encode.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_size_t]
    L.ref_t2dm_encode.restype = C.c_size_t
    L.ref_t2dm_decode.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_void_p]
    L.ref_t2dm_decode.restype = C.c_int
    return L


def ref_encode(L, a):
    a = np.ascontiguousarray(a)
    dims = (C.c_uint64 * a.ndim)(*a.shape)
    cap = 64 + a.nbytes
    buf = C.create_string_buffer(cap)
    n = L.ref_t2dm_encode(1 if a.dtype == np.float64 else 0, a.ndim, dims, a.ctypes.data, buf, cap)
    assert n > 0
    return buf.raw[:n]


def ref_decode(L, b, like=None):
    off = C.c_size_t(0)
    out = np.empty_like(like) if like is not None else None
    k = L.ref_t2dm_decode(b, len(b), C.byref(off), None if out is None else out.ctypes.data)
    return (None if k < 0 else REF_KINDS[k]), off.value, out


def test_reference_examples():
    # test_tensor_io.cpp: a 1x1x1 grid is 20 bytes, a 2x3 double grid 72, dims little endian
    assert len(t2dm.encode(np.zeros((1,), np.float32))) == 20
    b = t2dm.encode(np.arange(1, 7, dtype=np.float64).reshape(2, 3))
    assert len(b) == 8 + 16 + 48 and b[:4] == b"T2DM" and b[6] == 2 and b[8] == 2 and b[16] == 3
    g = t2dm.decode(t2dm.encode(np.random.default_rng(3).standard_normal((14, 14))))
    assert g.shape == (14, 14)


def test_bytes_identical_to_reference(ref):
    rng = np.random.default_rng(7)
    for trial in range(60):
        nd = int(rng.integers(1, 4))
        shape = tuple(int(v) for v in rng.integers(1, 10, size=nd))
        dt = np.float64 if trial % 2 else np.float32
        a = rng.standard_normal(shape).astype(dt)
        ours = t2dm.encode(a)
        assert ours == ref_encode(ref, a), shape
        kind, _, back = ref_decode(ref, ours, like=a)
        assert kind is None and np.array_equal(back, a)
        assert np.array_equal(t2dm.decode(ref_encode(ref, a)), a)


def _valid():
    return bytearray(t2dm.encode(np.array([[1, 2], [3, 4]], np.float32)))


@pytest.mark.parametrize("case", ["magic", "version", "dtype", "ndim0", "ndim9", "dim0", "truncated_dims",
                                  "truncated_payload", "inf", "nan", "header_only"])
def test_error_kinds_match_reference(ref, case):
    b = _valid()
    if case == "magic":
        b[0] = ord("X")
    elif case == "version":
        b[4] = 9
    elif case == "dtype":
        b[5] = 7
    elif case == "ndim0":
        b[6] = 0
    elif case == "ndim9":
        b[6] = 9
    elif case == "dim0":
        b[8:16] = (0).to_bytes(8, "little")
    elif case == "truncated_dims":
        b = b[:12]
    elif case == "truncated_payload":
        b = b[:-5]
    elif case == "inf":
        b[-4:] = np.array([np.inf], np.float32).tobytes()
    elif case == "nan":
        b[-8:-4] = np.array([np.nan], np.float32).tobytes()
    elif case == "header_only":
        b = b[:5]
    kind, off, _ = ref_decode(ref, bytes(b))
    with pytest.raises(t2dm.T2dmError) as ei:
        t2dm.decode(bytes(b))
    assert ei.value.kind == kind and ei.value.offset == off, (case, kind, off, ei.value)


def test_v2_batched_round_trip(tmp_path):
    rng = np.random.default_rng(11)
    for shape in [(3, 4, 5, 2), (2, 1, 3, 1, 2), (1, 2, 3, 4, 5, 6, 1, 2)]:
        for dt in (np.float32, np.float64):
            a = rng.standard_normal(shape).astype(dt)
            b = t2dm.encode(a)
            assert b[4] == 2  # version 2: more than 3 dims
            assert np.array_equal(t2dm.decode(b), a)
            p = tmp_path / "t.t2dm"
            assert t2dm.write(p, a) == len(b)
            assert np.array_equal(t2dm.read(p), a)
    with pytest.raises(ValueError):
        t2dm.encode(np.zeros((1,) * 9, np.float32))
    with pytest.raises(t2dm.T2dmError) as ei:
        t2dm.read(tmp_path / "missing.t2dm")
    assert ei.value.kind == "Io"


def test_v1_reader_rejects_more_than_three_dims_as_reference(ref):
    """A version-1 header with ndim 4 is BadShape in the reference and here."""
    b = bytearray(t2dm.encode(np.zeros((2, 2, 2, 2), np.float32)))
    b[4] = 1
    kind, off, _ = ref_decode(ref, bytes(b))
    with pytest.raises(t2dm.T2dmError) as ei:
        t2dm.decode(bytes(b))
    assert (ei.value.kind, ei.value.offset) == (kind, off) == ("BadShape", 6)
