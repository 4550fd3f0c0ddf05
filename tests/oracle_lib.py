"""ctypes access to the CPU checkers under oracle/ (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -- our plain-C restatement, oracle/liboracle.so
* ``RefLib``  -- the reference library built from its own sources,
  oracle/_ref/libscan2d_ref.so (present wherever ``oracle/Makefile ref`` ran)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "liboracle.so")
REF_SO = os.path.join(REPO, "oracle", "_ref", "libscan2d_ref.so")

_P = C.c_void_p


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def _np_dtype(dtype: str):
    return np.float64 if dtype == "f64" else np.float32


@dataclass
class Instance:
    """One reference ``ScanInstance`` (fixtures.hpp:13-17) as numpy arrays."""

    h: int
    w: int
    n: int
    x: np.ndarray
    z: np.ndarray
    B: np.ndarray
    C: np.ndarray
    A: np.ndarray
    D: float
    bias: float


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        for suf, ct in (("f64", C.c_double), ("f32", C.c_float)):
            getattr(L, f"orc_random_instance_{suf}").argtypes = [C.c_int] * 3 + [C.c_uint64] + [_P] * 7
            getattr(L, f"orc_fill_normal_{suf}").argtypes = [C.c_uint64, C.c_size_t, _P]
            getattr(L, f"orc_fwd_{suf}").argtypes = [C.c_int] * 3 + [_P] * 5 + [ct, ct] + [_P] * 3
            getattr(L, f"orc_carries_{suf}").argtypes = [C.c_int] * 4 + [_P] * 4
            getattr(L, f"orc_bwd_{suf}").argtypes = [C.c_int] * 3 + [_P] * 5 + [ct, ct] + [_P] * 8
            getattr(L, f"orc_fwd_batch_{suf}").argtypes = [C.c_int64] + [C.c_int] * 5 + [_P] * 8 + [C.c_int]
            getattr(L, f"orc_bwd_batch_{suf}").argtypes = [C.c_int64] + [C.c_int] * 5 + [_P] * 15
        L.orc_fast_expf.argtypes = [C.c_float]
        L.orc_fast_expf.restype = C.c_float

    # -- fixtures -----------------------------------------------------------
    def random_instance(self, h, w, n, seed, dtype="f64") -> Instance:
        dt = _np_dtype(dtype)
        x = np.empty(h * w, dt)
        z = np.empty(h * w, dt)
        B = np.empty(h * w * n, dt)
        Cc = np.empty(h * w * n, dt)
        A = np.empty(n, dt)
        D = np.empty(1, dt)
        bias = np.empty(1, dt)
        getattr(self.lib, f"orc_random_instance_{dtype}")(
            h, w, n, C.c_uint64(seed), _ptr(x), _ptr(z), _ptr(B), _ptr(Cc), _ptr(A), _ptr(D), _ptr(bias))
        return Instance(h, w, n, x, z, B, Cc, A, float(D[0]), float(bias[0]))

    def fill_normal(self, seed, count, dtype="f64"):
        out = np.empty(count, _np_dtype(dtype))
        getattr(self.lib, f"orc_fill_normal_{dtype}")(C.c_uint64(seed), count, _ptr(out))
        return out

    # -- single scan ----------------------------------------------------------
    def fwd(self, inst: Instance, dtype="f64", states=False):
        dt = _np_dtype(dtype)
        h, w, n = inst.h, inst.w, inst.n
        y = np.empty(h * w, dt)
        hh = np.empty(h * w * n, dt) if states else None
        hs = np.empty(h * w * n, dt) if states else None
        a = [np.ascontiguousarray(v, dt) for v in (inst.x, inst.z, inst.B, inst.C, inst.A)]
        getattr(self.lib, f"orc_fwd_{dtype}")(h, w, n, *[_ptr(v) for v in a], inst.D, inst.bias,
                                              _ptr(y), _ptr(hh), _ptr(hs))
        return (y, hh, hs) if states else y

    def carries(self, inst: Instance, t: int, dtype="f64"):
        dt = _np_dtype(dtype)
        _, hh, hs = self.fwd(inst, dtype, states=True)
        kh, kw = -(-inst.h // t), -(-inst.w // t)
        ph = np.empty(kh * kw * t * inst.n, dt)
        pv = np.empty_like(ph)
        getattr(self.lib, f"orc_carries_{dtype}")(inst.h, inst.w, inst.n, t, _ptr(hh), _ptr(hs), _ptr(ph), _ptr(pv))
        return ph, pv

    def bwd(self, inst: Instance, dy: np.ndarray, dtype="f64"):
        dt = _np_dtype(dtype)
        h, w, n = inst.h, inst.w, inst.n
        out = dict(dx=np.empty(h * w, dt), dz=np.empty(h * w, dt), dA=np.empty(n, dt),
                   dB=np.empty(h * w * n, dt), dC=np.empty(h * w * n, dt))
        dD = np.empty(1, dt)
        dbias = np.empty(1, dt)
        a = [np.ascontiguousarray(v, dt) for v in (inst.x, inst.z, inst.B, inst.C, inst.A)]
        getattr(self.lib, f"orc_bwd_{dtype}")(h, w, n, *[_ptr(v) for v in a], inst.D, inst.bias,
                                              _ptr(np.ascontiguousarray(dy, dt)), _ptr(out["dx"]), _ptr(out["dz"]),
                                              _ptr(out["dA"]), _ptr(out["dB"]), _ptr(out["dC"]),
                                              _ptr(dD), _ptr(dbias))
        out["dD"] = float(dD[0])
        out["dbias"] = float(dbias[0])
        return out

    # -- batched (C-ABI layout) ---------------------------------------------
    def fwd_batch(self, S, P, G, h, w, n, x, z, B, Cc, A, D, bias, dtype="f32", threads=1):
        dt = _np_dtype(dtype)
        y = np.empty(S * h * w, dt)
        arrs = [np.ascontiguousarray(v, dt).reshape(-1) for v in (x, z, B, Cc, A, D, bias)]
        getattr(self.lib, f"orc_fwd_batch_{dtype}")(S, P, G, h, w, n, *[_ptr(v) for v in arrs], _ptr(y), threads)
        return y

    def bwd_batch(self, S, P, G, h, w, n, x, z, B, Cc, A, D, bias, dy, dtype="f32"):
        dt = _np_dtype(dtype)
        hw = h * w
        out = dict(dx=np.empty(S * hw, dt), dz=np.empty(S * hw, dt), dA=np.empty(P * n, dt),
                   dB=np.empty((S // G) * hw * n, dt), dC=np.empty((S // G) * hw * n, dt),
                   dD=np.empty(P, dt), dbias=np.empty(P, dt))
        arrs = [np.ascontiguousarray(v, dt).reshape(-1) for v in (x, z, B, Cc, A, D, bias, dy)]
        getattr(self.lib, f"orc_bwd_batch_{dtype}")(
            S, P, G, h, w, n, *[_ptr(v) for v in arrs], _ptr(out["dx"]), _ptr(out["dz"]), _ptr(out["dA"]),
            _ptr(out["dB"]), _ptr(out["dC"]), _ptr(out["dD"]), _ptr(out["dbias"]))
        return out


class RefLib:
    """The reference library itself (oracle/_ref/libscan2d_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        for suf, ct in (("f64", C.c_double), ("f32", C.c_float)):
            getattr(L, f"ref_random_instance_{suf}").argtypes = [C.c_int] * 3 + [C.c_uint64] + [_P] * 7
            getattr(L, f"ref_tiled_fwd_{suf}").argtypes = [C.c_int] * 4 + [_P] * 5 + [ct, ct] + [_P] * 3
            getattr(L, f"ref_tiled_fwd_{suf}").restype = C.c_int
            getattr(L, f"ref_tiled_bwd_{suf}").argtypes = [C.c_int] * 4 + [_P] * 5 + [ct, ct] + [_P] * 8
            getattr(L, f"ref_tiled_bwd_{suf}").restype = C.c_int
            getattr(L, f"ref_oracle_fwd_{suf}").argtypes = [C.c_int] * 3 + [_P] * 5 + [ct, ct] + [_P] * 3
            getattr(L, f"ref_batch_{suf}").argtypes = [C.c_int64] + [C.c_int] * 8 + [_P] * 10
            getattr(L, f"ref_batch_{suf}").restype = C.c_double
            if hasattr(L, f"ref_batch_grads_{suf}"):
                getattr(L, f"ref_batch_grads_{suf}").argtypes = [C.c_int64] + [C.c_int] * 5 + [_P] * 16
                getattr(L, f"ref_batch_grads_{suf}").restype = C.c_double
        L.ref_fill_normal_f64.argtypes = [C.c_uint64, C.c_size_t, _P]
        L.ref_fast_expf.argtypes = [C.c_float]
        L.ref_fast_expf.restype = C.c_float
        L.ref_gradcheck.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int, _P]
        L.ref_gradcheck.restype = C.c_int

    def random_instance(self, h, w, n, seed, dtype="f64") -> Instance:
        dt = _np_dtype(dtype)
        x = np.empty(h * w, dt)
        z = np.empty(h * w, dt)
        B = np.empty(h * w * n, dt)
        Cc = np.empty(h * w * n, dt)
        A = np.empty(n, dt)
        D = np.empty(1, dt)
        bias = np.empty(1, dt)
        getattr(self.lib, f"ref_random_instance_{dtype}")(
            h, w, n, C.c_uint64(seed), _ptr(x), _ptr(z), _ptr(B), _ptr(Cc), _ptr(A), _ptr(D), _ptr(bias))
        return Instance(h, w, n, x, z, B, Cc, A, float(D[0]), float(bias[0]))

    def fill_normal(self, seed, count):
        out = np.empty(count, np.float64)
        self.lib.ref_fill_normal_f64(C.c_uint64(seed), count, _ptr(out))
        return out

    def tiled_fwd(self, inst: Instance, t: int, dtype="f64"):
        dt = _np_dtype(dtype)
        h, w, n = inst.h, inst.w, inst.n
        kh, kw = -(-h // t), -(-w // t)
        y = np.empty(h * w, dt)
        ph = np.empty(kh * kw * t * n, dt)
        pv = np.empty_like(ph)
        a = [np.ascontiguousarray(v, dt) for v in (inst.x, inst.z, inst.B, inst.C, inst.A)]
        rc = getattr(self.lib, f"ref_tiled_fwd_{dtype}")(h, w, n, t, *[_ptr(v) for v in a], inst.D, inst.bias,
                                                         _ptr(y), _ptr(ph), _ptr(pv))
        assert rc == 0
        return y, ph, pv

    def tiled_bwd(self, inst: Instance, t: int, dy: np.ndarray, dtype="f64"):
        dt = _np_dtype(dtype)
        h, w, n = inst.h, inst.w, inst.n
        out = dict(dx=np.empty(h * w, dt), dz=np.empty(h * w, dt), dA=np.empty(n, dt),
                   dB=np.empty(h * w * n, dt), dC=np.empty(h * w * n, dt))
        dD = np.empty(1, dt)
        dbias = np.empty(1, dt)
        a = [np.ascontiguousarray(v, dt) for v in (inst.x, inst.z, inst.B, inst.C, inst.A)]
        rc = getattr(self.lib, f"ref_tiled_bwd_{dtype}")(
            h, w, n, t, *[_ptr(v) for v in a], inst.D, inst.bias, _ptr(np.ascontiguousarray(dy, dt)),
            _ptr(out["dx"]), _ptr(out["dz"]), _ptr(out["dA"]), _ptr(out["dB"]), _ptr(out["dC"]), _ptr(dD), _ptr(dbias))
        assert rc == 0
        out["dD"] = float(dD[0])
        out["dbias"] = float(dbias[0])
        return out

    def oracle_fwd(self, inst: Instance, dtype="f64"):
        dt = _np_dtype(dtype)
        h, w, n = inst.h, inst.w, inst.n
        y = np.empty(h * w, dt)
        hh = np.empty(h * w * n, dt)
        hs = np.empty(h * w * n, dt)
        a = [np.ascontiguousarray(v, dt) for v in (inst.x, inst.z, inst.B, inst.C, inst.A)]
        getattr(self.lib, f"ref_oracle_fwd_{dtype}")(h, w, n, *[_ptr(v) for v in a], inst.D, inst.bias,
                                                     _ptr(y), _ptr(hh), _ptr(hs))
        return y, hh, hs

    def gradcheck(self, h, w, n, seed, step=1e-6, tile=3):
        out = np.zeros(14, np.float64)
        k = self.lib.ref_gradcheck(h, w, n, C.c_uint64(seed), step, tile, _ptr(out))
        return out[: 2 * k].reshape(k, 2)

    def batch(self, S, P, G, h, w, n, t, threads, do_bwd, x, z, B, Cc, A, D, bias, dy=None,
              dtype="f32", want_y=False):
        dt = _np_dtype(dtype)
        arrs = [np.ascontiguousarray(v, dt).reshape(-1) for v in (x, z, B, Cc, A, D, bias)]
        dyp = np.ascontiguousarray(dy, dt).reshape(-1) if dy is not None else None
        y = np.empty(S * h * w, dt) if want_y else None
        secs = getattr(self.lib, f"ref_batch_{dtype}")(S, P, G, h, w, n, t, threads, int(do_bwd),
                                                        *[_ptr(v) for v in arrs], _ptr(dyp), _ptr(y), None)
        return secs, y


    def batch_grads(self, S, h, w, n, t, threads, x, z, B, Cc, A, D, bias, dy, dtype="f64"):
        """The reference's tiled forward + backward per scan (P == S, G == 1):
        y and every gradient group (GradBundle, engine.hpp:71-80)."""
        dt = _np_dtype(dtype)
        hw = h * w
        arrs = [np.ascontiguousarray(v, dt).reshape(-1) for v in (x, z, B, Cc, A, D, bias, dy)]
        out = dict(y=np.empty(S * hw, dt), dx=np.empty(S * hw, dt), dz=np.empty(S * hw, dt),
                   dA=np.empty(S * n, dt), dB=np.empty(S * hw * n, dt), dC=np.empty(S * hw * n, dt),
                   dD=np.empty(S, dt), dbias=np.empty(S, dt))
        getattr(self.lib, f"ref_batch_grads_{dtype}")(
            S, h, w, n, t, threads, *[_ptr(v) for v in arrs],
            *[_ptr(out[k]) for k in ("y", "dx", "dz", "dA", "dB", "dC", "dD", "dbias")])
        return out


def rel_error(got, expect) -> float:
    """Normwise error of tests/test_util.hpp:17-26: max|got-ref| / max(max|ref|, 1)."""
    got = np.asarray(got, np.float64).reshape(-1)
    expect = np.asarray(expect, np.float64).reshape(-1)
    if expect.size == 0:
        return 0.0
    return float(np.max(np.abs(got - expect)) / max(float(np.max(np.abs(expect))), 1.0))


def elem_stats(got, expect, floor=1e-3) -> dict:
    """Per-element relative error distribution (denominator max(|ref|, floor))."""
    got = np.asarray(got, np.float64).reshape(-1)
    expect = np.asarray(expect, np.float64).reshape(-1)
    e = np.abs(got - expect) / np.maximum(np.abs(expect), floor)
    if e.size == 0:
        return dict(p50=0.0, p99=0.0, max=0.0)
    return dict(p50=float(np.percentile(e, 50)), p99=float(np.percentile(e, 99)), max=float(e.max()))
