"""ctypes binding of the C ABI (include/scan2d_cuda.h) -> lib/libscan2d_cuda.so.

The library is built in-tree (``make -C paper_2412_00678_b200/csrc``, or
``__graft_entry__.build()``).  There is no CPU fallback: if the shared object is
missing this module raises at import time.  ``SCAN2D_LIB_PATH`` points the loader
at another build of the same library (A/B timing of kernel variants).
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCAN2D_LIB_PATH") or os.path.join(_PKG, "lib", "libscan2d_cuda.so")

OK, EINVAL, ESTALE, ECUDA, ENOMEM, EUNSUPPORTED = 0, 1, 2, 3, 4, 5
F32, F64 = 0, 1
OP_FWD, OP_BWD = 0, 1
VARIANT_NAIVE, VARIANT_FLAT1D = 1, 2
MAX_STATE_DIM = 2048

# every symbol include/scan2d_cuda.h declares
EXPORTED_SYMBOLS = (
    "scan2d_check_desc",
    "scan2d_workspace_bytes",
    "scan2d_residual_bytes",
    "scan2d_forward",
    "scan2d_backward",
    "scan2d_forward_band",
    "scan2d_backward_band",
    "scan2d_band_strips",
    "scan2d_forward_band_linked",
    "scan2d_backward_band_linked",
    "scan2d_ipc_export",
    "scan2d_ipc_open",
    "scan2d_ipc_close",
    "scan2d_train_host",
    "scan2d_fwd_f32",
    "scan2d_fwd_f64",
    "scan2d_bwd_f32",
    "scan2d_bwd_f64",
    "scan2d_plan_info",
    "scan2d_comparator_workspace_bytes",
    "scan2d_forward_variant",
    "scan2d_last_launch_count",
    "scan2d_status_string",
    "scan2d_version",
)


class Scan2dDesc(C.Structure):
    """Mirror of ``scan2d_desc`` (include/scan2d_cuda.h)."""

    _fields_ = [
        ("num_scans", C.c_int64),
        ("height", C.c_int32),
        ("width", C.c_int32),
        ("state_dim", C.c_int32),
        ("tile", C.c_int32),
        ("params_period", C.c_int32),
        ("bc_group", C.c_int32),
        ("dtype", C.c_int32),
        ("flags", C.c_int32),
    ]


class Scan2dError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA library must be built "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    D = C.POINTER(Scan2dDesc)
    lib.scan2d_check_desc.argtypes = [D]
    lib.scan2d_check_desc.restype = C.c_int
    lib.scan2d_workspace_bytes.argtypes = [D, C.c_int]
    lib.scan2d_workspace_bytes.restype = C.c_size_t
    lib.scan2d_residual_bytes.argtypes = [D]
    lib.scan2d_residual_bytes.restype = C.c_size_t
    lib.scan2d_forward.argtypes = [D] + [P] * 12 + [C.c_size_t, P]
    lib.scan2d_forward.restype = C.c_int
    lib.scan2d_backward.argtypes = [D] + [P] * 17 + [C.c_size_t, P]
    lib.scan2d_backward.restype = C.c_int
    lib.scan2d_forward_band.argtypes = [D] + [P] * 12 + [C.c_size_t, P]
    lib.scan2d_forward_band.restype = C.c_int
    lib.scan2d_backward_band.argtypes = [D] + [P] * 20 + [C.c_size_t, P]
    lib.scan2d_backward_band.restype = C.c_int
    lib.scan2d_band_strips.argtypes = [D]
    lib.scan2d_band_strips.restype = C.c_int
    lib.scan2d_forward_band_linked.argtypes = [D] + [P] * 13 + [C.c_int, P, C.c_size_t, P]
    lib.scan2d_forward_band_linked.restype = C.c_int
    lib.scan2d_backward_band_linked.argtypes = [D] + [P] * 21 + [C.c_int, P, C.c_size_t, P]
    lib.scan2d_backward_band_linked.restype = C.c_int
    lib.scan2d_ipc_export.argtypes = [P, P, C.POINTER(C.c_uint64)]
    lib.scan2d_ipc_export.restype = C.c_int
    lib.scan2d_ipc_open.argtypes = [P, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    lib.scan2d_ipc_open.restype = C.c_int
    lib.scan2d_ipc_close.argtypes = [P]
    lib.scan2d_ipc_close.restype = C.c_int
    lib.scan2d_train_host.argtypes = [D] + [P] * 16 + [C.c_int, P]
    lib.scan2d_train_host.restype = C.c_int
    for name, n_in in (("scan2d_fwd_f32", 12), ("scan2d_fwd_f64", 12)):
        getattr(lib, name).argtypes = [D] + [P] * n_in + [C.c_size_t, P]
        getattr(lib, name).restype = C.c_int
    for name in ("scan2d_bwd_f32", "scan2d_bwd_f64"):
        getattr(lib, name).argtypes = [D] + [P] * 17 + [C.c_size_t, P]
        getattr(lib, name).restype = C.c_int
    lib.scan2d_comparator_workspace_bytes.argtypes = [D, C.c_int]
    lib.scan2d_comparator_workspace_bytes.restype = C.c_size_t
    lib.scan2d_forward_variant.argtypes = [D, C.c_int] + [P] * 9 + [C.c_size_t, P]
    lib.scan2d_forward_variant.restype = C.c_int
    lib.scan2d_plan_info.argtypes = [D, C.c_int, C.POINTER(C.c_int64)]
    lib.scan2d_plan_info.restype = C.c_int
    lib.scan2d_last_launch_count.argtypes = []
    lib.scan2d_last_launch_count.restype = C.c_int
    lib.scan2d_status_string.argtypes = [C.c_int]
    lib.scan2d_status_string.restype = C.c_char_p
    lib.scan2d_version.argtypes = []
    lib.scan2d_version.restype = C.c_int
    return lib


lib = _load()


def status_string(status: int) -> str:
    return lib.scan2d_status_string(status).decode()


FLAG_ACCURATE = 1  # include/scan2d_cuda.h SCAN2D_FLAG_ACCURATE
FLAG_GROUP_RED = 2  # include/scan2d_cuda.h SCAN2D_FLAG_GROUP_RED


def make_desc(S, H, W, N, tile=16, params_period=None, bc_group=1, dtype=F32, accurate=False,
              group_red=False) -> Scan2dDesc:
    return Scan2dDesc(int(S), int(H), int(W), int(N), int(tile),
                      int(S if params_period is None else params_period), int(bc_group), int(dtype),
                      (FLAG_ACCURATE if accurate else 0) | (FLAG_GROUP_RED if group_red else 0))


def plan_info(desc: Scan2dDesc, op: int = OP_FWD) -> dict:
    out = (C.c_int64 * 8)()
    rc = lib.scan2d_plan_info(C.byref(desc), op, out)
    if rc != OK:
        raise Scan2dError(rc, "scan2d_plan_info")
    keys = ("spl_x100_plus_lpc", "cols_per_chunk", "scans_per_warp", "warps_per_scan",
            "cols_per_warp", "smem_bytes", "warps_total", "band_rows")
    return dict(zip(keys, [int(v) for v in out]))
