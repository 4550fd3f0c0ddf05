"""Host-side mirror of the reference scan API over the CUDA C ABI.

Mirrors ``scan2d::tiled_scan_2d_forward`` / ``tiled_scan_2d_backward``
(proj/include/scan2d/engine.hpp:82-102) with the same argument meaning and
error behaviour, batched over S independent scans:

=====================  =========================  ==================================
reference              here                       notes
=====================  =========================  ==================================
``Grid<T> x`` [H,W]    ``x`` [S,H,W]               S = batch x channel (model.cpp:177)
``inputs.z_raw``       ``z`` [S,H,W]
``inputs.b / .c``      ``B, C`` [S/G,H,W,N]        G = bc_group (1 = reference contract)
``params.a``           ``A`` [P,N]                 scan s uses row s % P
``params.d_skip/bias`` ``Dskip, bias`` [P]
``TileConfig``         ``tile``                    only shapes the optional carries
``threads``            ``threads``                 accepted, no effect (already deterministic)
``save_residuals``     ``save_residuals``          False -> saved.valid is False
``CarryState``         ``carries=True``            ph, pv [S,kh,kw,T,N]
=====================  =========================  ==================================

Errors: shape problems raise ``ValueError`` (std::invalid_argument,
engine.cpp:19-30, :163-164, :251-252); backward from an invalid saved state
raises ``RuntimeError`` (std::logic_error, engine.cpp:248-249).

All compute runs in libscan2d_cuda.so; torch is used for device memory and
the current CUDA stream only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _native as nat


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return nat.F32
    if t.dtype == torch.float64:
        return nat.F64
    raise ValueError(f"scan2d: dtype {t.dtype} unsupported (float32 / float64 only)")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _vptr(t):
    """A tensor, a raw device address (int, e.g. IPC-mapped peer memory) or None."""
    if t is None:
        return None
    if isinstance(t, int):
        return C.c_void_p(t)
    return C.c_void_p(t.data_ptr())


def _stream(device: torch.device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check(cond: bool, msg: str):
    if not cond:
        raise ValueError(msg)


@dataclass
class SavedForward:
    """Analogue of ``SavedForward<T>`` (engine.hpp:51-59).  Inputs are
    referenced, not deep-copied (autograd convention: do not modify them in
    place between forward and backward); ``residual`` holds the recompute
    checkpoints and boundary carries."""

    x: Optional[torch.Tensor] = None
    z: Optional[torch.Tensor] = None
    B: Optional[torch.Tensor] = None
    C: Optional[torch.Tensor] = None
    A: Optional[torch.Tensor] = None
    Dskip: Optional[torch.Tensor] = None
    bias: Optional[torch.Tensor] = None
    residual: Optional[torch.Tensor] = None
    desc: Optional[nat.Scan2dDesc] = None
    valid: bool = False


@dataclass
class TiledForwardResult:
    y: torch.Tensor
    saved: SavedForward = field(default_factory=SavedForward)
    ph: Optional[torch.Tensor] = None
    pv: Optional[torch.Tensor] = None


@dataclass
class GradBundle:
    """Analogue of ``GradBundle<T>`` (engine.hpp:71-80)."""

    dx: torch.Tensor
    dz_raw: torch.Tensor
    da: torch.Tensor
    db: torch.Tensor
    dc: torch.Tensor
    dd: torch.Tensor
    dbias: torch.Tensor


def _normalise(x, z, B, C_, A, Dskip, bias):
    """Accept single-scan reference shapes ([H,W], [H,W,N], [N], scalar) or batched ones."""
    if x.dim() == 2:
        x = x.unsqueeze(0)
    if z.dim() == 2:
        z = z.unsqueeze(0)
    if B.dim() == 3:
        B = B.unsqueeze(0)
    if C_.dim() == 3:
        C_ = C_.unsqueeze(0)
    if A.dim() == 1:
        A = A.unsqueeze(0)
    Dskip = Dskip.reshape(-1)
    bias = bias.reshape(-1)
    return x, z, B, C_, A, Dskip, bias


def make_desc_for(x, z, B, C_, A, Dskip, bias, tile: int, accurate: bool = False,
                  group_red: bool = False) -> nat.Scan2dDesc:
    """require_shapes (engine.cpp:21-30) + TileConfig (types.hpp:133-146) checks."""
    _check(x.dim() == 3, "scan input must be [S,H,W] (single channel per scan)")
    S, H, W = x.shape
    _check(tuple(z.shape) == (S, H, W), "input and selective grids must share H and W")
    _check(B.dim() == 4 and C_.dim() == 4, "B and C must be [S/G,H,W,N]")
    _check(tuple(B.shape[1:3]) == (H, W) and tuple(C_.shape[1:3]) == (H, W),
           "input and selective grids must share H and W")
    _check(B.shape == C_.shape, "SelectiveInputs: B and C must share N")
    N = B.shape[3]
    _check(A.dim() == 2 and A.shape[1] == N, "state dimension mismatch between inputs and params")
    _check(N <= nat.MAX_STATE_DIM, "state dimension too large")
    P = A.shape[0]
    _check(Dskip.numel() == P and bias.numel() == P, "Dskip / bias must have one entry per A row")
    _check(S % P == 0, "number of scans must be a multiple of the parameter rows")
    _check(B.shape[0] >= 1 and S % B.shape[0] == 0, "number of scans must be a multiple of B/C blocks")
    _check(tile > 0, "TileConfig: T must be positive")
    for t in (x, z, B, C_, A, Dskip, bias):
        _check(t.is_cuda, "scan2d: tensors must be CUDA tensors (no CPU fallback)")
        _check(t.dtype == x.dtype, "scan2d: all tensors must share one dtype")
        _check(t.device == x.device, "scan2d: all tensors must be on one device")
    G = S // B.shape[0]
    desc = nat.make_desc(S, H, W, N, tile=tile, params_period=P, bc_group=G, dtype=_dtype_code(x),
                         accurate=accurate, group_red=group_red)
    rc = nat.lib.scan2d_check_desc(C.byref(desc))
    if rc == nat.EINVAL:
        raise ValueError(nat.status_string(rc))
    if rc != nat.OK:
        raise nat.Scan2dError(rc, "scan2d_check_desc")
    return desc


def tiled_scan_2d_forward(x, z, B, C_, A, Dskip, bias, tile: int = 16, threads: int = 1,
                          save_residuals: bool = True, carries: bool = False,
                          counter=None, accurate: bool = False, group_red: bool = False) -> TiledForwardResult:
    """Batched ``tiled_scan_2d_forward`` (engine.hpp:88-94) on the GPU.

    ``accurate``: SCAN2D_FLAG_ACCURATE; ``group_red``: SCAN2D_FLAG_GROUP_RED
    for the backward of shared-B/C layouts (kept in ``saved``'s descriptor).

    ``counter`` (a dict) is filled with the reference element-transfer model
    (engine.cpp:222-229 == memsim.cpp:38-71) when given."""
    del threads  # results are thread-invariant by construction
    x, z, B, C_, A, Dskip, bias = _normalise(x, z, B, C_, A, Dskip, bias)
    x, z, B, C_, A, Dskip, bias = [t.contiguous() for t in (x, z, B, C_, A, Dskip, bias)]
    desc = make_desc_for(x, z, B, C_, A, Dskip, bias, tile, accurate, group_red)
    S, H, W = x.shape
    N = B.shape[3]
    dev = x.device
    y = torch.empty((S, H, W), dtype=x.dtype, device=dev)
    ph = pv = None
    if carries:
        kh, kw = -(-H // tile), -(-W // tile)
        ph = torch.empty((S, kh, kw, tile, N), dtype=x.dtype, device=dev)
        pv = torch.empty_like(ph)
    residual = None
    if save_residuals:
        residual = torch.empty(nat.lib.scan2d_residual_bytes(C.byref(desc)), dtype=torch.uint8, device=dev)
    wsb = nat.lib.scan2d_workspace_bytes(C.byref(desc), nat.OP_FWD)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        rc = nat.lib.scan2d_forward(C.byref(desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A), _ptr(Dskip),
                                    _ptr(bias), _ptr(y), _ptr(ph), _ptr(pv), _ptr(residual), _ptr(ws), wsb,
                                    _stream(dev))
    if rc == nat.EINVAL:
        raise ValueError(nat.status_string(rc))
    if rc != nat.OK:
        raise nat.Scan2dError(rc, "scan2d_forward")
    if counter is not None:
        _charge_counter(counter, S, H, W, N, tile)
    saved = SavedForward()
    if save_residuals:
        saved = SavedForward(x, z, B, C_, A, Dskip, bias, residual, desc, True)
    return TiledForwardResult(y=y, saved=saved, ph=ph, pv=pv)


def tiled_scan_2d_backward(saved: SavedForward, dy: torch.Tensor, threads: int = 1) -> GradBundle:
    """Batched ``tiled_scan_2d_backward`` (engine.hpp:100-102) on the GPU."""
    del threads
    if saved is None or not saved.valid:
        raise RuntimeError("tiled_scan_2d_backward: stale saved forward state")
    x = saved.x
    if dy.dim() == 2:
        dy = dy.unsqueeze(0)
    if tuple(dy.shape) != tuple(x.shape):
        raise ValueError("tiled_scan_2d_backward: dy shape mismatch")
    dy = dy.contiguous()
    _check(dy.dtype == x.dtype and dy.device == x.device, "dy must match the forward's dtype/device")
    desc = saved.desc
    S, H, W = x.shape
    N = saved.B.shape[3]
    P = saved.A.shape[0]
    dev = x.device
    dx = torch.empty_like(x)
    dz = torch.empty_like(x)
    dB = torch.empty_like(saved.B)
    dC = torch.empty_like(saved.C)
    dA = torch.empty((P, N), dtype=x.dtype, device=dev)
    dD = torch.empty((P,), dtype=x.dtype, device=dev)
    dbias = torch.empty((P,), dtype=x.dtype, device=dev)
    wsb = nat.lib.scan2d_workspace_bytes(C.byref(desc), nat.OP_BWD)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        rc = nat.lib.scan2d_backward(C.byref(desc), _ptr(x), _ptr(saved.z), _ptr(saved.B), _ptr(saved.C),
                                     _ptr(saved.A), _ptr(saved.Dskip), _ptr(saved.bias), _ptr(saved.residual),
                                     _ptr(dy), _ptr(dx), _ptr(dz), _ptr(dA), _ptr(dB), _ptr(dC), _ptr(dD),
                                     _ptr(dbias), _ptr(ws), wsb, _stream(dev))
    if rc == nat.ESTALE:
        raise RuntimeError("tiled_scan_2d_backward: " + nat.status_string(rc))
    if rc == nat.EINVAL:
        raise ValueError(nat.status_string(rc))
    if rc != nat.OK:
        raise nat.Scan2dError(rc, "scan2d_backward")
    return GradBundle(dx=dx, dz_raw=dz, da=dA, db=dB, dc=dC, dd=dD, dbias=dbias)


def _charge_counter(counter: dict, S, H, W, N, t):
    """Reference counting model per tile (engine.cpp:222-229), summed over S scans."""
    kh, kw = -(-H // t), -(-W // t)
    flat = -(-(t * t) // 32) * 32
    cells = H * W
    add = dict(payload_reads=S * (2 * cells + 2 * cells * N), payload_writes=S * cells,
               intermediate_traffic=0, carry_traffic=S * kh * kw * 4 * t * N,
               padding_elements=S * 2 * N * (kh * kw * flat - cells))
    for k, v in add.items():
        counter[k] = counter.get(k, 0) + v


class Scan2dOp:
    """Preallocated forward+backward for a fixed descriptor: keeps the
    workspaces, residual and output buffers across calls so a training loop
    enqueues exactly the library's kernels (no allocator traffic).

    ``accurate`` sets SCAN2D_FLAG_ACCURATE (fp32 exponentials by polynomial);
    ``group_red`` sets SCAN2D_FLAG_GROUP_RED (bc_group > 1: dB / dC summed in
    place by L2 reductions -- faster, summation order not fixed)."""

    def __init__(self, S, H, W, N, tile=16, params_period=None, bc_group=1, dtype=torch.float32,
                 device="cuda", with_backward=True, accurate=False, group_red=False):
        self.dev = torch.device(device)
        if self.dev.type == "cuda" and self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        code = nat.F64 if dtype == torch.float64 else nat.F32
        self.desc = nat.make_desc(S, H, W, N, tile=tile, params_period=params_period, bc_group=bc_group,
                                  dtype=code, accurate=accurate, group_red=group_red)
        rc = nat.lib.scan2d_check_desc(C.byref(self.desc))
        if rc != nat.OK:
            raise ValueError(nat.status_string(rc))
        P = S if params_period is None else params_period
        self.shape = (S, H, W, N, P, S // bc_group)
        e = lambda *s: torch.empty(s, dtype=dtype, device=self.dev)
        self.y = e(S, H, W)
        self.wsf_bytes = nat.lib.scan2d_workspace_bytes(C.byref(self.desc), nat.OP_FWD)
        self.wsf = torch.empty(max(self.wsf_bytes, 1), dtype=torch.uint8, device=self.dev)
        self.residual = None
        if with_backward:
            self.residual = torch.empty(nat.lib.scan2d_residual_bytes(C.byref(self.desc)), dtype=torch.uint8,
                                        device=self.dev)
            self.wsb_bytes = nat.lib.scan2d_workspace_bytes(C.byref(self.desc), nat.OP_BWD)
            self.wsb = torch.empty(max(self.wsb_bytes, 1), dtype=torch.uint8, device=self.dev)
            G = S // bc_group
            self.dx, self.dz = e(S, H, W), e(S, H, W)
            self.dB, self.dC = e(G, H, W, N), e(G, H, W, N)
            self.dA, self.dD, self.dbias = e(P, N), e(P), e(P)
        self.launches = 0
        self.check = True  # validate operands against the descriptor (benchmarks may turn it off)

    def _operands(self, x, z, B, C_, A, Dskip, bias, dy=None):
        """Shape / dtype / device / contiguity of every operand against the
        preallocated descriptor: a raw pointer goes to the C ABI, so a view or
        a wrong dtype would otherwise be read out of bounds silently."""
        S, H, W, N, P, G = self.shape
        want = [("x", x, (S, H, W)), ("z", z, (S, H, W)), ("B", B, (G, H, W, N)), ("C", C_, (G, H, W, N)),
                ("A", A, (P, N)), ("Dskip", Dskip, (P,)), ("bias", bias, (P,))]
        if dy is not None:
            want.append(("dy", dy, (S, H, W)))
        for name, t, shp in want:
            _check(isinstance(t, torch.Tensor), f"Scan2dOp: {name} must be a tensor")
            _check(tuple(t.shape) == shp, f"Scan2dOp: {name} has shape {tuple(t.shape)}, expected {shp}")
            _check(t.dtype == self.dtype, f"Scan2dOp: {name} has dtype {t.dtype}, expected {self.dtype}")
            _check(t.device == self.dev, f"Scan2dOp: {name} is on {t.device}, expected {self.dev}")
            _check(t.is_contiguous(), f"Scan2dOp: {name} must be contiguous")

    def forward(self, x, z, B, C_, A, Dskip, bias, save=True):
        if self.check:
            self._operands(x, z, B, C_, A, Dskip, bias)
        rc = nat.lib.scan2d_forward(C.byref(self.desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A), _ptr(Dskip),
                                    _ptr(bias), _ptr(self.y), None, None,
                                    _ptr(self.residual) if save else None, _ptr(self.wsf), self.wsf_bytes,
                                    _stream(self.dev))
        if rc != nat.OK:
            raise nat.Scan2dError(rc, "scan2d_forward")
        self.launches += nat.lib.scan2d_last_launch_count()
        return self.y

    def backward(self, x, z, B, C_, A, Dskip, bias, dy):
        if self.check:
            self._operands(x, z, B, C_, A, Dskip, bias, dy)
        rc = nat.lib.scan2d_backward(C.byref(self.desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A),
                                     _ptr(Dskip), _ptr(bias), _ptr(self.residual), _ptr(dy), _ptr(self.dx),
                                     _ptr(self.dz), _ptr(self.dA), _ptr(self.dB), _ptr(self.dC), _ptr(self.dD),
                                     _ptr(self.dbias), _ptr(self.wsb), self.wsb_bytes, _stream(self.dev))
        if rc != nat.OK:
            raise nat.Scan2dError(rc, "scan2d_backward")
        self.launches += nat.lib.scan2d_last_launch_count()
        return self.dx, self.dz, self.dA, self.dB, self.dC, self.dD, self.dbias

    def plan(self) -> dict:
        return nat.plan_info(self.desc)


class Scan2dFunction(torch.autograd.Function):
    """Autograd binding: y = scan2d(x, z, B, C, A, Dskip, bias)."""

    @staticmethod
    def forward(ctx, x, z, B, C_, A, Dskip, bias, tile: int = 16):
        res = tiled_scan_2d_forward(x, z, B, C_, A, Dskip, bias, tile=tile, save_residuals=True)
        ctx.saved_fwd = res.saved
        ctx.shapes = (x.shape, z.shape, B.shape, C_.shape, A.shape, Dskip.shape, bias.shape)
        return res.y.reshape(x.shape)

    @staticmethod
    def backward(ctx, dy):
        g = tiled_scan_2d_backward(ctx.saved_fwd, dy.reshape(ctx.saved_fwd.x.shape))
        shapes = ctx.shapes
        outs = (g.dx, g.dz_raw, g.db, g.dc, g.da, g.dd, g.dbias)
        return tuple(o.reshape(s) for o, s in zip(outs, shapes)) + (None,)


def scan2d(x, z, B, C_, A, Dskip, bias, tile: int = 16):
    return Scan2dFunction.apply(x, z, B, C_, A, Dskip, bias, tile)


class Scan2dBandOp:
    """One row band of a taller grid (SURVEY.md §8e row-band shard) over the
    C ABI's ``scan2d_forward_band`` / ``scan2d_backward_band``.

    ``forward`` takes ``h_top`` [S,W,N] (h of the row above the band; None for
    the first band) and returns ``(y, h_bottom)``; ``backward`` takes the same
    ``h_top``, ``dy`` and ``g_bottom`` (Abar G of the row below; None for the last
    band) and returns ``(dx, dz, dA, dB, dC, dD, dbias, g_top)``.  dA / dD / dbias
    are this band's partial sums.  Buffers are preallocated per descriptor."""

    def __init__(self, S, H, W, N, tile=16, dtype=torch.float32, device="cuda", with_backward=True):
        self.op = Scan2dOp(S, H, W, N, tile=tile, dtype=dtype, device=device, with_backward=with_backward)
        e = lambda *s: torch.empty(s, dtype=dtype, device=self.op.dev)
        self.h_bottom = e(S, W, N)
        self.g_top = e(S, W, N) if with_backward else None
        self.launches = 0

    @property
    def desc(self):
        return self.op.desc

    def _carry(self, t, name):
        if t is not None:
            S, H, W, N, _, _ = self.op.shape
            _check(tuple(t.shape) == (S, W, N) and t.dtype == self.op.dtype and t.device == self.op.dev
                   and t.is_contiguous(), f"Scan2dBandOp: {name} must be a contiguous [S,W,N] tensor "
                                          "of the op's dtype on its device")

    def forward(self, x, z, B, C_, A, Dskip, bias, h_top=None, save=True, link=None, h_bottom=None):
        """``link`` = (in_flags, out_flags, seq) selects the in-kernel hand-off
        (``scan2d_forward_band_linked``): flags as tensors or raw device
        pointers (ints, e.g. peer memory), ``h_bottom`` a tensor or raw pointer
        to write the band's last-row carry to (default: this op's buffer)."""
        o = self.op
        if o.check:
            o._operands(x, z, B, C_, A, Dskip, bias)
            self._carry(h_top, "h_top")
        if link is not None:
            lin, lout, seq = link
            hb = self.h_bottom if h_bottom is None else h_bottom
            rc = nat.lib.scan2d_forward_band_linked(
                C.byref(o.desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A), _ptr(Dskip), _ptr(bias),
                _ptr(h_top), _ptr(o.y), _vptr(hb), _ptr(o.residual) if save else None, _vptr(lin), _vptr(lout),
                int(seq), _ptr(o.wsf), o.wsf_bytes, _stream(o.dev))
            if rc != nat.OK:
                raise nat.Scan2dError(rc, "scan2d_forward_band_linked")
            self.launches += nat.lib.scan2d_last_launch_count()
            return o.y, hb
        rc = nat.lib.scan2d_forward_band(C.byref(o.desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A),
                                         _ptr(Dskip), _ptr(bias), _ptr(h_top), _ptr(o.y), _ptr(self.h_bottom),
                                         _ptr(o.residual) if save else None, _ptr(o.wsf), o.wsf_bytes,
                                         _stream(o.dev))
        if rc != nat.OK:
            raise nat.Scan2dError(rc, "scan2d_forward_band")
        self.launches += nat.lib.scan2d_last_launch_count()
        return o.y, self.h_bottom

    def backward(self, x, z, B, C_, A, Dskip, bias, h_top, dy, g_bottom=None, link=None, g_top=None):
        """``link`` = (in_flags, out_flags, seq): in-kernel hand-off
        (``scan2d_backward_band_linked``); ``g_top`` a tensor or raw pointer."""
        o = self.op
        if o.check:
            o._operands(x, z, B, C_, A, Dskip, bias, dy)
            self._carry(h_top, "h_top")
            if link is None:
                self._carry(g_bottom, "g_bottom")
        if link is not None:
            lin, lout, seq = link
            gt = self.g_top if g_top is None else g_top
            rc = nat.lib.scan2d_backward_band_linked(
                C.byref(o.desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A), _ptr(Dskip), _ptr(bias),
                _ptr(h_top), _ptr(o.residual), _ptr(dy), _vptr(g_bottom), _ptr(o.dx), _ptr(o.dz), _ptr(o.dA),
                _ptr(o.dB), _ptr(o.dC), _ptr(o.dD), _ptr(o.dbias), _vptr(gt), _vptr(lin), _vptr(lout), int(seq),
                _ptr(o.wsb), o.wsb_bytes, _stream(o.dev))
            if rc != nat.OK:
                raise nat.Scan2dError(rc, "scan2d_backward_band_linked")
            self.launches += nat.lib.scan2d_last_launch_count()
            return o.dx, o.dz, o.dA, o.dB, o.dC, o.dD, o.dbias, gt
        rc = nat.lib.scan2d_backward_band(C.byref(o.desc), _ptr(x), _ptr(z), _ptr(B), _ptr(C_), _ptr(A),
                                          _ptr(Dskip), _ptr(bias), _ptr(h_top), _ptr(o.residual), _ptr(dy),
                                          _ptr(g_bottom), _ptr(o.dx), _ptr(o.dz), _ptr(o.dA), _ptr(o.dB),
                                          _ptr(o.dC), _ptr(o.dD), _ptr(o.dbias), _ptr(self.g_top), _ptr(o.wsb),
                                          o.wsb_bytes, _stream(o.dev))
        if rc != nat.OK:
            raise nat.Scan2dError(rc, "scan2d_backward_band")
        self.launches += nat.lib.scan2d_last_launch_count()
        return o.dx, o.dz, o.dA, o.dB, o.dC, o.dD, o.dbias, self.g_top


def train_host(x, z, B, C_, A, Dskip, bias, dy=None, outs=None, chunks: int = 0, tile: int = 16,
               sync: bool = True, group_red: bool = False):
    """One training step with HOST (CPU, ideally pinned) tensors through the C
    ABI's ``scan2d_train_host``: chunked host->device copies, kernels and
    device->host copies overlap on three streams of the current device.
    Returns ``outs`` = (y, dx, dz, dA, dB, dC, dD, dbias) as host tensors
    (gradients None when ``dy`` is None).  B / C may be shared by groups of G
    scans ([S/G,H,W,N]) and A / Dskip / bias by the period P ([P,N], [P]) --
    the model layout; chunks are then cut at whole groups / periods.  With
    ``sync=False`` the call returns as soon as the work is enqueued and the
    outputs are valid only after ``torch.cuda.current_stream().synchronize()``."""
    _check(x.dim() == 3, "train_host: x must be [S,H,W]")
    S, H, W = x.shape
    _check(B.dim() == 4 and B.shape[0] >= 1 and S % B.shape[0] == 0, "train_host: B must be [S/G,H,W,N]")
    _check(A.dim() == 2 and A.shape[0] >= 1 and S % A.shape[0] == 0, "train_host: A must be [P,N], P dividing S")
    N = B.shape[-1]
    SB, P = B.shape[0], A.shape[0]
    ins = [("x", x, (S, H, W)), ("z", z, (S, H, W)), ("B", B, (SB, H, W, N)), ("C", C_, (SB, H, W, N)),
           ("A", A, (P, N)), ("Dskip", Dskip, (P,)), ("bias", bias, (P,))]
    if dy is not None:
        ins.append(("dy", dy, (S, H, W)))
    _check(x.dtype in (torch.float32, torch.float64), "train_host: dtype must be float32 or float64")
    for name, t, shp in ins:
        _check(tuple(t.shape) == shp, f"train_host: {name} has shape {tuple(t.shape)}, expected {shp}")
        _check(t.dtype == x.dtype, f"train_host: {name} must be {x.dtype}")
        _check(t.device.type == "cpu", f"train_host: {name} must be a host tensor")
        _check(t.is_contiguous(), f"train_host: {name} must be contiguous")
    code = nat.F64 if x.dtype == torch.float64 else nat.F32
    desc = nat.make_desc(S, H, W, N, tile=tile, params_period=P, bc_group=S // SB, dtype=code,
                         group_red=group_red)
    if outs is None:
        e = lambda *s: torch.empty(s, dtype=x.dtype).pin_memory()
        outs = (e(S, H, W),) + ((e(S, H, W), e(S, H, W), e(P, N), e(SB, H, W, N), e(SB, H, W, N), e(P), e(P))
                                if dy is not None else (None,) * 7)
    oshapes = [(S, H, W), (S, H, W), (S, H, W), (P, N), (SB, H, W, N), (SB, H, W, N), (P,), (P,)]
    for k, (t, shp) in enumerate(zip(outs, oshapes)):
        if k > 0 and dy is None:
            continue
        _check(t is not None and tuple(t.shape) == shp and t.dtype == x.dtype and t.device.type == "cpu"
               and t.is_contiguous(), f"train_host: output {k} must be a contiguous host {shp} tensor")
    dev = torch.device("cuda", torch.cuda.current_device())
    rc = nat.lib.scan2d_train_host(C.byref(desc), *[_ptr(t) for t in (x, z, B, C_, A, Dskip, bias, dy)],
                                   *[_ptr(t) for t in outs], int(chunks), _stream(dev))
    if rc != nat.OK:
        raise nat.Scan2dError(rc, "scan2d_train_host")
    if sync:
        torch.cuda.current_stream(dev).synchronize()
    return outs
