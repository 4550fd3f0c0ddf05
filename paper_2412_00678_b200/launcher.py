"""Multi-GPU launcher: one process per GPU, scans sharded across ranks.

SURVEY.md §8(e): the S = B x D scans are independent (engine.cpp has no
cross-call state), so the (batch x channel) space is partitioned into
contiguous per-rank ranges and every rank runs the single-GPU operator on its
own range -- no collective on the hot path (weak scaling).  Collectives are
used only off the timed path (gathering results for parity, max-reducing
timings).

Shard boundaries respect the layout quanta of the C ABI: parameters repeat
with period P (scan s uses row s % P) and B/C are shared by groups of G scans,
so every shard starts at a multiple of lcm(P', G) where P' = P when the
parameter table is per channel; a shard then sees the same parameter rows and
whole B/C groups as the global problem.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    s0: int  # first scan (inclusive)
    s1: int  # last scan (exclusive)

    @property
    def count(self) -> int:
        return self.s1 - self.s0


def shard_range(S: int, world: int, rank: int, quantum: int = 1) -> Shard:
    """Contiguous, quantum-aligned split of [0, S) over `world` ranks.

    Units of `quantum` scans are dealt as evenly as possible (the first
    `units % world` ranks get one extra unit); ranks may get an empty range
    when S / quantum < world."""
    if S < 1 or world < 1 or not (0 <= rank < world) or quantum < 1:
        raise ValueError("shard_range: bad arguments")
    if S % quantum:
        raise ValueError(f"shard_range: S={S} is not a multiple of the layout quantum {quantum}")
    units = S // quantum
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return Shard(rank, world, u0 * quantum, u1 * quantum)


def layout_quantum(S: int, params_period: int, bc_group: int) -> int:
    """Smallest shard granularity that keeps parameter rows and B/C groups intact."""
    p = params_period if params_period < S else 1  # per-scan params: any split works
    return math.lcm(p, bc_group)


def shard_views(shard: Shard, x, z, B, C, A, Dskip, bias, params_period: int, bc_group: int):
    """Slice the global operands (torch tensors or numpy arrays with the C-ABI
    layouts) down to one shard.  Per-scan parameter tables (P == S) are sliced;
    periodic ones (P < S) are shared unchanged because shards start at
    multiples of P."""
    S = x.shape[0]
    s0, s1 = shard.s0, shard.s1
    g0, g1 = s0 // bc_group, s1 // bc_group
    if params_period == S:
        A, Dskip, bias = A[s0:s1], Dskip[s0:s1], bias[s0:s1]
    return x[s0:s1], z[s0:s1], B[g0:g1], C[g0:g1], A, Dskip, bias


class ShardedScan2d:
    """Batch shard of ONE global problem (S scans, H x W, N states, parameter
    period P, B/C group G) over `world` ranks, one GPU each (
    BASELINE configs[3] "batch-sharded over 2/4/8 GPUs").

    Rank r owns the contiguous, layout-quantum-aligned scan range
    ``shard_range(S, world, r, layout_quantum(S, P, G))`` and runs the
    single-GPU operator on it (``op_factory(S_local, P_local, G)``, by default
    a preallocated ``Scan2dOp``).  The data path has no collective: scans are
    independent.  Off the timed path, ``gather`` assembles per-scan outputs on
    every rank (all_gather of equal-sized padded blocks) and
    ``reduce_shared_params`` sums the per-rank partial gradients of shared
    parameter rows (P < S) in rank order (deterministic)."""

    def __init__(self, S, H, W, N, rank, world, params_period=None, bc_group=1, op_factory=None, dist=None,
                 **op_kwargs):
        self.S, self.H, self.W, self.N = S, H, W, N
        self.P = S if params_period is None else params_period
        self.G = bc_group
        self.rank, self.world, self.dist = rank, world, dist
        self.quantum = layout_quantum(S, self.P, self.G)
        self.shard = shard_range(S, world, rank, self.quantum)
        self.shards = [shard_range(S, world, r, self.quantum) for r in range(world)]
        self.per_scan_params = self.P == S
        self.P_local = self.shard.count if self.per_scan_params else self.P
        if op_factory is None:
            from .api import Scan2dOp

            def op_factory(s_loc, p_loc, g):
                return Scan2dOp(s_loc, H, W, N, params_period=p_loc, bc_group=g, **op_kwargs)
        self.op = op_factory(self.shard.count, self.P_local, self.G) if self.shard.count > 0 else None

    def views(self, x, z, B, C, A, Dskip, bias):
        """This rank's slices of the global operands (C-ABI layouts)."""
        return shard_views(self.shard, x, z, B, C, A, Dskip, bias, self.P, self.G)

    def forward(self, *shard_ins, **kw):
        if self.op is None:  # empty shard (fewer layout quanta than ranks)
            return shard_ins[0].new_empty((0, self.H, self.W))
        return self.op.forward(*shard_ins, **kw)

    def backward(self, *shard_ins_and_dy):
        if self.op is None:
            x, A = shard_ins_and_dy[0], shard_ins_and_dy[4]
            e = lambda *s: x.new_zeros(s)  # noqa: E731
            p = 0 if self.per_scan_params else self.P
            H, W, N = self.H, self.W, self.N
            return e(0, H, W), e(0, H, W), A.new_zeros((p, N)), e(0, H, W, N), e(0, H, W, N), e(p), e(p)
        return self.op.backward(*shard_ins_and_dy)

    def gather(self, t, scans_per_row=1):
        """All-gather a per-scan output (leading dim = this rank's scans //
        scans_per_row, e.g. G for dB / dC) into the global tensor on every rank."""
        import torch

        counts = [sh.count // scans_per_row for sh in self.shards]
        if self.world == 1 or self.dist is None:
            return t
        m = max(counts)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(bufs, pad)
        return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)

    def gather_grads(self, grads):
        """(dx, dz, dA, dB, dC, dD, dbias) of this shard -> the global bundle:
        per-scan groups concatenated in scan order; shared parameter rows
        (P < S) summed over ranks in rank order."""
        dx, dz, dA, dB, dC, dD, dbias = grads
        out = [self.gather(dx), self.gather(dz)]
        if self.per_scan_params:
            pA, pD, pb = self.gather(dA), self.gather(dD), self.gather(dbias)
        else:
            pA, pD, pb = self.reduce_shared_params([dA, dD, dbias])
        out += [pA, self.gather(dB, self.G), self.gather(dC, self.G), pD, pb]
        return out

    def reduce_shared_params(self, parts):
        if self.world == 1 or self.dist is None:
            return parts
        return reduce_params(self.dist, parts, self.world)


# ---------------------------------------------------------------- row bands
#
# Optional row-band shard of ONE giant scan: rank r
# owns rows [r*H/world, (r+1)*H/world).  The vertical carry P^v (h of the
# previous band's last row, W x N per scan) is the only forward exchange; it
# flows r -> r+1.  The host-side plan below is what each rank executes; the
# exchange itself is a device-to-device copy over NVLink (peer access) or an
# NCCL send/recv, issued by bench / user code between the band launches.


@dataclass(frozen=True)
class RowBand:
    rank: int
    world: int
    r0: int
    r1: int

    @property
    def rows(self) -> int:
        return self.r1 - self.r0


def row_band(H: int, world: int, rank: int, align: int = 1) -> RowBand:
    """Rows of `rank`'s band: units of `align` rows dealt as evenly as possible
    (the last band takes the remainder).  Aligning bands to the kernels' tile
    height (32 * SH / N rows) makes the banded result bit-identical to the
    single-GPU one (include/scan2d_cuda.h, scan2d_forward_band)."""
    if H < world or align < 1:
        raise ValueError("row_band: fewer rows than ranks")
    units = -(-H // align)
    if units < world:
        raise ValueError("row_band: fewer aligned row units than ranks")
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return RowBand(rank, world, u0 * align, min(H, u1 * align))


def band_align(N: int, dtype_bytes: int = 4) -> int:
    """Tile height of the tile kernels: R = 32 * SH / N (SH = 2 fp32, 1 fp64)."""
    sh = 2 if dtype_bytes == 4 else 1
    return max(1, 32 * sh // N) if N in (4, 8, 16, 32) else 1


def row_band_schedule(H: int, world: int):
    """Ordered (sender, receiver, boundary_row) list of forward carry hand-offs:
    rank r sends h(r1 - 1, :, :) of its band to rank r + 1."""
    out = []
    for r in range(world - 1):
        b = row_band(H, world, r)
        out.append((r, r + 1, b.r1 - 1))
    return out


class RowBandPipeline:
    """Row-band shard of a batch of scans over `world` ranks (one GPU each).

    Rank r owns rows [r0, r1) of every scan (row_band) and runs ``op`` -- an
    object with ``forward(ins, h_top) -> (y, h_bottom)`` and ``backward(ins,
    h_top, dy, g_bottom) -> (grads..., g_top)`` for one chunk of scans, e.g. a
    ``Scan2dBandOp`` per chunk.  The only exchanges are the vertical carries:
    forward h_bottom of rank r -> h_top of rank r+1, backward g_top of rank r+1
    -> g_bottom of rank r, [S_chunk, W, N] per chunk, as point-to-point
    send/recv (NCCL over NVLink on GPUs, gloo on CPU).  The S scans are split
    into chunks so the ranks work as a pipeline: rank r computes chunk k while
    rank r+1 computes chunk k-1; efficiency nchunks / (nchunks + world - 1).
    Band partial sums of dA / dD / dbias are reduced over ranks in rank order
    by the caller (``reduce_params``)."""

    def __init__(self, rank: int, world: int, dist=None, streams=None):
        self.rank, self.world, self.dist = rank, world, dist
        self.streams = streams  # optional pool of torch.cuda.Stream (one chunk per stream)
        self.h_tops = {}

    def _ctx(self, k):
        import contextlib

        import torch

        if self.streams is None:
            return contextlib.nullcontext()
        return torch.cuda.stream(self.streams[k % len(self.streams)])

    def forward(self, op, chunks, carry_shape, make_empty, keep=True):
        """chunks: list of per-chunk input tuples; carry_shape(k) -> (S_k, W, N);
        make_empty(shape) -> tensor for received carries.  Returns per-chunk y.
        On GPUs every chunk runs on its own stream of the pool, so chunks overlap
        on the device and the receive of chunk k+1 overlaps chunk k's kernels."""
        ys, pending = [], []
        for k, ins in enumerate(chunks):
            with self._ctx(k):
                h_top = None
                if self.rank > 0:
                    h_top = make_empty(carry_shape(k))
                    self.dist.irecv(h_top, src=self.rank - 1).wait()
                self.h_tops[k] = h_top
                y, h_bot = op(k).forward(*ins, h_top=h_top)
                if keep:
                    ys.append(y.clone())
                if self.rank < self.world - 1:
                    pending.append(self.dist.isend(h_bot, dst=self.rank + 1))
        for p in pending:
            p.wait()
        self._join()
        return ys

    def backward(self, op, chunks, dys, carry_shape, make_empty, keep=True):
        """Reverse carries; returns per-chunk gradient tuples (band partial sums
        for the parameter gradients)."""
        outs, pending = [], []
        for k, ins in enumerate(chunks):
            with self._ctx(k):
                g_bot = None
                if self.rank < self.world - 1:
                    g_bot = make_empty(carry_shape(k))
                    self.dist.irecv(g_bot, src=self.rank + 1).wait()
                res = op(k).backward(*ins, h_top=self.h_tops.get(k), dy=dys[k], g_bottom=g_bot)
                *grads, g_top = res
                if keep:
                    outs.append(tuple(g.clone() for g in grads))
                if self.rank > 0:
                    pending.append(self.dist.isend(g_top, dst=self.rank - 1))
        for p in pending:
            p.wait()
        self._join()
        return outs

    def _join(self):
        if self.streams is not None:
            import torch

            cur = torch.cuda.current_stream()
            for st in self.streams:
                cur.wait_stream(st)


def reduce_params(dist, parts, world: int):
    """Deterministic sum of per-rank parameter-gradient partials (dA, dD, dbias):
    gather to every rank, add in rank order."""
    import torch

    out = []
    for t in parts:
        bufs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(bufs, t.contiguous())
        acc = bufs[0].clone()
        for b in bufs[1:]:
            acc += b
        out.append(acc)
    return out


class LinkedRowBands:
    """Row-band shard with the carry hand-off done inside the kernels
    (``scan2d_forward_band_linked`` / ``scan2d_backward_band_linked``; SURVEY.md
    §8e): rank r owns rows ``row_band(H, world, r, band_align(N))`` of all S
    scans on its own GPU.

    Setup (off the hot path): every rank allocates its receive buffers --
    ``h_top`` [S,W,N] plus forward flags (written by rank r-1) and ``g_bottom``
    [S,W,N] plus backward flags (written by rank r+1) -- exports them as CUDA
    IPC handles, all-gathers the handles over ``dist`` and opens its
    neighbours'.  A forward then stores each (scan, 16-column strip)'s last-row
    state straight into rank r+1's ``h_top`` over NVLink and releases rank
    r+1's flag for that strip; rank r+1's strip acquires the flag right before
    it first reads ``h_top``.  The backward does the same upwards with
    ``Abar G``.  Per call: kernels only -- no host synchronisation, no
    collective, no scan-chunk pipeline; strips start as soon as their
    producer strip is done.

    Ordering across calls: a producer must not overwrite a receive buffer
    before the consumer has read it.  In a training step (forward, then
    backward) the backward's reverse hand-off orders the next forward after
    the consumer's forward; forward-only loops call ``step_barrier()``
    between steps."""

    def __init__(self, S, H, W, N, rank, world, dist=None, device="cuda", dtype=None, with_backward=True):
        import torch

        from . import _native as nat
        from .api import Scan2dBandOp

        self.nat, self.torch = nat, torch
        self.rank, self.world, self.dist = rank, world, dist
        dtype = torch.float32 if dtype is None else dtype
        self.band = row_band(H, world, rank, band_align(N, 4 if dtype == torch.float32 else 8))
        self.S, self.W, self.N = S, W, N
        self.op = Scan2dBandOp(S, self.band.rows, W, N, dtype=dtype, device=device, with_backward=with_backward)
        self.strips = nat.lib.scan2d_band_strips(ctypes_byref(self.op.desc))
        dev = self.op.op.dev
        self.h_top = torch.zeros((S, W, N), dtype=dtype, device=dev) if rank > 0 else None
        self.g_bottom = torch.zeros((S, W, N), dtype=dtype, device=dev) if rank < world - 1 else None
        self.f_in = torch.zeros(S * self.strips, dtype=torch.int32, device=dev) if rank > 0 else None
        self.b_in = torch.zeros(S * self.strips, dtype=torch.int32, device=dev) if rank < world - 1 else None
        self._opened = []
        self.peer = {"h_next": None, "f_next": None, "g_prev": None, "b_prev": None}
        if world > 1:
            mine = {k: (self._export(t) if t is not None else None)
                    for k, t in (("h_top", self.h_top), ("f_in", self.f_in), ("g_bottom", self.g_bottom),
                                 ("b_in", self.b_in))}
            allh = [None] * world
            dist.all_gather_object(allh, mine)
            if rank < world - 1:
                self.peer["h_next"] = self._open(allh[rank + 1]["h_top"])
                self.peer["f_next"] = self._open(allh[rank + 1]["f_in"])
            if rank > 0:
                self.peer["g_prev"] = self._open(allh[rank - 1]["g_bottom"])
                self.peer["b_prev"] = self._open(allh[rank - 1]["b_in"])
        self.seq_f = 0
        self.seq_b = 0

    def _export(self, t):
        import ctypes as C

        h = (C.c_ubyte * 64)()
        off = C.c_uint64(0)
        rc = self.nat.lib.scan2d_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off))
        if rc != self.nat.OK:
            raise self.nat.Scan2dError(rc, "scan2d_ipc_export")
        return bytes(h), off.value

    def _open(self, exported):
        import ctypes as C

        handle, off = exported
        p, base = C.c_void_p(), C.c_void_p()
        rc = self.nat.lib.scan2d_ipc_open((C.c_ubyte * 64).from_buffer_copy(handle), off, C.byref(p), C.byref(base))
        if rc != self.nat.OK:
            raise self.nat.Scan2dError(rc, "scan2d_ipc_open")
        self._opened.append(base.value)
        return p.value

    def views(self, x, z, B, C, dy=None):
        """This rank's rows of the global per-cell operands."""
        r0, r1 = self.band.r0, self.band.r1
        out = [t[:, r0:r1].contiguous() for t in (x, z, B, C)]
        if dy is not None:
            out.append(dy[:, r0:r1].contiguous())
        return out

    def forward(self, x, z, B, C, A, Dskip, bias, save=True):
        self.seq_f += 1
        link = (self.f_in, self.peer["f_next"], self.seq_f)
        y, _ = self.op.forward(x, z, B, C, A, Dskip, bias, h_top=self.h_top, save=save, link=link,
                               h_bottom=self.peer["h_next"])
        return y

    def backward(self, x, z, B, C, A, Dskip, bias, dy):
        """Gradients of this band; dA / dDskip / dbias are band partial sums
        (``reduce_params`` adds them over ranks in rank order)."""
        self.seq_b += 1
        link = (self.b_in, self.peer["b_prev"], self.seq_b)
        out = self.op.backward(x, z, B, C, A, Dskip, bias, self.h_top, dy, g_bottom=self.g_bottom, link=link,
                               g_top=self.peer["g_prev"])
        return out[:-1]

    def step_barrier(self):
        self.torch.cuda.current_stream(self.op.op.dev).synchronize()
        if self.dist is not None and self.world > 1:
            self.dist.barrier()

    def close(self):
        for p in self._opened:
            self.nat.lib.scan2d_ipc_close(ctypes_vp(p))
        self._opened = []


def ctypes_byref(x):
    import ctypes as C

    return C.byref(x)


def ctypes_vp(p):
    import ctypes as C

    return C.c_void_p(p)
