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
