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


def row_band(H: int, world: int, rank: int) -> RowBand:
    if H < world:
        raise ValueError("row_band: fewer rows than ranks")
    base, extra = divmod(H, world)
    r0 = rank * base + min(rank, extra)
    return RowBand(rank, world, r0, r0 + base + (1 if rank < extra else 0))


def row_band_schedule(H: int, world: int):
    """Ordered (sender, receiver, boundary_row) list of forward carry hand-offs:
    rank r sends h(r1 - 1, :, :) of its band to rank r + 1."""
    out = []
    for r in range(world - 1):
        b = row_band(H, world, r)
        out.append((r, r + 1, b.r1 - 1))
    return out
