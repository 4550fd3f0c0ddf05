"""Row-band shard: band planning, the numpy band restatement
against the oracle, the gloo world-size-2 pipeline (CPU), and the CUDA band
entry points chained on one GPU against the single-band result (-m gpu)."""
import os

import numpy as np
import pytest
import torch

from band_ref import band_backward, band_forward
from oracle_lib import Oracle, rel_error
from paper_2412_00678_b200.launcher import RowBandPipeline, band_align, reduce_params, row_band
from scan_cases import make_batch, oracle_bwd, oracle_fwd


def _inputs(b, s0=0, s1=None, r0=0, r1=None):
    s1 = b.S if s1 is None else s1
    r1 = b.H if r1 is None else r1
    return (b.x[s0:s1, r0:r1], b.z[s0:s1, r0:r1], b.B[s0:s1, r0:r1], b.C[s0:s1, r0:r1], b.A[s0:s1], b.D[s0:s1],
            b.bias[s0:s1])


def test_row_band_plan_covers_rows_aligned():
    for H, world, al in [(1024, 8, 4), (200, 3, 4), (37, 2, 1), (64, 8, 8)]:
        bands = [row_band(H, world, r, al) for r in range(world)]
        assert bands[0].r0 == 0 and bands[-1].r1 == H
        for a, b in zip(bands, bands[1:]):
            assert a.r1 == b.r0 and a.r1 % al == 0
    assert band_align(16) == 4 and band_align(4) == 16 and band_align(16, 8) == 2 and band_align(1) == 1
    with pytest.raises(ValueError):
        row_band(3, 4, 0)


def test_band_reference_matches_oracle():
    orc = Oracle()
    b = make_batch(orc, 3, 9, 7, 4, seed0=31, dtype="f64")
    y, _ = band_forward(*_inputs(b))
    assert rel_error(y, oracle_fwd(orc, b, "f64")) < 1e-12
    dx, dz, dA, dB, dC, dD, dbias, _ = band_backward(*_inputs(b), None, b.dy)
    ref = oracle_bwd(orc, b, "f64")
    for k, v in dict(dx=dx, dz=dz, dA=dA, dB=dB, dC=dC, dD=dD, dbias=dbias).items():
        assert rel_error(v, ref[k]) < 1e-11, k


def test_band_chain_equals_full_grid():
    orc = Oracle()
    b = make_batch(orc, 2, 12, 5, 3, seed0=7, dtype="f64")
    y_full, _ = band_forward(*_inputs(b))
    full = band_backward(*_inputs(b), None, b.dy)
    cuts = [0, 4, 5, 12]
    ys, tops = [], [None]
    for r0, r1 in zip(cuts, cuts[1:]):
        y, hb = band_forward(*_inputs(b, r0=r0, r1=r1), tops[-1])
        ys.append(y)
        tops.append(hb)
    np.testing.assert_allclose(np.concatenate(ys, axis=1), y_full, rtol=1e-13, atol=1e-13)
    g = None
    parts = []
    for k in range(len(cuts) - 2, -1, -1):
        r0, r1 = cuts[k], cuts[k + 1]
        out = band_backward(*_inputs(b, r0=r0, r1=r1), tops[k], b.dy[:, r0:r1], g)
        g = out[-1]
        parts.append((r0, r1, out))
    for idx, name in [(0, "dx"), (1, "dz"), (3, "dB"), (4, "dC")]:
        got = np.concatenate([o[idx] for _, _, o in sorted(parts)], axis=1)
        np.testing.assert_allclose(got, full[idx], rtol=1e-12, atol=1e-12, err_msg=name)
    for idx in (2, 5, 6):
        np.testing.assert_allclose(sum(o[idx] for _, _, o in parts), full[idx], rtol=1e-12, atol=1e-12)


class _NumpyBandOp:
    """CPU compute backend for the gloo pipeline test (test infrastructure)."""

    def forward(self, x, z, B, C, A, D, bias, h_top=None):
        y, hb = band_forward(*[t.numpy() for t in (x, z, B, C, A, D, bias)],
                             None if h_top is None else h_top.numpy())
        return torch.from_numpy(y), torch.from_numpy(hb)

    def backward(self, x, z, B, C, A, D, bias, h_top=None, dy=None, g_bottom=None):
        out = band_backward(*[t.numpy() for t in (x, z, B, C, A, D, bias)],
                            None if h_top is None else h_top.numpy(), dy.numpy(),
                            None if g_bottom is None else g_bottom.numpy())
        return tuple(torch.from_numpy(np.ascontiguousarray(o)) for o in out)


def _gloo_worker(rank, world, port, path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    b = make_batch(orc, 4, 10, 6, 4, seed0=100, dtype="f64")
    band = row_band(b.H, world, rank, align=2)
    chunks, dys = [], []
    for s0 in (0, 2):
        ins = _inputs(b, s0, s0 + 2, band.r0, band.r1)
        chunks.append(tuple(torch.from_numpy(np.ascontiguousarray(t)) for t in ins))
        dys.append(torch.from_numpy(np.ascontiguousarray(b.dy[s0:s0 + 2, band.r0:band.r1])))
    pipe = RowBandPipeline(rank, world, dist)
    op = _NumpyBandOp()
    shape = lambda k: (2, b.W, b.N)
    mk = lambda s: torch.empty(s, dtype=torch.float64)
    ys = pipe.forward(lambda k: op, chunks, shape, mk)
    grads = pipe.backward(lambda k: op, chunks, dys, shape, mk)
    dA = torch.cat([g[2] for g in grads])
    dD = torch.cat([g[5] for g in grads])
    dbias = torch.cat([g[6] for g in grads])
    dA, dD, dbias = reduce_params(dist, [dA, dD, dbias], world)
    np.savez(f"{path}.{rank}.npz", r0=band.r0, r1=band.r1, y=torch.cat(ys).numpy(),
             dx=torch.cat([g[0] for g in grads]).numpy(), dB=torch.cat([g[3] for g in grads]).numpy(),
             dA=dA.numpy(), dD=dD.numpy(), dbias=dbias.numpy())
    dist.destroy_process_group()


def test_gloo_rowband_pipeline_world2(tmp_path):
    import torch.multiprocessing as mp

    port = 29500 + os.getpid() % 1000
    path = str(tmp_path / "rb")
    mp.spawn(_gloo_worker, args=(2, port, path), nprocs=2, join=True)
    orc = Oracle()
    b = make_batch(orc, 4, 10, 6, 4, seed0=100, dtype="f64")
    y_ref = oracle_fwd(orc, b, "f64")
    ref = oracle_bwd(orc, b, "f64")
    for rank in range(2):
        d = np.load(f"{path}.{rank}.npz")
        r0, r1 = int(d["r0"]), int(d["r1"])
        assert rel_error(d["y"], y_ref[:, r0:r1]) < 1e-12
        assert rel_error(d["dx"], ref["dx"].reshape(b.S, b.H, b.W)[:, r0:r1]) < 1e-11
        assert rel_error(d["dB"], ref["dB"].reshape(b.S, b.H, b.W, b.N)[:, r0:r1]) < 1e-11
        for k in ("dA", "dD", "dbias"):
            assert rel_error(d[k], ref[k]) < 1e-11, k


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cuda_band_chain_bitwise(dtype):
    from paper_2412_00678_b200.api import Scan2dBandOp, Scan2dOp
    from scan_cases import batch_to_torch

    orc = Oracle()
    S, H, W, N = 3, 40, 48, 16
    b = make_batch(orc, S, H, W, N, seed0=500, dtype=dtype)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    tdt = x.dtype
    full = Scan2dOp(S, H, W, N, dtype=tdt, device="cuda")
    y_full = full.forward(x, z, B, C, A, D, bias).clone()
    g_full = [t.clone() for t in full.backward(x, z, B, C, A, D, bias, dy)]
    al = band_align(N, 4 if dtype == "f32" else 8)
    bands = [row_band(H, 3, r, al) for r in range(3)]
    ops, tops, ys = [], [None], []
    sl = lambda t, bd: t[:, bd.r0:bd.r1].contiguous()
    for bd in bands:
        op = Scan2dBandOp(S, bd.rows, W, N, dtype=tdt, device="cuda")
        y, hb = op.forward(sl(x, bd), sl(z, bd), sl(B, bd), sl(C, bd), A, D, bias, h_top=tops[-1])
        ys.append(y.clone())
        tops.append(hb.clone())
        ops.append(op)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(ys, dim=1), y_full)
    g, outs = None, {}
    for k in range(2, -1, -1):
        bd = bands[k]
        res = ops[k].backward(sl(x, bd), sl(z, bd), sl(B, bd), sl(C, bd), A, D, bias, tops[k], sl(dy, bd), g)
        g = res[-1].clone()
        outs[k] = [t.clone() for t in res[:-1]]
    torch.cuda.synchronize()
    for idx, name in [(0, "dx"), (1, "dz"), (3, "dB"), (4, "dC")]:
        got = torch.cat([outs[k][idx] for k in range(3)], dim=1)
        assert torch.equal(got, g_full[idx]), name
    for idx in (2, 5, 6):
        tot = outs[0][idx] + outs[1][idx] + outs[2][idx]
        assert rel_error(tot.cpu().numpy(), g_full[idx].cpu().numpy()) < (1e-5 if dtype == "f32" else 1e-12)


def _full_and_bands(dtype, S, H, W, N, nb, seed):
    from paper_2412_00678_b200.api import Scan2dOp
    from scan_cases import batch_to_torch

    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=seed, dtype=dtype)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    full = Scan2dOp(S, H, W, N, dtype=x.dtype, device="cuda")
    y_full = full.forward(x, z, B, C, A, D, bias).clone()
    g_full = [t.clone() for t in full.backward(x, z, B, C, A, D, bias, dy)]
    torch.cuda.synchronize()
    bands = [row_band(H, nb, r, band_align(N, 4 if dtype == "f32" else 8)) for r in range(nb)]
    return (x, z, B, C, A, D, bias), dy, y_full, g_full, bands


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cuda_linked_bands_in_kernel_handoff(dtype):
    """Three bands on three streams, linked in-kernel (scan2d_*_band_linked):
    every consumer band is launched BEFORE its producer, so only the per-strip
    flags order them; y, dx, dz, dB, dC must equal the single-grid run bit for
    bit, twice in a row (the flags' sequence number advances)."""
    from paper_2412_00678_b200 import _native as nat
    from paper_2412_00678_b200.api import Scan2dBandOp

    S, H, W, N = 3, 40, 48, 16
    (x, z, B, C, A, D, bias), dy, y_full, g_full, bands = _full_and_bands(dtype, S, H, W, N, 3, 700)
    tdt = x.dtype
    ops = [Scan2dBandOp(S, bd.rows, W, N, dtype=tdt, device="cuda") for bd in bands]
    strips = nat.lib.scan2d_band_strips(__import__("ctypes").byref(ops[0].desc))
    hbuf = [torch.zeros((S, W, N), dtype=tdt, device="cuda") for _ in range(2)]  # band k -> k+1
    gbuf = [torch.zeros((S, W, N), dtype=tdt, device="cuda") for _ in range(2)]  # band k+1 -> k
    ff = [torch.zeros(S * strips, dtype=torch.int32, device="cuda") for _ in range(2)]
    bf = [torch.zeros(S * strips, dtype=torch.int32, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(3)]
    sl = lambda t, bd: t[:, bd.r0:bd.r1].contiguous()  # noqa: E731
    ins = [(sl(x, bd), sl(z, bd), sl(B, bd), sl(C, bd), A, D, bias) for bd in bands]
    dys = [sl(dy, bd) for bd in bands]
    torch.cuda.synchronize()
    for seq in (1, 2):
        for k in (2, 1, 0):  # consumers first
            with torch.cuda.stream(streams[k]):
                ops[k].forward(*ins[k], h_top=hbuf[k - 1] if k > 0 else None,
                               link=(ff[k - 1] if k > 0 else None, ff[k] if k < 2 else None, seq),
                               h_bottom=hbuf[k] if k < 2 else None)
        for k in (0, 1, 2):  # backward consumers (upper bands) first
            with torch.cuda.stream(streams[k]):
                ops[k].backward(*ins[k], hbuf[k - 1] if k > 0 else None, dys[k],
                                g_bottom=gbuf[k] if k < 2 else None,
                                link=(bf[k] if k < 2 else None, bf[k - 1] if k > 0 else None, seq),
                                g_top=gbuf[k - 1] if k > 0 else None)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat([o.op.y for o in ops], dim=1), y_full), seq
        for idx, name in [(0, "dx"), (1, "dz"), (3, "dB"), (4, "dC")]:
            got = torch.cat([[o.op.dx, o.op.dz, o.op.dA, o.op.dB, o.op.dC][idx] for o in ops], dim=1)
            assert torch.equal(got, g_full[idx]), (seq, name)
        for idx, t in ((2, "dA"), (5, "dD"), (6, "dbias")):
            parts = [[o.op.dx, o.op.dz, o.op.dA, o.op.dB, o.op.dC, o.op.dD, o.op.dbias][idx] for o in ops]
            tot = parts[0] + parts[1] + parts[2]
            assert rel_error(tot.cpu().numpy(), g_full[idx].cpu().numpy()) < (1e-5 if dtype == "f32" else 1e-12), t


def _ipc_worker(rank, world, port, path):
    import torch.distributed as dist

    from paper_2412_00678_b200.launcher import LinkedRowBands
    from scan_cases import batch_to_torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    S, H, W, N = 2, 24, 40, 16
    b = make_batch(Oracle(), S, H, W, N, seed0=710, dtype="f32")
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    lb = LinkedRowBands(S, H, W, N, rank, world, dist=dist, device="cuda:0")
    xs, zs, Bs, Cs, dys = lb.views(x, z, B, C, dy)
    for _ in range(2):
        y = lb.forward(xs, zs, Bs, Cs, A, D, bias).clone()
        g = [t.clone() for t in lb.backward(xs, zs, Bs, Cs, A, D, bias, dys)]
        lb.step_barrier()
    torch.cuda.synchronize()
    np.savez(f"{path}.{rank}.npz", r0=lb.band.r0, r1=lb.band.r1, y=y.cpu().numpy(),
             **{k: v.cpu().numpy() for k, v in zip(("dx", "dz", "dA", "dB", "dC", "dD", "dbias"), g)})
    lb.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_cuda_linked_bands_ipc_two_processes(tmp_path):
    """Two processes (one band each) linked through CUDA IPC handles exchanged
    over gloo -- the multi-GPU setup, here with both processes on cuda:0."""
    import torch.multiprocessing as mp

    S, H, W, N = 2, 24, 40, 16
    (x, z, B, C, A, D, bias), dy, y_full, g_full, bands = _full_and_bands("f32", S, H, W, N, 2, 710)
    port = 29700 + os.getpid() % 1000
    path = str(tmp_path / "ipc")
    mp.spawn(_ipc_worker, args=(2, port, path), nprocs=2, join=True)
    parts = [np.load(f"{path}.{r}.npz") for r in range(2)]
    y = np.concatenate([p["y"] for p in parts], axis=1)
    assert np.array_equal(y, y_full.cpu().numpy())
    for idx, k in [(0, "dx"), (1, "dz"), (3, "dB"), (4, "dC")]:
        assert np.array_equal(np.concatenate([p[k] for p in parts], axis=1), g_full[idx].cpu().numpy()), k
    for idx, k in [(2, "dA"), (5, "dD"), (6, "dbias")]:
        assert rel_error(parts[0][k] + parts[1][k], g_full[idx].cpu().numpy()) < 1e-5, k
