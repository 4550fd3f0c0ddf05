"""Batch shard of one global problem over ranks (BASELINE
configs[3] "batch-sharded over 2/4/8 GPUs"): shard planning, the shard views
of the C-ABI layouts, and world-size-2 runs that shard a batch, run every
shard, gather the results and compare them with the oracle on the whole batch:
  * CPU, gloo, the oracle as the per-shard compute backend (host logic);
  * -m gpu: two processes sharing cuda:0 (gloo for the gather), the CUDA
    operator per shard; per-scan outputs must equal the unsharded GPU run bit
    for bit, and everything must match the fp64 oracle."""
import os

import numpy as np
import pytest
import torch

from oracle_lib import Oracle, rel_error
from paper_2412_00678_b200.launcher import ShardedScan2d, layout_quantum, shard_range, shard_views
from scan_cases import make_batch, oracle_bwd, oracle_fwd

NAMES = ("dx", "dz", "dA", "dB", "dC", "dD", "dbias")


def test_shard_plan_covers_batch():
    for S, world, q in [(128, 8, 1), (12288, 8, 1), (12, 5, 3), (7, 4, 1), (24, 3, 6), (3, 8, 1)]:
        shards = [shard_range(S, world, r, q) for r in range(world)]
        assert shards[0].s0 == 0 and shards[-1].s1 == S
        for a, b in zip(shards, shards[1:]):
            assert a.s1 == b.s0 and a.s1 % q == 0
        counts = [sh.count for sh in shards]
        assert max(counts) - min(counts) <= q
    assert layout_quantum(12, 4, 3) == 12 and layout_quantum(12, 12, 3) == 3 and layout_quantum(8, 8, 1) == 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 0, 3)


def test_shard_views_layouts():
    orc = Oracle()
    b = make_batch(orc, 12, 3, 4, 2, seed0=9, dtype="f64", P=4, G=3)
    q = layout_quantum(12, 4, 3)
    for world in (1, 2, 3):
        for r in range(world):
            sh = shard_range(12, world, r, q)
            x, z, B, C, A, D, bias = shard_views(sh, b.x, b.z, b.B, b.C, b.A, b.D, b.bias, 4, 3)
            assert x.shape[0] == sh.count and B.shape[0] == sh.count // 3
            assert A.shape[0] == 4  # periodic parameter table shared unchanged
            if sh.count:
                np.testing.assert_array_equal(B[0], b.B[sh.s0 // 3])


class _OracleOp:
    """Per-shard CPU compute backend (test infrastructure): the oracle."""

    def __init__(self, orc, S, P, G, H, W, N):
        self.orc, self.dims = orc, (S, P, G, H, W, N)

    def forward(self, x, z, B, C, A, D, bias, save=True):
        S, P, G, H, W, N = self.dims
        y = self.orc.fwd_batch(S, P, G, H, W, N, *[t.numpy() for t in (x, z, B, C, A, D, bias)], dtype="f64")
        return torch.from_numpy(y.reshape(S, H, W))

    def backward(self, x, z, B, C, A, D, bias, dy):
        S, P, G, H, W, N = self.dims
        g = self.orc.bwd_batch(S, P, G, H, W, N, *[t.numpy() for t in (x, z, B, C, A, D, bias, dy)], dtype="f64")
        shp = dict(dx=(S, H, W), dz=(S, H, W), dA=(P, N), dB=(S // G, H, W, N), dC=(S // G, H, W, N),
                   dD=(P,), dbias=(P,))
        return [torch.from_numpy(np.asarray(g[k]).reshape(shp[k])) for k in NAMES]


# (S, H, W, N, P, G); the last has one layout quantum only (rank 1's shard is empty)
CASES = [(10, 6, 9, 4, 10, 1), (12, 5, 7, 3, 4, 2), (12, 5, 7, 3, 4, 3)]


def _worker(rank, world, port, path, case, backend_gpu):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S, H, W, N, P, G = case
    orc = Oracle()
    dt = "f32" if backend_gpu else "f64"
    b = make_batch(orc, S, H, W, N, seed0=300, dtype=dt, P=P, G=G)
    glob = [torch.from_numpy(np.ascontiguousarray(v)) for v in (b.x, b.z, b.B, b.C, b.A, b.D, b.bias)]
    dy = torch.from_numpy(np.ascontiguousarray(b.dy))
    if backend_gpu:
        factory = None  # Scan2dOp on cuda:0 (both ranks share the one GPU)
        sh = ShardedScan2d(S, H, W, N, rank, world, params_period=P, bc_group=G, dist=dist, device="cuda:0")
        glob = [t.cuda() for t in glob]
        dy = dy.cuda()
    else:
        factory = lambda s, p, g: _OracleOp(orc, s, p, g, H, W, N)  # noqa: E731
        sh = ShardedScan2d(S, H, W, N, rank, world, params_period=P, bc_group=G, dist=dist, op_factory=factory)
    ins = [t.contiguous() for t in sh.views(*glob)]
    dy_l = dy[sh.shard.s0:sh.shard.s1].contiguous()
    y = sh.forward(*ins).clone()
    grads = [t.clone() for t in sh.backward(*ins, dy_l)]
    if backend_gpu:
        torch.cuda.synchronize()
        y, grads = y.cpu(), [t.cpu() for t in grads]
    y_all = sh.gather(y)
    g_all = sh.gather_grads(grads)
    if rank == 0:
        np.savez(path, y=y_all.numpy(), **{k: v.numpy() for k, v in zip(NAMES, g_all)})
    dist.destroy_process_group()


def _spawn(tmp_path, case, gpu):
    import torch.multiprocessing as mp

    port = 29600 + (os.getpid() + 17 * case[0] + 5 * case[5] + (7 if gpu else 0)) % 1000
    path = str(tmp_path / f"bs_{case[0]}_{case[5]}.npz")
    mp.spawn(_worker, args=(2, port, path, case, gpu), nprocs=2, join=True)
    return np.load(path)


@pytest.mark.parametrize("case", CASES)
def test_gloo_batch_shard_world2(tmp_path, case):
    S, H, W, N, P, G = case
    d = _spawn(tmp_path, case, gpu=False)
    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=300, dtype="f64", P=P, G=G)
    assert rel_error(d["y"], oracle_fwd(orc, b, "f64")) < 1e-13
    ref = oracle_bwd(orc, b, "f64")
    for k in NAMES:
        assert rel_error(d[k].reshape(-1), np.asarray(ref[k]).reshape(-1)) < 1e-12, k


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES + [(6, 40, 200, 16, 6, 1)])
def test_cuda_batch_shard_world2(tmp_path, case):
    from paper_2412_00678_b200.api import Scan2dOp
    from scan_cases import batch_to_torch

    S, H, W, N, P, G = case
    d = _spawn(tmp_path, case, gpu=True)
    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=300, dtype="f32", P=P, G=G)
    # the unsharded GPU run on the same inputs
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    op = Scan2dOp(S, H, W, N, params_period=P, bc_group=G, device="cuda")
    y = op.forward(x, z, B, C, A, D, bias).cpu().numpy()
    g = [t.cpu().numpy() for t in op.backward(x, z, B, C, A, D, bias, dy)]
    np.testing.assert_array_equal(d["y"], y)
    for k, v in zip(NAMES, g):
        if k in ("dx", "dz") or (k in ("dB", "dC") and G == 1) or (k in ("dA", "dD", "dbias") and P == S):
            np.testing.assert_array_equal(d[k], v, err_msg=k)  # per-scan outputs: identical bits
    assert rel_error(d["y"], oracle_fwd(orc, b, "f64")) <= 1e-4
    ref = oracle_bwd(orc, b, "f64")
    for k in NAMES:
        assert rel_error(d[k].reshape(-1), np.asarray(ref[k]).reshape(-1)) <= 1e-4, k
