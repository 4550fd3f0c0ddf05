"""bench.py's output contract (one JSON line from rank 0, keys the driver reads),
at N = 1 and through torchrun at N = 2.  The two-rank case shares cuda:0 via the
SCAN2D_BENCH_SHARED_GPU test hook (gloo for the timing collectives), so the
launch / max-over-ranks / rank-0-prints logic runs on a one-GPU box."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _run(cmd, env=None, timeout=600):
    e = dict(os.environ, **(env or {}))
    p = subprocess.run(cmd, cwd=REPO, env=e, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return lines


@pytest.mark.gpu
def test_bench_single_gpu_line():
    lines = _run([sys.executable, "bench.py", "--workload", "cfg1", "--steps", "3", "--warmup", "3", "--no-cpu"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] >= 3
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_one_line():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2",
           "--workload", "cfg1", "--steps", "3", "--warmup", "3", "--no-cpu"]
    lines = _run(cmd, env={"SCAN2D_BENCH_SHARED_GPU": "1"})
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert "x2" in d["config"]["parallelism"]


def test_bench_reference_arm_two_ranks():  # CPU only: the reference arm never touches a GPU
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29542", "bench.py", "--gpus", "2",
           "--workload", "cfg1", "--steps", "1", "--warmup", "1", "--impl", "reference"]
    lines = _run(cmd)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["cores"] >= 1
    # the config dict is the one the ours arm prints (the driver compares them)
    sys.path.insert(0, REPO)
    import bench

    assert d["config"] == bench.build_config("cfg1", 2, "weak")[0]


def test_bench_config_shared_by_both_arms():
    sys.path.insert(0, REPO)
    import bench

    for wl in bench.WORKLOADS:
        for world in (1, 2, 8):
            cfg, S_global, per_gpu = bench.build_config(wl, world, bench.SCALING[wl])
            assert sum(per_gpu) == S_global and cfg["S_per_gpu"] == per_gpu
            assert cfg["workload"] == wl and "l2" in cfg
