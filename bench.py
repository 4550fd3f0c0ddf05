#!/usr/bin/env python
"""bench.py -- throughput of the B200 2D selective scan (fwd + bwd) vs the CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl ours|reference]

One "step" = one training pass of the hot path over one batch: scan2d_forward
(saving the residual) followed by scan2d_backward, on synthetic inputs
resident in HBM (the `value`).  `e2e` repeats the step through the same C ABI
from pinned HOST buffers with every input copied in and every output
(y and all gradients) copied back inside the timed region -- the drop-in
replacement of the reference call, whose arguments and results live on the host.

Workloads (BASELINE.json configs):
  cfg1  S=64   16x16   N=16 fwd           (configs[0], the CPU-oracle case)
  cfg2  S=128  200x200 N=16 fwd+bwd       (configs[1], DEFAULT: WSI MIL scale)
  cfg3  S=12288 56x56  N=1  fwd+bwd       (configs[2], VMamba stage 1, B=64 D=192)
  cfg4a..d  B=64 N=1 fwd+bwd: 56x56 D=96, 28x28 D=192, 14x14 D=384, 7x7 D=768
  cfg5  S=256  1024x1024 N=16 fwd         (configs[4], giga-pixel slide)

Multi-GPU (torchrun, one rank per GPU): every rank processes its own S scans
(weak scaling, no collective on the data path); timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

METRIC = "2D sel-scan Gelem/s & HBM GB/s (% roofline) at 1/2/4/8 B200 vs CPU ref"

WORKLOADS = {
    "cfg1": dict(S=64, H=16, W=16, N=16, bwd=False, desc="B=1 D=64 N=16 16x16 fwd (configs[0])"),
    "cfg2": dict(S=128, H=200, W=200, N=16, bwd=True, desc="WSI MIL: B=1 D=128 N=16 200x200 fwd+bwd (configs[1])"),
    "cfg3": dict(S=64 * 192, H=56, W=56, N=1, bwd=True, desc="VMamba stage-1: B=64 D=192 N=1 56x56 fwd+bwd (configs[2])"),
    "cfg4a": dict(S=64 * 96, H=56, W=56, N=1, bwd=True, desc="VMamba sweep: B=64 D=96 N=1 56x56 fwd+bwd (configs[3])"),
    "cfg4b": dict(S=64 * 192, H=28, W=28, N=1, bwd=True, desc="VMamba sweep: B=64 D=192 N=1 28x28 fwd+bwd (configs[3])"),
    "cfg4c": dict(S=64 * 384, H=14, W=14, N=1, bwd=True, desc="VMamba sweep: B=64 D=384 N=1 14x14 fwd+bwd (configs[3])"),
    "cfg4d": dict(S=64 * 768, H=7, W=7, N=1, bwd=True, desc="VMamba sweep: B=64 D=768 N=1 7x7 fwd+bwd (configs[3])"),
    "cfg5": dict(S=256, H=1024, W=1024, N=16, bwd=False, desc="giga-pixel: B=1 D=256 N=16 1024x1024 fwd (configs[4])"),
    # the 2DMamba block layout of cfg2 (model.cpp:150-193): B / C shared by the D = 128 channels of the
    # batch item (G = 128), A / D / bias per channel -- SURVEY.md §8f row 2
    "cfg2m": dict(S=128, H=200, W=200, N=16, G=128, bwd=True,
                  desc="WSI MIL model layout: B=1 D=128 N=16 200x200, B/C shared by the 128 channels, fwd+bwd"),
}

# How `--gpus N` scales each workload (ShardedScan2d: contiguous scan ranges,
# no collective on the data path).  "weak": the global batch is N x the
# single-GPU batch (N slides / images -- per-GPU work fixed); "strong": the
# BASELINE batch itself is split over the N GPUs (configs[3], "batch-sharded
# over 2/4/8 GPUs").
SCALING = {"cfg1": "weak", "cfg2": "weak", "cfg2m": "weak", "cfg5": "weak", "cfg3": "strong", "cfg4a": "strong",
           "cfg4b": "strong", "cfg4c": "strong", "cfg4d": "strong"}

L2_BYTES = 126 * 1024 * 1024
NVML_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def alg_bytes(wl, es=4):
    """Reference counting model (memsim.cpp:45-46): per scan
    fwd = es*H*W*(3+2N) (x, z, B, C in; y out), bwd = es*H*W*(5+4N)
    (x, z, dy, B, C in; dx, dz, dB, dC out).  With B / C shared by groups of G
    scans (the model layout) the B / C / dB / dC terms count once per group:
    fwd = es*H*W*(3S + 2N S/G), bwd = es*H*W*(5S + 4N S/G)."""
    hw = wl["H"] * wl["W"]
    S, N, G = wl["S"], wl["N"], wl.get("G", 1)
    return es * hw * (3 * S + 2 * N * S // G), es * hw * (5 * S + 4 * N * S // G)


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy_ burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    p = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload, {})
    except Exception:
        return {}


class ClockSampler:
    """NVML clocks / throttle reasons sampled in a background thread."""

    def __init__(self, index=0, period=0.01):
        self.samples = []
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        self._t = None

    def start(self):
        if not self.ok:
            return
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while not self._stop.is_set():
            try:
                clk = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), clk, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self, t0, t1):
        win = [s for s in self.samples if t0 <= s[0] <= t1] or self.samples
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        bits = 0
        for s in win:
            bits |= s[2]
        reasons = [v for k, v in NVML_REASONS.items() if bits & k and k != 0x1]
        return {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(win)}


# ----------------------------------------------------------------- inputs


def synth_inputs(torch, wl, dev, seed, dtype):
    """random_instance distribution (fixtures.hpp:20-37): x, z, B, C ~ N(0,1),
    A ~ -U(0.05, 0.95), D ~ N(0,1), bias ~ U(-0.5, 0.5); dy ~ N(0,1)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    S, H, W, N = wl["S"], wl["H"], wl["W"], wl["N"]
    r = lambda *s: torch.randn(*s, generator=g, device=dev, dtype=dtype)
    u = lambda *s: torch.rand(*s, generator=g, device=dev, dtype=dtype)
    x, z = r(S, H, W), r(S, H, W)
    G = wl.get("G", 1)
    B, C = r(S // G, H, W, N), r(S // G, H, W, N)
    A = -(0.05 + 0.9 * u(S, N))
    D = r(S)
    bias = u(S) - 0.5
    dy = r(S, H, W)
    return [x, z, B, C, A, D, bias], dy


def host_inputs_np(wl, S_sample, seed=1234):
    import numpy as np

    rng = np.random.default_rng(seed)
    H, W, N = wl["H"], wl["W"], wl["N"]
    f = lambda *s: rng.standard_normal(s, dtype=np.float32)
    x, z, B, C = f(S_sample, H, W), f(S_sample, H, W), f(S_sample, H, W, N), f(S_sample, H, W, N)
    A = -(0.05 + 0.9 * rng.random((S_sample, N), dtype=np.float32))
    D = f(S_sample)
    bias = rng.random(S_sample, dtype=np.float32) - 0.5
    dy = f(S_sample, H, W)
    return x, z, B, C, A, D, bias, dy


# ------------------------------------------------------------ CPU reference


class CpuReference:
    """Reference CPU engine (oracle/_ref/libscan2d_ref.so: the reference's own
    tiled_scan_2d_forward/backward, threads=1 per scan, scans spread over all
    host cores in contiguous blocks -- the model.cpp:177 pattern) on a bounded
    sample of the workload.  Falls back to the oracle port (kind "port") when
    the reference library was not built."""

    def __init__(self, wl, target_s=10.0):
        sys.path.insert(0, os.path.join(REPO, "tests"))
        self.wl = wl
        self.kind = "reference"
        try:
            from oracle_lib import RefLib

            self.ref = RefLib()
        except Exception:
            from oracle_lib import Oracle

            self.ref = None
            self.orc = Oracle()
            self.kind = "port"
        cores = os.cpu_count() or 1
        self.t1 = self._run(1, 1, host_inputs_np(wl, 1, seed=99))
        threads = cores if (self.ref is not None or not wl["bwd"]) else 1
        k = int(max(threads, min(wl["S"], target_s * threads / max(self.t1, 1e-6) / 4)))
        self.k = min(k, wl["S"])
        self.threads = min(threads, self.k)
        self.arrs = host_inputs_np(wl, self.k, seed=7)

    def _run(self, S_, threads, arrs):
        wl = self.wl
        H, W, N, bwd = wl["H"], wl["W"], wl["N"], wl["bwd"]
        x, z, B, C, A, D, bias, dy = arrs
        if self.ref is not None:
            secs, _ = self.ref.batch(S_, S_, 1, H, W, N, 16, threads, bwd, x, z, B, C, A, D, bias, dy)
            return secs
        t0 = time.perf_counter()
        self.orc.fwd_batch(S_, S_, 1, H, W, N, x, z, B, C, A, D, bias, dtype="f32", threads=threads)
        if bwd:
            self.orc.bwd_batch(S_, S_, 1, H, W, N, x, z, B, C, A, D, bias, dy, dtype="f32")
        return time.perf_counter() - t0

    def step(self):
        """One timed pass over the sample; returns seconds."""
        return self._run(self.k, self.threads, self.arrs)

    def gelem_s(self, secs):
        return self.k * self.wl["H"] * self.wl["W"] / secs / 1e9

    def describe(self, secs, reps):
        wl = self.wl
        return {"value": self.gelem_s(secs), "unit": "Gelem/s", "cores": self.threads, "kind": self.kind,
                "sample": (f"{self.k} of {wl['S']} scans ({'fwd+bwd' if wl['bwd'] else 'fwd'}, T=16, "
                           f"tiled_scan_2d_* threads=1 per scan) over {self.threads} host threads, "
                           f"median of {reps} passes; one scan single-threaded {self.t1 * 1e3:.2f} ms")}


def cpu_reference(wl, target_s=10.0, reps=3, parity_dev=None):
    cr = CpuReference(wl, target_s)
    med = statistics.median(cr.step() for _ in range(reps))  # robust to the host's occasional slow pass
    out = cr.describe(med, reps)
    if parity_dev is not None and cr.ref is not None:
        out["parity"] = parity_vs_reference(cr, parity_dev)
    return out


def parity_vs_reference(cr, dev, max_scans=16):
    """North_star parity report on the CPU sample's own inputs: y and (for a
    training workload) every gradient group of the GPU path against the
    reference library's fp64 engine (normwise error of test_util.hpp:17-26 and
    the per-element distribution), with the reference's own fp32 engine on the
    same inputs beside it for scale."""
    import numpy as np
    import torch

    from oracle_lib import elem_stats, rel_error
    from paper_2412_00678_b200.api import Scan2dOp

    wl = cr.wl
    k = min(cr.k, max_scans)
    H, W, N = wl["H"], wl["W"], wl["N"]
    x, z, B, C, A, D, bias, dy = [a[:k] for a in cr.arrs]
    bwd = wl["bwd"]
    t = [torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (x, z, B, C, A, D, bias)]
    op = Scan2dOp(k, H, W, N, tile=16, device=dev, with_backward=bwd)
    got = {"y": op.forward(*t, save=bwd).cpu().numpy()}
    if bwd:
        g = op.backward(*t, torch.from_numpy(np.ascontiguousarray(dy)).to(dev))
        for name, v in zip(("dx", "dz", "dA", "dB", "dC", "dD", "dbias"), g):
            got[name] = v.cpu().numpy()
    refs = {}
    for dt in ("f64", "f32"):
        cast = np.float64 if dt == "f64" else np.float32
        arrs = [np.asarray(v, cast) for v in (x, z, B, C, A, D, bias, dy)]
        if bwd:
            refs[dt] = cr.ref.batch_grads(k, H, W, N, 16, cr.threads, *arrs, dtype=dt)
        else:
            _, y_ = cr.ref.batch(k, k, 1, H, W, N, 16, cr.threads, False, *arrs[:7], dtype=dt, want_y=True)
            refs[dt] = {"y": y_}
    groups = {}
    for name, v in got.items():
        r64 = refs["f64"][name]
        groups[name] = {"normwise_rel": rel_error(v, r64), "elem_rel": elem_stats(v, r64),
                        "reference_f32_normwise_rel": rel_error(refs["f32"][name], r64)}
    worst = max(gv["normwise_rel"] for gv in groups.values())
    return {"scans": k, "against": "reference tiled_scan_2d_forward/backward<double> (oracle/_ref)",
            "tolerance": 1e-4, "worst_normwise_rel": worst, "pass": bool(worst <= 1e-4),
            "normwise_rel": groups["y"]["normwise_rel"], "elem_rel": groups["y"]["elem_rel"],
            "reference_f32": {"normwise_rel": groups["y"]["reference_f32_normwise_rel"]},
            "groups": groups}


# ----------------------------------------------------------------- main


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f32", choices=["f32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-accurate", action="store_true", help="skip the accurate-mode side measurement")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunks", type=int, default=0, help="0 = library heuristic")
    ap.add_argument("--rowband", action="store_true",
                    help="row-band shard: every rank owns H/world rows of all S scans (cfg5 mode), vertical "
                         "carries handed to the neighbouring GPU by the kernels (NVLink peer stores + flags)")
    ap.add_argument("--api", default="cabi", choices=["cabi", "shim"],
                    help="shim: time the reference's own C++ API (one scan per call, host Grid operands) served "
                         "by libscan2d_engine_cuda.so over all host cores (lib/bench_shim)")
    ap.add_argument("--compare", action="store_true",
                    help="Table 3: tiled vs naive-2D vs flat-1D operators at 14^2/56^2/200^2, D=1 N=16")
    ap.add_argument("--bc-reduce", choices=["red", "fixed"], default="red",
                    help="shared-B/C workloads (G > 1): dB / dC group sums by in-kernel L2 reductions "
                         "(SCAN2D_FLAG_GROUP_RED; summation order not fixed) or per-scan gradients + a "
                         "fixed-order reduction kernel (bit-reproducible)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: global batch = N x the workload's; strong: the workload's batch split over N "
                         "GPUs (default per workload, see SCALING)")
    args = ap.parse_args()
    if args.compare:
        return compare_main(args)
    if args.api == "shim":
        return shim_main(args)
    wl = dict(WORKLOADS[args.workload])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    scaling = args.scaling or SCALING[args.workload]
    config, S_global, per_gpu = build_config(args.workload, world, scaling, args.bc_reduce)

    if args.rowband and args.impl == "ours":
        return rowband_main(args, wl, rank, world, local, config)

    if args.impl == "reference":
        if rank != 0:
            return 0
        cr = CpuReference(wl, target_s=2.0)
        for _ in range(args.warmup):
            cr.step()
        times = [cr.step() for _ in range(args.steps)]
        mean_s = statistics.median(times)  # typical pass: host passes show occasional +40 % outliers
        value = cr.gelem_s(mean_s)
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": args.dtype,
                "data": "synthetic (random_instance distribution)", "config": config,
                "cpu_baseline": dict(cr.describe(mean_s, args.steps), value=value),
                "e2e": {"value": value, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch

    dist, local = init_dist(torch, world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2412_00678_b200.api import Scan2dOp

    from paper_2412_00678_b200.launcher import ShardedScan2d

    dtype = torch.float32
    sharded = ShardedScan2d(S_global, wl["H"], wl["W"], wl["N"], rank, world, dist=dist,
                            bc_group=wl.get("G", 1), tile=16, dtype=dtype, device=dev, with_backward=wl["bwd"],
                            group_red=args.bc_reduce == "red")
    shard = sharded.shard
    wl_local = dict(wl, S=shard.count)  # this rank's contiguous scan range of the global batch
    assert [sh.count for sh in sharded.shards] == per_gpu
    ins, dy = synth_inputs(torch, wl_local, dev, 1234 + shard.s0, dtype)
    op = sharded.op

    def step():
        op.forward(*ins, save=wl["bwd"])
        if wl["bwd"]:
            op.backward(*ins, dy)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
        op.check = False  # operands validated on the first step; no host checks in the timed loop
    torch.cuda.synchronize()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op.launches = 0
    torch.cuda.synchronize()
    barrier()
    t_host0 = time.perf_counter()
    # inputs smaller than 2x L2: flush L2 between timed steps (a 512 MB write,
    # outside the per-step events) and time the steps by their own events
    fb0, _ = alg_bytes(wl_local)
    flush = fb0 < 2 * L2_BYTES
    scratch = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev) if flush else None
    e_start.record(stream)
    for k in range(args.steps):
        if flush:
            scratch.fill_(k & 0xff)
        e0, e1, e2 = evs[k]
        e0.record(stream)
        op.forward(*ins, save=wl["bwd"])
        e1.record(stream)
        if wl["bwd"]:
            op.backward(*ins, dy)
        e2.record(stream)
    e_end.record(stream)
    torch.cuda.synchronize()
    t_host1 = time.perf_counter()
    barrier()
    launches = op.launches
    total_ms = (sum(a.elapsed_time(c) for a, _, c in evs) if flush else e_start.elapsed_time(e_end))
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b, _ in evs)
    bwd_ms = statistics.mean(b.elapsed_time(c) for _, b, c in evs) if wl["bwd"] else 0.0
    if dist is not None:
        total_ms, fwd_ms, bwd_ms = max_over_ranks(torch, dist, dev, [total_ms, fwd_ms, bwd_ms])
    sampler.stop()
    clocks = sampler.summary(t_host0, t_host1)
    ms_per_step = total_ms / args.steps
    elems = S_global * wl["H"] * wl["W"]  # the whole job: every rank's scans
    value = elems / (ms_per_step * 1e-3) / 1e9

    fb, bb = alg_bytes(wl_local)  # the dominant kernel's launch on one GPU
    peak, peak_src = measured_peak()
    traffic = ncu_traffic(args.workload)
    # kernel family the library picks (scan2d_capi.cu: rows1_shape, use_tile_*)
    if wl["N"] == 1 and wl["W"] <= 128:
        family = "rows1"
    elif op.plan()["cols_per_chunk"] == 1 and wl["N"] in (4, 8, 16, 32):
        family = "tile2"
    else:
        family = None
    kname = lambda d: f"scan2d_{d}_{family}_kernel" if family else f"scan2d_{d}_kernel"
    if wl["bwd"]:
        dom_name, dom_bytes, dom_ms = kname("bwd"), bb, bwd_ms
    else:
        dom_name, dom_bytes, dom_ms = kname("fwd"), fb, fwd_ms
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    roof = {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_src, "frac_of_nominal_8000": achieved / 8000.0,
            "traffic": (None if traffic.get(dom_name, {}).get("dram_bytes_per_launch") is None else
                        traffic[dom_name]["dram_bytes_per_launch"] * shard.count / wl["S"]),
            "algorithmic_bytes_per_launch": dom_bytes,
            "launch_ms": dom_ms}
    extra = {"fwd_ms": fwd_ms, "fwd_gbs": fb / (fwd_ms * 1e-3) / 1e9, "fwd_frac": fb / (fwd_ms * 1e-3) / 1e9 / peak}
    if wl["bwd"]:
        extra.update({"bwd_ms": bwd_ms, "bwd_gbs": bb / (bwd_ms * 1e-3) / 1e9,
                      "bwd_frac": bb / (bwd_ms * 1e-3) / 1e9 / peak})
    extra["plan"] = op.plan()
    # the accurate-exponential mode (SCAN2D_FLAG_ACCURATE: fp32 error at or below
    # the reference fp32 engine's) on the same inputs, for its cost
    if not args.no_accurate:
        aop = Scan2dOp(shard.count, wl["H"], wl["W"], wl["N"], tile=16, dtype=dtype, device=dev,
                       with_backward=wl["bwd"], accurate=True, bc_group=wl.get("G", 1),
                       group_red=args.bc_reduce == "red")
        aop.check = False
        for _ in range(3):
            aop.forward(*ins, save=wl["bwd"])
            if wl["bwd"]:
                aop.backward(*ins, dy)
        aev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a0, a1, a2 in aev:
            if flush:
                scratch.fill_(1)
            a0.record(stream)
            aop.forward(*ins, save=wl["bwd"])
            a1.record(stream)
            if wl["bwd"]:
                aop.backward(*ins, dy)
            a2.record(stream)
        torch.cuda.synchronize()
        afwd = statistics.median(a.elapsed_time(b) for a, b, _ in aev)
        abwd = statistics.median(b.elapsed_time(c) for _, b, c in aev) if wl["bwd"] else 0.0
        extra["accurate_mode"] = {"flag": "SCAN2D_FLAG_ACCURATE", "fwd_ms": afwd, "bwd_ms": abwd,
                                  "step_ms": afwd + abwd, "value": shard.count * wl["H"] * wl["W"] /
                                  ((afwd + abwd) * 1e-3) / 1e9 * world}
        del aop
    extra["gstate_updates_per_s"] = value * wl["N"]
    extra["inputs_vs_l2"] = f"inputs {fb / 1e6:.0f} MB {'>' if fb > L2_BYTES else '<='} L2 {L2_BYTES / 1e6:.0f} MB"

    # ---- e2e through the C ABI with HOST operands (scan2d_train_host: the
    #      reference call's contract -- host data in, host results out -- with the
    #      copies pipelined against the kernels inside the library)
    e2e = None
    if not args.no_e2e:
        from paper_2412_00678_b200.api import train_host

        hin = [t.cpu().pin_memory() for t in ins]
        hdy = dy.cpu().pin_memory() if wl["bwd"] else None
        red = wl.get("G", 1) > 1 and args.bc_reduce == "red"
        outs = train_host(*hin, dy=hdy, chunks=args.e2e_chunks, group_red=red)
        torch.cuda.synchronize()
        h2d = sum(t.numel() * t.element_size() for t in hin) + (hdy.numel() * 4 if wl["bwd"] else 0)
        d2h = sum(t.numel() * t.element_size() for t in outs if t is not None)
        barrier()
        k2 = max(1, args.e2e_steps)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ea.record(stream)
        for _ in range(k2):
            train_host(*hin, dy=hdy, outs=outs, chunks=args.e2e_chunks, group_red=red)
            stream.synchronize()
        eb.record(stream)
        torch.cuda.synchronize()
        e_ms = ea.elapsed_time(eb) / k2
        if dist is not None:
            (e_ms,) = max_over_ranks(torch, dist, dev, [e_ms])
        e2e = {"value": elems / (e_ms * 1e-3) / 1e9, "unit": "Gelem/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms, "steps": k2, "chunks": args.e2e_chunks,
               "path": "C ABI scan2d_train_host: pinned host operands, H2D / kernels / D2H pipelined over "
                       "scan chunks on three streams; inputs+dy in, y+all gradients out"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference(wl, parity_dev=dev)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "Gelem/s", "cores": 0, "kind": "unavailable", "sample": str(exc)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (random_instance distribution, generated on device)",
                "config": config, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, **extra}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


# Table 3 of the paper: CUDA operators, one feature map per
# call (D = 1), N = 16, throughput in feature maps per second.
PAPER_TABLE3 = {"cub_1d": {14: 49e3, 56: 12e3, 200: 3e3}, "naive_2d": {14: 0.2e3, 56: 0.06e3, 200: 0.02e3},
                "tiled_2d": {14: 40e3, 56: 6e3, 200: 1e3}}


def compare_main(args):
    """Table 3 on B200: the tiled operator against the two comparators behind
    the same C ABI (naive 2D: N horizontal state maps in HBM, engine.cpp:412-487;
    flat 1D: block scan of the row-major flattening, engine.cpp:489-526), D = 1,
    N = 16, at 14^2 / 56^2 / 200^2.  Each call is one forward on S maps; K calls
    are captured in a CUDA graph and replayed, so the time is the device's (no
    Python launch overhead).  maps/s = S * K / time.  S = 1 is the paper's
    "single dimensional feature input"; S = 128 the batched throughput."""
    import ctypes as C

    import torch

    from paper_2412_00678_b200 import _native as nat
    from paper_2412_00678_b200.api import Scan2dOp

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    rows = []
    K = 20
    for hw in (14, 56, 200):
        for S in (1, 128):
            wl = dict(S=S, H=hw, W=hw, N=16)
            ins, _ = synth_inputs(torch, wl, dev, 77, torch.float32)
            y = torch.empty(S, hw, hw, device=dev)
            desc = nat.make_desc(S, hw, hw, 16)
            op = Scan2dOp(S, hw, hw, 16, device=dev, with_backward=False)
            op.check = False
            ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
            calls = {"tiled_2d": lambda: op.forward(*ins, save=False)}
            for name, var in (("naive_2d", nat.VARIANT_NAIVE), ("cub_1d", nat.VARIANT_FLAT1D)):
                wsb = nat.lib.scan2d_comparator_workspace_bytes(C.byref(desc), var)
                ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)

                def call(var=var, ws=ws, wsb=wsb):
                    rc = nat.lib.scan2d_forward_variant(
                        C.byref(desc), var, *[ptr(t) for t in ins], ptr(y), ptr(ws), wsb,
                        C.c_void_p(torch.cuda.current_stream().cuda_stream))
                    if rc != nat.OK:
                        raise RuntimeError(f"scan2d_forward_variant: {nat.status_string(rc)}")
                calls[name] = call
            for name, fn in calls.items():
                if name == "naive_2d" and hw == 200 and S == 128:
                    continue  # 26 GB of state maps: beyond the point of the comparison
                side = torch.cuda.Stream(dev)
                side.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.stream(side):
                    for _ in range(3):
                        fn()
                torch.cuda.current_stream(dev).wait_stream(side)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(K):
                        fn()
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 5
                e0.record()
                for _ in range(reps):
                    g.replay()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / (reps * K)
                rows.append({"variant": name, "hw": hw, "maps_per_call": S, "us_per_call": ms * 1e3,
                             "maps_per_s": S / (ms * 1e-3),
                             "paper_maps_per_s": PAPER_TABLE3[name][hw] if S == 1 else None})
    print(json.dumps({"compare": "Table 3 (PAPER.md:280-282) on one B200: D=1 N=16 fp32 forward, CUDA-graph "
                                 "replay of 20 calls (device time), inputs L2-resident like the paper's repeated "
                                 "inference calls", "rows": rows}), flush=True)
    return 0


def shim_main(args):
    """The drop-in path at the reference contract: the workload's scans through
    scan2d::tiled_scan_2d_forward / tiled_scan_2d_backward (engine.hpp:88-102)
    with host Grid operands, one call per scan, spread over all host cores --
    the same call pattern as the reference arm -- served by the CUDA engine
    shim.  4 host threads: the best of 1 / 4 / 8 / 16 measured on the B200 box
    (the path is bound by host memory traffic: the reference API's deep copies
    and fresh output vectors, plus the staging copies).  Prints one JSON line
    with the e2e throughput."""
    import subprocess

    wl = dict(WORKLOADS[args.workload])
    exe = os.path.join(REPO, "paper_2412_00678_b200", "lib", "bench_shim")
    cmd = [exe, "--scans", str(wl["S"]), "--height", str(wl["H"]), "--width", str(wl["W"]),
           "--state-dim", str(wl["N"]), "--threads", str(min(4, os.cpu_count() or 1)), "--reps", str(args.steps),
           "--warmup", str(max(args.warmup, 1))] + ([] if wl["bwd"] else ["--forward-only"])
    out = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
    print(json.dumps({"metric": METRIC, "api": "shim", "value": out["gelem_per_s"], "unit": "Gelem/s",
                      "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 1),
                      "ms_per_step": out["seconds_per_pass"] * 1e3, "higher_is_better": True,
                      "config": {"workload": args.workload, "desc": wl["desc"]},
                      "e2e": {"value": out["gelem_per_s"], "unit": "Gelem/s",
                              "h2d_bytes_per_step": out["h2d_bytes_per_pass"],
                              "d2h_bytes_per_step": out["d2h_bytes_per_pass"]},
                      "detail": out}), flush=True)
    return 0


def build_config(workload, world, scaling, bc_reduce="red"):
    """The `config` dict of a bench line -- computed from the workload alone, so
    both arms (ours and `--impl reference`) print the identical dict."""
    wl = WORKLOADS[workload]
    S_global = wl["S"] * world if scaling == "weak" else wl["S"]
    # largest per-GPU shard (launcher.shard_range with the layout quantum),
    # computed here so the reference arm imports nothing of the package (no repo
    # .so loaded on its path)
    q = wl.get("G", 1)
    units = S_global // q
    base, extra = divmod(units, world)
    per_gpu = [(base + (1 if r < extra else 0)) * q for r in range(world)]
    fb0, _ = alg_bytes(dict(wl, S=max(per_gpu)))
    config = {"workload": workload, "desc": wl["desc"], "S_global": S_global, "S_per_gpu": per_gpu, "H": wl["H"],
              "W": wl["W"], "N": wl["N"], "tile": 16, "pass": "fwd+bwd" if wl["bwd"] else "fwd",
              "parallelism": (f"batch-sharded x{world} ({scaling} scaling: contiguous scan ranges per GPU, "
                              "no collective on the data path)"),
              "l2": l2_policy(fb0)}
    if q > 1:
        config["bc_group"] = q
        config["bc_reduce"] = ("in-kernel L2 reductions (SCAN2D_FLAG_GROUP_RED)" if bc_reduce == "red" else
                               "per-scan dB/dC + fixed-order reduction kernel")
    return config, S_global, per_gpu


def l2_policy(fwd_bytes):
    """How the timed loop keeps L2 from serving repeated inputs (the same
    string in both arms' config)."""
    if fwd_bytes < 2 * L2_BYTES:
        return ("inputs {:.0f} MB < 2x L2: L2 flushed (512 MB write) between timed steps, steps timed by their "
                "own events".format(fwd_bytes / 1e6))
    return "inputs {:.0f} MB > 2x L2 (2 x 126 MB): no flush needed".format(fwd_bytes / 1e6)


def init_dist(torch, world, local):
    """One process per GPU over NCCL.  SCAN2D_BENCH_SHARED_GPU=1 is a test hook
    for one-GPU boxes: every rank uses cuda:0 and the timing collectives go over
    gloo (NCCL refuses two ranks on one device); numbers from it are not bench
    values."""
    if world <= 1:
        return None, local
    import torch.distributed as dist

    if os.environ.get("SCAN2D_BENCH_SHARED_GPU") == "1":
        dist.init_process_group("gloo")
        return dist, 0
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist, local


def max_over_ranks(torch, dist, dev, vals):
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([float(v) for v in vals], device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def rowband_main(args, wl, rank, world, local, config):
    """Row-band shard: rank r owns rows row_band(H, world, r) of every
    scan on its own GPU (LinkedRowBands): the kernels hand the vertical carries
    to the neighbouring GPU themselves -- forward h of the band's last row into
    rank r+1's buffer, backward Abar G of its first row into rank r-1's, over
    NVLink peer memory (CUDA IPC), with one system-scope release/acquire flag
    per (scan, 16-column strip).  No collective and no host step on the data
    path; ranks only meet at a barrier between forward-only steps (the
    ordering a receive buffer needs, LinkedRowBands docstring)."""
    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        if os.environ.get("SCAN2D_BENCH_SHARED_GPU") == "1":
            dist.init_process_group("gloo")
            local = 0
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2412_00678_b200.launcher import LinkedRowBands

    S, H, W, N = wl["S"], wl["H"], wl["W"], wl["N"]
    lb = LinkedRowBands(S, H, W, N, rank, world, dist=dist, device=dev, with_backward=wl["bwd"])
    band = lb.band
    bw = dict(wl, H=band.rows)
    ins, dy = synth_inputs(torch, bw, dev, 1234 + rank, torch.float32)
    lb.op.op.check = False

    def step():
        lb.forward(*ins, save=wl["bwd"])
        if wl["bwd"]:
            lb.backward(*ins, dy)
        else:
            lb.step_barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        (ms,) = max_over_ranks(torch, dist, dev, [ms])
        dist.barrier()
    if rank == 0:
        fb, bb = alg_bytes(wl)
        config.update({"parallelism": f"row-band x{world} (in-kernel NVLink carry hand-off, per-strip flags)",
                       "band_rows": band.rows, "S_global": S, "S_per_gpu": [S] * world})
        line = {"metric": METRIC, "value": S * H * W / (ms * 1e-3) / 1e9, "unit": "Gelem/s", "n_gpus": world,
                "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (random_instance distribution, generated on device)", "config": config,
                "hbm_gbs_per_gpu": (fb + (bb if wl["bwd"] else 0)) / world / (ms * 1e-3) / 1e9}
        print(json.dumps(line), flush=True)
    lb.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
