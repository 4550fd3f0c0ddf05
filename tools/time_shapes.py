"""Time forward (training, residual saved; and inference) and backward for arbitrary shapes.

usage: python tools/time_shapes.py S,H,W,N[,G] ...   (fp32, CUDA events, inputs resident;
G = scans sharing one B/C block, the model.cpp layout)
Prints ms and algorithmic GB/s (memsim.cpp:45-46 counting) per direction.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_00678_b200.api import Scan2dOp  # noqa: E402


def run(S, H, W, N, G=1, reps=10):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    r = lambda *s: torch.randn(*s, generator=g, device=dev)
    x, z, B, C, dy = r(S, H, W), r(S, H, W), r(S // G, H, W, N), r(S // G, H, W, N), r(S, H, W)
    A = -(0.05 + 0.9 * torch.rand(S, N, generator=g, device=dev))
    D, bias = r(S), torch.rand(S, generator=g, device=dev) - 0.5
    op = Scan2dOp(S, H, W, N, tile=16, bc_group=G, device=dev, with_backward=True)
    ins = (x, z, B, C, A, D, bias)
    for _ in range(3):
        op.forward(*ins, save=True)
        op.backward(*ins, dy)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(reps):
        ev[0].record()
        op.forward(*ins, save=True)
        ev[1].record()
        op.backward(*ins, dy)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    ti = 0.0
    for _ in range(reps):  # inference forward (no residual)
        ev[0].record()
        op.forward(*ins, save=False)
        ev[1].record()
        torch.cuda.synchronize()
        ti += ev[0].elapsed_time(ev[1])
    tf, tb, ti = tf / reps, tb / reps, ti / reps
    # per-scan B/C (G = 1): memsim.cpp:45-46; shared B/C: B/C bytes once per group
    cells = H * W * 4
    fb = cells * (3 * S + 2 * N * (S // G))
    bb = cells * (5 * S + 4 * N * (S // G))
    return {"shape": [S, H, W, N, G], "fwd_ms": round(tf, 4), "fwd_infer_ms": round(ti, 4), "bwd_ms": round(tb, 4),
            "fwd_gbs": round(fb / tf / 1e6, 1), "bwd_gbs": round(bb / tb / 1e6, 1), "plan_f": op.plan()}


if __name__ == "__main__":
    for a in sys.argv[1:]:
        print(json.dumps(run(*[int(v) for v in a.split(",")])), flush=True)
