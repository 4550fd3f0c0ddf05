"""Diagnostics: fp32 gradient error of the GPU path against the fp64 oracle on
a family of shapes, beside the reference's own fp32 arithmetic (the oracle's
fp32 restatement) on the same inputs.  Worst case per gradient group.

usage: python tools/dbias_probe.py N H W S n_seeds [seed0]"""
import sys, os
import numpy as np
import torch
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
from oracle_lib import Oracle, rel_error  # noqa: E402
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd  # noqa: E402
from paper_2412_00678_b200 import tiled_scan_2d_backward, tiled_scan_2d_forward  # noqa: E402

N, H, W, S, n = [int(v) for v in sys.argv[1:6]]
seed0 = int(sys.argv[6]) if len(sys.argv) > 6 else 9000
orc = Oracle()
worst = {}
for k in range(n):
    b = make_batch(orc, S, H, W, N, seed0=seed0 + 31 * k, dtype="f32")
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    res = tiled_scan_2d_forward(x, z, B, C, A, D, bias)
    g = tiled_scan_2d_backward(res.saved, dy)
    torch.cuda.synchronize()
    ref = oracle_bwd(orc, b, "f64")
    r32 = oracle_bwd(orc, b, "f32")
    yr = oracle_fwd(orc, b, "f64")
    ref["y"] = yr
    r32["y"] = oracle_fwd(orc, b, "f32")
    got = dict(y=res.y, dx=g.dx, dz=g.dz_raw, dA=g.da, dB=g.db, dC=g.dc, dD=g.dd, dbias=g.dbias)
    for key, t in got.items():
        e = rel_error(t.cpu().numpy().reshape(-1), np.asarray(ref[key]).reshape(-1))
        e32 = rel_error(np.asarray(r32[key]).reshape(-1), np.asarray(ref[key]).reshape(-1))
        if e > worst.get(key, (0, 0, 0))[0]:
            worst[key] = (e, e32, seed0 + 31 * k)
for key, (e, e32, sd) in worst.items():
    print(f"{key:6s} gpu {e:.2e}  ref-f32 {e32:.2e}  (seed0 {sd})")
