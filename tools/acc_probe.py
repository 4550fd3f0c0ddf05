"""Diagnostics: fp32 normwise error (vs the fp64 oracle) of the default and the
accurate-exponential mode, beside the reference's own fp32 engine.
usage: python tools/acc_probe.py"""
import sys, os, time
import numpy as np
import torch
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
from oracle_lib import Oracle, rel_error  # noqa: E402
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd  # noqa: E402
from paper_2412_00678_b200 import tiled_scan_2d_backward, tiled_scan_2d_forward  # noqa: E402

orc = Oracle()
for (S, H, W, N) in [(4, 200, 200, 16), (16, 56, 56, 1), (32, 16, 16, 16), (4, 60, 90, 8), (2, 64, 64, 32)]:
    b = make_batch(orc, S, H, W, N, seed0=9000, dtype="f32")
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    ref = oracle_bwd(orc, b, "f64"); ref["y"] = oracle_fwd(orc, b, "f64")
    r32 = oracle_bwd(orc, b, "f32"); r32["y"] = oracle_fwd(orc, b, "f32")
    rows = {}
    for acc in (False, True):
        res = tiled_scan_2d_forward(x, z, B, C, A, D, bias, accurate=acc)
        g = tiled_scan_2d_backward(res.saved, dy)
        torch.cuda.synchronize()
        got = dict(y=res.y, dx=g.dx, dz=g.dz_raw, dA=g.da, dB=g.db, dC=g.dc, dD=g.dd, dbias=g.dbias)
        rows[acc] = {k: rel_error(v.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1)) for k, v in got.items()}
    rf = {k: rel_error(np.asarray(r32[k]).reshape(-1), np.asarray(ref[k]).reshape(-1)) for k in rows[False]}
    print(f"S={S} {H}x{W} N={N}")
    for k in rows[False]:
        print(f"  {k:6s} fast {rows[False][k]:.2e}  accurate {rows[True][k]:.2e}  ref-f32 {rf[k]:.2e}")
