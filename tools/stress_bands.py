"""Randomised row-band sweep on the GPU (not part of the pytest suite): a grid
split into k aligned row bands (scan2d_forward_band / scan2d_backward_band,
vertical carries passed band to band) must reproduce the single-band run bit
for bit for y, dx, dz, dB, dC, and dA / dDskip / dbias up to the order of the
band sum.

usage: python tools/stress_bands.py <n_cases> [seed]"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from oracle_lib import Oracle, rel_error  # noqa: E402
from scan_cases import batch_to_torch, make_batch  # noqa: E402
from paper_2412_00678_b200.api import Scan2dBandOp, Scan2dOp  # noqa: E402
from paper_2412_00678_b200.launcher import band_align, row_band  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    rng = np.random.default_rng(seed)
    orc = Oracle()
    fails, t0 = 0, time.time()
    for c in range(n):
        N = int(rng.choice([4, 8, 16, 32]))
        dt = str(rng.choice(["f32", "f64"]))
        al = band_align(N, 4 if dt == "f32" else 8)
        nb = int(rng.integers(2, 6))
        H = int(rng.integers(nb * al, nb * al + 3 * al + 7))
        W = 4 * int(rng.integers(1, 75))  # band entry points need 16-byte aligned rows
        S = int(rng.integers(1, 5))
        label = f"#{c} S={S} {H}x{W} N={N} {dt} bands={nb} align={al}"
        try:
            b = make_batch(orc, S, H, W, N, seed0=700 + c, dtype=dt)
            (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
            tdt = x.dtype
            full = Scan2dOp(S, H, W, N, dtype=tdt, device="cuda")
            y_full = full.forward(x, z, B, C, A, D, bias).clone()
            g_full = [t.clone() for t in full.backward(x, z, B, C, A, D, bias, dy)]
            bands = [row_band(H, nb, r, al) for r in range(nb)]
            bands = [bd for bd in bands if bd.rows > 0]
            sl = lambda t, bd: t[:, bd.r0:bd.r1].contiguous()
            ops, tops, ys = [], [None], []
            for bd in bands:
                op = Scan2dBandOp(S, bd.rows, W, N, dtype=tdt, device="cuda")
                y, hb = op.forward(sl(x, bd), sl(z, bd), sl(B, bd), sl(C, bd), A, D, bias, h_top=tops[-1])
                ys.append(y.clone())
                tops.append(hb.clone())
                ops.append(op)
            g, outs = None, {}
            for k in range(len(bands) - 1, -1, -1):
                bd = bands[k]
                res = ops[k].backward(sl(x, bd), sl(z, bd), sl(B, bd), sl(C, bd), A, D, bias, tops[k],
                                      sl(dy, bd), g)
                g = res[-1].clone()
                outs[k] = [t.clone() for t in res[:-1]]
            torch.cuda.synchronize()
            bad = []
            if not torch.equal(torch.cat(ys, dim=1), y_full):
                bad.append("y")
            for idx, name in [(0, "dx"), (1, "dz"), (3, "dB"), (4, "dC")]:
                if not torch.equal(torch.cat([outs[k][idx] for k in range(len(bands))], dim=1), g_full[idx]):
                    bad.append(name)
            for idx, name in [(2, "dA"), (5, "dD"), (6, "dbias")]:
                tot = sum(outs[k][idx] for k in range(len(bands)))
                if rel_error(tot.cpu().numpy(), g_full[idx].cpu().numpy()) > (1e-4 if dt == "f32" else 1e-12):
                    bad.append(name)
            if bad:
                fails += 1
                print("FAIL", label, bad, flush=True)
        except Exception as exc:  # noqa: BLE001
            fails += 1
            print("ERROR", label, repr(exc)[:200], flush=True)
    print(f"bands: {n} cases, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
