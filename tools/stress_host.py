"""Randomised sweep of the host-operand path (scan2d_train_host: chunked,
ramped, three streams) against the device path: per-scan and per-group
outputs must be identical; parameter gradients that the host path sums over
chunks (shared parameters, P < S) agree to 1e-6 (normwise) -- the model
layout (shared B/C, G > 1; shared parameters) on a third of the cases.

usage: python tools/stress_host.py <n_cases> [seed]"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2412_00678_b200.api import Scan2dOp, train_host  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rng = np.random.default_rng(seed)
    fails, t0 = 0, time.time()
    for c in range(n):
        model = rng.random() < 0.33
        G = int(rng.choice([1, 2, 3, 4, 8])) if model else 1
        Pd = int(rng.choice([1, 2, 3])) if model else 1  # S / P
        S = G * Pd * int(rng.integers(1, 8)) if model else int(rng.integers(1, 70))
        P = S // Pd
        if model and S % G:  # keep G | S
            G = 1
        H = int(rng.integers(1, 40))
        W = int(rng.integers(1, 120))
        N = int(rng.choice([1, 4, 8, 16, 16, 32, 40]))
        dt = torch.float32 if rng.random() < 0.8 else torch.float64
        chunks = int(rng.choice([0, 1, 2, 3, 5, 8, 13]))
        bwd = rng.random() < 0.85
        label = f"#{c} S={S} {H}x{W} N={N} P={P} G={G} {dt} chunks={chunks} bwd={bwd}"
        try:
            g = torch.Generator(device="cuda").manual_seed(c)
            r = lambda *s: torch.randn(*s, generator=g, device="cuda", dtype=dt)
            x, z, B, C, dy = r(S, H, W), r(S, H, W), r(S // G, H, W, N), r(S // G, H, W, N), r(S, H, W)
            A = -(0.05 + 0.9 * torch.rand(P, N, generator=g, device="cuda", dtype=dt))
            D, bias = r(P), torch.rand(P, generator=g, device="cuda", dtype=dt) - 0.5
            ins = (x, z, B, C, A, D, bias)
            op = Scan2dOp(S, H, W, N, dtype=dt, device="cuda", with_backward=bwd, params_period=P, bc_group=G)
            y = op.forward(*ins, save=bwd).clone()
            grads = [t.clone() for t in op.backward(*ins, dy)] if bwd else []
            hin = [t.cpu().pin_memory() for t in ins]
            outs = train_host(*hin, dy=dy.cpu().pin_memory() if bwd else None, chunks=chunks)
            torch.cuda.synchronize()
            bad = []
            if not torch.equal(outs[0], y.cpu()):
                bad.append("y")
            if bwd:
                # host outs: y, dx, dz, dA, dB, dC, dD, dbias; device grads: dx, dz, dA, dB, dC, dD, dbias
                for name, ho, dg in zip(("dx", "dz", "dA", "dB", "dC", "dD", "dbias"), outs[1:], grads):
                    if name in ("dA", "dD", "dbias") and P < S:  # summed over chunks in another order
                        den = max(float(torch.linalg.vector_norm(dg.double())), 1e-30)
                        if float(torch.linalg.vector_norm(ho.double() - dg.cpu().double())) / den > 1e-6:
                            bad.append(name)
                    elif not torch.equal(ho, dg.cpu()):
                        bad.append(name)
            if bad:
                fails += 1
                print("FAIL", label, bad, flush=True)
        except Exception as exc:  # noqa: BLE001
            fails += 1
            print("ERROR", label, repr(exc)[:200], flush=True)
    print(f"host: {n} cases, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
