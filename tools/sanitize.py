"""Small fwd+bwd runs of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck).  usage: compute-sanitizer --tool T python tools/sanitize.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_00678_b200.api import Scan2dOp, train_host  # noqa: E402

dev = torch.device("cuda", 0)
for (S, H, W, N) in [(2, 9, 40, 16), (3, 9, 212, 16), (2, 6, 40, 4), (2, 5, 20, 32), (5, 9, 56, 1), (9, 7, 7, 1),
                     (2, 5, 21, 64), (1, 3, 8, 200)]:
    for dt in (torch.float32, torch.float64):
        g = torch.Generator(device=dev).manual_seed(1)
        r = lambda *s: torch.randn(*s, generator=g, device=dev, dtype=dt)
        x, z, B, C, dy = r(S, H, W), r(S, H, W), r(S, H, W, N), r(S, H, W, N), r(S, H, W)
        A = -(0.05 + 0.9 * torch.rand(S, N, generator=g, device=dev, dtype=dt))
        D, bias = r(S), torch.rand(S, generator=g, device=dev, dtype=dt) - 0.5
        op = Scan2dOp(S, H, W, N, dtype=dt, device=dev)
        op.forward(x, z, B, C, A, D, bias)
        op.backward(x, z, B, C, A, D, bias, dy)
        torch.cuda.synchronize()
        print("ok", S, H, W, N, dt, flush=True)
g = torch.Generator(device=dev).manual_seed(2)
S, H, W, N = 33, 8, 16, 16  # two chunks of 17 / 16 scans, ends split into 1/8,1/8,1/4,1/2 pieces
r = lambda *s: torch.randn(*s, generator=g, device=dev)
hin = [t.cpu().pin_memory() for t in (r(S, H, W), r(S, H, W), r(S, H, W, N), r(S, H, W, N),
                                      -(0.05 + 0.9 * torch.rand(S, N, generator=g, device=dev)), r(S),
                                      torch.rand(S, generator=g, device=dev) - 0.5)]
train_host(*hin, dy=r(S, H, W).cpu().pin_memory(), chunks=2)
torch.cuda.synchronize()
print("ok host path")
