"""Small fwd+bwd runs of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck).  usage: compute-sanitizer --tool T python tools/sanitize.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_00678_b200.api import (Scan2dOp, tiled_scan_2d_backward, tiled_scan_2d_forward,  # noqa: E402
                                       train_host)

dev = torch.device("cuda", 0)
for (S, H, W, N) in [(2, 9, 40, 16), (3, 9, 212, 16), (2, 6, 40, 4), (2, 5, 20, 32), (5, 9, 56, 1), (9, 7, 7, 1),
                     (2, 5, 21, 64), (1, 3, 8, 200), (2, 9, 14, 16), (3, 7, 7, 8)]:
    for dt in (torch.float32, torch.float64):
      for acc in ((False, True) if dt == torch.float32 else (False,)):
        g = torch.Generator(device=dev).manual_seed(1)
        r = lambda *s: torch.randn(*s, generator=g, device=dev, dtype=dt)
        x, z, B, C, dy = r(S, H, W), r(S, H, W), r(S, H, W, N), r(S, H, W, N), r(S, H, W)
        A = -(0.05 + 0.9 * torch.rand(S, N, generator=g, device=dev, dtype=dt))
        D, bias = r(S), torch.rand(S, generator=g, device=dev, dtype=dt) - 0.5
        op = Scan2dOp(S, H, W, N, dtype=dt, device=dev, accurate=acc)
        op.forward(x, z, B, C, A, D, bias)
        op.backward(x, z, B, C, A, D, bias, dy)
        # reference CarryState emission (tile kernels emit it too)
        res = tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=5, carries=True)
        tiled_scan_2d_backward(res.saved, dy)
        torch.cuda.synchronize()
        print("ok", S, H, W, N, dt, "accurate" if acc else "", flush=True)
# shared B/C (G > 1) with the in-kernel group reductions and shared parameters (P < S)
for (S, H, W, N, P, G) in [(4, 9, 40, 16, 2, 4), (6, 9, 212, 16, 3, 3), (4, 6, 20, 4, 4, 2)]:
    for red in (False, True):
        g = torch.Generator(device=dev).manual_seed(4)
        r = lambda *s: torch.randn(*s, generator=g, device=dev)
        x, z, dy = r(S, H, W), r(S, H, W), r(S, H, W)
        B, C_ = r(S // G, H, W, N), r(S // G, H, W, N)
        A = -(0.05 + 0.9 * torch.rand(P, N, generator=g, device=dev))
        D, bias = r(P), torch.rand(P, generator=g, device=dev) - 0.5
        op = Scan2dOp(S, H, W, N, params_period=P, bc_group=G, device=dev, group_red=red)
        op.forward(x, z, B, C_, A, D, bias)
        op.backward(x, z, B, C_, A, D, bias, dy)
        torch.cuda.synchronize()
        print("ok shared", S, H, W, N, P, G, "group_red" if red else "", flush=True)
# comparators (naive 2D, flat 1D block scan)
import ctypes as C  # noqa: E402

from paper_2412_00678_b200 import _native as nat  # noqa: E402

for (S, H, W, N) in [(2, 30, 40, 16), (1, 14, 14, 16), (2, 7, 9, 3)]:
    g = torch.Generator(device=dev).manual_seed(3)
    r = lambda *s: torch.randn(*s, generator=g, device=dev)
    ins = [r(S, H, W), r(S, H, W), r(S, H, W, N), r(S, H, W, N), -(0.05 + 0.9 * torch.rand(S, N, generator=g, device=dev)),
           r(S), torch.rand(S, generator=g, device=dev) - 0.5]
    y = torch.empty(S, H, W, device=dev)
    d = nat.make_desc(S, H, W, N)
    for var in (nat.VARIANT_NAIVE, nat.VARIANT_FLAT1D):
        wsb = nat.lib.scan2d_comparator_workspace_bytes(C.byref(d), var)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
        rc = nat.lib.scan2d_forward_variant(C.byref(d), var, *[C.c_void_p(t.data_ptr()) for t in ins],
                                            C.c_void_p(y.data_ptr()), C.c_void_p(ws.data_ptr()), wsb,
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
    torch.cuda.synchronize()
    print("ok comparators", S, H, W, N, flush=True)
g = torch.Generator(device=dev).manual_seed(2)
S, H, W, N = 33, 8, 16, 16  # two chunks of 17 / 16 scans, ends split into 1/8,1/8,1/4,1/2 pieces
r = lambda *s: torch.randn(*s, generator=g, device=dev)
hin = [t.cpu().pin_memory() for t in (r(S, H, W), r(S, H, W), r(S, H, W, N), r(S, H, W, N),
                                      -(0.05 + 0.9 * torch.rand(S, N, generator=g, device=dev)), r(S),
                                      torch.rand(S, generator=g, device=dev) - 0.5)]
train_host(*hin, dy=r(S, H, W).cpu().pin_memory(), chunks=2)
torch.cuda.synchronize()
print("ok host path")
