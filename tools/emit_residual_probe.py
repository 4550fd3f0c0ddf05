"""Diagnostics: a training forward WITH CarryState emission into a residual
buffer pre-filled with NaN, then the backward, against the fp64 oracle -- every
residual entry the backward reads must have been written by the forward."""
import ctypes as C
import sys, os
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle_lib import Oracle, rel_error
from scan_cases import make_batch, batch_to_torch, oracle_bwd
from paper_2412_00678_b200 import _native as nat

orc = Oracle()
p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
bad = 0
for (S, H, W, N) in [(1, 4, 5, 2), (1, 5, 4, 3), (2, 9, 13, 4), (1, 7, 7, 16), (1, 30, 40, 8), (3, 20, 200, 16),
                     (2, 33, 29, 6), (1, 12, 300, 1), (2, 40, 70, 1)]:
    for T in (1, 2, 3, 16):
        for dt in ("f64", "f32"):
            for emit in (True, False):
                b = make_batch(orc, S, H, W, N, seed0=7, dtype=dt)
                (x, z, B, Cc, A, D, bias), dy = batch_to_torch(b, device="cuda")
                d = nat.make_desc(S, H, W, N, tile=T, dtype=nat.F64 if dt == "f64" else nat.F32)
                res = torch.full((nat.lib.scan2d_residual_bytes(C.byref(d)) // 4,), float("nan"), device="cuda")
                wf = torch.empty(max(nat.lib.scan2d_workspace_bytes(C.byref(d), 0), 16), dtype=torch.uint8, device="cuda")
                wb = torch.empty(max(nat.lib.scan2d_workspace_bytes(C.byref(d), 1), 16), dtype=torch.uint8, device="cuda")
                y = torch.empty_like(x)
                kh, kw = -(-H // T), -(-W // T)
                ph = torch.empty((S, kh, kw, T, N), dtype=x.dtype, device="cuda") if emit else None
                pv = torch.empty_like(ph) if emit else None
                rc = nat.lib.scan2d_forward(C.byref(d), p(x), p(z), p(B), p(Cc), p(A), p(D), p(bias), p(y), p(ph), p(pv),
                                            p(res), p(wf), wf.numel(), st())
                assert rc == 0, rc
                g = [torch.empty_like(t) for t in (x, x, A, B, Cc, D, bias)]
                rc = nat.lib.scan2d_backward(C.byref(d), p(x), p(z), p(B), p(Cc), p(A), p(D), p(bias), p(res), p(dy),
                                             *[p(t) for t in g], p(wb), wb.numel(), st())
                assert rc == 0, rc
                torch.cuda.synchronize()
                ref = oracle_bwd(orc, b, "f64")
                errs = {k: rel_error(t.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1))
                        for k, t in zip(("dx", "dz", "dA", "dB", "dC", "dD", "dbias"), g)}
                w = max(errs.values())
                if not w <= (1e-10 if dt == "f64" else 1e-4):
                    bad += 1
                    print("BAD", S, H, W, N, T, dt, "emit" if emit else "noemit", {k: f"{v:.1e}" for k, v in errs.items()})
print("bad", bad)
