"""Diagnostics: CUDA-event fwd / bwd times of one workload through Scan2dOp.
usage: python tools/time_fb.py S H W N [reps] [G]   (env P = params period, GROUP_RED=1)"""
import sys, os, statistics
import torch
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2412_00678_b200.api import Scan2dOp  # noqa: E402

S, H, W, N = [int(v) for v in sys.argv[1:5]]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 30
G = int(sys.argv[6]) if len(sys.argv) > 6 else 1
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
r = lambda *s: torch.randn(*s, device=dev, generator=g)
P = int(os.environ.get("P", S // G if G > 1 else S))
x, z, dy = r(S, H, W), r(S, H, W), r(S, H, W)
B, C = r(S // G, H, W, N), r(S // G, H, W, N)
A = -(0.05 + 0.9 * torch.rand(P, N, device=dev, generator=g))
D, bias = r(P), 0.5 * r(P)
op = Scan2dOp(S, H, W, N, device=dev, params_period=P, bc_group=G,
              group_red=os.environ.get("GROUP_RED", "0") == "1")
op.check = False
ins = (x, z, B, C, A, D, bias)
for _ in range(3):
    op.forward(*ins); op.backward(*ins, dy)
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
torch.cuda.synchronize()
for e in ev:
    e[0].record(); op.forward(*ins); e[1].record(); op.backward(*ins, dy); e[2].record()
torch.cuda.synchronize()
f = statistics.median(a.elapsed_time(b) for a, b, _ in ev)
b_ = statistics.median(b.elapsed_time(c) for _, b, c in ev)
fb = 4 * S * H * W * (3 + 2 * N) if G == 1 else 4 * H * W * (S * 3 + (S // G) * 2 * N)
bb = 4 * S * H * W * (5 + 4 * N) if G == 1 else 4 * H * W * (S * 5 + (S // G) * 4 * N)
print(f"S={S} {H}x{W} N={N} G={G}: fwd {f*1e3:.1f} us ({fb/f/1e6:.0f} GB/s)  bwd {b_*1e3:.1f} us ({bb/b_/1e6:.0f} GB/s)  plan {op.plan()}")
