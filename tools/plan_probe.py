"""Diagnostics: the plan the library picks for a descriptor (both directions).
usage: python tools/plan_probe.py S H W N"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_00678_b200 import _native as nat  # noqa: E402
S, H, W, N = [int(v) for v in sys.argv[1:5]]
d = nat.make_desc(S, H, W, N)
print("fwd", nat.plan_info(d, nat.OP_FWD))
print("bwd", nat.plan_info(d, nat.OP_BWD))
