"""Diagnostics: CarryState emission (ph / pv) of tiled_scan_2d_forward against
the fp64 oracle over reference tile sizes T in {1, 2, 3, 6, 16} (GPU).
usage: python tools/emit_probe.py"""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle_lib import Oracle, rel_error
from scan_cases import make_batch, batch_to_torch, oracle_bwd
import paper_2412_00678_b200 as s2d
orc = Oracle()
for (S,H,W,N) in [(1,4,5,2),(1,5,4,3),(2,9,13,4),(1,7,7,16),(1,30,40,8)]:
  for T in (1,2,3,6,16):
    for dt in ("f64","f32"):
        b = make_batch(orc, S, H, W, N, seed0=7, dtype=dt)
        (x,z,B,C,A,D,bias), dy = batch_to_torch(b, device="cuda")
        r = s2d.tiled_scan_2d_forward(x,z,B,C,A,D,bias, tile=T, carries=True)
        g = s2d.tiled_scan_2d_backward(r.saved, dy)
        r2 = s2d.tiled_scan_2d_forward(x,z,B,C,A,D,bias, tile=T, carries=False)
        g2 = s2d.tiled_scan_2d_backward(r2.saved, dy)
        ref = oracle_bwd(orc, b, "f64")
        e = {k: rel_error(v.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1)) for k,v in dict(dx=g.dx,dz=g.dz_raw,dA=g.da,dB=g.db,dC=g.dc,dD=g.dd,dbias=g.dbias).items()}
        e2 = {k: rel_error(v.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1)) for k,v in dict(dx=g2.dx,dz=g2.dz_raw,dA=g2.da,dB=g2.db,dC=g2.dc,dD=g2.dd,dbias=g2.dbias).items()}
        w, w2 = max(e.values()), max(e2.values())
        flag = "BAD" if w > (1e-10 if dt=="f64" else 1e-4) else "ok"
        print(flag, S,H,W,N,T,dt, f"emit {w:.2e} noemit {w2:.2e}", max(e, key=e.get))
