#!/usr/bin/env python
"""Generate the golden vectors under tests/golden/ from the REFERENCE library.

Runs only where the reference sources exist (this container): it needs
oracle/_ref/libscan2d_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src/*.cpp.  The outputs are small .npz files committed to
the repository, so the GPU box (which has no /root/reference) can check the
CUDA path against the reference's own numbers.

Cases mirror the reference tests (proj/tests/test_engine.cpp,
proj/tests/test_backward.cpp) plus BASELINE.json configs[0] (64 scans of
16x16, N=16, seeds 1000..1063).  Inputs come from the reference generator
random_instance (fixtures.hpp:20-37); dy from Rng(seed ^ 0x5eed).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib  # noqa: E402

FWD_CASES = [  # (h, w, n, tiles, seed)   test_engine.cpp:12-44, :84-97
    (11, 7, 4, (64,), 42),
    (6, 9, 3, (1,), 43),
    (8, 8, 2, (3,), 44),
    (13, 10, 5, (1, 2, 3, 8, 13), 45),
    (33, 29, 6, (8,), 48),
    (23, 17, 3, (8,), 1000 + 23 * 31 + 17),
]
BWD_CASES = [  # (h, w, n, tile, seed)    test_backward.cpp:11-74, gradcheck instances
    (5, 6, 3, 2, 60),
    (7, 4, 2, 3, 62),
    (5, 4, 3, 3, 0),
    (4, 5, 2, 6, 7),
    (17, 13, 4, 4, 63),
    (16, 16, 16, 16, 1000),
]


def main():
    ref = RefLib()
    out = {}
    for h, w, n, tiles, seed in FWD_CASES:
        for dt in ("f64", "f32"):
            inst = ref.random_instance(h, w, n, seed, dt)
            key = f"fwd_{h}x{w}_n{n}_s{seed}_{dt}"
            out[key + "_x"] = inst.x
            out[key + "_B"] = inst.B
            for t in tiles:
                y, ph, pv = ref.tiled_fwd(inst, t, dt)
                out[f"{key}_t{t}_y"] = y
                out[f"{key}_t{t}_ph"] = ph
                out[f"{key}_t{t}_pv"] = pv
    for h, w, n, t, seed in BWD_CASES:
        for dt in ("f64", "f32"):
            inst = ref.random_instance(h, w, n, seed, dt)
            dy = ref.fill_normal(seed ^ 0x5EED, h * w).astype(np.float64 if dt == "f64" else np.float32)
            g = ref.tiled_bwd(inst, t, dy, dt)
            key = f"bwd_{h}x{w}_n{n}_s{seed}_t{t}_{dt}"
            for k, v in g.items():
                out[f"{key}_{k}"] = np.asarray(v)
    # configs[0]: S=64 scans, 16x16, N=16, T=16, seed 1000+s, fp32 forward
    ys = []
    for s in range(64):
        inst = ref.random_instance(16, 16, 16, 1000 + s, "f32")
        y, _, _ = ref.tiled_fwd(inst, 16, "f32")
        ys.append(y)
    out["cfg1_y_f32"] = np.stack(ys)
    # gradcheck group errors of the reference itself (test_backward.cpp:39-54)
    out["gradcheck_5x4_n3_s0_t3"] = ref.gradcheck(5, 4, 3, 0, 1e-6, 3)
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
