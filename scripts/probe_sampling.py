"""Probe: config-2 epochs and device time to 1e-6 per sampling mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
S = capi.System(A, b)
W = S.max_resident_warps()
bb = float(b @ b)
for name, smp in [("with_replacement", capi.WITH_REPLACEMENT), ("slice_shuffle", capi.SLICE_SHUFFLE)]:
    for seed in (3, 4, 5):
        t = S.solve(threads=W, epochs=300, target=1e-12 * bb, sampling=smp, seed=seed, want_x=False)
        st = S.stats()
        print(f"{name:17s} seed {seed}: epochs {t['epoch_index'][-1]:3d}  solve {st['solve_ms']:.2f} ms  "
              f"worker {st['worker_ms']:.2f} ms  per-epoch worker {st['worker_ms'] / t['epoch_index'][-1] * 1e3:.1f} us",
              flush=True)
