"""Dev probe: config-5 solve with and without the X download (host wall per call)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, B, Xs = capi.generate_fixed_theta(500000, 250000, 20, seed=1005, k=64)
B = B.astype(np.float32)
bb = float((B.astype(np.float64) ** 2).sum())
S = capi.MultiRHS(A, B, 0, 64)
W = S.max_resident_warps()
for want in (False, True, False, True):
    ts = []
    for k in range(4):
        t0 = time.perf_counter()
        S.solve(threads=W, epochs=400, target=1e-10 * bb, seed=k, want_x=want)
        ts.append(1e3 * (time.perf_counter() - t0))
    print("want_x", want, "ms per call", [round(t, 2) for t in ts], flush=True)
