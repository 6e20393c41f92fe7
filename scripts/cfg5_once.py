"""Dev: one config-5 tolerance solve after a warm-up (for ncu launch lists)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, B, Xs = capi.generate_fixed_theta(500000, 250000, 20, seed=1005, k=64)
B = B.astype(np.float32)
bb = float((B.astype(np.float64) ** 2).sum())
S = capi.MultiRHS(A, B, 0, 64)
for seed in (1, 2):
    t = S.solve(threads=4096, epochs=400, target=1e-10 * bb, seed=seed, sampling=capi.SLICE_SHUFFLE)
print(S.stats(), list(t["epoch_index"]))
