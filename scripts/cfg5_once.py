"""Dev: one config-5 tolerance solve after a warm-up (for ncu launch lists).
KL=<columns> (default 64) solves a narrower shard (the multi-GPU widths)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

kl = int(os.environ.get("KL", "64"))
A, B, Xs = capi.generate_fixed_theta(500000, 250000, 20, seed=1005, k=64)
B = B.astype(np.float32)
bb = float((B[:, :kl].astype(np.float64) ** 2).sum())
S = capi.MultiRHS(A, B, 0, kl)
W = S.max_resident_warps()
for seed in (1, 2):
    t = S.solve(threads=W, epochs=400, target=1e-10 * bb, seed=seed, sampling=capi.SLICE_SHUFFLE, want_x=False)
print(W, S.stats(), list(t["epoch_index"]))
