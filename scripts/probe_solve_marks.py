"""Dev probe: ASYRK_PROFILE_SOLVE host timestamps of a few config-2 resident solves."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200_000, 100_000, 30, seed=1002)
bb = float(b @ b)
S = capi.System(A, b)
W = S.max_resident_warps()
kw = dict(threads=W, gamma=1.0, epochs=2000, target=1e-12 * bb, sampling=capi.SLICE_SHUFFLE, snapshot_interval=1,
          want_x=False)
for k in range(4):
    S.solve(seed=k, **kw)
os.environ["ASYRK_PROFILE_SOLVE"] = "1"
print("---", flush=True)
for k in range(2):
    S.solve(seed=100 + k, **kw)
    print("library solve_ms", S.stats()["solve_ms"], flush=True)
