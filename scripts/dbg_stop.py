"""Dev probe: early-stop path of the deterministic and async solves."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(2000, 1000, 10, seed=3)
S = capi.System(A, b)
for ep, tgt in [(5, 0.0), (500, 0.0), (500, 1e-6 * float(b @ b)), (20, 1e-6 * float(b @ b))]:
    try:
        t = S.rk_solve(max_epochs=ep, seed=3, target=tgt)
        print("ok", ep, tgt, t["epoch_index"][-1])
    except Exception as e:
        print("ERR", ep, tgt, e)
