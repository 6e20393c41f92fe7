"""One cfg1 deterministic solve (for ncu launch lists)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402
A, b, _ = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
S = capi.System(A, b)
S.rk_solve(max_epochs=20, seed=42)
print(S.stats())
