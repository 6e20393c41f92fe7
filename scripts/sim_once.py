"""One Monte-Carlo call (acceptance C2 shape) for ncu captures."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(1200, 60, 5, 77)
with capi.System(A, b) as S:
    for _ in range(2):
        S.monte_carlo_ratios(np.zeros(60), gamma=0.15, tau=5, delay="uniform_random", iterations=2000, runs=1000,
                             base_seed=99)
