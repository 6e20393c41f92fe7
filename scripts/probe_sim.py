"""Time the device Monte-Carlo delay simulator against the reference's CPU
monte_carlo_ratios on acceptance criterion 2's shape (acceptance.cpp:137-155:
1000 runs x 2000 iterations, uniform delays tau=5, single component, m=1200,
n=60)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(1200, 60, 5, 77)
kw = dict(gamma=0.15, tau=5, delay="uniform_random", iterations=2000, base_seed=99)
for runs in [1000, 4000]:
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = capi.monte_carlo_ratios(A, b, np.zeros(60), runs=runs, **kw)
        dt = time.perf_counter() - t
        print(f"device runs={runs}: {dt*1e3:.1f} ms  ({runs*2000/dt/1e6:.1f} M iterations/s)")
with capi.System(A, b) as S:
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = S.monte_carlo_ratios(np.zeros(60), runs=1000, **kw)
        dt = time.perf_counter() - t
        print(f"device resident runs=1000: {dt*1e3:.1f} ms")
Ac = oracle.C.from_arrays(1200, 60, A.row_ptr, A.col_idx, A.values)
t = time.perf_counter()
rc = oracle.C.monte_carlo(Ac, b, np.zeros(60), runs=100, **kw)
dt = time.perf_counter() - t
print(f"oracle C (1 thread) runs=100: {dt*1e3:.1f} ms -> 1000 runs ~{dt*1e4:.0f} ms")
if oracle.REF is not None:
    Ar, _ = oracle.REF.build(1200, 60, np.repeat(np.arange(1200), 5), A.col_idx, A.values, True, None)
    t = time.perf_counter()
    rr = oracle.REF.monte_carlo(Ar, b, np.zeros(60), runs=100, **kw)
    dt = time.perf_counter() - t
    print(f"reference (1 thread) runs=100: {dt*1e3:.1f} ms -> 1000 runs ~{dt*1e4:.0f} ms")
    r100 = capi.monte_carlo_ratios(A, b, np.zeros(60), runs=100, **kw)
    print("bitwise vs reference:", np.array_equal(rr["mean_r_sq"], r100["mean_r_sq"]))
