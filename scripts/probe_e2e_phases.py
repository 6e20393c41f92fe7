"""Probe: phases of the one-shot host-buffer call at config 2 (ASYRK_PROFILE_CREATE=1
prints the synchronized create phases; the remainder is solve + readback)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
bb = float(b @ b)
W = 3552
for k in range(int(os.environ.get('CALLS', '4'))):
    t0 = time.perf_counter()
    r = capi.solve_parallel_host(A, b, threads=W, gamma=1.0, epochs=2000, target=1e-12 * bb,
                                 sampling=capi.SLICE_SHUFFLE, seed=2000 + k)
    print(f"call {k}: {1e3 * (time.perf_counter() - t0):.2f} ms, epochs {r['epoch_index'][-1]}", flush=True)
t0 = time.perf_counter()
S = capi.System(A, b)
t1 = time.perf_counter()
r = S.solve(threads=W, gamma=1.0, epochs=2000, target=1e-12 * bb, sampling=capi.SLICE_SHUFFLE, seed=7)
t2 = time.perf_counter()
S.close()
t3 = time.perf_counter()
print(f"create {1e3*(t1-t0):.2f} ms, solve {1e3*(t2-t1):.2f} ms (device {S.stats()['solve_ms'] if False else 0}), "
      f"destroy {1e3*(t3-t2):.2f} ms")
