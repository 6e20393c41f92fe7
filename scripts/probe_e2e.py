"""e2e phase breakdown on config 2: system build (upload + pack + SELL), solve, one-shot call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
target = 1e-12 * float(b @ b)
print("host cores", len(os.sched_getaffinity(0)))
W = 2664
kw = dict(threads=W, gamma=1.0, epochs=2000, target=target, sampling=capi.WITH_REPLACEMENT, snapshot_interval=1)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S = capi.System(A, b)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = S.solve(seed=5 + rep, want_x=True, **kw)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del S
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    r2 = capi.solve_parallel_host(A, b, seed=9 + rep, **kw)
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.2f} ms  solve {1e3*(t2-t1):7.2f} ms  destroy {1e3*(t3-t2):6.2f} ms  "
          f"one-shot {1e3*(t4-t3):7.2f} ms  epochs {int(r['epoch_index'][-1])}/{int(r2['epoch_index'][-1])}")
