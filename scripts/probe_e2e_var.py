"""Per-call wall times of the one-shot e2e path (config 2)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
target = 1e-12 * float(b @ b)
S = capi.System(A, b)
S.solve(threads=2664, epochs=2000, target=target, sampling=capi.WITH_REPLACEMENT, seed=1)
S.close()
for k in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = capi.solve_parallel_host(A, b, threads=2664, gamma=1.0, epochs=2000, target=target,
                                 sampling=capi.WITH_REPLACEMENT, seed=2000 + k)
    print(f"call {k}: {1e3*(time.perf_counter()-t0):.2f} ms epochs {int(r['epoch_index'][-1])}", flush=True)
