"""Probe: one-shot create (upload) time vs stager threads / chunk (env set by the caller)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
best = 1e9
for k in range(6):
    t0 = time.perf_counter()
    S = capi.System(A, b)
    t1 = time.perf_counter()
    S.close()
    best = min(best, t1 - t0)
print(f"threads={os.environ.get('ASYRK_STAGER_THREADS', 'default')} chunk_kb={os.environ.get('ASYRK_STAGE_CHUNK_KB', '8192')}"
      f" nt={'off' if os.environ.get('ASYRK_NO_NT_STAGING') else 'on'}: create {1e3 * best:.2f} ms (nproc {os.cpu_count()})",
      flush=True)
