"""Probe: per-event latency of the deterministic dataflow kernel on a pure
dependency chain (every row shares column 0, so event q waits for q-1):
worker time per event vs row length (slope = per-entry cost, intercept =
fixed cost per event on the critical path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1401_4780_b200 import capi  # noqa: E402

m, n = 20000, 4000
rng = np.random.default_rng(0)
for th in [int(t) for t in os.environ.get("THETAS", "2,4,8,16,24,32,48,64").split(",")]:
    cols = np.stack([np.concatenate([[0], 1 + rng.choice(n - 1, th - 1, replace=False)]) for _ in range(m)])
    cols.sort(axis=1)
    v = rng.standard_normal((m, th))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    A = capi.HostCsr(m, n, np.arange(m + 1) * th, cols.ravel(), v.ravel())
    b = np.zeros(m)
    with capi.System(A, rng.standard_normal(m)) as S:
        best = 1e9
        for _ in range(3):
            S.rk_solve(max_epochs=2, seed=1)
            best = min(best, S.stats()["worker_ms"] / 2)
    print(f"poll {os.environ.get('ASYRK_DET_POLL_NS', '32')} theta {th:3d}: {best*1e6/m:7.1f} ns per chained event ({best:.3f} ms/epoch)", flush=True)
