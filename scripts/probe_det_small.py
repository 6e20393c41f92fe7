"""Probe: where the deterministic path's time goes on a small, tightly coupled
system (the lsq augmented system) — device solve stats per epoch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1401_4780_b200 import capi  # noqa: E402

m, n, th = 4000, 1000, 10
A, b, xs = capi.generate_fixed_theta(m, n, th, seed=7)
b = b + 0.5 * np.random.default_rng(7).standard_normal(m)
sv = capi.dense_svd(A)
sr = float(sv["sigma"][sv["rank"] - 1])
phi, zeta = capi.lsq_optimal_params(sr)
aug = capi.lsq_augment(A, b, zeta, phi)
At, bt = aug["a_tilde"], aug["b_tilde"]
print("augmented", At.m, At.n, At.nnz, "max row", int(np.diff(At.row_ptr).max()))
S = capi.System(At, bt)
for ep in [1, 10, 104]:
    for rep in range(2):
        t0 = time.perf_counter()
        t = S.rk_solve(max_epochs=ep, seed=1)
        dt = time.perf_counter() - t0
    st = S.stats()
    print(f"epochs {ep}: wall {dt*1e3:.2f} ms  solve {st['solve_ms']:.2f} worker {st['worker_ms']:.2f} "
          f"monitor {st['monitor_ms']:.2f} launches {st['kernel_launches']}  per-epoch {dt*1e3/ep:.3f} ms", flush=True)
A2, b2, _ = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
S2 = capi.System(A2, b2)
for rep in range(2):
    t0 = time.perf_counter()
    S2.rk_solve(max_epochs=20, seed=42)
    dt = time.perf_counter() - t0
st = S2.stats()
print(f"cfg1: wall {dt*1e3:.2f} ms solve {st['solve_ms']:.2f} worker {st['worker_ms']:.2f} monitor {st['monitor_ms']:.2f}")
