"""Probe: device dense SVD and lsq_solve timings (det vs async) against the
reference lsq_solve on the host, on a noisy fixed-theta system."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402

for (m, n, th) in [(2000, 1000, 10), (4000, 1000, 10)]:
    A, b, xs = capi.generate_fixed_theta(m, n, th, seed=7)
    b = b + 0.5 * np.random.default_rng(7).standard_normal(m)
    t0 = time.perf_counter()
    sv = capi.dense_svd(A)
    t_svd = time.perf_counter() - t0
    t0 = time.perf_counter()
    sv = capi.dense_svd(A)
    t_svd2 = time.perf_counter() - t0
    sr = float(sv["sigma"][sv["rank"] - 1])
    print(f"{m}x{n}: dense_svd {t_svd*1e3:.1f} ms (again {t_svd2*1e3:.1f}), sweeps {sv['sweeps']}, sigma_r {sr:.4g}",
          flush=True)
    bb = float(b @ b)
    for thr, g in [(1, 1.0), (64, 1.0), (256, 1.0), (512, 1.0), (512, 0.5), (1024, 0.5), (1024, 0.25)]:
        t0 = time.perf_counter()
        try:
            r = capi.lsq_solve(A, b, sigma_r=sr, max_epochs=20000, target=1e-20 * bb, seed=1, threads=thr, gamma=g)
        except capi.AsyrkError as e:
            print(f"  threads {thr} gamma {g}: {e}", flush=True)
            continue
        dt = time.perf_counter() - t0
        print(f"  threads {thr} gamma {g}: {dt*1e3:.1f} ms, epochs {r['trace']['epoch_index'][-1]}, grad {r['grad_norm']:.3e}",
              flush=True)
    if oracle.REF is not None:
        rows = np.repeat(np.arange(m), np.diff(A.row_ptr))
        Ar, _ = oracle.REF.build(m, n, rows, A.col_idx, A.values, True, None)
        t0 = time.perf_counter()
        rr = oracle.REF.lsq_solve(Ar, b, sr, max_epochs=20000, target=1e-20 * bb, seed=1)
        print(f"  reference lsq_solve (1 core): {(time.perf_counter()-t0)*1e3:.1f} ms, epochs "
              f"{rr['trace']['epoch_index'][-1]}, grad {rr['grad_norm']:.3e}", flush=True)
