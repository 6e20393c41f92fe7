"""Dev probe: config-5 worker / monitor cost per epoch (1 GPU, all 64 columns).

Runs fixed 6-epoch solves (every boundary evaluated) and full tolerance solves,
prints per-epoch worker and monitor times from the library's own event timers.
Set ASYRK_MRHS_ROWS2=1 for the 2-rows-in-flight worker (A/B).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, B, Xs = capi.generate_fixed_theta(500000, 250000, 20, seed=1005, k=64)
B = B.astype(np.float32)
bb = float((B.astype(np.float64) ** 2).sum())
kls = [int(v) for v in os.environ.get("KLS", "64").split(",")]
for kl in kls:
    S = capi.MultiRHS(A, B, 0, kl)
    bbk = float((B[:, :kl].astype(np.float64) ** 2).sum())
    for W in [int(v) for v in os.environ.get("WARPS", "4096").split(",")]:
        for samp, nm in [(capi.WITH_REPLACEMENT, "with_replacement"), (capi.SLICE_SHUFFLE, "slice_shuffle")]:
            S.solve(threads=W, epochs=2, target=0.0, seed=1, sampling=samp)
            S.solve(threads=W, epochs=6, target=0.0, seed=2, sampling=samp)
            st = S.stats()
            wl = st["worker_launches"]
            per_w = st["worker_ms"] / wl
            per_m = (st["solve_ms"] - st["worker_ms"]) / (wl + 1)
            t0 = time.perf_counter()
            t = S.solve(threads=W, epochs=400, target=1e-10 * bbk, seed=3, sampling=samp)
            wall = time.perf_counter() - t0
            st2 = S.stats()
            print(json.dumps({"kl": kl, "warps": W, "sampling": nm, "rows2": bool(os.environ.get("ASYRK_MRHS_ROWS2")),
                              "worker_ms_per_epoch": round(per_w, 4), "monitor_ms_per_eval": round(per_m, 4),
                              "solve_ms": round(st2["solve_ms"], 3), "host_wall_ms": round(1e3 * wall, 3),
                              "epochs": int(t["epoch_index"][-1]), "records": len(t["epoch_index"]),
                              "record_epochs": [int(e) for e in t["epoch_index"]],
                              "worker_ms": round(st2["worker_ms"], 3),
                              "rel": float(np.sqrt(t["r_sq"][-1] / bbk))}), flush=True)
    S.close()
