"""Dev probe: config-5 worker / monitor cost per epoch (1 GPU).

Runs fixed 6-epoch solves (every boundary evaluated) and tolerance solves per
(kl, warps, sampling), prints per-epoch worker and monitor times from the
library's event timers and the multi-RHS x-side ceiling at the same shape.
Env: KLS, WARPS, SAMPLINGS; ASYRK_MRHS_ROWS (1/2/4) / ASYRK_MRHS_NOSTREAM /
ASYRK_MRHS_MINB select worker variants (A/B).
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
variant = {k: os.environ[k] for k in ("ASYRK_MRHS_ROWS", "ASYRK_MRHS_NOSTREAM", "ASYRK_MRHS_MINB", "ASYRK_MRHS_BATCH", "ASYRK_MRHS_ROWPAR", "ASYRK_MRHS_CSC_MONITOR") if k in os.environ}
kls = [int(v) for v in os.environ.get("KLS", "64").split(",")]
samps = os.environ.get("SAMPLINGS", "slice_shuffle").split(",")
for kl in kls:
    S = capi.MultiRHS(A, B, 0, kl)
    bbk = float((B[:, :kl].astype(np.float64) ** 2).sum())
    for W in ([int(v) for v in os.environ["WARPS"].split(",")] if "WARPS" in os.environ
              else [S.max_resident_warps()]):
        rowpar = kl in (8, 16, 32) and not any(k in os.environ for k in ("ASYRK_MRHS_ROWS", "ASYRK_MRHS_BATCH")) \
            and os.environ.get("ASYRK_MRHS_ROWPAR", "") != "0"
        rx = max(S.microbench_xside(W // (128 // kl) if rowpar else W, 64) for _ in range(2))  # on the shard's own X
        for nm in samps:
            samp = capi.SLICE_SHUFFLE if nm == "slice_shuffle" else capi.WITH_REPLACEMENT
            S.solve(threads=W, epochs=2, target=0.0, seed=1, sampling=samp, want_x=False)
            S.solve(threads=W, epochs=6, target=0.0, seed=2, sampling=samp, want_x=False)
            st = S.stats()
            wl = st["worker_launches"]
            per_w = st["worker_ms"] / wl
            per_m = (st["solve_ms"] - st["worker_ms"]) / (wl + 1)
            t0 = time.perf_counter()
            t = S.solve(threads=W, epochs=400, target=1e-10 * bbk, seed=3, sampling=samp, want_x=False)
            wall = time.perf_counter() - t0
            st2 = S.stats()
            print(json.dumps({"kl": kl, "warps": W, "sampling": nm, "variant": variant,
                              "worker_ms_per_epoch": round(per_w, 4), "monitor_ms_per_eval": round(per_m, 4),
                              "worker_proj_per_s": A.m / (per_w * 1e-3), "R_x_mrhs_proj_per_s": rx,
                              "frac_of_R_x": A.m / (per_w * 1e-3) / rx,
                              "solve_ms": round(st2["solve_ms"], 3), "host_wall_ms": round(1e3 * wall, 3),
                              "epochs": int(t["epoch_index"][-1]), "records": len(t["epoch_index"]),
                              "record_epochs": [int(e) for e in t["epoch_index"]],
                              "worker_ms": round(st2["worker_ms"], 3),
                              "rel": float(np.sqrt(t["r_sq"][-1] / bbk))}), flush=True)
    S.close()
