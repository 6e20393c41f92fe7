"""Probe: deterministic worker time vs ASYRK_DET_POLL_NS (set per process)."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    from paper_1401_4780_b200 import capi
    A, b, _ = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
    S = capi.System(A, b)
    A0, b0, _ = capi.generate_fixed_theta(4000, 1000, 10, seed=7)
    b0 = b0 + 0.5 * np.random.default_rng(7).standard_normal(4000)
    aug = capi.lsq_augment(A0, b0, 0.6, 1.0)
    S2 = capi.System(aug["a_tilde"], aug["b_tilde"])
    out = []
    for SS, ep in [(S, 20), (S2, 50)]:
        best = 1e9
        for _ in range(3):
            SS.rk_solve(max_epochs=ep, seed=42)
            best = min(best, SS.stats()["worker_ms"] / ep)
        out.append(best)
    print(f"poll_ns {os.environ.get('ASYRK_DET_POLL_NS')}: cfg1 {out[0]:.3f} ms/epoch, lsq-aug {out[1]:.3f} ms/epoch",
          flush=True)
else:
    for p in [0, 16, 32, 64, 128, 256, 512]:
        subprocess.run([sys.executable, __file__, "x"], env=dict(os.environ, ASYRK_DET_POLL_NS=str(p)))
