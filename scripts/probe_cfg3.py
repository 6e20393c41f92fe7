"""Config 3: worker rate (isolated and in the solve) vs the x-side ceiling at n=1M, theta=50."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

for prec, nm in [(capi.F32, "f32"), (capi.F64, "f64")]:
    for W in [2664, 3552]:
        r = [capi.microbench_xside(1000000, 50, prec, W, 256, mode) for mode in (0, 1, 2)]
        print(f"xside n=1M theta=50 {nm} W={W}: gather+red {r[0]:.3e}  gather {r[1]:.3e}  red {r[2]:.3e} proj/s")
A, b, xs = capi.generate_fixed_theta(2000000, 1000000, 50, seed=1003, dist="uniform")
for prec, nm in [(capi.F32, "f32"), (capi.F32X64, "f32x64")]:
    S = capi.System(A, b, precision=prec)
    print(nm, "max resident warps", S.max_resident_warps())
    for W in [2664, S.max_resident_warps()]:
        t = S.solve(threads=W, epochs=400, target=1e-10 * float(b @ b), sampling=capi.WITH_REPLACEMENT, seed=3,
                    precision=prec, want_x=False)
        st = S.stats()
        print(f"  {nm} W={W}: solve {st['solve_ms']:.1f} ms epochs {int(t['epoch_index'][-1])} "
              f"worker {st['projections']/(st['worker_ms']*1e-3):.3e} proj/s (worker share {st['worker_ms']/st['solve_ms']:.2f})")
    S.close()
