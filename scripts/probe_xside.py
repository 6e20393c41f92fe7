"""Dev probe: x-side roofline microbenchmark (R_x) at config-2 shape.

  python scripts/probe_xside.py        sweep warps x {1, 2 rows in flight} x modes
  python scripts/probe_xside.py ncu    one launch pair per shape for ncu --set full
                                       (2 rows in flight and 1, f64, all resident warps)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "ncu":
    for mode in (16, 0):
        print(f"mode {mode}: {capi.microbench_xside(100000, 30, capi.F64, 3552, 256, mode):.3e} proj/s")
    sys.exit(0)
for prec, nm in [(capi.F64, "f64"), (capi.F32, "f32")]:
    for W in [1184, 2368, 3552, 4736, 9472]:
        for rows in (1, 2):
            off = 16 if rows == 2 else 0
            r = [capi.microbench_xside(100000, 30, prec, W, 512, mode + off) for mode in (0, 1, 2)]
            print(f"{nm} W={W} rows={rows}: gather+red {r[0]:.3e}  gather {r[1]:.3e}  red {r[2]:.3e} proj/s")
