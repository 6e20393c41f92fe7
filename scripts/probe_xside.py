"""Dev probe: x-side roofline microbenchmark (R_x) at config-2 shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

for prec, nm in [(capi.F64, "f64"), (capi.F32, "f32")]:
    for W in [1184, 2368, 3552, 4736, 9472]:
        r = [capi.microbench_xside(100000, 30, prec, W, 512, mode) for mode in (0, 1, 2)]
        print(f"{nm} W={W}: gather+red {r[0]:.3e}  gather {r[1]:.3e}  red {r[2]:.3e} proj/s")
