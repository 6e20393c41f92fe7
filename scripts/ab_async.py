"""Dev A/B: config-2 async solve time (device events, L2 flushed between
solves) with the library ASYRK_LIB points at. Prints median ms per solve and
median epochs over 20 solves after 3 warm-ups."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

samp = {"slice": capi.SLICE_SHUFFLE, "uniform": capi.WITH_REPLACEMENT}[sys.argv[1] if len(sys.argv) > 1 else "slice"]
A, b, xs = capi.generate_fixed_theta(200_000, 100_000, 30, seed=2024)
bb = float(b @ b)
stream = torch.cuda.Stream()
S = capi.System(A, b, stream=stream.cuda_stream)
W = S.max_resident_warps()
kw = dict(threads=W, gamma=1.0, epochs=2000, target=1e-12 * bb, sampling=samp, snapshot_interval=1, want_x=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts, eps = [], []
for k in range(23):
    with torch.cuda.stream(stream):
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    r = S.solve(seed=1000 + k, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    if k >= 3:
        ts.append(e0.elapsed_time(e1))
        eps.append(int(r["epoch_index"][-1]))
print(os.environ.get("ASYRK_LIB", "default"), sys.argv[1:], "median ms", round(statistics.median(ts), 4),
      "min", round(min(ts), 4), "median epochs", statistics.median(eps), "ms/epoch", round(statistics.median(ts) / statistics.median(eps), 5))
