"""Dev probe: where the gap between the bench's event bracket around
System.solve and the library's own solve timer goes (config 2, resident
system): event bracket, host wall of the call, library solve_ms, and the
same through a raw ctypes call with preallocated trace buffers."""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(200_000, 100_000, 30, seed=1002)
bb = float(b @ b)
stream = torch.cuda.Stream()
S = capi.System(A, b, stream=stream.cuda_stream)
W = S.max_resident_warps()
kw = dict(threads=W, gamma=1.0, epochs=2000, target=1e-12 * bb, sampling=capi.SLICE_SHUFFLE, snapshot_interval=1,
          want_x=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = capi.lib()


def bracket(call, n=20):
    ev, wall, lib = [], [], []
    for k in range(n + 3):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        call(k)
        e1.record(stream)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        if k >= 3:
            ev.append(e0.elapsed_time(e1))
            wall.append(1e3 * (t1 - t0))
            lib.append(S.stats()["solve_ms"])
    return statistics.median(ev), statistics.median(wall), statistics.median(lib)


print("System.solve: event %.4f ms, host wall %.4f ms, library solve_ms %.4f ms" % bracket(
    lambda k: S.solve(seed=1000 + k, **kw)))
c = capi._run_config(**{k: v for k, v in kw.items() if k != "want_x"})
cap = 2002
tr = capi._Trace(0, cap, want_x=False)


def raw(k):
    c.seed = 1000 + k
    capi.check(L.asyrk_system_solve(S.h, None, C.byref(c), C.byref(tr.out), None))


print("raw ctypes:   event %.4f ms, host wall %.4f ms, library solve_ms %.4f ms" % bracket(raw))
