"""Dev A/B: config-1 deterministic solve time with a given build of the
library (path argument), raw ctypes so older builds with fewer symbols load.
Prints the median of 5 solve_ms (library event timer) after 2 warm-ups."""
import ctypes as C
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200.capi import CsrView, RkConfig, SolveStats, TraceOut  # noqa: E402

path = sys.argv[1]
reassoc = len(sys.argv) > 2 and sys.argv[2] == "reassoc"
L = C.CDLL(path)
i64, f64 = C.POINTER(C.c_int64), C.POINTER(C.c_double)
m, n, th = 20000, 10000, 20
rp, ci, v, rn = np.zeros(m + 1, np.int64), np.zeros(m * th, np.int64), np.zeros(m * th), np.zeros(m)
b, xs, norm = np.zeros(m), np.zeros(n), C.c_int32()
p = lambda a, t: a.ctypes.data_as(t)  # noqa: E731
assert L.asyrk_generate_fixed_theta(C.c_int64(m), C.c_int64(n), C.c_int64(th), C.c_uint64(1001), C.c_int32(0),
                                    C.c_double(0.0), C.c_int64(1), C.c_int32(0), p(rp, i64), p(ci, i64), p(v, f64),
                                    p(rn, f64), p(b, f64), p(xs, f64), C.byref(norm)) == 0
view = CsrView(m, n, m * th, p(rp, i64), p(ci, i64), p(v, f64), p(rn, f64), norm.value)
h = C.c_void_p()
assert L.asyrk_system_create(C.byref(view), p(b, f64), C.c_int32(0), None, C.byref(h)) == 0
cap = 24
bufs = [np.zeros(cap, np.int64), np.zeros(cap), np.zeros(cap), np.zeros(cap), np.zeros(cap), np.zeros(cap, np.int64)]
x = np.zeros(n)
times = []
for k in range(7):
    cfg = RkConfig(20, 0.0, 42, 0, None, 1 if reassoc else 0)
    tr = TraceOut(cap, 0, p(bufs[0], i64), p(bufs[1], f64), p(bufs[2], f64), p(bufs[3], f64), p(bufs[4], f64),
                  p(bufs[5], i64), p(x, f64))
    assert L.asyrk_system_rk_solve(h, None, C.byref(cfg), C.byref(tr)) == 0
    st = SolveStats()
    L.asyrk_system_last_stats(h, C.byref(st))
    if k >= 2:
        times.append(st.solve_ms)
print(path, "reassoc" if reassoc else "bitwise", "median solve_ms", statistics.median(times), times,
      "x checksum", float(x.sum()))
