"""Time the multithreaded Matrix Market reader/writer against the reference's
(single-threaded ifstream / fprintf) on a config-2-sized instance."""
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402

m, n, th = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (200000, 100000, 30)))
A, b, xs = capi.generate_fixed_theta(m, n, th, seed=1002)
d = tempfile.mkdtemp()
p, q, c = os.path.join(d, "a.mtx"), os.path.join(d, "r.mtx"), os.path.join(d, "a.csr")
t = time.perf_counter(); capi.write_matrix_market(p, A); tw = time.perf_counter() - t
t = time.perf_counter(); B = capi.read_matrix_market(p); tr = time.perf_counter() - t
t = time.perf_counter(); capi.write_csr_cache(c, A); tcw = time.perf_counter() - t
t = time.perf_counter(); C2 = capi.read_csr_cache(c); tcr = time.perf_counter() - t
print(f"{m}x{n} theta={th}: file {os.path.getsize(p)/1e6:.0f} MB; ours write {tw:.2f} s read {tr:.2f} s; "
      f"cache write {tcw:.2f} s read {tcr:.2f} s; threads {os.cpu_count()}")
R = oracle.REF
if R is not None:
    Ar, _ = R.build(m, n, np.repeat(np.arange(m), th), A.col_idx, A.values, False, None)
    t = time.perf_counter(); R.write_mtx(Ar, q); rw = time.perf_counter() - t
    t = time.perf_counter(); Rr = R.read_mtx(p); rr = time.perf_counter() - t
    same = open(p, "rb").read() == open(q, "rb").read()
    print(f"reference write {rw:.2f} s read {rr:.2f} s; identical bytes {same}; "
          f"speedup write {rw/tw:.1f}x read {rr/tr:.1f}x")
