"""Dev probe: latency/throughput of the deterministic dataflow worker."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402


def csr(m, n, cols_per_row, rng):
    th = cols_per_row.shape[1]
    v = rng.standard_normal((m, th))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return capi.HostCsr(m, n, np.arange(m + 1) * th, cols_per_row.ravel(), v.ravel())


rng = np.random.default_rng(0)
# (a) fully dependent chain: two rows over the same 20 columns
A = csr(2, 20, np.tile(np.arange(20), (2, 1)), rng)
S = capi.System(A, rng.standard_normal(2))
E = 20000
S.solve(threads=1, epochs=E, snapshot_interval=E, sampling=capi.WITH_REPLACEMENT)
st = S.stats()
print(f"chain: {st['worker_ms']*1e3/(2*E):.3f} us/event  (worker {st['worker_ms']:.1f} ms)")
# (b) independent rows: disjoint supports
m = 20000
A = csr(m, 20 * m, np.arange(20 * m).reshape(m, 20), rng)
S = capi.System(A, rng.standard_normal(m))
S.solve(threads=1, epochs=20, snapshot_interval=20, sampling=capi.SLICE_SHUFFLE)
st = S.stats()
print(f"independent: {st['worker_ms']*1e3/(20*m):.3f} us/event  (worker {st['worker_ms']:.1f} ms, n={20*m} -> "
      f"{'smem' if 20*m*12 < 200*1024 else 'serial kernel'})")
m, n = 20000, 10000
A = csr(m, n, np.sort(np.stack([rng.choice(n, 20, replace=False) for _ in range(m)]), axis=1), rng)
S = capi.System(A, rng.standard_normal(m))
S.solve(threads=1, epochs=20, snapshot_interval=20, sampling=capi.WITH_REPLACEMENT)
st = S.stats()
print(f"config1-like: {st['worker_ms']*1e3/(20*m):.3f} us/event  (worker {st['worker_ms']:.1f} ms)")
