"""Dev probe (history: the coefficient-forwarding kernel it A/B'd lives in
commit 4426b6e and was removed as slower; today it times the tolerance mode):
config-1 tolerance-mode solve against the bitwise mode: median solve_ms of 5 after 2
warm-ups, relative difference of final_x, run-to-run reproducibility; plus
ragged-row systems (E = 2, 4 lanes' slots)."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
with capi.System(A, b) as S:
    for mode in (False, True):
        ts, xs_ = [], []
        for k in range(7):
            r = S.rk_solve(max_epochs=20, seed=42, sampling=capi.RK_UNIFORM, reassociate=mode)
            if k >= 2:
                ts.append(S.stats()["solve_ms"])
            xs_.append(r["final_x"])
        if not mode:
            exact = xs_[-1]
        same = all(np.array_equal(xs_[0], x) for x in xs_)
        rel = np.linalg.norm(xs_[-1] - exact) / np.linalg.norm(exact)
        print(f"cfg1 {'tolerance' if mode else 'bitwise'} fwd_env={os.environ.get('ASYRK_DET_FORWARD')} "
              f"median {statistics.median(ts):.2f} ms {[round(t, 2) for t in ts]} rel {rel:.3e} reproducible {same}",
              flush=True)

if os.environ.get("PROBE_RAGGED", "1") == "0":
    sys.exit(0)
rng = np.random.default_rng(5)
for maxlen in (50, 120):
    m, n = 6000, 3000
    lens = rng.integers(1, maxlen, size=m)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int64)
    v = rng.standard_normal(rp[-1])
    Ar = capi.HostCsr(m, n, rp, ci, v)
    xstar = rng.standard_normal(n)
    br = np.zeros(m)
    for i in range(m):
        br[i] = v[rp[i]:rp[i + 1]] @ xstar[ci[rp[i]:rp[i + 1]]]
    with capi.System(Ar, br) as S:
        for samp in (capi.RK_UNIFORM, capi.RK_SHUFFLE, capi.RK_NORM_PROPORTIONAL):
            e = S.rk_solve(max_epochs=6, seed=9, sampling=samp)["final_x"]
            f = S.rk_solve(max_epochs=6, seed=9, sampling=samp, reassociate=True)["final_x"]
            print(f"ragged maxlen {maxlen} sampling {samp}: rel {np.linalg.norm(f - e) / np.linalg.norm(e):.3e}", flush=True)
