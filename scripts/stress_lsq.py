"""Randomized bit-identity stress of lsq_solve (σ_r supplied: augment + device
rk_solve) against the unmodified reference lsq_solve (oracle/_ref).
Usage: python scripts/stress_lsq.py [cases] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402


def main():
    if oracle.REF is None:
        print("oracle/_ref not built")
        return 1
    R = oracle.REF
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    t0 = time.time()
    bad = skipped = 0
    for c in range(cases):
        m = int(rng.integers(4, 300))
        n = int(rng.integers(2, max(3, m)))
        lo = min(max(1.5 / n, 0.02), 0.9)
        delta = float(rng.uniform(lo, max(0.6, lo + 0.05)))
        try:
            Ar, b, _ = R.gen_sparse_gaussian(m, n, delta, int(rng.integers(1, 10**6)))
        except oracle.OracleError:
            skipped += 1
            continue
        b = b + float(rng.choice([0.0, 0.3])) * rng.standard_normal(m)
        e = Ar.export()
        A = capi.HostCsr(m, n, e["row_ptr"], e["col_idx"], e["values"], e["row_norm"], normalized=e["normalized"])
        if np.bincount(A.col_idx, minlength=n).min() == 0:
            skipped += 1
            continue
        D = np.zeros((m, n))
        for i in range(m):
            D[i, A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.values[A.row_ptr[i]:A.row_ptr[i + 1]]
        s = np.linalg.svd(D, compute_uv=False)
        sr = float(s[s > 1e-10 * s[0]][-1])
        kw = dict(max_epochs=int(rng.integers(1, 200)), target=float(rng.choice([0.0, 1e-12])),
                  seed=int(rng.integers(0, 2**31)), sampling=str(rng.choice(["uniform", "shuffle"])))
        zeta = float(rng.choice([0.0, 0.0, 0.4]))
        got = capi.lsq_solve(A, b, sigma_r=sr, zeta=zeta, max_epochs=kw["max_epochs"], target=kw["target"],
                             seed=kw["seed"], sampling=capi.RK_UNIFORM if kw["sampling"] == "uniform" else capi.RK_SHUFFLE)
        want = R.lsq_solve(Ar, b, sr, zeta=zeta, **kw)
        ok = np.array_equal(got["x_ls"], want["x_ls"]) and np.array_equal(got["y"], want["y"])
        ok &= got["grad_norm"] == want["grad_norm"] and np.array_equal(got["trace"]["r_sq"], want["trace"]["r_sq"])
        if not ok:
            bad += 1
            print(f"MISMATCH case {c}: m={m} n={n} delta={delta:.3f} {kw} zeta={zeta}", flush=True)
    print(f"{cases} cases ({skipped} draws skipped), {bad} mismatches, {time.time() - t0:.1f} s", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
