"""Randomized stress of the async path: random systems, warp counts,
samplings, precisions, snapshot intervals and record modes. Checks that each
solve returns (no hang, no crash), that its last record's r_sq matches an
independent evaluation of the returned iterate (the record belongs to that
iterate: the stopping-snapshot restore), that records are ordered, and that
instrumented runs pass the increment audit.
Usage: python scripts/stress_async.py [cases] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    t0 = time.time()
    bad = nonfinite = 0
    for c in range(cases):
        m = int(rng.integers(200, 60000))
        n = int(rng.integers(10, max(11, m // 2)))
        th = int(rng.integers(2, min(n, 70)))
        A, b, xs = capi.generate_fixed_theta(m, n, th, seed=int(rng.integers(1, 10**6)))
        prec = int(rng.choice([capi.F64, capi.F64, capi.F32, capi.F32X64]))
        with capi.System(A, b, precision=prec) as S:
            W = S.max_resident_warps()
            threads = int(rng.choice([2, 32, 256, min(W, max(2, m // 8)), W]))
            samp = int(rng.choice([capi.WITH_REPLACEMENT, capi.SLICE_SHUFFLE]))
            if samp == capi.SLICE_SHUFFLE:
                threads = min(threads, m)
            gamma = 1.0 if threads <= m // 16 else 0.5
            interval = int(rng.choice([1, 1, 2, 3]))
            instr = rng.random() < 0.2
            every = rng.random() < 0.3
            bb = float(b @ b)
            tol = 1e-10 if prec == capi.F64 else 1e-8
            try:
                t = S.solve(threads=threads, gamma=gamma, epochs=int(rng.integers(1, 400)), target=tol * bb,
                            sampling=samp, seed=int(rng.integers(0, 2**31)), snapshot_interval=interval,
                            precision=prec, instrument=instr, record_every_boundary=every, x_star=xs)
            except capi.AsyrkError as e:
                if "NonFinite" in str(e):
                    nonfinite += 1
                    continue
                print(f"ERROR case {c}: {e}", flush=True)
                bad += 1
                continue
        ep = t["epoch_index"]
        ok = bool(np.all(np.diff(ep) > 0))
        # the monitor evaluates the system's stored values: fp32 for the fp32 layouts
        vals = A.values if prec == capi.F64 else A.values.astype(np.float32).astype(np.float64)
        Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, vals)
        rs, _ = oracle.C.residuals(Ao, t["final_x"], b)
        diverged = not (t["r_sq"][-1] <= bb)
        ok &= abs(rs - t["r_sq"][-1]) <= 1e-9 * rs + 1e-300 or diverged
        if instr and not diverged:
            ok &= bool(t["instrument"]["consistent"])
        if not ok:
            bad += 1
            print(f"MISMATCH case {c}: m={m} n={n} th={th} prec={prec} threads={threads} samp={samp} "
                  f"interval={interval} every={every} instr={instr} rec={t['r_sq'][-1]:.6g} eval={rs:.6g} "
                  f"epochs={list(ep[-3:])}", flush=True)
    print(f"{cases} cases, {bad} failures, {nonfinite} NonFinite (staleness), {time.time() - t0:.1f} s", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
