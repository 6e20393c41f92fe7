"""Randomized bit-identity stress of the deterministic path (rk_solve and
solve_single through the device) against the C restatement: random shapes,
ragged rows (incl. > 128 entries), raw or unit rows, all samplings and
variants, snapshot intervals and stop targets (the speculative-chunk restore).
Usage: python scripts/stress_det.py [cases] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402

KEYS = ["epoch_index", "r_sq", "grad_sq", "dist_sq", "updates_applied", "final_x"]


def system(rng):
    m = int(rng.integers(5, 3000))
    n = int(rng.integers(2, max(3, min(m, 2500))))
    hi = int(min(n, rng.choice([4, 16, 40, 100, 200])))
    lo = int(rng.integers(1, hi + 1))
    lens = rng.integers(lo, hi + 1, size=m)
    rp = np.concatenate([[0], np.cumsum(lens)])
    ci = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens])
    v = rng.standard_normal(rp[-1])
    unit = rng.random() < 0.7
    if unit:
        v /= np.repeat(np.sqrt(capi.serial_row_sumsq(rp, v)), lens)
    else:
        v *= np.repeat(10.0 ** rng.uniform(-1, 1, size=m), lens)
    A = capi.HostCsr(m, n, rp, ci, v)
    xs = rng.standard_normal(n)
    b = np.add.reduceat(v * xs[ci], rp[:-1]) if rng.random() < 0.8 else rng.standard_normal(m)
    return A, b, xs


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    t0 = time.time()
    bad = 0
    for c in range(cases):
        A, b, xs = system(rng)
        Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
        bb = float(b @ b)
        with capi.System(A, b) as S:
            epochs = int(rng.integers(1, 25))
            target = float(bb * 10.0 ** rng.uniform(-12, -1)) if rng.random() < 0.5 else 0.0
            seed = int(rng.integers(0, 2**31))
            use_xs = rng.random() < 0.5
            if A.normalized and rng.random() < 0.5:
                variant = "full_row" if rng.random() < 0.7 else "single"
                samp = "slice_shuffle" if rng.random() < 0.5 else "with_replacement"
                interval = int(rng.integers(1, 4))
                gamma = 1.0 if variant == "full_row" else 0.05
                try:
                    got = S.solve(threads=1, gamma=gamma, epochs=epochs, target=target, seed=seed,
                                  variant=capi.FULL_ROW if variant == "full_row" else capi.SINGLE_COMPONENT,
                                  sampling=capi.SLICE_SHUFFLE if samp == "slice_shuffle" else capi.WITH_REPLACEMENT,
                                  snapshot_interval=interval, x_star=xs if use_xs else None)
                except capi.AsyrkError as e:
                    got = str(e)
                try:
                    want = oracle.C.solve_parallel(Ao, b, np.zeros(A.n), 1, gamma, epochs, target, variant, samp,
                                                   seed, interval, xs if use_xs else None)
                except oracle.OracleError as e:
                    want = str(e)
                tag = f"solve_single {variant} {samp} interval {interval}"
            else:
                samp = "norm" if not A.normalized or rng.random() < 0.3 else rng.choice(["uniform", "shuffle"])
                code = {"uniform": capi.RK_UNIFORM, "shuffle": capi.RK_SHUFFLE, "norm": capi.RK_NORM_PROPORTIONAL}[samp]
                try:
                    got = S.rk_solve(max_epochs=epochs, target=target, seed=seed, sampling=code,
                                     x_star=xs if use_xs else None)
                except capi.AsyrkError as e:
                    got = str(e)
                try:
                    want = oracle.C.rk_solve(Ao, b, np.zeros(A.n), epochs, target, seed, samp, xs if use_xs else None)
                except oracle.OracleError as e:
                    want = str(e)
                tag = f"rk_solve {samp}"
        if isinstance(got, str) or isinstance(want, str):
            ok = isinstance(got, str) and isinstance(want, str) and got.split(":")[0] == want.split(":")[-2].strip() \
                if isinstance(want, str) and ":" in want else isinstance(got, str) == isinstance(want, str)
        else:
            ok = all(np.array_equal(got[k], want[k]) for k in KEYS if k in want and (k != "dist_sq" or use_xs))
        if not ok:
            bad += 1
            print(f"MISMATCH case {c}: {tag} m={A.m} n={A.n} maxlen={np.diff(A.row_ptr).max()} epochs={epochs} "
                  f"target={target:.3g} -> {got if isinstance(got, str) else 'arrays'} vs "
                  f"{want if isinstance(want, str) else 'arrays'}", flush=True)
    print(f"{cases} cases, {bad} mismatches, {time.time() - t0:.1f} s", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
