"""Dev probe: quick GPU checks of the hot path (not part of the test suite)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1401_4780_b200 import capi
import oracle

def cfg1():
    A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
    S = capi.System(A, b)
    t = time.time(); got = S.rk_solve(max_epochs=20, seed=42, sampling=capi.RK_UNIFORM, x_star=xs); t = time.time() - t
    st = S.stats()
    Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
    t2 = time.time(); want = oracle.C.rk_solve(Ao, b, np.zeros(A.n), 20, 0.0, 42, "uniform", xs); t2 = time.time() - t2
    print("cfg1 det: bitwise x", np.array_equal(got["final_x"], want["final_x"]), "r_sq", np.array_equal(got["r_sq"], want["r_sq"]),
          "g", np.array_equal(got["grad_sq"], want["grad_sq"]), "d", np.array_equal(got["dist_sq"], want["dist_sq"]),
          f"gpu {t*1e3:.1f} ms host-wall, solve {st['solve_ms']:.1f} ms, worker {st['worker_ms']:.1f} ms; cpu oracle {t2*1e3:.1f} ms")
    print("   maxdiff x", np.max(np.abs(got["final_x"]-want["final_x"])), "rel res", (got["r_sq"][-1]/(b@b))**.5)
    for th in [2048, 9472]:
        r = S.solve(threads=th, epochs=300, target=1e-16*(b@b), sampling=capi.WITH_REPLACEMENT, seed=3)
        st = S.stats()
        print(f"cfg1 async W={th}: epochs {r['epoch_index'][-1]} rel {(r['r_sq'][-1]/(b@b))**.5:.2e} solve {st['solve_ms']:.2f} ms worker {st['worker_ms']:.2f} ms proj/s {st['projections']/st['worker_ms']*1e3:.3e}")

def cfg2():
    A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
    S = capi.System(A, b)
    bb = float(b @ b)
    lam, it = S.power_iteration(1e-6)
    print(f"cfg2 lambda_max {lam:.5f} iters {it} tau_max {200000/(2*np.e*lam)-1:.0f}")
    print("resident warps", S.max_resident_warps())
    for samp in [capi.WITH_REPLACEMENT, capi.SLICE_SHUFFLE]:
        for th in [148, 1184, 2368, 4736, 9472]:
            r = S.solve(threads=th, epochs=200, target=1e-12*bb, sampling=samp, seed=5, x_star=xs)
            st = S.stats()
            rel = (r['r_sq'][-1]/bb)**.5
            err = (r['dist_sq'][-1]/(xs@xs))**.5
            print(f"cfg2 samp={samp} W={th} res={st['resident_warps']}: epochs {r['epoch_index'][-1]} rel {rel:.2e} xerr {err:.2e} "
                  f"solve {st['solve_ms']:.2f} ms worker {st['worker_ms']:.2f} ms ({st['worker_launches']} launches) "
                  f"proj/s(worker) {st['projections']/st['worker_ms']*1e3:.3e} proj/s(solve) {st['projections']/st['solve_ms']*1e3:.3e}")
    # e2e one-shot
    t = time.time(); r = capi.solve_parallel_host(A, b, threads=4736, epochs=200, target=1e-12*bb, sampling=capi.WITH_REPLACEMENT, seed=5); t = time.time()-t
    print(f"cfg2 e2e one-shot {t*1e3:.1f} ms epochs {r['epoch_index'][-1]}")

if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg1", "cfg2"]
    for w in which:
        globals()[w]()
