"""Row-length and size coverage of the device kernels that the reference-test
instances (all rows <= 32 nonzeros, n <= 1500) never reach:

  * worker_kernel<E=2> / <E=4> (rows of 33..64 / 65..128 entries) and
    worker_kernel_long (rows > 128 entries, looped), worker.cu:105-302;
  * det_dataflow_kernel<E=2> / <E=4>, and det_serial_kernel, the deterministic
    twin used when a row exceeds 128 entries or x does not fit in shared
    memory (det.cu:247-318);
  * ragged rows mixing 1-entry rows with the longest ones.

Parity bar as in test_gpu_parity.py: rk_solve / solve_single (threads == 1)
are BIT-IDENTICAL to the C restatement (oracle.C, itself pinned to the
reference's golden vectors in test_oracle.py); the async worker reaches the
relative-residual tolerance with ||x - x*|| / ||x*|| within 10x of it.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")
KEYS = ["epoch_index", "r_sq", "grad_sq", "dist_sq", "updates_applied", "final_x"]


def ragged(m, n, lo, hi, seed, normalize=True):
    """Consistent system b = A x* with row lengths uniform in [lo, hi]."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, size=m)
    lens[0], lens[-1] = lo, hi  # both extremes present
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int64)
    v = rng.standard_normal(rp[-1])
    if normalize:
        nrm = np.sqrt(np.add.reduceat(v * v, rp[:-1]))
        v /= np.repeat(nrm, lens)
    else:
        v *= np.repeat(10.0 ** rng.uniform(-1, 1, size=m), lens)
    A = capi.HostCsr(m, n, rp, ci, v)
    xs = rng.standard_normal(n)
    b = np.add.reduceat(v * xs[ci], rp[:-1])
    return A, b, xs


# name: (m, n, min row length, max row length, async workers; 0 = every resident warp)
# — the comment says which kernels each case selects
CASES = {
    "e2_33to64": (3000, 800, 33, 64, 32),        # worker E=2, det dataflow E=2
    "e4_1to128": (3000, 800, 1, 128, 32),        # worker E=4, det dataflow E=4, 1-entry rows
    "long_1to400": (2400, 600, 1, 400, 32),      # worker_kernel_long, det_serial_kernel
    "wide_n_30000": (150000, 30000, 8, 16, 0),   # x exceeds shared memory -> det_serial_kernel
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request):
    m, n, lo, hi, threads = CASES[request.param]
    A, b, xs = ragged(m, n, lo, hi, seed=100 + list(CASES).index(request.param))
    S = capi.System(A, b)
    Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
    yield request.param, A, b, xs, S, Ao, threads or S.max_resident_warps()
    S.close()


@pytest.mark.parametrize("sampling,code", [("uniform", capi.RK_UNIFORM), ("shuffle", capi.RK_SHUFFLE),
                                           ("norm", capi.RK_NORM_PROPORTIONAL)])
def test_rk_solve_bit_identical(case, sampling, code):
    nm, A, b, xs, S, Ao, threads = case
    epochs = 3
    got = S.rk_solve(max_epochs=epochs, seed=77, sampling=code, x_star=xs)
    want = oracle.C.rk_solve(Ao, b, np.zeros(A.n), epochs, 0.0, 77, sampling, xs)
    for k in KEYS:
        assert np.array_equal(got[k], want[k]), (nm, k)


@pytest.mark.parametrize("variant", ["full_row", "single"])
def test_solve_single_bit_identical(case, variant):
    nm, A, b, xs, S, Ao, threads = case
    gamma = 1.0 if variant == "full_row" else 0.05
    v = capi.FULL_ROW if variant == "full_row" else capi.SINGLE_COMPONENT
    got = S.solve(threads=1, gamma=gamma, epochs=3, variant=v, sampling=capi.SLICE_SHUFFLE, seed=9,
                  snapshot_interval=2, x_star=xs, instrument=True)
    want = oracle.C.solve_parallel(Ao, b, np.zeros(A.n), 1, gamma, 3, 0.0, variant, "slice_shuffle", 9, 2, xs,
                                   instrument=True)
    for k in KEYS:
        assert np.array_equal(got[k], want[k]), (nm, k)
    assert got["instrument"]["row_updates"] == want["instrument"]["row_updates"] == 3 * A.m


@pytest.mark.parametrize("sampling", [capi.WITH_REPLACEMENT, capi.SLICE_SHUFFLE])
def test_async_reaches_tolerance(case, sampling):
    nm, A, b, xs, S, Ao, threads = case
    bb = float(b @ b)
    t = S.solve(threads=threads, epochs=2000, target=1e-16 * bb, sampling=sampling, seed=5,
                x_star=xs)
    rel = float(np.sqrt(t["r_sq"][-1] / bb))
    err = float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))
    assert rel <= 1e-8 and err <= 1e-7, (nm, rel, err, len(t["r_sq"]))
    rs, _ = oracle.C.residuals(Ao, t["final_x"], b)
    assert abs(rs - t["r_sq"][-1]) <= 1e-9 * max(rs, 1e-300) + 1e-30


def test_instrumented_async_long_rows(case):
    nm, A, b, xs, S, Ao, threads = case
    t = S.solve(threads=min(threads, 256), epochs=4, seed=3, instrument=True)
    rep = t["instrument"]
    assert rep["consistent"] and rep["max_abs_error"] <= rep["tolerance"], (nm, rep)
    assert rep["row_updates"] == 4 * A.m


def test_raw_rows_norm_proportional_async():
    A, b, xs = ragged(4000, 700, 1, 300, seed=12, normalize=False)
    assert not A.normalized
    with capi.System(A, b) as S:
        bb = float(b @ b)
        t = S.solve(threads=64, epochs=3000, target=1e-16 * bb,
                    sampling=capi.NORM_PROPORTIONAL, seed=8, x_star=xs)
        rel = float(np.sqrt(t["r_sq"][-1] / bb))
        err = float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))
        assert rel <= 1e-8 and err <= 1e-7, (rel, err)
