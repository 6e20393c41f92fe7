"""GPU parity suite: the sm_100a path through the C ABI (and the pybind
module with the reference's signatures) against the reference's own outputs
(tests/golden/golden.npz from oracle/_ref) and the C restatement (oracle/).

Bar (BASELINE.json north_star): the deterministic worker reproduces the
reference's iterates within 1e-12 relative — we assert BIT-IDENTITY of
final_x and of every record's r_sq / grad_sq / dist_sq, which is stronger;
the async workers reach the same relative-residual tolerance with
||x - x*|| / ||x*|| within 10x that tolerance.
"""
import numpy as np
import pytest

import oracle
from conftest import triplets

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")
KEYS = ["epoch_index", "r_sq", "grad_sq", "dist_sq", "updates_applied", "final_x"]


def host_csr(inst):
    return capi.HostCsr(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"], inst["row_norm"])


@pytest.fixture(scope="module")
def systems(instances):
    out = {nm: capi.System(host_csr(inst), inst["b"]) for nm, inst in instances.items()}
    yield out
    for s in out.values():
        s.close()


# ---------------------------------------------------------------- deterministic worker: bit-identical
@pytest.mark.parametrize("sampling,code", [("uniform", capi.RK_UNIFORM), ("shuffle", capi.RK_SHUFFLE),
                                           ("norm", capi.RK_NORM_PROPORTIONAL)])
def test_rk_solve_bit_identical_to_reference(golden, instances, systems, sampling, code):
    for nm, inst in instances.items():
        epochs = 40 if inst["m"] <= 200 else 10
        t = systems[nm].rk_solve(max_epochs=epochs, seed=31337, sampling=code, x_star=inst["x_star"])
        q = f"rk/{nm}/{sampling}/"
        for k in KEYS:
            assert np.array_equal(t[k], golden[q + k]), (nm, k)


@pytest.mark.parametrize("variant", ["full_row", "single"])
@pytest.mark.parametrize("sampling", ["slice_shuffle", "with_replacement"])
def test_solve_parallel_single_worker_bit_identical(golden, instances, systems, variant, sampling):
    for nm, inst in instances.items():
        t = systems[nm].solve(
            threads=1, gamma=1.0 if variant == "full_row" else 0.05, epochs=13, target=0.0,
            variant=capi.FULL_ROW if variant == "full_row" else capi.SINGLE_COMPONENT,
            sampling=capi.SLICE_SHUFFLE if sampling == "slice_shuffle" else capi.WITH_REPLACEMENT,
            seed=21, snapshot_interval=3, x_star=inst["x_star"], instrument=True)
        q = f"par/{nm}/{variant}_{sampling}/"
        for k in KEYS:
            assert np.array_equal(t[k], golden[q + k]), (nm, k)
        ins = t["instrument"]
        ref = golden[q + "instrument"]
        assert ins["row_updates"] == ref[0] and ins["increments"] == ref[1]
        assert ins["max_abs_error"] == ref[2] and ins["tolerance"] == ref[3] and ins["consistent"] == bool(ref[4])


def test_pybind_reference_signatures_bit_identical(golden, instances):
    import paper_1401_4780_b200 as pkg

    inst = instances["accept5_200x80"]
    rows, cols, vals = triplets(inst)
    t = pkg.solve_rk(inst["m"], inst["n"], rows.tolist(), cols.tolist(), vals.tolist(), inst["b"].tolist(),
                     epochs=40, seed=31337, sampling="shuffle")
    assert np.array_equal(np.array(t["final_x"]), golden["rk/accept5_200x80/shuffle/final_x"])
    assert np.array_equal(np.array(t["r_sq"]), golden["rk/accept5_200x80/shuffle/r_sq"])
    # acceptance C5 (acceptance.cpp:230-270): one slice_shuffle worker == serial shuffled solver
    p = pkg.solve_parallel(inst["m"], inst["n"], rows.tolist(), cols.tolist(), vals.tolist(), inst["b"].tolist(),
                           threads=1, gamma=1.0, epochs=40, seed=31337)
    assert np.array_equal(np.array(p["final_x"]), np.array(t["final_x"]))
    assert np.array_equal(np.array(p["r_sq"]), np.array(t["r_sq"]))
    assert p["instrument"]["consistent"] is True
    assert p["instrument"]["row_updates"] == 40 * inst["m"]


def test_config1_full_size_bit_identical():
    # BASELINE config 1: 20000 x 10000, theta 20, uniform seeded sequence, 20 epochs
    A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
    S = capi.System(A, b)
    got = S.rk_solve(max_epochs=20, seed=42, sampling=capi.RK_UNIFORM, x_star=xs)
    Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
    want = oracle.C.rk_solve(Ao, b, np.zeros(A.n), 20, 0.0, 42, "uniform", xs)
    for k in KEYS:
        assert np.array_equal(got[k], want[k]), k
    # 1e-12 relative bar of north_star, stated explicitly
    assert np.max(np.abs(got["final_x"] - want["final_x"])) <= 1e-12 * np.max(np.abs(want["final_x"]))
    # slice_shuffle single worker on the same instance (solve_single, parallel.cpp:111-210)
    got2 = S.solve(threads=1, epochs=5, sampling=capi.SLICE_SHUFFLE, seed=7, snapshot_interval=2)
    want2 = oracle.C.solve_parallel(Ao, b, np.zeros(A.n), 1, 1.0, 5, 0.0, "full_row", "slice_shuffle", 7, 2)
    assert np.array_equal(got2["final_x"], want2["final_x"])
    assert np.array_equal(got2["epoch_index"], [0, 2, 4, 5])
    S.close()


def test_deterministic_stops_on_target_like_reference(instances, systems):
    inst = instances["repl_40x20"]
    Ao = oracle.C.from_arrays(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"])
    target = 1e-6 * float(inst["b"] @ inst["b"])
    got = systems["repl_40x20"].rk_solve(max_epochs=500, seed=3, target=target)
    want = oracle.C.rk_solve(Ao, inst["b"], np.zeros(inst["n"]), 500, target, 3, "uniform")
    assert np.array_equal(got["epoch_index"], want["epoch_index"])
    assert np.array_equal(got["final_x"], want["final_x"])


# ---------------------------------------------------------------- device building blocks
def test_residuals_and_spmv_bit_identical(golden, instances, systems):
    for nm, inst in instances.items():
        S = systems[nm]
        x = golden[f"res/{nm}/x"]
        assert np.array_equal(np.array(S.residuals(x)), golden[f"res/{nm}/vals"]), nm
        assert np.array_equal(S.multiply(x), golden[f"res/{nm}/Ax"]), nm
        assert np.array_equal(S.multiply_transpose(golden[f"res/{nm}/r_in"]), golden[f"res/{nm}/ATr"]), nm


def test_power_iteration(golden, instances, systems):
    for nm, inst in instances.items():
        lam, it = systems[nm].power_iteration(1e-10)
        ref = golden[f"pow/{nm}"][0]
        assert abs(lam - ref) <= 1e-8 * ref, nm  # test_stats.cpp:47-62 uses 1e-6


# ---------------------------------------------------------------- async warp-workers
def _rel(t, b):
    return float(np.sqrt(t["r_sq"][-1] / float(b @ b)))


@pytest.mark.parametrize("threads", [2, 4])
@pytest.mark.parametrize("variant", ["full_row", "single"])
def test_instrumented_async_run_is_consistent(instances, systems, threads, variant):
    # test_parallel.cpp:62-85 (and acceptance C9): x_final == x0 + sum of applied increments
    S = systems["instr_48x16"]
    t = S.solve(threads=threads, gamma=0.9 if variant == "full_row" else 0.05, epochs=40, seed=5,
                variant=capi.FULL_ROW if variant == "full_row" else capi.SINGLE_COMPONENT, instrument=True)
    rep = t["instrument"]
    assert rep["consistent"] and rep["max_abs_error"] <= rep["tolerance"]
    assert rep["row_updates"] == 40 * 48  # exact epochs (reference: within [40*48, 40*48+T))
    assert rep["increments"] >= rep["row_updates"]
    assert t["updates_applied"][-1] == rep["row_updates"]


def test_acceptance_c9_eight_workers(instances, systems):
    S = systems["accept9_2000x1500"]
    t = S.solve(threads=8, gamma=0.9, epochs=50, seed=11, instrument=True)
    assert t["instrument"]["consistent"]


@pytest.mark.parametrize("sampling", [capi.WITH_REPLACEMENT, capi.SLICE_SHUFFLE])
def test_async_converges(instances, systems, sampling):
    # test_parallel.cpp:87-98: with-replacement T=2 reaches r_sq <= 1e-10
    inst = instances["repl_40x20"]
    t = systems["repl_40x20"].solve(threads=2, sampling=sampling, gamma=1.0, epochs=200, target=1e-12)
    assert t["r_sq"][-1] <= 1e-10


def test_divergent_step_is_reported(systems):
    # test_parallel.cpp:100-109
    with pytest.raises(capi.AsyrkError, match="NonFinite"):
        systems["diverge_20x10"].solve(threads=1, gamma=1000.0, epochs=200)
    with pytest.raises(capi.AsyrkError, match="NonFinite"):
        systems["diverge_20x10"].solve(threads=4, gamma=1000.0, epochs=200)


def test_start_at_solution_returns_immediately(instances, systems):
    # test_parallel.cpp:111-119
    inst = instances["at_solution_20x10"]
    t = systems["at_solution_20x10"].solve(x0=inst["x_star"], threads=4, epochs=50)
    assert len(t["r_sq"]) == 1 and t["r_sq"][0] <= 1e-30


def test_config_validation(systems):
    # test_parallel.cpp:121-132 + validate_config parallel.cpp:56-80
    S = systems["snap_24x12"]
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        S.solve(threads=0)
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        S.solve(threads=1, snapshot_interval=0)
    with pytest.raises(capi.AsyrkError, match="InvalidGamma"):
        S.solve(threads=2, gamma=0.0)
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        S.solve(threads=100, sampling=capi.SLICE_SHUFFLE)  # m = 24 < threads


def test_snapshot_interval_keeps_endpoints(systems):
    # test_parallel.cpp:45-60
    t = systems["snap_24x12"].solve(threads=1, epochs=10, snapshot_interval=4)
    assert list(t["epoch_index"]) == [0, 4, 8, 10] and t["updates_applied"][-1] == 240
    t = systems["snap_24x12"].solve(threads=3, epochs=10, snapshot_interval=4)
    assert list(t["epoch_index"]) == [0, 4, 8, 10] and t["updates_applied"][-1] == 240


def test_unnormalized_rows_need_norm_proportional():
    # test_kaczmarz.cpp:124-137 on the device: uniform refuses raw rows, norm-proportional solves them
    A = capi.HostCsr(2, 2, [0, 1, 2], [0, 1], [2.0, 1.0])
    S = capi.System(A, np.array([2.0, 1.0]))
    with pytest.raises(capi.AsyrkError, match="NotNormalized"):
        S.rk_solve(max_epochs=5)
    t = S.rk_solve(max_epochs=60, sampling=capi.RK_NORM_PROPORTIONAL)
    assert t["r_sq"][-1] <= 1e-20
    with pytest.raises(capi.AsyrkError, match="NotNormalized"):
        S.solve(threads=2, epochs=5, sampling=capi.WITH_REPLACEMENT)
    t = S.solve(threads=2, epochs=60, sampling=capi.NORM_PROPORTIONAL)
    assert t["r_sq"][-1] <= 1e-20
    S.close()


def test_config2_async_reaches_tolerance():
    # BASELINE config 2 at full size: rel residual 1e-6, ||x-x*||/||x*|| within 10x
    A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
    S = capi.System(A, b)
    bb = float(b @ b)
    for sampling in (capi.WITH_REPLACEMENT, capi.SLICE_SHUFFLE):
        t = S.solve(threads=S.max_resident_warps(), epochs=300, target=1e-12 * bb, sampling=sampling, seed=3,
                    x_star=xs)
        rel = _rel(t, b)
        err = float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))
        assert rel <= 1e-6 and err <= 1e-5, (sampling, rel, err)
        # the device record agrees with an independent CPU evaluation of the final iterate
        Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
        rs, _ = oracle.C.residuals(Ao, t["final_x"], b)
        assert abs(rs - t["r_sq"][-1]) <= 1e-9 * rs
    S.close()


def test_config3_full_size_fp32():
    # BASELINE config 3 at full size: 2M x 1M, theta 50, U(-1,1) values, fp32 x
    # and atomics, all resident warps -> rel residual 1e-5, error within 10x
    A, b, xs = capi.generate_fixed_theta(2000000, 1000000, 50, seed=1003, dist="uniform")
    bb = float(b @ b)
    with capi.System(A, b, precision=capi.F32) as S:
        t = S.solve(threads=S.max_resident_warps(capi.F32), epochs=300, target=1e-10 * bb,
                    sampling=capi.SLICE_SHUFFLE, seed=1, precision=capi.F32, x_star=xs, want_x=False)
    rel = _rel(t, b)
    err = float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))
    assert rel <= 1e-5 and err <= 1e-4, (rel, err)


def test_config3_fp32_and_fp64x():
    # BASELINE config 3 shape at 1/10 scale: U(-1,1) values, fp32 x / fp32 atomics, and fp64-x variant
    A, b, xs = capi.generate_fixed_theta(200000, 100000, 50, seed=1003, dist="uniform")
    bb = float(b @ b)
    for prec in (capi.F32, capi.F32X64):
        S = capi.System(A, b, precision=prec)
        t = S.solve(threads=4096, epochs=300, target=1e-10 * bb, sampling=capi.WITH_REPLACEMENT, seed=1,
                    precision=prec, x_star=xs)
        rel = _rel(t, b)
        err = float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))
        assert rel <= 1e-5 and err <= 1e-4, (prec, rel, err)
        S.close()


@pytest.mark.parametrize("m,n", [(100000, 25000), (400000, 100000)])
def test_config4_alias_sampling_raw_rows(m, n):
    # BASELINE config 4 (full size, and at 1/4 scale): rows scaled log-uniform in
    # [0.1, 10], P(i) ~ ||a_i||^2
    A, b, xs = capi.generate_fixed_theta(m, n, 25, seed=1004, scale_decades=1.0)
    assert not A.normalized
    S = capi.System(A, b)
    bb = float(b @ b)
    t = S.solve(threads=2048, epochs=300, target=1e-12 * bb, sampling=capi.NORM_PROPORTIONAL, seed=2, x_star=xs)
    rel = _rel(t, b)
    err = float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))
    assert rel <= 1e-6 and err <= 1e-5, (rel, err)
    S.close()


def test_one_shot_host_entry_points(instances):
    inst = instances["accept5_200x80"]
    A = host_csr(inst)
    t = capi.rk_solve_host(A, inst["b"], max_epochs=40, seed=31337, sampling=capi.RK_SHUFFLE)
    Ao = oracle.C.from_arrays(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"])
    want = oracle.C.rk_solve(Ao, inst["b"], np.zeros(inst["n"]), 40, 0.0, 31337, "shuffle")
    assert np.array_equal(t["final_x"], want["final_x"])
    t = capi.solve_parallel_host(A, inst["b"], threads=16, epochs=300, target=1e-20, seed=4,
                                 sampling=capi.WITH_REPLACEMENT)
    assert t["r_sq"][-1] <= 1e-20


def test_record_modes_of_the_overlapped_monitor():
    # default: the monitor records the latest boundary it can (the reference's
    # coordinator, parallel.cpp:388-399) — records are a strictly increasing
    # subset of the boundaries plus the final one; record_every_boundary: all
    A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
    S = capi.System(A, b)
    bb = float(b @ b)
    kw = dict(threads=S.max_resident_warps(), epochs=400, target=1e-12 * bb, sampling=capi.WITH_REPLACEMENT,
              x_star=xs, want_x=False)
    t = S.solve(seed=3, **kw)
    ep = np.asarray(t["epoch_index"])
    assert ep[0] == 0 and np.all(np.diff(ep) > 0) and t["r_sq"][-1] <= 1e-12 * bb
    u = S.solve(seed=3, record_every_boundary=1, **kw)
    eu = np.asarray(u["epoch_index"])
    assert np.array_equal(eu, np.arange(len(eu))) and u["r_sq"][-1] <= 1e-12 * bb
    for r in (t, u):
        assert np.sqrt(r["dist_sq"][-1] / float(xs @ xs)) <= 1e-5
    S.close()


def test_cpp_drop_in_caller_runs(tmp_path):
    # the C++ drop-in API end to end (tests/cpp/drop_in_caller.cpp): rk_solve and
    # solve_single bit-identical to the C restatement, async converged with a
    # consistent audit, exact stats, projector distance, lsq, error codes
    import subprocess

    from test_host import _build_drop_in_caller
    out = subprocess.run([_build_drop_in_caller(tmp_path)], check=True, capture_output=True, text=True).stdout
    res = {ln.split()[0]: ln.split()[1:] for ln in out.splitlines() if ln.strip()}
    # rebuild the same system as the caller (triplet order, normalize_rows) for the oracle
    m, n = 60, 24
    xs = np.sin(0.7 * np.arange(n) + 0.3)
    trip = {}
    for i in range(m):
        for q in range(6):
            j = (i * 7 + q * 5 + (i * q) % 3) % n
            if (i, j) not in trip:
                trip[(i, j)] = np.cos(1.3 * i + 0.9 * q) + 0.1 * (q + 1)
    keys = sorted(trip)
    rows = np.array([k[0] for k in keys])
    cols = np.array([k[1] for k in keys])
    vals = np.array([trip[k] for k in keys])
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=m))])
    b0 = np.zeros(m)
    for i in range(m):  # CsrMatrix::row_dot order
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s += vals[k] * xs[cols[k]]
        b0[i] = s
    norms = np.sqrt(capi.serial_row_sumsq(rp, vals))
    vn = vals / np.repeat(norms, np.diff(rp))
    bn = b0 / norms
    Ao = oracle.C.from_arrays(m, n, rp, cols, vn)
    want = oracle.C.rk_solve(Ao, bn, np.zeros(n), 30, 0.0, 5, "uniform", xs)
    got = np.array([float(v) for v in res["rk_final_x"]])
    assert np.array_equal(got, want["final_x"])
    want1 = oracle.C.solve_parallel(Ao, bn, np.zeros(n), 1, 1.0, 12, 0.0, "full_row", "slice_shuffle", 9, 1)
    assert np.array_equal(np.array([float(v) for v in res["single_final_x"]]), want1["final_x"])
    assert float(res["async_r_sq"][0]) <= 1e-24 and res["async_r_sq"][2] == "1"
    assert float(res["stats"][4]) > 0.0  # lambda_min from the exact spectrum
    rec, d, pd = (float(v) for v in res["projector"])
    assert abs(rec - d) <= 1e-9 * max(d, 1e-30) and abs(pd - d) <= 1e-9 * max(d, 1e-30)
    assert float(res["lsq"][0]) <= 1e-6 and float(res["lsq"][1]) <= 1e-6
    assert res["error"] == ["InvalidArgument"]
