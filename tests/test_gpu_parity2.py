"""Parity cases added in round 2 (VERDICT r01 "close the parity gaps"):

* the device alias table's draw frequencies (ref tests/test_kaczmarz.cpp:153-169,
  weights {1, 2, 3}, 2e5 draws within 0.005) and on config-4-shaped weights;
* slice_shuffle draws are exact permutations of each worker's slice per pass
  (ref parallel.cpp:355-363);
* sweep_threads through the C ABI and the C++ API (ref tests/test_parallel.cpp:134-156);
* Trace::to_jsonl / to_csv byte-identical to the reference's serializers
  (ref trace.cpp:33-112) on the same trace content;
* BASELINE config 1 at full size against the reference's own rk_solve
  (oracle/_ref), bit for bit;
* config 3's fp64-x variant at full size.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _diag_system(w):
    """m = len(w) rows, row i = sqrt(w_i) e_i: row_norm^2 = w_i (the alias weights)."""
    m = len(w)
    A = capi.HostCsr(m, m, np.arange(m + 1, dtype=np.int64), np.arange(m, dtype=np.int64), np.sqrt(np.asarray(w)))
    return A, np.ones(m)


def test_device_alias_reproduces_target_distribution():
    # ref tests/test_kaczmarz.cpp:153-169: weights {1, 2, 3}, 200000 draws, |freq - w/6| < 0.005
    w = [1.0, 2.0, 3.0]
    A, b = _diag_system(w)
    with capi.System(A, b) as S:
        rows = S.sample_rows(capi.NORM_PROPORTIONAL, seed=123, warps=100, per_warp=2000)
    cnt = np.bincount(rows.ravel(), minlength=3)
    assert cnt.sum() == 200000
    for i in range(3):
        assert abs(cnt[i] / 200000 - w[i] / 6.0) < 0.005


def test_device_alias_config4_weights():
    # config 4's row weights (log-uniform norms over [0.1, 10]) on 4000 rows:
    # every row's count within 5 sigma of N w_i / sum w over 4e6 draws, and the
    # draws of two seeds differ
    A, b, _ = capi.generate_fixed_theta(4000, 2000, 25, seed=1004, scale_decades=1.0)
    w = capi.serial_row_sumsq(A.row_ptr, A.values)
    p = w / w.sum()
    with capi.System(A, b) as S:
        rows = S.sample_rows(capi.NORM_PROPORTIONAL, seed=7, warps=2000, per_warp=2000)
        rows2 = S.sample_rows(capi.NORM_PROPORTIONAL, seed=8, warps=2000, per_warp=2000)
    N = rows.size
    cnt = np.bincount(rows.ravel(), minlength=A.m)
    sd = np.sqrt(N * p * (1 - p))
    assert np.all(np.abs(cnt - N * p) <= 5 * sd + 1)
    assert not np.array_equal(rows, rows2)


def test_slice_shuffle_draws_are_slice_permutations():
    A, b, _ = capi.generate_fixed_theta(10007, 5000, 8, seed=3)
    W = 37
    with capi.System(A, b) as S:
        for epoch in (0, 5):
            lens = [(w + 1) * A.m // W - w * A.m // W for w in range(W)]
            per = 2 * max(lens)
            rows = S.sample_rows(capi.SLICE_SHUFFLE, seed=11, warps=W, per_warp=per, epoch=epoch)
            seen = []
            for w in range(W):
                lo, L = w * A.m // W, lens[w]
                first, second = rows[w, :L], rows[w, L:2 * L]
                assert np.array_equal(np.sort(first), np.arange(lo, lo + L))
                assert np.array_equal(np.sort(second), np.arange(lo, lo + L))  # the next pass: another permutation
                assert not np.array_equal(first, second)
                seen.append(first)
            assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(A.m))  # an epoch visits every row once


def test_with_replacement_draws_are_uniform():
    A, b, _ = capi.generate_fixed_theta(1000, 500, 8, seed=3)
    with capi.System(A, b) as S:
        rows = S.sample_rows(capi.WITH_REPLACEMENT, seed=1, warps=500, per_warp=2000)
    cnt = np.bincount(rows.ravel(), minlength=1000)
    N = rows.size
    p = 1e-3
    assert np.all(np.abs(cnt - N * p) <= 5 * np.sqrt(N * p * (1 - p)) + 1)


def test_sweep_threads_c_abi():
    # ref tests/test_parallel.cpp:134-156 through asyrk_sweep_threads
    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    Ar, b, _ = R.gen_instance(60, 30, 0.2, 97)
    e = Ar.export()
    A = capi.HostCsr(60, 30, e["row_ptr"], e["col_idx"], e["values"], e["row_norm"], e["normalized"])
    rep = capi.sweep_threads(A, b, [1, 2], gamma=1.0, epochs=30)
    assert len(rep) == 2
    assert rep[0]["threads"] == 1 and rep[0]["speedup"] == 1.0 and rep[0]["wall_seconds"] > 0.0
    assert rep[1]["threads"] == 2 and rep[1]["speedup"] > 0.0
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.sweep_threads(A, b, [2, 4], gamma=1.0, epochs=30)


def _build(tmp_path, name):
    exe = str(tmp_path / name)
    lib = os.path.join(ROOT, "paper_1401_4780_b200")
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-o", exe, "-L", lib, "-lasyrk_b200",
                    f"-Wl,-rpath,{lib}"], check=True, capture_output=True)
    return exe


def test_cpp_sweep_threads_and_trace_serialization(tmp_path):
    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    Ar, b, xs = R.gen_instance(60, 30, 0.2, 97)
    inst = tmp_path / "inst"
    inst.mkdir()
    R.write_instance(Ar, b, xs, dict(m=60, n=30, delta=0.2, seed=97, consistent=True, noise_level=0.0), str(inst))
    outd = tmp_path / "out"
    outd.mkdir()
    res = subprocess.run([_build(tmp_path, "sweep_trace_caller"), str(inst), str(outd)], check=True,
                         capture_output=True, text=True).stdout
    lines = [ln.split() for ln in res.splitlines() if ln.strip()]
    kv = {ln[0]: ln[1:] for ln in lines}
    sweeps = [ln[1:] for ln in lines if ln[0] == "sweep"]
    # ref tests/test_parallel.cpp:134-156
    assert kv["sweep_entries"] == ["2"]
    assert sweeps[0][0] == "1" and float(sweeps[0][4]) == 1.0 and float(sweeps[0][1]) > 0.0
    assert sweeps[1][0] == "2" and float(sweeps[1][4]) > 0.0
    assert kv["sweep_json_has_speedup"] == ["1"] and kv["sweep_csv_header"] == ["1"]
    assert kv["sweep_error"] == ["InvalidArgument"]
    assert kv["roundtrip"] == ["1"]
    # the reference's serializers (trace.cpp:33-112) on the same trace content
    for name in ("rk", "async"):
        ours_j = (outd / f"{name}.jsonl").read_text()
        ours_c = (outd / f"{name}.csv").read_text()
        ref_j, ref_c = R.trace_roundtrip(ours_j)
        assert ours_j == ref_j, name
        assert ours_c == ref_c, name
        assert '"dist_sq"' in ours_j  # x_star given: the optional field is serialized


def test_config1_full_size_bitwise_vs_reference():
    # BASELINE configs[0] at full size: 20000 x 10000, theta 20, uniform seeded
    # sequence, 20 epochs / 1e-8 — final_x and every record bit for bit against
    # the unmodified reference rk_solve (oracle/_ref)
    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
    target = 1e-16 * float(b @ b)
    Ah, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, normalize=True)
    want = R.rk_solve(Ah, b, np.zeros(A.n), 20, target, 42, "uniform", xs)
    with capi.System(A, b) as S:
        got = S.rk_solve(max_epochs=20, target=target, seed=42, sampling=capi.RK_UNIFORM, x_star=xs)
    assert np.array_equal(got["final_x"], want["final_x"])
    for k in ("epoch_index", "r_sq", "grad_sq", "dist_sq", "updates_applied"):
        assert np.array_equal(got[k], want[k]), k


def test_config3_fp64x_full_size():
    # BASELINE configs[2], fp64-x variant at full size: 2M x 1M, theta 50, fp32
    # values with fp64 x / atomics, async to 1e-5, error within 10x
    A, b, xs = capi.generate_fixed_theta(2000000, 1000000, 50, seed=1003, dist="uniform")
    bb = float(b @ b)
    with capi.System(A, b, precision=capi.F32X64) as S:
        t = S.solve(threads=S.max_resident_warps(), epochs=400, target=1e-10 * bb, sampling=capi.SLICE_SHUFFLE,
                    seed=1, x_star=xs, want_x=True, precision=capi.F32X64)
        rs, _ = S.residuals(t["final_x"])
    assert np.sqrt(t["r_sq"][-1] / bb) < 1e-5
    assert np.sqrt(t["dist_sq"][-1] / float(xs @ xs)) < 1e-4
    assert abs(rs - t["r_sq"][-1]) <= 1e-6 * rs  # the record is the returned iterate's residual


@pytest.mark.parametrize("sampling,name", [(0, "uniform"), (2, "shuffle"), (1, "norm")])
def test_deterministic_multi_rhs_columns_equal_reference_rk_solve(sampling, name):
    # SURVEY.md §8c, config 5's parity definition: column j of the deterministic
    # multi-RHS run == the reference rk_solve(A, B[:, j]) with the same sequence
    # (kaczmarz.cpp:128-227), bit for bit, for every sampling; the records are
    # the per-column exact values summed in column order
    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    k = 6
    raw = name == "norm"
    A, B, Xs = capi.generate_fixed_theta(3000, 1500, 12, seed=1005, k=k, scale_decades=1.0 if raw else 0.0)
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    Ah, _ = R.build(A.m, A.n, rows, A.col_idx, A.values, normalize=not raw)
    E = 6
    with capi.System(A, B[:, 0]) as S:
        got = S.rk_solve_multi(B, max_epochs=E, target=0.0, seed=17, sampling=sampling, X_star=Xs)
    assert list(got["epoch_index"]) == list(range(E + 1))
    r_sum = np.zeros(E + 1)
    g_sum = np.zeros(E + 1)
    d_sum = np.zeros(E + 1)
    for j in range(k):
        want = R.rk_solve(Ah, np.ascontiguousarray(B[:, j]), np.zeros(A.n), E, 0.0, 17, name,
                          np.ascontiguousarray(Xs[:, j]))
        assert np.array_equal(got["X"][:, j], want["final_x"]), j
        r_sum += want["r_sq"]  # column order, as the device adds them
        g_sum += want["grad_sq"]
        d_sum += want["dist_sq"]
    assert np.array_equal(got["r_sq"], r_sum)
    assert np.array_equal(got["grad_sq"], g_sum)
    assert np.array_equal(got["dist_sq"], d_sum)
    assert np.array_equal(got["updates_applied"], A.m * np.arange(E + 1))


def test_deterministic_multi_rhs_global_stop_and_x0():
    # a global target stops all columns together at the first epoch whose summed
    # r_sq meets it; a nonzero X0 per column is each column's own start
    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    k = 4
    A, B, Xs = capi.generate_fixed_theta(2000, 1000, 10, seed=9, k=k)
    X0 = np.random.default_rng(1).standard_normal((A.n, k))
    Ah, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, normalize=True)
    with capi.System(A, B[:, 0]) as S:
        free = S.rk_solve_multi(B, X0=X0, max_epochs=30, target=0.0, seed=3)
        tgt = float(free["r_sq"][12]) * 1.0000001
        got = S.rk_solve_multi(B, X0=X0, max_epochs=30, target=tgt, seed=3)
    assert int(got["epoch_index"][-1]) == 12
    for j in range(k):
        want = R.rk_solve(Ah, np.ascontiguousarray(B[:, j]), np.ascontiguousarray(X0[:, j]), 12, 0.0, 3, "uniform")
        assert np.array_equal(got["X"][:, j], want["final_x"]), j


def test_config1_reassociated_mode_within_1e12():
    # north_star: "a deterministic single-worker mode that consumes the
    # reference's seeded row-index sequence must reproduce the reference's
    # iterates within 1e-12 relative (fp64)": det_reassociate = 1 (warp-tree dot,
    # reciprocal coefficient, fused update) on config 1 at full size against
    # the unmodified reference rk_solve; deterministic run to run; the bitwise
    # default is unchanged
    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
    Ah, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, normalize=True)
    want = R.rk_solve(Ah, b, np.zeros(A.n), 20, 0.0, 42, "uniform")
    with capi.System(A, b) as S:
        fast = S.rk_solve(max_epochs=20, seed=42, sampling=capi.RK_UNIFORM, reassociate=True)
        fast2 = S.rk_solve(max_epochs=20, seed=42, sampling=capi.RK_UNIFORM, reassociate=True)
        exact = S.rk_solve(max_epochs=20, seed=42, sampling=capi.RK_UNIFORM)
    rel = np.linalg.norm(fast["final_x"] - want["final_x"]) / np.linalg.norm(want["final_x"])
    assert rel <= 1e-12, rel
    assert np.all(np.abs(fast["r_sq"] - want["r_sq"]) <= 1e-12 * want["r_sq"])
    assert np.array_equal(fast["final_x"], fast2["final_x"])  # reproducible
    assert np.array_equal(exact["final_x"], want["final_x"])  # the default stays bitwise


def test_sigma_sorted_columns_bitwise():
    # the monitor's column copy is sigma-sorted (positions by decreasing column
    # length, kernels.h CscDev): every column still sums its entries in
    # ascending row order, so A^T r and the residual records stay bit-identical
    # to the serial reference (csr.cpp:80-92, 140-160) on skewed column
    # lengths, empty columns and n not a multiple of 32
    rng = np.random.default_rng(21)
    m, n = 3000, 1001
    pop = rng.pareto(1.2, size=n) + 0.05
    pop[rng.choice(n, size=60, replace=False)] = 0.0  # empty columns
    pop /= pop.sum()
    lens = rng.integers(1, 40, size=m)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(n, size=k, replace=False, p=pop)) for k in lens]).astype(np.int64)
    v = rng.standard_normal(rp[-1])
    v /= np.repeat(np.sqrt(np.add.reduceat(v * v, rp[:-1])), lens)  # unit rows (rk_solve's uniform sampling)
    A = capi.HostCsr(m, n, rp, ci, v)
    b = rng.standard_normal(m)
    x = rng.standard_normal(n)
    r = rng.standard_normal(m)
    Ao = oracle.C.from_arrays(m, n, rp, ci, v)
    with capi.System(A, b) as S:
        assert np.array_equal(S.multiply_transpose(r), oracle.C.multiply_transpose(Ao, r))
        assert np.array_equal(S.multiply(x), oracle.C.multiply(Ao, x))
        assert S.residuals(x) == oracle.C.residuals(Ao, x, b)
        # the deterministic path's records (exact monitor: serial g^2 in column order)
        t = S.rk_solve(max_epochs=3, seed=5)
    ref = oracle.C.rk_solve(Ao, b, np.zeros(n), 3, seed=5)
    for k in ("r_sq", "grad_sq", "final_x"):
        assert np.array_equal(t[k], ref[k]), k


@pytest.mark.parametrize("epochs", [1, 50])
def test_async_solve_x0_meets_target(epochs):
    # record 0 (of x0, taken beside the first worker launch, read with record 1 —
    # system.cu run_scheduled): when x0 already meets the target the solve
    # returns x0 with one record at epoch 0 and no updates, whatever ran after it
    # on the device; a one-chunk solve takes the same path after its loop
    A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=31)
    bb = float(b @ b)
    with capi.System(A, b) as S:
        W = S.max_resident_warps()
        t = S.solve(x0=xs, threads=W, epochs=epochs, target=1e-6 * bb, seed=1)
        assert list(t["epoch_index"]) == [0]
        assert int(t["updates_applied"][-1]) == 0
        assert np.array_equal(t["final_x"], xs)
        # from zero, a one-epoch budget records boundaries 0 and 1 and applies m updates
        t = S.solve(threads=W, epochs=1, target=1e-6 * bb, seed=1)
        assert list(t["epoch_index"]) == [0, 1]
        assert int(t["updates_applied"][-1]) == A.m
        assert t["r_sq"][1] < t["r_sq"][0] == pytest.approx(bb, rel=1e-12)


def test_scheduled_solve_fuses_unrecorded_epochs():
    # the epochs between two scheduled evaluations run as one worker launch
    # (system.cu run_scheduled): fewer launches than epochs, the records still
    # sit at exact boundaries (updates = m x epoch at every record), every epoch
    # of work is credited, and the worker time is a part of the solve time
    A, b, xs = capi.generate_fixed_theta(40000, 20000, 30, seed=41)
    bb = float(b @ b)
    with capi.System(A, b) as S:
        W = S.max_resident_warps()
        t = S.solve(threads=W, epochs=500, target=1e-12 * bb, sampling=capi.SLICE_SHUFFLE, seed=2, x_star=xs)
        st = S.stats()
    ep = [int(e) for e in t["epoch_index"]]
    assert ep[0] == 0 and ep == sorted(ep) and t["r_sq"][-1] <= 1e-12 * bb
    assert all(int(u) == A.m * e for u, e in zip(t["updates_applied"], ep))
    assert st["projections"] == A.m * ep[-1]
    assert st["worker_launches"] < ep[-1]
    assert 0.0 < st["worker_ms"] <= st["solve_ms"]
    Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
    rs, _ = oracle.C.residuals(Ao, t["final_x"], b)
    assert abs(rs - t["r_sq"][-1]) <= 1e-9 * rs
