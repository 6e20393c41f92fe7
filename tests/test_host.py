"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/*.h declares, the pybind module mirrors the reference
signatures and error convention, the config generator's contract holds, and
the product fails loudly (no CPU fallback) when no device is present."""
import inspect
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADERS = [os.path.join(ROOT, "include", "asyrk_cuda.h"), os.path.join(ROOT, "include", "asyrk_datagen.h"),
           os.path.join(ROOT, "include", "asyrk_io.h"), os.path.join(ROOT, "include", "asyrk_dense.h")]


def declared_functions():
    names = set()
    for h in HEADERS:
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for mt in re.finditer(r"\b(asyrk_[a-z0-9_]+)\s*\(", text):
            names.add(mt.group(1))
    return names


def test_c_abi_exports_every_declared_symbol():
    from paper_1401_4780_b200 import capi

    L = capi.lib()
    declared = declared_functions()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/ but not exported"
    assert set(capi.EXPORTED) <= declared
    assert L.asyrk_abi_version() == 2


def test_exported_symbols_via_nm():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1401_4780_b200",
                                                                     "libasyrk_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert declared_functions() <= exported


def test_kernels_are_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1401_4780_b200",
                                                                  "libasyrk_b200.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pybind_signatures_match_reference():
    import paper_1401_4780_b200 as pkg

    doc = pkg.solve_parallel.__doc__
    for arg in ["m", "n", "rows", "cols", "vals", "b", "threads", "gamma", "epochs", "target", "seed", "variant"]:
        assert f"{arg}:" in doc
    for arg, default in [("threads", "1"), ("gamma", "1.0"), ("epochs", "100"), ("target", "0.0"), ("seed", "0"),
                         ("variant", "'full-row'")]:
        assert re.search(rf"\b{arg}: [^=]*= {re.escape(default)}[,)]", doc), arg
    doc = pkg.solve_rk.__doc__
    for arg, default in [("epochs", "100"), ("target", "0.0"), ("seed", "0"), ("sampling", "'uniform'")]:
        assert re.search(rf"\b{arg}: [^=]*= {re.escape(default)}[,)]", doc), arg


@pytest.mark.parametrize(
    "rows,cols,vals,code",
    [
        ([0, 0], [1, 1], [1.0, 2.0], "DuplicateEntry"),
        ([0, 2], [1, 1], [1.0, 2.0], "IndexOutOfRange"),
        ([0], [1], [1.0], "ZeroRow"),
        ([0, 1], [0], [1.0, 1.0], "DimensionMismatch"),
    ],
)
def test_host_validation_errors_surface_as_value_error(rows, cols, vals, code):
    import paper_1401_4780_b200 as pkg

    with pytest.raises(ValueError, match=code):
        pkg.solve_parallel(2, 2, rows, cols, vals, [1.0, 1.0], threads=2)
    with pytest.raises(ValueError, match=code):
        pkg.solve_rk(2, 2, rows, cols, vals, [1.0, 1.0])


def test_bad_variant_and_sampling_names():
    import paper_1401_4780_b200 as pkg

    with pytest.raises(ValueError, match="InvalidArgument"):
        pkg.solve_parallel(2, 2, [0, 1], [0, 1], [1.0, 1.0], [1.0, 1.0], variant="diagonal")
    with pytest.raises(ValueError, match="InvalidArgument"):
        pkg.solve_rk(2, 2, [0, 1], [0, 1], [1.0, 1.0], [1.0, 1.0], sampling="sorted")


def test_no_silent_cpu_fallback():
    from paper_1401_4780_b200 import capi

    A, b, _ = capi.generate_fixed_theta(64, 32, 4, seed=1)
    try:
        s = capi.System(A, b)
    except capi.AsyrkError as e:
        assert e.name == "ThreadSpawnFailure" and "CUDA" in str(e)
        return
    s.close()
    pytest.skip("a CUDA device is present; the GPU suite covers this path")


def test_generator_contract():
    from paper_1401_4780_b200 import capi

    m, n, th = 3000, 1000, 20
    A, b, xs = capi.generate_fixed_theta(m, n, th, seed=5, threads=4)
    A2, b2, xs2 = capi.generate_fixed_theta(m, n, th, seed=5, threads=1)
    assert np.array_equal(A.values, A2.values) and np.array_equal(b, b2)  # thread-count independent
    assert np.array_equal(A.row_ptr, np.arange(m + 1) * th)
    cols = A.col_idx.reshape(m, th)
    assert np.all(np.diff(cols, axis=1) > 0) and cols.min() >= 0 and cols.max() < n
    assert A.normalized and np.all(np.abs(A.row_norm - 1.0) <= 1e-12)
    dense_b = (A.values.reshape(m, th) * xs[cols]).sum(axis=1)
    assert np.allclose(b, dense_b, rtol=1e-12, atol=1e-12)
    # config 4 style: log-uniform row scaling -> raw norms in [0.1, 10]
    A4, b4, _ = capi.generate_fixed_theta(m, n, 25, seed=9, scale_decades=1.0)
    assert not A4.normalized and A4.row_norm.min() >= 0.1 - 1e-12 and A4.row_norm.max() <= 10 + 1e-9
    # uniform values, multi-RHS layout
    A3, B3, X3 = capi.generate_fixed_theta(500, 200, 10, seed=3, dist="uniform", k=4)
    assert B3.shape == (500, 4) and X3.shape == (200, 4)
    v = A3.values.reshape(500, 10)
    assert np.allclose(B3, np.einsum("it,itk->ik", v, X3[A3.col_idx.reshape(500, 10)]), rtol=1e-12, atol=1e-12)


def test_generator_rejects_bad_shapes():
    from paper_1401_4780_b200 import capi

    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.generate_fixed_theta(10, 5, 6, seed=1)


def test_corollary_tau_bound():
    import paper_1401_4780_b200 as pkg

    # 2e*lambda*(tau+1)/m <= 1  (stepsize.cpp:64-69); SURVEY probe: cfg2 lambda 6.076 -> tau_max 6054
    assert pkg.max_feasible_tau(200000, 6.076) == 6053  # m/(2e*lambda) - 1 = 6053.6
    lam = 6.076
    t = pkg.max_feasible_tau(200000, lam)
    assert 2 * np.e * lam * (t + 1) / 200000 <= 1 < 2 * np.e * lam * (t + 2) / 200000


def test_pybind_stats_and_simulate_signatures_match_reference():
    # ref/bindings/module.cpp:286-310
    import paper_1401_4780_b200 as pkg

    doc = pkg.simulate.__doc__
    for arg in ["m", "n", "rows", "cols", "vals", "b", "iterations", "tau", "gamma"]:
        assert f"{arg}:" in doc
    for arg, default in [("delay", "'uniform'"), ("variant", "'single'"), ("seed", "0")]:
        assert re.search(rf"\b{arg}: [^=]*= {re.escape(default)}[,)]", doc), arg
    for fn, extra in [(pkg.system_stats, []), (pkg.step_params, ["tau"])]:
        for arg in ["m", "n", "rows", "cols", "vals"] + extra:
            assert f"{arg}:" in fn.__doc__
    # module.cpp:311-316
    for arg in ["m", "n", "rows", "cols", "vals", "b"]:
        assert f"{arg}:" in pkg.lsq.__doc__
    for arg, default in [("epochs", "5000"), ("target", "0.0"), ("seed", "0")]:
        assert re.search(rf"\b{arg}: [^=]*= {re.escape(default)}[,)]", pkg.lsq.__doc__), arg


def test_host_csr_row_norms_are_serial_sums():
    # csr.cpp:53-61: the cached norm is sqrt of a storage-order serial sum; a
    # pairwise sum differs in the last ulp for many rows and would change every
    # projection coefficient of the deterministic path
    import math

    from paper_1401_4780_b200 import capi
    rng = np.random.default_rng(4)
    lens = rng.integers(1, 200, size=300)
    rp = np.concatenate([[0], np.cumsum(lens)])
    v = rng.standard_normal(rp[-1])
    A = capi.HostCsr(300, 250, rp, np.zeros(rp[-1], np.int64), v)
    want = []
    for i in range(300):
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s += v[k] * v[k]
        want.append(math.sqrt(s))
    assert np.array_equal(A.row_norm, np.array(want))


def _build_drop_in_caller(tmp_path):
    import subprocess
    exe = str(tmp_path / "drop_in_caller")
    lib = os.path.join(ROOT, "paper_1401_4780_b200")
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "drop_in_caller.cpp"), "-o", exe, "-L", lib, "-lasyrk_b200",
                    f"-Wl,-rpath,{lib}"], check=True, capture_output=True)
    return exe


def test_cpp_drop_in_caller_compiles_against_the_headers(tmp_path):
    # a reference-style C++ caller (tests/cpp/drop_in_caller.cpp) builds against
    # include/asyrk/*.hpp and links libasyrk_b200.so (run on the GPU in test_gpu_parity.py)
    assert os.path.exists(_build_drop_in_caller(tmp_path))


def test_bench_reference_arm_json_contract():
    # bench.py --impl reference runs the reference's own CPU path (oracle/_ref)
    # and prints one JSON line with the contract's keys (a CPU-only workload here)
    import json
    import subprocess
    import sys
    ref = os.path.join(ROOT, "oracle", "_ref", "libasyrk_ref.so")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "mc",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"]:
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_host_vectors_are_length_checked():
    # the C ABI copies n (or m) doubles from the caller's pointers: short
    # vectors are rejected before the call with the reference's
    # DimensionMismatch (parallel.cpp:57-61), no device needed
    from paper_1401_4780_b200 import capi

    A, b, xs = capi.generate_fixed_theta(200, 100, 5, seed=1)
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.solve_parallel_host(A, b[:-1], threads=4, epochs=2)
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.solve_parallel_host(A, b, x0=np.zeros(99), threads=4, epochs=2)
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.solve_parallel_host(A, b, x_star=xs[:50], threads=4, epochs=2)
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.sweep_threads(A, b[:10], [1, 2])
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.simulate(A, b, np.zeros(3), 1.0, 0, "fixed", 10, 1, "full_row")
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.MultiRHS(A, np.zeros((10, 4), np.float32), 0, 4)


def test_trace_serializers_match_the_reference_bytes(tmp_path):
    # Trace::to_jsonl / to_csv (host/trace.cpp, doubles through grisu2.hpp) vs the
    # reference's (trace.cpp:33-112, nlohmann/json) on the same trace content:
    # 40000 doubles over many magnitudes, integral values, powers of two,
    # subnormals, negatives and the fixed / exponent layout boundaries
    import subprocess

    import oracle

    R = oracle.REF
    if R is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(11)
    vals = [rng.standard_normal(8000) * 10.0 ** rng.integers(-30, 30, 8000),
            rng.random(8000), np.exp(rng.uniform(-700, 700, 8000)),
            np.ldexp(1.0, rng.integers(-1070, 1020, 4000)).astype(float),
            np.round(rng.uniform(-1e6, 1e6, 4000)), rng.uniform(0, 1, 4000) * 1e-310,
            np.array([1e-4, 1e-5, 9.999e-5, 1e15, 1e16, 123456789012345.0, 1234567890123456.0, 0.1, 1.0, 2.0,
                      5e-324, 1.7976931348623157e308, 2.2250738585072014e-308, 0.0, -0.0, 3.0, 100.0])]
    v = np.concatenate(vals)
    v = v[np.isfinite(v)]
    src = tmp_path / "v.bin"
    v.tofile(src)
    exe = str(tmp_path / "trace_dump")
    lib = os.path.join(ROOT, "paper_1401_4780_b200")
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "trace_dump.cpp"), "-o", exe, "-L", lib, "-lasyrk_b200",
                    f"-Wl,-rpath,{lib}"], check=True, capture_output=True)
    subprocess.run([exe, str(src), str(tmp_path / "t.jsonl"), str(tmp_path / "t.csv")], check=True)
    ours_j = (tmp_path / "t.jsonl").read_text()
    ours_c = (tmp_path / "t.csv").read_text()
    ref_j, ref_c = R.trace_roundtrip(ours_j)
    if ours_j != ref_j:  # name the first differing number
        for a, b in zip(ours_j.split(","), ref_j.split(",")):
            assert a == b
    assert ours_j == ref_j
    assert ours_c == ref_c


def test_csr_from_coo_matches_from_triplets(tmp_path):
    # the pybind drop-in path assembles the CSR straight from the coordinate
    # arrays (host/csr_coo.hpp, parallel passes when already sorted): same
    # arrays and row norms as CsrMatrix::from_triplets (ref csr.cpp:9-63), or the
    # same error, on sorted / unsorted / zero-valued / out-of-range / duplicate input
    import subprocess

    exe = str(tmp_path / "csr_coo_check")
    lib = os.path.join(ROOT, "paper_1401_4780_b200")
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "csr_coo_check.cpp"), "-o", exe, "-L", lib, "-lasyrk_b200",
                    f"-Wl,-rpath,{lib}"], check=True, capture_output=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    assert out.startswith("ok 48"), out
