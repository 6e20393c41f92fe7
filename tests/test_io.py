"""Instance I/O (ref/src/io.cpp:41-183) through the C ABI
(include/asyrk_io.h). Host-only: runs in the CPU suite. Files written here are
BYTE-IDENTICAL to the reference's writers, and parsing the reference's files
gives BIT-IDENTICAL arrays (oracle/_ref, the unmodified reference io.cpp);
the test cases follow ref tests/test_io_datagen.cpp:101-188."""
import os

import numpy as np
import pytest

import oracle

capi = pytest.importorskip("paper_1401_4780_b200.capi")
R = oracle.REF
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built")


def host_of(inst):
    return capi.HostCsr(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"], inst["row_norm"])


def same_csr(a, b):
    return (a.m == b.m and a.n == b.n and np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64)))


@needs_ref
def test_matrix_market_bytes_and_parse_match_reference(tmp_path, instances):
    for nm, inst in instances.items():
        A = host_of(inst)
        ours, ref = str(tmp_path / f"{nm}.ours.mtx"), str(tmp_path / f"{nm}.ref.mtx")
        capi.write_matrix_market(ours, A)
        Ar, _ = R.build(inst["m"], inst["n"], np.repeat(np.arange(inst["m"]), np.diff(inst["row_ptr"])),
                        inst["col_idx"], inst["values"], False, None)
        R.write_mtx(Ar, ref)
        assert open(ours, "rb").read() == open(ref, "rb").read(), nm
        back = capi.read_matrix_market(ref)
        e = R.read_mtx(ours).export()
        assert same_csr(back, capi.HostCsr(inst["m"], inst["n"], e["row_ptr"], e["col_idx"], e["values"])), nm
        assert same_csr(back, A) and np.array_equal(back.row_norm, A.row_norm), nm


@needs_ref
def test_awkward_values_round_trip(tmp_path):
    # test_io_datagen.cpp:113-123
    rows, cols = np.array([0, 0, 1, 1]), np.array([0, 1, 0, 1])
    vals = np.array([1.0 / 3.0, -2.5e-13, 1e17, -7.000000000000001])
    A = capi.HostCsr(2, 2, [0, 2, 4], cols, vals)
    p, q = str(tmp_path / "M.mtx"), str(tmp_path / "M.ref.mtx")
    capi.write_matrix_market(p, A)
    Ar, _ = R.build(2, 2, rows, cols, vals, False, None)
    R.write_mtx(Ar, q)
    assert open(p, "rb").read() == open(q, "rb").read()
    assert np.array_equal(capi.read_matrix_market(q).values.view(np.uint64), vals.view(np.uint64))


def _err(fn):
    with pytest.raises(capi.AsyrkError) as e:
        fn()
    return str(e.value)


@needs_ref
def test_malformed_files_match_reference_errors(tmp_path):
    # test_io_datagen.cpp:125-143, plus the other io.cpp failure paths
    cases = {
        "banner": "%%NotMatrixMarket\n2 2 1\n1 1 1.0\n",
        "zero_based": "%%MatrixMarket matrix coordinate real general\n2 2 2\n0 1 1.0\n1 1 1.0\n",
        "truncated": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n",
        "type": "%%MatrixMarket matrix array real general\n2 2\n",
        "size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
        "dims": "%%MatrixMarket matrix coordinate real general\n0 2 0\n",
        "junk_value": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 x\n2 2 1.0\n",
        "empty": "",
    }
    for nm, text in cases.items():
        p = str(tmp_path / f"{nm}.mtx")
        open(p, "w").write(text)
        ours = _err(lambda: capi.read_matrix_market(p))
        with pytest.raises(oracle.OracleError) as e:
            R.read_mtx(p)
        assert ours.startswith("IoError: ") and str(e.value).endswith(ours[len("IoError: "):]), (nm, ours, str(e.value))
    assert "cannot open" in _err(lambda: capi.read_matrix_market(str(tmp_path / "missing.mtx")))


@needs_ref
def test_comments_blank_lines_and_entry_layout(tmp_path):
    # comments/blank lines before the size line; entries may span lines;
    # unsorted entries and explicit zeros go through from_triplets
    text = ("%%MatrixMarket matrix coordinate real general\n%c1\n\n% c2\n3 3 6\n"
            "3 3 2.5\n1 2 -1e-300\n2 1 0.0 1 1 +4\n3 1\n7\n2 3 1.5\n")
    p = str(tmp_path / "c.mtx")
    open(p, "w").write(text)
    A = capi.read_matrix_market(p)
    e = R.read_mtx(p).export()
    assert same_csr(A, capi.HostCsr(3, 3, e["row_ptr"], e["col_idx"], e["values"]))
    assert A.nnz == 5  # the explicit zero is dropped
    open(p, "w").write(text.replace("2 3 1.5\n", "3 2 1.5\n"))  # row 2 is left with only the zero
    with pytest.raises(oracle.OracleError) as e:
        R.read_mtx(p)
    ours = _err(lambda: capi.read_matrix_market(p))
    assert ours.startswith("ZeroRow: ") and str(e.value).endswith(ours[len("ZeroRow: "):])


@needs_ref
def test_vectors_bytes_and_values(tmp_path):
    # test_io_datagen.cpp:145-154
    v = np.array([0.1, -3.0, 1e-17, 123456789.123456789, -0.0, 5e-324, 1.7976931348623157e308])
    p, q = str(tmp_path / "v.txt"), str(tmp_path / "v.ref.txt")
    capi.write_vector(p, v)
    R.write_vector(q, v)
    assert open(p, "rb").read() == open(q, "rb").read()
    assert np.array_equal(capi.read_vector(q).view(np.uint64), v.view(np.uint64))
    open(p, "w").write("1.5\n2.5 oops\n")
    assert "non-numeric content" in _err(lambda: capi.read_vector(p))
    with pytest.raises(oracle.OracleError, match="non-numeric content"):
        R.read_vector(p)
    assert "cannot open" in _err(lambda: capi.read_vector(str(tmp_path / "nope.txt")))


@needs_ref
@pytest.mark.parametrize("consistent", [True, False])
def test_instance_directories_match_reference(tmp_path, instances, consistent):
    # test_io_datagen.cpp:156-188
    inst = instances["seed_30x15"]
    A = host_of(inst)
    xs = inst["x_star"] if consistent else None
    spec = dict(m=inst["m"], n=inst["n"], delta=0.25, seed=43, consistent=consistent,
                noise_level=0.0 if consistent else 0.2)
    ours, ref = str(tmp_path / "ours"), str(tmp_path / "ref")
    capi.write_instance(ours, A, inst["b"], xs, spec)
    Ar, _ = R.build(inst["m"], inst["n"], np.repeat(np.arange(inst["m"]), np.diff(inst["row_ptr"])),
                    inst["col_idx"], inst["values"], True, None)
    R.write_instance(Ar, inst["b"], xs, spec, ref)
    names = sorted(os.listdir(ours))
    assert names == sorted(os.listdir(ref)) == (["A.mtx", "b.txt", "meta.json"] + (["xstar.txt"] if consistent else []))
    for f in names:
        assert open(os.path.join(ours, f), "rb").read() == open(os.path.join(ref, f), "rb").read(), f
    back = capi.read_instance(ref)
    assert same_csr(back["A"], A) and back["A"].normalized
    assert np.array_equal(back["b"].view(np.uint64), inst["b"].view(np.uint64))
    assert (back["x_star"] is None) == (not consistent)
    assert back["spec"] == spec
    rr = R.read_instance(ours)
    assert rr["spec"] == spec and np.array_equal(rr["b"], inst["b"])


def test_corrupted_instance_is_io_error(tmp_path, instances):
    inst = instances["seed_30x15"]
    d = str(tmp_path / "inst")
    capi.write_instance(d, host_of(inst), inst["b"], inst["x_star"], dict(delta=0.25, seed=43))
    with open(os.path.join(d, "b.txt"), "a") as f:
        f.write("1.5\n")
    assert "A and b dimensions disagree" in _err(lambda: capi.read_instance(d))


def test_binary_cache_round_trip(tmp_path):
    A, b, xs = capi.generate_fixed_theta(3000, 1000, 9, seed=8)
    p = str(tmp_path / "a.csr")
    capi.write_csr_cache(p, A)
    B = capi.read_csr_cache(p)
    assert same_csr(A, B) and np.array_equal(A.row_norm, B.row_norm) and B.normalized
    raw = bytearray(open(p, "rb").read())
    open(p, "wb").write(raw[:-8])
    assert "truncated or inconsistent cache" in _err(lambda: capi.read_csr_cache(p))
    raw[0] = ord("X")
    open(p, "wb").write(raw)
    assert "not an ASYRKCSR cache" in _err(lambda: capi.read_csr_cache(p))


@needs_ref
def test_parallel_reader_on_a_large_file(tmp_path):
    # > 1 MB of text: the multithreaded tokenizer splits the entry list
    A, b, xs = capi.generate_fixed_theta(40000, 15000, 12, seed=3)
    p = str(tmp_path / "big.mtx")
    capi.write_matrix_market(p, A)
    assert os.path.getsize(p) > (8 << 20)
    e = R.read_mtx(p).export()
    B = capi.read_matrix_market(p)
    assert same_csr(B, capi.HostCsr(A.m, A.n, e["row_ptr"], e["col_idx"], e["values"])) and same_csr(A, B)
    v = np.random.default_rng(0).standard_normal(300000)
    q = str(tmp_path / "big.txt")
    capi.write_vector(q, v)
    assert np.array_equal(capi.read_vector(q), v)
