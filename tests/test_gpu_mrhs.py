"""GPU tests of the multi-right-hand-side path (BASELINE config 5 shape at
reduced size): convergence of every column to the tolerance, the sharded
protocol with the global stop test (two shards on one GPU, norms summed on
the host between step and commit — the all-reduce a multi-GPU run does with
NCCL), and the device records against an independent CPU evaluation."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")
from paper_1401_4780_b200.mrhs import CudaShardBackend, shard_columns, solve_sharded  # noqa: E402

TOL = 1e-5


@pytest.fixture(scope="module")
def problem():
    A, B, Xs = capi.generate_fixed_theta(50000, 25000, 20, seed=1005, k=64)
    return A, B.astype(np.float32), Xs


def _residual(A, X, B):
    m = A.m
    v = A.values.reshape(m, -1)
    c = A.col_idx.reshape(m, -1)
    AX = np.einsum("it,itk->ik", v, X[c].astype(np.float64))
    return AX - B


def test_single_gpu_all_columns_converge(problem):
    A, B, Xs = problem
    S = capi.MultiRHS(A, B, 0, 64)
    bb = float((B.astype(np.float64) ** 2).sum())
    t = S.solve(threads=2048, epochs=400, target=TOL * TOL * bb, seed=3, X_star=Xs)
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    R = _residual(A, t["X"], B)
    rel = np.sqrt((R * R).sum() / bb)
    assert rel <= 2 * TOL  # independent fp64 evaluation of the fp32 iterate
    assert abs((R * R).sum() - t["r_sq"][-1]) <= 0.05 * t["r_sq"][-1]
    err = np.linalg.norm(t["X"] - Xs) / np.linalg.norm(Xs)
    assert err <= 10 * TOL
    assert np.sqrt(t["dist_sq"][-1]) / np.linalg.norm(Xs) <= 10 * TOL
    # every column individually reaches the tolerance band
    col_rel = np.sqrt((R * R).sum(axis=0) / (B.astype(np.float64) ** 2).sum(axis=0))
    assert col_rel.max() <= 10 * TOL
    S.close()


def test_config5_full_size_all_columns():
    # BASELINE config 5 at full size on one GPU: 500k x 250k, theta 20, k = 64
    # fp32 right-hand sides -> global ||R||_F / ||B||_F < 1e-5, error within 10x
    A, B, Xs = capi.generate_fixed_theta(500000, 250000, 20, seed=1005, k=64)
    B = B.astype(np.float32)
    bb = float((B.astype(np.float64) ** 2).sum())
    S = capi.MultiRHS(A, B, 0, 64)
    t = S.solve(threads=4096, epochs=400, target=TOL * TOL * bb, seed=3, X_star=Xs)
    S.close()
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    assert np.sqrt(t["dist_sq"][-1]) / np.linalg.norm(Xs) <= 10 * TOL
    R = _residual(A, t["X"], B)
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL  # independent fp64 evaluation


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_protocol_global_stop(problem, world):
    A, B, Xs = problem
    bb = float((B.astype(np.float64) ** 2).sum())
    shards = [CudaShardBackend(A, B, *shard_columns(64, world, r)) for r in range(world)]

    # host-side "all-reduce" over the in-process shards (NCCL sums in place on each rank)
    def make_all_reduce(pending=[]):
        def all_reduce(t):
            pending.append(t)
            if len(pending) == world:
                tot = sum(p.clone() for p in pending)
                for p in pending:
                    p.copy_(tot)
                pending.clear()
        return all_reduce

    ar = make_all_reduce()
    cfg = dict(threads=1024, epochs=400, target=TOL * TOL * bb, X_star=Xs)
    for r, s in enumerate(shards):
        s.begin(seed=10 + r, **cfg)
    for s in shards:
        ar(s.norms())
    for s in shards:
        s.commit(False)
    evaluated = 0
    for _ in range(400):
        stops = [s.stopped() for s in shards]
        assert len(set(stops)) == 1  # identical global decision
        if stops[0]:
            break
        for s in shards:
            s.step()
        dues = [s.due() for s in shards]
        assert len(set(dues)) == 1  # identical schedule (a function of the all-reduced records)
        if dues[0]:
            evaluated += 1
            for s in shards:
                ar(s.norms())
            for s in shards:
                s.commit(True)
    res = [s.finish() for s in shards]
    assert all(np.array_equal(res[0]["epoch_index"], r["epoch_index"]) for r in res)
    assert all(np.array_equal(res[0]["r_sq"], r["r_sq"]) for r in res)
    assert len(res[0]["r_sq"]) == evaluated + 1  # boundary 0 + every evaluated boundary
    X = np.concatenate([r["X"] for r in res], axis=1)
    R = _residual(A, X, B)
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL
    assert np.linalg.norm(X - Xs) / np.linalg.norm(Xs) <= 10 * TOL
    for s in shards:
        s.close()


def test_solve_sharded_single_rank(problem):
    A, B, Xs = problem
    bb = float((B.astype(np.float64) ** 2).sum())
    be = CudaShardBackend(A, B, 0, 64)
    t = solve_sharded(be, all_reduce=lambda x: None, threads=2048, epochs=400, target=TOL * TOL * bb, seed=9)
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    be.close()


def test_bad_shard_width_rejected(problem):
    A, B, _ = problem
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.MultiRHS(A, B, 0, 48)


def test_slice_shuffle_sampling_converges(problem):
    # the reference's default ParSampling (parallel.cpp:355-363): each worker
    # reshuffles its slice of the rows every pass
    A, B, Xs = problem
    S = capi.MultiRHS(A, B, 0, 64)
    bb = float((B.astype(np.float64) ** 2).sum())
    t = S.solve(threads=2048, epochs=400, target=TOL * TOL * bb, seed=4, X_star=Xs, sampling=capi.SLICE_SHUFFLE)
    S.close()
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    R = _residual(A, t["X"], B)
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL
    assert np.linalg.norm(t["X"] - Xs) / np.linalg.norm(Xs) <= 10 * TOL
    # exact epochs: every launch processes m row events per epoch
    assert int(t["updates_applied"][-1]) == A.m * int(t["epoch_index"][-1])


@pytest.mark.parametrize("kl", [2, 4, 8, 16, 32])
def test_narrow_shards_converge(problem, kl):
    # the shard widths of 32 / 16 / 8 / 4 / 2 GPUs (float2 and float4 lane layouts;
    # the row-parallel worker and monitor at 8 / 16 / 32 columns)
    A, B, Xs = problem
    S = capi.MultiRHS(A, B, 0, kl)
    bb = float((B[:, :kl].astype(np.float64) ** 2).sum())
    t = S.solve(threads=2048, epochs=400, target=TOL * TOL * bb, seed=5)
    S.close()
    R = _residual(A, t["X"], B[:, :kl])
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL


def test_monitor_schedule_records(problem):
    # tolerance runs evaluate a subset of boundaries (the last one meets the
    # target, the one before did not); a fixed epoch budget (target 0) and
    # record_every_boundary evaluate every boundary
    A, B, Xs = problem
    bb = float((B.astype(np.float64) ** 2).sum())
    S = capi.MultiRHS(A, B, 0, 64)
    t = S.solve(threads=2048, epochs=400, target=TOL * TOL * bb, seed=3)
    ep = t["epoch_index"]
    assert ep[0] == 0 and np.all(np.diff(ep) > 0)
    assert t["r_sq"][-1] <= TOL * TOL * bb < t["r_sq"][-2]
    assert len(ep) < ep[-1] + 1
    t2 = S.solve(threads=2048, epochs=7, target=0.0, seed=3)
    assert list(t2["epoch_index"]) == list(range(8))
    t3 = S.solve(threads=2048, epochs=400, target=TOL * TOL * bb, seed=3, record_every_boundary=1)
    assert list(t3["epoch_index"]) == list(range(int(t3["epoch_index"][-1]) + 1))
    S.close()


def test_native_nccl_driver_one_rank(problem):
    # asyrk_mrhs_solve_nccl with a 1-rank communicator the library builds from
    # its own unique id: the NCCL all-reduce path of a multi-GPU job, on one GPU
    A, B, Xs = problem
    bb = float((B.astype(np.float64) ** 2).sum())
    assert capi.nccl_version() >= 21800
    comm = capi.NcclComm(1, capi.nccl_unique_id(), 0)
    S = capi.MultiRHS(A, B, 0, 64)
    t = S.solve_nccl(comm, threads=2048, epochs=400, target=TOL * TOL * bb, seed=3, X_star=Xs,
                     sampling=capi.SLICE_SHUFFLE)
    S.close()
    comm.close()
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    R = _residual(A, t["X"], B)
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL
    assert np.sqrt(t["dist_sq"][-1]) / np.linalg.norm(Xs) <= 10 * TOL


def test_solve_devices_single_process():
    # asyrk_mrhs_solve_devices: one process, ncclCommInitAll over the listed
    # GPUs; on a 1-GPU box the device list is [0] (NCCL with one rank)
    import torch

    A, B, Xs = capi.generate_fixed_theta(20000, 10000, 20, seed=77, k=8)
    B = B.astype(np.float32)
    bb = float((B.astype(np.float64) ** 2).sum())
    devs = list(range(min(torch.cuda.device_count(), 2)))
    t = capi.mrhs_solve_devices(A, B, devs, threads=1024, epochs=400, target=TOL * TOL * bb, seed=3, X_star=Xs)
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    st = t["stats"]  # device 0's timings and counts
    assert st["solve_ms"] > 0.0 and 0.0 < st["worker_ms"] <= st["solve_ms"] and st["worker_launches"] >= 1
    R = _residual(A, t["X"], B)
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL
    assert np.linalg.norm(t["X"] - Xs) / np.linalg.norm(Xs) <= 10 * TOL


def test_solve_devices_two_gpus():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    A, B, Xs = capi.generate_fixed_theta(50000, 25000, 20, seed=1005, k=64)
    B = B.astype(np.float32)
    bb = float((B.astype(np.float64) ** 2).sum())
    t = capi.mrhs_solve_devices(A, B, [0, 1], threads=2048, epochs=400, target=TOL * TOL * bb, seed=3)
    R = _residual(A, t["X"], B)
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL


@pytest.mark.parametrize("kl", [8, 32])
def test_row_parallel_ragged_rows(kl):
    # rows of 1..30 nonzeros: the row-parallel kernels read records whose length
    # is a multiple of 4 as int4 / float4 and the others entry by entry (mrhs.cu
    # row_gather / row_scatter); both kinds of rows in one system
    rng = np.random.default_rng(17)
    m, n = 30000, 12000
    lens = rng.integers(1, 31, size=m)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int64)
    v = rng.standard_normal(rp[-1])
    v /= np.repeat(np.sqrt(np.add.reduceat(v * v, rp[:-1])), lens)
    A = capi.HostCsr(m, n, rp, ci, v)
    Xs = rng.standard_normal((n, kl))
    row = np.repeat(np.arange(m), lens)
    B = np.zeros((m, kl))
    np.add.at(B, row, v[:, None] * Xs[ci])
    B = B.astype(np.float32)
    bb = float((B.astype(np.float64) ** 2).sum())
    S = capi.MultiRHS(A, B, 0, kl)
    t = S.solve(threads=min(S.max_resident_warps(), m // 8), epochs=600, target=TOL * TOL * bb, seed=3)
    S.close()
    R = -B.astype(np.float64)
    np.add.at(R, row, v[:, None] * t["X"][ci].astype(np.float64))
    assert np.sqrt(t["r_sq"][-1] / bb) <= TOL
    assert np.sqrt((R * R).sum() / bb) <= 2 * TOL
