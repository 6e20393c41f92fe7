"""Multi-rank host logic of the RHS-sharded solve (paper_1401_4780_b200/mrhs.py)
on CPU: world_size 2 over gloo (127.0.0.1). The per-rank numerical backend
here is a small numpy Kaczmarz — test infrastructure standing in for the GPU
shard so that sharding, the all-reduced global stop and the identical
per-rank traces are checked without a GPU (the GPU backend is exercised in
tests/test_gpu_mrhs.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_4780_b200 import capi
from paper_1401_4780_b200.mrhs import shard_columns, solve_sharded


class NumpyShard:
    """Serial RK on columns [c0, c1) of X/B; same protocol as CudaShardBackend,
    including the library's monitor schedule (asyrk_monitor_schedule_next, the
    host arithmetic the native drivers use): only the boundaries it picks are
    evaluated and all-reduced."""

    def __init__(self, A, B, c0, c1):
        self.A, self.B = A, B[:, c0:c1].copy()
        self.c0, self.c1 = c0, c1

    def begin(self, threads=1, gamma=1.0, epochs=100, target=0.0, snapshot_interval=1, seed=0, X0=None,
              X_star=None, **_):
        m, n = self.A.shape
        self.X = np.zeros((n, self.c1 - self.c0))
        self.target, self.epochs, self.interval = target, epochs, snapshot_interval
        self.max_chunks = (epochs + snapshot_interval - 1) // snapshot_interval if epochs > 0 else 0
        self.rng = np.random.default_rng(seed)
        self.epoch, self.stop, self.records = 0, False, []
        self.b, self.next_mon, self.is_due = 0, 1, True
        self._norms = torch.zeros(3, dtype=torch.float64)
        self._measure()

    def _measure(self):
        R = self.A @ self.X - self.B
        self._norms[0] = float((R * R).sum())
        G = self.A.T @ R
        self._norms[1] = float((G * G).sum())
        self.local_r_sq = float(self._norms[0])

    def norms(self):
        return self._norms

    def commit(self, advance):
        if self.stop or not self.is_due:
            return
        self.is_due = False
        rs, gs = float(self._norms[0]), float(self._norms[1])
        self.records.append((self.b, self.epoch, rs, gs))
        if rs <= self.target or self.epoch >= self.epochs:
            self.stop = True
        bd = [r[0] for r in self.records[-2:]]
        rq = [r[2] for r in self.records[-2:]]
        self.next_mon = capi.monitor_schedule_next(self.target, bd, rq)

    def step(self):
        if self.stop:
            return
        m = self.A.shape[0]
        span = min(self.interval, self.epochs - self.epoch)
        for i in self.rng.integers(0, m, size=span * m):
            a = self.A[i]
            res = a @ self.X - self.B[i]
            self.X -= np.outer(a, res) / (a @ a)
        self.epoch += span
        self.b += 1
        self.is_due = self.b >= self.next_mon or self.b >= self.max_chunks
        if self.is_due:
            self._measure()

    def due(self):
        return self.is_due

    def stopped(self):
        return self.stop or self.b >= self.max_chunks

    def finish(self):
        return dict(epoch_index=np.array([r[1] for r in self.records]), r_sq=np.array([r[2] for r in self.records]),
                    X=self.X, local_r_sq=self.local_r_sq)


def _problem():
    rng = np.random.default_rng(5)
    m, n, k = 60, 30, 4
    A = rng.standard_normal((m, n)) * (rng.random((m, n)) < 0.3)
    A[np.arange(m), rng.integers(0, n, m)] += 1.0
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    Xs = rng.standard_normal((n, k))
    return A, A @ Xs, Xs


def _rank_main(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, B, Xs = _problem()
    c0, c1 = shard_columns(B.shape[1], world, rank)
    be = NumpyShard(A, B, c0, c1)
    target = (1e-5) ** 2 * float((B * B).sum())
    tr = solve_sharded(be, threads=1, epochs=400, target=target, seed=100 + rank)
    out[rank] = dict(c=(c0, c1), epochs=tr["epoch_index"].tolist(), r_sq=tr["r_sq"].tolist(),
                     local=tr["local_r_sq"], X=tr["X"])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_monitor_schedule_host_arithmetic():
    # asyrk_monitor_schedule_next (csrc/schedule.h): the next boundary while
    # fewer than two records exist / the residual did not drop / every boundary
    # is requested / the target is 0; else the first boundary at or after the
    # predicted crossing, at least 1 and at most the max gap
    nx = capi.monitor_schedule_next
    assert nx(1e-6, [0], [1.0]) == 1
    assert nx(1e-6, [3, 4], [1.0, 2.0]) == 5
    assert nx(1e-6, [3, 4], [1.0, 0.5], every=True) == 5
    assert nx(0.0, [3, 4], [1.0, 0.5]) == 5
    # r halves per boundary: the crossing is 30 boundaries away -> there, capped at the max gap (24)
    assert nx(2.0 ** -30, [3, 4], [2.0, 1.0]) == 4 + 24
    assert nx(2.0 ** -30, [3, 4], [2.0, 1.0], max_gap=40) == 4 + 30
    assert nx(2.0 ** -20, [3, 4], [2.0, 1.0]) == 4 + 20
    assert nx(2.0 ** -5.5, [3, 4], [2.0, 1.0]) == 4 + 6  # the first boundary at or after the crossing
    assert nx(2.0 ** -5, [3, 4], [2.0, 1.0]) == 4 + 5  # (a crossing on a boundary: that boundary)
    assert nx(2.0 ** -1, [3, 4], [2.0, 1.0]) == 4 + 1  # at most 1 away: the next one
    assert nx(0.9, [3, 4], [2.0, 1.0]) == 4 + 1


def test_shard_columns_cover_and_split_evenly():
    for world in (1, 2, 4, 8):
        spans = [shard_columns(64, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 64
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert len({c1 - c0 for c0, c1 in spans}) == 1
    with pytest.raises(ValueError, match="InvalidArgument"):
        shard_columns(64, 3, 0)


def test_two_rank_gloo_global_stop():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_rank_main, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    A, B, Xs = _problem()
    # disjoint shards covering all right-hand sides
    assert res[0]["c"] == (0, 2) and res[1]["c"] == (2, 4)
    # the all-reduced stop test makes both ranks stop at the same snapshot with identical records
    assert res[0]["epochs"] == res[1]["epochs"]
    assert res[0]["r_sq"] == res[1]["r_sq"]
    # the monitor schedule (a function of the all-reduced records) evaluated the
    # same subset of boundaries on both ranks: fewer records than epochs, the
    # last one meets the target and the one before it did not
    ep, rq = res[0]["epochs"], res[0]["r_sq"]
    target = (1e-5) ** 2 * float((B * B).sum())
    assert ep[0] == 0 and len(ep) < ep[-1] + 1
    assert rq[-1] <= target < rq[-2]
    # the recorded residual is the global one: sum of the shards' residuals
    assert res[0]["r_sq"][-1] == pytest.approx(res[0]["local"] + res[1]["local"], rel=1e-12)
    X = np.concatenate([res[0]["X"], res[1]["X"]], axis=1)
    rel = np.linalg.norm(A @ X - B) / np.linalg.norm(B)
    assert rel <= 1e-5
    assert np.linalg.norm(X - Xs) / np.linalg.norm(Xs) <= 1e-4
