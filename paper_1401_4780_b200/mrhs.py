"""Multi-GPU orchestration of the multi-right-hand-side AsyRK (BASELINE config 5).

One process per GPU (torchrun). The k right-hand sides are split into
contiguous column shards, one per rank; A is replicated. Every rank runs its
own lock-free warp-workers on its columns — there is no data-path exchange.
The only collective is the stopping test: after each snapshot the ranks
all-reduce (sum) their shard's {||R||_F^2, ||A^T R||_F^2, ||X - X*||_F^2}
(NCCL on the solve stream for CUDA tensors), then every rank's device-side
commit takes the same global decision ||R||_F^2 <= tol^2 ||B||_F^2.

The loop is written against a small backend protocol so that the host logic
(sharding, the global stop, identical records on every rank) is testable on
CPU with gloo (tests/test_multirank.py); the product backend is
capi.MultiRHS. There is no CPU fallback: without the CUDA library the
backend cannot be created.
"""
from __future__ import annotations

import numpy as np


def shard_columns(k_total: int, world: int, rank: int):
    """Contiguous equal column blocks [c0, c1); k_total must split evenly."""
    if k_total % world:
        raise ValueError(f"InvalidArgument: {k_total} right-hand sides do not split over {world} ranks")
    kl = k_total // world
    return rank * kl, (rank + 1) * kl


class _DeviceDoubles:
    """__cuda_array_interface__ view of a device double[n] owned by the library."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


class CudaShardBackend:
    """capi.MultiRHS behind the protocol used by solve_sharded."""

    def __init__(self, A, B, c0, c1, stream=None):
        import torch

        from . import capi

        # the shard's kernels run on torch's current stream, so the all-reduce
        # (NCCL / torch ops on the norms tensor) is stream-ordered with them
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
            if stream == 0:
                stream = 1  # torch's default stream is the legacy stream: cudaStreamLegacy == (cudaStream_t)0x1
        self.impl = capi.MultiRHS(A, B, c0, c1, stream=stream)
        self._norms = None

    def begin(self, **cfg):
        self.impl.begin(**cfg)

    def norms(self):
        import torch

        if self._norms is None:
            self._norms = torch.as_tensor(_DeviceDoubles(self.impl.norms_ptr(), 3), device="cuda")
        return self._norms

    def commit(self, advance):
        self.impl.commit(advance)

    def step(self):
        self.impl.step()

    def stopped(self):
        return self.impl.stopped()

    def finish(self):
        return self.impl.finish()

    def close(self):
        self.impl.close()


def solve_sharded(backend, group=None, all_reduce=None, **cfg):
    """Run one multi-RHS solve on this rank's shard with a global stop test.

    all_reduce(tensor) sums in place over the ranks (default:
    torch.distributed.all_reduce when a process group is initialized, else a
    no-op, i.e. a single-rank solve). cfg: RunConfig fields (threads, gamma,
    epochs, target = tol^2 * ||B||_F^2 over ALL columns, snapshot_interval,
    seed) plus X0 / X_star.
    """
    if all_reduce is None:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            def all_reduce(t):
                dist.all_reduce(t, group=group)
        else:
            def all_reduce(t):
                return None
    backend.begin(**cfg)
    all_reduce(backend.norms())
    backend.commit(False)
    epochs = int(cfg.get("epochs", 100))
    interval = max(int(cfg.get("snapshot_interval", 1)), 1)
    max_chunks = (epochs + interval - 1) // interval if epochs > 0 else 0
    if not backend.stopped():
        for _ in range(max_chunks):
            backend.step()
            all_reduce(backend.norms())
            backend.commit(True)
            if backend.stopped():
                break
    return backend.finish()


def relative_residual(trace, B_frob_sq):
    return float(np.sqrt(trace["r_sq"][-1] / B_frob_sq))
