"""Multi-GPU orchestration of the multi-right-hand-side AsyRK (BASELINE config 5).

One process per GPU (torchrun). The k right-hand sides are split into
contiguous column shards, one per rank; A is replicated. Every rank runs its
own lock-free warp-workers on its columns — there is no data-path exchange.
The only collective is the stopping test: after each snapshot the ranks
all-reduce (sum) their shard's {||R||_F^2, ||A^T R||_F^2, ||X - X*||_F^2}
(NCCL on the solve stream for CUDA tensors), then every rank's device-side
commit takes the same global decision ||R||_F^2 <= tol^2 ||B||_F^2.
Snapshots are taken at the boundaries the host-driven monitor schedule picks
(csrc/schedule.h); backend.due() says whether a step ended at one.

The same loop runs natively (no Python per epoch) through
capi.MultiRHS.solve_nccl (one process per GPU, an NCCL communicator the
library creates from a unique id the ranks share) and capi.mrhs_solve_devices
(one process, several GPUs); solve_sharded_native below wires the former to
torch.distributed.

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

    def due(self):
        return self.impl.due()

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
    for _ in range(max_chunks):
        if backend.stopped():
            break
        backend.step()
        # only the boundaries the monitor schedule evaluates carry norms; the
        # schedule is a function of the all-reduced records, so every rank
        # takes the same branch
        if backend.due():
            all_reduce(backend.norms())
            backend.commit(True)
    return backend.finish()


def relative_residual(trace, B_frob_sq):
    return float(np.sqrt(trace["r_sq"][-1] / B_frob_sq))


def solve_sharded_native(shard, group=None, **cfg):
    """This rank's shard through the native NCCL driver (asyrk_mrhs_solve_nccl):
    rank 0 creates the NCCL unique id, torch.distributed broadcasts it, the
    library builds its own communicator on the current device, and the whole
    loop (workers, monitor, ncclAllReduce, commit) runs in C++. With no
    process group: a 1-rank communicator."""
    import torch
    import torch.distributed as dist

    from . import capi

    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = capi.nccl_unique_id() if rank == 0 else bytes(capi.NCCL_UNIQUE_ID_BYTES)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, src=0, group=group)
        uid = bytes(t.cpu().tolist())
    else:
        world, rank, uid = 1, 0, capi.nccl_unique_id()
    comm = capi.NcclComm(world, uid, rank)
    try:
        return shard.solve_nccl(comm, **cfg)
    finally:
        comm.close()
