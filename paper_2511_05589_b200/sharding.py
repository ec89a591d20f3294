"""Data-parallel sharding of the loss path over GPUs.

Rows are independent and advantages are group-local (grpo.hpp:51-65,
trainer.hpp:136-140), so whole prompt groups shard with no exchange in the
data path. Every rank scales by the GLOBAL token count (grpo.hpp:135), which
the host knows from the batch (TrainBatch::total_tokens, rollout.hpp:84-90).
After the kernels one allreduce(sum) of four fp64 scalars — objective,
tokens, stale tokens, clipped tokens — gives every rank the batch loss
-objective / T_global.
"""
from __future__ import annotations

import numpy as np


def lpt_shard(group_tokens, world: int) -> list[list[int]]:
    """Deterministic longest-processing-time assignment of whole groups.

    Groups are taken in descending token count (ties: lower group id first)
    and each goes to the least-loaded rank (ties: lower rank). Returns, per
    rank, its group ids in ascending (batch) order.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(group_tokens)), key=lambda g: (-int(group_tokens[g]), g))
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for g in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(g)
        load[r] += int(group_tokens[g])
    return [sorted(x) for x in out]


def shard_arrays(tok_off, group_off, per_token: dict, per_traj: dict, groups):
    """Rank-local packed arrays for a list of group ids (batch order kept).

    per_token / per_traj map names to global arrays indexed by packed token /
    trajectory. Returns (tok_off, group_off, per_token_local, per_traj_local,
    token_index) where token_index maps local tokens to global packed indices.
    """
    tok_off = np.asarray(tok_off, np.int64)
    group_off = np.asarray(group_off, np.int64)
    trajs = np.concatenate([np.arange(group_off[g], group_off[g + 1]) for g in groups]) \
        if len(groups) else np.zeros(0, np.int64)
    lens = tok_off[trajs + 1] - tok_off[trajs]
    l_tok_off = np.zeros(len(trajs) + 1, np.int64)
    l_tok_off[1:] = np.cumsum(lens)
    sizes = np.asarray([group_off[g + 1] - group_off[g] for g in groups], np.int64)
    l_group_off = np.zeros(len(groups) + 1, np.int64)
    l_group_off[1:] = np.cumsum(sizes)
    token_index = np.concatenate([np.arange(tok_off[i], tok_off[i + 1]) for i in trajs]) \
        if len(trajs) else np.zeros(0, np.int64)
    pt = {k: np.asarray(v)[token_index] for k, v in per_token.items()}
    pj = {k: np.asarray(v)[trajs] for k, v in per_traj.items()}
    return l_tok_off, l_group_off, pt, pj, token_index


def allreduce_scalars(out4, group=None):
    """SUM-allreduce of the four per-rank fp64 scalars (in place). Works with
    NCCL on CUDA tensors and gloo on CPU tensors; a no-op without a process
    group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out4, op=dist.ReduceOp.SUM, group=group)
    return out4


def loss_from_scalars(out4, total_tokens: int) -> float:
    """grpo.hpp:183: loss = -objective * (1 / T)."""
    return -float(out4[0]) * (1.0 / float(total_tokens))


class NcclScalars:
    """The C-ABI form of the collective (copris_allreduce_scalars), for callers
    that drive NCCL themselves instead of through torch.distributed — the C++
    trainer's path. ``NcclScalars.init_all([0, 1, ...])`` builds one
    communicator per GPU in this process (ncclCommInitAll);
    ``NcclScalars(device, n_ranks, uid, rank)`` joins a multi-process group
    whose 128-byte id came from ``NcclScalars.unique_id()`` on rank 0."""

    def __init__(self, device: int = None, n_ranks: int = None, uid: bytes = None,
                 rank: int = None, *, _comm=None):
        import ctypes as C
        from . import _lib as L
        from .grpo import _raise
        self._lib, self._raise = L.load(), _raise
        if _comm is not None:
            self.comm = _comm
            return
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        rc = self._lib.copris_nccl_comm_init_rank(device, n_ranks, buf, rank, C.byref(h))
        if rc:
            self._raise(rc, self._lib)
        self.comm = h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from . import _lib as L
        from .grpo import _raise
        lib = L.load()
        buf = (C.c_uint8 * 128)()
        rc = lib.copris_nccl_unique_id(buf)
        if rc:
            _raise(rc, lib)
        return bytes(buf)

    @classmethod
    def init_all(cls, devices) -> list["NcclScalars"]:
        import ctypes as C
        from . import _lib as L
        from .grpo import _raise
        lib = L.load()
        n = len(devices)
        devs = (C.c_int32 * n)(*devices)
        comms = (C.c_void_p * n)()
        rc = lib.copris_nccl_comm_init_all(n, devs, comms)
        if rc:
            _raise(rc, lib)
        return [cls(_comm=C.c_void_p(comms[i])) for i in range(n)]

    def allreduce(self, out4, stream=None):
        """SUM-allreduce of a device f64[4] (in place) on `stream` (default: current)."""
        import ctypes as C
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(out4.device)
        rc = self._lib.copris_allreduce_scalars(self.comm, C.c_void_p(out4.data_ptr()),
                                                C.c_void_p(s.cuda_stream))
        if rc:
            self._raise(rc, self._lib)
        return out4

    def close(self):
        if self.comm:
            rc = self._lib.copris_nccl_comm_destroy(self.comm)
            self.comm = None
            if rc:
                self._raise(rc, self._lib)
