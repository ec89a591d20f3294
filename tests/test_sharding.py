"""CPU: whole-group sharding and the scalar allreduce.

Multi-process with the gloo backend (world_size 2, 127.0.0.1): each rank runs
the CPU oracle (as the checker stands in for the kernels here, which need a
GPU) on its LPT shard with the GLOBAL token count, the four scalars are
summed with sharding.allreduce_scalars, and the result must equal the
unsharded batch."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_05589_b200.sharding import (allreduce_scalars, loss_from_scalars, lpt_shard,
                                           shard_arrays)
from paper_2511_05589_b200.workload import make_host_batch


def test_lpt_is_deterministic_balanced_and_complete():
    rng = np.random.default_rng(0)
    toks = rng.integers(100, 10000, 200)
    for world in (1, 2, 4, 8):
        a = lpt_shard(toks, world)
        assert a == lpt_shard(toks, world)
        flat = sorted(g for r in a for g in r)
        assert flat == list(range(200))
        loads = [int(toks[r].sum()) if r else 0 for r in a]
        # LPT bound: max load <= mean + largest item
        assert max(loads) <= sum(loads) / world + toks.max()
        assert all(r == sorted(r) for r in a)


def test_lpt_tie_breaks():
    assert lpt_shard([5, 5, 5, 5], 2) == [[0, 2], [1, 3]]
    assert lpt_shard([1, 9], 3) == [[1], [0], []]


def test_shard_arrays_roundtrip():
    hb = make_host_batch(3, 6, 4, 50, mu=math.log(10), sigma=0.5, lmax=30)
    shards = lpt_shard(hb.group_tokens(), 3)
    seen = []
    for groups in shards:
        tok_off, group_off, pt, pj, idx = shard_arrays(
            hb.tok_off, hb.group_off, {"target": hb.target, "stage": hb.stage},
            {"reward": hb.reward}, groups)
        assert tok_off[-1] == len(idx) == len(pt["target"])
        np.testing.assert_array_equal(pt["target"], hb.target[idx])
        assert group_off[-1] == len(pj["reward"])
        seen.append(idx)
    allidx = np.sort(np.concatenate(seen))
    np.testing.assert_array_equal(allidx, np.arange(hb.n_tok))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        o = Oracle()
        hb = make_host_batch(11, 6, 4, 40, mu=math.log(8), sigma=0.7, lmax=20)
        rng = np.random.default_rng(5)
        z = rng.normal(0, 2, (hb.n_tok, 40))
        cur = o.logprob_gather(z, hb.target)
        blp = np.where(hb.stage < hb.cur_stage, cur + rng.uniform(-0.3, 0.3, hb.n_tok), cur)
        adv = o.advantages(hb.reward, hb.group_off)
        groups = lpt_shard(hb.group_tokens(), world)[rank]
        tok_off, group_off, pt, pj, idx = shard_arrays(
            hb.tok_off, hb.group_off, {"target": hb.target, "stage": hb.stage, "blp": blp},
            {"adv": adv}, groups)
        obj, stale, clipped = 0.0, 0, 0
        if len(idx):
            r = o.is_loss(z[idx], tok_off, pt["target"], pt["stage"], hb.cur_stage, pt["blp"],
                          pj["adv"])
            obj, stale, clipped = r.objective, r.stale_tokens, r.clipped_tokens
        out4 = torch.tensor([obj, float(len(idx)), float(stale), float(clipped)], dtype=torch.float64)
        allreduce_scalars(out4)
        if rank == 0:
            full = o.is_loss(z, hb.tok_off, hb.target, hb.stage, hb.cur_stage, blp, adv)
            q.put((loss_from_scalars(out4, hb.n_tok), full.loss, out4.tolist(), hb.n_tok,
                   full.stale_tokens, full.clipped_tokens))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_scalar_allreduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    loss, full_loss, out4, T, stale, clipped = res
    assert out4[1] == T and out4[2] == stale and out4[3] == clipped
    assert abs(loss - full_loss) <= 1e-12 * max(1.0, abs(full_loss))
