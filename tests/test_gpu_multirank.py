"""GPU, two or more devices: the sharded loss over a REAL multi-rank NCCL
communicator, against the unsharded CPU oracle.

  * one process, one thread per GPU (the reference runs one Trainer per
    std::thread, copris_cli.cpp:98-115): communicators from
    copris_nccl_comm_init_all, the four scalars reduced by
    copris_allreduce_scalars;
  * one process per GPU (the torchrun layout bench.py uses): NCCL through
    torch.distributed, a 127.0.0.1 rendezvous.

Both skip when fewer than two GPUs are visible (the build box has one; the
same sharding is checked on one GPU by test_gpu_fullsize.py and on CPU under
gloo by test_sharding.py)."""
import math
import os
import socket
import threading

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")]


def _problem(oracle, V=32000, P=8, G=4):
    from paper_2511_05589_b200.workload import make_host_batch, make_logits, stale_logprobs
    hb = make_host_batch(11, P, G, V, mu=math.log(64), sigma=1.0, lmax=256)
    logits = make_logits(hb.n_tok, V, hb.target, 11)  # host bf16
    z64 = logits.double().numpy()
    cur = oracle.logprob_gather(z64, hb.target)
    blp = stale_logprobs(cur, hb.stage, hb.cur_stage, 11)
    adv = oracle.advantages(hb.reward, hb.group_off)
    ref = oracle.is_loss(z64, hb.tok_off, hb.target, hb.stage, hb.cur_stage, blp.astype(np.float64),
                         adv, want_dlogits=False)
    return hb, logits, blp, ref


def _rank_loss(rank, world, hb, logits, blp):
    """This rank's shard: fused loss with the GLOBAL token count, then the
    deterministic reduction into a device f64[4]."""
    from paper_2511_05589_b200 import ClipConfig, Copris
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.sharding import lpt_shard, shard_arrays
    torch.cuda.set_device(rank)
    ctx = Copris(rank)
    groups = lpt_shard(hb.group_tokens(), world)[rank]
    t_off, g_off, pt, pj, idx = shard_arrays(hb.tok_off, hb.group_off,
                                             {"target": hb.target, "stage": hb.stage, "blp": blp},
                                             {"reward": hb.reward}, groups)
    dev = torch.device("cuda", rank)
    b = upload(ctx, t_off, g_off, pt["target"], pt["blp"], hb.cur_stage, stage=pt["stage"],
               reward=pj["reward"], device=dev)
    n = len(idx)
    lg = logits[torch.from_numpy(idx)].to(dev)
    outs = ctx.alloc_outputs(n, dev)
    dl = torch.empty_like(lg)
    ctx.loss_chunk_fused(lg, b, ClipConfig(), outs, dlogits=dl, total_tokens=hb.n_tok)
    out4 = torch.zeros(4, dtype=torch.float64, device=dev)
    ctx.reduce(outs, n, out4)
    ctx.check()
    return ctx, out4


def test_sharded_loss_nccl_init_all_threads(oracle):
    from paper_2511_05589_b200.sharding import NcclScalars, loss_from_scalars
    from parity_util import assert_loss_close
    world = min(torch.cuda.device_count(), 4)
    hb, logits, blp, ref = _problem(oracle)
    comms = NcclScalars.init_all(list(range(world)))
    got, errs = [None] * world, []

    def rank_main(r):
        try:
            ctx, out4 = _rank_loss(r, world, hb, logits, blp)
            comms[r].allreduce(out4)
            torch.cuda.synchronize(r)
            got[r] = out4.cpu()
            ctx.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for c in comms:
        c.close()
    assert not errs, errs
    for r in range(1, world):
        assert torch.equal(got[r], got[0])  # every rank holds the same sums
    assert int(got[0][1]) == hb.n_tok
    assert int(got[0][2]) == ref.stale_tokens and int(got[0][3]) == ref.clipped_tokens
    assert_loss_close(loss_from_scalars(got[0], hb.n_tok), ref.loss, ref.obj, hb.n_tok,
                      what=f"{world} ranks, copris_allreduce_scalars")


def _proc_main(rank, world, port, q):
    import torch.distributed as dist
    from oracle.oracle import Oracle
    from paper_2511_05589_b200.sharding import allreduce_scalars, loss_from_scalars
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    hb, logits, blp, ref = _problem(Oracle())
    _, out4 = _rank_loss(rank, world, hb, logits, blp)
    allreduce_scalars(out4)
    torch.cuda.synchronize()
    q.put((rank, dist.get_world_size(), out4.cpu().numpy().tolist(), ref.loss,
           ref.stale_tokens, ref.clipped_tokens, float(np.abs(ref.obj).sum()), hb.n_tok))
    dist.destroy_process_group()


def test_sharded_loss_nccl_one_process_per_gpu():
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sums = {tuple(r[2]) for r in res}
    assert len(sums) == 1  # identical on every rank
    _, ws, s4, ref_loss, stale, clipped, sabs, T = res[0]
    assert ws == world and int(s4[1]) == T and int(s4[2]) == stale and int(s4[3]) == clipped
    loss = -s4[0] * (1.0 / T)
    assert abs(loss - ref_loss) <= 1e-5 * max(abs(ref_loss), sabs / T)
