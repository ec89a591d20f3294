"""GPU: re-entrancy of the C-ABI (SURVEY.md §8(b) "Threading": the reference runs
one Trainer per std::thread, copris_cli.cpp:98-115, so the replacement keeps no
global mutable state — every call takes an explicit context and stream).

Several contexts on several host threads, each on its own CUDA stream, run the
whole path (packing, advantages, the fused loss, the reduction, the device error
check) at the same time; every result must be bitwise the one the same context
computes alone, and match the CPU oracle."""
import threading

import pytest
import torch

from parity_util import Case

pytestmark = pytest.mark.gpu

# several vocab sizes on the same kernel (fused_tma_kernel: 256 .. 32,000) with
# different shared-memory sizes: the per-function smem attribute is process-wide,
# so a thread lowering it under another thread's launch fails that launch
SPECS = [(11, 32000), (12, 151936), (13, 4099), (14, 32000), (15, 256), (16, 151936),
         (17, 1024), (18, 8000)]


def _run(ctx, case, stream, fused=True):
    with torch.cuda.stream(stream):
        logits = case.logits_gpu()
        batch = case.upload(ctx)
        res = ctx.grpo_step_loss(logits, batch, case.clip(), coef=True, fused=fused, stream=stream)
        stream.synchronize()
        return (res.loss, res.token_count, res.stale_tokens, res.clipped_tokens,
                res.cur_lp.cpu(), res.obj.cpu(), res.flags.cpu(),
                res.dlogits.view(torch.int16).cpu() if res.dlogits is not None else None), res


def _same(a, b):
    assert a[:4] == b[:4]
    for x, y in zip(a[4:], b[4:]):
        assert torch.equal(x, y)


@pytest.mark.parametrize("fused", [True, False])
def test_contexts_on_threads_bitwise(oracle, fused):
    from paper_2511_05589_b200 import Copris
    cases = [Case(oracle, seed=s, P=4, G=4, V=v, lmax=96) for s, v in SPECS]
    ctxs = [Copris(0) for _ in cases]
    streams = [torch.cuda.Stream() for _ in cases]
    alone = [_run(ctx, c, s, fused)[0] for ctx, c, s in zip(ctxs, cases, streams)]
    cases[1].check(_run(ctxs[1], cases[1], streams[1], fused)[1], torch.bfloat16, what="alone")

    results, errors = [None] * len(cases), []
    start = threading.Barrier(len(cases))

    def worker(i):
        try:
            start.wait()
            for _ in range(5):
                out, res = _run(ctxs[i], cases[i], streams[i], fused)
                _same(out, alone[i])
            results[i] = res
        except BaseException as e:  # surfaced below
            errors.append((i, e))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for case, res in zip(cases, results):
        case.check(res, torch.bfloat16, what="threaded")


def test_error_state_is_per_thread_and_per_context(oracle):
    """A contract violation detected on one context/thread does not leak into a
    concurrent healthy one (device error word per context, last-error message
    thread-local)."""
    from paper_2511_05589_b200 import Copris
    from paper_2511_05589_b200.errors import ContractViolation
    good = Case(oracle, seed=21, P=4, G=4, V=32000, lmax=64)
    bad = Case(oracle, seed=22, P=4, G=4, V=32000, lmax=64)
    ctx_good, ctx_bad = Copris(0), Copris(0)
    s_good, s_bad = torch.cuda.Stream(), torch.cuda.Stream()
    ref = _run(ctx_good, good, s_good)[0]
    outcome = {}

    def run_bad():
        with torch.cuda.stream(s_bad):
            logits = bad.logits_gpu()
            batch = bad.upload(ctx_bad)
            batch.target[3] = bad.V + 5  # token out of vocabulary
            try:
                ctx_bad.grpo_step_loss(logits, batch, bad.clip(), stream=s_bad)
                outcome["bad"] = None
            except ContractViolation as e:
                outcome["bad"] = str(e)

    def run_good():
        outs = [_run(ctx_good, good, s_good)[0] for _ in range(3)]
        outcome["good"] = outs

    ts = [threading.Thread(target=run_bad), threading.Thread(target=run_good)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert outcome["bad"] is not None and "token out of vocabulary" in outcome["bad"]
    for o in outcome["good"]:
        _same(o, ref)
    # the failed context is usable again after the error was reported
    _same(_run(ctx_bad, good, s_bad)[0], ref)


def test_host_dropin_on_threads_bitwise(oracle):
    """The host-buffer drop-in (copris_grpo_step_loss_host: pinned host arrays in,
    3-stream chunked pipeline, host loss and dlogits out) from several threads,
    each with its own context and workspace: bitwise the single-threaded result."""
    import math
    import numpy as np
    from paper_2511_05589_b200 import Copris
    from paper_2511_05589_b200.grpo import HostWorkspace
    specs = [(31, 32000), (32, 151936), (33, 8000), (34, 32000)]
    cases = [Case(oracle, seed=s, P=4, G=4, V=v, mu=math.log(20), lmax=64) for s, v in specs]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    ctxs = [Copris(0) for _ in cases]
    wss = [HostWorkspace(ctx, chunk_rows=37, vocab=c.V, max_tokens=c.hb.n_tok, max_traj=c.hb.n_traj,
                         dlogits_dtype=torch.bfloat16) for ctx, c in zip(ctxs, cases)]

    def call(i):
        c, hb = cases[i], cases[i].hb
        dl = torch.empty((hb.n_tok, c.V), dtype=torch.bfloat16).pin_memory()
        out = wss[i].grpo_step_loss(c.logits_cpu.pin_memory(), pin(hb.tok_off), pin(hb.target),
                                    pin(hb.stage.view(np.int32)), pin(c.blp), hb.cur_stage,
                                    rewards=pin(hb.reward), group_off=pin(hb.group_off),
                                    cfg=c.clip(), dlogits=dl)
        return out, dl

    alone = [call(i) for i in range(len(cases))]
    errors = []
    start = threading.Barrier(len(cases))

    def worker(i):
        try:
            start.wait()
            for _ in range(3):
                out, dl = call(i)
                assert out == alone[i][0]
                assert torch.equal(dl.view(torch.int16), alone[i][1].view(torch.int16))
        except BaseException as e:  # surfaced below
            errors.append((i, e))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i, c in enumerate(cases):
        assert alone[i][0]["token_count"] == c.hb.n_tok
        assert alone[i][0]["stale_tokens"] == c.ref.stale_tokens
    for ws in wss:
        ws.close()
