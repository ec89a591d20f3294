"""GPU: scheduler -> packed batch -> device pipeline, end to end.

The C++ rollout engine replays the reference's recorded event stream; every
batch it forms is packed, uploaded, and run through the device pipeline
(terminal rewards -> group advantages -> fused IS-corrected loss) and checked
against the CPU oracle on the same inputs."""
import gzip
import json
import os

import numpy as np
import pytest
import torch

from parity_util import assert_loss_close, assert_rows_close, assert_scalar_close

pytestmark = pytest.mark.gpu

STREAM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "engine_stream.jsonl.gz")


def _events(name):
    out, on = [], False
    with gzip.open(STREAM, "rt") as f:
        for line in f:
            ev = json.loads(line)
            if ev["op"] == "create":
                on = ev["scenario"] == name
            if on:
                out.append(ev)
    return out


@pytest.mark.parametrize("scenario", ["copris_c128_staleness1", "copris_c64_staleness2_h16",
                                      "naive_partial"])
def test_engine_batches_through_the_device_pipeline(ctx, oracle, scenario):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.engine import RolloutEngine
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import make_logits

    ev = _events(scenario)
    c = ev[0]
    V = c["vocab"]
    eng = RolloutEngine(mode=c["mode"], concurrency=c["concurrency"], batch_prompts=c["batch_prompts"],
                        rollouts_per_prompt=c["rollouts"], max_response_len=c["horizon"],
                        max_staleness=c["staleness"], vocab=V, seed=c["seed"])
    checked = 0
    for e in ev[1:]:
        op = e["op"]
        if op == "begin_stage":
            eng.begin_stage(e["version"])
        elif op == "append":
            eng.append_token(e["id"], e["token"], e["logprob"])
        elif op == "complete":
            eng.complete_trajectory(e["id"])
        elif op == "refill":
            eng.refill_active()
        elif op == "early_terminate":
            b = eng.early_terminate()
            d = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a if dt is None else a.view(dt))).cuda()
            # rewards and advantages on the device (grpo.hpp:35-65)
            reward = ctx.terminal_rewards(d(b.tokens), d(b.tok_off), d(b.terminated), d(b.answer_target),
                                          V - 1).cpu().numpy()
            np.testing.assert_array_equal(
                reward, oracle.terminal_rewards(b.tokens, b.tok_off, b.terminated, b.answer_target, V - 1))
            batch = upload(ctx, b.tok_off, b.group_off, b.tokens, b.buffered_lp, b.rollout_version,
                           seg_off=b.seg_off, seg_ver=b.seg_ver, reward=reward)
            np.testing.assert_array_equal(batch.stage.cpu().numpy().view(np.uint32), b.stage)
            adv = oracle.advantages(reward, b.group_off)
            np.testing.assert_array_equal(batch.adv.cpu().numpy(), adv)
            T = b.total_tokens
            logits = make_logits(T, V, b.tokens, 100 + checked, "cpu", torch.float32)
            res = ctx.grpo_step_loss(logits.cuda(), batch, ClipConfig(), dlogits_dtype=torch.float32)
            ref = oracle.is_loss(logits.double().numpy(), b.tok_off, b.tokens, b.stage,
                                 b.rollout_version, b.buffered_lp.astype(np.float64), adv)
            assert res.stale_tokens == ref.stale_tokens
            assert res.offpolicy_fraction == b.offpolicy_token_fraction()
            assert_scalar_close(res.cur_lp.cpu().numpy(), ref.cur_lp, what="cur_lp")
            # buffered log-probs here are arbitrary recorded values: ratios can sit anywhere,
            # so only the unguarded clip decisions may differ (none expected at this size)
            np.testing.assert_array_equal((res.flags.cpu().numpy() >> 1) & 1, ref.clipped)
            assert_loss_close(res.loss, ref.loss, ref.obj, T)
            atol = (V + 8) * 2.0 ** -52 * np.abs(ref.weight) / T
            assert_rows_close(res.dlogits.cpu().numpy(), ref.dlogits, row_atol=atol, what="dlogits")
            checked += 1
    assert checked >= 10
