"""GPU: clip-branch flips, fp32 device arithmetic vs the reference's fp64
(grpo.hpp:147-152), on inputs WITHOUT the synthetic guard band.

The device computes the ratio as expf(cur - behav) in fp32 from fp32 log-probs
(token_math.cuh) and the branch `u <= c` in fp64 on that ratio; the reference
does everything in fp64. A token whose ratio lies within a few fp32 ulps of
1 - eps_lo or 1 + eps_hi can take the other branch. The parity tests keep a
1e-4 guard band around the thresholds (workload.stale_logprobs) so their clip
masks are bit-exact; these tests drop it and COUNT the flips:

  * the reference Trainer's own batches (tests/golden/trainer_*.json, captured
    unmodified, never guarded): GPU flags vs the reference's branch on its fp64
    values (the oracle on the fp64 table, pinned bit-for-bit to the reference);
  * 4M synthetic tokens with guard = 0 (V = 64, fp32 stale log-probs):
    GPU vs the oracle on the same inputs.

Each test prints one JSON line (run with -s to collect them)."""
import json

import numpy as np
import pytest
import torch

from golden_io import all_steps, packed_step

pytestmark = pytest.mark.gpu


def _branch_stats(ratio_lo_hi, log_ratio, flips_mask):
    lo, hi = ratio_lo_hi
    d = np.minimum(np.abs(log_ratio - np.log(lo)), np.abs(log_ratio - np.log(hi)))
    return {"min_log_distance_to_threshold": float(d.min()) if d.size else None,
            "within_1e-6": int((d < 1e-6).sum()), "within_1e-4": int((d < 1e-4).sum()),
            "flips": int(flips_mask.sum())}


def test_reference_trainer_batches_unguarded(ctx, oracle):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.packing import upload
    tot = dict(steps=0, tokens=0, stale=0, clipped_ref=0, clipped_gpu=0, flips=0)
    near = []
    for name, step, fx, st in all_steps():
        ps = packed_step(fx, st)
        c = ps.clip
        if c["kl_coeff"] > 0:
            continue  # same branch logic; the KL term needs the snapshot log-probs
        batch = upload(ctx, ps.tok_off, ps.group_off, ps.target, ps.buffered_lp.astype(np.float32),
                       ps.cur_stage, stage=ps.stage, reward=ps.reward, adv_epsilon=c["adv_epsilon"])
        logits = torch.from_numpy(ps.logits.astype(np.float32)).cuda()
        cfg = ClipConfig(c["clip_low"], c["clip_high"], 0.0, c["entropy_coeff"], c["adv_epsilon"])
        res = ctx.grpo_step_loss(logits, batch, cfg, is_enabled=ps.is_enabled, dlogits_dtype=torch.float32)
        # the reference's branch: fp64 table, fp64 stored log-probs
        ref = oracle.is_loss(ps.logits, ps.tok_off, ps.target, ps.stage, ps.cur_stage, ps.buffered_lp,
                             ps.adv, c["clip_low"], c["clip_high"], 0.0, c["entropy_coeff"],
                             ps.is_enabled, want_dlogits=False)
        np.testing.assert_array_equal(ref.cur_lp, ps.current_lp)  # pinned to the fixture
        gpu_clip = (res.flags.cpu().numpy() >> 1) & 1
        flips = gpu_clip != ref.clipped
        tot["steps"] += 1
        tot["tokens"] += len(ps.target)
        tot["stale"] += int(res.stale_tokens)
        tot["clipped_ref"] += int(ref.clipped.sum())
        tot["clipped_gpu"] += int(gpu_clip.sum())
        tot["flips"] += int(flips.sum())
        near.append(ps.current_lp - ps.stored_lp)
    lr = np.concatenate(near)
    tot.update({k: v for k, v in _branch_stats((0.8, 1.28), lr, np.zeros(0, bool)).items() if k != "flips"})
    print(json.dumps({"clip_flips": "reference_trainer_fixtures", **tot}))
    assert tot["steps"] > 0 and tot["clipped_ref"] > 0
    assert tot["flips"] == 0


def test_synthetic_unguarded_4m_tokens(ctx, oracle):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import make_host_batch, make_logits, stale_logprobs
    V = 64
    hb = make_host_batch(11, 2048, 8, V, fixed_len=256, stages=(1, 2), stale_prob=1.0)
    T = hb.n_tok
    target = torch.from_numpy(hb.target).cuda()
    logits = make_logits(T, V, target, 11, device="cuda", dtype=torch.bfloat16)
    cur, _ = ctx.sequence_logprobs(logits, target)
    blp = stale_logprobs(cur.cpu().numpy(), hb.stage, hb.cur_stage, 11, guard=0.0)
    batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, blp, hb.cur_stage, stage=hb.stage,
                   reward=hb.reward)
    res = ctx.grpo_step_loss(logits, batch, ClipConfig())
    adv = oracle.advantages(hb.reward, hb.group_off)
    ref = oracle.is_loss(logits.float().cpu().numpy(), hb.tok_off, hb.target, hb.stage, hb.cur_stage,
                         blp.astype(np.float64), adv, want_dlogits=False)
    gpu_clip = (res.flags.cpu().numpy() >> 1) & 1
    flips = gpu_clip != ref.clipped
    stale = hb.stage < hb.cur_stage
    lr = (ref.cur_lp - blp.astype(np.float64))[stale]
    stats = _branch_stats((0.8, 1.28), lr, flips)
    out = {"clip_flips": "synthetic_unguarded", "tokens": int(T), "stale": int(stale.sum()),
           "clipped_ref": int(ref.clipped.sum()), "clipped_gpu": int(gpu_clip.sum()), **stats}
    if stats["flips"]:
        # a flip changes the objective by |u - c|, which is ~|r - threshold| |A|: tiny
        idx = np.nonzero(flips)[0]
        out["flip_log_distance"] = [float(np.min(np.abs(
            (ref.cur_lp[i] - float(blp[i])) - np.log([0.8, 1.28])))) for i in idx[:16]]
        out["loss_abs_err"] = abs(res.loss - ref.loss)
    print(json.dumps(out))
    assert stats["flips"] <= max(1, T // 100_000)
    assert stats["flips"] <= stats["within_1e-6"] + 1
