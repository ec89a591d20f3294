"""GPU: full-size parity at BASELINE config #2 shapes through size-independent
properties (the oracle cannot run 10^10-element rows in test time):

  * whole prompt groups (>= 1 group, ~24k rows) at V = 151,936 of the config-#2
    batch: dlogits rows sum to zero (sum_k coef (1[k=y] - p_k) = 0), the target
    entry equals coef (1 - exp(cur_lp)), every off-target entry is
    -coef p_k with p_k = exp(z_k - lse) (checked on sampled columns);
  * 48 sampled rows against the CPU oracle in full;
  * stale/clipped counts and the loss agree with the per-token outputs;
  * bit-identical reruns and chunk-size invariance at full size.
"""

import numpy as np
import pytest
import torch

from parity_util import assert_rows_close, assert_scalar_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def big(ctx):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import CONFIGS, make_host_batch, make_logits, stale_logprobs
    cfg = dict(CONFIGS["grpo_128x8_v151936"])
    P, G, V = cfg.pop("P"), cfg.pop("G"), cfg.pop("vocab")
    hb = make_host_batch(1, 8, G, V, **cfg)          # prompt groups of the config
    # whole groups, at least one, up to ~24k tokens (7 GB of bf16 logits)
    g_full = 1
    while g_full < len(hb.group_off) - 1 and hb.tok_off[hb.group_off[g_full + 1]] <= 24576:
        g_full += 1
    n_traj = int(hb.group_off[g_full])
    T = int(hb.tok_off[n_traj])
    tok_off = hb.tok_off[: n_traj + 1]
    group_off = hb.group_off[: g_full + 1]
    target = hb.target[:T]
    stage = hb.stage[:T]
    logits = make_logits(T, V, torch.from_numpy(target).cuda(), 7, device="cuda")
    cur, lse = ctx.sequence_logprobs(logits, torch.from_numpy(target).cuda())
    blp = stale_logprobs(cur.cpu().numpy(), stage, hb.cur_stage, 7)
    batch = upload(ctx, tok_off, group_off, target, blp, hb.cur_stage, stage=stage,
                   reward=hb.reward[:n_traj])
    res = ctx.grpo_step_loss(logits, batch, ClipConfig(), coef=True)
    return dict(hb=hb, T=T, V=V, logits=logits, batch=batch, res=res, target=target, stage=stage,
                blp=blp, tok_off=tok_off, group_off=group_off)


def test_rows_sum_to_zero_and_target_entry(big):
    res, T, V = big["res"], big["T"], big["V"]
    dl = res.dlogits.float()
    coef = res.coef.float()
    rs = dl.sum(dim=1)
    scale = coef.abs() * 1.0
    # bf16 rounding of V entries: sum error ~ sqrt(V) * 2^-9 * |coef| / V ... bounded by 2^-8 |coef|
    assert torch.all(rs.abs() <= 4e-3 * scale + 1e-30), float((rs.abs() / (scale + 1e-30)).max())
    y = torch.from_numpy(big["target"]).cuda().long()
    dy = dl[torch.arange(T, device="cuda"), y]
    expect = coef * -torch.expm1(res.cur_lp.float())
    assert torch.all((dy - expect).abs() <= 2 ** -7 * expect.abs() + 1e-30)


def test_sampled_columns_match_softmax(big):
    res, T, V = big["res"], big["T"], big["V"]
    g = torch.Generator(device="cpu").manual_seed(3)
    cols = torch.randint(0, V, (T, 8), generator=g).cuda()
    z = big["logits"].gather(1, cols).float()
    p = torch.exp(z - res.lse[:, None])
    expect = -res.coef.float()[:, None] * p
    y = torch.from_numpy(big["target"]).cuda().long()[:, None]
    expect = torch.where(cols == y, res.coef.float()[:, None] * -torch.expm1(res.cur_lp.float())[:, None], expect)
    got = res.dlogits.gather(1, cols).float()
    rowmax = res.coef.float().abs()[:, None]
    assert torch.all((got - expect).abs() <= 2 ** -7 * expect.abs() + 1e-5 * rowmax + 1e-30)


def test_sampled_rows_against_oracle(big, oracle):
    res, T, V = big["res"], big["T"], big["V"]
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(T, 48, replace=False))
    z = big["logits"][torch.from_numpy(rows).cuda()].double().cpu().numpy()
    tgt = big["target"][rows]
    ref_cur = oracle.logprob_gather(z, tgt)
    assert_scalar_close(res.cur_lp.cpu().numpy()[rows], ref_cur, what="cur_lp rows")
    # per-row dlogits = coef (onehot - softmax) with the kernel's coef
    coef = res.coef.cpu().numpy()[rows]
    e = np.exp(z - z.max(1, keepdims=True))
    p = e / e.sum(1, keepdims=True)
    ref = -coef[:, None] * p
    others = np.where(np.arange(V)[None, :] == tgt[:, None], 0.0, e).sum(1) / e.sum(1)
    ref[np.arange(len(rows)), tgt] = coef * others
    got = res.dlogits[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    assert_rows_close(got, ref, bf16=True, what="sampled rows")


def test_counts_and_loss_consistent(big):
    res, T = big["res"], big["T"]
    stale = int((big["stage"] < big["hb"].cur_stage).sum())
    assert res.stale_tokens == stale
    flags = res.flags.cpu().numpy()
    assert res.clipped_tokens == int(((flags >> 1) & 1).sum())
    obj = res.obj.cpu().numpy()
    assert abs(res.objective - obj.sum()) <= 1e-9 * max(1.0, np.abs(obj).sum())
    assert res.loss == -res.objective * (1.0 / T)


def test_full_size_determinism_and_chunking(ctx, big):
    from paper_2511_05589_b200 import ClipConfig
    res, T = big["res"], big["T"]
    again = ctx.grpo_step_loss(big["logits"], big["batch"], ClipConfig())
    assert again.loss == res.loss
    assert torch.equal(again.dlogits, res.dlogits)
    outs = ctx.alloc_outputs(T, big["logits"].device)
    dl = torch.empty_like(big["logits"])
    step = 5000
    for a in range(0, T, step):
        b = min(T, a + step)
        ctx.loss_chunk_fused(big["logits"][a:b], big["batch"], ClipConfig(), outs, dlogits=dl[a:b],
                             row_base=a, total_tokens=T)
    ctx.check()
    assert torch.equal(dl, res.dlogits)
    assert torch.equal(outs["obj"], res.obj)


def test_v32000_claimed_rows_against_oracle(ctx, oracle):
    """V = 32,000 (config #5) with 8,192 rows: far more rows than the TMA
    kernel's 444 CTAs, so almost every row is CLAIMED from the per-launch
    counter at run time. Every per-token output and the loss against the CPU
    oracle, dlogits on sampled rows; a rerun (a different row-to-CTA
    assignment) is bitwise identical."""
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import make_host_batch, make_logits, stale_logprobs
    from parity_util import assert_loss_close
    V = 32000
    hb = make_host_batch(3, 16, 8, V, fixed_len=64)
    T = hb.n_tok
    tgt = torch.from_numpy(hb.target).cuda()
    logits = make_logits(T, V, tgt, 3, device="cuda")
    z64 = logits.double().cpu().numpy()
    cur = oracle.logprob_gather(z64, hb.target)
    blp = stale_logprobs(cur, hb.stage, hb.cur_stage, 3)
    adv = oracle.advantages(hb.reward, hb.group_off)
    ref = oracle.is_loss(z64, hb.tok_off, hb.target, hb.stage, hb.cur_stage, blp.astype(np.float64),
                         adv, want_dlogits=False)
    batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, blp, hb.cur_stage, stage=hb.stage,
                   reward=hb.reward)
    res = ctx.grpo_step_loss(logits, batch, ClipConfig(), coef=True)
    assert ctx.last_launch()["kernel"] == "fused_tma_kernel"
    assert_scalar_close(res.cur_lp.cpu().numpy(), ref.cur_lp, what="cur_lp")
    assert_scalar_close(res.obj.cpu().numpy(), ref.obj, what="obj")
    np.testing.assert_array_equal((res.flags.cpu().numpy() >> 1) & 1, ref.clipped)
    assert res.stale_tokens == ref.stale_tokens and res.clipped_tokens == ref.clipped_tokens
    assert_loss_close(res.loss, ref.loss, ref.obj, T)
    rows = np.sort(np.random.default_rng(4).choice(T, 64, replace=False))
    coef = res.coef.cpu().numpy()[rows]
    z = z64[rows]
    e = np.exp(z - z.max(axis=1, keepdims=True))
    p = e / e.sum(axis=1, keepdims=True)
    want = -coef[:, None] * p
    want[np.arange(len(rows)), hb.target[rows]] = coef * (1.0 - p[np.arange(len(rows)), hb.target[rows]])
    got = res.dlogits[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    assert_rows_close(got, want, bf16=True, what="sampled rows",
                      row_atol=(V + 8) * 2.0 ** -52 * np.abs(coef))
    again = ctx.grpo_step_loss(logits, batch, ClipConfig(), coef=True)
    assert torch.equal(again.dlogits.view(torch.int16), res.dlogits.view(torch.int16))
    assert torch.equal(again.obj, res.obj) and again.loss == res.loss
