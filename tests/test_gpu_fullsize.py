"""GPU: full-size parity at BASELINE config #2, #3 and #4 shapes.

  * configs #2 (128 x 8, sigma 1, 2 stages) and #3 (sigma 1.5, 3-4 stages),
    V = 151,936: whole prompt groups of the config batch (~24k rows): EVERY
    row's cur_lp, behaviour log-prob, objective term, coef and flags against
    the CPU oracle (oracle_per_token, host threads), the loss, and dlogits on
    sampled rows rebuilt from the ORACLE's coefficients; plus size-independent
    properties over all rows (dlogits rows sum to zero, the target entry is
    coef (1 - p_y), off-target entries -coef p_k on sampled columns);
  * config #4 (512 x 16, sharded by prompt group): whole groups LPT-sharded
    over 2 and 4 ranks (one context per rank on this GPU, T_global passed to
    every rank, the four scalars summed): per-token outputs and dlogits
    bitwise those of the unsharded run, loss and counts equal to the oracle;
  * bit-identical reruns and chunk-size invariance at full size.
"""

import numpy as np
import pytest
import torch

from parity_util import assert_rows_close, assert_scalar_close

pytestmark = pytest.mark.gpu


def assert_rel_close(gpu, ref, rtol=1e-5, atol=1e-300, what=""):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(gpu - ref) - (rtol * np.abs(ref) + atol)
    assert np.all(err <= 0), f"{what}: {int((err > 0).sum())} out of tolerance, worst excess {err.max():.3e}"


@pytest.fixture(scope="module", params=["grpo_128x8_v151936", "grpo_128x8_v151936_longtail_4stage"])
def big(ctx, request):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import CONFIGS, make_host_batch, make_logits, stale_logprobs
    cfg = dict(CONFIGS[request.param])
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
    assert ctx.last_launch()["kernel"] == "fused_pair_kernel"
    return dict(hb=hb, T=T, V=V, logits=logits, batch=batch, res=res, target=target, stage=stage,
                blp=blp, tok_off=tok_off, group_off=group_off, n_traj=n_traj, name=request.param)


@pytest.fixture(scope="module")
def big_oracle(big, oracle):
    """The oracle's per-token outputs over every row of `big` (host threads)."""
    from parity_util import oracle_per_token
    adv = oracle.advantages(big["hb"].reward[:big["n_traj"]], big["group_off"])
    return oracle_per_token(oracle, big["logits"].cpu(), big["tok_off"], big["target"], big["stage"],
                            big["hb"].cur_stage, big["blp"], adv)


def test_all_rows_against_oracle(big, big_oracle):
    """every row at the config's shape against the oracle, not
    against the kernel's own intermediates."""
    from parity_util import assert_loss_close
    res, T, ref = big["res"], big["T"], big_oracle
    what = big["name"]
    assert_scalar_close(res.cur_lp.cpu().numpy(), ref["cur_lp"], what=f"{what} cur_lp")
    assert_scalar_close(res.behav.cpu().numpy(), ref["behav"], what=f"{what} behav")
    assert_scalar_close(res.obj.cpu().numpy(), ref["obj"], what=f"{what} obj")
    # coef = -w / T (policy.hpp:188 with scale -inv_t): relative, it is ~1/T
    assert_rel_close(res.coef.cpu().numpy(), -ref["weight"] / T, rtol=1e-5, what=f"{what} coef")
    flags = res.flags.cpu().numpy()
    np.testing.assert_array_equal(flags & 1, (big["stage"] < big["hb"].cur_stage).astype(np.uint8))
    np.testing.assert_array_equal((flags >> 1) & 1, ref["clipped"])
    assert res.clipped_tokens == int(ref["clipped"].sum())
    assert_loss_close(res.loss, -ref["obj"].sum() / T, ref["obj"], T, what=f"{what} loss")


def test_rows_sum_to_zero_and_target_entry(big):
    res, T, V = big["res"], big["T"], big["V"]
    dl = res.dlogits.float()
    coef = res.coef.float()
    rs = dl.sum(dim=1)
    # exact rows sum to zero (sum_k coef (1[k=y] - p_k) = 0); each bf16 entry is
    # within one ulp (2^-7 relative at most) of its exact value, so the sum of
    # the rounded entries is within 2^-7 sum_k |d_k| of zero
    tol = 2.0 ** -7 * dl.abs().sum(dim=1)
    assert torch.all(rs.abs() <= tol + 1e-30), float((rs.abs() / (tol + 1e-30)).max())
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


def test_sampled_rows_against_oracle(big, big_oracle, oracle):
    res, T, V = big["res"], big["T"], big["V"]
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(T, 48, replace=False))
    # rows with a nonzero coefficient first: those carry a softmax to check
    w = big_oracle["weight"]
    live = np.flatnonzero(w != 0.0)
    rows = np.sort(np.unique(np.concatenate([rows[:16], rng.choice(live, min(32, len(live)), replace=False)])))
    z = big["logits"][torch.from_numpy(rows).cuda()].double().cpu().numpy()
    tgt = big["target"][rows]
    ref_cur = oracle.logprob_gather(z, tgt)
    assert_scalar_close(res.cur_lp.cpu().numpy()[rows], ref_cur, what="cur_lp rows")
    # per-row dlogits = coef (onehot - softmax) with the ORACLE's coef -w/T
    coef = -w[rows] / T
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
    with ctx.options(fused_impl="tma"):
        _claimed_rows_checks(ctx, logits, batch, ref, hb, T, z64, V)


def _claimed_rows_checks(ctx, logits, batch, ref, hb, T, z64, V):
    from paper_2511_05589_b200 import ClipConfig
    from parity_util import assert_loss_close
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


def test_config4_sharded_equals_unsharded(ctx, oracle):
    """BASELINE config #4 (512 x 16, max 16k tokens, sharded by prompt group)
    on this GPU: whole groups of the config's batch, LPT-sharded over 2 and 4
    ranks, one context per rank, T_global passed to each, the four scalars
    summed (the allreduce). Rows are independent and every rank scales by the
    global T, so each shard's per-token outputs and dlogits are bitwise the
    unsharded run's; the loss and counts equal the oracle's over all rows."""
    from paper_2511_05589_b200 import ClipConfig, Copris
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.sharding import loss_from_scalars, lpt_shard, shard_arrays
    from paper_2511_05589_b200.workload import CONFIGS, make_host_batch, make_logits, stale_logprobs
    from parity_util import assert_loss_close, oracle_per_token
    cfg = dict(CONFIGS["grpo_512x16_v151936"])
    P, G, V = cfg.pop("P"), cfg.pop("G"), cfg.pop("vocab")
    cfg.pop("strong")
    cfg["mu"], cfg["lmax"] = np.log(512.0), 2048  # the config's shape law, lengths scaled to test size
    hb = make_host_batch(4, 8, G, V, **cfg)       # 8 prompt groups x 16 responses
    T = hb.n_tok
    tgt = torch.from_numpy(hb.target).cuda()
    logits = make_logits(T, V, tgt, 4, device="cuda")
    cur, _ = ctx.sequence_logprobs(logits, tgt)
    blp = stale_logprobs(cur.cpu().numpy(), hb.stage, hb.cur_stage, 4)
    whole = upload(ctx, hb.tok_off, hb.group_off, hb.target, blp, hb.cur_stage, stage=hb.stage,
                   reward=hb.reward)
    full = ctx.grpo_step_loss(logits, whole, ClipConfig(), coef=True)
    adv = oracle.advantages(hb.reward, hb.group_off)
    ref = oracle_per_token(oracle, logits.cpu(), hb.tok_off, hb.target, hb.stage, hb.cur_stage, blp, adv)
    assert_loss_close(full.loss, -ref["obj"].sum() / T, ref["obj"], T, what="config #4 unsharded")
    assert full.clipped_tokens == int(ref["clipped"].sum())
    for world in (2, 4):
        shards = lpt_shard(hb.group_tokens(), world)
        total = torch.zeros(4, dtype=torch.float64)
        for rank in range(world):
            rctx = Copris(0)  # one context per rank
            t_off, g_off, pt, pj, idx = shard_arrays(
                hb.tok_off, hb.group_off, {"target": hb.target, "stage": hb.stage, "blp": blp},
                {"reward": hb.reward}, shards[rank])
            n = len(idx)
            b = upload(rctx, t_off, g_off, pt["target"], pt["blp"], hb.cur_stage, stage=pt["stage"],
                       reward=pj["reward"])
            gi = torch.from_numpy(idx).cuda()
            part = rctx.grpo_step_loss(logits[gi], b, ClipConfig(), coef=True, total_tokens=T)
            assert torch.equal(part.cur_lp, full.cur_lp[gi])
            assert torch.equal(part.obj, full.obj[gi]) and torch.equal(part.coef, full.coef[gi])
            assert torch.equal(part.flags, full.flags[gi])
            assert torch.equal(part.dlogits.view(torch.int16), full.dlogits[gi].view(torch.int16))
            total += torch.tensor([part.objective, part.token_count, part.stale_tokens,
                                   part.clipped_tokens], dtype=torch.float64)
            rctx.close()
        assert int(total[1]) == T and int(total[3]) == full.clipped_tokens
        assert int(total[2]) == full.stale_tokens
        assert_loss_close(loss_from_scalars(total, T), -ref["obj"].sum() / T, ref["obj"], T,
                          what=f"config #4 over {world} ranks")
