"""GPU parity: the sm_100a path, called through the C-ABI, against the CPU
oracle (oracle/copris_oracle.c, itself pinned to the reference) on the same
seeded inputs. Tolerances: tests/parity_util.py."""
import math

import numpy as np
import pytest
import torch

from parity_util import Case, assert_loss_close, assert_rows_close, assert_scalar_close, exact_dlogits

pytestmark = pytest.mark.gpu

BF16, F32 = torch.bfloat16, torch.float32


def run(ctx, case, dl_dtype=BF16, fused=True, **kw):
    batch = case.upload(ctx)
    return case, ctx.grpo_step_loss(case.logits_gpu(), batch, case.clip(), is_enabled=case.is_enabled,
                                    behav_mode=case.behav_mode, fused=fused,
                                    dlogits_dtype=dl_dtype, coef=True, **kw)


# (V, logits dtype, forced implementation or None, expected kernel, expected cluster)
PAIR = ("fused_pair_kernel", 2)
QUAD = ("fused_quad_kernel", 4)
SHAPES = [
    # Qwen2.5 vocab: the CTA-pair kernel for bf16 logits, with f16 exponentials
    # (bf16 dlogits) or the raw logits (fp32 dlogits) staged in TMEM
    (151936, BF16, None, (PAIR, PAIR), None),
    (151936, BF16, "pair+pl0", (PAIR, PAIR), None),   # no lookahead: pass 2 right after the row
    (151936, BF16, "pair+pl1", (PAIR, PAIR), None),
    (151936, BF16, "pair+st1", (PAIR, PAIR), None),  # 32-byte stores in pass 2 (lane-pair swap)
    (151936, BF16, "pair+bst0", (PAIR, PAIR), None),  # f16 exponentials in TMEM (round-2 first version)
    (151936, BF16, "pair+bst0+st1", (PAIR, PAIR), None),
    (32000, BF16, "solo+bst0", "fused_solo_kernel", 1),
    (200000, BF16, "pair+st1", (PAIR, PAIR), None),
    (151936, BF16, "pair+pl3+slots3", (PAIR, PAIR), None),  # short ring: producer waits on slots
    (200000, BF16, None, (PAIR, PAIR), None),
    (151952, BF16, "pair+st1", (PAIR, PAIR), None),  # second half not 32-byte aligned: 16-byte stores there         # 7 slots per half-row: the TMEM ring wraps every row
    (80000, BF16, None, (PAIR, PAIR), None),          # 8-warp pair CTAs (2 per SM): 5 slots per half
    (40000, BF16, "pair", (PAIR, PAIR), None),        # 80 KB rows, forced pair (the solo's range)
    (40000, BF16, None, "fused_solo_kernel", 1),      # 80 KB rows: solo by default
    (57344, BF16, None, "fused_solo_kernel", 1),      # largest solo row: 7 slots of 8,192 columns
    (57360, BF16, None, (PAIR, PAIR), None),          # one vector more: the pair kernel
    (114688, BF16, None, (PAIR, PAIR), None),         # largest half row for 8-warp pair CTAs
    (114704, BF16, None, (PAIR, PAIR), None),         # first 16-warp pair width
    (229376, BF16, None, (PAIR, PAIR), None),         # widest pair row: 7 slots per half
    (229392, BF16, None, (QUAD, QUAD), None),         # one vector more: a 4-CTA cluster per row
    (256000, BF16, None, (QUAD, QUAD), None),         # Gemma-size vocabulary
    (458752, BF16, None, (QUAD, QUAD), None),         # widest quad row: 7 slots per quarter
    (458768, BF16, None, "fused_stream_la_kernel", 1),  # wider: the ring kernel (any width)
    (151944, BF16, None, "fused_stream_la_kernel", 1),  # 16-byte rows but V % 16 != 0: the ring kernel
    (151936, BF16, "stream", "fused_stream_la_kernel", 1),  # the ring kernel forced for bf16 too
    (151936, BF16, "stream+la0", "fused_stream_la_kernel", 1),  # same without the lookahead
    (151936, BF16, "stream+la5", "fused_stream_la_kernel", 1),
    (32000, BF16, None, "fused_solo_kernel", 1),      # 64 KB rows: one CTA per row, exponentials in TMEM
    (32000, BF16, "tma", "fused_tma_kernel", 1),      # 64 KB rows resident, several CTAs/SM
    (32000, BF16, "stream", "fused_stream_la_kernel[resident]", 1),  # 3 rows fit the ring: no L2 re-read
    (32000, BF16, "stream+res0", "fused_stream_la_kernel", 1),  # 2 segments/row: lookahead = whole row
    (32000, BF16, "stream+la1+res0", "fused_stream_la_kernel", 1),
    (20000, BF16, "stream", "fused_stream_la_kernel[resident]", 1),  # partial last segment
    (32000, BF16, "stream+la0+res0", "fused_stream_la_kernel", 1),
    (80000, BF16, "tma", "fused_tma_kernel", 1),      # 160 KB rows: one 16-warp CTA per row
    (32000, BF16, "solo", "fused_solo_kernel", 1),    # one CTA per row, exponentials in TMEM
    (32000, BF16, "solo+pl0", "fused_solo_kernel", 1),
    (48000, BF16, "solo", "fused_solo_kernel", 1),    # 6 slots per row (PW 8: 16 KB slots), partial last slot
    (4096, BF16, "solo", "fused_solo_kernel", 1),     # one partial slot per row
    (256, BF16, "solo", "fused_solo_kernel", 1),      # tiny rows
    (151936, F32, None, "fused_stream_la_kernel", 1),
    (151936, F32, "stream+la0", "fused_stream_la_kernel", 1),
    (32000, F32, None, "fused_stream_la_kernel", 1),
    (256, BF16, None, "fused_tma_kernel", 1),
    (4099, BF16, None, "fused_generic_kernel", 1),    # odd vocab: unaligned rows
    (100, F32, None, "fused_generic_kernel", 1),
    (6, F32, None, "fused_generic_kernel", 1),        # desk vocab
]

# the context options every test starts from (copris_ctx_set_option)
DEFAULT_OPTS = dict(fused_impl=0, lookahead=2, resident=1, slots=0, pair_lookahead=3, pair_st256=0,
                    pair_bf16_stage=1)


@pytest.fixture
def impl(ctx):
    def set_impl(name):
        """name = implementation[+laN][+resN]: the context's fused_impl and the
        stream kernel's lookahead (0 = pass 2 right after pass 1) / resident mode."""
        opts = dict(DEFAULT_OPTS)
        if name and "+" in name:
            name, *rest = name.split("+")
            for o in rest:
                if o.startswith("la"):
                    opts["lookahead"] = int(o[2:])
                elif o.startswith("res"):
                    opts["resident"] = int(o[3:])
                elif o.startswith("pl"):
                    opts["pair_lookahead"] = int(o[2:])
                elif o.startswith("slots"):
                    opts["slots"] = int(o[5:])
                elif o.startswith("st"):
                    opts["pair_st256"] = int(o[2:])
                elif o.startswith("bst"):
                    opts["pair_bf16_stage"] = int(o[3:])
        if name:
            opts["fused_impl"] = name
        for k, v in opts.items():
            ctx.set_option(k, v)
    yield set_impl
    for k, v in DEFAULT_OPTS.items():
        ctx.set_option(k, v)


@pytest.mark.parametrize("V,dtype,force,kernel,cluster", SHAPES)
@pytest.mark.parametrize("dl_dtype", [BF16, F32])
def test_fused_matches_oracle(ctx, oracle, impl, V, dtype, force, kernel, cluster, dl_dtype):
    if cluster is None:  # (bf16-dlogits kernel, fp32-dlogits kernel)
        kernel, cluster = kernel[0] if dl_dtype == BF16 else kernel[1]
    impl(force)
    P, G = (2, 4) if V > 50000 else (4, 4)
    case = Case(oracle, seed=V % 97 + 3, P=P, G=G, V=V, dtype=dtype, mu=math.log(10), lmax=24)
    _, res = run(ctx, case, dl_dtype)
    info = ctx.last_launch()
    assert info["kernel"] == kernel and info["cluster"] == cluster, info
    case.check(res, dl_dtype, what=f"V={V} {dtype}->{dl_dtype}")


@pytest.mark.parametrize("V,dtype", [(151936, BF16), (32000, BF16), (4099, BF16), (32000, F32)])
def test_unfused_matches_oracle(ctx, oracle, V, dtype):
    case = Case(oracle, seed=11, P=2, G=4, V=V, dtype=dtype, mu=math.log(10), lmax=24)
    _, res = run(ctx, case, F32, fused=False)
    assert ctx.last_launch()["kernel"] == "bwd_kernel"
    case.check(res, F32, what=f"unfused V={V}")


@pytest.mark.parametrize("V,force", [(151936, None), (151936, "stream+la0"), (80000, "tma"),
                                     (32000, None), (32000, "stream"), (4099, None)])
def test_kl_and_entropy(ctx, oracle, impl, V, force):
    impl(force)
    case = Case(oracle, seed=5, P=2, G=4, V=V, mu=math.log(10), lmax=24, kl_coeff=0.1,
                entropy_coeff=0.01)
    for fused in (True, False):
        _, res = run(ctx, case, F32, fused=fused)
        case.check(res, F32, what=f"kl+entropy V={V} fused={fused} impl={force}")


def test_is_off_every_ratio_is_one(ctx, oracle):
    """trainer.hpp:149 / acceptance C3: with IS off the behaviour IS the
    recomputed log-prob, bit for bit, so every ratio is exactly 1."""
    case = Case(oracle, seed=7, P=2, G=4, V=32000, is_enabled=False, stale_prob=1.0)
    _, res = run(ctx, case, F32)
    cur, beh = res.cur_lp.cpu().numpy(), res.behav.cpu().numpy()
    np.testing.assert_array_equal(cur.view(np.uint32), beh.view(np.uint32))
    assert res.clipped_tokens == 0
    case.check(res, F32, what="IS off")


def test_current_stage_ratio_exactly_one(ctx, oracle):
    """Current-stage tokens take the recomputed log-prob (RECOMPUTED mode),
    stale tokens their buffered one; the select is bit-exact."""
    case = Case(oracle, seed=8, P=4, G=4, V=32000, stages=(2, 4), stale_prob=1.0)
    _, res = run(ctx, case, F32)
    cur, beh = res.cur_lp.cpu().numpy(), res.behav.cpu().numpy()
    stale = case.hb.stage < case.hb.cur_stage
    np.testing.assert_array_equal(beh[~stale].view(np.uint32), cur[~stale].view(np.uint32))
    np.testing.assert_array_equal(beh[stale].view(np.uint32), case.blp[stale].view(np.uint32))
    # weight = ratio * adv = adv exactly for unclipped current tokens
    coef = res.coef.cpu().numpy()
    tok_traj = np.repeat(np.arange(case.hb.n_traj), np.diff(case.hb.tok_off))
    expect = -case.adv[tok_traj] * (1.0 / case.hb.n_tok)
    np.testing.assert_array_equal(coef[~stale], expect[~stale])


def test_recorded_mode(ctx, oracle):
    case = Case(oracle, seed=9, P=2, G=4, V=32000, behav_mode=1)
    _, res = run(ctx, case, F32)
    np.testing.assert_array_equal(res.behav.cpu().numpy().view(np.uint32), case.blp.view(np.uint32))
    case.check(res, F32, what="recorded")


def test_zero_advantages_zero_loss_and_grad(ctx, oracle):
    """test_grpo.cpp:293-303: A=0 -> loss 0 and gradient exactly 0."""
    case = Case(oracle, seed=10, P=2, G=4, V=151936, reward=1.0)
    assert np.all(case.adv == 0.0)
    _, res = run(ctx, case, BF16)
    assert res.loss == 0.0
    assert torch.count_nonzero(res.dlogits).item() == 0


def test_advantages_and_rewards_bit_exact(ctx, oracle):
    from paper_2511_05589_b200.workload import make_host_batch
    hb = make_host_batch(3, 64, 8, 100, mu=math.log(20), sigma=1.0, lmax=64)
    rew = torch.from_numpy(hb.reward).cuda()
    goff = torch.from_numpy(hb.group_off).cuda()
    adv = ctx.compute_advantages(rew, goff, 1e-6).cpu().numpy()
    np.testing.assert_array_equal(adv, oracle.advantages(hb.reward, hb.group_off))
    # terminal rewards (grpo.hpp:35-47) on random EOS placement
    rng = np.random.default_rng(0)
    eos = 99
    toks = hb.target.copy()
    ends = hb.tok_off[1:] - 1
    toks[ends[rng.random(len(ends)) < 0.5]] = eos
    ans = rng.integers(0, 4, hb.n_traj).astype(np.int32)
    toks[hb.tok_off[:-1]] = rng.integers(0, 4, hb.n_traj)
    term = np.ones(hb.n_traj, np.uint8)
    got = ctx.terminal_rewards(torch.from_numpy(toks).cuda(), torch.from_numpy(hb.tok_off).cuda(),
                               torch.from_numpy(term).cuda(), torch.from_numpy(ans).cuda(), eos)
    np.testing.assert_array_equal(got.cpu().numpy(),
                                  oracle.terminal_rewards(toks, hb.tok_off, term, ans, eos))


def test_group_of_one_is_config_error(ctx):
    from paper_2511_05589_b200 import ConfigError
    rew = torch.zeros(3, dtype=torch.float64, device="cuda")
    goff = torch.tensor([0, 2, 3], device="cuda")
    with pytest.raises(ConfigError, match="advantage group size must be >= 2"):
        ctx.compute_advantages(rew, goff)


def test_out_of_vocab_token_is_contract_violation(ctx, oracle):
    from paper_2511_05589_b200 import ContractViolation
    case = Case(oracle, seed=12, P=2, G=4, V=32000)
    batch = case.upload(ctx)
    batch.target[3] = 32000
    with pytest.raises(ContractViolation, match="token out of vocabulary"):
        ctx.grpo_step_loss(case.logits_gpu(), batch, case.clip())
    ctx.check()  # the error word was cleared


def test_nonfinite_buffered_logprob_is_contract_violation(ctx, oracle):
    from paper_2511_05589_b200 import ContractViolation
    case = Case(oracle, seed=13, P=2, G=4, V=32000, stale_prob=1.0)
    batch = case.upload(ctx)
    stale_idx = int(np.flatnonzero(case.hb.stage < case.hb.cur_stage)[0])
    batch.buffered_lp[stale_idx] = float("-inf")
    with pytest.raises(ContractViolation, match="token_ratio requires finite log-probs"):
        ctx.grpo_step_loss(case.logits_gpu(), batch, case.clip())


def test_config_errors(ctx, oracle):
    from paper_2511_05589_b200 import ClipConfig, ConfigError, ContractViolation
    case = Case(oracle, seed=14, P=2, G=4, V=256)
    batch = case.upload(ctx)
    with pytest.raises(ConfigError):
        ctx.grpo_step_loss(case.logits_gpu(), batch, ClipConfig(clip_low=0.0))
    with pytest.raises(ContractViolation, match="reference log-probs required"):
        ctx.grpo_step_loss(case.logits_gpu(), batch, ClipConfig(kl_coeff=0.1))


def test_deterministic_and_chunk_invariant(ctx, oracle):
    """Reruns are bitwise identical (fixed-order reductions, no float atomics)
    and processing the batch in chunks changes nothing."""
    case = Case(oracle, seed=15, P=4, G=4, V=151936, mu=math.log(16), lmax=40)
    batch = case.upload(ctx)
    logits = case.logits_gpu()
    r1 = ctx.grpo_step_loss(logits, batch, case.clip())
    r2 = ctx.grpo_step_loss(logits, batch, case.clip())
    assert r1.loss == r2.loss
    assert torch.equal(r1.dlogits, r2.dlogits)
    # chunked
    T = batch.n_tok
    outs = ctx.alloc_outputs(T, logits.device)
    dl = torch.empty_like(logits)
    for a in range(0, T, 37):
        b = min(T, a + 37)
        ctx.loss_chunk_fused(logits[a:b], batch, case.clip(), outs, dlogits=dl[a:b], row_base=a,
                             total_tokens=T)
    out4 = torch.empty(4, dtype=torch.float64, device="cuda")
    ctx.reduce(outs, T, out4)
    ctx.check()
    assert -out4[0].item() * (1.0 / T) == r1.loss
    assert torch.equal(dl, r1.dlogits)
    assert torch.equal(outs["cur_lp"], r1.cur_lp)
    # the unfused K1 -> K2 -> K3 pipeline, chunked, equals its one-shot run
    u1 = ctx.grpo_step_loss(logits, batch, case.clip(), fused=False)
    outs = ctx.alloc_outputs(T, logits.device)
    for a in range(0, T, 37):
        b = min(T, a + 37)
        ctx.loss_chunk_unfused(logits[a:b], batch, case.clip(), outs, dlogits=dl[a:b], row_base=a,
                               total_tokens=T)
    ctx.reduce(outs, T, out4)
    ctx.check()
    assert -out4[0].item() * (1.0 / T) == u1.loss
    assert torch.equal(dl, u1.dlogits)
    case.check(u1, torch.bfloat16, what="unfused one-shot")


def test_padded_rows(ctx, oracle):
    for ld, kernel in ((32008, "fused_solo_kernel"), (32001, "fused_generic_kernel")):
        case = Case(oracle, seed=16, P=2, G=4, V=32000, ld=ld)
        _, res = run(ctx, case, F32)
        assert ctx.last_launch()["kernel"] == kernel
        case.check(res, F32, what=f"ld={ld}")


@pytest.mark.parametrize("dl_dtype", [F32, BF16])
def test_saturated_rows_one_minus_p(ctx, oracle, dl_dtype):
    """Rows whose target saturates (p_y -> 1) keep 1-p_y accurate (the target
    is excluded from the running sum): checked on every 64th row; bf16
    dlogits run the CTA-pair kernel, where the saturated target also stays out
    of every warp's staging maximum."""
    case = Case(oracle, seed=17, P=4, G=4, V=151936, fixed_len=32)
    _, res = run(ctx, case, dl_dtype)
    sat = np.arange(case.hb.n_tok) % 64 == 0
    assert sat.any()
    dl = res.dlogits.float().cpu().numpy()[sat]
    coef = -case.ref.weight / case.hb.n_tok
    exact = exact_dlogits(case.z64[sat], case.hb.target[sat], coef[sat])
    assert_rows_close(dl, exact, bf16=dl_dtype == BF16, what="saturated rows vs cancellation-free fp64")
    assert_scalar_close(res.cur_lp.cpu().numpy()[sat], case.ref.cur_lp[sat], rtol=1e-6,
                        what="saturated cur_lp")


def test_logprob_gather_k1(ctx, oracle):
    for V, dtype in ((151936, BF16), (4099, F32), (6, F32)):
        case = Case(oracle, seed=18, P=2, G=4, V=V, dtype=dtype)
        lp, lse = ctx.sequence_logprobs(case.logits_gpu(), torch.from_numpy(case.hb.target).cuda())
        ctx.check()
        assert_scalar_close(lp.cpu().numpy(), case.ref.cur_lp, what=f"K1 V={V}")


@pytest.mark.parametrize("n,off", [(100_000, 0), (100_003, 0), (100_003, 1), (3, 0)])
def test_behaviour_concat_k2_bit_exact(ctx, oracle, n, off):
    """16-byte vector path (aligned), its scalar tail (n % 4) and the scalar
    kernel (inputs offset by one element, so not 16-byte aligned)."""
    rng = np.random.default_rng(1)
    stage = rng.integers(0, 6, n + off).astype(np.uint32)
    blp = rng.standard_normal(n + off).astype(np.float32)
    cur = rng.standard_normal(n + off).astype(np.float32)
    d = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda()[off:]
    stage, blp, cur = stage[off:], blp[off:], cur[off:]
    for is_on in (True, False):
        for mode in (0, 1):
            behav, flags = ctx.concat_segments(d(np.concatenate([np.zeros(off, np.uint32), stage])), 5,
                                               d(np.concatenate([np.zeros(off, np.float32), blp])),
                                               d(np.concatenate([np.zeros(off, np.float32), cur])),
                                               is_on, mode)
            ref, n_stale = oracle.behaviour(stage, 5, blp, cur, is_on, mode)
            np.testing.assert_array_equal(behav.cpu().numpy(), ref.astype(np.float32))
            np.testing.assert_array_equal(flags.cpu().numpy(), (stage < 5).astype(np.uint8))
            assert int(flags.sum().item()) == n_stale


@pytest.mark.parametrize("n,off", [(1_000_003, 0), (1_000_003, 1), (5, 0), (4099, 3)])
def test_reduce_vector_and_scalar_paths(ctx, n, off):
    """copris_loss_reduce: vectorized (aligned) and scalar (offset) kernels give
    exact integer counts and the fp64 sum within rounding; reruns are bitwise."""
    rng = np.random.default_rng(2)
    obj = torch.from_numpy(rng.standard_normal(n + off)).cuda()
    flags = torch.from_numpy(rng.integers(0, 8, n + off).astype(np.uint8)).cuda()
    outs = {"obj": obj[off:], "flags": flags[off:]}
    out4 = torch.empty(4, dtype=torch.float64, device="cuda")
    ctx.reduce(outs, n, out4)
    first = out4.clone()
    ctx.reduce(outs, n, out4)
    assert torch.equal(first, out4)
    f = flags[off:].cpu().numpy()
    o = obj[off:].cpu().numpy()
    assert out4[1].item() == n - int(((f >> 2) & 1).sum())
    assert out4[2].item() == int((f & 1).sum())
    assert out4[3].item() == int(((f >> 1) & 1).sum())
    assert abs(out4[0].item() - float(np.sum(o))) <= 1e-12 * max(1.0, float(np.abs(o).sum()))


def test_expand_segments(ctx):
    from paper_2511_05589_b200.workload import make_host_batch
    hb = make_host_batch(4, 8, 4, 100, mu=math.log(30), sigma=1.0, lmax=100, stages=(3, 4),
                         stale_prob=1.0)
    st = ctx.expand_segments(torch.from_numpy(hb.seg_off).cuda(),
                             torch.from_numpy(hb.seg_ver.view(np.int32)).cuda(), hb.n_tok)
    np.testing.assert_array_equal(st.cpu().numpy().view(np.uint32), hb.stage)
    tt = ctx.token_traj(torch.from_numpy(hb.tok_off).cuda(), hb.n_tok).cpu().numpy()
    np.testing.assert_array_equal(tt, np.repeat(np.arange(hb.n_traj), np.diff(hb.tok_off)))


@pytest.mark.parametrize("V,dl_dtype", [(32000, F32), (151936, BF16)])
def test_host_buffer_dropin(ctx, oracle, V, dl_dtype):
    """copris_grpo_step_loss_host: host arrays in (pinned), 3-stream chunked
    pipeline, host loss/counts/dlogits out — same numbers as the oracle (bf16
    dlogits at V = 151,936: the bench's e2e path)."""
    from paper_2511_05589_b200.grpo import HostWorkspace
    case = Case(oracle, seed=19, P=4, G=4, V=V, mu=math.log(20), lmax=64)
    hb = case.hb
    T = hb.n_tok
    ws = HostWorkspace(ctx, chunk_rows=29, vocab=V, max_tokens=T, max_traj=hb.n_traj,
                       dlogits_dtype=dl_dtype)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    logits = case.logits_cpu.pin_memory()
    dl = torch.empty((T, V), dtype=dl_dtype).pin_memory()
    cur = torch.empty(T, dtype=F32).pin_memory()
    out = ws.grpo_step_loss(logits, pin(hb.tok_off), pin(hb.target), pin(hb.stage.view(np.int32)),
                            pin(case.blp), hb.cur_stage, rewards=pin(hb.reward),
                            group_off=pin(hb.group_off), cfg=case.clip(), dlogits=dl, cur_lp=cur)
    ref = case.ref
    assert out["token_count"] == T
    assert out["stale_tokens"] == ref.stale_tokens
    assert out["clipped_tokens"] == ref.clipped_tokens
    assert_scalar_close(cur.numpy(), ref.cur_lp, what="host cur_lp")
    from parity_util import assert_loss_close
    assert_loss_close(out["loss"], ref.loss, ref.obj, T, what="host loss")
    atol = (V + 8) * 2.0 ** -52 * np.abs(ref.weight) / T
    assert_rows_close(dl.float().numpy(), ref.dlogits, bf16=dl_dtype == BF16, what="host dlogits",
                      row_atol=atol)
    # errors keep the reference's semantics
    from paper_2511_05589_b200 import ConfigError
    bad = pin(np.array([0, 1, 3], np.int64))
    with pytest.raises(ConfigError, match="advantage group size must be >= 2"):
        ws.grpo_step_loss(logits[:3], pin(np.array([0, 1, 2, 3], np.int64)), pin(hb.target[:3]),
                          pin(hb.stage[:3].view(np.int32)), pin(case.blp[:3]), hb.cur_stage,
                          rewards=pin(np.zeros(3)), group_off=bad, cfg=case.clip())
    ws.close()


@pytest.mark.parametrize("V,force", [(151936, None), (151936, "stream+la0"), (151936, "stream+la5"),
                                     (32000, None), (32000, "stream")])
def test_forward_only_matches_forward_backward(ctx, oracle, impl, V, force):
    """want_grad=False skips the dlogits pass (the producer drops pass 2 from the
    ring): the forward outputs must be bitwise those of the full call."""
    impl(force)
    case = Case(oracle, seed=21, P=2, G=4, V=V, mu=math.log(10), lmax=24)
    batch = case.upload(ctx)
    full = ctx.grpo_step_loss(case.logits_gpu(), batch, case.clip(), coef=True)
    fwd = ctx.grpo_step_loss(case.logits_gpu(), batch, case.clip(), coef=True, want_grad=False)
    assert fwd.dlogits is None
    assert fwd.loss == full.loss and fwd.clipped_tokens == full.clipped_tokens
    assert torch.equal(fwd.cur_lp, full.cur_lp) and torch.equal(fwd.coef, full.coef)


@pytest.mark.parametrize("rows", [1, 37, 73, 74, 75, 148, 149, 300])
def test_pair_rows_around_the_grid(ctx, oracle, impl, rows):
    """Row counts around the pair kernel's persistent grid (74 CTA pairs): a
    single row, clusters with one row next to clusters with several; all
    against the oracle."""
    impl(None)
    case = Case(oracle, seed=rows, P=1, G=2, V=151936, fixed_len=(rows + 1) // 2)
    _, res = run(ctx, case, BF16)
    assert ctx.last_launch()["kernel"] == "fused_pair_kernel"
    case.check(res, BF16, what=f"rows={case.hb.n_tok}")


@pytest.mark.parametrize("half", [37, 74, 75, 148, 150])
def test_stream_rows_around_the_grid(ctx, oracle, impl, half):
    """Row counts around the persistent grid (148 SMs): 74 .. 300 rows, i.e. CTAs
    with one row (no lookahead row) next to CTAs with two; all against the oracle."""
    impl("stream")
    case = Case(oracle, seed=half, P=1, G=2, V=151936, fixed_len=half)
    _, res = run(ctx, case, F32)
    assert ctx.last_launch()["kernel"] == "fused_stream_la_kernel"
    case.check(res, F32, what=f"rows={case.hb.n_tok}")


@pytest.mark.parametrize("V,force", [(151936, None), (80000, "tma"), (32000, None),
                                     (32000, "stream"), (4099, None)])
@pytest.mark.parametrize("fused", [True, False])
def test_loss_mask_equals_deletion(ctx, oracle, impl, V, force, fused):
    """copris_loss_batch.loss_mask: a masked token is left out of the loss as
    if it were not in the batch. Checked against the oracle run on the batch
    with the masked tokens deleted (advantages come from the rewards, so they
    do not change), with one trajectory masked entirely."""
    impl(force)
    case = Case(oracle, seed=13, P=2, G=4, V=V, mu=math.log(10), lmax=24)
    hb = case.hb
    rng = np.random.default_rng(5)
    keep = rng.random(hb.n_tok) > 0.3
    keep[hb.tok_off[1]:hb.tok_off[2]] = False
    csum = np.concatenate([[0], np.cumsum(keep)])
    tok_off2 = csum[hb.tok_off].astype(np.int64)
    T2 = int(keep.sum())
    ref = oracle.is_loss(case.z64[keep], tok_off2, hb.target[keep], hb.stage[keep], hb.cur_stage,
                         case.blp[keep].astype(np.float64), case.adv, **case.cfg)
    batch = case.upload(ctx)
    batch.loss_mask = torch.from_numpy(keep.astype(np.uint8)).cuda()
    res = ctx.grpo_step_loss(case.logits_gpu(), batch, case.clip(), fused=fused,
                             dlogits_dtype=torch.float32)
    assert res.token_count == T2
    assert res.stale_tokens == ref.stale_tokens and res.clipped_tokens == ref.clipped_tokens
    flags = res.flags.cpu().numpy()
    np.testing.assert_array_equal(flags[~keep], 4)
    np.testing.assert_array_equal(flags[keep] & 1, (hb.stage[keep] < hb.cur_stage).astype(np.uint8))
    np.testing.assert_array_equal((flags[keep] >> 1) & 1, ref.clipped)
    # log-probs are still produced for every token
    assert_scalar_close(res.cur_lp.cpu().numpy(), case.ref.cur_lp, what="masked cur_lp")
    obj = res.obj.cpu().numpy()
    assert np.all(obj[~keep] == 0.0)
    assert_scalar_close(obj[keep], ref.obj, what="masked obj")
    assert_loss_close(res.loss, ref.loss, ref.obj, T2, what="masked loss")
    dl = res.dlogits.cpu().numpy()
    assert np.all(dl[~keep] == 0.0)
    atol = (V + 8) * 2.0 ** -52 * np.abs(ref.weight) / T2
    assert_rows_close(dl[keep], ref.dlogits, what="masked dlogits", row_atol=atol)


@pytest.mark.parametrize("V", [151936, 32000])
def test_cuda_graph_replay_bitwise(ctx, oracle, V):
    """The chunk launches and the reduction are capturable in a CUDA graph (no
    host sync, no allocation inside the C-ABI calls); replaying the graph
    gives bitwise the eager results."""
    case = Case(oracle, seed=17, P=2, G=4, V=V, mu=math.log(10), lmax=24)
    batch = case.upload(ctx)
    logits = case.logits_gpu()
    T = batch.n_tok
    chunk = max(1, T // 3)

    def launches(outs, dl, out4):
        for r0 in range(0, T, chunk):
            n = min(chunk, T - r0)
            ctx.loss_chunk_fused(logits[r0:r0 + n], batch, case.clip(), outs, dlogits=dl[r0:r0 + n],
                                 row_base=r0, total_tokens=T)
        ctx.reduce(outs, T, out4)

    eager = ctx.alloc_outputs(T, logits.device)
    dl_e = torch.empty_like(logits)
    o4_e = torch.empty(4, dtype=torch.float64, device=logits.device)
    launches(eager, dl_e, o4_e)
    ctx.check()

    outs = ctx.alloc_outputs(T, logits.device)
    dl = torch.zeros_like(logits)
    o4 = torch.zeros(4, dtype=torch.float64, device=logits.device)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        launches(outs, dl, o4)
    torch.cuda.current_stream().wait_stream(side)
    with torch.cuda.graph(g):
        launches(outs, dl, o4)
    for _ in range(3):
        dl.zero_()
        o4.zero_()
        g.replay()
    torch.cuda.synchronize()
    ctx.check()
    assert torch.equal(dl.view(torch.int16), dl_e.view(torch.int16))
    assert torch.equal(o4, o4_e)
    for k in ("cur_lp", "obj", "flags"):
        assert torch.equal(outs[k], eager[k]), k
    assert_loss_close(-o4[0].item() / T, case.ref.loss, case.ref.obj, T, what="graph loss")


@pytest.mark.parametrize("V,dtype", [(151936, BF16), (32000, BF16), (4099, BF16), (151936, F32),
                                     (32000, F32), (6, F32)])
def test_k1_equals_loss_recompute_bitwise(ctx, oracle, V, dtype):
    """test_policy.cpp:157-172 on the GPU: the log-probs K1 (sequence_logprobs,
    what a sampler records) returns are bitwise the ones the loss kernel
    recomputes, so a current-stage token's ratio is exactly 1 in either
    behaviour mode; K1 is the fused kernels in gather-only mode."""
    case = Case(oracle, seed=19, P=2, G=4, V=V, dtype=dtype, mu=math.log(10), lmax=24)
    logits = case.logits_gpu()
    lp, lse = ctx.sequence_logprobs(logits, torch.from_numpy(case.hb.target).cuda())
    # bf16 dlogits: the kernel K1 shares its pass 1 with (the pair kernel at
    # V = 151,936 with bf16 logits; fp32 dlogits run the ring kernel there)
    _, res = run(ctx, case, BF16 if dtype == BF16 else F32)
    assert torch.equal(lp.view(torch.int32), res.cur_lp.view(torch.int32))
    assert torch.equal(lse.view(torch.int32), res.lse.view(torch.int32))
    assert_scalar_close(lp.cpu().numpy(), case.ref.cur_lp, what=f"K1 V={V}")


def test_pair_and_ring_kernels_agree(ctx, oracle, impl):
    """At V = 151,936 the CTA-pair kernel and the ring kernel (exponentials
    recomputed from an L2 re-read) split the log-sum-exp differently:
    per-token outputs agree to fp32 rounding, the pair kernel's bf16 dlogits
    (TMEM-staged f16 exponentials) are within one bf16 ulp of the ring
    kernel's fp32 dlogits, its fp32 dlogits (TMEM-staged raw logits) within
    1e-5 of the row's max, and branch decisions are identical."""
    case = Case(oracle, seed=29, P=2, G=8, V=151936, mu=math.log(24), lmax=64)
    _, a = run(ctx, case, BF16)
    assert ctx.last_launch()["kernel"] == "fused_pair_kernel"
    _, a32 = run(ctx, case, F32)
    assert ctx.last_launch()["kernel"] == "fused_pair_kernel"
    impl("stream")
    _, b = run(ctx, case, F32)
    assert ctx.last_launch()["kernel"] == "fused_stream_la_kernel"
    assert_scalar_close(a.cur_lp.cpu().numpy(), b.cur_lp.cpu().numpy(), rtol=2e-6, what="cur_lp")
    assert torch.equal(a.flags, b.flags) and torch.equal(a32.flags, b.flags)
    assert torch.equal(a.cur_lp, a32.cur_lp)  # same pass 1 in both pair modes
    ref = b.dlogits.double().cpu().numpy()
    assert_rows_close(a.dlogits.float().cpu().numpy(), ref, bf16=True, what="pair vs ring dlogits")
    assert_rows_close(a32.dlogits.double().cpu().numpy(), ref, what="pair f32 vs ring f32 dlogits")


@pytest.mark.parametrize("n_tok,masked,force,V,kernel", [
    (2048, False, "tma", 32000, "fused_tma_kernel"), (1000, False, "tma", 32000, "fused_tma_kernel"),
    (4099, True, "tma", 32000, "fused_tma_kernel"), (8192, False, "tma", 32000, "fused_tma_kernel"),
    (8193, False, "tma", 32000, "fused_tma_kernel"),
    (2048, False, None, 32000, "fused_solo_kernel"), (4099, True, None, 32000, "fused_solo_kernel"),
    (8192, False, None, 32000, "fused_solo_kernel"), (8193, False, "solo", 32000, "fused_solo_kernel"),
    (1000, True, None, 151936, "fused_pair_kernel"), (2048, False, None, 151936, "fused_pair_kernel")])
def test_fused_reduction_bitwise(ctx, oracle, impl, n_tok, masked, force, V, kernel):
    """copris_loss_out.out4: a one-chunk step of <= 8,192 tokens is reduced by
    the loss launch's last CTA (ONE launch); larger ones by the separate
    reduction. Either way out4 is bitwise copris_loss_reduce's result (same
    tiles, same fixed order), reruns are bitwise identical, and the loss
    matches the oracle."""
    impl(force)
    case = Case(oracle, seed=n_tok, P=1, G=n_tok // 256 + 1, V=V, fixed_len=256)
    hb = case.hb
    batch = case.upload(ctx)
    n = min(n_tok, hb.n_tok)
    logits = case.logits_gpu()[:n]
    keep = np.random.default_rng(1).random(hb.n_tok) > 0.2
    if masked:
        batch.loss_mask = torch.from_numpy(keep.astype(np.uint8)).cuda()
    outs = ctx.alloc_outputs(hb.n_tok, logits.device)
    dl = torch.empty((n, case.V), dtype=torch.bfloat16, device="cuda")
    T = hb.n_tok
    fused4 = torch.full((4,), -1.0, dtype=torch.float64, device="cuda")
    ctx.loss_chunk_fused(logits, batch, case.clip(), outs, dlogits=dl, total_tokens=T, out4=fused4)
    info = ctx.last_launch()
    assert info["kernel"] == kernel and info["fused_reduce"] == (n <= 8192)
    sep4 = torch.zeros(4, dtype=torch.float64, device="cuda")
    ctx.reduce(outs, n, sep4)
    ctx.check()
    assert torch.equal(fused4, sep4)
    again = torch.zeros(4, dtype=torch.float64, device="cuda")
    ctx.loss_chunk_fused(logits, batch, case.clip(), outs, dlogits=dl, total_tokens=T, out4=again)
    torch.cuda.synchronize()
    assert torch.equal(again, fused4)
    k = keep[:n] if masked else np.ones(n, bool)
    obj = outs["obj"].cpu().numpy()[:n]
    assert int(fused4[1]) == int(k.sum())
    assert abs(fused4[0].item() - obj.sum()) <= 1e-12 * max(1.0, np.abs(obj).sum())
    if n == hb.n_tok and not masked:
        assert_loss_close(-fused4[0].item() / T, case.ref.loss, case.ref.obj, T, what="fused out4")


@pytest.mark.parametrize("V,force,kernel", [(32000, "tma", "fused_tma_kernel"),
                                            (32000, None, "fused_solo_kernel"),
                                            (80000, None, "fused_pair_kernel"),
                                            (151936, None, "fused_pair_kernel"),
                                            (256000, None, "fused_quad_kernel")])
def test_claim_counter_rearmed_across_launch_kinds(ctx, oracle, impl, V, force, kernel):
    """Rows after each CTA's (cluster's) first are CLAIMED from a per-context
    counter that the launch's last CTA rearms (no memset node): the TMA kernel
    and the pair family (solo / pair / quad, whose rank-0 producer publishes the
    cluster's row sequence through DSMEM). K1 (gather-only) and loss launches of
    more rows than resident CTAs, interleaved with the other kernel kind on the
    same context, must each give bitwise what a fresh context with the static
    row stride (pair_dynamic = 0) gives."""
    from paper_2511_05589_b200 import Copris
    impl(force)
    P, G, L = (2, 8, 256) if V <= 32000 else (2, 4, 256)   # 4,096 / 2,048 rows > resident CTAs
    case = Case(oracle, seed=41, P=P, G=G, V=V, fixed_len=L)
    logits = case.logits_gpu()
    tgt = torch.from_numpy(case.hb.target).cuda()
    fresh = Copris(0)
    if force:
        fresh.set_option("fused_impl", force)
    fresh.set_option("pair_dynamic", 0)
    lp0, _ = fresh.sequence_logprobs(logits, tgt)
    _, r0 = run(fresh, case, BF16)
    other = "solo" if force == "tma" else "tma"
    for _ in range(3):
        lp, _ = ctx.sequence_logprobs(logits, tgt)
        _, r = run(ctx, case, BF16)
        assert ctx.last_launch()["kernel"] == kernel
        assert torch.equal(lp, lp0)
        assert torch.equal(r.cur_lp, r0.cur_lp) and torch.equal(r.flags, r0.flags)
        assert torch.equal(r.dlogits.view(torch.int16), r0.dlogits.view(torch.int16))
        assert r.loss == r0.loss
        # the other kind on the same counter in between
        ctx.set_option("fused_impl", other)
        run(ctx, case, BF16)
        ctx.set_option("fused_impl", force or "auto")
    case.check(r0, BF16, what=f"claim counter V={V}")


def _mask_vocab(logits, hb):
    """-inf logits (a masked vocabulary): ~10% of each row's non-target columns,
    row 0 everything but the target (p_y = 1 exactly), row 1 everything but the
    target and one other column."""
    g = torch.Generator().manual_seed(5)
    T, V = logits.shape[0], logits.shape[1]
    m = torch.rand((T, V), generator=g) < 0.1
    m[0, :] = True
    m[1, :] = True
    m[1, (int(hb.target[1]) + 7) % V] = False
    m[torch.arange(T), torch.from_numpy(hb.target).long()] = False
    logits.masked_fill_(m, float("-inf"))


@pytest.mark.parametrize("V,force,kernel", [(151936, None, "fused_pair_kernel"),
                                            (32000, None, "fused_solo_kernel"),
                                            (32000, "tma", "fused_tma_kernel"),
                                            (151936, "stream", "fused_stream_la_kernel")])
@pytest.mark.parametrize("dl_dtype", [BF16, F32])
def test_masked_vocabulary_minus_inf(ctx, oracle, impl, V, force, kernel, dl_dtype):
    """-inf logits: zero probability, zero dlogits, and a row whose only finite
    logit is the target has log-prob exactly 0 (policy.hpp:114-120 with
    exp(-inf) = 0); every kernel, K1 and the unfused path against the oracle.
    (With the entropy term on, the reference's h -= p log p is NaN at p = 0,
    grpo.hpp:172; the kernels take the limit 0 there.)"""
    impl(force)
    case = Case(oracle, seed=43, P=2, G=4, V=V, mu=math.log(10), lmax=24, edit_logits=_mask_vocab)
    _, res = run(ctx, case, dl_dtype)
    assert ctx.last_launch()["kernel"] == kernel
    case.check(res, dl_dtype, what=f"masked vocab V={V} {force}")
    assert res.cur_lp[0].item() == 0.0
    dl = res.dlogits.float()
    inf_cols = torch.isinf(case.logits_gpu().float())
    assert torch.all(dl[inf_cols] == 0)
    # K1 (sequence_logprobs) and the unfused path on the same rows
    lp, lse = ctx.sequence_logprobs(case.logits_gpu(), torch.from_numpy(case.hb.target).cuda())
    assert_scalar_close(lp.cpu().numpy(), case.ref.cur_lp, what="K1 masked vocab")
    assert torch.isfinite(lse).all()
    if force is None:
        _, ru = run(ctx, case, F32, fused=False)
        case.check(ru, F32, what=f"unfused masked vocab V={V}")



def _special_rows(logits, hb):
    """Rows the reference's own KATs single out (test_policy.cpp:52-65): an
    all-equal row (p = 1/V), a row spanning +-300 (LSE stability), a row whose
    target is far below the rest (log-prob ~ -600; the reference takes log(p), so
    its log-prob is only finite while p > 1e-308: no further)."""
    T, V = logits.shape
    y = torch.from_numpy(hb.target).long()
    for r in range(0, T, 5):
        logits[r] = 0.0
    for r in range(1, T, 5):
        logits[r] = torch.linspace(-300.0, 300.0, V)
    for r in range(2, T, 5):
        logits[r, y[r]] = -600.0


@pytest.mark.parametrize("V,force,kernel", [(151936, None, "fused_pair_kernel"),
                                            (32000, None, "fused_solo_kernel"),
                                            (32000, "tma", "fused_tma_kernel"),
                                            (151936, "stream", "fused_stream_la_kernel"),
                                            (4099, None, "fused_generic_kernel")])
def test_empty_trajectories_and_special_rows(ctx, oracle, impl, V, force, kernel):
    """Zero-length trajectories inside groups (they count for the group's
    advantages, grpo.hpp:51-65, and add no token), uniform rows, +-300 rows and
    targets far below the row maximum, through every kernel against the oracle."""
    impl(force)
    case = Case(oracle, seed=47, P=3, G=4, V=V, mu=math.log(8), lmax=16, empty=[1, 4, 5, 10],
                edit_logits=_special_rows)
    assert np.any(np.diff(case.hb.tok_off) == 0)
    for dl_dtype in (BF16, F32):
        _, res = run(ctx, case, dl_dtype)
        assert ctx.last_launch()["kernel"] == kernel
        case.check(res, dl_dtype, what=f"empty trajectories / special rows V={V} {force}")
    uni = np.arange(0, case.hb.n_tok, 5)
    assert_scalar_close(res.cur_lp.cpu().numpy()[uni], np.full(len(uni), -math.log(V)), rtol=2e-6,
                        what="uniform rows: -log V")



def _far_off_policy(blp, cur, hb):
    """Stale tokens whose behaviour log-prob is 120 below / above the current
    one: ratios e^120 and e^-120 (fp32 exp overflows at e^88)."""
    stale = np.nonzero(hb.stage < hb.cur_stage)[0]
    blp[stale[0::4]] = cur[stale[0::4]] - 120.0
    blp[stale[1::4]] = cur[stale[1::4]] + 120.0


def test_far_off_policy_ratios(ctx, oracle, impl):
    """Ratios e^+-120 (grpo.hpp:71 takes exp in fp64): the objective, the fp64
    coefficient and the loss match the reference's; positive advantages take
    the clipped branch (zero gradient), negative ones the unclipped branch with
    |w| ~ e^120 (beyond any f32/bf16 dlogits, whose rows are not compared)."""
    impl(None)
    case = Case(oracle, seed=53, P=2, G=4, V=151936, mu=math.log(12), lmax=24, stale_prob=1.0,
                edit_blp=_far_off_policy)
    _, res = run(ctx, case, F32)
    ref = case.ref
    assert_scalar_close(res.obj.cpu().numpy(), ref.obj, what="obj")
    np.testing.assert_array_equal((res.flags.cpu().numpy() >> 1) & 1, ref.clipped)
    coef = res.coef.cpu().numpy()
    want = -ref.weight / case.hb.n_tok
    assert_scalar_close(coef, want, what="coef")
    assert np.isfinite(res.loss) and np.isfinite(ref.loss)
    assert_loss_close(res.loss, ref.loss, ref.obj, case.hb.n_tok, what="far off-policy loss")
    assert np.abs(coef).max() > 1e40  # the e^120 rows are there



@pytest.mark.parametrize("V,force,kernel,targets", [
    # pair: half boundary at column 75,968 (nvec0 = 9,496 vectors), slots of 16,384 columns
    (151936, None, "fused_pair_kernel", [0, 1, 7, 8, 16383, 16384, 75959, 75967, 75968, 75969,
                                         75968 + 16383, 75968 + 16384, 151935, 151934]),
    (151952, None, "fused_pair_kernel", [0, 75975, 75976, 75977, 151951]),  # odd nvec0
    (32000, None, "fused_solo_kernel", [0, 1, 16383, 16384, 31999, 31998]),
    (32000, "tma", "fused_tma_kernel", [0, 1, 16383, 16384, 31999]),
    # quad: quarters of 8,000 vectors (64,000 columns)
    (256000, None, "fused_quad_kernel", [0, 63999, 64000, 64001, 127999, 128000, 191999, 192000,
                                         192000 + 16384, 255999]),
])
@pytest.mark.parametrize("dl_dtype", [BF16, F32])
def test_target_at_vector_slot_and_half_boundaries(ctx, oracle, impl, V, force, kernel, targets,
                                                   dl_dtype):
    """Target columns on every boundary the kernels split rows at (16-byte
    vector, ring slot, CTA-pair half, last column): the target is kept out of
    the running sums by the thread that owns it, and its one-hot term is
    written by that thread — against the oracle, bf16 and f32 dlogits."""
    impl(force)
    case = Case(oracle, seed=59, P=2, G=4, V=V, mu=math.log(10), lmax=24, targets=targets)
    _, res = run(ctx, case, dl_dtype)
    assert ctx.last_launch()["kernel"] == kernel
    case.check(res, dl_dtype, what=f"boundary targets V={V} {force}")


@pytest.mark.parametrize("V,kernel", [(151936, "fused_pair_kernel"), (32000, "fused_solo_kernel")])
@pytest.mark.parametrize("mode", ["kl", "is_off", "recorded", "kl_recorded"])
def test_pair_and_solo_token_math_modes(ctx, oracle, impl, V, kernel, mode):
    """The default kernels at both vocabularies in every token-math mode they
    take: KL against the
    version-0 snapshot's log-probs (grpo.hpp:158-162), IS off (trainer.hpp:149),
    recorded behaviour (concat_segments verbatim), KL with recorded behaviour."""
    impl(None)
    kw = dict(kl_coeff=0.1 if mode.startswith("kl") else 0.0, is_enabled=mode != "is_off",
              behav_mode=1 if mode.endswith("recorded") else 0)
    case = Case(oracle, seed=61, P=2, G=4, V=V, mu=math.log(12), lmax=24, **kw)
    for dl_dtype in (BF16, F32):
        _, res = run(ctx, case, dl_dtype)
        assert ctx.last_launch()["kernel"] == kernel
        case.check(res, dl_dtype, what=f"{mode} V={V}")


@pytest.mark.parametrize("V,kernel,cluster", [(32000, "fused_solo_kernel", 1),
                                              (80000, "fused_pair_kernel", 2),
                                              (151936, "fused_pair_kernel", 2),
                                              (256000, "fused_quad_kernel", 4)])
def test_entropy_on_pair_family(ctx, oracle, impl, V, kernel, cluster):
    """The entropy bonus (grpo.hpp:168-181) in the solo / pair / quad kernels:
    raw logits staged in TMEM, u = sum e (z - m) exchanged with each warp's
    (m, s) partial, pass 2 through row_grad's p (log p + H) term; with KL on
    too, bf16 and fp32 dlogits, against the oracle."""
    impl(None)
    P, G = (2, 4) if V > 50000 else (4, 4)
    case = Case(oracle, seed=V % 89 + 7, P=P, G=G, V=V, mu=math.log(12), lmax=24, kl_coeff=0.1,
                entropy_coeff=0.01)
    for dl_dtype in (BF16, F32):
        _, res = run(ctx, case, dl_dtype)
        info = ctx.last_launch()
        assert info["kernel"] == kernel and info["cluster"] == cluster, info
        case.check(res, dl_dtype, what=f"entropy V={V} {dl_dtype}")
    # forward only (no dlogits): the same objective
    _, rf = run(ctx, case, BF16, want_grad=False)
    assert ctx.last_launch()["kernel"] == kernel and rf.dlogits is None
    assert_loss_close(rf.loss, case.ref.loss, case.ref.obj, case.hb.n_tok, what=f"entropy fwd V={V}")


@pytest.mark.parametrize("V,kernel", [(151936, "fused_pair_kernel"), (32000, "fused_solo_kernel")])
def test_entropy_masked_vocabulary_pair_vs_stream(ctx, oracle, impl, V, kernel):
    """-inf logits with the entropy term on: the reference's h -= p log p is NaN
    at p = 0 (grpo.hpp:172), the kernels take the limit 0 there. The pair-family
    kernel against the streaming kernel (the same limit, its entropy arithmetic
    pinned to the oracle on finite rows): finite, and equal within fp32 rounding."""
    case = Case(oracle, seed=43, P=2, G=4, V=V, mu=math.log(10), lmax=24, edit_logits=_mask_vocab,
                entropy_coeff=0.01)
    out = {}
    for force, kern in ((None, kernel), ("stream", "fused_stream_la_kernel")):
        impl(force)
        _, res = run(ctx, case, F32)
        assert ctx.last_launch()["kernel"].startswith(kern)
        out[kern] = res
    a, b = out[kernel], out["fused_stream_la_kernel"]
    for r in (a, b):
        assert math.isfinite(r.loss) and torch.isfinite(r.dlogits).all() and torch.isfinite(r.obj).all()
    np.testing.assert_allclose(a.cur_lp.cpu().numpy(), b.cur_lp.cpu().numpy(), rtol=0, atol=2e-5)
    np.testing.assert_allclose(a.obj.cpu().numpy(), b.obj.cpu().numpy(), rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(a.dlogits.cpu().numpy(), b.dlogits.cpu().numpy(), rtol=1e-4, atol=1e-9)
    inf_cols = torch.isinf(case.logits_gpu().float())
    assert torch.all(a.dlogits[inf_cols] == 0)
