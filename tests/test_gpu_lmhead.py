"""GPU: LM-head forward on tcgen05 with fused log-softmax partials
 and the loss path behind it.

Parity is split at the bf16 logits the GEMM stores:
  * GEMM: stored logits vs the fp64 product of the same bf16 inputs, within
    bf16 rounding + fp32-accumulation error (|err| <= 2^-8 |z| + H 2^-23 sum|x w|);
  * statistics: (cur_lp, lse) from the partials vs K1 (sequence_logprobs) on the
    stored logits, and the whole loss path vs the CPU oracle on the stored logits
    (the usual 1e-5 relative bar);
  * backward: dhidden / dweight vs fp64 products of the kernel's own dlogits.
"""
import numpy as np
import pytest
import torch

from parity_util import assert_loss_close, assert_scalar_close

pytestmark = pytest.mark.gpu


LM_DEFAULTS = dict(lmhead_impl=0, lmhead_tma_store=1, gemm_wide=1, gemm_mc=0, gemm_splits=0,
                   dw_kchunk=8192)


@pytest.fixture(params=["pair", "1sm"], autouse=True)
def impl(request, ctx):
    """Both kernels: the CTA-pair (cta_group::2) default and the 1-SM variant
    (the context's lmhead_impl option); every option is reset afterwards."""
    ctx.set_option("lmhead_impl", request.param)
    yield request.param
    for k, v in LM_DEFAULTS.items():
        ctx.set_option(k, v)


def _inputs(T, H, V, seed, scale=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = (torch.randn(T, H, generator=g) * scale).to(torch.bfloat16)
    w = (torch.randn(V, H, generator=g) / H ** 0.5 * 2.0).to(torch.bfloat16)
    tgt = torch.randint(0, V, (T,), generator=g, dtype=torch.int32)
    return x.cuda(), w.cuda(), tgt.cuda()


def _check_logits(lg, x, w):
    ref = x.double() @ w.double().t()
    bound = (x.double().abs() @ w.double().abs().t()) * x.shape[1] * 2.0 ** -23
    err = (lg.double() - ref).abs()
    assert torch.all(err <= 2.0 ** -8 * ref.abs() + bound + 1e-30), float((err - 2.0 ** -8 * ref.abs() - bound).max())


@pytest.mark.parametrize("T,H,V", [(1, 64, 256), (64, 64, 100), (130, 64, 300), (257, 192, 1000), (300, 520, 4099),
                                   (512, 1024, 32000), (129, 4096, 151936)])
def test_lmhead_logits_and_partials(ctx, impl, T, H, V):
    x, w, tgt = _inputs(T, H, V, T + H + V)
    lg, part = ctx.lmhead_logits(x, w, tgt)
    pair = "lmhead_fwd_pair_kernel<tma_store>" if V % 8 == 0 else "lmhead_fwd_pair_kernel"
    assert ctx.last_launch()["kernel"] == (pair if impl == "pair" else "lmhead_fwd_kernel")
    torch.cuda.synchronize()
    rows = torch.arange(T, device="cuda") if T * V <= 2 ** 26 else torch.randperm(T, device="cuda")[:32]
    _check_logits(lg[rows], x[rows], w)
    lp, lse = ctx.lse_merge(part, lg, tgt)
    ref_lp, ref_lse = ctx.sequence_logprobs(lg, tgt)
    ctx.check()
    assert_scalar_close(lp.cpu().numpy(), ref_lp.cpu().numpy(), what="cur_lp (partials vs K1)")
    assert_scalar_close(lse.cpu().numpy(), ref_lse.cpu().numpy(), what="lse (partials vs K1)")


def test_lmhead_saturated_rows(ctx):
    """A dominant target logit (p_y -> 1): cur_lp stays accurate (target excluded from sums)."""
    T, H, V = 64, 128, 2048
    x, w, tgt = _inputs(T, H, V, 5)
    w = w.clone()
    x = x.clone()
    # row r points along the target's weight row, scaled so z_y - max_other ~ 20..40
    wy = w[tgt.long()].float()
    x = (wy / wy.norm(dim=1, keepdim=True) * torch.linspace(8, 16, T, device="cuda")[:, None] *
         (H ** 0.5) / 2.0).to(torch.bfloat16)
    lg, part = ctx.lmhead_logits(x, w, tgt)
    lp, lse = ctx.lse_merge(part, lg, tgt)
    ref_lp, _ = ctx.sequence_logprobs(lg, tgt)
    ctx.check()
    assert float(lp.abs().max()) < 1e-3
    assert_scalar_close(lp.cpu().numpy(), ref_lp.cpu().numpy(), what="saturated cur_lp")


@pytest.mark.parametrize("chunk", [4096, 100])
@pytest.mark.parametrize("dhidden_impl,dweight_impl,loss_impl,fwd_impl", [
    ("cublas", "cublas", "lse", "tcgen05"), ("tcgen05", "tcgen05", "lse", "tcgen05"),
    ("cublas", "cublas", "fused", "tcgen05"), ("tcgen05", "tcgen05", "fused", "tcgen05"),
    ("cublas", "cublas", "fused", "cublas"), ("tcgen05", "tcgen05", "fused", "cublas")])
def test_lmhead_loss_path_against_oracle(ctx, oracle, chunk, dhidden_impl, dweight_impl, loss_impl,
                                         fwd_impl, impl):
    """The LM-head step against the oracle on the logits the step computed.
    loss_impl "fused": the forward stores logits only and the one-pass fused
    loss kernel runs on them (the CTA-pair tcgen05 forward's TMA-store epilogue
    has the logits-only mode; the 1-SM forward runs the "lse" path only);
    fwd_impl "cublas": a plain library GEMM forward (the step's default)."""
    if loss_impl == "fused" and fwd_impl == "tcgen05" and impl == "1sm":
        with pytest.raises(Exception, match="logits-only"):
            _lmhead_oracle_case(ctx, oracle, chunk, dhidden_impl, dweight_impl, loss_impl, fwd_impl)
        return
    _lmhead_oracle_case(ctx, oracle, chunk, dhidden_impl, dweight_impl, loss_impl, fwd_impl)


def _lmhead_oracle_case(ctx, oracle, chunk, dhidden_impl, dweight_impl, loss_impl, fwd_impl):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.lmhead import lmhead_grpo_step_loss
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import stale_logprobs
    rng = np.random.default_rng(3)
    n_traj, G = 8, 4
    lens = rng.integers(5, 60, n_traj)
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(tok_off[-1])
    H, V = 256, 1000
    x, w, tgt = _inputs(T, H, V, 11)
    target = tgt.cpu().numpy()
    stage = np.zeros(T, np.uint32)
    for i in range(n_traj):
        a, b = tok_off[i], tok_off[i + 1]
        stage[a:a + (b - a) // 2] = 1 if i % 2 else 2
        stage[a + (b - a) // 2:b] = 2
    if fwd_impl == "cublas":
        # the step's own chunking, so the library GEMM picks the same kernels
        lg_full = torch.cat([torch.mm(x[a:a + chunk], w.t()) for a in range(0, T, chunk)])
    else:
        lg_full, _ = ctx.lmhead_logits(x, w, tgt)
    cur, _ = ctx.sequence_logprobs(lg_full, tgt)
    blp = stale_logprobs(cur.cpu().numpy(), stage, 2, 7)
    reward = (rng.random(n_traj) < 0.5).astype(np.float64)
    group_off = np.arange(0, n_traj + 1, G, dtype=np.int64)
    batch = upload(ctx, tok_off, group_off, target, blp, 2, stage=stage, reward=reward)
    res = lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=chunk, coef=True,
                                dhidden_impl=dhidden_impl, dweight_impl=dweight_impl,
                                loss_impl=loss_impl, fwd_impl=fwd_impl)
    z = lg_full.double().cpu().numpy()
    adv = batch.adv.cpu().numpy()
    ref = oracle.is_loss(z, tok_off, target, stage, 2, blp.astype(np.float64), adv)
    assert res.stale_tokens == ref.stale_tokens
    assert_scalar_close(res.cur_lp.cpu().numpy(), ref.cur_lp, what="cur_lp")
    np.testing.assert_array_equal((res.flags.cpu().numpy() >> 1) & 1, ref.clipped)
    assert_loss_close(res.loss, ref.loss, ref.obj, T)
    # backward: dlogits (oracle, fp64) -> dhidden, dweight
    dl = torch.from_numpy(ref.dlogits)
    xd, wd = x.double().cpu(), w.double().cpu()
    dh_ref = dl @ wd
    dw_ref = dl.t() @ xd
    # the kernel's dlogits are bf16 (2^-9 relative) and the GEMMs accumulate in fp32
    tol_h = 2.0 ** -7 * (dl.abs() @ wd.abs()) + 1e-12
    tol_w = 2.0 ** -7 * (dl.abs().t() @ xd.abs()) + 1e-12
    assert torch.all((res.dhidden.double().cpu() - dh_ref).abs() <= tol_h)
    assert torch.all((res.dweight.double().cpu() - dw_ref).abs() <= tol_w)


def test_lmhead_matches_logits_path(ctx):
    """Same batch through (a) lmhead path and (b) grpo_step_loss on the stored
    logits: identical objective terms within fp32 rounding, dlogits within bf16."""
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.lmhead import lmhead_grpo_step_loss
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import stale_logprobs
    T, H, V = 2000, 512, 32000
    x, w, tgt = _inputs(T, H, V, 2)
    tok_off = np.linspace(0, T, 17).astype(np.int64)
    group_off = np.arange(0, 17, 4, dtype=np.int64)
    stage = (np.arange(T) % 3 == 0).astype(np.uint32) + 1
    lg, _ = ctx.lmhead_logits(x, w, tgt)
    cur, _ = ctx.sequence_logprobs(lg, tgt)
    blp = stale_logprobs(cur.cpu().numpy(), stage, 2, 3)
    reward = (np.arange(16) % 3 == 0).astype(np.float64)
    batch = upload(ctx, tok_off, group_off, tgt.cpu().numpy(), blp, 2, stage=stage, reward=reward)
    a = lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=777, loss_impl="lse",
                              fwd_impl="tcgen05")
    b = ctx.grpo_step_loss(lg.contiguous(), batch, ClipConfig())
    assert a.stale_tokens == b.stale_tokens and a.clipped_tokens == b.clipped_tokens
    assert abs(a.loss - b.loss) <= 1e-6 * max(1e-12, float(b.obj.abs().sum()) / T)
    dh = b.dlogits.float() @ w.float()
    assert torch.allclose(a.dhidden.float(), dh, rtol=2e-2, atol=1e-3 * float(dh.abs().max()))


def test_lmhead_loss_mask_equals_deletion(ctx, oracle):
    """A token mask on the LM-head path divides by the UNMASKED count (the
    masked token mean, as grpo_step_loss does): the result equals the oracle
    run on the batch with the masked tokens deleted (lmhead.py:80)."""
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.lmhead import lmhead_grpo_step_loss
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import stale_logprobs
    from parity_util import assert_loss_close
    T, H, V = 600, 256, 4096
    x, w, tgt = _inputs(T, H, V, 31)
    tok_off = np.linspace(0, T, 9).astype(np.int64)
    group_off = np.arange(0, 9, 4, dtype=np.int64)
    stage = (np.arange(T) % 3 == 0).astype(np.uint32) + 1
    lg, _ = ctx.lmhead_logits(x, w, tgt)
    z64 = lg.double().cpu().numpy()
    cur = oracle.logprob_gather(z64, tgt.cpu().numpy())
    blp = stale_logprobs(cur, stage, 2, 7)
    reward = (np.arange(8) % 3 == 0).astype(np.float64)
    batch = upload(ctx, tok_off, group_off, tgt.cpu().numpy(), blp, 2, stage=stage, reward=reward)
    keep = np.random.default_rng(3).random(T) > 0.35
    batch.loss_mask = torch.from_numpy(keep.astype(np.uint8)).cuda()
    res = lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=250, loss_impl="lse",
                                fwd_impl="tcgen05")
    csum = np.concatenate([[0], np.cumsum(keep)])
    adv = oracle.advantages(reward, group_off)
    ref = oracle.is_loss(z64[keep], csum[tok_off].astype(np.int64), tgt.cpu().numpy()[keep],
                         stage[keep], 2, blp[keep].astype(np.float64), adv, want_dlogits=False)
    assert res.token_count == int(keep.sum())
    assert res.clipped_tokens == ref.clipped_tokens and res.stale_tokens == ref.stale_tokens
    assert_loss_close(res.loss, ref.loss, ref.obj, int(keep.sum()), what="lmhead masked loss")
    # and the same batch through the logits path gives the same masked mean
    b = ctx.grpo_step_loss(lg.contiguous(), batch, ClipConfig())
    assert abs(res.loss - b.loss) <= 1e-6 * max(1e-12, float(b.obj.abs().sum()) / keep.sum())


def test_lmhead_argument_errors(ctx):
    """C-ABI validation: misaligned strides/pointers, short ld, partial-width mismatch."""
    from paper_2511_05589_b200.grpo import _p
    T, H, V = 16, 64, 300
    x, w, tgt = _inputs(T, H, V, 1)
    lib = ctx.lib
    lg = torch.empty((T, 304), dtype=torch.bfloat16, device="cuda")
    part = torch.empty((T, 2, 2), dtype=torch.float32, device="cuda")
    s = ctx._stream()
    ok = lib.copris_lmhead_logits(ctx.h, _p(x), H, _p(w), H, T, H, V, _p(tgt), _p(lg), 304, _p(part), s)
    assert ok == 0
    assert lib.copris_lmhead_logits(ctx.h, _p(x), H, _p(w), H, T, H, V, _p(tgt), _p(lg), 300,
                                    _p(part), s) != 0  # ld_logits % 8
    assert b"ld_logits" in lib.copris_last_error()
    assert lib.copris_lmhead_logits(ctx.h, _p(x), 60, _p(w), H, T, H, V, _p(tgt), _p(lg), 304,
                                    _p(part), s) != 0  # ld_hidden < hidden_dim
    xo = torch.empty(T * H + 8, dtype=torch.bfloat16, device="cuda")[1:1 + T * H]
    assert lib.copris_lmhead_logits(ctx.h, _p(xo), H, _p(w), H, T, H, V, _p(tgt), _p(lg), 304,
                                    _p(part), s) != 0  # misaligned hidden
    assert b"aligned" in lib.copris_last_error()
    lp = torch.empty(T, dtype=torch.float32, device="cuda")
    assert lib.copris_lse_merge(ctx.h, _p(part), 3, _p(lg), 304, _p(tgt), T, V, _p(lp), None, s) != 0
    assert b"n_vt" in lib.copris_last_error()
    assert lib.copris_lmhead_logits(ctx.h, _p(x), H, _p(w), H, 0, H, V, _p(tgt), _p(lg), 304,
                                    _p(part), s) == 0  # empty is a no-op
    ctx.check()


def test_lmhead_token_out_of_vocabulary(ctx):
    from paper_2511_05589_b200 import ContractViolation
    T, H, V = 8, 64, 300
    x, w, tgt = _inputs(T, H, V, 2)
    tgt[3] = V
    lg, part = ctx.lmhead_logits(x, w, tgt)
    ctx.lse_merge(part, lg, tgt)
    with pytest.raises(ContractViolation, match="token out of vocabulary"):
        ctx.check()


@pytest.mark.parametrize("T,H,V", [(300, 512, 4096), (256, 256, 1000), (1024, 4096, 151936)])
@pytest.mark.parametrize("variant", ["wide", "pair", "mc"])
def test_lmhead_dhidden_tcgen05(ctx, T, H, V, variant, monkeypatch):
    """LM-head backward dhidden = dlogits @ W on the CTA-pair tcgen05 kernel
    (B = W^T, split-K with a fixed-order sum): the default 256 x 512 tiles vs the
    fp32 product within bf16 rounding of the output, bitwise on a rerun; the
    256 x 256 tile (pair) and the multicast 4-CTA variant (mc) at the same split
    count are bitwise the default (same k order for every output element)."""
    g = torch.Generator(device="cuda").manual_seed(T + H)
    ldv = (V + 7) // 8 * 8
    dl = (torch.randn((T, ldv), device="cuda", generator=g) * 1e-3).to(torch.bfloat16)[:, :V]
    w = (torch.randn((V, H), device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    wt = w.t().contiguous()
    if ldv != V:
        wt = torch.nn.functional.pad(wt, (0, ldv - V))[:, :V]
    for k in ("gemm_wide", "gemm_mc", "gemm_splits"):
        ctx.set_option(k, LM_DEFAULTS[k])
    out = ctx.lmhead_dhidden(dl, wt)
    assert ctx.last_launch()["kernel"].endswith(",wide>")
    torch.cuda.synchronize()
    ref = dl.float() @ w.float()
    err = (out.float() - ref).abs()
    tol = 2.0 ** -8 * ref.abs() + 1e-3 * ref.abs().max()
    assert bool((err <= tol).all()), float((err - tol).max())
    again = ctx.lmhead_dhidden(dl, wt)
    assert torch.equal(again.view(torch.int16), out.view(torch.int16))
    if variant != "wide":
        ctx.set_option("gemm_splits", 2)
        base = ctx.lmhead_dhidden(dl, wt)
        small_ref = ctx.lmhead_dhidden(dl[:1], wt)
        ctx.set_option("gemm_mc" if variant == "mc" else "gemm_wide", 1 if variant == "mc" else 0)
        multi = ctx.lmhead_dhidden(dl, wt)
        assert ctx.last_launch()["kernel"].endswith(f",{variant}>" if variant == "mc" else "<gemm>")
        assert torch.equal(multi.view(torch.int16), base.view(torch.int16))
        small = ctx.lmhead_dhidden(dl[:1], wt)
        assert torch.equal(small.view(torch.int16), small_ref.view(torch.int16))


@pytest.mark.parametrize("T,H,V", [(300, 512, 4096), (257, 192, 1000), (64, 520, 300), (1, 64, 256),
                                   (4100, 1024, 32000), (1024, 4096, 151936)])
def test_lmhead_dweight_tcgen05(ctx, T, H, V):
    """LM-head backward dW += dlogits^T @ hidden on the CTA-pair tcgen05 kernel
    with both operands MN-major (the token dimension is the reduction): vs the
    fp64 product within fp32-accumulation error, accumulation into an existing
    dW, ragged T/H/V (TMA zero fill), and bitwise on a rerun."""
    g = torch.Generator(device="cuda").manual_seed(T + H + V)
    ldv = (V + 7) // 8 * 8
    dl = (torch.randn((T, ldv), device="cuda", generator=g) * 1e-3).to(torch.bfloat16)[:, :V]
    x = torch.randn((T, H), device="cuda", generator=g).to(torch.bfloat16)
    dw0 = torch.randn((V, H), device="cuda", generator=g)
    out = ctx.lmhead_dweight(dl, x, out=dw0.clone())
    torch.cuda.synchronize()
    if V * H <= 1 << 24:
        ref = dw0.double() + dl.double().t() @ x.double()
        bound = (dl.double().abs().t() @ x.double().abs())
    else:  # fp32 on the GPU for the big case (its own error is inside the bound)
        ref = (dw0 + dl.float().t() @ x.float()).double()
        bound = (dl.float().abs().t() @ x.float().abs()).double()
    tol = (T + 2) * 2.0 ** -23 * bound + 2.0 ** -23 * dw0.double().abs() + 1e-30
    err = (out.double() - ref).abs()
    assert bool((err <= tol).all()), float((err - tol).max())
    again = ctx.lmhead_dweight(dl, x, out=dw0.clone())
    assert torch.equal(again.view(torch.int32), out.view(torch.int32))


def test_lmhead_dweight_token_chunks(ctx, monkeypatch):
    """The token reduction in several ordered launches (dw_kchunk option): the
    same bound plus one fp32 rounding of dW per launch, bitwise on a rerun."""
    ctx.set_option("dw_kchunk", 128)
    T, H, V = 300, 256, 1000
    g = torch.Generator(device="cuda").manual_seed(5)
    dl = (torch.randn((T, V), device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    x = torch.randn((T, H), device="cuda", generator=g).to(torch.bfloat16)
    dw0 = torch.randn((V, H), device="cuda", generator=g)
    out = ctx.lmhead_dweight(dl, x, out=dw0.clone())
    torch.cuda.synchronize()
    ref = dw0.double() + dl.double().t() @ x.double()
    bound = dl.double().abs().t() @ x.double().abs()
    tol = (T + 2) * 2.0 ** -23 * bound + 3 * 2.0 ** -23 * (dw0.double().abs() + bound) + 1e-30
    err = (out.double() - ref).abs()
    assert bool((err <= tol).all()), float((err - tol).max())
    again = ctx.lmhead_dweight(dl, x, out=dw0.clone())
    assert torch.equal(again.view(torch.int32), out.view(torch.int32))


def test_lmhead_dweight_strided(ctx):
    """Row strides larger than the logical widths on every operand: dlogits and
    hidden as column slices of wider buffers, dW rows padded; the padding is
    neither read into the product nor written."""
    T, H, V = 200, 264, 1000
    g = torch.Generator(device="cuda").manual_seed(9)
    dl_full = (torch.randn((T, V + 24), device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    x_full = torch.randn((T, H + 8), device="cuda", generator=g).to(torch.bfloat16)
    dl, x = dl_full[:, :V], x_full[:, :H]
    dw_full = torch.full((V, H + 12), 7.0, device="cuda")
    dw = dw_full[:, :H]
    dw.zero_()
    ctx.lmhead_dweight(dl, x, out=dw)
    torch.cuda.synchronize()
    ref = dl.double().t() @ x.double()
    bound = dl.double().abs().t() @ x.double().abs()
    assert bool(((dw.double() - ref).abs() <= (T + 2) * 2.0 ** -23 * bound + 1e-30).all())
    assert bool((dw_full[:, H:] == 7.0).all())


def test_lmhead_dweight_errors(ctx):
    dl = torch.zeros((8, 64), dtype=torch.bfloat16, device="cuda")
    x = torch.zeros((8, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        ctx.lmhead_dweight(dl, x[:4])
    with pytest.raises(ValueError, match="bad row strides"):
        ctx.lmhead_dweight(dl, x, out=torch.zeros((64, 66), device="cuda")[:, :64])


@pytest.mark.parametrize("impl", ["pair"], indirect=True)  # the TMA-store epilogue is the pair kernel's
@pytest.mark.parametrize("T,H,V", [(1, 64, 256), (130, 64, 300), (257, 192, 1000), (300, 520, 4099),
                                   (129, 64, 1064), (1024, 4096, 151936)])
def test_lmhead_tma_store_epilogue_bitwise(ctx, T, H, V, impl, monkeypatch):
    """The forward with the logits leaving through swizzled staging boxes and TMA
    stores (the default when V % 8 == 0): logits and LSE partials bitwise the
    register-store epilogue's (lmhead_tma_store = 0), ragged T included; at
    V % 8 != 0 the register-store epilogue runs (TMA would clip at 16-byte
    granularity and write the row padding)."""
    x, w, tgt = _inputs(T, H, V, 23)
    ldv = (V + 7) // 8 * 8
    lg0 = torch.full((T, ldv), 3.0, dtype=torch.bfloat16, device="cuda")
    lg1 = lg0.clone()
    nvt = int(ctx.lib.copris_lmhead_num_vtiles(V))
    p0 = torch.empty((T, nvt, 2), dtype=torch.float32, device="cuda")
    p1 = torch.empty_like(p0)
    ctx.set_option("lmhead_tma_store", 0)
    ctx.lmhead_logits(x, w, tgt, logits=lg0[:, :V], partials=p0)
    assert ctx.last_launch()["kernel"] == "lmhead_fwd_pair_kernel"
    ctx.set_option("lmhead_tma_store", 1)
    ctx.lmhead_logits(x, w, tgt, logits=lg1[:, :V], partials=p1)
    assert ctx.last_launch()["kernel"] == ("lmhead_fwd_pair_kernel<tma_store>" if V % 8 == 0
                                           else "lmhead_fwd_pair_kernel")
    torch.cuda.synchronize()
    assert torch.equal(lg1.view(torch.int16), lg0.view(torch.int16))  # padding untouched too
    assert torch.equal(p1.view(torch.int32), p0.view(torch.int32))


@pytest.mark.parametrize("impl", ["pair"], indirect=True)
@pytest.mark.parametrize("T,H,V", [(130, 64, 1000), (1024, 4096, 151936)])
def test_lmhead_logits_only_bitwise(ctx, T, H, V, impl):
    """partials = NULL: the forward stores the logits only (no exponentials in
    the epilogue) — bitwise the logits of the statistics-producing call."""
    x, w, tgt = _inputs(T, H, V, 29)
    a, pa = ctx.lmhead_logits(x, w, tgt)
    b, pb = ctx.lmhead_logits(x, w, None, stats=False)
    torch.cuda.synchronize()
    assert pb is None and pa is not None
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
