"""Shared helpers for the parity tests: synthetic cases and tolerance checks.

Tolerances (BASELINE.json north_star: "within 1e-5 relative tolerance (fp32
accumulation) for log-probs, ratios, loss and gradients"), made row-scaled the
way the reference's own checks are (test_grpo.cpp:341, acceptance_main.cpp:95):
  * per-token scalars  |gpu - ref| <= 1e-5 * max(1, |ref|)
  * f32 dlogits rows   |gpu - ref| <= 1e-5 * max_k |ref_row|
  * bf16 dlogits rows  |gpu - ref| <= 2^-7 |ref| + 1e-5 * max_k |ref_row|
                       (one bf16 ulp at the top of a binade; the pair kernel's
                       bf16-staged path is within 3 * 2^-9 by construction)
  * loss               |gpu - ref| <= 1e-5 * max(|ref|, sum_t |obj_t| / T)
Bit-exact: stage/stale flags, clip masks, behaviour select, advantages.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from paper_2511_05589_b200.workload import make_host_batch, make_logits, stale_logprobs

RTOL = 1e-5


def max_rel_scalar(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(gpu - ref) / np.maximum(1.0, np.abs(ref)), initial=0.0))


def assert_scalar_close(gpu, ref, rtol=RTOL, what=""):
    e = max_rel_scalar(gpu, ref)
    assert e <= rtol, f"{what}: max scaled error {e:.3e} > {rtol}"


def assert_rows_close(gpu, ref, bf16=False, rtol=RTOL, what="", row_atol=None):
    """row_atol: per-row absolute slack for the reference's OWN rounding — its
    one-hot entry is -w*p_y + w in fp64 (policy.hpp:193-194), which cancels when
    p_y -> 1 and is then only accurate to ~|w| * 2^-52."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    rowmax = np.abs(ref).max(axis=1, keepdims=True)
    tol = rtol * rowmax + 1e-300
    if row_atol is not None:
        tol = tol + np.asarray(row_atol, np.float64).reshape(-1, 1)
    if bf16:
        tol = tol + 2.0 ** -7 * np.abs(ref)
    bad = np.abs(gpu - ref) > tol
    if bad.any():
        i, k = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} entries out of tolerance; first row {i} col {k}: "
                             f"gpu {gpu[i, k]!r} ref {ref[i, k]!r} rowmax {rowmax[i, 0]!r}")


def assert_loss_close(gpu_loss, ref_loss, ref_obj, T, rtol=RTOL, what="loss"):
    scale = max(abs(ref_loss), float(np.abs(ref_obj).sum()) / T, 1e-300)
    assert abs(gpu_loss - ref_loss) <= rtol * scale, \
        f"{what}: gpu {gpu_loss!r} ref {ref_loss!r} (scale {scale:.3e})"


def with_empty_trajectories(hb, idx):
    """The batch with every token of trajectories `idx` removed (zero-length
    trajectories stay in their groups: they count for the group advantage but
    contribute no token)."""
    from dataclasses import replace
    idx = set(int(i) for i in idx)
    keep = np.ones(hb.n_tok, bool)
    for i in idx:
        keep[hb.tok_off[i]:hb.tok_off[i + 1]] = False
    before = np.concatenate([[0], np.cumsum(~keep)])  # dropped tokens before each offset
    tok_off = hb.tok_off - before[hb.tok_off]
    seg_off = hb.seg_off - before[hb.seg_off]
    nonempty = np.diff(seg_off) > 0
    seg_off = np.concatenate([[0], seg_off[1:][nonempty]]).astype(np.int64)
    return replace(hb, tok_off=tok_off.astype(np.int64), target=hb.target[keep], stage=hb.stage[keep],
                   seg_off=seg_off, seg_ver=hb.seg_ver[nonempty])


class Case:
    """A seeded synthetic batch plus its oracle result."""

    def __init__(self, oracle, seed=1, P=2, G=4, V=512, fixed_len=None, mu=math.log(12),
                 sigma=0.6, lmax=48, stages=(1, 2), stale_prob=0.6, dtype=torch.bfloat16,
                 ld=None, clip_low=0.2, clip_high=0.28, kl_coeff=0.0, entropy_coeff=0.0,
                 is_enabled=True, behav_mode=0, reward=None, edit_logits=None, empty=None,
                 edit_blp=None, targets=None):
        hb = make_host_batch(seed, P, G, V, mu=mu, sigma=sigma, lmax=lmax, fixed_len=fixed_len,
                             stages=stages, stale_prob=stale_prob)
        if targets is not None:  # chosen target columns, cycled over the tokens
            t = np.asarray(targets, np.int32)
            hb.target[:] = t[np.arange(hb.n_tok) % len(t)]
        if empty is not None:
            hb = with_empty_trajectories(hb, empty)
        if reward is not None:
            hb.reward[:] = reward
        self.hb = hb
        self.V = V
        self.dtype = dtype
        self.ld = ld
        logits = make_logits(hb.n_tok, V, hb.target, seed, "cpu", dtype, ld=ld)
        if edit_logits is not None:  # e.g. masked vocabulary entries (-inf)
            edit_logits(logits, hb)
        self.logits_cpu = logits  # may be a padded view
        self.z64 = logits.double().numpy()
        cur = oracle.logprob_gather(self.z64, hb.target)
        self.blp = stale_logprobs(cur, hb.stage, hb.cur_stage, seed, clip_low, clip_high)
        if edit_blp is not None:  # e.g. tokens far off policy
            edit_blp(self.blp, cur, hb)
        self.adv = oracle.advantages(hb.reward, hb.group_off)
        self.ref_lp = None
        if kl_coeff > 0.0:
            ref_logits = make_logits(hb.n_tok, V, hb.target, seed + 101, "cpu", dtype)
            self.ref_lp = oracle.logprob_gather(ref_logits.double().numpy(), hb.target).astype(np.float32)
        self.cfg = dict(clip_low=clip_low, clip_high=clip_high, kl_coeff=kl_coeff,
                        entropy_coeff=entropy_coeff)
        self.is_enabled = is_enabled
        self.behav_mode = behav_mode
        self.ref = oracle.is_loss(self.z64, hb.tok_off, hb.target, hb.stage, hb.cur_stage,
                                  self.blp.astype(np.float64), self.adv, is_enabled=is_enabled,
                                  ref_lp=None if self.ref_lp is None else self.ref_lp.astype(np.float64),
                                  behav_mode=behav_mode, **self.cfg)

    def logits_gpu(self):
        if self.ld is None:
            return self.logits_cpu.cuda()
        base = self.logits_cpu.as_strided((self.hb.n_tok, self.ld), (self.ld, 1)).cuda()
        return base[:, :self.V]

    def upload(self, ctx):
        from paper_2511_05589_b200.packing import upload
        hb = self.hb
        return upload(ctx, hb.tok_off, hb.group_off, hb.target, self.blp, hb.cur_stage,
                      seg_off=hb.seg_off, seg_ver=hb.seg_ver, reward=hb.reward,
                      ref_lp=self.ref_lp)

    def clip(self):
        from paper_2511_05589_b200 import ClipConfig
        return ClipConfig(**self.cfg)

    def check(self, res, dl_dtype, what=""):
        ref, hb = self.ref, self.hb
        T = hb.n_tok
        assert res.token_count == T
        cur = res.cur_lp.cpu().numpy()
        assert_scalar_close(cur, ref.cur_lp, what=f"{what} cur_lp")
        if res.behav is not None:
            assert_scalar_close(res.behav.cpu().numpy(), ref.behav, what=f"{what} behav")
        flags = res.flags.cpu().numpy()
        np.testing.assert_array_equal(flags & 1, (hb.stage < hb.cur_stage).astype(np.uint8),
                                      err_msg=f"{what} stale flags")
        np.testing.assert_array_equal((flags >> 1) & 1, ref.clipped, err_msg=f"{what} clip mask")
        assert res.stale_tokens == ref.stale_tokens
        assert res.clipped_tokens == ref.clipped_tokens
        assert_scalar_close(res.obj.cpu().numpy(), ref.obj, what=f"{what} obj")
        assert_loss_close(res.loss, ref.loss, ref.obj, T, what=f"{what} loss")
        if res.dlogits is not None:
            dl = res.dlogits.float().cpu().numpy()
            # the reference's p_y = e_y / sum_k e_k carries up to ~V ulps of error,
            # which its one-hot entry w - w*p_y inherits (policy.hpp:193-194)
            atol = (self.V + 8) * 2.0 ** -52 * (np.abs(ref.weight) + self.cfg["entropy_coeff"]) / T
            beta = self.cfg["kl_coeff"]
            if beta > 0.0:
                # w = r A + beta (e^d - 1) can cancel; its error follows the
                # conditioning of its terms in cur (an fp32 log-prob on the
                # device): dw ~ (|r A| + beta e^d) dcur, dcur ~ 2e-6 max(1, |cur|)
                cur = ref.cur_lp
                r = np.exp(cur - ref.behav)
                adv_t = np.repeat(self.adv, np.diff(hb.tok_off))
                ed = np.exp(self.ref_lp.astype(np.float64) - cur)
                atol = atol + (np.abs(r * adv_t) + beta * ed) * 2e-6 * np.maximum(1.0, np.abs(cur)) / T
            assert_rows_close(dl, ref.dlogits, bf16=(dl_dtype == torch.bfloat16),
                              what=f"{what} dlogits", row_atol=atol)


def exact_dlogits(z64, target, coef):
    """fp64 dlogits WITHOUT the reference's cancellation: the one-hot entry is
    coef * sum_{k != y} p_k instead of coef - coef * p_y."""
    z = np.asarray(z64, np.float64)
    e = np.exp(z - z.max(axis=1, keepdims=True))
    S = e.sum(axis=1, keepdims=True)
    p = e / S
    d = -coef[:, None] * p
    rows = np.arange(len(target))
    mask = np.ones_like(e, dtype=bool)
    mask[rows, target] = False
    others = np.where(mask, e, 0.0).sum(axis=1)
    d[rows, target] = coef * others / S[:, 0]
    return d


def oracle_per_token(oracle, logits_cpu, tok_off, target, stage, cur_stage, blp, adv,
                     chunk=256, threads=None, **cfg):
    """The CPU oracle's per-token outputs (cur_lp, behav, obj, weight, clipped)
    over ALL rows of a large batch, computed on host threads in row chunks.

    Per-token results depend only on the token's logits row, its stage and
    buffered log-prob and its trajectory's advantage, so each chunk [a, b) is
    presented to the oracle as the trajectories' pieces inside it (each piece
    keeping its trajectory's advantage). ``logits_cpu`` is a bf16/f32 torch
    tensor; rows are widened to fp64 one chunk at a time. The loss and the
    dlogits coefficients are formed by the caller from obj / weight with the
    batch's own T (grpo.hpp:135,183)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    tok_off = np.asarray(tok_off, np.int64)
    T = int(tok_off[-1])
    out = {k: np.zeros(T, np.float64) for k in ("cur_lp", "behav", "obj", "weight")}
    out["clipped"] = np.zeros(T, np.uint8)

    def work(a):
        b = min(T, a + chunk)
        t_lo = int(np.searchsorted(tok_off, a, side="right")) - 1
        t_hi = int(np.searchsorted(tok_off, b, side="left"))
        sub = np.clip(tok_off[t_lo:t_hi + 1], a, b) - a
        z = logits_cpu[a:b].double().numpy()
        r = oracle.is_loss(z, sub, target[a:b], stage[a:b], cur_stage,
                           np.asarray(blp[a:b], np.float64), np.asarray(adv[t_lo:t_hi], np.float64),
                           want_dlogits=False, **cfg)
        for k in ("cur_lp", "behav", "obj", "weight", "clipped"):
            out[k][a:b] = getattr(r, k)

    n = threads or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=n) as ex:
        list(ex.map(work, range(0, T, chunk)))
    return out
