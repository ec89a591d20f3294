"""LM-head + IS-corrected GRPO loss over hidden states.

The reference's policy is a table (policy.hpp:110-121: the logits row of token
t is ``row(class, t)``); in an LLM the same row is ``hidden[t] @ W^T``. This
module runs the loss path of grpo.hpp:117-185 with that producer in front and
its backward behind, chunked over tokens so the [T x V] logits exist only one
chunk at a time:

  per chunk of rows (default: loss_impl="fused", fwd_impl="cublas")
    logits = hidden @ W^T  (plain GEMM; or copris_lmhead_logits, tcgen05, logits only)
    copris_is_loss_fused   the one-pass loss: cur_lp, behaviour, objective,
                           dlogits IN PLACE over the logits (CTA-pair kernel)
    dhidden = dlogits @ W  and  dW += dlogits^T @ hidden   (plain GEMMs, or tcgen05)
  copris_loss_reduce -> loss, counts
  loss_impl="lse" instead: copris_lmhead_logits (tcgen05, logits + LSE partials in
  the epilogue) -> copris_lse_merge -> copris_behaviour_concat -> copris_is_loss_bwd.

The loss is a kernel in libcopris_b200.so; the GEMMs are plain library GEMMs by
default, or this library's tcgen05 kernels (DESIGN.md §3b for the measurements).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib as L
from .errors import ConfigError, ContractViolation
from .grpo import ClipConfig, Copris, PackedBatch, _p


@dataclass
class LmHeadStepResult:
    loss: float
    token_count: int
    objective: float
    stale_tokens: int
    clipped_tokens: int
    cur_lp: torch.Tensor
    lse: torch.Tensor
    obj: torch.Tensor
    flags: torch.Tensor
    dhidden: Optional[torch.Tensor]
    dweight: Optional[torch.Tensor]
    coef: Optional[torch.Tensor] = None


def lmhead_grpo_step_loss(ctx: Copris, *args, stream=None, **kw) -> "LmHeadStepResult":
    """See _lmhead_grpo_step_loss; with ``stream`` every buffer is allocated on it."""
    if stream is None:
        return _lmhead_grpo_step_loss(ctx, *args, stream=None, **kw)
    with torch.cuda.stream(stream):
        return _lmhead_grpo_step_loss(ctx, *args, stream=stream, **kw)


def _lmhead_grpo_step_loss(ctx: Copris, hidden: torch.Tensor, weight: torch.Tensor,
                          batch: PackedBatch, cfg: ClipConfig = None, *, chunk_rows: int = 8192,
                          is_enabled: bool = True, behav_mode: int = L.COPRIS_BEHAV_RECOMPUTED,
                          total_tokens: Optional[int] = None, want_grad: bool = True,
                          dweight: Optional[torch.Tensor] = None, coef: bool = False,
                          dhidden_impl: str = "cublas", weight_t: Optional[torch.Tensor] = None,
                          dweight_impl: str = "cublas", loss_impl: str = "fused",
                          fwd_impl: str = "cublas", stream=None) -> LmHeadStepResult:
    """grpo.hpp:117-185 with logits = hidden @ weight^T (bf16 in, fp32 accumulate).

    ``dweight`` (fp32 [V x H]) is accumulated into when given (zeros otherwise).
    ``dhidden_impl="tcgen05"`` computes dhidden = dlogits @ weight on the
    CTA-pair tcgen05 kernel (copris_lmhead_dhidden, 256 x 512 tiles; needs
    weight^T, passed as ``weight_t`` or transposed here once) and
    ``dweight_impl="tcgen05"`` accumulates dweight += dlogits^T @ hidden on the
    same kernel with MN-major operands (copris_lmhead_dweight). Alone, both are
    within a few percent of cuBLAS (dhidden faster at 8K-token chunks); inside
    this power-capped step the cuBLAS GEMMs measured faster, so they are the
    default.

    ``loss_impl``: "fused" (default) — the forward stores the logits only and
    the one-pass fused loss kernel (copris_is_loss_fused: the CTA-pair kernel,
    one exponential per element) writes dlogits in place; "lse" — the tcgen05
    forward's epilogue emits the softmax statistics, then lse_merge -> K2 -> K3
    (one streaming pass that recomputes the exponentials).
    ``fwd_impl``: "cublas" (default) — the forward is a plain library GEMM;
    "tcgen05" — copris_lmhead_logits (the CTA-pair tcgen05 kernel). Defaults
    are the fastest measured combination in a sustained, power-capped step
    (cuBLAS GEMMs around the one-pass loss kernel; the tcgen05
    kernels run 2-10% slower there, at lower clocks for the same power).
    """
    cfg = cfg or ClipConfig()
    cfg.validate()
    if batch.n_traj == 0:
        raise ConfigError("grpo_step_loss requires a non-empty batch")
    if batch.n_tok == 0:
        raise ConfigError("grpo_step_loss batch has no tokens")
    T, H = hidden.shape
    V = weight.shape[0]
    if T != batch.n_tok:
        raise ContractViolation("log-prob vectors must align with token count")
    if weight.shape[1] != H:
        raise ContractViolation("hidden and weight disagree on the hidden size")
    # the masked token mean divides by the UNMASKED count, as grpo_step_loss does
    T_glob = total_tokens if total_tokens is not None else batch.loss_tokens()
    if T_glob <= 0:
        raise ConfigError("grpo_step_loss batch has no tokens")
    dev = hidden.device
    chunk = max(1, min(chunk_rows, T))
    ldv = (V + 7) // 8 * 8
    buf = torch.empty((chunk, ldv), dtype=torch.bfloat16, device=dev)[:, :V]
    nvt = int(ctx.lib.copris_lmhead_num_vtiles(V))
    part = torch.empty((chunk, nvt, 2), dtype=torch.float32, device=dev) if loss_impl == "lse" else None
    outs = ctx.alloc_outputs(T, dev, coef=coef)
    dhidden = torch.empty_like(hidden) if want_grad else None
    if want_grad and dweight is None:
        dweight = torch.zeros((V, H), dtype=torch.float32, device=dev)
    s = ctx._stream(stream)
    if want_grad and dhidden_impl == "tcgen05" and weight_t is None:
        weight_t = weight.t().contiguous()
    elif dhidden_impl not in ("cublas", "tcgen05"):
        raise ValueError("dhidden_impl must be 'cublas' or 'tcgen05'")
    if dweight_impl not in ("cublas", "tcgen05"):
        raise ValueError("dweight_impl must be 'cublas' or 'tcgen05'")
    if loss_impl not in ("lse", "fused"):
        raise ValueError("loss_impl must be 'lse' or 'fused'")
    if fwd_impl not in ("cublas", "tcgen05"):
        raise ValueError("fwd_impl must be 'cublas' or 'tcgen05'")
    if loss_impl == "lse" and fwd_impl != "tcgen05":
        raise ValueError("loss_impl='lse' needs the statistics of fwd_impl='tcgen05'")
    for a in range(0, T, chunk):
        n = min(chunk, T - a)
        sl = slice(a, a + n)
        lg = buf[:n]
        if loss_impl == "fused":
            if fwd_impl == "tcgen05":
                ctx.lmhead_logits(hidden[sl], weight, None, logits=lg, stats=False, stream=stream)
            else:
                with torch.cuda.stream(stream) if stream is not None else _null():
                    torch.mm(hidden[sl], weight.t(), out=lg)
            ctx.loss_chunk_fused(lg, batch, cfg, outs, dlogits=lg if want_grad else None, row_base=a,
                                 total_tokens=T_glob, is_enabled=is_enabled, behav_mode=behav_mode,
                                 stream=stream)
        else:
            ctx.lmhead_logits(hidden[sl], weight, batch.target[sl], logits=lg, partials=part[:n],
                              stream=stream)
            ctx.lse_merge(part[:n], lg, batch.target[sl], out_lp=outs["cur_lp"][sl],
                          out_lse=outs["lse"][sl], stream=stream)
            ctx._call(ctx.lib.copris_behaviour_concat(
                ctx.h, _p(batch.stage[sl]), batch.cur_stage, _p(batch.buffered_lp[sl]),
                _p(outs["cur_lp"][sl]), int(is_enabled), behav_mode, n, _p(outs["behav"][sl]), None,
                s))
            b, c, o = ctx._structs(lg, batch, cfg, is_enabled, behav_mode, T_glob, a,
                                   lg if want_grad else None, outs)
            ctx._call(ctx.lib.copris_is_loss_bwd(ctx.h, C.byref(b), C.byref(c), _p(outs["cur_lp"]),
                                                 _p(outs["lse"]), _p(outs["behav"]), C.byref(o), s))
        if want_grad:
            # dlogits now sits in `lg`: the LM-head backward (plain GEMMs)
            if dhidden_impl == "tcgen05":
                ctx.lmhead_dhidden(lg, weight_t, out=dhidden[sl], stream=stream)
            if dweight_impl == "tcgen05":
                ctx.lmhead_dweight(lg, hidden[sl], out=dweight, stream=stream)
            with torch.cuda.stream(stream) if stream is not None else _null():
                if dhidden_impl == "cublas":
                    torch.mm(lg, weight, out=dhidden[sl])
                if dweight_impl == "cublas":
                    torch.addmm(dweight, lg.t(), hidden[sl], out_dtype=torch.float32, out=dweight)
    out4 = torch.empty(4, dtype=torch.float64, device=dev)
    ctx.reduce(outs, T, out4, stream=stream)
    ctx.check(stream)
    o4 = out4.cpu().tolist()
    res = LmHeadStepResult(loss=-o4[0] * (1.0 / T_glob), token_count=int(o4[1]), objective=o4[0],
                           stale_tokens=int(o4[2]), clipped_tokens=int(o4[3]),
                           cur_lp=outs["cur_lp"], lse=outs["lse"], obj=outs["obj"],
                           flags=outs["flags"], dhidden=dhidden, dweight=dweight,
                           coef=outs.get("coef"))
    return res


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
