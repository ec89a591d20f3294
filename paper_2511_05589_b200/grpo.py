"""Host-side mirror of the reference's loss entry points over the C-ABI.

Reference surface (``/root/reference/proj/include/copris``) -> here:

  ClipConfig                       grpo.hpp:15-28     -> ClipConfig
  sequence_logprobs                policy.hpp:160-173 -> Copris.sequence_logprobs   (K1)
  concat_segments / IS-off         trajectory.hpp:69-75, trainer.hpp:149
                                                      -> Copris.concat_segments     (K2)
  terminal_reward                  grpo.hpp:35-47     -> Copris.terminal_rewards
  compute_advantages               grpo.hpp:51-65     -> Copris.compute_advantages  (K3a)
  grpo_step_loss / GrpoStepResult  grpo.hpp:94-185    -> Copris.grpo_step_loss      (K3 / fused)
  offpolicy_token_fraction         rollout.hpp:99-110 -> GrpoStepResult.stale_tokens / token_count

Device memory and streams come from PyTorch (plumbing); every computation is a
kernel in libcopris_b200.so. Errors raise the reference's exception types with
the reference's messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib as L
from .errors import ConfigError, ContractViolation, CudaError


def _raise(rc: int, lib) -> None:
    msg = lib.copris_last_error().decode()
    if rc == L.COPRIS_E_CONTRACT:
        raise ContractViolation(msg)
    if rc == L.COPRIS_E_CONFIG:
        raise ConfigError(msg)
    if rc == L.COPRIS_E_CUDA:
        raise CudaError(msg)
    raise ValueError(msg)


def _p(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _on_stream(fn):
    """Run the method with `stream` as torch's current stream, so the buffers it
    allocates (outputs, split-K work, zero-filled dweight) are allocated and
    initialised on the stream the kernels run on: the caching allocator then
    cannot hand a dropped work buffer to another stream while the kernel still
    writes it (grpo.py:213)."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *args, stream=None, **kw):
        if stream is None:
            return fn(self, *args, stream=None, **kw)
        with torch.cuda.stream(stream):
            return fn(self, *args, stream=stream, **kw)
    return wrapped


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return L.COPRIS_BF16
    if dt == torch.float32:
        return L.COPRIS_F32
    raise ValueError(f"unsupported dtype {dt} (bf16 or f32)")


@dataclass
class ClipConfig:
    """grpo.hpp:15-28 (defaults = configs/desk.json:17-23)."""
    clip_low: float = 0.2
    clip_high: float = 0.28
    kl_coeff: float = 0.0
    entropy_coeff: float = 0.0
    adv_epsilon: float = 1e-6

    def validate(self) -> None:  # grpo.hpp:20-25
        if self.clip_low <= 0.0 or self.clip_high <= 0.0:
            raise ConfigError("grpo.clip_low and grpo.clip_high must be > 0")
        if self.kl_coeff < 0.0:
            raise ConfigError("grpo.kl_coeff must be >= 0")
        if self.adv_epsilon <= 0.0:
            raise ConfigError("grpo.adv_epsilon must be > 0")


@dataclass
class PackedBatch:
    """Packed stage-tagged batch in device memory (include/copris_b200.h layout).

    Token t is row t of the batch's logits. All tensors live on one device.
    """
    tok_off: torch.Tensor       # [n+1] int64
    group_off: torch.Tensor     # [P+1] int64
    target: torch.Tensor        # [T] int32
    stage: torch.Tensor         # [T] int32 (uint32 semantics)
    buffered_lp: torch.Tensor   # [T] f32
    tok_traj: torch.Tensor      # [T] int32
    adv: torch.Tensor           # [n] f64
    cur_stage: int
    ref_lp: Optional[torch.Tensor] = None  # [T] f32, for kl_coeff > 0
    group_off_host: Optional[list] = None
    loss_mask: Optional[torch.Tensor] = None  # [T] uint8, 0 = token left out of the loss

    def loss_tokens(self) -> int:
        """Tokens the loss averages over (the masked token mean)."""
        return self.n_tok if self.loss_mask is None else int(self.loss_mask.count_nonzero())

    @property
    def n_tok(self) -> int:
        return int(self.target.numel())

    @property
    def n_traj(self) -> int:
        return int(self.tok_off.numel()) - 1


@dataclass
class GrpoStepResult:
    """grpo.hpp:102-106 plus the scalars the trainer reads (trainer.hpp:167,177)."""
    loss: float
    dlogits: Optional[torch.Tensor]
    token_count: int
    objective: float
    stale_tokens: int
    clipped_tokens: int
    cur_lp: torch.Tensor
    behav: Optional[torch.Tensor]
    obj: torch.Tensor
    flags: torch.Tensor
    coef: Optional[torch.Tensor] = None
    lse: Optional[torch.Tensor] = None

    @property
    def offpolicy_fraction(self) -> float:  # rollout.hpp:99-110
        return self.stale_tokens / self.token_count if self.token_count else 0.0


class Copris:
    """One C-ABI context bound to a CUDA device (re-entrant, no global state)."""

    def __init__(self, device: int | torch.device | None = None):
        self.lib = L.load()
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = int(device)
        h = C.c_void_p()
        rc = self.lib.copris_ctx_create(self.device, C.byref(h))
        if rc:
            _raise(rc, self.lib)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.copris_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing -------------------------------------------------------------
    def _stream(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    def _call(self, rc):
        if rc:
            _raise(rc, self.lib)

    def check(self, stream=None) -> None:
        """Synchronise and raise any device-detected contract violation."""
        self._call(self.lib.copris_ctx_check(self.h, self._stream(stream)))

    # kernel selection / tunables of THIS context (copris_ctx_set_option); the
    # COPRIS_* environment is read once, when the context is created
    _NAMED = {"fused_impl": {"auto": 0, "stream": 1, "tma": 2, "pair": 3, "solo": 4},
              "lmhead_impl": {"pair": 0, "1sm": 1}}

    def set_option(self, name: str, value) -> None:
        if isinstance(value, str):
            value = self._NAMED[name][value]
        self._call(self.lib.copris_ctx_set_option(self.h, name.encode(), int(value)))

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        self._call(self.lib.copris_ctx_get_option(self.h, name.encode(), C.byref(v)))
        return v.value

    def options(self, **kw):
        """Context manager: set options, restore the previous values on exit."""
        import contextlib

        @contextlib.contextmanager
        def cm():
            old = {k: self.get_option(k) for k in kw}
            try:
                for k, v in kw.items():
                    self.set_option(k, v)
                yield self
            finally:
                for k, v in old.items():
                    self.set_option(k, v)
        return cm()

    def last_launch(self) -> dict:
        cl, grid, sms = C.c_int(), C.c_int(), C.c_int()
        name = C.c_char_p()
        self._call(self.lib.copris_ctx_last_launch(self.h, C.byref(cl), C.byref(grid),
                                                   C.byref(sms), C.byref(name)))
        return {"cluster": cl.value, "grid": grid.value, "num_sms": sms.value,
                "kernel": name.value.decode() if name.value else "",
                "fused_reduce": bool(self.lib.copris_ctx_last_fused_reduce(self.h))}

    # -- K1 -----------------------------------------------------------------------
    @_on_stream
    def sequence_logprobs(self, logits: torch.Tensor, target: torch.Tensor, stream=None,
                          out_lp=None, out_lse=None):
        """policy.hpp:160-173 over packed rows -> (cur_lp f32 [T], lse f32 [T])."""
        n, v = logits.shape
        lp = out_lp if out_lp is not None else torch.empty(n, dtype=torch.float32, device=logits.device)
        lse = out_lse if out_lse is not None else torch.empty(n, dtype=torch.float32, device=logits.device)
        self._call(self.lib.copris_logprob_gather(
            self.h, _p(logits), logits.stride(0), _dtype_code(logits.dtype), _p(target), n, v,
            _p(lp), _p(lse), self._stream(stream)))
        return lp, lse

    # -- LM-head forward + log-softmax partials (tcgen05) ---------------------------
    @_on_stream
    def lmhead_logits(self, hidden: torch.Tensor, weight: torch.Tensor, target: Optional[torch.Tensor],
                      logits: Optional[torch.Tensor] = None,
                      partials: Optional[torch.Tensor] = None, stream=None, stats: bool = True):
        """logits = bf16(hidden @ weight^T) and per-256-column LSE partials
        (float2 per (token, tile), target column excluded); ``stats=False``:
        logits only (no partials, ``target`` unused)."""
        n, h = hidden.shape
        v = weight.shape[0]
        if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
            raise ValueError("hidden and weight must be bf16")
        nvt = int(self.lib.copris_lmhead_num_vtiles(v))
        if logits is None:
            ld = (v + 7) // 8 * 8
            logits = torch.empty((n, ld), dtype=torch.bfloat16, device=hidden.device)[:, :v]
        if stats and partials is None:
            partials = torch.empty((n, nvt, 2), dtype=torch.float32, device=hidden.device)
        if not stats:
            partials = None
        self._call(self.lib.copris_lmhead_logits(
            self.h, _p(hidden), hidden.stride(0), _p(weight), weight.stride(0), n, h, v,
            _p(target) if stats else None, _p(logits), logits.stride(0),
            _p(partials) if stats else None, self._stream(stream)))
        return logits, partials

    @_on_stream
    def lmhead_dhidden(self, dlogits: torch.Tensor, weight_t: torch.Tensor,
                       out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """dhidden = dlogits @ weight (bf16) on the tcgen05 pair kernel; weight_t
        is weight^T [H x V] contiguous (transpose once per optimizer step)."""
        n, V = dlogits.shape
        H = weight_t.shape[0]
        if out is None:
            out = torch.empty((n, H), dtype=torch.bfloat16, device=dlogits.device)
        splits = int(self.lib.copris_lmhead_dhidden_splits(self.h, n, H))
        work = torch.empty((max(1, splits), n, H), dtype=torch.float32, device=dlogits.device)
        self._call(self.lib.copris_lmhead_dhidden(
            self.h, _p(dlogits), dlogits.stride(0), _p(weight_t), weight_t.stride(0), n, H, V,
            _p(out), out.stride(0), _p(work), self._stream(stream)))
        return out

    @_on_stream
    def lmhead_dweight(self, dlogits: torch.Tensor, hidden: torch.Tensor,
                       out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """dweight (fp32 [V x H]) += dlogits^T @ hidden on the tcgen05 pair kernel
        (MN-major operands; zeros first when ``out`` is None)."""
        n, V = dlogits.shape
        H = hidden.shape[1]
        if hidden.shape[0] != n:
            raise ValueError("dlogits and hidden must have the same number of rows")
        if out is None:
            out = torch.zeros((V, H), dtype=torch.float32, device=dlogits.device)
        self._call(self.lib.copris_lmhead_dweight(
            self.h, _p(dlogits), dlogits.stride(0), _p(hidden), hidden.stride(0), n, H, V,
            _p(out), out.stride(0), self._stream(stream)))
        return out

    @_on_stream
    def lse_merge(self, partials: torch.Tensor, logits: torch.Tensor, target: torch.Tensor,
                  out_lp=None, out_lse=None, stream=None):
        """(cur_lp, lse) from lmhead partials — what sequence_logprobs gives on the logits."""
        n, v = logits.shape
        lp = out_lp if out_lp is not None else torch.empty(n, dtype=torch.float32, device=logits.device)
        lse = out_lse if out_lse is not None else torch.empty(n, dtype=torch.float32, device=logits.device)
        self._call(self.lib.copris_lse_merge(
            self.h, _p(partials), partials.shape[1], _p(logits), logits.stride(0), _p(target), n, v,
            _p(lp), _p(lse), self._stream(stream)))
        return lp, lse

    # -- K2 -----------------------------------------------------------------------
    @_on_stream
    def expand_segments(self, seg_off: torch.Tensor, seg_ver: torch.Tensor, n_tok: int,
                        stream=None) -> torch.Tensor:
        out = torch.empty(n_tok, dtype=torch.int32, device=seg_off.device)
        self._call(self.lib.copris_expand_segments(self.h, _p(seg_off), _p(seg_ver),
                                                   seg_ver.numel(), _p(out), self._stream(stream)))
        return out

    @_on_stream
    def concat_segments(self, stage, cur_stage: int, buffered_lp, cur_lp, is_enabled=True,
                        behav_mode=L.COPRIS_BEHAV_RECOMPUTED, stream=None):
        """trajectory.hpp:69-75 + trainer.hpp:149 -> (behav f32 [T], flags u8 [T])."""
        n = stage.numel()
        behav = torch.empty(n, dtype=torch.float32, device=stage.device)
        flags = torch.empty(n, dtype=torch.uint8, device=stage.device)
        self._call(self.lib.copris_behaviour_concat(
            self.h, _p(stage), cur_stage, _p(buffered_lp), _p(cur_lp), int(is_enabled),
            behav_mode, n, _p(behav), _p(flags), self._stream(stream)))
        return behav, flags

    # -- K3a ----------------------------------------------------------------------
    @_on_stream
    def terminal_rewards(self, tokens, tok_off, terminated, answer_target, eos_token: int,
                         stream=None) -> torch.Tensor:
        n = tok_off.numel() - 1
        out = torch.empty(n, dtype=torch.float64, device=tokens.device)
        self._call(self.lib.copris_terminal_rewards(
            self.h, _p(tokens), _p(tok_off), n, _p(terminated), _p(answer_target), eos_token,
            _p(out), self._stream(stream)))
        return out

    @_on_stream
    def compute_advantages(self, rewards: torch.Tensor, group_off: torch.Tensor,
                           adv_epsilon: float = 1e-6, group_off_host=None,
                           stream=None) -> torch.Tensor:
        """grpo.hpp:51-65 for every group at once (fp64, bit-identical)."""
        host = group_off_host if group_off_host is not None else group_off.cpu().tolist()
        host_arr = (C.c_int64 * len(host))(*host)
        out = torch.empty_like(rewards, dtype=torch.float64)
        self._call(self.lib.copris_group_advantages(
            self.h, _p(rewards), C.cast(host_arr, C.c_void_p), _p(group_off), len(host) - 1,
            adv_epsilon, _p(out), self._stream(stream)))
        return out

    @_on_stream
    def token_traj(self, tok_off: torch.Tensor, n_tok: int, stream=None) -> torch.Tensor:
        out = torch.empty(n_tok, dtype=torch.int32, device=tok_off.device)
        self._call(self.lib.copris_token_traj(self.h, _p(tok_off), tok_off.numel() - 1, n_tok,
                                              _p(out), self._stream(stream)))
        return out

    # -- K3 -----------------------------------------------------------------------
    def _structs(self, logits, batch: PackedBatch, cfg: ClipConfig, is_enabled, behav_mode,
                 total_tokens, row_base, dlogits, outs, out4=None):
        n_rows, v = logits.shape
        b = L.LossBatch(_p(logits), logits.stride(0), _dtype_code(logits.dtype), v, n_rows,
                        row_base, _p(batch.target), _p(batch.stage), _p(batch.buffered_lp),
                        _p(batch.ref_lp), _p(batch.tok_traj), _p(batch.adv), batch.cur_stage, 0,
                        _p(batch.loss_mask))
        c = L.LossCfg(cfg.clip_low, cfg.clip_high, cfg.kl_coeff, cfg.entropy_coeff,
                      int(is_enabled), behav_mode, total_tokens)
        o = L.LossOut(_p(dlogits), dlogits.stride(0) if dlogits is not None else 0,
                      _dtype_code(dlogits.dtype) if dlogits is not None else 0, 0,
                      _p(outs.get("cur_lp")), _p(outs.get("lse")), _p(outs.get("behav")),
                      _p(outs["obj"]), _p(outs.get("coef")), _p(outs["flags"]), _p(out4))
        return b, c, o

    def alloc_outputs(self, n_tok: int, device, coef=False, lse=True, behav=True):
        f = lambda dt: torch.empty(n_tok, dtype=dt, device=device)
        outs = {"cur_lp": f(torch.float32), "obj": f(torch.float64), "flags": f(torch.uint8)}
        if lse:
            outs["lse"] = f(torch.float32)
        if behav:
            outs["behav"] = f(torch.float32)
        if coef:
            outs["coef"] = f(torch.float64)
        return outs

    def loss_chunk_fused(self, logits, batch, cfg, outs, *, dlogits=None, row_base=0,
                         total_tokens=None, is_enabled=True,
                         behav_mode=L.COPRIS_BEHAV_RECOMPUTED, out4=None, stream=None):
        """Launch the fused kernel on one chunk of rows (no sync). ``out4`` (a
        device f64[4], with the LAST chunk) also reduces rows [0, row_base + n)
        — in the same launch for small batches (copris_loss_out.out4)."""
        T = total_tokens if total_tokens is not None else batch.loss_tokens()
        b, c, o = self._structs(logits, batch, cfg, is_enabled, behav_mode, T, row_base, dlogits,
                                outs, out4)
        self._call(self.lib.copris_is_loss_fused(self.h, C.byref(b), C.byref(c), C.byref(o),
                                                 self._stream(stream)))

    def loss_chunk_unfused(self, logits, batch, cfg, outs, *, dlogits=None, row_base=0,
                           total_tokens=None, is_enabled=True,
                           behav_mode=L.COPRIS_BEHAV_RECOMPUTED, out4=None, stream=None):
        """K1 -> K2 -> K3 on one chunk of rows (no sync); ``out4`` as for the fused path."""
        T = total_tokens if total_tokens is not None else batch.loss_tokens()
        n = logits.shape[0]
        sl = slice(row_base, row_base + n)
        cur, lse = outs["cur_lp"][sl], outs["lse"][sl]
        self.sequence_logprobs(logits, batch.target[sl], stream=stream, out_lp=cur, out_lse=lse)
        behav = outs["behav"][sl]
        self._call(self.lib.copris_behaviour_concat(
            self.h, _p(batch.stage[sl]), batch.cur_stage, _p(batch.buffered_lp[sl]), _p(cur),
            int(is_enabled), behav_mode, n, _p(behav), None, self._stream(stream)))
        b, c, o = self._structs(logits, batch, cfg, is_enabled, behav_mode, T, row_base, dlogits,
                                outs, out4)
        # K3 indexes its per-token inputs by the packed index: pass the full arrays
        self._call(self.lib.copris_is_loss_bwd(self.h, C.byref(b), C.byref(c), _p(outs["cur_lp"]),
                                               _p(outs["lse"]), _p(outs["behav"]), C.byref(o),
                                               self._stream(stream)))

    def reduce(self, outs, n_tok: int, out4: torch.Tensor, row_base=0, stream=None):
        obj = outs["obj"][row_base:row_base + n_tok]
        flags = outs["flags"][row_base:row_base + n_tok]
        self._call(self.lib.copris_loss_reduce(self.h, _p(obj), _p(flags), n_tok, _p(out4),
                                               self._stream(stream)))

    @_on_stream
    def grpo_step_loss(self, logits: torch.Tensor, batch: PackedBatch, cfg: ClipConfig = None,
                       *, is_enabled: bool = True, behav_mode: int = L.COPRIS_BEHAV_RECOMPUTED,
                       fused: bool = True, dlogits: Optional[torch.Tensor] = None,
                       dlogits_dtype: Optional[torch.dtype] = None, want_grad: bool = True,
                       total_tokens: Optional[int] = None, coef: bool = False,
                       stream=None) -> GrpoStepResult:
        """grpo.hpp:117-185 over a resident [T x V] logits tensor.

        loss = -(1/T) sum_t obj_t; dlogits rows = d loss / d logits. ``total_tokens``
        overrides T (the GLOBAL token count when the batch is a shard). With
        ``batch.loss_mask`` T counts the unmasked tokens and masked tokens are
        left out as if absent (obj 0, zero dlogits row, not counted).
        """
        cfg = cfg or ClipConfig()
        cfg.validate()
        if batch.n_traj == 0:
            raise ConfigError("grpo_step_loss requires a non-empty batch")
        if batch.n_tok == 0:
            raise ConfigError("grpo_step_loss batch has no tokens")
        if logits.shape[0] != batch.n_tok:
            raise ContractViolation("log-prob vectors must align with token count")
        T = total_tokens if total_tokens is not None else batch.loss_tokens()
        if T == 0:
            raise ConfigError("grpo_step_loss batch has no tokens")
        if want_grad and dlogits is None:
            dlogits = torch.empty(logits.shape, dtype=dlogits_dtype or logits.dtype,
                                  device=logits.device)
        outs = self.alloc_outputs(batch.n_tok, logits.device, coef=coef)
        run = self.loss_chunk_fused if fused else self.loss_chunk_unfused
        out4 = torch.empty(4, dtype=torch.float64, device=logits.device)
        # one call: the reduction rides along (in the loss launch when small)
        run(logits, batch, cfg, outs, dlogits=dlogits if want_grad else None, row_base=0,
            total_tokens=T, is_enabled=is_enabled, behav_mode=behav_mode, out4=out4, stream=stream)
        self.check(stream)
        o = out4.cpu().tolist()
        return GrpoStepResult(loss=-o[0] * (1.0 / T), dlogits=dlogits if want_grad else None,
                              token_count=int(o[1]), objective=o[0], stale_tokens=int(o[2]),
                              clipped_tokens=int(o[3]), cur_lp=outs["cur_lp"],
                              behav=outs.get("behav"), obj=outs["obj"], flags=outs["flags"],
                              coef=outs.get("coef"), lse=outs.get("lse"))


class HostWorkspace:
    """Device workspace for the host-buffer drop-in copris_grpo_step_loss_host
    (host arrays in, host loss/counts/dlogits out; chunked, 3-stream pipeline)."""

    def __init__(self, ctx: Copris, chunk_rows: int, vocab: int, max_tokens: int, max_traj: int,
                 logits_dtype=torch.bfloat16, dlogits_dtype=torch.bfloat16):
        self.ctx = ctx
        self.vocab = vocab
        self.logits_dtype, self.dlogits_dtype = logits_dtype, dlogits_dtype
        h = C.c_void_p()
        ctx._call(ctx.lib.copris_workspace_create(ctx.h, chunk_rows, vocab, _dtype_code(logits_dtype),
                                                  _dtype_code(dlogits_dtype), max_tokens, max_traj,
                                                  C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.copris_workspace_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def grpo_step_loss(self, logits: torch.Tensor, tok_off, target, stage, buffered_lp,
                       cur_stage: int, *, adv=None, rewards=None, group_off=None,
                       adv_epsilon: float = 1e-6, ref_lp=None, cfg: ClipConfig = None,
                       is_enabled: bool = True, behav_mode: int = L.COPRIS_BEHAV_RECOMPUTED,
                       total_tokens: int = 0, dlogits: Optional[torch.Tensor] = None,
                       cur_lp: Optional[torch.Tensor] = None) -> dict:
        """All tensors are CPU tensors (pin them for overlapped copies)."""
        cfg = cfg or ClipConfig()
        cfg.validate()
        n_tok, v = logits.shape
        hb = L.HostBatch(_p(logits), logits.stride(0), _dtype_code(logits.dtype), v, n_tok,
                         tok_off.numel() - 1, _p(tok_off), _p(target), _p(stage), _p(buffered_lp),
                         _p(ref_lp), _p(adv), _p(rewards), _p(group_off),
                         (group_off.numel() - 1) if group_off is not None else 0, adv_epsilon,
                         cur_stage, 0)
        c = L.LossCfg(cfg.clip_low, cfg.clip_high, cfg.kl_coeff, cfg.entropy_coeff, int(is_enabled),
                      behav_mode, total_tokens)
        r = L.HostResult(_p(dlogits), dlogits.stride(0) if dlogits is not None else 0,
                         _dtype_code(dlogits.dtype) if dlogits is not None else 0, 0, _p(cur_lp),
                         0.0, 0.0, 0, 0, 0)
        self.ctx._call(self.ctx.lib.copris_grpo_step_loss_host(self.ctx.h, self.h, C.byref(hb),
                                                               C.byref(c), C.byref(r)))
        return {"loss": r.loss, "objective": r.objective, "token_count": r.token_count,
                "stale_tokens": r.stale_tokens, "clipped_tokens": r.clipped_tokens}
