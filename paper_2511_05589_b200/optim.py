"""The steps after the gradient: Adam with decoupled
weight decay on the device (AdamOptimizer, grpo.hpp:187-240; bit-identical
fp64) and the CPRSCKPT checkpoint format (io.hpp:397-438; byte-identical)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import ConfigError
from .grpo import Copris, _raise


@dataclass
class AdamConfig:
    """grpo.hpp:187-201."""
    lr: float = 5e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01

    def validate(self) -> None:
        if self.lr < 0.0:
            raise ConfigError("optimizer.lr must be >= 0")
        if not (0.0 <= self.beta1 < 1.0 and 0.0 <= self.beta2 < 1.0):
            raise ConfigError("optimizer betas must lie in [0, 1)")
        if self.eps <= 0.0:
            raise ConfigError("optimizer.eps must be > 0")
        if self.weight_decay < 0.0:
            raise ConfigError("optimizer.weight_decay must be >= 0")


class HostAdamOptimizer:
    """The whole AdamOptimizer object for a HOST parameter table (grpo.hpp:205-235)
    through copris_adam_host_*: the moments stay on the device, each update is one
    blocking call on fp64 numpy arrays (params updated in place) and bumps `version`."""

    def __init__(self, ctx: Copris, cfg: AdamConfig | None = None):
        self.ctx, self.cfg = ctx, cfg or AdamConfig()
        self.cfg.validate()
        self.h = None
        self.n = 0
        self.version = 0

    def update(self, params: np.ndarray, grad: np.ndarray) -> None:
        from .errors import ContractViolation
        if grad.size != params.size:
            raise ContractViolation("gradient shape mismatch")
        if params.dtype != np.float64 or grad.dtype != np.float64 or not params.flags.c_contiguous:
            raise ValueError("contiguous fp64 arrays expected (the reference's precision)")
        grad = np.ascontiguousarray(grad)
        if self.h is None:
            c = L.AdamCfg(self.cfg.lr, self.cfg.beta1, self.cfg.beta2, self.cfg.eps, self.cfg.weight_decay)
            h = C.c_void_p()
            self.ctx._call(self.ctx.lib.copris_adam_host_create(self.ctx.h, params.size, C.byref(c),
                                                                C.byref(h)))
            self.h, self.n = h, params.size
        self.ctx._call(self.ctx.lib.copris_adam_host_update(self.h, params.ctypes.data, grad.ctypes.data,
                                                            params.size))
        self.version += 1

    @property
    def t(self) -> int:
        if self.h is None:
            return 0
        t = C.c_int64()
        self.ctx._call(self.ctx.lib.copris_adam_host_steps(self.h, C.byref(t)))
        return t.value

    def close(self) -> None:
        if self.h is not None:
            self.ctx.lib.copris_adam_host_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AdamOptimizer:
    """AdamOptimizer::update on device fp64 tensors; each update bumps `version`."""

    def __init__(self, ctx: Copris, cfg: AdamConfig | None = None):
        self.ctx, self.cfg = ctx, cfg or AdamConfig()
        self.m = self.v = None
        self.t = 0
        self.version = 0

    def update(self, params: torch.Tensor, grad: torch.Tensor, stream=None) -> None:
        from .errors import ContractViolation
        if grad.numel() != params.numel():
            raise ContractViolation("gradient shape mismatch")
        if params.dtype != torch.float64 or grad.dtype != torch.float64:
            raise ValueError("fp64 tensors expected (the reference's precision)")
        if self.m is None:
            self.m = torch.zeros_like(params)
            self.v = torch.zeros_like(params)
        self.t += 1
        c = L.AdamCfg(self.cfg.lr, self.cfg.beta1, self.cfg.beta2, self.cfg.eps, self.cfg.weight_decay)
        p = lambda t: C.c_void_p(t.data_ptr())
        self.ctx._call(self.ctx.lib.copris_adam_update(self.ctx.h, p(params), p(grad), p(self.m), p(self.v),
                                                       params.numel(), self.t, C.byref(c),
                                                       self.ctx._stream(stream)))
        self.version += 1


def write_checkpoint(path: str, logits, dims, version: int, seed: int) -> None:
    """io.hpp:397-411: magic CPRSCKPT, schema, version, seed, dims[4], fp64 table."""
    lib = L.load()
    a = np.ascontiguousarray(logits.detach().cpu().numpy() if isinstance(logits, torch.Tensor) else logits,
                             dtype=np.float64)
    d = (C.c_int32 * 4)(*dims)
    rc = lib.copris_checkpoint_write(path.encode(), a.ctypes.data_as(C.c_void_p), d, version, seed)
    if rc:
        _raise(rc, lib)


def read_checkpoint(path: str):
    """io.hpp:413-438 -> (logits fp64 [Q*H*V], dims, version, seed)."""
    lib = L.load()
    d = (C.c_int32 * 4)()
    ver, sd = C.c_uint64(), C.c_uint64()
    rc = lib.copris_checkpoint_read(path.encode(), None, d, C.byref(ver), C.byref(sd))
    if rc:
        _raise(rc, lib)
    out = np.zeros(d[0] * d[1] * d[2], np.float64)
    rc = lib.copris_checkpoint_read(path.encode(), out.ctypes.data_as(C.c_void_p), d, C.byref(ver), C.byref(sd))
    if rc:
        _raise(rc, lib)
    return out, tuple(d), ver.value, sd.value
