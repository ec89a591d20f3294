"""ctypes bindings for the CPU checker — TEST INFRASTRUCTURE ONLY.

Two checkers live here:
  * ``Oracle``    — oracle/build/libcopris_oracle.so, the C restatement
                    (copris_oracle.c) of the reference hot path;
  * ``Reference`` — oracle/_ref/libcopris_ref.so, the reference's own headers
                    compiled read-only through oracle/ref_harness.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg / reference
arm may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libcopris_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcopris_ref.so")

E_CONTRACT, E_CONFIG = 1, 2


class ContractViolation(Exception):
    """Mirror of copris::ContractViolation (common.hpp:9-12)."""


class ConfigError(Exception):
    """Mirror of copris::ConfigError (common.hpp:15-18)."""


def _raise(rc: int, msg: str):
    if rc == E_CONTRACT:
        raise ContractViolation(msg)
    if rc == E_CONFIG:
        raise ConfigError(msg)
    raise RuntimeError(msg)


def build_oracle() -> None:
    """Compile the checker libraries (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
U32 = C.c_uint32
D = C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _oracle_batch(C.Structure):
    _fields_ = [("logits", P), ("ld", I64), ("vocab", I32), ("n_tok", I64), ("n_traj", I64),
                ("tok_off", P), ("target", P), ("stage", P), ("cur_stage", U32),
                ("buffered_lp", P), ("ref_lp", P), ("adv", P)]


class _oracle_cfg(C.Structure):
    _fields_ = [("clip_low", D), ("clip_high", D), ("kl_coeff", D), ("entropy_coeff", D),
                ("is_enabled", C.c_int), ("behav_mode", C.c_int)]


class _oracle_result(C.Structure):
    _fields_ = [("loss", D), ("objective", D), ("dlogits", P), ("cur_lp", P), ("behav", P),
                ("weight", P), ("clipped", P), ("obj", P), ("stale_tokens", I64),
                ("clipped_tokens", I64)]


@dataclass
class LossResult:
    loss: float
    objective: float = 0.0
    dlogits: np.ndarray | None = None
    cur_lp: np.ndarray | None = None
    behav: np.ndarray | None = None
    weight: np.ndarray | None = None
    clipped: np.ndarray | None = None
    obj: np.ndarray | None = None
    stale_tokens: int = 0
    clipped_tokens: int = 0
    seconds: float = 0.0
    extra: dict = field(default_factory=dict)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """The C restatement (oracle/copris_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        self.lib = C.CDLL(path)
        L = self.lib
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_logprob_gather.argtypes = [P, I64, P, I64, I32, P]
        L.oracle_behaviour.argtypes = [P, U32, P, P, C.c_int, C.c_int, I64, P, P]
        L.oracle_behaviour.restype = None
        L.oracle_advantages.argtypes = [P, P, I64, D, P]
        L.oracle_terminal_rewards.argtypes = [P, P, I64, P, P, I32, P]
        L.oracle_is_loss.argtypes = [C.POINTER(_oracle_batch), C.POINTER(_oracle_cfg),
                                     C.POINTER(_oracle_result)]

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.oracle_last_error().decode())

    def logprob_gather(self, logits, target):
        logits = _f64(logits)
        target = np.ascontiguousarray(target, dtype=np.int32)
        n, v = logits.shape
        out = np.zeros(n, np.float64)
        self._check(self.lib.oracle_logprob_gather(_ptr(logits), v, _ptr(target), n, v, _ptr(out)))
        return out

    def behaviour(self, stage, cur_stage, buffered_lp, cur_lp, is_enabled=True, behav_mode=0):
        stage = np.ascontiguousarray(stage, dtype=np.uint32)
        buffered_lp, cur_lp = _f64(buffered_lp), _f64(cur_lp)
        out = np.zeros(len(stage), np.float64)
        stale = C.c_int64(0)
        self.lib.oracle_behaviour(_ptr(stage), cur_stage, _ptr(buffered_lp), _ptr(cur_lp),
                                  int(is_enabled), behav_mode, len(stage), _ptr(out),
                                  C.byref(stale))
        return out, stale.value

    def advantages(self, rewards, group_off, adv_epsilon=1e-6):
        rewards = _f64(rewards)
        group_off = np.ascontiguousarray(group_off, dtype=np.int64)
        out = np.zeros(len(rewards), np.float64)
        self._check(self.lib.oracle_advantages(_ptr(rewards), _ptr(group_off), len(group_off) - 1,
                                               adv_epsilon, _ptr(out)))
        return out

    def terminal_rewards(self, tokens, tok_off, terminated, answer_target, eos_token):
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
        terminated = np.ascontiguousarray(terminated, dtype=np.uint8)
        answer_target = np.ascontiguousarray(answer_target, dtype=np.int32)
        out = np.zeros(len(tok_off) - 1, np.float64)
        self._check(self.lib.oracle_terminal_rewards(_ptr(tokens), _ptr(tok_off), len(tok_off) - 1,
                                                     _ptr(terminated), _ptr(answer_target),
                                                     eos_token, _ptr(out)))
        return out

    def is_loss(self, logits, tok_off, target, stage, cur_stage, buffered_lp, adv,
                clip_low=0.2, clip_high=0.28, kl_coeff=0.0, entropy_coeff=0.0,
                is_enabled=True, ref_lp=None, want_dlogits=True, behav_mode=0) -> LossResult:
        logits = _f64(logits)
        n, v = logits.shape
        tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
        target = np.ascontiguousarray(target, dtype=np.int32)
        stage = np.ascontiguousarray(stage, dtype=np.uint32)
        buffered_lp, adv, ref_lp = _f64(buffered_lp), _f64(adv), _f64(ref_lp)
        b = _oracle_batch(_ptr(logits), v, v, n, len(tok_off) - 1, _ptr(tok_off), _ptr(target),
                          _ptr(stage), cur_stage, _ptr(buffered_lp), _ptr(ref_lp), _ptr(adv))
        cfg = _oracle_cfg(clip_low, clip_high, kl_coeff, entropy_coeff, int(is_enabled), behav_mode)
        res = LossResult(0.0)
        res.dlogits = np.zeros((n, v), np.float64) if want_dlogits else None
        res.cur_lp = np.zeros(n, np.float64)
        res.behav = np.zeros(n, np.float64)
        res.weight = np.zeros(n, np.float64)
        res.clipped = np.zeros(n, np.uint8)
        res.obj = np.zeros(n, np.float64)
        out = _oracle_result(0.0, 0.0, _ptr(res.dlogits), _ptr(res.cur_lp), _ptr(res.behav),
                             _ptr(res.weight), _ptr(res.clipped), _ptr(res.obj), 0, 0)
        self._check(self.lib.oracle_is_loss(C.byref(b), C.byref(cfg), C.byref(out)))
        res.loss, res.objective = out.loss, out.objective
        res.stale_tokens, res.clipped_tokens = out.stale_tokens, out.clipped_tokens
        return res


class Reference:
    """The reference's own code (oracle/_ref/libcopris_ref.so)."""

    available = os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_logprob_gather.argtypes = [P, I64, P, I64, I32, P]
        L.ref_advantages.argtypes = [P, P, I64, D, P]
        L.ref_terminal_rewards.argtypes = [P, P, I64, P, P, I32, P]
        L.ref_is_loss.argtypes = [P, I64, I32, I64, P, P, P, U32, P, P, P, D, D, D, D, C.c_int,
                                  C.c_int, P, P, P, P, P]
        L.ref_adam.argtypes = [P, P, P, C.c_int, D, D, D, D, D]
        L.ref_write_checkpoint.argtypes = [C.c_char_p, P, P, C.c_uint64, C.c_uint64]
        L.ref_read_checkpoint.argtypes = [C.c_char_p, P, P, C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64)]

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.ref_last_error().decode())

    def logprob_gather(self, logits, target):
        logits = _f64(logits)
        target = np.ascontiguousarray(target, dtype=np.int32)
        n, v = logits.shape
        out = np.zeros(n, np.float64)
        self._check(self.lib.ref_logprob_gather(_ptr(logits), v, _ptr(target), n, v, _ptr(out)))
        return out

    def advantages(self, rewards, group_off, adv_epsilon=1e-6):
        rewards = _f64(rewards)
        group_off = np.ascontiguousarray(group_off, dtype=np.int64)
        out = np.zeros(len(rewards), np.float64)
        self._check(self.lib.ref_advantages(_ptr(rewards), _ptr(group_off), len(group_off) - 1,
                                            adv_epsilon, _ptr(out)))
        return out

    def terminal_rewards(self, tokens, tok_off, terminated, answer_target, eos_token):
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
        terminated = np.ascontiguousarray(terminated, dtype=np.uint8)
        answer_target = np.ascontiguousarray(answer_target, dtype=np.int32)
        out = np.zeros(len(tok_off) - 1, np.float64)
        self._check(self.lib.ref_terminal_rewards(_ptr(tokens), _ptr(tok_off), len(tok_off) - 1,
                                                  _ptr(terminated), _ptr(answer_target),
                                                  eos_token, _ptr(out)))
        return out

    def is_loss(self, logits, tok_off, target, stage, cur_stage, buffered_lp, adv,
                clip_low=0.2, clip_high=0.28, kl_coeff=0.0, entropy_coeff=0.0,
                is_enabled=True, ref_logits=None, current_from_recompute=True,
                want_dlogits=True) -> LossResult:
        logits = _f64(logits)
        n, v = logits.shape
        tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
        target = np.ascontiguousarray(target, dtype=np.int32)
        stage = np.ascontiguousarray(stage, dtype=np.uint32)
        buffered_lp, adv, ref_logits = _f64(buffered_lp), _f64(adv), _f64(ref_logits)
        loss = C.c_double(0.0)
        secs = C.c_double(0.0)
        res = LossResult(0.0)
        res.dlogits = np.zeros((n, v), np.float64) if want_dlogits else None
        res.cur_lp = np.zeros(n, np.float64)
        res.behav = np.zeros(n, np.float64)
        self._check(self.lib.ref_is_loss(
            _ptr(logits), v, v, len(tok_off) - 1, _ptr(tok_off), _ptr(target), _ptr(stage),
            cur_stage, _ptr(buffered_lp), _ptr(ref_logits), _ptr(adv), clip_low, clip_high,
            kl_coeff, entropy_coeff, int(is_enabled), int(current_from_recompute),
            C.byref(loss), _ptr(res.dlogits), _ptr(res.cur_lp), _ptr(res.behav), C.byref(secs)))
        res.loss, res.seconds = loss.value, secs.value
        return res

    def adam(self, dims, params, grads, lr=5e-2, b1=0.9, b2=0.999, eps=1e-8, wd=0.01):
        """AdamOptimizer::update applied len(grads) times (grpo.hpp:203-233)."""
        d = np.ascontiguousarray(dims, np.int32)
        p = np.array(params, np.float64)
        g = np.ascontiguousarray(grads, np.float64)
        self._check(self.lib.ref_adam(_ptr(d), _ptr(p), _ptr(g), len(g), lr, b1, b2, eps, wd))
        return p

    def write_checkpoint(self, path, dims, logits, version, seed):
        d = np.ascontiguousarray(dims, np.int32)
        a = np.ascontiguousarray(logits, np.float64)
        self._check(self.lib.ref_write_checkpoint(path.encode(), _ptr(d), _ptr(a), version, seed))

    def read_checkpoint(self, path, n):
        d = np.zeros(4, np.int32)
        out = np.zeros(n, np.float64)
        ver, seed = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_read_checkpoint(path.encode(), _ptr(d), _ptr(out), C.byref(ver),
                                                 C.byref(seed)))
        return out, tuple(int(x) for x in d), ver.value, seed.value
