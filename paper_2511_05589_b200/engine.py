"""Host rollout buffer / concurrency-controlled scheduler over the C-ABI.

Mirrors the reference RolloutEngine (rollout.hpp:125-386): begin_stage,
refill_active, append_token, complete_trajectory, batch_ready,
early_terminate, and its queries. The implementation is C++
(include/copris_b200/rollout.hpp) with bit-exact decisions; early_terminate
returns the formed batch already packed for the device (include/copris_b200.h
layout), ready for packing.upload / the loss kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .grpo import _raise

SYNCHRONOUS, NAIVE_PARTIAL, COPRIS = 0, 1, 2
_LISTS = {"in_flight": 0, "resume_queue": 1, "buffered": 2, "consumed": 3, "evicted": 4}


@dataclass
class PackedTrainBatch:
    """TrainBatch (rollout.hpp:75-95) in the packed layout."""
    rollout_version: int
    group_off: np.ndarray
    group_ids: np.ndarray
    group_class: np.ndarray
    traj_ids: np.ndarray
    tok_off: np.ndarray
    tokens: np.ndarray
    seg_off: np.ndarray
    seg_ver: np.ndarray
    buffered_lp: np.ndarray
    stage: np.ndarray
    terminated: np.ndarray
    answer_target: np.ndarray

    @property
    def total_tokens(self) -> int:
        return int(self.tok_off[-1])

    def offpolicy_token_fraction(self, version: int | None = None) -> float:  # rollout.hpp:99-110
        v = self.rollout_version if version is None else version
        n = len(self.stage)
        return float((self.stage < v).sum()) / n if n else 0.0


class RolloutEngine:
    def __init__(self, mode=COPRIS, concurrency=16, batch_prompts=4, rollouts_per_prompt=4,
                 max_response_len=8, max_staleness=0, num_classes=4, horizon=None, vocab=6,
                 answer_vocab=4, seed=1):
        self.lib = L.load()
        cfg = L.EngineCfg(mode, concurrency, batch_prompts, rollouts_per_prompt, max_response_len,
                          max_staleness, num_classes,
                          horizon if horizon is not None else max_response_len, vocab,
                          answer_vocab, seed)
        h = C.c_void_p()
        self._call(self.lib.copris_engine_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.cap = max(1024, 4 * max(concurrency, batch_prompts * rollouts_per_prompt))

    def _call(self, rc):
        if rc:
            _raise(rc, self.lib)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.copris_engine_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _ids(self, fn, *args):
        buf = (C.c_uint64 * self.cap)()
        n = C.c_int64()
        # cap >= max(concurrency, B*N), the admission bound the C-ABI checks
        # before the engine admits anything
        self._call(fn(self.h, *args, buf, self.cap, C.byref(n)))
        return list(buf[: n.value])

    def begin_stage(self, version: int) -> list[int]:
        return self._ids(self.lib.copris_engine_begin_stage, C.c_uint64(version))

    def refill_active(self) -> list[int]:
        return self._ids(self.lib.copris_engine_refill_active)

    def append_token(self, traj_id: int, token: int, logprob: float) -> bool:
        term = C.c_int32()
        self._call(self.lib.copris_engine_append_token(self.h, traj_id, token, logprob, C.byref(term)))
        return bool(term.value)

    def complete_trajectory(self, traj_id: int) -> bool:
        ready = C.c_int32()
        self._call(self.lib.copris_engine_complete(self.h, traj_id, C.byref(ready)))
        return bool(ready.value)

    def batch_ready(self) -> bool:
        return bool(self.stats()["batch_ready"])

    def early_terminate(self) -> PackedTrainBatch:
        sizes = (C.c_int64 * 4)()
        self._call(self.lib.copris_engine_early_terminate(self.h, sizes))
        g, n, t, s = (int(x) for x in sizes)
        a = {
            "group_off": np.zeros(g + 1, np.int64), "group_ids": np.zeros(g, np.uint64),
            "group_class": np.zeros(g, np.int32), "traj_ids": np.zeros(n, np.uint64),
            "tok_off": np.zeros(n + 1, np.int64), "tokens": np.zeros(t, np.int32),
            "seg_off": np.zeros(s + 1, np.int64), "seg_ver": np.zeros(s, np.uint32),
            "buffered_lp": np.zeros(t, np.float32), "stage": np.zeros(t, np.uint32),
            "terminated": np.zeros(n, np.uint8), "answer_target": np.zeros(n, np.int32),
        }
        ph = L.PackedHostC(0, *[C.c_void_p(a[k].ctypes.data) for k in (
            "group_off", "group_ids", "group_class", "traj_ids", "tok_off", "tokens", "seg_off",
            "seg_ver", "buffered_lp", "stage", "terminated", "answer_target")])
        self._call(self.lib.copris_engine_batch_copy(self.h, C.byref(ph)))
        return PackedTrainBatch(rollout_version=int(ph.rollout_version), **a)

    def ids(self, which: str) -> list[int]:
        return self._ids(self.lib.copris_engine_list, _LISTS[which])

    def stats(self) -> dict:
        out = (C.c_int64 * 7)()
        self._call(self.lib.copris_engine_stats(self.h, out))
        keys = ("in_flight", "buffered_partial", "buffered_complete", "total_admitted",
                "stage_version", "batch_ready", "stage_tokens_in_buffer")
        return dict(zip(keys, (int(x) for x in out)))
