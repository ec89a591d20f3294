"""Host -> device packing of stage-tagged trajectories.

The reference keeps ragged per-trajectory vectors (Trajectory / LogProbSegment,
trajectory.hpp:13-65; TrainBatch, rollout.hpp:75-95). The device layout is the
packed SoA of include/copris_b200.h. Per-token stage ids are expanded on the
device from the segment tables (K2 copris_expand_segments), per-token
trajectory ids from tok_off, advantages from rewards (K3a).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from .grpo import Copris, PackedBatch


@dataclass
class LogProbSegment:
    """trajectory.hpp:15-18."""
    policy_version: int
    logprobs: list = field(default_factory=list)


@dataclass
class Trajectory:
    """trajectory.hpp:37-65 (the fields the loss path reads)."""
    traj_id: int = 0
    group_id: int = 0
    tokens: list = field(default_factory=list)
    terminated: bool = False
    segments: list = field(default_factory=list)
    target_token: int = 0  # Question::target_token of its prompt

    def token_count(self) -> int:
        return len(self.tokens)

    def stage_span(self) -> int:
        return len(self.segments)

    def check_invariants(self) -> None:  # trajectory.hpp:51-64
        from .errors import ContractViolation
        total, prev, first = 0, 0, True
        for seg in self.segments:
            if not seg.logprobs:
                raise ContractViolation("log-prob segment must be non-empty")
            if not first and not seg.policy_version > prev:
                raise ContractViolation("segment versions must strictly increase")
            prev, first = seg.policy_version, False
            total += len(seg.logprobs)
        if total != len(self.tokens):
            raise ContractViolation("segment lengths must sum to token count")


def concat_segments_host(traj: Trajectory) -> list:
    """trajectory.hpp:69-75 on the host (used to fill buffered_lp)."""
    out = []
    for seg in traj.segments:
        out.extend(seg.logprobs)
    return out


@dataclass
class PackedHost:
    tok_off: np.ndarray
    group_off: np.ndarray
    target: np.ndarray
    seg_off: np.ndarray
    seg_ver: np.ndarray
    buffered_lp: np.ndarray
    terminated: np.ndarray
    answer_target: np.ndarray


def pack_groups(groups: Sequence[Sequence[Trajectory]]) -> PackedHost:
    """Pack groups (batch order) of members (ascending traj_id) into SoA."""
    tok_off, group_off, seg_off = [0], [0], [0]
    target, seg_ver, blp, term, ans = [], [], [], [], []
    for g in groups:
        for t in g:
            target.extend(t.tokens)
            for seg in t.segments:
                seg_off.append(seg_off[-1] + len(seg.logprobs))
                seg_ver.append(seg.policy_version)
                blp.extend(seg.logprobs)
            tok_off.append(len(target))
            term.append(1 if t.terminated else 0)
            ans.append(t.target_token)
        group_off.append(len(tok_off) - 1)
    return PackedHost(np.asarray(tok_off, np.int64), np.asarray(group_off, np.int64),
                      np.asarray(target, np.int32), np.asarray(seg_off, np.int64),
                      np.asarray(seg_ver, np.uint32), np.asarray(blp, np.float32),
                      np.asarray(term, np.uint8), np.asarray(ans, np.int32))


def _dev(a, device):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def upload(ctx: Copris, tok_off, group_off, target, buffered_lp, cur_stage: int, *,
           stage=None, seg_off=None, seg_ver=None, adv=None, reward=None,
           adv_epsilon: float = 1e-6, ref_lp=None, device=None) -> PackedBatch:
    """Copy a packed host batch to the device and derive the per-token
    metadata there. Give either per-token ``stage`` or segment tables, and
    either ``adv`` or ``reward`` (advantages are then computed on the device)."""
    device = device if device is not None else torch.device("cuda", ctx.device)
    d_tok_off = _dev(np.asarray(tok_off, np.int64), device)
    d_group_off = _dev(np.asarray(group_off, np.int64), device)
    d_target = _dev(np.asarray(target, np.int32), device)
    n_tok = int(d_target.numel())
    if stage is not None:
        d_stage = _dev(np.asarray(stage, np.uint32).view(np.int32), device)
    else:
        d_stage = ctx.expand_segments(_dev(np.asarray(seg_off, np.int64), device),
                                      _dev(np.asarray(seg_ver, np.uint32).view(np.int32), device),
                                      n_tok)
    d_blp = _dev(np.asarray(buffered_lp, np.float32), device)
    d_tok_traj = ctx.token_traj(d_tok_off, n_tok)
    if adv is not None:
        d_adv = _dev(np.asarray(adv, np.float64), device)
    else:
        d_adv = ctx.compute_advantages(_dev(np.asarray(reward, np.float64), device), d_group_off,
                                       adv_epsilon, group_off_host=[int(x) for x in group_off])
    d_ref = _dev(np.asarray(ref_lp, np.float32), device) if ref_lp is not None else None
    return PackedBatch(d_tok_off, d_group_off, d_target, d_stage, d_blp, d_tok_traj, d_adv,
                       int(cur_stage), d_ref, [int(x) for x in group_off])
