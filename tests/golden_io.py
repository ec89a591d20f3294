"""Loaders for the committed golden fixtures (tests/golden/).

``trainer_*.json`` were captured from the UNMODIFIED reference Trainer by
oracle/gen_golden.cpp (regenerate with ``tests/golden/make_golden.sh``). Each
captured step holds exactly what the reference passed to grpo_step_loss
(trainer.hpp:133-176) and what it returned. ``packed_step`` lays a step out in
the packed row-per-token form the GPU path consumes: token t of member i reads
the table row (class_i, t) (policy.hpp:31-33).
"""
from __future__ import annotations

import glob
import json
import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def trainer_fixtures():
    return sorted(glob.glob(os.path.join(GOLDEN, "trainer_*.json")))


def load(path):
    with open(path) as f:
        return json.load(f)


@dataclass
class PackedStep:
    vocab: int
    logits: np.ndarray          # [T, V] fp64 — gathered table rows
    ref_logits: np.ndarray      # [T, V] fp64 — version-0 snapshot rows (KL)
    tok_off: np.ndarray         # [n+1] int64
    group_off: np.ndarray       # [P+1] int64
    target: np.ndarray          # [T] int32
    stage: np.ndarray           # [T] uint32
    buffered_lp: np.ndarray     # [T] fp64  (concat_segments)
    cur_stage: int
    adv: np.ndarray             # [n] fp64
    reward: np.ndarray          # [n] fp64
    answer_target: np.ndarray   # [n] int32
    terminated: np.ndarray      # [n] uint8
    rows: np.ndarray            # [T] int64 table row index per token
    current_lp: np.ndarray      # [T] reference item.current_lp
    stored_lp: np.ndarray       # [T] reference item.stored_lp
    ref_lp: np.ndarray          # [T] reference item.ref_lp (empty if KL off)
    loss: float
    grad: np.ndarray            # [Q*H*V] reference table gradient
    clip: dict
    is_enabled: bool
    offpolicy_fraction: float
    eos: int


def packed_step(fx, step) -> PackedStep:
    pol = fx["policy"]
    Q, H, V = pol["num_classes"], pol["horizon"], pol["vocab"]
    table = np.asarray(step["params"], np.float64).reshape(Q * H, V)
    ref_table = np.asarray(fx["reference_params"], np.float64).reshape(Q * H, V)
    tok_off, group_off = [0], [0]
    target, stage, blp, adv, reward, rows, ans, term = [], [], [], [], [], [], [], []
    cur, sto, rlp = [], [], []
    for g in step["groups"]:
        for m in g["members"]:
            toks = m["tokens"]
            for t in range(len(toks)):
                rows.append(g["class_id"] * H + t)
            target += toks
            for s in m["segments"]:
                stage += [s["version"]] * len(s["logprobs"])
                blp += s["logprobs"]
            adv.append(m["advantage"])
            reward.append(m["reward"])
            ans.append(g["target_token"])
            term.append(1 if m["terminated"] else 0)
            cur += m["current_lp"]
            sto += m["stored_lp"]
            rlp += m["ref_lp"]
            tok_off.append(len(target))
        group_off.append(len(adv))
    rows = np.asarray(rows, np.int64)
    return PackedStep(
        vocab=V, logits=table[rows], ref_logits=ref_table[rows],
        tok_off=np.asarray(tok_off, np.int64), group_off=np.asarray(group_off, np.int64),
        target=np.asarray(target, np.int32), stage=np.asarray(stage, np.uint32),
        buffered_lp=np.asarray(blp, np.float64), cur_stage=step["rollout_version"],
        adv=np.asarray(adv, np.float64), reward=np.asarray(reward, np.float64),
        answer_target=np.asarray(ans, np.int32), terminated=np.asarray(term, np.uint8),
        rows=rows, current_lp=np.asarray(cur, np.float64), stored_lp=np.asarray(sto, np.float64),
        ref_lp=np.asarray(rlp, np.float64), loss=step["loss"],
        grad=np.asarray(step["grad"], np.float64), clip=fx["clip"],
        is_enabled=fx["is_enabled"], offpolicy_fraction=step["offpolicy_fraction"],
        eos=V - 1)


def all_steps():
    for path in trainer_fixtures():
        fx = load(path)
        for step in fx["steps"]:
            yield os.path.basename(path), step["step"], fx, step


def scatter_table(ps: PackedStep, dlogits: np.ndarray) -> np.ndarray:
    """Tabular adapter: scatter-add per-token dlogits rows into the table, in
    batch order (Appendix A.7 of SURVEY.md)."""
    V = ps.vocab
    grad = np.zeros_like(ps.grad).reshape(-1, V)
    for t, r in enumerate(ps.rows):
        grad[r] += dlogits[t]
    return grad.reshape(-1)
