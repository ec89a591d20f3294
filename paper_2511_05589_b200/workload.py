"""Synthetic workloads of the BASELINE.json configs.

Shapes follow the reference's own length law and batch structure:
  * lengths   lognormal(mu, sigma) rounded and clamped to [1, Lmax] — the
              rule of drawn_length (cluster.hpp:57-65);
  * batch     P prompt groups x G members, packed group by group, members in
              ascending id (TrainBatch, rollout.hpp:75-95);
  * stages    K segments per trajectory at uniform split points, versions
              cur_stage-K+1 .. cur_stage; only the last is current
              (LogProbSegment, trajectory.hpp:13-65);
  * rewards   Bernoulli(0.5) per trajectory (acceptance_main.cpp:60);
  * logits    ~N(0, 2^2) bf16, target logit +4, one row in 64 saturated (+30);
  * stale log-probs = current log-prob + U(-0.3, 0.3) (acceptance_main.cpp:66)
              pushed out of a 1e-4 guard band around log(1 - clip_low) and
              log(1 + clip_high) so fp32 and fp64 agree on every clip branch.
This is input generation, not a checker: nothing here computes the loss.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class HostBatch:
    tok_off: np.ndarray      # [n+1] int64
    group_off: np.ndarray    # [P+1] int64
    target: np.ndarray       # [T] int32
    stage: np.ndarray        # [T] uint32
    reward: np.ndarray       # [n] f64
    cur_stage: int
    vocab: int
    seg_off: np.ndarray      # [n_seg+1] int64 token offsets of segments
    seg_ver: np.ndarray      # [n_seg] uint32

    @property
    def n_tok(self) -> int:
        return int(self.tok_off[-1])

    @property
    def n_traj(self) -> int:
        return len(self.tok_off) - 1

    def group_tokens(self) -> np.ndarray:
        return self.tok_off[self.group_off[1:]] - self.tok_off[self.group_off[:-1]]


CONFIGS = {
    # BASELINE.json configs[1]: 128 prompts x 8, max 8k, vocab 151,936, 2 stages
    "grpo_128x8_v151936": dict(P=128, G=8, mu=math.log(2048), sigma=1.0, lmax=8192,
                               vocab=151936, stages=(1, 2), stale_prob=0.5),
    # configs[2]: long tail, 3-4 stages per trajectory
    "grpo_128x8_v151936_longtail_4stage": dict(P=128, G=8, mu=math.log(2048), sigma=1.5,
                                               lmax=8192, vocab=151936, stages=(3, 4),
                                               stale_prob=1.0),
    # configs[3]: 512 x 16, max 16k, ONE global batch sharded over 1/2/4/8 GPUs
    # (strong scaling: P is the global prompt count, not per rank)
    "grpo_512x16_v151936": dict(P=512, G=16, mu=math.log(4096), sigma=1.0, lmax=16384,
                                vocab=151936, stages=(1, 2), stale_prob=0.5, strong=True),
}
# configs[4]: vocab 32,000 short-response sweep (fixed lengths 256 .. 4k) at
# 128 x 8 per GPU, plus a one-group variant (8 trajectories) that exposes the
# per-step launch and reduction overhead
for _L in (256, 512, 1024, 2048, 4096):
    CONFIGS[f"grpo_128x8_v32000_L{_L}"] = dict(P=128, G=8, fixed_len=_L, vocab=32000,
                                                stages=(1, 2), stale_prob=0.5)
    CONFIGS[f"grpo_1x8_v32000_L{_L}"] = dict(P=1, G=8, fixed_len=_L, vocab=32000,
                                              stages=(1, 2), stale_prob=0.5)

BASELINE_INDEX = {"grpo_128x8_v151936": 1, "grpo_128x8_v151936_longtail_4stage": 2,
                  "grpo_512x16_v151936": 3}


def describe(name: str) -> str:
    """One-line workload description for bench output (BASELINE.json configs[i])."""
    c = CONFIGS[name]
    idx = BASELINE_INDEX.get(name, 4)
    if "fixed_len" in c:
        shape = f"{c['P']} prompts x {c['G']} responses, fixed length {c['fixed_len']}"
    else:
        shape = f"{c['P']} prompts x {c['G']} responses, lognormal lengths max {c['lmax']}"
    k0, k1 = c["stages"]
    stages = f"{k0}-{k1} rollout stages" if k0 != k1 else f"{k0} rollout stages"
    per = "global batch sharded by prompt group" if c.get("strong") else "per GPU"
    return f"{name} (BASELINE.json configs[{idx}]: {shape}, vocab {c['vocab']}, {stages}) {per}"


def make_host_batch(seed: int, P: int, G: int, vocab: int, mu: float = 0.0, sigma: float = 0.0,
                    lmax: int = 8192, fixed_len: int | None = None, stages=(1, 2),
                    stale_prob: float = 0.5, cur_stage: int = 7) -> HostBatch:
    rng = np.random.default_rng(seed)
    n = P * G
    if fixed_len is not None:
        lengths = np.full(n, fixed_len, np.int64)
    else:
        lengths = np.clip(np.rint(np.exp(mu + sigma * rng.standard_normal(n))), 1, lmax).astype(np.int64)
    tok_off = np.zeros(n + 1, np.int64)
    tok_off[1:] = np.cumsum(lengths)
    group_off = np.arange(0, n + 1, G, dtype=np.int64)
    T = int(tok_off[-1])
    target = rng.integers(0, vocab, T, dtype=np.int64).astype(np.int32)
    stage = np.empty(T, np.uint32)
    seg_off, seg_ver = [0], []
    kmin, kmax = stages
    for i in range(n):
        L = int(lengths[i])
        k = 1
        if rng.random() < stale_prob:
            k = int(rng.integers(kmin, kmax + 1))
        k = max(1, min(k, L))
        cuts = np.sort(rng.choice(np.arange(1, L), size=k - 1, replace=False)) if k > 1 else []
        bounds = [0, *[int(c) for c in cuts], L]
        for j in range(k):
            ver = cur_stage - (k - 1 - j)
            a, b = tok_off[i] + bounds[j], tok_off[i] + bounds[j + 1]
            stage[a:b] = ver
            seg_off.append(int(b))
            seg_ver.append(ver)
    reward = rng.integers(0, 2, n).astype(np.float64)
    return HostBatch(tok_off, group_off, target, stage, reward, cur_stage, vocab,
                     np.asarray(seg_off, np.int64), np.asarray(seg_ver, np.uint32))


def make_logits(n_rows: int, vocab: int, target, seed: int, device="cpu",
                dtype=torch.bfloat16, row0: int = 0, ld: int | None = None) -> torch.Tensor:
    """~N(0, 2^2) logits, target logit +4, every 64th packed row saturated (+30).

    ``target`` is indexed by chunk-local row; ``row0`` is the packed index of
    row 0 (it selects which rows saturate). ``ld`` > vocab pads rows.
    """
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    width = ld if ld is not None else vocab
    z = torch.empty((n_rows, width), dtype=torch.float32, device=device)
    z.normal_(0.0, 2.0, generator=g)
    z = z[:, :vocab]
    tgt = torch.as_tensor(target, device=device).long()
    rows = torch.arange(n_rows, device=device)
    boost = torch.full((n_rows,), 4.0, device=device)
    boost[(rows + row0) % 64 == 0] = 30.0
    z[rows, tgt] += boost
    full = torch.zeros((n_rows, width), dtype=dtype, device=device)
    full[:, :vocab] = z.to(dtype)
    return full[:, :vocab] if ld is not None else full


def stale_logprobs(cur_lp: np.ndarray, stage: np.ndarray, cur_stage: int, seed: int,
                   clip_low: float = 0.2, clip_high: float = 0.28,
                   guard: float = 1e-4) -> np.ndarray:
    """buffered_lp: current log-prob for current-stage tokens (what the
    sampler records), current + U(-0.3,0.3) for stale ones, kept at least
    ``guard`` away from the clip thresholds in log-ratio space."""
    rng = np.random.default_rng(seed + 7919)
    cur = np.asarray(cur_lp, np.float64)
    noise = rng.uniform(-0.3, 0.3, cur.shape)
    for thr in (math.log(1.0 - clip_low), math.log(1.0 + clip_high)):
        # log ratio = cur - blp = -noise
        close = np.abs(-noise - thr) < guard
        noise[close] += np.where(-noise[close] > thr, -2 * guard, 2 * guard)
    out = np.where(np.asarray(stage) < cur_stage, cur + noise, cur)
    return out.astype(np.float32)
