"""CPU: the host rollout scheduler is bit-exact
with the reference RolloutEngine (rollout.hpp:125-386).

  * replay: tests/golden/engine_stream.jsonl.gz is the reference engine's own
    event stream (8 scenarios: copris / naive_partial / synchronous, staleness
    eviction, groups of 2..8), recorded by oracle/engine_check.cpp. Every call is
    replayed through the C-ABI engine and every decision (admissions, refills,
    batch formation and order, members, resume queue, evictions) must match;
  * direct: oracle/_ref/engine_check drives the reference engine and the C++
    engine side by side and compares ~14M decisions/queries (when built).
"""
import gzip
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2511_05589_b200 import ConfigError, ContractViolation
from paper_2511_05589_b200.engine import RolloutEngine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STREAM = os.path.join(ROOT, "tests", "golden", "engine_stream.jsonl.gz")
CHECK = os.path.join(ROOT, "oracle", "_ref", "engine_check")


def _scenarios():
    cur = None
    with gzip.open(STREAM, "rt") as f:
        for line in f:
            ev = json.loads(line)
            if ev["op"] == "create":
                if cur:
                    yield cur
                cur = [ev]
            else:
                cur.append(ev)
    if cur:
        yield cur


SCEN = list(_scenarios())


@pytest.mark.parametrize("events", SCEN, ids=[s[0]["scenario"] for s in SCEN])
def test_replay_reference_event_stream(events):
    c = events[0]
    eng = RolloutEngine(mode=c["mode"], concurrency=c["concurrency"], batch_prompts=c["batch_prompts"],
                        rollouts_per_prompt=c["rollouts"], max_response_len=c["horizon"],
                        max_staleness=c["staleness"], vocab=c["vocab"], seed=c["seed"])
    batches = 0
    for ev in events[1:]:
        op = ev["op"]
        if op == "begin_stage":
            assert eng.begin_stage(ev["version"]) == ev["admitted"]
        elif op == "append":
            eng.append_token(ev["id"], ev["token"], ev["logprob"])
        elif op == "complete":
            assert eng.complete_trajectory(ev["id"]) == ev["ready"]
        elif op == "refill":
            assert eng.refill_active() == ev["admitted"]
        elif op == "early_terminate":
            b = eng.early_terminate()
            assert b.rollout_version == ev["version"]
            assert [int(g) for g in b.group_ids] == [g["group"] for g in ev["groups"]]
            assert [int(x) for x in b.group_class] == [g["class"] for g in ev["groups"]]
            members = [int(x) for x in b.traj_ids]
            assert members == [m for g in ev["groups"] for m in g["members"]]
            assert eng.ids("resume_queue") == ev["resume"]
            batches += 1
        elif op == "end":
            assert eng.ids("evicted") == ev["evicted"]
            assert len(eng.ids("consumed")) == ev["consumed"]
    assert batches >= 10


def test_packed_batch_layout_matches_segments():
    """early_terminate packs members in batch order: stage ids expand the
    segment versions, buffered_lp is concat_segments (trajectory.hpp:69-75)."""
    events = SCEN[2]  # copris with staleness eviction: multi-stage trajectories
    c = events[0]
    eng = RolloutEngine(mode=c["mode"], concurrency=c["concurrency"], batch_prompts=c["batch_prompts"],
                        rollouts_per_prompt=c["rollouts"], max_response_len=c["horizon"],
                        max_staleness=c["staleness"], vocab=c["vocab"], seed=c["seed"])
    appended = {}
    multi = 0
    for ev in events[1:]:
        if ev["op"] == "begin_stage":
            eng.begin_stage(ev["version"])
            version = ev["version"]
        elif ev["op"] == "append":
            eng.append_token(ev["id"], ev["token"], ev["logprob"])
            appended.setdefault(ev["id"], []).append((ev["token"], ev["logprob"], version))
        elif ev["op"] == "complete":
            eng.complete_trajectory(ev["id"])
        elif ev["op"] == "refill":
            eng.refill_active()
        elif ev["op"] == "early_terminate":
            b = eng.early_terminate()
            for i, tid in enumerate(b.traj_ids):
                a, z = b.tok_off[i], b.tok_off[i + 1]
                recs = appended[int(tid)]
                assert list(b.tokens[a:z]) == [r[0] for r in recs]
                np.testing.assert_array_equal(b.buffered_lp[a:z], np.float32([r[1] for r in recs]))
                np.testing.assert_array_equal(b.stage[a:z], np.uint32([r[2] for r in recs]))
                multi += len(set(r[2] for r in recs)) > 1
            assert b.offpolicy_token_fraction() == float((b.stage < b.rollout_version).mean())
    assert multi > 0


def test_engine_errors_follow_the_reference():
    eng = RolloutEngine(concurrency=4, batch_prompts=1, rollouts_per_prompt=2, max_response_len=3)
    ids = eng.begin_stage(0)
    with pytest.raises(ContractViolation, match="previous stage still has in-flight trajectories"):
        eng.begin_stage(1)
    with pytest.raises(ContractViolation, match="token out of vocabulary"):
        eng.append_token(ids[0], 6, -1.0)
    with pytest.raises(ContractViolation, match="cannot complete an unterminated trajectory"):
        eng.complete_trajectory(ids[0])
    with pytest.raises(ContractViolation, match="early_terminate before B groups are done"):
        eng.early_terminate()
    with pytest.raises(ContractViolation, match="unknown trajectory id"):
        eng.append_token(999, 0, -1.0)
    with pytest.raises(ConfigError, match="naive_partial initial dispatch"):
        RolloutEngine(mode=1, concurrency=2, batch_prompts=4, rollouts_per_prompt=4)
    with pytest.raises(ConfigError, match="engine.concurrency must be >= 1"):
        RolloutEngine(concurrency=0)


def test_side_by_side_with_the_reference_engine():
    assert os.path.exists(CHECK), "oracle/_ref/engine_check not built (needs /root/reference at build time)"
    p = subprocess.run([CHECK], capture_output=True, text=True, timeout=300)
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert p.returncode == 0 and res["mismatches"] == 0, p.stderr[-2000:]
    assert res["checks"] > 1_000_000


def test_small_id_buffer_leaves_engine_untouched():
    """copris_engine_begin_stage / _refill_active check the caller's id buffer
    against the admission bound max(concurrency, B*N) BEFORE admitting: a
    too-small buffer fails with COPRIS_E_INVALID and the engine state is
    unchanged, so the same call then succeeds (engine_capi.cpp:70)."""
    import ctypes as C
    from paper_2511_05589_b200 import _lib as L
    eng = RolloutEngine(concurrency=12, batch_prompts=2, rollouts_per_prompt=4,
                        max_response_len=8, vocab=6, seed=3)
    ref = RolloutEngine(concurrency=12, batch_prompts=2, rollouts_per_prompt=4,
                        max_response_len=8, vocab=6, seed=3)
    small = (C.c_uint64 * 4)()
    n = C.c_int64()
    rc = eng.lib.copris_engine_begin_stage(eng.h, C.c_uint64(1), small, 4, C.byref(n))
    assert rc == L.COPRIS_E_INVALID
    assert eng.begin_stage(1) == ref.begin_stage(1)
    rc = eng.lib.copris_engine_refill_active(eng.h, small, 4, C.byref(n))
    assert rc == L.COPRIS_E_INVALID
    assert eng.refill_active() == ref.refill_active()
