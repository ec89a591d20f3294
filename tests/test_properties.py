"""Property tests (hypothesis) of the host-side data path that feeds the
kernels: LPT sharding of whole prompt groups and the
rank-local packed arrays built from it. CPU only."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2511_05589_b200.sharding import lpt_shard, shard_arrays

group_tokens = st.lists(st.integers(min_value=0, max_value=10_000), min_size=0, max_size=64)


@settings(max_examples=200, deadline=None)
@given(group_tokens, st.integers(min_value=1, max_value=9))
def test_lpt_assigns_every_group_once_and_balances(gt, world):
    shards = lpt_shard(gt, world)
    assert len(shards) == world
    flat = [g for s in shards for g in s]
    assert sorted(flat) == list(range(len(gt)))           # each group exactly once
    assert all(s == sorted(s) for s in shards)             # batch order within a rank
    assert shards == lpt_shard(list(gt), world)            # deterministic
    loads = [sum(gt[g] for g in s) for s in shards]
    # list-scheduling bound: no rank exceeds the mean by more than one group
    if gt:
        assert max(loads) <= sum(gt) / world + max(gt) + 1e-9


@st.composite
def packed_batches(draw):
    n_groups = draw(st.integers(min_value=0, max_value=12))
    sizes = [draw(st.integers(min_value=1, max_value=5)) for _ in range(n_groups)]
    lens = [draw(st.integers(min_value=0, max_value=9)) for _ in range(sum(sizes))]
    world = draw(st.integers(min_value=1, max_value=5))
    return sizes, lens, world


@settings(max_examples=200, deadline=None)
@given(packed_batches())
def test_shard_arrays_partition_the_tokens(batch):
    sizes, lens, world = batch
    group_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(tok_off[-1])
    n = len(lens)
    target = np.arange(T, dtype=np.int32) * 7 + 3
    reward = np.arange(n, dtype=np.float64) + 0.5
    gt = tok_off[group_off[1:]] - tok_off[group_off[:-1]]
    seen = []
    for groups in lpt_shard(gt, world):
        l_tok, l_grp, pt, pj, idx = shard_arrays(tok_off, group_off, {"target": target},
                                                 {"reward": reward}, groups)
        assert l_tok[0] == 0 and l_tok[-1] == len(idx) and np.all(np.diff(l_tok) >= 0)
        assert l_grp[0] == 0 and l_grp[-1] == len(pj["reward"])
        np.testing.assert_array_equal(pt["target"], target[idx])
        # each local trajectory keeps its length and its reward
        trajs = [t for g in groups for t in range(group_off[g], group_off[g + 1])]
        np.testing.assert_array_equal(np.diff(l_tok), np.asarray(lens, np.int64)[trajs]
                                      if trajs else np.zeros(0, np.int64))
        np.testing.assert_array_equal(pj["reward"], reward[trajs] if trajs else np.zeros(0))
        seen.extend(idx.tolist())
    assert sorted(seen) == list(range(T))                  # every token on exactly one rank
