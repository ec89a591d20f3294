"""CPU: the oracle (oracle/copris_oracle.c) pinned against the reference.

  * golden fixtures captured from the UNMODIFIED reference Trainer
    (tests/golden/trainer_*.json): loss, log-probs, behaviour log-probs,
    advantages, rewards and the off-policy fraction must match BIT FOR BIT;
    the table gradient (scatter-add of per-token rows) within 1e-15;
  * the reference's own known-answer tests (test_policy.cpp, test_grpo.cpp),
    restated against the oracle;
  * the reference compiled from its headers (oracle/_ref, when built) on
    random inputs, bit for bit.
"""
import math

import numpy as np
import pytest

from golden_io import all_steps, packed_step, scatter_table

STEPS = list(all_steps())


@pytest.mark.parametrize("name,step,fx,st", STEPS, ids=[f"{n}-{s}" for n, s, _, _ in STEPS])
def test_oracle_reproduces_reference_trainer(oracle, name, step, fx, st):
    ps = packed_step(fx, st)
    c = ps.clip
    res = oracle.is_loss(ps.logits, ps.tok_off, ps.target, ps.stage, ps.cur_stage,
                         ps.buffered_lp, ps.adv, c["clip_low"], c["clip_high"], c["kl_coeff"],
                         c["entropy_coeff"], ps.is_enabled,
                         ref_lp=ps.ref_lp if c["kl_coeff"] > 0 else None)
    assert res.loss == ps.loss                                 # grpo.hpp:183, bitwise
    np.testing.assert_array_equal(res.cur_lp, ps.current_lp)   # policy.hpp:160-173
    np.testing.assert_array_equal(res.behav, ps.stored_lp)     # trajectory.hpp:69-75 / trainer.hpp:149
    g = scatter_table(ps, res.dlogits)
    assert np.abs(g - ps.grad).max() <= 1e-15 * max(1.0, np.abs(ps.grad).max())
    adv = oracle.advantages(ps.reward, ps.group_off, c["adv_epsilon"])
    np.testing.assert_array_equal(adv, ps.adv)                 # grpo.hpp:51-65
    rew = oracle.terminal_rewards(ps.target, ps.tok_off, ps.terminated, ps.answer_target, ps.eos)
    np.testing.assert_array_equal(rew, ps.reward)              # grpo.hpp:35-47
    assert res.stale_tokens / len(ps.target) == ps.offpolicy_fraction  # rollout.hpp:99-110


def test_golden_fixtures_cover_the_stage_structure():
    """The fixtures exercise multi-stage trajectories, IS off, KL+entropy and
    long-tail lengths (BASELINE configs #1 and the K=3-4 stage case)."""
    max_span, names = 0, set()
    for name, _, fx, st in STEPS:
        names.add(name)
        for g in st["groups"]:
            for m in g["members"]:
                max_span = max(max_span, len(m["segments"]))
    assert max_span >= 4
    assert {"trainer_b16_c48_is_off.json", "trainer_b16_c48_kl_entropy.json",
            "trainer_lognormal_h64_c128.json"} <= names


# ---- known-answer tests restated from the reference's own suite -------------------

def test_zero_logits_uniform(oracle):  # test_policy.cpp:52-57
    z = np.zeros((3, 5))
    lp = oracle.logprob_gather(z, [0, 2, 4])
    assert np.all(np.abs(np.exp(lp) - 0.2) < 1e-15)


def test_saturated_logits(oracle):  # test_policy.cpp:59-65
    z = np.zeros((1, 4))
    z[0, 3] = 1e6
    assert np.exp(oracle.logprob_gather(z, [3]))[0] >= 1 - 1e-6


def test_logprobs_vs_long_double(oracle):  # test_policy.cpp:67-75,174-186
    rng = np.random.default_rng(0)
    for _ in range(50):
        z = rng.uniform(-3, 3, (4, 6))
        tgt = rng.integers(0, 6, 4)
        zl = z.astype(np.longdouble)
        e = np.exp(zl - zl.max(1, keepdims=True))
        ref = np.log(e[np.arange(4), tgt] / e.sum(1))
        assert np.all(np.abs(oracle.logprob_gather(z, tgt) - ref.astype(np.float64)) < 1e-12)


def test_empty_sequence(oracle):  # test_policy.cpp:151-155
    assert oracle.logprob_gather(np.zeros((0, 4)), np.zeros(0, np.int32)).size == 0


def test_out_of_vocab(oracle):  # policy.hpp:169
    from oracle.oracle import ContractViolation
    with pytest.raises(ContractViolation, match="token out of vocabulary"):
        oracle.logprob_gather(np.zeros((1, 4)), [4])


def test_uniform_rewards_zero_advantage(oracle):  # test_grpo.cpp:94-97
    assert np.all(oracle.advantages([1.0, 1.0, 1.0, 1.0], [0, 4]) == 0.0)


def test_two_member_group(oracle):  # test_grpo.cpp:99-106
    a = oracle.advantages([1.0, 0.0], [0, 2])
    assert abs(a[0] - 1) < 3e-6 and abs(a[1] + 1) < 3e-6


def test_balanced_group(oracle):  # test_grpo.cpp:108-115
    a = oracle.advantages([1.0, 1.0, 0.0, 0.0], [0, 4])
    assert np.all(np.abs(np.abs(a) - 1) < 3e-6)


def test_advantages_sum_to_zero(oracle):  # test_grpo.cpp:117-128
    rng = np.random.default_rng(17)
    for _ in range(100):
        g = int(rng.integers(2, 16))
        r = rng.integers(0, 2, g).astype(float)
        assert abs(oracle.advantages(r, [0, g]).sum()) < 1e-9


def test_group_of_one(oracle):  # test_grpo.cpp:130-133
    from oracle.oracle import ConfigError
    with pytest.raises(ConfigError):
        oracle.advantages([1.0], [0, 1])


def _single(oracle, cur_lp_logits_row, adv, blp, stage=0, cur_stage=1, **kw):
    z = np.asarray(cur_lp_logits_row, float)[None, :]
    return oracle.is_loss(z, [0, 1], [0], [stage], cur_stage, [blp], [adv], **kw)


def test_clipped_objective_kats(oracle):  # test_grpo.cpp:169-175
    # choose logits so that cur_lp = log(0.5) for token 0 of a binary row
    z = [0.0, 0.0]
    lp = math.log(0.5)
    for ratio, adv, expect in ((1.0, 0.7, 0.7), (1.0, -2.0, -2.0), (2.0, 1.0, 1.28),
                               (0.5, -1.0, -0.8)):
        r = _single(oracle, z, adv, lp - math.log(ratio))
        assert abs(r.objective - expect) < 1e-12, (ratio, adv, r.objective)


def test_on_policy_ratio_exactly_one(oracle):  # test_grpo.cpp:142-167, C3
    rng = np.random.default_rng(3)
    z = rng.normal(size=(6, 7))
    tgt = rng.integers(0, 7, 6)
    cur = oracle.logprob_gather(z, tgt)
    stage = np.array([3, 3, 3, 5, 5, 5], np.uint32)
    blp = cur.copy()
    blp[:3] += 0.1  # stale segment recorded under an older policy
    r = oracle.is_loss(z, [0, 6], tgt, stage, 5, blp, [0.7])
    ratios = np.exp(r.cur_lp - r.behav)
    assert np.all(ratios[3:] == 1.0)
    assert np.all(np.abs(ratios[:3] - np.exp(-0.1)) < 1e-12)


def test_zero_advantage_zero_loss_and_grad(oracle):  # test_grpo.cpp:293-303
    rng = np.random.default_rng(4)
    z = rng.normal(size=(8, 5))
    tgt = rng.integers(0, 5, 8)
    r = oracle.is_loss(z, [0, 4, 8], tgt, np.zeros(8, np.uint32), 1,
                       rng.normal(size=8) - 2.0, [0.0, 0.0])
    assert r.loss == 0.0 and np.all(r.dlogits == 0.0)


def test_empty_batch_is_config_error(oracle):  # test_grpo.cpp:305-310
    from oracle.oracle import ConfigError
    with pytest.raises(ConfigError):
        oracle.is_loss(np.zeros((0, 3)), [0], np.zeros(0, np.int32), np.zeros(0, np.uint32), 0,
                       np.zeros(0), np.zeros(0))


def test_gradient_matches_finite_differences(oracle):  # test_grpo.cpp:312-343, C1
    rng = np.random.default_rng(5)
    worst = 0.0
    for trial in range(20):
        T, V = 6, 5
        z = rng.uniform(-1, 1, (T, V))
        tgt = rng.integers(0, V, T)
        tok_off = [0, 3, 6]
        stage = np.array([0, 0, 1, 0, 1, 1], np.uint32)
        adv = rng.normal(size=2)
        cur = oracle.logprob_gather(z, tgt)
        blp = cur + rng.uniform(-0.3, 0.3, T)
        kw = dict(kl_coeff=0.1, entropy_coeff=0.01) if trial % 5 == 4 else {}
        ref_lp = cur + 0.05 if kw else None
        # stored log-probs are recorded values, constant in z (RECORDED mode)
        kw["behav_mode"] = 1
        r = oracle.is_loss(z, tok_off, tgt, stage, 1, blp, adv, ref_lp=ref_lp, **kw)
        h = 1e-5
        fd = np.zeros_like(z)
        for i in range(T):
            for k in range(V):
                zp, zm = z.copy(), z.copy()
                zp[i, k] += h
                zm[i, k] -= h
                lp = oracle.is_loss(zp, tok_off, tgt, stage, 1, blp, adv, ref_lp=ref_lp, **kw).loss
                lm = oracle.is_loss(zm, tok_off, tgt, stage, 1, blp, adv, ref_lp=ref_lp, **kw).loss
                fd[i, k] = (lp - lm) / (2 * h)
        worst = max(worst, np.abs(fd - r.dlogits).max() / max(1.0, np.abs(fd).max()))
    assert worst < 1e-4


# ---- the reference itself, compiled from its headers (oracle/_ref) -----------------

@pytest.mark.parametrize("seed", range(6))
def test_oracle_equals_compiled_reference(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(2, 300))
    n_traj = 4
    lens = rng.integers(1, 12, n_traj)
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(tok_off[-1])
    z = rng.normal(0, 2, (T, V))
    tgt = rng.integers(0, V, T).astype(np.int32)
    stage = np.zeros(T, np.uint32)
    for i in range(n_traj):  # 1-3 segments per trajectory
        k = int(rng.integers(1, 4))
        cuts = np.sort(rng.integers(tok_off[i], tok_off[i + 1], k - 1)) if k > 1 else []
        ver = 9 - k
        start = tok_off[i]
        for c in list(cuts) + [tok_off[i + 1]]:
            stage[start:c] = ver
            start, ver = c, ver + 1
        stage[start:tok_off[i + 1]] = 8
    cur = oracle.logprob_gather(z, tgt)
    blp = np.where(stage < 8, cur + rng.uniform(-0.3, 0.3, T), cur)
    adv = oracle.advantages(rng.integers(0, 2, n_traj).astype(float), [0, 2, 4])
    kl = 0.1 if seed % 3 == 2 else 0.0
    ent = 0.01 if seed % 2 == 1 else 0.0
    zr = z + rng.normal(0, 0.1, z.shape)
    ref_lp = oracle.logprob_gather(zr, tgt) if kl else None
    for is_on in (True, False):
        o = oracle.is_loss(z, tok_off, tgt, stage, 8, blp, adv, kl_coeff=kl, entropy_coeff=ent,
                           is_enabled=is_on, ref_lp=ref_lp)
        r = reference.is_loss(z, tok_off, tgt, stage, 8, blp, adv, kl_coeff=kl, entropy_coeff=ent,
                              is_enabled=is_on, ref_logits=zr if kl else None)
        assert o.loss == r.loss
        np.testing.assert_array_equal(o.cur_lp, r.cur_lp)
        np.testing.assert_array_equal(o.behav, r.behav)
        np.testing.assert_array_equal(o.dlogits, r.dlogits)
    np.testing.assert_array_equal(oracle.advantages([1.0, 0.0, 1.0, 1.0], [0, 2, 4]),
                                  reference.advantages([1.0, 0.0, 1.0, 1.0], [0, 2, 4]))
