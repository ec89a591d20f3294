"""GPU path vs the reference's own Trainer batches (tests/golden/trainer_*.json,
captured from the unmodified reference through Trainer::set_inspector).

The table logits are fp64 in the reference; the GPU reads them as f32, so
log-probs/loss/grad are compared within 1e-5 (row-scaled), while advantages,
rewards, stale masks and clip masks must be exact."""
import numpy as np
import pytest
import torch

from golden_io import all_steps, packed_step, scatter_table
from parity_util import assert_loss_close, assert_scalar_close

pytestmark = pytest.mark.gpu

STEPS = list(all_steps())


@pytest.mark.parametrize("name,step,fx,st", STEPS, ids=[f"{n}-{s}" for n, s, _, _ in STEPS])
@pytest.mark.parametrize("fused", [True, False])
def test_trainer_batch(ctx, oracle, name, step, fx, st, fused):
    from paper_2511_05589_b200 import ClipConfig
    from paper_2511_05589_b200.packing import upload
    ps = packed_step(fx, st)
    c = ps.clip
    kl = c["kl_coeff"] > 0
    ref_lp = None
    if kl:  # ref log-probs of the version-0 snapshot, as the GPU would get them from K1
        ref_lp = ps.ref_lp.astype(np.float32)
    batch = upload(ctx, ps.tok_off, ps.group_off, ps.target, ps.buffered_lp.astype(np.float32),
                   ps.cur_stage, stage=ps.stage, reward=ps.reward, adv_epsilon=c["adv_epsilon"],
                   ref_lp=ref_lp)
    # advantages recomputed on the device from the rewards: bit-exact
    np.testing.assert_array_equal(batch.adv.cpu().numpy(), ps.adv)
    logits = torch.from_numpy(ps.logits.astype(np.float32)).cuda()
    cfg = ClipConfig(c["clip_low"], c["clip_high"], c["kl_coeff"], c["entropy_coeff"],
                     c["adv_epsilon"])
    res = ctx.grpo_step_loss(logits, batch, cfg, is_enabled=ps.is_enabled, fused=fused,
                             dlogits_dtype=torch.float32)
    # oracle on the same f32-rounded logits (what the GPU saw)
    ref = oracle.is_loss(ps.logits.astype(np.float32).astype(np.float64), ps.tok_off, ps.target,
                         ps.stage, ps.cur_stage, ps.buffered_lp.astype(np.float32).astype(np.float64),
                         ps.adv, c["clip_low"], c["clip_high"], c["kl_coeff"], c["entropy_coeff"],
                         ps.is_enabled, ref_lp=None if ref_lp is None else ref_lp.astype(np.float64))
    assert_scalar_close(res.cur_lp.cpu().numpy(), ps.current_lp, what="cur_lp vs reference")
    assert_scalar_close(res.behav.cpu().numpy(), ps.stored_lp, what="stored_lp vs reference")
    assert_loss_close(res.loss, ps.loss, ref.obj, len(ps.target), what="loss vs reference")
    # off-policy fraction (rollout.hpp:99-110) from the stale flags: exact
    assert res.stale_tokens / res.token_count == ps.offpolicy_fraction
    np.testing.assert_array_equal((res.flags.cpu().numpy() >> 1) & 1, ref.clipped)
    # tabular adapter: scatter-add the per-token rows into the reference's table
    g = scatter_table(ps, res.dlogits.double().cpu().numpy())
    scale = np.abs(ps.grad).max()
    assert np.abs(g - ps.grad).max() <= 1e-5 * scale, "table gradient vs reference"
