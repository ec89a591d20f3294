"""GPU: the reference training loop with the GPU loss AND the GPU Adam in it.

oracle/_ref/trainer_loop_check (reference headers + include/copris_b200/
grpo_dropin.hpp, linked against libcopris_b200.so) restates Trainer::train_step
(trainer.hpp:120-178) with grpo_step_loss -> DropIn (trainer.hpp:176) and
adam_.update -> AdamDropIn (trainer.hpp:177), so the GPU gradient and update
drive the next rollout, and runs it beside the UNMODIFIED reference Trainer.
While the two runs form the same batches (ids, tokens, segment versions and
lengths) the losses must agree within 1e-5 (relative); the step at which the
scheduler first forms a different batch is reported, not asserted — the runs
are chaotic in the sampled tokens (a gradient that differs in the 7th digit
moves a token once a uniform draw lands that close to a CDF boundary). Plus
the GPU form of acceptance criterion C2 (acceptance_main.cpp:105-121): the
synchronous GPU loop against the reference's standalone on-policy loop."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "trainer_loop_check")
CASES = {"desk", "b16_c48", "b16_c48_is_off", "b16_c48_kl_entropy", "v64_h16_c128", "desk_synchronous"}


def test_reference_trainer_loop_with_gpu_loss_and_adam():
    assert os.path.exists(EXE), "oracle/_ref/trainer_loop_check not built (needs /root/reference at build time)"
    p = subprocess.run([EXE, "30"], capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert lines, p.stderr
    summaries = {l["case"]: l for l in lines if l.get("summary")}
    assert set(summaries) == CASES | {"c2_sync_vs_reference_loop"}, sorted(summaries)
    bad = [l for l in lines if not l["ok"]] if lines else []
    assert not bad, bad[:3]
    assert p.returncode == 0, p.stderr
    for name in CASES:
        s = summaries[name]
        # the first batch is formed before any update: identical by construction
        assert s["lockstep_steps"] >= 1, s
        assert s["worst_loss_rel_err_lockstep"] <= 1e-5, s
    print(json.dumps(list(summaries.values())))
