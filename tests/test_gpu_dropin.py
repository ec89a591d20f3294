"""GPU: the reference Trainer with the C++ drop-in at its grpo_step_loss seam.

oracle/_ref/dropin_check (built from the UNMODIFIED reference headers plus
include/copris_b200/grpo_dropin.hpp, linked against libcopris_b200.so) runs
reference Trainer steps and, with the exact arguments trainer.hpp:176 passes,
compares the reference grpo_step_loss with the GPU path: loss within 1e-5 and
the table gradient within 1e-5 of its max, on every captured step; then runs
every case again on its own std::thread with its own context (the reference
CLI's one-Trainer-per-thread mode, copris_cli.cpp:98-115) and requires the GPU
losses to be bitwise the sequential ones."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_check")


def test_reference_trainer_with_gpu_dropin():
    assert os.path.exists(EXE), "oracle/_ref/dropin_check not built (hard failure, see conftest.reference)"
    p = subprocess.run([EXE, "--threads"], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert lines, p.stderr
    bad = [l for l in lines if not l["ok"]]
    assert not bad, bad[:3]
    assert p.returncode == 0, p.stderr
    cases = {"desk", "b16_c48", "b16_c48_is_off", "b16_c48_kl_entropy", "v64_h16_c128"}
    assert {l["case"] for l in lines if l["mode"] == "sequential"} == cases
    assert {l["case"] for l in lines if l["mode"] == "threaded_vs_sequential"} == cases
