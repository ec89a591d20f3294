"""Adam (grpo.hpp:187-240) and CPRSCKPT checkpoints (io.hpp:397-438).

CPU: our checkpoint writer produces the reference's bytes exactly and both
readers accept each other's files; GPU: the Adam kernel reproduces the
reference optimizer bit for bit over several steps."""
import os

import numpy as np
import pytest

from paper_2511_05589_b200 import ConfigError
from paper_2511_05589_b200.optim import AdamConfig, read_checkpoint, write_checkpoint


def test_checkpoint_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    dims = (3, 5, 7, 2)
    logits = rng.normal(size=3 * 5 * 7)
    p = str(tmp_path / "c.bin")
    write_checkpoint(p, logits, dims, version=42, seed=777)
    back, d, v, s = read_checkpoint(p)
    assert d == dims and v == 42 and s == 777
    np.testing.assert_array_equal(back, logits)
    assert os.path.getsize(p) == 8 + 4 + 8 + 8 + 16 + 8 * logits.size


def test_checkpoint_matches_reference_bytes(tmp_path, reference):
    rng = np.random.default_rng(1)
    dims = (4, 8, 6, 4)
    logits = rng.normal(size=4 * 8 * 6)
    mine, theirs = str(tmp_path / "mine.bin"), str(tmp_path / "ref.bin")
    write_checkpoint(mine, logits, dims, 9, 123)
    reference.write_checkpoint(theirs, dims, logits, 9, 123)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    back, d, v, s = reference.read_checkpoint(mine, logits.size)
    np.testing.assert_array_equal(back, logits)
    assert (d, v, s) == (dims, 9, 123)


def test_checkpoint_errors(tmp_path):
    p = str(tmp_path / "bad.bin")
    open(p, "wb").write(b"NOTACKPT" + b"\0" * 40)
    with pytest.raises(ConfigError, match="bad checkpoint magic"):
        read_checkpoint(p)
    good = str(tmp_path / "good.bin")
    write_checkpoint(good, np.zeros(2 * 2 * 3), (2, 2, 3, 1), 0, 0)
    data = open(good, "rb").read()
    open(p, "wb").write(data[:-8])
    with pytest.raises(ConfigError, match="truncated checkpoint"):
        read_checkpoint(p)
    with pytest.raises(ConfigError, match="cannot read checkpoint"):
        read_checkpoint(str(tmp_path / "missing.bin"))


def test_adam_config_validation():
    for bad in (dict(lr=-1), dict(beta1=1.0), dict(beta2=-0.1), dict(eps=0.0), dict(weight_decay=-1)):
        with pytest.raises(ConfigError):
            AdamConfig(**bad).validate()


@pytest.mark.gpu
def test_adam_kernel_bit_identical_to_reference(ctx, reference):
    import torch
    from paper_2511_05589_b200.optim import AdamOptimizer
    rng = np.random.default_rng(2)
    dims = (4, 8, 6, 4)
    n = 4 * 8 * 6
    params = rng.normal(size=n)
    grads = rng.normal(size=(3, n))
    cfg = AdamConfig(lr=3e-2, weight_decay=0.01)
    opt = AdamOptimizer(ctx, cfg)
    p = torch.from_numpy(params.copy()).cuda()
    for k in range(3):
        opt.update(p, torch.from_numpy(grads[k]).cuda())
    ref = reference.adam(dims, params, grads, lr=3e-2, wd=0.01)
    np.testing.assert_array_equal(p.cpu().numpy(), ref)
    assert opt.version == 3


@pytest.mark.gpu
def test_host_adam_bit_identical_to_reference(ctx, reference):
    """copris_adam_host (the AdamDropIn behind trainer.hpp:177) on host arrays:
    bitwise the reference AdamOptimizer over several updates; size mismatch is
    the reference's ContractViolation."""
    from paper_2511_05589_b200.errors import ContractViolation
    from paper_2511_05589_b200.optim import HostAdamOptimizer
    rng = np.random.default_rng(5)
    dims = (4, 8, 6, 4)
    n = 4 * 8 * 6
    params = rng.normal(size=n)
    grads = rng.normal(size=(4, n))
    opt = HostAdamOptimizer(ctx, AdamConfig(lr=3e-2, weight_decay=0.01))
    p = params.copy()
    for k in range(4):
        opt.update(p, grads[k].copy())
    np.testing.assert_array_equal(p, reference.adam(dims, params, grads, lr=3e-2, wd=0.01))
    assert opt.version == 4 and opt.t == 4
    with pytest.raises(ContractViolation, match="gradient shape mismatch"):
        opt.update(np.zeros(n + 1), np.zeros(n + 1))
    opt.close()
