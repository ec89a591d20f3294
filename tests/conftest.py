import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    # a hard failure, not a skip: the reference-compiled checkers travel with the
    # snapshot (oracle/_ref/ is git-ignored, not gpurun-ignored), so a missing
    # build means the parity evidence is missing
    assert Reference.available, "oracle/_ref/libcopris_ref.so not built: run __graft_entry__.build() with /root/reference present"
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    import torch
    from paper_2511_05589_b200 import Copris
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return Copris(0)
