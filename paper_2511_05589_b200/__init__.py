"""B200-native CoPRIS IS-corrected loss path (arXiv 2511.05589).

The product is libcopris_b200.so (hand-written sm_100a CUDA behind the C-ABI in
include/copris_b200.h). This package is the host-side mirror of the reference's
loss entry points over that ABI; there is no CPU compute path.
"""
from ._lib import (COPRIS_BEHAV_RECOMPUTED, COPRIS_BEHAV_RECORDED, COPRIS_FLAG_CLIPPED,
                   COPRIS_FLAG_STALE, LIB_PATH, load)
from .errors import ConfigError, ContractViolation, CudaError
from .grpo import ClipConfig, Copris, GrpoStepResult, PackedBatch

__all__ = [
    "COPRIS_BEHAV_RECOMPUTED", "COPRIS_BEHAV_RECORDED", "COPRIS_FLAG_CLIPPED",
    "COPRIS_FLAG_STALE", "LIB_PATH", "load", "ConfigError", "ContractViolation", "CudaError",
    "ClipConfig", "Copris", "GrpoStepResult", "PackedBatch",
]
