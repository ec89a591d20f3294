"""Exception types mirroring the reference's (common.hpp:8-22)."""


class ContractViolation(Exception):
    """copris::ContractViolation — a precondition or structural invariant failed."""


class ConfigError(Exception):
    """copris::ConfigError — invalid or inconsistent configuration / empty batch."""


class CudaError(RuntimeError):
    """A CUDA runtime or launch failure inside libcopris_b200.so."""
