"""ctypes binding of the product C-ABI (include/copris_b200.h).

The shared library is built in-tree (paper_2511_05589_b200/libcopris_b200.so,
``make -C paper_2511_05589_b200/csrc``). There is no fallback: if the library
is missing, loading raises, and every compute entry point needs a B200.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COPRIS_LIB_PATH") or os.path.join(HERE, "libcopris_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "copris_b200.h")

COPRIS_OK, COPRIS_E_CONTRACT, COPRIS_E_CONFIG, COPRIS_E_CUDA, COPRIS_E_INVALID = range(5)
COPRIS_BF16, COPRIS_F32 = 0, 1
COPRIS_BEHAV_RECOMPUTED, COPRIS_BEHAV_RECORDED = 0, 1
COPRIS_FLAG_STALE, COPRIS_FLAG_CLIPPED, COPRIS_FLAG_MASKED = 1, 2, 4

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U32 = C.c_uint32
D = C.c_double


class LossBatch(C.Structure):
    _fields_ = [("logits", P), ("ld", I64), ("logits_dtype", I32), ("vocab", I32),
                ("n_rows", I64), ("row_base", I64), ("target", P), ("stage", P),
                ("buffered_lp", P), ("ref_lp", P), ("tok_traj", P), ("adv", P),
                ("cur_stage", U32), ("_pad", U32), ("loss_mask", P)]


class LossCfg(C.Structure):
    _fields_ = [("clip_low", D), ("clip_high", D), ("kl_coeff", D), ("entropy_coeff", D),
                ("is_enabled", I32), ("behav_mode", I32), ("total_tokens", I64)]


class LossOut(C.Structure):
    _fields_ = [("dlogits", P), ("ld_dlogits", I64), ("dlogits_dtype", I32), ("_pad", I32),
                ("cur_lp", P), ("lse", P), ("behav", P), ("obj", P), ("coef", P), ("flags", P),
                ("out4", P)]


class HostBatch(C.Structure):
    _fields_ = [("logits", P), ("ld", I64), ("logits_dtype", I32), ("vocab", I32),
                ("n_tok", I64), ("n_traj", I64), ("tok_off", P), ("target", P), ("stage", P),
                ("buffered_lp", P), ("ref_lp", P), ("adv", P), ("rewards", P), ("group_off", P),
                ("n_groups", I64), ("adv_epsilon", D), ("cur_stage", U32), ("_pad", U32)]


class HostResult(C.Structure):
    _fields_ = [("dlogits", P), ("ld_dlogits", I64), ("dlogits_dtype", I32), ("_pad", I32),
                ("cur_lp", P), ("loss", D), ("objective", D), ("token_count", I64),
                ("stale_tokens", I64), ("clipped_tokens", I64)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", D), ("beta1", D), ("beta2", D), ("eps", D), ("weight_decay", D)]


class EngineCfg(C.Structure):
    _fields_ = [("mode", I32), ("concurrency", I32), ("batch_prompts", I32),
                ("rollouts_per_prompt", I32), ("max_response_len", I32), ("max_staleness", I32),
                ("num_classes", I32), ("horizon", I32), ("vocab", I32), ("answer_vocab", I32),
                ("seed", C.c_uint64)]


class PackedHostC(C.Structure):
    _fields_ = [("rollout_version", C.c_uint64), ("group_off", P), ("group_ids", P),
                ("group_class", P), ("traj_ids", P), ("tok_off", P), ("tokens", P), ("seg_off", P),
                ("seg_ver", P), ("buffered_lp", P), ("stage", P), ("terminated", P),
                ("answer_target", P)]


_SIGS = {
    "copris_abi_version": ([], C.c_int),
    "copris_last_error": ([], C.c_char_p),
    "copris_ctx_create": ([C.c_int, C.POINTER(P)], C.c_int),
    "copris_ctx_destroy": ([P], C.c_int),
    "copris_ctx_check": ([P, P], C.c_int),
    "copris_logprob_gather": ([P, P, I64, I32, P, I64, I32, P, P, P], C.c_int),
    "copris_lmhead_num_vtiles": ([I32], I32),
    "copris_lmhead_logits": ([P, P, I64, P, I64, I64, I32, I32, P, P, I64, P, P], C.c_int),
    "copris_lse_merge": ([P, P, I32, P, I64, P, I64, I32, P, P, P], C.c_int),
    "copris_lmhead_dhidden_splits": ([P, I64, I32], I32),
    "copris_lmhead_dhidden": ([P, P, I64, P, I64, I64, I32, I32, P, I64, P, P], C.c_int),
    "copris_allreduce_scalars": ([P, P, P], C.c_int),
    "copris_nccl_comm_init_all": ([I32, P, P], C.c_int),
    "copris_nccl_unique_id": ([P], C.c_int),
    "copris_nccl_comm_init_rank": ([I32, I32, P, I32, P], C.c_int),
    "copris_nccl_comm_destroy": ([P], C.c_int),
    "copris_lmhead_dweight": ([P, P, I64, P, I64, I64, I32, I32, P, I64, P], C.c_int),
    "copris_expand_segments": ([P, P, P, I64, P, P], C.c_int),
    "copris_behaviour_concat": ([P, P, U32, P, P, I32, I32, I64, P, P, P], C.c_int),
    "copris_terminal_rewards": ([P, P, P, I64, P, P, I32, P, P], C.c_int),
    "copris_group_advantages": ([P, P, P, P, I64, D, P, P], C.c_int),
    "copris_token_traj": ([P, P, I64, I64, P, P], C.c_int),
    "copris_is_loss_fused": ([P, C.POINTER(LossBatch), C.POINTER(LossCfg), C.POINTER(LossOut), P],
                             C.c_int),
    "copris_is_loss_bwd": ([P, C.POINTER(LossBatch), C.POINTER(LossCfg), P, P, P,
                            C.POINTER(LossOut), P], C.c_int),
    "copris_loss_reduce": ([P, P, P, I64, P, P], C.c_int),
    "copris_workspace_create": ([P, I64, I32, I32, I32, I64, I64, C.POINTER(P)], C.c_int),
    "copris_workspace_destroy": ([P], C.c_int),
    "copris_grpo_step_loss_host": ([P, P, C.POINTER(HostBatch), C.POINTER(LossCfg),
                                    C.POINTER(HostResult)], C.c_int),
    "copris_ctx_trace_read": ([P, P, C.c_int], C.c_int),
    "copris_ctx_set_option": ([P, C.c_char_p, I64], C.c_int),
    "copris_ctx_last_fused_reduce": ([P], C.c_int),
    "copris_ctx_get_option": ([P, C.c_char_p, C.POINTER(I64)], C.c_int),
    "copris_adam_update": ([P, P, P, P, P, I64, I64, C.POINTER(AdamCfg), P], C.c_int),
    "copris_adam_host_create": ([P, I64, C.POINTER(AdamCfg), C.POINTER(P)], C.c_int),
    "copris_adam_host_update": ([P, P, P, I64], C.c_int),
    "copris_adam_host_steps": ([P, C.POINTER(I64)], C.c_int),
    "copris_adam_host_destroy": ([P], C.c_int),
    "copris_checkpoint_write": ([C.c_char_p, P, P, C.c_uint64, C.c_uint64], C.c_int),
    "copris_checkpoint_read": ([C.c_char_p, P, P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], C.c_int),
    "copris_engine_create": ([C.POINTER(EngineCfg), C.POINTER(P)], C.c_int),
    "copris_engine_destroy": ([P], C.c_int),
    "copris_engine_begin_stage": ([P, C.c_uint64, P, I64, C.POINTER(I64)], C.c_int),
    "copris_engine_refill_active": ([P, P, I64, C.POINTER(I64)], C.c_int),
    "copris_engine_append_token": ([P, C.c_uint64, I32, D, C.POINTER(I32)], C.c_int),
    "copris_engine_complete": ([P, C.c_uint64, C.POINTER(I32)], C.c_int),
    "copris_engine_early_terminate": ([P, P], C.c_int),
    "copris_engine_batch_copy": ([P, C.POINTER(PackedHostC)], C.c_int),
    "copris_engine_list": ([P, I32, P, I64, C.POINTER(I64)], C.c_int),
    "copris_engine_stats": ([P, P], C.c_int),
    "copris_ctx_last_launch": ([P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_char_p)], C.c_int),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libcopris_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C paper_2511_05589_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def declared_symbols(header: str = HEADER) -> list[str]:
    """Function names declared by include/copris_b200.h."""
    import re
    with open(header) as f:
        text = f.read()
    return sorted(set(re.findall(r"^COPRIS_API\s+[\w\s\*]+?\b(copris_\w+)\s*\(", text, re.M)))
