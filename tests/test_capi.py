"""CPU checks of the C-ABI boundary: the library loads, exports exactly what
include/copris_b200.h declares, the ctypes layouts match the C structs, and
compute entry points fail loudly (never silently) without a GPU."""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

from paper_2511_05589_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = L.load()
    declared = L.declared_symbols()
    assert len(declared) >= 15, declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/copris_b200.h but not exported"
    assert set(declared) == set(L._SIGS), "ctypes signatures out of sync with the header"
    assert lib.copris_abi_version() == 3


def test_exports_nothing_else():
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(L.declared_symbols()), exported ^ set(L.declared_symbols())


def test_struct_layouts_match_header():
    src = r'''
#include <stddef.h>
#include <stdio.h>
#include "copris_b200.h"
#define F(T, m) printf(#T "." #m " %zu\n", offsetof(T, m));
int main(void) {
  printf("copris_loss_batch %zu\n", sizeof(copris_loss_batch));
  printf("copris_loss_cfg %zu\n", sizeof(copris_loss_cfg));
  printf("copris_loss_out %zu\n", sizeof(copris_loss_out));
  printf("copris_host_batch %zu\n", sizeof(copris_host_batch));
  printf("copris_host_result %zu\n", sizeof(copris_host_result));
  F(copris_loss_batch, cur_stage) F(copris_loss_batch, adv) F(copris_loss_batch, tok_traj)
  F(copris_loss_cfg, total_tokens) F(copris_loss_cfg, behav_mode)
  F(copris_loss_out, flags) F(copris_loss_out, cur_lp) F(copris_loss_out, out4)
  F(copris_host_batch, adv_epsilon) F(copris_host_batch, cur_stage) F(copris_host_batch, group_off)
  F(copris_host_result, loss) F(copris_host_result, clipped_tokens)
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), c, "-o", exe],
                       check=True)
        got = dict(l.rsplit(" ", 1) for l in subprocess.run([exe], capture_output=True, text=True,
                                                             check=True).stdout.splitlines())
    assert int(got["copris_loss_batch"]) == C.sizeof(L.LossBatch)
    assert int(got["copris_loss_cfg"]) == C.sizeof(L.LossCfg)
    assert int(got["copris_loss_out"]) == C.sizeof(L.LossOut)
    assert int(got["copris_host_batch"]) == C.sizeof(L.HostBatch)
    assert int(got["copris_host_result"]) == C.sizeof(L.HostResult)
    for key, val in got.items():
        if "." in key:
            struct, field = key.split(".")
            cls = {"copris_loss_batch": L.LossBatch, "copris_loss_cfg": L.LossCfg,
                   "copris_loss_out": L.LossOut, "copris_host_batch": L.HostBatch,
                   "copris_host_result": L.HostResult}[struct]
            assert getattr(cls, field).offset == int(val), key


def test_header_compiles_as_c_and_cpp():
    for compiler, std in (("gcc", "-std=c99"), ("g++", "-std=c++17")):
        with tempfile.TemporaryDirectory() as d:
            src = os.path.join(d, "h.c" if compiler == "gcc" else "h.cpp")
            open(src, "w").write('#include "copris_b200.h"\nint main(void){return 0;}\n')
            subprocess.run([compiler, std, "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                            src, "-o", os.path.join(d, "h")], check=True)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = L.load()
    h = C.c_void_p()
    rc = lib.copris_ctx_create(0, C.byref(h))
    assert rc == L.COPRIS_E_CUDA
    assert lib.copris_last_error()
    from paper_2511_05589_b200 import Copris, CudaError
    with pytest.raises((CudaError, RuntimeError, AssertionError)):
        Copris(0)


def test_null_arguments_are_rejected_without_a_gpu():
    lib = L.load()
    assert lib.copris_is_loss_fused(None, None, None, None, None) == L.COPRIS_E_INVALID
    assert lib.copris_ctx_check(None, None) == L.COPRIS_E_INVALID
    assert b"null" in lib.copris_last_error()
