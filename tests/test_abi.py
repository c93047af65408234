"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/spngd_b200.h; compute entry points fail loudly (no CPU
fallback) when no CUDA device is present."""
import ctypes as C
import os
import re

import pytest
import torch

from paper_2002_06015_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spngd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spngd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["spngd_factor_sym_batched", "spngd_damp_and_invert_batched", "spngd_spd_inverse_batched",
                 "spngd_precondition_update_batched", "spngd_bn_solve_update_batched", "spngd_bn_moments_batched",
                 "spngd_stat_distance_batched", "spngd_reduce_scatter_mean", "spngd_all_gather", "spngd_opt_step"]:
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(N.EXPORTS) <= set(declared_symbols())


def test_library_is_sm100a_only():
    assert b"sm_100a" in N.lib().spngd_version()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    h = C.c_void_p()
    rc = N.lib().spngd_ctx_create(0, None, C.byref(h))
    assert rc == 100  # SPNGD_ERR_CUDA
    assert b"no CPU fallback" in N.lib().spngd_last_error()
