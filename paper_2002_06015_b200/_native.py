"""ctypes binding of libspngd_b200.so (the C ABI declared in include/spngd_b200.h).

The library is built in-tree by ``make -C paper_2002_06015_b200`` (see
``__graft_entry__.build``).  There is no fallback: if the library or a CUDA
device is missing, loading or the first call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspngd_b200.so")

_i64 = C.c_int64
_fp = C.c_void_p


class FactorReq(C.Structure):
    _fields_ = [("x", _fp), ("dim", _i64), ("hw", _i64), ("layout", _i64), ("lo", _i64),
                ("hi", _i64), ("scale", C.c_double), ("packed_out", _fp)]


class BnFullReq(C.Structure):
    _fields_ = [("gg", _fp), ("gb", _fp), ("c", _i64), ("lo", _i64), ("hi", _i64), ("packed_out", _fp)]


class BnFullUpdateReq(C.Structure):
    _fields_ = [("finv", _fp), ("ld", _i64), ("grad", _fp), ("c", _i64), ("gamma", _fp), ("beta", _fp),
                ("vgamma", _fp), ("vbeta", _fp), ("pg_out", _fp), ("pb_out", _fp)]


class BnGradReq(C.Structure):
    _fields_ = [("dy", _fp), ("xhat", _fp), ("M", _i64), ("c", _i64), ("S", _i64), ("gg", _fp), ("gb", _fp)]


class BnBackwardReq(C.Structure):
    _fields_ = [("dy", _fp), ("xhat", _fp), ("M", _i64), ("c", _i64), ("S", _i64), ("gg", _fp), ("gb", _fp),
                ("out3c", _fp), ("payload", _fp)]


class BnMomentsReq(C.Structure):
    _fields_ = [("gg", _fp), ("gb", _fp), ("c", _i64), ("lo", _i64), ("hi", _i64), ("out3c", _fp)]


class SpdReq(C.Structure):
    _fields_ = [("packed", _fp), ("n", _i64), ("damping", C.c_float), ("damping_dev", _fp),
                ("dense_out", _fp), ("ld", _i64), ("packed_out", _fp)]


class KronReq(C.Structure):
    _fields_ = [("A_packed", _fp), ("G_packed", _fp), ("a", _i64), ("g", _i64),
                ("Ainv_dense", _fp), ("lda", _i64), ("Ginv_dense", _fp), ("ldg", _i64),
                ("Ainv_packed", _fp), ("Ginv_packed", _fp), ("pi_out", _fp)]


class PrecondReq(C.Structure):
    _fields_ = [("Ginv", _fp), ("ldg", _i64), ("Ainv", _fp), ("lda", _i64), ("dW", _fp),
                ("g", _i64), ("a", _i64), ("P_out", _fp), ("W", _fp), ("V", _fp),
                ("rescale", C.c_int)]


class BnUpdateReq(C.Structure):
    _fields_ = [("m3c", _fp), ("grad", _fp), ("c", _i64), ("gamma", _fp), ("beta", _fp),
                ("vgamma", _fp), ("vbeta", _fp), ("pg_out", _fp), ("pb_out", _fp)]


class StatReq(C.Structure):
    _fields_ = [("x", _fp), ("x1", _fp), ("x2", _fp), ("n", _i64), ("kind", _i64), ("out4", _fp)]


class LayerDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("a", _i64), ("g", _i64), ("hw", _i64)]


class LayoutEntry(C.Structure):
    _fields_ = [("owner", C.c_int32), ("pad_", C.c_int32), ("off_A", _i64), ("off_G", _i64),
                ("off_M", _i64), ("off_dW", _i64), ("off_W", _i64)]


class OptConfig(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("rescale", C.c_int32), ("stale", C.c_int32),
                ("stale_alpha", C.c_double), ("batch", _i64), ("fisher_mode", C.c_int32),
                ("elem_size", C.c_int32), ("sgd", C.c_int32), ("bn_mode", C.c_int32),
                ("wgrad", C.c_int32), ("pad_", C.c_int32)]


class ConvGeom(C.Structure):  # spngd_conv_geom
    _fields_ = [("c_in", _i64), ("h", _i64), ("w", _i64), ("k", _i64), ("stride", _i64), ("pad", _i64)]


class Im2colReq(C.Structure):
    _fields_ = [("x", C.c_void_p), ("out", C.c_void_p), ("batch", _i64), ("geom", ConvGeom)]


class HostInput(C.Structure):  # spngd_host_input
    _fields_ = [("layer", C.c_int32), ("which", C.c_int32), ("host", C.c_void_p)]


class LedgerRowC(C.Structure):  # spngd_ledger_row
    _fields_ = [("step", _i64), ("stage", C.c_int32), ("collective", C.c_int32), ("id_kind", C.c_int32),
                ("layer", C.c_int32), ("elements", _i64), ("bytes", _i64), ("skipped", C.c_int32),
                ("pad_", C.c_int32)]


# status codes (include/spngd_b200.h) -> reference exception names (errors.hpp)
STATUS_NAMES = {
    1: "ShapeMismatch", 2: "NotPositiveDefinite", 3: "SingularBlock", 4: "ZeroReference",
    5: "EmptyBatch", 6: "MissingMcPass", 7: "StaleBeyondLimit", 8: "RefreshOutOfTurn",
    9: "IndivisibleBatch", 10: "MissingOwner", 11: "EmptyAccumulation", 100: "CudaError",
    101: "NcclError", 102: "InvalidArgument",
}

EXPORTS = [
    "spngd_last_error", "spngd_ctx_last_error", "spngd_version", "spngd_ctx_create", "spngd_ctx_destroy", "spngd_ctx_sync",
    "spngd_ctx_stream", "spngd_copy", "spngd_host_alloc", "spngd_host_free", "spngd_event_time",
    "spngd_factor_sym_batched", "spngd_bn_moments_batched", "spngd_bn_grad_reduce_batched",
    "spngd_bn_full_moments_batched", "spngd_bn_full_solve_update_batched",
    "spngd_spd_inverse_batched", "spngd_damp_and_invert_batched",
    "spngd_precondition_update_batched", "spngd_bn_solve_update_batched",
    "spngd_stat_distance_batched", "spngd_tracker_create", "spngd_tracker_destroy",
    "spngd_tracker_should_refresh", "spngd_tracker_on_refresh", "spngd_tracker_state",
    "spngd_nccl_unique_id", "spngd_ctx_init_comm", "spngd_reduce_scatter_mean", "spngd_all_gather",
    "spngd_plan_layout", "spngd_opt_create", "spngd_opt_destroy", "spngd_opt_buffer", "spngd_opt_owner", "spngd_opt_step",
    "spngd_opt_phase_ms", "spngd_opt_launch_count", "spngd_opt_stale_info", "spngd_opt_set_overlap", "spngd_opt_sync",
    "spngd_opt_enable_bn_inputs", "spngd_bn_backward_stats_batched", "spngd_opt_enable_raw_inputs_ex",
]


def build():
    subprocess.check_call(["make", "-s", "-j8", "-C", _HERE], stdout=subprocess.DEVNULL)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C {_HERE}` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def _declare(L):
    P = C.c_void_p
    sig = {
        "spngd_last_error": (C.c_char_p, []),
        "spngd_ctx_last_error": (C.c_char_p, [C.c_void_p]),
        "spngd_version": (C.c_char_p, []),
        "spngd_ctx_create": (C.c_int, [C.c_int, P, C.POINTER(P)]),
        "spngd_ctx_destroy": (None, [P]),
        "spngd_ctx_sync": (C.c_int, [P]),
        "spngd_ctx_stream": (P, [P]),
        "spngd_copy": (C.c_int, [P, P, P, C.c_size_t]),
        "spngd_host_alloc": (C.c_int, [C.POINTER(P), C.c_size_t]),
        "spngd_host_free": (None, [P]),
        "spngd_event_time": (C.c_int, [P, C.POINTER(P), C.c_int, C.POINTER(C.c_float)]),
        "spngd_factor_sym_batched": (C.c_int, [P, C.c_int, C.POINTER(FactorReq)]),
        "spngd_bn_moments_batched": (C.c_int, [P, C.c_int, C.POINTER(BnMomentsReq)]),
        "spngd_bn_grad_reduce_batched": (C.c_int, [P, C.c_int, C.POINTER(BnGradReq)]),
        "spngd_bn_full_moments_batched": (C.c_int, [P, C.c_int, C.POINTER(BnFullReq)]),
        "spngd_bn_full_solve_update_batched": (C.c_int, [P, C.c_int, C.POINTER(BnFullUpdateReq), C.c_double,
                                                         C.c_double]),
        "spngd_spd_inverse_batched": (C.c_int, [P, C.c_int, C.POINTER(SpdReq), C.POINTER(C.c_int)]),
        "spngd_damp_and_invert_batched": (C.c_int, [P, C.c_int, C.POINTER(KronReq), C.c_double,
                                                   C.POINTER(C.c_int)]),
        "spngd_precondition_update_batched": (C.c_int, [P, C.c_int, C.POINTER(PrecondReq),
                                                        C.c_double, C.c_double]),
        "spngd_bn_solve_update_batched": (C.c_int, [P, C.c_int, C.POINTER(BnUpdateReq), C.c_double,
                                                    C.c_double, C.c_double]),
        "spngd_stat_distance_batched": (C.c_int, [P, C.c_int, C.POINTER(StatReq)]),
        "spngd_tracker_create": (P, [C.c_char_p, C.c_double]),
        "spngd_tracker_destroy": (None, [P]),
        "spngd_tracker_should_refresh": (C.c_int, [P, _i64]),
        "spngd_tracker_on_refresh": (C.c_int, [P, _i64, C.c_int, C.c_double, C.c_double, C.c_int,
                                               C.c_double, C.c_double, C.POINTER(_i64),
                                               C.POINTER(C.c_int)]),
        "spngd_tracker_state": (None, [P] + [C.POINTER(_i64)] * 4),
        "spngd_nccl_unique_id": (C.c_int, [P]),
        "spngd_ctx_init_comm": (C.c_int, [P, C.c_int, C.c_int, P]),
        "spngd_reduce_scatter_mean": (C.c_int, [P, P, P, _i64]),
        "spngd_all_gather": (C.c_int, [P, P, P, _i64]),
        "spngd_plan_layout_ex": (C.c_int, [C.POINTER(LayerDesc), C.c_int, C.c_int, C.c_int, C.POINTER(LayoutEntry),
                                           C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
        "spngd_plan_layout": (C.c_int, [C.POINTER(LayerDesc), C.c_int, C.c_int, C.POINTER(LayoutEntry),
                                        C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
        "spngd_opt_create": (C.c_int, [P, C.POINTER(LayerDesc), C.c_int, C.POINTER(OptConfig),
                                       C.POINTER(P)]),
        "spngd_opt_destroy": (None, [P]),
        "spngd_opt_buffer": (P, [P, C.c_int, C.c_int, C.POINTER(_i64)]),
        "spngd_opt_owner": (C.c_int, [P, C.c_int]),
        "spngd_opt_step": (C.c_int, [P, _i64, C.c_double, C.c_double]),
        "spngd_opt_phase_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
        "spngd_opt_set_overlap": (C.c_int, [P, C.c_int]),
        "spngd_opt_sync": (C.c_int, [P]),
        "spngd_opt_enable_bn_inputs": (C.c_int, [P, C.POINTER(C.c_int64)]),
        "spngd_opt_enable_raw_inputs_ex": (C.c_int, [P, C.POINTER(ConvGeom), C.c_int]),
        "spngd_bn_backward_stats_batched": (C.c_int, [P, C.c_int, C.POINTER(BnBackwardReq)]),
        "spngd_opt_launch_count": (_i64, [P]),
        "spngd_opt_stale_info": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
                                           C.POINTER(C.c_int)]),
        "spngd_ledger_step_rows": (_i64, [C.POINTER(LayerDesc), C.c_int, C.c_int, _i64, C.POINTER(C.c_ubyte),
                                          C.c_int, C.c_int, C.POINTER(LedgerRowC), _i64]),
        "spngd_opt_step_host": (C.c_int, [P, _i64, C.c_double, C.c_double, C.POINTER(HostInput), C.c_int,
                                           C.c_void_p]),
        "spngd_opt_ipc_handle": (C.c_int, [P, C.c_void_p]),
        "spngd_opt_attach_peers": (C.c_int, [P, C.c_void_p]),
        "spngd_opt_enable_raw_inputs": (C.c_int, [P, C.POINTER(ConvGeom)]),
        "spngd_im2col_batched": (C.c_int, [P, C.c_int, C.POINTER(Im2colReq)]),
        "spngd_opt_ledger": (_i64, [P, C.POINTER(LedgerRowC), _i64]),
        "spngd_opt_ledger_clear": (C.c_int, [P]),
        "spngd_opt_wire_bytes": (C.c_int, [P, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
        "spngd_synth_normal": (C.c_int, [P, P, _i64, C.c_uint64, C.c_float, C.c_float, C.c_int]),
        "spngd_synth_conv_capture": (C.c_int, [P, P] + [_i64] * 7 + [C.c_uint64, C.c_int, C.c_float,
                                                                      C.c_float]),
        "spngd_synth_bn_pairs": (C.c_int, [P, P, P, _i64, C.c_uint64]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(L, name):
            continue  # reported by tests/test_abi.py
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
