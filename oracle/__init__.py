"""fp64 CPU oracle for the SP-NGD optimizer step — TEST INFRASTRUCTURE ONLY.

ctypes bindings over ``oracle/liboracle.so`` (built from ``spngd_oracle.cpp``
by ``oracle/Makefile``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs import this module,
always as the checker or as the timed CPU baseline, never as the product.

Each wrapper names the reference function it restates; see the C++ source for
file:line citations into /root/reference/proj.  Errors come back as the
reference's exception names (errors.hpp:10-85) via :class:`OracleError`.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

_ERR = {1: "ShapeMismatch", 2: "NotPositiveDefinite", 3: "SingularBlock",
        4: "ZeroReference", 5: "EmptyBatch"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.kind = _ERR.get(code, f"code{code}")
        super().__init__(f"{where}: {self.kind}")


def build() -> str:
    src = os.path.join(_HERE, "spngd_oracle.cpp")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_i64 = C.c_int64


class OrLayer(C.Structure):
    _fields_ = [("is_conv", _i64), ("a", _i64), ("g", _i64), ("hw", _i64),
                ("batch", _i64), ("act", _fp), ("grad", _fp), ("dW", _fp),
                ("W", _fp), ("V", _fp), ("W_out", _dp), ("V_out", _dp),
                ("Ainv_out", _dp), ("Ginv_out", _dp), ("P_out", _dp),
                ("seconds", C.c_double * 4), ("status", C.c_int)]


def _declare(L):
    sig = {
        "or_packed_size": (_i64, [_i64]),
        "or_packed_offset": (_i64, [_i64, _i64, _i64]),
        "or_unpack": (None, [_dp, _i64, _dp]),
        "or_pack": (None, [_dp, _i64, _dp]),
        "or_spd_inverse": (C.c_int, [_dp, _i64, C.c_double, _dp]),
        "or_spd_inverse_fast": (C.c_int, [_dp, _i64, C.c_double, _dp]),
        "or_inv2x2": (C.c_int, [C.c_double] * 4 + [_dp]),
        "or_kron_matvec": (C.c_int, [_dp, _dp, _i64, _i64, _dp, _dp]),
        "or_avg_eigenvalue": (C.c_double, [_dp, _i64]),
        "or_frob_norm": (C.c_double, [_dp, _i64]),
        "or_rel_frob_distance": (C.c_int, [_dp, _dp, _i64, _dp]),
        "or_mean_outer": (C.c_int, [_dp, _i64, _i64, _i64, _i64, C.c_double, C.c_int, _dp]),
        "or_factor_A_f32": (C.c_int, [_fp, _i64, _i64, _i64, _i64, _i64, C.c_int, _dp]),
        "or_factor_G_f32": (C.c_int, [_fp, _i64, _i64, _i64, _i64, _i64, C.c_int, _dp]),
        "or_build_bn_block": (C.c_int, [_dp, _dp, _i64, _i64, _i64, C.c_int, _dp]),
        "or_bn_grad_reduce": (C.c_int, [C.POINTER(C.c_float), C.POINTER(C.c_float), _i64, _i64, _i64, _dp, _dp]),
        "or_build_bn_full": (C.c_int, [_dp, _dp, _i64, _i64, _i64, C.c_int, _dp]),
        "or_damp_and_invert": (C.c_int, [_dp, _dp, _i64, _i64, C.c_double, _dp, _dp, _dp]),
        "or_damp_bn": (C.c_int, [_dp, _i64, C.c_double, _dp]),
        "or_precondition_bn": (C.c_int, [_dp, _i64, _dp, _dp, C.c_double, _dp, _dp]),
        "or_precondition_bn_full": (C.c_int, [_dp, _i64, _dp, _dp, _dp, _dp]),
        "or_ngd_update": (None, [_dp, _dp, _dp, _i64, C.c_double, C.c_double, _dp, _dp]),
        "or_rescale": (None, [_dp, _dp, _i64, _i64, _dp, _dp]),
        "or_weighted_norm": (C.c_double, [_dp, _dp, _i64]),
        "or_similar": (C.c_int, [_dp, _dp, _dp, _i64, C.c_double]),
        "or_im2col": (None, [_dp] + [_i64] * 6 + [_dp]),
        "or_rng_derive": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "or_rng_fill": (None, [C.c_uint64, C.c_int, _i64, _dp]),
        "or_sizeof_layer": (_i64, []),
        "or_kfac_layers": (C.c_int, [C.POINTER(OrLayer), _i64, C.c_double, C.c_double,
                                     C.c_double, C.c_int, C.c_int, C.c_int]),
        "or_synth_normal": (None, [C.c_uint64, _i64, _i64, _fp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    assert L.or_sizeof_layer() == C.sizeof(OrLayer), "OrLayer ABI mismatch"


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(_fp)


def _check(rc, where):
    if rc:
        raise OracleError(rc, where)


def packed_size(n):
    return n * (n + 1) // 2


def pack(dense):
    """SymMatrix::pack (linalg.cpp:7-16): upper triangle, row-major."""
    dense, p = _d(dense)
    n = dense.shape[0]
    out = np.empty(packed_size(n))
    lib().or_pack(p, n, out.ctypes.data_as(_dp))
    return out


def unpack(packed, n):
    """SymMatrix::unpack (linalg.cpp:18-27)."""
    packed, p = _d(packed)
    out = np.empty((n, n))
    lib().or_unpack(p, n, out.ctypes.data_as(_dp))
    return out


def spd_inverse(packed, n, damping, fast=False):
    """spd_inverse (linalg.cpp:29-48) -> packed (M + d I)^-1."""
    packed, p = _d(packed)
    out = np.empty(packed_size(n))
    f = lib().or_spd_inverse_fast if fast else lib().or_spd_inverse
    _check(f(p, n, damping, out.ctypes.data_as(_dp)), "spd_inverse")
    return out


def inv2x2(a, b, c, d):
    """inv2x2 (linalg.cpp:50-56)."""
    out = np.empty(4)
    _check(lib().or_inv2x2(a, b, c, d, out.ctypes.data_as(_dp)), "inv2x2")
    return tuple(out)


def kron_matvec(gp, ap, dg, da, x):
    """kron_matvec (linalg.cpp:58-62): G X A."""
    gp, g_ = _d(gp)
    ap, a_ = _d(ap)
    x, x_ = _d(x)
    if x.shape != (dg, da):
        raise OracleError(1, "kron_matvec")
    out = np.empty((dg, da))
    _check(lib().or_kron_matvec(g_, a_, dg, da, x_, out.ctypes.data_as(_dp)), "kron_matvec")
    return out


def avg_eigenvalue(p, n):
    p, p_ = _d(p)
    return lib().or_avg_eigenvalue(p_, n)


def frob_norm(p, n):
    p, p_ = _d(p)
    return lib().or_frob_norm(p_, n)


def rel_frob_distance(a, b, n):
    a, a_ = _d(a)
    b, b_ = _d(b)
    out = C.c_double()
    _check(lib().or_rel_frob_distance(a_, b_, n, C.byref(out)), "rel_frob_distance")
    return out.value


def mean_outer(stacked, r, lo, hi, denom, compensated=False):
    """mean_outer (fisher.cpp:55-75); stacked is 2-D row-major."""
    stacked, s_ = _d(stacked)
    cols = stacked.shape[1]
    dim = cols if r == 1 else r
    out = np.empty(packed_size(dim))
    _check(lib().or_mean_outer(s_, cols, r, lo, hi, denom, int(compensated),
                               out.ctypes.data_as(_dp)), "mean_outer")
    return out


def factor_A(act, is_conv, a, hw, lo, hi, compensated=False):
    """factor_A (fisher.cpp:92-114) on an fp32 capture (net.hpp:84-101)."""
    act, a_ = _f(act)
    out = np.empty(packed_size(a))
    _check(lib().or_factor_A_f32(a_, int(is_conv), a, hw, lo, hi, int(compensated),
                                 out.ctypes.data_as(_dp)), "factor_A")
    return out


def factor_G(grad, is_conv, g, hw, lo, hi, compensated=False):
    """factor_G (fisher.cpp:116-145)."""
    grad, g_ = _f(grad)
    out = np.empty(packed_size(g))
    _check(lib().or_factor_G_f32(g_, int(is_conv), g, hw, lo, hi, int(compensated),
                                 out.ctypes.data_as(_dp)), "factor_G")
    return out


def build_bn_block(gg, gb, lo, hi, compensated=False):
    """build_bn_block (fisher.cpp:147-185) -> interleaved 3c payload."""
    gg, g_ = _d(gg)
    gb, b_ = _d(gb)
    c = gg.shape[1]
    out = np.empty(3 * c)
    _check(lib().or_build_bn_block(g_, b_, c, lo, hi, int(compensated),
                                   out.ctypes.data_as(_dp)), "build_bn_block")
    return out


def bn_grad_reduce(dy, xhat, M, c, S):
    """Per-sample BN gamma/beta gradients (net.cpp:467-475) -> (gg, gb), M x c."""
    dy = np.ascontiguousarray(dy, dtype=np.float32)
    xh = np.ascontiguousarray(xhat, dtype=np.float32)
    if dy.size != M * c * S or xh.size != M * c * S:
        raise OracleError(1, "bn_grad_reduce")
    gg = np.empty(M * c)
    gb = np.empty(M * c)
    fp = C.POINTER(C.c_float)
    _check(lib().or_bn_grad_reduce(dy.ctypes.data_as(fp), xh.ctypes.data_as(fp), M, c, S,
                                   gg.ctypes.data_as(_dp), gb.ctypes.data_as(_dp)), "bn_grad_reduce")
    return gg.reshape(M, c), gb.reshape(M, c)


def build_bn_full(gg, gb, lo, hi, compensated=False):
    gg, g_ = _d(gg)
    gb, b_ = _d(gb)
    c = gg.shape[1]
    out = np.empty(packed_size(2 * c))
    _check(lib().or_build_bn_full(g_, b_, c, lo, hi, int(compensated),
                                  out.ctypes.data_as(_dp)), "build_bn_full")
    return out


def damp_and_invert(A, G, da, dg, lam):
    """damp_and_invert (fisher.cpp:218-228) -> (pi, A_inv, G_inv) packed."""
    A, a_ = _d(A)
    G, g_ = _d(G)
    pi = C.c_double()
    Ai = np.empty(packed_size(da))
    Gi = np.empty(packed_size(dg))
    _check(lib().or_damp_and_invert(a_, g_, da, dg, lam, C.byref(pi),
                                    Ai.ctypes.data_as(_dp), Gi.ctypes.data_as(_dp)),
           "damp_and_invert")
    return pi.value, Ai, Gi


def damp_bn(m3c, lam):
    m3c, m_ = _d(m3c)
    out = np.empty_like(m3c)
    _check(lib().or_damp_bn(m_, m3c.size // 3, lam, out.ctypes.data_as(_dp)), "damp_bn")
    return out


def precondition_bn(m3c, gg, gb, lam):
    """precondition_bn (fisher.cpp:259-276)."""
    m3c, m_ = _d(m3c)
    gg, g_ = _d(gg)
    gb, b_ = _d(gb)
    c = gg.size
    if gb.size != c or m3c.size != 3 * c:
        raise OracleError(1, "precondition_bn")
    pg = np.empty(c)
    pb = np.empty(c)
    _check(lib().or_precondition_bn(m_, c, g_, b_, lam, pg.ctypes.data_as(_dp),
                                    pb.ctypes.data_as(_dp)), "precondition_bn")
    return pg, pb


def precondition_bn_full(finv, gg, gb):
    finv, f_ = _d(finv)
    gg, g_ = _d(gg)
    gb, b_ = _d(gb)
    c = gg.size
    pg = np.empty(c)
    pb = np.empty(c)
    _check(lib().or_precondition_bn_full(f_, c, g_, b_, pg.ctypes.data_as(_dp),
                                         pb.ctypes.data_as(_dp)), "precondition_bn_full")
    return pg, pb


def ngd_update(p, delta, v, eta, momentum):
    """ngd_step's per-tensor update (fisher.cpp:332-333)."""
    p, p_ = _d(p)
    delta, d_ = _d(delta)
    v, v_ = _d(v)
    np_ = np.empty_like(p)
    nv = np.empty_like(p)
    lib().or_ngd_update(p_, d_, v_, p.size, eta, momentum, np_.ctypes.data_as(_dp),
                        nv.ctypes.data_as(_dp))
    return np_, nv


def rescale(w_new, w_old, d_out):
    """rescale_weights (schemes.cpp:116-119) + velocity fix (dist.cpp:621-632)."""
    w_new, n_ = _d(w_new)
    w_old, o_ = _d(w_old)
    w = np.empty_like(w_new)
    v = np.empty_like(w_new)
    lib().or_rescale(n_, o_, w_new.size, d_out, w.ctypes.data_as(_dp), v.ctypes.data_as(_dp))
    return w, v


def similar(x, ref, w, alpha):
    """stale.hpp:56-64."""
    x, x_ = _d(x)
    ref, r_ = _d(ref)
    w, w_ = _d(w)
    if x.size != ref.size:
        raise OracleError(1, "similar")
    return bool(lib().or_similar(x_, r_, w_, x.size, alpha))


def im2col(x, c, h, w, k, stride, pad):
    """im2col (net.cpp:199-219)."""
    x, x_ = _d(x)
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    out = np.empty((c * k * k, ho * wo))
    lib().or_im2col(x_, c, h, w, k, stride, pad, out.ctypes.data_as(_dp))
    return out


def rng_derive(seed, tag):
    return lib().or_rng_derive(seed, tag)


def rng_normal(seed, n):
    """n draws of Rng(seed).normal() (rng.cpp:36-45)."""
    out = np.empty(n)
    lib().or_rng_fill(seed, 1, n, out.ctypes.data_as(_dp))
    return out


def rng_uniform(seed, n):
    out = np.empty(n)
    lib().or_rng_fill(seed, 0, n, out.ctypes.data_as(_dp))
    return out


def synth_normal(key, offset, n):
    """Counter-based stream shared with the device generator (synth.cu)."""
    out = np.empty(n, dtype=np.float32)
    lib().or_synth_normal(key, offset, n, out.ctypes.data_as(_fp))
    return out


def random_spd(n, seed, eps=0.5):
    """oracles::random_spd (tests/oracles.hpp:42-49) drawn from Rng(seed)."""
    m = rng_normal(seed, n * n).reshape(n, n)
    s = m @ m.T / n + eps * np.eye(n)
    return 0.5 * (s + s.T)


def kfac_layers(layers, lam, eta, momentum, rescale=True, fast_inverse=True, threads=1):
    """Whole-layer Stage-4 restatement over OrLayer records (timed baseline)."""
    arr = (OrLayer * len(layers))(*layers)
    rc = lib().or_kfac_layers(arr, len(layers), lam, eta, momentum, int(rescale),
                              int(fast_inverse), threads)
    for i in range(len(layers)):
        layers[i] = arr[i]
    _check(rc, "kfac_layers")
    return layers
