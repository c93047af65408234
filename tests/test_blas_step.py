"""The BLAS/LAPACK fp64 restatement that bench.py times as the CPU baseline
(oracle/blas_step.py) computes the same step as the line-by-line oracle
(oracle/spngd_oracle.cpp, pinned by tests/test_oracle_kat.py): factors,
damped inverses, preconditioning, update + rescale, unit BN."""
import ctypes as C

import numpy as np

import oracle as O
from oracle import blas_step as B
from paper_2002_06015_b200 import workloads as W

LAM, ETA, MOM = 2.5e-4, 1.25e-2, 0.993


def test_blas_step_matches_oracle():
    layers = [W.conv(3, 8, 3, 1, 8), W.bn(8), W.conv(8, 16, 3, 2, 8), W.fc(64, 10)]
    batch = 4
    bs = B.BlasStep(layers, batch, seed=3)
    for d in bs.data:  # fp32-representable inputs, as the oracle reads them
        for k in ("act", "grad", "dW", "W", "V", "gg", "gb"):
            if hasattr(d, k):
                setattr(d, k, getattr(d, k).astype(np.float32).astype(np.float64))
    t = [0.0, 0.0, 0.0]
    for l, d in zip(layers, bs.data):
        if l.kind == "bn":
            w, v = B.bn_layer(d, LAM, ETA, MOM, t)
            m3 = O.build_bn_block(d.gg, d.gb, 0, batch)
            pg, pb = O.precondition_bn(m3, d.dW[:l.g], d.dW[l.g:], LAM)
            want_w, want_v = O.ngd_update(d.W, np.concatenate([pg, pb]), d.V, ETA, MOM)
        else:
            w, v = B.kfac_layer(d, LAM, ETA, MOM, t)
            f32 = [np.ascontiguousarray(x, dtype=np.float32).reshape(-1) for x in (d.act, d.grad, d.dW, d.W, d.V)]
            rec = O.OrLayer()
            want_w, want_v = np.empty(l.g * l.a), np.empty(l.g * l.a)
            rec.is_conv, rec.a, rec.g, rec.hw, rec.batch = int(l.kind == "conv"), l.a, l.g, l.hw, batch
            rec.act, rec.grad, rec.dW, rec.W, rec.V = [x.ctypes.data_as(C.POINTER(C.c_float)) for x in f32]
            rec.W_out = want_w.ctypes.data_as(C.POINTER(C.c_double))
            rec.V_out = want_v.ctypes.data_as(C.POINTER(C.c_double))
            O.kfac_layers([rec], LAM, ETA, MOM, rescale=True, fast_inverse=False, threads=1)
        for got, want in ((w, want_w), (v, want_v)):
            err = np.linalg.norm(np.ravel(got) - want) / np.linalg.norm(want)
            assert err <= 1e-10, f"{l}: {err:.2e}"


def test_sample_classes_include_every_4608_factor():
    layers = W.resnet50()
    idx = B.sample_classes(layers)
    big = [i for i, l in enumerate(layers) if l.kind != "bn" and max(l.a, l.g) == 4608]
    assert len(big) == 3 and set(big) <= set(idx)
    classes = {(l.kind, l.a, l.g, l.hw) for l in layers}
    assert {(layers[i].kind, layers[i].a, layers[i].g, layers[i].hw) for i in idx} == classes
