"""Parity at the factors that dominate the inverse: the
ResNet-50 layer-4 / layer-3 shapes with n = 2048 / 2304 / 4608 factors at
B = 32 (A rank-deficient for the 4608 layers: K = 32 * 49 = 1568 < 4608), and
the config-5 damped-inverse sweep inputs at n = 2048 / 4096 / 4608, against
the fp64 oracle (oracle/spngd_oracle.cpp; numpy/LAPACK fp64 for the sweep's
4096/4608 inverses, pinned to the oracle at n = 2048).  Gate: relative
Frobenius <= 1e-4 (north_star) on inverses, preconditioned gradients and
updated weights/velocities."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

from paper_2002_06015_b200 import spngd as P  # noqa: E402
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import ACT, DW, GRAD, V, Optimizer  # noqa: E402
from paper_2002_06015_b200.step import W as WB  # noqa: E402

ETA, MOM, LAM = 1.25e-2, 0.993, 2.5e-4
GATE = 1e-4
# (a, g, hw) = (4608, 512, 49) x3, (2304, 256, 196) x6, (512, 2048, 49) x3, (1024, 2048, 49) x1
LAYERS = [W.conv(512, 512, 3, 1, 7), W.conv(256, 256, 3, 1, 14), W.conv(512, 2048, 1, 1, 7),
          W.conv(1024, 2048, 1, 2, 14)]
BATCH = 32


def rel(a, b):
    a = np.asarray(a, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


@pytest.fixture(scope="module")
def r50_big(cuda_dev):
    """One step of the optimizer over the four layer shapes, the captures it
    consumed, and the oracle's inverses / preconditioned gradients / weights."""
    opt = Optimizer(LAYERS, BATCH, lam=LAM)
    opt.synth(seed=11)
    before = [{w: opt.download(li, w).numpy().copy() for w in (ACT, GRAD, DW, WB, V)} for li in range(len(LAYERS))]
    opt.step(1, ETA, MOM)
    opt.sync()
    after = [(opt.download(li, WB).numpy().copy(), opt.download(li, V).numpy().copy()) for li in range(len(LAYERS))]
    opt.close()
    recs, outs = [], []
    for l, b in zip(LAYERS, before):
        r = O.OrLayer()
        o = {k: np.empty(n) for k, n in (("W", l.g * l.a), ("V", l.g * l.a), ("P", l.g * l.a),
                                           ("Ai", l.a * (l.a + 1) // 2), ("Gi", l.g * (l.g + 1) // 2))}
        r.is_conv, r.a, r.g, r.hw, r.batch = 1, l.a, l.g, l.hw, BATCH
        r.act, r.grad, r.dW, r.W, r.V = [b[k].ctypes.data_as(C.POINTER(C.c_float)) for k in (ACT, GRAD, DW, WB, V)]
        r.W_out, r.V_out, r.P_out = [o[k].ctypes.data_as(C.POINTER(C.c_double)) for k in ("W", "V", "P")]
        r.Ainv_out, r.Ginv_out = [o[k].ctypes.data_as(C.POINTER(C.c_double)) for k in ("Ai", "Gi")]
        recs.append(r)
        outs.append(o)
    O.kfac_layers(recs, LAM, ETA, MOM, rescale=True, fast_inverse=True, threads=min(len(recs), threads()))
    return before, after, outs


def test_resnet50_large_layers_step(r50_big):
    """spngd_opt_step on the layers whose factors dominate the inverse
    (4608^2 A with K < a, 2304^2 A, 2048^2 G): updated W and V vs the oracle."""
    _, after, outs = r50_big
    for l, (w, v), o in zip(LAYERS, after, outs):
        ew, ev = rel(w, o["W"]), rel(v, o["V"])
        assert ew <= GATE and ev <= GATE, f"{l}: W {ew:.2e} V {ev:.2e}"


def test_resnet50_large_layers_primitives(r50_big):
    """factor_A/factor_G -> damp_and_invert -> precondition (the reference's
    Stage-4 primitives, fisher.cpp:92-145, 218-228, 255-257) on the same
    captures: A^-1, G^-1 and the preconditioned gradient vs the oracle."""
    before, _, outs = r50_big
    blocks, dws = [], []
    for l, b in zip(LAYERS, before):
        act = torch.from_numpy(b[ACT]).cuda()
        grad = torch.from_numpy(b[GRAD]).cuda()
        A = P.factor_sym(act, l.a, l.hw, 1, 0, BATCH, 1.0 / (BATCH * l.hw))
        G = P.factor_sym(grad, l.g, l.hw, 1, 0, BATCH, 1.0 / BATCH)
        blocks.append(P.KroneckerBlock(A=P.SymMatrix(l.a, A), G=P.SymMatrix(l.g, G)))
        dws.append(torch.from_numpy(b[DW]).cuda().reshape(l.g, l.a))
    info = []
    P.damp_and_invert_batched(blocks, LAM, info=info)
    assert info == [0] * len(LAYERS)
    for l, blk, dw, o in zip(LAYERS, blocks, dws, outs):
        ea = O.rel_frob_distance(blk.A_inv.data.cpu().numpy().astype(np.float64), o["Ai"], l.a)
        eg = O.rel_frob_distance(blk.G_inv.data.cpu().numpy().astype(np.float64), o["Gi"], l.g)
        ep = rel(P.precondition(blk, dw).cpu().numpy().reshape(-1), o["P"])
        assert max(ea, eg, ep) <= GATE, f"{l}: A^-1 {ea:.2e} G^-1 {eg:.2e} P {ep:.2e}"


def sweep_matrix(n, kind, seed):
    """SURVEY.md §8d config 5 inputs, fp32 on the device: (i) random SPD,
    (ii) A = X X^T / K from ReLU activations with K < n and K > n."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        if kind == "random_spd":
            x = torch.randn(n, n, device="cuda", generator=g) / n ** 0.5
            m = x @ x.T + 0.5 * torch.eye(n, device="cuda")
        else:
            k = n // 2 if kind == "relu_K<n" else 2 * n
            x = torch.relu(torch.randn(n, k, device="cuda", generator=g))
            m = x @ x.T / k
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    iu = torch.triu_indices(n, n, device="cuda")
    return m[iu[0], iu[1]].contiguous().float()


DAMP = float(np.float32(2.5e-4 ** 0.5))  # damp_and_invert's A-side damping with pi = 1


def fp64_inverse(packed, n, damp):
    m = O.unpack(packed.cpu().numpy().astype(np.float64), n)
    m[np.diag_indices(n)] += damp
    return np.linalg.inv(m)


@pytest.mark.parametrize("n,kind", [(2048, "relu_K<n"), (4096, "relu_K<n"), (4608, "relu_K<n"),
                                    (4608, "relu_K>n"), (4608, "random_spd")])
def test_inverse_sweep_large(cuda_dev, n, kind):
    """Config-5 sweep rows at the sizes that missed the gate in round 1
    (relu K<n: 1.19e-4 at 4096, 1.27e-4 at 4608, cond up to 4.7e4): batched
    spd_inverse (two matrices per call) vs the fp64 inverse of the same fp32
    input."""
    pk = [sweep_matrix(n, kind, 1000 * n + i) for i in range(2)]
    info = []
    outs = P.spd_inverse_batched([P.SymMatrix(n, p) for p in pk], DAMP, info=info)
    assert info == [0, 0]
    for p, o in zip(pk, outs):
        want = fp64_inverse(p, n, DAMP)
        got = O.unpack(o.data.cpu().numpy().astype(np.float64), n)
        err = rel(got, want)
        assert err <= GATE, f"n={n} {kind}: {err:.3e}"


def test_sweep_reference_pinned_to_oracle(cuda_dev):
    """The LAPACK fp64 inverse used above agrees with the oracle's restated
    spd_inverse (linalg.cpp:29-48) at n = 2048, and so does the GPU result."""
    n = 2048
    p = sweep_matrix(n, "relu_K<n", 77)
    pn = p.cpu().numpy().astype(np.float64)
    want = O.spd_inverse(pn, n, DAMP, fast=True)
    lap = fp64_inverse(p, n, DAMP)
    assert O.rel_frob_distance(O.pack(lap), want, n) <= 1e-10
    got = P.spd_inverse_batched([P.SymMatrix(n, p)], DAMP)[0]
    assert O.rel_frob_distance(got.data.cpu().numpy().astype(np.float64), want, n) <= GATE


def test_info_names_failing_factor(cuda_dev):
    """A non-PD matrix in a batch of 5: NotPositiveDefinite, info[] marks
    exactly that request, and the message names it (fisher.cpp:48-51
    layer_tag, linalg.cpp:37-40)."""
    n = 256
    mats = [P.SymMatrix(n, sweep_matrix(n, "random_spd", 5 + i)) for i in range(5)]
    bad = mats[3].data.clone()
    bad[0] = -1.0  # M[0][0] = -1: first pivot -1 + d < 0
    mats[3] = P.SymMatrix(n, bad)
    info = []
    with pytest.raises(P.NotPositiveDefinite) as e:
        P.spd_inverse_batched(mats, DAMP, info=info)
    assert info == [0, 0, 0, P.SPNGD_ERR_NOT_POSITIVE_DEFINITE, 0]
    assert "request 3" in str(e.value) and "n=256" in str(e.value)
    # damp_and_invert: the G factor of block 1 is the bad one
    blocks = [P.KroneckerBlock(A=P.SymMatrix(n, sweep_matrix(n, "random_spd", 20 + i)),
                               G=P.SymMatrix(n, sweep_matrix(n, "random_spd", 30 + i))) for i in range(3)]
    gbad = blocks[1].G.data.clone()
    gbad[0] = -1e3
    blocks[1].G = P.SymMatrix(n, gbad)
    info = []
    with pytest.raises(P.NotPositiveDefinite) as e:
        P.damp_and_invert_batched(blocks, LAM, info=info)
    assert info == [0, P.SPNGD_ERR_NOT_POSITIVE_DEFINITE, 0]
    assert "request 1" in str(e.value) and "G factor" in str(e.value)
