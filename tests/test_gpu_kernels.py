"""GPU parity of each hot-path kernel against the fp64 oracle (same inputs).

Tolerances: packed factors <= 1e-6 relative Frobenius; inverses,
preconditioned gradients and updated weights <= 1e-4 (BASELINE north_star).
"""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2002_06015_b200")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def rel_packed(a, b, n):
    return O.rel_frob_distance(np.asarray(a, np.float64), np.asarray(b, np.float64), n)


def conv_capture(batch, c, h, w, k, stride, pad, seed, relu=True):
    ctx = P.context()
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    x = torch.empty(batch * c * k * k * ho * wo, device="cuda")
    P.check(P._native.lib().spngd_synth_conv_capture(ctx.h, x.data_ptr(), batch, c, h, w, k, stride, pad,
                                                     seed, int(relu), 1.0, 0.0))
    torch.cuda.synchronize()
    return x, c * k * k, ho * wo


@pytest.mark.parametrize("d,batch", [(5, 6), (64, 32), (256, 128), (784, 128), (1000, 32)])
def test_fc_factor_matches_oracle(cuda_dev, d, batch):
    x = torch.randn(batch, d, device="cuda")
    got = P.factor_sym(x, d, 1, 0, 0, batch, 1.0 / batch).cpu().numpy()
    want = O.factor_A(x.cpu().numpy(), False, d, 1, 0, batch)
    assert rel_packed(got, want, d) <= 1e-6


@pytest.mark.parametrize("shape", [
    (4, 2, 4, 4, 3, 1, 1),        # reference conv_net shape (test_fisher.cpp:25-32)
    (3, 8, 7, 7, 3, 1, 1),        # hw = 49 (scalar, non-multiple-of-4 segments)
    (2, 64, 14, 14, 3, 1, 1),     # a = 576, hw = 196
    (2, 128, 28, 28, 3, 2, 1),    # a = 1152, hw = 196, stride 2
    (2, 3, 224, 224, 7, 2, 3),    # ResNet-50 conv1: a = 147, K = 25088 -> split-K
    (1, 512, 7, 7, 3, 1, 1),      # a = 4608, hw = 49 (largest A factor)
])
def test_conv_factor_A_matches_oracle(cuda_dev, shape):
    batch, c, h, w, k, s, p = shape
    x, a, hw = conv_capture(batch, c, h, w, k, s, p, 1234 + c)
    got = P.factor_sym(x, a, hw, 1, 0, batch, 1.0 / (batch * hw)).cpu().numpy()
    want = O.factor_A(x.cpu().numpy(), True, a, hw, 0, batch)
    assert rel_packed(got, want, a) <= 1e-6


def test_factor_subrange_and_errors(cuda_dev):
    x, a, hw = conv_capture(6, 2, 4, 4, 3, 1, 1, 99)
    xn = x.cpu().numpy()
    for lo, hi in [(0, 2), (2, 6), (1, 4)]:
        got = P.factor_sym(x, a, hw, 1, lo, hi, 1.0 / ((hi - lo) * hw)).cpu().numpy()
        assert rel_packed(got, O.factor_A(xn, True, a, hw, lo, hi), a) <= 1e-6
    with pytest.raises(P.EmptyBatch):
        P.factor_sym(x, a, hw, 1, 2, 2, 1.0)


def test_ctx_last_error_is_per_context(cuda_dev):
    """spngd_last_error(ctx) -- a failure on one context
    is readable from that context (and not from another) after the call."""
    from paper_2002_06015_b200.spngd import Context
    L = P._native.lib()
    ctx = P.context()
    other = Context(0)
    x, a, hw = conv_capture(6, 2, 4, 4, 3, 1, 1, 99)
    with pytest.raises(P.EmptyBatch):
        P.factor_sym(x, a, hw, 1, 2, 2, 1.0)
    msg = L.spngd_ctx_last_error(ctx.h).decode()
    assert "empty sample range" in msg, msg
    assert msg == L.spngd_last_error().decode()
    assert L.spngd_ctx_last_error(other.h).decode() == ""


def test_conv_factor_G_scaling(cuda_dev):
    batch, g, hw = 5, 64, 196
    gr = torch.randn(batch * g * hw, device="cuda") / np.sqrt(batch * hw)
    got = P.factor_sym(gr, g, hw, 1, 0, batch, 1.0 / batch).cpu().numpy()
    want = O.factor_G(gr.cpu().numpy(), True, g, hw, 0, batch)
    assert rel_packed(got, want, g) <= 1e-6


@pytest.mark.parametrize("n", [1, 3, 9, 64, 128, 129, 147, 300, 576, 1152])
def test_spd_inverse_random_spd(cuda_dev, n):
    s = O.random_spd(n, 7 + n)
    packed = O.pack(s)
    got, dense = P.spd_inverse(P.SymMatrix(n, torch.tensor(packed, dtype=torch.float32, device="cuda")), 0.3,
                               dense=True)
    want = O.spd_inverse(packed.astype(np.float32).astype(np.float64), n, 0.3)
    assert rel_packed(got.data.cpu().numpy(), want, n) <= 1e-5
    d = dense.cpu().numpy()
    assert np.array_equal(d, d.T)  # exactly symmetric (test_linalg.cpp:79-84)


def test_spd_inverse_relu_activation_factor(cuda_dev):
    """Ill-conditioned A from post-ReLU im2col at the reference
    damping: the hard case for the 1e-4 gate."""
    x, a, hw = conv_capture(4, 64, 14, 14, 3, 2, 1, 77)  # a = 576, K = 4*49 = 196 < a
    A = P.factor_sym(x, a, hw, 1, 0, 4, 1.0 / (4 * hw))
    d = float(np.sqrt(2.5e-4) * 3.8)
    got = P.spd_inverse(P.SymMatrix(a, A), d).data.cpu().numpy()
    want = O.spd_inverse(A.cpu().numpy().astype(np.float64), a, d)
    assert rel_packed(got, want, a) <= 1e-4


def test_spd_inverse_rejects_broken(cuda_dev):
    bad = np.eye(3)
    bad[1, 1] = np.nan
    with pytest.raises(P.NotPositiveDefinite):
        P.spd_inverse(P.SymMatrix(3, torch.tensor(O.pack(bad), dtype=torch.float32, device="cuda")), 1.0)
    with pytest.raises(P.NotPositiveDefinite):
        P.spd_inverse(P.SymMatrix(3, torch.tensor(O.pack(-2 * np.eye(3)), dtype=torch.float32, device="cuda")),
                      0.5)
    with pytest.raises(P.NotPositiveDefinite):  # large, fails in a deep Schur complement
        m = -np.eye(300)
        P.spd_inverse(P.SymMatrix(300, torch.tensor(O.pack(m), dtype=torch.float32, device="cuda")), 0.5)


def test_damp_and_invert_worked_example(cuda_dev):  # test_fisher.cpp:231-249
    b = P.KroneckerBlock(A=P.SymMatrix.pack(4 * torch.eye(2, device="cuda")),
                         G=P.SymMatrix.pack(torch.eye(3, device="cuda")))
    P.damp_and_invert(b, 1.0)
    assert abs(b.pi - 2.0) < 1e-6
    assert torch.allclose(b.A_inv.unpack(), torch.eye(2, device="cuda") / 6, atol=1e-7)
    assert torch.allclose(b.G_inv.unpack(), torch.eye(3, device="cuda") * 2 / 3, atol=1e-7)
    z = P.KroneckerBlock(A=P.SymMatrix(2), G=P.SymMatrix.pack(torch.eye(3, device="cuda")))
    P.damp_and_invert(z, 0.25)
    assert z.pi == 1.0
    with pytest.raises(P.NotPositiveDefinite):
        P.damp_and_invert(z, 0.0)


@pytest.mark.parametrize("g,a", [(7, 5), (64, 147), (128, 1152), (512, 4608 // 4)])
def test_precondition_matches_oracle(cuda_dev, g, a):
    rng = np.random.default_rng(g + a)
    A = O.pack(O.random_spd(a, 11 + a))
    G = O.pack(O.random_spd(g, 13 + g))
    b = P.KroneckerBlock(A=P.SymMatrix(a, torch.tensor(A, dtype=torch.float32, device="cuda")),
                         G=P.SymMatrix(g, torch.tensor(G, dtype=torch.float32, device="cuda")))
    P.damp_and_invert(b, 2.5e-4)
    pi, Ai, Gi = O.damp_and_invert(A.astype(np.float32).astype(np.float64),
                                   G.astype(np.float32).astype(np.float64), a, g, 2.5e-4)
    assert abs(b.pi - pi) / pi < 1e-6
    assert rel_packed(b.A_inv.data.cpu().numpy(), Ai, a) <= 1e-4
    assert rel_packed(b.G_inv.data.cpu().numpy(), Gi, g) <= 1e-4
    dW = rng.standard_normal((g, a)).astype(np.float32)
    got = P.precondition(b, torch.tensor(dW, device="cuda")).cpu().numpy()
    want = O.kron_matvec(Gi, Ai, g, a, dW.astype(np.float64))
    assert rel(got, want) <= 1e-4


def test_precondition_update_rescale_matches_oracle(cuda_dev):
    g, a = 64, 576
    rng = np.random.default_rng(5)
    x, _, hw = conv_capture(4, 64, 14, 14, 3, 2, 1, 5)
    gr = torch.randn(4 * g * hw, device="cuda") / np.sqrt(4 * hw)
    A = P.factor_sym(x, a, hw, 1, 0, 4, 1.0 / (4 * hw))
    G = P.factor_sym(gr, g, hw, 1, 0, 4, 1.0 / 4)
    b = P.KroneckerBlock(A=P.SymMatrix(a, A), G=P.SymMatrix(g, G))
    P.damp_and_invert(b, 2.5e-4)
    W = (rng.standard_normal((g, a)) * np.sqrt(2 / a)).astype(np.float32)
    V = (0.01 * rng.standard_normal((g, a))).astype(np.float32)
    dW = (rng.standard_normal((g, a)) / np.sqrt(a)).astype(np.float32)
    Wt, Vt = torch.tensor(W, device="cuda"), torch.tensor(V, device="cuda")
    P.kron_update(b, torch.tensor(dW, device="cuda"), Wt, Vt, 1.25e-2, 0.993, rescale=True)
    An, Gn = A.cpu().numpy().astype(np.float64), G.cpu().numpy().astype(np.float64)
    pi, Ai, Gi = O.damp_and_invert(An, Gn, a, g, 2.5e-4)
    Pw = O.kron_matvec(Gi, Ai, g, a, dW.astype(np.float64))
    nw, nv = O.ngd_update(W, Pw, V, 1.25e-2, 0.993)
    rw, rv = O.rescale(nw, W, g)
    assert rel(Wt.cpu().numpy(), rw.reshape(g, a)) <= 1e-4
    assert rel(Vt.cpu().numpy(), rv.reshape(g, a)) <= 1e-4


def test_bn_moments_and_update(cuda_dev):
    m, c, lam = 64, 300, 2.5e-4
    gg = torch.randn(m, c, device="cuda")
    gb = 0.6 * gg + 0.8 * torch.randn(m, c, device="cuda")
    cap = P.CaptureBuffer(m, [P.LayerCapture(bn_ggamma_true=gg, bn_gbeta_true=gb)])
    net = P.NetworkSpec([P.LayerSpec.batch_norm(c)])
    blk = P.build_bn_block(cap, net, 0)
    want = O.build_bn_block(gg.cpu().numpy(), gb.cpu().numpy(), 0, m)
    assert rel(blk.m3c.cpu().numpy(), want) <= 1e-6
    xg, xb = torch.randn(c, device="cuda"), torch.randn(c, device="cuda")
    pg, pb = P.precondition_bn(blk, xg, xb, lam)
    wg, wb = O.precondition_bn(blk.m3c.cpu().numpy(), xg.cpu().numpy(), xb.cpu().numpy(), lam)
    assert rel(pg.cpu().numpy(), wg) <= 1e-5 and rel(pb.cpu().numpy(), wb) <= 1e-5
    with pytest.raises(P.ShapeMismatch):
        P.precondition_bn(blk, torch.zeros(c + 1, device="cuda"), xb, lam)
    with pytest.raises(P.ShapeMismatch):
        P.factor_A(cap, net, 0)


def test_bn_singular_block(cuda_dev):
    blk = P.UnitBnBlock(m3c=torch.zeros(3, device="cuda"))
    with pytest.raises(P.SingularBlock):
        P.precondition_bn(blk, torch.ones(1, device="cuda"), torch.ones(1, device="cuda"), 1e-20)


def test_stat_distance_matches_oracle(cuda_dev):
    n = 300
    x = torch.randn(n * (n + 1) // 2, device="cuda")
    x1 = x + 0.05 * torch.randn_like(x)
    d = P.stat_distances(x, x1, None, n, 0)
    w = np.concatenate([[1.0] + [2.0] * (n - 1 - i) for i in range(n)])
    xn, x1n = x.cpu().numpy().astype(np.float64), x1.cpu().numpy().astype(np.float64)
    assert d[0] == pytest.approx(np.sqrt((w * (xn - x1n) ** 2).sum()), rel=1e-6)
    assert d[1] == pytest.approx(np.sqrt((w * x1n * x1n).sum()), rel=1e-6)
    ref = np.zeros(6)
    assert O.similar(xn[:6], x1n[:6], np.ones(6), 0.5) == (np.linalg.norm(xn[:6] - x1n[:6]) /
                                                           np.linalg.norm(x1n[:6]) < 0.5)


def test_bn_grad_reduce_matches_oracle(cuda_dev):
    """per-sample BN gradients (net.cpp:467-475) from dY and
    x_hat in one batched launch; odd S (scalar path), S % 4 == 0 (float4 path),
    a large S and single-channel / single-sample edges."""
    shapes = [(4, 16, 49), (3, 8, 196), (2, 4, 3136), (1, 1, 12544), (5, 1, 1), (2, 3, 4)]
    g = torch.Generator(device="cuda").manual_seed(11)
    items, host = [], []
    for M, c, S in shapes:
        dy = torch.randn(M, c * S, device="cuda", generator=g)
        xh = torch.randn(M, c * S, device="cuda", generator=g)
        items.append((dy, xh, M, c, S))
        host.append((dy.cpu().numpy(), xh.cpu().numpy(), M, c, S))
    outs = P.bn_grad_reduce_batched(items)
    for (gg, gb), (dy, xh, M, c, S) in zip(outs, host):
        wg, wb = O.bn_grad_reduce(dy, xh, M, c, S)
        scale = np.sqrt(S)  # fp32 accumulation of S terms
        assert np.abs(gg.cpu().numpy() - wg).max() <= 2e-6 * scale * max(1.0, np.abs(wg).max())
        assert np.abs(gb.cpu().numpy() - wb).max() <= 2e-6 * scale * max(1.0, np.abs(wb).max())
    with pytest.raises(P.EmptyBatch):
        P.bn_grad_reduce(items[0][0], items[0][1], 0, 16, 49)


@pytest.mark.parametrize("m,c,lam", [(64, 16, 2.5e-4), (32, 32, 1e-2), (8, 1, 2.5e-4)])
def test_bn_full_block_matches_oracle(cuda_dev, m, c, lam):
    """BnMode::Full: build_bn_full (fisher.cpp:187-216),
    damp_bn_full (:248-253), precondition_bn_full (:278-296) and the BN update
    of ngd_step (:346-359) against the fp64 oracle."""
    torch.manual_seed(1000 * m + c)  # fixed inputs: the c = 1 case compares a 1-element beta
    gg = torch.randn(m, c, device="cuda")
    gb = 0.6 * gg + 0.8 * torch.randn(m, c, device="cuda")
    cap = P.CaptureBuffer(m, [P.LayerCapture(bn_ggamma_true=gg, bn_gbeta_true=gb)])
    net = P.NetworkSpec([P.LayerSpec.batch_norm(c)])
    blk = P.build_bn_full(cap, net, 0)
    want_f = O.build_bn_full(gg.cpu().numpy(), gb.cpu().numpy(), 0, m)
    assert rel(blk.F.data.cpu().numpy(), want_f) <= 1e-6
    P.damp_bn_full(blk, lam)
    finv = O.spd_inverse(want_f, 2 * c, lam)
    xg, xb = torch.randn(c, device="cuda"), torch.randn(c, device="cuda")
    pg, pb = P.precondition_bn_full(blk, xg, xb)
    wg, wb = O.precondition_bn_full(finv, xg.cpu().numpy(), xb.cpu().numpy())
    assert rel(pg.cpu().numpy(), wg) <= 1e-4 and rel(pb.cpu().numpy(), wb) <= 1e-4
    gamma, beta = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
    vg, vb = 0.01 * torch.randn(c, device="cuda"), 0.01 * torch.randn(c, device="cuda")
    g0, b0, vg0, vb0 = gamma.cpu().numpy(), beta.cpu().numpy(), vg.cpu().numpy(), vb.cpu().numpy()
    P.bn_full_update(blk, torch.cat([xg, xb]).contiguous(), gamma, beta, vg, vb, 1.25e-2, 0.993)
    ng, nvg = O.ngd_update(g0, wg, vg0, 1.25e-2, 0.993)
    nb, nvb = O.ngd_update(b0, wb, vb0, 1.25e-2, 0.993)
    assert rel(gamma.cpu().numpy(), ng) <= 1e-4 and rel(beta.cpu().numpy(), nb) <= 1e-4
    with pytest.raises(P.ShapeMismatch):
        P.precondition_bn_full(blk, torch.zeros(c + 1, device="cuda"), xb)


def test_pair_sm_factor_kernel_subprocess(cuda_dev):
    """The opt-in 2-CTA (cta_group::2) factor SYRK (SPNGD_PAIR=1, gemm_pair.cu)
    passes the same factor parity tests (run in a subprocess: the switch is read
    once per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SPNGD_PAIR="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-k",
                        "conv_factor_A or fc_factor", os.path.join(root, "tests", "test_gpu_kernels.py")],
                       env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
