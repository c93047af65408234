"""Pins the fp64 oracle to the reference's own known-answer and identity tests.

The reference ships no golden bit-vectors; its hot-path tests
are math-defined.  Each case below ports one of them (cited file:line under
/root/reference/proj/tests) onto the oracle with the reference's tolerance,
so the oracle that judges the CUDA path is itself anchored to the reference.
"""
import numpy as np
import pytest

import oracle as O


def random_symmetric(n, seed):
    v = O.rng_normal(seed, n * n).reshape(n, n)
    return np.triu(v) + np.triu(v, 1).T


def dense_kron(g, a):  # tests/oracles.hpp:32-40
    return np.kron(g, a)


# ---- test_linalg.cpp ------------------------------------------------------
def test_packed_sizes():  # test_linalg.cpp:23-29
    assert [O.packed_size(n) for n in (1, 2, 4, 6, 10)] == [1, 3, 10, 21, 55]


def test_pack_unpack_roundtrip_and_layout():  # test_linalg.cpp:31-64
    for n in (1, 2, 3, 7, 12):
        s = random_symmetric(n, 101 + n)
        p = O.pack(s)
        assert p.size == O.packed_size(n)
        assert np.array_equal(O.unpack(p, n), s)
    m = np.array([[1.0, 2.0], [99.0, 3.0]])
    assert list(O.pack(m)) == [1.0, 2.0, 3.0]
    # (0,0),(0,1),(0,2),(1,1),(1,2),(2,2)
    assert [O.lib().or_packed_offset(3, i, j) for i, j in
            [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]] == list(range(6))
    assert O.lib().or_packed_offset(3, 2, 0) == 2


def test_spd_inverse_multiply_back():  # test_linalg.cpp:66-77
    for n in (1, 3, 6, 9):
        s = O.random_spd(n, 7 + n)
        inv = O.unpack(O.spd_inverse(O.pack(s), n, 0.3), n)
        assert np.abs(inv @ (s + 0.3 * np.eye(n)) - np.eye(n)).max() < 1e-10
        inv_f = O.unpack(O.spd_inverse(O.pack(s), n, 0.3, fast=True), n)
        assert np.abs(inv_f - inv).max() < 1e-12


def test_spd_inverse_symmetric_exactly():  # test_linalg.cpp:79-84
    u = O.unpack(O.spd_inverse(O.pack(O.random_spd(5, 8)), 5, 1e-3), 5)
    assert np.array_equal(u, u.T)


def test_spd_inverse_rejects_broken():  # test_linalg.cpp:86-94
    bad = np.eye(3)
    bad[1, 1] = np.nan
    with pytest.raises(O.OracleError, match="NotPositiveDefinite"):
        O.spd_inverse(O.pack(bad), 3, 1.0)
    with pytest.raises(O.OracleError, match="NotPositiveDefinite"):
        O.spd_inverse(O.pack(-2 * np.eye(3)), 3, 0.5)


def test_inv2x2_known_answer():  # test_linalg.cpp:96-104
    a, b, c, d = O.inv2x2(4.0, 7.0, 2.0, 6.0)
    assert np.allclose([a, b, c, d], [0.6, -0.7, -0.2, 0.4], rtol=1e-12, atol=0)
    for args in [(1.0, 2.0, 2.0, 4.0), (0.0, 0.0, 0.0, 0.0)]:
        with pytest.raises(O.OracleError, match="SingularBlock"):
            O.inv2x2(*args)


def test_kron_matvec_equals_dense_kronecker():  # test_linalg.cpp:106-116
    gd, ad = O.random_spd(4, 21), O.random_spd(3, 22)
    x = O.rng_normal(23, 12).reshape(4, 3)
    got = O.kron_matvec(O.pack(gd), O.pack(ad), 4, 3, x)
    want = dense_kron(gd, ad) @ x.reshape(-1)
    assert np.abs(got.reshape(-1) - want).max() < 1e-12
    with pytest.raises(O.OracleError, match="ShapeMismatch"):  # :118-122
        O.kron_matvec(O.pack(gd), O.pack(ad), 4, 3, np.zeros((3, 4)))


def test_avg_eigenvalue():  # test_linalg.cpp:124-129
    m = np.array([[4.0, 1.0, 0.0], [1.0, 2.0, 0.5], [0.0, 0.5, 6.0]])
    assert O.avg_eigenvalue(O.pack(m), 3) == pytest.approx(4.0, rel=1e-15)


def test_frob_and_rel_distance():  # test_linalg.cpp:131-154
    for n in (1, 2, 5, 8):
        s = random_symmetric(n, 31 + n)
        assert O.frob_norm(O.pack(s), n) == pytest.approx(np.linalg.norm(s), rel=1e-13)
    od = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert O.frob_norm(O.pack(od), 2) == pytest.approx(np.sqrt(2.0), rel=1e-15)
    a, b = random_symmetric(5, 41), random_symmetric(5, 42)
    want = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert O.rel_frob_distance(O.pack(a), O.pack(b), 5) == pytest.approx(want, rel=1e-12)
    with pytest.raises(O.OracleError, match="ZeroReference"):
        O.rel_frob_distance(O.pack(a), np.zeros(15), 5)


# ---- test_fisher.cpp ------------------------------------------------------
def mean_outer_dense(stacked, r, lo, hi, denom):  # test_fisher.cpp:60-74
    dim = stacked.shape[1] if r == 1 else r
    acc = np.zeros((dim, dim))
    for s in range(lo, hi):
        blk = stacked[s:s + 1] if r == 1 else stacked[s * r:(s + 1) * r]
        acc += blk.T @ blk if r == 1 else blk @ blk.T
    return acc / denom


def test_fc_factor_A_and_G():  # test_fisher.cpp:89-119
    rng = np.random.default_rng(20250801)
    x = rng.random((6, 5)).astype(np.float32)
    A = O.factor_A(x, False, 5, 1, 0, 6)
    assert np.abs(O.unpack(A, 5) - mean_outer_dense(x.astype(np.float64), 1, 0, 6, 6.0)).max() <= 1e-14
    g = rng.standard_normal((6, 7)).astype(np.float32)
    G = O.factor_G(g, False, 7, 1, 0, 6)
    assert np.abs(O.unpack(G, 7) - mean_outer_dense(g.astype(np.float64), 1, 0, 6, 6.0)).max() <= 1e-14


def conv_capture(m, c, h, w, k, stride, pad, seed):
    rng = np.random.default_rng(seed)
    xs = rng.random((m, c * h * w))
    cols = [O.im2col(xs[s], c, h, w, k, stride, pad) for s in range(m)]
    return xs, np.concatenate(cols, axis=0)


def test_conv_im2col_capture_and_scaling():  # test_fisher.cpp:121-169
    m = 5
    xs, act = conv_capture(m, 2, 4, 4, 3, 1, 1, 20250803)
    # direct check of the im2col index order (net.cpp:207): row = ch*9+ky*3+kx
    x0 = xs[0].reshape(2, 4, 4)
    cols = act[:18]
    assert cols[1 * 9 + 1 * 3 + 1, 0 * 4 + 0] == x0[1, 0, 0]
    assert cols[0 * 9 + 0 * 3 + 0, 0] == 0.0  # padded corner
    A = O.factor_A(act.astype(np.float32), True, 18, 16, 0, m)
    want = mean_outer_dense(act.astype(np.float32).astype(np.float64), 18, 0, m, m * 16.0)
    assert np.abs(O.unpack(A, 18) - want).max() <= 1e-13
    rng = np.random.default_rng(20250804)
    grad = rng.standard_normal((m * 4, 4)).astype(np.float32)
    G = O.factor_G(grad, True, 4, 4, 0, m)
    wantG = mean_outer_dense(grad.astype(np.float64), 4, 0, m, float(m))
    assert np.abs(O.unpack(G, 4) - wantG).max() <= 1e-13
    # mis-scaling G by hw would be caught
    assert np.abs(O.unpack(G, 4) - wantG / 4).max() > 1e-3


def test_subrange_shard_means_recombine():  # test_fisher.cpp:171-197
    m = 6
    _, act = conv_capture(m, 2, 4, 4, 3, 1, 1, 20250805)
    act = act.astype(np.float32)
    lo = O.unpack(O.factor_A(act, True, 18, 16, 0, 2), 18)
    hi = O.unpack(O.factor_A(act, True, 18, 16, 2, m), 18)
    full = O.unpack(O.factor_A(act, True, 18, 16, 0, m), 18)
    assert np.abs(full - (2 * lo + 4 * hi) / 6).max() <= 1e-12
    with pytest.raises(O.OracleError, match="EmptyBatch"):  # :199-229
        O.factor_A(act, True, 18, 16, 2, 2)


def test_compensated_matches_plain():  # test_dist.cpp:596-618 (<=1e-10)
    _, act = conv_capture(6, 2, 4, 4, 3, 1, 1, 7)
    act = act.astype(np.float32)
    a = O.factor_A(act, True, 18, 16, 0, 6, compensated=False)
    b = O.factor_A(act, True, 18, 16, 0, 6, compensated=True)
    assert np.abs(a - b).max() <= 1e-10


def test_damped_inverse_worked_example():  # test_fisher.cpp:231-249, acceptance.cpp:124-140
    pi, Ai, Gi = O.damp_and_invert(O.pack(4 * np.eye(2)), O.pack(np.eye(3)), 2, 3, 1.0)
    assert abs(pi - 2.0) <= 1e-15
    assert np.abs(O.unpack(Ai, 2) - np.eye(2) / 6).max() <= 1e-15
    assert np.abs(O.unpack(Gi, 3) - np.eye(3) * 2 / 3).max() <= 1e-15


def test_pi_guard_and_lambda_positive():  # test_fisher.cpp:251-276
    pi, Ai, _ = O.damp_and_invert(np.zeros(3), O.pack(np.eye(3)), 2, 3, 0.25)
    assert pi == 1.0
    assert np.abs(O.unpack(Ai, 2) - 2 * np.eye(2)).max() <= 1e-15
    pi2, _, _ = O.damp_and_invert(O.pack(np.eye(2)), np.zeros(6), 2, 3, 0.25)
    assert pi2 == 1.0
    for lam in (0.0, -1.0):
        with pytest.raises(O.OracleError, match="NotPositiveDefinite"):
            O.damp_and_invert(np.zeros(3), O.pack(np.eye(3)), 2, 3, lam)
    with pytest.raises(O.OracleError, match="NotPositiveDefinite"):
        O.damp_bn(np.zeros(6), 0.0)


@pytest.mark.parametrize("trial", range(10))
def test_precondition_vs_dense_kron_inverse(trial):  # test_fisher.cpp:278-306, acceptance.cpp:142-176
    rng = np.random.default_rng(501 + trial)
    da, dg = 2 + rng.integers(5), 2 + rng.integers(5)
    lam = 0.1 if trial % 2 == 0 else 1.0
    A, G = O.random_spd(da, 600 + trial), O.random_spd(dg, 700 + trial)
    pi, Ai, Gi = O.damp_and_invert(O.pack(A), O.pack(G), da, dg, lam)
    root = np.sqrt(lam)
    Ad = A + pi * root * np.eye(da)
    Gd = G + root / pi * np.eye(dg)
    X = rng.standard_normal((dg, da))
    want = np.linalg.solve(dense_kron(Gd, Ad), X.reshape(-1))
    got = O.kron_matvec(Gi, Ai, dg, da, X)
    assert np.abs(got.reshape(-1) - want).max() <= 1e-8
    rt = O.kron_matvec(Gi, Ai, dg, da, Gd @ X @ Ad)
    assert np.abs(rt - X).max() <= 1e-8


def test_unit_bn_moments_and_full_diagonal():  # test_fisher.cpp:308-346
    rng = np.random.default_rng(20250807)
    m, c = 6, 3
    gg, gb = rng.standard_normal((m, c)), rng.standard_normal((m, c))
    u = O.build_bn_block(gg, gb, 0, m)
    for ch in range(c):
        assert u[3 * ch] == pytest.approx((gg[:, ch] ** 2).sum() / m, rel=1e-14)
        assert u[3 * ch + 1] == pytest.approx((gg[:, ch] * gb[:, ch]).sum() / m, rel=1e-14)
        assert u[3 * ch + 2] == pytest.approx((gb[:, ch] ** 2).sum() / m, rel=1e-14)
    F = O.unpack(O.build_bn_full(gg, gb, 0, m), 2 * c)
    for ch in range(c):
        assert F[2 * ch, 2 * ch] == u[3 * ch]
        assert F[2 * ch, 2 * ch + 1] == u[3 * ch + 1]
        assert F[2 * ch + 1, 2 * ch + 1] == u[3 * ch + 2]
    assert abs(F[0, 2]) > 0


def test_damp_bn_precondition_bn_vs_2x2_inverse():  # test_fisher.cpp:348-398
    rng = np.random.default_rng(47)
    c = 4
    a, b = rng.standard_normal(c), rng.standard_normal(c)
    m3 = np.stack([a * a + 0.1, a * b, b * b + 0.1], 1).reshape(-1)
    lam = 0.05
    inv = O.damp_bn(m3, lam)
    gg, gb = rng.standard_normal(c), rng.standard_normal(c)
    pg, pb = O.precondition_bn(m3, gg, gb, lam)
    for ch in range(c):
        Fi = np.linalg.inv(np.array([[m3[3 * ch] + lam, m3[3 * ch + 1]],
                                     [m3[3 * ch + 1], m3[3 * ch + 2] + lam]]))
        assert inv[3 * ch] == pytest.approx(Fi[0, 0], rel=1e-12)
        assert inv[3 * ch + 1] == pytest.approx(Fi[0, 1], rel=1e-12)
        assert inv[3 * ch + 2] == pytest.approx(Fi[1, 1], rel=1e-12)
        sol = Fi @ np.array([gg[ch], gb[ch]])
        assert pg[ch] == pytest.approx(sol[0], rel=1e-12)
        assert pb[ch] == pytest.approx(sol[1], rel=1e-12)
    with pytest.raises(O.OracleError, match="ShapeMismatch"):
        O.precondition_bn(m3, np.zeros(c + 1), gb, lam)


def test_full_bn_solve():  # test_fisher.cpp:400-434
    rng = np.random.default_rng(20250808)
    m, c, lam = 8, 3, 0.02
    gg, gb = rng.standard_normal((m, c)), rng.standard_normal((m, c))
    F = O.build_bn_full(gg, gb, 0, m)
    Finv = O.spd_inverse(F, 2 * c, lam)
    xg, xb = rng.standard_normal(c), rng.standard_normal(c)
    pg, pb = O.precondition_bn_full(Finv, xg, xb)
    u = np.stack([xg, xb], 1).reshape(-1)
    sol = np.linalg.solve(O.unpack(F, 2 * c) + lam * np.eye(2 * c), u)
    assert np.allclose(pg, sol[0::2], rtol=1e-10, atol=0)
    assert np.allclose(pb, sol[1::2], rtol=1e-10, atol=0)


def test_plain_and_identity_step_exact():  # test_fisher.cpp:436-511
    rng = np.random.default_rng(71)
    p, g, v = (rng.standard_normal(20) for _ in range(3))
    np_, nv = O.ngd_update(p, g, v, 0.07, 0.9)
    assert np.array_equal(np_, p - 0.07 * g + 0.9 * v)
    assert np.array_equal(nv, np_ - p)
    # identity preconditioners (A_inv = I, G_inv = I) reproduce the plain step
    X = g.reshape(4, 5)
    P = O.kron_matvec(O.pack(np.eye(4)), O.pack(np.eye(5)), 4, 5, X)
    assert np.array_equal(P, X)


def test_preconditioned_step_vs_dense_ngd():  # test_fisher.cpp:513-553
    rng = np.random.default_rng(20250809)
    x = rng.random((8, 5)).astype(np.float32)
    gr = rng.standard_normal((8, 7)).astype(np.float32)
    A, G = O.factor_A(x, False, 5, 1, 0, 8), O.factor_G(gr, False, 7, 1, 0, 8)
    lam = 0.1
    pi, Ai, Gi = O.damp_and_invert(A, G, 5, 7, lam)
    W, dW = rng.standard_normal((7, 5)), rng.standard_normal((7, 5))
    v = 0.01 * rng.standard_normal((7, 5))
    delta = O.kron_matvec(Gi, Ai, 7, 5, dW)
    np_, _ = O.ngd_update(W, delta, v, 0.2, 0.9)
    root = np.sqrt(lam)
    Ad = O.unpack(A, 5) + pi * root * np.eye(5)
    Gd = O.unpack(G, 7) + root / pi * np.eye(7)
    dv = np.linalg.solve(dense_kron(Gd, Ad), dW.reshape(-1)).reshape(7, 5)
    assert np.abs(np_.reshape(7, 5) - (W - 0.2 * dv + 0.9 * v)).max() <= 1e-8


def test_unit_bn_vs_dense_block_acceptance4():  # acceptance.cpp:181-233
    lam = 2.5e-4
    rng = np.random.default_rng(601)
    worst = 0.0
    for c in range(1, 33):
        g = rng.standard_normal((64, c))
        b = 0.6 * g + 0.8 * rng.standard_normal((64, c))
        m3 = O.build_bn_block(g, b, 0, 64)
        xg, xb = rng.standard_normal(c), rng.standard_normal(c)
        pg, pb = O.precondition_bn(m3, xg, xb, lam)
        F = np.zeros((2 * c, 2 * c))
        for ch in range(c):
            F[2 * ch, 2 * ch] = m3[3 * ch]
            F[2 * ch, 2 * ch + 1] = F[2 * ch + 1, 2 * ch] = m3[3 * ch + 1]
            F[2 * ch + 1, 2 * ch + 1] = m3[3 * ch + 2]
        sol = np.linalg.solve(F + lam * np.eye(2 * c), np.stack([xg, xb], 1).reshape(-1))
        worst = max(worst, np.abs(pg - sol[0::2]).max(), np.abs(pb - sol[1::2]).max())
    assert worst <= 1e-10


def test_rescale_norm_and_idempotence():  # test_schemes.cpp:239-259
    w = O.rng_normal(51, 6 * 11)
    r, _ = O.rescale(w, w, 6)
    assert np.linalg.norm(r) == pytest.approx(np.sqrt(12.0), rel=1e-9)
    assert np.abs(r / np.linalg.norm(r) - w / np.linalg.norm(w)).max() <= 1e-12
    r2, _ = O.rescale(r, r, 6)
    assert np.abs(r2 - r).max() <= 1e-8
    z, _ = O.rescale(np.zeros(12), np.zeros(12), 3)
    assert (z == 0).all()


# ---- test_stale.cpp (similarity) -------------------------------------------
def test_similar_strict_threshold_and_weights():  # test_stale.cpp:79-110
    ref = np.array([3.0, 0.0, 4.0])
    x = ref.copy()
    x[1] = 1.0
    w1 = np.ones(3)
    assert O.similar(x, ref, w1, 0.25)
    assert not O.similar(x, ref, w1, 0.2)
    assert not O.similar(ref, ref, w1, 0.0)
    assert O.similar(np.zeros(2), np.zeros(2), np.ones(2), 0.5)
    assert not O.similar(np.array([1e-3, 0.0]), np.zeros(2), np.ones(2), 0.5)
    w = np.array([1.0, 2.0, 1.0])
    x = ref.copy()
    x[1] = 0.5
    assert not O.similar(x, ref, w, 0.13)
    assert O.similar(x, ref, w, 0.15)


# ---- cross-check against an independent numpy/scipy fp64 path ---------------
def test_oracle_vs_numpy_at_resnet_like_shape():
    """Independent check: im2col conv factors + damped inverse vs numpy."""
    rng = np.random.default_rng(9)
    m, c, h, w = 3, 8, 7, 7
    xs = np.maximum(rng.standard_normal((m, c * h * w)), 0)
    act = np.concatenate([O.im2col(xs[s], c, h, w, 3, 1, 1) for s in range(m)]).astype(np.float32)
    a = c * 9
    A = O.factor_A(act, True, a, 49, 0, m)
    Ad = sum(act[s * a:(s + 1) * a].astype(np.float64) @ act[s * a:(s + 1) * a].astype(np.float64).T
             for s in range(m)) / (m * 49)
    assert np.abs(O.unpack(A, a) - Ad).max() / np.abs(Ad).max() < 1e-13
    Ai = O.unpack(O.spd_inverse(A, a, 0.05), a)
    assert np.abs(Ai - np.linalg.inv(Ad + 0.05 * np.eye(a))).max() / np.abs(Ai).max() < 1e-10


def test_synth_stream_deterministic():
    a = O.synth_normal(1234, 0, 1000)
    b = O.synth_normal(1234, 500, 500)
    assert np.array_equal(a[500:], b)
    assert abs(a.mean()) < 0.1 and abs(a.std() - 1) < 0.1


def test_bn_grad_reduce_oracle():  # net.cpp:467-475 per-sample gamma/beta gradients
    rng = np.random.default_rng(3)
    M, c, S = 3, 5, 7
    dy = rng.standard_normal((M, c * S)).astype(np.float32)
    xh = rng.standard_normal((M, c * S)).astype(np.float32)
    gg, gb = O.bn_grad_reduce(dy, xh, M, c, S)
    d3 = dy.astype(np.float64).reshape(M, c, S)
    x3 = xh.astype(np.float64).reshape(M, c, S)
    assert np.allclose(gg, (d3 * x3).sum(-1), rtol=0, atol=1e-12)
    assert np.allclose(gb, d3.sum(-1), rtol=0, atol=1e-12)
    with pytest.raises(O.OracleError):
        O.bn_grad_reduce(dy[:0], xh[:0], 0, c, S)   # EmptyBatch
