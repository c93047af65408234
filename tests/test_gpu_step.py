"""Whole-step parity (accumulate_microsteps Stages 2-5 at K = 1) against the
fp64 oracle on identical device-generated inputs, rel. Frobenius <= 1e-4 on the
updated weights / velocities (north_star gate).  Full-size MLP (config 1);
ResNet-18/50 checked on a layer sample (the fp64 oracle needs minutes per
4608^2 inverse)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import ACT, BN_GB, BN_GG, DW, GRAD, V, Optimizer  # noqa: E402
from paper_2002_06015_b200.step import (BN_GB_SAMPLED, BN_GG_SAMPLED, EMPIRICAL, GRAD_SAMPLED,  # noqa: E402
                                        ONE_MC)
from paper_2002_06015_b200.step import W as WB  # noqa: E402

ETA, MOM, LAM = 1.25e-2, 0.993, 2.5e-4


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def oracle_layer(l, batch, before):
    act, grad, dW, W0, V0 = (before[k] for k in (ACT, GRAD, DW, WB, V))
    if GRAD_SAMPLED in before:  # factor_G(OneMC) reads grad_sampled (fisher.cpp:127-132)
        grad = before[GRAD_SAMPLED]
    rec = O.OrLayer()
    wo, vo = np.empty(l.g * l.a), np.empty(l.g * l.a)
    rec.is_conv, rec.a, rec.g, rec.hw, rec.batch = int(l.kind == "conv"), l.a, l.g, l.hw, batch
    rec.act, rec.grad, rec.dW, rec.W, rec.V = [b.ctypes.data_as(C.POINTER(C.c_float)) for b in (act, grad, dW, W0, V0)]
    rec.W_out = wo.ctypes.data_as(C.POINTER(C.c_double))
    rec.V_out = vo.ctypes.data_as(C.POINTER(C.c_double))
    O.kfac_layers([rec], LAM, ETA, MOM, rescale=True, fast_inverse=True, threads=1)
    return wo, vo


def oracle_bn(l, batch, before):
    c = l.g
    gg, gb = (BN_GG_SAMPLED, BN_GB_SAMPLED) if BN_GG_SAMPLED in before else (BN_GG, BN_GB)  # fisher.cpp:158-159
    m3 = O.build_bn_block(before[gg].reshape(batch, c), before[gb].reshape(batch, c), 0, batch)
    g2 = before[DW].astype(np.float64)
    pg, pb = O.precondition_bn(m3, g2[:c], g2[c:], LAM)
    return O.ngd_update(before[WB], np.concatenate([pg, pb]), before[V], ETA, MOM)


def run_and_check(layers, batch, check_layers, fisher_mode=EMPIRICAL):
    opt = Optimizer(layers, batch, lam=LAM, fisher_mode=fisher_mode)
    opt.synth(seed=3)
    before = {}
    for li in check_layers:
        l = layers[li]
        ws = [BN_GG, BN_GB, DW, WB, V] if l.kind == "bn" else [ACT, GRAD, DW, WB, V]
        if fisher_mode == ONE_MC:
            ws += [BN_GG_SAMPLED, BN_GB_SAMPLED] if l.kind == "bn" else [GRAD_SAMPLED]
        before[li] = {w: opt.download(li, w).numpy() for w in ws}
    opt.step(1, ETA, MOM)
    opt.sync()
    worst = 0.0
    for li in check_layers:
        l = layers[li]
        wo, vo = (oracle_bn if l.kind == "bn" else oracle_layer)(l, batch, before[li])
        ew = rel(opt.download(li, WB).numpy(), wo)
        ev = rel(opt.download(li, V).numpy(), vo)
        assert ew <= 1e-4 and ev <= 1e-4, f"layer {li} {l}: W {ew:.2e} V {ev:.2e}"
        worst = max(worst, ew, ev)
    ph = opt.phase_ms()
    assert all(v >= 0 for v in ph.values())
    opt.close()
    return worst


def test_mlp_full_step(cuda_dev):
    layers, batch, _ = W.CONFIGS["mlp"]
    run_and_check(layers(), batch, range(3))


def test_small_convnet_full_step(cuda_dev):
    layers = [W.conv(3, 16, 3, 1, 16), W.bn(16), W.conv(16, 32, 3, 2, 16), W.bn(32), W.conv(32, 32, 1, 1, 8),
              W.bn(32), W.fc(32 * 4, 10)]
    run_and_check(layers, 16, range(len(layers)))


def test_one_mc_full_step(cuda_dev):
    """FisherMode::OneMC (dist.cpp:476-480): G and the BN moments come from the
    sampled-label captures; dW stays the true-label gradient.  The sampled
    buffers differ from the true ones, so a step that read the wrong capture
    misses the oracle by O(1)."""
    layers = [W.conv(3, 16, 3, 1, 16), W.bn(16), W.conv(16, 32, 3, 2, 16), W.bn(32), W.fc(32 * 64, 10)]
    run_and_check(layers, 16, range(len(layers)), fisher_mode=ONE_MC)
    from paper_2002_06015_b200.spngd import MissingMcPass
    opt = Optimizer(layers, 16, lam=LAM)
    try:
        with pytest.raises(MissingMcPass):
            opt.ptr(0, GRAD_SAMPLED)
    finally:
        opt.close()


def test_resnet18_sampled_layers(cuda_dev):
    layers = W.resnet18_cifar()
    pick = [0, 1, 2, 5, 8, len(layers) - 1]
    run_and_check(layers, 128, pick)


def test_resnet50_sampled_layers(cuda_dev):
    layers = W.resnet50()
    # conv1 (147x64, K = 401,408 split-K), a 576 3x3, a 1152 3x3, BN, the FC.
    idx = {(l.a, l.g, l.hw): i for i, l in reversed(list(enumerate(layers)))}
    pick = [0, 1, idx[(576, 64, 3136)], idx[(1152, 128, 784)], len(layers) - 1]
    run_and_check(layers, 32, pick)


def test_overlapped_schedule_is_bitwise_phase_serial(cuda_dev):
    """The single-GPU wave schedule (inverse recursion of the largest factors
    overlapping the remaining factor SYRKs) runs the same kernels on the same
    inputs as the phase-serial schedule: results must be bit-identical."""
    layers = W.resnet50()
    outs = []
    for overlap in (True, False):
        opt = Optimizer(layers, 8, lam=LAM)
        opt.set_overlap(overlap)
        opt.synth(seed=5)
        for s in range(2):
            opt.step(s + 1, ETA, MOM)
        opt.sync()
        outs.append([(opt.download(li, WB).numpy().copy(), opt.download(li, V).numpy().copy())
                     for li in range(len(layers))])
        opt.close()
    for li, ((w0, v0), (w1, v1)) in enumerate(zip(*outs)):
        assert np.array_equal(w0, w1) and np.array_equal(v0, v1), f"layer {li} {layers[li]}"


def test_sgd_step(cuda_dev):
    """OptimizerConfig::sgd (ngd_step with blocks == nullptr, fisher.cpp:320-333,
    348-356): W' = W - eta g + m V, V' = W' - W for every layer, no statistics,
    no rescale; the ledger ships only grads and weights."""
    layers = [W.conv(3, 16, 3, 1, 16), W.bn(16), W.fc(16 * 256, 10)]
    opt = Optimizer(layers, 8, lam=LAM, sgd=True)
    try:
        opt.synth(seed=4)
        before = {li: {w: opt.download(li, w).numpy().astype(np.float64) for w in (DW, WB, V)}
                  for li in range(len(layers))}
        opt.step(1, ETA, MOM)
        opt.sync()
        for li in range(len(layers)):
            b = before[li]
            wn = b[WB] - ETA * b[DW] + MOM * b[V]
            assert rel(opt.download(li, WB).numpy(), wn) <= 1e-6
            assert np.allclose(opt.download(li, V).numpy(), wn - b[WB], atol=1e-6)
        ids = [r.statistic_id for r in opt.ledger().rows()]
        assert ids == ["grad:0", "grad:1", "grad:2", "w:0", "w:1", "w:2"]
        assert opt.launch_count() == 1
    finally:
        opt.close()


def test_accumulate_microsteps_equals_concatenated_batch(cuda_dev):
    """accumulate_microsteps (dist.cpp:446-508) averages the per-micro shard
    means of n equal micro-batches: mean_mi(1/m sum_{s in mi}) = 1/(n m) sum_all.
    The device step therefore takes n micro-batches as one capture of n*m
    samples in micro order (batch = n*m); here the oracle restates the
    reference's per-micro accumulation literally and the step must match it."""
    n_micro, m = 3, 4
    layers = [W.conv(3, 8, 3, 1, 8), W.fc(8 * 64, 10)]
    opt = Optimizer(layers, n_micro * m, lam=LAM)
    try:
        opt.synth(seed=9)
        before = {li: {w: opt.download(li, w).numpy() for w in (ACT, GRAD, DW, WB, V)} for li in range(2)}
        opt.step(1, ETA, MOM)
        opt.sync()
        for li, l in enumerate(layers):
            b = before[li]
            conv = l.kind == "conv"
            hw = l.hw if conv else 1
            act = b[ACT].astype(np.float64).reshape(n_micro * m * l.a, hw) if conv else \
                b[ACT].astype(np.float64).reshape(n_micro * m, l.a)
            grad = b[GRAD].astype(np.float64).reshape(n_micro * m * l.g, hw) if conv else \
                b[GRAD].astype(np.float64).reshape(n_micro * m, l.g)
            A = sum(O.factor_A(act, conv, l.a, hw, mi * m, (mi + 1) * m) for mi in range(n_micro)) / n_micro
            G = sum(O.factor_G(grad, conv, l.g, hw, mi * m, (mi + 1) * m) for mi in range(n_micro)) / n_micro
            _, Ai, Gi = O.damp_and_invert(A, G, l.a, l.g, LAM)
            delta = O.kron_matvec(Gi, Ai, l.g, l.a, b[DW].astype(np.float64).reshape(l.g, l.a)).reshape(-1)
            wn, _ = O.ngd_update(b[WB], delta, b[V], ETA, MOM)
            wr, vr = O.rescale(wn, b[WB], l.g)
            assert rel(opt.download(li, WB).numpy(), wr) <= 1e-4
            assert rel(opt.download(li, V).numpy(), vr) <= 1e-4
    finally:
        opt.close()


@pytest.mark.parametrize("stale", [False, True])
def test_full_bn_mode_step(cuda_dev, stale):
    """BnMode::FullBlockDiag2c inside the step (dist.cpp:572-586; build_bn_full,
    damp_bn_full, precondition_bn_full + the BN update, fisher.cpp:187-216,
    248-253, 278-296, 346-359): F from the interleaved per-sample pairs by the
    SYRK engine, (F + lambda I)^-1 by the batched Cholesky, v = T^T (T u).
    rel. Frobenius <= 1e-4 on F^-1, the updated gamma/beta and velocities."""
    from paper_2002_06015_b200.step import AINV, BN_FULL, BN_M3C
    # B > 2c keeps F + lambda I well conditioned; with B < 2c (rank-deficient F,
    # cond ~ |F| / lambda) fp32 inverses lose ~cond * 2^-24 like the config-5
    # K < n sweep inputs
    layers = [W.conv(3, 16, 3, 1, 8), W.bn(16, 64), W.conv(16, 48, 3, 1, 8), W.bn(48, 64), W.fc(48, 10), W.bn(40)]
    B = 160
    opt = Optimizer(layers, B, lam=LAM, bn_mode=BN_FULL, stale=stale)
    try:
        opt.synth(seed=11)
        bns = [li for li, l in enumerate(layers) if l.kind == "bn"]
        before = {li: {w: opt.download(li, w).numpy() for w in (BN_GG, BN_GB, DW, WB, V)} for li in bns}
        opt.step(1, ETA, MOM)
        opt.sync()
        for li in bns:
            c, b = layers[li].g, before[li]
            F = O.build_bn_full(b[BN_GG].reshape(B, c), b[BN_GB].reshape(B, c), 0, B)
            got_F = opt.download(li, BN_M3C).numpy()
            assert rel(got_F, F) <= 1e-5
            finv = O.spd_inverse(F, 2 * c, LAM)
            assert rel(opt.download(li, AINV).numpy(), O.unpack(finv, 2 * c)) <= 1e-4
            g2 = b[DW].astype(np.float64)
            pg, pb = O.precondition_bn_full(finv, g2[:c], g2[c:])
            wo, vo = O.ngd_update(b[WB], np.concatenate([pg, pb]), b[V], ETA, MOM)
            assert rel(opt.download(li, WB).numpy(), wo) <= 1e-4, li
            assert rel(opt.download(li, V).numpy(), vo) <= 1e-4, li
        ids = [r.statistic_id for r in opt.ledger().rows() if r.statistic_id.startswith("F:")]
        assert ids == ["F:1", "F:3", "F:5"]
        if stale:  # steps 2, 3 refresh (Fibonacci 1, 2, 3), 4 does not: every path runs
            for step in (2, 3, 4):
                opt.step(step, ETA, MOM)
            opt.sync()
            assert all(np.isfinite(opt.download(li, WB).numpy()).all() for li in bns)
    finally:
        opt.close()


@pytest.mark.parametrize("fisher_mode", [EMPIRICAL, ONE_MC])
def test_wgrad_in_step(cuda_dev, fisher_mode):
    """cfg.wgrad: the step forms grad_payload itself
    (dist.cpp:315-391: conv sum_s G_s A_s^T / m, FC grad^T act / m, BN column
    means) from the true-label captures -- also under OneMC, where G reads the
    sampled capture -- then preconditions with it.  rel. Frobenius <= 1e-5 on
    dW (fp64 reference), <= 1e-4 on the updated weights."""
    layers = [W.conv(3, 16, 3, 1, 10), W.bn(16, 100), W.conv(16, 32, 3, 2, 10), W.fc(32 * 25, 10)]
    B = 12
    opt = Optimizer(layers, B, lam=LAM, wgrad=True, fisher_mode=fisher_mode)
    try:
        opt.synth(seed=21)
        ws = {li: [ACT, GRAD, WB, V] + ([GRAD_SAMPLED] if fisher_mode == ONE_MC else []) for li in (0, 2, 3)}
        ws[1] = [BN_GG, BN_GB, WB, V] + ([BN_GG_SAMPLED, BN_GB_SAMPLED] if fisher_mode == ONE_MC else [])
        before = {li: {w: opt.download(li, w).numpy() for w in ws[li]} for li in ws}
        opt.step(1, ETA, MOM)
        opt.sync()
        for li, l in enumerate(layers):
            b = before[li]
            if l.kind == "bn":
                c = l.g
                want = np.concatenate([b[BN_GG].reshape(B, c).astype(np.float64).mean(0),
                                       b[BN_GB].reshape(B, c).astype(np.float64).mean(0)])
            elif l.kind == "conv":
                act = b[ACT].astype(np.float64).reshape(B, l.a, l.hw)
                grad = b[GRAD].astype(np.float64).reshape(B, l.g, l.hw)
                want = np.einsum("sgp,sap->ga", grad, act).reshape(-1) / B
            else:
                act = b[ACT].astype(np.float64).reshape(B, l.a)
                grad = b[GRAD].astype(np.float64).reshape(B, l.g)
                want = (grad.T @ act).reshape(-1) / B
            got = opt.download(li, DW).numpy()
            assert rel(got, want) <= 1e-5, (li, rel(got, want))
            b[DW] = want.astype(np.float32)
            wo, vo = (oracle_bn if l.kind == "bn" else oracle_layer)(l, B, b)
            assert rel(opt.download(li, WB).numpy(), wo) <= 1e-4, li
            assert rel(opt.download(li, V).numpy(), vo) <= 1e-4, li
    finally:
        opt.close()


@pytest.mark.parametrize("implicit,wgrad", [(False, False), (True, False), (True, True)])
def test_raw_inputs_step(cuda_dev, implicit, wgrad):
    """spngd_opt_enable_raw_inputs(_ex): the step takes each
    conv layer's raw input (net.cpp:199-219: padding, stride 2, 7x7, 1x1
    stride 2; 1x1 stride 1 aliases the capture) and either expands it on the
    device (the capture must equal the oracle's im2col bit for bit) or, with
    implicit=True, the A-factor SYRK (and the in-step wgrad GEMM) gather the
    im2col operand straight from it and no capture exists.  A factor,
    gradient payload and the updated weights vs the oracle on the oracle's
    im2col of the same raw tensor."""
    from paper_2002_06015_b200.step import A_PACKED, RAW_ACT
    layers = [W.conv(3, 8, 7, 2, 20), W.bn(8, 100), W.conv(8, 16, 3, 1, 10), W.conv(16, 32, 1, 1, 10),
              W.conv(32, 16, 1, 2, 10), W.fc(16 * 25, 10), W.conv(128, 64, 3, 1, 8)]  # a = 1152: 2-CTA SYRK
    B = 6
    opt = Optimizer(layers, B, lam=LAM, wgrad=wgrad)
    try:
        opt.enable_raw_inputs(implicit=implicit)
        opt.synth(seed=31)
        raws = {li: opt.download(li, RAW_ACT).numpy() for li, l in enumerate(layers) if l.kind == "conv"}
        before = {li: {w: opt.download(li, w).numpy() for w in (GRAD, DW, WB, V)} for li in raws}
        opt.step(1, ETA, MOM)
        opt.sync()
        for li, x in raws.items():
            l = layers[li]
            cap = np.concatenate([O.im2col(x.reshape(B, l.c_in * l.h_in * l.w_in)[s], l.c_in, l.h_in, l.w_in, l.k,
                                           l.stride, l.pad) for s in range(B)])
            if not implicit:
                got = opt.download(li, ACT).numpy().reshape(B * l.a, l.hw)
                assert np.array_equal(got, cap.astype(np.float32)), li
            A = O.factor_A(cap, True, l.a, l.hw, 0, B)
            assert rel(opt.download(li, A_PACKED).numpy(), A) <= 1e-5, li
            b = dict(before[li])
            b[ACT] = cap.astype(np.float32).reshape(-1)
            if wgrad:  # grad_payload conv branch (dist.cpp:341-361): sum_s G_s A_s^T / m
                g = b[GRAD].astype(np.float64).reshape(B, l.g, l.hw)
                a = cap.reshape(B, l.a, l.hw)
                dw = np.einsum("sgp,sap->ga", g, a) / B
                assert rel(opt.download(li, DW).numpy(), dw.reshape(-1)) <= 1e-5, li
                b[DW] = opt.download(li, DW).numpy()
            wo, vo = oracle_layer(l, B, b)
            assert rel(opt.download(li, WB).numpy(), wo) <= 1e-4, li
            assert rel(opt.download(li, V).numpy(), vo) <= 1e-4, li
        # 1x1 stride-1 convs alias the capture; with implicit im2col every other
        # conv's capture is gone
        assert opt.ptr(3, RAW_ACT)[0] == opt.ptr(3, ACT)[0]
        for li in (0, 2, 4, 6):
            assert (opt.ptr(li, ACT)[0] is None) == implicit, li
    finally:
        opt.close()


@pytest.mark.parametrize("raw", [False, True])
def test_step_host_equals_device_step(cuda_dev, raw):
    """spngd_opt_step_host: the same step fed from pinned host buffers, the H2D
    copies overlapped wave by wave with the SYRKs (and im2col of raw inputs),
    is bit-identical to the step on device-resident inputs."""
    # conv(256, 64, 3) has a = 2304 > 1536: an earlier wave, so its precondition
    # runs beside the last inverse wave and its weights stream back early
    layers = [W.conv(3, 16, 3, 1, 12), W.bn(16, 144), W.conv(16, 64, 3, 2, 12), W.conv(64, 256, 1, 1, 6),
              W.bn(256, 36), W.fc(256 * 36, 10), W.conv(256, 64, 3, 1, 6)]
    B = 8
    outs = []
    for host in (False, True):
        opt = Optimizer(layers, B, lam=LAM)
        try:
            if raw:
                opt.enable_raw_inputs()
            opt.synth(seed=41)
            if host:
                keep = []
                ins = []
                for li, w in opt.input_buffers():
                    t = opt.download(li, w).pin_memory()
                    keep.append(t)
                    ins.append((li, w, t.data_ptr()))
                for li, w in opt.input_buffers():  # clobber the device copies: the step must use the host inputs
                    opt.upload(li, w, torch.full((opt.numel(li, w),), 7.0))
                wout = torch.empty(opt.ptr(0, 12)[1], dtype=torch.float32).pin_memory()
                opt.step_host(1, ins, wout.data_ptr(), ETA, MOM)
                opt.sync()
                for li in range(len(layers)):  # the weights read back with the step
                    off = (opt.ptr(li, WB)[0] - opt.ptr(0, 12)[0]) // 4
                    w = opt.download(li, WB).numpy()
                    assert np.array_equal(wout.numpy()[off:off + w.size], w), li
            else:
                opt.step(1, ETA, MOM)
                opt.sync()
            outs.append([opt.download(li, WB).numpy() for li in range(len(layers))])
        finally:
            opt.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def _params(opt, layers):
    return [(opt.download(li, WB).numpy().copy(), opt.download(li, V).numpy().copy()) for li in range(len(layers))]


def test_failed_step_names_layer_and_updates_nothing(cuda_dev):
    """A non-finite capture makes layer 2's A factor fail in damp_and_invert:
    the step raises NotPositiveDefinite naming layer 2 / its A factor and no
    parameter of any layer changes -- the reference throws in Stage 4 before
    ngd_step (dist.cpp:597-601)."""
    from paper_2002_06015_b200.spngd import NotPositiveDefinite
    layers = [W.conv(3, 16, 3, 1, 16), W.bn(16), W.conv(16, 32, 3, 2, 16), W.bn(32), W.fc(32 * 64, 10)]
    opt = Optimizer(layers, 8, lam=LAM)
    try:
        opt.set_overlap(False)
        opt.synth(seed=4)
        act = opt.download(2, ACT)
        act[5] = float("nan")
        opt.upload(2, ACT, act)
        before = _params(opt, layers)
        opt.step(1, ETA, MOM)
        with pytest.raises(NotPositiveDefinite) as e:
            opt.sync()
        assert "layer 2" in str(e.value) and "A factor" in str(e.value), str(e.value)
        after = _params(opt, layers)
        for li, ((w0, v0), (w1, v1)) in enumerate(zip(before, after)):
            assert np.array_equal(w0, w1) and np.array_equal(v0, v1), f"layer {li} was updated"
    finally:
        opt.close()


def test_singular_bn_block_updates_nothing(cuda_dev):
    """damp_bn's SingularBlock (fisher.cpp:230-246): a BN layer with all-zero
    per-sample gradients and lambda = 1e-16 has det(F + lambda I) < 1e-30;
    every channel is checked before any parameter is written."""
    from paper_2002_06015_b200.spngd import SingularBlock
    # every Kronecker factor full rank (K = 8 * 64 > a, g), so only the BN block fails
    layers = [W.conv(3, 16, 3, 1, 8), W.bn(16), W.conv(16, 8, 1, 1, 8)]
    opt = Optimizer(layers, 8, lam=1e-16)
    try:
        opt.set_overlap(False)
        opt.synth(seed=6)
        z = torch.zeros(8 * 16)
        opt.upload(1, BN_GG, z)
        opt.upload(1, BN_GB, z)
        before = _params(opt, layers)
        opt.step(1, ETA, MOM)
        with pytest.raises(SingularBlock) as e:
            opt.sync()
        assert "layer 1" in str(e.value), str(e.value)
        after = _params(opt, layers)
        for li, ((w0, v0), (w1, v1)) in enumerate(zip(before, after)):
            assert np.array_equal(w0, w1) and np.array_equal(v0, v1), f"layer {li} was updated"
    finally:
        opt.close()


def test_failed_step_under_wave_schedule_updates_nothing(cuda_dev, monkeypatch):
    """Failure atomicity with the wave schedule on: the early precondition
    part (the FC layer, wave 1) writes W and V while the last wave's SYRK and
    recursion still run; the conv layer's A factor (n = 576, last wave) then
    reports a non-positive pivot at its final leaf (SPNGD_TEST_FAIL_N hook).
    The step must raise naming layer 0 and leave every parameter as it was:
    phase 4 restores the snapshot taken at step start (dist.cpp:597-601)."""
    from paper_2002_06015_b200.spngd import NotPositiveDefinite
    monkeypatch.setenv("SPNGD_TEST_FAIL_N", "576")
    # conv: a = 576 (last wave), K = 32 * 112^2 -> a long last-wave SYRK; fc: a = 1600 (wave 1, early part)
    layers = [W.conv(64, 64, 3, 1, 112), W.fc(1600, 8)]
    opt = Optimizer(layers, 32, lam=LAM)
    try:
        opt.synth(seed=9)
        before = _params(opt, layers)
        opt.step(1, ETA, MOM)
        with pytest.raises(NotPositiveDefinite) as e:
            opt.sync()
        assert "layer 0" in str(e.value) and "A factor" in str(e.value), str(e.value)
        after = _params(opt, layers)
        for li, ((w0, v0), (w1, v1)) in enumerate(zip(before, after)):
            assert np.array_equal(w0, w1) and np.array_equal(v0, v1), f"layer {li} was updated"
    finally:
        opt.close()
    # without the hook the same optimizer updates both layers (the early part did run)
    monkeypatch.delenv("SPNGD_TEST_FAIL_N")
    opt = Optimizer(layers, 32, lam=LAM)
    try:
        opt.synth(seed=9)
        before = _params(opt, layers)
        opt.step(1, ETA, MOM)
        opt.sync()
        after = _params(opt, layers)
        for li, ((w0, _), (w1, _)) in enumerate(zip(before, after)):
            assert not np.array_equal(w0, w1), f"layer {li} was not updated"
    finally:
        opt.close()


@pytest.mark.parametrize("overlap", [True, False])
def test_bn_backward_inputs_in_step(cuda_dev, overlap):
    """SURVEY §8f row 1 inside the step: BN layers take dY / x_hat; the fused
    launch forms the per-sample capture (net.cpp:467-475), the moments
    (fisher.cpp:147-185) and the BN payload (dist.cpp:364-371).  Updated BN
    parameters vs the oracle chain bn_grad_reduce -> build_bn_block ->
    precondition_bn -> ngd_step; Kronecker layers unchanged in meaning."""
    from paper_2002_06015_b200.step import BN_DY, BN_XHAT
    layers = [W.conv(3, 16, 3, 1, 16), W.bn(16), W.conv(16, 32, 3, 2, 16), W.bn(32), W.conv(32, 32, 1, 1, 8),
              W.bn(32), W.fc(32 * 64, 10)]
    batch = 16
    opt = Optimizer(layers, batch, lam=LAM)
    try:
        opt.set_overlap(overlap)
        opt.enable_bn_inputs()
        opt.synth(seed=9)
        before = {}
        for li, l in enumerate(layers):
            ws = [BN_DY, BN_XHAT, WB, V] if l.kind == "bn" else [ACT, GRAD, DW, WB, V]
            before[li] = {w: opt.download(li, w).numpy() for w in ws}
        opt.step(1, ETA, MOM)
        opt.sync()
        for li, l in enumerate(layers):
            b = before[li]
            if l.kind != "bn":
                wo, vo = oracle_layer(l, batch, b)
                assert rel(opt.download(li, WB).numpy(), wo) <= 1e-4
                continue
            c, S = l.g, opt.bn_spatial[li]
            gg, gb = O.bn_grad_reduce(b[BN_DY], b[BN_XHAT], batch, c, S)
            # the captures the step formed
            assert rel(opt.download(li, BN_GG).numpy(), gg.reshape(-1)) <= 1e-5
            assert rel(opt.download(li, BN_GB).numpy(), gb.reshape(-1)) <= 1e-5
            m3 = O.build_bn_block(gg, gb, 0, batch)
            dW = np.concatenate([gg.mean(0), gb.mean(0)])  # grad_payload BN branch
            assert rel(opt.download(li, DW).numpy(), dW) <= 1e-5
            pg, pb = O.precondition_bn(m3, dW[:c], dW[c:], LAM)
            wo, vo = O.ngd_update(b[WB], np.concatenate([pg, pb]), b[V], ETA, MOM)
            ew, ev = rel(opt.download(li, WB).numpy(), wo), rel(opt.download(li, V).numpy(), vo)
            assert ew <= 1e-4 and ev <= 1e-4, f"layer {li}: W {ew:.2e} V {ev:.2e}"
    finally:
        opt.close()


def test_bn_backward_stats_entry_point(cuda_dev):
    """spngd_bn_backward_stats_batched on the ResNet-50 BN shapes (B = 32):
    captures, moments and payload vs the oracle on a few layers."""
    import ctypes as C
    from paper_2002_06015_b200 import _native as N
    from paper_2002_06015_b200.spngd import check, context
    layers = W.resnet50()
    shapes, prev = [], None
    for l in layers:
        if l.kind == "conv":
            prev = l
        elif l.kind == "bn":
            shapes.append((l.g, prev.hw))
    B = 32
    g = torch.Generator(device="cuda").manual_seed(1)
    bufs, reqs = [], []
    for c, S in shapes:
        dy = torch.randn(B * c * S, device="cuda", generator=g) / (B * S) ** 0.5
        xh = torch.randn(B * c * S, device="cuda", generator=g)
        gg, gb = torch.empty(B * c, device="cuda"), torch.empty(B * c, device="cuda")
        m3, pay = torch.empty(3 * c, device="cuda"), torch.empty(2 * c, device="cuda")
        bufs.append((dy, xh, gg, gb, m3, pay))
        reqs.append(N.BnBackwardReq(dy.data_ptr(), xh.data_ptr(), B, c, S, gg.data_ptr(), gb.data_ptr(), m3.data_ptr(),
                                    pay.data_ptr()))
    arr = (N.BnBackwardReq * len(reqs))(*reqs)
    check(N.lib().spngd_bn_backward_stats_batched(context().h, len(reqs), arr))
    for k in (0, 1, 10, len(shapes) - 1):
        (c, S), (dy, xh, gg, gb, m3, pay) = shapes[k], bufs[k]
        wgg, wgb = O.bn_grad_reduce(dy.cpu().numpy(), xh.cpu().numpy(), B, c, S)
        assert rel(gg.cpu().numpy(), wgg.reshape(-1)) <= 1e-5
        assert rel(gb.cpu().numpy(), wgb.reshape(-1)) <= 1e-5
        # moments / payload of the fp32 captures (what build_bn_block would read)
        cg, cb = gg.cpu().numpy().reshape(B, c), gb.cpu().numpy().reshape(B, c)
        assert rel(m3.cpu().numpy(), O.build_bn_block(cg, cb, 0, B)) <= 1e-6
        assert rel(pay.cpu().numpy(), np.concatenate([cg.astype(np.float64).mean(0), cb.astype(np.float64).mean(0)])) <= 1e-6
