"""Stale-statistics gating fused into spngd_opt_step (BASELINE config 4).

Gating follows accumulate_microsteps (dist.cpp:431-444 due sets, 514-537 RS of
due statistics only, 588-601 rebuild + re-invert both factors of a touched
layer) with the StaleTracker schedule of stale.hpp:78-132.  The expected refresh
pattern is computed here from fp64 oracle statistics with a restatement of the
tracker (test infrastructure), and the fused step must match it step by step:
which statistics refreshed, the next refresh step, the statistics the owner
holds, and the inverses formed from them (<= 1e-4, north_star gate).  The layers
change on different schedules so partial refreshes (some statistics due, some
not) are exercised.
"""
import numpy as np
import pytest
import torch

import oracle as O
from oracle import ledger as OL

pytestmark = pytest.mark.gpu

from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import (A_PACKED, ACT, AINV, BN_GB, BN_GG, BN_M3C, DW, G_PACKED, GINV, GRAD,  # noqa: E402
                                        Optimizer)

LAYERS = [W.conv(8, 16, 3, 1, 8), W.bn(16), W.fc(64, 10)]
B = 4
ALPHA = 0.1
LAM = 2.5e-4


class PyTracker:
    """StaleTracker (stale.hpp:92-132) with next_interval (stale.hpp:78-88)."""

    def __init__(self):
        self.t_x, self.delta, self.delta_prev, self.x1, self.x2 = 1, 1, 1, None, None

    def refresh(self, x, w, step):
        if self.x1 is None or not O.similar(x, self.x1, w, ALPHA):
            nd = max(1, self.delta // 2)
        elif self.x2 is None or not O.similar(x, self.x2, w, ALPHA):
            nd = self.delta
        else:
            nd = self.delta + self.delta_prev
        self.x2, self.x1 = self.x1, x
        self.delta_prev, self.delta = self.delta, nd
        self.t_x = step + nd


def packed_weights(n):
    w = np.full(n * (n + 1) // 2, 2.0)
    off = 0
    for i in range(n):
        w[off] = 1.0          # diagonal (packed row i starts at (i, i))
        off += n - i
    return w


def bn_weights(c):
    return np.tile([1.0, 2.0, 1.0], c)


def captures(step, rng_seed):
    """Per-layer host captures for `step`: conv/FC constant except a jump at
    step 5 (conv) ; BN jumps at step 2 and stays.  Tiny noise (1e-6) keeps
    'constant' statistics similar but not bit-identical."""
    out = []
    for li, l in enumerate(LAYERS):
        if l.kind == "bn":
            base = 1 + (step >= 2)
            g = np.random.default_rng(100 * li + base).standard_normal((B, l.g)).astype(np.float32)
            b = (0.6 * g + 0.8 * np.random.default_rng(100 * li + base + 50).standard_normal((B, l.g))).astype(
                np.float32)
            out.append(dict(gg=g, gb=b))
            continue
        base = 1 + (step >= 5 and l.kind == "conv")
        hw = l.hw if l.kind == "conv" else 1
        r = np.random.default_rng(100 * li + base)
        act = np.maximum(r.standard_normal((B * l.a, hw)), 0).astype(np.float32)
        grad = (r.standard_normal((B * l.g, hw)) / np.sqrt(B * hw)).astype(np.float32)
        noise = np.random.default_rng(rng_seed + step)
        act = (act * (1 + 1e-6 * noise.standard_normal(act.shape))).astype(np.float32)
        out.append(dict(act=act, grad=grad))
    return out


def host_stats(l, cap):
    if l.kind == "bn":
        return dict(F=O.build_bn_block(cap["gg"].astype(np.float64), cap["gb"].astype(np.float64), 0, B))
    conv = l.kind == "conv"
    hw = l.hw if conv else 1
    act = cap["act"].reshape(B * l.a, hw) if conv else cap["act"].reshape(B, l.a)
    grad = cap["grad"].reshape(B * l.g, hw) if conv else cap["grad"].reshape(B, l.g)
    return dict(A=O.factor_A(act, conv, l.a, hw, 0, B), G=O.factor_G(grad, conv, l.g, hw, 0, B))


def test_stale_gating_matches_tracker_schedule(cuda_dev):
    opt = Optimizer(LAYERS, B, lam=LAM, stale=True, stale_alpha=ALPHA)
    try:
        opt.synth(3)
        trackers = {(li, k): PyTracker() for li, l in enumerate(LAYERS) for k in (("F",) if l.kind == "bn" else ("A", "G"))}
        held = {}
        saw_partial = False
        for step in range(1, 12):
            caps = captures(step, 7)
            for li, (l, cap) in enumerate(zip(LAYERS, caps)):
                if l.kind == "bn":
                    opt.upload(li, BN_GG, torch.from_numpy(cap["gg"].reshape(-1)))
                    opt.upload(li, BN_GB, torch.from_numpy(cap["gb"].reshape(-1)))
                else:
                    opt.upload(li, ACT, torch.from_numpy(cap["act"].reshape(-1)))
                    opt.upload(li, GRAD, torch.from_numpy(cap["grad"].reshape(-1)))
            due = {}
            for (li, k), tr in trackers.items():
                due[(li, k)] = step == tr.t_x
                if due[(li, k)]:
                    x = host_stats(LAYERS[li], caps[li])[k]
                    w = bn_weights(LAYERS[li].g) if k == "F" else packed_weights(LAYERS[li].a if k == "A" else LAYERS[li].g)
                    tr.refresh(x, w, step)
                    held[(li, k)] = x
            saw_partial |= 0 < sum(due.values()) < len(due)
            opt.step(step, 1.25e-2, 0.993)
            opt.sync()
            # CommLedger rows of this step (dist.cpp:511-537, 661-662) follow the same decisions
            plan_due = [due[(li, k)] for li, l in enumerate(LAYERS) for k in (("F",) if l.kind == "bn" else ("A", "G"))]
            want_rows = OL.step_rows(LAYERS, 1, step, plan_due, 4)
            got_rows = [(r.step, r.stage, r.collective, r.statistic_id, r.elements, r.bytes, r.skipped)
                        for r in opt.ledger().rows() if r.step == step]
            assert got_rows == want_rows, step
            for (li, k), tr in trackers.items():
                info = opt.stale_info(li, k)
                assert info["refreshed"] == due[(li, k)], (step, li, k)
                which = {"A": A_PACKED, "G": G_PACKED, "F": BN_M3C}[k]
                got = opt.download(li, which).numpy().astype(np.float64)
                want = held[(li, k)]
                assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want), (step, li, k)
                assert info["t_x"] == tr.t_x, (step, li, k, info, tr.t_x)
        assert saw_partial
        # inverses of the conv layer come from the held (stale) statistics
        l = LAYERS[0]
        pi, ai, gi = O.damp_and_invert(held[(0, "A")], held[(0, "G")], l.a, l.g, LAM)
        got_a = opt.download(0, AINV).numpy().astype(np.float64)
        got_g = opt.download(0, GINV).numpy().astype(np.float64)
        want_a, want_g = O.unpack(ai, l.a), O.unpack(gi, l.g)
        assert np.linalg.norm(got_a - want_a) <= 1e-4 * np.linalg.norm(want_a)
        assert np.linalg.norm(got_g - want_g) <= 1e-4 * np.linalg.norm(want_g)
    finally:
        opt.close()


def test_stale_constant_inputs_equal_plain_step(cuda_dev):
    """With constant captures every refresh rebuilds identical statistics, so
    the gated step must produce bit-identical weights to the ungated one."""
    ws = []
    for stale in (False, True):
        opt = Optimizer(LAYERS, B, lam=LAM, stale=stale)
        try:
            opt.synth(5)
            for step in range(1, 7):
                opt.step(step, 1.25e-2, 0.993)
            opt.sync()
            ws.append([opt.download(li, 3).numpy() for li in range(len(LAYERS))])
            if stale:
                assert [opt.stale_info(0, "A")["t_x"], opt.stale_info(2, "G")["t_x"]] == [8, 8]  # 1,2,3,5,8
        finally:
            opt.close()
    for a, b in zip(*ws):
        assert np.array_equal(a, b)


def test_stale_partial_refresh_replans_large_classes(cuda_dev):
    """Partial refreshes whose due subset changes from step to step, in a size
    class large enough for 2-CTA recursion rounds (three 4608-wide FC layers):
    each re-planned recursion covers only the due members, and its plan may
    choose 2-CTA / single-CTA rounds differently from the full class plan (the
    re-plan buffers are sized for either).  Each layer's captures jump at its
    own step, so the due subsets differ; held statistics and the inverses
    formed from them match the fp64 oracle (dist.cpp:588-601 re-invert both).
    (The descriptor-upload ordering bug a drifting ResNet-50 stream exposed is
    covered by scripts/stale_bench.py --drift, profiles/r02_configs/.)"""
    layers = [W.fc(4608, 16) for _ in range(3)]
    bq = 8
    jumps = [3, 4, 6]
    lam = 0.1  # rank-8 factors: keeps cond(A + dI) ~1e3 so the fp32 inverse meets 1e-4 without refinement

    def caps(step):
        out = []
        for li, l in enumerate(layers):
            r = np.random.default_rng(1000 * li + 1 + (step >= jumps[li]))
            act = np.maximum(r.standard_normal((bq, l.a)), 0).astype(np.float32)
            grad = r.standard_normal((bq, l.g)).astype(np.float32)
            out.append((act, grad))
        return out

    opt = Optimizer(layers, bq, lam=lam, stale=True, stale_alpha=ALPHA)
    try:
        trackers = {(li, k): PyTracker() for li in range(len(layers)) for k in ("A", "G")}
        held, subsets = {}, set()
        for step in range(1, 10):
            cs = caps(step)
            for li, (act, grad) in enumerate(cs):
                opt.upload(li, ACT, torch.from_numpy(act.reshape(-1)))
                opt.upload(li, GRAD, torch.from_numpy(grad.reshape(-1)))
            due = {}
            for (li, k), tr in trackers.items():
                due[(li, k)] = step == tr.t_x
                if due[(li, k)]:
                    act, grad = cs[li]
                    l = layers[li]
                    x = (O.factor_A(act.astype(np.float64), False, l.a, 1, 0, bq) if k == "A"
                         else O.factor_G(grad.astype(np.float64), False, l.g, 1, 0, bq))
                    tr.refresh(x, packed_weights(l.a if k == "A" else l.g), step)
                    held[(li, k)] = x
            touched = tuple(li for li in range(len(layers)) if due[(li, "A")] or due[(li, "G")])
            if 0 < len(touched) < len(layers):
                subsets.add(touched)
            opt.step(step, 1.25e-2, 0.993)
            opt.sync()
            for (li, k) in trackers:
                assert opt.stale_info(li, k)["refreshed"] == due[(li, k)], (step, li, k)
        assert len(subsets) >= 2, subsets
        for li, l in enumerate(layers):
            # damp_and_invert (fisher.cpp:218-228) with the blocked fp64 inverse of the oracle
            ea = np.trace(O.unpack(held[(li, "A")], l.a)) / l.a
            eg = np.trace(O.unpack(held[(li, "G")], l.g)) / l.g
            pi = np.sqrt(ea / eg) if min(ea, eg) >= 1e-12 else 1.0
            ai = O.spd_inverse(held[(li, "A")], l.a, pi * np.sqrt(lam), fast=True)
            gi = O.spd_inverse(held[(li, "G")], l.g, np.sqrt(lam) / pi, fast=True)
            got_a = opt.download(li, AINV).numpy().astype(np.float64)
            want_a = O.unpack(ai, l.a)
            assert np.linalg.norm(got_a - want_a) <= 1e-4 * np.linalg.norm(want_a), li
            got_g = opt.download(li, GINV).numpy().astype(np.float64)
            want_g = O.unpack(gi, l.g)
            assert np.linalg.norm(got_g - want_g) <= 1e-4 * np.linalg.norm(want_g), li
    finally:
        opt.close()
