"""Communication ledger (CommLedger, dist.hpp:16-56, dist.cpp:42-133): the
native host planner against the oracle restatement (oracle/ledger.py) and the
reference's own ledger tests (tests/test_dist.cpp:214-272, acceptance.cpp:296-338,
test_dist.cpp:497-571)."""
import io
import random

import pytest

from oracle import ledger as OL
from paper_2002_06015_b200 import spngd as S
from paper_2002_06015_b200 import workloads as W


def _tuples(rows):
    return [(r.step, r.stage, r.collective, r.statistic_id, r.elements, r.bytes, r.skipped) for r in rows]


def small_net():  # test_dist.cpp:18-25: conv(1,3,3,1,1), bn(3), fc(3,5) on 1x4x4
    return [W.conv(1, 3, 3, 1, 4), W.bn(3, 16), W.fc(3, 5)]


@pytest.mark.parametrize("world", [1, 2, 8])
@pytest.mark.parametrize("bn_full", [False, True])
def test_planner_matches_oracle(world, bn_full):
    rng = random.Random(world * 7 + bn_full)
    for net in (small_net(), W.mlp(), W.resnet18_cifar(), W.resnet50()):
        n_stats = len(OL.plan_statistics(net))
        for trial in range(4):
            due = None if trial == 0 else [rng.random() < 0.5 for _ in range(n_stats)]
            es = rng.choice([2, 4, 8])
            got = S.ledger_step_rows(net, world, 3 + trial, due, es, bn_full)
            want = OL.step_rows(net, world, 3 + trial, due, es, bn_full)
            assert _tuples(got) == want


@pytest.mark.parametrize("world", [1, 4])
def test_sgd_ledger_has_no_statistics(world):
    """OptimizerConfig::sgd: plan_statistics is empty (dist.cpp:258), grads and weights still ship."""
    net = small_net()
    got = _tuples(S.ledger_step_rows(net, world, 2, sgd=True))
    assert got == OL.step_rows(net, world, 2, sgd=True)
    assert [r[3] for r in got] == ["grad:0", "grad:1", "grad:2", "w:0", "w:1", "w:2"]


def test_symmetry_kat():
    """acceptance.cpp:318-338: fc(4,6)+fc(6,10) at K=2 ships tri(4)+tri(6)+tri(6)+tri(10)."""
    net = [W.fc(4, 6), W.fc(6, 10)]
    rows = S.ledger_step_rows(net, 2, 1)
    shipped = sum(r.elements for r in rows if r.statistic_id[0] in "AG")
    assert shipped == 10 + 21 + 21 + 55


def test_stale_skip_pattern_and_report():
    """test_dist.cpp:497-571: off-schedule steps ship no statistic bytes but the rest;
    the Fibonacci refresh trace {1,2,3,5} / skip {4}."""
    net = small_net()
    n_stats = len(OL.plan_statistics(net))
    led = S.CommLedger()
    for step in range(1, 6):
        due = [step != 4] * n_stats
        for r in S.ledger_step_rows(net, 2, step, due, 4):
            led.record(r.step, r.stage, r.collective, r.statistic_id, r.elements, r.bytes, r.skipped)
    real, skip = {}, {}
    for r in led.rows():
        if r.statistic_id[:2] in ("A:", "G:", "F:"):
            (skip if r.skipped else real).setdefault(r.statistic_id, []).append(r.step)
            if r.skipped:
                assert r.elements == 0 and r.bytes == 0
    for i in ("A:0", "G:0", "F:1", "A:2", "G:2"):
        assert real[i] == [1, 2, 3, 5] and skip[i] == [4]
    rep = S.ledger_report(led)
    assert rep.steps == 5
    assert sum(r.bytes for r in led.rows() if r.step == 4 and r.statistic_id[:2] in ("A:", "G:", "F:")) == 0
    assert rep.reduction_rate < 1.0 and rep.stat_bytes < rep.stat_bytes_every_step
    assert rep.stat_bytes * 5 == rep.stat_bytes_every_step * 4
    # disabled staleness: nothing skipped, rate 1 (test_dist.cpp:574-594)
    full = S.CommLedger(S.ledger_step_rows(net, 2, 1) + S.ledger_step_rows(net, 2, 2))
    assert not any(r.skipped for r in full.rows())
    assert S.ledger_report(full).reduction_rate == 1.0


def test_report_kat():
    """test_dist.cpp:214-242."""
    L = S.CommLedger()
    L.record(1, 2, "RSV_A", "A:0", 10, 40, False)
    L.record(1, 3, "RSV_G_F_grad", "G:0", 6, 24, False)
    L.record(1, 3, "RSV_G_F_grad", "grad:0", 20, 80, False)
    L.record(1, 5, "AGV_params", "w:0", 20, 80, False)
    L.record(2, 2, "RSV_A", "A:0", 0, 0, True)
    L.record(2, 3, "RSV_G_F_grad", "G:0", 6, 24, False)
    L.record(2, 3, "RSV_G_F_grad", "grad:0", 20, 80, False)
    L.record(2, 5, "AGV_params", "w:0", 20, 80, False)
    rep = S.ledger_report(L)
    assert (rep.steps, rep.total_bytes, rep.stat_bytes, rep.grad_bytes, rep.param_bytes) == (2, 408, 88, 160, 160)
    assert rep.stat_bytes_every_step == 128
    assert rep.reduction_rate == pytest.approx(88.0 / 128.0, rel=1e-15)
    assert rep.per_step_bytes == [(1, 224), (2, 184)]
    E = S.CommLedger()
    E.record(1, 2, "RSV_A", "A:0", 0, 0, True)
    assert S.ledger_report(E).reduction_rate == 1.0


def test_csv_roundtrip_and_errors():
    """test_dist.cpp:244-273."""
    L = S.CommLedger()
    L.record(3, 2, "RSV_A", "A:1", 45, 180, False)
    L.record(3, 3, "RSV_G_F_grad", "F:2", 0, 0, True)
    f = io.StringIO()
    L.write_csv(f)
    rows = S.read_ledger_csv(io.StringIO(f.getvalue()))
    assert len(rows) == 2
    assert (rows[0].step, rows[0].stage, rows[0].collective, rows[0].statistic_id, rows[0].elements,
            rows[0].bytes, rows[0].skipped) == (3, 2, "RSV_A", "A:1", 45, 180, False)
    assert rows[1].skipped
    hdr = "step,stage,collective,statistic_id,elements,bytes,skipped\n"
    for bad in ("step,stage\n1,2\n", hdr + "1,2,x\n", hdr + "one,2,RSV_A,A:0,3,12,0\n", ""):
        with pytest.raises(S.ParseError):
            S.read_ledger_csv(io.StringIO(bad))


def test_planner_rejects_bad_arguments():
    from paper_2002_06015_b200 import _native as N
    from paper_2002_06015_b200.step import layer_descs
    arr = layer_descs(small_net())
    assert N.lib().spngd_ledger_step_rows(arr, 3, 0, 1, None, 4, 0, None, 0) < 0
    assert N.lib().spngd_ledger_step_rows(arr, 0, 1, 1, None, 4, 0, None, 0) < 0


@pytest.mark.parametrize("world", [1, 3, 8])
def test_layout_entries_hold_their_payloads(world):
    """Owner-major layout (spngd_plan_layout_ex): every statistic / gradient /
    weight entry fits before the next one of its owner, 64-float aligned, inside
    the padded segment; full BN sizes F as the packed 2c x 2c block."""
    from paper_2002_06015_b200.step import plan_layout
    net = W.resnet18_cifar()
    for bn_full in (False, True):
        ents, seg_st, seg_gr, seg_ag = plan_layout(net, world, bn_full)
        spans = {}
        for li, (l, e) in enumerate(zip(net, ents)):
            assert 0 <= e["owner"] < world
            if l.kind == "bn":
                c = l.g
                stat = [(e["M"], (2 * c) * (2 * c + 1) // 2 if bn_full else 3 * c)]
                g_len = 2 * c
            else:
                stat = [(e["A"], l.a * (l.a + 1) // 2), (e["G"], l.g * (l.g + 1) // 2)]
                g_len = l.g * l.a
            for region, items, seg in (("st", stat, seg_st), ("gr", [(e["dW"], g_len)], seg_gr),
                                       ("ag", [(e["W"], g_len)], seg_ag)):
                for off, n in items:
                    assert off % 64 == 0 and off + n <= seg
                    spans.setdefault((region, e["owner"]), []).append((off, off + n))
        for iv in spans.values():
            iv.sort()
            assert all(a[1] <= b[0] for a, b in zip(iv, iv[1:]))
