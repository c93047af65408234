"""CommLedger restatement — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pure-Python restatement of the rows `accumulate_microsteps` records per step
(/root/reference/proj/src/dist.cpp), used by tests/test_ledger.py as the
checker for the native host planner `spngd_ledger_step_rows`:

* plan_statistics (dist.cpp:256-269): per layer "A:l","G:l" or "F:l".
* stat payload lengths (dist.cpp:271-295): A/G packed n(n+1)/2, unit BN 3c,
  full BN packed 2c(2c+1)/2; grad_payload (dist.cpp:315-391) g*a or 2c.
* reduce_scatter_v (dist.cpp:181-220) records one row per payload with
  elements = size if K > 1 else 0, bytes = elements * elem_size; all_gather_v
  (dist.cpp:222-237) likewise.
* stage 2 RSV_A over due A, then skipped A rows (dist.cpp:511-520); stage 3
  RSV_G_F_grad over due G/F then grad:0..L-1, then skipped G/F rows
  (dist.cpp:522-537); stage 5 AGV_params w:0..L-1 (dist.cpp:646-662).
"""
from __future__ import annotations


def plan_statistics(layers, spngd=True):  # dist.cpp:256-269
    plans = []
    if not spngd:
        return plans
    for li, l in enumerate(layers):
        if l.kind == "bn":
            plans.append((f"F:{li}", li, "F"))
        else:
            plans.append((f"A:{li}", li, "A"))
            plans.append((f"G:{li}", li, "G"))
    return plans


def _stat_len(l, kind, bn_full):  # dist.cpp:271-295
    if kind == "A":
        return l.a * (l.a + 1) // 2
    if kind == "G":
        return l.g * (l.g + 1) // 2
    c = l.g
    return (2 * c) * (2 * c + 1) // 2 if bn_full else 3 * c


def _grad_len(l):  # dist.cpp:315-391
    return 2 * l.g if l.kind == "bn" else l.g * l.a


def step_rows(layers, K, step, due=None, elem_size=4, bn_full=False, sgd=False):
    """[(step, stage, collective, id, elements, bytes, skipped)] of one step."""
    plans = plan_statistics(layers, not sgd)
    due_map = {p[0]: (True if due is None else bool(due[i])) for i, p in enumerate(plans)}
    rows = []

    def reduce_scatter_v(payloads, stage, coll):  # dist.cpp:181-220 ledger part
        for pid, size in payloads:
            elems = size if K > 1 else 0
            rows.append((step, stage, coll, pid, elems, elems * elem_size, False))

    # Stage 2
    rsv_a = [(pid, _stat_len(layers[li], kind, bn_full)) for pid, li, kind in plans
             if kind == "A" and due_map[pid]]
    reduce_scatter_v(rsv_a, 2, "RSV_A")
    for pid, li, kind in plans:
        if kind == "A" and not due_map[pid]:
            rows.append((step, 2, "RSV_A", pid, 0, 0, True))
    # Stage 3
    rsv_g = [(pid, _stat_len(layers[li], kind, bn_full)) for pid, li, kind in plans
             if kind != "A" and due_map[pid]]
    rsv_g += [(f"grad:{li}", _grad_len(l)) for li, l in enumerate(layers)]
    reduce_scatter_v(rsv_g, 3, "RSV_G_F_grad")
    for pid, li, kind in plans:
        if kind != "A" and not due_map[pid]:
            rows.append((step, 3, "RSV_G_F_grad", pid, 0, 0, True))
    # Stage 5 (all_gather_v, dist.cpp:222-237)
    for li, l in enumerate(layers):
        elems = _grad_len(l) if K > 1 else 0
        rows.append((step, 5, "AGV_params", f"w:{li}", elems, elems * elem_size, False))
    return rows
