"""Stale-statistics scheduler (host logic in libspngd_b200.so) against the
reference's own traces (tests/test_stale.cpp:112-242).  Similarity norms are
computed here with numpy exactly as stale.hpp:49-64 does; on the GPU they
come from the K8 kernel (tests/test_gpu_kernels.py)."""
import ctypes as C

import numpy as np
import pytest

from paper_2002_06015_b200 import _native as N

REASONS = ["FirstBuild", "Dissimilar1", "Dissimilar2", "SimilarBoth"]


class Tracker:
    def __init__(self, id, alpha):
        self.h = N.lib().spngd_tracker_create(id.encode(), alpha)
        self.x1 = self.x2 = None

    def __del__(self):
        N.lib().spngd_tracker_destroy(self.h)

    def should_refresh(self, step):
        return bool(N.lib().spngd_tracker_should_refresh(self.h, step))

    def on_refresh(self, x, step):
        x = np.asarray(x, float)
        d = [0.0] * 4
        if self.x1 is not None:
            d[0], d[1] = np.linalg.norm(x - self.x1), np.linalg.norm(self.x1)
        if self.x2 is not None:
            d[2], d[3] = np.linalg.norm(x - self.x2), np.linalg.norm(self.x2)
        iv, rs = C.c_int64(), C.c_int()
        rc = N.lib().spngd_tracker_on_refresh(self.h, step, int(self.x1 is not None), d[0], d[1],
                                              int(self.x2 is not None), d[2], d[3], C.byref(iv), C.byref(rs))
        if rc:
            raise RuntimeError(N.STATUS_NAMES.get(rc))
        self.x2, self.x1 = self.x1, x
        return iv.value, REASONS[rs.value]

    def state(self):
        v = [C.c_int64() for _ in range(4)]
        N.lib().spngd_tracker_state(self.h, *[C.byref(x) for x in v])
        return [x.value for x in v]


def drive(tr, steps, fn):
    trace = []
    for s in range(1, steps + 1):
        if tr.should_refresh(s):
            iv, why = tr.on_refresh(fn(s), s)
            trace.append((s, iv, why))
    return trace


def test_constant_statistics_fibonacci():  # test_stale.cpp:141-166
    tr = Tracker("A:0", 0.1)
    trace = drive(tr, 60, lambda s: [2.0, -1.0, 0.5])
    assert [t[0] for t in trace] == [1, 2, 3, 5, 8, 13, 21, 34, 55]
    assert [t[1] for t in trace] == [1, 1, 2, 3, 5, 8, 13, 21, 34]
    assert trace[0][2] == "FirstBuild" and trace[1][2] == "Dissimilar2"
    assert all(t[2] == "SimilarBoth" for t in trace[2:])
    assert tr.state() == [89, 34, 21, 9]


def test_ever_changing_refresh_every_step():  # test_stale.cpp:168-180
    tr = Tracker("G:1", 0.1)
    trace = drive(tr, 12, lambda s: [5.0 if s % 2 == 0 else -5.0, 1.0])
    assert [t[0] for t in trace] == list(range(1, 13))
    assert all(t[1] == 1 for t in trace)
    assert all(t[2] == "Dissimilar1" for t in trace[1:])


def test_alpha_zero_refreshes_every_step():  # test_stale.cpp:182-190
    tr = Tracker("F:2", 0.0)
    trace = drive(tr, 10, lambda s: [1.0, 1.0])
    assert len(trace) == 10 and all(t[1] == 1 for t in trace)


def test_shift_halves_then_regrows():  # test_stale.cpp:192-220
    tr = Tracker("A:3", 0.1)
    for s in range(1, 9):
        if tr.should_refresh(s):
            tr.on_refresh([5.0, 0.0], s)
    assert tr.state()[1] == 5 and tr.state()[0] == 13
    assert tr.on_refresh([50.0, 10.0], 13) == (2, "Dissimilar1")
    assert tr.on_refresh([50.0, 10.0], 15) == (2, "Dissimilar2")
    assert tr.on_refresh([50.0, 10.0], 17) == (4, "SimilarBoth")
    assert tr.state()[0] == 21


def test_refresh_out_of_turn():  # test_stale.cpp:222-232
    tr = Tracker("A:0", 0.1)
    assert not tr.should_refresh(0) and not tr.should_refresh(2)
    with pytest.raises(RuntimeError, match="RefreshOutOfTurn"):
        tr.on_refresh([1.0], 2)
    tr.on_refresh([1.0], 1)
    with pytest.raises(RuntimeError, match="RefreshOutOfTurn"):
        tr.on_refresh([1.0], 1)
