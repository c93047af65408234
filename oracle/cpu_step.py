"""Timed CPU baseline of the SP-NGD step: the fp64 oracle restatement of the
reference path (TEST/BASELINE INFRASTRUCTURE, see oracle/__init__.py).

The reference (single-threaded C++/Eigen, proj/CMakeLists.txt:26) cannot be
built here (no Eigen), so the baseline is the restated path `or_kfac_layers`:
factor_A/factor_G (mean_outer, fisher.cpp:55-145) -> damp_and_invert
(Cholesky inverse, linalg.cpp:29-48) -> precondition (linalg.cpp:58-62) ->
update + rescale (fisher.cpp:332-333, schemes.cpp:116-119), layer-parallel
over host threads as SPEC.md:285-286 allows.

A full ResNet-50 step is minutes of fp64 CPU work, so each timed step runs a
bounded SAMPLE of the workload's layers at a reduced batch and extrapolates
each phase by its algorithmic flops (SURVEY.md §8d formulas).
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import OrLayer, kfac_layers

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


def _layer_flops(l, batch):
    K = batch * l.hw
    a, g = l.a, l.g
    return ((a * (a + 1) + g * (g + 1)) * K, a ** 3 + g ** 3, 2 * g * g * a + 2 * g * a * a)


def choose_sample(layers, max_dim=1152):
    """Distinct (a, g, hw) Kronecker shape classes with a, g <= max_dim."""
    seen, out = set(), []
    for l in layers:
        if l.kind == "bn":
            continue
        key = (l.a, l.g, l.hw)
        if key in seen or max(l.a, l.g) > max_dim:
            continue
        seen.add(key)
        out.append(l)
    return out


class CpuStep:
    def __init__(self, layers, batch, sample_batch=2, threads=1, max_dim=1152, seed=0):
        self.layers, self.batch = layers, batch
        self.sample = choose_sample(layers, max_dim)
        self.sample_batch = min(sample_batch, batch)
        self.threads = threads
        rng = np.random.default_rng(seed)
        self.bufs = []
        self.recs = []
        for l in self.sample:
            sb = self.sample_batch
            act = np.maximum(rng.standard_normal(sb * l.a * l.hw, dtype=np.float32), 0)
            grad = (rng.standard_normal(sb * l.g * l.hw, dtype=np.float32) / np.sqrt(sb * l.hw)).astype(np.float32)
            dW = (rng.standard_normal(l.g * l.a, dtype=np.float32) / np.sqrt(l.a)).astype(np.float32)
            W = (rng.standard_normal(l.g * l.a, dtype=np.float32) * np.sqrt(2 / l.a)).astype(np.float32)
            V = (0.01 * rng.standard_normal(l.g * l.a, dtype=np.float32)).astype(np.float32)
            Wo = np.empty(l.g * l.a)
            self.bufs.append((act, grad, dW, W, V, Wo))
        full = np.array([_layer_flops(l, batch) for l in layers if l.kind != "bn"]).sum(0)
        samp = np.array([_layer_flops(l, self.sample_batch) for l in self.sample]).sum(0)
        self.scale = full / samp

    def _records(self):
        recs = []
        for l, (act, grad, dW, W, V, Wo) in zip(self.sample, self.bufs):
            r = OrLayer()
            r.is_conv = int(l.kind == "conv")
            r.a, r.g, r.hw, r.batch = l.a, l.g, l.hw, self.sample_batch
            r.act = act.ctypes.data_as(_fp)
            r.grad = grad.ctypes.data_as(_fp)
            r.dW = dW.ctypes.data_as(_fp)
            r.W = W.ctypes.data_as(_fp)
            r.V = V.ctypes.data_as(_fp)
            r.W_out = Wo.ctypes.data_as(_dp)
            recs.append(r)
        return recs

    def run(self, lam=2.5e-4, eta=1.25e-2, momentum=0.993):
        """One timed sample; returns (estimated full-step ms, per-phase ms dict)."""
        recs = self._records()
        t0 = time.perf_counter()
        kfac_layers(recs, lam, eta, momentum, rescale=True, fast_inverse=True, threads=self.threads)
        wall = time.perf_counter() - t0
        per = np.array([[r.seconds[0], r.seconds[1], r.seconds[2] + r.seconds[3]] for r in recs]).sum(0)
        # Layer-parallel wall time split across phases in proportion to the
        # single-layer phase seconds, then each phase scaled by its flop ratio.
        frac = per / max(per.sum(), 1e-12)
        est = float((wall * frac * self.scale).sum() * 1e3)
        phases = dict(zip(["factor", "inverse", "precondition_update"], (wall * frac * self.scale * 1e3).tolist()))
        return est, phases, wall

    def describe(self):
        return (f"{len(self.sample)} distinct layer shapes with a,g <= 1152 "
                f"({', '.join(f'{l.a}x{l.g}@{l.hw}' for l in self.sample)}), batch {self.sample_batch}, "
                f"{self.threads} thread(s), extrapolated per phase by algorithmic flops to the full "
                f"{sum(1 for l in self.layers if l.kind != 'bn')}-layer step at batch {self.batch}")


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"
