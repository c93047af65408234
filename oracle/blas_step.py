"""Timed CPU baseline of the SP-NGD optimizer step (TEST/BASELINE
INFRASTRUCTURE: only bench.py's cpu_baseline leg, its --impl reference arm
and tests/ use this module; the product never imports oracle/).

The reference (proj/, C++20 + Eigen3, single-threaded, proj/CMakeLists.txt:26)
cannot be built here: Eigen3 is absent.  This module restates
the reference's per-layer Stage-4 path in fp64 with the same algorithm at
the level of its Eigen calls, each mapped to the LAPACK/BLAS routine Eigen
itself would use (scipy-openblas, the closest stand-in for Eigen's blocked
kernels):

  factor_A / factor_G  fisher.cpp:55-145   mean_outer: per sample s, add the
                                           s-th block's Gram matrix into the
                                           accumulator (dsyrk, beta = 1) --
                                           the reference adds per-sample row
                                           dots in sample order -- then / denom
  avg_eigenvalue, pi   linalg.cpp:64-69, fisher.cpp:221-226
  spd_inverse          linalg.cpp:29-48    unpack, + d I, finite check,
                                           Eigen::LLT (dpotrf), solve(I)
                                           (dpotrs on the identity: the same
                                           7n^3/3 flops), finite check,
                                           (X + X^T)/2
  precondition         linalg.cpp:58-62    G * X * A, left to right (dgemm)
  ngd_step + rescale   fisher.cpp:332-333, schemes.cpp:116-119, dist.cpp:621-633
  unit BN              fisher.cpp:147-185, 259-276, 346-357

Layers run one after another (the reference's loop, dist.cpp:539-633); BLAS
threads = all host cores for the headline CPU number, 1 for the faithful
single-threaded variant.  Synthetic inputs: one pool
of fp64 N(0,1) draws viewed per layer (the step's cost does not depend on the
values; every factor is a Gram matrix + damping, so every inverse succeeds).
"""
from __future__ import annotations

import os
import time

import numpy as np
import scipy.linalg.blas as blas
import scipy.linalg.lapack as lapack

POOL = 64 << 20  # doubles (512 MB): larger than any single layer's capture at B = 32


def _pool(seed=0):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal(POOL)
    return p


class LayerData:
    """Views of the per-layer synthetic inputs in the reference layouts
    (net.hpp:84-101): conv act (M*a) x hw stacked, grad (M*g) x hw; FC act
    M x a, grad M x g; dW, W, V g x a; BN per-sample (g_gamma, g_beta) M x c."""

    def __init__(self, l, batch, pool, off):
        self.l, self.batch = l, batch
        n = POOL

        def take(count):
            nonlocal off
            if count > n:  # larger than the pool (ResNet-18 CIFAR at batch 128): repeat it
                return np.resize(pool, count)
            if off + count > n:
                off = 0
            v = pool[off:off + count]
            off += count
            return v

        B = batch
        if l.kind == "bn":
            c = l.g
            self.gg = take(B * c).reshape(B, c)
            self.gb = take(B * c).reshape(B, c)
            self.dW = take(2 * c) * 0.1
            self.W = np.concatenate([np.ones(c), np.zeros(c)])
            self.V = take(2 * c) * 0.01
        else:
            a, g, hw = l.a, l.g, l.hw
            self.act = np.maximum(take(B * a * hw), 0.0).reshape(B, a, hw)
            self.grad = take(B * g * hw).reshape(B, g, hw) / np.sqrt(B * hw)
            self.dW = take(g * a).reshape(g, a) / np.sqrt(a)
            self.W = take(g * a).reshape(g, a) * np.sqrt(2.0 / a)
            self.V = take(g * a).reshape(g, a) * 0.01
        self.end = off


def mean_outer_conv(x, denom):
    """fisher.cpp:55-75 with r > 1: sum over samples of block_s block_s^T."""
    n = x.shape[1]
    acc = np.zeros((n, n), order="F")
    for s in range(x.shape[0]):
        acc = blas.dsyrk(1.0, x[s].T, beta=1.0, c=acc, trans=1, lower=0, overwrite_c=1)
    return acc / denom


def mean_outer_rows(x, denom):
    """fisher.cpp:55-75 with r == 1 (FC): rows are the vectors."""
    n = x.shape[1]
    acc = blas.dsyrk(1.0, np.asfortranarray(x), trans=1, lower=0)
    return acc / denom


def spd_inverse(upper, d):
    """linalg.cpp:29-48 on the upper-filled dense factor."""
    n = upper.shape[0]
    m = np.triu(upper)
    m = m + np.triu(m, 1).T
    m[np.diag_indices(n)] += d
    if not np.isfinite(m).all():
        raise FloatingPointError("spd_inverse: non-finite entries in input")
    c, info = lapack.dpotrf(m, lower=1, clean=0, overwrite_a=1)
    if info != 0:
        raise FloatingPointError("spd_inverse: Cholesky factorization failed")
    x, info = lapack.dpotrs(c, np.eye(n), lower=1, overwrite_b=1)
    if info != 0 or not np.isfinite(x).all():
        raise FloatingPointError("spd_inverse: inverse has non-finite entries")
    return 0.5 * (x + x.T)


def kfac_layer(d: LayerData, lam, eta, mom, t):
    l, B = d.l, d.batch
    t0 = time.perf_counter()
    if l.kind == "conv":
        A = mean_outer_conv(d.act, B * l.hw)
        G = mean_outer_conv(d.grad, B)
    else:
        A = mean_outer_rows(d.act.reshape(B, -1), B)
        G = mean_outer_rows(d.grad.reshape(B, -1), B)
    t1 = time.perf_counter()
    ea, eg = np.trace(A) / l.a, np.trace(G) / l.g
    pi = 1.0 if (ea < 1e-12 or eg < 1e-12) else np.sqrt(ea / eg)
    Ai = spd_inverse(A, pi * np.sqrt(lam))
    Gi = spd_inverse(G, np.sqrt(lam) / pi)
    t2 = time.perf_counter()
    P = (Gi @ d.dW) @ Ai
    t3 = time.perf_counter()
    nw = d.W - eta * P + mom * d.V
    s = np.sqrt(2.0 * l.g) / (np.linalg.norm(nw) + 1e-9)
    rw = s * nw
    rv = rw - d.W
    t4 = time.perf_counter()
    t[0] += t1 - t0
    t[1] += t2 - t1
    t[2] += t3 - t2 + t4 - t3
    return rw, rv


def bn_layer(d: LayerData, lam, eta, mom, t):
    t0 = time.perf_counter()
    B, c = d.batch, d.l.g
    fgg = (d.gg * d.gg).sum(0) / B
    fgb = (d.gg * d.gb).sum(0) / B
    fbb = (d.gb * d.gb).sum(0) / B
    t1 = time.perf_counter()
    a, b, dd = fgg + lam, fgb, fbb + lam
    det = a * dd - b * b
    if (np.abs(det) < 1e-30).any():
        raise FloatingPointError("inv2x2: determinant below 1e-30")
    gg, gb = d.dW[:c], d.dW[c:]
    pg = (dd * gg - b * gb) / det
    pb = (-b * gg + a * gb) / det
    nw = d.W - eta * np.concatenate([pg, pb]) + mom * d.V
    t2 = time.perf_counter()
    t[0] += t1 - t0
    t[2] += t2 - t1
    return nw, nw - d.W


class BlasStep:
    """One SP-NGD step over `layers` at `batch` on this host."""

    def __init__(self, layers, batch, seed=0):
        self.layers, self.batch = layers, batch
        pool = _pool(seed)
        off = 0
        self.data = []
        for l in layers:
            ld = LayerData(l, batch, pool, off)
            off = ld.end
            self.data.append(ld)

    def run(self, lam=2.5e-4, eta=1.25e-2, mom=0.993, subset=None):
        """Returns (wall ms, per-phase ms, per-layer ms) of one step (or of the
        layer subset)."""
        t = [0.0, 0.0, 0.0]
        idx = range(len(self.layers)) if subset is None else subset
        per = []
        t0 = time.perf_counter()
        for i in idx:
            d = self.data[i]
            ti = time.perf_counter()
            (bn_layer if d.l.kind == "bn" else kfac_layer)(d, lam, eta, mom, t)
            per.append((time.perf_counter() - ti) * 1e3)
        wall = (time.perf_counter() - t0) * 1e3
        return wall, {"factor": t[0] * 1e3, "inverse": t[1] * 1e3, "precondition_update": t[2] * 1e3}, per


def sample_classes(layers, include_all=(4608,)):
    """One layer per distinct (kind, a, g, hw) class, plus every layer whose
    a or g is in include_all (all three 4608^2 factors)."""
    seen, out = set(), []
    for i, l in enumerate(layers):
        key = (l.kind, l.a, l.g, l.hw)
        if key not in seen or l.a in include_all or l.g in include_all:
            seen.add(key)
            out.append(i)
    return out


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


def blas_threads(n):
    """Context manager limiting the BLAS pools (numpy's and scipy's OpenBLAS)."""
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=n, user_api="blas")
