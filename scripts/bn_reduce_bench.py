"""fused BN per-sample reduction (net.cpp:467-475) over all
53 ResNet-50 BN layers at B=32 (2.85 GB of dY + x_hat per pass), one batched
launch (spngd_bn_grad_reduce_batched).  Reports achieved HBM GB/s against the
measured copy bandwidth in MEASURED_PEAKS.json.

python scripts/bn_reduce_bench.py [--batch 32] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2002_06015_b200 import spngd as P  # noqa: E402
from paper_2002_06015_b200 import workloads as W  # noqa: E402


def bn_shapes(layers):
    """(c, S) of every BN layer: S = h_out * w_out of the conv it follows."""
    out, prev = [], None
    for l in layers:
        if l.kind == "conv":
            prev = l
        elif l.kind == "bn":
            out.append((l.g, prev.hw))
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--reps", type=int, default=10)
    a = p.parse_args()
    shapes = bn_shapes(W.resnet50())
    M = a.batch
    g = torch.Generator(device="cuda").manual_seed(3)
    items = []
    for c, S in shapes:
        dy = torch.randn(M, c * S, device="cuda", generator=g)
        xh = torch.randn(M, c * S, device="cuda", generator=g)
        items.append((dy, xh, M, c, S))
    nbytes = sum(2 * M * c * S * 4 for c, S in shapes) + sum(2 * M * c * 4 for c, _ in shapes)
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")  # > L2 between reps (inputs exceed L2 anyway)
    P.bn_grad_reduce_batched(items)  # warm-up
    ts = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.bn_grad_reduce_batched(items)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    gbs = nbytes / ms / 1e6
    print(json.dumps({"metric": "BN per-sample reduction (net.cpp:467-475), ResNet-50 53 BN layers",
                      "per_gpu_batch": M, "bytes": nbytes, "ms": round(ms, 4), "achieved_GBps": round(gbs, 1),
                      "peak_GBps": peaks["hbm_gbs"], "frac": round(gbs / peaks["hbm_gbs"], 3),
                      "timing": "CUDA events around the batched C-ABI call (includes its task upload and sync)",
                      "data": "synthetic N(0,1)"}))


if __name__ == "__main__":
    main()
