"""BASELINE config 5: damped-inverse sweep (spd_inverse, linalg.cpp:29-48),
n in {64, 128, 256, 512, 1024, 2048, 4096, 4608}, batched per call.

python scripts/inverse_sweep.py [--batch 4] [--reps 3]

Inputs: (i) well-conditioned random SPD, (ii) A-type
factors X X^T / K from ReLU activations with K < n and K > n.  Damping
sqrt(lambda) = sqrt(2.5e-4): the A-side damping of damp_and_invert with pi = 1.  Timing is the
batched C-ABI call (spngd_spd_inverse_batched: unpack + damping, recursive
Cholesky inverse, pack), median of `reps`, device-synchronised wall time.
Accuracy: rel. Frobenius vs a torch fp64 inverse of the same fp32 input on one
matrix per size (north_star gate 1e-4).  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_06015_b200 import spngd as P  # noqa: E402

SIZES = [64, 128, 256, 512, 1024, 2048, 4096, 4608]
DAMP = 2.5e-4 ** 0.5   # damp_and_invert damping pi*sqrt(lambda) with pi = 1 (fisher.cpp:218-228)


def make(n, kind, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if kind == "random_spd":
        x = torch.randn(n, n, device="cuda", generator=g) / n ** 0.5
        m = x @ x.T + 0.5 * torch.eye(n, device="cuda")
    else:
        k = n // 2 if kind == "relu_K<n" else 2 * n
        x = torch.relu(torch.randn(n, k, device="cuda", generator=g))
        m = x @ x.T / k
    return m


def packed(m):
    n = m.shape[0]
    iu = torch.triu_indices(n, n, device=m.device)
    return m[iu[0], iu[1]].contiguous().float()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=4)
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    rows = []
    for kind in ("random_spd", "relu_K<n", "relu_K>n"):
        for n in SIZES:
            mats = [make(n, kind, 1000 * n + i) for i in range(a.batch)]
            syms = [P.SymMatrix(n, packed(m)) for m in mats]
            failures = 0
            ts = []
            outs = None
            for rep in range(a.reps + 1):  # first call: warm-up (plans, scratch pool, tensor maps)
                if rep:
                    torch.cuda.synchronize()
                t0 = time.perf_counter()
                try:
                    o = P.spd_inverse_batched(syms, DAMP)  # one spngd_spd_inverse_batched call
                except P.NotPositiveDefinite:
                    failures += 1
                    continue
                torch.cuda.synchronize()
                if rep:
                    ts.append(time.perf_counter() - t0)
                outs = o
            if outs is None:
                rows.append(dict(kind=kind, n=n, batch=a.batch, failures=failures))
                print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
                continue
            ms = sorted(ts)[len(ts) // 2] * 1e3
            m0 = mats[0].double().cpu() + DAMP * torch.eye(n, dtype=torch.float64)
            want = torch.linalg.inv(m0)
            iu = torch.triu_indices(n, n)
            got = torch.zeros(n, n, dtype=torch.float64)
            got[iu[0], iu[1]] = outs[0].data.double().cpu()
            got = got + got.T - torch.diag(torch.diag(got))
            err = float(torch.linalg.norm(got - want) / torch.linalg.norm(want))
            cond = float(torch.linalg.cond(m0))
            flops = a.batch * float(n) ** 3
            rows.append(dict(kind=kind, n=n, batch=a.batch, ms=round(ms, 3), gflops=round(flops / ms / 1e6, 1),
                             rel_err=float(f"{err:.3e}"), cond=float(f"{cond:.3e}"), failures=failures))
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"metric": "damped SPD inverse sweep (config 5)", "damping": DAMP, "n_gpus": 1,
                      "flops_basis": "n^3 per inverse (potrf + trtri + lauum)", "rows": rows}))


if __name__ == "__main__":
    main()
