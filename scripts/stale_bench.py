"""BASELINE config 4: stale-gated ResNet-50 SP-NGD steps (StaleTracker,
stale.hpp:78-132; gating dist.cpp:431-444, 514-537, 588-601).

python scripts/stale_bench.py [--batch 32] [--steps 13] [--gpus N under torchrun]

Synthetic captures are held fixed, so every statistic follows the Fibonacci
refresh pattern (steps 1, 2, 3, 5, 8, 13, ...).  --drift EPS makes the capture
stream drift slowly instead: after every step each layer's captures are scaled
in place on the device by (1 + EPS * N(0, 1)) (one draw per layer and buffer),
so statistics change by ~2 EPS per step and the trackers' intervals adapt.  Prints one JSON line with the
refresh-step and non-refresh-step device milliseconds (max over ranks; the sum
of the six phase event intervals) and their amortised mean over the run.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import Comm, Optimizer  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--steps", type=int, default=13)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--drift", type=float, default=0.0)
    a = p.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    layers = W.resnet50()
    opt = Optimizer(layers, a.batch, device=local, world=world, rank=rank, nccl_id=nccl_id, stale=True)
    opt.synth(42)
    from paper_2002_06015_b200.step import ACT, BN_GB, BN_GG, GRAD

    class _Dev:  # zero-copy torch view of a library device buffer
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}

    drift_bufs = []
    if a.drift > 0:
        for li, l in enumerate(layers):
            for w in ((BN_GG, BN_GB) if l.kind == "bn" else (ACT, GRAD)):
                p_, _ = opt.ptr(li, w)
                drift_bufs.append(torch.as_tensor(_Dev(p_, opt.numel(li, w)), device=f"cuda:{local}"))
    gen = torch.Generator().manual_seed(1234 + rank)
    rows = []
    for step in range(1, a.steps + 1):
        opt.step(step, 1.25e-2, 0.993)
        ph = opt.phase_ms()
        total = sum(ph.values())
        stats = [(li, w) for li, l in enumerate(layers) for w in (("F",) if l.kind == "bn" else ("A", "G"))]
        n_ref = sum(opt.stale_info(li, w)["refreshed"] for li, w in stats)
        refreshed = n_ref > 0
        t = torch.tensor([total], dtype=torch.float64)
        if pg:
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
        rows.append((step, refreshed, float(t.item()), {k: round(v, 3) for k, v in ph.items()}, n_ref))
        if drift_bufs:  # outside the step's events: the next step's inputs
            opt.sync()
            for b in drift_bufs:
                b.mul_(1.0 + a.drift * float(torch.randn(1, generator=gen)))
            torch.cuda.synchronize()
    # CommLedger of the run (dist.cpp:42-133): the reference's Fig. 6 reduction
    # rate of statistic traffic (stale-gated bytes / every-step counterfactual)
    from paper_2002_06015_b200.spngd import ledger_report
    rep = ledger_report(opt.ledger())
    ledger = {"steps": rep.steps, "stat_bytes": rep.stat_bytes, "stat_bytes_every_step": rep.stat_bytes_every_step,
              "reduction_rate": round(rep.reduction_rate, 4), "grad_bytes": rep.grad_bytes,
              "param_bytes": rep.param_bytes, "total_bytes": rep.total_bytes,
              "note": "reference ledger semantics: elements are 0 at one worker (dist.cpp:214)"}
    opt.close()
    if rank == 0:
        ref = [r[2] for r in rows[1:] if r[1]]       # step 1 includes graph capture
        non = [r[2] for r in rows if not r[1]]
        out = {
            "metric": "ResNet-50 SP-NGD stale-gated step ms (config 4)",
            "n_gpus": world, "per_gpu_batch": a.batch, "alpha": 0.1,
            "refresh_steps": [r[0] for r in rows if r[1]],
            "refresh_step_ms": round(sorted(ref)[len(ref) // 2], 3) if ref else None,
            "non_refresh_step_ms": round(sorted(non)[len(non) // 2], 3) if non else None,
            "amortized_ms": round(sum(r[2] for r in rows[1:]) / max(1, len(rows) - 1), 3),
            "per_step": [dict(step=r[0], refreshed=r[1], stats_refreshed=r[4], ms=round(r[2], 3), phases=r[3])
                         for r in rows],
            "data": ("synthetic, captures drifting by (1 + %g N(0,1)) per layer and step" % a.drift) if a.drift > 0
                    else "synthetic, captures held fixed (Fibonacci refresh pattern)",
            "stats": len(stats),
            "ledger": ledger,
        }
        print(json.dumps(out), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
