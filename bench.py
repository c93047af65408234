#!/usr/bin/env python
"""Benchmark: ResNet-50 SP-NGD optimizer-step ms (factor+invert+precondition) @ N GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config resnet50|resnet18|mlp]

One process per GPU (torchrun for N > 1, rendezvous on 127.0.0.1).  A "step"
is one SP-NGD optimizer step over one synthetic per-rank batch (32 images/GPU,
weak scaling): factors + BN moments, NCCL reduce-scatter to layer owners,
damped Cholesky inverses, preconditioning + momentum/rescale update, BN 2x2
solve, NCCL all-gather.  Rank 0 prints one JSON line.

--gpus N without torchrun re-executes itself under torch.distributed.run with
N ranks.  --impl reference times the reference path's fp64 CPU restatement
(oracle/blas_step.py; the reference itself needs Eigen, which is absent) on
the full configuration on all host cores; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-50 SP-NGD optimizer-step ms (factor+invert+precondition) @1/2/4/8 GPU"
UNIT = "ms"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="resnet50", choices=["resnet50", "resnet18", "mlp"])
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-raw-e2e", action="store_true")
    p.add_argument("--lam", type=float, default=2.5e-4)
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(config):
    from paper_2002_06015_b200 import workloads as W
    fn, batch, desc = W.CONFIGS[config]
    return fn(), batch, desc


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return m["bf16_tflops"], m["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- CPU legs
# The reference (C++/Eigen, single-threaded) cannot be built here (no Eigen,
# SURVEY.md §8c); its path is timed as the fp64 BLAS/LAPACK restatement in
# oracle/blas_step.py (validated against the line-by-line oracle in
# tests/test_blas_step.py) on the full configuration.
def cpu_full_step(layers, batch, threads, warmup, steps, budget_s):
    """Times whole steps of the restated reference path on `threads` BLAS
    threads: `warmup` untimed steps, then up to `steps` timed steps while the
    time budget lasts (at least one).  Returns (median ms, phases, n timed)."""
    from oracle.blas_step import BlasStep, blas_threads
    bs = BlasStep(layers, batch)
    runs = []
    with blas_threads(threads):
        for _ in range(warmup):
            bs.run()
        t0 = time.time()
        for _ in range(max(1, steps)):
            runs.append(bs.run())
            if time.time() - t0 > budget_s:
                break
    runs.sort(key=lambda r: r[0])
    wall, phases, _ = runs[len(runs) // 2]
    return wall, phases, len(runs), bs


def cpu_single_thread(bs, layers, batch):
    """the faithful single-threaded path on a layer sample
    (one layer per distinct shape class plus all three 4608^2 factors); the
    full-step figure adds each remaining layer at its class's measured time."""
    from oracle.blas_step import blas_threads, sample_classes
    sub = sample_classes(layers)
    with blas_threads(1):
        wall, phases, per = bs.run(subset=sub)
    cls = {}
    for i, ms in zip(sub, per):
        l = layers[i]
        cls.setdefault((l.kind, l.a, l.g, l.hw), ms)
    est = sum(per) + sum(cls[(l.kind, l.a, l.g, l.hw)] for i, l in enumerate(layers) if i not in set(sub))
    return {"sample_ms": round(wall, 1), "sample_layers": len(sub), "cores": 1,
            "phases_ms": {k: round(v, 1) for k, v in phases.items()},
            "full_step_ms_est": round(est, 1),
            "sample": f"{len(sub)} of {len(layers)} layers (one per (kind, a, g, hw) class + all 4608^2 factors), "
                      f"batch {batch}; full step = sample + remaining layers at their class's measured time"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.blas_step import cpu_model, host_threads
    layers, batch, desc = workload(args.config)
    threads = host_threads()
    t0 = time.time()
    budget = float(os.environ.get("SPNGD_REF_BUDGET_S", "150"))
    warm = min(args.warmup, 1)
    value, phases, steps, _ = cpu_full_step(layers, batch, threads, warm, args.steps, budget)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": round(value, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "global_batch": batch * args.gpus, "per_gpu_batch": batch,
                   "parallelism": f"host BLAS threads x{threads} (one rank's shard)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"the full {len(layers)}-layer step (no sampling), {steps} timed step(s) after "
                                   f"{warm} warm-up, median",
                         "phases_ms": {k: round(v, 1) for k, v in phases.items()}},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("reference C++/Eigen is not buildable here (no Eigen3); timed its fp64 restatement "
                 "oracle/blas_step.py (Eigen's LLT/solve(I)/GEMM/row-dot calls as LAPACK/BLAS, per-sample "
                 "factor accumulation as in mean_outer), steps capped by a %.0f s budget" % budget),
        "wall_s": round(time.time() - t0, 1),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.path = index, None, f"/tmp/spngd_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import ctypes as C

    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
        pg = dist
    from paper_2002_06015_b200 import _native as N
    from paper_2002_06015_b200 import workloads as W
    from paper_2002_06015_b200.spngd import check
    from paper_2002_06015_b200.step import ALL_WEIGHTS, Comm, Optimizer, ACT, GRAD, DW, BN_GG, BN_GB

    layers, batch, desc = workload(args.config)
    def new_nccl_id():
        if world == 1:
            return None
        obj = [Comm.unique_id() if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        return obj[0]

    nccl_id = new_nccl_id()
    opt = Optimizer(layers, batch, lam=args.lam, device=local, world=world, rank=rank, nccl_id=nccl_id)
    p2p = world > 1 and os.environ.get("SPNGD_NO_P2P") is None
    if p2p:  # Stage 5 as NVLink stores fused into the owners' rescale pass
        opt.attach_peers(pg)
    opt.synth(seed=42)
    L = N.lib()

    def barrier():
        if pg:
            pg.barrier()

    for s in range(args.warmup):
        opt.step(s + 1)
    opt.sync()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ev = (C.c_void_p * 2)()
    ms = C.c_float()
    t_wall = time.time()
    check(L.spngd_event_time(opt.ctx, ev, 0, C.byref(ms)))
    for s in range(args.steps):
        opt.step(args.warmup + s + 1)
    check(L.spngd_event_time(opt.ctx, ev, 1, C.byref(ms)))
    opt.sync()
    wall_s = time.time() - t_wall
    clocks = sampler.stop()
    step_ms = ms.value / args.steps
    phases = opt.phase_ms()  # last step, device events
    launches = opt.launch_count()
    owners = [opt.owner(li) for li in range(len(layers))]
    barrier()
    if pg:
        import torch
        t = torch.tensor([step_ms], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        step_ms = float(t.item())

    # ---- e2e through the public API with host-resident inputs (pinned) ----
    def measure_e2e(o, step0):
        bufs = []  # (device ptr, host ptr, bytes)
        for li, w in o.input_buffers():
            p, _ = o.ptr(li, w)
            nbytes = o.numel(li, w) * 4
            hp = C.c_void_p()
            check(L.spngd_host_alloc(C.byref(hp), nbytes))
            check(L.spngd_copy(o.ctx, hp, C.c_void_p(p), nbytes))
            bufs.append((p, hp, nbytes))
        wp, wcount = o.ptr(0, ALL_WEIGHTS)
        out_bytes = wcount * 4
        hw_out = C.c_void_p()
        check(L.spngd_host_alloc(C.byref(hw_out), out_bytes))
        o.sync()
        h2d = sum(b for _, _, b in bufs)
        times = []
        ins = [(li, w, hp.value) for (li, w), (_, hp, _) in zip(o.input_buffers(), bufs)]
        for s in range(args.e2e_steps):
            barrier()
            ev2 = (C.c_void_p * 2)()
            check(L.spngd_event_time(o.ctx, ev2, 0, C.byref(ms)))
            # spngd_opt_step_host: H2D of this step's inputs (copy stream, wave
            # order) overlapped with the step, D2H of the weights at the end
            o.step_host(step0 + s, ins, hw_out.value)
            check(L.spngd_event_time(o.ctx, ev2, 1, C.byref(ms)))
            times.append(ms.value)
        o.sync()
        v = sorted(times)[len(times) // 2] if times else float("nan")
        if pg:
            t = torch.tensor([v], dtype=torch.float64)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            v = float(t.item())
        for _, hp, _ in bufs:
            L.spngd_host_free(hp)
        L.spngd_host_free(hw_out)
        return v, h2d, out_bytes

    e2e, h2d, out_bytes = measure_e2e(opt, args.warmup + args.steps + 1)
    # Same step fed the raw conv inputs instead of the im2col captures (the
    # device forms the captures, spngd_opt_enable_raw_inputs): fewer H2D bytes.
    e2e_raw = None
    if args.e2e_steps > 0 and any(l.kind == "conv" for l in layers) and not args.no_raw_e2e:
        opt_r = Optimizer(layers, batch, lam=args.lam, device=local, world=world, rank=rank,
                          nccl_id=new_nccl_id())
        opt_r.enable_raw_inputs()
        if p2p:
            opt_r.attach_peers(pg)
        opt_r.synth(seed=42)
        for s in range(args.warmup):
            opt_r.step(s + 1)
        opt_r.sync()
        v, h2d_r, ob_r = measure_e2e(opt_r, args.warmup + 1)
        e2e_raw = {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": h2d_r, "d2h_bytes_per_step": ob_r,
                   "inputs": "raw conv layer inputs (B x c_in x h x w) expanded on the device by im2col "
                             "(spngd_opt_enable_raw_inputs); 1x1 stride-1 inputs are the captures themselves"}

        def device_ms(o, step0, n=5):
            ev4 = (C.c_void_p * 2)()
            check(L.spngd_event_time(o.ctx, ev4, 0, C.byref(ms)))
            for s in range(n):
                o.step(step0 + s)
            check(L.spngd_event_time(o.ctx, ev4, 1, C.byref(ms)))
            return ms.value / n

        e2e_raw["device_ms_explicit_im2col"] = round(device_ms(opt_r, args.warmup + args.e2e_steps + 1), 3)
        opt_r.close()
        # the same step with implicit im2col (no capture; the
        # GEMMs gather from the raw inputs), device time with resident inputs
        opt_i = Optimizer(layers, batch, lam=args.lam, device=local, world=world, rank=rank, nccl_id=new_nccl_id())
        opt_i.enable_raw_inputs(implicit=True)
        if p2p:
            opt_i.attach_peers(pg)
        opt_i.synth(seed=42)
        for s in range(args.warmup):
            opt_i.step(s + 1)
        e2e_raw["device_ms_implicit_im2col"] = round(device_ms(opt_i, args.warmup + 1), 3)
        opt_i.close()

    # ---- phase-serial pass (single GPU): the factor SYRK launch alone, for
    # the roofline (in the overlapped schedule it shares the GPU with the
    # inverse recursion, so its event span is not one kernel's duration).
    serial = None
    if True:
        opt.set_overlap(False)
        t0 = args.warmup + args.steps + args.e2e_steps + 1
        for s in range(3):
            opt.step(t0 + s)
        ev3 = (C.c_void_p * 2)()
        check(L.spngd_event_time(opt.ctx, ev3, 0, C.byref(ms)))
        for s in range(3):
            opt.step(t0 + 3 + s)
        check(L.spngd_event_time(opt.ctx, ev3, 1, C.byref(ms)))
        opt.sync()
        serial = {"ms_per_step": round(ms.value / 3, 4),
                  "phases_ms_last_step": {k: round(v, 3) for k, v in opt.phase_ms().items()}}
        opt.set_overlap(True)

    if rank == 0:
        bf16, hbm, basis = peaks()
        ff, fi, fp = W.flops(layers, batch)
        # Dominant kernel: the grouped 3xTF32 factor GEMM (one launch per step).
        # achieved = algorithmic SYRK-half flops / its CUDA-event duration.  Each
        # fp32-accurate product costs 3 tf32 MMAs; dense tf32 peak = bf16 / 2,
        # so the 3xTF32-effective peak is bf16 / 6 (of measured).
        fac_ms = serial["phases_ms_last_step"]["factor_gemm"] if serial else phases["factor_gemm"]
        t_fac = fac_ms * 1e-3
        achieved = ff / t_fac / 1e12
        peak = bf16 / 6.0
        roofline = {"bound": "tensor", "kernel": "gemm_tf32x3_kernel (factor SYRK, grouped)",
                    "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": "TFLOP/s",
                    "frac": round(achieved / peak, 4), "traffic": load_traffic(),
                    "algorithmic": f"{ff / 1e9:.1f} GF per launch (SURVEY §8d F_fac, SYRK-half)",
                    "peak_basis": f"bf16 {bf16} TF/s {basis} / 2 (tf32) / 3 (3xTF32 products)",
                    "launch_ms": round(fac_ms, 3),
                    "launch_timing": ("CUDA events around the factor SYRK launch in a phase-serial pass of the "
                                      "same optimizer (overlap off)" if serial else
                                      "CUDA events around the factor SYRK launch in the timed steps"),
                    "step_share": round(fac_ms / max(sum((serial or {}).get("phases_ms_last_step", phases).values()),
                                                     1e-9), 3)}
        # The other two tensor-core phases of north_star's target, from the
        # same phase-serial pass (CUDA events on the library stream; each span
        # is the phase's grouped GEMM launches plus its small helpers).
        sp = (serial or {}).get("phases_ms_last_step", phases)
        if world > 1:  # owner-local phases: this rank's (rank 0's) owned layers' flops
            fp = fi = 0.0
            for li, l in enumerate(layers):
                if l.kind != "bn" and owners[li] == 0:
                    fi += l.a ** 3 + l.g ** 3
                    fp += 2 * l.g * l.g * l.a + 2 * l.g * l.a * l.a
        rooflines = {
            "factor_syrk": {k: roofline[k] for k in ("achieved", "peak", "frac", "launch_ms")},
            "precondition": {"achieved": round(fp / (sp["precondition_update"] * 1e-3) / 1e12, 2),
                             "peak": round(peak, 2), "unit": "TFLOP/s",
                             "frac": round(fp / (sp["precondition_update"] * 1e-3) / 1e12 / peak, 4),
                             "span_ms": sp["precondition_update"],
                             "algorithmic": f"{fp / 1e9:.1f} GF (SURVEY §8d F_pre = sum 2g^2a + 2ga^2"
                                            + (", rank 0's owned layers)" if world > 1 else ")"),
                             "span": "four triangular 3xTF32 GEMM launches (T_A, T_A^T, T_G, T_G^T) with the "
                                     "momentum/velocity/norm epilogue + rescale + BN det check + BN solve/update"},
            "inverse": {"achieved": round(fi / (sp["inverse"] * 1e-3) / 1e12, 2), "peak": round(peak, 2),
                        "unit": "TFLOP/s", "frac": round(fi / (sp["inverse"] * 1e-3) / 1e12 / peak, 4),
                        "span_ms": sp["inverse"],
                        "algorithmic": f"{fi / 1e9:.1f} GF (SURVEY §8d F_inv = sum a^3 + g^3"
                                       + (", rank 0's owned layers)" if world > 1 else ")"),
                        "span": "pi + unpack/damping + every recursion round (leaves + grouped 3xTF32 GEMMs) of "
                                "all 108 factors, size classes on concurrent streams"},
        }
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle.blas_step import cpu_model, host_threads
            thr = host_threads()
            v, ph, nsteps, bs = cpu_full_step(layers, batch, thr, 0, 1, 0.0)
            single = cpu_single_thread(bs, layers, batch)
            del bs
            cpu = {"value": round(v, 1), "unit": UNIT, "cores": thr, "kind": "port", "cpu": cpu_model(),
                   "sample": f"the full {len(layers)}-layer step at batch {batch} (no sampling), one timed step, "
                             "fp64 BLAS/LAPACK restatement of the reference path (oracle/blas_step.py)",
                   "phases_ms": {k: round(x, 1) for k, x in ph.items()},
                   "single_thread": single}
        line = {
            "metric": METRIC, "value": round(step_ms, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32 (3xTF32 tensor-core products; fp32 leaf factorization)",
            "data": "synthetic (device-generated captures, SURVEY.md §8d)",
            "config": {"workload": desc, "model": args.config, "global_batch": batch * world,
                       "per_gpu_batch": batch, "seq_len": None, "parallelism": f"hybrid dp/mp x{world}",
                       "lambda": args.lam, "eta": 1.25e-2, "momentum": 0.993, "rescale": True,
                       "l2": f"inputs > L2: {W.capture_bytes(layers, batch) / 1e9:.2f} GB of captures per step"},
            "phases_ms_last_step": overlap_labels(phases, world),
            "schedule": "waves: inverse recursion of the largest factors runs on high-priority streams while the "
                        "remaining factor SYRKs run" + ("; per-wave owner reductions on a comm stream" if world > 1 else "")
                        + ("; Stage 5 as NVLink peer stores fused into the rescale pass" if p2p else ""),
            "phase_serial": serial,
            "e2e_raw_inputs": e2e_raw,
            "e2e": ({"value": round(e2e, 3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": out_bytes}
                    if args.e2e_steps > 0 else None),
            "gpu_launches": launches * args.steps,
            "roofline": roofline,
            "rooflines": rooflines,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "wall_s_timed": round(wall_s, 3),
        }
        print(json.dumps(line), flush=True)
    opt.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def overlap_labels(phases, world):
    """The six event spans of an overlapped (wave) step, named by what runs in
    them: in that schedule the inverse recursion runs beside the factor SYRKs,
    so the phase-serial names (factor_gemm, ..., inverse) do not apply."""
    v = list(phases.values())
    if world > 1:
        names = ["factor_syrk_waves (earlier waves' inverses overlapped)", "last_wave_reduce_and_bn_moments",
                 "comm_join_and_early_precondition (layers of the earlier waves)",
                 "inverse_tail (last wave's recursion)", "precondition_update_late_and_bn", "all_gather"]
    else:  # one GPU: every precondition part runs inside the schedule, per inverse class
        names = ["factor_syrk_waves (earlier waves' inverses overlapped)", "last_wave_reduce_and_bn_moments",
                 "inverse_tail_and_precondition (parts as their inverse classes finish)",
                 "join", "status_restore_and_bn_update", "all_gather (none at P=1)"]
    return {n: round(x, 3) for n, x in zip(names, v)}


def load_traffic():
    """dram bytes per launch of the factor GEMM from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "factor_gemm_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1), same arguments."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        return run_reference(args)
    if world_env is None and args.gpus > 1:
        relaunch(args)
    world = int(world_env or 1)
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU"}),
              flush=True)
        return 2
    if world > 1:  # NCCL's init lines (ranks, transports) stay in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
