"""K-invariance of the NCCL path (tests/test_dist.cpp:363-387 analogue).

torchrun --nproc-per-node 2 scripts/multi_gpu_check.py [--mode default|wgrad|bn_full|one_mc|sgd|host|p2p...]
                                                        [--layers toy|r50]
Every rank runs one step at P = 2 on its own shard; rank 0 then replays the
same step at P = 1 over the concatenated batch (mean dW) and compares all
updated weights.  Replicas must be bit-identical across ranks, and the step's
CommLedger rows must equal the oracle restatement at P (oracle/ledger.py).
Modes: the optimizer configurations of DESIGN.md §3.6 (wgrad forms dW on each
rank from its shard; host feeds the rank's inputs through spngd_opt_step_host).
--layers r50: a ResNet-50 layer sample with the dominant factors (a 4608^2
A with K < a, a 2304^2 A, a 2048^2 G, conv1, BN, the FC) at 32 images in
total; rank 0 then also checks every Kronecker layer's updated weights
against the fp64 oracle (or_kfac_layers) on the concatenated batch.
Exit 0 on pass.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import ACT, BN_GB, BN_GG, DW, GRAD, V, Comm, Optimizer  # noqa: E402
from paper_2002_06015_b200.step import BN_GB_SAMPLED, BN_GG_SAMPLED, GRAD_SAMPLED  # noqa: E402
from oracle import ledger as OL  # noqa: E402
from paper_2002_06015_b200.step import W as WB  # noqa: E402

LAYERS = [W.conv(16, 32, 3, 1, 16), W.bn(32), W.conv(32, 64, 3, 2, 16), W.bn(64), W.conv(64, 128, 3, 1, 8),
          W.bn(128), W.conv(128, 256, 3, 2, 8), W.bn(256), W.fc(1024, 10),
          W.conv(256, 256, 3, 1, 4), W.conv(512, 512, 3, 1, 4)]  # inverse waves 1 and 0
B = 8
R50_LAYERS = [W.conv(3, 64, 7, 2, 224), W.bn(64), W.conv(256, 256, 3, 1, 14), W.bn(256),
              W.conv(512, 512, 3, 1, 7), W.bn(512), W.conv(512, 2048, 1, 1, 7), W.fc(2048, 1000)]


MODES = {"default": {}, "wgrad": {"wgrad": True}, "bn_full": {"bn_mode": 1}, "one_mc": {"fisher_mode": 1},
         "sgd": {"sgd": True}, "host": {}, "p2p": {}, "p2p_sgd": {"sgd": True},
         "p2p_bn_full": {"bn_mode": 1}, "p2p_wgrad": {"wgrad": True}, "p2p_host": {}}


def main():
    mode = sys.argv[sys.argv.index("--mode") + 1] if "--mode" in sys.argv else "default"
    kw = MODES[mode]
    global B, LAYERS
    r50 = "--layers" in sys.argv and sys.argv[sys.argv.index("--layers") + 1] == "r50"
    if mode.endswith("bn_full"):
        B = 320  # 2c <= 512 < P*B: full-rank F, so fp32 summation order stays below the 1e-4 gate
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if r50:
        LAYERS, B = R50_LAYERS, 32 // world
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    opt = Optimizer(LAYERS, B, device=local, world=world, rank=rank, nccl_id=obj[0], **kw)
    if mode.startswith("p2p"):
        opt.attach_peers(dist)
    opt.synth(seed=11)
    inputs = {}

    def in_whichs(l):
        ws = [BN_GG, BN_GB, DW] if l.kind == "bn" else [ACT, GRAD, DW]
        if kw.get("fisher_mode") == 1:
            ws += [BN_GG_SAMPLED, BN_GB_SAMPLED] if l.kind == "bn" else [GRAD_SAMPLED]
        return ws

    for li, l in enumerate(LAYERS):
        inputs[li] = {w: opt.download(li, w).numpy() for w in in_whichs(l)}
        inputs[li][WB] = opt.download(li, WB).numpy()
        if opt.owner(li) == rank:
            inputs[li][V] = opt.download(li, V).numpy()
    if mode.endswith("host"):
        keep = [opt.download(li, w).pin_memory() for li, w in opt.input_buffers()]
        for li, w in opt.input_buffers():
            opt.upload(li, w, torch.full((opt.numel(li, w),), 3.0))
        opt.step_host(1, [(li, w, t.data_ptr()) for (li, w), t in zip(opt.input_buffers(), keep)])
    else:
        opt.step(1)
    opt.sync()
    rows = [(r.step, r.stage, r.collective, r.statistic_id, r.elements, r.bytes, r.skipped)
            for r in opt.ledger().rows()]
    want_rows = OL.step_rows(LAYERS, world, 1, None, 4, bn_full=kw.get("bn_mode") == 1, sgd=kw.get("sgd", False))
    ledger_ok = rows == want_rows and all(r[4] > 0 for r in rows)
    wire = opt.wire_bytes()
    after = [opt.download(li, WB).numpy() for li in range(len(LAYERS))]
    owners = [opt.owner(li) for li in range(len(LAYERS))]
    gathered = [None] * world
    dist.all_gather_object(gathered, (inputs, after))
    ok = True
    if rank == 0:
        for r in range(1, world):
            for li in range(len(LAYERS)):
                if not np.array_equal(gathered[r][1][li], after[li]):
                    print(f"replica mismatch rank {r} layer {li}")
                    ok = False
        ref = Optimizer(LAYERS, B * world, device=local, **kw)
        for li, l in enumerate(LAYERS):
            ws = [w for w in in_whichs(l) if w != DW]
            for w in ws:
                ref.upload(li, w, torch.from_numpy(np.concatenate([gathered[r][0][li][w] for r in range(world)])))
            ref.upload(li, DW, torch.from_numpy(np.mean([gathered[r][0][li][DW] for r in range(world)], axis=0)))
            ref.upload(li, WB, torch.from_numpy(inputs[li][WB]))
            vown = gathered[owners[li]][0][li][V]
            ref.upload(li, V, torch.from_numpy(vown))
        ref.step(1)
        ref.sync()
        worst = 0.0
        for li in range(len(LAYERS)):
            want = ref.download(li, WB).numpy().astype(np.float64)
            err = np.linalg.norm(after[li] - want) / np.linalg.norm(want)
            worst = max(worst, err)
            print(f"layer {li} {LAYERS[li].kind} owner {owners[li]} rel {err:.2e}")
        ok = ok and worst <= 1e-4
        if r50 and not kw.get("sgd"):  # the fp64 oracle on the concatenated batch (Stage 2-5, dist.cpp:406-675)
            import ctypes as C
            import oracle as O
            recs, outs, keep = [], [], []
            for li, l in enumerate(LAYERS):
                if l.kind == "bn":
                    continue
                cat = lambda w: np.ascontiguousarray(np.concatenate([gathered[r][0][li][w] for r in range(world)]),
                                                     dtype=np.float32)
                bufs = [cat(ACT), cat(GRAD),
                        np.mean([gathered[r][0][li][DW] for r in range(world)], axis=0).astype(np.float32),
                        inputs[li][WB].astype(np.float32), gathered[owners[li]][0][li][V].astype(np.float32)]
                rec = O.OrLayer()
                out = np.empty(l.g * l.a)
                rec.is_conv, rec.a, rec.g, rec.hw, rec.batch = int(l.kind == "conv"), l.a, l.g, l.hw, B * world
                rec.act, rec.grad, rec.dW, rec.W, rec.V = [b.ctypes.data_as(C.POINTER(C.c_float)) for b in bufs]
                rec.W_out = out.ctypes.data_as(C.POINTER(C.c_double))
                recs.append(rec)
                outs.append((li, out))
                keep.append(bufs)
            O.kfac_layers(recs, 2.5e-4, 1.25e-2, 0.993, rescale=True, fast_inverse=True,
                          threads=min(len(recs), os.cpu_count() or 1))
            for li, want in outs:
                err = np.linalg.norm(after[li] - want) / np.linalg.norm(want)
                print(f"oracle layer {li} ({LAYERS[li].a}x{LAYERS[li].g}) rel {err:.2e}")
                ok = ok and err <= 1e-4
        print("ledger rows match the oracle at P =", world, ledger_ok, "| NCCL bytes", wire)
        ok = ok and ledger_ok
        ph = opt.phase_ms()
        print("phases", {k: round(v, 3) for k, v in ph.items()})
        print("PASS" if ok else "FAIL", f"mode {mode} worst {worst:.2e}")
        ref.close()
    opt.close()
    t = torch.tensor([1 if ok else 0])
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(0 if t.item() else 1)


if __name__ == "__main__":
    main()
