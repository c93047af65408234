"""The N > 1 schedule on CPU: world_size 2 over gloo.

Mirrors the reference's ClusterSim tests (tests/test_dist.cpp:94-129 mean
order, :363-387 K-invariance; acceptance.cpp:237-292 replicas identical):
each rank builds its shard statistics with the fp64 oracle, packs them into
the owner-major reduce-scatter buffer laid out by the library's own
`spngd_plan_layout`, reduces (mean), owners run Stage 4 and write their
weights into the all-gather buffer, and every rank must end with the same
weights as the single-process full-batch step.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2002_06015_b200 import workloads as W
from paper_2002_06015_b200.step import plan_layout

LAYERS = [W.conv(3, 8, 3, 1, 6), W.bn(8), W.conv(8, 16, 3, 2, 6), W.bn(16), W.fc(16 * 9, 5)]
M_PER_RANK, WORLD = 4, 2
LAM, ETA, MOM = 2.5e-4, 1.25e-2, 0.993


def shard_inputs(rank):
    rng = np.random.default_rng(100 + rank)
    out = []
    for l in LAYERS:
        if l.kind == "bn":
            gg = rng.standard_normal((M_PER_RANK, l.g))
            out.append(dict(gg=gg, gb=0.6 * gg + 0.8 * rng.standard_normal((M_PER_RANK, l.g)),
                            dW=0.1 * rng.standard_normal(2 * l.g)))
        else:
            act = np.maximum(rng.standard_normal(M_PER_RANK * l.a * l.hw), 0).astype(np.float32)
            grad = (rng.standard_normal(M_PER_RANK * l.g * l.hw) / np.sqrt(M_PER_RANK * l.hw)).astype(np.float32)
            out.append(dict(act=act, grad=grad, dW=rng.standard_normal(l.g * l.a) / np.sqrt(l.a)))
    return out


def params():
    rng = np.random.default_rng(7)
    ps = []
    for l in LAYERS:
        if l.kind == "bn":
            ps.append(dict(W=np.concatenate([np.ones(l.g), np.zeros(l.g)]), V=np.zeros(2 * l.g)))
        else:
            ps.append(dict(W=rng.standard_normal(l.g * l.a) * np.sqrt(2 / l.a),
                           V=0.01 * rng.standard_normal(l.g * l.a)))
    return ps


def stats(l, d, n):
    if l.kind == "bn":
        return dict(M=O.build_bn_block(d["gg"], d["gb"], 0, n), dW=d["dW"])
    conv = l.kind == "conv"
    return dict(A=O.factor_A(d["act"], conv, l.a, l.hw, 0, n), G=O.factor_G(d["grad"], conv, l.g, l.hw, 0, n),
                dW=d["dW"])


def stage4(l, s, p):
    """Owner-local update (dist.cpp:539-633) with the oracle."""
    if l.kind == "bn":
        c = l.g
        pg, pb = O.precondition_bn(s["M"], s["dW"][:c], s["dW"][c:], LAM)
        w, _ = O.ngd_update(p["W"], np.concatenate([pg, pb]), p["V"], ETA, MOM)
        return w
    pi, Ai, Gi = O.damp_and_invert(s["A"], s["G"], l.a, l.g, LAM)
    P = O.kron_matvec(Gi, Ai, l.g, l.a, s["dW"].reshape(l.g, l.a)).reshape(-1)
    nw, _ = O.ngd_update(p["W"], P, p["V"], ETA, MOM)
    w, _ = O.rescale(nw, p["W"], l.g)
    return w


def full_batch_reference():
    shards = [shard_inputs(r) for r in range(WORLD)]
    ps = params()
    outs = []
    for li, l in enumerate(LAYERS):
        if l.kind == "bn":
            d = dict(gg=np.concatenate([s[li]["gg"] for s in shards]), gb=np.concatenate([s[li]["gb"] for s in shards]),
                     dW=np.mean([s[li]["dW"] for s in shards], axis=0))
        else:
            d = dict(act=np.concatenate([s[li]["act"] for s in shards]),
                     grad=np.concatenate([s[li]["grad"] for s in shards]),
                     dW=np.mean([s[li]["dW"] for s in shards], axis=0))
        outs.append(stage4(l, stats(l, d, WORLD * M_PER_RANK), ps[li]))
    return outs


def worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        lay, seg_st, seg_gr, seg_ag = plan_layout(LAYERS, WORLD)
        mine = shard_inputs(rank)
        # send buffer: [WORLD x statistics segment | WORLD x gradient segment]
        send = np.zeros(WORLD * (seg_st + seg_gr))
        for li, l in enumerate(LAYERS):
            st = stats(l, mine[li], M_PER_RANK)
            for key in ("A", "G", "M", "dW"):
                if key in st:
                    v = st[key]
                    base = (WORLD * seg_st + lay[li]["owner"] * seg_gr) if key == "dW" else lay[li]["owner"] * seg_st
                    send[base + lay[li][key]: base + lay[li][key] + v.size] = v
        t = torch.from_numpy(send)
        dist.all_reduce(t)                    # reduce_scatter_v = per-owner mean (dist.cpp:204-213)
        full = (t / WORLD).numpy()
        recv_st = full[rank * seg_st:(rank + 1) * seg_st]
        recv_gr = full[WORLD * seg_st + rank * seg_gr: WORLD * seg_st + (rank + 1) * seg_gr]
        ps = params()
        ag = np.zeros(WORLD * seg_ag)
        for li, l in enumerate(LAYERS):
            if lay[li]["owner"] != rank:
                continue
            s = {}
            if l.kind == "bn":
                s["M"] = recv_st[lay[li]["M"]: lay[li]["M"] + 3 * l.g]
                s["dW"] = recv_gr[lay[li]["dW"]: lay[li]["dW"] + 2 * l.g]
            else:
                s["A"] = recv_st[lay[li]["A"]: lay[li]["A"] + l.a * (l.a + 1) // 2]
                s["G"] = recv_st[lay[li]["G"]: lay[li]["G"] + l.g * (l.g + 1) // 2]
                s["dW"] = recv_gr[lay[li]["dW"]: lay[li]["dW"] + l.g * l.a]
            w = stage4(l, s, ps[li])
            off = rank * seg_ag + lay[li]["W"]
            ag[off: off + w.size] = w
        parts = [torch.zeros(seg_ag, dtype=torch.float64) for _ in range(WORLD)]
        dist.all_gather(parts, torch.from_numpy(ag[rank * seg_ag:(rank + 1) * seg_ag]))  # all_gather_v
        full = torch.cat(parts).numpy()
        got = []
        for li, l in enumerate(LAYERS):
            off = lay[li]["owner"] * seg_ag + lay[li]["W"]
            n = 2 * l.g if l.kind == "bn" else l.g * l.a
            got.append(full[off: off + n].copy())
        q.put((rank, got, [e["owner"] for e in lay]))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_world2_reduce_scatter_owner_update_all_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(WORLD):
        r, got, owners = q.get(timeout=300)
        res[r] = (got, owners)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(res[0][1]) == {0, 1}            # both ranks own work
    want = full_batch_reference()
    for li in range(len(LAYERS)):
        a, b = res[0][0][li], res[1][0][li]
        assert np.array_equal(a, b)            # replicas identical (acceptance.cpp:237-292)
        assert np.abs(a - want[li]).max() <= 1e-9 * max(1.0, np.abs(want[li]).max())  # K-invariance


def test_layout_every_payload_owned_once():
    for world in (1, 2, 4, 8):
        lay, seg_st, seg_gr, seg_ag = plan_layout(W.resnet50(), world)
        for r in range(world):
            for keys in (("A", "G", "M"), ("dW",)):  # statistics region, gradient region
                offs = [e[k] for e in lay if e["owner"] == r for k in keys if e[k] >= 0]
                assert len(offs) == len(set(offs))   # no two payloads share an offset
        assert all(0 <= e["owner"] < world for e in lay)
        assert seg_st % 64 == 0 and seg_gr % 64 == 0 and seg_ag % 64 == 0
