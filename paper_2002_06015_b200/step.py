"""Whole-step optimizer over the C ABI (spngd_opt_*), the drop-in for
`accumulate_microsteps` / `run_step` (src/dist.cpp:406-682) at n = 1 micro-step.

One `Optimizer` per rank (one process per GPU).  Inputs (captures, BN per-sample
gradient pairs, this rank's shard-mean weight gradient) and state (weights,
velocity) are device buffers owned by the library; `buffer()` exposes them.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import torch

from . import _native as N
from .spngd import check
from .workloads import Layer

(ACT, GRAD, DW, W, V, BN_GG, BN_GB, AINV, GINV, A_PACKED, G_PACKED, BN_M3C, ALL_WEIGHTS,
 GRAD_SAMPLED, BN_GG_SAMPLED, BN_GB_SAMPLED, RAW_ACT, BN_DY, BN_XHAT) = range(19)
EMPIRICAL, ONE_MC = 0, 1  # FisherMode (fisher.hpp:14)
BN_UNIT, BN_FULL = 0, 1   # BnMode (fisher.hpp:18)
PHASES = ["factor_gemm", "factor_reduce_bn", "reduce_scatter", "inverse", "precondition_update", "all_gather"]


def _mix(*xs) -> int:
    h = 0x9E3779B97F4A7C15
    for x in xs:
        h = (h ^ (int(x) & 0xFFFFFFFFFFFFFFFF)) * 0xBF58476D1CE4E5B9 & 0xFFFFFFFFFFFFFFFF
        h ^= h >> 31
    return h


def layer_descs(layers: List[Layer]):
    descs = []
    for l in layers:
        kind = {"fc": 0, "conv": 1, "bn": 2}[l.kind]
        descs.append(N.LayerDesc(kind, 0, l.a if l.kind != "bn" else 0, l.g, l.hw if l.kind == "conv" else 1))
    return (N.LayerDesc * len(descs))(*descs)


def plan_layout(layers: List[Layer], world: int, bn_full: bool = False):
    """Owners and owner-major RS/AG offsets (spngd_plan_layout_ex, host only;
    bn_full sizes BN statistics as the packed 2c x 2c block).

    Returns (entries, seg_stat, seg_grad, seg_ag): A/G/M offsets are within the
    owner's statistics segment, dW within the owner's gradient segment; the
    send buffer is [world * seg_stat | world * seg_grad]."""
    arr = layer_descs(layers)
    out = (N.LayoutEntry * len(layers))()
    seg_st, seg_gr, seg_ag = C.c_int64(), C.c_int64(), C.c_int64()
    check(N.lib().spngd_plan_layout_ex(arr, len(layers), world, 1 if bn_full else 0, out, C.byref(seg_st),
                                       C.byref(seg_gr), C.byref(seg_ag)))
    return [dict(owner=e.owner, A=e.off_A, G=e.off_G, M=e.off_M, dW=e.off_dW, W=e.off_W) for e in out], \
        seg_st.value, seg_gr.value, seg_ag.value


class Comm:
    """NCCL communicator bootstrap: rank 0's unique id is shared by the caller
    (torch.distributed object broadcast), then spngd_ctx_init_comm."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(N.lib().spngd_nccl_unique_id(buf))
        return buf.raw


class Optimizer:
    def __init__(self, layers: List[Layer], batch: int, lam: float = 2.5e-4, rescale: bool = True,
                 device: int = 0, world: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                 stream=None, stale: bool = False, stale_alpha: float = 0.1, fisher_mode: int = EMPIRICAL,
                 elem_size: int = 4, sgd: bool = False, bn_mode: int = 0,
                 wgrad: bool = False):
        self.layers, self.batch, self.lam = layers, batch, lam
        self.fisher_mode, self.sgd, self.bn_mode = fisher_mode, sgd, bn_mode
        self.world, self.rank, self.device = world, rank, device
        L = N.lib()
        self.ctx = C.c_void_p()
        check(L.spngd_ctx_create(device, stream, C.byref(self.ctx)))
        if world > 1:
            check(L.spngd_ctx_init_comm(self.ctx, world, rank, C.create_string_buffer(nccl_id, 128)))
        arr = layer_descs(layers)
        cfg = N.OptConfig(lam, int(rescale), int(stale), stale_alpha, batch, int(fisher_mode), int(elem_size), int(sgd), int(bn_mode), int(wgrad), 0)
        self.h = C.c_void_p()
        check(L.spngd_opt_create(self.ctx, arr, len(layers), C.byref(cfg), C.byref(self.h)))

    def close(self):
        L = N.lib()
        if getattr(self, "h", None):
            L.spngd_opt_destroy(self.h)
            self.h = None
        if getattr(self, "ctx", None):
            L.spngd_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- buffers --------------------------------------------------------------
    def numel(self, li: int, which: int) -> int:
        l, B = self.layers[li], self.batch
        if which == ACT:
            return B * l.a * l.hw
        if which == RAW_ACT:
            return B * (l.c_in * l.h_in * l.w_in if l.kind == "conv" else l.a)
        if which in (GRAD, GRAD_SAMPLED):
            return B * l.g * l.hw
        if which in (DW, W, V):
            return 2 * l.g if l.kind == "bn" else l.g * l.a
        if which in (BN_GG, BN_GB, BN_GG_SAMPLED, BN_GB_SAMPLED):
            return B * l.g
        if which in (BN_DY, BN_XHAT):
            return B * l.g * self.bn_spatial[li]
        if which == A_PACKED:
            return l.a * (l.a + 1) // 2
        if which == G_PACKED:
            return l.g * (l.g + 1) // 2
        if which == BN_M3C:
            return (2 * l.g) * (2 * l.g + 1) // 2 if self.bn_mode == BN_FULL else 3 * l.g
        raise ValueError(which)

    def ptr(self, li: int, which: int):
        if which in (GRAD_SAMPLED, BN_GG_SAMPLED, BN_GB_SAMPLED) and self.fisher_mode != ONE_MC:
            from .spngd import MissingMcPass
            raise MissingMcPass(f"layer {li}: no sampled-label backward (fisher_mode is Empirical)")
        ld = C.c_int64()
        p = N.lib().spngd_opt_buffer(self.h, li, which, C.byref(ld))
        return p, ld.value

    def owner(self, li: int) -> int:
        return N.lib().spngd_opt_owner(self.h, li)

    def download(self, li: int, which: int) -> torch.Tensor:
        """Copies a buffer to a CPU float32 tensor (synchronizes)."""
        p, ld = self.ptr(li, which)
        if not p:
            raise ValueError(f"layer {li} buffer {which} not available on rank {self.rank}")
        if which in (AINV, GINV):
            l = self.layers[li]
            n = (2 * l.g if l.kind == "bn" else l.a) if which == AINV else l.g
            t = torch.empty(n, ld, dtype=torch.float32).pin_memory()
            check(N.lib().spngd_copy(self.ctx, C.c_void_p(t.data_ptr()), C.c_void_p(p), t.numel() * 4))
            self.sync()
            return t[:, :n].clone()
        n = self.numel(li, which)
        t = torch.empty(n, dtype=torch.float32).pin_memory()
        check(N.lib().spngd_copy(self.ctx, C.c_void_p(t.data_ptr()), C.c_void_p(p), n * 4))
        self.sync()
        return t.clone()

    def upload(self, li: int, which: int, host: torch.Tensor):
        p, _ = self.ptr(li, which)
        h = host.contiguous().float()
        if h.numel() != self.numel(li, which):
            raise ValueError("size mismatch")
        h = h.pin_memory()
        check(N.lib().spngd_copy(self.ctx, C.c_void_p(p), C.c_void_p(h.data_ptr()), h.numel() * 4))
        self.sync()

    def sync(self):
        # spngd_opt_sync: a failed step names its layer (fisher.cpp:48-51 layer_tag)
        check(N.lib().spngd_opt_sync(self.h) if getattr(self, "h", None) else N.lib().spngd_ctx_sync(self.ctx))

    # ---- synthetic inputs -------------------------
    def synth(self, seed: int = 42):
        """Per-layer synthetic inputs generated in place on the device:
        conv/FC inputs ReLU(N(0,1)) laid out as the reference im2col capture,
        output grads N(0,1)/sqrt(B hw), BN pairs g ~ N, b = 0.6 g + 0.8 N,
        dW ~ N(0,1)/sqrt(a), W He-normal (identical on every rank), V = 0.01 N,
        gamma = 1, beta = 0.  Captures and dW differ per rank (distinct shards)."""
        L, B, r = N.lib(), self.batch, self.rank
        for li, l in enumerate(self.layers):
            if l.kind == "bn" and getattr(self, "bn_spatial", None):
                n = B * l.g * self.bn_spatial[li]
                dy, _ = self.ptr(li, BN_DY)
                xh, _ = self.ptr(li, BN_XHAT)
                check(L.spngd_synth_normal(self.ctx, dy, n, _mix(seed, li, 8, r), float((B * self.bn_spatial[li]) ** -0.5),
                                           0.0, 0))
                check(L.spngd_synth_normal(self.ctx, xh, n, _mix(seed, li, 9, r), 1.0, 0.0, 0))
            if l.kind == "bn":
                gg, _ = self.ptr(li, BN_GG)
                gb, _ = self.ptr(li, BN_GB)
                check(L.spngd_synth_bn_pairs(self.ctx, gg, gb, B * l.g, _mix(seed, li, 5, r)))
                if self.fisher_mode == ONE_MC:
                    sg, _ = self.ptr(li, BN_GG_SAMPLED)
                    sb, _ = self.ptr(li, BN_GB_SAMPLED)
                    check(L.spngd_synth_bn_pairs(self.ctx, sg, sb, B * l.g, _mix(seed, li, 7, r)))
                dw, _ = self.ptr(li, DW)
                check(L.spngd_synth_normal(self.ctx, dw, 2 * l.g, _mix(seed, li, 2, r), 0.1, 0.0, 0))
                w, _ = self.ptr(li, W)
                check(L.spngd_synth_normal(self.ctx, w, l.g, 0, 0.0, 1.0, 0))  # gamma = 1
                check(L.spngd_synth_normal(self.ctx, C.c_void_p(w + 4 * l.g), l.g, 0, 0.0, 0.0, 0))  # beta = 0
                continue
            act, _ = self.ptr(li, ACT)
            if l.kind == "conv" and getattr(self, "raw_inputs", False):
                raw, _ = self.ptr(li, RAW_ACT)  # same counters as the capture kernel: im2col(raw) == capture
                check(L.spngd_synth_normal(self.ctx, raw, B * l.c_in * l.h_in * l.w_in, _mix(seed, li, 0, r), 1.0, 0.0,
                                           1))
            elif l.kind == "conv":
                check(L.spngd_synth_conv_capture(self.ctx, act, B, l.c_in, l.h_in, l.w_in, l.k, l.stride, l.pad,
                                                 _mix(seed, li, 0, r), 1, 1.0, 0.0))
            else:
                check(L.spngd_synth_normal(self.ctx, act, B * l.a, _mix(seed, li, 0, r), 1.0, 0.0, 1))
            grad, _ = self.ptr(li, GRAD)
            check(L.spngd_synth_normal(self.ctx, grad, B * l.g * l.hw, _mix(seed, li, 1, r),
                                       float((B * l.hw) ** -0.5), 0.0, 0))
            if self.fisher_mode == ONE_MC:
                gs, _ = self.ptr(li, GRAD_SAMPLED)
                check(L.spngd_synth_normal(self.ctx, gs, B * l.g * l.hw, _mix(seed, li, 6, r),
                                           float((B * l.hw) ** -0.5), 0.0, 0))
            dw, _ = self.ptr(li, DW)
            check(L.spngd_synth_normal(self.ctx, dw, l.g * l.a, _mix(seed, li, 2, r), float(l.a ** -0.5), 0.0, 0))
            w, _ = self.ptr(li, W)
            check(L.spngd_synth_normal(self.ctx, w, l.g * l.a, _mix(seed, li, 3), float((2.0 / l.a) ** 0.5), 0.0, 0))
            v, _ = self.ptr(li, V)
            if v:
                check(L.spngd_synth_normal(self.ctx, v, l.g * l.a, _mix(seed, li, 4), 0.01, 0.0, 0))
        self.sync()

    # ---- the step -----------------------------------------------------------------
    def step(self, step: int, eta: float = 1.25e-2, momentum: float = 0.993):
        check(N.lib().spngd_opt_step(self.h, step, eta, momentum))

    def step_host(self, step: int, inputs, weights_out=None, eta: float = 1.25e-2, momentum: float = 0.993):
        """The step fed from host memory (spngd_opt_step_host): `inputs` is a list
        of (layer, which, host pointer) -- pinned memory makes the transfer
        asynchronous and, with the wave schedule, overlapped with the step;
        `weights_out` (host pointer, optional) receives every weight replica."""
        arr = (N.HostInput * max(len(inputs), 1))(*[N.HostInput(li, w, hp) for li, w, hp in inputs])
        check(N.lib().spngd_opt_step_host(self.h, step, eta, momentum, arr, len(inputs), weights_out))

    def phase_ms(self):
        out = (C.c_float * 6)()
        check(N.lib().spngd_opt_phase_ms(self.h, out))
        return dict(zip(PHASES, list(out)))

    def attach_peers(self, pg):
        """Stages 2-3 (statistics) and 5 over NVLink peer memory
        (spngd_opt_attach_peers): exchanges the replica / inbox buffers' IPC handles over the torch.distributed group `pg` (the
        control plane) and attaches them.  Call on every rank before the first step."""
        h = C.create_string_buffer(128)
        check(N.lib().spngd_opt_ipc_handle(self.h, h))
        allh = [None] * self.world
        pg.all_gather_object(allh, h.raw)
        buf = C.create_string_buffer(b"".join(allh), 128 * self.world)
        check(N.lib().spngd_opt_attach_peers(self.h, buf))

    def enable_bn_inputs(self, spatial=None):
        """SURVEY §8f row 1 in the step: every BN layer takes the backward's dY
        and x_hat (BN_DY / BN_XHAT, B x (c*S)); one launch per step forms the
        per-sample capture, the moments and the BN gradient payload
        (spngd_opt_enable_bn_inputs).  `spatial`: S per layer (default: the
        h_out*w_out of the conv each BN layer follows).  Before the first step."""
        if spatial is None:
            spatial, prev = [], 1
            for l in self.layers:
                if l.kind == "conv":
                    prev = l.hw
                spatial.append(prev if l.kind == "bn" else 0)
        arr = (C.c_int64 * len(self.layers))(*spatial)
        check(N.lib().spngd_opt_enable_bn_inputs(self.h, arr))
        self.bn_spatial = list(spatial)

    def enable_raw_inputs(self, implicit: bool = False):
        """The step takes each conv layer's raw input (RAW_ACT, B x c_in x h x w)
        and forms the im2col capture on the device (net.cpp:199-219), or with
        implicit=True never forms it: the factor / wgrad GEMMs gather the
        operand from the raw input (spngd_opt_enable_raw_inputs_ex).  Call
        before the first step."""
        g = (N.ConvGeom * len(self.layers))()
        for i, l in enumerate(self.layers):
            if l.kind == "conv":
                g[i] = N.ConvGeom(l.c_in, l.h_in, l.w_in, l.k, l.stride, l.pad)
        check(N.lib().spngd_opt_enable_raw_inputs_ex(self.h, g, int(implicit)))
        self.raw_inputs = True

    def input_buffers(self):
        """(layer, which) of every per-step input the host supplies: raw conv
        inputs when enabled (else the im2col captures), grads, BN pairs, dW."""
        out = []
        for li, l in enumerate(self.layers):
            if l.kind == "bn" and getattr(self, "bn_spatial", None):
                out += [(li, BN_DY), (li, BN_XHAT)]  # the step forms the captures and the BN dW
            elif l.kind == "bn":
                out += [(li, BN_GG), (li, BN_GB), (li, DW)]
            else:
                a = RAW_ACT if (getattr(self, "raw_inputs", False) and l.kind == "conv") else ACT
                out += [(li, a), (li, GRAD), (li, DW)]
        return out

    def ledger(self):
        """The CommLedger rows every step appended (dist.cpp:511-537, 661-662)."""
        from .spngd import CommLedger, _row_from_c
        L = N.lib()
        n = L.spngd_opt_ledger(self.h, None, 0)
        out = (N.LedgerRowC * max(n, 1))()
        L.spngd_opt_ledger(self.h, out, n)
        return CommLedger([_row_from_c(out[i]) for i in range(n)])

    def clear_ledger(self):
        check(N.lib().spngd_opt_ledger_clear(self.h))

    def wire_bytes(self):
        """Bytes this rank handed to NCCL in the last step: statistics, gradients, all-gather."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(N.lib().spngd_opt_wire_bytes(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return dict(stat=a.value, grad=b.value, all_gather=c.value)

    def launch_count(self) -> int:
        return N.lib().spngd_opt_launch_count(self.h)

    def set_overlap(self, on: bool):
        """Single-GPU wave schedule (inverse recursion of the largest factors
        overlapping the remaining factor SYRKs); off = phase-serial.  Same
        kernels and inputs either way (spngd_opt_set_overlap)."""
        check(N.lib().spngd_opt_set_overlap(self.h, int(on)))

    def stale_info(self, layer: int, which: str):
        """Tracker state of statistic which in {"A", "G", "F"} of `layer`
        (StaleTracker t_X / delta / refresh count) and whether it refreshed
        in the last step."""
        tx, d, rc, due = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        check(N.lib().spngd_opt_stale_info(self.h, layer, {"A": 0, "G": 1, "F": 2}[which], C.byref(tx), C.byref(d),
                                           C.byref(rc), C.byref(due)))
        return dict(t_x=tx.value, delta=d.value, refreshes=rc.value, refreshed=bool(due.value))
