"""Reference-shaped Python API over the B200 C ABI.

Mirrors the public functions of the reference library (`spngd`, C++20) that
sit on the optimizer-step hot path, with the same names, argument meaning and
error behaviour (include/spngd/fisher.hpp:56-124, linalg.hpp:60-77,
stale.hpp:92-132, errors.hpp:10-85).  Tensors are torch CUDA fp32 tensors in
the reference layouts; every computation runs in libspngd_b200.so kernels.
The only torch calls here allocate outputs and move layouts (plumbing).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import torch

from . import _native as N


# ---- errors (include/spngd/errors.hpp:10-85) --------------------------------
class Error(RuntimeError):
    pass


class ShapeMismatch(Error):
    pass


class NotPositiveDefinite(Error):
    pass


class SingularBlock(Error):
    pass


class ZeroReference(Error):
    pass


class EmptyBatch(Error):
    pass


class MissingMcPass(Error):
    pass


class StaleBeyondLimit(Error):
    pass


class RefreshOutOfTurn(Error):
    pass


class IndivisibleBatch(Error):
    pass


class MissingOwner(Error):
    pass


class EmptyAccumulation(Error):
    pass


class CudaError(Error):
    pass


class ParseError(Error):  # errors.hpp: ledger / manifest parsing
    pass


# status codes of include/spngd_b200.h (spngd_status)
SPNGD_OK, SPNGD_ERR_SHAPE_MISMATCH, SPNGD_ERR_NOT_POSITIVE_DEFINITE, SPNGD_ERR_SINGULAR_BLOCK = 0, 1, 2, 3
_ERRORS = {1: ShapeMismatch, 2: NotPositiveDefinite, 3: SingularBlock, 4: ZeroReference,
           5: EmptyBatch, 6: MissingMcPass, 7: StaleBeyondLimit, 8: RefreshOutOfTurn,
           9: IndivisibleBatch, 10: MissingOwner, 11: EmptyAccumulation, 100: CudaError,
           101: Error, 102: Error}


def check(rc: int):
    if rc:
        msg = N.lib().spngd_last_error().decode()
        raise _ERRORS.get(rc, Error)(msg)


# ---- context -----------------------------------------------------------------
class Context:
    """One per device; wraps spngd_ctx on torch's current stream."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        self.device = device
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        # torch's default stream has handle 0, which spngd_ctx_create reads as
        # "no stream" (a private non-blocking stream, unordered with torch's
        # work).  Pass cudaStreamLegacy (0x1) instead so calls are stream-ordered
        # after the torch kernels that produced their inputs.
        handle = s.cuda_stream if s.cuda_stream else 1
        h = C.c_void_p()
        check(N.lib().spngd_ctx_create(device, C.c_void_p(handle), C.byref(h)))
        self.h = h

    def sync(self):
        check(N.lib().spngd_ctx_sync(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                N.lib().spngd_ctx_destroy(self.h)
        except Exception:
            pass


_CTX = {}


def context(device=None) -> Context:
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the SP-NGD step has no CPU fallback")
    d = torch.cuda.current_device() if device is None else device
    if d not in _CTX:
        _CTX[d] = Context(d)
    return _CTX[d]


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ShapeMismatch("expected a contiguous float32 CUDA tensor")
    return C.c_void_p(t.data_ptr())


def packed_size(n: int) -> int:
    return n * (n + 1) // 2


# ---- types mirroring net.hpp / fisher.hpp ------------------------------------
FC, CONV, BN = "fc", "conv", "bn"


@dataclass
class LayerSpec:  # net.hpp:13-31
    kind: str
    d_in: int = 0
    d_out: int = 0
    c_in: int = 0
    c_out: int = 0
    kernel: int = 0
    stride: int = 1
    padding: int = 0
    channels: int = 0

    @staticmethod
    def fc(d_in, d_out):
        return LayerSpec(FC, d_in=d_in, d_out=d_out)

    @staticmethod
    def conv(c_in, c_out, kernel, stride=1, padding=0):
        return LayerSpec(CONV, c_in=c_in, c_out=c_out, kernel=kernel, stride=stride, padding=padding)

    @staticmethod
    def batch_norm(channels):
        return LayerSpec(BN, channels=channels)

    @property
    def a(self):  # Kronecker A dimension (dist.cpp:551-555)
        return self.d_in if self.kind == FC else self.c_in * self.kernel * self.kernel

    @property
    def g(self):
        return self.d_out if self.kind == FC else self.c_out

    def describe(self):
        return f"{self.kind}({self.a}->{self.g})" if self.kind != BN else f"bn({self.channels})"


@dataclass
class NetworkSpec:  # net.hpp:39-43
    layers: List[LayerSpec]


@dataclass
class LayerCapture:  # net.hpp:84-101
    act: Optional[torch.Tensor] = None
    grad_true: Optional[torch.Tensor] = None
    grad_sampled: Optional[torch.Tensor] = None
    bn_ggamma_true: Optional[torch.Tensor] = None
    bn_gbeta_true: Optional[torch.Tensor] = None
    bn_ggamma_sampled: Optional[torch.Tensor] = None
    bn_gbeta_sampled: Optional[torch.Tensor] = None
    rows_per_sample: int = 0
    grad_rows_per_sample: int = 0
    h_out: int = 1
    w_out: int = 1


@dataclass
class CaptureBuffer:  # net.hpp:114-119
    batch_size: int
    layers: List[LayerCapture]


class SymMatrix:
    """Packed upper-triangle symmetric matrix (linalg.hpp:24-55) on the GPU."""

    def __init__(self, dim: int, data: Optional[torch.Tensor] = None, device=None):
        self.dim = dim
        self.data = data if data is not None else torch.zeros(
            packed_size(dim), dtype=torch.float32, device=device or "cuda")

    def unpack(self) -> torch.Tensor:
        n = self.dim
        iu = torch.triu_indices(n, n, device=self.data.device)
        d = torch.zeros(n, n, dtype=self.data.dtype, device=self.data.device)
        d[iu[0], iu[1]] = self.data
        d[iu[1], iu[0]] = self.data
        return d

    @staticmethod
    def pack(dense: torch.Tensor) -> "SymMatrix":
        n = dense.shape[0]
        if dense.shape != (n, n):
            raise ShapeMismatch("pack: matrix is not square")
        iu = torch.triu_indices(n, n, device=dense.device)
        return SymMatrix(n, dense[iu[0], iu[1]].contiguous().float())


class FisherMode:
    Empirical = "emp"
    OneMC = "1mc"


@dataclass
class KroneckerBlock:  # fisher.hpp:24-31
    layer: int = -1
    A: Optional[SymMatrix] = None
    G: Optional[SymMatrix] = None
    A_inv: Optional[SymMatrix] = None
    G_inv: Optional[SymMatrix] = None
    A_inv_dense: Optional[torch.Tensor] = None
    G_inv_dense: Optional[torch.Tensor] = None
    pi: float = 1.0
    lam: float = 0.0
    fresh_step_a: int = -1
    fresh_step_g: int = -1


@dataclass
class FullBnBlock:  # fisher.hpp:45-51: full 2c x 2c block (BnMode::Full)
    layer: int = -1
    F: Optional["SymMatrix"] = None
    F_inv: Optional["SymMatrix"] = None
    F_inv_dense: Optional[torch.Tensor] = None
    lam: float = 0.0
    fresh_step: int = -1


@dataclass
class UnitBnBlock:  # fisher.hpp:36-42, moments interleaved (fgg, fgb, fbb)
    layer: int = -1
    m3c: Optional[torch.Tensor] = None
    lam: float = 0.0
    fresh_step: int = -1

    @property
    def fgg(self):
        return self.m3c[0::3]

    @property
    def fgb(self):
        return self.m3c[1::3]

    @property
    def fbb(self):
        return self.m3c[2::3]


# ---- K1 / K2 -----------------------------------------------------------------
def _check_layer(cap: CaptureBuffer, net: NetworkSpec, layer: int, who: str):
    if layer < 0 or layer >= len(net.layers):  # fisher.cpp:38-44
        raise ShapeMismatch(f"{who}: layer index out of range")
    if len(cap.layers) != len(net.layers):
        raise ShapeMismatch(f"{who}: capture does not match network")


def _range(cap, lo, hi, who):
    hi = cap.batch_size if hi is None else hi
    if lo < 0 or hi > cap.batch_size or hi <= lo:  # fisher.cpp:46-49
        raise EmptyBatch(f"{who}: empty sample range")
    return lo, hi


def factor_requests(cap: CaptureBuffer, net: NetworkSpec, reqs):
    """Builds FactorReq structs for [(layer, 'A'|'G', lo, hi, mode, out)]."""
    out = []
    for layer, which, lo, hi, mode, dst in reqs:
        who = f"factor_{which}"
        _check_layer(cap, net, layer, who)
        lo, hi = _range(cap, lo, hi, who)
        L, lc = net.layers[layer], cap.layers[layer]
        tag = f"layer {layer} ({L.describe()})"
        if L.kind == BN:
            raise ShapeMismatch(f"{who}: {tag} has no Kronecker factors")
        n = hi - lo
        if which == "A":
            x = lc.act
            if x is None or x.numel() == 0:
                raise EmptyBatch(f"{who}: {tag}: no captured activations")
            dim = L.a
            hw = lc.h_out * lc.w_out
            scale = 1.0 / n if L.kind == FC else 1.0 / (n * hw)  # fisher.cpp:104-108
        else:
            if mode == FisherMode.OneMC:
                x = lc.grad_sampled
                if x is None or x.numel() == 0:
                    raise MissingMcPass(f"{who}: {tag}: no sampled-label backward was run")
            else:
                x = lc.grad_true
                if x is None or x.numel() == 0:
                    raise EmptyBatch(f"{who}: {tag}: no captured gradients")
            dim = L.g
            hw = lc.h_out * lc.w_out
            scale = 1.0 / n  # fisher.cpp:138-139
        layout = 0 if L.kind == FC else 1
        out.append(N.FactorReq(x.data_ptr(), dim, hw, layout, lo, hi, scale, dst.data_ptr()))
    return out


def factor_A(cap: CaptureBuffer, net: NetworkSpec, layer: int, lo: int = 0, hi: Optional[int] = None,
             compensated: bool = False) -> SymMatrix:
    """fisher.hpp:56-59.  `compensated` is accepted for signature parity; the
    device path always accumulates tiles in fp32 TMEM and partials in fp64."""
    L = net.layers[layer] if 0 <= layer < len(net.layers) else None
    dim = L.a if L is not None and L.kind != BN else 0
    out = torch.empty(max(packed_size(dim), 1), dtype=torch.float32, device="cuda")
    reqs = factor_requests(cap, net, [(layer, "A", lo, hi, FisherMode.Empirical, out)])
    arr = (N.FactorReq * 1)(*reqs)
    check(N.lib().spngd_factor_sym_batched(context().h, 1, arr))
    return SymMatrix(dim, out)


def factor_G(cap: CaptureBuffer, net: NetworkSpec, layer: int, mode=FisherMode.Empirical, lo: int = 0,
             hi: Optional[int] = None, compensated: bool = False) -> SymMatrix:
    """fisher.hpp:63-67."""
    L = net.layers[layer] if 0 <= layer < len(net.layers) else None
    dim = L.g if L is not None and L.kind != BN else 0
    out = torch.empty(max(packed_size(dim), 1), dtype=torch.float32, device="cuda")
    reqs = factor_requests(cap, net, [(layer, "G", lo, hi, mode, out)])
    arr = (N.FactorReq * 1)(*reqs)
    check(N.lib().spngd_factor_sym_batched(context().h, 1, arr))
    return SymMatrix(dim, out)


def factor_sym(x: torch.Tensor, dim: int, hw: int, layout: int, lo: int, hi: int, scale: float) -> torch.Tensor:
    """Raw K1 entry: scale * sum_s X_s X_s^T, packed (spngd_factor_sym_batched)."""
    out = torch.empty(packed_size(dim), dtype=torch.float32, device=x.device)
    arr = (N.FactorReq * 1)(N.FactorReq(x.data_ptr(), dim, hw, layout, lo, hi, scale, out.data_ptr()))
    check(N.lib().spngd_factor_sym_batched(context().h, 1, arr))
    return out


def build_bn_block(cap: CaptureBuffer, net: NetworkSpec, layer: int, mode=FisherMode.Empirical, lo: int = 0,
                   hi: Optional[int] = None, compensated: bool = False) -> UnitBnBlock:
    """fisher.hpp:71-76 -> interleaved 3c moments on the device."""
    _check_layer(cap, net, layer, "build_bn_block")
    lo, hi = _range(cap, lo, hi, "build_bn_block")
    L, lc = net.layers[layer], cap.layers[layer]
    if L.kind != BN:
        raise ShapeMismatch(f"build_bn_block: layer {layer} ({L.describe()}) is not BatchNorm")
    if mode == FisherMode.OneMC:
        gg, gb = lc.bn_ggamma_sampled, lc.bn_gbeta_sampled
        if gg is None or gg.numel() == 0:
            raise MissingMcPass("build_bn_block: no sampled-label backward was run")
    else:
        gg, gb = lc.bn_ggamma_true, lc.bn_gbeta_true
        if gg is None or gg.numel() == 0:
            raise EmptyBatch("build_bn_block: no captured gradients")
    c = L.channels
    out = torch.empty(3 * c, dtype=torch.float32, device=gg.device)
    arr = (N.BnMomentsReq * 1)(N.BnMomentsReq(gg.data_ptr(), gb.data_ptr(), c, lo, hi, out.data_ptr()))
    check(N.lib().spngd_bn_moments_batched(context().h, 1, arr))
    return UnitBnBlock(layer=layer, m3c=out)


def bn_grad_reduce(dy: torch.Tensor, xhat: torch.Tensor, M: int, c: int, S: int):
    """Per-sample BN parameter gradients of the backward (net.cpp:467-475):
    dY, x_hat M x (c*S) -> (gg, gb) M x c, the bn_ggamma/bn_gbeta capture."""
    return bn_grad_reduce_batched([(dy, xhat, M, c, S)])[0]


def bn_grad_reduce_batched(items):
    """bn_grad_reduce over several BN layers in one launch; items are
    (dy, xhat, M, c, S) tuples."""
    reqs, outs = [], []
    for dy, xh, M, c, S in items:
        _ptr(dy), _ptr(xh)  # contiguous float32 CUDA tensors
        if M > 0 and (dy.numel() != M * c * S or xh.numel() != M * c * S):
            raise ShapeMismatch("bn_grad_reduce: dY / x_hat must be M x (c*S)")
        gg = torch.empty(M, c, dtype=torch.float32, device=dy.device)
        gb = torch.empty(M, c, dtype=torch.float32, device=dy.device)
        reqs.append(N.BnGradReq(dy.data_ptr(), xh.data_ptr(), M, c, S, gg.data_ptr(), gb.data_ptr()))
        outs.append((gg, gb))
    if reqs:
        arr = (N.BnGradReq * len(reqs))(*reqs)
        check(N.lib().spngd_bn_grad_reduce_batched(context().h, len(reqs), arr))
    return outs


# ---- K3 / K4 -------------------------------------------------------------------
def spd_inverse(m: SymMatrix, damping: float, dense: bool = False):
    """linalg.hpp:60: (m + damping I)^-1, packed (and dense if requested)."""
    n = m.dim
    if n == 0:
        raise ShapeMismatch("spd_inverse: empty matrix")
    out = torch.empty(packed_size(n), dtype=torch.float32, device=m.data.device)
    ld = (n + 31) // 32 * 32
    dn = torch.empty(n, ld, dtype=torch.float32, device=m.data.device) if dense else None
    req = N.SpdReq(m.data.data_ptr(), n, damping, None, dn.data_ptr() if dense else None, ld,
                   out.data_ptr())
    arr = (N.SpdReq * 1)(req)
    check(N.lib().spngd_spd_inverse_batched(context().h, 1, arr, None))
    res = SymMatrix(n, out)
    return (res, dn[:, :n]) if dense else res


def spd_inverse_batched(ms: List[SymMatrix], damping: float, info: list = None) -> List[SymMatrix]:
    """spd_inverse (linalg.hpp:60) over many matrices in one batched call.
    `info` (a list) receives the per-request status codes; the raised
    NotPositiveDefinite names the first failing request."""
    reqs, outs = [], []
    for m in ms:
        if m.dim == 0:
            raise ShapeMismatch("spd_inverse: empty matrix")
        out = torch.empty(packed_size(m.dim), dtype=torch.float32, device=m.data.device)
        reqs.append(N.SpdReq(m.data.data_ptr(), m.dim, damping, None, None, 0, out.data_ptr()))
        outs.append(SymMatrix(m.dim, out))
    if reqs:
        arr = (N.SpdReq * len(reqs))(*reqs)
        inf = (C.c_int * len(reqs))()
        rc = N.lib().spngd_spd_inverse_batched(context().h, len(reqs), arr, inf)
        if info is not None:
            info[:] = list(inf)
        check(rc)
    return outs


def damp_and_invert_batched(blocks: List[KroneckerBlock], lam: float, info: list = None):
    """damp_and_invert (fisher.cpp:218-228) for many blocks in one batched call.
    `info` (a list) receives the per-block status codes."""
    if not (lam > 0.0):
        raise NotPositiveDefinite("damp_and_invert: lambda must be > 0")
    reqs, keep = [], []
    for b in blocks:
        a, g = b.A.dim, b.G.dim
        if a == 0 or g == 0:
            raise ShapeMismatch("avg_eigenvalue: empty matrix")
        dev = b.A.data.device
        lda, ldg = (a + 31) // 32 * 32, (g + 31) // 32 * 32
        Ad = torch.empty(a, lda, dtype=torch.float32, device=dev)
        Gd = torch.empty(g, ldg, dtype=torch.float32, device=dev)
        Ap = torch.empty(packed_size(a), dtype=torch.float32, device=dev)
        Gp = torch.empty(packed_size(g), dtype=torch.float32, device=dev)
        pi = torch.empty(1, dtype=torch.float32, device=dev)
        reqs.append(N.KronReq(b.A.data.data_ptr(), b.G.data.data_ptr(), a, g, Ad.data_ptr(), lda,
                              Gd.data_ptr(), ldg, Ap.data_ptr(), Gp.data_ptr(), pi.data_ptr()))
        keep.append((b, Ad, Gd, Ap, Gp, pi))
    arr = (N.KronReq * len(reqs))(*reqs)
    inf = (C.c_int * len(reqs))()
    rc = N.lib().spngd_damp_and_invert_batched(context().h, len(reqs), arr, lam, inf)
    if info is not None:
        info[:] = list(inf)
    check(rc)
    for b, Ad, Gd, Ap, Gp, pi in keep:
        b.A_inv, b.G_inv = SymMatrix(b.A.dim, Ap), SymMatrix(b.G.dim, Gp)
        b.A_inv_dense, b.G_inv_dense = Ad, Gd
        b.pi = float(pi.item())
        b.lam = lam
    return blocks


def damp_and_invert(block: KroneckerBlock, lam: float):
    """fisher.hpp:85."""
    damp_and_invert_batched([block], lam)


def damp_bn(block: UnitBnBlock, lam: float):
    """fisher.hpp:88; the step recomputes the 2x2 inverse per use (fisher.cpp:268-270)."""
    if not (lam > 0.0):
        raise NotPositiveDefinite("damp_bn: lambda must be > 0")
    block.lam = lam


# ---- K5 / K6 / K7 ------------------------------------------------------------
def _dense_inv(b: KroneckerBlock, which: str):
    d = b.A_inv_dense if which == "A" else b.G_inv_dense
    if d is None:
        raise StaleBeyondLimit("precondition: Kronecker block never inverted")
    return d


def precondition(block: KroneckerBlock, grad: torch.Tensor) -> torch.Tensor:
    """fisher.hpp:93: G_inv * grad * A_inv."""
    g, a = block.G.dim, block.A.dim
    if grad.shape != (g, a):
        raise ShapeMismatch("kron_matvec: X must be dim(G) x dim(A)")
    Ad, Gd = _dense_inv(block, "A"), _dense_inv(block, "G")
    P = torch.empty(g, a, dtype=torch.float32, device=grad.device)
    req = N.PrecondReq(Gd.data_ptr(), Gd.shape[1], Ad.data_ptr(), Ad.shape[1], grad.contiguous().data_ptr(),
                       g, a, P.data_ptr(), None, None, 0)
    arr = (N.PrecondReq * 1)(req)
    check(N.lib().spngd_precondition_update_batched(context().h, 1, arr, 0.0, 0.0))
    return P


def kron_update(block: KroneckerBlock, grad: torch.Tensor, W: torch.Tensor, V: torch.Tensor, eta: float,
                momentum: float, rescale: bool) -> torch.Tensor:
    """Fused K5+K6 for one layer: W, V updated in place; returns P."""
    g, a = block.G.dim, block.A.dim
    Ad, Gd = _dense_inv(block, "A"), _dense_inv(block, "G")
    P = torch.empty(g, a, dtype=torch.float32, device=grad.device)
    req = N.PrecondReq(Gd.data_ptr(), Gd.shape[1], Ad.data_ptr(), Ad.shape[1], grad.contiguous().data_ptr(),
                       g, a, P.data_ptr(), W.data_ptr(), V.data_ptr(), int(rescale))
    arr = (N.PrecondReq * 1)(req)
    check(N.lib().spngd_precondition_update_batched(context().h, 1, arr, eta, momentum))
    return P


def build_bn_full(cap: CaptureBuffer, net: NetworkSpec, layer: int, mode=FisherMode.Empirical, lo: int = 0,
                  hi: Optional[int] = None) -> FullBnBlock:
    """fisher.hpp:79-81 (build_bn_full, fisher.cpp:187-216): F = E[u u^T] over the
    interleaved (g_gamma, g_beta) per-sample vector, packed 2c x 2c."""
    _check_layer(cap, net, layer, "build_bn_full")
    lo, hi = _range(cap, lo, hi, "build_bn_full")
    L, lc = net.layers[layer], cap.layers[layer]
    if L.kind != BN:
        raise ShapeMismatch(f"build_bn_full: layer {layer} ({L.describe()}) is not BatchNorm")
    if mode == FisherMode.OneMC:
        gg, gb = lc.bn_ggamma_sampled, lc.bn_gbeta_sampled
        if gg is None or gg.numel() == 0:
            raise MissingMcPass("build_bn_full: no sampled-label backward was run")
    else:
        gg, gb = lc.bn_ggamma_true, lc.bn_gbeta_true
        if gg is None or gg.numel() == 0:
            raise EmptyBatch("build_bn_full: no captured gradients")
    c = L.channels
    out = torch.empty(packed_size(2 * c), dtype=torch.float32, device=gg.device)
    arr = (N.BnFullReq * 1)(N.BnFullReq(gg.data_ptr(), gb.data_ptr(), c, lo, hi, out.data_ptr()))
    check(N.lib().spngd_bn_full_moments_batched(context().h, 1, arr))
    return FullBnBlock(layer=layer, F=SymMatrix(2 * c, out))


def damp_bn_full(block: FullBnBlock, lam: float):
    """fisher.hpp:90 (fisher.cpp:248-253): F_inv = (F + lam I)^-1."""
    if not (lam > 0.0):
        raise NotPositiveDefinite("damp_bn_full: lambda must be > 0")
    block.F_inv, block.F_inv_dense = spd_inverse(block.F, lam, dense=True)
    block.lam = lam


def precondition_bn_full(block: FullBnBlock, grad_gamma: torch.Tensor, grad_beta: torch.Tensor):
    """fisher.cpp:278-296: (pg, pb) = F_inv (g_gamma, g_beta) interleaved."""
    c = grad_gamma.numel()
    if grad_beta.numel() != c or block.F is None or block.F.dim != 2 * c:
        raise ShapeMismatch("precondition_bn_full: gradient length mismatch")
    if block.F_inv_dense is None:
        raise StaleBeyondLimit("precondition_bn_full: block never inverted")
    grad = torch.cat([grad_gamma.reshape(-1), grad_beta.reshape(-1)]).float().contiguous()
    pg = torch.empty(c, dtype=torch.float32, device=grad.device)
    pb = torch.empty(c, dtype=torch.float32, device=grad.device)
    d = block.F_inv_dense
    req = N.BnFullUpdateReq(d.data_ptr(), d.stride(0), grad.data_ptr(), c, None, None, None, None, pg.data_ptr(),
                            pb.data_ptr())
    arr = (N.BnFullUpdateReq * 1)(req)
    check(N.lib().spngd_bn_full_solve_update_batched(context().h, 1, arr, 0.0, 0.0))
    return pg, pb


def bn_full_update(block: FullBnBlock, grad2c: torch.Tensor, gamma, beta, vgamma, vbeta, eta, momentum):
    """precondition_bn_full + the BN branch of ngd_step (fisher.cpp:346-359), in place."""
    c = grad2c.numel() // 2
    if block.F_inv_dense is None:
        raise StaleBeyondLimit("precondition_bn_full: block never inverted")
    d = block.F_inv_dense
    req = N.BnFullUpdateReq(d.data_ptr(), d.stride(0), grad2c.data_ptr(), c, gamma.data_ptr(), beta.data_ptr(),
                            vgamma.data_ptr(), vbeta.data_ptr(), None, None)
    arr = (N.BnFullUpdateReq * 1)(req)
    check(N.lib().spngd_bn_full_solve_update_batched(context().h, 1, arr, eta, momentum))


def precondition_bn(block: UnitBnBlock, grad_gamma: torch.Tensor, grad_beta: torch.Tensor, lam: float):
    """fisher.hpp:96-99: per channel (F_c + lam I)^-1 (g_gamma, g_beta)."""
    c = block.m3c.numel() // 3
    if grad_gamma.numel() != c or grad_beta.numel() != c:
        raise ShapeMismatch("precondition_bn: gradient length mismatch")
    grad = torch.cat([grad_gamma.reshape(-1), grad_beta.reshape(-1)]).float().contiguous()
    pg = torch.empty(c, dtype=torch.float32, device=grad.device)
    pb = torch.empty(c, dtype=torch.float32, device=grad.device)
    req = N.BnUpdateReq(block.m3c.data_ptr(), grad.data_ptr(), c, None, None, None, None, pg.data_ptr(),
                        pb.data_ptr())
    arr = (N.BnUpdateReq * 1)(req)
    check(N.lib().spngd_bn_solve_update_batched(context().h, 1, arr, lam, 0.0, 0.0))
    return pg, pb


def bn_update(block: UnitBnBlock, grad2c: torch.Tensor, gamma, beta, vgamma, vbeta, lam, eta, momentum):
    """Fused K7: 2x2 solve + BN branch of ngd_step (fisher.cpp:336-357), in place."""
    c = block.m3c.numel() // 3
    req = N.BnUpdateReq(block.m3c.data_ptr(), grad2c.data_ptr(), c, gamma.data_ptr(), beta.data_ptr(),
                        vgamma.data_ptr(), vbeta.data_ptr(), None, None)
    arr = (N.BnUpdateReq * 1)(req)
    check(N.lib().spngd_bn_solve_update_batched(context().h, 1, arr, lam, eta, momentum))


# ---- K8 + stale scheduler (stale.hpp) ------------------------------------------
def stat_distances(x: torch.Tensor, x1: Optional[torch.Tensor], x2: Optional[torch.Tensor], n: int,
                   kind: int = 0):
    """(||x-x1||_w, ||x1||_w, ||x-x2||_w, ||x2||_w) with packed weights (stale.hpp:23-51)."""
    out = torch.zeros(4, dtype=torch.float64, device=x.device)
    req = N.StatReq(x.data_ptr(), x1.data_ptr() if x1 is not None else None,
                    x2.data_ptr() if x2 is not None else None, n, kind, out.data_ptr())
    arr = (N.StatReq * 1)(req)
    check(N.lib().spngd_stat_distance_batched(context().h, 1, arr))
    return out.tolist()


REASONS = ["FirstBuild", "Dissimilar1", "Dissimilar2", "SimilarBoth"]


class StaleTracker:
    """stale.hpp:92-132: refresh exactly at t_X, then advance by the interval.
    Snapshots live on the device; similarity is computed by K8."""

    def __init__(self, id: str, alpha: float):
        self._h = N.lib().spngd_tracker_create(id.encode(), alpha)
        self.id, self.alpha = id, alpha
        self.x1 = self.x2 = None

    def __del__(self):
        try:
            N.lib().spngd_tracker_destroy(self._h)
        except Exception:
            pass

    def should_refresh(self, step: int) -> bool:
        return bool(N.lib().spngd_tracker_should_refresh(self._h, step))

    def on_refresh(self, x: torch.Tensor, step: int, n: Optional[int] = None, kind: int = 0):
        n = n if n is not None else x.numel()
        d = stat_distances(x, self.x1, self.x2, n, kind) if self.x1 is not None else [0, 0, 0, 0]
        interval, reason = C.c_int64(), C.c_int()
        check(N.lib().spngd_tracker_on_refresh(self._h, step, int(self.x1 is not None), d[0], d[1],
                                               int(self.x2 is not None), d[2], d[3],
                                               C.byref(interval), C.byref(reason)))
        self.x2, self.x1 = self.x1, x.clone()
        return interval.value, REASONS[reason.value]

    def _state(self):
        v = [C.c_int64() for _ in range(4)]
        N.lib().spngd_tracker_state(self._h, *[C.byref(x) for x in v])
        return [x.value for x in v]

    @property
    def t_x(self):
        return self._state()[0]

    @property
    def delta(self):
        return self._state()[1]

    @property
    def delta_prev(self):
        return self._state()[2]

    @property
    def refresh_count(self):
        return self._state()[3]

    def ever_built(self):
        return self.refresh_count > 0


# ---- communication ledger (include/spngd/dist.hpp:16-56, src/dist.cpp:42-133) ----
LEDGER_HEADER = "step,stage,collective,statistic_id,elements,bytes,skipped"  # dist.cpp:14-15
_COLLECTIVES = {0: "RSV_A", 1: "RSV_G_F_grad", 2: "AGV_params"}
_ID_KINDS = {0: "A", 1: "G", 2: "F", 3: "grad", 4: "w"}


@dataclass
class LedgerRow:  # dist.hpp:19-27
    step: int = 0
    stage: int = 0
    collective: str = ""
    statistic_id: str = ""
    elements: int = 0
    bytes: int = 0
    skipped: bool = False


def _row_from_c(r) -> LedgerRow:
    return LedgerRow(r.step, r.stage, _COLLECTIVES[r.collective], f"{_ID_KINDS[r.id_kind]}:{r.layer}",
                     r.elements, r.bytes, bool(r.skipped))


class CommLedger:  # dist.hpp:29-40
    def __init__(self, rows: Optional[List[LedgerRow]] = None):
        self._rows: List[LedgerRow] = list(rows or [])

    def record(self, step, stage, collective, id, elements, bytes, skipped):  # dist.cpp:42-46
        self._rows.append(LedgerRow(step, stage, collective, id, elements, bytes, bool(skipped)))

    def rows(self) -> List[LedgerRow]:
        return self._rows

    def size(self) -> int:
        return len(self._rows)

    def write_csv(self, f) -> None:  # dist.cpp:48-54
        f.write(LEDGER_HEADER + "\n")
        for r in self._rows:
            f.write(f"{r.step},{r.stage},{r.collective},{r.statistic_id},{r.elements},{r.bytes},"
                    f"{1 if r.skipped else 0}\n")


def ledger_step_rows(net_layers, world: int, step: int, due=None, elem_size: int = 4,
                     bn_full: bool = False, sgd: bool = False) -> List[LedgerRow]:
    """Rows one accumulate_microsteps call appends (dist.cpp:511-537, 646-662),
    computed by the native library's host planner (spngd_ledger_step_rows).
    `net_layers` are workloads.Layer; `due` per statistic in plan_statistics
    order (dist.cpp:256-269), None = all due."""
    from .step import layer_descs
    L = N.lib()
    arr = layer_descs(net_layers)
    d = None
    if due is not None:
        d = (C.c_ubyte * len(due))(*[1 if x else 0 for x in due])
    flags = (1 if bn_full else 0) | (2 if sgd else 0)  # SPNGD_LEDGER_BN_FULL | SPNGD_LEDGER_SGD
    n = L.spngd_ledger_step_rows(arr, len(net_layers), world, step, d, elem_size, flags, None, 0)
    if n < 0:
        check(int(-n))
    out = (N.LedgerRowC * max(n, 1))()
    L.spngd_ledger_step_rows(arr, len(net_layers), world, step, d, elem_size, flags, out, n)
    return [_row_from_c(out[i]) for i in range(n)]


def _is_statistic_id(i: str) -> bool:  # dist.cpp:22-24
    return i.startswith("A:") or i.startswith("G:") or i.startswith("F:")


@dataclass
class LedgerReport:  # dist.hpp:42-52
    steps: int = 0
    total_bytes: int = 0
    stat_bytes: int = 0
    grad_bytes: int = 0
    param_bytes: int = 0
    stat_bytes_every_step: int = 0
    reduction_rate: float = 1.0
    per_step_bytes: list = field(default_factory=list)


def ledger_report(rows) -> LedgerReport:  # dist.cpp:56-86
    if isinstance(rows, CommLedger):
        rows = rows.rows()
    rep = LedgerReport()
    steps, per_step, full = set(), {}, {}
    for r in rows:
        steps.add(r.step)
        per_step[r.step] = per_step.get(r.step, 0) + r.bytes
        rep.total_bytes += r.bytes
        if _is_statistic_id(r.statistic_id):
            if not r.skipped:
                rep.stat_bytes += r.bytes
                full[r.statistic_id] = r.bytes
        elif r.statistic_id.startswith("grad:"):
            rep.grad_bytes += r.bytes
        elif r.statistic_id.startswith("w:"):
            rep.param_bytes += r.bytes
    rep.steps = len(steps)
    for b in full.values():
        rep.stat_bytes_every_step += b * rep.steps
    rep.reduction_rate = 1.0 if rep.stat_bytes_every_step == 0 else rep.stat_bytes / rep.stat_bytes_every_step
    rep.per_step_bytes = sorted(per_step.items())
    return rep


def read_ledger_csv(f) -> List[LedgerRow]:  # dist.cpp:92-133
    lines = f.read().split("\n")
    if not lines or lines == [""]:
        raise ParseError("ledger: empty file")
    if lines[0].rstrip("\r") != LEDGER_HEADER:
        raise ParseError("ledger: unrecognized header")
    rows = []
    for lineno, line in enumerate(lines[1:], start=2):
        line = line.rstrip("\r")
        if not line:
            continue
        parts = line.split(",")
        if len(parts) != 7:
            raise ParseError(f"ledger: line {lineno}: expected 7 fields")
        try:
            rows.append(LedgerRow(int(parts[0]), int(parts[1]), parts[2], parts[3], int(parts[4]), int(parts[5]),
                                  int(parts[6]) != 0))
        except ValueError:
            raise ParseError(f"ledger: line {lineno}: malformed numeric field") from None
    return rows
