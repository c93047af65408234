"""Accuracy diagnostics of the GPU path vs the fp64 oracle (development tool).

Separates error sources on an ill-conditioned post-ReLU factor: factor
construction, the damped inverse, fp32 LAPACK as a yardstick, preconditioning
and the fused update.
"""
import sys

import numpy as np
import scipy.linalg as sl
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2002_06015_b200 as P  # noqa: E402


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def conv_capture(batch, c, h, w, k, stride, pad, seed):
    ctx = P.context()
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    x = torch.empty(batch * c * k * k * ho * wo, device="cuda")
    P.check(P._native.lib().spngd_synth_conv_capture(ctx.h, x.data_ptr(), batch, c, h, w, k, stride, pad,
                                                     seed, 1, 1.0, 0.0))
    torch.cuda.synchronize()
    return x, c * k * k, ho * wo


def case(batch, c, h, w, k, s, p, g, seed=77, lam=2.5e-4):
    x, a, hw = conv_capture(batch, c, h, w, k, s, p, seed)
    gr = torch.randn(batch * g * hw, device="cuda", generator=torch.Generator("cuda").manual_seed(seed)) / np.sqrt(batch * hw)
    A = P.factor_sym(x, a, hw, 1, 0, batch, 1.0 / (batch * hw))
    G = P.factor_sym(gr, g, hw, 1, 0, batch, 1.0 / batch)
    An = O.factor_A(x.cpu().numpy(), True, a, hw, 0, batch)
    Gn = O.factor_G(gr.cpu().numpy(), True, g, hw, 0, batch)
    print(f"case a={a} g={g} K={batch * hw}")
    print(f"  factor A rel {O.rel_frob_distance(A.cpu().numpy().astype(np.float64), An, a):.2e}  "
          f"G rel {O.rel_frob_distance(G.cpu().numpy().astype(np.float64), Gn, g):.2e}")
    # inverse on identical (our fp32) factors
    A64 = A.cpu().numpy().astype(np.float64)
    G64 = G.cpu().numpy().astype(np.float64)
    pi, Ai, Gi = O.damp_and_invert(A64, G64, a, g, lam)
    Ad = O.unpack(A64, a) + pi * np.sqrt(lam) * np.eye(a)
    print(f"  pi {pi:.4f} damping {pi * np.sqrt(lam):.4e} cond(A+dI) {np.linalg.cond(Ad):.3e}")
    b = P.KroneckerBlock(A=P.SymMatrix(a, A), G=P.SymMatrix(g, G))
    P.damp_and_invert(b, lam)
    ea = O.rel_frob_distance(b.A_inv.data.cpu().numpy().astype(np.float64), Ai, a)
    eg = O.rel_frob_distance(b.G_inv.data.cpu().numpy().astype(np.float64), Gi, g)
    print(f"  GPU inverse rel: A {ea:.2e}  G {eg:.2e}")
    Ad32 = Ad.astype(np.float32)
    c32 = sl.cho_factor(Ad32)
    inv32 = sl.cho_solve(c32, np.eye(a, dtype=np.float32))
    print(f"  LAPACK fp32 (spotrf+spotrs) A inverse rel: {relf(inv32, O.unpack(Ai, a)):.2e}")
    rng = np.random.default_rng(1)
    dW = (rng.standard_normal((g, a)) / np.sqrt(a)).astype(np.float32)
    Pg = P.precondition(b, torch.tensor(dW, device="cuda")).cpu().numpy()
    Pw = O.kron_matvec(Gi, Ai, g, a, dW.astype(np.float64))
    print(f"  precondition rel {relf(Pg, Pw):.2e}  |P|/|dW| {np.linalg.norm(Pw) / np.linalg.norm(dW):.3e}")
    # P with exact (oracle) inverses run through numpy fp32 for reference
    W = (rng.standard_normal((g, a)) * np.sqrt(2 / a)).astype(np.float32)
    V = (0.01 * rng.standard_normal((g, a))).astype(np.float32)
    Wt, Vt = torch.tensor(W, device="cuda"), torch.tensor(V, device="cuda")
    P.kron_update(b, torch.tensor(dW, device="cuda"), Wt, Vt, 1.25e-2, 0.993, rescale=True)
    nw, nv = O.ngd_update(W, Pw, V, 1.25e-2, 0.993)
    rw, rv = O.rescale(nw, W, g)
    print(f"  |eta P|/|W| {1.25e-2 * np.linalg.norm(Pw) / np.linalg.norm(W):.3e}")
    print(f"  updated W rel {relf(Wt.cpu().numpy(), rw.reshape(g, a)):.2e}  V rel {relf(Vt.cpu().numpy(), rv.reshape(g, a)):.2e}")


if __name__ == "__main__":
    case(4, 64, 14, 14, 3, 2, 1, 64)
    case(32, 64, 14, 14, 3, 2, 1, 64)
    case(32, 512, 7, 7, 3, 1, 1, 512)
