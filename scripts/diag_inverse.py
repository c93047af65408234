"""Development diagnostic: spd_inverse on rank-deficient ReLU factors
(X X^T / K, K = n/2) -- accuracy / pivot failures by n and damping."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2002_06015_b200 import spngd as P  # noqa: E402


def packed(m):
    n = m.shape[0]
    iu = torch.triu_indices(n, n, device=m.device)
    return m[iu[0], iu[1]].contiguous().float()


for n in [int(a) for a in sys.argv[1:]]:
    g = torch.Generator(device="cuda").manual_seed(1000 * n)
    k = n // 2
    x = torch.relu(torch.randn(n, k, device="cuda", generator=g))
    torch.backends.cuda.matmul.allow_tf32 = False
    m = x @ x.T / k
    for damp in (0.0158, 0.05, 0.2):
        md = m.double() + damp * torch.eye(n, device="cuda", dtype=torch.float64)
        L = torch.linalg.cholesky(md)
        piv = torch.diagonal(L) ** 2
        try:
            out = P.spd_inverse(P.SymMatrix(n, packed(m)), damp)
            iu = torch.triu_indices(n, n, device="cuda")
            got = torch.zeros(n, n, dtype=torch.float64, device="cuda")
            got[iu[0], iu[1]] = out.data.double()
            got = got + got.T - torch.diag(torch.diag(got))
            want = torch.linalg.inv(md.cpu()).cuda()
            err = float(torch.linalg.norm(got - want) / torch.linalg.norm(want))
            print(f"n={n} damp={damp}: min fp64 pivot {float(piv.min()):.3e} at {int(piv.argmin())}, rel err {err:.3e}")
        except Exception as e:
            print(f"n={n} damp={damp}: min fp64 pivot {float(piv.min()):.3e} at {int(piv.argmin())}, FAILED {type(e).__name__}")


def batched(n, nb, seed0=0):
    torch.backends.cuda.matmul.allow_tf32 = False
    ms = []
    for i in range(nb):
        g = torch.Generator(device="cuda").manual_seed(1000 * n + i + seed0)
        x = torch.relu(torch.randn(n, n // 2, device="cuda", generator=g))
        ms.append(x @ x.T / (n // 2))
    damp = 0.0158
    try:
        outs = P.spd_inverse_batched([P.SymMatrix(n, packed(m)) for m in ms], damp)
    except Exception as e:
        print(f"batched n={n} x{nb}: FAILED {type(e).__name__}")
        for i, m in enumerate(ms):
            try:
                P.spd_inverse(P.SymMatrix(n, packed(m)), damp)
                print(f"   matrix {i} alone: ok")
            except Exception as e2:
                print(f"   matrix {i} alone: FAILED {type(e2).__name__}")
        return
    iu = torch.triu_indices(n, n, device="cuda")
    for i, (m, o) in enumerate(zip(ms, outs)):
        got = torch.zeros(n, n, dtype=torch.float64, device="cuda")
        got[iu[0], iu[1]] = o.data.double()
        got = got + got.T - torch.diag(torch.diag(got))
        want = torch.linalg.inv((m.double() + damp * torch.eye(n, device="cuda", dtype=torch.float64)).cpu()).cuda()
        print(f"batched n={n} x{nb} matrix {i}: rel err {float(torch.linalg.norm(got - want) / torch.linalg.norm(want)):.3e}")


if len(sys.argv) == 1 or True:
    for n, nb in ((2048, 4), (2048, 2), (1024, 4), (512, 3)):
        batched(n, nb)
