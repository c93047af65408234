"""Development diagnostic: repeated batched spd_inverse calls; counts failures
and large errors (race hunting)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2002_06015_b200 import spngd as P  # noqa: E402

n, nb, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
torch.backends.cuda.matmul.allow_tf32 = False
ms = []
for i in range(nb):
    g = torch.Generator(device="cuda").manual_seed(7 + i)
    x = torch.randn(n, n, device="cuda", generator=g) / n ** 0.5
    ms.append(x @ x.T + 0.5 * torch.eye(n, device="cuda"))
iu = torch.triu_indices(n, n, device="cuda")
syms = [P.SymMatrix(n, m[iu[0], iu[1]].contiguous()) for m in ms]
ref = None
fails, bad = 0, 0
for r in range(reps):
    try:
        outs = P.spd_inverse_batched(syms, 0.0158)
    except Exception:
        fails += 1
        continue
    cur = torch.stack([o.data for o in outs])
    if ref is None:
        ref = cur.clone()
    elif not torch.equal(cur, ref):
        bad += 1
print(f"n={n} x{nb}: {reps} calls, {fails} failures, {bad} results differing from the first call")
