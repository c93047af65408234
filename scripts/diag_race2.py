"""Development diagnostic: alternate batched spd_inverse sizes; results must be
identical to the first call of each size."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2002_06015_b200 import spngd as P  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
sizes = [int(a) for a in sys.argv[2:]] or [512, 1024, 256, 2048]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
data = {}
for n in sizes:
    ms = []
    for i in range(4):
        g = torch.Generator(device="cuda").manual_seed(7 + i + n)
        x = torch.randn(n, n, device="cuda", generator=g) / n ** 0.5
        ms.append(x @ x.T + 0.5 * torch.eye(n, device="cuda"))
    iu = torch.triu_indices(n, n, device="cuda")
    data[n] = [P.SymMatrix(n, m[iu[0], iu[1]].contiguous()) for m in ms]
torch.cuda.synchronize()
ref, fails, bad = {}, 0, 0
for r in range(reps):
    for n in sizes:
        try:
            outs = P.spd_inverse_batched(data[n], 0.0158)
        except Exception:
            fails += 1
            print(f"rep {r} n={n}: FAILED")
            continue
        cur = torch.stack([o.data for o in outs])
        if n not in ref:
            ref[n] = cur.clone()
        elif not torch.equal(cur, ref[n]):
            bad += 1
            print(f"rep {r} n={n}: differs, max abs diff {float((cur - ref[n]).abs().max()):.3e}")
print(f"sizes {sizes}: {reps} rounds, {fails} failures, {bad} differing")
