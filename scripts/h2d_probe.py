"""PCIe H2D probe: the e2e inputs of bench.py (ResNet-50 B=32) copied as one
pinned buffer vs as the per-input pieces spngd_opt_step_host issues, on one
stream and on two; CUDA events around each variant."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import Optimizer  # noqa: E402

opt = Optimizer(W.resnet50(), 32)
sizes = [opt.numel(li, w) * 4 for li, w in opt.input_buffers()]
opt.close()
total = sum(sizes)
host = torch.empty(total // 4, dtype=torch.float32).pin_memory()
dev = torch.empty(total // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(kind):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    cur = torch.cuda.current_stream()
    if kind == "one":
        dev.copy_(host, non_blocking=True)
    else:
        for st in (s1, s2):
            st.wait_stream(cur)
        off, k = 0, 0
        for b in sizes:
            n = b // 4
            st = s1 if (kind == "pieces" or k % 2 == 0) else s2
            with torch.cuda.stream(st):
                dev[off:off + n].copy_(host[off:off + n], non_blocking=True)
            off += n
            k += 1
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


out = {"bytes": total, "pieces": len(sizes)}
for kind in ("one", "pieces", "pieces_2streams"):
    ts = sorted(run(kind) for _ in range(5))
    out[kind] = {"ms": round(ts[2], 3), "GB/s": round(total / ts[2] / 1e6, 1)}
print(json.dumps(out))
