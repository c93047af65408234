"""Factor-GEMM timing through the Optimizer's device events (development tool)."""
import sys
sys.path.insert(0, ".")
from paper_2002_06015_b200 import workloads as W
from paper_2002_06015_b200.step import Optimizer

def run(name, layers, batch, reps=5):
    opt = Optimizer(layers, batch)
    opt.synth(1)
    for s in range(2):
        opt.step(s + 1)
    t = []
    for s in range(reps):
        opt.step(s + 3)
        t.append(opt.phase_ms()["factor_gemm"])
    ff, _, _ = W.flops(layers, batch)
    ms = sorted(t)[len(t) // 2]
    print(f"{name}: factor GEMM {ms:.3f} ms  {ff / ms / 1e9:.1f} TF/s algorithmic", flush=True)
    opt.close()

run("a=4096 K=8192", [W.conv(4096, 32, 1, 1, 64)], 2)
run("a=2048 K=16384", [W.conv(2048, 32, 1, 1, 128)], 1)
run("a=1024 K=65536", [W.conv(1024, 32, 1, 1, 256)], 1)
run("resnet50 b32", W.resnet50(), 32, reps=3)
