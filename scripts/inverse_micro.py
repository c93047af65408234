"""Inverse-phase time per matrix size class, in isolation (development tool)."""
import sys
sys.path.insert(0, ".")
from paper_2002_06015_b200 import workloads as W
from paper_2002_06015_b200.step import Optimizer


def run(name, layers, batch=32, reps=3):
    opt = Optimizer(layers, batch)
    opt.synth(1)
    for s in range(2):
        opt.step(s + 1)
    t = []
    for s in range(reps):
        opt.step(s + 3)
        t.append(opt.phase_ms())
    ms = sorted(x["inverse"] for x in t)[len(t) // 2]
    print(f"{name}: inverse {ms:.3f} ms   precond {t[-1]['precondition_update']:.3f}", flush=True)
    opt.close()


run("3x 4608 (+3x 512 G)", [W.conv(512, 512, 3, 1, 7)] * 3)
run("1x 4608 (+1x 512 G)", [W.conv(512, 512, 3, 1, 7)])
run("6x 2304 (+6x 256 G)", [W.conv(256, 256, 3, 1, 14)] * 6)
run("1x 2304", [W.conv(256, 256, 3, 1, 14)])
run("1x 1152", [W.conv(128, 128, 3, 1, 28)])
run("1x 576", [W.conv(64, 64, 3, 1, 56)])
run("1x 128 (leaf only)", [W.conv(128, 128, 1, 1, 28)])
run("resnet50", W.resnet50())
