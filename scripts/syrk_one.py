"""The ResNet-50 B=32 factor SYRK alone (phase-serial optimizer step, 3 steps) -- ncu target."""
import sys
sys.path.insert(0, ".")
from paper_2002_06015_b200 import workloads as W
from paper_2002_06015_b200.step import Optimizer

opt = Optimizer(W.resnet50(), 32)
opt.set_overlap(False)
opt.synth(1)
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    opt.step(s + 1)
opt.sync()
print(opt.phase_ms())
opt.close()
