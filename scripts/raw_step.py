"""Two ResNet-50 B=32 steps with raw conv inputs (device im2col), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import Optimizer  # noqa: E402

opt = Optimizer(W.resnet50(), 32)
opt.enable_raw_inputs()
opt.synth(42)
for s in (1, 2):
    opt.step(s)
opt.sync()
opt.close()
print("ok")
