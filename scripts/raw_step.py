"""One phase-serial ResNet-50 B=32 step with raw conv inputs, for ncu:
--implicit gathers the im2col operand inside the GEMMs (no capture),
otherwise im2col_kernel expands it first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.step import Optimizer  # noqa: E402

opt = Optimizer(W.resnet50(), 32)
opt.set_overlap(False)
opt.enable_raw_inputs(implicit="--implicit" in sys.argv)
opt.synth(42)
opt.step(1)
opt.sync()
print(opt.phase_ms())
opt.close()
