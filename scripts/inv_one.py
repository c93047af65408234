"""One optimizer step on a single 3x3 512->512 conv layer (A = 4608^2): inverse-round profiling target."""
import sys
sys.path.insert(0, ".")
from paper_2002_06015_b200 import workloads as W
from paper_2002_06015_b200.step import Optimizer

opt = Optimizer([W.conv(512, 512, 3, 1, 7)], 32)
opt.synth(1)
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    opt.step(s + 1)
opt.sync()
print(opt.phase_ms())
opt.close()
