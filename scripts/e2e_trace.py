"""Timeline of one spngd_opt_step_host step (ResNet-50 B=32, pinned host inputs):
SPNGD_STEP_TRACE=1 events per wave / inverse class / precondition part plus the
landing of the last H2D copy, against the step start.  Diagnosis of the e2e
tail (what runs after the PCIe stream ends)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2002_06015_b200 import _native as N  # noqa: E402
from paper_2002_06015_b200 import workloads as W  # noqa: E402
from paper_2002_06015_b200.spngd import check  # noqa: E402
from paper_2002_06015_b200.step import ALL_WEIGHTS, Optimizer  # noqa: E402

L = N.lib()
o = Optimizer(W.resnet50(), 32)
o.synth(1)
bufs = []
for li, w in o.input_buffers():
    p, _ = o.ptr(li, w)
    nbytes = o.numel(li, w) * 4
    hp = C.c_void_p()
    check(L.spngd_host_alloc(C.byref(hp), nbytes))
    check(L.spngd_copy(o.ctx, hp, C.c_void_p(p), nbytes))
    bufs.append(hp)
_, wcount = o.ptr(0, ALL_WEIGHTS)
hw_out = C.c_void_p()
check(L.spngd_host_alloc(C.byref(hw_out), wcount * 4))
ins = [(li, w, hp.value) for (li, w), hp in zip(o.input_buffers(), bufs)]
for s in range(4):
    o.step_host(s + 1, ins, hw_out.value)
    o.sync()
print(o.phase_ms())
o.close()
