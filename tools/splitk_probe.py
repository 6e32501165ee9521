import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan
L = next(l for l in workloads.resnet50(32) if l.name == sys.argv[1])
genes = [int(v) for v in sys.argv[2:9]]
plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
plan.set_config(1, genes)
x, w, b = workloads.generate(L, "bf16", "uniform", seed=1)
xd = x.permute(0, 2, 3, 1).contiguous().cuda(); wd = w.permute(0, 2, 3, 1).contiguous().cuda(); bd = b.cuda()
y = torch.empty(plan.y_shape(), dtype=xd.dtype, device="cuda")
plan.run(xd, wd, bd, y); torch.cuda.synchronize()
ws = plan._ws
times = []
for i in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.run(xd, wd, bd, y); e1.record(); torch.cuda.synchronize()
    times.append(round(e0.elapsed_time(e1) * 1e3, 1))
print("times", times)
# counters live at the tail of the used workspace region: check all zero in the last few KB
tail = ws[-65536:].view(torch.int32)
print("nonzero int32 in ws tail:", int((tail != 0).sum()))
