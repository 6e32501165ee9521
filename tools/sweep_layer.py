"""Time one ResNet-50 layer (N=32 bf16 NHWC) under a list of UMMA configs (or every valid config
of a small grid). Prints median us (L2 flushed before each rep) -- quick A/B for kernel work.
usage: python tools/sweep_layer.py LAYER [genes ...]  |  LAYER grid"""
import sys, os, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan
from paper_2008_04567_b200.selector import time_fn

name = sys.argv[1]
net = os.environ.get("NET", "resnet50")
dt = os.environ.get("DT", "bf16")
batch = int(os.environ.get("BATCH", {"resnet50": "32", "vgg16": "64", "mobilenet_v2": "1"}[net]))
L = next(l for l in getattr(workloads, net)(batch) if l.name == name)
plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype=dt)
x, w, b = workloads.generate(L, dt, "uniform", seed=1)
xd = x.permute(0, 2, 3, 1).contiguous().cuda(); wd = w.permute(0, 2, 3, 1).contiguous().cuda(); bd = b.cuda()
y = torch.empty(plan.y_shape(), dtype=xd.dtype, device="cuda")
fl = 2 * L.n * L.k * plan.p * plan.q * (L.c // L.groups) * L.r * L.s
if len(sys.argv) > 2 and sys.argv[2] == "grid":
    cfgs = [list(c) for c in itertools.product([64, 128, 256], [3, 4, 6], [1], [0, 1], [0], [1, 2], [128, 256])]
elif len(sys.argv) > 2 and sys.argv[2] == "grid2":   # wider: pairs, 4 accumulators, split-K
    cfgs = [list(c) for c in itertools.product([64, 128, 192, 256], [3, 4, 6], [1, 2], [0, 1, 2, 3], [0],
                                               [1, 2, 4], [128, 256])]
elif len(sys.argv) > 2:
    vals = [int(v) for v in sys.argv[2:]]
    cfgs = [vals[i:i + 7] for i in range(0, len(vals), 7)]
else:
    cfgs = [plan.config[1]]
print(name, "default", plan.config)
for g in cfgs:
    if not plan.config_valid(plan.config[0], g):
        continue
    plan.set_config(plan.config[0], g)
    try:
        if os.environ.get("B2B"):   # 30 back-to-back runs between two events (warm L2, 0.1-us resolution)
            for _ in range(3):
                plan.run(xd, wd, bd, y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(30):
                plan.run(xd, wd, bd, y)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e3 / 30
        else:
            t = time_fn(lambda: plan.run(xd, wd, bd, y), warmup=3, reps=15)
        torch.cuda.synchronize()
    except Exception as e:
        print(g, "FAILED", e)
        raise
    print(f"{str(g):40s} {t:8.1f} us {fl / t / 1e6:8.1f} TF/s", flush=True)
