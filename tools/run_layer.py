"""Run one ResNet-50 (N=32 bf16 NHWC) layer a few times with a given config -- a short command
for ncu captures:  python tools/run_layer.py s4b1.c2 [genes...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan

name = sys.argv[1]
reps = int(os.environ.get("REPS", "3"))
net = os.environ.get("NET", "resnet50")
batch = int(os.environ.get("BATCH", {"resnet50": "32", "vgg16": "64", "mobilenet_v2": "1"}.get(net, "8")))
L = next(l for l in getattr(workloads, net)(batch) if l.name == name)
plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc",
                  dtype=os.environ.get("DT", "bf16"))
if len(sys.argv) > 2:
    plan.set_config(1, [int(v) for v in sys.argv[2:9]])
elif os.environ.get("CFG_JSON"):   # the layer's config from a bench --configs-out file
    import json
    plan.set_config(*json.load(open(os.environ["CFG_JSON"]))[name])
x, w, b = workloads.generate(L, plan.dtype, "uniform", seed=1)
xd = x.permute(0, 2, 3, 1).contiguous().cuda(); wd = w.permute(0, 2, 3, 1).contiguous().cuda(); bd = b.cuda()
y = torch.empty(plan.y_shape(), dtype=xd.dtype, device="cuda")
for _ in range(reps):
    plan.run(xd, wd, bd, y)
torch.cuda.synchronize()
print(name, plan.config)
