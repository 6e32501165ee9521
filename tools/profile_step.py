"""One bench step (all 53 ResNet-50 convs, N=32 bf16 NHWC) with the configs bench.py chose
(--configs-in JSON), for ncu launch lists:  ncu --metrics ... python tools/profile_step.py cfg.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan

cfgs = json.load(open(sys.argv[1])) if len(sys.argv) > 1 else {}
steps = int(os.environ.get("STEPS", "2"))
units = []
for i, L in enumerate(workloads.resnet50(32)):
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    if L.name in cfgs:
        plan.set_config(*cfgs[L.name])
    for c in range(L.count):
        x, w, b = workloads.generate(L, "bf16", "uniform", seed=workloads.config_seed(1, i) + 7919 * c)
        units.append((L.name, plan, x.permute(0, 2, 3, 1).contiguous().cuda(), w.permute(0, 2, 3, 1).contiguous().cuda(),
                      b.cuda(), torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda")))
for s in range(steps):
    for (nm, plan, x, w, b, y) in units:
        plan.run(x, w, b, y)
torch.cuda.synchronize()
print("layers", [u[0] for u in units])
