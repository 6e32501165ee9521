"""One bench step (all 53 ResNet-50 convs, N=32 bf16 NHWC, per-conv buffers as bench.py) captured in
ONE CUDA graph and launched once -- for `ncu --graph-profiling graph`, which measures the whole graph
as one result (DRAM bytes of a step for bench.py's roofline.traffic).
    ncu --graph-profiling graph --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        python tools/step_graph_ncu.py CONFIGS_JSON"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
from paper_2008_04567_b200 import Conv2dPlan

cfgs = json.load(open(sys.argv[1]))
units = []
for i, L in enumerate(workloads.resnet50(32)):
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    plan.set_config(*cfgs[L.name])
    for c in range(L.count):
        x, w, b = workloads.generate(L, "bf16", "uniform", seed=workloads.config_seed(1, i) + 7919 * c)
        units.append((plan, x.permute(0, 2, 3, 1).contiguous().cuda(), w.permute(0, 2, 3, 1).contiguous().cuda(),
                      b.cuda(), torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda")))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for (p, x, w, b, y) in units:   # eager pass: weight packing, workspaces
        p.run(x, w, b, y, stream=s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for (p, x, w, b, y) in units:
        p.run(x, w, b, y, stream=s)
torch.cuda.synchronize()
with torch.cuda.stream(s):
    g.replay()
torch.cuda.synchronize()
print("replayed one step graph of", len(units), "convs")
