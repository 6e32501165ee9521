"""Which kernels the box's cuDNN runs for each ResNet-50 N=32 bf16 layer (fused conv+bias+ReLU on
channels_last), with their device durations from a CUPTI trace (torch.profiler), next to ours --
the kernel names carry cuDNN's tile shapes. usage: python tools/cudnn_kernels.py [CFG_JSON]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import workloads
from paper_2008_04567_b200 import Conv2dPlan
from paper_2008_04567_b200.selector import cudnn_conv_fn

cfgs = json.load(open(sys.argv[1])) if len(sys.argv) > 1 else {}
for i, L in enumerate(workloads.resnet50(int(os.environ.get("BATCH", "32")))):
    x, w, b = workloads.generate(L, "bf16", "uniform", seed=1)
    xd = x.permute(0, 2, 3, 1).contiguous().cuda(); wd = w.permute(0, 2, 3, 1).contiguous().cuda(); bd = b.cuda()
    f = cudnn_conv_fn(xd, wd, bd, L.stride, L.pad, L.dil, L.groups, "nhwc", "bf16", fused=True)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    if L.name in cfgs:
        plan.set_config(*cfgs[L.name])
    y = torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda")
    for _ in range(5):
        f(); plan.run(xd, wd, bd, y)
    torch.cuda.synchronize()
    flush = torch.empty(300 << 20, dtype=torch.uint8, device="cuda")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            flush.zero_(); f()
            flush.zero_(); plan.run(xd, wd, bd, y)
        torch.cuda.synchronize()
    ks = {}
    for e in prof.events():
        if str(e.device_type).endswith("CUDA") and "elementwise" not in e.name and "fill" not in e.name.lower() \
                and "Memset" not in e.name:
            ks.setdefault(e.name, []).append(e.time_range.end - e.time_range.start)
    print(f"== {L.name} (x{L.count})")
    for n, v in ks.items():
        print(f"   {sum(v) / len(v):7.2f} us  x{len(v)}  {n[:200]}")
