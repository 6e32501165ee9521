"""Run one fused depthwise+pointwise plan (for ncu / timeline captures): python tools/run_dwpw.py
N C HW STRIDE K [genes as comma list] -- MobileNet-like 3x3 pad 1, bf16, uniform inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
from paper_2008_04567_b200 import DwPwPlan


def main():
    n, c, hw, st, k = (int(v) for v in sys.argv[1:6])
    plan = DwPwPlan(n, c, hw, hw, k, 3, 3, st, 1, 1, dtype="bf16")
    if len(sys.argv) > 6:
        plan.set_config(1, [int(v) for v in sys.argv[6].split(",")])
    L = workloads.ConvLayer("dw", n, c, hw, hw, c, 3, 3, st, 1, 1, c)
    x, w_dw, b_dw = workloads.generate(L, "bf16", "uniform", seed=1)
    w_pw = torch.randn(k, c).to(torch.bfloat16).cuda()
    b_pw = torch.zeros(k, dtype=torch.bfloat16).cuda()
    xd = x.permute(0, 2, 3, 1).contiguous().cuda()
    args = (xd, w_dw.contiguous().cuda(), b_dw.cuda(), w_pw, b_pw)
    for _ in range(3):
        plan.run(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.run(*args)
    e1.record()
    torch.cuda.synchronize()
    print("config", plan.config, "us/launch (warm, back to back)", e0.elapsed_time(e1) * 100)


if __name__ == "__main__":
    main()
