"""Measure split-K configs (SPLIT_K 2-16) of the deep ResNet-50 N=32 layers with the tuner protocol."""
import itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_2008_04567_b200 import Conv2dPlan
for name in ['s5b1.c2', 's5b0.c2', 's5b1.c1', 's4b1.c2']:
    L = next(l for l in workloads.resnet50(32) if l.name == name)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    res = []
    for g in itertools.product([64, 128, 256], [4, 6, 8], [2, 4, 8, 16], [0, 1, 2, 3], [0, 4, 5, 6], [1, 2], [128, 256]):
        g = list(g)
        if not plan.config_valid(1, g):
            continue
        plan.set_config(1, g)
        try:
            res.append((plan.measure(3, 7), g))
        except Exception as e:
            pass
    res.sort()
    print(name, len(res), res[:5], flush=True)
