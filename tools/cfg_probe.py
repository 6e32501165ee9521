"""Time one layer under a list of configs with the tuner's protocol (wpk_conv2d_measure: L2 evicted,
globaltimer-bracketed reps, interquartile mean).  usage:
    python tools/cfg_probe.py LAYER "g0,g1,...,g6" ["..."]   (NET / BATCH / DT env as elsewhere)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_2008_04567_b200 import Conv2dPlan

name = sys.argv[1]
net = os.environ.get("NET", "resnet50")
batch = int(os.environ.get("BATCH", {"resnet50": "32", "vgg16": "64", "mobilenet_v2": "1"}[net]))
dt = os.environ.get("DT", "bf16")
L = next(l for l in getattr(workloads, net)(batch) if l.name == name)
plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype=dt)
fl = 2 * L.n * L.k * plan.p * plan.q * (L.c // L.groups) * L.r * L.s
tag = os.environ.get("TAG", "")
for c in sys.argv[2:]:
    g = [int(v) for v in c.split(",")]
    if not plan.config_valid(1, g):
        print(f"{tag} {name} {g} invalid", flush=True)
        continue
    plan.set_config(1, g)
    us = plan.measure(3, 21, True)
    print(f"{tag} {name} {str(g):36s} {us:8.2f} us {fl / us / 1e6:7.1f} TF/s", flush=True)
