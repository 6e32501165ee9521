"""Time every unique layer of a workload in given configs with the tuner's protocol
(wpk_conv2d_measure: globaltimer-bracketed reps, L2 evicted before each, interquartile mean).
Quick A/B of kernel changes / environment knobs across processes:
    WPK_L2PF=0 python tools/ab_layers.py CFG_JSON [--net resnet50 --batch 32 --dtype bf16] > a.json
CFG_JSON maps layer name -> [family, genes] (bench.py --configs-out); missing layers use the default."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan

ap = argparse.ArgumentParser()
ap.add_argument("cfg", nargs="?")
ap.add_argument("--net", default="resnet50")
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--reps", type=int, default=21)
ap.add_argument("--layers", default=None)
ap.add_argument("--tag", default=os.environ.get("TAG", ""))
a = ap.parse_args()
cfgs = json.load(open(a.cfg)) if a.cfg else {}
if "layers" in cfgs and isinstance(cfgs["layers"], dict):
    cfgs = cfgs["layers"]
out = {}
for L in getattr(workloads, a.net)(a.batch):
    if a.layers and L.name not in a.layers.split(","):
        continue
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype=a.dtype)
    if L.name in cfgs:
        plan.set_config(*cfgs[L.name])
    us = plan.measure(3, a.reps, True)
    fl = 2 * L.n * L.k * plan.p * plan.q * (L.c // L.groups) * L.r * L.s
    out[L.name] = {"us": us, "count": L.count, "tflops": fl / us / 1e6, "config": plan.config}
    print(f"{a.tag} {L.name:10s} {us:8.2f} us {fl / us / 1e6:7.1f} TF/s {plan.config}", flush=True)
tot = sum(v["us"] * v["count"] for v in out.values())
print(f"{a.tag} SUM {tot:.1f} us", flush=True)
json.dump(out, sys.stdout if False else open(os.environ.get("AB_OUT", "/dev/null"), "w"))
