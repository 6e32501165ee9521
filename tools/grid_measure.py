"""Measure every valid tcgen05 config of a grid on given ResNet-50 N=32 bf16 layers with the tuner's
protocol (wpk_conv2d_measure, rotating cold copies) -- how close the GA's pick is to the grid's best.
usage: python tools/grid_measure.py CONFIGS_JSON LAYER [LAYER ...] > out.json
(GRID_KG_ONLY=1: only the K-group producers A_MODE 5 / 6)"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_2008_04567_b200 import Conv2dPlan

picked = json.load(open(sys.argv[1]))
out = {}
for name in sys.argv[2:]:
    L = next(l for l in workloads.resnet50(32) if l.name == name)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    res = []
    amodes = [5, 6] if os.environ.get("GRID_KG_ONLY") else [0, 4, 5, 6]
    for g in itertools.product([64, 128, 192, 256], [4, 6, 8], [1, 2], range(8), amodes, [1, 2], [128, 256]):
        g = list(g)
        if not plan.config_valid(1, g):
            continue
        plan.set_config(1, g)
        try:
            res.append((plan.measure(3, 7), g))
        except Exception:
            pass
    res.sort()
    pk = picked.get(name)
    pk_us = None
    if pk:
        plan.set_config(*pk)
        pk_us = plan.measure(3, 11)
    rank = sum(1 for us, _ in res if pk_us is not None and us < pk_us)
    out[name] = {"n_valid": len(res), "best": res[:8], "picked": pk, "picked_us": pk_us, "picked_rank": rank}
    print(name, len(res), "best", res[0], "picked", pk, pk_us, "rank", rank, file=sys.stderr, flush=True)
json.dump(out, sys.stdout, indent=1)
