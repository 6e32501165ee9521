"""NEXT-2 measurement: the paper's JIT code generation against the precompiled
template of the same genes (SIMT family) and the exact-fp32 implicit GEMM (GEMM32), per layer of
the paper's per-convolution workload (ResNet-18 at N=1, fp32, NCHW as in PAPER.md:142), each GA-tuned
with the same budget; tuning wall time with NVRTC compile time (multi-threaded, cached) included.
Timing: the tuner's protocol (wpk_conv2d_measure). Writes JSON + a markdown table.

    python tools/jit_suite.py OUT_PREFIX [--net resnet18] [--batch 1] [--budget 48]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
from paper_2008_04567_b200 import Conv2dPlan, _lib as L_, selector

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--net", default="resnet18")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--budget", type=int, default=48)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--layout", default="nchw")
a = ap.parse_args()

rows = []
for i, L in enumerate(getattr(workloads, a.net)(a.batch)):
    fl = 2 * L.n * L.k * ((L.h + 2 * L.pad - L.dil * (L.r - 1) - 1) // L.stride + 1) * \
        ((L.w + 2 * L.pad - L.dil * (L.s - 1) - 1) // L.stride + 1) * (L.c // L.groups) * L.r * L.s
    row = {"layer": L.name, "gflop": fl / 1e9}
    for fam in ["simt", "jit", "gemm32"]:
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout=a.layout,
                          dtype=a.dtype)
        if fam == "gemm32" and a.dtype != "f32":
            continue
        s0 = L_.jit_stats()
        t0 = time.perf_counter()
        res = plan.tune("ga", a.budget, seed=i, family=fam, finalists=2)
        secs = time.perf_counter() - t0
        s1 = L_.jit_stats()
        us = plan.measure(3, 21, True)
        row[fam] = {"us": us, "genes": res.genes, "tune_s": secs, "measured": res.measured,
                    "compiles": s1["compiles"] - s0["compiles"], "compile_s": s1["compile_seconds"] - s0["compile_seconds"]}
    x, w, b = workloads.generate(L, a.dtype, "uniform", seed=7)
    xd, wd, bd = x.cuda(), w.cuda(), b.cuda()
    f = selector.cudnn_conv_fn(xd, wd, bd, L.stride, L.pad, L.dil, L.groups, a.layout, a.dtype, fused=False)
    row["cudnn_us"] = selector.time_fn(f)
    rows.append(row)
    print(json.dumps(row), flush=True)

json.dump(rows, open(a.out + ".json", "w"), indent=1)
with open(a.out + ".md", "w") as fp:
    fp.write(f"# JIT family vs precompiled template ({a.net} N={a.batch}, {a.dtype}, {a.layout}; GA budget {a.budget} "
             "per family per layer; tuner timing protocol; cuDNN: median of 11 flushed event-timed runs)\n\n")
    fp.write("| layer | GFLOP | SIMT us | JIT us | JIT/SIMT speed-up | GEMM32 us | cuDNN us | JIT tune s (compile s, compiles) | SIMT tune s |\n|---|---|---|---|---|---|---|---|---|\n")
    tot = {"simt": 0.0, "jit": 0.0, "gemm32": 0.0, "cudnn": 0.0, "jt": 0.0, "jc": 0.0, "st": 0.0}
    for r in rows:
        g = r.get("gemm32", {}).get("us", float("nan"))
        fp.write(f"| {r['layer']} | {r['gflop']:.3f} | {r['simt']['us']:.1f} | {r['jit']['us']:.1f} | "
                 f"{r['simt']['us'] / r['jit']['us']:.2f} | {g:.1f} | {r['cudnn_us']:.1f} | "
                 f"{r['jit']['tune_s']:.1f} ({r['jit']['compile_s']:.1f}, {r['jit']['compiles']}) | {r['simt']['tune_s']:.1f} |\n")
        tot["simt"] += r["simt"]["us"]; tot["jit"] += r["jit"]["us"]; tot["cudnn"] += r["cudnn_us"]
        tot["gemm32"] += r.get("gemm32", {}).get("us", 0.0)
        tot["jt"] += r["jit"]["tune_s"]; tot["jc"] += r["jit"]["compile_s"]; tot["st"] += r["simt"]["tune_s"]
    fp.write(f"| **sum** | | {tot['simt']:.1f} | {tot['jit']:.1f} | {tot['simt'] / tot['jit']:.2f} | {tot['gemm32']:.1f} | "
             f"{tot['cudnn']:.1f} | {tot['jt']:.1f} ({tot['jc']:.1f}) | {tot['st']:.1f} |\n")
print(open(a.out + ".md").read())
