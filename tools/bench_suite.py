"""Supplementary per-layer measurements for the other BASELINE.json configs (not the bench.py
contract line): each unique layer is tuned (GA, or RL for VGG-16 as configs[2] says), then timed
with the selector protocol (3 warm-ups, 11 event-timed reps, read-based L2 flush, median) next to
the same-box cuDNN. Writes JSON + a markdown table.

    python tools/bench_suite.py OUT_PREFIX [--nets vgg16,mobilenet_v2,resnet50_n1,resnet50_tf32] [--budget 32]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
from paper_2008_04567_b200 import Conv2dPlan, selector

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) \
    else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}

NETS = {
    "vgg16": (lambda: workloads.vgg16(64), "f16", "rl"),
    "mobilenet_v2": (lambda: workloads.mobilenet_v2(1), "bf16", "ga"),
    "mobilenet_v2_n32": (lambda: workloads.mobilenet_v2(32), "bf16", "ga"),
    "mobilenet_v2_n128": (lambda: workloads.mobilenet_v2(128), "bf16", "ga"),
    "resnet50_n1": (lambda: workloads.resnet50(1), "bf16", "ga"),
    "resnet18_n1": (lambda: workloads.resnet18(1), "bf16", "ga"),
    "table1_n1": (lambda: workloads.table1(1), "bf16", "rl"),
    "resnet50_tf32": (lambda: workloads.resnet50(32), "tf32", "ga"),
    "resnet50_f32_n8": (lambda: workloads.resnet50(8), "f32", "ga"),   # exact-fp32 CUDA-core path
    "resnext50_grouped_bf16_n8": (lambda: workloads.resnext50_grouped(8), "bf16", "ga"),   # general groups (SIMT)
    "resnext50_grouped_f32_n8": (lambda: workloads.resnext50_grouped(8), "f32", "ga"),
    # NEXT-4: e4m3 operands / bf16 output (tcgen05 kind::f8f6f4). cuDNN has no fp8 conv through torch:
    # the competitor columns are cuDNN bf16 and our own tuned bf16 kernel on the same (rounded) inputs
    "resnet50_fp8": (lambda: workloads.resnet50(32), "fp8", "ga"),
    # NEXT-4 grouped convs on the tensor cores (gconv_tc.cu): every groups-per-tile choice measured
    "resnext50_grouped_tc_bf16_n8": (lambda: workloads.resnext50_grouped(8), "bf16", "tc_sweep"),
}


def _fp8_row(i, L, plan, res, budget):
    """Own e4m3 kernel vs own bf16 kernel vs cuDNN bf16, all with the selector protocol."""
    x, w, b = workloads.generate(L, "fp8", "uniform", seed=workloads.config_seed(2, i))
    xd = x.permute(0, 2, 3, 1).contiguous().cuda()
    wd = w.permute(0, 2, 3, 1).contiguous().cuda()
    bd = b.cuda()
    yd = torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda")
    xs = selector.rotating_copies(xd, yd.numel() * yd.element_size())
    ys = [yd] + [torch.empty_like(yd) for _ in xs[1:]]
    own = selector.time_rotating([lambda i=i: plan.run(xs[i], wd, bd, ys[i]) for i in range(len(xs))])
    # the same layer in bf16 (own tuned kernel, cuDNN) on the e4m3 values widened to bf16 (exact)
    p16 = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype="bf16")
    p16.tune("ga", budget, seed=i)
    x16, w16 = xd.to(torch.bfloat16), wd.to(torch.bfloat16)
    sel = selector.select(p16, x16, w16, bd, torch.empty_like(yd), L.stride, L.pad, L.dil, L.groups)
    return own, sel, xd, wd, bd, yd


def run_net(name, budget):
    make, dtype, search = NETS[name]
    layers = make()
    rows = []
    t_tune = 0.0
    for i, L in enumerate(layers):
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc",
                          dtype=dtype)
        fam = plan.config[0]
        t0 = time.perf_counter()
        kw = dict(seed=i)
        if search == "rl":
            kw.update(rl_envs=4, rl_horizon=16)
        if search == "tc_sweep":   # the tcgen05 grouped kernel: its only gene is BLOCK_N
            best = None
            for bn in (16, 32, 64, 96, 128, 192, 256):
                genes = [bn, 2, 1, 0, 1, 1, 128]
                if plan.config_valid(1, genes):
                    plan.set_config(1, genes)
                    us = plan.measure()
                    if best is None or us < best[0]:
                        best = (us, genes)
            plan.set_config(1, best[1])
            from paper_2008_04567_b200.conv import TuneResult
            res = TuneResult(1, best[1], best[0], 7, 1, 0.0)
        else:
            res = plan.tune(search if fam != 2 else "ga", budget, **kw)
        t_tune += time.perf_counter() - t0
        extra = {}
        if dtype == "fp8":
            own, sel16, xd, wd, bd, yd = _fp8_row(i, L, plan, res, budget)
            sel = selector.Selection(own, sel16.cudnn_us, sel16.cudnn_variant + " (bf16)",
                                     "wpk" if own <= sel16.cudnn_us else "cudnn")
            extra = {"bf16_wpk_us": sel16.own_us, "fp8_speedup_vs_own_bf16": sel16.own_us / own}
        else:
            x, w, b = workloads.generate(L, dtype, "uniform", seed=workloads.config_seed(2, i))
            xd = x.permute(0, 2, 3, 1).contiguous().cuda()
            wd = w.permute(0, 2, 3, 1).contiguous().cuda()
            bd = b.cuda()
            yd = torch.empty(plan.y_shape(), dtype=xd.dtype, device="cuda")
            sel = selector.select(plan, xd, wd, bd, yd, L.stride, L.pad, L.dil, L.groups)
        fl = 2 * L.n * L.k * plan.p * plan.q * (L.c // L.groups) * L.r * L.s
        by = (xd.element_size() * (xd.numel() + wd.numel()) + yd.element_size() * (bd.numel() + yd.numel()))
        # f32 runs on the CUDA cores: 148 SMs x 128 FP32 lanes x 2 flop/FMA x max SM clock (74.4 TF/s);
        # tf32 = half and fp8 = twice the measured bf16 figure (the guide's nominal ratios)
        peak_tf = (148 * 128 * 2 * PEAKS["sm_max_mhz"] / 1e6 if dtype == "f32"
                   else PEAKS["bf16_tflops"] * {"tf32": 0.5, "fp8": 2.0}.get(dtype, 1.0))
        rows.append({"layer": L.name, "count": L.count, "n": L.n, "dtype": dtype, "family": res.family, **extra,
                     "config": res.genes, "wpk_us": sel.own_us, "cudnn_us": sel.cudnn_us,
                     "cudnn_variant": sel.cudnn_variant, "speedup_vs_cudnn": sel.cudnn_us / sel.own_us,
                     "selector": sel.choice, "gflop": fl / 1e9, "mbytes": by / 1e6,
                     "wpk_tflops": fl / (sel.own_us * 1e-6) / 1e12,
                     "pct_tensor_peak": fl / (sel.own_us * 1e-6) / 1e12 / peak_tf,
                     "wpk_gbs": by / (sel.own_us * 1e-6) / 1e9,
                     "pct_hbm_peak": by / (sel.own_us * 1e-6) / 1e9 / PEAKS["hbm_gbs"],
                     "tune_measured": res.measured})
        print(json.dumps(rows[-1]), flush=True)
    return {"net": name, "dtype": dtype, "search": search, "budget": budget, "tuning_seconds_1gpu": t_tune,
            "layers": rows,
            "sum_wpk_us": sum(r["wpk_us"] * r["count"] for r in rows),
            "sum_cudnn_us": sum(r["cudnn_us"] * r["count"] for r in rows),
            "sum_selector_us": sum(min(r["wpk_us"], r["cudnn_us"]) * r["count"] for r in rows),
            "peak_source": "MEASURED_PEAKS.json (tf32 = half the bf16 figure; f32 = FP32 FMA peak at sm_max_mhz)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--nets", default="vgg16,mobilenet_v2,resnet50_n1,resnet50_tf32")
    ap.add_argument("--budget", type=int, default=32)
    a = ap.parse_args()
    res = [run_net(n, a.budget) for n in a.nets.split(",")]
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        for r in res:
            f.write(f"\n### {r['net']} ({r['dtype']}, {r['search']}-tuned, budget {r['budget']}/layer; "
                    f"tuning {r['tuning_seconds_1gpu']:.1f} s on 1 GPU)\n\n")
            f.write("| layer | x | GFLOP | MB | wpk us | cuDNN us | speedup | TF/s | % peak (f32: FMA) | GB/s | % HBM | config |\n")
            f.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for L in r["layers"]:
                f.write(f"| {L['layer']} | {L['count']} | {L['gflop']:.3f} | {L['mbytes']:.2f} | {L['wpk_us']:.1f} | "
                        f"{L['cudnn_us']:.1f} | {L['speedup_vs_cudnn']:.2f} | {L['wpk_tflops']:.1f} | "
                        f"{100 * L['pct_tensor_peak']:.1f} | {L['wpk_gbs']:.0f} | {100 * L['pct_hbm_peak']:.1f} | "
                        f"{L['family']}:{L['config']} |\n")
            f.write(f"\nsum (x count): wpk {r['sum_wpk_us']:.0f} us, cuDNN {r['sum_cudnn_us']:.0f} us, "
                    f"selector {r['sum_selector_us']:.0f} us\n")
    print("wrote", a.out + ".json", a.out + ".md")


if __name__ == "__main__":
    main()
