"""NEXT-1 measurement: the residual epilogue y = relu(conv(x) + b + z) against cuDNN's fused
torch.cudnn_convolution_add_relu (and the unfused conv2d + add + relu), per layer on the last 1x1
conv of every ResNet-50 bottleneck block (N=32 bf16 NHWC, the shapes that carry the shortcut), and
one whole bottleneck block (c1 -> c2 -> c3 + shortcut, chained through L2-resident activations) in
one CUDA graph each. Same flushed event protocol as the selector.
usage: python tools/residual_bench.py OUT_PREFIX [--budget B]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

import workloads
from paper_2008_04567_b200 import Conv2dPlan
from paper_2008_04567_b200.selector import time_fn


def nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous().cuda()


def cudnn_add_relu(x, w, b, z, stride, pad):
    xt, wt, zt = x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), z.permute(0, 3, 1, 2)
    return lambda: torch.cudnn_convolution_add_relu(xt, wt, zt, 1.0, b, (stride, stride), (pad, pad), (1, 1), 1)


def unfused(x, w, b, z, stride, pad):
    xt, wt, zt = x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), z.permute(0, 3, 1, 2)
    return lambda: F.relu_(F.conv2d(xt, wt, b, stride, pad) + zt)


def per_layer(budget):
    rows = []
    layers = {L.name: L for L in workloads.resnet50(32)}
    for i, name in enumerate(["s2b0.c3", "s3b0.c3", "s4b0.c3", "s5b0.c3"]):
        L = layers[name]
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16",
                          epilogue="bias_add_relu")
        res = plan.tune("ga", budget, seed=i)
        x, w, b = workloads.generate(L, "bf16", "uniform", seed=100 + i)
        xd, wd, bd = nhwc(x), nhwc(w), b.cuda()
        z = torch.randn(L.n, plan.p, plan.q, L.k, generator=torch.Generator().manual_seed(7)).to(torch.bfloat16).cuda()
        y = torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda")
        torch.backends.cudnn.benchmark = True
        t_wpk = time_fn(lambda: plan.run(xd, wd, bd, y, z=z))
        t_fused = time_fn(cudnn_add_relu(xd, wd, bd, z, L.stride, L.pad))
        t_unf = time_fn(unfused(xd, wd, bd, z, L.stride, L.pad))
        ref = torch.cudnn_convolution_add_relu(xd.permute(0, 3, 1, 2), wd.permute(0, 3, 1, 2), z.permute(0, 3, 1, 2),
                                               1.0, bd, (L.stride,) * 2, (L.pad,) * 2, (1, 1), 1)
        err = ((y.float() - ref.permute(0, 2, 3, 1).float()).norm() / ref.float().norm()).item()
        fl = 2 * L.n * L.k * plan.p * plan.q * L.c * L.r * L.s
        rows.append({"layer": name, "config": res.genes, "wpk_us": t_wpk, "cudnn_add_relu_us": t_fused,
                     "cudnn_unfused_us": t_unf, "speedup_vs_fused": t_fused / t_wpk, "wpk_tflops": fl / t_wpk / 1e6,
                     "rel_err_vs_cudnn": err})
        print(json.dumps(rows[-1]), flush=True)
    return rows


def block(budget):
    """Bottleneck s3b1 (C=512 -> 128 -> 128 -> 512 at 28x28) chained: wpk's three convs (the last with
    the residual epilogue) vs cuDNN's conv_relu, conv_relu, conv_add_relu, each set in one CUDA graph."""
    n, h = 32, 28
    specs = [(512, 128, 1, 0), (128, 128, 3, 1), (128, 512, 1, 0)]
    plans, ws, bs = [], [], []
    for i, (c, k, r, p) in enumerate(specs):
        epi = "bias_add_relu" if i == 2 else "bias_relu"
        plan = Conv2dPlan(n, c, h, h, k, r, r, 1, p, layout="nhwc", dtype="bf16", epilogue=epi)
        plan.tune("ga", budget, seed=10 + i)
        g = torch.Generator().manual_seed(20 + i)
        ws.append((torch.randn(k, r, r, c, generator=g) * (2.0 / (c * r * r)) ** 0.5).to(torch.bfloat16).cuda())
        bs.append((torch.randn(k, generator=g) * 0.1).cuda().float().to(torch.bfloat16))
        plans.append(plan)
    x = torch.randn(n, h, h, 512, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
    a1 = torch.empty(n, h, h, 128, dtype=torch.bfloat16, device="cuda")
    a2 = torch.empty_like(a1)
    y = torch.empty(n, h, h, 512, dtype=torch.bfloat16, device="cuda")

    def wpk_block():
        plans[0].run(x, ws[0], bs[0], a1)
        plans[1].run(a1, ws[1], bs[1], a2)
        plans[2].run(a2, ws[2], bs[2], y, z=x)

    xt = x.permute(0, 3, 1, 2)
    wt = [w.permute(0, 3, 1, 2) for w in ws]

    def cudnn_block():
        t1 = torch.cudnn_convolution_relu(xt, wt[0], bs[0], (1, 1), (0, 0), (1, 1), 1)
        t2 = torch.cudnn_convolution_relu(t1, wt[1], bs[1], (1, 1), (1, 1), (1, 1), 1)
        return torch.cudnn_convolution_add_relu(t2, wt[2], xt, 1.0, bs[2], (1, 1), (0, 0), (1, 1), 1)

    out = {}
    for nm, fn in (("wpk", wpk_block), ("cudnn", cudnn_block)):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            r = fn()
        out[nm + "_us"] = time_fn(gr.replay)
        if nm == "cudnn":
            gr.replay()
            torch.cuda.synchronize()
            ref = r.permute(0, 2, 3, 1)
    out["rel_err_vs_cudnn"] = ((y.float() - ref.float()).norm() / ref.float().norm()).item()
    out["speedup"] = out["cudnn_us"] / out["wpk_us"]
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--budget", type=int, default=32)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    res = {"per_layer": per_layer(a.budget), "block_s3b1": block(a.budget)}
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("| layer (N=32 bf16 NHWC, residual epilogue) | wpk us | cuDNN conv_add_relu us | cuDNN conv2d+add+relu us | "
                "speedup vs fused cuDNN | TF/s | config |\n|---|---|---|---|---|---|---|\n")
        for r in res["per_layer"]:
            f.write(f"| {r['layer']} | {r['wpk_us']:.1f} | {r['cudnn_add_relu_us']:.1f} | {r['cudnn_unfused_us']:.1f} | "
                    f"{r['speedup_vs_fused']:.2f} | {r['wpk_tflops']:.0f} | {r['config']} |\n")
        b = res["block_s3b1"]
        f.write(f"\nbottleneck block s3b1 (1x1 -> 3x3 -> 1x1 + shortcut, chained, one CUDA graph each): wpk "
                f"{b['wpk_us']:.1f} us, cuDNN {b['cudnn_us']:.1f} us (speedup {b['speedup']:.2f}, rel. error vs "
                f"cuDNN {b['rel_err_vs_cudnn']:.1e})\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
