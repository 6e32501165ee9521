"""Test helpers: run a layer through the product (C ABI via the binding) and through the oracle on
the same seeded inputs, and compare. Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import workloads

TOL = {"f32": 1e-5, "tf32": 5e-3, "bf16": 2e-2, "f16": 2e-2,   # BASELINE.json north_star
       "fp8": 2e-2}   # e4m3 operands (the oracle sees the same rounded values), bf16 output: the bf16 bound


def to_layout(x, w, layout):
    if layout == "nhwc":
        return x.permute(0, 2, 3, 1).contiguous(), w.permute(0, 2, 3, 1).contiguous()
    return x.contiguous(), w.contiguous()


def from_layout(y, layout):
    return y.permute(0, 3, 1, 2).contiguous() if layout == "nhwc" else y


def run_product(L: workloads.ConvLayer, dtype, layout, x, w, b, config=None, epilogue="bias_relu"):
    from paper_2008_04567_b200 import Conv2dPlan
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout=layout,
                      epilogue=epilogue, dtype=dtype)
    if config is not None:
        plan.set_config(*config)
    xl, wl = to_layout(x, w, layout)
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda() if b is not None else None)
    torch.cuda.synchronize()
    return from_layout(y.cpu(), layout), plan


def oracle_full(L, x, w, b, epilogue="bias_relu"):
    if epilogue == "none":
        b = None
    return oracle.conv2d(x, w, b, stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups,
                         relu=(epilogue == "bias_relu"))


def canon_bits(t: torch.Tensor) -> torch.Tensor:
    """Bit pattern with -0 canonicalised to +0 (reading c7)."""
    t = t.clone()
    t[t == 0] = 0
    if t.dtype == torch.float32:
        return t.view(torch.int32)
    return t.view(torch.int16)


def assert_bit_exact(got: torch.Tensor, ref_f64: np.ndarray):
    ref = torch.from_numpy(ref_f64).to(got.dtype)    # RN(double -> dtype): exact ints stay exact
    bad = (canon_bits(got) != canon_bits(ref))
    if bad.any():
        idx = bad.nonzero()[0].tolist()
        raise AssertionError(f"{int(bad.sum())} of {bad.numel()} outputs differ; first at {idx}: "
                             f"got {got[tuple(idx)].item()} want {ref[tuple(idx)].item()}")


def rel_error(dtype, got: torch.Tensor, ref: np.ndarray) -> float:
    g = got.double().numpy()
    if dtype == "f32":
        return float(np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-30))
    return float(np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30))
