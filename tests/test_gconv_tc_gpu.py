"""GPU parity of the tensor-core grouped convolution (gconv_tc.cu: the tcgen05 family's A_MODE 1 for
1 < groups < C) against the oracle (PAPER.md:47's definition with groups,
oracle/conv_oracle.c). Exact-integer inputs: every product and partial sum is an integer < 2^24, so
the fp32 accumulation is exact and the output equals RN(oracle) bit for bit; uniform inputs within
the 16-bit normwise bound."""
import pytest
import torch

import oracle
import workloads
from workloads import ConvLayer

from _util import TOL, assert_bit_exact, from_layout, rel_error, to_layout

pytestmark = pytest.mark.gpu

LAYERS = [
    ConvLayer("rx_s2", 2, 128, 15, 13, 128, 3, 3, 1, 1, 1, 32),     # ResNeXt stage 2: C/g = K/g = 4
    ConvLayer("rx_s3s2", 2, 256, 15, 15, 256, 3, 3, 2, 1, 1, 32),   # stage 3 (strided): 8 per group
    ConvLayer("rx_s4", 1, 512, 9, 11, 512, 3, 3, 1, 1, 1, 32),      # 16 per group
    ConvLayer("rx_s5", 2, 1024, 7, 7, 1024, 3, 3, 1, 1, 1, 32),     # 32 per group
    ConvLayer("g2mult", 2, 24, 13, 12, 40, 3, 3, 1, 1, 1, 2),       # C/g 12 (general gather), K/g 20
    ConvLayer("g4dil", 1, 32, 17, 17, 48, 3, 3, 1, 2, 2, 4),        # dilation 2, K/g 12
    ConvLayer("g8_1x1", 3, 64, 9, 7, 64, 1, 1, 1, 0, 1, 8),         # grouped 1x1
]


def _np(L):
    return max(16, -(-(L.k // L.groups) // 16) * 16)


def _valid_bns(plan, L):
    return [bn for bn in (16, 32, 64, 96, 128, 192, 256) if plan.config_valid(1, [bn, 2, 1, 0, 1, 1, 128])]


@pytest.fixture(scope="module", autouse=True)
def _setup():
    oracle.build()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("layer", LAYERS, ids=lambda l: l.name)
def test_gconv_tc_every_tile_int_bit_exact(layer, dtype):
    """Every valid groups-per-tile choice (BLOCK_N = groups/tile x the per-group MMA width)."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = layer
    x, w, b = workloads.generate(L, dtype, "int", seed=101)
    ref = oracle.conv2d(x, w, b, stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype=dtype)
    bns = _valid_bns(plan, L)
    assert bns and all(bn % _np(L) == 0 for bn in bns)
    xl, wl = to_layout(x, w, "nhwc")
    xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
    for bn in bns:
        plan.set_config(1, [bn, 2, 1, 0, 1, 1, 128])
        y = plan.run(xl, wl, bc)
        torch.cuda.synchronize()
        assert_bit_exact(from_layout(y.cpu(), "nhwc"), ref)


@pytest.mark.parametrize("layer", LAYERS, ids=lambda l: l.name)
def test_gconv_tc_uniform_tolerance(layer):
    from paper_2008_04567_b200 import Conv2dPlan
    L = layer
    x, w, b = workloads.generate(L, "bf16", "uniform", seed=102)
    ref = oracle.conv2d(x, w, b, stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype="bf16")
    plan.set_config(1, [_valid_bns(plan, L)[-1], 2, 1, 0, 1, 1, 128])
    xl, wl = to_layout(x, w, "nhwc")
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda())
    torch.cuda.synchronize()
    assert rel_error("bf16", from_layout(y.cpu(), "nhwc"), ref) <= TOL["bf16"]


@pytest.mark.parametrize("epilogue", ["none", "bias", "bias_add_relu"])
def test_gconv_tc_epilogues(epilogue):
    from paper_2008_04567_b200 import Conv2dPlan
    L = LAYERS[1]
    x, w, b = workloads.generate(L, "bf16", "int", seed=103)
    p = (L.h + 2 * L.pad - 2 - 1) // L.stride + 1
    z = torch.randint(-5, 6, (L.n, L.k, p, p), generator=torch.Generator().manual_seed(104)).to(torch.bfloat16)
    if epilogue == "bias_add_relu":
        ref = oracle.conv2d(x, w, b, stride=L.stride, pad=L.pad, groups=L.groups, residual=z)
    else:
        ref = oracle.conv2d(x, w, b if epilogue == "bias" else None, stride=L.stride, pad=L.pad, groups=L.groups,
                            relu=False)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc",
                      epilogue=epilogue, dtype="bf16")
    plan.set_config(1, [64, 2, 1, 0, 1, 1, 128])
    xl, wl = to_layout(x, w, "nhwc")
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda() if epilogue != "none" else None,
                 z=z.permute(0, 2, 3, 1).contiguous().cuda() if epilogue == "bias_add_relu" else None)
    torch.cuda.synchronize()
    assert_bit_exact(from_layout(y.cpu(), "nhwc"), ref)


def test_gconv_tc_matches_grouped_cuda_core_kernel():
    """Same outputs as the CUDA-core grouped kernel (the DW family's default) on exact-integer inputs."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = LAYERS[0]
    x, w, b = workloads.generate(L, "bf16", "int", seed=105)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype="bf16")
    assert plan.config[0] == 2
    xl, wl = to_layout(x, w, "nhwc")
    xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
    y0 = plan.run(xl, wl, bc).clone()
    plan.set_config(1, [256, 2, 1, 0, 1, 1, 128])
    y1 = plan.run(xl, wl, bc)
    torch.cuda.synchronize()
    assert torch.equal(y0.view(torch.int16), y1.view(torch.int16))


def test_gconv_tc_resnext_n8_sampled():
    """A full-size ResNeXt-50 32x4d grouped layer at N=8 (stage 2: 56x56, C = K = 128, 32 groups):
    sampled outputs (every border pixel of every image x 8 channels + 65,536 interior points)."""
    import numpy as np
    from paper_2008_04567_b200 import Conv2dPlan
    L = workloads.resnext50_grouped(8)[0]
    x, w, b = workloads.generate(L, "bf16", "uniform", seed=106)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc", dtype="bf16")
    plan.set_config(1, [_valid_bns(plan, L)[-1], 2, 1, 0, 1, 1, 128])
    xl, wl = to_layout(x, w, "nhwc")
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda())
    torch.cuda.synchronize()
    pts = workloads.parity_points(L, plan.p, plan.q, interior=65536, seed=107, border_channels=8)
    ref = oracle.conv2d_points(x, w, b, pts.numpy(), stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups, nthreads=8)
    got = y.cpu()[pts[:, 0], pts[:, 2], pts[:, 3], pts[:, 1]].double().numpy()
    assert float(np.linalg.norm(got - ref) / np.linalg.norm(ref)) <= TOL["bf16"]
