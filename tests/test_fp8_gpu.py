"""GPU parity of the FP8 path (NEXT-4: tcgen05.mma kind::f8f6f4): x and w in OCP
e4m3, bias / residual / output in bf16, fp32 accumulate (include/wpk.h WPK_FP8E4M3).

The oracle (oracle/conv_oracle.c, PAPER.md:47's definition) sees the same e4m3-rounded inputs as
float64, so the only differences are the fp32 accumulation order and the one RN conversion to bf16:
exact-integer inputs (x, w in {-1,0,1} are e4m3 values; every partial sum an integer < 2^24) must be
bit-exact, uniform inputs within the bf16 normwise bound (reading c10)."""
import itertools

import pytest
import torch

import oracle
import workloads
from workloads import ConvLayer

from _util import TOL, assert_bit_exact, from_layout, oracle_full, rel_error, run_product, to_layout

pytestmark = pytest.mark.gpu

LAYERS = [
    ConvLayer("3x3s1", 2, 64, 14, 14, 96, 3, 3, 1, 1),
    ConvLayer("3x3c256", 2, 256, 9, 11, 200, 3, 3, 1, 1),     # 2 K blocks of 128 channels per tap, K tail
    ConvLayer("3x3s2", 2, 128, 15, 13, 64, 3, 3, 2, 1),
    ConvLayer("1x1", 3, 256, 7, 9, 40, 1, 1, 1, 0),            # tiled A (plain GEMM)
    ConvLayer("1x1s2", 2, 64, 14, 14, 128, 1, 1, 2, 0),
    ConvLayer("dil2", 1, 32, 17, 17, 48, 3, 3, 1, 2, 2),
    ConvLayer("7x7s2c3", 2, 3, 30, 30, 64, 7, 7, 2, 3),        # C = 3: channels zero-padded to 16 bytes
    ConvLayer("c24", 1, 24, 12, 20, 24, 5, 3, 1, 1),           # C not a multiple of 16
]


@pytest.fixture(scope="module", autouse=True)
def _setup():
    oracle.build()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("layer", LAYERS, ids=lambda l: l.name)
def test_fp8_default_int_bit_exact(layer, layout):
    x, w, b = workloads.generate(layer, "fp8", "int", seed=81)
    assert x.dtype == torch.float8_e4m3fn and b.dtype == torch.bfloat16
    y, plan = run_product(layer, "fp8", layout, x, w, b)
    assert plan.config[0] == 1 and y.dtype == torch.bfloat16
    assert_bit_exact(y, oracle_full(layer, x, w, b))


@pytest.mark.parametrize("layer", LAYERS, ids=lambda l: l.name)
def test_fp8_default_uniform_tolerance(layer):
    x, w, b = workloads.generate(layer, "fp8", "uniform", seed=82)
    y, _ = run_product(layer, "fp8", "nhwc", x, w, b)
    err = rel_error("fp8", y, oracle_full(layer, x, w, b))
    assert err <= TOL["fp8"], err


@pytest.mark.parametrize("epilogue", ["none", "bias", "bias_relu"])
def test_fp8_epilogues(epilogue):
    L = LAYERS[0]
    x, w, b = workloads.generate(L, "fp8", "int", seed=83)
    y, _ = run_product(L, "fp8", "nhwc", x, w, b if epilogue != "none" else None, epilogue=epilogue)
    assert_bit_exact(y, oracle_full(L, x, w, b, epilogue))


def test_fp8_every_config_bit_exact():
    """Every valid tcgen05 config of a sweep (1-CTA and pair tiles, BLOCK_M 128/256, split-K in L2 and
    in a cluster, 1/2/4 accumulators, dual accumulators, round-robin producers) on a shape with M, K
    and channel-block tails: bit-identical outputs in exact-integer mode."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = ConvLayer("sweep8", 2, 192, 11, 13, 200, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, "fp8", "int", seed=84)
    ref = oracle_full(L, x, w, b)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="fp8")
    xl, wl = to_layout(x, w, "nhwc")
    xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
    n = 0
    for genes in itertools.product([16, 32, 64, 128, 192, 256], [2, 4, 6], [1, 2, 4], range(8), [0, 4, 5, 6], [1, 2, 4],
                                   [128, 256]):
        genes = list(genes)
        if not plan.config_valid(1, genes):
            continue
        plan.set_config(1, genes)
        y = plan.run(xl, wl, bc)
        torch.cuda.synchronize()
        assert_bit_exact(from_layout(y.cpu(), "nhwc"), ref)
        n += 1
    assert n > 100
    for am in (1, 2, 3):   # gather / explicit-im2col producers are not instantiated for e4m3
        assert not plan.config_valid(1, [128, 4, 1, 0, am, 2, 128])


def test_fp8_residual_epilogue():
    """y = relu(conv + b + z) with a bf16 residual z, TMA-store and direct (NCHW) epilogues."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = ConvLayer("r8", 2, 64, 11, 13, 128, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, "fp8", "int", seed=85)
    g = torch.Generator().manual_seed(86)
    z = torch.randint(-6, 7, (L.n, L.k, 11, 13), generator=g).to(torch.bfloat16)
    ref = oracle.conv2d(x, w, b, stride=1, pad=1, residual=z)
    for layout in ("nhwc", "nchw"):
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout=layout,
                          epilogue="bias_add_relu", dtype="fp8")
        xl, wl = to_layout(x, w, layout)
        zl = z.permute(0, 2, 3, 1).contiguous() if layout == "nhwc" else z
        y = plan.run(xl.cuda(), wl.cuda(), b.cuda(), z=zl.cuda())
        torch.cuda.synchronize()
        assert_bit_exact(from_layout(y.cpu(), layout), ref)


def test_fp8_tune_then_parity():
    """GA over the e4m3 space (the tuner fills e4m3 operands and bf16 bias itself); the chosen config
    is bit-exact."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = ConvLayer("t8", 4, 256, 14, 14, 256, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, "fp8", "int", seed=87)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="fp8")
    res = plan.tune("ga", 16, seed=3)
    assert res.measured >= 1 and res.best_us < float("inf")
    xl, wl = to_layout(x, w, "nhwc")
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda())
    torch.cuda.synchronize()
    assert_bit_exact(from_layout(y.cpu(), "nhwc"), oracle_full(L, x, w, b))


def test_fp8_resnet50_sampled():
    """A full-size ResNet-50 N=32 3x3 layer (s4b1.c2) in e4m3: sampled outputs (every border pixel of
    every image x 8 channels + 65,536 interior points) against the oracle point by point."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = [l for l in workloads.resnet50(32) if l.name == "s4b1.c2"][0]
    x, w, b = workloads.generate(L, "fp8", "uniform", seed=workloads.config_seed(2, 16))
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="fp8")
    xl, wl = to_layout(x, w, "nhwc")
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda())
    torch.cuda.synchronize()
    p, q = y.shape[1], y.shape[2]
    pts = workloads.parity_points(L, p, q, interior=65536, seed=88, border_channels=8)
    ref = oracle.conv2d_points(x, w, b, pts.numpy(), stride=L.stride, pad=L.pad, nthreads=8)
    yc = y.cpu()
    got = yc[pts[:, 0], pts[:, 2], pts[:, 3], pts[:, 1]].double().numpy()
    import numpy as np
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert err <= TOL["fp8"], err


def test_fp8_plan_rejections():
    """Groups > 1 and the CUDA-core families have no e4m3 kernel: WPK_ERR_UNSUPPORTED at plan time,
    and the SIMT / GEMM32 / DW families are invalid configs of an fp8 plan."""
    from paper_2008_04567_b200 import Conv2dPlan
    with pytest.raises(Exception, match="FP8"):
        Conv2dPlan(1, 32, 8, 8, 32, 3, 3, 1, 1, groups=32, layout="nhwc", dtype="fp8")
    plan = Conv2dPlan(1, 32, 8, 8, 32, 3, 3, 1, 1, layout="nhwc", dtype="fp8")
    assert not plan.config_valid(0, [16, 4, 4, 1, 1, 1, 1])
    assert not plan.config_valid(3, [64, 64, 16, 4, 1, 0, 0])
