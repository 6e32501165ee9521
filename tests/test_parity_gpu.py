"""GPU parity: the CUDA path through the C ABI vs the oracle on the same seeded inputs.

Exact-integer mode (x, w in {-1,0,1}, b in {-4..4}) must be bit-exact on every precision path
(reading c11); uniform mode must meet BASELINE.json's tolerances: fp32 max-rel 1e-5, TF32
normwise 5e-3, bf16/fp16 normwise 2e-2."""
import itertools
import os

import numpy as np
import pytest
import torch

import oracle
import workloads
from workloads import ConvLayer

from _util import TOL, assert_bit_exact, from_layout, oracle_full, rel_error, run_product, to_layout

pytestmark = pytest.mark.gpu

SMALL = [
    ConvLayer("cfg1", 1, 3, 8, 8, 8, 3, 3, 1, 1),
    ConvLayer("3x3s1", 2, 64, 14, 14, 96, 3, 3, 1, 1),
    ConvLayer("3x3s2", 2, 64, 15, 13, 64, 3, 3, 2, 1),
    ConvLayer("1x1", 3, 128, 7, 9, 40, 1, 1, 1, 0),
    ConvLayer("1x1s2", 2, 64, 14, 14, 128, 1, 1, 2, 0),
    ConvLayer("dil2", 1, 32, 17, 17, 48, 3, 3, 1, 2, 2),
    ConvLayer("7x7s2c3", 2, 3, 30, 30, 64, 7, 7, 2, 3),
    ConvLayer("5x3_asym", 1, 16, 12, 20, 24, 5, 3, 1, 1),
    ConvLayer("valid", 1, 64, 12, 10, 256, 3, 3, 1, 0),
]


@pytest.fixture(scope="module", autouse=True)
def _setup():
    oracle.build()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16", "f16"])
@pytest.mark.parametrize("layer", SMALL, ids=lambda l: l.name)
def test_default_config_int_bit_exact(layer, dtype, layout):
    x, w, b = workloads.generate(layer, dtype, "int", seed=11)
    y, plan = run_product(layer, dtype, layout, x, w, b)
    assert_bit_exact(y, oracle_full(layer, x, w, b))


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16", "f16"])
@pytest.mark.parametrize("layer", SMALL, ids=lambda l: l.name)
def test_default_config_uniform_tolerance(layer, dtype, layout):
    x, w, b = workloads.generate(layer, dtype, "uniform", seed=12)
    y, plan = run_product(layer, dtype, layout, x, w, b)
    err = rel_error(dtype, y, oracle_full(layer, x, w, b))
    assert err <= TOL[dtype], err


@pytest.mark.parametrize("epilogue", ["none", "bias", "bias_relu"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_epilogues(dtype, epilogue):
    L = SMALL[1]
    x, w, b = workloads.generate(L, dtype, "int", seed=13)
    y, _ = run_product(L, dtype, "nhwc", x, w, b if epilogue != "none" else None, epilogue=epilogue)
    assert_bit_exact(y, oracle_full(L, x, w, b, epilogue))


def _umma_space():
    bns = [16, 32, 64, 96, 128, 192, 256]
    out = []
    for bn, st, sp, ra, amode, acc, bm in itertools.product(bns, [2, 4, 6], [1, 2, 4], [0, 1, 2, 3, 4, 5, 6, 7], [0, 1, 2, 4, 5, 6],
                                                          [1, 2, 4], [128, 256]):
        out.append((bn, st, sp, ra, amode, acc, bm))
    return out


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_umma_every_config_bit_exact(dtype):
    """Every valid UMMA config in a sweep of the space on one shape with an M tail, K tail and
    several K blocks: exact-integer outputs must be bit-identical (a tiling can change speed,
    never values)."""
    L = ConvLayer("sweep", 2, 64, 11, 13, 200, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, dtype, "int", seed=14)
    ref = oracle_full(L, x, w, b)
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype=dtype)
    xl, wl = to_layout(x, w, "nhwc")
    xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
    n = 0
    for genes in _umma_space():
        if not plan.config_valid(1, genes):
            continue
        plan.set_config(1, genes)
        y = plan.run(xl, wl, bc)
        torch.cuda.synchronize()
        assert_bit_exact(from_layout(y.cpu(), "nhwc"), ref)
        n += 1
    assert n > 100


@pytest.mark.parametrize("env", [{}, {"WPK_EPI_DIRECT": "1"}, {"WPK_A_IM2COL": "1"}])
@pytest.mark.parametrize("dtype", ["bf16", "f16", "tf32"])
def test_umma_1x1_and_epilogue_paths(dtype, env, monkeypatch):
    """1x1 layers (tiled A path), split-K partials through the TMA store, the direct epilogue."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    for L in [ConvLayer("1x1a", 2, 128, 9, 11, 192, 1, 1, 1, 0), ConvLayer("1x1b", 1, 256, 7, 7, 72, 1, 1, 1, 0)]:
        x, w, b = workloads.generate(L, dtype, "int", seed=21)
        ref = oracle_full(L, x, w, b)
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype=dtype)
        xl, wl = to_layout(x, w, "nhwc")
        xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
        for genes in [(64, 4, 1, 0, 0, 2, 128), (128, 3, 2, 1, 0, 2, 128), (256, 2, 4, 0, 0, 1, 128),
                      (32, 4, 1, 0, 0, 2, 128), (96, 5, 2, 0, 0, 2, 128), (192, 3, 1, 1, 0, 2, 128),
                      (64, 4, 1, 0, 1, 2, 128), (128, 4, 2, 0, 1, 2, 128), (64, 4, 1, 0, 0, 2, 256),
                      (128, 3, 2, 0, 0, 1, 256), (96, 4, 1, 1, 0, 2, 256), (32, 4, 2, 0, 1, 2, 256),
                      (64, 4, 1, 0, 2, 2, 128), (128, 3, 2, 0, 2, 2, 256), (256, 2, 1, 0, 2, 1, 128),
                      (128, 4, 1, 2, 0, 2, 256), (256, 3, 1, 3, 0, 2, 256), (64, 4, 1, 2, 1, 2, 256),
                      (32, 4, 1, 2, 0, 1, 256), (192, 3, 1, 2, 0, 2, 256)]:
            if not plan.config_valid(1, list(genes)):
                continue
            plan.set_config(1, list(genes))
            y = plan.run(xl, wl, bc)
            torch.cuda.synchronize()
            assert_bit_exact(from_layout(y.cpu(), "nhwc"), ref)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_cta_pair_configs(dtype):
    """tcgen05 CTA pairs (cta_group::2): 3x3 and strided shapes with M and K tails, with split-K
    (per-CTA-half fixup counters) and 1/2/4 accumulator stages."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    for L in [ConvLayer("p3", 2, 64, 17, 19, 160, 3, 3, 1, 1), ConvLayer("p3s2", 3, 128, 15, 15, 96, 3, 3, 2, 1)]:
        x, w, b = workloads.generate(L, dtype, "int", seed=29)
        ref = oracle_full(L, x, w, b)
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype=dtype)
        xl, wl = to_layout(x, w, "nhwc")
        xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
        n = 0
        for bn, st, mode, acc, sp, am in itertools.product([32, 64, 128, 256], [2, 4], [2, 3], [1, 2, 4], [1, 2, 4],
                                                           [0, 5]):
            genes = [bn, st, sp, mode, am, acc, 256]
            if not plan.config_valid(1, genes):
                continue
            plan.set_config(1, genes)
            y = plan.run(xl, wl, bc)
            torch.cuda.synchronize()
            assert_bit_exact(from_layout(y.cpu(), "nhwc"), ref)
            n += 1
        assert n >= 8


def test_simt_every_tile_template():
    L = ConvLayer("simt", 2, 6, 9, 11, 10, 3, 3, 2, 1)
    x, w, b = workloads.generate(L, "f32", "int", seed=15)
    ref = oracle_full(L, x, w, b)
    from paper_2008_04567_b200 import Conv2dPlan
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nchw", dtype="f32")
    xc, wc, bc = x.cuda(), w.cuda(), b.cuda()
    for tx, ty, tz, trz in itertools.product([1, 2, 4], [1, 2, 4], [1, 2, 4], [1, 2, 4, 8]):
        for T in [(8, 4, 2), (32, 1, 1), (1, 1, 32)]:
            genes = list(T) + [tx, ty, tz, trz]
            plan.set_config(0, genes)
            y = plan.run(xc, wc, bc)
            torch.cuda.synchronize()
            assert_bit_exact(y.cpu(), ref)


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_gemm32_every_template(layout):
    """Exact-fp32 implicit GEMM (WPK_FAMILY_GEMM32): every (BLOCK_M, BLOCK_N, BLOCK_K, THREAD_TILE)
    instantiation with and without split-K, vector (C % 4 == 0) and scalar operand loads, ragged M/K/R*S*C tails, all
    epilogues: bit-exact in integer mode, within 1e-5 max-rel in uniform mode."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    layers = [ConvLayer("g3", 2, 20, 13, 11, 72, 3, 3, 1, 1), ConvLayer("g3s2", 1, 7, 17, 15, 130, 3, 3, 2, 1),
              ConvLayer("g1", 3, 36, 9, 7, 40, 1, 1, 1, 0), ConvLayer("gdil", 1, 12, 14, 16, 24, 3, 5, 1, 2, 2)]
    for li, L in enumerate(layers):
        epi = ["none", "bias", "bias_relu", "bias_relu"][li]
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, layout=layout, epilogue=epi,
                          dtype="f32")
        assert plan.config[0] == 3
        ran = 0
        for mode in ("int", "uniform"):
            x, w, b = workloads.generate(L, "f32", mode, seed=60 + li)
            ref = oracle.conv2d(x, w, b if epi != "none" else None, stride=L.stride, pad=L.pad, dil=L.dil,
                                relu=(epi == "bias_relu"))
            xl, wl = to_layout(x, w, layout)
            xl, wl, bc = xl.cuda(), wl.cuda(), (b.cuda() if epi != "none" else None)
            for bm, bn, bk, tt, sk in itertools.product([64, 128], [64, 128], [8, 16], [4, 8], [1, 2, 8]):
                if not plan.config_valid(3, [bm, bn, bk, tt, sk, 0, 0]):
                    assert sk == 8, (L.name, bm, bn, bk, tt, sk)   # only an empty split is invalid
                    continue
                ran += 1
                plan.set_config(3, [bm, bn, bk, tt, sk, 0, 0])
                y = from_layout(plan.run(xl, wl, bc).cpu(), layout)
                torch.cuda.synchronize()
                if mode == "int":
                    assert_bit_exact(y, ref)
                else:
                    assert rel_error("f32", y, ref) <= TOL["f32"], (L.name, bm, bn, bk, tt)
        assert ran >= 2 * 32, L.name


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16", "f16"])
def test_general_groups(dtype, layout):
    """Grouped conv with 1 < groups (ResNeXt-style C/g = 4, g = 2, channel multiplier 2): the
    grouped-kernel default and other output vectors / pixels per thread, and two SIMT tile
    templates: bit-exact in integer mode, within tolerance in uniform mode."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    layers = [ConvLayer("g32x4", 2, 128, 9, 11, 128, 3, 3, 1, 1, 1, 32), ConvLayer("g2s2", 1, 24, 13, 12, 40, 3, 3, 2, 1, 1, 2),
              ConvLayer("gmult", 2, 16, 8, 8, 32, 3, 3, 1, 1, 1, 16)]
    for L in layers:
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout=layout, dtype=dtype)
        assert plan.config[0] == 2, L.name
        tiles = [None, (2, [1, 2, 64, 1, 0, 0, 0]), (2, [2, 4, 128, 1, 0, 0, 0]), (2, [4, 1, 512, 1, 0, 0, 0]),
                 (0, [8, 8, 4, 2, 1, 2, 1]), (0, [32, 2, 2, 1, 2, 1, 1])]
        for mode in ("int", "uniform"):
            x, w, b = workloads.generate(L, dtype, mode, seed=71)
            ref = oracle.conv2d(x, w, b, stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups)
            xl, wl = to_layout(x, w, layout)
            xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
            for cfg in tiles:
                if cfg is not None:
                    if not plan.config_valid(*cfg):
                        assert cfg[0] == 2 and (L.k // L.groups) % cfg[1][0], (L.name, cfg)
                        continue
                    plan.set_config(*cfg)
                y = from_layout(plan.run(xl, wl, bc).cpu(), layout)
                torch.cuda.synchronize()
                if mode == "int":
                    assert_bit_exact(y, ref)
                else:
                    assert rel_error(dtype, y, ref) <= TOL[dtype], (L.name, cfg)


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_depthwise(dtype, layout):
    for L in [ConvLayer("dw", 2, 96, 15, 15, 96, 3, 3, 2, 1, 1, 96), ConvLayer("dw1", 1, 32, 12, 12, 32, 3, 3, 1, 1, 1, 32)]:
        x, w, b = workloads.generate(L, dtype, "int", seed=16)
        y, plan = run_product(L, dtype, layout, x, w, b)
        assert plan.config[0] == 2
        assert_bit_exact(y, oracle_full(L, x, w, b))
        from paper_2008_04567_b200 import Conv2dPlan
        for genes in itertools.product([1, 2, 4, 8], [1, 2, 4], [64, 256], [1]):
            if plan.config_valid(2, list(genes) + [0, 0, 0]):
                plan.set_config(2, list(genes) + [0, 0, 0])
                from _util import to_layout, from_layout
                xl, wl = to_layout(x, w, layout)
                yy = plan.run(xl.cuda(), wl.cuda(), b.cuda())
                torch.cuda.synchronize()
                assert_bit_exact(from_layout(yy.cpu(), layout), oracle_full(L, x, w, b))


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_depthwise_nhwc_sliding_window(dtype):
    """The NHWC 3x3 sliding-window depthwise kernel (VEC_C 8, 16-bit, stride 1 / 2) against the oracle
    (exact-integer: bit-exact; uniform: tolerance) and against the generic kernel on the same inputs
    (NCHW plan): the same per-output order (taps in (r, s) order, fp32 FMA, bias after the sum), so the
    outputs are bit-identical up to the sign of zero. Ragged Q (not a multiple of PIX), every epilogue."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import canon_bits, from_layout, to_layout
    for L in [ConvLayer("mb", 2, 144, 19, 17, 144, 3, 3, 1, 1, 1, 144), ConvLayer("mbs2", 3, 96, 21, 23, 96, 3, 3, 2, 1, 1, 96),
              ConvLayer("c8", 1, 8, 9, 11, 8, 3, 3, 1, 1, 1, 8)]:
        for epi in ("none", "bias", "bias_relu", "bias_add_relu"):
            for mode in ("int", "uniform"):
                x, w, b = workloads.generate(L, dtype, mode, seed=17)
                p, q = (L.h + 2 - 2 - 1) // L.stride + 1, (L.w + 2 - 2 - 1) // L.stride + 1
                z = torch.randint(-3, 4, (L.n, L.k, p, q), generator=torch.Generator().manual_seed(18)).to(x.dtype)
                bb = b if epi != "none" else None
                if epi == "bias_add_relu":
                    ref = oracle.conv2d(x, w, b, stride=L.stride, pad=1, groups=L.groups, residual=z)
                else:
                    ref = oracle.conv2d(x, w, bb, stride=L.stride, pad=1, groups=L.groups, relu=(epi == "bias_relu"))
                outs = {}
                for layout in ("nhwc", "nchw"):
                    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, 3, 3, L.stride, 1, 1, L.groups, layout=layout,
                                      epilogue=epi, dtype=dtype)
                    xl, wl = to_layout(x, w, layout)
                    zl = z.permute(0, 2, 3, 1).contiguous() if layout == "nhwc" else z
                    # NHWC VEC_C 8: the sliding-window kernel; NHWC VEC_C 4 and NCHW VEC_C 1: the generic one
                    for vec, pix in ([(8, 1), (8, 2), (8, 4), (4, 2)] if layout == "nhwc" else [(1, 1), (1, 4)]):
                        plan.set_config(2, [vec, pix, 128, 1, 0, 0, 0])
                        y = plan.run(xl.cuda(), wl.cuda(), bb.cuda() if bb is not None else None,
                                     z=zl.cuda() if epi == "bias_add_relu" else None)
                        torch.cuda.synchronize()
                        y = from_layout(y.cpu(), layout)
                        if mode == "int":
                            assert_bit_exact(y, ref)
                        else:
                            assert rel_error(dtype, y, ref) <= TOL[dtype]
                        outs[(layout, vec, pix)] = y
                base = canon_bits(outs[("nchw", 1, 1)])
                for key, y in outs.items():
                    assert torch.equal(canon_bits(y), base), (L.name, epi, mode, key)


def test_run_host_matches_device():
    L = SMALL[1]
    x, w, b = workloads.generate(L, "bf16", "int", seed=17)
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    xl, wl = to_layout(x, w, "nhwc")
    yh = torch.empty(plan.y_shape(), dtype=torch.bfloat16).pin_memory()
    plan.run_host(xl.pin_memory(), wl.cuda(), b.cuda(), yh)
    yd = plan.run(xl.cuda(), wl.cuda(), b.cuda())
    torch.cuda.synchronize()
    assert torch.equal(yh, yd.cpu())
    # the async variant on a side stream: valid after that stream is synchronised
    ya = torch.zeros_like(yh).pin_memory()
    st = torch.cuda.Stream()
    plan.run_host_async(xl.pin_memory(), wl.cuda(), b.cuda(), ya, stream=st)
    st.synchronize()
    assert torch.equal(ya, yh)


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_gather_producer_small_c(dtype, layout):
    """A_MODE 2 (fused im2col gather into swizzled smem) on small-C shapes incl. conv1-like 7x7/s2."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    for L in [ConvLayer("c3", 2, 3, 30, 30, 64, 7, 7, 2, 3), ConvLayer("c5", 1, 5, 17, 13, 40, 3, 3, 1, 1, 2),
              ConvLayer("c24", 3, 24, 15, 15, 144, 1, 1, 2, 0)]:
        x, w, b = workloads.generate(L, dtype, "int", seed=23)
        ref = oracle_full(L, x, w, b)
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, layout=layout, dtype=dtype)
        xl, wl = to_layout(x, w, layout)
        xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
        for genes in [(64, 4, 1, 0, 2, 2, 128), (128, 3, 2, 1, 2, 2, 256), (32, 6, 1, 0, 2, 1, 128)]:
            if not plan.config_valid(1, list(genes)):
                continue
            plan.set_config(1, list(genes))
            y = plan.run(xl, wl, bc)
            torch.cuda.synchronize()
            assert_bit_exact(from_layout(y.cpu(), layout), ref)


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["bf16", "f16", "tf32"])
def test_segment_gather_small_c(dtype, layout):
    """A_MODE 3 (pixel-segment gather, C <= 4): conv1-like 7x7/s2, VGG conv1_1-like 3x3/s1,
    MobileNet stem-like 3x3/s2, C=1 with dilation, C=4 5x5/s3, ragged M and K tails."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    for L in [ConvLayer("c3s2", 2, 3, 30, 30, 64, 7, 7, 2, 3), ConvLayer("c3s1", 1, 3, 19, 21, 72, 3, 3, 1, 1),
              ConvLayer("stem", 3, 3, 17, 17, 32, 3, 3, 2, 1), ConvLayer("c1d2", 2, 1, 23, 20, 40, 3, 3, 1, 2, 2),
              ConvLayer("c4s3", 1, 4, 31, 29, 24, 5, 5, 3, 0), ConvLayer("c2", 1, 2, 9, 9, 16, 2, 4, 1, 1)]:
        x, w, b = workloads.generate(L, dtype, "int", seed=29)
        ref = oracle_full(L, x, w, b)
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, layout=layout, dtype=dtype)
        xl, wl = to_layout(x, w, layout)
        xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
        ran = 0
        for genes in [(64, 4, 1, 0, 3, 2, 128), (128, 3, 2, 1, 3, 2, 256), (32, 6, 1, 0, 3, 1, 128),
                      (16, 3, 1, 0, 3, 4, 256)]:
            if not plan.config_valid(1, list(genes)):
                continue
            plan.set_config(1, list(genes))
            y = plan.run(xl, wl, bc)
            torch.cuda.synchronize()
            assert_bit_exact(from_layout(y.cpu(), layout), ref)
            ran += 1
        assert ran >= 2, L.name


@pytest.mark.parametrize("layer", workloads.resnet50(32), ids=lambda l: l.name)
def test_resnet50_n32_sampled_bf16(layer):
    """Full-size bench layers (BASELINE.json configs[1], N=32 bf16 NHWC, default config): sampled
    outputs (every border pixel of every image x all channels + 65,536 interior points) vs the oracle."""
    x, w, b = workloads.generate(layer, "bf16", "int", seed=workloads.config_seed(1, 0))
    y, plan = run_product(layer, "bf16", "nhwc", x, w, b)
    pts = workloads.parity_points(layer, plan.p, plan.q, 65536, seed=1).numpy()
    ref = oracle.conv2d_points(x, w, b, pts, stride=layer.stride, pad=layer.pad, nthreads=os.cpu_count() or 8)
    got = y[pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    assert_bit_exact(got, ref)


_TUNED_F32 = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r1e_suite_f32.json")


@pytest.mark.parametrize("layer", workloads.resnet50(8), ids=lambda l: l.name)
def test_resnet50_n8_f32_tuned_configs_sampled(layer):
    """Exact fp32 at full size in the GA-tuned GEMM32 configs of profiles/r1e_suite_f32.json (split-K
    up to 8): sampled outputs bit-exact in integer mode, within fp32 max-rel 1e-5 in uniform mode."""
    import json
    r = {row["layer"]: row for row in json.load(open(_TUNED_F32))[0]["layers"]}[layer.name]
    for mode in ("int", "uniform"):
        x, w, b = workloads.generate(layer, "f32", mode, seed=workloads.config_seed(2, 3))
        y, plan = run_product(layer, "f32", "nhwc", x, w, b, config=(r["family"], r["config"]))
        pts = workloads.random_points(layer, plan.p, plan.q, 2048, seed=3).numpy()
        ref = oracle.conv2d_points(x, w, b, pts, stride=layer.stride, pad=layer.pad, nthreads=8)
        got = y[pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]].double().numpy()
        if mode == "int":
            assert np.array_equal(got, ref)
        else:
            assert np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30) <= TOL["f32"]


def _residual_case(L, dtype, layout, seed):
    """x, w, b and a residual z (NCHW, y's shape) in exact-integer mode, plus the oracle output."""
    x, w, b = workloads.generate(L, dtype, "int", seed=seed)
    p = (L.h + 2 * L.pad - L.dil * (L.r - 1) - 1) // L.stride + 1
    q = (L.w + 2 * L.pad - L.dil * (L.s - 1) - 1) // L.stride + 1
    g = torch.Generator().manual_seed(seed + 1)
    z = torch.randint(-6, 7, (L.n, L.k, p, q), generator=g).to(workloads.torch_dtype(dtype))
    ref = oracle.conv2d(x, w, b, stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups, residual=z)
    return x, w, b, z, ref


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16", "f16"])
def test_residual_epilogue(dtype, layout):
    """Epilogue 3, y = relu(conv + b + z): every family (GEMM32 incl. split-K and SIMT for f32, tcgen05
    with TMA-store and direct epilogues, pairs, both gathers, depthwise and grouped) is bit-exact
    against the oracle."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout
    cases = [(ConvLayer("r3", 2, 64, 11, 13, 128, 3, 3, 1, 1), None),
             (ConvLayer("r1", 1, 96, 9, 7, 200, 1, 1, 1, 0), None),
             (ConvLayer("rdw", 2, 32, 10, 9, 32, 3, 3, 2, 1, 1, 32), None),
             (ConvLayer("rgrp", 2, 32, 10, 9, 48, 3, 3, 1, 1, 1, 4), None)]
    for L, _ in cases:
        x, w, b, z, ref = _residual_case(L, dtype, layout, seed=41)
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout=layout,
                          epilogue="bias_add_relu", dtype=dtype)
        xl, wl = to_layout(x, w, layout)
        zl = z.permute(0, 2, 3, 1).contiguous() if layout == "nhwc" else z.contiguous()
        xl, wl, bc, zc = xl.cuda(), wl.cuda(), b.cuda(), zl.cuda()
        configs = [plan.config]
        if dtype == "f32" and L.groups == 1:   # the paper's SIMT template, GEMM32 default and split-K
            configs += [(0, [16, 4, 4, 1, 1, 1, 1]), (0, [8, 8, 4, 2, 1, 2, 4]), (3, [64, 64, 8, 4, 2, 0, 0]),
                        (3, [128, 64, 16, 8, 4, 0, 0])]
        if plan.config[0] == 1:
            configs += [(1, [128, 4, 1, 0, 0, 2, 128]), (1, [64, 3, 1, 1, 0, 4, 256]), (1, [256, 3, 1, 2, 0, 1, 256])]
            assert not plan.config_valid(1, [128, 4, 2, 0, 0, 2, 128])   # residual plans: SPLIT_K = 1 only
        ran = 0
        for fam, genes in configs:
            if not plan.config_valid(fam, list(genes)):
                continue
            plan.set_config(fam, list(genes))
            y = plan.run(xl, wl, bc, z=zc)
            torch.cuda.synchronize()
            assert_bit_exact(from_layout(y.cpu(), layout), ref)
            ran += 1
        assert ran >= 1, L.name
        with pytest.raises(Exception):   # a residual plan refuses the plain run entry point
            plan.run(xl, wl, bc)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_residual_plan_tunes(dtype):
    """A residual-epilogue plan can be tuned (the tuner supplies a z buffer to every candidate) and
    its chosen config is bit-exact."""
    from paper_2008_04567_b200 import Conv2dPlan
    L = ConvLayer("rt", 2, 64, 14, 14, 128, 1, 1, 1, 0)
    x, w, b, z, ref = _residual_case(L, dtype, "nhwc", seed=43)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", epilogue="bias_add_relu",
                      dtype=dtype)
    res = plan.tune("ga", 12, seed=1)
    assert res.measured >= 1 and res.best_us < float("inf")
    xl, wl = x.permute(0, 2, 3, 1).contiguous().cuda(), w.permute(0, 2, 3, 1).contiguous().cuda()
    y = plan.run(xl, wl, b.cuda(), z=z.permute(0, 2, 3, 1).contiguous().cuda())
    torch.cuda.synchronize()
    assert_bit_exact(y.cpu().permute(0, 3, 1, 2).contiguous(), ref)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_fold_batchnorm(dtype):
    """wpk_conv2d_fold_batchnorm vs the oracle's float64 fold: folded weights/bias within one
    rounding of the dtype, and the folded conv within the dtype tolerance of BN(conv) (oracle)."""
    from paper_2008_04567_b200 import Conv2dPlan
    from _util import to_layout, from_layout, rel_error
    L = ConvLayer("bn", 2, 32, 9, 9, 48, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, dtype, "uniform", seed=51)
    g = torch.Generator().manual_seed(52)
    gamma = torch.rand(L.k, generator=g) + 0.5
    beta = torch.rand(L.k, generator=g) - 0.5
    mean = torch.rand(L.k, generator=g) - 0.5
    var = torch.rand(L.k, generator=g) + 0.2
    eps = 1e-5
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype=dtype)
    xl, wl = to_layout(x, w, "nhwc")
    wf, bf = plan.fold_batchnorm(wl.cuda(), b.cuda(), gamma.cuda(), beta.cuda(), mean.cuda(), var.cuda(), eps)
    torch.cuda.synchronize()
    wo, bo = oracle.fold_batchnorm(w, b, gamma, beta, mean, var, eps)
    # one rounding of the dtype (bf16/f16), or a few fp32 ulps of the fp32 fold (s_k then w * s_k)
    ulp = {"f32": 2.0 ** -21, "bf16": 2.0 ** -7, "f16": 2.0 ** -10}[dtype]
    wf_nchw = wf.permute(0, 3, 1, 2).cpu().double().numpy()
    tiny = {"f32": 2.0 ** -149, "bf16": 2.0 ** -133, "f16": 2.0 ** -24}[dtype]   # subnormal spacing
    assert np.all(np.abs(wf_nchw - wo) <= 1.01 * ulp * np.abs(wo) + tiny)
    # b' = (b - mean) s + beta can cancel: bound by the magnitude of its terms (two fp32 roundings
    # inside, one rounding of the dtype at the end)
    sk = gamma.double().numpy() / np.sqrt(var.double().numpy() + eps)
    mag = np.abs(b.double().numpy() - mean.double().numpy()) * sk + np.abs(beta.double().numpy())
    assert np.all(np.abs(bf.cpu().double().numpy() - bo) <= 1.01 * ulp * mag + 4 * 2.0 ** -24 * mag + tiny)
    y = plan.run(xl.cuda(), wf, bf)
    torch.cuda.synchronize()
    t = oracle.conv2d(x, w, b, stride=1, pad=1, relu=False)
    ref = np.maximum(gamma.double().numpy()[None, :, None, None] * (t - mean.double().numpy()[None, :, None, None])
                     / np.sqrt(var.double().numpy() + eps)[None, :, None, None] + beta.double().numpy()[None, :, None, None], 0)
    assert rel_error(dtype, from_layout(y.cpu(), "nhwc"), ref) <= TOL[dtype]


@pytest.mark.parametrize("case", range(24))
def test_random_shapes_random_configs(case):
    """Seeded random shapes (N, C, H, W, K, R, S, stride, pad, dilation, groups in {1, C}, layout,
    dtype) x the plan's default config and 3 random valid configs of its family: exact-integer
    inputs, bit-exact against the oracle."""
    from paper_2008_04567_b200 import Conv2dPlan, _lib as L
    from _util import to_layout, from_layout
    rng = np.random.default_rng(9000 + case)
    dtype = ["f32", "tf32", "bf16", "f16"][case % 4]
    layout = ["nhwc", "nchw"][(case // 4) % 2]
    dw = case % 6 == 5
    c = int(rng.choice([3, 8, 16, 64, 96, 128]))
    k = c if dw else int(rng.choice([8, 24, 64, 80, 128, 200]))
    r, s = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    st, pd, dl = int(rng.integers(1, 3)), int(rng.integers(0, 3)), int(rng.integers(1, 3))
    h = dl * (r - 1) + 1 + int(rng.integers(0, 12))
    w_ = dl * (s - 1) + 1 + int(rng.integers(0, 12))
    n = int(rng.integers(1, 4))
    Lc = ConvLayer(f"rand{case}", n, c, h, w_, k, r, s, st, pd, dl, c if dw else 1)
    x, w, b = workloads.generate(Lc, dtype, "int", seed=case)
    ref = oracle_full(Lc, x, w, b)
    plan = Conv2dPlan(Lc.n, Lc.c, Lc.h, Lc.w, Lc.k, Lc.r, Lc.s, Lc.stride, Lc.pad, Lc.dil, Lc.groups,
                      layout=layout, dtype=dtype)
    xl, wl = to_layout(x, w, layout)
    xl, wl, bc = xl.cuda(), wl.cuda(), b.cuda()
    fam = plan.config[0]
    names, doms = L.family_describe(["simt", "umma", "dw", "gemm32"][fam])
    configs = [plan.config]
    tries = 0
    while len(configs) < 4 and tries < 400:
        tries += 1
        genes = [int(rng.choice(d)) for d in doms]
        if plan.config_valid(fam, genes):
            configs.append((fam, genes))
    for fam_, genes in configs:
        plan.set_config(fam_, list(genes))
        y = plan.run(xl, wl, bc)
        torch.cuda.synchronize()
        assert_bit_exact(from_layout(y.cpu(), layout), ref)


@pytest.mark.parametrize("dtype", ["bf16", "f16", "tf32"])
@pytest.mark.parametrize("layout", ["nhwc", "nchw"])
def test_umma_dual_accumulators(dtype, layout):
    """MODE bit 2 (two accumulators per 128-row tile, even / odd K steps, summed by the epilogue):
    bit-exact on exact-integer inputs through the TMA-store and the direct (NCHW) epilogues, within
    tolerance on uniform inputs, and with the residual epilogue."""
    from paper_2008_04567_b200 import Conv2dPlan
    import oracle
    L = ConvLayer("dual", 3, 128, 14, 14, 192, 3, 3, 1, 1)
    for mode in ["int", "uniform"]:
        x, w, b = workloads.generate(L, dtype, mode, seed=31)
        ref = oracle_full(L, x, w, b)
        for genes in ([128, 4, 1, 4, 0, 2, 128], [64, 5, 1, 5, 0, 1, 128], [192, 3, 1, 4, 0, 1, 128]):
            y, plan = run_product(L, dtype, layout, x, w, b, config=(1, genes))
            assert plan.config[1][3] == genes[3]
            if mode == "int":
                assert_bit_exact(y, ref)
            else:
                assert rel_error(dtype, y, ref) <= TOL[dtype]
    # residual epilogue through the dual variant
    x, w, b = workloads.generate(L, dtype, "int", seed=32)
    z = torch.randint(-3, 4, (L.n, L.k, 14, 14)).to(x.dtype)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout=layout, dtype=dtype,
                      epilogue="bias_add_relu")
    plan.set_config(1, [128, 4, 1, 4, 0, 2, 128])
    xl, wl = to_layout(x, w, layout)
    zl = z.permute(0, 2, 3, 1).contiguous() if layout == "nhwc" else z
    yd = plan.run(xl.cuda(), wl.cuda(), b.cuda(), z=zl.cuda())
    torch.cuda.synchronize()
    assert_bit_exact(from_layout(yd.cpu(), layout), oracle.conv2d(x, w, b, stride=1, pad=1, residual=z))
