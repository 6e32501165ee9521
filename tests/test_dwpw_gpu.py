"""GPU parity of the fused depthwise + pointwise kernel (wpk_dwpw_plan / wpk_dwpw_run; SURVEY.md
8(f) NEXT-4, the MobileNet block; PAPER.md:15 / :35 operator fusion).

The reference is the oracle chain written out: t = RN_dtype(oracle.conv2d(x, w_dw, b_dw, groups=C))
(the depthwise conv exactly as the unfused path stores it), then y = oracle.conv2d(t, w_pw, b_pw)
(reading "fused dw+pw" in DESIGN.md). Exact-integer inputs: every depthwise output is an integer
|t| <= R*S + 4, exact in bf16/fp16, and every pointwise sum an integer < 2^24, so the GPU result must
equal RN(oracle) bit for bit; uniform inputs within the 16-bit normwise bound."""
import itertools

import numpy as np
import pytest
import torch

import oracle
import workloads
from workloads import ConvLayer

from _util import TOL, assert_bit_exact, rel_error

pytestmark = pytest.mark.gpu

# (name, n, c, h, w, k_out, stride, pad, dil): MobileNet-V2-like depthwise widths (C = 6 x C_in),
# ragged channel blocks (144 = 2.25 x 64, 24 < 64), stride 2, dilation, odd spatial sizes
CASES = [
    ("mb_s1", 2, 144, 14, 14, 24, 1, 1, 1),
    ("mb_s2", 2, 96, 15, 13, 24, 2, 1, 1),
    ("mb_wide", 1, 576, 7, 9, 160, 1, 1, 1),
    ("c24", 3, 24, 11, 10, 40, 1, 1, 1),
    ("dil2", 1, 64, 12, 12, 72, 1, 2, 2),
    ("k200", 2, 128, 9, 11, 200, 1, 1, 1),
]


@pytest.fixture(scope="module", autouse=True)
def _setup():
    oracle.build()
    torch.cuda.set_device(0)


def _inputs(case, dtype, mode, seed):
    name, n, c, h, w, k, st, pad, dil = case
    dwl = ConvLayer(name + "_dw", n, c, h, w, c, 3, 3, st, pad, dil, c)
    x, w_dw, b_dw = workloads.generate(dwl, dtype, mode, seed=seed)
    p = (h + 2 * pad - dil * 2 - 1) // st + 1
    q = (w + 2 * pad - dil * 2 - 1) // st + 1
    pwl = ConvLayer(name + "_pw", n, c, p, q, k, 1, 1, 1, 0)
    _, w_pw, b_pw = workloads.generate(pwl, dtype, mode, seed=seed + 1)
    return x, w_dw, b_dw, w_pw, b_pw, (st, pad, dil)


def _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, dt, dw_epi="bias_relu", pw_epi="bias"):
    st, pad, dil = conv
    c = x.shape[1]
    t = oracle.conv2d(x, w_dw, b_dw if dw_epi != "none" else None, stride=st, pad=pad, dil=dil, groups=c,
                      relu=(dw_epi == "bias_relu"))
    t = torch.from_numpy(t).to(dt)                       # the depthwise result as the I/O dtype stores it
    return oracle.conv2d(t, w_pw, b_pw if pw_epi != "none" else None, relu=(pw_epi == "bias_relu"))


def _run(plan, x, w_dw, b_dw, w_pw, b_pw, dw_epi="bias_relu", pw_epi="bias"):
    xd = x.permute(0, 2, 3, 1).contiguous().cuda()
    y = plan.run(xd, w_dw.contiguous().cuda(), b_dw.cuda() if dw_epi != "none" else None,
                 w_pw.contiguous().cuda(), b_pw.cuda() if pw_epi != "none" else None)
    torch.cuda.synchronize()
    return y.cpu().permute(0, 3, 1, 2).contiguous()


def _plan(case, dtype, dw_epi="bias_relu", pw_epi="bias"):
    from paper_2008_04567_b200 import DwPwPlan
    name, n, c, h, w, k, st, pad, dil = case
    return DwPwPlan(n, c, h, w, k, 3, 3, st, pad, dil, dw_epilogue=dw_epi, pw_epilogue=pw_epi, dtype=dtype)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_dwpw_default_int_bit_exact(case, dtype):
    """Both fused kernels (A_MODE 1, the default: one tile per CTA; A_MODE 0: the persistent kernel's
    depthwise producer) bit-exact against the oracle chain."""
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, dtype, "int", seed=91)
    plan = _plan(case, dtype)
    assert plan.config[0] == 1
    ref = _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, workloads.torch_dtype(dtype))
    assert_bit_exact(_run(plan, x, w_dw, b_dw, w_pw, b_pw), ref)
    g = plan.config[1]
    if g[4] == 1:
        plan.set_config(1, [g[0], 4, 1, 0, 0, 2, 128])
        assert_bit_exact(_run(plan, x, w_dw, b_dw, w_pw, b_pw), ref)


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_dwpw_uniform_tolerance(case):
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "uniform", seed=92)
    y = _run(_plan(case, "bf16"), x, w_dw, b_dw, w_pw, b_pw)
    err = rel_error("bf16", y, _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, torch.bfloat16))
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("dw_epi,pw_epi", [("none", "none"), ("bias", "bias_relu"), ("bias_relu", "bias_relu"),
                                           ("bias_relu", "bias")])
def test_dwpw_epilogues(dw_epi, pw_epi):
    case = CASES[0]
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "int", seed=93)
    y = _run(_plan(case, "bf16", dw_epi, pw_epi), x, w_dw, b_dw, w_pw, b_pw, dw_epi, pw_epi)
    assert_bit_exact(y, _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, torch.bfloat16, dw_epi, pw_epi))


def test_dwpw_every_config_bit_exact():
    """Every valid config of a sweep (BLOCK_N covering K_out, STAGES, SPLIT_K through L2, raster,
    accumulator stages, BLOCK_M 128 / 256): the tiling changes speed, never values."""
    case = ("sweep", 2, 200, 11, 13, 136, 1, 1, 1)    # C = 200: 4 channel blocks, the last one 8 wide
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "int", seed=94)
    ref = _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, torch.bfloat16)
    plan = _plan(case, "bf16")
    xd = x.permute(0, 2, 3, 1).contiguous().cuda()
    args = (w_dw.cuda(), b_dw.cuda(), w_pw.contiguous().cuda(), b_pw.cuda())
    n = 0
    for genes in itertools.product([16, 32, 64, 96, 128, 192, 256], [2, 4, 7], [1, 2, 4], [0, 1], [0, 1], [1, 2, 4],
                                   [128, 256]):
        genes = list(genes)
        if not plan.config_valid(1, genes):
            continue
        plan.set_config(1, genes)
        y = plan.run(xd, *args)
        torch.cuda.synchronize()
        assert_bit_exact(y.cpu().permute(0, 3, 1, 2).contiguous(), ref)
        n += 1
    assert n >= 40
    assert not plan.config_valid(1, [128, 4, 1, 2, 0, 2, 256])   # no CTA pairs
    assert plan.config_valid(1, [192, 2, 1, 0, 1, 1, 128])       # A_MODE 1: the one-tile-per-CTA kernel
    assert not plan.config_valid(1, [128, 4, 1, 0, 4, 2, 128])   # A_MODE 0 / 1 only


def test_dwpw_equals_unfused_product_chain():
    """The fused kernel equals the library's own unfused chain (depthwise family -> bf16 t ->
    tcgen05 1x1) bit for bit on exact-integer inputs."""
    from paper_2008_04567_b200 import Conv2dPlan
    case = CASES[1]
    name, n, c, h, w, k, st, pad, dil = case
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "int", seed=95)
    y = _run(_plan(case, "bf16"), x, w_dw, b_dw, w_pw, b_pw)
    pdw = Conv2dPlan(n, c, h, w, c, 3, 3, st, pad, dil, c, layout="nhwc", dtype="bf16")
    t = pdw.run(x.permute(0, 2, 3, 1).contiguous().cuda(), w_dw.permute(0, 2, 3, 1).contiguous().cuda(), b_dw.cuda())
    ppw = Conv2dPlan(n, c, pdw.p, pdw.q, k, 1, 1, 1, 0, layout="nhwc", epilogue="bias", dtype="bf16")
    y2 = ppw.run(t, w_pw.permute(0, 2, 3, 1).contiguous().cuda(), b_pw.cuda())
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), y2.cpu().permute(0, 3, 1, 2).contiguous().view(torch.int16))


def test_dwpw_tune_then_parity():
    """The tuner measures fused candidates (it allocates the depthwise operands itself); the chosen
    config is bit-exact."""
    case = ("t", 4, 144, 28, 28, 32, 1, 1, 1)
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "int", seed=96)
    plan = _plan(case, "bf16")
    res = plan.tune("ga", 16, seed=2)
    assert res.measured >= 1 and res.best_us < float("inf") and res.genes[4] in (0, 1)
    y = _run(plan, x, w_dw, b_dw, w_pw, b_pw)
    assert_bit_exact(y, _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, torch.bfloat16))


def test_dwpw_mobilenet_v2_n32_sampled():
    """A full-size MobileNet-V2 N=32 block pair (the 56x56 stride-1 dw 3x3 over 144 channels into the
    1x1 projection to 24): sampled outputs (every border pixel of every image x 8 channels + 65,536
    interior points) against the oracle chain, point by point on the pointwise side."""
    case = ("mb32", 32, 144, 56, 56, 24, 1, 1, 1)
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "uniform", seed=97)
    y = _run(_plan(case, "bf16"), x, w_dw, b_dw, w_pw, b_pw)
    t = oracle.conv2d(x, w_dw, b_dw, stride=1, pad=1, groups=144, nthreads=8)
    t = torch.from_numpy(t).to(torch.bfloat16)
    L = ConvLayer("mb32_pw", 32, 144, 56, 56, 24, 1, 1, 1, 0)
    pts = workloads.parity_points(L, 56, 56, interior=65536, seed=98, border_channels=8)
    ref = oracle.conv2d_points(t, w_pw, b_pw, pts.numpy(), relu=False, nthreads=8)
    got = y[pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]].double().numpy()
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("splits", [2, 4, 8])
def test_dwpw_one_tile_kernel_split_k(splits):
    """A_MODE 1 with SPLIT_K: the 64-channel chunks of a deep block (C = 960) split over CTAs, fp32
    partials summed in split order by the reduction kernel (bias / epilogue there): bit-exact on
    exact-integer inputs, within tolerance on uniform inputs."""
    case = ("deep", 2, 960, 7, 9, 160, 1, 1, 1)
    genes = [192, 2, splits, 0, 1, 1, 128]
    for mode in ("int", "uniform"):
        plan = _plan(case, "bf16")   # a fresh plan: the packed depthwise weights are cached per pointer
        assert plan.config_valid(1, genes)
        plan.set_config(1, genes)
        x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", mode, seed=99)
        ref = _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, torch.bfloat16)
        y = _run(plan, x, w_dw, b_dw, w_pw, b_pw)
        if mode == "int":
            assert_bit_exact(y, ref)
        else:
            assert rel_error("bf16", y, ref) <= TOL["bf16"]


def test_dwpw_tune_sparse_space_k320():
    """K_out = 320 leaves only a handful of valid fused configs in the 7-gene space: the GA's rejection
    sampler falls back to the expert-template default instead of failing (reading "sparse spaces"),
    and the tuned plan is bit-exact."""
    case = ("k320", 2, 960, 7, 7, 320, 1, 1, 1)
    x, w_dw, b_dw, w_pw, b_pw, conv = _inputs(case, "bf16", "int", seed=111)
    plan = _plan(case, "bf16")
    res = plan.tune("ga", 16, seed=5)
    assert res.measured >= 1 and res.best_us < float("inf")
    assert_bit_exact(_run(plan, x, w_dw, b_dw, w_pw, b_pw),
                     _oracle_chain(x, w_dw, b_dw, w_pw, b_pw, conv, torch.bfloat16))
