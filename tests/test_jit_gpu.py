"""JIT family on the GPU: generated + NVRTC-compiled kernels match the oracle (bit-exact on
exact-integer inputs, within tolerance on uniform inputs), agree bit for bit with the precompiled
SIMT family for the same genes, and the tuner searches the JIT space with multi-threaded
compilation and its cache."""
import pytest
import torch

import workloads
from workloads import ConvLayer
from _util import TOL, assert_bit_exact, oracle_full, rel_error, run_product

pytestmark = pytest.mark.gpu

SHAPES = [
    ConvLayer("j3x3", 2, 13, 9, 11, 24, 3, 3, 1, 1),
    ConvLayer("j_s2_d2", 3, 8, 17, 15, 10, 3, 3, 2, 2, dil=2),
    ConvLayer("j1x1", 2, 40, 7, 7, 33, 1, 1, 1, 0),
    ConvLayer("j7x7", 1, 3, 20, 20, 16, 7, 7, 2, 3),
    ConvLayer("jgrp", 2, 12, 8, 8, 18, 3, 3, 1, 1, groups=3),
]
GENES = [[8, 4, 4, 2, 1, 2, 4], [16, 4, 2, 1, 2, 1, 1], [4, 8, 8, 1, 1, 4, 8]]


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("L", SHAPES, ids=lambda l: l.name)
def test_jit_bit_exact_integer_mode(L, layout, dtype):
    x, w, b = workloads.generate(L, dtype, "int", seed=21)
    ref = oracle_full(L, x, w, b)
    for genes in GENES:
        y, plan = run_product(L, dtype, layout, x, w, b, config=("jit", genes))
        assert plan.config[0] == 4
        assert_bit_exact(y, ref)


@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16"])
def test_jit_uniform_tolerance(dtype):
    L = ConvLayer("ju", 2, 64, 14, 14, 48, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, dtype, "uniform", seed=22)
    y, _ = run_product(L, dtype, "nhwc", x, w, b, config=("jit", [16, 4, 4, 1, 2, 2, 8]))
    assert rel_error(dtype, y, oracle_full(L, x, w, b)) <= TOL[dtype]


def test_jit_equals_simt_bit_for_bit():
    L = ConvLayer("jsame", 2, 32, 12, 12, 40, 3, 3, 1, 1)
    for dtype in ["f32", "bf16"]:
        x, w, b = workloads.generate(L, dtype, "uniform", seed=23)
        genes = [8, 4, 4, 2, 2, 1, 1]
        yj, _ = run_product(L, dtype, "nchw", x, w, b, config=("jit", genes))
        ys, _ = run_product(L, dtype, "nchw", x, w, b, config=("simt", genes))
        assert torch.equal(yj.view(torch.int16 if dtype != "f32" else torch.int32),
                           ys.view(torch.int16 if dtype != "f32" else torch.int32))


def test_jit_residual_epilogue():
    from paper_2008_04567_b200 import Conv2dPlan
    import oracle
    L = ConvLayer("jres", 2, 16, 8, 8, 16, 3, 3, 1, 1)
    x, w, b = workloads.generate(L, "f32", "int", seed=24)
    z = torch.randint(-3, 4, (L.n, L.k, 8, 8)).float()
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nchw", dtype="f32",
                      epilogue="bias_add_relu")
    plan.set_config("jit", [8, 8, 2, 1, 1, 2, 2])
    y = plan.run(x.cuda(), w.cuda(), b.cuda(), z=z.cuda())
    torch.cuda.synchronize()
    ref = oracle.conv2d(x, w, b, stride=1, pad=1, residual=z)
    assert_bit_exact(y.cpu(), ref)


def test_jit_tune_compiles_then_hits_cache(tmp_path):
    from paper_2008_04567_b200 import Conv2dPlan, _lib as L_
    L = ConvLayer("jt", 4, 32, 14, 14, 64, 3, 3, 1, 1)
    s0 = L_.jit_stats()
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    res = plan.tune("ga", 12, seed=5, family="jit", warmup=1, reps=3, finalists=0, ga_pop=6, ga_pool=6,
                    ga_elites=1, log_path=str(tmp_path / "log.jsonl"))
    assert res.family == 4 and res.measured <= 12 and res.best_us > 0
    s1 = L_.jit_stats()
    assert s1["compiles"] - s0["compiles"] >= 1 and s1["failures"] == s0["failures"]
    assert "jit_compile_seconds" in open(tmp_path / "log.jsonl").read()
    x, w, b = workloads.generate(L, "bf16", "int", seed=25)
    y, _ = run_product(L, "bf16", "nhwc", x, w, b, config=("jit", res.genes))
    assert_bit_exact(y, oracle_full(L, x, w, b))
    # the same search again: every candidate is already compiled
    plan2 = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    plan2.tune("ga", 12, seed=5, family="jit", warmup=1, reps=3, finalists=0, ga_pop=6, ga_pool=6, ga_elites=1)
    assert L_.jit_stats()["compiles"] == s1["compiles"]
