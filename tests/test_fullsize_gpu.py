"""Full-size parity at the BASELINE.json configurations, in the tuned configurations the suites and
the bench report ("Full-tensor parity for configs 1, 2 (N=1), 4, and for small
shapes. Sampled parity for N>=32: all border rows/columns + >= 65,536 random interior outputs per
layer"; each sampled output is an independent dot product, so the check is exact per element).

  * ResNet-50 N=32 bf16 (configs[1]) in the bench's committed tuned configs;
  * ResNet-50 N=32 TF32 (configs[1]) and VGG-16 N=64 fp16 (configs[2], RL-tuned) in the suite's
    committed tuned configs (profiles/r2_suite_tuned_configs.json), sampled;
  * MobileNet-V2 N=32 bf16 in its suite configs, sampled;
  * ResNet-50 N=1 bf16 (configs[1]) and MobileNet-V2 N=1 bf16 (configs[3]): the WHOLE output tensor.

Exact-integer inputs must be bit-exact (reading c11); uniform inputs must meet BASELINE.json's
tolerances (bf16/fp16 normwise 2e-2, TF32 normwise 5e-3) on the same points."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import workloads

from _util import TOL, assert_bit_exact, oracle_full, rel_error, run_product

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = json.load(open(os.path.join(ROOT, "profiles", "r2_suite_tuned_configs.json")))
BENCH_CFG = os.path.join(ROOT, "profiles", "bench_tuned_configs.json")
NCPU = os.cpu_count() or 8


@pytest.fixture(scope="module", autouse=True)
def _setup():
    oracle.build()
    torch.cuda.set_device(0)


def _sampled_check(layer, dtype, mode, y, x, w, b, seed, border_channels=None):
    """y: the product's output in NCHW (CPU). Compares all-border + 65,536 interior points."""
    p, q = y.shape[2], y.shape[3]
    pts = workloads.parity_points(layer, p, q, 65536, seed=seed, border_channels=border_channels)
    ref = oracle.conv2d_points(x, w, b, pts.numpy(), stride=layer.stride, pad=layer.pad, dil=layer.dil,
                               groups=layer.groups, nthreads=NCPU)
    got = y[pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    if mode == "int":
        assert_bit_exact(got, ref)
    else:
        err = rel_error(dtype, got, ref)
        assert err <= TOL[dtype], (layer.name, err)
    return int(pts.shape[0])


def _bench_configs():
    if os.path.exists(BENCH_CFG):
        return json.load(open(BENCH_CFG))
    return json.load(open(os.path.join(ROOT, "profiles", "r1k_tuned_configs.json")))


@pytest.mark.parametrize("mode", ["int", "uniform"])
@pytest.mark.parametrize("layer", workloads.resnet50(32), ids=lambda l: l.name)
def test_resnet50_n32_bf16_bench_configs(layer, mode):
    fam, genes = _bench_configs()[layer.name]
    x, w, b = workloads.generate(layer, "bf16", mode, seed=workloads.config_seed(1, 40))
    y, _ = run_product(layer, "bf16", "nhwc", x, w, b, config=(fam, genes))
    assert _sampled_check(layer, "bf16", mode, y, x, w, b, seed=1) >= 65536


@pytest.mark.parametrize("mode", ["int", "uniform"])
@pytest.mark.parametrize("layer", workloads.resnet50(32), ids=lambda l: l.name)
def test_resnet50_n32_tf32_suite_configs(layer, mode):
    fam, genes = SUITE["resnet50_tf32"]["layers"][layer.name]
    x, w, b = workloads.generate(layer, "tf32", mode, seed=workloads.config_seed(1, 60))
    y, _ = run_product(layer, "tf32", "nhwc", x, w, b, config=(fam, genes))
    _sampled_check(layer, "tf32", mode, y, x, w, b, seed=2)


@pytest.mark.parametrize("mode", ["int", "uniform"])
@pytest.mark.parametrize("layer", workloads.vgg16(64), ids=lambda l: l.name)
def test_vgg16_n64_f16_rl_suite_configs(layer, mode):
    fam, genes = SUITE["vgg16"]["layers"][layer.name]
    x, w, b = workloads.generate(layer, "f16", mode, seed=workloads.config_seed(2, 60))
    y, _ = run_product(layer, "f16", "nhwc", x, w, b, config=(fam, genes))
    # 224x224 layers: 892 border pixels x 64 images -> all K channels of every border pixel
    _sampled_check(layer, "f16", mode, y, x, w, b, seed=3)


@pytest.mark.parametrize("mode", ["int", "uniform"])
@pytest.mark.parametrize("layer", workloads.resnet50(1), ids=lambda l: l.name)
def test_resnet50_n1_bf16_suite_configs_full_tensor(layer, mode):
    fam, genes = SUITE["resnet50_n1"]["layers"][layer.name]
    x, w, b = workloads.generate(layer, "bf16", mode, seed=workloads.config_seed(1, 80))
    y, _ = run_product(layer, "bf16", "nhwc", x, w, b, config=(fam, genes))
    ref = oracle.conv2d(x, w, b, stride=layer.stride, pad=layer.pad, dil=layer.dil, groups=layer.groups,
                        nthreads=NCPU)
    if mode == "int":
        assert_bit_exact(y, ref)
    else:
        assert rel_error("bf16", y, ref) <= TOL["bf16"]


@pytest.mark.parametrize("mode", ["int", "uniform"])
@pytest.mark.parametrize("layer", workloads.mobilenet_v2(1), ids=lambda l: l.name)
def test_mobilenet_v2_n1_bf16_suite_configs_full_tensor(layer, mode):
    fam, genes = SUITE["mobilenet_v2"]["layers"][layer.name]
    x, w, b = workloads.generate(layer, "bf16", mode, seed=workloads.config_seed(3, 80))
    y, _ = run_product(layer, "bf16", "nhwc", x, w, b, config=(fam, genes))
    ref = oracle_full(layer, x, w, b)
    if mode == "int":
        assert_bit_exact(y, ref)
    else:
        assert rel_error("bf16", y, ref) <= TOL["bf16"]



@pytest.mark.parametrize("mode", ["int", "uniform"])
@pytest.mark.parametrize("layer", workloads.mobilenet_v2(32), ids=lambda l: l.name)
def test_mobilenet_v2_n32_bf16_suite_configs(layer, mode):
    fam, genes = SUITE["mobilenet_v2_n32"]["layers"][layer.name]
    x, w, b = workloads.generate(layer, "bf16", mode, seed=workloads.config_seed(3, 90))
    y, _ = run_product(layer, "bf16", "nhwc", x, w, b, config=(fam, genes))
    _sampled_check(layer, "bf16", mode, y, x, w, b, seed=5)
