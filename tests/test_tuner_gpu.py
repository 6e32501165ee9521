"""Measured-mode tuning on the GPU: the sharded evaluator times real kernels with CUDA events;
the chosen config is valid, runs correctly, and is no slower than the default (within noise)."""
import pytest
import torch

import workloads
from workloads import ConvLayer
from _util import assert_bit_exact, oracle_full, run_product, to_layout, from_layout

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("search", ["ga", "random", "rl"])
def test_measured_tune_bf16(search, tmp_path):
    L = ConvLayer("t", 8, 64, 28, 28, 128, 3, 3, 1, 1)
    from paper_2008_04567_b200 import Conv2dPlan
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    default = plan.config
    rec = str(tmp_path / "rec.jsonl")
    kw = dict(rl_hidden=[64, 64, 64, 64], rl_horizon=8, rl_envs=4) if search == "rl" else {}
    res = plan.tune(search, 24, seed=1, record_path=rec, warmup=2, reps=5, **kw)
    assert res.measured <= 24 and res.best_us > 0
    assert len(open(rec).read().splitlines()) == res.measured
    x, w, b = workloads.generate(L, "bf16", "int", seed=3)
    xl, wl = to_layout(x, w, "nhwc")
    y = plan.run(xl.cuda(), wl.cuda(), b.cuda())
    torch.cuda.synchronize()
    assert_bit_exact(from_layout(y.cpu(), "nhwc"), oracle_full(L, x, w, b))
    # replaying the recorded timing set reproduces the same choice without touching the GPU
    plan2 = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
    res2 = plan2.tune(search, 24, seed=1, eval_mode="replay", replay_path=rec, **kw)
    assert res2.genes == res.genes and res2.best_us == res.best_us
