"""System-level selection: the per-layer choice between the
tuned WPK kernel and the box's cuDNN is made with the tuner's timing protocol, persisted next to
the tuning cache, and USED: SelectedConv2d dispatches every call to the chosen implementation.
Also the binding's argument checks on y / b / host buffers (a wrong buffer must raise, never reach
the kernel)."""
import os

import pytest
import torch

import oracle
import workloads
from workloads import ConvLayer

from _util import TOL, rel_error

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _setup():
    oracle.build()
    torch.cuda.set_device(0)


def _case(L, dtype, epilogue="bias_relu", seed=5):
    from paper_2008_04567_b200 import Conv2dPlan
    x, w, b = workloads.generate(L, dtype, "uniform", seed=seed)
    plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, layout="nhwc", dtype=dtype,
                      epilogue=epilogue)
    xd = x.permute(0, 2, 3, 1).contiguous().cuda()
    wd = w.permute(0, 2, 3, 1).contiguous().cuda()
    return plan, x, w, b, xd, wd, b.cuda()


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_dispatch_both_choices_match_oracle(dtype):
    from paper_2008_04567_b200.selector import SelectedConv2d
    L = ConvLayer("s", 4, 64, 14, 14, 128, 3, 3, 1, 1)
    plan, x, w, b, xd, wd, bd = _case(L, dtype)
    ref = oracle.conv2d(x, w, b, stride=1, pad=1)
    sc = SelectedConv2d(plan, L.stride, L.pad, L.dil)
    for choice, variant in (("wpk", None), ("cudnn", "cudnn_convolution_relu"), ("cudnn", "conv2d+relu_")):
        sc.choice, sc.variant, sc._fns = choice, variant, {}
        y = sc(xd, wd, bd)
        torch.cuda.synchronize()
        assert tuple(y.shape) == plan.y_shape()
        got = y.permute(0, 3, 1, 2).float().cpu()
        assert rel_error(dtype, got, ref) <= TOL[dtype], (choice, variant)


def test_select_persists_and_reloads(tmp_path):
    from paper_2008_04567_b200.selector import SelectedConv2d
    L = ConvLayer("s", 8, 256, 14, 14, 256, 1, 1, 1, 0)
    plan, x, w, b, xd, wd, bd = _case(L, "bf16")
    sc = SelectedConv2d(plan, L.stride, L.pad, L.dil, cache_dir=str(tmp_path))
    sel = sc.select(xd, wd, bd, reps=5)
    assert sel.choice in ("wpk", "cudnn")
    assert sel.choice == ("wpk" if sel.own_us <= sel.cudnn_us else "cudnn")    # ties -> own kernel
    files = os.listdir(tmp_path)
    assert len(files) == 1 and files[0].startswith("sel_")
    sc2 = SelectedConv2d(plan, L.stride, L.pad, L.dil, cache_dir=str(tmp_path))
    assert sc2.load() and sc2.choice == sel.choice
    # the choice was made for the plan's config: another config invalidates it
    fam, genes = plan.config
    alt = None
    for bn in (64, 128, 256):
        for st in (2, 3, 4):
            g = [bn, st] + list(genes[2:])
            if g != list(genes) and plan.config_valid(fam, g):
                alt = g
                break
        if alt:
            break
    assert alt is not None
    plan.set_config(fam, alt)
    assert not SelectedConv2d(plan, L.stride, L.pad, L.dil, cache_dir=str(tmp_path)).load()
    # dispatching through the loaded choice gives the right answer
    plan.set_config(fam, genes)
    y = sc2(xd, wd, bd)
    torch.cuda.synchronize()
    ref = oracle.conv2d(x, w, b)
    assert rel_error("bf16", y.permute(0, 3, 1, 2).float().cpu(), ref) <= TOL["bf16"]


def test_selected_step_in_cuda_graph():
    """Mixed dispatch (one layer on each implementation) captured in ONE CUDA graph, as the bench's
    selector_step does, replays to the oracle's values."""
    from paper_2008_04567_b200.selector import SelectedConv2d
    la = ConvLayer("a", 2, 64, 14, 14, 64, 3, 3, 1, 1)
    lb = ConvLayer("b", 2, 64, 14, 14, 256, 1, 1, 1, 0)
    pa, xa, wa, ba, xda, wda, bda = _case(la, "bf16", seed=7)
    pb, xb, wb, bb, xdb, wdb, bdb = _case(lb, "bf16", seed=8)
    sa, sb = SelectedConv2d(pa, 1, 1, 1), SelectedConv2d(pb, 1, 0, 1)
    sa.choice, sb.choice, sb.variant = "wpk", "cudnn", "cudnn_convolution_relu"
    ya = torch.empty(pa.y_shape(), dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.Stream()
    outs = {}

    def step():
        sa(xda, wda, bda, ya, stream=st)
        outs["b"] = sb(xdb, wdb, bdb, stream=st)
    with torch.cuda.stream(st):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        step()
    ya.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert rel_error("bf16", ya.permute(0, 3, 1, 2).float().cpu(), oracle.conv2d(xa, wa, ba, pad=1)) <= TOL["bf16"]
    assert rel_error("bf16", outs["b"].permute(0, 3, 1, 2).float().cpu(), oracle.conv2d(xb, wb, bb)) <= TOL["bf16"]


def test_binding_rejects_bad_buffers():
    L = ConvLayer("s", 2, 64, 8, 8, 64, 3, 3, 1, 1)
    plan, x, w, b, xd, wd, bd = _case(L, "bf16")
    with pytest.raises(ValueError):
        plan.run(xd, wd, bd, torch.empty(1, dtype=torch.bfloat16, device="cuda"))          # y too small
    with pytest.raises(ValueError):
        plan.run(xd, wd, bd, torch.empty(plan.y_shape(), dtype=torch.float16, device="cuda"))  # y dtype
    with pytest.raises(ValueError):
        plan.run(xd, wd, bd.float())                                                       # bias dtype
    with pytest.raises(ValueError):
        plan.run(xd, wd, bd[:10])                                                          # bias shape
    yh = torch.empty(plan.y_shape(), dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        plan.run_host(xd, wd, bd, yh)                                                      # x_host on the GPU
    with pytest.raises(ValueError):
        plan.run_host(xd.cpu(), wd, bd, torch.empty(3, dtype=torch.bfloat16))               # y_host too small
    plan.run_host(xd.cpu(), wd, bd, yh)                                                    # the right buffers work
    ref = oracle.conv2d(x, w, b, pad=1)
    assert rel_error("bf16", yh.permute(0, 3, 1, 2).float(), ref) <= TOL["bf16"]
