"""Host cost of one Conv2dPlan.run() call, split: Python wrapper + ctypes, C entry (validation,
workspace, geometry), kernel launch. usage: python tools/host_overhead.py"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan

L = next(l for l in workloads.resnet50(32) if l.name == "s4b1.c2")
plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
x, w, b = workloads.generate(L, "bf16", "uniform", seed=1)
xd = x.permute(0, 2, 3, 1).contiguous().cuda(); wd = w.permute(0, 2, 3, 1).contiguous().cuda(); bd = b.cuda()
y = torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda")
plan.run(xd, wd, bd, y); torch.cuda.synchronize()
N = 300
s = torch.cuda.current_stream().cuda_stream
lib = plan.lib
args = [plan.handle, ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(wd.data_ptr()), ctypes.c_void_p(bd.data_ptr()),
        ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(s)]
def timeit(f):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(N): f()
    t1 = time.perf_counter(); torch.cuda.synchronize()
    return (t1 - t0) / N * 1e6
print(f"plan.run (Python wrapper + C + launch): {timeit(lambda: plan.run(xd, wd, bd, y)):.1f} us")
print(f"raw ctypes wpk_conv2d_run:              {timeit(lambda: lib.wpk_conv2d_run(*args)):.1f} us")
print(f"ctypes trivial call (last_launch_count): {timeit(lambda: lib.wpk_conv2d_last_launch_count(plan.handle)):.1f} us")
k = torch.empty(1, device="cuda")
print(f"torch tiny kernel launch (k.add_(1)):   {timeit(lambda: k.add_(1)):.1f} us")
