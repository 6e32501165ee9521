"""Per-conv phases inside the bench's whole-step CUDA graph (globaltimer stamps written by CTA
threads; needs the debug hook wpk_debug_set_plan_timeline): for each conv, relative to the step
start: first CTA start, median CTA setup done, first stage full, last CTA end. Shows the bubbles
between consecutive kernels under programmatic dependent launch.
usage: python tools/step_timeline.py CONFIGS_JSON"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the production library compiles the stamps out: use the timeline build (make -C
# paper_2008_04567_b200/csrc timeline)
_TL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2008_04567_b200",
                   "libwpk_timeline.so")
if not os.environ.get("WPK_LIB"):
    if not os.path.exists(_TL):
        sys.exit(f"{_TL} missing: run `make -C paper_2008_04567_b200/csrc -j16 timeline`")
    os.environ["WPK_LIB"] = _TL
import numpy as np
import torch
import workloads
from paper_2008_04567_b200 import Conv2dPlan, _lib

cfgs = json.load(open(sys.argv[1]))
lib = _lib.load()
lib.wpk_debug_set_plan_timeline.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
units = []
for i, L in enumerate(workloads.resnet50(32)):
    for c in range(L.count):
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
        plan.set_config(*cfgs[L.name])
        x, w, b = workloads.generate(L, "bf16", "uniform", seed=workloads.config_seed(1, i) + 7919 * c)
        dbg = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
        lib.wpk_debug_set_plan_timeline(plan.handle, ctypes.c_void_p(dbg.data_ptr()))
        units.append((f"{L.name}#{c}", plan, x.permute(0, 2, 3, 1).contiguous().cuda(),
                      w.permute(0, 2, 3, 1).contiguous().cuda(), b.cuda(),
                      torch.empty(plan.y_shape(), dtype=torch.bfloat16, device="cuda"), dbg))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for u in units:
        u[1].run(*u[2:6], stream=st)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for u in units:
        u[1].run(*u[2:6], stream=st)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for u in units:
    u[6].zero_()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
rows = []
for u in units:
    t = u[6].view(148, 64).cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]
    rows.append((u[0], t[:, 0].min(), np.median(t[:, 1]), t[:, 2][t[:, 2] > 0].min() if (t[:, 2] > 0).any() else 0,
                 t[:, 6].max(), len(t), t[:, 7][t[:, 7] > 0].min() if (t[:, 7] > 0).any() else 0))
t0 = rows[0][1]
print(f"{'conv':10s} {'start':>8s} {'setup':>8s} {'1stfull':>8s} {'end':>8s} {'dur':>7s} {'gap':>7s} CTAs "
      f"{'wait':>7s} {'load':>7s}  (us from step start; wait = previous end -> first griddepcontrol.wait return, "
      f"load = that -> first full stage)")
prev_end = None
for (nm, s0, su, ff, e, n, wr) in rows:
    gap = (s0 - prev_end) / 1e3 if prev_end is not None else 0.0
    wt = (wr - prev_end) / 1e3 if (prev_end is not None and wr > 0) else float("nan")
    ld = (ff - wr) / 1e3 if (wr > 0 and ff > 0) else float("nan")
    print(f"{nm:10s} {(s0 - t0) / 1e3:8.2f} {(su - t0) / 1e3:8.2f} {(ff - t0) / 1e3:8.2f} {(e - t0) / 1e3:8.2f} "
          f"{(e - s0) / 1e3:7.2f} {gap:7.2f} {n} {wt:7.2f} {ld:7.2f}")
    prev_end = e
print(f"step span {(rows[-1][4] - t0) / 1e3:.1f} us")
