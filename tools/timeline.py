"""Per-CTA timeline of one tcgen05 conv launch (globaltimer ns, relative to the earliest CTA start):
start, setup done, first full stage, first tile MMAs issued, first tile epilogue done, all epilogues
done, CTA end.  usage: python tools/timeline.py LAYER [genes]
Note: the "end" stamp (thread 0 after the final CTA barrier) reads earlier than the epilogue warps'
"epi_all_done" stamp although a shared-memory flag written by the epilogue before the barrier is
always visible to thread 0 after it (checked): compare stamps within one warp's role only."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the production library compiles the stamps out: use the timeline build (make -C
# paper_2008_04567_b200/csrc timeline)
_TL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2008_04567_b200",
                   "libwpk_timeline.so")
if not os.environ.get("WPK_LIB"):
    if not os.path.exists(_TL):
        sys.exit(f"{_TL} missing: run `make -C paper_2008_04567_b200/csrc -j16 timeline`")
    os.environ["WPK_LIB"] = _TL
import torch, numpy as np
import workloads
from paper_2008_04567_b200 import Conv2dPlan, _lib

name = sys.argv[1]
net = os.environ.get("NET", "resnet50")
batch = int(os.environ.get("BATCH", {"resnet50": "32", "vgg16": "64", "mobilenet_v2": "1"}[net]))
L = next(l for l in getattr(workloads, net)(batch) if l.name == name)
plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype="bf16")
if len(sys.argv) > 2:
    plan.set_config(1, [int(v) for v in sys.argv[2:9]])
x, w, b = workloads.generate(L, "bf16", "uniform", seed=1)
xd = x.permute(0, 2, 3, 1).contiguous().cuda(); wd = w.permute(0, 2, 3, 1).contiguous().cuda(); bd = b.cuda()
y = torch.empty(plan.y_shape(), dtype=xd.dtype, device="cuda")
dbg = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.wpk_debug_set_timeline.argtypes = [ctypes.c_void_p]
for i in range(3):
    plan.run(xd, wd, bd, y)
torch.cuda.synchronize()
lib.wpk_debug_set_timeline(ctypes.c_void_p(dbg.data_ptr()))
flush = torch.ones(300 << 20, dtype=torch.uint8, device="cuda")
torch.sum(flush.view(torch.int32), dtype=torch.int64)
plan.run(xd, wd, bd, y)
torch.cuda.synchronize()
lib.wpk_debug_set_timeline(None)
t64 = dbg.view(148, 64).cpu().numpy().astype(np.float64)
t = t64[:, :16]
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t[:, :7] - t0) / 1000.0
names = ["start", "setup", "1st_full", "1st_mma_done", "1st_epi_done", "epi_all_done", "end"]
print(name, plan.config, "CTAs", len(t))
for i, n in enumerate(names):
    col = rel[:, i]
    col = col[col > -1e6]
    print(f"  {n:14s} min {col.min():8.2f}  median {np.median(col):8.2f}  max {col.max():8.2f} us")
if int(os.environ.get("WPK_DBG_FLAGS", "0")) & 128:   # MMA-loop cycle accounting, first tile
    c = t64[t64[:, 0] > 0][:, 60:64]
    nkb = np.maximum(c[:, 3], 1)
    print("  MMA loop, clk per K block (median over CTAs): wait %.0f  issue %.0f  total %.0f  (kb %d)" % (
        np.median(c[:, 0] / nkb), np.median(c[:, 1] / nkb), np.median(c[:, 2] / nkb), int(np.median(c[:, 3]))))
if int(os.environ.get("WPK_DBG_FLAGS", "0")) & 8:   # per-K-block stamps of the first tile, CTA 0
    r0 = t64[0]
    print("  CTA0 first tile, us:  A issued / B issued / stage full (MMA)")
    for kb in range(16):
        a_, b_, f_ = r0[16 + kb], r0[32 + kb], r0[48 + kb]
        if f_ > 0:
            print(f"   kb {kb:2d}  {(a_ - t0) / 1e3:7.2f} {(b_ - t0) / 1e3:7.2f} {(f_ - t0) / 1e3:7.2f}")
    sys.exit(0)
ev = t64[t64[:, 0] > 0][:, 16:64].reshape(-1, 8, 6)
print("  per-tile events of CTA 0 (us): tempty_ok, 1st_full, mma_commit, epi_tfull_ok, epi_done, [mma_seen_done]")
for it in range(8):
    row = ev[0, it, :6] if ev[0, it, 5] > 0 else ev[0, it, :5]
    if row[0] > 0:
        print("   tile", it, np.round((row - t0) / 1000.0, 2))
sk = t64[t64[:, 0] > 0][:, 56:60]
if (sk > 0).any():   # split-K (EK_SPLIT) first work item: publish / owner wait start / wait done / done
    for i, n in [(0, "splitk_published"), (3, "owner_wait_start"), (1, "owner_saw_all"), (2, "owner_done")]:
        col = sk[:, i]
        col = (col[col > 0] - t0) / 1000.0
        if len(col):
            print(f"  {n:16s} min {col.min():8.2f}  median {np.median(col):8.2f}  max {col.max():8.2f} us  (n={len(col)})")
fx = t[:, 8:14]
if os.environ.get("SPLITK_FIX") and (fx[:, 0] > 0).any():
    sel = fx[:, 0] > 0
    r = (fx[sel][:, [0, 1, 2, 3, 5]] - t0) / 1000.0
    for i, n in enumerate(["fix_enter", "fix_bulkwait", "fix_bar1", "fix_flag", "fix_final_done"]):
        col = r[:, i]
        col = col[col > 0]
        if len(col):
            print(f"  {n:14s} min {col.min():8.2f}  median {np.median(col):8.2f}  max {col.max():8.2f} us  (n={len(col)})")
    print("  final passes per CTA:", np.bincount(fx[sel][:, 4].astype(int)))
    slow = np.argmax(t[:, 5])
    print("  slowest CTA row (us):", np.round((t[slow, :14] - t0) / 1000.0, 2))

# event-timed duration of the same launch vs the in-kernel span, and host cost of one run() call
import time
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.sum(flush.view(torch.int32), dtype=torch.int64)
e0.record(); plan.run(xd, wd, bd, y); e1.record(); torch.cuda.synchronize()
print(f"  event-timed run: {e0.elapsed_time(e1) * 1e3:.2f} us; kernel span {rel.max():.2f} us")
# back-to-back
e0.record()
for i in range(50):
    plan.run(xd, wd, bd, y)
e1.record(); torch.cuda.synchronize()
print(f"  50 back-to-back runs: {e0.elapsed_time(e1) * 1e3 / 50:.2f} us each")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(200):
    plan.run(xd, wd, bd, y)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"  host time per run() call: {(t1 - t0) / 200 * 1e6:.1f} us")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    plan.run(xd, wd, bd, y)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(50):
            plan.run(xd, wd, bd, y, stream=s)
torch.cuda.synchronize()
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"  graph of 50 runs: {e0.elapsed_time(e1) * 1e3 / 50:.2f} us each")
