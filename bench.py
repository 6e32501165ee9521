"""bench.py -- the driver's benchmark contract for the WPK hot path on B200.

One step = one forward pass of every ResNet-50 v1.5 convolution (53 convs, 23 unique shapes) at
N=32 per GPU, bf16 NHWC, fused bias+ReLU (BASELINE.json configs[1], N=32 bf16 -- the largest
single-GPU case the metric is quoted on), each layer running the config chosen by the per-layer
GA tuner (§2.3) before the timed region. value = whole-job conv TFLOP/s
(2*N*K*P*Q*C*R*S summed over layers and ranks / max-over-ranks device time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl wpk|reference] [--tune-budget B]

N>1 runs under torchrun: every rank processes its own N=32 shard (the N=256 batch split along N,
BASELINE.json configs[4]; weak scaling) and the GA population is sharded over the ranks with an
NCCL all-gather of fitness records (paper_2008_04567_b200/dist.py).
"""
from __future__ import annotations

import argparse
import tempfile
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv2d TFLOP/s per layer (% of B200 peak) vs same-box cuDNN; tuning time 1/2/4/8 GPU"
PEAK_FALLBACK = {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}   # B200_PROFILING.md fallback


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(PEAK_FALLBACK), "fallback (B200_PROFILING.md)"


def layer_flops(L, p, q):
    return 2 * L.n * L.k * p * q * (L.c // L.groups) * L.r * L.s


def layer_bytes(L, p, q, elem):
    return elem * (L.n * L.c * L.h * L.w + L.k * (L.c // L.groups) * L.r * L.s + L.k + L.n * L.k * p * q)


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every 5 ms (the timed
    region of a default run is tens of ms), else nvidia-smi every 100 ms."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self.source = "nvidia-smi"
        self.nv = self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(index)
            self.source = "nvml"
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _sample_nvml(self):
        nv, h = self.nv, self.h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        return [str(sm), str(mx), "", *("Active" if r & b else "Not Active" for b in bits)]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self.nv is not None:
                    self.rows.append(self._sample_nvml())
                    self._stop.wait(0.005)
                    continue
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                self.nv = None   # fall back to nvidia-smi
            self._stop.wait(0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# -------------------------------------------------------------------------------------------------
# reference arm: the oracle (test infrastructure) timed on the host cores
# -------------------------------------------------------------------------------------------------
def oracle_sample_step(layers, per_layer_points, nthreads, seed=0):
    """One bounded sample of the workload through the oracle: `per_layer_points` outputs of every
    unique layer (x 'count'), computed one by one. Returns (flops, seconds)."""
    import oracle
    import workloads
    flops, secs = 0.0, 0.0
    for i, L in enumerate(layers):
        x, w, b = workloads.generate(L, "bf16", "uniform", seed=workloads.config_seed(1, i))
        p, q = oracle.out_dims(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups)
        pts = workloads.random_points(L, p, q, per_layer_points, seed=seed + i).numpy()[-per_layer_points:]
        t0 = time.perf_counter()
        for _ in range(L.count):
            oracle.conv2d_points(x, w, b, pts, stride=L.stride, pad=L.pad, nthreads=nthreads)
        secs += time.perf_counter() - t0
        flops += L.count * len(pts) * 2.0 * (L.c // L.groups) * L.r * L.s
    return flops, secs


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import workloads
    oracle.build()
    layers = workloads.resnet50(32)
    cores = os.cpu_count() or 1
    pts = args.ref_points
    for _ in range(args.warmup):
        oracle_sample_step(layers, max(pts // 8, 16), cores)
    tot_f, tot_s = 0.0, 0.0
    for k in range(args.steps):
        f, s = oracle_sample_step(layers, pts, cores, seed=100 + k)
        tot_f += f
        tot_s += s
    tflops = tot_f / tot_s / 1e12
    sample = (f"{pts} sampled outputs x 53 ResNet-50 convs (N=32 bf16-rounded inputs, float64 oracle) "
              f"per step, computed one by one")
    line = {"impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "resnet50_convs_n32_bf16_nhwc_bias_relu (sampled)",
                                            "global_batch": 32, "parallelism": "host cores"},
            "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------------------------------------
# WPK arm
# -------------------------------------------------------------------------------------------------
class Dist:
    """Process-group plumbing. NCCL over NVLink by default; gloo (CPU tensors) when
    WPK_BENCH_BACKEND=gloo or when fewer GPUs than ranks are visible -- the ranks then share the
    visible devices round-robin, which runs the N>1 code path (sharded tuner exchange, max-over-ranks
    timing) on one GPU as a smoke test (tests/test_nsplit_gpu.py)."""

    def __init__(self):
        import torch
        self.world, self.rank, self.local = dist_env()
        ndev = max(1, torch.cuda.device_count())
        self.backend = os.environ.get("WPK_BENCH_BACKEND") or ("nccl" if ndev >= self.world else "gloo")
        self.dev_index = self.local % ndev
        torch.cuda.set_device(self.dev_index)
        self.dev = torch.device("cuda", self.dev_index)
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")
            self.pg = dist.group.WORLD

    def max(self, v: float) -> float:
        """Max over ranks (every rank gets the same value, so rank-local decisions agree)."""
        if self.pg is None:
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.pg is not None:
            import torch.distributed as dist
            dist.barrier()


def _capture(units, stream, fn=None):
    """One CUDA graph holding every conv of the step in order (fn(unit) issues one conv)."""
    import torch
    fn = fn or (lambda u: u[1].run(u[2], u[3], u[4], u[5], stream=stream))
    with torch.cuda.stream(stream):           # eager pass: packs weights, sizes workspaces
        for u in units:
            fn(u)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for u in units:
            fn(u)
    torch.cuda.synchronize()
    return g


def _graph_ms(g, stream, reps, warmup=2):
    import torch
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _step_ms(units, stream, D, reps=12):
    """Device time of one whole-step graph replay, max over ranks (graph refinement)."""
    g = _capture(units, stream)
    ms = D.max(_graph_ms(g, stream, reps))
    del g
    return ms


def graph_refine(args, layers, plans, units, records, stream, D):
    """System-level refinement after the per-operator search (implementations are
    selected per operator, here in the context of the whole graph): the tuner times each candidate
    alone, but inside the step graph a conv's config also decides how early the next conv's CTAs
    start on idle SMs (programmatic dependent launch). For each layer, in order, the next-best
    measured configs (top --graph-refine by the tuner's beta) are tried in the whole-step graph and
    kept if the step gets >= 0.5% faster. Step times are max-reduced over ranks and every rank holds
    the same gathered tuning records, so all ranks take the same decisions."""
    base = _step_ms(units, stream, D)
    tried, changed = 0, []
    for i, L in enumerate(layers):
        path = records.get(i)
        if not path or not os.path.exists(path):
            continue
        recs = [json.loads(l) for l in open(path) if l.strip()]
        recs = [r for r in recs if r.get("beta_us") is not None and r["beta_us"] < 1e30]
        recs.sort(key=lambda r: r["beta_us"])
        cur = (plans[i].config[0], list(plans[i].config[1]))
        alts, seen = [], {(cur[0], tuple(cur[1]))}
        for r in recs:
            key = (r["family"], tuple(r["genes"]))
            if key not in seen:
                seen.add(key)
                alts.append(key)
            if len(alts) >= args.graph_refine:
                break
        for fam, genes in alts:
            plans[i].set_config(fam, list(genes))
            t = _step_ms(units, stream, D)
            tried += 1
            if t < base * 0.995:
                base, cur = t, (fam, list(genes))
                changed.append(L.name)
        plans[i].set_config(cur[0], list(cur[1]))
        os.remove(path)
    return {"tried": tried, "changed": changed, "step_ms_after": base}


def kernel_trace(graph, stream, replays=3):
    """Per-launch device intervals of the step graph's kernels, recorded by CUPTI (torch.profiler)
    over `replays` back-to-back replays right after the timed region. Returns a list of steps, each a
    list of (kernel name, start_us, end_us) in launch order."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        with torch.cuda.stream(stream):
            for _ in range(replays):
                graph.replay()
        torch.cuda.synchronize()
    ks = []
    for e in prof.events():
        if str(getattr(e, "device_type", "")).endswith("CUDA") and e.time_range.end > e.time_range.start:
            nm = e.name
            if nm.startswith("Memcpy") or nm.startswith("Memset"):
                continue
            ks.append((nm, float(e.time_range.start), float(e.time_range.end)))
    ks.sort(key=lambda k: k[1])
    if not ks or len(ks) % replays:
        return None
    per = len(ks) // replays
    return [ks[r * per:(r + 1) * per] for r in range(replays)]


def _union(iv):
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in sorted(iv):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def trace_summary(steps):
    """The conv kernel's share of the step: union of its launch intervals / the step's span."""
    if not steps:
        return None
    shares, spans, conv_us, launches = [], [], [], []
    names = {}
    for st in steps:
        span = max(e for _, _, e in st) - min(s for _, s, _ in st)
        conv = [(s, e) for (n, s, e) in st if "umma_conv_kernel" in n]
        u = _union(conv)
        shares.append(u / span)
        spans.append(span)
        conv_us.append(u)
        launches.append(len(conv))
        for (n, s, e) in st:
            short = n.split("(")[0].split("<")[0].replace("void ", "").replace("wpk::", "")
            d = names.setdefault(short, {"launches": 0, "busy_us": 0.0})
            d["launches"] += 1
            d["busy_us"] += e - s
    k = len(steps)
    for d in names.values():
        d["launches"] //= k
        d["busy_us"] /= k
    return {"share": statistics.mean(shares), "span_us": statistics.mean(spans), "conv_busy_us": statistics.mean(conv_us),
            "conv_launches": launches[0], "kernels": names, "replays": k}


def latency_floor_us(stream, reps=51):
    """Empty-kernel floor on this box: event-timed single launch of a 0-cycle spin kernel (median),
    and the per-kernel cost of 64 such kernels back to back inside one CUDA graph."""
    import torch
    with torch.cuda.stream(stream):
        for _ in range(5):
            torch.cuda._sleep(0)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.cuda._sleep(0)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(64):
            torch.cuda._sleep(0)
    per = _graph_ms(g, stream, 20) * 1e3 / 64
    del g
    return {"event_single_launch_us": statistics.median(ts), "in_graph_per_kernel_us": per,
            "how": "torch.cuda._sleep(0) (an empty spin kernel); CUDA events advance in ~2 us steps here"}


def cpu_baseline_with_parity(layers, plans, units, args, rank):
    """The oracle on the host cores (cpu_baseline) over a bounded sample of THIS run's workload: for
    every unique layer, the bench's own inputs of its first conv and a seeded sample of output points
    -- every border pixel of every image (a rotating subset of channels) plus interior draws. The
    same points are read back from the outputs the timed graph wrote, so the leg doubles as the
    bench's parity check of the tuned configs (normwise error vs the bf16 tolerance 2e-2, and the
    worst per-layer error)."""
    import numpy as np
    import oracle
    import workloads
    oracle.build()
    cores = os.cpu_count() or 1
    flops = secs = 0.0
    worst, npts, rows = 0.0, 0, []
    for i, L in enumerate(layers):
        unit = next(u for u in units if u[0] == i)
        _, plan, xd, wd, bd, yd = unit
        x = xd.permute(0, 3, 1, 2).cpu()     # NCHW views of the bench's own tensors
        w = wd.permute(0, 3, 1, 2).cpu()
        b = bd.cpu()
        pts = workloads.parity_points(L, plan.p, plan.q, args.cpu_interior_points, seed=1000 + i,
                                      border_channels=args.cpu_border_channels)
        t0 = time.perf_counter()
        ref = oracle.conv2d_points(x, w, b, pts.numpy(), stride=L.stride, pad=L.pad, dil=L.dil, groups=L.groups,
                                   nthreads=cores)
        secs += time.perf_counter() - t0
        flops += len(pts) * 2.0 * (L.c // L.groups) * L.r * L.s
        y = yd.cpu()                          # NHWC [n, p, q, k]
        got = y[pts[:, 0], pts[:, 2], pts[:, 3], pts[:, 1]].double().numpy()
        err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
        worst = max(worst, err)
        npts += len(pts)
        rows.append({"layer": L.name, "points": int(len(pts)), "normwise_err": err, "config": plans[i].config[1]})
    cpu = {"value": flops / secs / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
           "sample": (f"per unique layer: every border pixel of every image x {args.cpu_border_channels} rotating "
                      f"channels + {args.cpu_interior_points} interior points of the bench's own inputs "
                      f"({npts} outputs over 23 layers), float64 7-loop oracle, OpenMP over points; {secs:.1f} s")}
    parity = {"ok": worst <= 2e-2, "max_normwise_err": worst, "tolerance": 2e-2, "points": npts,
              "layers": rows, "what": "bench outputs of the timed graph (tuned configs) vs the oracle on the same inputs"}
    return cpu, parity


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="wpk", choices=["wpk", "reference"])
    ap.add_argument("--batch", type=int, default=32, help="images per GPU")
    ap.add_argument("--tune-budget", type=int, default=128, help="distinct configs measured per unique layer")
    ap.add_argument("--graph-refine", type=int, default=3,
                    help="after the search, try each layer's next-best N measured configs in the whole-step graph")
    ap.add_argument("--ga-pop", type=int, default=16,
                    help="GA population, fixed for every world size (16 divides evenly over 1/2/4/8 ranks; "
                         "profiles/r1c_search_compare.md: with the paper's 48 a budget of 48 is one random generation)")
    ap.add_argument("--search", default="ga", choices=["ga", "rl", "random", "none"])
    ap.add_argument("--no-cudnn", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-points", type=int, default=1024)
    ap.add_argument("--cpu-interior-points", type=int, default=262144,
                    help="interior oracle outputs per unique layer for cpu_baseline / parity")
    ap.add_argument("--cpu-border-channels", type=int, default=8,
                    help="channels per border pixel (rotating over K) in the cpu_baseline / parity sample")
    ap.add_argument("--layers-json", default=None, help="also write the full line + per-layer table here")
    ap.add_argument("--trace-out", default=None, help="write the per-launch CUPTI trace of the step graph here")
    ap.add_argument("--configs-out", default=None, help="write the per-layer chosen configs (JSON)")
    ap.add_argument("--configs-in", default=None, help="use these per-layer configs instead of tuning")
    ap.add_argument("--cache-dir", default=None, help="tuning + selection cache directory (PAPER.md:179)")
    args = ap.parse_args()
    if os.environ.get("WPK_BENCH_WATCHDOG"):   # tests: dump every thread's stack and exit instead of hanging
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["WPK_BENCH_WATCHDOG"]), exit=True)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import workloads
    from paper_2008_04567_b200 import Conv2dPlan
    from paper_2008_04567_b200 import selector
    from paper_2008_04567_b200 import dist as wdist

    D = Dist()
    world, rank, dev = D.world, D.rank, D.dev
    peaks, peak_src = load_peaks()
    layers = workloads.resnet50(args.batch)
    stream = torch.cuda.Stream(dev)

    # ---- plans, inputs (resident in HBM), tuning -------------------------------------------------
    t_tune0 = time.perf_counter()
    units = []           # one entry per conv of the network (53), sharing the layer's plan
    plans = []
    tune_info = []
    records = {}         # layer index -> the tuner's measurement records (graph refinement)
    for i, L in enumerate(layers):
        plan = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc",
                          dtype="bf16", device=D.dev_index)
        if args.configs_in:
            fam, genes = json.load(open(args.configs_in))[L.name]
            plan.set_config(fam, genes)
        elif args.search != "none" and args.tune_budget > 0:
            ex = wdist.make_exchange(D.pg) if world > 1 else {}
            if args.search == "ga":   # small population -> several generations within the budget
                ex.update(ga_pop=args.ga_pop, ga_pool=args.ga_pop, ga_elites=2)
            if args.graph_refine > 0:   # every rank holds the same gathered records
                rec = os.path.join(tempfile.gettempdir(), f"wpk_bench_rec_{os.getpid()}_{rank}_{i}.jsonl")
                if os.path.exists(rec):
                    os.remove(rec)
                ex["record_path"] = rec
                records[i] = rec
            if args.cache_dir:
                ex["cache_dir"] = args.cache_dir
            res = plan.tune(args.search, args.tune_budget, seed=i, rank=rank, world=world, **ex)
            tune_info.append({"layer": L.name, "best_us": res.best_us, "measured": res.measured,
                              "family": res.family, "genes": res.genes, "seconds": res.seconds})
        plans.append(plan)
        for c in range(L.count):
            x, w, b = workloads.generate(L, "bf16", "uniform", seed=workloads.config_seed(1, i) + 7919 * c + rank)
            xd = x.permute(0, 2, 3, 1).contiguous().to(dev)
            wd = w.permute(0, 2, 3, 1).contiguous().to(dev)
            bd = b.to(dev)
            yd = torch.empty(plan.y_shape(), dtype=torch.bfloat16, device=dev)
            units.append((i, plan, xd, wd, bd, yd))
    torch.cuda.synchronize()
    search_seconds = D.max(time.perf_counter() - t_tune0)
    refine_info = graph_refine(args, layers, plans, units, records, stream, D) if records else None
    tune_seconds = D.max(time.perf_counter() - t_tune0)
    if args.configs_out and rank == 0:
        json.dump({L.name: list(plans[i].config) for i, L in enumerate(layers)}, open(args.configs_out, "w"))

    total_flops = sum(layer_flops(L, plans[i].p, plans[i].q) * L.count for i, L in enumerate(layers))

    # Per-conv graphs (instrumented per-layer pass) and the step graph: ONE graph holding all convs in
    # order -- no per-conv launch gaps, and the kernels' programmatic-dependent-launch attribute
    # becomes a programmatic edge, so each conv's prologue overlaps its predecessor's tail.
    graphs, graph_launches = [], []
    for u in units:
        graphs.append(_capture([u], stream))
        graph_launches.append(u[1].last_launch_count())
    step_graph = _capture(units, stream)
    launches_per_step = sum(graph_launches)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step_graph.replay()
    torch.cuda.synchronize()

    # ---- timed region ------------------------------------------------------------------------------
    D.barrier()
    torch.cuda.synchronize()
    with ClockSampler(D.dev_index) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                step_graph.replay()
        t1.record(stream)
        torch.cuda.synchronize()
    ms = D.max(t0.elapsed_time(t1))
    D.barrier()
    launches = launches_per_step * args.steps
    ms_per_step = ms / args.steps
    value = total_flops * world * args.steps / (ms * 1e-3) / 1e12

    # ---- the conv kernel's share of the step: CUPTI trace of the same graph, same run ------------------
    trace = None
    try:
        trace = kernel_trace(step_graph, stream)
    except Exception as ex:   # profiler unavailable: the line says so
        trace = None
        trace_err = str(ex)[:200]
    tsum = trace_summary(trace)
    if args.trace_out and rank == 0 and trace:
        json.dump({"summary": tsum, "steps": trace}, open(args.trace_out, "w"))

    # ---- per-layer split: per-conv graphs between events (instrumented pass, no cross-conv overlap) -----
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in units]
          for _ in range(min(args.steps, 10))]
    with torch.cuda.stream(stream):
        for k in range(len(ev)):
            for j, g in enumerate(graphs):
                ev[k][j][0].record(stream)
                g.replay()
                ev[k][j][1].record(stream)
    torch.cuda.synchronize()
    per_unit_ms = [statistics.mean(ev[k][j][0].elapsed_time(ev[k][j][1]) for k in range(len(ev)))
                   for j in range(len(units))]
    per_layer_ms = [0.0] * len(layers)
    for j, (i, *_rest) in enumerate(units):
        per_layer_ms[i] += per_unit_ms[j]
    iso_ms = sum(per_unit_ms)

    # ---- roofline --------------------------------------------------------------------------------------
    peak = float(peaks.get("bf16_tflops", PEAK_FALLBACK["bf16_tflops"]))
    hbm = float(peaks.get("hbm_gbs", PEAK_FALLBACK["hbm_gbs"]))
    # Per-launch floor of the mixed step: each conv is bound by max(FLOPs / tensor peak, algorithmic
    # bytes / HBM peak); frac = that floor summed over the step / the timed step.
    t_roof_ms, n_tensor = 0.0, 0
    roof_rows = {}
    for j, (i, *_rest) in enumerate(units):
        L, pl = layers[i], plans[i]
        tf = layer_flops(L, pl.p, pl.q) / (peak * 1e12) * 1e3
        tb = layer_bytes(L, pl.p, pl.q, 2) / (hbm * 1e9) * 1e3
        t_roof_ms += max(tf, tb)
        n_tensor += tf >= tb
        roof_rows[i] = (tf * 1e3, tb * 1e3)
    conv_ms = (tsum["conv_busy_us"] / tsum["span_us"]) * ms_per_step if tsum else None
    achieved = total_flops / (conv_ms * 1e-3) / 1e12 if conv_ms else total_flops / (ms_per_step * 1e-3) / 1e12
    bytes_step = sum(layer_bytes(layers[i], plans[i].p, plans[i].q, 2) for (i, *_r) in units)
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_step_range.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic = pj["dram_bytes_per_step"]
            traffic_src = (f"{os.path.relpath(prof, ROOT)}: ncu range capture of one step-graph replay "
                           f"(configs {pj.get('configs_file')}; this run's configs "
                           f"{'match' if pj.get('configs') == {L.name: list(plans[i].config) for i, L in enumerate(layers)} else 'differ (re-tuned)'})")
        except Exception:
            traffic = None
    roofline = {
        "bound": "mixed", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": t_roof_ms / ms_per_step, "traffic": traffic,
        "frac_definition": ("sum over the 53 launches of max(FLOPs / tensor peak, bytes / HBM peak) "
                            f"({t_roof_ms * 1e3:.1f} us) / the timed step ({ms_per_step * 1e3:.1f} us); "
                            f"{n_tensor} launches tensor-bound, {len(units) - n_tensor} HBM-bound at the measured peaks"),
        "tensor_frac": achieved / peak,
        "achieved_from": ("conv FLOPs per step / the conv kernel's busy time in the step (step time x its share of "
                          f"the step graph, {tsum['share']:.3f}, CUPTI trace of the same graph in this run)") if tsum
                         else "conv FLOPs per step / step time (no kernel trace available)",
        "algorithmic_bytes_per_step": bytes_step,
        "hbm_gbs_achieved": bytes_step / (ms_per_step * 1e-3) / 1e9,
        "traffic_unit": "DRAM bytes read+write per step (all launches)", "traffic_source": traffic_src,
        "kernel": "umma_conv_kernel (all 53 conv launches of a step)",
        "peak_source": peak_src + " bf16 burst (the timed region runs at max SM clock; see clocks)",
        "hbm_peak_gbs": hbm,
        "isolated_sum_us": iso_ms * 1e3,
    }

    # ---- e2e through the public API with host buffers ----------------------------------------------
    host = []
    h2d = d2h = 0
    for (i, plan, xd, wd, bd, yd) in units:
        xh = xd.cpu().pin_memory()
        yh = torch.empty(yd.shape, dtype=yd.dtype).pin_memory()
        host.append((plan, xh, wd, bd, yh))
        h2d += xh.numel() * xh.element_size()
        d2h += yh.numel() * yh.element_size()
    # Layers go round-robin over several streams (each plan always on the same one) through the async
    # host-buffer call, so one layer's H2D copy overlaps another's kernel and D2H copy.
    n_e2e = int(os.environ.get("WPK_E2E_STREAMS", "6"))   # 1: 9.7, 3: 14.7, 6: 16.6, 12: 16.7 TF/s (same box)
    e2e_streams = [torch.cuda.Stream(device=dev) for _ in range(n_e2e)]
    for j, (plan, xh, wd, bd, yh) in enumerate(host):     # warm-up of the host path
        plan.run_host(xh, wd, bd, yh, stream=e2e_streams[j % n_e2e])
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 5))
    D.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for es in e2e_streams:
        es.wait_stream(stream)
    for _ in range(e2e_steps):
        for j, (plan, xh, wd, bd, yh) in enumerate(host):
            plan.run_host_async(xh, wd, bd, yh, stream=e2e_streams[j % n_e2e])
    for es in e2e_streams:
        stream.wait_stream(es)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = D.max(e0.elapsed_time(e1))
    e2e_value = total_flops * world * e2e_steps / (e2e_ms * 1e-3) / 1e12
    del host

    floor = latency_floor_us(stream)

    # ---- per-layer table vs same-box cuDNN, the per-layer selector choice (outside the timed region) ----
    table, sels = [], []
    for i, L in enumerate(layers):
        plan = plans[i]
        _, _, xd, wd, bd, yd = next(u for u in units if u[0] == i)
        fl = layer_flops(L, plan.p, plan.q)
        tf_us, tb_us = roof_rows[i]
        row = {"layer": L.name, "count": L.count, "gflop": fl / 1e9,
               "wpk_us_graph": per_layer_ms[i] / L.count * 1e3,
               "t_roof_us": max(tf_us, tb_us), "bound": "tensor" if tf_us >= tb_us else "hbm",
               "config": plan.config[1], "family": plan.config[0]}
        if row["t_roof_us"] < 5.0:
            row["latency_floor_us"] = floor["event_single_launch_us"]
        sc = selector.SelectedConv2d(plan, L.stride, L.pad, L.dil, cache_dir=args.cache_dir)
        if rank == 0 and not args.no_cudnn:
            with torch.cuda.stream(stream):
                sel = sc.select(xd, wd, bd, yd)
            row.update({"wpk_us": sel.own_us, "cudnn_us": sel.cudnn_us, "cudnn_variant": sel.cudnn_variant,
                        "speedup_vs_cudnn": sel.cudnn_us / sel.own_us, "selector": sel.choice,
                        "wpk_tflops": fl / (sel.own_us * 1e-6) / 1e12,
                        "pct_peak": fl / (sel.own_us * 1e-6) / 1e12 / peak,
                        "pct_of_roofline": row["t_roof_us"] / sel.own_us})
        sels.append(sc)
        table.append(row)

    # ---- the same step through the box's cuDNN, and through the per-layer selector (rank 0) --------------
    cudnn_step = selector_step = None
    if rank == 0 and not args.no_cudnn:
        try:
            fns = [selector.cudnn_conv_fn(xd, wd, bd, layers[i].stride, layers[i].pad, layers[i].dil, layers[i].groups,
                                          "nhwc", "bf16", fused=True) for (i, plan, xd, wd, bd, yd) in units]
            cg = _capture(list(range(len(fns))), stream, fn=lambda j: fns[j]())
            cms = _graph_ms(cg, stream, args.steps, warmup=args.warmup)
            cudnn_step = {"ms_per_step": cms, "value": total_flops / (cms * 1e-3) / 1e12, "unit": "TFLOP/s",
                          "wpk_speedup": cms / ms_per_step,
                          "how": "torch.cudnn_convolution_relu on channels_last bf16, the 53 convs in one CUDA graph, "
                                 "cudnn.benchmark=True, same warm-up and step count"}
            del cg
        except Exception as ex:   # the competitor is optional context, never a reason to fail the bench
            cudnn_step = {"error": str(ex)[:200]}
        try:
            sg = _capture(units, stream, fn=lambda u: sels[u[0]](u[2], u[3], u[4], u[5], stream=stream))
            sms = _graph_ms(sg, stream, args.steps, warmup=args.warmup)
            n_cudnn = sum(1 for (i, *_r) in units if sels[i].choice == "cudnn")
            selector_step = {"ms_per_step": sms, "value": total_flops / (sms * 1e-3) / 1e12, "unit": "TFLOP/s",
                             "convs_on_cudnn": n_cudnn, "convs_on_wpk": len(units) - n_cudnn,
                             "how": "each conv dispatched by SelectedConv2d to its selected implementation "
                                    "(PAPER.md:140), the 53 convs in one CUDA graph, same warm-up and step count"}
            del sg
        except Exception as ex:
            selector_step = {"error": str(ex)[:200]}

    # ---- CPU oracle baseline + parity of this run's outputs (rank 0, N=1 only) ------------------------
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        with torch.cuda.stream(stream):
            step_graph.replay()               # the outputs of the timed graph itself
        torch.cuda.synchronize()
        cpu, parity = cpu_baseline_with_parity(layers, plans, units, args, rank)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"resnet50_v1.5_all_53_convs_n{args.batch}_bf16_nhwc_bias_relu",
                       "global_batch": args.batch * world, "per_gpu_batch": args.batch,
                       "parallelism": f"dp{world} (batch split along N)", "tune": args.search,
                       "tune_budget_per_layer": args.tune_budget, "ga_pop": args.ga_pop,
                       "backend": D.backend if world > 1 else None,
                       "l2": "inputs larger than L2 (1.44 GB per step; every conv has its own buffers)"},
            "parity": (parity or {}).get("ok"),
            "roofline": roofline,
            "cudnn_step": cudnn_step,
            "selector_step": selector_step,
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": "wpk_conv2d_run_host_async per conv on " + str(n_e2e) + " round-robin streams (pinned host x in, host y out)"},
            "gpu_launches": launches,
            "gpu_launches_per_step": launches_per_step,
            "tuning_seconds": tune_seconds, "search_seconds": search_seconds,
            "graph_refine": refine_info,
            "latency_floor": floor,
            "kernel_trace": tsum,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "parity_detail": parity,
            "layers": table,
            "tune": tune_info,
        }
        if args.layers_json:
            json.dump(line, open(args.layers_json, "w"), indent=1)
        # the JSON line itself stays compact: the per-layer parity rows go to --layers-json only
        if parity:
            line["parity_detail"] = {k: v for k, v in parity.items() if k != "layers"}
        print(json.dumps(line), flush=True)
    if D.pg is not None:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
