"""System-level exploration (§2.5): per operator, keep the faster of WPK's own tuned
kernel and a third-party implementation -- here the same box's cuDNN reached through torch
(BASELINE.json north_star). Ties go to the own kernel (reading c25).

The timing protocol is the one the tuner uses (wpk_tune_options.l2_flush = 2): W
warm-ups, then R reps, each one CUDA graph of P calls on P cold copies of the input between CUDA
events, interquartile mean of span / P. The C library never sees torch: the choice lives here,
in SelectedConv2d, which persists it next to the tuning cache and dispatches each call to it.
"""
from __future__ import annotations

import json
import os
import statistics
from dataclasses import dataclass

import torch
import torch.nn.functional as F

_FLUSH = {}


def l2_flush_buffer(device) -> torch.Tensor:
    dev = torch.device(device)
    if dev not in _FLUSH:
        l2 = getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20)
        _FLUSH[dev] = torch.ones(2 * max(l2, 64 << 20), dtype=torch.uint8, device=dev)
    return _FLUSH[dev]


def l2_flush(buf: torch.Tensor):
    """Evict L2 by READING a 2x-L2 buffer (a write-based flush would leave ~L2-size dirty lines whose
    write-back would then be charged to the timed kernel)."""
    torch.sum(buf.view(torch.int32), dtype=torch.int64)


def time_fn(fn, warmup: int = 3, reps: int = 11, flush: bool = True, stream=None) -> float:
    """Median microseconds of fn() over `reps` event-timed runs on `stream` (L2 flushed before each)."""
    stream = stream or torch.cuda.current_stream()
    buf = l2_flush_buffer(stream.device) if flush else None
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            fn()
        ts = []
        for _ in range(reps):
            if buf is not None:
                l2_flush(buf)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def rotating_copies(t: torch.Tensor, other_bytes: int = 0, cap: int = 64) -> list:
    """P copies of t (the first is t itself) with P * (|t| + other_bytes) >= 2 x L2, <= cap, <= 3 GB:
    a graph that cycles through them reads every input cold."""
    l2 = getattr(torch.cuda.get_device_properties(t.device), "L2_cache_size", 126 << 20)
    foot = t.numel() * t.element_size() + other_bytes
    p = max(2, min(cap, -(-2 * l2 // max(foot, 1))))
    while p > 2 and p * foot > (3 << 30):
        p -= 1
    return [t] + [t.clone() for _ in range(p - 1)]


def time_rotating(fns, warmup: int = 3, reps: int = 11, stream=None) -> float:
    """Microseconds per call: the P callables (each bound to its own cold input copy) are captured in
    one CUDA graph, replayed `reps` times between CUDA events; interquartile mean of span / P. The
    same protocol as the tuner's (wpk_tune_options.l2_flush = 2): the events' ~2-us steps are spread
    over P calls, and consecutive calls overlap as in a network step."""
    stream = stream or torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for _ in range(max(1, warmup)):
            for f in fns:
                f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for f in fns:
            f()
    torch.cuda.synchronize()
    ts = []
    with torch.cuda.stream(stream):
        g.replay()
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / len(fns))
    del g
    ts.sort()
    lo, hi = len(ts) // 4, len(ts) - len(ts) // 4
    return sum(ts[lo:hi]) / (hi - lo)


def cudnn_conv_fn(x, w, b, stride, pad, dil, groups, layout, dtype, fused: bool, z=None, epilogue="bias_relu"):
    """cuDNN competitor: NHWC tensors are passed as channels_last views (no copies). The returned
    callable gives the output in the caller's layout (an NHWC view of cuDNN's channels_last result).
    epilogue: "bias_relu" (default), "bias", "none", or "bias_add_relu" with the residual z."""
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = (dtype == "tf32")
    torch.backends.cuda.matmul.allow_tf32 = (dtype == "tf32")
    nhwc = layout == "nhwc"
    if nhwc:
        xt = x.permute(0, 3, 1, 2)             # logical NCHW view of channels_last memory
        wt = w.permute(0, 3, 1, 2)
        zt = z.permute(0, 3, 1, 2) if z is not None else None
    else:
        xt, wt, zt = x, w, z
    st, pd, dl = (stride, stride), (pad, pad), (dil, dil)
    if epilogue == "bias_add_relu":
        if fused and hasattr(torch, "cudnn_convolution_add_relu"):
            def g():
                return torch.cudnn_convolution_add_relu(xt, wt, zt, 1.0, b, st, pd, dl, groups)
        else:
            def g():
                return F.relu_(F.conv2d(xt, wt, b, stride, pad, dil, groups).add_(zt))
    elif epilogue in ("bias", "none"):
        bb = b if epilogue == "bias" else None

        def g():
            return F.conv2d(xt, wt, bb, stride, pad, dil, groups)
    elif fused and b is not None and hasattr(torch, "cudnn_convolution_relu"):
        def g():
            return torch.cudnn_convolution_relu(xt, wt, b, st, pd, dl, groups)
    else:
        def g():
            return F.relu_(F.conv2d(xt, wt, b, stride, pad, dil, groups))
    if not nhwc:
        return g

    def f():
        return g().permute(0, 2, 3, 1)           # NHWC view (channels_last memory: no copy)
    return f


@dataclass
class Selection:
    own_us: float
    cudnn_us: float
    cudnn_variant: str
    choice: str          # "wpk" or "cudnn"


_VARIANT_NAMES = {("bias_relu", True): "cudnn_convolution_relu", ("bias_relu", False): "conv2d+relu_",
                  ("bias_add_relu", True): "cudnn_convolution_add_relu", ("bias_add_relu", False): "conv2d+add_+relu_",
                  ("bias", True): "conv2d", ("bias", False): "conv2d", ("none", True): "conv2d",
                  ("none", False): "conv2d"}


def select(plan, x, w, b, y, stride, pad, dil, groups, warmup=3, reps=11, z=None) -> Selection:
    """Time the plan's current config and both cuDNN variants with the same protocol (time_rotating:
    a graph over cold input copies); pick the argmin (ties -> wpk)."""
    xs = rotating_copies(x, y.numel() * y.element_size())
    ys = [y] + [torch.empty_like(y) for _ in xs[1:]]
    own = time_rotating([lambda i=i: plan.run(xs[i], w, b, ys[i], z=z) for i in range(len(xs))], warmup, reps)
    best, variant = float("inf"), "none"
    for fused in (False, True):
        try:
            fns = [cudnn_conv_fn(xi, w, b, stride, pad, dil, groups, plan.layout, plan.dtype, fused, z=z,
                                 epilogue=plan.epilogue) for xi in xs]
            fns[0]()
            t = time_rotating(fns, warmup, reps)
        except (RuntimeError, TypeError):
            continue
        if t < best:
            best, variant = t, _VARIANT_NAMES[(plan.epilogue, fused)]
    choice = "wpk" if own <= best else "cudnn"
    return Selection(own, best, variant, choice)


def _device_tag(device) -> str:
    p = torch.cuda.get_device_properties(device)
    return "".join(ch if ch.isalnum() else "_" for ch in f"{p.name}_sm{p.multi_processor_count}")


class SelectedConv2d:
    """One convolution of the optimized inference plan (§2.5: "If the third-party
    implementation is superior, we will use this ... implementation in our optimized inference
    plan"): a tuned WPK plan plus the system-level choice between it and the box's cuDNN, made by
    `select` (same protocol as the tuner, ties -> WPK) and persisted next to the tuning cache.

    __call__ dispatches: "wpk" runs the plan (libwpk.so kernels, into y if given); "cudnn" runs the
    chosen cuDNN variant through torch and returns its own output tensor in the plan's layout (an
    NHWC view of channels_last memory for NHWC plans; y is not written)."""

    def __init__(self, plan, stride=1, pad=0, dil=1, cache_dir: str | None = None):
        self.plan, self.stride, self.pad, self.dil = plan, stride, pad, dil
        self.groups = plan.groups
        self.cache_dir = cache_dir
        self.choice = "wpk"          # until a selection is made or loaded
        self.variant = None
        self.selection: Selection | None = None
        self._fns = {}

    # -- persistence -----------------------------------------------------------------------------
    def key(self) -> str:
        pl = self.plan
        return (f"sel_n{pl.n}_c{pl.c}_h{pl.h}_w{pl.w}_k{pl.k}_r{pl.r}_s{pl.s}_st{self.stride}_p{self.pad}"
                f"_d{self.dil}_g{pl.groups}_{pl.layout}_{pl.epilogue}_{pl.dtype}_{_device_tag(pl.device)}")

    def _path(self):
        return os.path.join(self.cache_dir, self.key() + ".json") if self.cache_dir else None

    def save(self):
        path = self._path()
        if path is None or self.selection is None:
            return
        os.makedirs(self.cache_dir, exist_ok=True)
        fam, genes = self.plan.config
        rec = {"choice": self.choice, "cudnn_variant": self.variant, "own_us": self.selection.own_us,
               "cudnn_us": self.selection.cudnn_us, "family": fam, "genes": genes}
        tmp = f"{path}.tmp{os.getpid()}"
        with open(tmp, "w") as f:
            json.dump(rec, f)
        os.replace(tmp, path)

    def load(self) -> bool:
        """Adopt a persisted choice if it was made for the plan's current config."""
        path = self._path()
        if path is None or not os.path.exists(path):
            return False
        rec = json.load(open(path))
        fam, genes = self.plan.config
        if rec.get("family") != fam or list(rec.get("genes", [])) != list(genes):
            return False
        self.choice, self.variant = rec["choice"], rec.get("cudnn_variant")
        self.selection = Selection(rec["own_us"], rec["cudnn_us"], self.variant or "none", self.choice)
        return True

    # -- selection and dispatch ------------------------------------------------------------------
    def select(self, x, w, b, y=None, z=None, warmup=3, reps=11) -> Selection:
        if y is None:
            y = torch.empty(self.plan.y_shape(), dtype=x.dtype, device=x.device)
        sel = select(self.plan, x, w, b, y, self.stride, self.pad, self.dil, self.groups, warmup, reps, z=z)
        self.selection, self.choice, self.variant = sel, sel.choice, sel.cudnn_variant
        self.save()
        return sel

    def __call__(self, x, w, b, y=None, z=None, stream=None):
        if self.choice == "wpk":
            return self.plan.run(x, w, b, y, stream=stream, z=z)
        key = (x.data_ptr(), w.data_ptr(), None if b is None else b.data_ptr(), None if z is None else z.data_ptr())
        f = self._fns.get(key)
        if f is None:
            fused = self.variant in ("cudnn_convolution_relu", "cudnn_convolution_add_relu")
            f = cudnn_conv_fn(x, w, b, self.stride, self.pad, self.dil, self.groups, self.plan.layout,
                              self.plan.dtype, fused, z=z, epilogue=self.plan.epilogue)
            self._fns[key] = f
        if stream is not None:
            with torch.cuda.stream(stream):
                return f()
        return f()
