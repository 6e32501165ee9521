"""System-level exploration (§2.5): per operator, keep the faster of WPK's own tuned
kernel and a third-party implementation -- here the same box's cuDNN reached through torch
(BASELINE.json north_star). Ties go to the own kernel (reading c25).

The timing protocol is the one the tuner uses: W warm-ups, then R CUDA-event-timed
reps with an L2 flush before each, median. The C library never sees torch; this module only
records which implementation a layer should dispatch to.
"""
from __future__ import annotations

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


def cudnn_conv_fn(x, w, b, stride, pad, dil, groups, layout, dtype, fused: bool):
    """cuDNN competitor: NHWC tensors are passed as channels_last views (no copies)."""
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = (dtype == "tf32")
    torch.backends.cuda.matmul.allow_tf32 = (dtype == "tf32")
    if layout == "nhwc":
        xt = x.permute(0, 3, 1, 2)             # logical NCHW view of channels_last memory
        wt = w.permute(0, 3, 1, 2)
    else:
        xt, wt = x, w
    if fused and b is not None and hasattr(torch, "cudnn_convolution_relu"):
        def f():
            return torch.cudnn_convolution_relu(xt, wt, b, (stride, stride), (pad, pad), (dil, dil), groups)
    else:
        def f():
            return F.relu_(F.conv2d(xt, wt, b, stride, pad, dil, groups))
    return f


@dataclass
class Selection:
    own_us: float
    cudnn_us: float
    cudnn_variant: str
    choice: str          # "wpk" or "cudnn"


def select(plan, x, w, b, y, stride, pad, dil, groups, warmup=3, reps=11) -> Selection:
    """Time the plan's current config and both cuDNN variants; pick the argmin (ties -> wpk)."""
    own = time_fn(lambda: plan.run(x, w, b, y), warmup, reps)
    best, variant = float("inf"), "none"
    for fused in (False, True):
        try:
            f = cudnn_conv_fn(x, w, b, stride, pad, dil, groups, plan.layout, plan.dtype, fused)
            f()
            t = time_fn(f, warmup, reps)
        except (RuntimeError, TypeError):
            continue
        if t < best:
            best, variant = t, ("cudnn_convolution_relu" if fused else "conv2d+relu_")
    choice = "wpk" if own <= best else "cudnn"
    return Selection(own, best, variant, choice)
