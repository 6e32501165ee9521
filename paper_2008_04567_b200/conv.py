"""Python face of the C ABI: a per-layer plan object that marshals torch tensors to
wpk_conv2d_run / wpk_conv2d_tune. Every step of the convolution runs in libwpk.so kernels; torch
only allocates device memory and provides streams (BASELINE.json north_star).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L

# dtype of b / z / y; x and w use _TORCH_IN_DT (they differ for "fp8": e4m3 operands, bf16 output)
_TORCH_DT = {"f32": torch.float32, "tf32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16,
             "fp8": torch.bfloat16}
_TORCH_IN_DT = dict(_TORCH_DT, fp8=torch.float8_e4m3fn)


def output_dims(n, c, h, w, k, r, s, stride=1, pad=0, dil=1, groups=1):
    lib = L.load()
    shp = L.make_shape(n, c, h, w, k, r, s, stride, pad, dil, groups)
    p, q = ctypes.c_int32(), ctypes.c_int32()
    L.check(lib.wpk_conv2d_output_dims(ctypes.byref(shp), ctypes.byref(p), ctypes.byref(q)))
    return p.value, q.value


@dataclass
class TuneResult:
    family: int
    genes: list
    best_us: float
    measured: int
    rounds: int
    seconds: float


class Conv2dPlan:
    """wpk_conv2d_plan + run/tune for one convolution layer.

    Layouts: "nchw" -> x [N,C,H,W], w [K,C/g,R,S], y [N,K,P,Q];  "nhwc" -> x [N,H,W,C],
    w [K,R,S,C/g], y [N,P,Q,K] (dense tensors, i.e. a permuted channels_last tensor must be made
    contiguous in that order)."""

    def __init__(self, n, c, h, w, k, r, s, stride=1, pad=0, dil=1, groups=1, layout="nchw",
                 epilogue="bias_relu", dtype="bf16", device: int | None = None):
        self.lib = L.load()
        self.dtype, self.layout, self.epilogue = dtype, layout, epilogue
        self.device = torch.cuda.current_device() if device is None else device
        self.shape = L.make_shape(n, c, h, w, k, r, s, stride, pad, dil, groups, layout, epilogue)
        self.n, self.c, self.h, self.w, self.k, self.r, self.s = n, c, h, w, k, r, s
        self.groups = groups
        h_ = ctypes.c_void_p()
        L.check(self.lib.wpk_conv2d_plan(ctypes.byref(self.shape), L.DTYPES[dtype], self.device, ctypes.byref(h_)))
        self.handle = h_
        self.p, self.q = output_dims(n, c, h, w, k, r, s, stride, pad, dil, groups)
        self._ws = None
        self._ws_bytes = -1
        # per-call checks against precomputed values (the eager call path is host-latency bound)
        self._tdt = _TORCH_DT[dtype]
        self._idt = _TORCH_IN_DT[dtype]
        self._xs, self._wsh, self._ys = torch.Size(self.x_shape()), torch.Size(self.w_shape()), torch.Size(self.y_shape())
        self._hval = self.handle.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.wpk_conv2d_destroy(h)
            self.handle = None

    # -- config ----------------------------------------------------------------------------------
    @property
    def config(self):
        fam = ctypes.c_int32()
        genes = (ctypes.c_int32 * L.NUM_GENES)()
        L.check(self.lib.wpk_conv2d_get_config(self.handle, ctypes.byref(fam), genes))
        return fam.value, list(genes)

    def set_config(self, family, genes):
        fam = L.FAMILIES[family] if isinstance(family, str) else int(family)
        arr = (ctypes.c_int32 * L.NUM_GENES)(*genes)
        L.check(self.lib.wpk_conv2d_set_config(self.handle, fam, arr))
        self._ws_bytes = -1

    def jit_compile(self, genes) -> int:
        """Generate + NVRTC-compile this shape's JIT-family kernel for `genes` (no GPU needed);
        returns the cubin size in bytes (cached per process / on disk)."""
        arr = (ctypes.c_int32 * L.NUM_GENES)(*genes)
        n = ctypes.c_size_t()
        L.check(self.lib.wpk_jit_compile(self.handle, arr, ctypes.byref(n)))
        return n.value

    def config_valid(self, family, genes) -> bool:
        fam = L.FAMILIES[family] if isinstance(family, str) else int(family)
        arr = (ctypes.c_int32 * L.NUM_GENES)(*genes)
        return bool(self.lib.wpk_conv2d_config_valid(self.handle, fam, arr))

    def workspace_bytes(self) -> int:
        b = ctypes.c_size_t()
        L.check(self.lib.wpk_conv2d_workspace_size(self.handle, ctypes.byref(b)))
        return b.value

    def _ensure_workspace(self):
        if self._ws_bytes >= 0:      # sized for the current config (set_config / tune reset it)
            return
        need = self.workspace_bytes()
        if need != self._ws_bytes:
            self._ws = torch.empty(max(need, 16), dtype=torch.uint8, device=f"cuda:{self.device}")
            L.check(self.lib.wpk_conv2d_set_workspace(self.handle, ctypes.c_void_p(self._ws.data_ptr()), need))
            self._ws_bytes = need

    # -- shapes ----------------------------------------------------------------------------------
    def x_shape(self):
        return (self.n, self.c, self.h, self.w) if self.layout == "nchw" else (self.n, self.h, self.w, self.c)

    def w_shape(self):
        cpg = self.c // self.groups
        return (self.k, cpg, self.r, self.s) if self.layout == "nchw" else (self.k, self.r, self.s, cpg)

    def y_shape(self):
        return (self.n, self.k, self.p, self.q) if self.layout == "nchw" else (self.n, self.p, self.q, self.k)

    # -- run -------------------------------------------------------------------------------------
    def run(self, x: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None, y: torch.Tensor | None = None,
            stream: torch.cuda.Stream | None = None, z: torch.Tensor | None = None) -> torch.Tensor:
        """y = epilogue(conv(x, w)); for epilogue "bias_add_relu" z is the residual (y's shape)."""
        dt, it = self._tdt, self._idt
        for t, nm, shp in ((x, "x", self._xs), (w, "w", self._wsh)):
            if t.dtype is not it or t.shape != shp or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{nm}: expected contiguous cuda {it} of shape {tuple(shp)}, got {t.dtype} {tuple(t.shape)}")
        if y is None:
            y = torch.empty(self._ys, dtype=dt, device=x.device)
        elif y.dtype is not dt or y.shape != self._ys or not y.is_cuda or not y.is_contiguous():
            raise ValueError(f"y: expected contiguous cuda {dt} of shape {tuple(self._ys)}, got {y.dtype} {tuple(y.shape)}")
        if b is not None and (b.dtype is not dt or b.shape != (self.k,) or not b.is_cuda or not b.is_contiguous()):
            raise ValueError(f"b: expected contiguous cuda {dt} of shape ({self.k},), got {b.dtype} {tuple(b.shape)}")
        if self._ws_bytes < 0:
            self._ensure_workspace()
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        if self.epilogue != "bias_add_relu":   # fast path: plain integers for the c_void_p arguments
            st = self.lib.wpk_conv2d_run(self._hval, x.data_ptr(), w.data_ptr(),
                                         b.data_ptr() if b is not None else None, y.data_ptr(), s)
            if st != 0:
                L.check(st)
            return y
        bp = ctypes.c_void_p(b.data_ptr()) if b is not None else None
        if self.epilogue == "bias_add_relu":
            if z is None or z.dtype != dt or tuple(z.shape) != self.y_shape() or not z.is_contiguous() or not z.is_cuda:
                raise ValueError(f"z: expected contiguous cuda {dt} of shape {self.y_shape()}")
            L.check(self.lib.wpk_conv2d_run_residual(self.handle, ctypes.c_void_p(x.data_ptr()),
                                                     ctypes.c_void_p(w.data_ptr()), bp, ctypes.c_void_p(z.data_ptr()),
                                                     ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(s)))
            return y
        L.check(self.lib.wpk_conv2d_run(self.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                        bp, ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(s)))
        return y

    def _check_host(self, x_host, w, b, y_host):
        dt, it = self._tdt, self._idt
        for t, nm, shp, tdt in ((x_host, "x_host", self._xs, it), (y_host, "y_host", self._ys, dt)):
            if t.dtype is not tdt or t.shape != shp or t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{nm}: expected contiguous CPU {tdt} of shape {tuple(shp)}, got "
                                 f"{t.dtype} {tuple(t.shape)} on {t.device}")
        if w.dtype is not it or w.shape != self._wsh or not w.is_cuda or not w.is_contiguous():
            raise ValueError(f"w: expected contiguous cuda {it} of shape {tuple(self._wsh)}")
        if b is not None and (b.dtype is not dt or b.shape != (self.k,) or not b.is_cuda or not b.is_contiguous()):
            raise ValueError(f"b: expected contiguous cuda {dt} of shape ({self.k},)")

    def run_host(self, x_host: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None, y_host: torch.Tensor,
                 stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """x_host/y_host are (pinned) CPU tensors; H2D + conv + D2H inside, then stream sync."""
        self._check_host(x_host, w, b, y_host)
        self._ensure_workspace()
        s = (stream or torch.cuda.current_stream(w.device)).cuda_stream
        bp = ctypes.c_void_p(b.data_ptr()) if b is not None else None
        L.check(self.lib.wpk_conv2d_run_host(self.handle, ctypes.c_void_p(x_host.data_ptr()),
                                             ctypes.c_void_p(w.data_ptr()), bp,
                                             ctypes.c_void_p(y_host.data_ptr()), ctypes.c_void_p(s)))
        return y_host

    def run_host_async(self, x_host: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None, y_host: torch.Tensor,
                       stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """run_host without the final stream sync: y_host is valid after the stream is synchronised."""
        self._check_host(x_host, w, b, y_host)
        self._ensure_workspace()
        s = (stream or torch.cuda.current_stream(w.device)).cuda_stream
        bp = ctypes.c_void_p(b.data_ptr()) if b is not None else None
        L.check(self.lib.wpk_conv2d_run_host_async(self.handle, ctypes.c_void_p(x_host.data_ptr()),
                                                   ctypes.c_void_p(w.data_ptr()), bp,
                                                   ctypes.c_void_p(y_host.data_ptr()), ctypes.c_void_p(s)))
        return y_host

    def fold_batchnorm(self, w: torch.Tensor, b: torch.Tensor | None, gamma: torch.Tensor, beta: torch.Tensor,
                       mean: torch.Tensor, var: torch.Tensor, eps: float = 1e-5, w_out: torch.Tensor | None = None,
                       b_out: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None):
        """(w', b') with conv(x, w') + b' == BN(conv(x, w) + b) (inference BN; fp32 [K] statistics)."""
        dt = _TORCH_DT[self.dtype]
        if w_out is None:
            w_out = torch.empty_like(w)
        if b_out is None:
            b_out = torch.empty(self.k, dtype=dt, device=w.device)
        f32 = [t.float().contiguous() for t in (gamma, beta, mean, var)]
        s = (stream or torch.cuda.current_stream(w.device)).cuda_stream
        bp = ctypes.c_void_p(b.data_ptr()) if b is not None else None
        L.check(self.lib.wpk_conv2d_fold_batchnorm(self.handle, ctypes.c_void_p(w.data_ptr()), bp,
                                                   *[ctypes.c_void_p(t.data_ptr()) for t in f32], ctypes.c_float(eps),
                                                   ctypes.c_void_p(w_out.data_ptr()), ctypes.c_void_p(b_out.data_ptr()),
                                                   ctypes.c_void_p(s)))
        self._f32_keep = f32   # alive until the stream has consumed them (next call replaces)
        return w_out, b_out

    def last_launch_count(self) -> int:
        return int(self.lib.wpk_conv2d_last_launch_count(self.handle))

    def invalidate(self):
        L.check(self.lib.wpk_conv2d_invalidate(self.handle))

    # -- tune ------------------------------------------------------------------------------------
    def tune(self, search: str = "ga", budget: int = 64, opts: L.TuneOptions | None = None, **kw) -> TuneResult:
        o = opts if opts is not None else make_options(**kw)
        L.check(self.lib.wpk_conv2d_tune(self.handle, L.SEARCHES[search], int(budget), ctypes.byref(o)))
        self._ws_bytes = -1
        return self.tune_stats()

    def measure(self, warmup: int = 3, reps: int = 11, l2_flush: int | bool = 2) -> float:
        """Microseconds of the current config under the tuner's timing protocol (wpk_conv2d_measure).
        l2_flush: 2 (default) rotating cold buffer copies in one graph per rep, 1 flush before each
        single launch, 0 warm; True means 2, False 0."""
        mode = (2 if l2_flush else 0) if isinstance(l2_flush, bool) else int(l2_flush)
        us = ctypes.c_double()
        L.check(self.lib.wpk_conv2d_measure(self.handle, int(warmup), int(reps), mode, ctypes.byref(us)))
        return us.value

    def tune_stats(self) -> TuneResult:
        best, secs = ctypes.c_double(), ctypes.c_double()
        meas, rounds = ctypes.c_int32(), ctypes.c_int32()
        L.check(self.lib.wpk_conv2d_tune_stats(self.handle, ctypes.byref(best), ctypes.byref(meas),
                                               ctypes.byref(rounds), ctypes.byref(secs)))
        fam, genes = self.config
        return TuneResult(fam, genes, best.value, meas.value, rounds.value, secs.value)


class DwPwPlan(Conv2dPlan):
    """Fused depthwise + pointwise convolution (wpk_dwpw_plan / wpk_dwpw_run; SURVEY.md 8(f) NEXT-4,
    the MobileNet block): y = pw_epilogue(RN(dw_epilogue(dwconv(x, w_dw) + b_dw)) (*) w_pw + b_pw) in
    one tcgen05 kernel. NHWC only: x [N,H,W,C], w_dw [C,R,S] (or [C,R,S,1] / [C,1,R,S]), b_dw [C],
    w_pw [K,C] (or [K,1,1,C] / [K,C,1,1]), b_pw [K], y [N,P,Q,K]. Tuning, configs and the workspace
    go through the inherited Conv2dPlan calls."""

    def __init__(self, n, c, h, w, k_out, r=3, s=3, stride=1, pad=1, dil=1, dw_epilogue="bias_relu",
                 pw_epilogue="bias", dtype="bf16", device: int | None = None):
        self.lib = L.load()
        self.dtype, self.layout, self.epilogue = dtype, "nhwc", pw_epilogue
        self.dw_epilogue = dw_epilogue
        self.device = torch.cuda.current_device() if device is None else device
        self.shape = L.make_shape(n, c, h, w, c, r, s, stride, pad, dil, c, "nhwc", dw_epilogue)
        self.n, self.c, self.h, self.w, self.k, self.r, self.s = n, c, h, w, k_out, r, s
        self.groups = 1
        h_ = ctypes.c_void_p()
        L.check(self.lib.wpk_dwpw_plan(ctypes.byref(self.shape), int(k_out), L.EPILOGUES[pw_epilogue],
                                       L.DTYPES[dtype], self.device, ctypes.byref(h_)))
        self.handle = h_
        self.p, self.q = output_dims(n, c, h, w, c, r, s, stride, pad, dil, c)
        self._ws = None
        self._ws_bytes = -1
        self._tdt = self._idt = _TORCH_DT[dtype]
        self._xs, self._ys = torch.Size((n, h, w, c)), torch.Size((n, self.p, self.q, k_out))
        self._hval = self.handle.value

    def x_shape(self):
        return tuple(self._xs)

    def y_shape(self):
        return tuple(self._ys)

    def run(self, x, w_dw, b_dw, w_pw, b_pw, y=None, stream=None, z=None):
        dt = self._tdt
        checks = ((x, "x", self.n * self.h * self.w * self.c), (w_dw, "w_dw", self.c * self.r * self.s),
                  (w_pw, "w_pw", self.k * self.c))
        if tuple(x.shape) != tuple(self._xs):
            raise ValueError(f"x: expected shape {tuple(self._xs)}, got {tuple(x.shape)}")
        for t, nm, numel in checks:
            if t.dtype is not dt or t.numel() != numel or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{nm}: expected contiguous cuda {dt} with {numel} elements, got {t.dtype} "
                                 f"{tuple(t.shape)}")
        for t, nm, numel in ((b_dw, "b_dw", self.c), (b_pw, "b_pw", self.k)):
            if t is not None and (t.dtype is not dt or t.numel() != numel or not t.is_cuda or not t.is_contiguous()):
                raise ValueError(f"{nm}: expected contiguous cuda {dt} [{numel}]")
        if y is None:
            y = torch.empty(self._ys, dtype=dt, device=x.device)
        elif y.dtype is not dt or y.shape != self._ys or not y.is_cuda or not y.is_contiguous():
            raise ValueError(f"y: expected contiguous cuda {dt} of shape {tuple(self._ys)}")
        if self._ws_bytes < 0:
            self._ensure_workspace()
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        L.check(self.lib.wpk_dwpw_run(self._hval, x.data_ptr(), w_dw.data_ptr(), ptr(b_dw), w_pw.data_ptr(),
                                      ptr(b_pw), y.data_ptr(), s))
        return y


def make_options(**kw) -> L.TuneOptions:
    """wpk_tune_options with defaults, overridden by keyword arguments (field names of wpk.h)."""
    o = L.TuneOptions()
    L.load().wpk_tune_options_init(ctypes.byref(o))
    keep = []
    for k, v in kw.items():
        if k in ("record_path", "replay_path", "log_path", "cache_dir"):
            v = v.encode() if v is not None else None
            keep.append(v)
        elif k == "eval_mode" and isinstance(v, str):
            v = L.EVAL_MODES[v]
        elif k == "family" and isinstance(v, str):
            v = L.FAMILIES[v]
        elif k == "synthetic":
            arr = (ctypes.c_double * (1 + 2 * L.NUM_GENES))(*v)
            v = arr
        elif k == "rl_hidden":
            v = (ctypes.c_int32 * 4)(*v)
        setattr(o, k, v)
    o._keep = keep
    return o
