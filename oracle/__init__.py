"""oracle/ -- TEST INFRASTRUCTURE ONLY (task rule ③).

A plain, slow, obviously-correct CPU implementation of what the hot path computes:

  * `conv2d`, `conv2d_points`  -- the forward convolution + bias + ReLU in double precision
    (oracle/conv_oracle.c, a 7-loop written from PAPER.md:47 and SURVEY.md §8(c) Part 1);
  * `oracle.search`            -- the paper's search arithmetic step by step: GA Eq. (1)-(2),
    roulette inverse sampling, elitism, convergence (§2.3); the RL-search
    moving average, reward, GAE and PPO loss/gradient (§2.4).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
import this package. The product package (paper_2008_04567_b200) never imports it and shares no
code with it; both consume inputs from `workloads/` only.

Parity-unpinned functions: none in this package (every function has a pin in
tests/test_oracle_conv.py or tests/test_oracle_search.py); kernel *speed* is unpinned
 and is not an oracle function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, OpenMP for the outer (n,k) loop only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i32p = ctypes.POINTER(ctypes.c_int32)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.wpk_oracle_conv2d.argtypes = [i32p, dp, dp, dp, dp, ctypes.c_int]
        lib.wpk_oracle_conv2d_res.argtypes = [i32p, dp, dp, dp, dp, dp, ctypes.c_int]
        lib.wpk_oracle_conv2d_points.argtypes = [i32p, dp, dp, dp, ctypes.POINTER(ctypes.c_int64),
                                                 ctypes.c_int64, dp, ctypes.c_int]
        lib.wpk_oracle_out_dims.argtypes = [i32p, i32p, i32p]
        _lib = lib
    return _lib


EPI_NONE, EPI_BIAS, EPI_BIAS_RELU, EPI_BIAS_ADD_RELU = 0, 1, 2, 3


def _shape(n, c, h, w, k, r, s, stride, pad, dil, groups, epilogue):
    sh, sw = (stride, stride) if np.isscalar(stride) else stride
    ph, pw = (pad, pad) if np.isscalar(pad) else pad
    dh, dw = (dil, dil) if np.isscalar(dil) else dil
    return np.array([n, c, h, w, k, r, s, sh, sw, ph, pw, dh, dw, groups, epilogue], dtype=np.int32)


def _as_f64(a):
    if a is None:
        return None
    try:  # torch tensor (any dtype, incl. bf16) -> exact float64 copy
        import torch
        if isinstance(a, torch.Tensor):
            return np.ascontiguousarray(a.detach().to("cpu", torch.float64).numpy())
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def out_dims(n, c, h, w, k, r, s, stride=1, pad=0, dil=1, groups=1):
    sh = _shape(n, c, h, w, k, r, s, stride, pad, dil, groups, 0)
    p, q = ctypes.c_int32(), ctypes.c_int32()
    _load().wpk_oracle_out_dims(sh.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                ctypes.byref(p), ctypes.byref(q))
    return p.value, q.value


def conv2d(x, w, b=None, stride=1, pad=0, dil=1, groups=1, relu=True, nthreads=1, residual=None):
    """y[N,K,P,Q] (float64) for x[N,C,H,W], w[K,C/g,R,S], b[K] (NCHW/KCRS). With residual
    z[N,K,P,Q]: y = max(conv + b + z, 0) (epilogue 3, the ResNet block's residual-add fusion)."""
    if residual is not None:
        return _conv2d_res(x, w, b, residual, stride, pad, dil, groups, nthreads)
    x, w, b = _as_f64(x), _as_f64(w), _as_f64(b)
    n, c, h, wd = x.shape
    k, cpg, r, s = w.shape
    if cpg * groups != c:
        raise ValueError("C/groups mismatch")
    epi = EPI_NONE if b is None else (EPI_BIAS_RELU if relu else EPI_BIAS)
    if b is None:
        b = np.zeros(k)
    sh = _shape(n, c, h, wd, k, r, s, stride, pad, dil, groups, epi)
    p, q = out_dims(n, c, h, wd, k, r, s, stride, pad, dil, groups)
    if p < 1 or q < 1:
        raise ValueError("empty output")
    y = np.zeros((n, k, p, q), dtype=np.float64)
    rc = _load().wpk_oracle_conv2d(sh.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   _ptr(x), _ptr(w), _ptr(b), _ptr(y), int(nthreads))
    if rc != 0:
        raise ValueError("invalid shape")
    return y


def _conv2d_res(x, w, b, z, stride, pad, dil, groups, nthreads):
    x, w, b, z = _as_f64(x), _as_f64(w), _as_f64(b), _as_f64(z)
    n, c, h, wd = x.shape
    k, cpg, r, s = w.shape
    if b is None:
        b = np.zeros(k)
    sh = _shape(n, c, h, wd, k, r, s, stride, pad, dil, groups, EPI_BIAS_ADD_RELU)
    p, q = out_dims(n, c, h, wd, k, r, s, stride, pad, dil, groups)
    if p < 1 or q < 1 or z.shape != (n, k, p, q):
        raise ValueError("empty output or residual shape mismatch")
    y = np.zeros((n, k, p, q), dtype=np.float64)
    rc = _load().wpk_oracle_conv2d_res(sh.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       _ptr(x), _ptr(w), _ptr(b), _ptr(z), _ptr(y), int(nthreads))
    if rc != 0:
        raise ValueError("invalid shape")
    return y


def conv2d_points(x, w, b, pts, stride=1, pad=0, dil=1, groups=1, relu=True, nthreads=1):
    """y at the given (n,k,p,q) points (int64 array [npts,4]); float64 [npts]."""
    x, w, b = _as_f64(x), _as_f64(w), _as_f64(b)
    n, c, h, wd = x.shape
    k, cpg, r, s = w.shape
    epi = EPI_NONE if b is None else (EPI_BIAS_RELU if relu else EPI_BIAS)
    if b is None:
        b = np.zeros(k)
    sh = _shape(n, c, h, wd, k, r, s, stride, pad, dil, groups, epi)
    pts = np.ascontiguousarray(np.asarray(pts, dtype=np.int64).reshape(-1, 4))
    out = np.zeros(pts.shape[0], dtype=np.float64)
    rc = _load().wpk_oracle_conv2d_points(
        sh.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _ptr(x), _ptr(w), _ptr(b),
        pts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pts.shape[0], _ptr(out), int(nthreads))
    if rc != 0:
        raise ValueError("invalid points/shape")
    return out


def fold_batchnorm(w, b, gamma, beta, mean, var, eps):
    """Inference batch-norm folded into (w, b), in float64 (SURVEY.md 8(f) NEXT-1b):
    s_k = gamma_k / sqrt(var_k + eps); w'[k] = w[k] * s_k; b'_k = (b_k - mean_k) * s_k + beta_k.
    Test infrastructure only."""
    w, gamma, beta, mean, var = (_as_f64(t) for t in (w, gamma, beta, mean, var))
    b = np.zeros(w.shape[0]) if b is None else _as_f64(b)
    s = gamma / np.sqrt(var + eps)
    return w * s.reshape((-1,) + (1,) * (w.ndim - 1)), (b - mean) * s + beta
