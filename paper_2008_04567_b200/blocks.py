"""NEXT-1 composition: a ResNet bottleneck block (1x1 -> 3x3 -> 1x1 + shortcut) whose every operator is
one fused kernel of the library ("write one CUDA kernel function for the fused operator";
PAPER.md:35 operator fusion): inference batch-norm is folded into each conv's weights and bias once
(wpk_conv2d_fold_batchnorm), conv1 / conv2 carry bias + ReLU in their epilogue, and conv3 carries the
shortcut add + ReLU (WPK_EPI_BIAS_ADD_RELU, y = relu(conv(x) + b + z)); a projection shortcut is a
fourth plan with the bias-only epilogue. Activations are NHWC in the plan dtype and stay on the device
(L2-resident between the chained convs). Argument marshalling and plan bookkeeping only: every
arithmetic step runs in libwpk.so (no torch compute on this path).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .conv import Conv2dPlan


@dataclass
class BN:
    """Inference batch-norm statistics of one conv's output channels (fp32 [K])."""
    gamma: torch.Tensor
    beta: torch.Tensor
    mean: torch.Tensor
    var: torch.Tensor
    eps: float = 1e-5


class Bottleneck:
    """ResNet v1.5 bottleneck on NHWC activations: stride on the 3x3 (torchvision convention).
    Weights are passed NHWC-packed ([K][R][S][C], torch channels_last) in the plan dtype, with
    optional conv bias and a BN per conv; fold() turns them into the fused kernels' (w', b')."""

    def __init__(self, n, c_in, h, w, mid, c_out, stride=1, dtype="bf16", device=None):
        self.n, self.c_in, self.h, self.w, self.mid, self.c_out, self.stride = n, c_in, h, w, mid, c_out, stride
        self.dtype = dtype
        self.ho, self.wo = (h - 1) // stride + 1, (w - 1) // stride + 1
        kw = dict(layout="nhwc", dtype=dtype, device=device)
        self.c1 = Conv2dPlan(n, c_in, h, w, mid, 1, 1, 1, 0, epilogue="bias_relu", **kw)
        self.c2 = Conv2dPlan(n, mid, h, w, mid, 3, 3, stride, 1, epilogue="bias_relu", **kw)
        self.c3 = Conv2dPlan(n, mid, self.ho, self.wo, c_out, 1, 1, 1, 0, epilogue="bias_add_relu", **kw)
        self.proj = stride != 1 or c_in != c_out
        self.ds = Conv2dPlan(n, c_in, h, w, c_out, 1, 1, stride, 0, epilogue="bias", **kw) if self.proj else None
        self.params = None
        self._bufs = None

    def plans(self):
        return [p for p in (self.c1, self.c2, self.c3, self.ds) if p is not None]

    def fold(self, weights, biases, bns, stream=None):
        """weights / biases / bns: lists for (c1, c2, c3[, ds]); bias entries may be None. Folds
        each BN into its conv on the device (one small kernel each) and keeps (w', b')."""
        self.params = []
        for plan, w, b, bn in zip(self.plans(), weights, biases, bns):
            if bn is None:
                if b is None:
                    b = torch.zeros(plan.k, dtype=w.dtype, device=w.device)
                self.params.append((w, b))
            else:
                self.params.append(plan.fold_batchnorm(w, b, bn.gamma, bn.beta, bn.mean, bn.var, bn.eps,
                                                       stream=stream))
        return self

    def tune(self, search="ga", budget=32, **kw):
        return [p.tune(search, budget, **kw) for p in self.plans()]

    def _buffers(self, x):
        key = (x.device, x.dtype)
        if self._bufs is None or self._bufs[0] != key:
            e = dict(dtype=x.dtype, device=x.device)
            self._bufs = (key, torch.empty(self.c1.y_shape(), **e), torch.empty(self.c2.y_shape(), **e),
                          torch.empty(self.ds.y_shape(), **e) if self.ds is not None else None)
        return self._bufs[1:]

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """x: [N][H][W][C_in] NHWC -> y: [N][Ho][Wo][C_out]; 3 (or 4) kernel launches on `stream`."""
        if self.params is None:
            raise RuntimeError("Bottleneck.fold() first")
        t1, t2, sc = self._buffers(x)
        (w1, b1), (w2, b2), (w3, b3) = self.params[:3]
        if y is None:
            y = torch.empty(self.c3.y_shape(), dtype=x.dtype, device=x.device)
        self.c1.run(x, w1, b1, t1, stream=stream)
        self.c2.run(t1, w2, b2, t2, stream=stream)
        if self.ds is not None:
            wd, bd = self.params[3]
            self.ds.run(x, wd, bd, sc, stream=stream)
        else:
            sc = x
        self.c3.run(t2, w3, b3, y, stream=stream, z=sc)
        return y

    __call__ = forward
