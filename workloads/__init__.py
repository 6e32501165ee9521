"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds ONLY layer-shape tables and seeded input generators. It contains none of the
method's arithmetic (no convolution, no output-size formula used for checking, no search logic),
so both `oracle/` and the CUDA path may consume its outputs without sharing code (task rule ③).

Input recipe:
  * uniform mode:  x ~ U[-1,1),  w ~ U[-a,a) with a = sqrt(3/K_g), K_g = (C/g)*R*S,  b ~ U[-0.1,0.1)
  * int mode:      x, w ~ uniform over {-1,0,1},  b ~ uniform over {-4..4}
    (every partial sum is an integer < 2^24, so fp32 accumulation is exact on every path)
  * generation is fp32 on the CPU from torch.Generator().manual_seed(seed), then cast to the dtype.
  * seed = 4567 + 1000*config_id + layer_index.

Layer tables: ResNet-50 v1.5 (torchvision; stride on the 3x3), VGG-16, MobileNet-V2 (1.0, 224),
the paper's Table 1 (VALID chain) and BASELINE.json config 1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict, replace

import torch


@dataclass(frozen=True)
class ConvLayer:
    name: str
    n: int
    c: int
    h: int
    w: int
    k: int
    r: int
    s: int
    stride: int = 1
    pad: int = 0
    dil: int = 1
    groups: int = 1
    count: int = 1          # how many times this exact shape occurs in the network

    def with_batch(self, n: int) -> "ConvLayer":
        return replace(self, n=n)

    def as_dict(self) -> dict:
        return asdict(self)


# --- BASELINE.json configs[0]: N=1 C=3 H=W=8 K=8 R=S=3 stride 1 pad 1, fp32, bias+ReLU -------------
CONFIG1 = ConvLayer("config1", 1, 3, 8, 8, 8, 3, 3, 1, 1)


def _rn50(n: int) -> list[ConvLayer]:
    L = ConvLayer
    rows = [
        # name,        C,    H,   K,   R, stride, pad, count
        ("conv1",      3,  224,   64,  7, 2, 3, 1),
        ("s2b0.c1",   64,   56,   64,  1, 1, 0, 1),
        ("s2b0.c2",   64,   56,   64,  3, 1, 1, 3),
        ("s2b0.c3",   64,   56,  256,  1, 1, 0, 4),
        ("s2b1.c1",  256,   56,   64,  1, 1, 0, 2),
        ("s3b0.c1",  256,   56,  128,  1, 1, 0, 1),
        ("s3b0.c2",  128,   56,  128,  3, 2, 1, 1),
        ("s3b0.c3",  128,   28,  512,  1, 1, 0, 4),
        ("s3b0.ds",  256,   56,  512,  1, 2, 0, 1),
        ("s3b1.c1",  512,   28,  128,  1, 1, 0, 3),
        ("s3b1.c2",  128,   28,  128,  3, 1, 1, 3),
        ("s4b0.c1",  512,   28,  256,  1, 1, 0, 1),
        ("s4b0.c2",  256,   28,  256,  3, 2, 1, 1),
        ("s4b0.c3",  256,   14, 1024,  1, 1, 0, 6),
        ("s4b0.ds",  512,   28, 1024,  1, 2, 0, 1),
        ("s4b1.c1", 1024,   14,  256,  1, 1, 0, 5),
        ("s4b1.c2",  256,   14,  256,  3, 1, 1, 5),
        ("s5b0.c1", 1024,   14,  512,  1, 1, 0, 1),
        ("s5b0.c2",  512,   14,  512,  3, 2, 1, 1),
        ("s5b0.c3",  512,    7, 2048,  1, 1, 0, 3),
        ("s5b0.ds", 1024,   14, 2048,  1, 2, 0, 1),
        ("s5b1.c1", 2048,    7,  512,  1, 1, 0, 2),
        ("s5b1.c2",  512,    7,  512,  3, 1, 1, 2),
    ]
    return [L(nm, n, c, h, h, k, r, r, st, p, 1, 1, cnt) for (nm, c, h, k, r, st, p, cnt) in rows]


def resnet50(n: int = 32) -> list[ConvLayer]:
    """23 unique ResNet-50 v1.5 conv shapes (53 convs with multiplicity)."""
    return _rn50(n)


def resnet18(n: int = 1) -> list[ConvLayer]:
    """The 11 unique ResNet-18 conv shapes (20 convs with multiplicity) -- the network of the
    paper's per-convolution comparison (SURVEY.md 8(f) NEXT-3b; the paper labels
    them C1-C12 as TVM does). torchvision layout: stride on the first 3x3 of a stage, 1x1
    stride-2 downsample."""
    L = ConvLayer
    rows = [
        # name,      C,   H,   K,  R, stride, pad, count
        ("conv1",     3, 224,  64, 7, 2, 3, 1),
        ("s2.c",     64,  56,  64, 3, 1, 1, 4),
        ("s3b0.c1",  64,  56, 128, 3, 2, 1, 1),
        ("s3b0.ds",  64,  56, 128, 1, 2, 0, 1),
        ("s3.c",    128,  28, 128, 3, 1, 1, 3),
        ("s4b0.c1", 128,  28, 256, 3, 2, 1, 1),
        ("s4b0.ds", 128,  28, 256, 1, 2, 0, 1),
        ("s4.c",    256,  14, 256, 3, 1, 1, 3),
        ("s5b0.c1", 256,  14, 512, 3, 2, 1, 1),
        ("s5b0.ds", 256,  14, 512, 1, 2, 0, 1),
        ("s5.c",    512,   7, 512, 3, 1, 1, 3),
    ]
    out = [L(nm, n, c, h, h, k, r, r, st, p, 1, 1, cnt) for (nm, c, h, k, r, st, p, cnt) in rows]
    return out


def resnext50_grouped(n: int = 8) -> list[ConvLayer]:
    """The grouped 3x3 convs of ResNeXt-50 32x4d (groups 32, 4..32 channels per group; stride 2 on
    the first block of stages 3-5) -- the general-groups workload of SURVEY.md 8(f) NEXT-4."""
    L = ConvLayer
    rows = [
        # name,      C,   H, stride, count
        ("s2.g",    128, 56, 1, 3),
        ("s3b0.g",  256, 56, 2, 1),
        ("s3.g",    256, 28, 1, 3),
        ("s4b0.g",  512, 28, 2, 1),
        ("s4.g",    512, 14, 1, 5),
        ("s5b0.g", 1024, 14, 2, 1),
        ("s5.g",   1024,  7, 1, 2),
    ]
    return [L(nm, n, c, h, h, c, 3, 3, st, 1, 1, 32, cnt) for (nm, c, h, st, cnt) in rows]


def vgg16(n: int = 64) -> list[ConvLayer]:
    rows = [("conv1_1", 3, 224, 64, 1), ("conv1_2", 64, 224, 64, 1),
            ("conv2_1", 64, 112, 128, 1), ("conv2_2", 128, 112, 128, 1),
            ("conv3_1", 128, 56, 256, 1), ("conv3_2", 256, 56, 256, 2),
            ("conv4_1", 256, 28, 512, 1), ("conv4_2", 512, 28, 512, 2),
            ("conv5_x", 512, 14, 512, 3)]
    return [ConvLayer(nm, n, c, h, h, k, 3, 3, 1, 1, 1, 1, cnt) for (nm, c, h, k, cnt) in rows]


def mobilenet_v2(n: int = 1) -> list[ConvLayer]:
    """MobileNet-V2 (width 1.0, 224): stem, 17 inverted-residual blocks, final 1x1. Unique shapes."""
    layers: list[ConvLayer] = []
    layers.append(ConvLayer("stem", n, 3, 224, 224, 32, 3, 3, 2, 1))
    h, cin = 112, 32
    blocks = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
              (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
    bi = 0
    for t, cout, reps, s0 in blocks:
        for i in range(reps):
            s = s0 if i == 0 else 1
            hid = cin * t
            if t != 1:
                layers.append(ConvLayer(f"b{bi}.expand", n, cin, h, h, hid, 1, 1, 1, 0))
            layers.append(ConvLayer(f"b{bi}.dw", n, hid, h, h, hid, 3, 3, s, 1, 1, hid))
            h = h // s
            layers.append(ConvLayer(f"b{bi}.project", n, hid, h, h, cout, 1, 1, 1, 0))
            cin = cout
            bi += 1
    layers.append(ConvLayer("final", n, 320, 7, 7, 1280, 1, 1, 1, 0))
    # merge identical shapes (computationally identical convs)
    uniq: dict[tuple, ConvLayer] = {}
    for L in layers:
        key = (L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups)
        if key in uniq:
            uniq[key] = replace(uniq[key], count=uniq[key].count + 1)
        else:
            uniq[key] = L
    return list(uniq.values())


@dataclass(frozen=True)
class DwPwBlock:
    """A depthwise conv and the 1x1 projection that consumes it (the fused-operator unit of
    wpk_dwpw_*): y = project(relu(dw(x) + b_dw)) + b_pw (MobileNet-V2's projection is linear)."""
    name: str
    dw: ConvLayer
    k_out: int
    count: int = 1


def mobilenet_v2_dwpw(n: int = 1) -> list[DwPwBlock]:
    """The 17 (depthwise 3x3 -> 1x1 projection) pairs of MobileNet-V2 (width 1.0, 224), merged by
    shape: the fused-operator view of mobilenet_v2() (same dw / project shapes)."""
    h, cin = 112, 32
    blocks = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
              (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
    out: dict[tuple, DwPwBlock] = {}
    bi = 0
    for t, cout, reps, s0 in blocks:
        for i in range(reps):
            s = s0 if i == 0 else 1
            hid = cin * t
            dw = ConvLayer(f"b{bi}.dw", n, hid, h, h, hid, 3, 3, s, 1, 1, hid)
            key = (hid, h, s, cout)
            if key in out:
                out[key] = replace(out[key], count=out[key].count + 1)
            else:
                out[key] = DwPwBlock(f"b{bi}", dw, cout)
            h = h // s
            cin = cout
            bi += 1
    return list(out.values())


def table1(n: int = 1) -> list[ConvLayer]:
    """PAPER.md:162-177 Table 1 ("Convolutions on which RL-search outperforms genetic search").
    Padding is VALID: the table's H/W chain is self-consistent only without padding."""
    rows = [("conv1a", 112, 96, 3, 64, 1), ("conv1b", 110, 94, 64, 96, 2),
            ("conv2", 54, 46, 96, 128, 2), ("conv3", 26, 22, 128, 256, 2),
            ("conv4", 12, 10, 256, 512, 1)]
    return [ConvLayer(nm, n, ci, h, w, co, 3, 3, st, 0) for (nm, h, w, ci, co, st) in rows]


def config_seed(config_id: int, layer_index: int) -> int:
    return 4567 + 1000 * config_id + layer_index


# element type of b / z / y per dtype name; x and w use _DT_IN ("fp8" = OCP e4m3 operands with a
# bf16 bias and output, the library's WPK_FP8E4M3)
_DT = {"f32": torch.float32, "tf32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16,
       "fp8": torch.bfloat16}
_DT_IN = dict(_DT, fp8=torch.float8_e4m3fn)


def torch_dtype(dtype: str) -> torch.dtype:
    """Element type of b / z / y for `dtype` (x / w: torch_in_dtype)."""
    return _DT[dtype]


def torch_in_dtype(dtype: str) -> torch.dtype:
    return _DT_IN[dtype]


def generate(layer: ConvLayer, dtype: str = "f32", mode: str = "uniform", seed: int = 0,
             bias: bool = True):
    """Seeded CPU tensors in canonical NCHW / KCRS layout, already rounded to `dtype`.

    Returns (x[N,C,H,W], w[K,C/g,R,S], b[K] or None), torch CPU tensors: x and w of
    torch_in_dtype(dtype), b of torch_dtype(dtype) (they differ only for "fp8"). The fp32 draws are
    rounded to nearest by torch's cast; the uniform ranges stay inside e4m3's finite range (|v| <= 1).
    """
    g = torch.Generator().manual_seed(int(seed))
    cpg = layer.c // layer.groups
    xs = (layer.n, layer.c, layer.h, layer.w)
    ws = (layer.k, cpg, layer.r, layer.s)
    if mode == "uniform":
        kg = cpg * layer.r * layer.s
        a = math.sqrt(3.0 / kg)
        x = torch.rand(xs, generator=g, dtype=torch.float32) * 2 - 1
        w = (torch.rand(ws, generator=g, dtype=torch.float32) * 2 - 1) * a
        b = (torch.rand((layer.k,), generator=g, dtype=torch.float32) * 2 - 1) * 0.1
    elif mode == "int":
        x = torch.randint(-1, 2, xs, generator=g).to(torch.float32)
        w = torch.randint(-1, 2, ws, generator=g).to(torch.float32)
        b = torch.randint(-4, 5, (layer.k,), generator=g).to(torch.float32)
    elif mode == "ones":
        x = torch.ones(xs)
        w = torch.ones(ws)
        b = torch.zeros(layer.k)
    else:
        raise ValueError(mode)
    dt, it = _DT[dtype], _DT_IN[dtype]
    return x.to(it), w.to(it), (b.to(dt) if bias else None)


def random_points(layer: ConvLayer, p: int, q: int, count: int, seed: int):
    """Seeded sample of output coordinates (n,k,p,q): every border position of image 0 /
    channel 0..min(K,4)-1 plus `count` uniform interior draws. p, q are the output sizes."""
    g = torch.Generator().manual_seed(int(seed) + 77)
    pts = []
    for kk in range(min(layer.k, 4)):
        for pp in range(p):
            for qq in range(q):
                if pp in (0, p - 1) or qq in (0, q - 1):
                    pts.append((0, kk, pp, qq))
    n = torch.randint(0, layer.n, (count,), generator=g)
    k = torch.randint(0, layer.k, (count,), generator=g)
    pp = torch.randint(0, p, (count,), generator=g)
    qq = torch.randint(0, q, (count,), generator=g)
    pts += list(zip(n.tolist(), k.tolist(), pp.tolist(), qq.tolist()))
    return torch.tensor(pts, dtype=torch.int64)


def parity_points(layer: ConvLayer, p: int, q: int, interior: int = 65536, seed: int = 0,
                  border_channels: int | None = None):
    """Seeded full-size parity sample of output coordinates (n, k, p, q) ("all
    border rows/columns + >= 65,536 random interior outputs per layer"): every border pixel
    (p in {0, P-1} or q in {0, Q-1}) of EVERY image, for every output channel (or, with
    border_channels=c, for c channels per pixel rotating through all K), plus `interior` uniform
    draws from the non-border pixels (all pixels when P or Q <= 2). Returns an int64 [count, 4]."""
    g = torch.Generator().manual_seed(int(seed) + 4567)
    pp, qq = torch.meshgrid(torch.arange(p), torch.arange(q), indexing="ij")
    border = (pp == 0) | (pp == p - 1) | (qq == 0) | (qq == q - 1)
    bp, bq = pp[border], qq[border]                       # [nb]
    nb = bp.numel()
    if border_channels is None or border_channels >= layer.k:
        ks = torch.arange(layer.k)
        n_idx = torch.arange(layer.n).view(-1, 1, 1).expand(layer.n, nb, layer.k)
        k_idx = ks.view(1, 1, -1).expand(layer.n, nb, layer.k)
        p_idx = bp.view(1, -1, 1).expand(layer.n, nb, layer.k)
        q_idx = bq.view(1, -1, 1).expand(layer.n, nb, layer.k)
    else:
        c = border_channels
        n_idx = torch.arange(layer.n).view(-1, 1, 1).expand(layer.n, nb, c)
        off = (torch.arange(layer.n).view(-1, 1, 1) * nb + torch.arange(nb).view(1, -1, 1)) * c
        k_idx = (off + torch.arange(c).view(1, 1, -1)) % layer.k
        p_idx = bp.view(1, -1, 1).expand(layer.n, nb, c)
        q_idx = bq.view(1, -1, 1).expand(layer.n, nb, c)
    bpts = torch.stack([n_idx.reshape(-1), k_idx.reshape(-1), p_idx.reshape(-1), q_idx.reshape(-1)], 1)
    inner = ~border if (p > 2 and q > 2) else torch.ones_like(border)
    ip, iq = pp[inner], qq[inner]
    sel = torch.randint(0, ip.numel(), (interior,), generator=g)
    n = torch.randint(0, layer.n, (interior,), generator=g)
    k = torch.randint(0, layer.k, (interior,), generator=g)
    ipts = torch.stack([n, k, ip[sel], iq[sel]], 1)
    return torch.cat([bpts, ipts]).to(torch.int64)
