"""NEXT-1 composition: a chained ResNet bottleneck block (BN folded into every conv, bias+ReLU
epilogues, the shortcut add fused into the last conv) against the oracle chain on the same inputs,
with the block's intermediate activations rounded to the I/O dtype exactly where the product stores
them (bf16 tolerance 2e-2 normwise, BASELINE.json)."""
import pytest
import torch

import oracle
from _util import TOL, rel_error

pytestmark = pytest.mark.gpu


def _rt(a, dt):
    """float64 numpy -> the I/O dtype (RN) -> float64 torch: where the product rounds."""
    return torch.from_numpy(a).to(dt).double()


@pytest.mark.parametrize("cfg", [(2, 64, 14, 14, 32, 64, 1), (2, 64, 14, 14, 32, 128, 2), (1, 128, 9, 11, 64, 256, 1)],
                         ids=["identity", "proj_s2", "proj_s1"])
def test_bottleneck_chain_matches_oracle(cfg):
    from paper_2008_04567_b200.blocks import BN, Bottleneck
    n, cin, h, w, mid, cout, stride = cfg
    dt = torch.bfloat16
    g = torch.Generator().manual_seed(7)

    def u(*shape, a=1.0):
        return (torch.rand(*shape, generator=g, dtype=torch.float64) * 2 - 1) * a

    def bn(k):
        return BN(gamma=(0.5 + torch.rand(k, generator=g)).float(), beta=(0.2 * u(k)).float(),
                  mean=(0.1 * u(k)).float(), var=(0.5 + torch.rand(k, generator=g)).float())

    blk = Bottleneck(n, cin, h, w, mid, cout, stride, dtype="bf16")
    shapes = [(mid, cin, 1, 1), (mid, mid, 3, 3), (cout, mid, 1, 1)] + ([(cout, cin, 1, 1)] if blk.proj else [])
    ws = [u(*s, a=(3.0 / (s[1] * s[2] * s[3])) ** 0.5).to(dt) for s in shapes]
    bs = [(0.1 * u(s[0])).to(dt) for s in shapes]
    bns = [bn(s[0]) for s in shapes]
    x = u(n, cin, h, w).to(dt)
    # product: NHWC activations and [K][R][S][C] weights
    blk.fold([wi.permute(0, 2, 3, 1).contiguous().cuda() for wi in ws], [bi.cuda() for bi in bs],
             [BN(*(t.cuda() for t in (b.gamma, b.beta, b.mean, b.var)), b.eps) for b in bns])
    y = blk(x.permute(0, 2, 3, 1).contiguous().cuda())
    torch.cuda.synchronize()
    got = y.permute(0, 3, 1, 2).cpu()
    # oracle chain: folds in float64, rounds folded weights / biases and stored activations to bf16
    folded = []
    for wi, bi, b in zip(ws, bs, bns):
        wf, bf = oracle.fold_batchnorm(wi, bi, b.gamma, b.beta, b.mean, b.var, b.eps)
        folded.append((_rt(wf, dt), _rt(bf, dt)))
    (w1, b1), (w2, b2), (w3, b3) = folded[:3]
    t1 = _rt(oracle.conv2d(x, w1, b1, stride=1, pad=0), dt)
    t2 = _rt(oracle.conv2d(t1, w2, b2, stride=stride, pad=1), dt)
    if blk.proj:
        wd, bd = folded[3]
        sc = _rt(oracle.conv2d(x, wd, bd, stride=stride, pad=0, relu=False), dt)
    else:
        sc = x.double()
    ref = oracle.conv2d(t2, w3, b3, stride=1, pad=0, residual=sc)
    err = rel_error("bf16", got, ref)
    assert err <= TOL["bf16"], err
    # an independent check of the fusion: the same block through torch fp64 reference ops
    import torch.nn.functional as F
    r1 = F.relu(F.conv2d(x.double(), w1, b1)).to(dt).double()
    r2 = F.relu(F.conv2d(r1, w2, b2, stride=stride, padding=1)).to(dt).double()
    rs = F.conv2d(x.double(), *folded[3], stride=stride).to(dt).double() if blk.proj else x.double()
    r3 = F.relu(F.conv2d(r2, w3, b3) + rs)
    assert rel_error("bf16", got, r3.numpy()) <= TOL["bf16"]
