"""Pins for the convolution oracle. CPU only.

Each test checks the oracle against something other than itself: hand-computed values
(tests/golden/conv_hand_examples.json), closed forms, identities, a naive matmul, and torch's
float64 CPU convolution (a library routine)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "conv_hand_examples.json")))


def _arr(v):
    return np.array(v, dtype=np.float64)


@pytest.mark.parametrize("key", ["p1_scalar", "p2_pad1", "p2_pad0", "p2_stride2", "p2_bias_relu",
                                 "p3_flip_detector"])
def test_hand_examples(oracle_lib, key):
    g = GOLD[key]
    b = _arr(g["b"]) if "b" in g else None
    y = oracle.conv2d(_arr(g["x"]), _arr(g["w"]), b, stride=g["stride"], pad=g["pad"])
    np.testing.assert_array_equal(y, _arr(g["y"]))


def test_dilation_example(oracle_lib):
    g = GOLD["p4_dilation"]
    x = np.arange(1, g["x_range"] + 1, dtype=np.float64).reshape(1, 1, g["hw"], g["hw"])
    y = oracle.conv2d(x, np.ones((1, 1, 3, 3)), None, pad=g["pad"], dil=g["dil"])
    assert y.shape == (1, 1, 5, 5)
    np.testing.assert_array_equal(y[0, 0, 0], g["row0"])
    assert y[0, 0, 2, 2] == g["centre"]


def test_config1_all_ones_closed_form(oracle_lib):
    g = GOLD["p5_config1_all_ones"]
    L = workloads.CONFIG1
    x, w, b = workloads.generate(L, "f32", "ones")
    y = oracle.conv2d(x, w, b, stride=1, pad=1)
    assert y.shape == (1, 8, 8, 8)
    assert y[0, 0, 0, 0] == g["corner"] and y[0, 5, 0, 3] == g["edge"] and y[0, 7, 4, 4] == g["interior"]
    assert y.sum() == g["sum"]

    # general closed form y = C * cnt_h(p) * cnt_w(q), cnt = number of in-bounds taps
    def cnt(p, n=8):
        return sum(1 for r in range(3) if 0 <= p - 1 + r < n)
    for p in range(8):
        for q in range(8):
            assert (y[0, :, p, q] == 3 * cnt(p) * cnt(q)).all()


def test_delta_filter_shift_identity(oracle_lib):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 3, 9, 7))
    for (c0, r0, s0, stride, pad, dil) in [(1, 0, 2, 1, 1, 1), (2, 2, 1, 2, 2, 1), (0, 1, 1, 1, 0, 2),
                                           (1, 1, 1, 1, 1, 1)]:
        w = np.zeros((4, 3, 3, 3))
        w[:, c0, r0, s0] = 1.0
        y = oracle.conv2d(x, w, None, stride=stride, pad=pad, dil=dil)
        P, Q = y.shape[2:]
        for p in range(P):
            for q in range(Q):
                hi, wi = p * stride - pad + r0 * dil, q * stride - pad + s0 * dil
                want = x[:, c0, hi, wi] if (0 <= hi < 9 and 0 <= wi < 7) else 0.0
                for k in range(4):
                    np.testing.assert_array_equal(y[:, k, p, q], want)
    # centre delta with pad (R-1)/2 is the identity
    w = np.zeros((3, 3, 3, 3))
    for c in range(3):
        w[c, c, 1, 1] = 1.0
    np.testing.assert_array_equal(oracle.conv2d(x, w, None, pad=1), x)


def _naive_matmul(A, B):
    n, m = len(A), len(B[0])
    out = [[0.0] * m for _ in range(n)]
    for i in range(n):
        for j in range(m):
            s = 0.0
            for t in range(len(B)):
                s += A[i][t] * B[t][j]
            out[i][j] = s
    return np.array(out)


def test_1x1_is_matmul(oracle_lib):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 5, 4, 6))
    w = rng.standard_normal((7, 5, 1, 1))
    y = oracle.conv2d(x, w, None)
    for n in range(2):
        X = x[n].reshape(5, -1)                            # [C, H*W]
        want = _naive_matmul(w[:, :, 0, 0].tolist(), X.tolist())
        np.testing.assert_allclose(y[n].reshape(7, -1), want, rtol=1e-13, atol=1e-13)
    # stride 2 1x1 == matmul on the subsampled pixels
    y2 = oracle.conv2d(x, w, None, stride=2)
    for n in range(2):
        X = x[n][:, ::2, ::2].reshape(5, -1)
        want = _naive_matmul(w[:, :, 0, 0].tolist(), X.tolist())
        np.testing.assert_allclose(y2[n].reshape(7, -1), want, rtol=1e-13, atol=1e-13)


def test_groups_is_concatenation_and_depthwise(oracle_lib):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((1, 6, 7, 7))
    w = rng.standard_normal((9, 2, 3, 3))
    y = oracle.conv2d(x, w, None, pad=1, groups=3)
    for g in range(3):
        yg = oracle.conv2d(x[:, 2 * g:2 * g + 2], w[3 * g:3 * g + 3], None, pad=1)
        np.testing.assert_array_equal(y[:, 3 * g:3 * g + 3], yg)
    wd = rng.standard_normal((6, 1, 3, 3))
    yd = oracle.conv2d(x, wd, None, stride=2, pad=1, groups=6)
    for c in range(6):
        np.testing.assert_array_equal(yd[:, c:c + 1], oracle.conv2d(x[:, c:c + 1], wd[c:c + 1], None,
                                                                     stride=2, pad=1))


def test_linearity_and_explicit_padding(oracle_lib):
    rng = np.random.default_rng(4)
    x1, x2 = rng.standard_normal((2, 2, 3, 6, 5))
    w1, w2 = rng.standard_normal((2, 4, 3, 3, 3))
    a, c = 0.7, -1.3
    y = oracle.conv2d(a * x1 + c * x2, w1, None, pad=1)
    np.testing.assert_allclose(y, a * oracle.conv2d(x1, w1, None, pad=1) + c * oracle.conv2d(x2, w1, None, pad=1),
                               rtol=1e-12, atol=1e-12)
    y = oracle.conv2d(x1, a * w1 + c * w2, None, pad=1)
    np.testing.assert_allclose(y, a * oracle.conv2d(x1, w1, None, pad=1) + c * oracle.conv2d(x1, w2, None, pad=1),
                               rtol=1e-12, atol=1e-12)
    xp = np.pad(x1, ((0, 0), (0, 0), (1, 1), (1, 1)))
    np.testing.assert_array_equal(oracle.conv2d(x1, w1, None, pad=1), oracle.conv2d(xp, w1, None, pad=0))


@pytest.mark.parametrize("case", range(12))
def test_vs_torch_float64(oracle_lib, case):
    g = torch.Generator().manual_seed(100 + case)
    ri = lambda lo, hi: int(torch.randint(lo, hi + 1, (1,), generator=g))
    groups = [1, 1, 2, 3][case % 4]
    c = groups * ri(1, 4)
    k = groups * ri(1, 4)
    if case % 5 == 0:              # depthwise
        groups, c, k = 4, 4, 4
    r, s = ri(1, 4), ri(1, 4)
    stride, pad, dil = (ri(1, 3), ri(1, 2)), (ri(0, 2), ri(0, 2)), (ri(1, 2), ri(1, 2))
    h = dil[0] * (r - 1) + 1 + ri(0, 6)
    w_ = dil[1] * (s - 1) + 1 + ri(0, 6)
    x = torch.randn(ri(1, 3), c, h, w_, generator=g, dtype=torch.float64)
    w = torch.randn(k, c // groups, r, s, generator=g, dtype=torch.float64)
    b = torch.randn(k, generator=g, dtype=torch.float64)
    want = torch.relu(torch.nn.functional.conv2d(x, w, b, stride, pad, dil, groups)).numpy()
    got = oracle.conv2d(x.numpy(), w.numpy(), b.numpy(), stride, pad, dil, groups)
    assert got.shape == want.shape
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_points_match_full(oracle_lib):
    L = workloads.ConvLayer("t", 2, 8, 9, 9, 16, 3, 3, 2, 1)
    x, w, b = workloads.generate(L, "f32", "uniform", seed=5)
    y = oracle.conv2d(x, w, b, stride=2, pad=1)
    pts = workloads.random_points(L, y.shape[2], y.shape[3], 50, seed=5).numpy()
    got = oracle.conv2d_points(x, w, b, pts, stride=2, pad=1)
    want = y[pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    np.testing.assert_array_equal(got, want)


def test_table1_is_a_valid_chain(oracle_lib):
    """p11: Table 1 is self-consistent only under VALID padding."""
    rows = workloads.table1()
    for a, b in zip(rows, rows[1:]):
        p, q = oracle.out_dims(a.n, a.c, a.h, a.w, a.k, a.r, a.s, a.stride, 0)
        assert (p, q) == (b.h, b.w) and a.k == b.c
        ps, qs = oracle.out_dims(a.n, a.c, a.h, a.w, a.k, a.r, a.s, a.stride, 1)   # SAME-style pad
        assert (ps, qs) != (b.h, b.w)


def test_invalid_shapes_rejected(oracle_lib):
    with pytest.raises(ValueError):
        oracle.conv2d(np.ones((1, 1, 2, 2)), np.ones((1, 1, 3, 3)), None)      # empty output
    with pytest.raises(ValueError):
        oracle.conv2d(np.ones((1, 3, 4, 4)), np.ones((2, 2, 1, 1)), None, groups=2)


# ---- residual-add epilogue (epilogue 3: y = max(conv + b + z, 0)) ----------
def test_residual_closed_forms(oracle_lib):
    """Pins of the residual epilogue against forms that do not go through it: z = 0 is the
    bias+ReLU epilogue; a per-channel constant z folds into the bias (so z is indexed by k and added
    before the ReLU); a 1x1 identity filter gives relu(x + b + z) written out in numpy; z = -(conv+b)
    gives exactly zero."""
    rng = np.random.default_rng(5)
    x = rng.integers(-3, 4, size=(2, 4, 6, 5)).astype(np.float64)
    w = rng.integers(-2, 3, size=(6, 4, 3, 3)).astype(np.float64)
    b = rng.integers(-4, 5, size=6).astype(np.float64)
    base = oracle_lib.conv2d(x, w, b, stride=1, pad=1, relu=True)
    pre = oracle_lib.conv2d(x, w, b, stride=1, pad=1, relu=False)
    z0 = np.zeros_like(base)
    assert np.array_equal(oracle_lib.conv2d(x, w, b, stride=1, pad=1, residual=z0), base)
    cst = rng.integers(-5, 6, size=6).astype(np.float64)
    zc = np.broadcast_to(cst[None, :, None, None], base.shape).copy()
    assert np.array_equal(oracle_lib.conv2d(x, w, b, stride=1, pad=1, residual=zc),
                          oracle_lib.conv2d(x, w, b + cst, stride=1, pad=1, relu=True))
    assert np.array_equal(oracle_lib.conv2d(x, w, b, stride=1, pad=1, residual=-pre), np.zeros_like(base))
    eye = np.zeros((4, 4, 1, 1))
    eye[np.arange(4), np.arange(4)] = 1.0
    z = rng.integers(-6, 7, size=x.shape).astype(np.float64)
    bi = rng.integers(-4, 5, size=4).astype(np.float64)
    want = np.maximum(x + bi[None, :, None, None] + z, 0.0)
    assert np.array_equal(oracle_lib.conv2d(x, eye, bi, residual=z), want)


def test_residual_vs_torch_float64(oracle_lib):
    g = torch.Generator().manual_seed(11)
    x = torch.randn(2, 5, 9, 7, generator=g, dtype=torch.float64)
    w = torch.randn(8, 5, 3, 3, generator=g, dtype=torch.float64)
    b = torch.randn(8, generator=g, dtype=torch.float64)
    ref0 = torch.nn.functional.conv2d(x, w, b, stride=2, padding=1)
    z = torch.randn(ref0.shape, generator=g, dtype=torch.float64)
    ref = torch.relu(ref0 + z).numpy()
    got = oracle_lib.conv2d(x, w, b, stride=2, pad=1, residual=z)
    assert np.abs(got - ref).max() < 1e-12


def test_fold_batchnorm_closed_form(oracle_lib):
    """conv(x, w') + b' equals batch-norm applied to conv(x, w) + b, written out directly
    (gamma * (t - mean) / sqrt(var + eps) + beta per output channel)."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((2, 3, 7, 6))
    w = rng.standard_normal((5, 3, 3, 3))
    b = rng.standard_normal(5)
    gamma, beta = rng.standard_normal(5), rng.standard_normal(5)
    mean, var, eps = rng.standard_normal(5), rng.uniform(0.1, 2.0, 5), 1e-3
    t = oracle_lib.conv2d(x, w, b, stride=1, pad=1, relu=False)
    bn = gamma[None, :, None, None] * (t - mean[None, :, None, None]) / np.sqrt(var + eps)[None, :, None, None] \
        + beta[None, :, None, None]
    wf, bf = oracle.fold_batchnorm(w, b, gamma, beta, mean, var, eps)
    got = oracle_lib.conv2d(x, wf, bf, stride=1, pad=1, relu=False)
    assert np.abs(got - bn).max() < 1e-12
    # gamma = sqrt(var + eps), beta = mean, b = mean: the identity fold
    wi, bi = oracle.fold_batchnorm(w, mean, np.sqrt(var + eps), mean, mean, var, eps)
    assert np.allclose(wi, w, rtol=1e-15, atol=0) and np.allclose(bi, mean, rtol=1e-15, atol=1e-15)
