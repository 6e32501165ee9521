"""Pins for the search oracle. CPU only.

Formula examples come from tests/golden/search_formula_examples.json (paper formulas, SPEC worked
examples, with S:258's erratum corrected by hand). The PPO gradient is pinned by central finite
differences; GAE by the explicit double sum; the GA by the whole-space enumeration optimum and
by dominance over random search on a synthetic surface with a known optimum."""
import json
import math
import os

import numpy as np
import pytest

from oracle import search as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "search_formula_examples.json")))


def test_eq1_eq2_roulette():
    g = GOLD["eq1"]
    np.testing.assert_allclose(S.selection_probabilities(g["f"]), g["p"], rtol=0, atol=1e-15)
    g = GOLD["eq2"]
    np.testing.assert_allclose(S.cumulative_probabilities(g["p"]), g["P"], rtol=0, atol=1e-15)
    g = GOLD["roulette"]
    for v, want in g["cases"]:
        assert S.roulette(g["P"], v) + 1 == want
    assert S.selection_probabilities([2.0]) == [1.0]
    assert S.selection_probabilities([3.0] * 4) == [0.25] * 4


def test_alpha_reward():
    for betas, want in GOLD["alpha"]["cases"]:
        a, out = 0.0, []
        for t, b in enumerate(betas, start=1):
            a = S.alpha_update(a, b, t)
            out.append(a)
        np.testing.assert_allclose(out, want, rtol=1e-15)
    for a, b, want in GOLD["reward"]["cases"]:
        assert S.reward(a, b) == pytest.approx(want, abs=1e-15)
    # constant beta: alpha strictly decreasing for t >= 2
    a, prev = 0.0, None
    for t in range(1, 12):
        a = S.alpha_update(a, 10.0, t)
        if t >= 2:
            assert a < prev
        prev = a


def test_gae_example_and_double_sum():
    g = GOLD["gae"]
    A, d = S.gae(g["r"], g["v"], g["gamma"], g["mu"])
    np.testing.assert_allclose(d, g["delta"], atol=1e-12)
    assert A[0] == pytest.approx(g["A0"], abs=1e-12)
    rng = np.random.default_rng(0)
    for _ in range(1000):
        T = int(rng.integers(1, 17))
        r = rng.standard_normal(T).tolist()
        v = rng.standard_normal(T + 1).tolist()
        gm, mu = float(rng.uniform(0.5, 1)), float(rng.uniform(0, 1))
        A, _ = S.gae(r, v, gm, mu)
        np.testing.assert_allclose(A, S.gae_explicit(r, v, gm, mu), rtol=0, atol=1e-10)
    A, d = S.gae([1.0, 2.0], [0.0, 0.0, 0.0], 1.0, 1.0)     # telescoping
    assert A[0] == d[0] + d[1]


def test_decode_action():
    doms = [list(range(8))] * 7
    for a, gi, vi in GOLD["decode"]["cases"]:
        assert S.decode_action(a, doms) == (gi, vi)
    with pytest.raises(IndexError):
        S.decode_action(56, doms)


def test_rng_properties():
    # counter-based: same (seed, stream, ctr) -> same draw; uniform_oc in (0,1]
    assert S.draw(1, 2, 3) == S.draw(1, 2, 3) and S.draw(1, 2, 3) != S.draw(1, 2, 4)
    us = [S.uniform_oc(S.draw(7, 0, i)) for i in range(20000)]
    assert min(us) > 0 and max(us) <= 1 and abs(np.mean(us) - 0.5) < 0.01
    ks = [S.randint(S.draw(7, 1, i), 6) for i in range(60000)]
    cnt = np.bincount(ks, minlength=6)
    assert cnt.min() > 9500 and cnt.max() < 10500
    # multinomial via roulette matches softmax probabilities within 3 sigma
    logits = np.array([0.3, -1.0, 2.0, 0.0])
    p = np.exp(S.log_softmax(logits))
    P = S.cumulative_probabilities(p.tolist())
    n = 100000
    c = np.bincount([S.roulette(P, S.uniform_oc(S.draw(9, 0, i))) for i in range(n)], minlength=4)
    sig = np.sqrt(n * p * (1 - p))
    assert (np.abs(c - n * p) < 3 * sig + 1).all()


# --- PPO gradient check (p15) ------------------------------------------------------------------
def _tiny_params(rng, dims):
    return [(rng.standard_normal((dims[i + 1], dims[i])) * 0.5, rng.standard_normal(dims[i + 1]) * 0.1)
            for i in range(len(dims) - 1)]


@pytest.mark.parametrize("trial", range(10))
def test_ppo_gradient_finite_differences(trial):
    rng = np.random.default_rng(trial)
    A = 3
    dims = [4, 8, 8, 8, 8, A + 1]
    params = _tiny_params(rng, dims)
    B = 6
    obs = rng.standard_normal((B, 4))
    actions = rng.integers(0, A, B)
    old_logp = np.log(rng.uniform(0.2, 0.5, B))
    adv = rng.standard_normal(B)
    v_old = rng.standard_normal(B)
    consts = S.PPOConsts(c1=0.15, c2=0.5, clip=0.2)
    loss, grads = S.ppo_grad(params, obs, actions, old_logp, adv, v_old, consts)
    h = 1e-4
    worst = 0.0
    for l in range(5):
        for which in (0, 1):
            P = params[l][which]
            G = grads[l][which]
            it = np.nditer(P, flags=["multi_index"])
            for _ in it:
                idx = it.multi_index
                old = P[idx]
                P[idx] = old + h
                lp, _ = S.ppo_objective(params, obs, actions, old_logp, adv, v_old, consts)
                P[idx] = old - h
                lm, _ = S.ppo_objective(params, obs, actions, old_logp, adv, v_old, consts)
                P[idx] = old
                fd = -(lp - lm) / (2 * h)
                worst = max(worst, abs(fd - G[idx]) / max(1e-3, abs(fd) + abs(G[idx])))
    assert worst < 1e-4


def test_entropy_uniform_and_degenerate():
    A = 5
    pr = np.exp(S.log_softmax(np.zeros(A)))
    assert -(pr * np.log(pr)).sum() == pytest.approx(math.log(A), abs=1e-12)
    lp = S.log_softmax(np.array([0.0, -1e4, -1e4]))
    assert -(np.exp(lp) * lp).sum() == pytest.approx(0.0, abs=1e-12)


def test_ppo_ratio_one_gives_mean_adv():
    rng = np.random.default_rng(5)
    params = _tiny_params(rng, [4, 8, 8, 8, 8, 4])
    obs = rng.standard_normal((7, 4))
    out, _ = S.mlp_forward(params, obs)
    lp = S.log_softmax(out[:, :3])
    acts = rng.integers(0, 3, 7)
    adv = rng.standard_normal(7)
    L, parts = S.ppo_objective(params, obs, acts, lp[np.arange(7), acts], adv, out[:, 3] - adv,
                               S.PPOConsts(c1=0.0, c2=0.0))
    assert L == pytest.approx(adv.mean(), abs=1e-12)        # L^clip at ratio 1 = mean(A)


# --- GA / random search behaviour (p16) --------------------------------------------------------
T_DOM = [1, 2, 4, 8, 16, 32]
TILE_DOM = [1, 2, 4]
RZ_DOM = [1, 2]
DOMAINS = [T_DOM, T_DOM, T_DOM, TILE_DOM, TILE_DOM, TILE_DOM, RZ_DOM]


def valid(c):
    return c[0] * c[1] * c[2] <= 1024


def surface(seed):
    rng = np.random.default_rng(seed)
    cstar = [d[int(rng.integers(len(d)))] for d in DOMAINS]
    while not valid(cstar):
        cstar = [d[int(rng.integers(len(d)))] for d in DOMAINS]
    wts = rng.uniform(0.05, 1.0, len(DOMAINS))
    base = 10.0

    def f(c):
        return base + sum(wi * (math.log2(ci) - math.log2(si)) ** 2 for wi, ci, si in zip(wts, c, cstar))
    return f, tuple(cstar), base


def test_space_size_and_validity():
    sp = S.enumerate_space(DOMAINS, valid)
    assert 0 < len(sp) <= 10 ** 4
    assert (32, 32, 2, 1, 1, 1, 1) not in sp and (16, 8, 4, 1, 1, 1, 1) in sp
    rng = S.Rng(3, 0)
    for _ in range(2000):
        c = S._sample_valid(DOMAINS, valid, rng, 10000)
        assert valid(c) and all(v in d for v, d in zip(c, DOMAINS))


def test_ga_near_optimum():
    hits = 0
    for seed in range(20):
        f, cstar, base = surface(seed)
        opt = min(f(c) for c in S.enumerate_space(DOMAINS, valid))
        assert opt == base
        res = S.ga_run(DOMAINS, valid, f, seed=seed, budget=2000)
        hits += res.best_beta <= 1.05 * opt
    assert hits >= 18


def test_ga_and_elitism_invariants():
    f, _, _ = surface(1)
    res = S.ga_run(DOMAINS, valid, f, seed=11, budget=600)
    bests = [h["best_beta"] for h in res.history]
    assert all(b2 <= b1 for b1, b2 in zip(bests, bests[1:]))
    assert len(res.measured) <= 600 and len(set(res.measured)) == len(res.measured)
    for h in res.history:
        assert all(valid(tuple(c)) for c in h["pop"])
    # the elites of generation g reappear in generation g+1
    for h0, h1 in zip(res.history, res.history[1:]):
        order = sorted(range(len(h0["pop"])), key=lambda i: (h0["beta"][i], i))
        assert h0["pop"][order[0]] in h1["pop"]
    # determinism: byte-identical history
    assert json.dumps(S.ga_run(DOMAINS, valid, f, seed=11, budget=600).history) == json.dumps(res.history)


def test_ga_degenerate_cases():
    one = [[4], [4], [4], [1], [1], [1], [1]]
    res = S.ga_run(one, valid, lambda c: 3.0, seed=0, budget=10)
    assert res.best == (4, 4, 4, 1, 1, 1, 1) and len(res.history) == 1
    f, _, _ = surface(2)
    res = S.ga_run(DOMAINS, valid, f, seed=0, budget=1000, params=S.GAParams(eps=math.inf))
    assert len(res.history) == 1
    res = S.ga_run(DOMAINS, valid, f, seed=0, budget=1)
    assert len(res.measured) == 1


def test_ga_beats_random():
    wins = 0
    for seed in range(20):
        f, _, _ = surface(100 + seed)
        ga = S.ga_run(DOMAINS, valid, f, seed=seed, budget=512)
        rnd = S.random_run(DOMAINS, valid, f, seed=seed, budget=512)
        wins += ga.best_beta <= rnd.best_beta
    assert wins >= 18


# --- pins added in round 2 for the functions that had only self-consistency checks ----------------
def test_observation_hand_vector():
    """O_conv entry order of PAPER.md:89-93: (N, C_in, C_out, K_h, K_w, H, W, Stride, Padding,
    T_x, T_y, T_z, Tile_x, Tile_y, Tile_z, Tile_rz, alpha_t), with the log2(1+v) feature scaling of
    DESIGN.md reading c24b. Every size entry is 2^j - 1 with a different j, so log2(1+v) = j is
    exact and a swapped pair (C_in/C_out, H/W, K_h/K_w, a gene pair) changes the vector."""
    shape9 = (1, 3, 7, 15, 31, 63, 127, 255, 1)          # padding 1 = SAME
    genes = (0, 1, 3, 7, 15, 31, 63)
    o = S.observation(shape9, genes, 511.0)
    want = [1, 2, 3, 4, 5, 6, 7, 8, 1, 0, 1, 2, 3, 4, 5, 6, 9]   # written out by hand
    assert o.shape == (17,)
    assert o.tolist() == [float(v) for v in want]
    assert S.observation(shape9[:8] + (0,), genes, 0.0)[8] == 0.0 and S.observation(shape9, genes, 0.0)[16] == 0.0


# SELU constants (Klambauer et al. 2017), written out: lambda, alpha and lambda*alpha
SELU_LAMBDA = 1.0507009873554804934
SELU_ALPHA = 1.6732632423543772848
SELU_LAMBDA_ALPHA = 1.7580993408473768599


def test_selu_constants():
    assert float(S.selu(np.array(1.0))) == pytest.approx(SELU_LAMBDA, rel=1e-15)
    assert float(S.selu(np.array(-50.0))) == pytest.approx(-SELU_LAMBDA_ALPHA, rel=1e-15)
    assert float(S.selu(np.array(math.log(0.5)))) == pytest.approx(-SELU_LAMBDA_ALPHA / 2, rel=1e-14)
    assert SELU_LAMBDA * SELU_ALPHA == pytest.approx(SELU_LAMBDA_ALPHA, rel=1e-15)


def test_mlp_forward_hand_network():
    """A 1-unit-per-layer network whose pre-activations are chosen so each activation has a closed
    form: tanh(atanh 0.5) = 0.5, tanh(atanh 0.6) = 0.6, selu(1) = lambda, selu(ln 0.5) = -lambda*alpha/2,
    then the linear head. The order tanh, tanh, selu, selu of PAPER.md:99 is what produces these
    numbers (any other order gives e.g. selu(atanh 0.5) = 0.577 in layer 1)."""
    z1 = 0.54930614433405484570        # atanh(0.5)
    z2 = 0.69314718055994530942        # atanh(0.6) = ln 2
    params = [
        (np.array([[2 * z1]]), np.array([0.0])),                    # obs 0.5 -> z1
        (np.array([[2 * z2]]), np.array([0.0])),                    # h1 0.5  -> z2
        (np.array([[0.0]]), np.array([1.0])),                       # -> z3 = 1
        (np.array([[0.0]]), np.array([math.log(0.5)])),            # -> z4 = ln 0.5
        (np.array([[2.0], [-1.0]]), np.array([0.25, 0.0])),        # linear head, A = 1 logit + value
    ]
    out, cache = S.mlp_forward(params, np.array([[0.5]]))
    h = [float(v[0, 0]) for v in cache["h"][1:]]
    assert h[0] == pytest.approx(0.5, abs=1e-15)
    assert h[1] == pytest.approx(0.6, abs=1e-15)
    assert h[2] == pytest.approx(SELU_LAMBDA, abs=1e-15)
    assert h[3] == pytest.approx(-SELU_LAMBDA_ALPHA / 2, abs=1e-15)
    np.testing.assert_allclose(out[0], [0.25 - SELU_LAMBDA_ALPHA, SELU_LAMBDA_ALPHA / 2], rtol=0, atol=1e-15)
    # inverted dropout after the 4th hidden layer: a dropped unit zeroes the head's input
    out0, _ = S.mlp_forward(params, np.array([[0.5]]), mask=np.array([[0.0]]), keep=0.85)
    np.testing.assert_allclose(out0[0], [0.25, 0.0], atol=0)
    out1, _ = S.mlp_forward(params, np.array([[0.5]]), mask=np.array([[1.0]]), keep=0.5)
    np.testing.assert_allclose(out1[0], [0.25 - 2 * SELU_LAMBDA_ALPHA, SELU_LAMBDA_ALPHA], atol=1e-14)


def _const_head(A, V):
    """A network whose output ignores the input: logits all 0 (uniform policy), value V."""
    dims = [1, 1, 1, 1, 1]
    ps = [(np.zeros((dims[i + 1], dims[i])), np.zeros(dims[i + 1])) for i in range(4)]
    ps.append((np.zeros((A + 1, 1)), np.array([0.0] * A + [V])))
    return ps


def test_ppo_objective_hand_values():
    """L = mean[L^clip - c1 L^VF + c2 S] with the paper's c1 = 0.15, c2 = 20,
    L^VF = (V - (A + V_old))^2 (reading c20), on a uniform 2-action policy (S = ln 2) and value 1.
    Values worked by hand:
      ratio 1 (old logp = ln 1/2): L^clip = adv = (0.5, -0.5); V^target = (0.5, 0.5) -> L^VF = 0.25
        L = 0 - 0.15*0.25 + 20 ln 2 = 13.825443611198906
      ratio 2 (old logp = ln 1/4), clip 0.2: L^clip = (min(1.0, 0.6), min(-1.0, -0.6)) = (0.6, -1.0)
        L = -0.2 - 0.0375 + 20 ln 2 = 13.625443611198906"""
    params = _const_head(2, 1.0)
    obs = np.zeros((2, 1))
    acts = np.array([0, 1])
    adv = np.array([0.5, -0.5])
    v_old = np.array([0.0, 1.0])
    c = S.PPOConsts()
    assert (c.c1, c.c2) == (0.15, 20.0)
    L, parts = S.ppo_objective(params, obs, acts, np.log([0.5, 0.5]), adv, v_old, c)
    np.testing.assert_allclose(parts["ent"], [math.log(2)] * 2, rtol=1e-15)
    np.testing.assert_allclose(parts["lvf"], [0.25, 0.25], rtol=1e-15)
    assert L == pytest.approx(13.825443611198906, abs=1e-12)
    L2, parts2 = S.ppo_objective(params, obs, acts, np.log([0.25, 0.25]), adv, v_old, c)
    np.testing.assert_allclose(parts2["lclip"], [0.6, -1.0], rtol=1e-14)
    assert L2 == pytest.approx(13.625443611198906, abs=1e-12)
    # the value term alone: c2 = 0, V = 3, targets 0.5 -> L = mean(adv) - c1 * 6.25
    L3, _ = S.ppo_objective(_const_head(2, 3.0), obs, acts, np.log([0.5, 0.5]), adv, v_old,
                            S.PPOConsts(c1=0.15, c2=0.0))
    assert L3 == pytest.approx(-0.15 * 6.25, abs=1e-14)


def test_random_run_hand_enumerated_space():
    """Random search: uniform valid samples, best-ever. On a 3-gene space with one
    invalid corner, enumerated by hand: {1,2}^3 minus (2,2,2) = 7 valid configs."""
    doms = [[1, 2], [1, 2], [1, 2]]
    ok = lambda c: c[0] * c[1] * c[2] <= 4
    space = [(1, 1, 1), (1, 1, 2), (1, 2, 1), (1, 2, 2), (2, 1, 1), (2, 1, 2), (2, 2, 1)]
    assert sorted(S.enumerate_space(doms, ok)) == space
    cost = {c: 10.0 + i for i, c in enumerate([(2, 1, 2), (1, 1, 1), (2, 2, 1), (1, 2, 2),
                                                 (1, 1, 2), (2, 1, 1), (1, 2, 1)])}
    f = lambda c: cost[c]
    # budget >= |space|: every valid config measured once, never the invalid one, exact optimum
    for seed in range(5):
        res = S.random_run(doms, ok, f, seed=seed, budget=10)
        assert sorted(res.measured) == space
        assert res.best == (2, 1, 2) and res.best_beta == 10.0
    # budget 3: three distinct valid configs, best = min of those measured
    for seed in range(20):
        res = S.random_run(doms, ok, f, seed=seed, budget=3)
        assert len(res.measured) == 3 == len(set(res.measured))
        assert all(c in space for c in res.measured)
        assert res.best_beta == min(cost[c] for c in res.measured)
    # uniform over the valid configs: the first measured config of 7000 seeds, 3-sigma per cell
    first = [S.random_run(doms, ok, f, seed=s, budget=1).measured[0] for s in range(7000)]
    cnt = [first.count(c) for c in space]
    sig = math.sqrt(7000 * (1 / 7) * (6 / 7))
    assert all(abs(n - 1000) < 3.5 * sig for n in cnt), cnt
