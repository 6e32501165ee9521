"""oracle/search.py -- TEST INFRASTRUCTURE ONLY.

The paper's search arithmetic, written out step by step in the paper's order and notation, in
float64 numpy / pure Python. Used to pin the C++ tuner (paper_2008_04567_b200/csrc/tune_*.cpp).

GA: PAPER.md:60-82 (§2.3).  RL-search: PAPER.md:83-121 (§2.4).  Readings of silent/garbled
points follow SURVEY.md §8(c) c13-c24 and are listed in DESIGN.md "Readings".

Random numbers: a counter-based generator (SplitMix64 finaliser over (seed, stream, counter)),
implemented independently here and in the product (task rule ③ "each side implements the same
counter-based generator"):
    mix64(z)        = SplitMix64 finaliser of z + golden-gamma
    draw(s, st, c)  = mix64(mix64(s ^ (st * 0xD1B54A32D192ED03)) ^ c)
    uniform_oc(u)   = ((u >> 11) + 1) * 2^-53          in (0, 1]
    uniform_co(u)   = (u >> 11) * 2^-53                 in [0, 1)
    randint(u, n)   = ((u >> 11) * n) >> 53             in [0, n)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1


def mix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def draw(seed: int, stream: int, ctr: int) -> int:
    return mix64(mix64((seed ^ ((stream * 0xD1B54A32D192ED03) & M64)) & M64) ^ (ctr & M64))


def uniform_oc(u: int) -> float:
    return ((u >> 11) + 1) * 2.0 ** -53


def uniform_co(u: int) -> float:
    return (u >> 11) * 2.0 ** -53


def randint(u: int, n: int) -> int:
    return ((u >> 11) * n) >> 53


class Rng:
    """One (seed, stream) counter stream."""

    def __init__(self, seed: int, stream: int):
        self.seed, self.stream, self.ctr = seed, stream, 0

    def next(self) -> int:
        u = draw(self.seed, self.stream, self.ctr)
        self.ctr += 1
        return u


# ----------------------------------------------------------------------------------------------
# GA formulas
# ----------------------------------------------------------------------------------------------
def fitness(beta: float) -> float:
    """f(a_i) = 1/beta (reading c13: "the function of runtime"); failed -> 0."""
    return 0.0 if not math.isfinite(beta) else 1.0 / beta


def selection_probabilities(f):
    """Eq. (1): p(a_i) = f(a_i) / sum_i f(a_i)."""
    tot = sum(f)
    return [fi / tot for fi in f]


def cumulative_probabilities(p):
    """Eq. (2): P(a_i) = sum_{j<=i} p(a_j)."""
    out, acc = [], 0.0
    for pi in p:
        acc += pi
        out.append(acc)
    return out


def roulette(P, v: float) -> int:
    """the i-th individual is selected if P(a_{i-1}) < v <= P(a_i), P(a_0)=0.
    Returns the 0-based index; v above the last (rounded) P selects the last individual."""
    prev = 0.0
    for i, Pi in enumerate(P):
        if prev < v <= Pi:
            return i
        prev = Pi
    return len(P) - 1


# ----------------------------------------------------------------------------------------------
# GA run (Step1..Step4)
# ----------------------------------------------------------------------------------------------
@dataclass
class GAParams:
    pop: int = 48            # |a| = |a'|   (reading c15)
    elites: int = 4          # k
    pool: int = 0            # m; 0 -> m = |a| (reading c14)
    mutation: float = 0.1    # per-gene resample probability (c15)
    eps: float = 0.02        # convergence: (max beta - min beta)/min beta < eps (c15)
    max_gen: int = 50        # G
    max_reject: int = 10000  # Step1 rejection bound
    child_retries: int = 100


@dataclass
class SearchResult:
    best: tuple | None
    best_beta: float
    history: list = field(default_factory=list)   # one dict per generation / evaluation batch
    measured: list = field(default_factory=list)  # configs in measurement order


def _sample_valid(domains, valid, rng: Rng, max_reject: int):
    """Step1 sampler: each gene uniform over its domain; reject until valid."""
    for _ in range(max_reject):
        cfg = tuple(d[randint(rng.next(), len(d))] for d in domains)
        if valid(cfg):
            return cfg
    raise RuntimeError("ExhaustedSampling")


class _Memo:
    """Reading c16: config -> beta memoised within one tune; budget counts distinct configs."""

    def __init__(self, evaluate, budget: int):
        self.evaluate, self.budget, self.table, self.order = evaluate, budget, {}, []

    def measure_batch(self, cfgs):
        """Measure the new distinct configs of `cfgs` in first-occurrence order, up to budget.
        Returns the list of configs actually measured in this batch."""
        new = []
        for c in cfgs:
            if c not in self.table and c not in new:
                new.append(c)
        room = self.budget - len(self.order)
        new = new[:max(room, 0)]
        for c in new:
            self.table[c] = float(self.evaluate(c))
            self.order.append(c)
        return new

    @property
    def exhausted(self):
        return len(self.order) >= self.budget


def ga_run(domains, valid, evaluate, seed: int, budget: int, params: GAParams | None = None):
    """The GA of PAPER.md §2.3. Stream g (generation number) drives generation g's draws."""
    prm = params or GAParams()
    memo = _Memo(evaluate, budget)
    res = SearchResult(None, math.inf)
    m_pool = prm.pool if prm.pool > 0 else prm.pop

    # Step1: random valid population
    rng = Rng(seed, 0)
    pop = [_sample_valid(domains, valid, rng, prm.max_reject) for _ in range(prm.pop)]
    gen = 0
    while True:
        # Step2: fitness by measured runtime (memoised)
        memo.measure_batch(pop)
        pop = [c for c in pop if c in memo.table]        # drop unmeasured (budget ran out)
        betas = [memo.table[c] for c in pop]
        for c in memo.order[len(res.measured):]:
            res.measured.append(c)
            b = memo.table[c]
            if b < res.best_beta:                        # best-ever; ties keep the first
                res.best, res.best_beta = c, b
        fin = [b for b in betas if math.isfinite(b)]
        spread = ((max(fin) - min(fin)) / min(fin)) if fin else math.inf
        res.history.append({"gen": gen, "pop": [list(c) for c in pop], "beta": betas,
                            "best_beta": res.best_beta,
                            "mean_beta": (sum(fin) / len(fin)) if fin else math.inf,
                            "spread": spread, "measured": len(memo.order)})
        # Step4: stop when the runtimes are close enough, or on budget / G
        if spread < prm.eps or memo.exhausted or gen + 1 >= prm.max_gen or not pop:
            break
        if not fin:
            break
        # Step3
        rng = Rng(seed, gen + 1)
        f = [fitness(b) for b in betas]
        p = selection_probabilities(f)                               # Eq. (1)
        order = sorted(range(len(pop)), key=lambda i: (-p[i], i))   # decreasing p, stable
        k = min(prm.elites, len(pop))
        nxt = [pop[i] for i in order[:k]]                            # elites, unchanged
        poolidx = order[:min(m_pool, len(pop))]
        psum = sum(p[i] for i in poolidx)
        P = cumulative_probabilities([p[i] / psum for i in poolidx])  # Eq. (2), renormalised
        while len(nxt) < prm.pop:
            child = None
            for _ in range(prm.child_retries):
                a = pop[poolidx[roulette(P, uniform_oc(rng.next()))]]
                b = pop[poolidx[roulette(P, uniform_oc(rng.next()))]]
                genes = []
                for gi in range(len(domains)):                       # uniform crossover
                    genes.append(a[gi] if (rng.next() >> 63) == 0 else b[gi])
                for gi, d in enumerate(domains):                     # per-gene mutation
                    if uniform_co(rng.next()) < prm.mutation:
                        genes[gi] = d[randint(rng.next(), len(d))]
                cand = tuple(genes)
                if valid(cand):
                    child = cand
                    break
            if child is None:
                child = _sample_valid(domains, valid, rng, prm.max_reject)
            nxt.append(child)
        pop = nxt
        gen += 1
    return res


def random_run(domains, valid, evaluate, seed: int, budget: int, batch: int = 48,
               max_draw_factor: int = 100):
    """Random search baseline: uniform valid samples, best-ever. Samples are drawn
    in batches of `batch` new distinct configs (so that a batch can be measured in parallel,
    SURVEY.md §8(e)); duplicates cost no budget (reading c16)."""
    memo = _Memo(evaluate, budget)
    res = SearchResult(None, math.inf)
    rng = Rng(seed, 0)
    draws, limit = 0, max_draw_factor * max(budget, 1)
    rounds = 0
    while not memo.exhausted and draws < limit:
        room = budget - len(memo.order)
        b = []
        while len(b) < min(batch, room) and draws < limit:
            c = _sample_valid(domains, valid, rng, 10000)
            draws += 1
            if c not in memo.table and c not in b:
                b.append(c)
        for c in memo.measure_batch(b):
            res.measured.append(c)
            if memo.table[c] < res.best_beta:
                res.best, res.best_beta = c, memo.table[c]
        rounds += 1
        res.history.append({"round": rounds, "measured": len(memo.order), "best_beta": res.best_beta})
    return res


def enumerate_space(domains, valid):
    """Whole-space enumeration (the brute-force oracle for regret checks)."""
    out = [()]
    for d in domains:
        out = [c + (v,) for c in out for v in d]
    return [c for c in out if valid(c)]


# ----------------------------------------------------------------------------------------------
# RL-search formulas
# ----------------------------------------------------------------------------------------------
def alpha_update(alpha_prev: float, beta: float, t: int) -> float:
    """alpha_t = (alpha_{t-1} * 0.8 + beta_t) / t, alpha_0 = 0 (reading c17)."""
    return (alpha_prev * 0.8 + beta) / t


def reward(alpha_prev: float, beta: float) -> float:
    """r_t = alpha_{t-1} - min{beta_t, 2 alpha_{t-1}}."""
    return alpha_prev - min(beta, 2.0 * alpha_prev)


def gae(r, v, gamma: float, mu: float):
    """PAPER.md:109-113 by backward recursion A_t = delta_t + (gamma mu) A_{t+1} (reading c19);
    v has len(r)+1 entries (bootstrap value last)."""
    T = len(r)
    delta = [r[t] + gamma * v[t + 1] - v[t] for t in range(T)]
    A = [0.0] * T
    acc = 0.0
    for t in range(T - 1, -1, -1):
        acc = delta[t] + gamma * mu * acc
        A[t] = acc
    return A, delta


def gae_explicit(r, v, gamma: float, mu: float):
    """The explicit sum A_t = sum_{l=0}^{T-t-1} (gamma mu)^l delta_{t+l}."""
    T = len(r)
    delta = [r[t] + gamma * v[t + 1] - v[t] for t in range(T)]
    return [sum((gamma * mu) ** l * delta[t + l] for l in range(T - t)) for t in range(T)]


def decode_action(a: int, domains):
    """an action updates one parameter; flattened (gene, value-index) decode."""
    for gi, d in enumerate(domains):
        if a < len(d):
            return gi, a
        a -= len(d)
    raise IndexError("action out of range")


def observation(shape9, genes, alpha_us: float):
    """O_conv: (N, C_in, C_out, K_h, K_w, H, W, Stride, Padding, 7 genes, alpha).
    Feature scaling (reading): log2(1+v) for every size / gene, padding as 0/1,
    log2(1+alpha in microseconds)."""
    n, cin, cout, kh, kw, h, w, stride, padding = shape9
    raw = [n, cin, cout, kh, kw, h, w, stride]
    o = [math.log2(1.0 + v) for v in raw] + [1.0 if padding else 0.0]
    o += [math.log2(1.0 + g) for g in genes]
    o.append(math.log2(1.0 + alpha_us))
    return np.array(o, dtype=np.float64)


# --- policy/value network ------------------------------------------------------
SELU_A = 1.6732632423543772848170429916717
SELU_L = 1.0507009873554804934193349852946


def selu(z):
    return SELU_L * np.where(z > 0, z, SELU_A * (np.exp(z) - 1.0))


def dselu(z):
    return SELU_L * np.where(z > 0, 1.0, SELU_A * np.exp(z))


ACTS = ("tanh", "tanh", "selu", "selu")   # PAPER.md:99 ("tahn, tahn, selu and selu"; c22)


def mlp_forward(params, obs, mask=None, keep: float = 1.0):
    """params = [(W1,b1),...,(W5,b5)], W_l of shape [out,in]. obs [B,17].
    Hidden layers tanh,tanh,selu,selu; dropout (inverted, `mask`/keep) after the 4th hidden layer;
    linear output of width A+1 (A logits, then the value). Returns (out, cache)."""
    h = obs
    cache = {"h": [obs], "z": []}
    for l in range(4):
        W, b = params[l]
        z = h @ W.T + b
        h = np.tanh(z) if ACTS[l] == "tanh" else selu(z)
        cache["z"].append(z)
        cache["h"].append(h)
    if mask is not None:
        h = h * mask / keep
    cache["hd"] = h
    W, b = params[4]
    out = h @ W.T + b
    return out, cache


def log_softmax(logits):
    m = logits.max(axis=-1, keepdims=True)
    z = logits - m
    return z - np.log(np.exp(z).sum(axis=-1, keepdims=True))


@dataclass
class PPOConsts:
    c1: float = 0.15
    c2: float = 20.0
    clip: float = 0.2    # reading c24


def ppo_objective(params, obs, actions, old_logp, adv, v_old, consts: PPOConsts,
                  mask=None, keep: float = 1.0):
    """L = mean_t[ L^clip - c1 L^VF + c2 S ], L^VF = (V - (A + V_old))^2 (c20).
    Returns (L, parts)."""
    out, cache = mlp_forward(params, obs, mask, keep)
    A = out.shape[1] - 1
    logits, V = out[:, :A], out[:, A]
    lp = log_softmax(logits)
    pi = np.exp(lp)
    lpa = lp[np.arange(len(actions)), actions]
    ratio = np.exp(lpa - old_logp)
    lclip = np.minimum(ratio * adv, np.clip(ratio, 1 - consts.clip, 1 + consts.clip) * adv)
    vt = adv + v_old
    lvf = (V - vt) ** 2
    ent = -(pi * lp).sum(axis=1)
    L = np.mean(lclip - consts.c1 * lvf + consts.c2 * ent)
    return L, {"out": out, "cache": cache, "lp": lp, "pi": pi, "ratio": ratio, "adv": adv,
               "vt": vt, "ent": ent, "lclip": lclip, "lvf": lvf}


def ppo_grad(params, obs, actions, old_logp, adv, v_old, consts: PPOConsts,
             mask=None, keep: float = 1.0):
    """Gradient of the LOSS  -L  (the quantity minimised) w.r.t. every parameter, by manual
    backpropagation through the network of mlp_forward. Returns (loss, grads like params)."""
    L, pr = ppo_objective(params, obs, actions, old_logp, adv, v_old, consts, mask, keep)
    B = obs.shape[0]
    out, lp, pi, ratio = pr["out"], pr["lp"], pr["pi"], pr["ratio"]
    A = out.shape[1] - 1
    V = out[:, A]
    # dL/dlogits and dL/dV  (L is the mean objective); loss = -L
    g_out = np.zeros_like(out)
    # clip term: derivative of min(r*adv, clip(r)*adv) w.r.t. log pi(a)
    unclipped = ratio * adv
    clipped = np.clip(ratio, 1 - consts.clip, 1 + consts.clip) * adv
    use_unclipped = unclipped <= clipped
    inside = (ratio >= 1 - consts.clip) & (ratio <= 1 + consts.clip)
    d_lpa = np.where(use_unclipped, ratio * adv, np.where(inside, ratio * adv, 0.0))
    # when both are equal (ratio inside the clip range) the min is r*adv either way
    onehot = np.zeros((B, A))
    onehot[np.arange(B), actions] = 1.0
    g_logits = d_lpa[:, None] * (onehot - pi)
    # entropy: S = -sum pi lp ; dS/dz_j = -pi_j (lp_j + S)
    S = pr["ent"]
    g_logits += consts.c2 * (-pi * (lp + S[:, None]))
    g_out[:, :A] = g_logits
    g_out[:, A] = -consts.c1 * 2.0 * (V - pr["vt"])
    g_out /= B
    g_out = -g_out                                    # loss = -L
    cache = pr["cache"]
    grads = [None] * 5
    W5, _ = params[4]
    hd = cache["hd"]
    grads[4] = (g_out.T @ hd, g_out.sum(axis=0))
    gh = g_out @ W5
    if mask is not None:
        gh = gh * mask / keep
    for l in range(3, -1, -1):
        z = cache["z"][l]
        gz = gh * ((1.0 - np.tanh(z) ** 2) if ACTS[l] == "tanh" else dselu(z))
        hin = cache["h"][l]
        W, _ = params[l]
        grads[l] = (gz.T @ hin, gz.sum(axis=0))
        gh = gz @ W
    return -L, grads
