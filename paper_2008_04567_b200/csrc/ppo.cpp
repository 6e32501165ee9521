// RL-search (§2.4, lines 83-121): PPO over one-gene-at-a-time actions.
//
//  * observation O_conv: 9 operator-shape entries, the 7 genes of the current
//    config, and the runtime moving average alpha_t; feature scaling log2(1+v) (DESIGN.md c24b);
//  * policy/value network: FC 512, 1024, 1024, 512 with tanh, tanh, selu, selu,
//    dropout (keep probability rl_keep_prob, DESIGN.md c22) and a linear output of A logits + 1
//    value (shared trunk, DESIGN.md c24);
//  * actions: multinomial over A = sum of the gene-domain sizes; action a sets one gene to one
//    value ("an action updates one parameter at a time");
//  * alpha_t = (alpha_{t-1}*0.8 + beta_t)/t (EMA variant behind rl_alpha_mode, c17);
//  * reward r_t = alpha_{t-1} - min{beta_t, 2 alpha_{t-1}};
//  * GAE by backward recursion (c19); loss L = E[L^clip - c1 L^VF + c2 S]
//    with c1 = 0.15, c2 = 20, minimised as -L with Adam.
// All arithmetic is float64; matrix loops assign each output element to one thread with a fixed
// summation order, so results do not depend on the OpenMP thread count.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "tune.h"

namespace wpk {

static const double SELU_A = 1.6732632423543772848170429916717;
static const double SELU_L = 1.0507009873554804934193349852946;

struct MLP {
    int dims[6];
    std::vector<double> p;     // W1, b1, ..., W5, b5 (W_l is [dims[l+1]][dims[l]])
    size_t off_w[5], off_b[5];
    void setup(const int *d) {
        std::memcpy(dims, d, sizeof dims);
        size_t o = 0;
        for (int l = 0; l < 5; ++l) {
            off_w[l] = o;
            o += (size_t)dims[l + 1] * dims[l];
            off_b[l] = o;
            o += dims[l + 1];
        }
        p.assign(o, 0.0);
    }
    size_t size() const { return p.size(); }
};

// Y[B][O] = X[B][I] W[O][I]^T + b
static void linear_fwd(const double *X, const double *W, const double *b, double *Y, int B, int I, int O) {
#pragma omp parallel for schedule(static) if ((long long)B * O * I > 200000)
    for (long long bo = 0; bo < (long long)B * O; ++bo) {
        const int bb = (int)(bo / O), o = (int)(bo % O);
        const double *x = X + (size_t)bb * I, *w = W + (size_t)o * I;
        double s = 0;
        for (int i = 0; i < I; ++i) s += x[i] * w[i];
        Y[bo] = s + b[o];
    }
}
// dW[O][I] += G^T X ; db[O] += sum_b G ; dX[B][I] = G W
static void linear_bwd(const double *X, const double *W, const double *G, double *dW, double *db, double *dX, int B,
                       int I, int O) {
#pragma omp parallel for schedule(static) if ((long long)B * O * I > 200000)
    for (int o = 0; o < O; ++o) {
        double *dw = dW + (size_t)o * I;
        double sb = 0;
        for (int bb = 0; bb < B; ++bb) {
            const double g = G[(size_t)bb * O + o];
            sb += g;
            const double *x = X + (size_t)bb * I;
            for (int i = 0; i < I; ++i) dw[i] += g * x[i];
        }
        db[o] += sb;
    }
    if (!dX) return;
#pragma omp parallel for schedule(static) if ((long long)B * O * I > 200000)
    for (long long bi = 0; bi < (long long)B * I; ++bi) {
        const int bb = (int)(bi / I), i = (int)(bi % I);
        double s = 0;
        const double *g = G + (size_t)bb * O;
        for (int o = 0; o < O; ++o) s += g[o] * W[(size_t)o * I + i];
        dX[bi] = s;
    }
}

struct Fwd {
    std::vector<double> h[5];    // h[0] = input, h[1..4] = activations
    std::vector<double> z[4];    // pre-activations
    std::vector<double> hd;      // after dropout
    std::vector<double> out;     // [B][A+1]
};

static void mlp_forward(const MLP &m, const double *obs, int B, const double *mask, double keep, Fwd &f) {
    f.h[0].assign(obs, obs + (size_t)B * m.dims[0]);
    for (int l = 0; l < 4; ++l) {
        const int I = m.dims[l], O = m.dims[l + 1];
        f.z[l].resize((size_t)B * O);
        linear_fwd(f.h[l].data(), m.p.data() + m.off_w[l], m.p.data() + m.off_b[l], f.z[l].data(), B, I, O);
        f.h[l + 1].resize((size_t)B * O);
        for (size_t i = 0; i < f.z[l].size(); ++i) {
            const double zz = f.z[l][i];
            f.h[l + 1][i] = (l < 2) ? std::tanh(zz) : SELU_L * (zz > 0 ? zz : SELU_A * (std::exp(zz) - 1.0));
        }
    }
    f.hd = f.h[4];
    if (mask)
        for (size_t i = 0; i < f.hd.size(); ++i) f.hd[i] = f.hd[i] * mask[i] / keep;
    f.out.resize((size_t)B * m.dims[5]);
    linear_fwd(f.hd.data(), m.p.data() + m.off_w[4], m.p.data() + m.off_b[4], f.out.data(), B, m.dims[4], m.dims[5]);
}

// Loss -L and its gradient; consts = {c1, c2, clip}.
static double ppo_loss_grad(const MLP &m, int B, const double *obs, const int32_t *act, const double *old_logp,
                            const double *adv, const double *v_old, const double *consts, const double *mask,
                            double keep, double *grad) {
    const double c1 = consts[0], c2 = consts[1], clip = consts[2];
    Fwd f;
    mlp_forward(m, obs, B, mask, keep, f);
    const int A = m.dims[5] - 1, OUT = m.dims[5];
    std::vector<double> gout((size_t)B * OUT, 0.0);
    double L = 0;
    for (int b = 0; b < B; ++b) {
        const double *lg = &f.out[(size_t)b * OUT];
        double mx = lg[0];
        for (int a = 1; a < A; ++a) mx = std::max(mx, lg[a]);
        double se = 0;
        for (int a = 0; a < A; ++a) se += std::exp(lg[a] - mx);
        const double lse = std::log(se);
        std::vector<double> lp(A), pi(A);
        for (int a = 0; a < A; ++a) { lp[a] = lg[a] - mx - lse; pi[a] = std::exp(lp[a]); }
        double S = 0;
        for (int a = 0; a < A; ++a) S -= pi[a] * lp[a];
        const double ratio = std::exp(lp[act[b]] - old_logp[b]);
        const double cr = std::min(std::max(ratio, 1 - clip), 1 + clip);
        const double unc = ratio * adv[b], clp = cr * adv[b];
        const double lclip = std::min(unc, clp);
        const double V = lg[A], vt = adv[b] + v_old[b];
        const double lvf = (V - vt) * (V - vt);
        L += lclip - c1 * lvf + c2 * S;
        const bool inside = ratio >= 1 - clip && ratio <= 1 + clip;
        const double d_lpa = (unc <= clp) ? ratio * adv[b] : (inside ? ratio * adv[b] : 0.0);
        double *g = &gout[(size_t)b * OUT];
        for (int a = 0; a < A; ++a) {
            double ga = d_lpa * ((a == act[b] ? 1.0 : 0.0) - pi[a]);
            ga += c2 * (-pi[a] * (lp[a] + S));
            g[a] = -ga / B;
        }
        g[A] = -(-c1 * 2.0 * (V - vt)) / B;
    }
    L /= B;
    if (grad) {
        std::fill(grad, grad + m.size(), 0.0);
        std::vector<double> gh((size_t)B * m.dims[4]);
        linear_bwd(f.hd.data(), m.p.data() + m.off_w[4], gout.data(), grad + m.off_w[4], grad + m.off_b[4], gh.data(),
                   B, m.dims[4], OUT);
        if (mask)
            for (size_t i = 0; i < gh.size(); ++i) gh[i] = gh[i] * mask[i] / keep;
        for (int l = 3; l >= 0; --l) {
            const int I = m.dims[l], O = m.dims[l + 1];
            std::vector<double> gz((size_t)B * O);
            for (size_t i = 0; i < gz.size(); ++i) {
                const double zz = f.z[l][i];
                double d;
                if (l < 2) { const double t = std::tanh(zz); d = 1.0 - t * t; }
                else d = SELU_L * (zz > 0 ? 1.0 : SELU_A * std::exp(zz));
                gz[i] = gh[i] * d;
            }
            std::vector<double> gin;
            if (l > 0) gin.resize((size_t)B * I);
            linear_bwd(f.h[l].data(), m.p.data() + m.off_w[l], gz.data(), grad + m.off_w[l], grad + m.off_b[l],
                       l > 0 ? gin.data() : nullptr, B, I, O);
            gh.swap(gin);
        }
    }
    return -L;
}

static void gae(int T, const double *r, const double *v, double gamma, double mu, double *adv) {
    double acc = 0;
    for (int t = T - 1; t >= 0; --t) {
        const double delta = r[t] + gamma * v[t + 1] - v[t];
        acc = delta + gamma * mu * acc;
        adv[t] = acc;
    }
}

static void observation(const ConvDesc &d, const int *genes, double alpha_us, double *o) {
    const double raw[8] = {(double)d.n, (double)d.c, (double)d.k, (double)d.r,
                           (double)d.s, (double)d.h, (double)d.w, (double)d.sh};
    for (int i = 0; i < 8; ++i) o[i] = std::log2(1.0 + raw[i]);
    o[8] = (d.ph > 0 || d.pw > 0) ? 1.0 : 0.0;
    for (int g = 0; g < WPK_NUM_GENES; ++g) o[9 + g] = std::log2(1.0 + genes[g]);
    o[16] = std::log2(1.0 + (std::isfinite(alpha_us) ? alpha_us : 1e9));
}

// ---------------------------------------------------------------------------------------------------
// the RL-search loop
// ---------------------------------------------------------------------------------------------------
struct Adam {
    std::vector<double> m, v;
    long long t = 0;
    void step(std::vector<double> &p, const std::vector<double> &g, double lr) {
        if (m.empty()) { m.assign(p.size(), 0.0); v.assign(p.size(), 0.0); }
        ++t;
        const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
        const double c1 = 1 - std::pow(b1, (double)t), c2 = 1 - std::pow(b2, (double)t);
#pragma omp parallel for schedule(static) if (p.size() > 100000)
        for (long long i = 0; i < (long long)p.size(); ++i) {
            m[i] = b1 * m[i] + (1 - b1) * g[i];
            v[i] = b2 * v[i] + (1 - b2) * g[i] * g[i];
            p[i] -= lr * (m[i] / c1) / (std::sqrt(v[i] / c2) + eps);
        }
    }
};

wpk_status rl_search(TuneCtx &t) {
    const wpk_tune_options &o = t.o;
    const ConvDesc &d = t.plan->d;
    const int E = std::max(1, o.rl_envs), T = std::max(1, o.rl_horizon);
    std::vector<int> dsz;
    int A = 0;
    for (int g = 0; g < WPK_NUM_GENES; ++g) { dsz.push_back((int)t.sp->dom[g].size()); A += dsz.back(); }
    int dims[6] = {17, o.rl_hidden[0], o.rl_hidden[1], o.rl_hidden[2], o.rl_hidden[3], A + 1};
    for (int i = 1; i < 5; ++i)
        if (dims[i] < 1) return fail(WPK_ERR_INVALID_ARGUMENT, "bad rl_hidden");
    MLP net;
    net.setup(dims);
    Rng init(o.seed, 8);
    for (int l = 0; l < 5; ++l) {   // uniform(-sqrt(6/(in+out)), +) (Glorot); output layer scaled down
        const double a = std::sqrt(6.0 / (dims[l] + dims[l + 1])) * (l == 4 ? 0.1 : 1.0);
        for (size_t i = 0; i < (size_t)dims[l + 1] * dims[l]; ++i)
            net.p[net.off_w[l] + i] = (2 * uniform_co(init.next()) - 1) * a;
    }
    Adam adam;
    Rng rng(o.seed, 7);
    // initial configs of the E environments
    std::vector<Config> cur(E);
    Rng r0(o.seed, 0);
    for (int e = 0; e < E; ++e)
        if (!sample_valid(t, r0, &cur[e])) return fail(WPK_ERR_EXHAUSTED, "RL: no valid initial config");
    if (o.seed_default && t.has_default) cur[0] = t.default_cfg;   // env 0 starts from the expert default
    t.measure_batch(cur);
    if (t.err != WPK_OK) return t.err;
    std::vector<double> alpha(E, 0.0);
    std::vector<long long> tstep(E, 0);
    const long long max_steps = 50LL * std::max(t.budget, 1);
    long long steps = 0;
    const double keep = o.rl_keep_prob > 0 ? o.rl_keep_prob : 1.0;
    const double consts[3] = {o.rl_c1, o.rl_c2, o.rl_clip};
    while (!t.exhausted() && steps < max_steps && !t.stop()) {
        // ---- rollout of T steps in each of the E environments ----
        std::vector<double> bobs, blogp, br, bv;
        std::vector<int32_t> bact;
        bobs.reserve((size_t)E * T * 17);
        for (int st = 0; st < T; ++st) {
            std::vector<double> obs((size_t)E * 17);
            for (int e = 0; e < E; ++e) observation(d, cur[e].genes, alpha[e], &obs[(size_t)e * 17]);
            Fwd f;
            mlp_forward(net, obs.data(), E, nullptr, 1.0, f);
            std::vector<Config> prop(E);
            std::vector<int> acts(E);
            std::vector<double> lps(E), vals(E);
            for (int e = 0; e < E; ++e) {
                const double *lg = &f.out[(size_t)e * (A + 1)];
                double mx = lg[0];
                for (int a = 1; a < A; ++a) mx = std::max(mx, lg[a]);
                double se = 0;
                for (int a = 0; a < A; ++a) se += std::exp(lg[a] - mx);
                const double v = uniform_oc(rng.next());   // multinomial by inverse sampling
                double acc = 0, prev = 0;
                int a_sel = A - 1;
                for (int a = 0; a < A; ++a) {
                    acc += std::exp(lg[a] - mx) / se;
                    if (prev < v && v <= acc) { a_sel = a; break; }
                    prev = acc;
                }
                acts[e] = a_sel;
                lps[e] = lg[a_sel] - mx - std::log(se);
                vals[e] = lg[A];
                int g = 0, rem = a_sel;
                while (rem >= dsz[g]) { rem -= dsz[g]; ++g; }   // decode
                Config c = cur[e];
                c.genes[g] = t.sp->dom[g][rem];
                prop[e] = t.valid(c) ? c : cur[e];             // invalid -> config unchanged
            }
            t.measure_batch(prop);
            if (t.err != WPK_OK) return t.err;
            for (int e = 0; e < E; ++e) {
                auto it = t.memo.find(prop[e]);
                if (it == t.memo.end()) continue;               // budget ran out mid-step
                double beta = it->second;
                const double a_prev = alpha[e];
                if (!std::isfinite(beta)) beta = a_prev > 0 ? 2 * a_prev : (t.best_beta < 1e299 ? 2 * t.best_beta : 1e6);
                const double r = a_prev - std::min(beta, 2 * a_prev);
                tstep[e] += 1;
                alpha[e] = (o.rl_alpha_mode == 0) ? (a_prev * 0.8 + beta) / (double)tstep[e]
                                                  : (tstep[e] == 1 ? beta : 0.8 * a_prev + 0.2 * beta);
                bobs.insert(bobs.end(), &obs[(size_t)e * 17], &obs[(size_t)e * 17 + 17]);
                bact.push_back(acts[e]);
                blogp.push_back(lps[e]);
                br.push_back(r);
                bv.push_back(vals[e]);
                cur[e] = prop[e];
            }
            ++steps;
            if (t.exhausted()) break;
        }
        t.rounds++;
        const int B = (int)br.size();
        if (B == 0) break;
        // ---- GAE per environment (transitions are interleaved e-major per step) ----
        std::vector<double> bootstrap(E);
        {
            std::vector<double> obs((size_t)E * 17);
            for (int e = 0; e < E; ++e) observation(d, cur[e].genes, alpha[e], &obs[(size_t)e * 17]);
            Fwd f;
            mlp_forward(net, obs.data(), E, nullptr, 1.0, f);
            for (int e = 0; e < E; ++e) bootstrap[e] = f.out[(size_t)e * (A + 1) + A];
        }
        std::vector<double> adv(B);
        if (B % E == 0) {
            const int Tn = B / E;
            std::vector<double> rr(Tn), vv(Tn + 1), aa(Tn);
            for (int e = 0; e < E; ++e) {
                for (int s2 = 0; s2 < Tn; ++s2) { rr[s2] = br[(size_t)s2 * E + e]; vv[s2] = bv[(size_t)s2 * E + e]; }
                vv[Tn] = bootstrap[e];
                gae(Tn, rr.data(), vv.data(), o.rl_gamma, o.rl_mu, aa.data());
                for (int s2 = 0; s2 < Tn; ++s2) adv[(size_t)s2 * E + e] = aa[s2];
            }
        } else {
            std::vector<double> vv(bv);
            vv.push_back(0.0);
            gae(B, br.data(), vv.data(), o.rl_gamma, o.rl_mu, adv.data());
        }
        std::vector<double> vbase(bv);   // value-target base: V_target = A_raw + V_old (reading c20)
        if (o.rl_adv_norm) {   // advantage normalisation (PPO reference implementations; DESIGN.md c24)
            const std::vector<double> raw(adv);
            double mu = 0, var = 0;
            for (double v : adv) mu += v;
            mu /= B;
            for (double v : adv) var += (v - mu) * (v - mu);
            const double sd = std::sqrt(var / B) + 1e-8;
            for (double &v : adv) v = (v - mu) / sd;
            for (int j = 0; j < B; ++j) vbase[j] = bv[j] + raw[j] - adv[j];   // keeps V_target unnormalised
        }
        // every rl_restart_every updates, environments restart from the best-ever config
        if (o.rl_restart_every > 0 && t.have_best && t.rounds % o.rl_restart_every == 0)
            for (int e = 0; e < E; ++e) cur[e] = t.best;
        // ---- PPO epochs over shuffled minibatches (dropout active in the update forward) ----
        const int mb = std::max(1, std::min(o.rl_minibatch, B));
        std::vector<int> idx(B);
        std::vector<double> grad(net.size());
        double last_loss = 0;
        for (int ep = 0; ep < std::max(1, o.rl_epochs); ++ep) {
            std::iota(idx.begin(), idx.end(), 0);
            for (int i = B - 1; i > 0; --i) std::swap(idx[i], idx[randint(rng.next(), (uint64_t)i + 1)]);
            for (int s0 = 0; s0 < B; s0 += mb) {
                const int n = std::min(mb, B - s0);
                std::vector<double> ob((size_t)n * 17), lp(n), ad(n), vo(n), mask((size_t)n * dims[4]);
                std::vector<int32_t> ac(n);
                for (int i = 0; i < n; ++i) {
                    const int j = idx[s0 + i];
                    std::copy(&bobs[(size_t)j * 17], &bobs[(size_t)j * 17 + 17], &ob[(size_t)i * 17]);
                    lp[i] = blogp[j]; ad[i] = adv[j]; vo[i] = vbase[j]; ac[i] = bact[j];
                }
                for (auto &mv : mask) mv = (uniform_co(rng.next()) < keep) ? 1.0 : 0.0;
                last_loss = ppo_loss_grad(net, n, ob.data(), ac.data(), lp.data(), ad.data(), vo.data(), consts,
                                          keep < 1.0 ? mask.data() : nullptr, keep, grad.data());
                if (o.rl_lr > 0) adam.step(net.p, grad, o.rl_lr);
            }
        }
        double rsum = 0;
        for (double v : br) rsum += v;
        char buf[512];
        snprintf(buf, sizeof buf,
                 "{\"update\": %d, \"steps\": %lld, \"measured\": %zu, \"best_beta\": %.17g, \"mean_reward\": %.9g, "
                 "\"alpha0\": %.9g, \"loss\": %.9g}",
                 t.rounds, steps, t.order.size(), t.best_beta, rsum / B, alpha[0], last_loss);
        log_line(t, buf);
    }
    return WPK_OK;
}

}  // namespace wpk

using namespace wpk;

extern "C" {

wpk_status wpk_ppo_loss_grad(const int32_t *dims, const double *params, int32_t batch, const double *obs,
                             const int32_t *actions, const double *old_logp, const double *adv, const double *v_old,
                             const double *consts, const double *mask, double keep, double *loss, double *grad) {
    if (!dims || !params || !obs || !actions || !old_logp || !adv || !v_old || !consts || !loss || batch < 1)
        return fail(WPK_ERR_INVALID_ARGUMENT, "NULL argument");
    MLP m;
    m.setup(dims);
    std::copy(params, params + m.size(), m.p.begin());
    *loss = ppo_loss_grad(m, batch, obs, actions, old_logp, adv, v_old, consts, mask, keep, grad);
    return WPK_OK;
}

wpk_status wpk_gae(int32_t T, const double *r, const double *v, double gamma, double mu, double *adv) {
    if (T < 1 || !r || !v || !adv) return fail(WPK_ERR_INVALID_ARGUMENT, "bad argument");
    gae(T, r, v, gamma, mu, adv);
    return WPK_OK;
}

wpk_status wpk_observation(const wpk_conv2d_shape *shape, const int32_t *genes, double alpha_us, double *obs17) {
    if (!shape || !genes || !obs17) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL argument");
    ConvDesc d{};
    d.n = shape->n; d.c = shape->c; d.k = shape->k; d.r = shape->r; d.s = shape->s; d.h = shape->h; d.w = shape->w;
    d.sh = shape->stride_h; d.ph = shape->pad_h; d.pw = shape->pad_w;
    observation(d, genes, alpha_us, obs17);
    return WPK_OK;
}

}  // extern "C"
