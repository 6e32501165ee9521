// wpk_conv2d_tune: the per-operator automated search (§2.3 genetic search, §2.4
// RL-search, plus the random-search baseline of PAPER.md:161) over the plan's kernel-family gene
// space, with fitness from CUDA-event kernel time.
//
// Candidate evaluation ("compile ... then execute them to get the runtime") is pure
// measurement here: tiles are runtime parameters, so nothing is compiled per candidate. The new
// distinct candidates of a generation are sharded over ranks (index j -> rank j mod world) and
// their fitness records are all-gathered through the wpk_exchange_fn callback (NCCL via torch in
// practice); every rank then runs the identical deterministic searcher update.
#include <cuda_runtime.h>
#include <unistd.h>

#include <cctype>
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "tune.h"
#include "jit.h"

namespace wpk {

void fill_random_device(void *p, size_t n, int dtype, uint64_t seed, void *stream);   // run.cu
void timestamp_device(unsigned long long *dst, void *stream);                          // run.cu
void l2_flush_device(const void *buf, size_t bytes, void *sink, void *stream);          // run.cu

double wall_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool TuneCtx::time_up() const { return o.max_seconds > 0 && wall_seconds() - t_start > o.max_seconds; }

std::string genes_json(const Config &c) {
    std::string s = "[";
    for (int g = 0; g < WPK_NUM_GENES; ++g) s += (g ? "," : "") + std::to_string(c.genes[g]);
    return s + "]";
}

static std::string dbl(double v) {
    if (!std::isfinite(v)) return "Infinity";
    char b[64];
    snprintf(b, sizeof b, "%.17g", v);
    return b;
}

void log_line(TuneCtx &t, const std::string &s) {
    if (t.log && t.o.rank == 0) {
        fputs(s.c_str(), t.log);
        fputc('\n', t.log);
        fflush(t.log);
    }
}

// ---------------------------------------------------------------------------------------------------
// measured evaluator (W warm-ups + R device-timestamped reps, interquartile mean; L2 flushed before each rep)
// ---------------------------------------------------------------------------------------------------
struct GpuBench {
    cudaStream_t st = nullptr;
    void *x = nullptr, *w = nullptr, *b = nullptr, *y = nullptr, *z = nullptr, *ws = nullptr, *flush = nullptr;
    void *wdw = nullptr, *bdw = nullptr;   // fused depthwise+pointwise plans: the depthwise weights / bias
    // rotating mode (l2_flush == 2): P copies of x and y, one timed rep = one CUDA graph of P
    // back-to-back convs over all copies, so every launch reads an input last touched P launches ago
    // (P x footprint >= 2 x L2: cold) and one stamp pair spans P launches (the device timestamps
    // advance in ~2-us steps here, as coarse as a small layer)
    std::vector<void *> xr, yr;
    unsigned long long *stamps = nullptr;   // [2 * reps] device timestamps
    size_t ws_bytes = 0, flush_bytes = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    bool ok = false;
    std::string err;

    bool init(Plan &p) {
        const ConvDesc &d = p.d;
        if (cudaSetDevice(p.device) != cudaSuccess) return fail_("cudaSetDevice");
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return fail_("stream");
        const size_t e = d.in_elem(), eo = d.elem();   // x / w and y / b / z element bytes
        size_t xb = (size_t)d.n * d.c * d.h * d.w * e, wb = (size_t)d.k * (d.c / d.g) * d.r * d.s * e;
        size_t yb = (size_t)d.M() * d.k * eo;
        if (cudaMalloc(&x, xb) || cudaMalloc(&w, wb) || cudaMalloc(&b, d.k * eo + 16) || cudaMalloc(&y, yb))
            return fail_("cudaMalloc of tuning buffers");
        fill_random_device(x, xb / e, d.dtype, 1, st);
        fill_random_device(w, wb / e, d.dtype, 2, st);
        fill_random_device(b, d.k, d.out_dtype(), 3, st);
        if (d.fused_dw) {   // w / b above are the pointwise [K][C] (C = d.c) and [K]; add the depthwise ones
            const size_t wdb = (size_t)d.c * d.r * d.s * e;
            if (cudaMalloc(&wdw, wdb) || cudaMalloc(&bdw, d.c * e + 16))
                return fail_("cudaMalloc of the depthwise buffers");
            fill_random_device(wdw, wdb / e, d.dtype, 5, st);
            fill_random_device(bdw, d.c, d.dtype, 6, st);
        }
        if (d.epilogue == WPK_EPI_BIAS_ADD_RELU) {   // a residual plan reads z of y's shape
            if (cudaMalloc(&z, yb)) return fail_("cudaMalloc of the residual buffer");
            fill_random_device(z, yb / eo, d.out_dtype(), 4, st);
        }
        flush_bytes = (size_t)2 * device_l2_bytes(p.device);
        if (cudaMalloc(&flush, flush_bytes + 256)) return fail_("cudaMalloc of the L2 flush buffer");
        cudaMemsetAsync(flush, 1, flush_bytes + 256, st);
        if (cudaEventCreate(&e0) || cudaEventCreate(&e1)) return fail_("events");
        if (cudaMalloc(&stamps, 2 * 1024 * sizeof(unsigned long long))) return fail_("cudaMalloc of timestamps");
        if (cudaStreamSynchronize(st)) return fail_("init sync");
        ok = true;
        return true;
    }
    bool fail_(const char *m) {
        cudaError_t e = cudaGetLastError();
        err = std::string(m) + ": " + cudaGetErrorString(e);
        return false;
    }
    bool init_rotation(Plan &p) {   // lazily, on the first rotating measurement
        if (!xr.empty()) return true;
        const ConvDesc &d = p.d;
        const size_t xb = (size_t)d.n * d.c * d.h * d.w * d.in_elem(), yb = (size_t)d.M() * d.k * d.elem();
        const size_t foot = xb + yb;
        size_t P = (2 * (size_t)device_l2_bytes(p.device) + foot - 1) / foot;
        P = std::max<size_t>(2, std::min<size_t>(P, 64));
        while (P > 2 && P * foot > ((size_t)3 << 30)) --P;   // <= 3 GB of copies
        for (size_t i = 0; i < P; ++i) {
            void *xx = nullptr, *yy = nullptr;
            if (cudaMalloc(&xx, xb) || cudaMalloc(&yy, yb)) {
                if (xx) cudaFree(xx);
                cudaGetLastError();
                break;
            }
            cudaMemcpyAsync(xx, x, xb, cudaMemcpyDeviceToDevice, st);
            xr.push_back(xx);
            yr.push_back(yy);
        }
        if (xr.size() < 2) return fail_("cudaMalloc of the rotating buffers");
        return cudaStreamSynchronize(st) == cudaSuccess;
    }
    ~GpuBench() {
        for (void *ptr : xr) cudaFree(ptr);
        for (void *ptr : yr) cudaFree(ptr);
        for (void *ptr : {x, w, b, y, z, ws, flush, wdw, bdw, (void *)stamps})
            if (ptr) cudaFree(ptr);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (st) cudaStreamDestroy(st);
    }
    // Wait for the stream with a host watchdog (a hung kernel aborts the tune, not the box).
    bool sync_with_deadline(double seconds) {
        double t0 = wall_seconds();
        while (true) {
            cudaError_t q = cudaStreamQuery(st);
            if (q == cudaSuccess) return true;
            if (q != cudaErrorNotReady) { err = cudaGetErrorString(q); return false; }
            if (wall_seconds() - t0 > seconds) { err = "candidate exceeded the watchdog deadline"; return false; }
        }
    }
    // Rotating mode: microseconds per conv of a graph of P back-to-back convs on P cold buffer copies
    // (interquartile mean over reps), the graph's kernels overlapping through PDL as in a network step.
    double measure_rotating(Plan &p, const Config &cfg, int warmup, int reps, bool *fatal) {
        if (!init_rotation(p)) { *fatal = true; return INFINITY; }
        const size_t P = xr.size();
        for (int i = 0; i < std::max(1, warmup); ++i)   // eager: weight packing, workspace state, first-use maps
            if (launch_conv(p, cfg, xr[i % P], w, b, yr[i % P], st, (char *)ws, ws_bytes, z, wdw, bdw) < 0) return INFINITY;
        if (!sync_with_deadline(10.0)) { *fatal = true; return INFINITY; }
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { *fatal = true; return INFINITY; }
        bool ok = true;
        for (size_t i = 0; i < P && ok; ++i)
            ok = launch_conv(p, cfg, xr[i], w, b, yr[i], st, (char *)ws, ws_bytes, z, wdw, bdw) >= 0;
        if (cudaStreamEndCapture(st, &g) != cudaSuccess || !ok || !g) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return INFINITY;
        }
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
            cudaGraphDestroy(g);
            cudaGetLastError();
            return INFINITY;
        }
        cudaGraphDestroy(g);
        std::vector<unsigned long long> hs(2 * (size_t)reps);
        cudaGraphLaunch(ge, st);   // one untimed pass of the graph
        for (int i = 0; i < reps; ++i) {
            timestamp_device(stamps + 2 * i, st);
            cudaGraphLaunch(ge, st);
            timestamp_device(stamps + 2 * i + 1, st);
        }
        const bool done = sync_with_deadline(30.0);
        cudaGraphExecDestroy(ge);
        if (!done || cudaMemcpy(hs.data(), stamps, hs.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) {
            *fatal = true;
            return INFINITY;
        }
        std::vector<double> t;
        for (int i = 0; i < reps; ++i) t.push_back((double)(hs[2 * i + 1] - hs[2 * i]) * 1e-3 / (double)P);
        std::sort(t.begin(), t.end());
        const size_t lo = t.size() / 4, hi = t.size() - t.size() / 4;
        double sum = 0;
        for (size_t i = lo; i < hi; ++i) sum += t[i];
        return sum / (double)(hi - lo);
    }
    // Returns the median microseconds, +inf on a recoverable failure; sets *fatal on a sticky error.
    // l2mode: 0 warm (no eviction), 1 read-flush of a 2 x L2 buffer before each single-launch rep,
    // 2 rotating cold buffers (measure_rotating).
    double measure(Plan &p, const Config &cfg, int warmup, int reps, int l2mode, bool *fatal) {
        const bool l2flush = (l2mode == 1);
        size_t need = workspace_bytes(p, cfg, false);
        if (need > ws_bytes) {
            if (ws) cudaFree(ws);
            ws = nullptr;
            ws_bytes = 0;
            if (cudaMalloc(&ws, need) != cudaSuccess) { cudaGetLastError(); return INFINITY; }
            ws_bytes = need;
        }
        p.reset_ws_state();
        if (l2mode == 2) return measure_rotating(p, cfg, warmup, reps, fatal);
        for (int i = 0; i < warmup; ++i)
            if (launch_conv(p, cfg, x, w, b, y, st, (char *)ws, ws_bytes, z, wdw, bdw) < 0) return INFINITY;
        if (!sync_with_deadline(10.0)) { *fatal = true; return INFINITY; }
        // Each rep is bracketed by two 1-thread kernels that write %globaltimer (256-ns steps; CUDA
        // events on this part advance in ~2-us steps, too coarse for 5-30 us layers). The constant
        // launch latency of the closing stamp is the same for every candidate of a layer.
        std::vector<float> t;
        std::vector<unsigned long long> hs(2 * (size_t)reps);
        for (int i = 0; i < reps; ++i) {
            if (l2flush) l2_flush_device(flush, flush_bytes, (char *)flush + flush_bytes, st);
            timestamp_device(stamps + 2 * i, st);
            if (launch_conv(p, cfg, x, w, b, y, st, (char *)ws, ws_bytes, z, wdw, bdw) < 0) return INFINITY;
            timestamp_device(stamps + 2 * i + 1, st);
            if (!sync_with_deadline(10.0)) { *fatal = true; return INFINITY; }
        }
        if (cudaMemcpy(hs.data(), stamps, hs.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) {
            *fatal = true;
            return INFINITY;
        }
        for (int i = 0; i < reps; ++i) t.push_back((float)((double)(hs[2 * i + 1] - hs[2 * i]) * 1e-3));
        // mean of the middle half: the median's robustness to outliers, finer than one timer step
        std::sort(t.begin(), t.end());
        const size_t lo = t.size() / 4, hi = t.size() - t.size() / 4;
        double s = 0;
        for (size_t i = lo; i < hi; ++i) s += t[i];
        return s / (double)(hi - lo);
    }
};

// ---------------------------------------------------------------------------------------------------
// replay records: one JSON object per line {"family": f, "genes": [...], "beta_us": v}
// ---------------------------------------------------------------------------------------------------
static bool parse_record(const char *line, Config *c, double *beta) {
    const char *g = strstr(line, "\"genes\"");
    const char *b = strstr(line, "\"beta_us\"");
    const char *f = strstr(line, "\"family\"");
    if (!g || !b) return false;
    g = strchr(g, '[');
    if (!g) return false;
    ++g;
    for (int i = 0; i < WPK_NUM_GENES; ++i) {
        char *end;
        c->genes[i] = (int)strtol(g, &end, 10);
        if (end == g) return false;
        g = end;
        while (*g == ',' || *g == ' ') ++g;
    }
    b = strchr(b, ':');
    if (!b) return false;
    ++b;
    while (*b == ' ') ++b;
    if (!strncmp(b, "Infinity", 8) || !strncmp(b, "null", 4)) *beta = INFINITY;
    else *beta = strtod(b, nullptr);
    c->family = 0;
    if (f && (f = strchr(f, ':'))) c->family = (int)strtol(f + 1, nullptr, 10);
    return true;
}

static bool load_replay(TuneCtx &t, const char *path) {
    FILE *fp = fopen(path, "r");
    if (!fp) return false;
    char buf[4096];
    while (fgets(buf, sizeof buf, fp)) {
        Config c;
        double beta;
        if (parse_record(buf, &c, &beta)) t.replay[c] = beta;
    }
    fclose(fp);
    return true;
}

// ---------------------------------------------------------------------------------------------------
// sharded batch evaluation
// ---------------------------------------------------------------------------------------------------
struct Rec {
    int32_t idx;
    int32_t status;
    double beta;
};
static_assert(sizeof(Rec) == 16, "record layout");

static int32_t config_hash(const Config &c) {
    uint32_t h = 2166136261u ^ (uint32_t)c.family;
    for (int g = 0; g < WPK_NUM_GENES; ++g) h = (h ^ (uint32_t)c.genes[g]) * 16777619u;
    return (int32_t)(h & 0x7fffffff);
}

static double evaluate_one(TuneCtx &t, const Config &c, int32_t *status) {
    *status = 0;
    if (!t.valid(c)) { *status = 1; return INFINITY; }
    switch (t.o.eval_mode) {
    case WPK_EVAL_REPLAY: {
        auto it = t.replay.find(c);
        if (it == t.replay.end()) { *status = 2; return INFINITY; }
        return it->second;
    }
    case WPK_EVAL_SYNTHETIC: {   // SPEC.md:235-249 surface, log2(1+gene) so that 0-valued genes are defined
        const double *s = t.o.synthetic;
        double v = s[0];
        for (int g = 0; g < WPK_NUM_GENES; ++g) {
            double dlt = std::log2(1.0 + c.genes[g]) - std::log2(1.0 + s[1 + WPK_NUM_GENES + g]);
            v += s[1 + g] * dlt * dlt;
        }
        return v;
    }
    default: {
        bool fatal = false;
        double b = t.gb->measure(*t.plan, c, t.o.warmup, t.o.reps, t.o.l2_flush, &fatal);
        if (fatal) { t.err = WPK_ERR_CUDA; set_error("tune: " + t.gb->err); *status = 3; }
        else if (!std::isfinite(b)) *status = 4;
        return b;
    }
    }
}

std::vector<Config> TuneCtx::measure_batch(const std::vector<Config> &cfgs) {
    std::vector<Config> fresh;
    for (const Config &c : cfgs) {
        if (memo.count(c)) continue;
        if (std::find(fresh.begin(), fresh.end(), c) != fresh.end()) continue;
        fresh.push_back(c);
    }
    int room = budget - (int)order.size();
    if ((int)fresh.size() > room) fresh.resize(std::max(room, 0));
    // every rank computes the same `fresh` (replicated state), so all ranks exchange or none do
    if (fresh.empty() || err != WPK_OK) return {};
    const int n = (int)fresh.size(), world = std::max(1, o.world), rank = o.rank;
    const int per = (n + world - 1) / world;
    // per rank: `per` fitness records + one flags record {idx -2, status = bit0 time-up | bit1 fatal}
    std::vector<Rec> send(per + 1), recv((size_t)(per + 1) * world);
    if (o.eval_mode == WPK_EVAL_MEASURED && family == WPK_FAMILY_JIT && err == WPK_OK) {
        // this rank's share of the generation is compiled on all host cores first
        // (NVRTC, cached), then measured one by one on the GPU
        std::vector<Config> mine;
        for (int i = 0; i < per; ++i)
            if (rank + i * world < n) mine.push_back(fresh[rank + i * world]);
        const double c0 = wall_seconds();
        jit_precompile(plan->d, mine, 0);
        compile_seconds += wall_seconds() - c0;
    }
    for (int i = 0; i < per; ++i) {
        int j = rank + i * world;
        if (j < n && err == WPK_OK) {
            int32_t st;
            double b = evaluate_one(*this, fresh[j], &st);
            send[i] = Rec{j, st, b};
        } else {
            send[i] = Rec{j < n ? j : -1, j < n ? 3 : 0, INFINITY};   // after a fatal error: not measured
        }
    }
    send[per] = Rec{-2, (time_up() ? 1 : 0) | (err != WPK_OK ? 2 : 0), 0.0};
    std::vector<double> beta(n, INFINITY);
    if (world > 1) {
        if (!o.exchange || o.exchange(o.exchange_ctx, send.data(), (per + 1) * sizeof(Rec), recv.data()) != 0) {
            err = WPK_ERR_INTERNAL;
            set_error("tune: exchange (all-gather of fitness records) failed");
            return {};
        }
        int32_t flags = 0;
        for (const Rec &r : recv)
            if (r.idx == -2) flags |= r.status;
        if (flags & 1) stop_all = true;
        if ((flags & 2) && err == WPK_OK) {
            err = WPK_ERR_CUDA;
            set_error("tune: another rank hit a fatal CUDA error; all ranks stop");
        }
        if (err != WPK_OK) return {};
    } else {
        recv = send;
        if (err != WPK_OK) return {};
    }
    for (const Rec &r : recv)
        if (r.idx >= 0 && r.idx < n) beta[r.idx] = r.beta;
    for (int j = 0; j < n; ++j) {
        memo[fresh[j]] = beta[j];
        order.push_back(fresh[j]);
        if (rec && o.eval_mode == WPK_EVAL_MEASURED) {   // the gathered table: identical on every rank
            fprintf(rec, "{\"family\": %d, \"genes\": %s, \"beta_us\": %s}\n", fresh[j].family,
                    genes_json(fresh[j]).c_str(), dbl(beta[j]).c_str());
        }
        if (beta[j] < best_beta) {   // best-ever; ties keep the first measured
            best_beta = beta[j];
            best = fresh[j];
            have_best = true;
        }
    }
    if (rec) fflush(rec);
    return fresh;
}

// Step1 sampler: each gene uniform over its domain, rejection until valid.
bool sample_valid(TuneCtx &t, Rng &rng, Config *out, int max_reject) {
    for (int i = 0; i < max_reject; ++i) {
        Config c;
        c.family = t.family;
        for (int g = 0; g < WPK_NUM_GENES; ++g) {
            const auto &d = t.sp->dom[g];
            c.genes[g] = d[randint(rng.next(), d.size())];
        }
        if (t.valid(c)) { *out = c; return true; }
    }
    return false;
}

// ---------------------------------------------------------------------------------------------------
// GA, step by step as oracle/search.py ga_run
// ---------------------------------------------------------------------------------------------------
static int roulette(const std::vector<double> &P, double v) {
    double prev = 0.0;
    for (size_t i = 0; i < P.size(); ++i) {
        if (prev < v && v <= P[i]) return (int)i;
        prev = P[i];
    }
    return (int)P.size() - 1;
}

static wpk_status ga_search(TuneCtx &t) {
    const wpk_tune_options &o = t.o;
    const int popsize = std::max(1, o.ga_pop);
    const int m_pool = o.ga_pool > 0 ? o.ga_pool : popsize;
    std::vector<Config> pop;
    Rng rng(o.seed, 0);
    for (int i = 0; i < popsize; ++i) {                      // Step1
        Config c;
        if (!sample_valid(t, rng, &c)) {
            // a sparse space (e.g. a fused depthwise+pointwise plan with K_out = 320): the rejection
            // sampler (10^4 draws) found nothing -- fall back to the expert template
            // when there is one (reading "sparse spaces" in DESIGN.md)
            if (!t.has_default) return fail(WPK_ERR_EXHAUSTED, "GA Step1: no valid config sampled");
            c = t.default_cfg;
        }
        pop.push_back(c);
    }
    // The expert template default replaces the first random individual, so a search
    // never returns something slower than the untuned plan (opt-out: seed_default = 0).
    if (o.seed_default && t.has_default) pop[0] = t.default_cfg;
    for (int gen = 0;; ++gen) {
        t.measure_batch(pop);                                 // Step2 (memoised, sharded)
        if (t.err != WPK_OK) return t.err;
        std::vector<Config> kept;
        std::vector<double> betas;
        for (const Config &c : pop) {
            auto it = t.memo.find(c);
            if (it != t.memo.end()) { kept.push_back(c); betas.push_back(it->second); }
        }
        pop.swap(kept);
        double mn = INFINITY, mx = -INFINITY, sum = 0;
        int nf = 0;
        for (double b : betas)
            if (std::isfinite(b)) { mn = std::min(mn, b); mx = std::max(mx, b); sum += b; ++nf; }
        const double spread = nf ? (mx - mn) / mn : INFINITY;
        t.rounds = gen + 1;
        {
            std::string s = "{\"gen\": " + std::to_string(gen) + ", \"pop\": [";
            for (size_t i = 0; i < pop.size(); ++i) s += (i ? "," : "") + genes_json(pop[i]);
            s += "], \"beta\": [";
            for (size_t i = 0; i < betas.size(); ++i) s += (i ? "," : "") + dbl(betas[i]);
            s += "], \"best_beta\": " + dbl(t.best_beta) + ", \"mean_beta\": " + dbl(nf ? sum / nf : INFINITY) +
                 ", \"spread\": " + dbl(spread) + ", \"measured\": " + std::to_string(t.order.size()) + "}";
            log_line(t, s);
        }
        // Step4: runtimes close enough, budget, generation cap
        if (spread < o.ga_eps || t.exhausted() || gen + 1 >= o.ga_max_gen || pop.empty() || nf == 0 || t.stop())
            break;
        // Step3
        Rng r(o.seed, (uint64_t)gen + 1);
        const int n = (int)pop.size();
        std::vector<double> f(n), p(n);
        double tot = 0;
        for (int i = 0; i < n; ++i) f[i] = std::isfinite(betas[i]) ? 1.0 / betas[i] : 0.0;
        for (int i = 0; i < n; ++i) tot += f[i];
        for (int i = 0; i < n; ++i) p[i] = f[i] / tot;          // Eq. (1)
        std::vector<int> idx(n);
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return p[a] > p[b]; });
        const int k = std::min(o.ga_elites, n);
        std::vector<Config> nxt;
        for (int i = 0; i < k; ++i) nxt.push_back(pop[idx[i]]);  // elites
        const int m = std::min(m_pool, n);
        double psum = 0;
        for (int i = 0; i < m; ++i) psum += p[idx[i]];
        std::vector<double> P(m);
        double acc = 0;
        for (int i = 0; i < m; ++i) { acc += p[idx[i]] / psum; P[i] = acc; }   // Eq. (2), renormalised
        while ((int)nxt.size() < popsize) {
            bool got = false;
            Config child;
            for (int tr = 0; tr < 100 && !got; ++tr) {
                const Config &a = pop[idx[roulette(P, uniform_oc(r.next()))]];
                const Config &b = pop[idx[roulette(P, uniform_oc(r.next()))]];
                Config c;
                c.family = t.family;
                for (int g = 0; g < WPK_NUM_GENES; ++g) c.genes[g] = ((r.next() >> 63) == 0) ? a.genes[g] : b.genes[g];
                for (int g = 0; g < WPK_NUM_GENES; ++g)
                    if (uniform_co(r.next()) < o.ga_mutation) {
                        const auto &d = t.sp->dom[g];
                        c.genes[g] = d[randint(r.next(), d.size())];
                    }
                if (t.valid(c)) { child = c; got = true; }
            }
            if (!got && !sample_valid(t, r, &child)) {
                if (!t.has_default) return fail(WPK_ERR_EXHAUSTED, "GA: no valid child");
                child = t.default_cfg;   // sparse space: the expert template (memoised, costs no budget again)
            }
            nxt.push_back(child);
        }
        pop.swap(nxt);
    }
    return WPK_OK;
}

// Random search (PAPER.md:161 baseline): batches of uniform valid samples, best-ever.
static wpk_status random_search(TuneCtx &t) {
    Rng rng(t.o.seed, 0);
    long long draws = 0;
    if (t.o.seed_default && t.has_default) t.measure_batch({t.default_cfg});
    const long long limit = 100LL * std::max(t.budget, 1);
    const int batch = std::max(1, t.o.ga_pop);
    while (!t.exhausted() && draws < limit && !t.stop()) {
        std::vector<Config> b;
        const int room = t.budget - (int)t.order.size();
        while ((int)b.size() < std::min(batch, room) && draws < limit) {
            Config c;
            if (!sample_valid(t, rng, &c)) return fail(WPK_ERR_EXHAUSTED, "random search: no valid config");
            ++draws;
            if (!t.memo.count(c) && std::find(b.begin(), b.end(), c) == b.end()) b.push_back(c);
        }
        t.measure_batch(b);
        if (t.err != WPK_OK) return t.err;
        ++t.rounds;
        log_line(t, "{\"round\": " + std::to_string(t.rounds) + ", \"measured\": " + std::to_string(t.order.size()) +
                        ", \"best_beta\": " + dbl(t.best_beta) + "}");
    }
    return WPK_OK;
}

// ---------------------------------------------------------------------------------------------------
// tuning-result cache ("a caching mechanism to reuse search results")
// ---------------------------------------------------------------------------------------------------
static std::string cache_key(const Plan &p, int family, int measured_mode) {
    const ConvDesc &d = p.d;
    char b[512];
    std::string dev = "offline";
    if (measured_mode) {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, p.device) == cudaSuccess) {
            char t[400];
            snprintf(t, sizeof t, "%.200s_sm%d_cc%d%d", prop.name, prop.multiProcessorCount, prop.major, prop.minor);
            dev = t;
            for (char &ch : dev)
                if (!isalnum((unsigned char)ch)) ch = '_';
        } else {
            cudaGetLastError();
        }
    }
    snprintf(b, sizeof b, "n%d_c%d_h%d_w%d_k%d_r%d_s%d_st%dx%d_p%dx%d_d%dx%d_g%d_l%d_e%d_t%d_f%d_", d.n, d.c, d.h, d.w,
             d.k, d.r, d.s, d.sh, d.sw, d.ph, d.pw, d.dh, d.dw, d.g, d.layout, d.epilogue, d.dtype, family);
    std::string key(b);
    if (d.fused_dw) key += "dwpw" + std::to_string(d.dw_epi) + "_";   // fused depthwise+pointwise operator
    return key + dev + "_abi" + std::to_string(WPK_ABI_VERSION);
}

static bool cache_lookup(const std::string &path, int budget, Config *cfg, double *beta) {
    FILE *fp = fopen(path.c_str(), "r");
    if (!fp) return false;
    char buf[2048];
    size_t n = fread(buf, 1, sizeof buf - 1, fp);
    fclose(fp);
    buf[n] = 0;
    const char *bb = strstr(buf, "\"budget\"");
    if (!bb || !(bb = strchr(bb, ':')) || atoi(bb + 1) < budget) return false;
    return parse_record(buf, cfg, beta);
}

static void cache_store(const std::string &path, const Config &cfg, double beta, int budget, int search) {
    const std::string tmp = path + ".tmp" + std::to_string((long long)getpid());
    FILE *fp = fopen(tmp.c_str(), "w");
    if (!fp) return;
    fprintf(fp, "{\"family\": %d, \"genes\": %s, \"beta_us\": %s, \"budget\": %d, \"search\": %d}\n", cfg.family,
            genes_json(cfg).c_str(), dbl(beta).c_str(), budget, search);
    fclose(fp);
    rename(tmp.c_str(), path.c_str());
}

}  // namespace wpk

using namespace wpk;

extern "C" wpk_status wpk_conv2d_measure(wpk_plan plan, int32_t warmup, int32_t reps, int32_t l2_flush, double *us) {
    if (!plan || !us) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (reps < 1 || reps > 1024 || warmup < 0) return fail(WPK_ERR_INVALID_ARGUMENT, "bad timing protocol");
    Plan *p = reinterpret_cast<Plan *>(plan);
    GpuBench gb;
    if (!gb.init(*p)) return fail(WPK_ERR_CUDA, "measure: " + gb.err);
    bool fatal = false;
    const Config cfg = p->cfg;
    *us = gb.measure(*p, cfg, warmup, reps, l2_flush, &fatal);
    p->reset_ws_state();   // the measurement ran on its own workspace
    if (fatal) return fail(WPK_ERR_CUDA, "measure: " + gb.err);
    if (!std::isfinite(*us)) return fail(WPK_ERR_CUDA, "measure: the launch failed: " + std::string(wpk_last_error()));
    return WPK_OK;
}

extern "C" wpk_status wpk_conv2d_tune(wpk_plan plan, wpk_search search, int32_t budget, const wpk_tune_options *opts) {
    if (!plan) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL plan");
    if (budget < 1) return fail(WPK_ERR_INVALID_ARGUMENT, "budget must be >= 1");
    if (search < WPK_SEARCH_GA || search > WPK_SEARCH_RANDOM) return fail(WPK_ERR_INVALID_ARGUMENT, "bad search");
    Plan *p = reinterpret_cast<Plan *>(plan);
    TuneCtx t;
    t.plan = p;
    if (opts) {
        if (opts->struct_size != sizeof(wpk_tune_options))
            return fail(WPK_ERR_INVALID_ARGUMENT, "wpk_tune_options.struct_size mismatch");
        t.o = *opts;
    } else {
        wpk_tune_options_init(&t.o);
    }
    if (t.o.world < 1 || t.o.rank < 0 || t.o.rank >= t.o.world) return fail(WPK_ERR_INVALID_ARGUMENT, "bad rank/world");
    if (t.o.world > 1 && !t.o.exchange) return fail(WPK_ERR_INVALID_ARGUMENT, "world > 1 needs an exchange callback");
    if (t.o.reps < 1 || t.o.reps > 1024 || t.o.warmup < 0) return fail(WPK_ERR_INVALID_ARGUMENT, "bad timing protocol");
    t.family = (t.o.family == WPK_FAMILY_AUTO) ? default_family(p->d) : t.o.family;
    std::string why;
    if (!family_applicable(p->d, t.family, &why)) return fail(WPK_ERR_INVALID_ARGUMENT, "family not applicable: " + why);
    t.sp = &family_space(t.family);
    t.budget = budget;
    {
        Config dc = default_config(p->d, t.family);
        t.has_default = (dc.family == t.family) && config_valid(p->d, dc, nullptr);
        t.default_cfg = dc;
    }
    t.t_start = wall_seconds();
    // the JIT family's cubins go to the tuning cache directory too, unless WPK_JIT_CACHE_DIR chose one
    if (t.family == WPK_FAMILY_JIT && t.o.cache_dir && t.o.cache_dir[0] && !getenv("WPK_JIT_CACHE_DIR"))
        jit_set_cache_dir(t.o.cache_dir);
    std::string cpath;
    if (t.o.cache_dir && t.o.cache_dir[0]) {
        cpath = std::string(t.o.cache_dir) + "/" + cache_key(*p, t.family, t.o.eval_mode == WPK_EVAL_MEASURED) + ".json";
        Config hit;
        double hb = 0;
        bool use = cache_lookup(cpath, budget, &hit, &hb) && config_valid(p->d, hit, nullptr);
        if (t.o.world > 1) {   // collective: a hit counts only if every rank read the same record
            Rec mine{use ? 1 : 0, use ? config_hash(hit) : 0, use ? hb : 0.0};
            std::vector<Rec> all(t.o.world);
            if (t.o.exchange(t.o.exchange_ctx, &mine, sizeof(Rec), all.data()) != 0)
                return fail(WPK_ERR_INTERNAL, "tune: cache-decision exchange failed");
            for (const Rec &r : all)
                if (r.idx != 1 || r.status != mine.status || r.beta != mine.beta) use = false;
        }
        if (use) {
            p->cfg = hit;
            p->reset_ws_state();
            p->best_us = hb;
            p->measured = 0;
            p->rounds = 0;
            p->tune_seconds = wall_seconds() - t.t_start;
    if (t.family == WPK_FAMILY_JIT)
        log_line(t, "{\"jit_compile_seconds\": " + dbl(t.compile_seconds) + ", \"tune_seconds\": " + dbl(p->tune_seconds) + "}");
            return WPK_OK;
        }
    }
    if (t.o.eval_mode == WPK_EVAL_REPLAY) {
        if (!t.o.replay_path || !load_replay(t, t.o.replay_path))
            return fail(WPK_ERR_INVALID_ARGUMENT, "replay mode needs a readable replay_path");
    }
    GpuBench gb;
    if (t.o.eval_mode == WPK_EVAL_MEASURED) {
        if (!gb.init(*p)) return fail(WPK_ERR_CUDA, "tune: " + gb.err);
        t.gb = &gb;
    }
    if (t.o.record_path) t.rec = fopen(t.o.record_path, "a");   // per-rank path (caller's choice)
    if (t.o.log_path && t.o.rank == 0) t.log = fopen(t.o.log_path, "w");
    wpk_status st;
    if (search == WPK_SEARCH_GA) st = ga_search(t);
    else if (search == WPK_SEARCH_RANDOM) st = random_search(t);
    else st = rl_search(t);
    struct Closer {   // history files stay open through the finalist re-timing
        TuneCtx &t;
        ~Closer() {
            if (t.rec) fclose(t.rec);
            if (t.log) fclose(t.log);
        }
    } closer{t};
    if (st != WPK_OK) return st;
    if (!t.have_best || !std::isfinite(t.best_beta)) return fail(WPK_ERR_EXHAUSTED, "every candidate failed");
    // Finalists (SURVEY.md 8(d) protocol item 2): the top-k measured configs are re-timed on every
    // rank and the lowest median across ranks wins. Deterministic given the gathered table: every
    // rank holds the same memo, ranks the same finalists and sees the same all-gathered timings.
    if (t.o.eval_mode == WPK_EVAL_MEASURED && t.o.finalists > 0 && t.order.size() > 1) {
        std::vector<int> idx(t.order.size());
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return t.memo[t.order[a]] < t.memo[t.order[b]]; });
        std::vector<Config> fin;
        for (int i : idx)
            if ((int)fin.size() < t.o.finalists && std::isfinite(t.memo[t.order[i]])) fin.push_back(t.order[i]);
        const int k = (int)fin.size(), world = std::max(1, t.o.world);
        std::vector<Rec> mine(k), all((size_t)k * world);
        for (int i = 0; i < k; ++i) {
            bool fatal = false;
            double b = (t.err == WPK_OK) ? gb.measure(*p, fin[i], t.o.warmup, t.o.reps, t.o.l2_flush, &fatal) : INFINITY;
            if (fatal && t.err == WPK_OK) { t.err = WPK_ERR_CUDA; set_error("tune: " + gb.err); }
            mine[i] = Rec{i, (fatal || t.err != WPK_OK) ? 3 : 0, b};
        }
        if (world > 1) {
            if (t.o.exchange(t.o.exchange_ctx, mine.data(), k * sizeof(Rec), all.data()) != 0)
                return fail(WPK_ERR_INTERNAL, "tune: finalist exchange failed");
        } else {
            all = mine;
        }
        for (const Rec &r : all)
            if (r.status == 3) return fail(WPK_ERR_CUDA, "tune: a rank failed while re-timing the finalists");
        int besti = -1;
        double bestm = INFINITY;
        for (int i = 0; i < k; ++i) {
            std::vector<double> v;
            for (int r = 0; r < world; ++r) v.push_back(all[(size_t)r * k + i].beta);
            std::sort(v.begin(), v.end());
            const double med = (v.size() & 1) ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
            log_line(t, "{\"finalist\": " + std::to_string(i) + ", \"genes\": " + genes_json(fin[i]) +
                            ", \"search_beta\": " + dbl(t.memo[fin[i]]) + ", \"median_beta\": " + dbl(med) + "}");
            if (med < bestm) { bestm = med; besti = i; }   // ties keep the better search-time rank
        }
        if (besti >= 0) {
            t.best = fin[besti];
            t.best_beta = bestm;
        }
    }
    // every rank must have chosen the same config (replicated deterministic searcher state)
    if (t.o.world > 1) {
        Rec mine{t.best.family, 0, t.best_beta};
        int32_t h = 0;
        for (int g = 0; g < WPK_NUM_GENES; ++g) h = h * 1000003 + t.best.genes[g];
        mine.status = h;
        std::vector<Rec> all(t.o.world);
        if (t.o.exchange(t.o.exchange_ctx, &mine, sizeof(Rec), all.data()) != 0)
            return fail(WPK_ERR_INTERNAL, "tune: final exchange failed");
        for (const Rec &r : all)
            if (r.idx != mine.idx || r.status != mine.status || r.beta != mine.beta)
                return fail(WPK_ERR_INTERNAL, "tune: ranks disagree on the chosen config");
    }
    p->cfg = t.best;
    p->reset_ws_state();   // the tuning workspace is gone; the plan's own starts from scratch
    p->best_us = t.best_beta;
    if (!cpath.empty() && t.o.rank == 0) cache_store(cpath, t.best, t.best_beta, budget, (int)search);
    p->measured = (int)t.order.size();
    p->rounds = t.rounds;
    p->tune_seconds = wall_seconds() - t.t_start;
    if (t.family == WPK_FAMILY_JIT)
        log_line(t, "{\"jit_compile_seconds\": " + dbl(t.compile_seconds) + ", \"tune_seconds\": " + dbl(p->tune_seconds) + "}");
    return WPK_OK;
}
