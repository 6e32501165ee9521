// Tuner internals shared by tune.cpp (evaluator, GA, random search) and ppo.cpp (RL-search).
#pragma once
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "rng.h"
#include "wpk_internal.h"

namespace wpk {

struct GpuBench;   // measured-mode scratch state (tune.cpp)

// One tuning session: the memo table (reading c16), the budget of distinct measured configs, the
// sharded batch evaluator and the history/record files.
struct TuneCtx {
    Plan *plan = nullptr;
    wpk_tune_options o{};
    int family = 0;
    const Space *sp = nullptr;
    std::map<Config, double> memo;
    std::vector<Config> order;          // measurement order
    int budget = 0;
    std::map<Config, double> replay;
    FILE *rec = nullptr, *log = nullptr;
    GpuBench *gb = nullptr;
    wpk_status err = WPK_OK;
    double t_start = 0;
    // best-ever
    bool have_best = false;
    Config best;
    double best_beta = 1e300;
    int rounds = 0;
    double compile_seconds = 0;         // JIT family: host NVRTC time spent inside this tune
    bool has_default = false;
    Config default_cfg;

    bool exhausted() const { return (int)order.size() >= budget; }
    bool valid(const Config &c) const { return config_valid(plan->d, c, nullptr); }
    bool time_up() const;
    // Stop decisions are collective: with world > 1 every exchange also carries each rank's
    // (time-up, fatal-error) flags, OR-reduced, so all ranks leave the search at the same step and
    // never enter an all-gather that another rank skips. stop() is the searchers' check.
    bool stop_all = false;
    bool stop() const { return o.world > 1 ? stop_all : time_up(); }
    // Measure the new distinct configs of `cfgs` (first-occurrence order, truncated to the
    // remaining budget), sharded over ranks; returns the configs measured. Updates memo/best.
    std::vector<Config> measure_batch(const std::vector<Config> &cfgs);
};

bool sample_valid(TuneCtx &t, Rng &rng, Config *out, int max_reject = 10000);
wpk_status rl_search(TuneCtx &t);   // ppo.cpp
double wall_seconds();
void log_line(TuneCtx &t, const std::string &s);
std::string genes_json(const Config &c);

}  // namespace wpk
