"""Random vs GA vs RL search on measured B200 landscapes (the analogue of PAPER.md Fig. 3a / Table 1,
P:160-177): for each layer, every valid tcgen05 config is measured once on the GPU (a random search
whose budget is the number of valid configs, recorded as JSONL); then each searcher is replayed
(wpk_tune_options.eval_mode = REPLAY) on that fixed landscape for several budgets and seeds, so the
comparison is between search algorithms only, with no timing noise between them.

usage:  python tools/search_compare.py record OUTDIR      (GPU: writes OUTDIR/<layer>.jsonl)
        python tools/search_compare.py compare OUTDIR     (CPU: replays, prints a markdown table)
"""
import itertools
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_2008_04567_b200 import Conv2dPlan

DOM = [[16, 32, 64, 96, 128, 192, 256], [2, 3, 4, 5, 6, 7, 8], [1, 2, 4, 8, 16], [0, 1, 2, 3], [0, 1, 2, 3],
       [1, 2, 4], [128, 256]]   # include/wpk.h: the UMMA family's 7 gene domains
BUDGETS = [8, 16, 32, 64, 128]
SEEDS = range(10)


def layers():
    out = [(L, "table1_n1") for L in workloads.table1(1)]
    r50 = {L.name: L for L in workloads.resnet50(32)}
    out += [(r50[n], "resnet50_n32") for n in ("s3b1.c2", "s4b1.c1", "s5b0.c2")]
    return out


def make_plan(L, device=None):
    kw = {} if device is None else {"device": device}
    return Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, L.dil, L.groups, layout="nhwc",
                      dtype="bf16", **kw)


def record(outdir):
    os.makedirs(outdir, exist_ok=True)
    for L, tag in layers():
        plan = make_plan(L)
        nvalid = sum(plan.config_valid(1, list(g)) for g in itertools.product(*DOM))
        path = os.path.join(outdir, f"{tag}_{L.name}.jsonl")
        if os.path.exists(path):
            os.remove(path)
        res = plan.tune("random", nvalid, record_path=path, seed_default=0, warmup=2, reps=7)
        print(f"{tag} {L.name}: {nvalid} valid configs, {res.measured} measured, best {res.best_us:.2f} us "
              f"{res.genes}", flush=True)


def compare(outdir):
    rows = ["| workload | layer | valid | optimum us | budget | random | GA | RL |", "|---|---|---|---|---|---|---|---|"]
    summary = {}
    for L, tag in layers():
        path = os.path.join(outdir, f"{tag}_{L.name}.jsonl")
        if not os.path.exists(path):
            continue
        recs = [json.loads(l) for l in open(path) if l.strip()]
        betas = [r["beta_us"] for r in recs if r["beta_us"] is not None and r["beta_us"] < 1e30]
        opt = min(betas)
        plan = make_plan(L, device=0)
        for B in BUDGETS:
            cells = []
            for search in ("random", "ga", "rl"):
                ratios = []
                for sd in SEEDS:
                    r = plan.tune(search, B, eval_mode="replay", replay_path=path, seed=sd, seed_default=0)
                    ratios.append(r.best_us / opt)
                mean = statistics.mean(ratios)
                hit = sum(x <= 1.05 for x in ratios) / len(ratios)
                summary.setdefault((search, B), []).append(mean)
                cells.append(f"{mean:.3f} ({hit:.0%})")
            rows.append(f"| {tag} | {L.name} | {len(betas)} | {opt:.2f} | {B} | " + " | ".join(cells) + " |")
    rows.append("")
    rows.append("| budget | random | GA | RL |  (geometric-mean-free average of best/optimum over the layers) |")
    rows.append("|---|---|---|---|---|")
    for B in BUDGETS:
        vals = [statistics.mean(summary.get((s, B), [float("nan")])) for s in ("random", "ga", "rl")]
        rows.append(f"| {B} | " + " | ".join(f"{v:.3f}" for v in vals) + " | |")
    print("\n".join(rows))


if __name__ == "__main__":
    if sys.argv[1] == "record":
        record(sys.argv[2])
    else:
        compare(sys.argv[2])
