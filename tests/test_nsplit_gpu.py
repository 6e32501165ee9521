"""N-split forward: two processes with a gloo process group on ONE
GPU each run their shard of a batch; every shard's output must equal the same images of a
one-process run of the whole batch, bit for bit, in uniform (not only exact-integer) mode, with the
same kernel configuration on both sides. Also runs bench.py's N>1 code path (torchrun, gloo, one
device) as a smoke test of the sharded tuner exchange and the max-over-ranks timing."""
import json
import os
import subprocess
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import workloads
    from paper_2008_04567_b200 import Conv2dPlan
    from paper_2008_04567_b200.nsplit import shard_batch, shard_plan, shard_range
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {}
    cases = [(workloads.ConvLayer("s3b1.c2_n6", 6, 128, 28, 28, 128, 3, 3, 1, 1), "bf16", (1, [128, 4, 1, 0, 0, 2, 128])),
             (workloads.ConvLayer("s4b1.c1_n5", 5, 1024, 14, 14, 256, 1, 1, 1, 0), "bf16", (1, [128, 4, 2, 0, 0, 1, 128])),
             (workloads.ConvLayer("conv1_n3", 3, 3, 64, 64, 64, 7, 7, 2, 3), "bf16", None),
             (workloads.ConvLayer("tf32_n4", 4, 64, 20, 20, 96, 3, 3, 2, 1), "tf32", None)]
    for L, dtype, cfg in cases:
        x, w, b = workloads.generate(L, dtype, "uniform", seed=31)
        xn = x.permute(0, 2, 3, 1).contiguous()
        wn = w.permute(0, 2, 3, 1).contiguous().cuda()
        bc = b.cuda()
        full = Conv2dPlan(L.n, L.c, L.h, L.w, L.k, L.r, L.s, L.stride, L.pad, layout="nhwc", dtype=dtype)
        shard = shard_plan(L, rank, world, layout="nhwc", dtype=dtype)
        if cfg is None:
            cfg = full.config
        full.set_config(*cfg)
        shard.set_config(*cfg)
        y_full = full.run(xn.cuda(), wn, bc).cpu()
        y_shard = shard.run(shard_batch(xn, rank, world).cuda(), wn, bc).cpu()
        s, c = shard_range(L.n, rank, world)
        same = torch.equal(y_full[s:s + c].view(torch.int16 if dtype != "tf32" else torch.int32),
                           y_shard.view(torch.int16 if dtype != "tf32" else torch.int32))
        # every image is covered exactly once across ranks
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([c]))
        res[L.name] = {"bit_equal": bool(same), "start": s, "count": c, "total": int(sum(t.item() for t in counts))}
    json.dump(res, open(os.path.join(out_dir, f"rank{rank}.json"), "w"))
    dist.destroy_process_group()


def test_nsplit_shards_equal_single_process(tmp_path):
    world, port = 2, 29517
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    seen = {}
    for r in range(world):
        res = json.load(open(tmp_path / f"rank{r}.json"))
        for name, v in res.items():
            assert v["bit_equal"], (r, name)
            assert v["total"] > 0
            seen.setdefault(name, []).append((v["start"], v["count"], v["total"]))
    for name, parts in seen.items():
        parts.sort()
        assert parts[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert parts[-1][0] + parts[-1][1] == parts[0][2]


def test_bench_two_ranks_gloo_one_device(tmp_path):
    env = dict(os.environ, WPK_BENCH_BACKEND="gloo", OMP_NUM_THREADS="4", WPK_BENCH_WATCHDOG="420")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--tune-budget", "6", "--ga-pop", "4", "--no-cudnn",
           "--no-cpu-baseline", "--graph-refine", "1"]
    with open(tmp_path / "out.txt", "w") as fo, open(tmp_path / "err.txt", "w") as fe:
        try:
            rc = subprocess.run(cmd, env=env, stdout=fo, stderr=fe, timeout=600, cwd=ROOT).returncode
        except subprocess.TimeoutExpired:
            rc = "timeout"
    out, err = open(tmp_path / "out.txt").read(), open(tmp_path / "err.txt").read()
    assert rc == 0, (rc, err[-6000:])
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["global_batch"] == 64
