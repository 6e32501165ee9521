"""The wpk_exchange_fn all-gather used when candidate evaluation is sharded over GPUs
(BASELINE.json north_star: "GA population / RL rollout candidates are evaluated in parallel, one
candidate batch per GPU, with an NCCL all-gather of fitness values over NVLink").

torch.distributed owns the process group (ProcessGroupNCCL on GPUs, gloo for the CPU tests); the
C library only sees a C function pointer. Records are fixed-size and placed by rank, so the
gathered table is identical on every rank and the replicated searcher state stays in lock-step.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from ._lib import EXCHANGE_FN

_KEEP = []   # keep ctypes callbacks alive for the process lifetime


def make_exchange(group=None) -> dict:
    """Return {"exchange": fn} for make_options / Conv2dPlan.tune (pass rank and world too)."""
    backend = dist.get_backend(group)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")

    def _cb(ctx, send, nbytes, recv):
        try:
            src = torch.empty(nbytes, dtype=torch.uint8)
            ctypes.memmove(src.data_ptr(), send, nbytes)
            src = src.to(dev)
            out = torch.empty(nbytes * world, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(out, src, group=group)
            out = out.cpu()
            ctypes.memmove(recv, out.data_ptr(), nbytes * world)
            return 0
        except Exception:   # noqa: BLE001 -- any failure is reported to C as non-zero
            return 1

    fn = EXCHANGE_FN(_cb)
    _KEEP.append(fn)
    return {"exchange": fn}
