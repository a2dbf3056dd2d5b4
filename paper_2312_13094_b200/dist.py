"""Rank context: one process per GPU, torch.distributed for the control
plane (handle exchange, barriers, gathers), NVLink peer memory for the data
plane.

Replaces the SPEC's ``spawn_ranks`` / ``RankContext`` / ``Transport``
(SPEC.md:406-428): ranks are real processes launched by torchrun (the
paper's ``mpirun``); halo payloads move GPU-to-GPU through
CUDA IPC mappings (runtime_plan.py), never through the host.  A gloo
subgroup carries the small control messages so they work on CPU-only
test runs too.
"""
from __future__ import annotations

import os
from typing import Any, List, Optional

_CTX = None


class RankContext:
    def __init__(self):
        import torch
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        if self.dist is None and int(os.environ.get("WORLD_SIZE", "1")) > 1:
            import torch.distributed as d
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            d.init_process_group(backend=default_backend())
            self.dist = d
        if self.dist is not None:
            self.rank = self.dist.get_rank()
            self.size = self.dist.get_world_size()
            backend = self.dist.get_backend()
            self.ctrl = self.dist.new_group(backend="gloo") if backend != "gloo" else None
        else:
            self.rank, self.size, self.ctrl = 0, 1, None
        local = int(os.environ.get("LOCAL_RANK", self.rank))
        self.device = None
        if torch.cuda.is_available():
            n = torch.cuda.device_count()
            self.device = local % n if n else 0
            torch.cuda.set_device(self.device)

    # -- control plane -------------------------------------------------------
    def allgather(self, obj: Any) -> List[Any]:
        if self.size == 1:
            return [obj]
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.ctrl)
        return out

    def barrier(self):
        if self.size > 1:
            self.dist.barrier(group=self.ctrl)

    def allreduce_max(self, value: float) -> float:
        if self.size == 1:
            return value
        return max(self.allgather(value))


def default_backend() -> str:
    """Process-group backend for the control plane.  NCCL when every rank
    has its own GPU; gloo on CPU and when ranks are oversubscribed onto fewer
    GPUs (NCCL rejects two ranks on one device; the halo data plane is CUDA
    IPC either way, which works between processes sharing a device).
    ``SDMP_DIST_BACKEND`` overrides."""
    import torch
    forced = os.environ.get("SDMP_DIST_BACKEND")
    if forced:
        return forced
    if not torch.cuda.is_available():
        return "gloo"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return "nccl" if world <= torch.cuda.device_count() else "gloo"


class SelfContext(RankContext):
    """A one-rank world on this process's device (``Grid(..., comm="self")``):
    used to compute single-rank references inside a multi-rank job."""

    def __init__(self, device=None):
        import torch
        self.dist = None
        self.rank, self.size, self.ctrl = 0, 1, None
        self.device = device
        if self.device is None and torch.cuda.is_available():
            self.device = torch.cuda.current_device()


def context() -> RankContext:
    global _CTX
    if _CTX is None:
        _CTX = RankContext()
    return _CTX


def reset_context():
    """Drop the cached context (tests that re-initialise process groups)."""
    global _CTX
    _CTX = None
