"""The reference SPEC's operation names, mapped onto this
framework, so code written against the specified API finds them.

| SPEC operation | here |
|---|---|
| `allocate(spec, decomposition)` | :func:`allocate` -> a zero-initialised distributed ``Function`` / ``TimeFunction`` |
| `write_global(field, region, value)` | :func:`write_global` (= ``field.data[region] = value``, collective) |
| `gather(field)` | :func:`gather` (= ``field.data.gather()``) |
| `region_boxes`, `global_to_local`, ... | ``distfield`` / ``decomposition`` (same names) |
| `align_accesses`, `optimize_halospots`, `lower_mode` | ``compiler`` (same names) |
| `build_clusters(equations, decomposition)` | :func:`build_clusters` -> per-kernel halo requirements |
| `build_schedule_tree(clusters)` | :func:`build_schedule_tree` -> Listing-5/6 text |
| `spawn_ranks(nranks, topology, program)` | :func:`spawn_ranks` (CPU processes, gloo; GPU runs use torchrun) |
| `pack_region` / `unpack_region` | :func:`pack_region` / :func:`unpack_region` (device kernels, C-ABI ``sdmp_pack``/``sdmp_unpack``) |
| `halo_exchange`, `execute_plan_full` | ``Operator.apply(mpi="basic" / "diagonal" / "full")`` (the plan executor) |
| `diffusion_kernel`, `acoustic_kernel`, `elastic_kernel`, `tti_gxx_kernel` | :func:`diffusion_kernel` ... (``kernels`` factories) |
| `run_benchmark`, `verify_against_single_rank`, `efficiency`, `scaling_report` | ``bench_cli`` |
"""
from __future__ import annotations

import os
from typing import Callable, Optional, Sequence

from . import compiler as CP
from . import kernels as KD
from . import symbolics as S
from .api import Function, Grid, TimeFunction, _FUNCS


def allocate(spec: S.FieldSpec, decomposition=None, comm=None) -> Function:
    """a zero-initialised distributed field for ``spec``
    (FULL = local shape + 2 halo per axis, time_order + 1 buffers), on the
    ranks of the current job (``decomposition`` fixes the topology)."""
    if spec in _FUNCS:
        return _FUNCS[spec]
    topo = decomposition.topology.dims if decomposition is not None else None
    grid = Grid(spec.grid.shape, spec.grid.extent, topology=topo, comm=comm)
    if spec.time_order > 0:
        return TimeFunction(spec.name, grid, space_order=spec.space_order,
                            time_order=spec.time_order, halo=spec.halo)
    return Function(spec.name, grid, space_order=spec.space_order, halo=spec.halo)


def write_global(field: Function, region, value) -> None:
    """SPEC.md:232-240 (collective): write ``value`` into the global
    ``region`` (a tuple of slices / indices, or ``...``)."""
    field.data[region] = value


def gather(field: Function, buffer: Optional[int] = None):
    """SPEC.md:242-250 (collective): the global array."""
    return field.data.gather(buffer)


def build_clusters(equations: Sequence, decomposition) -> list:
    """kernels recognised from the solved updates with their
    halo requirement (field set and per-axis radius) per phase; empty
    requirements on one rank."""
    kernels = CP.recognise(list(equations))
    an = CP.halo_phases(kernels, decomposition.nranks)
    return [(ph.kernel, ph.halo) for ph in an.phases]


def build_schedule_tree(equations: Sequence, decomposition) -> str:
    """SPEC.md:338-346 + Listing 5/6: the time loop with its HaloSpots."""
    kernels = CP.recognise(list(equations))
    updates = [e for e in equations if isinstance(e, S.StencilEquation)]
    return CP.dump_plan(kernels, decomposition.nranks, None, updates)


def _spawn_worker(rank, nranks, port, program, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(nranks), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    from . import dist as D
    D.reset_context()
    try:
        q.put((rank, program(D.context())))
    except Exception as exc:  # noqa: BLE001 - reported with the rank
        q.put((rank, RuntimeError(f"rank {rank}: {exc!r}")))
    finally:
        dist.destroy_process_group()


def spawn_ranks(nranks: int, program: Callable, topology=None, timeout: float = 300.0) -> list:
    """run ``program(ctx)`` on ``nranks`` CPU processes (gloo
    control plane; ``ctx`` offers rank / size / barrier / allgather /
    allreduce_max) and return the per-rank results; a failing or hung rank
    raises naming the rank.  GPU jobs are launched one process per GPU by
    torchrun instead.  ``program`` must be picklable (module level)."""
    import socket

    import torch.multiprocessing as mp
    if topology is not None:
        n = 1
        for d in topology:
            n *= d
        if n != nranks:
            raise ValueError(f"topology {tuple(topology)} does not hold {nranks} ranks")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_spawn_worker, args=(r, nranks, port, program, q))
             for r in range(nranks)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in procs:
            r, v = q.get(timeout=timeout)
            out[r] = v
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.terminate()
    missing = [r for r in range(nranks) if r not in out]
    if missing:
        raise RuntimeError(f"ranks {missing} did not finish (watchdog {timeout} s)")
    for r in range(nranks):
        if isinstance(out[r], Exception):
            raise out[r]
    return [out[r] for r in range(nranks)]


def pack_region(field: Function, box, buffer: int = 0):
    """the FULL-coordinate ``box`` of time buffer ``buffer``
    as a contiguous row-major device tensor (``sdmp_pack``)."""
    import torch

    from . import runtime as R
    lo = list(box[0]) + [0] * (3 - len(box[0]))
    hi = list(box[1]) + [1] * (3 - len(box[1]))
    out = torch.empty(_vol(lo, hi), dtype=torch.float32, device=field.storage.device)
    if out.numel():
        R.pack(field.storage[buffer], field.full3, lo, hi, out)
        torch.cuda.synchronize()
    return out


def unpack_region(field: Function, box, buf, buffer: int = 0) -> None:
    """write a packed buffer back into ``box``."""
    from . import runtime as R
    lo, hi = list(box[0]) + [0] * (3 - len(box[0])), list(box[1]) + [1] * (3 - len(box[1]))
    if buf.numel() != _vol(lo, hi):
        raise ValueError(f"buffer of {buf.numel()} values does not match box {box}")
    if buf.numel():
        import torch
        R.unpack(field.storage[buffer], field.full3, lo, hi, buf)
        torch.cuda.synchronize()


def _vol(lo, hi):
    v = 1
    for a, b in zip(lo, hi):
        v *= max(0, b - a)
    return v


def diffusion_kernel(grid: Grid, so: int = 2, name: str = "u"):
    """SPEC.md:572-578."""
    return KD.diffusion_model(grid, so=so, name=name)


def acoustic_kernel(grid: Grid, so: int = 8, vp=None, name: str = "u"):
    """SPEC.md:580-585 (no damping)."""
    return KD.acoustic_model(grid, so=so, vp=vp, name=name)


def elastic_kernel(grid: Grid, so: int = 8):
    """the collocated velocity-stress system."""
    return KD.elastic_model(grid, so=so, collocated=True)


def tti_gxx_kernel(grid: Grid, so: int = 8, vp=None, name: str = "u"):
    """the single-field rotated operator G = D^T D."""
    return KD.rotated_model(grid, so=so, vp=vp, name=name)
