"""Benchmark driver API of the SPEC's ``bench_cli`` module:
RunConfig, MetricsRecord, run_benchmark, verify_against_single_rank,
efficiency, scaling_report and a CSV/JSON command line.

    python -m paper_2312_13094_b200.bench_cli --kernel acoustic --shape 64,64,64 \
        --so 8 --tn 20 --mode full --topology 2,1,1 --check --json

Under torchrun every rank runs the same command; rank 0 prints.  Runs execute
on the GPU through the Operator API (there is no CPU execution path; the
CPU reference is the oracle used by the tests).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys
import time
from dataclasses import asdict, dataclass, field
from typing import List, Optional, Sequence

import numpy as np

CSV_COLUMNS = ("kernel", "shape", "sdo", "ranks", "topology", "mode", "transport", "steps",
               "walltime_s", "gpts_per_s", "msgs_per_rank_step", "bytes_per_rank_step",
               "max_diff", "checksum")


@dataclass
class RunConfig:
    """SPEC.md:630-634."""
    kernel: str = "acoustic"
    shape: tuple = (64, 64, 64)
    sdo: int = 8
    steps: int = 20
    topology: Optional[tuple] = None
    mode: str = "diagonal"
    transport: str = "nvlink"
    check: bool = False
    seed: int = 0


@dataclass
class MetricsRecord:
    """throughput = DOMAIN points x timesteps / wall."""
    config: dict
    walltime_s: float
    gpts_per_s: float
    msgs_per_rank_step: int
    bytes_per_rank_step: int
    checksum: float
    max_diff: Optional[float] = None
    sections: dict = field(default_factory=dict)

    def row(self) -> dict:
        c = self.config
        return {"kernel": c["kernel"], "shape": "x".join(map(str, c["shape"])), "sdo": c["sdo"],
                "ranks": c.get("ranks", 1), "topology": ",".join(map(str, c.get("topology") or ())),
                "mode": c["mode"], "transport": c["transport"], "steps": c["steps"],
                "walltime_s": self.walltime_s, "gpts_per_s": self.gpts_per_s,
                "msgs_per_rank_step": self.msgs_per_rank_step,
                "bytes_per_rank_step": self.bytes_per_rank_step,
                "max_diff": self.max_diff, "checksum": self.checksum}


def efficiency(throughputs: Sequence[float]) -> List[float]:
    """SPEC.md:661-666 / PAPER.md:735-737: 100 * T(N) / (T(1) * N) for
    node multipliers N = 1, 2, 4, ... (index i -> N = 2**i)."""
    t1 = throughputs[0]
    return [100.0 * t / (t1 * (2 ** i)) for i, t in enumerate(throughputs)]


def scaling_report(kind: str, base_shape: Sequence[int], ranks: Sequence[int]) -> List[dict]:
    """strong keeps the global shape; weak doubles one axis
    per rank doubling, cycling axes (32^3 -> 64x32x32 -> 64x64x32)."""
    rows = []
    for r in ranks:
        shape = list(base_shape)
        if kind == "weak":
            doublings = int(round(math.log2(r)))
            for d in range(doublings):
                shape[d % len(shape)] *= 2
        elif kind != "strong":
            raise ValueError("kind must be 'strong' or 'weak'")
        rows.append({"ranks": r, "shape": tuple(shape)})
    return rows


def _build(cfg: RunConfig, comm=None):
    from . import Grid, Operator, SparseTimeFunction
    from . import kernels as KD
    from . import symbolics as S
    grid = Grid(cfg.shape, tuple(10.0 * (n - 1) for n in cfg.shape), topology=cfg.topology,
                comm=comm)
    nt = cfg.steps
    if cfg.kernel == "acoustic":
        kd = KD.acoustic_model(grid, so=cfg.sdo, name="u_bench" if comm is None else "u_ref")
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        src = KD.point_source(grid, [tuple(0.5 * e + 1.7 for e in grid.extent)], nt, dt,
                              f0=0.03, name="src_bench" if comm is None else "src_ref")
        terms = [src.inject(u.forward, expr=src * S.DT ** 2 / m)]
        out = [u]
    elif cfg.kernel == "damped":
        kd = KD.damped_acoustic_model(grid, so=cfg.sdo, nbl=max(2, min(cfg.shape) // 8),
                                      name="u_bench" if comm is None else "u_ref")
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        src = KD.point_source(grid, [tuple(0.5 * e + 1.7 for e in grid.extent)], nt, dt,
                              f0=0.03, name="src_bench" if comm is None else "src_ref")
        terms = [src.inject(u.forward, expr=src * S.DT ** 2 / m)]
        out = [u]
    elif cfg.kernel == "diffusion":
        kd = KD.diffusion_model(grid, so=cfg.sdo, name="u_bench" if comm is None else "u_ref")
        u = kd.fields["u"]
        rng = np.random.default_rng(cfg.seed)
        u.data[...] = np.float32(rng.random(cfg.shape))
        dt = float(np.float32(0.1 * min(grid.spacing) ** 2))
        terms, out = [], [u]
    elif cfg.kernel == "tti":
        kd = KD.tti_model(grid, so=cfg.sdo)
        kd.fields["p"].data[...] = np.float32(np.random.default_rng(cfg.seed).standard_normal(cfg.shape))
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
        terms, out = [], [kd.fields["p"], kd.fields["r"]]
    elif cfg.kernel in ("elastic", "visco"):
        kd = (KD.viscoelastic_model(grid, so=cfg.sdo) if cfg.kernel == "visco"
              else KD.elastic_model(grid, so=cfg.sdo))
        kd.fields["txx"].data[...] = np.float32(
            np.random.default_rng(cfg.seed).standard_normal(cfg.shape))
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1)))
        terms, out = [], [kd.fields[n] for n in KD.VNAMES + KD.TNAMES]
    else:
        raise ValueError(f"unknown kernel {cfg.kernel}")
    return grid, Operator([kd] + terms), out, dt


def run_benchmark(cfg: RunConfig) -> MetricsRecord:
    """SPEC.md:643-651 (GPU, through Operator.apply)."""
    import torch
    from . import api
    api._FUNCS.clear()
    grid, op, out, dt = _build(cfg)
    op.apply(time_M=0, dt=dt, mpi=cfg.mode)  # plan build + warm run
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op.apply(time_m=1, time_M=cfg.steps - 1, dt=dt, mpi=cfg.mode)
    wall = grid.ctx.allreduce_max(time.perf_counter() - t0)
    ep = op.plan(cfg.mode)
    msgs = ep.message_count()
    nbytes = 4 * sum(m.volume * len(a.spot.fields)
                     for a in ep.actions if a.kind == "post" for m in a.messages)
    fields = [f.data_gather() for f in out]
    checksum = float(sum(np.abs(f.astype(np.float64)).sum() for f in fields))
    npts = math.prod(cfg.shape) * (cfg.steps - 1)
    conf = asdict(cfg)
    conf["ranks"] = grid.ctx.size
    conf["topology"] = grid.topology
    rec = MetricsRecord(conf, wall, npts / wall / 1e9, msgs, int(nbytes), checksum)
    if cfg.check:
        rec.max_diff = verify_against_single_rank(cfg, fields)
    return rec


def verify_against_single_rank(cfg: RunConfig, fields=None) -> float:
    """max |gathered multi-rank - single-rank| (0.0 by
    construction; every rank runs the single-rank reference on its GPU)."""
    from . import api
    if fields is None:
        api._FUNCS.clear()
        _g, op, out, dt = _build(cfg)
        op.apply(time_M=cfg.steps - 1, dt=dt, mpi=cfg.mode)
        fields = [f.data_gather() for f in out]
    saved = dict(api._FUNCS)
    api._FUNCS.clear()
    _g, op, out, dt = _build(cfg, comm="self")
    op.apply(time_M=0, dt=dt, mpi="diagonal")
    op.apply(time_m=1, time_M=cfg.steps - 1, dt=dt, mpi="diagonal")
    ref = [f.data_gather() for f in out]
    api._FUNCS.clear()
    api._FUNCS.update(saved)
    return float(max(np.abs(a.astype(np.float64) - b).max() for a, b in zip(fields, ref)))


def to_csv(records: Sequence[MetricsRecord]) -> str:
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=CSV_COLUMNS)
    w.writeheader()
    for r in records:
        w.writerow(r.row())
    return buf.getvalue()


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--kernel", default="acoustic",
                    choices=["acoustic", "damped", "diffusion", "tti", "elastic", "visco"])
    ap.add_argument("--shape", default="64,64,64")
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--tn", type=int, default=20)
    ap.add_argument("--topology", default=None)
    ap.add_argument("--mode", default=os.environ.get("STENCIL_DMP_MODE", "diagonal"))
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--json", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--dump-plan", action="store_true")
    ap.add_argument("--ranks", type=int, default=None,
                    help="expected number of ranks (one per GPU, launched by torchrun)")
    ap.add_argument("--transport", default="nvlink",
                    help="halo transport: nvlink (CUDA-IPC peer stores / copy engines); the "
                         "SPEC's inproc/socket CPU transports have no GPU counterpart")
    a = ap.parse_args(argv)
    if a.transport != "nvlink":
        ap.error(f"transport {a.transport!r} is not available on the GPU path (use nvlink)")
    cfg = RunConfig(kernel=a.kernel, shape=tuple(int(x) for x in a.shape.split(",")), sdo=a.so,
                    steps=a.tn, mode=a.mode, check=a.check, seed=a.seed,
                    topology=tuple(int(x) for x in a.topology.split(",")) if a.topology else None)
    from .dist import context
    ctx = context()
    if a.ranks is not None and a.ranks != ctx.size:
        ap.error(f"--ranks {a.ranks} but {ctx.size} rank(s) were launched "
                 "(torchrun --nproc-per-node sets the rank count)")
    if a.dump_plan:
        _g, op, _o, _dt = _build(cfg)
        if ctx.rank == 0:
            print(op.dump(cfg.mode))
        return 0
    rec = run_benchmark(cfg)
    if ctx.rank == 0:
        text = json.dumps(rec.row()) if a.json else to_csv([rec])
        print(text)
        if a.out:
            with open(a.out, "w") as f:
                f.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
