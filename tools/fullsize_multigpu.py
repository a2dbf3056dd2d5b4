"""Multi-GPU == single-GPU, bitwise, at BASELINE sizes (C2: 1024^3 per GPU;
C4 elastic 1024^3 global; TTI / visco at the largest size a single GPU holds).

    torchrun --nproc-per-node N tools/fullsize_multigpu.py [--steps 20] [--mode full]

Every rank runs the decomposed problem and, on its own GPU, the same global
problem on a one-rank grid; each rank hashes its owned box in both runs
(order-independent integer hash of the fp32 bit patterns) and rank 0 prints
one JSON line.  Equal hashes on every rank = bitwise-equal wavefields.
"""
import argparse
import gc
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_13094_b200 import Grid, Operator  # noqa: E402
from paper_2312_13094_b200 import api  # noqa: E402
from paper_2312_13094_b200 import kernels as KD  # noqa: E402
from paper_2312_13094_b200 import symbolics as S  # noqa: E402
from paper_2312_13094_b200.dist import context  # noqa: E402

TOPOS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (4, 2, 1)}


def bit_hash(t):
    """Order-independent 64-bit hash of the fp32 bit patterns of ``t`` (with
    a position weight, so permutations differ)."""
    b = t.contiguous().view(torch.int32).reshape(-1).to(torch.int64)
    idx = torch.arange(b.numel(), device=b.device, dtype=torch.int64)
    w = idx * 2654435761 + 97531
    return int(((b + 0x9E3779B9) * w).sum())


def run(grid, tag, steps, mode, kernel):
    """Returns (fields to compare, receiver function or None)."""
    if kernel == "acoustic":
        kd = KD.acoustic_model(grid, so=8, name=f"u_{tag}")
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        ext = grid.extent
        src = KD.point_source(grid, [tuple(0.5 * e + 3.7 for e in ext)], steps, dt, f0=0.02,
                              name=f"src_{tag}")
        rec = KD.receiver_line(grid, 64, steps, name=f"rec_{tag}")
        op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
        out = [u]
    else:
        so = 16 if kernel == "visco" else 8
        kd = {"tti": KD.tti_model, "elastic": KD.elastic_model,
              "visco": KD.viscoelastic_model}[kernel](grid, so=so)
        ext = grid.extent
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2 if kernel == "tti" else 0.1)))
        tgt = kd.fields["p"] if kernel == "tti" else kd.fields["txx"]
        src = KD.point_source(grid, [tuple(0.5 * e + 3.7 for e in ext)], steps, dt, f0=0.02,
                              name=f"src_{tag}")
        rec = KD.receiver_line(grid, 64, steps, name=f"rec_{tag}")
        obs = kd.fields["p"] if kernel == "tti" else kd.fields["vz"]
        op = Operator([kd, src.inject(tgt.forward, expr=src * S.DT), rec.interpolate(obs)])
        names = ["p", "r"] if kernel == "tti" else list(KD.VNAMES + KD.TNAMES)
        out = [kd.fields[n] for n in names]
    op.apply(time_M=steps - 1, dt=dt, mpi=mode)
    return out, rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--mode", default="full")
    ap.add_argument("--kernel", default="acoustic", choices=["acoustic", "tti", "elastic", "visco"])
    ap.add_argument("--shape", default=None, help="global shape (default n x topology)")
    a = ap.parse_args()
    ctx = context()
    N = ctx.size
    topo = TOPOS[N]
    shape = tuple(a.n * p for p in topo)
    if a.shape:
        shape = tuple(int(x) for x in a.shape.split(","))
    h = 10.0
    g = Grid(shape, tuple(h * (s - 1) for s in shape), topology=topo)
    fields, rec = run(g, "dist", a.steps, a.mode, a.kernel)
    ext = g.local_extent
    mine = [bit_hash(f._domain_view(f._latest)) for f in fields]
    traces = rec.data.copy()
    del fields
    api._FUNCS.clear()
    gc.collect()
    torch.cuda.empty_cache()
    g1 = Grid(shape, tuple(h * (s - 1) for s in shape), comm="self")
    fields1, rec1 = run(g1, "single", a.steps, a.mode, a.kernel)
    box = tuple(slice(lo, hi) for lo, hi in ext)
    ref = [bit_hash(f._domain_view(f._latest)[box]) for f in fields1]
    res = ctx.allgather({"rank": ctx.rank, "box": ext, "hash": mine, "hash_single": ref,
                         "equal": mine == ref})
    tr_equal = bool(np.array_equal(traces, rec1.data))
    if ctx.rank == 0:
        print(json.dumps({"kernel": a.kernel, "shape": shape, "topology": topo, "mode": a.mode,
                          "steps": a.steps,
                          "ranks": res, "all_equal": all(r["equal"] for r in res),
                          "traces_equal": tr_equal}), flush=True)
    return 0 if all(r["equal"] for r in res) and tr_equal else 1


if __name__ == "__main__":
    sys.exit(main())
