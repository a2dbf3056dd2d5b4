"""One acoustic shot (BASELINE C1-style): layered velocity, absorbing layer,
Ricker source, line of receivers, on one or more B200s.

    python examples/acoustic_shot.py --size 256 --nt 200 --so 8
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 examples/acoustic_shot.py --size 512
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_13094_b200 import Grid, Operator, kernels as KD, symbolics as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=256, help="grid points per axis")
ap.add_argument("--nt", type=int, default=200)
ap.add_argument("--so", type=int, default=8)
ap.add_argument("--nbl", type=int, default=20, help="absorbing layer width (0: none)")
ap.add_argument("--mode", default="full")
a = ap.parse_args()

n = a.size
grid = Grid((n, n, n), (10.0 * (n - 1),) * 3)
kd = (KD.damped_acoustic_model(grid, so=a.so, nbl=a.nbl) if a.nbl > 0
      else KD.acoustic_model(grid, so=a.so))
u, m = kd.fields["u"], kd.fields["m"]
dt = float(np.float32(KD.critical_dt(4.5, grid.spacing)))
ext = grid.extent
src = KD.point_source(grid, [(0.5 * ext[0] + 3.3, 0.5 * ext[1] - 2.1, 0.04 * ext[2])], a.nt, dt)
rec = KD.receiver_line(grid, 256, a.nt)
op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
first = op.apply(time_M=a.nt - 1, dt=dt, mpi=a.mode)  # builds the plan, captures graphs
u.data[...] = 0.0  # same shot again on the built plan (steady state)
summary = op.apply(time_M=a.nt - 1, dt=dt, mpi=a.mode)
if grid.ctx.rank == 0:
    print(f"{a.nt} steps of {n}^3 SO-{a.so} on {grid.ctx.size} GPU(s), topology "
          f"{grid.topology}, mode {a.mode}: {summary['gpts_s']:.1f} GPts/s "
          f"(first apply incl. plan build: {first['gpts_s']:.1f})")
    e = np.square(rec.data.astype(np.float64)).sum(0)
    print(f"receiver trace energy: max {e.max():.3e} at receiver {int(e.argmax())}, "
          f"{int((e > 0).sum())} of {e.size} receivers non-zero")
