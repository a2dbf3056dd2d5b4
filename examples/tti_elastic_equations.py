"""The paper's TTI pair and the SPEC's collocated elastic system written as
update equations with the public API, exactly as a Devito user would, and
run on one or more B200s.  The Operator recognises the equations (exact
rational probing against the families' templates) and runs the matching
sm_100a kernels: TTI SO <= 6 on the single-pass kernel, SO >= 8 on two
passes; elastic on the collocated velocity / stress pair.

    python examples/tti_elastic_equations.py --size 128 --nt 40 --so 8
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 examples/tti_elastic_equations.py
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_13094_b200 import (Eq, Function, Grid, Operator, TimeFunction,  # noqa: E402
                                   solve, symbolics as S)

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=128)
ap.add_argument("--nt", type=int, default=40)
ap.add_argument("--so", type=int, default=8)
ap.add_argument("--mode", default="full")
a = ap.parse_args()

n, so = a.size, a.so
h = 10.0
grid = Grid((n, n, n), (h * (n - 1),) * 3)
rng = np.random.default_rng(0)

# ---- TTI: m p.dt2 = epsp H0 p + delp Gzz r, m r.dt2 = delp H0 p + Gzz r
p = TimeFunction(name="p", grid=grid, space_order=so, time_order=2)
r = TimeFunction(name="r", grid=grid, space_order=so, time_order=2)
m = Function(name="m", grid=grid, space_order=so)
epsp = Function(name="epsp", grid=grid, space_order=so)
delp = Function(name="delp", grid=grid, space_order=so)
ax, ay, az = (Function(name=f"a{c}", grid=grid, space_order=so) for c in "xyz")
vp = 2.5
m.data[...] = 1.0 / vp ** 2
eps, dlt = 0.2, 0.08
epsp.data[...] = 1.0 + 2.0 * eps
delp.data[...] = math.sqrt(1.0 + 2.0 * dlt)
th, ph = math.radians(30.0), math.radians(20.0)
ax.data[...] = math.sin(th) * math.cos(ph)
ay.data[...] = math.sin(th) * math.sin(ph)
az.data[...] = math.cos(th)


def gzz(f):
    """sum_i D_i(a_i sum_j a_j D_j f): nested centred first derivatives."""
    a3 = (ax, ay, az)
    inner = S.add(*(S.mul(a3[j].at(), f.d(j)) for j in range(3)))
    return S.add(*(S.Deriv(S.mul(a3[i].at(), inner), i, 1) for i in range(3)))


h0 = p.laplace - gzz(p)
eq_p = Eq(p.forward, solve(Eq(m * p.dt2, epsp * h0 + delp * gzz(r)), p.forward))
eq_r = Eq(r.forward, solve(Eq(m * r.dt2, delp * h0 + gzz(r)), r.forward))
init = np.zeros((n, n, n), dtype=np.float32)
c = n // 2
init[c - 2:c + 3, c - 2:c + 3, c - 2:c + 3] = 1.0
p.data[...] = init
r.data[...] = init
dt = 0.2 * h / vp
tti = Operator([eq_p, eq_r])
s1 = tti.apply(time_M=a.nt - 1, dt=dt, mpi=a.mode)
if grid.ctx.rank == 0:
    print(f"TTI from equations -> {type(tti.kernels[0]).__name__}: {a.nt} steps of {n}^3 "
          f"SO-{so}, {grid.ctx.size} GPU(s), mode {a.mode}: {s1['gpts_s']:.1f} GPts/s")
pg = p.data_gather()
if grid.ctx.rank == 0:
    print(f"  |p| = {np.linalg.norm(pg):.4e}, max {np.abs(pg).max():.4e}")

# ---- collocated elastic: v.dt = b div(tau), tau.dt = lam tr(grad v) I + mu (grad v + grad v^T)
v = [TimeFunction(name=f"v{c}", grid=grid, space_order=so, time_order=1) for c in "xyz"]
names = ("txx", "tyy", "tzz", "txy", "txz", "tyz")
t = {nm: TimeFunction(name=nm, grid=grid, space_order=so, time_order=1) for nm in names}
b = Function(name="b", grid=grid, space_order=so)
lam = Function(name="lam", grid=grid, space_order=so)
mu = Function(name="mu", grid=grid, space_order=so)
rho, vs = 2.0, vp / math.sqrt(3.0)
b.data[...] = 1.0 / rho
lam.data[...] = rho * (vp ** 2 - 2.0 * vs ** 2)
mu.data[...] = rho * vs ** 2
T = [[t["txx"], t["txy"], t["txz"]], [t["txy"], t["tyy"], t["tyz"]], [t["txz"], t["tyz"], t["tzz"]]]
eqs = [Eq(v[i].forward, solve(Eq(v[i].dt, b * S.add(*(T[i][j].d(j) for j in range(3)))),
                              v[i].forward)) for i in range(3)]
dv = lambda i, j: S.Deriv(v[i].forward, j, 1)  # noqa: E731
tr = S.add(*(dv(k, k) for k in range(3)))
for i, nm in enumerate(("txx", "tyy", "tzz")):
    eqs.append(Eq(t[nm].forward, solve(Eq(t[nm].dt, lam * tr + 2 * mu * dv(i, i)),
                                       t[nm].forward)))
for (i, j), nm in (((0, 1), "txy"), ((0, 2), "txz"), ((1, 2), "tyz")):
    eqs.append(Eq(t[nm].forward, solve(Eq(t[nm].dt, mu * (dv(i, j) + dv(j, i))), t[nm].forward)))
for nm in ("txx", "tyy", "tzz"):
    t[nm].data[...] = init
el = Operator(eqs)
s2 = el.apply(time_M=a.nt - 1, dt=0.1 * h / vp, mpi=a.mode)
if grid.ctx.rank == 0:
    kinds = [f"{type(k).__name__}({k.kind}, collocated={k.collocated})" for k in el.kernels]
    print(f"elastic from equations -> {kinds}: {s2['gpts_s']:.1f} GPts/s")
vz = v[2].data_gather()
if grid.ctx.rank == 0:
    print(f"  |vz| = {np.linalg.norm(vz):.4e}")
