"""ORACLE (test infrastructure) — kernel families as simulated-rank problems.

Each builder takes fp32-bound parameters (numpy float32 arrays / scalars,
the SAME values handed to the GPU plan) and returns a problem for
``oracle.runtime.Simulation``.  Arithmetic is fp64.
"""
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import decomp as D
from . import stencils as K


@dataclass
class Phase:
    exchange: List[Tuple[str, int]]
    radius: Tuple[int, ...]
    compute: Callable
    before: Optional[Callable] = None
    after: Optional[Callable] = None


@dataclass
class Problem:
    fields: dict
    halo: Tuple[int, ...]
    phases: List[Phase] = field(default_factory=list)


@dataclass
class SparseSpec:
    """Sources (inject) and receivers (interpolate) of one problem.

    ``src_amp[time, pid]`` fp32; ``scale`` ('m', C) -> C/m[node], or
    (None, C) -> C.  Receivers sample ``rec_field`` at tshift 0 (after the
    exchange, before the update — halo fresh), sources are added to the
    updated buffer (tshift +1) after compute."""
    grid_shape: tuple
    spacing: tuple
    src_coords: np.ndarray = None
    src_amp: np.ndarray = None
    src_field: str = "u"
    scale: tuple = (None, 1.0)
    rec_coords: np.ndarray = None
    rec_field: str = "u"


def _sparse_hooks(sim_shape, dims, sp: SparseSpec):
    """Before/after callables implementing SPEC.md:507-525 per rank."""
    nd = len(sp.grid_shape)
    extent = tuple(h * (n - 1) for h, n in zip(sp.spacing, sp.grid_shape))

    def owners(c):
        return D.owners_of_point(c, sp.grid_shape, extent, dims)

    src = []
    if sp.src_coords is not None:
        for pid, c in enumerate(np.asarray(sp.src_coords, dtype=np.float64)):
            corners, w = K.trilinear(c, sp.spacing, sp.grid_shape)
            src.append((pid, corners, w, owners(c)))
    rec = []
    if sp.rec_coords is not None:
        for pid, c in enumerate(np.asarray(sp.rec_coords, dtype=np.float64)):
            corners, w = K.trilinear(c, sp.spacing, sp.grid_shape)
            rec.append((pid, corners, w, owners(c)))

    def before(sim, rk, time):
        if not rec:
            return
        u = rk.buf(sp.rec_field, time, 0)
        row = sim.traces.setdefault(time, np.zeros(len(rec)))
        for pid, corners, w, own in rec:
            if own[0] == rk.rank:
                row[pid] = K.interpolate(u, rk.halo, [e[0] for e in rk.ext], corners, w)

    def after(sim, rk, time):
        if not src:
            return
        nodes = {}
        for pid, corners, w, own in src:
            if rk.rank not in own:
                continue
            for c, wi in zip(corners, w):
                if all(e0 <= ci < e1 for ci, (e0, e1) in zip(c, rk.ext)):
                    nodes.setdefault(c, []).append((pid, wi))
        if not nodes:
            return
        u = rk.buf(sp.src_field, time, 1)
        scale = None
        if sp.scale[0] == "m":
            scale = (sp.scale[1], rk.buf("m", time, 0))
        elif sp.scale[1] != 1.0:
            scale = (sp.scale[1], None)
        amps = np.asarray(sp.src_amp[time], dtype=np.float64)
        K.inject(u, rk.halo, [e[0] for e in rk.ext], nodes, amps, scale)

    return before, after


def star(nd, so, coeffs, A, B, C, with_m, sparse=None, shape=None, dims=None, halo=None):
    """Acoustic (time_order 2, A,B,C = 2,-1,dt^2) or diffusion
    (time_order 1, 1,0,dt) star stencil, radius so/2 per axis."""
    r = so // 2
    halo = tuple(halo) if halo is not None else (so,) * nd
    fields = {"u": 3 if B != 0.0 else 2}
    if with_m:
        fields["m"] = 1

    def compute(rk, box, time):
        u0 = rk.buf("u", time, 0)
        u2 = rk.buf("u", time, -1) if B != 0.0 else None
        m = rk.buf("m", time, 0) if with_m else None
        K.star_update(u0, u2, m, coeffs, A, B, C, box, rk.buf("u", time, 1))

    before = after = None
    if sparse is not None:
        before, after = _sparse_hooks(shape, dims or (1,) * nd, sparse)
    return Problem(fields, halo, [Phase([("u", 0)], (r,) * nd, compute, before, after)])


def var_star(nd, so, coeffs, with_prev=True, sparse=None, shape=None, dims=None, extra=()):
    """Variable-coefficient star (damped acoustic): static fields A, B, S
    (+ ``extra`` static fields, e.g. m for the source scaling)."""
    r = so // 2
    halo = (so,) * nd
    fields = {"u": 3 if with_prev else 2, "A": 1, "S": 1}
    fields.update({n: 1 for n in extra})
    if with_prev:
        fields["B"] = 1

    def compute(rk, box, time):
        b = lambda n, t=0: rk.buf(n, time, t)
        K.var_star_update(b("u"), b("u", -1) if with_prev else None, b("A"),
                          b("B") if with_prev else None, b("S"), coeffs, box, b("u", 1))

    before = after = None
    if sparse is not None:
        before, after = _sparse_hooks(shape, dims or (1,) * nd, sparse)
    return Problem(fields, halo, [Phase([("u", 0)], (r,) * nd, compute, before, after)])


def rotated(so, d1_c, dt2, sparse=None, shape=None, dims=None):
    """Single-field rotated operator (SPEC tti_gxx_kernel): fields u, m, a*."""
    fields = {"u": 3, "m": 1, "ax": 1, "ay": 1, "az": 1}

    def compute(rk, box, time):
        b = lambda n, t=0: rk.buf(n, time, t)
        K.rot_update(b("u"), b("u", -1), b("m"), (b("ax"), b("ay"), b("az")), d1_c, dt2, box,
                     b("u", 1))

    before = after = None
    if sparse is not None:
        before, after = _sparse_hooks(shape, dims or (1,) * 3, sparse)
    return Problem(fields, (so,) * 3, [Phase([("u", 0)], (so,) * 3, compute, before, after)])


def tti(so, lap_c, d1_c, dt2, sparse=None, shape=None, dims=None):
    halo = (so,) * 3
    fields = {"p": 3, "r": 3, "m": 1, "epsp": 1, "delp": 1, "ax": 1, "ay": 1, "az": 1}

    def compute(rk, box, time):
        b = lambda n, t=0: rk.buf(n, time, t)
        K.tti_update(b("p"), b("p", -1), b("r"), b("r", -1), b("m"), b("epsp"), b("delp"),
                     (b("ax"), b("ay"), b("az")), lap_c, d1_c, dt2, box,
                     b("p", 1), b("r", 1))

    before = after = None
    if sparse is not None:
        before, after = _sparse_hooks(shape, dims or (1,) * 3, sparse)
    return Problem(fields, halo, [Phase([("p", 0), ("r", 0)], (so,) * 3, compute, before, after)])


VNAMES = ("vx", "vy", "vz")
TNAMES = ("txx", "tyy", "tzz", "txy", "txz", "tyz")
RNAMES = ("rxx", "ryy", "rzz", "rxy", "rxz", "ryz")


def elastic(so, sc, dt, visco=False, sparse=None, shape=None, dims=None, collocated=False):
    """Staggered velocity-stress or its single-
    relaxation viscoelastic extension.  Two phases,
    two exchanges per step: stress before v, v before stress."""
    r = so // 2
    halo = (so,) * 3
    fields = {n: 2 for n in VNAMES + TNAMES}
    if visco:
        fields.update({n: 2 for n in RNAMES})
        fields.update({"b": 1, "l2m": 1, "mus": 1, "its": 1})
    else:
        fields.update({"b": 1, "lam": 1, "mu": 1})

    def phase_v(rk, box, time):
        b = lambda n, t=0: rk.buf(n, time, t)
        K.velocity_update([b(n) for n in VNAMES], [b(n) for n in TNAMES], b("b"), sc, dt,
                          box, [b(n, 1) for n in VNAMES], collocated)

    def phase_t(rk, box, time):
        b = lambda n, t=0: rk.buf(n, time, t)
        if visco:
            K.visco_stress_update([b(n, 1) for n in VNAMES], [b(n) for n in TNAMES],
                                  [b(n) for n in RNAMES], b("l2m"), b("mus"), b("its"),
                                  sc, dt, box, [b(n, 1) for n in TNAMES],
                                  [b(n, 1) for n in RNAMES])
        else:
            K.stress_update([b(n, 1) for n in VNAMES], [b(n) for n in TNAMES], b("lam"),
                            b("mu"), sc, dt, box, [b(n, 1) for n in TNAMES], collocated)

    before = after = None
    if sparse is not None:
        before, after = _sparse_hooks(shape, dims or (1,) * 3, sparse)
    return Problem(fields, halo, [
        Phase([(n, 0) for n in TNAMES], (r,) * 3, phase_v, before, None),
        Phase([(n, 1) for n in VNAMES], (r,) * 3, phase_t, None, after),
    ])
