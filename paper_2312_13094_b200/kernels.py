"""Kernel-family definitions and synthetic models (SPEC.md:560-623,
PAPER.md:964-1097).

Each ``*_model`` builds the fields of one family on a Grid, fills
synthetic material parameters on the device (decomposition-independent:
every value is a pure function of its global index) and returns a
``KernelDef`` whose ``kernels`` the Operator executes.  The acoustic and
diffusion families are ALSO recognised from user-written equations
(``Operator([Eq(u.forward, solve(m*u.dt2 - u.laplace, u.forward))])``).

Families (B200 kernels in csrc/):
  acoustic   u1 = 2u - u_prev + dt^2/m lap(u)                  star.cu
  diffusion  u1 = u + dt lap(u)                                 star.cu
  tti        two-field pseudo-acoustic, rotated nested D(aD)    tti.cu
  elastic    staggered velocity-stress (Virieux)                elastic.cu
  visco      + single-relaxation memory variables               elastic.cu
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import compiler as CP
from . import symbolics as S
from .api import (Eq, Function, Grid, Operator, SparseTimeFunction, TimeFunction, ricker,
                  solve)


@dataclass
class KernelDef:
    name: str
    fields: Dict[str, object]
    kernels: List[object]
    equations: List[object] = field(default_factory=list)
    bytes_per_point: int = 16
    working_set: int = 0  # arrays touched per step


# ---------------------------------------------------------------------------
# deterministic synthetic noise: pure function of the global index


def hash_uniform(gx, gy, gz, seed: int = 0):
    """U[0,1) from global indices (torch or numpy int64 arrays)."""
    h = (gx * 73856093) ^ (gy * 19349663) ^ (gz * 83492791) ^ (seed * 2654435761)
    h = h & 0xFFFFFFFF
    h = (h ^ (h >> 16)) * 0x45D9F3B & 0xFFFFFFFF
    h = (h ^ (h >> 16)) * 0x45D9F3B & 0xFFFFFFFF
    h = h ^ (h >> 16)
    return (h & 0xFFFFFF) / float(1 << 24)


def _vp_law(gx, gy, gz, nz, vmin=1.5, vmax=4.5, noise=0.01, seed=0):
    """vp(z) = vmin + (vmax - vmin) k/(nz-1), times (1 + noise U(-1,1))
    (SURVEY.md §8d C1 law), fp64, from global index grids."""
    base = vmin + (vmax - vmin) * gz.double() / max(nz - 1, 1)
    u = hash_uniform(gx, gy, gz, seed).double()
    return base * (1.0 + noise * (2.0 * u - 1.0))


def _fill(fns: Sequence[Function], f, max_points: int = 1 << 27):
    """Write ``f(gx, gy, gz)`` (a tuple of fp64 tensors, one per field) into
    the DOMAIN of each static field, slab by slab along x so the fp64 /
    int64 temporaries stay bounded (a 1536^3 TTI rank would otherwise need
    tens of GB of index grids)."""
    import torch
    ref = fns[0]
    ext = list(ref.grid.local_extent)
    dev = ref.storage.device
    while len(ext) < 3:
        ext.append((0, 1))
    (xa, xb), (ya, yb), (za, zb) = ext
    gy_ = torch.arange(ya, yb, device=dev, dtype=torch.int64)
    gz_ = torch.arange(za, zb, device=dev, dtype=torch.int64)
    chunk = max(1, max_points // max(1, (yb - ya) * (zb - za)))
    views = [fn._domain_view(0) for fn in fns]
    for x0 in range(xa, xb, chunk):
        x1 = min(xb, x0 + chunk)
        gx_ = torch.arange(x0, x1, device=dev, dtype=torch.int64)
        gx, gy, gz = torch.meshgrid(gx_, gy_, gz_, indexing="ij")
        vals = f(gx, gy, gz)
        for v, val in zip(views, vals):
            v[x0 - xa:x1 - xa].copy_(val.reshape(v[x0 - xa:x1 - xa].shape).to(v.dtype))
    for fn in fns:
        fn._version += 1


def layered_vp(fn: Function, vmin=1.5, vmax=4.5, noise=0.01, seed=0):
    """:func:`_vp_law` on this rank's DOMAIN (device tensor, DOMAIN shape;
    small grids only, the models fill slab by slab)."""
    import torch
    ext = list(fn.grid.local_extent)
    while len(ext) < 3:
        ext.append((0, 1))
    dev = fn.storage.device
    gx, gy, gz = torch.meshgrid(*[torch.arange(a, b, device=dev, dtype=torch.int64)
                                  for a, b in ext], indexing="ij")
    return _vp_law(gx, gy, gz, fn.grid.shape[-1], vmin, vmax, noise, seed)


def layered_vp_numpy(shape, vmin=1.5, vmax=4.5, noise=0.01, seed=0):
    """Host twin of :func:`layered_vp` over the global grid (oracle input)."""
    nd = len(shape)
    idx = np.meshgrid(*[np.arange(n, dtype=np.int64) for n in shape], indexing="ij")
    while len(idx) < 3:
        idx.append(np.zeros_like(idx[0]))
    gx, gy, gz = idx
    nz = shape[-1]
    base = vmin + (vmax - vmin) * gz.astype(np.float64) / max(nz - 1, 1)
    u = hash_uniform(gx, gy, gz, seed).astype(np.float64)
    return base * (1.0 + noise * (2.0 * u - 1.0))


def _set_domain(fn: Function, values):
    """Write a DOMAIN-shaped device tensor into buffer 0 of a static field."""
    v = fn._domain_view(0)
    v.copy_(values.reshape(v.shape).to(v.dtype))
    fn._version += 1


def critical_dt(vmax: float, spacing: Sequence[float], courant: float = 0.38) -> float:
    """CFL guard: dt = courant * min(h) / vmax."""
    return courant * min(spacing) / vmax


# ---------------------------------------------------------------------------
# acoustic / diffusion


def acoustic_model(grid: Grid, so: int = 8, vp=None, name: str = "u") -> KernelDef:
    """Isotropic acoustic:
    ``m u.dt2 - lap u = src``, m = 1/vp^2 (fp32)."""
    import torch
    u = TimeFunction(name=name, grid=grid, space_order=so, time_order=2)
    m = Function(name=f"m_{name}", grid=grid, space_order=so)
    nz = grid.shape[-1]
    if vp is None:
        _fill([m], lambda gx, gy, gz: (1.0 / _vp_law(gx, gy, gz, nz) ** 2,))
    else:
        _set_domain(m, (1.0 / vp ** 2).float())
    eq = Eq(u.forward, solve(m * u.dt2 - u.laplace, u.forward))
    return KernelDef("acoustic", {"u": u, "m": m}, [], [eq], bytes_per_point=16, working_set=4)


def damping_profile(n: int, nbl: int, h: float) -> np.ndarray:
    """1D absorbing-layer profile along one axis (the paper's ABC layer,
    PAPER.md:695): zero inside, (1.5 ln(1000) / nbl) (p - sin(2 pi p) / 2 pi) / h
    at relative depth p into a layer of nbl points at either end."""
    i = np.arange(n, dtype=np.float64)
    depth = np.maximum(np.maximum(nbl - i, i - (n - 1 - nbl)), 0.0) / max(nbl, 1)
    coeff = 1.5 * math.log(1000.0) / max(nbl, 1)
    return coeff * (depth - np.sin(2.0 * math.pi * depth) / (2.0 * math.pi)) / h


def damped_acoustic_model(grid: Grid, so: int = 8, nbl: int = 10, vp=None,
                          name: str = "u") -> KernelDef:
    """Acoustic with an absorbing boundary layer, written as the paper's
    operator ``m*u.dt2 - u.laplace + damp*u.dt`` and solved by the reference
    symbolics; runs as the variable-coefficient star family (24 B/pt)."""
    import torch
    u = TimeFunction(name=name, grid=grid, space_order=so, time_order=2)
    m = Function(name=f"m_{name}", grid=grid, space_order=so)
    damp = Function(name=f"damp_{name}", grid=grid, space_order=so)
    nz = grid.shape[-1]
    if vp is None:
        _fill([m], lambda gx, gy, gz: (1.0 / _vp_law(gx, gy, gz, nz) ** 2,))
    else:
        _set_domain(m, (1.0 / vp ** 2).float())
    profs = [torch.from_numpy(damping_profile(n, nbl, h)) for n, h in zip(grid.shape, grid.spacing)]
    while len(profs) < 3:
        profs.append(torch.zeros(1, dtype=torch.float64))

    def law(gx, gy, gz):
        dev = gx.device
        return (profs[0].to(dev)[gx] + profs[1].to(dev)[gy] + profs[2].to(dev)[gz],)

    _fill([damp], law)
    eq = Eq(u.forward, solve(m * u.dt2 - u.laplace + damp * u.dt, u.forward))
    return KernelDef("damped_acoustic", {"u": u, "m": m, "damp": damp}, [], [eq],
                     bytes_per_point=24, working_set=6)


def diffusion_model(grid: Grid, so: int = 2, name: str = "u") -> KernelDef:
    u = TimeFunction(name=name, grid=grid, space_order=so, time_order=1)
    eq = Eq(u.forward, solve(Eq(u.dt, u.laplace), u.forward))
    return KernelDef("diffusion", {"u": u}, [], [eq], bytes_per_point=8, working_set=2)


# ---------------------------------------------------------------------------
# TTI


def tti_model(grid: Grid, so: int = 8, vp=None) -> KernelDef:
    """Two-field TTI with synthetic eps/delta/theta/phi:
    eps = 0.25 k/(nz-1), delta = 0.4 eps, theta = 30 deg + 5 deg U, phi = 20 deg + 5 deg U.
    Bound parameters: epsp = 1 + 2 eps, delp = sqrt(1 + 2 delta),
    a = (sin t cos f, sin t sin f, cos t)."""
    import torch
    if grid.ndims != 3:
        raise ValueError("TTI is 3D")
    p = TimeFunction(name="p", grid=grid, space_order=so, time_order=2)
    r = TimeFunction(name="r", grid=grid, space_order=so, time_order=2)
    m = Function(name="m_tti", grid=grid, space_order=so)
    epsp = Function(name="epsp", grid=grid, space_order=so)
    delp = Function(name="delp", grid=grid, space_order=so)
    a = [Function(name=f"a{c}", grid=grid, space_order=so) for c in "xyz"]
    nz = grid.shape[-1]

    def law(gx, gy, gz):
        eps = 0.25 * gz.double() / max(nz - 1, 1)
        dlt = 0.4 * eps
        th = math.radians(30.0) + math.radians(5.0) * hash_uniform(gx, gy, gz, 11).double()
        ph = math.radians(20.0) + math.radians(5.0) * hash_uniform(gx, gy, gz, 12).double()
        out = (1.0 + 2.0 * eps, torch.sqrt(1.0 + 2.0 * dlt), torch.sin(th) * torch.cos(ph),
               torch.sin(th) * torch.sin(ph), torch.cos(th))
        if vp is None:
            out = (1.0 / _vp_law(gx, gy, gz, nz) ** 2,) + out
        return out

    _fill(([m] if vp is None else []) + [epsp, delp] + a, law)
    if vp is not None:
        _set_domain(m, (1.0 / vp ** 2).float())
    # the system as update equations (reference symbolics); the Operator
    # recognises the pair as the TTI family (compiler.recognise_tti)
    eqs = list(CP.tti_updates(p.spec, r.spec, m.spec, epsp.spec, delp.spec,
                              tuple(f.spec for f in a)))
    fields = {"p": p, "r": r, "m": m, "epsp": epsp, "delp": delp, "ax": a[0], "ay": a[1],
              "az": a[2]}
    return KernelDef("tti", fields, [], eqs, bytes_per_point=48, working_set=12)


def rotated_model(grid: Grid, so: int = 8, vp=None, name: str = "u") -> KernelDef:
    """The SPEC's tti_gxx_kernel: one field, m u_tt = G u
    with the rotated operator G = D^T D built from direction-cosine fields
    (theta, phi as in the TTI model), written with the reference symbolics
    and recognised by the compiler (28 B/pt)."""
    import torch
    if grid.ndims != 3:
        raise ValueError("the rotated operator is 3D")
    u = TimeFunction(name=name, grid=grid, space_order=so, time_order=2)
    m = Function(name=f"m_{name}", grid=grid, space_order=so)
    a = [Function(name=f"a{c}_{name}", grid=grid, space_order=so) for c in "xyz"]
    nz = grid.shape[-1]

    def law(gx, gy, gz):
        th = math.radians(30.0) + math.radians(5.0) * hash_uniform(gx, gy, gz, 11).double()
        ph = math.radians(20.0) + math.radians(5.0) * hash_uniform(gx, gy, gz, 12).double()
        out = (torch.sin(th) * torch.cos(ph), torch.sin(th) * torch.sin(ph), torch.cos(th))
        if vp is None:
            out = (1.0 / _vp_law(gx, gy, gz, nz) ** 2,) + out
        return out

    _fill(([m] if vp is None else []) + a, law)
    if vp is not None:
        _set_domain(m, (1.0 / vp ** 2).float())
    eq = CP.rotated_update(u.spec, m.spec, tuple(f.spec for f in a))
    return KernelDef("rotated", {"u": u, "m": m, "ax": a[0], "ay": a[1], "az": a[2]}, [], [eq],
                     bytes_per_point=28, working_set=7)


# ---------------------------------------------------------------------------
# staggered elastic / viscoelastic

VNAMES = ("vx", "vy", "vz")
TNAMES = ("txx", "tyy", "tzz", "txy", "txz", "tyz")
RNAMES = ("rxx", "ryy", "rzz", "rxy", "rxz", "ryz")


def _elastic_materials(gx, gy, gz, nz):
    """vp law as acoustic, vs = vp/sqrt(3), rho = 0.31 (1000 vp)^0.25 (g/cc,
    Gardner), lam = rho (vp^2 - 2 vs^2), mu = rho vs^2, b = 1/rho."""
    vp = _vp_law(gx, gy, gz, nz)
    vs = vp / math.sqrt(3.0)
    rho = 0.31 * (1000.0 * vp) ** 0.25
    return vp, vs, rho


def elastic_model(grid: Grid, so: int = 8, collocated: bool = False) -> KernelDef:
    """Velocity-stress elastic: the paper's staggered (Virieux) grid, or with
    ``collocated=True`` the SPEC's elastic_kernel (centred
    first derivatives on one grid)."""
    if grid.ndims != 3:
        raise ValueError("elastic is 3D")
    v = [TimeFunction(name=n, grid=grid, space_order=so, time_order=1) for n in VNAMES]
    t = [TimeFunction(name=n, grid=grid, space_order=so, time_order=1) for n in TNAMES]
    b = Function(name="b_el", grid=grid, space_order=so)
    lam = Function(name="lam", grid=grid, space_order=so)
    mu = Function(name="mu", grid=grid, space_order=so)
    nz = grid.shape[-1]

    def law(gx, gy, gz):
        vp, vs, rho = _elastic_materials(gx, gy, gz, nz)
        return 1.0 / rho, rho * (vp ** 2 - 2.0 * vs ** 2), rho * vs ** 2

    _fill([b, lam, mu], law)
    fields = {f.name: f for f in v + t}
    fields.update({"b": b, "lam": lam, "mu": mu})
    if collocated:
        # the SPEC's elastic_kernel as nine update equations (reference
        # symbolics); recognised as the collocated pair of phases
        # (compiler.recognise_elastic)
        eqs = CP.elastic_updates(tuple(f.spec for f in v), tuple(f.spec for f in t),
                                 b.spec, lam.spec, mu.spec)
        return KernelDef("elastic_collocated", fields, [], eqs, bytes_per_point=120,
                         working_set=21)
    # staggered (Virieux) offsets are half-integer: not expressible in the
    # reference symbolics (integer offsets) -> kernel descriptors
    kv = CP.StaggeredPhase("v", tuple(f.spec for f in v), tuple(f.spec for f in t),
                           (b.spec,), so=so)
    kt = CP.StaggeredPhase("t", tuple(f.spec for f in v), tuple(f.spec for f in t),
                           (lam.spec, mu.spec), so=so)
    return KernelDef("elastic", fields, [kv, kt], bytes_per_point=120, working_set=21)


def viscoelastic_model(grid: Grid, so: int = 16, qp: float = 100.0, qs: float = 50.0,
                       f0: float = 0.010) -> KernelDef:
    """Single relaxation.  tau_sigma / tau_eps from Q
    at f0 (Blanch-style single-SLS: tau_sigma = (sqrt(1+1/Q^2) - 1/Q) /
    (2 pi f0), tau_eps = 1/((2 pi f0)^2 tau_sigma)); bound per point:
    l2m = (lam + 2 mu) tau_ep/tau_s, mus = mu tau_es/tau_s, its = 1/tau_s."""
    if grid.ndims != 3:
        raise ValueError("viscoelastic is 3D")
    v = [TimeFunction(name=n, grid=grid, space_order=so, time_order=1) for n in VNAMES]
    s = [TimeFunction(name=n, grid=grid, space_order=so, time_order=1) for n in TNAMES]
    r = [TimeFunction(name=n, grid=grid, space_order=so, time_order=1) for n in RNAMES]
    b = Function(name="b_ve", grid=grid, space_order=so)
    l2m = Function(name="l2m", grid=grid, space_order=so)
    mus = Function(name="mus", grid=grid, space_order=so)
    its = Function(name="its", grid=grid, space_order=so)
    w0 = 2.0 * math.pi * f0

    def taus(q):
        ts = (math.sqrt(1.0 + 1.0 / q ** 2) - 1.0 / q) / w0
        te = 1.0 / (w0 * w0 * ts)
        return ts, te

    ts_p, te_p = taus(qp)
    ts_s, te_s = taus(qs)
    t_sigma = ts_p  # one stress relaxation time for P and S (PAPER.md Table)
    nz = grid.shape[-1]

    def law(gx, gy, gz):
        vp, vs, rho = _elastic_materials(gx, gy, gz, nz)
        lam = rho * (vp ** 2 - 2.0 * vs ** 2)
        mu_ = rho * vs ** 2
        return (1.0 / rho, (lam + 2.0 * mu_) * (te_p / t_sigma), mu_ * (te_s / t_sigma),
                rho * 0.0 + 1.0 / t_sigma)

    _fill([b, l2m, mus, its], law)
    kv = CP.StaggeredPhase("v", tuple(f.spec for f in v), tuple(f.spec for f in s),
                           (b.spec,), so=so)
    kt = CP.StaggeredPhase("visco_t", tuple(f.spec for f in v), tuple(f.spec for f in s),
                           (l2m.spec, mus.spec, its.spec), mem=tuple(f.spec for f in r), so=so)
    fields = {f.name: f for f in v + s + r}
    fields.update({"b": b, "l2m": l2m, "mus": mus, "its": its})
    return KernelDef("visco", fields, [kv, kt], bytes_per_point=172, working_set=37)


# ---------------------------------------------------------------------------
# sources / receivers


def point_source(grid: Grid, coords, nt: int, dt: float, f0: float = 0.010,
                 name: str = "src") -> SparseTimeFunction:
    """Ricker point source (f0 in kHz with dt in ms)."""
    src = SparseTimeFunction(name, grid, npoint=len(coords), nt=nt, coordinates=coords)
    t = np.arange(nt) * dt
    src.data[:] = np.float32(ricker(f0, t, 1.0 / f0))[:, None]
    return src


def receiver_line(grid: Grid, nrec: int, nt: int, depth_frac: float = 0.0079,
                  name: str = "rec") -> SparseTimeFunction:
    ext = grid.extent
    xs = np.linspace(5.0 * ext[0] / 2550.0, ext[0] - 5.0 * ext[0] / 2550.0, nrec)
    coords = np.zeros((nrec, grid.ndims))
    coords[:, 0] = xs
    if grid.ndims == 3:
        coords[:, 1] = 0.5 * ext[1] - 0.00019 * ext[1]
        coords[:, 2] = depth_frac * ext[2]
    else:
        coords[:, 1] = depth_frac * ext[1]
    return SparseTimeFunction(name, grid, npoint=nrec, nt=nt, coordinates=coords)
