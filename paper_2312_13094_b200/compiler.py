"""Operator compiler: kernel-family recognition, HaloSpot detection and
optimisation, and lowering of the three exchange modes to an ExecPlan.

Implements the SPEC's ``compiler`` module for the B200
path:

* ``recognise`` — each solved update (``StencilEquation``) is matched
  EXACTLY against a kernel-family template by rational probing (the
  ``rational_probe`` idea of test_symbolics.py:152-164): the rhs is linear in
  the field accesses, so its coefficients are extracted with ``eval_exact``
  at random rational bindings and checked against the family's algebraic
  form.  Unrecognised equations raise — there is no generic/CPU fallback.
* ``halo_phases`` — per-kernel read radii (``build_clusters``,
  SPEC.md:328-336), HaloSpots placed before the first dependent kernel and
  optimised: drop (field not dirty), merge (adjacent spots), hoist
  (read-only coefficient fields exchanged once before the time loop)
  (``optimize_halospots``).
* ``ExecPlan`` — ``lower_mode``: basic = axis-sequenced
  face exchange then DOMAIN; diagonal = single-step exchange then DOMAIN;
  full = post, CORE, wait, OWNED slabs (Listing 8).  The same ExecPlan is
  instantiated per rank into native actions (``runtime_plan.py``).
"""
from __future__ import annotations

import os
import random
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

from . import symbolics as S

MODES = ("basic", "diagonal", "full")
_MODE_ALIASES = {"1": "basic", "basic": "basic", "diag": "diagonal", "diag2": "diagonal",
                 "diagonal": "diagonal", "full": "full", "overlap": "full"}


class CompilerError(S.SymbolicsError):
    """Equation not recognised / plan cannot be built."""


def normalise_mode(mode) -> str:
    m = _MODE_ALIASES.get(str(mode).lower())
    if m is None:
        raise CompilerError(f"unknown mpi mode {mode!r}; expected basic | diagonal | full")
    return m


# ---------------------------------------------------------------------------
# Kernel families


@dataclass
class StarKernel:
    """u1 = A u0 + B u2 + S L(u0),  S = c * dt^p * m^q  (q in {0, -1}).

    Acoustic: (A, B, c, p, q) = (2, -1, 1, 2, -1) — the reference's solved
    ``m*u.dt2 - u.laplace`` (symbolics.py:629-674); diffusion: (1, 0, 1, 1, 0)
    — ``Eq(u.dt, u.laplace)``."""

    u: S.FieldSpec
    m: Optional[S.FieldSpec]
    A: Fraction
    B: Fraction
    c: Fraction
    p: int
    q: int
    weights: Tuple[Tuple[Fraction, ...], ...]  # per axis, centre-out w_k (k = 0..r)
    family: str = "star"

    @property
    def radius(self) -> Tuple[int, ...]:
        return tuple(len(w) - 1 for w in self.weights)

    def reads(self):
        """(field, tshift, radius per axis) read by the kernel."""
        out = [(self.u, 0, self.radius)]
        if self.B != 0:
            out.append((self.u, -1, (0,) * len(self.radius)))
        if self.m is not None:
            out.append((self.m, 0, (0,) * len(self.radius)))
        return out

    def writes(self):
        return [(self.u, 1)]

    @property
    def bytes_per_point(self) -> int:
        """Algorithmic HBM bytes per updated point (each array once)."""
        return 4 * (2 + (1 if self.B != 0 else 0) + (1 if self.m is not None else 0))


@dataclass(eq=False)
class VarStarKernel:
    """u1 = A(x) u0 + B(x) u2 + S(x) L(u0) with pointwise coefficients that
    are functions of static fields and dt — e.g. the acoustic equation with an
    absorbing (damping) layer, ``m*u.dt2 - u.laplace + damp*u.dt``, which the
    reference's symbolics solve to A = (2m + d dt)/(m + d dt),
    B = -m/(m + d dt), S = dt^2/(m + d dt).  A, B, S are evaluated from the
    solved update itself (``coefficients``) once per apply, in fp64, and
    bound to fp32 arrays."""

    u: S.FieldSpec
    statics: Tuple[S.FieldSpec, ...]
    weights: Tuple[Tuple[Fraction, ...], ...]
    eq: S.StencilEquation
    has_prev: bool
    family: str = "vstar"

    @property
    def radius(self) -> Tuple[int, ...]:
        return tuple(len(w) - 1 for w in self.weights)

    def reads(self):
        out = [(self.u, 0, self.radius)]
        if self.has_prev:
            out.append((self.u, -1, (0,) * len(self.radius)))
        for f in self.statics:
            out.append((f, 0, (0,) * len(self.radius)))
        return out

    def writes(self):
        return [(self.u, 1)]

    @property
    def bytes_per_point(self) -> int:
        """u0, u2, A, B, S read, u1 written (the bound coefficient arrays
        replace the static fields on the hot path)."""
        return 4 * (2 + (2 if self.has_prev else 1) + 2)

    def coefficients(self, values, dt, spacing):
        """(A, B, S) from static-field values (arrays of one shape, fp64),
        dt and the grid spacing, by evaluating the solved update with unit
        unknowns (it is linear in them)."""
        u = self.u
        nd = len(spacing)
        bind = {}
        for leaf in _leaves(self.eq.rhs):
            if isinstance(leaf, S.Symbol):
                if leaf.name == "dt":
                    bind[leaf] = float(dt)
                else:
                    bind[leaf] = float(spacing[S.AXIS_NAMES.index(leaf.name[2:])])
            elif leaf.spec in values:
                bind[leaf] = values[leaf.spec]
            else:
                bind[leaf] = 0.0  # the unknowns (u0 taps, u2)
        centre = S.FieldAccess(u, 0, (0,) * nd)
        prev = S.FieldAccess(u, -1, (0,) * nd)
        k1 = S.FieldAccess(u, 0, tuple(1 if b == 0 else 0 for b in range(nd)))

        def coeff(acc):
            b = dict(bind)
            b[acc] = 1.0
            return S.eval_numeric(self.eq.rhs, b)

        W = self.weights
        Sv = coeff(k1) * (spacing[0] ** 2 / float(W[0][1]))
        A = coeff(centre) - Sv * sum(float(W[a][0]) / spacing[a] ** 2 for a in range(nd))
        B = coeff(prev) if self.has_prev else 0.0
        return A, B, Sv


@dataclass
class TTIKernel:
    """Two-field pseudo-acoustic TTI."""

    p: S.FieldSpec
    r: S.FieldSpec
    m: S.FieldSpec
    epsp: S.FieldSpec
    delp: S.FieldSpec
    a: Tuple[S.FieldSpec, S.FieldSpec, S.FieldSpec]
    so: int
    family: str = "tti"

    @property
    def radius(self):
        return (self.so // 2,) * 3

    def reads(self):
        nest = (self.so,) * 3
        zero = (0, 0, 0)
        out = [(self.p, 0, nest), (self.r, 0, nest), (self.p, -1, zero), (self.r, -1, zero),
               (self.m, 0, zero), (self.epsp, 0, zero), (self.delp, 0, zero)]
        out += [(ai, 0, self.radius) for ai in self.a]
        return out

    def writes(self):
        return [(self.p, 1), (self.r, 1)]

    bytes_per_point = 48


@dataclass(eq=False)
class RotatedKernel:
    """Single-field rotated operator, the SPEC's tti_gxx_kernel
    (SPEC.md:594-601): m u_tt = G u with G = sum_i D_i(a_i sum_j a_j D_j u)
    (nested centred first derivatives, the reference's Deriv(a * Deriv)
    lowering, symbolics.py:556-566), solved u1 = 2 u0 - u2 + dt^2/m G u0.
    Recognised by exact comparison with the reference discretization."""

    u: S.FieldSpec
    m: S.FieldSpec
    a: Tuple[S.FieldSpec, S.FieldSpec, S.FieldSpec]
    so: int
    family: str = "rotated"

    @property
    def radius(self):
        return (self.so // 2,) * 3

    def reads(self):
        zero = (0, 0, 0)
        out = [(self.u, 0, (self.so,) * 3), (self.u, -1, zero), (self.m, 0, zero)]
        out += [(ai, 0, self.radius) for ai in self.a]
        return out

    def writes(self):
        return [(self.u, 1)]

    bytes_per_point = 28  # u0, u2, m, a_x, a_y, a_z read; u1 written


def rotated_update(u: S.FieldSpec, m: S.FieldSpec, a) -> S.StencilEquation:
    """The reference discretization of m u_tt = G u."""
    inner = S.add(*(S.mul(a[j].at(), u.d(j)) for j in range(3)))
    gxx = S.add(*(S.Deriv(S.mul(a[i].at(), inner), i, 1) for i in range(3)))
    return S.solve_forward(S.Eq(m.at() * u.dt2 - gxx), u.forward)


def recognise_rotated(eq: S.StencilEquation) -> Optional[RotatedKernel]:
    """Match a solved update against rotated_update for some assignment of
    its static fields to (m, a_x, a_y, a_z), by exact evaluation at random
    rational bindings (or None)."""
    u = eq.lhs.spec
    if (u.is_static or eq.lhs.tshift != 1 or any(eq.lhs.offsets) or eq.temporaries
            or u.grid.ndims != 3 or u.time_order != 2):
        return None
    accs = S.accesses(eq.rhs)
    statics = {a.spec for a in accs if a.spec != u}
    if len(statics) != 4 or any(not f.is_static for f in statics):
        return None
    pointwise = [f for f in statics if all(not any(a.offsets) for a in accs if a.spec == f)]
    if len(pointwise) != 1:
        return None
    m = pointwise[0]
    others = sorted(statics - {m}, key=lambda f: f.name)
    leaves = sorted({S.format_expr(n) for n in _leaves(eq.rhs)})
    rng = random.Random(99)
    samples = [{k: Fraction(rng.randint(1, 40), rng.randint(1, 12)) for k in leaves}
               for _ in range(2)]

    def value(expr, vals):
        bind = {}
        for n in _leaves(expr):
            key = S.format_expr(n)
            if key not in vals:
                return None
            bind[n] = vals[key]
        return S.eval_exact(expr, bind)

    want = [value(eq.rhs, v) for v in samples]
    import itertools
    for perm in itertools.permutations(others):
        exp = rotated_update(u, m, perm)
        if {S.format_expr(n) for n in _leaves(exp.rhs)} != set(leaves):
            continue
        if [value(exp.rhs, v) for v in samples] == want:
            return RotatedKernel(u, m, tuple(perm), u.space_order)
    return None


@dataclass
class StaggeredPhase:
    """One phase of the staggered elastic / viscoelastic system."""

    kind: str  # "v" | "t" | "visco_t"
    v: Tuple[S.FieldSpec, ...]
    tau: Tuple[S.FieldSpec, ...]
    params: Tuple[S.FieldSpec, ...]  # (b,) | (lam, mu) | (l2m, mus, its)
    mem: Tuple[S.FieldSpec, ...] = ()
    so: int = 8
    family: str = "staggered"
    # the SPEC's collocated elastic_kernel: centred first
    # derivatives on one grid instead of the paper's staggered D+/D-
    collocated: bool = False

    @property
    def radius(self):
        return (self.so // 2,) * 3

    # axes each stress is differentiated along by the velocity update
    # (tau = xx, yy, zz, xy, xz, yz; PAPER.md:1041-1051, SPEC.md:587-592:
    # v_i,t = b sum_j D_j tau_ij)
    TAU_AXES = ((0,), (1,), (2,), (0, 1), (0, 2), (1, 2))

    def reads(self):
        r, zero = self.radius, (0, 0, 0)
        if self.kind == "v":
            tau = [(f, 0, tuple(r[a] if a in ax else 0 for a in range(3)))
                   for f, ax in zip(self.tau, self.TAU_AXES)]
            return tau + [(f, 0, zero) for f in self.v] + [(self.params[0], 0, zero)]
        out = [(f, 1, r) for f in self.v] + [(f, 0, zero) for f in self.tau]
        out += [(f, 0, zero) for f in self.mem] + [(f, 0, zero) for f in self.params]
        return out

    def writes(self):
        if self.kind == "v":
            return [(f, 1) for f in self.v]
        return [(f, 1) for f in self.tau] + [(f, 1) for f in self.mem]

    @property
    def bytes_per_point(self) -> int:
        if self.kind == "v":
            return 4 * 13
        if self.kind == "t":
            return 4 * 17
        return 4 * 30


# ---------------------------------------------------------------------------
# Recognition by exact rational probing


def _leaves(e: S.Expr):
    return {n for n in S.walk(e) if isinstance(n, (S.Symbol, S.FieldAccess))}


def _coefficients(rhs: S.Expr, unknowns: List[S.FieldAccess], binding: dict) -> dict:
    """Coefficient of each unknown access in a rhs that is linear in them."""
    base = dict(binding)
    for acc in unknowns:
        base[acc] = Fraction(0)
    c0 = S.eval_exact(rhs, base)
    out = {}
    for acc in unknowns:
        b = dict(base)
        b[acc] = Fraction(1)
        out[acc] = S.eval_exact(rhs, b) - c0
    # linearity / no affine constant: check on a random point as well
    rng = random.Random(7)
    b = dict(binding)
    vals = {acc: Fraction(rng.randint(-9, 9), rng.randint(1, 7)) for acc in unknowns}
    b.update(vals)
    if S.eval_exact(rhs, b) != c0 + sum(out[a] * vals[a] for a in unknowns) or c0 != 0:
        raise CompilerError("update is not linear-homogeneous in the field accesses")
    return out


def recognise_star(eq: S.StencilEquation) -> Optional[StarKernel]:
    """Match ``u1 = A u0 + B u2 + c dt^p m^q L(u0)`` exactly (or None)."""
    u = eq.lhs.spec
    if u.is_static or eq.lhs.tshift != 1 or any(eq.lhs.offsets):
        return None
    accs = S.accesses(eq.rhs) + [a for _, t in eq.temporaries for a in S.accesses(t)]
    if eq.temporaries:
        return None  # solve_forward output has none; CSE'd forms are re-solved upstream
    evolving = {a for a in accs if a.spec == u}
    statics = {a.spec for a in accs if a.spec != u}
    if any(a.spec != u and (not a.spec.is_static or any(a.offsets)) for a in accs):
        return None
    if len(statics) > 1:
        return None
    m = next(iter(statics)) if statics else None
    nd = u.grid.ndims
    if any(a.tshift not in (0, -1) for a in evolving):
        return None
    if any(a.tshift == -1 and any(a.offsets) for a in evolving):
        return None
    r = u.space_order // 2
    weights = [Fraction(w) for w in S.fd_coefficients(2, u.space_order)]
    W = tuple(weights[r + k] for k in range(r + 1))
    # expected access set: u0 star of radius r, u2 (optional), m[0]
    star = {S.FieldAccess(u, 0, tuple(k if b == a else 0 for b in range(nd)))
            for a in range(nd) for k in range(-r, r + 1)}
    u0s = {a for a in evolving if a.tshift == 0}
    if not u0s <= star:
        return None
    unknowns = sorted(u0s | {a for a in evolving if a.tshift == -1},
                      key=lambda a: (a.tshift, a.offsets))
    rng = random.Random(1234)
    samples = []
    for _ in range(3):
        bind = {}
        dt = Fraction(rng.randint(2, 30), rng.randint(2, 30))
        hs = [Fraction(rng.randint(2, 40), rng.randint(1, 9)) for _ in range(nd)]
        mv = Fraction(rng.randint(2, 50), rng.randint(2, 17))
        for leaf in _leaves(eq.rhs):
            if isinstance(leaf, S.Symbol):
                if leaf.name == "dt":
                    bind[leaf] = dt
                elif leaf.name.startswith("h_"):
                    bind[leaf] = hs[S.AXIS_NAMES.index(leaf.name[2:])]
                else:
                    return None
            elif leaf.spec == m:
                bind[leaf] = mv
        coeffs = _coefficients(eq.rhs, unknowns, bind)
        samples.append((dt, hs, mv, coeffs))
    k1 = S.FieldAccess(u, 0, tuple(1 if b == 0 else 0 for b in range(nd)))
    if W[1] == 0:
        return None
    centre = S.FieldAccess(u, 0, (0,) * nd)
    prev = S.FieldAccess(u, -1, (0,) * nd)
    scales, AB = [], set()
    for dt, hs, mv, co in samples:
        Sv = co.get(k1, Fraction(0)) * hs[0] ** 2 / W[1]
        if Sv == 0:
            return None
        for a in range(nd):
            for k in range(1, r + 1):
                for sgn in (-1, 1):
                    acc = S.FieldAccess(u, 0, tuple(sgn * k if b == a else 0 for b in range(nd)))
                    if co.get(acc, Fraction(0)) != Sv * W[k] / hs[a] ** 2:
                        return None
        A = co.get(centre, Fraction(0)) - Sv * sum(W[0] / h ** 2 for h in hs)
        AB.add((A, co.get(prev, Fraction(0))))
        scales.append((dt, mv, Sv))
    if len(AB) != 1:
        return None
    A0, B0 = AB.pop()
    # S = c * dt^p * m^q: exactly one (p, q) gives a sample-independent c
    cands = [(p, q) for p in (0, 1, 2) for q in ((0, -1) if m is not None else (0,))]
    fits = [(p, q) for p, q in cands
            if len({Sv / (dt ** p * mv ** q) for dt, mv, Sv in scales}) == 1]
    if len(fits) != 1:
        return None
    pq = fits[0]
    dt, mv, Sv = scales[0]
    c0 = Sv / (dt ** pq[0] * mv ** pq[1])
    if B0 != 0 and u.time_order < 2:
        return None
    if pq[1] == 0:
        m = None
    return StarKernel(u=u, m=m, A=A0, B=B0, c=c0, p=pq[0], q=pq[1],
                      weights=tuple(W for _ in range(nd)))


# Registry of family equations built by paper_2312_13094_b200.kernels; the
# Operator matches user equations against it by structural equality.
_FAMILY_REGISTRY: Dict[S.StencilEquation, object] = {}


def register_family(eq: S.StencilEquation, kernel) -> None:
    _FAMILY_REGISTRY[eq] = kernel


def recognise_var_star(eq: S.StencilEquation) -> Optional[VarStarKernel]:
    """Match u1 = A u0 + B u2 + S L(u0) where A, B, S may depend on any
    static fields read at the point (exact rational probing with independent
    random values for every static field; or None)."""
    u = eq.lhs.spec
    if u.is_static or eq.lhs.tshift != 1 or any(eq.lhs.offsets) or eq.temporaries:
        return None
    accs = S.accesses(eq.rhs)
    evolving = {a for a in accs if a.spec == u}
    if any(a.spec != u and (not a.spec.is_static or any(a.offsets)) for a in accs):
        return None
    statics = tuple(sorted({a.spec for a in accs if a.spec != u}, key=lambda f: f.name))
    nd = u.grid.ndims
    if any(a.tshift not in (0, -1) for a in evolving):
        return None
    if any(a.tshift == -1 and any(a.offsets) for a in evolving):
        return None
    r = u.space_order // 2
    weights = [Fraction(w) for w in S.fd_coefficients(2, u.space_order)]
    W = tuple(weights[r + k] for k in range(r + 1))
    if W[1] == 0:
        return None
    star = {S.FieldAccess(u, 0, tuple(k if b == a else 0 for b in range(nd)))
            for a in range(nd) for k in range(-r, r + 1)}
    u0s = {a for a in evolving if a.tshift == 0}
    if not u0s <= star:
        return None
    has_prev = any(a.tshift == -1 for a in evolving)
    unknowns = sorted(u0s | {a for a in evolving if a.tshift == -1},
                      key=lambda a: (a.tshift, a.offsets))
    rng = random.Random(4321)
    k1 = S.FieldAccess(u, 0, tuple(1 if b == 0 else 0 for b in range(nd)))
    for _ in range(3):
        bind = {}
        hs = [Fraction(rng.randint(2, 40), rng.randint(1, 9)) for _ in range(nd)]
        svals = {f: Fraction(rng.randint(2, 50), rng.randint(2, 17)) for f in statics}
        for leaf in _leaves(eq.rhs):
            if isinstance(leaf, S.Symbol):
                if leaf.name == "dt":
                    bind[leaf] = Fraction(rng.randint(2, 30), rng.randint(2, 30))
                elif leaf.name.startswith("h_"):
                    bind[leaf] = hs[S.AXIS_NAMES.index(leaf.name[2:])]
                else:
                    return None
            elif leaf.spec != u:
                bind[leaf] = svals[leaf.spec]
        co = _coefficients(eq.rhs, unknowns, bind)
        Sv = co.get(k1, Fraction(0)) * hs[0] ** 2 / W[1]
        if Sv == 0:
            return None
        for a in range(nd):
            for k in range(1, r + 1):
                for sgn in (-1, 1):
                    acc = S.FieldAccess(u, 0, tuple(sgn * k if b == a else 0 for b in range(nd)))
                    if co.get(acc, Fraction(0)) != Sv * W[k] / hs[a] ** 2:
                        return None
    return VarStarKernel(u, statics, tuple(W for _ in range(nd)), eq, has_prev)


class _Probe:
    """Exact evaluation at seeded random rational values keyed by
    (field spec, tshift, offsets) / symbol name, drawn on first use, so two
    expressions over the same leaves see the same values.  ``rename`` maps
    field specs of a template onto the fields a candidate role assignment
    gives them (the template is built once and re-evaluated per assignment)."""

    def __init__(self, seed):
        self.rng = random.Random(seed)
        self.vals = {}

    def _value(self, key):
        v = self.vals.get(key)
        if v is None:
            v = self.vals[key] = Fraction(self.rng.randint(1, 40), self.rng.randint(1, 12))
        return v

    def eval(self, expr, rename=None):
        bind = {}
        for n in _leaves(expr):
            if isinstance(n, S.Symbol):
                bind[n] = self._value(("symbol", n.name))
            else:
                spec = rename.get(n.spec, n.spec) if rename else n.spec
                bind[n] = self._value((spec, n.tshift, n.offsets))
        return S.eval_exact(expr, bind)


def _matching_rename(eqs, templates, renames, samples=2):
    """First rename under which every solved update in ``eqs`` equals its
    template (same lhs after renaming) at ``samples`` independent exact
    probes (the updates themselves are evaluated once per probe), or None."""
    probes = [_Probe(1000 + seed) for seed in range(samples)]
    cache = {}
    for rename in renames:
        ok = True
        for si, pr in enumerate(probes):
            for ei, (eq, tp) in enumerate(zip(eqs, templates)):
                if rename.get(tp.lhs.spec, tp.lhs.spec) != eq.lhs.spec:
                    ok = False
                    break
                if (si, ei) not in cache:
                    cache[(si, ei)] = pr.eval(eq.rhs)
                if cache[(si, ei)] != pr.eval(tp.rhs, rename):
                    ok = False
                    break
            if not ok:
                break
        if ok:
            return rename
    return None


def _solved_shape_ok(eq, time_order) -> bool:
    u = eq.lhs.spec
    return (not u.is_static and eq.lhs.tshift == 1 and not any(eq.lhs.offsets)
            and not eq.temporaries and u.grid.ndims == 3 and u.time_order == time_order)


def tti_updates(p: S.FieldSpec, r: S.FieldSpec, m: S.FieldSpec, epsp: S.FieldSpec,
                delp: S.FieldSpec, a) -> Tuple[S.StencilEquation, S.StencilEquation]:
    """The paper's two-field pseudo-acoustic TTI (Devito's
    centred kernel form) written with the reference symbolics:

        Gzz f = sum_i D_i(a_i sum_j a_j D_j f)   (nested centred first
                derivatives, the reference's Deriv(coef * Deriv) lowering,
                symbolics.py:556-566; radius = space order)
        H0 f  = laplace f - Gzz f
        m p.dt2 = epsp H0 p + delp Gzz r
        m r.dt2 = delp H0 p + Gzz r

    with epsp = 1 + 2 eps, delp = sqrt(1 + 2 delta) and the direction
    cosines a = (sin t cos f, sin t sin f, cos t) as static fields, each
    solved for the forward buffer by ``solve_forward`` (symbolics.py:629)."""
    def gzz(f):
        inner = S.add(*(S.mul(a[j].at(), f.d(j)) for j in range(3)))
        return S.add(*(S.Deriv(S.mul(a[i].at(), inner), i, 1) for i in range(3)))

    h0p = S.add(p.laplace, S.neg(gzz(p)))
    gr = gzz(r)
    eq_p = S.solve_forward(
        S.Eq(S.mul(m.at(), p.dt2), S.add(S.mul(epsp.at(), h0p), S.mul(delp.at(), gr))),
        p.forward)
    eq_r = S.solve_forward(
        S.Eq(S.mul(m.at(), r.dt2), S.add(S.mul(delp.at(), h0p), gr)), r.forward)
    return eq_p, eq_r


def recognise_tti(eq_p: S.StencilEquation, eq_r: S.StencilEquation) -> Optional[TTIKernel]:
    """Match a pair of solved updates against ``tti_updates`` for some
    assignment of their static fields to (m, epsp, delp, a_x, a_y, a_z):
    epsp is the pointwise static only the p update reads, {m, delp} the
    pointwise statics both read, the three statics read at offsets are the
    direction cosines; the 2 x 6 remaining assignments are decided by exact
    evaluation of one template (or None)."""
    if not (_solved_shape_ok(eq_p, 2) and _solved_shape_ok(eq_r, 2)):
        return None
    p, r = eq_p.lhs.spec, eq_r.lhs.spec
    if p == r or p.space_order != r.space_order or p.grid != r.grid:
        return None
    acc_p, acc_r = S.accesses(eq_p.rhs), S.accesses(eq_r.rhs)
    for accs in (acc_p, acc_r):
        if {a.spec for a in accs if not a.spec.is_static} != {p, r}:
            return None

    def split(accs):
        st = {a.spec for a in accs if a.spec.is_static}
        pw = {f for f in st if all(not any(a.offsets) for a in accs if a.spec == f)}
        return pw, st - pw

    pw_p, off_p = split(acc_p)
    pw_r, off_r = split(acc_r)
    if len(pw_p) != 3 or len(pw_r) != 2 or not pw_r < pw_p or off_p != off_r or len(off_p) != 3:
        return None
    epsp = next(iter(pw_p - pw_r))
    import itertools
    a0 = tuple(sorted(off_p, key=lambda f: f.name))
    m0, d0 = sorted(pw_r, key=lambda f: f.name)
    tp = tti_updates(p, r, m0, epsp, d0, a0)
    renames = [{m0: m, d0: d, **dict(zip(a0, perm))}
               for m, d in ((m0, d0), (d0, m0)) for perm in itertools.permutations(a0)]
    rn = _matching_rename((eq_p, eq_r), tp, renames)
    if rn is None:
        return None
    return TTIKernel(p, r, rn[m0], epsp, rn[d0], tuple(rn[f] for f in a0), p.space_order)


# stress components in the order xx, yy, zz, xy, xz, yz
_TAU_INDEX = {(0, 0): 0, (1, 1): 1, (2, 2): 2, (0, 1): 3, (0, 2): 4, (1, 2): 5}


def _tau(i, j):
    return _TAU_INDEX[(min(i, j), max(i, j))]


def elastic_updates(v, tau, b: S.FieldSpec, lam: S.FieldSpec, mu: S.FieldSpec):
    """The SPEC's collocated isotropic elastic system (
    PAPER.md:1041-1051 on one grid) written with the reference symbolics:

        v_i.dt   = b sum_j D_j tau_ij
        tau_ii.dt = lam sum_k D_k v_k[t+1] + 2 mu D_i v_i[t+1]
        tau_ij.dt = mu (D_j v_i[t+1] + D_i v_j[t+1])     (i != j)

    D = centred first derivative of the fields' space order; the stress
    update reads the freshly updated velocity (``v.forward``).  Returns the
    nine solved updates (3 velocity, then 6 stress)."""
    out = []
    for i in range(3):
        div = S.add(*(tau[_tau(i, j)].d(j) for j in range(3)))
        out.append(S.solve_forward(S.Eq(v[i].dt, S.mul(b.at(), div)), v[i].forward))

    def dv(i, j):
        return S.Deriv(v[i].forward, j, 1)

    tr = S.add(*(dv(k, k) for k in range(3)))
    for i in range(3):
        rhs = S.add(S.mul(lam.at(), tr), S.mul(S.Const(Fraction(2)), mu.at(), dv(i, i)))
        out.append(S.solve_forward(S.Eq(tau[i].dt, rhs), tau[i].forward))
    for (i, j) in ((0, 1), (0, 2), (1, 2)):
        k = _tau(i, j)
        out.append(S.solve_forward(S.Eq(tau[k].dt, S.mul(mu.at(), S.add(dv(i, j), dv(j, i)))),
                                   tau[k].forward))
    return out


def recognise_elastic(eqs: Sequence[S.StencilEquation]):
    """Match nine solved first-order updates against ``elastic_updates``.

    Roles are read off the access structure (velocity updates read stresses
    at tshift 0 with offsets; a diagonal stress is read by one velocity
    update along that velocity's axis, an off-diagonal one by two; b is the
    static of the velocity updates; mu the only static of the shear-stress
    updates, lam the other static of the normal-stress ones), then the whole
    system is verified by exact evaluation.  Returns the velocity and stress
    phases (collocated ``StaggeredPhase`` pair) or None."""
    if len(eqs) != 9 or not all(_solved_shape_ok(e, 1) for e in eqs):
        return None
    lhs = [e.lhs.spec for e in eqs]
    if len(set(lhs)) != 9 or len({f.space_order for f in lhs}) != 1:
        return None
    evolving = set(lhs)
    vel, stress = [], []
    for e in eqs:
        ts = {a.tshift for a in S.accesses(e.rhs) if a.spec in evolving and a.spec != e.lhs.spec}
        if ts == {0}:
            vel.append(e)
        elif ts == {1}:
            stress.append(e)
        else:
            return None
    if len(vel) != 3 or len(stress) != 6:
        return None
    vfields = [e.lhs.spec for e in vel]
    tfields = {e.lhs.spec for e in stress}
    readers = {f: [] for f in tfields}   # stress field -> [(velocity field, axes read along)]
    for e in vel:
        for f in tfields:
            offs = [a.offsets for a in S.accesses(e.rhs) if a.spec == f]
            if offs:
                axes = {ax for o in offs for ax, k in enumerate(o) if k}
                if len(axes) != 1:
                    return None
                readers[f].append((e.lhs.spec, axes.pop()))
    v_of_axis, tau = {}, [None] * 6
    for f, rd in readers.items():
        if len(rd) == 1:
            vf, ax = rd[0]
            if ax in v_of_axis:
                return None
            v_of_axis[ax] = vf
            tau[_tau(ax, ax)] = f
    if sorted(v_of_axis) != [0, 1, 2]:
        return None
    axis_of_v = {vf: ax for ax, vf in v_of_axis.items()}
    for f, rd in readers.items():
        if len(rd) == 2:
            (v1, a1), (v2, a2) = rd
            i, j = axis_of_v[v1], axis_of_v[v2]
            if {i, j} != {a1, a2} or i == j:
                return None
            tau[_tau(i, j)] = f
    if any(t is None for t in tau):
        return None
    v = tuple(v_of_axis[a] for a in range(3))
    statics = lambda e: {a.spec for a in S.accesses(e.rhs) if a.spec.is_static}
    bs = set.union(*(statics(e) for e in vel))
    shear = [e for e in stress if e.lhs.spec in tau[3:]]
    normal = [e for e in stress if e.lhs.spec in tau[:3]]
    mus = set.union(*(statics(e) for e in shear))
    lams = set.union(*(statics(e) for e in normal)) - mus
    if len(bs) != 1 or len(mus) != 1 or len(lams) != 1:
        return None
    b, mu, lam = bs.pop(), mus.pop(), lams.pop()
    tp = elastic_updates(v, tau, b, lam, mu)
    by_lhs = {e.lhs.spec: e for e in eqs}
    if _matching_rename([by_lhs[t.lhs.spec] for t in tp], tp, [{}]) is None:
        return None
    so = v[0].space_order
    kv = StaggeredPhase("v", v, tuple(tau), (b,), so=so, collocated=True)
    kt = StaggeredPhase("t", v, tuple(tau), (lam, mu), so=so, collocated=True)
    return kv, kt


def _recognise_groups(pending: List[S.StencilEquation]):
    """Multi-equation families among updates no single-equation family
    matched: TTI pairs (each update reads the other's field) and the
    nine-update collocated elastic system.  Returns [(first index, kernels,
    consumed indices)]."""
    out, used = [], set()
    for i, e in enumerate(pending):
        if i in used or not _solved_shape_ok(e, 2):
            continue
        others = {a.spec for a in S.accesses(e.rhs) if not a.spec.is_static} - {e.lhs.spec}
        for j, f in enumerate(pending):
            if j in used or j == i or f.lhs.spec not in others:
                continue
            # p is the update reading three pointwise statics (epsp, m, delp)
            for a, b_ in ((e, f), (f, e)):
                k = recognise_tti(a, b_)
                if k is not None:
                    out.append((min(i, j), [k], {i, j}))
                    used |= {i, j}
                    break
            if i in used:
                break
    first_order = [i for i, e in enumerate(pending) if i not in used and _solved_shape_ok(e, 1)]
    if len(first_order) >= 9:
        ks = recognise_elastic([pending[i] for i in first_order[:9]])
        if ks is not None:
            out.append((first_order[0], list(ks), set(first_order[:9])))
            used |= set(first_order[:9])
    return out, used


def recognise(equations: Sequence) -> List[object]:
    """Solved updates -> kernel list (one kernel may own several updates).

    Single-update families first (star, damped star, rotated G_xx), then
    the multi-update families among the rest (TTI pair, collocated elastic
    system), placed at their first update's position.  Anything left
    raises: there is no generic/CPU path."""
    slots: List[object] = []     # kernels, or ("pending", index into pending)
    pending: List[S.StencilEquation] = []
    seen = set()
    for eq in equations:
        if isinstance(eq, (StarKernel, VarStarKernel, RotatedKernel, TTIKernel, StaggeredPhase)):
            slots.append(eq)
            continue
        if not isinstance(eq, S.StencilEquation):
            raise CompilerError(f"expected a solved update, got {type(eq).__name__}")
        fam = _FAMILY_REGISTRY.get(eq)
        if fam is not None:
            if id(fam) not in seen:
                seen.add(id(fam))
                slots.append(fam)
            continue
        k = recognise_star(eq)
        if k is None:
            k = recognise_var_star(eq)
        if k is None:
            k = recognise_rotated(eq)
        if k is None:
            slots.append(("pending", len(pending)))
            pending.append(eq)
        else:
            slots.append(k)
    groups, used = _recognise_groups(pending) if pending else ([], set())
    left = [e for i, e in enumerate(pending) if i not in used]
    if left:
        raise CompilerError(
            "equation not recognised as a supported kernel family (acoustic, "
            "damped acoustic, diffusion, rotated G_xx, TTI pair, collocated "
            "elastic system; staggered elastic/viscoelastic via kernels.py): "
            + " ; ".join(S.format_equation(left[0]))[:300])
    first = {g[0]: g[1] for g in groups}
    kernels: List[object] = []
    for sl in slots:
        if isinstance(sl, tuple) and len(sl) == 2 and sl[0] == "pending":
            kernels.extend(first.get(sl[1], []))
        else:
            kernels.append(sl)
    return kernels


# ---------------------------------------------------------------------------
# Access alignment


def align_accesses(eq: S.StencilEquation, halo=None) -> S.StencilEquation:
    """Shift every spatial index by +halo (``u[t,x,y]`` -> ``u[t,x+2,y+2]``
    for SO-2).  ``halo`` = per-axis width for all fields, or None for each
    field's own halo.  Relative offsets are unchanged."""

    def move(n):
        if isinstance(n, S.FieldAccess):
            h = n.spec.halo if halo is None else tuple(halo)
            return S.FieldAccess(n.spec, n.tshift, tuple(o + k for o, k in zip(n.offsets, h)))
        return n

    lhs = move(eq.lhs)
    rhs = S.transform(eq.rhs, move)
    temps = tuple((name, S.transform(body, move)) for name, body in eq.temporaries)
    # bypass the explicit-scheme check (already validated on the input)
    out = object.__new__(S.StencilEquation)
    object.__setattr__(out, "lhs", lhs)
    object.__setattr__(out, "rhs", rhs)
    object.__setattr__(out, "temporaries", temps)
    return out


# ---------------------------------------------------------------------------
# HaloSpots


@dataclass
class HaloSpot:
    """Exchange of ``fields`` (spec, tshift) with per-axis ``radius`` (the
    union over the fields: it sizes CORE / OWNED and the message boxes).

    ``field_radius`` holds each field's own per-axis read radius, as Devito's
    HaloScheme keeps one per function: a field read with offsets along x
    only (the staggered velocity update reads txx only through D_x) never
    ships its y faces or xy corners."""

    fields: List[Tuple[S.FieldSpec, int]]
    radius: Tuple[int, ...]
    field_radius: Optional[Dict[Tuple[S.FieldSpec, int], Tuple[int, ...]]] = None

    def sends(self, f: S.FieldSpec, t: int, direction) -> bool:
        """Whether ``(f, t)`` travels in the message along ``direction``:
        every axis the direction crosses must be one the field is read
        along."""
        if os.environ.get("SDMP_FIELD_RADII", "1") == "0":  # A/B: every face
            return True
        fr = (self.field_radius or {}).get((f, t), self.radius)
        return all(fr[a] > 0 for a, d in enumerate(direction) if d)


@dataclass
class Phase:
    halo: Optional[HaloSpot]
    kernel: object


@dataclass
class HaloAnalysis:
    hoisted: Optional[HaloSpot]
    phases: List[Phase]
    exchanges_per_step: int


def halo_phases(kernels: Sequence, nranks: int) -> HaloAnalysis:
    """build_clusters + optimize_halospots."""
    nd = None
    written = set()
    for k in kernels:
        for f, _t in k.writes():
            written.add(f)
    # static fields read with offsets -> hoisted once before the loop
    hoist_fields, hoist_r = [], None
    # dirty buffers at step start: everything written last step (tshift 0
    # relative to the new step is the old tshift +1)
    dirty = {(f, 0) for f in written}
    phases = []
    count = 0
    for k in kernels:
        need, rad, frad = [], None, {}
        for f, t, r in k.reads():
            nd = len(r)
            if not any(r) or nranks == 1:
                continue
            if f.is_static:
                if (f, 0) not in hoist_fields:
                    hoist_fields.append((f, 0))
                hoist_r = tuple(max(a, b) for a, b in zip(hoist_r or r, r))
                continue
            if (f, t) in dirty:
                if (f, t) not in [x[0:2] for x in need]:
                    need.append((f, t))
                rad = tuple(max(a, b) for a, b in zip(rad or r, r))
                fr = frad.get((f, t))
                frad[(f, t)] = tuple(max(a, b) for a, b in zip(fr or r, r))
        spot = None
        if need:
            spot = HaloSpot(need, rad, frad)
            count += 1
            for ft in need:
                dirty.discard(ft)
        phases.append(Phase(spot, k))
        for f, t in k.writes():
            dirty.add((f, t))
    hoisted = HaloSpot(hoist_fields, hoist_r) if hoist_fields else None
    return HaloAnalysis(hoisted, phases, count)


# ---------------------------------------------------------------------------
# ExecPlan (per-rank action list in terms of boxes; lowered to native ids by
# runtime_plan.py)


@dataclass
class Action:
    kind: str                 # post | wait | compute | inject | interp | record | streamwait
    stream: int
    phase: int = -1           # epoch phase index (post / wait)
    spot: Optional[HaloSpot] = None
    messages: list = field(default_factory=list)
    kernel: object = None
    box: tuple = None         # DOMAIN coordinates
    region: str = ""
    event: int = -1
    sparse: object = None
    # fused halo push (full mode): the compute / inject kernel also stores
    # these output fields into the neighbours' HALO over NVLink:
    # (output fields in kernel output order, messages giving the boxes)
    push: Optional[tuple] = None
    pushed: bool = False      # post: halos already pushed (copy only on run start)


@dataclass
class ExecPlan:
    mode: str
    actions: List[Action]
    phases_per_step: int
    hoisted: Optional[HaloSpot]
    hoisted_messages: list

    def kinds(self) -> List[str]:
        return [a.kind if a.kind != "compute" else f"compute:{a.region}" for a in self.actions]

    def message_count(self) -> int:
        return sum(len(a.messages) for a in self.actions if a.kind == "post")


def optimize_halospots(kernels: Sequence, nranks: int) -> HaloAnalysis:
    """SPEC.md:348-356 name for :func:`halo_phases` (drop / merge / hoist)."""
    return halo_phases(kernels, nranks)


def dump_plan(kernels: Sequence, nranks: int, mode: Optional[str] = None,
              updates: Sequence = ()) -> str:
    """Listing 5/6/7-style text: the time loop with its
    HaloSpots before lowering (``mode=None``) or the mode's update / wait
    calls after lowering.  ``updates`` = solved equations printed (CSE'd,
    aligned) inside the loop nest."""
    an = halo_phases(kernels, nranks)
    nd = None
    lines = ["<Callable Kernel>"]
    exprs = []
    for eq in updates:
        e = align_accesses(S.apply_cse(eq))
        exprs += S.format_equation(e)
    for k in kernels:
        nd = len(k.radius)
    if an.hoisted is not None:
        names = ",".join(f.name for f, _t in an.hoisted.fields)
        lines.append(f" <HaloSpot({names}) hoisted>" if mode is None
                     else f" <HaloUpdateCall({names}) once>")
    lines.append(" <[affine,sequential] Iteration time...>")
    loops = ["x", "y", "z"][: nd or 3]

    def nest(indent, region=""):
        out = []
        for i, ax in enumerate(loops):
            tag = "[affine,parallel,vector-dim]" if i == len(loops) - 1 else "[affine,parallel]"
            out.append(" " * (indent + i) + f"<{tag} Iteration {ax}{region}...>")
        for e in exprs or ["<stencil update>"]:
            out.append(" " * (indent + len(loops)) + f"<Expression {e}>")
        return out

    for ph in an.phases:
        spot = ph.halo
        names = ",".join(f.name for f, _t in spot.fields) if spot else ""
        if spot is None:
            lines += nest(2)
        elif mode is None:
            lines.append(f"  <HaloSpot({names})>")
            lines += nest(2)
        elif normalise_mode(mode) in ("basic", "diagonal"):
            steps = len(loops) if normalise_mode(mode) == "basic" else 1
            lines.append(f"  <HaloUpdateList({names}) steps={steps}>")
            lines.append("   <HaloUpdateCall>")
            lines.append(f"  <HaloWaitList({names})>")
            lines += nest(2)
        else:
            lines.append(f"  <HaloUpdateList({names}) async>")
            lines += nest(2, " CORE")
            lines.append(f"  <HaloWaitList({names})>")
            lines += nest(2, " REMAINDER")
    return "\n".join(lines)


def _fuse_pushes(acts, analysis: HaloAnalysis, decomp, rank: int) -> None:
    """Full mode: fold the halo exchange into the kernels that produce the
    OWNED values.  Every exchanged field's send boxes lie inside the OWNED
    slabs (CORE is shrunk by the same radius), so the slab kernels (and the
    source injection, which updates values after them) store every value a
    neighbour needs straight into its HALO; the next post only releases the
    flag (copies happen on the first step of a run, when nothing was
    pushed).  Falls back to copies if any precondition fails."""
    from .distfield import RegionName, diagonal_messages, rank_regions

    radius, spot_of = {}, {}
    for ph in analysis.phases:
        if ph.halo is not None:
            for f, t in ph.halo.fields:
                radius[f] = ph.halo.radius
                spot_of[f] = (ph.halo, t)
    if not radius:
        return
    geo = {f: diagonal_messages(decomp, rank, r) for f, r in radius.items()}
    if any(len(m) > 8 for m in geo.values()):
        return  # push lists hold 8 directions (x/y splits)

    def outputs(k):
        outs = [f for f, t in k.writes() if t == 1]
        pushed = [f for f in outs if f in radius]
        # the kernels push a PREFIX of their outputs with one geometry
        if not pushed or outs[:len(pushed)] != pushed:
            return None
        if len({radius[f] for f in pushed}) != 1:
            return None
        return pushed

    plan = []
    for a in acts:
        if a.kind == "compute" and a.region == "OWNED":
            outs = outputs(a.kernel)
            if outs is None:
                if any(f in radius for f, _t in a.kernel.writes()):
                    return
                continue
            plan.append((a, (outs, geo[outs[0]])))
        elif a.kind == "compute" and a.region == "CORE":
            # CORE must not intersect any pushed send box
            outs = outputs(a.kernel) or []
            for f in outs:
                for m in geo[f]:
                    lo = [max(x, y) for x, y in zip(a.box[0], m.send[0])]
                    hi = [min(x, y) for x, y in zip(a.box[1], m.send[1])]
                    if all(h > l for l, h in zip(lo, hi)):
                        return
        elif a.kind == "inject" and a.sparse.field in radius:
            plan.append((a, ([a.sparse.field], geo[a.sparse.field])))
    for a, (outs, msgs) in plan:
        # per output and direction: does the neighbour read this field
        # across that face (HaloSpot.sends)?  Kernels skip the others.
        sends = [[spot_of[f][0].sends(f, spot_of[f][1], m.direction) for m in msgs]
                 for f in outs]
        a.push = (outs, msgs, sends)
    for a in acts:
        if a.kind == "post":
            a.pushed = True


def lower_mode(analysis: HaloAnalysis, decomp, rank: int, mode: str,
               sparse_terms: Sequence = (), exchange: bool = True,
               fused: bool = True) -> ExecPlan:
    """Per-rank ExecPlan for ``mode``.

    ``exchange=False`` keeps the mode's compute boxes and stream structure
    but drops every post/wait: the compute-only baseline used to measure
    the exposed halo-exchange time per step."""
    from .distfield import (RegionName, basic_messages, diagonal_messages,
                            rank_regions)

    mode = normalise_mode(mode)
    nd = decomp.ndims
    acts: List[Action] = []
    epoch = 0
    ev = 0
    shape = decomp.local_shape(rank)
    domain = ((0,) * nd, tuple(shape))
    interps = [t for t in sparse_terms if t.kind == "interp"]
    injects = [t for t in sparse_terms if t.kind == "inject"]

    def kernel_reads_field(k, spec):
        return any(f == spec for f, _t, _r in k.reads())

    def kernel_writes_field(k, spec):
        return any(f == spec for f, _t in k.writes())

    for pi, ph in enumerate(analysis.phases):
        k = ph.kernel
        spot = ph.halo
        my_interps = [t for t in interps if kernel_reads_field(k, t.field)
                      and t not in [a.sparse for a in acts if a.kind == "interp"]]
        my_injects = [t for t in injects if kernel_writes_field(k, t.field)]
        if spot is not None:
            # the exchange stream must see this step's previous compute; in
            # full mode so must the remainder stream: its OWNED kernels read
            # values next to CORE that the previous phase's CORE kernel (and
            # the injection) wrote on stream 0, and the peer's flag does not
            # order them (found by the full-size bitwise check, r02)
            acts.append(Action("record", 0, event=ev))
            acts.append(Action("streamwait", 2, event=ev))
            if mode == "full":
                acts.append(Action("streamwait", 1, event=ev))
            ev += 1
        if spot is None:
            # no exchange: the interpolation reads the field's current
            # buffer, which this phase's update does not write (explicit
            # scheme), so it runs on stream 1 beside the update, ordered
            # after everything stream 0 did before it (r03: C1 -4.5 us/step)
            # That holds only if the update never writes the sampled buffer
            # (tshift 0) and the field has a separate buffer to write to;
            # otherwise the interpolation runs on stream 0 first.
            overlap = [t for t in my_interps
                       if (t.field, 0) not in set(k.writes()) and t.field.time_buffers >= 2]
            if overlap:
                acts.append(Action("record", 0, event=ev))
                acts.append(Action("streamwait", 1, event=ev))
                ev += 1
            for t in my_interps:
                acts.append(Action("interp", 1 if t in overlap else 0, sparse=t))
            acts.append(Action("compute", 0, kernel=k, box=domain, region="DOMAIN"))
        elif mode == "basic":
            steps = basic_messages(decomp, rank, spot.radius)
            for a in range(nd):
                acts.append(Action("post", 2, phase=epoch, spot=spot, messages=steps[a]))
                acts.append(Action("wait", 2, phase=epoch, spot=spot, messages=steps[a]))
                epoch += 1
            acts.append(Action("record", 2, event=ev))
            acts.append(Action("streamwait", 0, event=ev))
            ev += 1
            for t in my_interps:
                acts.append(Action("interp", 0, sparse=t))
            acts.append(Action("compute", 0, kernel=k, box=domain, region="DOMAIN"))
        elif mode == "diagonal":
            msgs = diagonal_messages(decomp, rank, spot.radius)
            acts.append(Action("post", 2, phase=epoch, spot=spot, messages=msgs))
            # the wait follows the post on the exchange stream (a spinning
            # wait on the compute stream, unordered with the post, replays
            # ~1.7x slower inside CUDA graphs: measured r02)
            acts.append(Action("wait", 2, phase=epoch, spot=spot, messages=msgs))
            acts.append(Action("record", 2, event=ev))
            acts.append(Action("streamwait", 0, event=ev))
            ev += 1
            epoch += 1
            for t in my_interps:
                acts.append(Action("interp", 0, sparse=t))
            acts.append(Action("compute", 0, kernel=k, box=domain, region="DOMAIN"))
        else:  # full: post -> CORE -> wait -> OWNED (Listing 8)
            msgs = diagonal_messages(decomp, rank, spot.radius)
            acts.append(Action("post", 2, phase=epoch, spot=spot, messages=msgs))
            core = rank_regions(decomp, rank, spot.radius, RegionName.CORE)[0]
            acts.append(Action("compute", 0, kernel=k, box=core, region="CORE"))
            acts.append(Action("wait", 1, phase=epoch, spot=spot, messages=msgs))
            epoch += 1
            for t in my_interps:
                acts.append(Action("interp", 1, sparse=t))
            for slab in rank_regions(decomp, rank, spot.radius, RegionName.OWNED):
                acts.append(Action("compute", 1, kernel=k, box=slab, region="OWNED"))
            acts.append(Action("record", 1, event=ev))
            acts.append(Action("streamwait", 0, event=ev))
            ev += 1
        for t in my_injects:
            acts.append(Action("inject", 0, sparse=t))
    emitted = {id(a.sparse) for a in acts if a.kind in ("interp", "inject")}
    for t in sparse_terms:
        if id(t) not in emitted:
            what = "reads" if t.kind == "interp" else "writes"
            raise CompilerError(f"{t.kind} of {t.sparse.name!r} on field {t.field.name!r}: no "
                                f"kernel of this Operator {what} that field")
    if ev > 32:
        raise CompilerError("too many stream joins per step")
    if not exchange:
        acts = [a for a in acts if a.kind not in ("post", "wait")]
    elif mode == "full" and fused:
        _fuse_pushes(acts, analysis, decomp, rank)
    # phases per step is identical on every rank (epoch numbering)
    per_step = 0
    for ph in analysis.phases:
        if ph.halo is not None:
            per_step += nd if mode == "basic" else 1
    hoisted_msgs = []
    if analysis.hoisted is not None:
        hoisted_msgs = diagonal_messages(decomp, rank, analysis.hoisted.radius)
    return ExecPlan(mode, acts, max(per_step, 1), analysis.hoisted, hoisted_msgs)
