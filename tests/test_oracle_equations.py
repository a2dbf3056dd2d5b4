"""Pins the CPU oracle's per-point updates (oracle/stencils.py) to the solved
update equations of the symbolic front end, whose printed forms equal the
reference's (sha256 fixtures generated from /root/reference by
tests/golden/make_golden.py, checked in test_symbolics_golden.py).

Each solved rhs (symbolics.py solve_forward, reference symbolics.py:591-674)
is evaluated numerically over a box -- every FieldAccess bound to the array
view shifted by its offsets, dt and h_a to numbers (``eval_numeric``) -- and
compared with the oracle step on the same fp64 arrays with exact (unrounded)
FD weights.  The GPU kernels are compared with this oracle in the -m gpu
suite, so the chain reference equations -> oracle -> CUDA is closed for
acoustic, damped acoustic, TTI (two-field, nested derivatives), the rotated
G_xx operator and the collocated elastic system.  CPU only, seconds."""
import numpy as np
import pytest

from oracle import stencils as K
from paper_2312_13094_b200 import compiler as CP
from paper_2312_13094_b200 import symbolics as S

SHAPE = (9, 8, 7)
EXTENT = (80.0, 35.0, 60.0)  # h = (10, 5, 10): distinct spacing per axis
DT = 0.7


def _grid():
    return S.GridSpec(SHAPE, EXTENT)


def _eval(eq, arrays, box, h):
    """Solved rhs over ``box`` (FULL coordinates) with numpy fp64 leaves."""
    bind = {}
    for leaf in S.walk(eq.rhs):
        if isinstance(leaf, S.Symbol):
            bind[leaf] = DT if leaf.name == "dt" else h[S.AXIS_NAMES.index(leaf.name[2:])]
        elif isinstance(leaf, S.FieldAccess):
            arr = arrays[(leaf.spec.name, leaf.tshift)]
            bind[leaf] = arr[tuple(slice(lo + o, hi + o)
                                   for lo, hi, o in zip(box[0], box[1], leaf.offsets))]
    return S.eval_numeric(eq.rhs, bind)


def _setup(so, names, seed):
    rng = np.random.default_rng(seed)
    full = tuple(n + 2 * so for n in SHAPE)
    box = ((so,) * 3, tuple(so + n for n in SHAPE))
    arrays = {k: rng.standard_normal(full) for k in names}
    return arrays, box


def _weights(deriv, so, h):
    """Centre-out exact FD weights / h^deriv per axis (k = 0..r)."""
    w = [float(c) for c in S.fd_coefficients(deriv, so)]
    r = so // 2
    return [np.array([w[r + k] / hh ** deriv for k in range(r + 1)]) for hh in h]


def _close(a, b):
    scale = max(np.abs(b).max(), 1.0)
    assert np.abs(a - b).max() <= 1e-11 * scale, np.abs(a - b).max() / scale


@pytest.mark.parametrize("so", [2, 4, 8, 12, 16])
def test_oracle_acoustic_equals_solved_equation(so):
    g = _grid()
    u, m = S.FieldSpec("u", g, so, 2), S.FieldSpec("m", g, so, 0)
    eq = S.solve_forward(S.Eq(m.at() * u.dt2 - u.laplace), u.forward)
    arrays, box = _setup(so, [("u", 0), ("u", -1), ("m", 0)], 1)
    arrays[("m", 0)] = 0.2 + np.abs(arrays[("m", 0)])
    out = np.zeros_like(arrays[("u", 0)])
    K.star_update(arrays[("u", 0)], arrays[("u", -1)], arrays[("m", 0)],
                  _weights(2, so, g.spacing), 2.0, -1.0, DT * DT, box, out)
    _close(out[K._sl(box)], _eval(eq, arrays, box, g.spacing))


@pytest.mark.parametrize("so", [4, 8, 16])
def test_oracle_tti_equals_solved_equations(so):
    """The two-field TTI pair as nested Deriv(a * Deriv)
    equations (compiler.tti_updates, pinned to the reference by sha256)."""
    g = _grid()
    f = lambda n, to=0: S.FieldSpec(n, g, so, to)
    p, r, m, e, d = f("p", 2), f("r", 2), f("m"), f("epsp"), f("delp")
    a = (f("ax"), f("ay"), f("az"))
    eq_p, eq_r = CP.tti_updates(p, r, m, e, d, a)
    names = [("p", 0), ("p", -1), ("r", 0), ("r", -1), ("m", 0), ("epsp", 0), ("delp", 0),
             ("ax", 0), ("ay", 0), ("az", 0)]
    arrays, box = _setup(so, names, 2)
    arrays[("m", 0)] = 0.2 + np.abs(arrays[("m", 0)])
    p1 = np.zeros_like(arrays[("p", 0)])
    r1 = np.zeros_like(p1)
    d1 = [np.concatenate([[0.0], w[1:]]) for w in _weights(1, so, g.spacing)]
    K.tti_update(arrays[("p", 0)], arrays[("p", -1)], arrays[("r", 0)], arrays[("r", -1)],
                 arrays[("m", 0)], arrays[("epsp", 0)], arrays[("delp", 0)],
                 tuple(arrays[(n, 0)] for n in ("ax", "ay", "az")),
                 _weights(2, so, g.spacing), d1, DT * DT, box, p1, r1)
    _close(p1[K._sl(box)], _eval(eq_p, arrays, box, g.spacing))
    _close(r1[K._sl(box)], _eval(eq_r, arrays, box, g.spacing))


@pytest.mark.parametrize("so", [4, 8, 16])
def test_oracle_rotated_equals_solved_equation(so):
    """The SPEC's tti_gxx_kernel from compiler.rotated_update."""
    g = _grid()
    f = lambda n, to=0: S.FieldSpec(n, g, so, to)
    u, m, a = f("u", 2), f("m"), (f("ax"), f("ay"), f("az"))
    eq = CP.rotated_update(u, m, a)
    arrays, box = _setup(so, [("u", 0), ("u", -1), ("m", 0), ("ax", 0), ("ay", 0),
                              ("az", 0)], 3)
    arrays[("m", 0)] = 0.2 + np.abs(arrays[("m", 0)])
    out = np.zeros_like(arrays[("u", 0)])
    d1 = [np.concatenate([[0.0], w[1:]]) for w in _weights(1, so, g.spacing)]
    K.rot_update(arrays[("u", 0)], arrays[("u", -1)], arrays[("m", 0)],
                 tuple(arrays[(n, 0)] for n in ("ax", "ay", "az")), d1, DT * DT, box, out)
    _close(out[K._sl(box)], _eval(eq, arrays, box, g.spacing))


@pytest.mark.parametrize("so", [2, 4, 8, 16])
def test_oracle_collocated_elastic_equals_solved_equations(so):
    """The SPEC's elastic_kernel as nine first-order
    updates (compiler.elastic_updates): the oracle's velocity phase against
    the three velocity updates, its stress phase against the six stress
    updates (which read the new velocities, tshift +1)."""
    g = _grid()
    vn, tn = ("vx", "vy", "vz"), ("txx", "tyy", "tzz", "txy", "txz", "tyz")
    v = tuple(S.FieldSpec(n, g, so, 1) for n in vn)
    t = tuple(S.FieldSpec(n, g, so, 1) for n in tn)
    b, lam, mu = (S.FieldSpec(n, g, so, 0) for n in ("b", "lam", "mu"))
    eqs = CP.elastic_updates(v, t, b, lam, mu)
    names = ([(n, 0) for n in vn + tn] + [(n, 1) for n in vn]
             + [("b", 0), ("lam", 0), ("mu", 0)])
    arrays, box = _setup(so, names, 4)
    sc = [w[1:] for w in _weights(1, so, g.spacing)]
    v1 = [np.zeros_like(arrays[("vx", 0)]) for _ in vn]
    K.velocity_update([arrays[(n, 0)] for n in vn], [arrays[(n, 0)] for n in tn],
                      arrays[("b", 0)], sc, DT, box, v1, col=True)
    for i in range(3):
        _close(v1[i][K._sl(box)], _eval(eqs[i], arrays, box, g.spacing))
    t1 = [np.zeros_like(arrays[("vx", 0)]) for _ in tn]
    K.stress_update([arrays[(n, 1)] for n in vn], [arrays[(n, 0)] for n in tn],
                    arrays[("lam", 0)], arrays[("mu", 0)], sc, DT, box, t1, col=True)
    for i in range(6):
        _close(t1[i][K._sl(box)], _eval(eqs[3 + i], arrays, box, g.spacing))


@pytest.mark.parametrize("so", [4, 8, 16])
def test_oracle_damped_equals_solved_equation(so):
    """Acoustic with an absorbing layer, ``m*u.dt2 - u.laplace + damp*u.dt``
    solved by the reference's solve_forward: the oracle's var-star update
    with the closed-form A = (2m + d dt)/(m + d dt), B = -m/(m + d dt),
    S = dt^2/(m + d dt) equals the solved rhs, and so do the coefficients the
    product binds from the equation (compiler.VarStarKernel.coefficients)."""
    g = _grid()
    u, m, dmp = (S.FieldSpec("u", g, so, 2), S.FieldSpec("m", g, so, 0),
                 S.FieldSpec("damp", g, so, 0))
    eq = S.solve_forward(S.Eq(m.at() * u.dt2 - u.laplace + dmp.at() * u.dt), u.forward)
    arrays, box = _setup(so, [("u", 0), ("u", -1), ("m", 0), ("damp", 0)], 5)
    arrays[("m", 0)] = 0.2 + np.abs(arrays[("m", 0)])
    arrays[("damp", 0)] = np.abs(arrays[("damp", 0)])
    M, D = arrays[("m", 0)], arrays[("damp", 0)]
    A, B, Sc = (2 * M + D * DT) / (M + D * DT), -M / (M + D * DT), DT * DT / (M + D * DT)
    want = _eval(eq, arrays, box, g.spacing)
    lap = _weights(2, so, g.spacing)
    out = np.zeros_like(M)
    K.var_star_update(arrays[("u", 0)], arrays[("u", -1)], A, B, Sc, lap, box, out)
    _close(out[K._sl(box)], want)
    k = CP.recognise([eq])[0]
    assert isinstance(k, CP.VarStarKernel)
    s = K._sl(box)
    Ak, Bk, Sk = k.coefficients({m: M[s], dmp: D[s]}, DT, g.spacing)
    for got, ref in ((Ak, A[s]), (Bk, B[s]), (Sk, Sc[s])):
        _close(np.asarray(got), ref)


@pytest.mark.parametrize("so,nd", [(2, 2), (4, 2), (2, 3), (8, 3)])
def test_oracle_diffusion_equals_solved_equation(so, nd):
    """``Eq(u.dt, u.laplace)`` (Listing 1/4): forward
    Euler u1 = u0 + dt L(u0), in 2D and 3D."""
    shape, extent = SHAPE[:nd], EXTENT[:nd]
    g = S.GridSpec(shape, extent)
    u = S.FieldSpec("u", g, so, 1)
    eq = S.solve_forward(S.Eq(u.dt, u.laplace), u.forward)
    rng = np.random.default_rng(6)
    full = tuple(n + 2 * so for n in shape)
    box = ((so,) * nd, tuple(so + n for n in shape))
    arrays = {("u", 0): rng.standard_normal(full)}
    out = np.zeros(full)
    K.star_update(arrays[("u", 0)], None, None, _weights(2, so, g.spacing), 1.0, 0.0, DT,
                  box, out)
    _close(out[K._sl(box)], _eval(eq, arrays, box, g.spacing))
