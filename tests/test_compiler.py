"""Host-side compiler: family recognition by exact probing, HaloSpot
optimisation (drop / merge / hoist), ExecPlan structure per mode
(acceptance 4, 5, 8) and the C-ABI surface."""
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from paper_2312_13094_b200 import compiler as CP
from paper_2312_13094_b200 import decomposition as DC
from paper_2312_13094_b200 import symbolics as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def acoustic_eq(so, nd=3, n=16):
    g = S.GridSpec((n,) * nd, (10.0 * (n - 1),) * nd)
    u = S.FieldSpec("u", g, so, 2)
    m = S.FieldSpec("m", g, so, 0)
    return S.solve_forward(S.Eq(m.at() * u.dt2 - u.laplace), u.forward), u, m


@pytest.mark.parametrize("so", [2, 4, 6, 8, 12, 16])
@pytest.mark.parametrize("nd", [2, 3])
def test_recognise_acoustic(so, nd):
    eq, u, m = acoustic_eq(so, nd)
    k = CP.recognise([eq])[0]
    assert isinstance(k, CP.StarKernel)
    assert (k.A, k.B, k.c, k.p, k.q) == (2, -1, 1, 2, -1)
    assert k.m == m and k.radius == (so // 2,) * nd
    assert k.weights[0] == tuple(S.fd_coefficients(2, so)[so // 2:])


def test_recognise_diffusion_and_variants():
    g = S.GridSpec((8, 8), (2.0, 2.0))
    u = S.FieldSpec("u", g, 2, 1)
    k = CP.recognise([S.solve_forward(S.Eq(u.dt, u.laplace), u.forward)])[0]
    assert (k.A, k.B, k.c, k.p, k.q, k.m) == (1, 0, 1, 1, 0, None)
    # scaled diffusion u.dt = 3 * lap -> c = 3
    k = CP.recognise([S.solve_forward(S.Eq(u.dt, 3 * u.laplace), u.forward)])[0]
    assert (k.A, k.c, k.p) == (1, 3, 1)
    # heat with coefficient: m u.dt = lap -> S = dt / m
    m = S.FieldSpec("m", g, 2, 0)
    k = CP.recognise([S.solve_forward(S.Eq(m.at() * u.dt, u.laplace), u.forward)])[0]
    assert (k.p, k.q, k.m) == (1, -1, m)


def test_recognise_rejects_unsupported():
    g = S.GridSpec((8, 8), (2.0, 2.0))
    u = S.FieldSpec("u", g, 2, 1)
    for eq in [S.Eq(u.dt, u.dx), S.Eq(u.dt, u.laplace + u.dx)]:
        with pytest.raises(CP.CompilerError):
            CP.recognise([S.solve_forward(eq, u.forward)])


def test_halospots_drop_merge_hoist():
    eq, u, m = acoustic_eq(8)
    k = CP.recognise([eq])[0]
    an = CP.halo_phases([k, k], nranks=4)
    # two consecutive readers of u[t0] without a write in between -> 1 spot
    assert an.phases[0].halo is not None and an.phases[1].halo is None
    assert an.exchanges_per_step == 1
    # single rank -> no spots at all
    assert CP.halo_phases([k], nranks=1).exchanges_per_step == 0
    # TTI: read-only direction cosines hoisted out of the time loop
    g = S.GridSpec((16,) * 3, (150.0,) * 3)
    f = lambda n, to=0: S.FieldSpec(n, g, 8, to)
    tti = CP.TTIKernel(f("p", 2), f("r", 2), f("mt"), f("e"), f("d"),
                       (f("ax"), f("ay"), f("az")), 8)
    an = CP.halo_phases([tti], nranks=2)
    assert an.hoisted is not None and {x[0].name for x in an.hoisted.fields} == {"ax", "ay", "az"}
    assert an.hoisted.radius == (4, 4, 4)
    assert an.phases[0].halo.radius == (8, 8, 8)
    assert {x[0].name for x in an.phases[0].halo.fields} == {"p", "r"}


def test_elastic_two_exchanges_per_step():
    g = S.GridSpec((16,) * 3, (150.0,) * 3)
    v = tuple(S.FieldSpec(n, g, 8, 1) for n in ("vx", "vy", "vz"))
    t = tuple(S.FieldSpec(n, g, 8, 1) for n in ("txx", "tyy", "tzz", "txy", "txz", "tyz"))
    b, lam, mu = (S.FieldSpec(n, g, 8, 0) for n in ("b", "lam", "mu"))
    kv = CP.StaggeredPhase("v", v, t, (b,), so=8)
    kt = CP.StaggeredPhase("t", v, t, (lam, mu), so=8)
    an = CP.halo_phases([kv, kt], nranks=8)
    assert an.exchanges_per_step == 2
    assert [x[1] for x in an.phases[0].halo.fields] == [0] * 6   # tau[t0] before v
    assert [x[1] for x in an.phases[1].halo.fields] == [1] * 3   # v[t1] before tau


@pytest.mark.parametrize("collocated", [False, True])
def test_stress_halos_only_along_their_derivative_axes(collocated):
    """Per-field halo radii (Devito's per-function HaloScheme): the velocity
    update reads each stress only along the axes it differentiates it
    (v_i,t = b sum_j D_j tau_ij), so txx ships x faces only, tyy y faces
    only, tzz none (z is never split), shears their two axes; velocities
    every face.  Posts and fused pushes carry exactly those (field, face)
    pairs, which cuts a (2,2,1) rank's stress halo bytes in half."""
    g = S.GridSpec((32,) * 3, (150.0,) * 3)
    v = tuple(S.FieldSpec(n, g, 8, 1) for n in ("vx", "vy", "vz"))
    t = tuple(S.FieldSpec(n, g, 8, 1) for n in ("txx", "tyy", "tzz", "txy", "txz", "tyz"))
    b, lam, mu = (S.FieldSpec(n, g, 8, 0) for n in ("b", "lam", "mu"))
    kv = CP.StaggeredPhase("v", v, t, (b,), so=8, collocated=collocated)
    kt = CP.StaggeredPhase("t", v, t, (lam, mu), so=8, collocated=collocated)
    d = DC.Decomposition.create((64, 64, 32), 4, (2, 2, 1))
    an = CP.halo_phases([kv, kt], d.nranks)
    spot_t, spot_v = an.phases[0].halo, an.phases[1].halo
    assert spot_t.radius == (4, 4, 4)
    faces = {"x": (1, 0, 0), "y": (0, 1, 0), "xy": (1, 1, 0)}
    want = {"txx": {"x"}, "tyy": {"y"}, "tzz": set(), "txy": {"x", "y", "xy"},
            "txz": {"x"}, "tyz": {"y"}}
    for f, tt in spot_t.fields:
        got = {k for k, dvec in faces.items() if spot_t.sends(f, tt, dvec)}
        assert got == want[f.name], f.name
    assert all(spot_v.sends(f, tt, dvec) for f, tt in spot_v.fields for dvec in faces.values())
    # basic: the x step ships txx, txy, txz; the y step tyy, txy, tyz
    posts = [a for a in CP.lower_mode(an, d, 0, "basic").actions
             if a.kind == "post" and a.spot is spot_t]
    shipped = [{f.name for f, tt in a.spot.fields
                if any(a.spot.sends(f, tt, m.direction) for m in a.messages)} for a in posts]
    assert shipped[:2] == [{"txx", "txy", "txz"}, {"tyy", "txy", "tyz"}]
    for mode in ("diagonal", "full"):
        p = CP.lower_mode(an, d, 0, mode)
        post = [a for a in p.actions if a.kind == "post"][0]
        full_vol = sum(m.volume * len(post.spot.fields) for m in post.messages)
        sent = sum(m.volume * sum(post.spot.sends(f, tt, m.direction)
                                  for f, tt in post.spot.fields) for m in post.messages)
        # rank 0 of (2,2,1): one x face, one y face, one corner per field
        assert 2 * sent < full_vol
        if mode == "full":
            slabs = [a for a in p.actions if a.kind == "compute" and a.region == "OWNED"
                     and a.kernel is kt]
            assert slabs
            for a in slabs:
                outs, msgs, sends = a.push
                for f, fs in zip(outs, sends):
                    for m, s_ in zip(msgs, fs):
                        assert s_ == spot_t.sends(f, 0, m.direction)


def plan_for(mode, dims=(2, 2, 1), rank=0, shape=(32, 32, 32)):
    eq, u, m = acoustic_eq(8, 3, 32)
    k = CP.recognise([eq])[0]
    d = DC.Decomposition.create(shape, int(np.prod(dims)), dims)
    an = CP.halo_phases([k], d.nranks)
    return CP.lower_mode(an, d, rank, mode)


def test_full_mode_listing8_order():
    p = plan_for("full")
    kinds = [a.kind if a.kind != "compute" else a.region for a in p.actions]
    post, core, wait = kinds.index("post"), kinds.index("CORE"), kinds.index("wait")
    owned = [i for i, k in enumerate(kinds) if k == "OWNED"]
    assert post < core < wait < min(owned)  # Listing 8 (acceptance 8)
    core_a = p.actions[core]
    wait_a = p.actions[wait]
    assert core_a.stream != wait_a.stream  # CORE overlaps the exchange
    assert p.phases_per_step == 1


def test_basic_and_diagonal_structure():
    b = plan_for("basic")
    posts = [a for a in b.actions if a.kind == "post"]
    assert len(posts) == 3 and b.phases_per_step == 3  # axis-sequenced x, y, z
    assert [len(a.messages) for a in posts] == [1, 1, 0]
    d = plan_for("diagonal")
    assert [len(a.messages) for a in d.actions if a.kind == "post"] == [3]
    assert [a.region for a in d.actions if a.kind == "compute"] == ["DOMAIN"]


def test_interior_message_counts_3d():
    for mode, want in (("basic", 6), ("diagonal", 26), ("full", 26)):
        p = plan_for(mode, dims=(3, 3, 3), rank=13, shape=(48, 48, 48))
        assert p.message_count() == want


def test_mode_aliases():
    assert CP.normalise_mode("diag2") == "diagonal"
    assert CP.normalise_mode("1") == "basic"
    assert CP.normalise_mode("FULL") == "full"
    with pytest.raises(CP.CompilerError):
        CP.normalise_mode("nope")


def test_c_abi_library_exports_every_declared_symbol():
    from paper_2312_13094_b200 import runtime as R
    lib = R.lib()
    with open(os.path.join(ROOT, "include", "sdmp.h")) as f:
        declared = set(re.findall(r"\b(sdmp_[a-z0-9_]+)\s*\(", f.read()))
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.sdmp_version() == 1
    # error path without touching a GPU
    assert lib.sdmp_plan_add_action(None, None, 0, None, 0) == -1
    assert b"null" in lib.sdmp_last_error()


def _format_access(eq):
    return S.format_equation(eq)


def test_align_accesses_spec_examples():
    g = S.GridSpec((8, 8), (7.0, 7.0))
    u = S.FieldSpec("u", g, 2, 1)
    eq = S.StencilEquation(u.forward, u.at() + u.at(offsets=(-1, 0)))
    al = CP.align_accesses(eq, (2, 2))
    accs = sorted((a.tshift, a.offsets) for a in S.accesses(al.rhs))
    assert accs == [(0, (1, 2)), (0, (2, 2))]           # u[t,x-1,y] -> u[t,x+1,y+2]
    assert al.lhs.offsets == (2, 2)                       # u[t,x,y] -> u[t,x+2,y+2]
    ident = CP.align_accesses(eq, (0, 0))
    assert S.format_equation(ident) == S.format_equation(eq)
    # default: each field's own halo (SO-2 -> 1)
    assert CP.align_accesses(eq).lhs.offsets == tuple(u.halo)


def test_dump_plan_listings():
    eq, u, m = acoustic_eq(8, 3, 32)
    k = CP.recognise([eq])[0]
    pre = CP.dump_plan([k], 4, None, [eq])
    assert "<HaloSpot(u)>" in pre and "Iteration time" in pre
    basic = CP.dump_plan([k], 4, "basic", [eq])
    assert "HaloUpdateCall" in basic and "HaloWaitList" in basic
    full = CP.dump_plan([k], 4, "full", [eq])
    assert full.index("CORE") < full.index("HaloWaitList") < full.index("REMAINDER")
    assert "HaloSpot" not in CP.dump_plan([k], 1, None, [eq])


@pytest.mark.parametrize("dims", [(4, 2, 1), (2, 2, 1), (4, 1, 1)])
def test_full_mode_fused_push_covers_every_send_box(dims):
    """Host logic of the fused exchange for every rank of the 8-GPU layout:
    each message's send box lies inside the union of the OWNED slabs that push
    it (so every halo value a neighbour reads is stored by a slab kernel), the
    push lists fit the 8-direction limit, and CORE never intersects a send box."""
    from paper_2312_13094_b200.distfield import diagonal_messages
    eq, u, m = acoustic_eq(8, 3, 32)
    k = CP.recognise([eq])[0]
    shape = tuple(32 * d for d in dims)
    d = DC.Decomposition.create(shape, int(np.prod(dims)), dims)
    an = CP.halo_phases([k], d.nranks)
    for rank in range(d.nranks):
        p = CP.lower_mode(an, d, rank, "full")
        posts = [a for a in p.actions if a.kind == "post"]
        assert posts and all(a.pushed for a in posts)
        slabs = [a for a in p.actions if a.kind == "compute" and a.region == "OWNED"]
        core = [a for a in p.actions if a.kind == "compute" and a.region == "CORE"]
        msgs = diagonal_messages(d, rank, k.radius)
        assert all(a.push is not None and len(a.push[1]) <= 8 for a in slabs)
        covered = np.zeros(d.local_shape(rank), dtype=bool)
        for a in slabs:
            covered[tuple(slice(lo, hi) for lo, hi in zip(*a.box))] = True
        for msg in msgs:
            box = tuple(slice(lo, hi) for lo, hi in zip(*msg.send))
            assert covered[box].all(), (rank, msg)
            for c in core:
                inter = [max(a0, b0) < min(a1, b1) for a0, a1, b0, b1 in
                         zip(c.box[0], c.box[1], msg.send[0], msg.send[1])]
                assert not all(inter), (rank, msg)


def test_dump_plan_tti_and_staggered():
    g = S.GridSpec((16,) * 3, (150.0,) * 3)
    f = lambda n, to=0, so=8: S.FieldSpec(n, g, so, to)
    tti = CP.TTIKernel(f("p", 2), f("r", 2), f("mt"), f("e"), f("d"), (f("ax"), f("ay"), f("az")), 8)
    txt = CP.dump_plan([tti], 2, "full")
    assert "HaloUpdateCall(ax,ay,az) once" in txt and "CORE" in txt
    v = tuple(f(n, 1) for n in ("vx", "vy", "vz"))
    t = tuple(f(n, 1) for n in ("txx", "tyy", "tzz", "txy", "txz", "tyz"))
    kv = CP.StaggeredPhase("v", v, t, (f("b"),), so=8)
    kt = CP.StaggeredPhase("t", v, t, (f("lam"), f("mu")), so=8)
    txt = CP.dump_plan([kv, kt], 4, "diagonal")
    assert txt.count("HaloWaitList") == 2  # tau before v, v before tau


def test_recognise_rotated_gxx_golden_form():
    """The SPEC's tti_gxx_kernel written as in tests/golden/make_golden.py
    (m u.dt2 - sum_i D_i(a_i sum_j a_j D_j u), solved by the reference
    symbolics) is recognised as the rotated family; a perturbed update is not."""
    g = S.GridSpec((16,) * 3, (150.0,) * 3)
    u = S.FieldSpec("u", g, 4, 2)
    m = S.FieldSpec("m", g, 4, 0)
    a = [S.FieldSpec(f"a{S.AXIS_NAMES[i]}", g, 4, 0) for i in range(3)]
    inner = S.add(*(S.mul(a[j].at(), u.d(j)) for j in range(3)))
    gxx = S.add(*(S.Deriv(S.mul(a[i].at(), inner), i, 1) for i in range(3)))
    eq = S.solve_forward(S.Eq(m.at() * u.dt2 - gxx), u.forward)
    k = CP.recognise([eq])[0]
    assert isinstance(k, CP.RotatedKernel) and k.m == m and [f.name for f in k.a] == ["ax", "ay", "az"]
    assert k.reads()[0] == (u, 0, (4, 4, 4))
    # swapped direction cosines in the inner derivative: a different operator
    bad_inner = S.add(S.mul(a[1].at(), u.d(0)), S.mul(a[0].at(), u.d(1)), S.mul(a[2].at(), u.d(2)))
    bad = S.add(*(S.Deriv(S.mul(a[i].at(), bad_inner), i, 1) for i in range(3)))
    with pytest.raises(CP.CompilerError):
        CP.recognise([S.solve_forward(S.Eq(m.at() * u.dt2 - bad), u.forward)])


# --- multi-update families written as equations -----------------------------

def _tti_fields(so, n=16):
    g = S.GridSpec((n,) * 3, (10.0 * (n - 1),) * 3)
    F = lambda name, to: S.FieldSpec(name, g, so, to)
    return (F("p", 2), F("r", 2), F("m", 0), F("epsp", 0), F("delp", 0),
            [F("ax", 0), F("ay", 0), F("az", 0)])


@pytest.mark.parametrize("so", [4, 8])
def test_recognise_tti_pair_from_equations(so):
    """The paper's two-field TTI written as Eqs is
    recognised as ONE TTI kernel whatever the equation order, and the roles
    of its static fields come out of the exact probe, not their names."""
    p, r, m, e, d, a = _tti_fields(so)
    eq_p, eq_r = CP.tti_updates(p, r, m, e, d, a)
    for eqs in ([eq_p, eq_r], [eq_r, eq_p]):
        ks = CP.recognise(eqs)
        assert len(ks) == 1 and isinstance(ks[0], CP.TTIKernel)
        k = ks[0]
        assert (k.p, k.r, k.m, k.epsp, k.delp, k.a, k.so) == (p, r, m, e, d, tuple(a), so)
    # the same system with m and delp (and two direction cosines) swapped
    eq_p2, eq_r2 = CP.tti_updates(p, r, d, e, m, [a[2], a[1], a[0]])
    k = CP.recognise([eq_p2, eq_r2])[0]
    assert (k.m, k.delp, k.a) == (d, m, (a[2], a[1], a[0]))
    # a user-written equivalent form: p.dt2 = (...)/m, solved by the reference solver
    gzz = lambda f: S.add(*(S.Deriv(S.mul(a[i].at(), S.add(*(S.mul(a[j].at(), f.d(j))
                                                                for j in range(3)))), i, 1)
                            for i in range(3)))
    h0 = p.laplace - gzz(p)
    user_p = S.solve_forward(S.Eq(p.dt2, (e.at() * h0 + d.at() * gzz(r)) / m.at()), p.forward)
    user_r = S.solve_forward(S.Eq(r.dt2, (d.at() * h0 + gzz(r)) / m.at()), r.forward)
    assert isinstance(CP.recognise([user_r, user_p])[0], CP.TTIKernel)


def test_tti_wrong_physics_rejected():
    p, r, m, e, d, a = _tti_fields(4)
    gzz = lambda f: S.add(*(S.Deriv(S.mul(a[i].at(), S.add(*(S.mul(a[j].at(), f.d(j))
                                                                for j in range(3)))), i, 1)
                            for i in range(3)))
    h0 = p.laplace - gzz(p)
    # sign flip on the coupling term: not the TTI system
    bad_p = S.solve_forward(S.Eq(m.at() * p.dt2, e.at() * h0 - d.at() * gzz(r)), p.forward)
    good_r = CP.tti_updates(p, r, m, e, d, a)[1]
    with pytest.raises(CP.CompilerError, match="not recognised"):
        CP.recognise([bad_p, good_r])


def _elastic_fields(so, n=16):
    g = S.GridSpec((n,) * 3, (10.0 * (n - 1),) * 3)
    F = lambda name, to: S.FieldSpec(name, g, so, to)
    v = [F(x, 1) for x in ("vx", "vy", "vz")]
    t = [F(x, 1) for x in ("txx", "tyy", "tzz", "txy", "txz", "tyz")]
    return v, t, F("b", 0), F("lam", 0), F("mu", 0)


@pytest.mark.parametrize("so", [4, 8, 16])
def test_recognise_collocated_elastic_from_equations(so):
    """The SPEC's elastic_kernel as nine Eqs -> the
    velocity and stress phases, in that order, with roles read off the
    access structure (field names are irrelevant)."""
    v, t, b, lam, mu = _elastic_fields(so)
    eqs = CP.elastic_updates(v, t, b, lam, mu)
    import random
    random.Random(so).shuffle(eqs)
    kv, kt = CP.recognise(eqs)
    assert (kv.kind, kt.kind) == ("v", "t") and kv.collocated and kt.collocated
    assert kv.v == tuple(v) and kv.tau == tuple(t) and kv.params == (b,)
    assert kt.params == (lam, mu) and kv.so == so
    # relabelled: components given in another order still map to their roles
    v2 = [v[1], v[2], v[0]]
    t2 = [t[1], t[2], t[0], t[5], t[3], t[4]]  # yy,zz,xx,(yz as xy)...
    eqs2 = CP.elastic_updates(v2, t2, b, lam, mu)
    kv2, kt2 = CP.recognise(eqs2)
    assert kv2.v == tuple(v2) and kv2.tau == tuple(t2)


def test_elastic_wrong_physics_rejected():
    v, t, b, lam, mu = _elastic_fields(4)
    eqs = CP.elastic_updates(v, t, b, lam, mu)
    # txy with a factor 2 on the shear strain: not the elastic system
    dv = lambda i, j: S.Deriv(v[i].forward, j, 1)
    bad = S.solve_forward(S.Eq(t[3].dt, S.mul(S.Const(Fraction(2)), mu.at(),
                                               S.add(dv(0, 1), dv(1, 0)))), t[3].forward)
    eqs = [bad if e.lhs.spec == t[3] else e for e in eqs]
    with pytest.raises(CP.CompilerError, match="not recognised"):
        CP.recognise(eqs)


def test_sparse_term_on_unused_field_raises():
    """A receiver on a field no kernel of the Operator reads (or a source
    into a field none writes) is an error, not a silently empty trace."""
    from paper_2312_13094_b200 import api
    grid = api.Grid((12, 12, 12), (110.0,) * 3, comm="self")
    u = api.TimeFunction("u_sp", grid, space_order=4, time_order=2)
    m = api.Function("m_sp", grid, space_order=4)
    w = api.TimeFunction("w_sp", grid, space_order=4, time_order=2)
    eq = S.solve_forward(S.Eq(m.at() * u.dt2 - u.laplace), u.forward)
    rec = api.SparseTimeFunction("rec_sp", grid, 2, 4, coordinates=[(10.0,) * 3, (20.0,) * 3])
    op = api.Operator([eq, rec.interpolate(w)])
    with pytest.raises(CP.CompilerError, match="no kernel"):
        op.plan("diagonal")
    op2 = api.Operator([eq, rec.interpolate(u)])
    assert any(a.kind == "interp" for a in op2.plan("diagonal").actions)
