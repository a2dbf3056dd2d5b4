"""End-to-end parity through the public API (Operator.apply -> libsdmp) vs
the oracle, single rank, every kernel family and every mpi mode.

Tolerance (north star): rel-L2 <= 1e-5 on wavefields and receiver traces,
max-abs reported in the assertion message.  Parameters are bound to fp32
once and the SAME fp32 values (read back from the device) feed the oracle.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import problems as P  # noqa: E402
from oracle.runtime import Simulation  # noqa: E402
from paper_2312_13094_b200 import (Eq, Function, Grid, Operator, SparseTimeFunction,  # noqa: E402
                                   TimeFunction, kernels as KD, solve, symbolics as S)

REL = 1e-5


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def star_coeffs(so, h):
    w = [float(c) for c in S.fd_coefficients(2, so)]
    r = so // 2
    return [np.float32([w[r + k] / (hh * hh) for k in range(r + 1)]).astype(np.float64)
            for hh in h]


@pytest.mark.parametrize("mode", ["basic", "diagonal", "full"])
def test_listing4_through_api(mode):
    nx = ny = 4
    dx = 2.0 / (nx - 1)
    dt = 0.25 * dx * dx / 0.5
    grid = Grid(shape=(nx, ny), extent=(2.0, 2.0))
    u = TimeFunction(name=f"u_l4_{mode}", grid=grid, space_order=2)
    u.data[1:-1, 1:-1] = 1
    op = Operator([Eq(u.forward, solve(Eq(u.dt, u.laplace), u.forward))])
    op.apply(time_M=1, dt=dt, mpi=mode)
    a, b = 0.5, -0.25
    want = np.array([[a, b, b, a], [b, a, a, b], [b, a, a, b], [a, b, b, a]])
    got = u.data[:]
    assert np.abs(got - want).max() < 1e-6, got


def run_acoustic(shape, so, steps, mode, tag, nrec=7):
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.acoustic_model(grid, so=so, name=f"u_{tag}")
    u, m = kd.fields["u"], kd.fields["m"]
    dt = np.float32(KD.critical_dt(4.6, grid.spacing))
    ext = grid.extent
    src = KD.point_source(grid, [tuple(0.5 * e + 1.3 for e in ext)], steps, float(dt),
                          f0=0.030, name=f"src_{tag}")
    rec = SparseTimeFunction(f"rec_{tag}", grid, nrec, steps,
                             coordinates=np.stack([np.linspace(5.0, ext[0] - 5.0, nrec)] +
                                                  [np.full(nrec, 0.37 * e) for e in ext[1:]], 1))
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
    op.apply(time_M=steps - 1, dt=float(dt), mpi=mode)
    return grid, u, m, src, rec, float(dt)


@pytest.mark.parametrize("so", [4, 8, 12, 16])
def test_acoustic_vs_oracle(so):
    shape, steps = (40, 36, 44), 30
    grid, u, m, src, rec, dt = run_acoustic(shape, so, steps, "diagonal", f"a{so}")
    mv = m.data_gather().astype(np.float64)
    C = float(np.float32(dt * dt))
    h = grid.spacing
    sp = P.SparseSpec(shape, h, src.coordinates, src.data.astype(np.float64), "u", ("m", C),
                      rec.coordinates, "u")
    prob = P.star(3, so, star_coeffs(so, h), 2.0, -1.0, C, True, sparse=sp, shape=shape)
    sim = Simulation(prob, shape)
    sim.write_global("m", mv)
    sim.run(0, steps - 1)
    want = sim.gather("u", steps % 3)
    got = u.data_gather()
    err = rel_l2(got, want)
    assert err <= REL, (err, np.abs(got - want).max())
    traces_want = np.array([sim.traces[t] for t in range(steps)])
    terr = rel_l2(rec.data, traces_want)
    assert terr <= REL, (terr, np.abs(rec.data - traces_want).max())
    assert np.abs(want).max() > 0 and np.abs(traces_want).max() > 0


def test_modes_bitwise_equal_single_rank():
    outs = []
    for mode in ("basic", "diagonal", "full"):
        _g, u, _m, _s, rec, _dt = run_acoustic((24, 20, 28), 8, 12, mode, f"mb_{mode}")
        outs.append((u.data_gather(), rec.data.copy()))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


@pytest.mark.parametrize("so", [4, 6, 8, 12, 16])
def test_tti_vs_oracle(so):
    shape, steps = (28, 24, 32), 10
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.tti_model(grid, so=so)
    p, r = kd.fields["p"], kd.fields["r"]
    rng = np.random.default_rng(0)
    init = np.float32(rng.standard_normal(shape))
    p.data[:] = init
    r.data[:] = 0.5 * init
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
    op = Operator([kd])
    op.apply(time_M=steps - 1, dt=dt)
    h = grid.spacing
    rr = so // 2
    d1 = [float(c) for c in S.fd_coefficients(1, so)]
    d1_c = [np.float32([0.0] + [d1[rr + k] / hh for k in range(1, rr + 1)]).astype(np.float64)
            for hh in h]
    sim = Simulation(P.tti(so, star_coeffs(so, h), d1_c, float(np.float32(dt * dt))), shape)
    for name in ("m", "epsp", "delp", "ax", "ay", "az"):
        sim.write_global(name, kd.fields[name].data_gather().astype(np.float64))
    sim.write_global("p", init.astype(np.float64))
    sim.write_global("r", 0.5 * init.astype(np.float64))
    sim.run(0, steps - 1)
    for name, fn in (("p", p), ("r", r)):
        want = sim.gather(name, steps % 3)
        got = fn.data_gather()
        err = rel_l2(got, want)
        assert err <= REL, (name, err, np.abs(got - want).max())


@pytest.mark.parametrize("visco,so", [(False, 4), (False, 8), (False, 12), (False, 16),
                                     (True, 4), (True, 8), (True, 16)])
def test_elastic_vs_oracle(visco, so):
    shape, steps = (24, 28, 20), 8
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.viscoelastic_model(grid, so=so) if visco else KD.elastic_model(grid, so=so)
    rng = np.random.default_rng(1)
    t0 = np.float32(rng.standard_normal(shape))
    kd.fields["txx"].data[:] = t0
    kd.fields["tzz"].data[:] = -t0
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1)))
    Operator([kd]).apply(time_M=steps - 1, dt=dt)
    h = grid.spacing
    sc = [np.float32([float(c) / hh for c in S.staggered_coefficients(so)]).astype(np.float64)
          for hh in h]
    sim = Simulation(P.elastic(so, sc, float(np.float32(dt)), visco=visco), shape)
    params = ("b", "l2m", "mus", "its") if visco else ("b", "lam", "mu")
    for name in params:
        sim.write_global(name, kd.fields[name].data_gather().astype(np.float64))
    sim.write_global("txx", t0.astype(np.float64))
    sim.write_global("tzz", -t0.astype(np.float64))
    sim.run(0, steps - 1)
    names = P.VNAMES + P.TNAMES + (P.RNAMES if visco else ())
    for name in names:
        want = sim.gather(name, steps % 2)
        got = kd.fields[name].data_gather()
        err = rel_l2(got, want)
        assert err <= REL, (name, err, np.abs(got - want).max())


@pytest.mark.parametrize("so,shape", [(4, (40, 36, 44)), (8, (40, 36, 44)), (12, (40, 36, 44)),
                                      (16, (40, 36, 44)), (14, (44, 60, 300)),
                                      (16, (90, 80, 300))])
def test_star_kernels_bitwise_equal_generic(so, shape, monkeypatch):
    """star_tma (one row per warp), star_tma2 (two rows per thread, register
    x-window, SO >= 12), star_tmem (x-window in tensor memory, SO-16) and the
    generic kernel give identical bits; the larger shapes run several y / z
    tiles, partial tiles and x chunks."""
    outs = []
    for variant in ("1", "0", "3", "4"):
        monkeypatch.setenv("SDMP_STAR_VARIANT", variant)
        import paper_2312_13094_b200.api as A
        A._FUNCS.clear()
        _g, u, _m, _s, rec, _dt = run_acoustic(shape, so, 8 if shape[2] < 100 else 24,
                                               "diagonal", f"sb{so}_{variant}")
        outs.append((u.data_gather(), rec.data.copy()))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])
    assert np.abs(outs[0][0]).max() > 0


@pytest.mark.parametrize("family,so", [("tti", 4), ("tti", 6), ("tti", 8), ("tti", 12),
                                       ("tti", 16), ("rotated", 4), ("rotated", 6),
                                       ("rotated", 8), ("rotated", 12), ("elastic", 8),
                                       ("elastic", 4), ("elastic", 16), ("visco", 16),
                                       ("visco", 8)])
def test_stream_kernels_bitwise_equal_generic(family, so, monkeypatch):
    """TMA streaming launches (thick boxes) and generic launches (thin OWNED
    slabs) share one per-point routine: results must agree bit for bit."""
    shape, steps = (40, 36, 44), 6
    outs = []
    for variant in ("1", "0"):
        monkeypatch.setenv("SDMP_TTI_VARIANT", variant)
        monkeypatch.setenv("SDMP_STAGGERED_VARIANT", variant)
        import paper_2312_13094_b200.api as A
        A._FUNCS.clear()
        grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
        if family == "tti":
            kd = KD.tti_model(grid, so=so)
            names = ("p", "r")
            dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
        elif family == "rotated":
            kd = KD.rotated_model(grid, so=so, name=f"urb{so}_{variant}")
            names = ("u", "u")
            dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
        else:
            kd = (KD.viscoelastic_model(grid, so=so) if family == "visco"
                  else KD.elastic_model(grid, so=so))
            names = KD.VNAMES + KD.TNAMES
            dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1)))
        rng = np.random.default_rng(7)
        kd.fields[names[0]].data[:] = np.float32(rng.standard_normal(shape))
        kd.fields[names[-1]].data[:] = np.float32(rng.standard_normal(shape))
        Operator([kd]).apply(time_M=steps - 1, dt=dt)
        outs.append([kd.fields[n].data_gather() for n in names])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
        assert np.abs(a).max() > 0


def test_graph_replay_long_run(monkeypatch):
    res = []
    for g in ("0", "1"):
        monkeypatch.setenv("SDMP_GRAPH", g)
        import paper_2312_13094_b200.api as A
        A._FUNCS.clear()
        shape = (24, 20, 28)
        grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
        kd = KD.acoustic_model(grid, so=8, name="ug")
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        steps = 23
        src = KD.point_source(grid, [tuple(0.5 * e + 1.3 for e in grid.extent)], steps, dt,
                              f0=0.03, name="srcg")
        rec = SparseTimeFunction("recg", grid, 5, steps,
                                 coordinates=[(5.0 + 40 * i, 60.0, 70.0) for i in range(5)])
        op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
        op.apply(time_M=2, dt=dt)          # first run: no graphs
        op.apply(time_m=3, time_M=steps - 1, dt=dt)  # 20 steps: 6 periods + 2
        res.append((u.data_gather(), rec.data.copy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert np.abs(res[1][1]).max() > 0


def test_static_field_update_between_applies():
    """dt^2/m is re-bound only when m changes (Data writes bump its version):
    changing m between two applies must give the same result as an operator
    built on the changed m from the start; an unchanged m is not re-bound."""
    shape, so, steps = (24, 20, 28), 8, 8

    def build(tag):
        grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
        kd = KD.acoustic_model(grid, so=so, name=f"u_{tag}")
        u, m = kd.fields["u"], kd.fields["m"]
        u.data[:, 10, 10, 14] = 1.0
        return u, m, Operator([kd])

    dt = float(np.float32(KD.critical_dt(4.6 * 1.5, (10.0,) * 3)))  # stable for m / 2 too
    u1, m1, op1 = build("sv1")
    op1.apply(time_M=0, dt=dt)           # binds dt^2/m with the original m
    m1.data[...] = m1.data[...] * np.float32(0.5)
    u1.data[...] = 0.0
    u1.data[:, 10, 10, 14] = 1.0
    op1.apply(time_M=steps - 1, dt=dt)
    u2, m2, op2 = build("sv2")
    m2.data[...] = m2.data[...] * np.float32(0.5)
    op2.apply(time_M=steps - 1, dt=dt)
    assert np.array_equal(u1.data_gather(), u2.data_gather())


@pytest.mark.parametrize("so", [4, 8, 16])
def test_damped_acoustic_vs_oracle(so):
    """Acoustic with an absorbing layer (m u.dt2 - lap u + damp u.dt, solved by
    the reference symbolics) -> variable-coefficient star; A, B, S bound on
    the device and the same fp32 values fed to the oracle."""
    shape, steps = (40, 36, 44), 30
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.damped_acoustic_model(grid, so=so, nbl=6, name=f"ud{so}")
    u, m = kd.fields["u"], kd.fields["m"]
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
    ext = grid.extent
    src = KD.point_source(grid, [tuple(0.5 * e + 1.3 for e in ext)], steps, dt, f0=0.030,
                          name=f"srcd{so}")
    rec = SparseTimeFunction(f"recd{so}", grid, 7, steps,
                             coordinates=np.stack([np.linspace(5.0, ext[0] - 5.0, 7)] +
                                                  [np.full(7, 0.37 * e) for e in ext[1:]], 1))
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
    assert type(op.kernels[0]).__name__ == "VarStarKernel"
    op.apply(time_M=steps - 1, dt=dt, mpi="full")
    plan = next(iter(op._plans.values()))
    _k, ufn, bufs = plan.var_bufs[0]
    dom = tuple(slice(hh, hh + n) for hh, n in zip(ufn.halo3, ufn.local3))
    coef = {n: b[dom].double().cpu().numpy() for n, b in bufs.items()}
    C = float(np.float32(dt * dt))
    h = grid.spacing
    sp = P.SparseSpec(shape, h, src.coordinates, src.data.astype(np.float64), "u", ("m", C),
                      rec.coordinates, "u")
    prob = P.var_star(3, so, star_coeffs(so, h), True, sparse=sp, shape=shape, extra=("m",))
    sim = Simulation(prob, shape)
    for n in ("A", "B", "S"):
        sim.write_global(n, coef[n])
    sim.write_global("m", m.data_gather().astype(np.float64))
    sim.run(0, steps - 1)
    want = sim.gather("u", steps % 3)
    got = u.data_gather()
    err = rel_l2(got, want)
    assert err <= REL, (err, np.abs(got - want).max())
    tw = np.array([sim.traces[t] for t in range(steps)])
    terr = rel_l2(rec.data, tw)
    assert terr <= REL, terr
    assert np.abs(tw).max() > 0 and np.abs(want).max() > 0
    # the layer damps: the coefficient arrays differ from the undamped (2, -1) inside it
    assert coef["A"].max() > 2.0 - 1e-6 and coef["B"].min() > -1.0 - 1e-6
    assert np.any(coef["B"] > -0.999)


@pytest.mark.parametrize("so,shape", [(4, (40, 36, 44)), (8, (40, 36, 44)), (8, (70, 80, 300)),
                                      (16, (40, 36, 44))])
def test_damped_kernels_bitwise_equal_generic(so, shape, monkeypatch):
    """The variable-coefficient (damped) family: the stream-engine kernel and
    the generic one-thread-per-point kernel give identical bits in every mode
    (r04 A/B: a star_tma variant with per-point A, B lost 1-1.5% to the
    engine at SO-4/8, profiles/round2_ab_damped_star.txt)."""
    outs = []
    for variant in ("1", "0"):
        monkeypatch.setenv("SDMP_STAR_VARIANT", variant)
        import paper_2312_13094_b200.api as A
        A._FUNCS.clear()
        grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
        kd = KD.damped_acoustic_model(grid, so=so, nbl=6, name=f"udb{so}_{variant}")
        u, m = kd.fields["u"], kd.fields["m"]
        steps = 12
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        ext = grid.extent
        src = KD.point_source(grid, [tuple(0.5 * e + 1.3 for e in ext)], steps, dt, f0=0.030,
                              name=f"srcdb{so}_{variant}")
        op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m)])
        res = []
        for mode in ("diagonal", "full"):
            u.data[...] = 0.0
            op.apply(time_M=steps - 1, dt=dt, mpi=mode)
            res.append(u.data_gather())
        outs.append(res)
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    assert np.abs(outs[0][0]).max() > 0


@pytest.mark.parametrize("so", [4, 6, 8, 12])
def test_rotated_gxx_vs_oracle(so):
    """The SPEC's tti_gxx_kernel (single-field rotated operator) through the
    public API vs the oracle on the same fp32 fields."""
    shape, steps = (28, 24, 32), 8
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.rotated_model(grid, so=so, name=f"ur{so}")
    u = kd.fields["u"]
    rng = np.random.default_rng(so)
    init = np.float32(rng.standard_normal(shape))
    u.data[:] = init
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
    op = Operator([kd])
    assert type(op.kernels[0]).__name__ == "RotatedKernel"
    op.apply(time_M=steps - 1, dt=dt, mpi="full")
    h = grid.spacing
    r = so // 2
    w1 = [float(c) for c in S.fd_coefficients(1, so)]
    d1 = [np.float32([0.0] + [w1[r + k] / hh for k in range(1, r + 1)]).astype(np.float64)
          for hh in h]
    sim = Simulation(P.rotated(so, d1, float(np.float32(dt * dt))), shape)
    for name in ("m", "ax", "ay", "az"):
        sim.write_global(name, kd.fields[name].data_gather().astype(np.float64))
    sim.write_global("u", init.astype(np.float64))
    sim.run(0, steps - 1)
    want = sim.gather("u", steps % 3)
    got = u.data_gather()
    err = rel_l2(got, want)
    assert err <= REL, (err, np.abs(got - want).max())


@pytest.mark.parametrize("so", [4, 8, 16])
def test_collocated_elastic_vs_oracle(so):
    """The SPEC's collocated elastic_kernel vs the oracle."""
    shape, steps = (24, 28, 20), 8
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.elastic_model(grid, so=so, collocated=True)
    rng = np.random.default_rng(2)
    t0 = np.float32(rng.standard_normal(shape))
    kd.fields["txx"].data[:] = t0
    kd.fields["tyz"].data[:] = 0.5 * t0
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1)))
    Operator([kd]).apply(time_M=steps - 1, dt=dt, mpi="full")
    r = so // 2
    w1 = [float(c) for c in S.fd_coefficients(1, so)]
    sc = [np.float32([w1[r + k] / hh for k in range(1, r + 1)]).astype(np.float64)
          for hh in grid.spacing]
    sim = Simulation(P.elastic(so, sc, float(np.float32(dt)), collocated=True), shape)
    for name in ("b", "lam", "mu"):
        sim.write_global(name, kd.fields[name].data_gather().astype(np.float64))
    sim.write_global("txx", t0.astype(np.float64))
    sim.write_global("tyz", 0.5 * t0.astype(np.float64))
    sim.run(0, steps - 1)
    for name in P.VNAMES + P.TNAMES:
        want = sim.gather(name, steps % 2)
        got = kd.fields[name].data_gather()
        err = rel_l2(got, want)
        assert err <= REL, (name, err, np.abs(got - want).max())
    assert np.abs(sim.gather("vx", steps % 2)).max() > 0


def test_acoustic_cfl_guard():
    """a dt above the stencil's leapfrog stability limit is
    refused at configuration time; the conservative critical_dt runs."""
    shape = (24, 20, 28)
    grid = Grid(shape=shape, extent=tuple(10.0 * (n - 1) for n in shape))
    kd = KD.acoustic_model(grid, so=8, name="u_cfl")
    op = Operator([kd])
    vmax = float(1.0 / np.sqrt(kd.fields["m"].data_gather().min()))
    with pytest.raises(ValueError, match="CFL"):
        op.apply(time_M=1, dt=0.6 * 10.0 / vmax)
    op.apply(time_M=1, dt=float(np.float32(KD.critical_dt(vmax, grid.spacing))))
