"""Pin the oracle against the paper/SPEC golden values before trusting it
(PAPER.md:271-298 Listings 3-4; SPEC.md worked examples), then check the
central oracle property: multi-rank == single-rank, bitwise, every mode."""
import itertools
import math

import numpy as np
import pytest

from oracle import decomp as D
from oracle import problems as P
from oracle import stencils as K
from oracle.runtime import Simulation
from paper_2312_13094_b200.symbolics import fd_coefficients, staggered_coefficients


def star_coeffs(nd, so, h):
    w = [float(c) for c in fd_coefficients(2, so)]
    r = so // 2
    return [np.float32([w[r + k] / (hh * hh) for k in range(r + 1)]).astype(np.float64)
            for hh in h]


def diffusion_listing(dims):
    h = (2.0 / 3.0, 2.0 / 3.0)
    dt = 0.25 * h[0] * h[1] / 0.5  # PAPER.md:155-158 -> 2/9
    prob = P.star(2, 2, star_coeffs(2, 2, h), 1.0, 0.0, dt, False)
    sim = Simulation(prob, (4, 4), dims, mode="diagonal")
    init = np.zeros((4, 4))
    init[1:-1, 1:-1] = 1.0
    sim.write_global("u", init)
    return sim


def test_listing3_rank_views():
    sim = diffusion_listing((2, 2))
    views = [rk.arrays["u"][0][2:4, 2:4] for rk in sim.ranks]
    want = [[[0, 0], [0, 1]], [[0, 0], [1, 0]], [[0, 1], [0, 0]], [[1, 0], [0, 0]]]
    for v, w in zip(views, want):
        assert np.array_equal(v, np.array(w, dtype=float))


@pytest.mark.parametrize("mode", ["basic", "diagonal", "full"])
def test_listing4_two_steps(mode):
    sim = diffusion_listing((2, 2))
    sim.mode = mode
    sim.run(0, 1)  # time_M=1 -> two iterations
    g = sim.gather("u", 0)
    a, b = 0.5, -0.25
    want = np.array([[a, b, b, a], [b, a, a, b], [b, a, a, b], [a, b, b, a]])
    assert np.max(np.abs(g - want)) < 1e-6
    views = [rk.arrays["u"][0][2:4, 2:4] for rk in sim.ranks]
    assert np.allclose(views[0], [[a, b], [b, a]])
    assert np.allclose(views[1], [[b, a], [a, b]])


def test_spec_examples_decomposition():
    assert D.default_topology(4, 2) == (2, 2)
    assert D.default_topology(16, 3) == (4, 2, 2)
    assert D.default_topology(1, 3) == (1, 1, 1)
    assert D.decompose_axis(5, 2) == [(0, 3), (3, 5)]
    assert D.decompose_axis(1024, 8) == [(128 * i, 128 * (i + 1)) for i in range(8)]
    assert D.global_to_local(((0, 2), (0, 2)), ((1, 3), (1, 3))) == ((1, 2), (1, 2))
    assert D.global_to_local(((2, 4), (2, 4)), ((1, 3), (1, 3))) == ((0, 1), (0, 1))
    # Fig. 4: interior point, shared edge, four-rank corner (4x4 nodes on 2x2)
    shape, extent = (8, 8), (7.0, 7.0)
    assert D.owners_of_point((1.2, 1.3), shape, extent, (2, 2)) == [0]
    assert D.owners_of_point((3.5, 1.3), shape, extent, (2, 2)) == [0, 2]
    assert D.owners_of_point((3.5, 3.5), shape, extent, (2, 2)) == [0, 1, 2, 3]


def test_spec_examples_regions_and_counts():
    core = D.core_mask((8, 8), [True, True], [True, True], (1, 1))
    assert core.sum() == 36
    slabs = D.owned_slabs_reference((8, 8), [True, True], [True, True], (1, 1))
    assert [((h[0] - l[0]) * (h[1] - l[1])) for l, h in slabs] == [8, 8, 6, 6]
    # interior rank message counts
    for nd, basic, diag in ((2, 4, 8), (3, 6, 26)):
        dims = (3,) * nd
        mid = D.coords_rank((1,) * nd, dims)
        shape = (12,) * nd
        assert sum(len(s) for s in D.basic_messages(shape, dims, mid, (1,) * nd)) == basic
        assert len(D.diag_messages(shape, dims, mid, (1,) * nd)) == diag


def test_spec_examples_sparse():
    _, w = K.trilinear((0.25, 0.75), (1.0, 1.0), (4, 4))
    assert np.allclose(w, [0.1875, 0.5625, 0.0625, 0.1875])
    f0, t0 = 10.0, 0.1
    assert abs(K.ricker(f0, t0, t0) - 1.0) < 1e-15
    assert abs(K.ricker(f0, t0 + 1.0 / (math.pi * f0 * math.sqrt(2.0)), t0)) < 1e-12
    assert abs(K.ricker(f0, t0 + 10.0 / f0, t0)) < 1e-12


def acoustic_problem(shape, dims, so=4, steps=6, seed=0):
    nd = len(shape)
    rng = np.random.default_rng(seed)
    h = (10.0,) * nd
    vp = 1.5 + rng.random(shape)
    dt = np.float32(0.3 * h[0] / 2.5)
    coeffs = star_coeffs(nd, so, h)
    extent = tuple(hh * (n - 1) for hh, n in zip(h, shape))
    src = np.array([[e * 0.47 + 0.3 for e in extent], [e * 0.5 for e in extent]])
    rec = np.array([[e * f for e in extent] for f in (0.1, 0.33, 0.5, 0.77)])
    amp = np.float32(rng.standard_normal((steps, len(src))))
    sp = P.SparseSpec(shape, h, src, amp, "u", ("m", float(np.float32(dt * dt))), rec, "u")
    prob = P.star(nd, so, coeffs, 2.0, -1.0, float(np.float32(dt * dt)), True,
                  sparse=sp, shape=shape, dims=dims)
    m = np.float32(1.0 / vp ** 2).astype(np.float64)
    return prob, m


@pytest.mark.parametrize("shape,dims", [((12, 10), (2, 1)), ((12, 11), (2, 2)),
                                        ((10, 9, 8), (2, 2, 1)), ((9, 8, 10), (1, 3, 1)),
                                        ((12, 10, 9), (2, 2, 2))])
@pytest.mark.parametrize("mode", ["basic", "diagonal", "full"])
def test_multirank_equals_single_rank_acoustic(shape, dims, mode):
    steps = 6
    results = []
    for dd in (None, dims):
        prob, m = acoustic_problem(shape, dd or (1,) * len(shape), steps=steps)
        sim = Simulation(prob, shape, dd, mode=mode)
        sim.write_global("m", m)
        sim.run(0, steps - 1)
        results.append((sim.gather("u", steps % 3), np.array([sim.traces[t] for t in range(steps)])))
    assert np.array_equal(results[0][0], results[1][0])
    assert np.array_equal(results[0][1], results[1][1])
    assert np.abs(results[0][0]).max() > 0


def test_injection_mass_conservation():
    # sum of field change == sum amplitudes * scale, every decomposition
    shape = (9, 9, 9)
    for dims in [(1, 1, 1), (2, 2, 1), (3, 1, 2)]:
        h = (1.0, 1.0, 1.0)
        coeffs = [np.zeros(2)] * 3
        src = np.array([[4.0, 4.0, 4.0], [3.5, 2.25, 6.75], [8.0, 8.0, 8.0]])
        amp = np.array([[1.0, 2.0, 0.5]])
        sp = P.SparseSpec(shape, h, src, amp, "u", (None, 1.0))
        prob = P.star(3, 2, coeffs, 1.0, 0.0, 0.0, False, sparse=sp, shape=shape, dims=dims)
        sim = Simulation(prob, shape, dims)
        sim.run(0, 0)
        assert abs(sim.gather("u", 1).sum() - 3.5) < 1e-12


@pytest.mark.parametrize("mode", ["basic", "full"])
def test_multirank_equals_single_rank_tti(mode):
    shape, dims, so = (10, 9, 11), (2, 2, 1), 4
    rng = np.random.default_rng(3)
    h = (10.0,) * 3
    d1 = [float(c) for c in fd_coefficients(1, so)]
    r = so // 2
    d1_c = [np.float32([0.0] + [d1[r + k] / hh for k in range(1, r + 1)]).astype(np.float64) for hh in h]
    lap_c = star_coeffs(3, so, h)
    th, ph = rng.random(shape) * 0.6, rng.random(shape) * 0.8
    vals = {"m": 1.0 / (2.0 + rng.random(shape)) ** 2, "epsp": 1 + 0.4 * rng.random(shape),
            "delp": np.sqrt(1 + 0.2 * rng.random(shape)), "ax": np.sin(th) * np.cos(ph),
            "ay": np.sin(th) * np.sin(ph), "az": np.cos(th)}
    init = rng.standard_normal(shape)
    out = []
    for dd in (None, dims):
        sim = Simulation(P.tti(so, lap_c, d1_c, 1.0), shape, dd, mode=mode)
        for k, v in vals.items():
            sim.write_global(k, np.float32(v).astype(np.float64))
        sim.exchange_static(["ax", "ay", "az"], (so // 2,) * 3)
        sim.write_global("p", init)
        sim.write_global("r", 0.5 * init)
        sim.run(0, 3)
        out.append((sim.gather("p", 4 % 3), sim.gather("r", 4 % 3)))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("visco", [False, True])
def test_multirank_equals_single_rank_elastic(visco):
    shape, dims, so = (10, 12, 9), (2, 3, 1), 4
    rng = np.random.default_rng(5)
    h = (5.0, 5.0, 5.0)
    sc = [np.float32([float(c) / hh for c in staggered_coefficients(so)]).astype(np.float64) for hh in h]
    txx0, vz0 = rng.standard_normal(shape), rng.standard_normal(shape)
    out = []
    for dd in (None, dims):
        sim = Simulation(P.elastic(so, sc, 0.3, visco=visco), shape, dd, mode="diagonal")
        mats = (("b", 0.5), ("l2m", 2.0), ("mus", 1.0), ("its", 0.2)) if visco else \
            (("b", 0.5), ("lam", 2.0), ("mu", 1.0))
        for k, s in mats:
            sim.write_global(k, s * (1 + 0.1 * np.random.default_rng(1).random(shape)))
        sim.write_global("txx", txx0)
        sim.write_global("vz", vz0)
        sim.run(0, 3)
        out.append([sim.gather(n, 0) for n in P.VNAMES + P.TNAMES])
    for a, b in zip(*out):
        assert np.array_equal(a, b)
