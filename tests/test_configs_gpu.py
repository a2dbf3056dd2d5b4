"""BASELINE configs as parity tests.

* C1 at FULL size: 3D isotropic acoustic SO-8, 256^3 fp32, 200 steps, Ricker
  point source + 256-receiver line, through ``Operator.apply`` on the GPU,
  against the oracle (numpy fp64 on the same fp32 parameters, threaded over
  x-slabs).  rel-L2 <= 1e-5 on the final wavefield and the traces; max-abs
  printed.
* C2-C5 DOWN-SCALED (same space order, topology and mpi mode as the config,
  about 64-128^3 per rank, 12-30 steps): the GPU single-rank run against the
  oracle's SIMULATED ranks executing the config's decomposition and mode
  (SPEC.md:395-483), so the decomposed algorithm is pinned to the same
  numbers.  (GPU multi-rank == GPU single-rank bitwise is
  tests/test_multigpu.py.)

Set ``SDMP_EVIDENCE=<dir>`` to also write each result as JSON there.
"""
import json
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import problems as P  # noqa: E402
from oracle.runtime import Simulation  # noqa: E402
from paper_2312_13094_b200 import Grid, Operator, SparseTimeFunction  # noqa: E402
from paper_2312_13094_b200 import kernels as KD  # noqa: E402
from paper_2312_13094_b200 import symbolics as S  # noqa: E402

REL = 1e-5
THREADS = min(os.cpu_count() or 1, 32)


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def report(name, res):
    print(json.dumps({"config": name, **res}))
    d = os.environ.get("SDMP_EVIDENCE")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"{name}.json"), "w") as f:
            json.dump({"config": name, **res}, f, indent=1)


def star_coeffs(so, h):
    w = [float(c) for c in S.fd_coefficients(2, so)]
    r = so // 2
    return [np.float32([w[r + k] / (hh * hh) for k in range(r + 1)]).astype(np.float64)
            for hh in h]


def d1_coeffs(so, h):
    r = so // 2
    d1 = [float(c) for c in S.fd_coefficients(1, so)]
    return [np.float32([0.0] + [d1[r + k] / hh for k in range(1, r + 1)]).astype(np.float64)
            for hh in h]


def acoustic_case(shape, steps, mode, dims, tag, nrec, src_xyz, rec_yz, f0, h=10.0, vmax=4.5):
    grid = Grid(shape, tuple(h * (n - 1) for n in shape), comm="self")
    kd = KD.acoustic_model(grid, so=8, name=f"u_{tag}")
    u, m = kd.fields["u"], kd.fields["m"]
    dt = float(np.float32(0.38 * h / (vmax * 1.01)))
    src = KD.point_source(grid, [src_xyz], steps, dt, f0=f0, name=f"src_{tag}")
    ext = grid.extent
    rc = np.stack([np.linspace(5.0, ext[0] - 5.0, nrec), np.full(nrec, rec_yz[0]),
                   np.full(nrec, rec_yz[1])], 1)
    rec = SparseTimeFunction(f"rec_{tag}", grid, nrec, steps, coordinates=rc)
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
    t0 = time.perf_counter()
    op.apply(time_M=steps - 1, dt=dt, mpi=mode)
    gpu_s = time.perf_counter() - t0
    got, traces = u.data_gather(), rec.data.copy()
    C = float(np.float32(dt * dt))
    sp = P.SparseSpec(shape, grid.spacing, src.coordinates, src.data.astype(np.float64), "u",
                      ("m", C), rc, "u")
    prob = P.star(3, 8, star_coeffs(8, grid.spacing), 2.0, -1.0, C, True, sparse=sp,
                  shape=shape, dims=dims)
    sim = Simulation(prob, shape, dims=dims, mode=mode, threads=THREADS)
    sim.write_global("m", m.data_gather().astype(np.float64))
    t0 = time.perf_counter()
    sim.run(0, steps - 1)
    cpu_s = time.perf_counter() - t0
    want = sim.gather("u", steps % 3)
    tw = np.array([sim.traces[t] for t in range(steps)])
    res = {"shape": list(shape), "steps": steps, "mode": mode, "oracle_ranks": list(dims),
           "wavefield_rel_l2": rel_l2(got, want),
           "wavefield_max_abs": float(np.abs(got - want).max()),
           "wavefield_max": float(np.abs(want).max()),
           "traces_rel_l2": rel_l2(traces, tw), "traces_max_abs": float(np.abs(traces - tw).max()),
           "traces_max": float(np.abs(tw).max()),
           "tolerance_rel_l2": REL, "gpu_apply_s_incl_plan_build": gpu_s,
           "oracle_s": cpu_s, "oracle_threads": THREADS}
    return res


def test_c1_fullsize_vs_oracle():
    """BASELINE configs[0] at full size."""
    res = acoustic_case((256, 256, 256), 200, "diagonal", (1, 1, 1), "c1", 256,
                        (1278.3, 1272.9, 101.7), (1277.5, 20.3), 0.010)
    report("C1_acoustic_so8_256cubed_200steps", res)
    assert res["wavefield_max"] > 0
    assert res["wavefield_rel_l2"] <= REL, res
    assert res["traces_rel_l2"] <= REL, res


def test_c2_downscaled_2x2_full():
    """C2 (acoustic SO-8 weak scaling, 1024^3 per GPU) down-scaled to 128^3
    per rank on the (2,2,1) topology in full mode."""
    shape = (256, 256, 128)
    ext = tuple(10.0 * (n - 1) for n in shape)
    # receiver line through the source depth, crossing the x split (the
    # wave reaches it within the 30 steps)
    res = acoustic_case(shape, 30, "full", (2, 2, 1), "c2", 64,
                        (0.5 * ext[0] + 3.7, 0.5 * ext[1] + 3.7, 0.5 * ext[2] + 3.7),
                        (0.5 * ext[1] + 2.5, 0.5 * ext[2] - 31.3), 0.030)
    assert res["traces_max"] > 1e-3 * res["wavefield_max"], res
    report("C2_acoustic_so8_128cubed_per_rank_2x2x1_full", res)
    assert res["wavefield_rel_l2"] <= REL and res["traces_rel_l2"] <= REL, res


def test_c3_downscaled_tti_2x1_full():
    """C3 (TTI SO-8, mpi=full core/remainder overlap) at 128^3 per rank on
    (2,1,1)."""
    so, steps, dims, mode = 8, 16, (2, 1, 1), "full"
    shape = (256, 128, 128)
    grid = Grid(shape, tuple(10.0 * (n - 1) for n in shape), comm="self")
    kd = KD.tti_model(grid, so=so)
    p, r = kd.fields["p"], kd.fields["r"]
    rng = np.random.default_rng(0)
    init = np.float32(rng.standard_normal(shape))
    p.data[:] = init
    r.data[:] = 0.5 * init
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
    Operator([kd]).apply(time_M=steps - 1, dt=dt, mpi=mode)
    h = grid.spacing
    prob = P.tti(so, star_coeffs(so, h), d1_coeffs(so, h), float(np.float32(dt * dt)),
                 shape=shape, dims=dims)
    sim = Simulation(prob, shape, dims=dims, mode=mode, threads=THREADS)
    for name in ("m", "epsp", "delp", "ax", "ay", "az"):
        sim.write_global(name, kd.fields[name].data_gather().astype(np.float64))
    sim.write_global("p", init.astype(np.float64))
    sim.write_global("r", 0.5 * init.astype(np.float64))
    # the direction cosines are read at offsets: their halos are exchanged
    # once before the time loop (the hoisted HaloSpot)
    sim.exchange_static(("ax", "ay", "az"), (so,) * 3)
    sim.run(0, steps - 1)
    res = {"shape": list(shape), "steps": steps, "mode": mode, "oracle_ranks": list(dims)}
    for name, fn in (("p", p), ("r", r)):
        want, got = sim.gather(name, steps % 3), fn.data_gather()
        res[f"{name}_rel_l2"] = rel_l2(got, want)
        res[f"{name}_max_abs"] = float(np.abs(got - want).max())
    report("C3_tti_so8_128cubed_per_rank_2x1x1_full", res)
    assert res["p_rel_l2"] <= REL and res["r_rel_l2"] <= REL, res


@pytest.mark.parametrize("visco", [False, True])
def test_c4_c5_downscaled_elastic(visco):
    """C4 (staggered elastic SO-8, (4,2,1), mpi=diag) and C5 (viscoelastic
    SO-16, (2,2,1), mpi=full) at 64^3 per rank, with a source in txx and a
    receiver line in vz."""
    if visco:
        so, dims, mode, shape, steps = 16, (2, 2, 1), "full", (128, 128, 64), 12
    else:
        so, dims, mode, shape, steps = 8, (4, 2, 1), "diagonal", (256, 128, 64), 16
    grid = Grid(shape, tuple(10.0 * (n - 1) for n in shape), comm="self")
    kd = KD.viscoelastic_model(grid, so=so) if visco else KD.elastic_model(grid, so=so)
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1)))
    ext = grid.extent
    src = KD.point_source(grid, [(0.5 * ext[0] + 0.3, 0.5 * ext[1] + 0.2, 0.4 * ext[2])], steps,
                          dt, f0=0.03, name=f"src_el{visco}")
    nrec = 17
    rc = np.stack([np.linspace(5.0, ext[0] - 5.0, nrec), np.full(nrec, 0.5 * ext[1] + 1.1),
                   np.full(nrec, 0.3 * ext[2])], 1)
    rec = SparseTimeFunction(f"rec_el{visco}", grid, nrec, steps, coordinates=rc)
    op = Operator([kd, src.inject(kd.fields["txx"].forward, expr=src * S.DT),
                   rec.interpolate(kd.fields["vz"])])
    op.apply(time_M=steps - 1, dt=dt, mpi=mode)
    h = grid.spacing
    sc = [np.float32([float(c) / hh for c in S.staggered_coefficients(so)]).astype(np.float64)
          for hh in h]
    sp = P.SparseSpec(shape, h, src.coordinates, src.data.astype(np.float64), "txx",
                      (None, float(np.float32(dt))), rc, "vz")
    prob = P.elastic(so, sc, float(np.float32(dt)), visco=visco, sparse=sp, shape=shape,
                     dims=dims)
    sim = Simulation(prob, shape, dims=dims, mode=mode, threads=THREADS)
    params = ("b", "l2m", "mus", "its") if visco else ("b", "lam", "mu")
    for name in params:
        sim.write_global(name, kd.fields[name].data_gather().astype(np.float64))
    sim.run(0, steps - 1)
    res = {"shape": list(shape), "steps": steps, "mode": mode, "oracle_ranks": list(dims),
           "so": so}
    worst = 0.0
    for name in P.VNAMES + P.TNAMES + (P.RNAMES if visco else ()):
        want, got = sim.gather(name, steps % 2), kd.fields[name].data_gather()
        e = rel_l2(got, want)
        res[f"{name}_rel_l2"] = e
        worst = max(worst, e)
    tw = np.array([sim.traces[t] for t in range(steps)])
    res["traces_rel_l2"] = rel_l2(rec.data, tw)
    res["worst_field_rel_l2"] = worst
    report(("C5_visco_so16_64cubed_per_rank_2x2x1_full" if visco
            else "C4_elastic_so8_64cubed_per_rank_4x2x1_diag"), res)
    assert np.abs(tw).max() > 0
    assert worst <= REL and res["traces_rel_l2"] <= REL, res
