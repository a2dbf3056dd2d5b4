"""BASELINE config C1 at full size: 3D isotropic acoustic SO-8, 256^3 fp32,
200 steps, Ricker point source + 256-receiver line, run on
the GPU through the public API and on the CPU oracle on identical fp32
parameters; reports rel-L2 / max-abs of the final wavefield and the traces
and the two timings.

    python tools/c1_parity.py [--steps 200] [--out profiles/r01_c1_parity.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--mode", default="diagonal")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from oracle import problems as P
    from oracle.runtime import Simulation
    from paper_2312_13094_b200 import Grid, Operator, SparseTimeFunction
    from paper_2312_13094_b200 import kernels as KD
    from paper_2312_13094_b200 import symbolics as S

    n, so, steps = a.n, 8, a.steps
    shape = (n, n, n)
    h = 10.0
    grid = Grid(shape, (h * (n - 1),) * 3)
    kd = KD.acoustic_model(grid, so=so)
    u, m = kd.fields["u"], kd.fields["m"]
    vmax = 4.5 * 1.01
    dt = float(np.float32(0.38 * h / vmax))
    src = KD.point_source(grid, [(1278.3, 1272.9, 101.7)], steps, dt, f0=0.010)
    rc = np.stack([np.linspace(5.0, 2545.0, 256), np.full(256, 1277.5), np.full(256, 20.3)], 1)
    rec = SparseTimeFunction("rec", grid, 256, steps, coordinates=rc)
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
    op.apply(time_M=steps - 1, dt=dt, mpi=a.mode)  # warm (plan build + first run)
    u.data[:] = 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op.apply(time_M=steps - 1, dt=dt, mpi=a.mode)
    gpu_s = time.perf_counter() - t0
    got = u.data_gather()
    traces = rec.data.copy()

    w = [float(c) for c in S.fd_coefficients(2, so)]
    r = so // 2
    coeffs = [np.float32([w[r + k] / (h * h) for k in range(r + 1)]).astype(np.float64)] * 3
    C = float(np.float32(dt * dt))
    sp = P.SparseSpec(shape, grid.spacing, src.coordinates, src.data.astype(np.float64), "u",
                      ("m", C), rc, "u")
    sim = Simulation(P.star(3, so, coeffs, 2.0, -1.0, C, True, sparse=sp, shape=shape), shape)
    sim.write_global("m", m.data_gather().astype(np.float64))
    t0 = time.perf_counter()
    sim.run(0, steps - 1)
    cpu_s = time.perf_counter() - t0
    want = sim.gather("u", steps % 3)
    tw = np.array([sim.traces[t] for t in range(steps)])
    rel = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    trel = float(np.linalg.norm(traces - tw) / np.linalg.norm(tw))
    res = {"config": "C1 acoustic SO-8 256^3 fp32, 200 steps, Ricker src + 256 receivers",
           "steps": steps, "mode": a.mode, "dt_ms": dt,
           "wavefield_rel_l2": rel, "wavefield_max_abs": float(np.abs(got - want).max()),
           "wavefield_max": float(np.abs(want).max()),
           "traces_rel_l2": trel, "traces_max_abs": float(np.abs(traces - tw).max()),
           "tolerance": 1e-5, "pass": rel <= 1e-5 and trel <= 1e-5,
           "gpu_apply_s": gpu_s, "gpu_gpts": n ** 3 * steps / gpu_s / 1e9,
           "cpu_oracle_s": cpu_s, "cpu_oracle_gpts": n ** 3 * steps / cpu_s / 1e9,
           "cpu_threads": 1}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
