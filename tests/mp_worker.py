"""Multi-GPU worker (launched by tests/test_multigpu.py under torchrun).

For every family and mpi mode: run the decomposed problem on the world,
gather, and compare BITWISE with the same problem run on a one-rank grid
(``comm="self"``) on this process's GPU (acceptance 3).
Also checks receiver traces and that full mode keeps the Listing-8 order
(post -> CORE -> wait -> OWNED) in the device trace.
Exit code 0 = all equal.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2312_13094_b200 import Grid, Operator, SparseTimeFunction  # noqa: E402
from paper_2312_13094_b200 import kernels as KD  # noqa: E402
from paper_2312_13094_b200 import symbolics as S  # noqa: E402
from paper_2312_13094_b200.dist import context  # noqa: E402


def acoustic(grid, tag, steps, so=8):
    kd = KD.acoustic_model(grid, so=so, name=f"u{tag}")
    u, m = kd.fields["u"], kd.fields["m"]
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
    ext = grid.extent
    # source near a rank corner, receivers crossing rank boundaries
    src = KD.point_source(grid, [tuple(0.5 * e + 0.3 for e in ext), (0.25 * ext[0], 0.5 * ext[1], 0.5 * ext[2])],
                          steps, dt, f0=0.03, name=f"src{tag}")
    nrec = 11
    rc = np.stack([np.linspace(5.0, ext[0] - 5.0, nrec), np.full(nrec, 0.5 * ext[1]),
                   np.full(nrec, 0.31 * ext[2])], 1)
    rec = SparseTimeFunction(f"rec{tag}", grid, nrec, steps, coordinates=rc)
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
    return op, dt, [u], rec


def diffusion(grid, tag, steps, so=4):
    kd = KD.diffusion_model(grid, so=so, name=f"ud{tag}")
    u = kd.fields["u"]
    u.data[...] = np.float32(np.random.default_rng(3).random(grid.shape))
    dt = float(np.float32(0.1 * min(grid.spacing) ** 2))
    return Operator([kd]), dt, [u], None


def damped(grid, tag, steps, so=8):
    kd = KD.damped_acoustic_model(grid, so=so, nbl=5, name=f"ud{tag}")
    u, m = kd.fields["u"], kd.fields["m"]
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
    ext = grid.extent
    src = KD.point_source(grid, [tuple(0.5 * e + 0.3 for e in ext)], steps, dt, f0=0.03,
                          name=f"srcd{tag}")
    rc = np.stack([np.linspace(5.0, ext[0] - 5.0, 7), np.full(7, 0.5 * ext[1]),
                   np.full(7, 0.31 * ext[2])], 1)
    rec = SparseTimeFunction(f"recd{tag}", grid, 7, steps, coordinates=rc)
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)])
    return op, dt, [u], rec


def rotated(grid, tag, steps, so=8):
    kd = KD.rotated_model(grid, so=so, name=f"ur{tag}")
    u = kd.fields["u"]
    u.data[:] = np.float32(np.random.default_rng(4).standard_normal(grid.shape))
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
    return Operator([kd]), dt, [u], None


def tti(grid, tag, steps, so=8):
    kd = KD.tti_model(grid, so=so)
    rng = np.random.default_rng(0)
    init = np.float32(rng.standard_normal(grid.shape))
    kd.fields["p"].data[:] = init
    kd.fields["r"].data[:] = 0.5 * init
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.2)))
    return Operator([kd]), dt, [kd.fields["p"], kd.fields["r"]], None


def elastic(grid, tag, steps, so=8, visco=False, collocated=False):
    kd = (KD.viscoelastic_model(grid, so=so) if visco
          else KD.elastic_model(grid, so=so, collocated=collocated))
    rng = np.random.default_rng(1)
    t0 = np.float32(rng.standard_normal(grid.shape))
    kd.fields["txx"].data[:] = t0
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1)))
    names = KD.VNAMES + KD.TNAMES
    # a source on a rank boundary (its injection is pushed into the
    # neighbour's halo in full mode) and receivers crossing ranks
    ext = grid.extent
    src = KD.point_source(grid, [(0.5 * ext[0] + 0.3, 0.5 * ext[1] + 0.2, 0.4 * ext[2])], steps, dt,
                          f0=0.03, name=f"src{tag}")
    rc = np.stack([np.linspace(5.0, ext[0] - 5.0, 9), np.full(9, 0.5 * ext[1]),
                   np.full(9, 0.3 * ext[2])], 1)
    rec = SparseTimeFunction(f"rec{tag}", grid, 9, steps, coordinates=rc)
    op = Operator([kd, src.inject(kd.fields["txx"].forward, expr=src * S.DT),
                   rec.interpolate(kd.fields["vz"])])
    return op, dt, [kd.fields[n] for n in names], rec


def full_order(op, dt, steps):
    """Device trace of two more full-mode steps: per phase, the post starts
    before the wait ends, CORE starts no later than the first OWNED slab, and
    every OWNED slab starts after the wait ended (Listing 8, SPEC.md:366,
    450-458; acceptance 8)."""
    nat = op._native("full", dt)
    nat.plan.set_tracing(True)
    nat.plan.run(steps, steps + 1, torch.cuda.current_stream())
    nat.plan.sync()
    nat.plan.set_tracing(False)
    rows = nat.plan.trace()
    eps = 2e-3
    problems = []
    phases = {}
    cur = 0
    for i, a in enumerate(nat.eplan.actions):
        if a.kind == "post":
            cur = a.phase
        j = nat.native_index[i]
        if j < 0:
            continue
        beg, dur = rows[j][3], rows[j][4]
        key = None
        if a.kind in ("post", "wait"):
            key = a.kind
        elif a.kind == "compute" and getattr(a, "region", None) in ("CORE", "OWNED"):
            key = a.region
        if key:
            phases.setdefault(cur, {}).setdefault(key, []).append((beg, beg + dur))
    for ph, d in phases.items():
        if "wait" not in d or "OWNED" not in d:
            continue
        wait_end = max(e for _b, e in d["wait"])
        own_beg = min(b for b, _e in d["OWNED"])
        if own_beg + eps < wait_end:
            problems.append(f"phase {ph}: OWNED starts {own_beg:.4f} before the wait ends {wait_end:.4f}")
        if "CORE" in d and min(b for b, _e in d["CORE"]) > own_beg + eps:
            problems.append(f"phase {ph}: CORE starts after OWNED")
        if "post" in d and min(b for b, _e in d["post"]) > wait_end + eps:
            problems.append(f"phase {ph}: post starts after the wait ended")
    return problems


def main():
    ctx = context()
    rank, size = ctx.rank, ctx.size
    topo = tuple(int(x) for x in os.environ.get("TOPO", f"{size},1,1").split(","))
    shape = tuple(int(x) for x in os.environ.get("SHAPE", "40,36,32").split(","))
    steps = int(os.environ.get("STEPS", "12"))
    failures = []
    order_problems = []
    memory_problems = []
    results = {}
    cases = [("acoustic", acoustic, {}), ("diffusion", diffusion, {}), ("damped", damped, {}),
             ("rotated", rotated, {}), ("tti", tti, {}),
             # SO-4: the single-pass kernels (csrc/tti_fused.cuh)
             ("rotated4", rotated, {"so": 4}), ("tti4", tti, {"so": 4}),
             ("elastic", elastic, {}), ("elastic_col", elastic, {"collocated": True}),
             ("visco", elastic, {"visco": True, "so": 16})]
    only = os.environ.get("FAMILIES")
    if only:
        # "<family><SO>" (e.g. acoustic2, elastic_col4) runs a family at
        # another space order (the SPEC.md:702 matrix over SDO {2, 4, 8})
        import re
        base = {c[0]: c for c in cases}
        picked = []
        for name in only.split(","):
            if name in base:
                picked.append(base[name])
                continue
            mt = re.fullmatch(r"([a-z_]+?)(\d+)", name)
            if mt and mt.group(1) in base:
                fam, build, kw = base[mt.group(1)]
                picked.append((name, build, dict(kw, so=int(mt.group(2)))))
            else:
                raise SystemExit(f"unknown family {name!r}")
        cases = picked
    for fam, build, kw in cases:
        for mode in ("basic", "diagonal", "full"):
            ext = tuple(10.0 * (n - 1) for n in shape)
            g = Grid(shape, ext, topology=topo)
            ref_g = Grid(shape, ext, comm="self")
            tag = f"{fam}_{mode}"
            # the multi-rank and single-rank problems need distinct field names
            op, dt, fields, rec = build(g, tag, steps, **kw)
            op.apply(time_M=steps - 1, dt=dt, mpi=mode)
            got = [f.data_gather() for f in fields]
            got_tr = rec.data.copy() if rec is not None else None
            if os.environ.get("SDMP_GUARD", "0") != "0":
                from memcheck_util import check_fields
                memory_problems.extend(f"{tag} rank {rank}: {n}: {p}" for n, p in
                                       check_fields(list(op.fields.values()), g.decomposition, rank))
            if mode == "full" and size > 1:
                order_problems.extend(f"{fam}: {p}" for p in full_order(op, dt, steps))
            # release the distributed fields before building the reference
            import paper_2312_13094_b200.api as A
            names_mr = [f.name for f in fields]
            del op, fields, rec
            A._FUNCS.clear()
            rop, rdt, rfields, rrec = build(ref_g, tag, steps, **kw)
            rop.apply(time_M=steps - 1, dt=rdt, mpi="diagonal")
            want = [f.data_gather() for f in rfields]
            ok = all(np.array_equal(a, b) for a, b in zip(got, want))
            if rrec is not None:
                ok = ok and np.array_equal(got_tr, rrec.data)
            maxdiff = max(float(np.abs(a - b).max()) for a, b in zip(got, want))
            results[tag] = {"equal": bool(ok), "max_abs": maxdiff,
                            "norm": float(np.linalg.norm(want[0]))}
            if not ok:
                failures.append(tag)
            del rop, rfields, rrec
            A._FUNCS.clear()
            torch.cuda.empty_cache()
    orders = ctx.allgather(order_problems)
    mem = [p for ps in ctx.allgather(memory_problems) for p in ps]
    if rank == 0:
        print(json.dumps({"topology": topo, "shape": shape, "results": results,
                          "order_ok": not any(orders), "order": orders,
                          "memory_ok": not mem, "memory": mem[:20],
                          "devices": torch.cuda.device_count(), "ranks": size}))
    ctx.barrier()
    return 1 if failures or any(orders) or mem else 0


if __name__ == "__main__":
    rc = main()
    sys.stdout.flush()
    os._exit(rc)
