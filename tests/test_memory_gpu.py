"""Memory-safety checks of every kernel family and mpi mode on one rank
(compute-sanitizer is closed on this pool; tests/memcheck_util.py): canary
guard zones around every field allocation and the exterior-halo-zero
invariant, after runs that exercise the TMA streaming kernels,
the generic kernels (full-mode OWNED slabs), sparse injection /
interpolation and the CUDA-graph replay.  The multi-rank versions (peer
stores, IPC copies) run in tests/test_multigpu.py with SDMP_GUARD=1."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

FAMILIES = [("acoustic", {}), ("diffusion", {}), ("damped", {}), ("rotated", {}), ("tti", {}),
            ("rotated4", {"so": 4}), ("tti4", {"so": 4}),
            ("elastic", {}), ("elastic_col", {"collocated": True}),
            ("visco", {"visco": True, "so": 16})]


@pytest.mark.parametrize("fam,kw", FAMILIES, ids=[f[0] for f in FAMILIES])
@pytest.mark.parametrize("mode", ["basic", "diagonal", "full"])
def test_guards_and_exterior_halo(fam, kw, mode, monkeypatch):
    monkeypatch.setenv("SDMP_GUARD", "1")
    import mp_worker as W
    from memcheck_util import check_fields
    from paper_2312_13094_b200 import Grid
    build = {"acoustic": W.acoustic, "diffusion": W.diffusion, "damped": W.damped,
             "rotated": W.rotated, "tti": W.tti, "rotated4": W.rotated,
             "tti4": W.tti}.get(fam, W.elastic)
    shape = (40, 36, 44)   # TMA-streamed DOMAIN boxes plus generic edges
    g = Grid(shape, tuple(10.0 * (n - 1) for n in shape), comm="self")
    op, dt, fields, rec = build(g, f"mem_{fam}_{mode}", 14, **kw)
    assert all(f._guard is not None for f in op.fields.values())
    op.apply(time_M=13, dt=dt, mpi=mode)
    assert all(np.isfinite(f.data_gather()).all() for f in fields)
    assert np.abs(fields[0].data_gather()).max() > 0
    problems = check_fields(list(op.fields.values()), g.decomposition, 0)
    assert not problems, problems


def test_guard_detects_overrun(monkeypatch):
    """The check itself: a deliberate write one float past the last buffer
    is caught by the guard, one into the exterior halo by the invariant."""
    monkeypatch.setenv("SDMP_GUARD", "1")
    from memcheck_util import check_fields
    from paper_2312_13094_b200 import Grid, TimeFunction
    g = Grid((16, 16, 16), (150.0,) * 3, comm="self")
    u = TimeFunction("u_guard", g, space_order=4, time_order=2)
    assert check_fields([u], g.decomposition, 0) == []
    flat, gz, n = u._guard
    flat[gz + n] = 1.0
    u.storage[1, 0, 0, 0] = 2.0
    probs = [p for _n, p in check_fields([u], g.decomposition, 0)]
    assert len(probs) == 2 and "guard" in probs[0] and "exterior" in probs[1], probs
