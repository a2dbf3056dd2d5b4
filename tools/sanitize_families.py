"""Small single-process run of every kernel family in every mpi mode (full
mode included: CORE / OWNED split, fused push bookkeeping, stream joins),
meant to run under compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_families.py

Uses tests/mp_worker.py's family builders on a one-rank grid.  Exit code 0
when every run completed (the sanitizer's own report is the evidence)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import mp_worker as W  # noqa: E402
from paper_2312_13094_b200 import Grid  # noqa: E402
from paper_2312_13094_b200 import api as A  # noqa: E402


def main():
    shape = tuple(int(x) for x in os.environ.get("SHAPE", "24,20,28").split(","))
    steps = int(os.environ.get("STEPS", "3"))
    fams = os.environ.get("FAMILIES")
    cases = [("acoustic", W.acoustic, {}), ("diffusion", W.diffusion, {}),
             ("damped", W.damped, {}), ("rotated", W.rotated, {}), ("tti", W.tti, {}),
             ("elastic", W.elastic, {}), ("elastic_col", W.elastic, {"collocated": True}),
             ("visco", W.elastic, {"visco": True, "so": 16})]
    if fams:
        cases = [c for c in cases if c[0] in fams.split(",")]
    for fam, build, kw in cases:
        for mode in ("basic", "diagonal", "full"):
            g = Grid(shape, tuple(10.0 * (n - 1) for n in shape), comm="self")
            op, dt, fields, rec = build(g, f"{fam}_{mode}", steps, **kw)
            op.apply(time_M=steps - 1, dt=dt, mpi=mode)
            assert all(np.isfinite(f.data_gather()).all() for f in fields), fam
            print(f"{fam} {mode}: ok", flush=True)
            A._FUNCS.clear()
    return 0


if __name__ == "__main__":
    sys.exit(main())
