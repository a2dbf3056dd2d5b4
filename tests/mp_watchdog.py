"""Watchdog check (launched by tests/test_multigpu.py under torchrun, 2 ranks):
rank 1 builds the plan (IPC handles exchanged) but never runs it, so rank 0's
halo wait cannot complete; with SDMP_TIMEOUT_MS=1500 rank 0 must get a
NativeError naming the watchdog instead of hanging."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SDMP_TIMEOUT_MS"] = "1500"

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_13094_b200 import Grid, Operator  # noqa: E402
from paper_2312_13094_b200 import kernels as KD  # noqa: E402
from paper_2312_13094_b200.dist import context  # noqa: E402
from paper_2312_13094_b200.runtime import NativeError  # noqa: E402


def main():
    ctx = context()
    grid = Grid((48, 32, 32), (470.0, 310.0, 310.0), topology=(2, 1, 1))
    kd = KD.acoustic_model(grid, so=8, name="uw")
    op = Operator([kd])
    dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
    plan = op._native("diagonal", dt)   # collective: both ranks build it
    result = {"rank": ctx.rank}
    if ctx.rank == 0:
        try:
            plan.run(0, 3)
            result["outcome"] = "completed"
        except NativeError as exc:
            result["outcome"] = "timeout" if "watchdog" in str(exc) else f"error: {exc}"
    ctx.barrier()
    out = ctx.allgather(result)
    if ctx.rank == 0:
        print(json.dumps(out))
    return 0


if __name__ == "__main__":
    rc = main()
    sys.stdout.flush()
    os._exit(rc)
