"""Kernel micro-benchmark: one star/TTI/elastic launch over a DOMAIN box,
timed with CUDA events on the launching stream (development tool; the
contract benchmark is bench.py).

    python tools/kbench.py --kernel star --n 1024 --so 8 --variant 3
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_13094_b200 import runtime as R  # noqa: E402
from paper_2312_13094_b200.symbolics import fd_coefficients  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="star")
    ap.add_argument("--n", type=int, nargs="+", default=[1024])
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--scale", action="store_true", help="m holds bound dt^2/m")
    a = ap.parse_args()
    if a.scale:
        a.variant |= R.VARIANT_M_IS_SCALE
    n = a.n * 3 if len(a.n) == 1 else a.n
    so = a.so
    r = so // 2
    full = tuple(x + 2 * so for x in n)
    lo = (so,) * 3
    hi = tuple(so + x for x in n)
    w = [float(c) for c in fd_coefficients(2, so)]
    coeffs = [np.float32([w[r + k] / 100.0 for k in range(r + 1)])] * 3
    u = [torch.zeros(full, device="cuda") for _ in range(3)]
    m = torch.ones(full, device="cuda")
    for t in u:
        t.normal_()
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(3):
        R.star_update(u[i % 3], u[(i + 2) % 3], m, u[(i + 1) % 3], full, lo, hi, (r,) * 3,
                      coeffs, 2.0, -1.0, 1e-3, variant=a.variant)
    torch.cuda.synchronize()
    times = []
    for i in range(a.iters):
        ev[0].record(s)
        R.star_update(u[i % 3], u[(i + 2) % 3], m, u[(i + 1) % 3], full, lo, hi, (r,) * 3,
                      coeffs, 2.0, -1.0, 1e-3, variant=a.variant)
        ev[1].record(s)
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]))
    pts = float(np.prod(n))
    t = float(np.median(times)) * 1e-3
    out = {"kernel": a.kernel, "n": n, "so": so, "variant": a.variant, "ms": t * 1e3,
           "gpts": pts / t / 1e9, "gbs_alg": 16 * pts / t / 1e9,
           "frac_hbm": 16 * pts / t / 1e9 / 6555.2, "min_ms": min(times)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
