"""NVLink transfer rates of the halo mechanisms (one process, GPU 0 -> GPU 1),
timed with CUDA events on the issuing stream of GPU 0:

* the copy engine (`sdmp_copy_box` engine 0, cudaMemcpy3DAsync), as used by
  diagonal / basic mode, for the BASELINE message shapes: an x-face (R
  planes) and a y-face (R rows) of a 1024^3 rank with halo 8, with and
  without whole-z rows (SDMP_WHOLE_Z);
* SM stores into peer memory (`sdmp_copy_box` engine 1, scalar stores; engine
  2, the batched post kernel with 16-byte stores -- the store path of the
  diagonal / basic default and, per point, of the fused full-mode push),
  same shapes;
* a plain 1 GiB contiguous peer copy as the link ceiling.

Prints one JSON line per case: bytes moved, ms, GB/s, fraction of 900 GB/s.

    python tools/nvlink_bw.py [--n 1024] [--r 4] [--reps 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_13094_b200 import runtime as R  # noqa: E402


def timed(fn, reps):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--r", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    n, r, h = a.n, a.r, 8
    full = (n + 2 * h, n + 2 * h, n + 2 * h)
    torch.cuda.set_device(0)
    src = torch.randn(full, device="cuda:0")
    dst = torch.zeros(full, device="cuda:1")
    R.check(R.lib().sdmp_enable_peer(1), "enable_peer")
    torch.cuda.set_device(1)
    R.check(R.lib().sdmp_enable_peer(0), "enable_peer")
    torch.cuda.set_device(0)
    cases = {
        # x-face: planes [n+h-r, n+h) -> receiver halo [0+h-r... ] (rows of n z)
        "x_face": ((n + h - r, h, h), (h - r, h, h), (r, n, n)),
        "y_face": ((h, n + h - r, h), (h, h - r, h), (n, r, n)),
        "xy_edge": ((n + h - r, n + h - r, h), (h - r, h - r, h), (r, r, n)),
    }
    out = []
    for name, (slo, dlo, ext) in cases.items():
        for whole_z in (False, True):
            s_lo, d_lo, e = list(slo), list(dlo), list(ext)
            if whole_z:
                s_lo[2], d_lo[2], e[2] = 0, 0, full[2]
            nbytes = 4 * e[0] * e[1] * e[2]
            for engine in (0, 1, 2):
                ms = timed(lambda: R.copy_box(src, full, s_lo, dst, full, d_lo, e, engine), a.reps)
                out.append({"case": name, "whole_z": whole_z,
                            "engine": ["copy engine (cudaMemcpy3DAsync)",
                                       "SM peer stores (one kernel per box)",
                                       "SM peer stores (batched post kernel, 16-byte)"][engine],
                            "bytes": nbytes, "ms": ms,
                            "gbs": nbytes / (ms * 1e-3) / 1e9,
                            "frac_of_900": nbytes / (ms * 1e-3) / 1e9 / 900.0})
    big_s = torch.empty(1 << 28, device="cuda:0")
    big_d = torch.empty(1 << 28, device="cuda:1")
    ms = timed(lambda: big_d.copy_(big_s, non_blocking=True), max(4, a.reps // 4))
    out.append({"case": "contiguous 1 GiB", "engine": "copy engine (torch peer copy)",
                "bytes": 4 << 28, "ms": ms, "gbs": (4 << 28) / (ms * 1e-3) / 1e9,
                "frac_of_900": (4 << 28) / (ms * 1e-3) / 1e9 / 900.0})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
