"""Parity at BASELINE sizes through size-independent properties (the CPU
oracle cannot run 1024^3; it is matched at small sizes and at C1 full size,
profiles/r01_c1_parity.json).

Mirror symmetry: on a model that depends on z only, with the source on the
x and y mirror planes, the exact solution is symmetric in x and y.  The
per-point update sums tap pairs (u[-k] + u[+k]) in the same k order at a
point and at its mirror image, and IEEE addition is commutative, so the
computed wavefield must be symmetric BITWISE - at full C2 size (1024^3 per
GPU, odd extents so the mirror planes are grid planes), through the TMA
kernels, the CUDA-graph replay and the sparse injection.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_13094_b200 import Grid, Operator  # noqa: E402
from paper_2312_13094_b200 import kernels as KD  # noqa: E402
from paper_2312_13094_b200 import symbolics as S  # noqa: E402


def test_c2_fullsize_mirror_symmetry():
    shape = (1023, 1023, 1024)
    h = 10.0
    grid = Grid(shape, tuple(h * (n - 1) for n in shape), comm="self")
    kd = KD.acoustic_model(grid, so=8, name="u_mirror")
    u, m = kd.fields["u"], kd.fields["m"]
    nz = shape[2]
    # vp(z) of the C1/C2 law without the hashed noise: symmetric in x and y
    KD._fill([m], lambda gx, gy, gz: (1.0 / (1.5 + 3.0 * gz.double() / (nz - 1)) ** 2,))
    steps = 40
    dt = float(np.float32(KD.critical_dt(4.5, grid.spacing)))
    src = KD.point_source(grid, [(511 * h, 511 * h, 300.3)], steps, dt, f0=0.025, name="src_mirror")
    op = Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / m)])
    op.apply(time_M=steps - 1, dt=dt, mpi="full")
    v = u._domain_view(u._latest)
    assert float(v.abs().max()) > 0
    assert torch.equal(v, v.flip(0)), "wavefield not mirror-symmetric in x"
    assert torch.equal(v, v.flip(1)), "wavefield not mirror-symmetric in y"
