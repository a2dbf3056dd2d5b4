"""SPEC.md kernels-module worked examples on the GPU path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_13094_b200 import Eq, Grid, Operator, TimeFunction, solve  # noqa: E402
from paper_2312_13094_b200 import kernels as KD  # noqa: E402
from paper_2312_13094_b200 import symbolics as S  # noqa: E402


def test_acoustic_zero_state_stays_zero():
    grid = Grid((24, 20, 16), (230.0, 190.0, 150.0))
    kd = KD.acoustic_model(grid, so=8, name="uz")
    Operator([kd]).apply(time_M=9, dt=float(np.float32(KD.critical_dt(4.6, grid.spacing))))
    assert not np.any(kd.fields["u"].data_gather())


def test_diffusion_constant_field_unchanged_interior():
    grid = Grid((16, 16), (15.0, 15.0))
    u = TimeFunction(name="uc", grid=grid, space_order=4)
    u.data[...] = 3.0
    Operator([Eq(u.forward, solve(Eq(u.dt, u.laplace), u.forward))]).apply(time_M=0, dt=0.1)
    g = u.data_gather()
    assert np.all(g[2:-2, 2:-2] == np.float32(3.0))  # Laplacian of a constant is 0


def test_acoustic_homogeneous_point_source_reflection_symmetric():
    """Ricker source at the centre of an odd grid, homogeneous m: the
    wavefield is symmetric under every axis reflection (bitwise: the per-point
    sums add tap pairs u[-k] + u[+k], commutative) and, to fp32 rounding,
    under axis permutations (max asymmetry)."""
    n = 41
    grid = Grid((n, n, n), (10.0 * (n - 1),) * 3)
    m = float(np.float32(1.0 / 2.5 ** 2))
    kd = KD.acoustic_model(grid, so=8, vp=torch.full((n, n, n), 2.5, dtype=torch.float64,
                                                     device="cuda"), name="ur")
    u = kd.fields["u"]
    steps = 30
    dt = float(np.float32(KD.critical_dt(2.5, grid.spacing)))
    c = 10.0 * (n - 1) / 2
    src = KD.point_source(grid, [(c, c, c)], steps, dt, f0=0.03, name="src_rs")
    Operator([kd, src.inject(u.forward, expr=src * S.DT ** 2 / kd.fields["m"])]).apply(
        time_M=steps - 1, dt=dt, mpi="full")
    g = u.data_gather().astype(np.float64)
    assert np.abs(g).max() > 0
    for ax in range(3):
        assert np.array_equal(g, np.flip(g, ax)), f"not symmetric under reflection of axis {ax}"
    scale = np.abs(g).max()
    for perm in ((1, 0, 2), (0, 2, 1), (2, 1, 0)):
        assert np.abs(g - np.transpose(g, perm)).max() <= 1e-5 * scale
    assert kd.fields["m"].data_gather().min() == np.float32(m)


def test_elastic_zero_state_stays_zero():
    grid = Grid((20, 20, 20), (190.0,) * 3)
    kd = KD.elastic_model(grid, so=4)
    Operator([kd]).apply(time_M=4, dt=float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.1))))
    for n in KD.VNAMES + KD.TNAMES:
        assert not np.any(kd.fields[n].data_gather())


def test_spec_pack_unpack_round_trip():
    """pack then unpack into an equal box of a zeroed field
    reproduces the values (row-major); empty box -> empty buffer."""
    from paper_2312_13094_b200 import api, spec as SP
    g = S.GridSpec((12, 10, 16), (110.0, 90.0, 150.0))
    a = SP.allocate(S.FieldSpec("pk_a", g, 4, 0), comm="self")
    b = SP.allocate(S.FieldSpec("pk_b", g, 4, 0), comm="self")
    a.storage.copy_(torch.randn_like(a.storage))
    box = ((3, 2, 5), (9, 7, 13))
    buf = SP.pack_region(a, box)
    assert buf.numel() == 6 * 5 * 8
    ref = a.storage[0][3:9, 2:7, 5:13].reshape(-1)
    assert torch.equal(buf, ref)
    SP.unpack_region(b, box, buf)
    assert torch.equal(b.storage[0][3:9, 2:7, 5:13], a.storage[0][3:9, 2:7, 5:13])
    assert SP.pack_region(a, ((3, 2, 5), (3, 7, 13))).numel() == 0
    with pytest.raises(ValueError):
        SP.unpack_region(b, box, buf[:-1])
