"""The SPEC operation names (paper_2312_13094_b200.spec) on CPU: allocate /
write_global / gather, build_clusters, build_schedule_tree, spawn_ranks,
kernel factories."""
import numpy as np
import pytest

from paper_2312_13094_b200 import kernels as KD
from paper_2312_13094_b200 import api
from paper_2312_13094_b200 import compiler as CP
from paper_2312_13094_b200 import decomposition as DC
from paper_2312_13094_b200 import spec as SP
from paper_2312_13094_b200 import symbolics as S


def _ring_program(ctx):
    # ring exchange of rank ids, reduce-sum -> 6 on 4 ranks
    ids = ctx.allgather(ctx.rank)
    return sum(ids)


def test_spawn_ranks_ring_sum():
    assert SP.spawn_ranks(4, _ring_program, topology=(2, 2)) == [6, 6, 6, 6]
    with pytest.raises(ValueError):
        SP.spawn_ranks(3, _ring_program, topology=(2, 2))


def test_allocate_write_gather_single_rank():
    api._FUNCS.clear()
    g = S.GridSpec((4, 4), (2.0, 2.0))
    u = S.FieldSpec("u_spec", g, 2, 2)
    f = SP.allocate(u, comm="self")
    assert f.storage.shape == (3, 8, 8, 1)  # time_order 2 -> 3 buffers; 4 + 2 * halo (= SO = 2)
    assert not f.storage.any()
    SP.write_global(f, (slice(1, 3), slice(1, 3)), 1.0)
    gl = SP.gather(f)
    assert gl.sum() == 4 and gl[1:3, 1:3].all()


def test_build_clusters_and_schedule_tree():
    g = S.GridSpec((16, 16), (15.0, 15.0))
    u = S.FieldSpec("u", g, 2, 1)
    eq = S.solve_forward(S.Eq(u.dt, u.laplace), u.forward)
    d4 = DC.Decomposition.create((16, 16), 4, (2, 2))
    d1 = DC.Decomposition.create((16, 16), 1, None)
    (k, spot), = SP.build_clusters([eq], d4)
    assert spot is not None and spot.radius == (1, 1) and [f.name for f, _ in spot.fields] == ["u"]
    (k1, spot1), = SP.build_clusters([eq], d1)
    assert spot1 is None
    tree = SP.build_schedule_tree([eq], d4)
    assert tree.index("Iteration time") < tree.index("HaloSpot(u)") < tree.index("Iteration x")
    assert "HaloSpot" not in SP.build_schedule_tree([eq], d1)


def test_kernel_factories_build_the_named_families():
    api._FUNCS.clear()
    grid = api.Grid((16, 16, 16), (150.0,) * 3, comm="self")
    ks = CP.recognise([api._as_update(q) for q in SP.tti_gxx_kernel(grid, so=4, name="w").equations])
    assert isinstance(ks[0], CP.RotatedKernel)
    el = SP.elastic_kernel(grid, so=4)
    assert el.kernels == [] and len(el.equations) == 9   # written as update equations
    kv, kt = CP.recognise([api._as_update(q) for q in el.equations])
    assert kv.collocated and kt.collocated and (kv.kind, kt.kind) == ("v", "t")
    tti = KD.tti_model(grid, so=4)
    assert tti.kernels == [] and len(tti.equations) == 2
    assert isinstance(CP.recognise(tti.equations)[0], CP.TTIKernel)
    ac = SP.acoustic_kernel(grid, so=4, name="ua")
    assert isinstance(CP.recognise([api._as_update(q) for q in ac.equations])[0], CP.StarKernel)


def _alloc_program(ctx):
    from paper_2312_13094_b200 import spec as SP2
    from paper_2312_13094_b200 import symbolics as S2
    from paper_2312_13094_b200 import decomposition as DC2
    g = S2.GridSpec((4, 4), (2.0, 2.0))
    u = S2.FieldSpec("u", g, 2, 2)
    f = SP2.allocate(u, DC2.Decomposition.create((4, 4), 4, (2, 2)))
    SP2.write_global(f, (slice(1, -1), slice(1, -1)), 1.0)
    return {"full": tuple(f.storage.shape), "view": f.data[:].tolist(),
            "gather": SP2.gather(f).tolist()}


def test_allocate_distributed_listing3():
    """SPEC.md:227 / Listing 3: 4x4 on 2x2 ranks, halo 2 -> 6x6 local
    buffers, 3 time buffers; the interior write gives the four printed views."""
    out = SP.spawn_ranks(4, _alloc_program, topology=(2, 2))
    want = [[[0, 0], [0, 1]], [[0, 0], [1, 0]], [[0, 1], [0, 0]], [[1, 0], [0, 0]]]
    for r in range(4):
        assert out[r]["full"] == (3, 6, 6, 1)
        assert out[r]["view"] == want[r]
    assert np.array(out[0]["gather"]).sum() == 4
