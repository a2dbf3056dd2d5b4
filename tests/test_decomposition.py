"""Product index maps vs the oracle, bit-exact (
SPEC.md:118-260, 358-366, 440-448)."""
import itertools

import numpy as np
import pytest

from oracle import decomp as OD
from oracle import problems as P
from oracle.runtime import Simulation
from paper_2312_13094_b200 import decomposition as PD
from paper_2312_13094_b200 import distfield as DF
from paper_2312_13094_b200.symbolics import GridSpec


@pytest.mark.parametrize("ndims", [2, 3])
def test_default_topology_matches_oracle(ndims):
    for n in range(1, 65):
        assert PD.default_topology(n, ndims).dims == OD.default_topology(n, ndims)


def test_spec_topology_examples():
    assert PD.default_topology(4, 2).dims == (2, 2)
    assert PD.default_topology(16, 3).dims == (4, 2, 2)
    assert PD.default_topology(1, 3).dims == (1, 1, 1)
    assert PD.default_topology(8, 3).dims == (2, 2, 2)


def test_decompose_axis_matches_oracle():
    for n in range(1, 40):
        for p in range(1, n + 1):
            assert PD.decompose_axis(n, p) == OD.decompose_axis(n, p)
    with pytest.raises(PD.DecompositionError):
        PD.decompose_axis(3, 4)


CASES = [((4, 4), (2, 2)), ((13, 7), (3, 2)), ((9, 10, 11), (2, 2, 2)),
         ((12, 9, 8), (4, 2, 1)), ((7, 7, 16), (1, 3, 2)), ((16, 16, 8), (2, 1, 1))]


@pytest.mark.parametrize("shape,dims", CASES)
def test_extents_coords_neighbours(shape, dims):
    d = PD.Decomposition.create(shape, int(np.prod(dims)), dims)
    for r in range(d.nranks):
        assert d.topology.coords(r) == OD.rank_coords(r, dims)
        assert d.extent(r) == OD.extents(shape, dims, r)
        assert d.neighbours(r) == OD.neighbour_table(dims, r)
        # symmetry
        for v, nb in d.neighbours(r).items():
            if nb is not None:
                assert d.neighbour(nb, tuple(-x for x in v)) == r
    # tiling: disjoint + complete
    cnt = np.zeros(shape, dtype=int)
    for r in range(d.nranks):
        cnt[tuple(slice(a, b) for a, b in d.extent(r))] += 1
    assert (cnt == 1).all()


@pytest.mark.parametrize("shape,dims", CASES)
@pytest.mark.parametrize("radius", [0, 1, 2])
def test_regions_match_bruteforce(shape, dims, radius):
    d = PD.Decomposition.create(shape, int(np.prod(dims)), dims)
    nd = len(shape)
    rad = (radius,) * nd
    halo = (max(radius, 1) + 1,) * nd
    for r in range(d.nranks):
        loc = d.local_shape(r)
        lo, hi = OD.side_flags(dims, r)
        if any(n < radius * (int(a) + int(b)) for n, a, b in zip(loc, lo, hi)):
            with pytest.raises(ValueError):
                DF.rank_regions(d, r, rad, DF.RegionName.CORE, halo)
            continue
        core = DF.rank_regions(d, r, rad, DF.RegionName.CORE, halo)
        owned = DF.rank_regions(d, r, rad, DF.RegionName.OWNED, halo)
        assert len(core) == 1
        cmask = OD.boxes_to_mask(core, loc)
        omask = OD.boxes_to_mask(owned, loc)
        assert np.array_equal(cmask.astype(bool), OD.core_mask(loc, lo, hi, rad))
        assert ((cmask + omask) == 1).all()  # disjoint, union = DOMAIN
        assert owned == OD.owned_slabs_reference(loc, lo, hi, rad)
        full = tuple(n + 2 * h for n, h in zip(loc, halo))
        hm = OD.boxes_to_mask(DF.rank_regions(d, r, rad, DF.RegionName.HALO, halo), full, halo)
        assert hm.max() <= 1
        want = np.zeros(full, dtype=int)
        grown = tuple(slice(0 if l else h, n + h + (h if u else 0))
                      for n, h, l, u in zip(loc, halo, lo, hi))
        want[grown] = 1
        want[tuple(slice(h, h + n) for n, h in zip(loc, halo))] = 0
        assert np.array_equal(hm, want)
        if radius == 0:
            assert core[0] == ((0,) * nd, loc) and owned == []


def _as_tuples(msgs):
    return sorted((m.peer, m.direction, m.send, m.recv) for m in msgs)


@pytest.mark.parametrize("shape,dims", CASES)
def test_messages_match_oracle(shape, dims):
    d = PD.Decomposition.create(shape, int(np.prod(dims)), dims)
    nd = len(shape)
    for rad in [(1,) * nd, (2,) * nd, tuple(range(1, nd + 1))]:
        if any(r > n for n, r in zip(min(d.local_shape(k) for k in range(d.nranks)), rad)):
            continue
        for r in range(d.nranks):
            assert _as_tuples(DF.diagonal_messages(d, r, rad)) == sorted(
                OD.diag_messages(shape, dims, r, rad))
            ps = DF.basic_messages(d, r, rad)
            os_ = OD.basic_messages(shape, dims, r, rad)
            assert [_as_tuples(s) for s in ps] == [sorted(s) for s in os_]
            for m in DF.diagonal_messages(d, r, rad):
                # slot is the receiver-side direction pointing back at us
                back = d.neighbour(m.peer, PD.directions(nd)[m.slot]
                                   if nd == 3 else tuple(-x for x in m.direction))
                assert back == r


def test_interior_message_counts():
    # SPEC.md:364-365 / 461 / acceptance 4
    for nd, basic, diag in ((2, 4, 8), (3, 6, 26)):
        dims = (3,) * nd
        d = PD.Decomposition.create((12,) * nd, 3 ** nd, dims)
        mid = d.topology.rank_of((1,) * nd)
        assert DF.message_counts(d, mid, (1,) * nd, "basic") == basic
        assert DF.message_counts(d, mid, (1,) * nd, "diagonal") == diag
        assert DF.message_counts(d, mid, (1,) * nd, "full") == diag


def test_weak_scaling_bytes_constant():
    # acceptance 9: interior-rank bytes per step constant along a weak series
    vols = []
    for dims in [(3, 3, 1), (3, 3, 2), (3, 3, 3)]:
        d = PD.Decomposition.create(tuple(16 * p for p in dims), int(np.prod(dims)), dims)
        mid = d.topology.rank_of(tuple(p // 2 for p in dims))
        vols.append(sum(m.volume for m in DF.diagonal_messages(d, mid, (2, 2, 2))))
    interior = [v for v, dims in zip(vols, [(3, 3, 1), (3, 3, 2), (3, 3, 3)])]
    assert interior[2] >= interior[0]
    # same topology, growing z depth per rank fixed -> identical volume
    v2 = []
    for nz in (1, 2):
        dims = (3, 3, 1)
        d = PD.Decomposition.create((48, 48, 16), 9, dims)
        v2.append(sum(m.volume for m in DF.diagonal_messages(d, 4, (2, 2, 2))))
    assert v2[0] == v2[1]


@pytest.mark.parametrize("mode", ["basic", "diagonal", "full"])
@pytest.mark.parametrize("shape,dims", [((12, 11), (2, 2)), ((10, 9, 12), (2, 2, 1)),
                                        ((12, 10, 9), (2, 2, 2)), ((15, 8, 8), (3, 1, 1))])
def test_product_messages_drive_oracle_to_single_rank_result(shape, dims, mode):
    """The product's message lists, applied by the oracle's simulated ranks,
    reproduce the single-rank result exactly."""
    from tests.test_oracle import acoustic_problem
    d = PD.Decomposition.create(shape, int(np.prod(dims)), dims)

    def product_msgs(rank, radius, m):
        conv = lambda ms: [(x.peer, x.direction, x.send, x.recv) for x in ms]
        if m == "basic":
            return [conv(s) for s in DF.basic_messages(d, rank, radius)]
        return [conv(DF.diagonal_messages(d, rank, radius))]

    out = []
    for dd, msgs in ((None, None), (dims, product_msgs)):
        prob, m = acoustic_problem(shape, dd or (1,) * len(shape), steps=5)
        sim = Simulation(prob, shape, dd, mode=mode, messages=msgs)
        sim.write_global("m", m)
        sim.run(0, 4)
        out.append(sim.gather("u", 5 % 3))
    assert np.array_equal(out[0], out[1])


def test_global_to_local_listing3():
    d = PD.Decomposition.create((4, 4), 4)
    region = (PD.normalise_slice(slice(1, -1), 4),) * 2
    views = []
    for r in range(4):
        loc = PD.global_to_local(d.extent(r), region)
        v = np.zeros((2, 2))
        v[tuple(slice(a, b) for a, b in loc)] = 1
        views.append(v.tolist())
    assert views == [[[0, 0], [0, 1]], [[0, 0], [1, 0]], [[0, 1], [0, 0]], [[1, 0], [0, 0]]]
    assert PD.global_to_local(((0, 2), (0, 2)), ((2, 4), (0, 4))) is None


def test_owners_match_oracle():
    rng = np.random.default_rng(0)
    for shape, dims in [((8, 8), (2, 2)), ((9, 10, 11), (2, 2, 2)), ((20, 12, 8), (4, 2, 1))]:
        extent = tuple(float(n - 1) * 2.5 for n in shape)
        g = GridSpec(shape, extent)
        d = PD.Decomposition.create(shape, int(np.prod(dims)), dims)
        for _ in range(200):
            c = tuple(rng.random() * e for e in extent)
            assert PD.owners_of_point(c, d, g) == OD.owners_of_point(c, shape, extent, dims)
        # boundary nodes exactly on the extent edges are legal
        corner = tuple(extent)
        assert PD.owners_of_point(corner, d, g) == OD.owners_of_point(corner, shape, extent, dims)
