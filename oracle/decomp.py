"""ORACLE (test infrastructure) — decomposition, regions and messages,
restated brute-force from SPEC.md so the product's box algebra
(paper_2312_13094_b200/decomposition.py, distfield.py) is checked
independently, cell by cell.
"""
import itertools
import math

import numpy as np


def default_topology(nranks, ndims):
    """exhaustive search over ordered factorisations;
    minimise max dim, tie -> lexicographically smallest descending tuple."""
    cands = [d for d in itertools.product(range(1, nranks + 1), repeat=ndims)
             if math.prod(d) == nranks]
    best = min(cands, key=lambda d: (max(d), sorted(d, reverse=True)))
    return tuple(sorted(best, reverse=True))


def decompose_axis(n, p):
    """sizes q+1 for the first n%p parts, q after."""
    if p > n:
        raise ValueError("nparts > npoints")
    sizes = [n // p + (1 if i < n % p else 0) for i in range(p)]
    out, s = [], 0
    for z in sizes:
        out.append((s, s + z))
        s += z
    return out


def rank_coords(rank, dims):
    """Row-major, last axis fastest (Listing 3)."""
    return tuple(int(c) for c in np.unravel_index(rank, dims))


def coords_rank(coords, dims):
    if any(c < 0 or c >= d for c, d in zip(coords, dims)):
        return None
    return int(np.ravel_multi_index(coords, dims))


def extents(shape, dims, rank):
    c = rank_coords(rank, dims)
    return tuple(decompose_axis(n, p)[ci] for n, p, ci in zip(shape, dims, c))


def neighbour_table(dims, rank):
    c = rank_coords(rank, dims)
    out = {}
    for v in itertools.product((-1, 0, 1), repeat=len(dims)):
        if any(v):
            out[v] = coords_rank(tuple(ci + vi for ci, vi in zip(c, v)), dims)
    return out


def global_to_local(ext, region):
    """SPEC.md:158-166."""
    out = []
    for (e0, e1), (r0, r1) in zip(ext, region):
        lo, hi = max(e0, r0), min(e1, r1)
        if hi <= lo:
            return None
        out.append((lo - e0, hi - e0))
    return tuple(out)


# --- regions, brute force -----------------------------------

def side_flags(dims, rank):
    c = rank_coords(rank, dims)
    return ([ci > 0 for ci in c], [ci < d - 1 for ci, d in zip(c, dims)])


def core_mask(shape, has_lo, has_hi, radius):
    """A DOMAIN cell is CORE iff every read within ``radius`` along each
    axis stays inside DOMAIN or crosses only a neighbour-less side."""
    m = np.ones(shape, dtype=bool)
    for a, n in enumerate(shape):
        idx = np.arange(n)
        ok = np.ones(n, dtype=bool)
        if has_lo[a]:
            ok &= idx - radius[a] >= 0
        if has_hi[a]:
            ok &= idx + radius[a] <= n - 1
        sl = [None] * len(shape)
        sl[a] = slice(None)
        m &= ok[tuple(sl)]
    return m


def boxes_to_mask(boxes, shape, offset=None):
    """Rasterise boxes (DOMAIN coords + ``offset``) into a counting mask."""
    offset = offset or (0,) * len(shape)
    cnt = np.zeros(shape, dtype=np.int32)
    for lo, hi in boxes:
        sl = tuple(slice(l + o, h + o) for l, h, o in zip(lo, hi, offset))
        cnt[sl] += 1
    return cnt


def owned_slabs_reference(shape, has_lo, has_hi, radius):
    """The SPEC's lexicographic OWNED slab rule: slab on axis a
    spans CORE on earlier axes and full DOMAIN on later ones."""
    nd = len(shape)
    core = [(radius[a] if has_lo[a] else 0, shape[a] - (radius[a] if has_hi[a] else 0))
            for a in range(nd)]
    slabs = []
    for a in range(nd):
        for side, present in ((0, has_lo[a]), (1, has_hi[a])):
            if not present or radius[a] == 0:
                continue
            lo, hi = [], []
            for b in range(nd):
                if b < a:
                    rng = core[b]
                elif b > a:
                    rng = (0, shape[b])
                else:
                    rng = (0, radius[a]) if side == 0 else (shape[a] - radius[a], shape[a])
                lo.append(rng[0]); hi.append(rng[1])
            if all(h > l for l, h in zip(lo, hi)):
                slabs.append((tuple(lo), tuple(hi)))
    return slabs


# --- messages -----------------------------------------------------------------

def diag_messages(shape, dims, rank, radius):
    """for each existing neighbour v, the sender's cells
    within ``radius`` of the shared face/edge/corner.  Returned as
    {peer: (v, send_box_domain, recv_box_in_peer_domain)}."""
    c = rank_coords(rank, dims)
    mine = extents(shape, dims, rank)
    out = []
    for v, peer in neighbour_table(dims, rank).items():
        if peer is None or any(vi and radius[a] == 0 for a, vi in enumerate(v)):
            continue
        theirs = extents(shape, dims, peer)
        send_lo, send_hi, recv_lo, recv_hi = [], [], [], []
        for a, vi in enumerate(v):
            n = mine[a][1] - mine[a][0]
            # global cells shipped along a, then shifted into peer coords
            if vi == 0:
                g0, g1 = mine[a]
            elif vi > 0:
                g0, g1 = mine[a][1] - radius[a], mine[a][1]
            else:
                g0, g1 = mine[a][0], mine[a][0] + radius[a]
            send_lo.append(g0 - mine[a][0]); send_hi.append(g1 - mine[a][0])
            recv_lo.append(g0 - theirs[a][0]); recv_hi.append(g1 - theirs[a][0])
        out.append((peer, v, (tuple(send_lo), tuple(send_hi)),
                    (tuple(recv_lo), tuple(recv_hi))))
    return out


def basic_messages(shape, dims, rank, radius):
    """axis a exchanged after axes < a, including the halo
    columns received so far on neighbour sides."""
    mine = extents(shape, dims, rank)
    has_lo, has_hi = side_flags(dims, rank)
    c = rank_coords(rank, dims)
    steps = []
    for a in range(len(dims)):
        msgs = []
        for s in (-1, 1):
            peer = coords_rank(tuple(ci + (s if b == a else 0) for b, ci in enumerate(c)), dims)
            if peer is None or radius[a] == 0:
                continue
            theirs = extents(shape, dims, peer)
            send_lo, send_hi, recv_lo, recv_hi = [], [], [], []
            for b in range(len(dims)):
                if b == a:
                    g0, g1 = ((mine[b][1] - radius[b], mine[b][1]) if s > 0
                              else (mine[b][0], mine[b][0] + radius[b]))
                elif b < a:
                    g0 = mine[b][0] - (radius[b] if has_lo[b] else 0)
                    g1 = mine[b][1] + (radius[b] if has_hi[b] else 0)
                else:
                    g0, g1 = mine[b]
                send_lo.append(g0 - mine[b][0]); send_hi.append(g1 - mine[b][0])
                recv_lo.append(g0 - theirs[b][0]); recv_hi.append(g1 - theirs[b][0])
            msgs.append((peer, tuple(s if b == a else 0 for b in range(len(dims))),
                         (tuple(send_lo), tuple(send_hi)), (tuple(recv_lo), tuple(recv_hi))))
        steps.append(msgs)
    return steps


def owners_of_point(coords, shape, extent, dims, support=1):
    """ranks whose owned node box grown by ``support``
    cells contains both corner nodes of the enclosing cell on every axis."""
    h = [e / (n - 1) for e, n in zip(extent, shape)]
    cell = [min(max(int(math.floor(x / hi)), 0), n - 2) for x, hi, n in zip(coords, h, shape)]
    out = []
    for r in range(math.prod(dims)):
        ext = extents(shape, dims, r)
        if all(e0 - support <= ci and ci + 1 <= e1 - 1 + support
               for ci, (e0, e1) in zip(cell, ext)):
            out.append(r)
    return out
