"""Region algebra (CORE / OWNED / HALO / DOMAIN / FULL) and halo-message
boxes for the three exchange modes.

Implements ``distfield.region_boxes`` and the message
geometry of ``runtime.halo_exchange`` (basic axis-sequenced
rule 376).  Boxes are half-open ``(lo, hi)`` tuples in DOMAIN coordinates:
index 0 is the first owned point, HALO cells are negative or >= n.  FULL
coordinates (the device layout) add the per-axis halo width
(``align_accesses``).

All of this is integer bookkeeping executed once at plan build; it is
checked bit-exactly against ``oracle/decomp.py``.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

from .decomposition import Decomposition, directions, direction_slot

Box = Tuple[Tuple[int, ...], Tuple[int, ...]]


class RegionName(enum.Enum):
    CORE = "CORE"
    OWNED = "OWNED"
    HALO = "HALO"
    DOMAIN = "DOMAIN"
    FULL = "FULL"


def box_volume(box: Box) -> int:
    v = 1
    for lo, hi in zip(*box):
        v *= max(0, hi - lo)
    return v


def box_empty(box: Box) -> bool:
    return any(hi <= lo for lo, hi in zip(*box))


def to_full(box: Box, halo: Sequence[int]) -> Box:
    """DOMAIN coordinates -> FULL (device array) coordinates."""
    lo, hi = box
    return (tuple(l + h for l, h in zip(lo, halo)), tuple(u + h for u, h in zip(hi, halo)))


def region_boxes(shape: Sequence[int], has_lo: Sequence[bool], has_hi: Sequence[bool],
                 radius: Sequence[int], name: RegionName,
                 halo: Optional[Sequence[int]] = None) -> List[Box]:
    """Disjoint boxes of region ``name`` for a rank with local ``shape``.

    CORE = DOMAIN shrunk by ``radius`` on sides that have a neighbour;
    OWNED = DOMAIN minus CORE as <= 2*ndims lexicographic slabs (axis-0
    slabs full width, later axes restricted to CORE's range on earlier
    axes); HALO = cells outside DOMAIN within ``halo`` on neighbour sides
    (SPEC.md:255), also split lexicographically so boxes stay disjoint.
    """
    nd = len(shape)
    if halo is None:
        halo = radius
    if any(r > h for r, h in zip(radius, halo)):
        raise ValueError("radius exceeds halo")
    dom = (tuple(0 for _ in shape), tuple(shape))
    if name is RegionName.DOMAIN:
        return [dom]
    if name is RegionName.FULL:
        return [(tuple(-h for h in halo), tuple(n + h for n, h in zip(shape, halo)))]
    core_lo = tuple(r if lo else 0 for r, lo in zip(radius, has_lo))
    core_hi = tuple(n - (r if hi else 0) for n, r, hi in zip(shape, radius, has_hi))
    if any(h < l for l, h in zip(core_lo, core_hi)):
        raise ValueError(f"radius {tuple(radius)} leaves no CORE in local shape "
                         f"{tuple(shape)} (use fewer ranks along that axis)")
    if name is RegionName.CORE:
        return [(core_lo, core_hi)]
    if name is RegionName.OWNED:
        inner_lo, inner_hi = core_lo, core_hi
        outer_lo, outer_hi = dom
        width_lo = [r if lo else 0 for r, lo in zip(radius, has_lo)]
        width_hi = [r if hi else 0 for r, hi in zip(radius, has_hi)]
    elif name is RegionName.HALO:
        inner_lo, inner_hi = dom
        outer_lo = tuple(-h if lo else 0 for h, lo in zip(halo, has_lo))
        outer_hi = tuple(n + (h if hi else 0) for n, h, hi in zip(shape, halo, has_hi))
        width_lo = [h if lo else 0 for h, lo in zip(halo, has_lo)]
        width_hi = [h if hi else 0 for h, hi in zip(halo, has_hi)]
    else:  # pragma: no cover
        raise ValueError(name)
    out = []
    for a in range(nd):
        for side in (0, 1):
            w = width_lo[a] if side == 0 else width_hi[a]
            if w == 0:
                continue
            lo, hi = [], []
            for b in range(nd):
                if b < a:
                    lo.append(inner_lo[b]); hi.append(inner_hi[b])
                elif b > a:
                    lo.append(outer_lo[b]); hi.append(outer_hi[b])
                elif side == 0:
                    lo.append(outer_lo[b]); hi.append(inner_lo[b])
                else:
                    lo.append(inner_hi[b]); hi.append(outer_hi[b])
            box = (tuple(lo), tuple(hi))
            if not box_empty(box):
                out.append(box)
    return out


def rank_regions(decomp: Decomposition, rank: int, radius: Sequence[int],
                 name: RegionName, halo: Optional[Sequence[int]] = None) -> List[Box]:
    nd = decomp.ndims
    return region_boxes(decomp.local_shape(rank),
                        [decomp.has_low(rank, a) for a in range(nd)],
                        [decomp.has_high(rank, a) for a in range(nd)],
                        radius, name, halo)


# ---------------------------------------------------------------------------
# Messages


@dataclass(frozen=True)
class Message:
    """One halo transfer from this rank to ``peer``.

    ``send`` is in the sender's DOMAIN coordinates; ``recv`` is where the
    same cells land in the *receiver's* DOMAIN coordinates.  ``slot`` is the
    receiver-side direction slot (the direction pointing back at the
    sender), used for completion flags.
    """

    peer: int
    direction: tuple
    send: Box
    recv: Box
    slot: int

    @property
    def volume(self) -> int:
        return box_volume(self.send)


def _axis_span(v: int, n: int, r: int, send: bool) -> Tuple[int, int]:
    if v < 0:
        return (0, r) if send else (-r, 0)
    if v > 0:
        return (n - r, n) if send else (n, n + r)
    return (0, n)


def diagonal_messages(decomp: Decomposition, rank: int,
                      radius: Sequence[int]) -> List[Message]:
    """Single-step exchange to every existing neighbour.

    Returns the messages this rank SENDS; receive boxes are expressed in
    the receiver's coordinates.  Axes with zero radius contribute no
    directions that move along them.
    """
    shape = decomp.local_shape(rank)
    out = []
    for v in directions(decomp.ndims):
        if any(vi != 0 and radius[a] == 0 for a, vi in enumerate(v)):
            continue
        peer = decomp.neighbour(rank, v)
        if peer is None:
            continue
        pshape = decomp.local_shape(peer)
        send_lo, send_hi, recv_lo, recv_hi = [], [], [], []
        for a, vi in enumerate(v):
            s0, s1 = _axis_span(vi, shape[a], radius[a], True)
            # receiver sees the data on its -v side
            r0, r1 = _axis_span(-vi, pshape[a], radius[a], False)
            send_lo.append(s0); send_hi.append(s1)
            recv_lo.append(r0); recv_hi.append(r1)
        out.append(Message(peer, tuple(v), (tuple(send_lo), tuple(send_hi)),
                           (tuple(recv_lo), tuple(recv_hi)),
                           direction_slot(tuple(-x for x in v))))
    return out


def basic_messages(decomp: Decomposition, rank: int,
                   radius: Sequence[int]) -> List[List[Message]]:
    """Axis-sequenced face exchange: one list per axis, in
    axis order.  On axes already exchanged the box spans the received halo
    on sides that have a neighbour (exterior halo columns, always zero, are
    not shipped — SURVEY.md Appendix B decision)."""
    nd = decomp.ndims
    shape = decomp.local_shape(rank)
    steps = []
    for a in range(nd):
        msgs = []
        if radius[a] == 0:
            steps.append(msgs)
            continue
        for s in (-1, 1):
            v = tuple(s if b == a else 0 for b in range(nd))
            peer = decomp.neighbour(rank, v)
            if peer is None:
                continue
            pshape = decomp.local_shape(peer)
            send_lo, send_hi, recv_lo, recv_hi = [], [], [], []
            for b in range(nd):
                if b == a:
                    s0, s1 = _axis_span(s, shape[b], radius[b], True)
                    r0, r1 = _axis_span(-s, pshape[b], radius[b], False)
                elif b < a:
                    # both ranks share the coordinate along b (same slab of
                    # the topology), so their b-neighbour sets coincide
                    lo = -radius[b] if decomp.has_low(rank, b) else 0
                    hi = shape[b] + (radius[b] if decomp.has_high(rank, b) else 0)
                    s0, s1 = lo, hi
                    r0, r1 = lo, hi
                else:
                    s0, s1 = 0, shape[b]
                    r0, r1 = 0, pshape[b]
                send_lo.append(s0); send_hi.append(s1)
                recv_lo.append(r0); recv_hi.append(r1)
            msgs.append(Message(peer, v, (tuple(send_lo), tuple(send_hi)),
                                (tuple(recv_lo), tuple(recv_hi)),
                                direction_slot(tuple(-x for x in v))))
        steps.append(msgs)
    return steps


def message_counts(decomp: Decomposition, rank: int, radius: Sequence[int],
                   mode: str) -> int:
    """Messages sent by ``rank`` per exchange epoch."""
    if mode == "basic":
        return sum(len(m) for m in basic_messages(decomp, rank, radius))
    return len(diagonal_messages(decomp, rank, radius))
