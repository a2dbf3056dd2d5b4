"""Memory-safety checks without compute-sanitizer (closed on this pool):

* guard zones (``SDMP_GUARD=1``: every field's buffers sit between two
  NaN-canary zones of at least one x-plane, api.Function.check_guard) catch
  writes past either end of a field allocation;
* the exterior-halo invariant (the exterior halo is zero
  forever, never written by exchange or compute) catches writes outside a
  kernel's box inside the allocation: on every side without a neighbour
  the halo (and the z padding) must still be exactly zero in every time
  buffer; sides with a neighbour may hold received halo values.
"""


def exterior_violations(fn, decomp, rank):
    """Number of nonzero cells of ``fn``'s buffers outside the region that
    may legitimately be written (DOMAIN, plus the whole halo on sides with a
    neighbour)."""
    import torch
    st = fn.storage
    nd = decomp.ndims
    keep = []
    for a in range(3):
        h, n = fn.halo3[a], fn.local3[a]
        if a < nd and a < 2:
            lo = 0 if decomp.has_low(rank, a) else h
            hi = h + n + (h if decomp.has_high(rank, a) else 0)
        else:
            lo, hi = h, h + n
        keep.append((lo, hi))
    mask = torch.ones(fn.full3, dtype=torch.bool, device=st.device)
    mask[keep[0][0]:keep[0][1], keep[1][0]:keep[1][1], keep[2][0]:keep[2][1]] = False
    return int(sum(int((st[b][mask] != 0).sum()) for b in range(st.shape[0])))


def check_fields(fields, decomp, rank):
    """[(field name, problem)] for guard or exterior-halo violations."""
    out = []
    for fn in fields:
        if not fn.check_guard():
            out.append((fn.name, "guard zone overwritten"))
        n = exterior_violations(fn, decomp, rank)
        if n:
            out.append((fn.name, f"{n} nonzero exterior-halo cells"))
    return out
