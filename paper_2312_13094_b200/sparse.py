"""Sparse points: multilinear weights, owner routing and the per-rank
device tables for deterministic inject / interpolate.

Routing rules:

* a point is replicated on every rank whose owned box grown by one cell
  contains its enclosing cell (``decomposition.owners_of_point``);
* injection adds only into nodes of the rank's own DOMAIN, so no node is
  counted twice; per node the contributions are summed in point-id order by
  one GPU thread (no float atomics -> bit-reproducible for any topology);
* interpolation is reported by the lowest-rank owner (reads at most one
  halo cell, fresh after the exchange).
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

from .decomposition import Decomposition, enclosing_cell, owners_of_point
from .symbolics import GridSpec


def multilinear_weights(coords: Sequence[float], grid: GridSpec):
    """Enclosing cell corners (row-major, last axis fastest) and weights
    (SPEC.md:497-505)."""
    cell = enclosing_cell(coords, grid)
    frac = [x / h - c for x, h, c in zip(coords, grid.spacing, cell)]
    corners, weights = [], []
    nd = grid.ndims
    for bits in range(1 << nd):
        b = [(bits >> (nd - 1 - a)) & 1 for a in range(nd)]
        w = 1.0
        for a in range(nd):
            w *= frac[a] if b[a] else 1.0 - frac[a]
        corners.append(tuple(c + bi for c, bi in zip(cell, b)))
        weights.append(w)
    return corners, weights


def _full_index(node, ext, halo3, full3):
    idx = [g - e0 + h for g, (e0, _e1), h in zip(node, ext, halo3)]
    idx += [0] * (3 - len(idx))
    return (idx[0] * full3[1] + idx[1]) * full3[2] + idx[2]


def injection_table(coords: np.ndarray, grid: GridSpec, decomp: Decomposition, rank: int,
                    halo3, full3):
    """CSR (node FULL index, ptr, pid, w) of this rank's owned nodes."""
    ext = decomp.extent(rank)
    per_node = {}
    for pid, c in enumerate(np.asarray(coords, dtype=np.float64)):
        if rank not in owners_of_point(c, decomp, grid):
            continue
        corners, weights = multilinear_weights(c, grid)
        for node, w in zip(corners, weights):
            if all(e0 <= g < e1 for g, (e0, e1) in zip(node, ext)):
                per_node.setdefault(node, []).append((pid, w))
    nodes = sorted(per_node)
    node_idx = np.array([_full_index(n, ext, halo3, full3) for n in nodes], dtype=np.int64)
    ptr = np.zeros(len(nodes) + 1, dtype=np.int32)
    pids, ws = [], []
    for i, n in enumerate(nodes):
        contrib = sorted(per_node[n])
        pids += [p for p, _ in contrib]
        ws += [w for _, w in contrib]
        ptr[i + 1] = len(pids)
    return node_idx, ptr, np.array(pids, dtype=np.int32), np.array(ws, dtype=np.float32)


def interpolation_table(coords: np.ndarray, grid: GridSpec, decomp: Decomposition, rank: int,
                        halo3, full3):
    """Points reported by this rank (lowest owner) -> (pids, idx, w)."""
    ext = decomp.extent(rank)
    pids, idx, ws = [], [], []
    for pid, c in enumerate(np.asarray(coords, dtype=np.float64)):
        own = owners_of_point(c, decomp, grid)
        if not own or own[0] != rank:
            continue
        corners, weights = multilinear_weights(c, grid)
        pids.append(pid)
        idx += [_full_index(n, ext, halo3, full3) for n in corners]
        ws += weights
    return (np.array(pids, dtype=np.int32), np.array(idx, dtype=np.int64),
            np.array(ws, dtype=np.float32))
