"""ORACLE (test infrastructure) — simulated SPMD ranks executing the three
exchange modes in fp64 numpy.

A *problem* (oracle/problems.py) supplies fields, per-step phases and sparse
terms; this module owns per-rank FULL buffers, the halo exchange and the
box schedule:

* basic    — per phase, axis-sequenced face exchange, then DOMAIN;
* diagonal — per phase, single-step exchange to all neighbours, then DOMAIN;
* full     — per phase, post, CORE, wait, OWNED slabs (Listing 8).

Message geometry comes from ``oracle.decomp`` by default; tests can inject
the product's message lists (``messages=``) to check them against the
single-rank result.
"""
import math

import numpy as np

from . import decomp as D


def _sl(box, halo):
    return tuple(slice(l + h, u + h) for l, u, h in zip(box[0], box[1], halo))


class Rank:
    def __init__(self, rank, problem, shape, dims):
        self.rank = rank
        self.ext = D.extents(shape, dims, rank)
        self.local = tuple(b - a for a, b in self.ext)
        self.halo = problem.halo
        full = tuple(n + 2 * h for n, h in zip(self.local, self.halo))
        self.arrays = {name: [np.zeros(full) for _ in range(nb)]
                       for name, nb in problem.fields.items()}
        self.has_lo, self.has_hi = D.side_flags(dims, rank)

    def buf(self, name, time, tshift=0):
        bufs = self.arrays[name]
        return bufs[(time + tshift) % len(bufs)]


class Simulation:
    def __init__(self, problem, shape, dims=None, mode="diagonal", messages=None, threads=1):
        self.p = problem
        # threads > 1: each compute box is cut into x-slabs evaluated
        # concurrently (numpy releases the GIL; every per-point update writes
        # only its own box of an output buffer it does not read, so slabs are
        # independent and the result is identical to one call)
        self.threads = max(1, int(threads))
        self._pool = None
        self.shape = tuple(shape)
        self.dims = tuple(dims) if dims else (1,) * len(shape)
        self.mode = mode
        self.nranks = math.prod(self.dims)
        self.ranks = [Rank(r, problem, self.shape, self.dims) for r in range(self.nranks)]
        self.messages = messages
        self.traces = {}
        self.msg_count = 0
        self.msg_cells = 0

    # -- data in/out ------------------------------------
    def write_global(self, name, array, buffers=None):
        array = np.asarray(array, dtype=np.float64)
        for rk in self.ranks:
            sl = tuple(slice(a, b) for a, b in rk.ext)
            bufs = rk.arrays[name] if buffers is None else [rk.arrays[name][b] for b in buffers]
            for arr in bufs:
                arr[_sl(((0,) * len(rk.local), rk.local), rk.halo)] = array[sl]

    def gather(self, name, buffer):
        out = np.zeros(self.shape)
        for rk in self.ranks:
            sl = tuple(slice(a, b) for a, b in rk.ext)
            out[sl] = rk.arrays[name][buffer][_sl(((0,) * len(rk.local), rk.local), rk.halo)]
        return out

    def exchange_static(self, names, radius):
        """Hoisted one-off exchange of read-only coefficient fields
        (optimize_halospots 'hoist')."""
        self._exchange([(n, 0) for n in names], radius, time=0)

    # -- exchange -----------------------------------------------------------
    def _msgs(self, rank, radius):
        if self.messages is not None:
            return self.messages(rank, radius, self.mode)
        if self.mode == "basic":
            return D.basic_messages(self.shape, self.dims, rank, radius)
        return [D.diag_messages(self.shape, self.dims, rank, radius)]

    def _exchange(self, fields, radius, time):
        if self.nranks == 1:
            return
        per_rank = [self._msgs(r, radius) for r in range(self.nranks)]
        nsteps = max(len(s) for s in per_rank)
        for step in range(nsteps):
            # snapshot sends first (all ranks post, then all receive)
            pending = []
            for r, steps in enumerate(per_rank):
                for peer, _v, sbox, rbox in (steps[step] if step < len(steps) else []):
                    src = self.ranks[r]
                    for name, tsh in fields:
                        data = src.buf(name, time, tsh)[_sl(sbox, src.halo)].copy()
                        pending.append((peer, name, tsh, rbox, data))
                    self.msg_count += 1
                    self.msg_cells += int(np.prod([h - l for l, h in zip(*sbox)]))
            for peer, name, tsh, rbox, data in pending:
                dst = self.ranks[peer]
                dst.buf(name, time, tsh)[_sl(rbox, dst.halo)] = data

    def _compute(self, ph, rk, fb, time):
        lo, hi = fb
        n0 = hi[0] - lo[0]
        if self.threads == 1 or n0 < 2 * self.threads:
            ph.compute(rk, fb, time)
            return
        if self._pool is None:
            from concurrent.futures import ThreadPoolExecutor
            self._pool = ThreadPoolExecutor(self.threads)
        cuts = np.linspace(lo[0], hi[0], self.threads + 1).astype(int)
        boxes = [((int(a),) + tuple(lo[1:]), (int(b),) + tuple(hi[1:]))
                 for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        list(self._pool.map(lambda b: ph.compute(rk, b, time), boxes))

    # -- time loop ----------------------------------------------------------
    def run(self, time_m, time_M):
        for time in range(time_m, time_M + 1):
            for ph in self.p.phases:
                self._exchange(ph.exchange, ph.radius, time)
                for rk in self.ranks:
                    if ph.before is not None:
                        ph.before(self, rk, time)
                    if self.mode == "full":
                        core = [(tuple(ph.radius[a] if rk.has_lo[a] else 0 for a in range(len(rk.local))),
                                 tuple(n - (ph.radius[a] if rk.has_hi[a] else 0)
                                       for a, n in enumerate(rk.local)))]
                        boxes = core + D.owned_slabs_reference(rk.local, rk.has_lo, rk.has_hi, ph.radius)
                    else:
                        boxes = [((0,) * len(rk.local), rk.local)]
                    for box in boxes:
                        if all(h > l for l, h in zip(*box)):
                            fb = tuple(tuple(x + h for x, h in zip(c, rk.halo)) for c in box)
                            self._compute(ph, rk, fb, time)
                    if ph.after is not None:
                        ph.after(self, rk, time)
