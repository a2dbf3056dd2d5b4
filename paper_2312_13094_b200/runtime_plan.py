"""Instantiate an ExecPlan on this rank's GPU: bind fp32 parameters once,
register local and peer (IPC-mapped) buffers, encode native actions, run.

This is the ``RankContext`` + ``execute_plan_full`` side of the SPEC
 for one process per B200: the plan executor in libsdmp
replays the action list; halo pushes go straight into the neighbours' HALO
regions over NVLink (peer pointers imported with cudaIpcOpenMemHandle).
"""
from __future__ import annotations

import math
import os
from fractions import Fraction
from typing import Dict, List

import numpy as np

from . import compiler as CP
from . import runtime as R
from . import sparse as SP
from . import symbolics as S
from .decomposition import direction_slot

NFLAGS = 32


def _f32(x) -> float:
    return float(np.float32(float(x)))


def star_binding(k: CP.StarKernel, spacing, dt):
    """fp32 parameters of the star kernel: coefficient table, A, B, C."""
    nd = len(spacing)
    coeffs = []
    for a in range(3):
        if a < nd:
            h = spacing[a]
            coeffs.append([_f32(float(w) / (h * h)) for w in k.weights[a]])
        else:
            coeffs.append([0.0])
    if k.p > 0 and dt is None:
        raise ValueError("this operator needs dt")
    C = _f32(float(k.c) * (float(dt) ** k.p if k.p else 1.0))
    return coeffs, _f32(k.A), _f32(k.B), C


def tti_binding(k: CP.TTIKernel, spacing, dt):
    r = k.so // 2
    w2 = [float(c) for c in S.fd_coefficients(2, k.so)]
    w1 = [float(c) for c in S.fd_coefficients(1, k.so)]
    lap = [[_f32(w2[r + j] / (h * h)) for j in range(r + 1)] for h in spacing]
    d1 = [[0.0] + [_f32(w1[r + j] / h) for j in range(1, r + 1)] for h in spacing]
    return lap, d1, _f32(float(dt) * float(dt))


def staggered_binding(k: CP.StaggeredPhase, spacing, dt):
    if k.collocated:  # centred first-derivative weights w_k, k = 1..R
        r = k.so // 2
        w1 = [float(x) for x in S.fd_coefficients(1, k.so)]
        c = [w1[r + j] for j in range(1, r + 1)]
    else:
        c = [float(x) for x in S.staggered_coefficients(k.so)]
    return [[_f32(ci / h) for ci in c] for h in spacing], _f32(dt)


class NativeOperatorPlan:
    def __init__(self, op, mode: str, dt, exchange: bool = True):
        torch = __import__("torch")
        self.op = op
        self.mode = mode
        self.dt = dt
        grid = op.grid
        self.ctx = ctx = grid.ctx
        self.rank = rank = ctx.rank
        decomp = grid.decomposition
        self.eplan = op.plan(mode, dt, exchange=exchange)
        ep = self.eplan
        self.plan = R.NativePlan(ctx.device or 0, ep.phases_per_step, rank)
        self.static = None
        self._seen = {}  # static-field versions the bound buffers reflect
        self.keep = []
        self.fid: Dict[S.FieldSpec, int] = {}
        for spec, fn in op.fields.items():
            self.fid[spec] = self.plan.add_field(fn.buffer_ptrs(), fn.full3)

        # -- peers: fields and flags --------------------------------------
        exchanged = []
        for a in ep.actions:
            if a.kind == "post":
                for f, _t in a.spot.fields:
                    if f not in exchanged:
                        exchanged.append(f)
        if ep.hoisted is not None:
            for f, _t in ep.hoisted.fields:
                if f not in exchanged:
                    exchanged.append(f)
        self.flags = R.flags_alloc(NFLAGS)
        self.plan.set_local_flags(self.flags)
        need_static = ep.hoisted is not None and decomp.nranks > 1
        if need_static:
            self.static = R.NativePlan(ctx.device or 0, 1, rank)
            self.static_flags = R.flags_alloc(NFLAGS)
            self.static.set_local_flags(self.static_flags)
            self.static_fid = {f: self.static.add_field(op.fields[f].buffer_ptrs(),
                                                        op.fields[f].full3)
                               for f, _t in ep.hoisted.fields}
        mine = {}
        if decomp.nranks > 1:
            for f in exchanged:
                fn = op.fields[f]
                mine[f.name] = ([R.ipc_export(p) for p in fn.buffer_ptrs()], fn.full3)
            flags_h = R.ipc_export(self.flags)
            sflags_h = R.ipc_export(self.static_flags) if need_static else None
            table = ctx.allgather((mine, flags_h, sflags_h))
        peers = set()
        for a in ep.actions:
            if a.kind == "post":
                peers |= {m.peer for m in a.messages}
        for m in ep.hoisted_messages:
            peers.add(m.peer)
        self.pfid = {}
        self.pflag = {}
        self.spfid, self.spflag = {}, {}
        for q in sorted(peers):
            fields_q, fh, sfh = table[q]
            for f in exchanged:
                handles, full = fields_q[f.name]
                ptrs = [R.ipc_import(h, off) for h, off in handles]
                self.pfid[(q, f)] = self.plan.add_field(ptrs, full)
                if need_static and f in self.static_fid:
                    self.spfid[(q, f)] = self.static.add_field(ptrs, full)
            self.pflag[q] = self.plan.add_flags(R.ipc_import(*fh))
            if need_static:
                self.spflag[q] = self.static.add_flags(R.ipc_import(*sfh))

        # -- bound parameters ------------------------------------------------
        self.scale_bufs = []  # (out tensor, m tensor, C)
        self.cfl = []         # (StarKernel, m Function): acoustic CFL guard
        self.var_bufs = []    # (VarStarKernel, u Function, {"A"|"B"|"S": tensor})
        self.kparams = {}
        spacing = grid.spacing
        for k in op.kernels:
            if isinstance(k, CP.StarKernel):
                coeffs, A, B, C = star_binding(k, spacing, dt)
                mid = -1
                variant = 0
                if k.m is not None:
                    mfn = op.fields[k.m]
                    sbuf = torch.zeros_like(mfn.storage[0])
                    self.scale_bufs.append((sbuf, mfn, C))
                    if (k.A, k.B, k.p, k.q) == (2, -1, 2, -1):
                        self.cfl.append((k, mfn))
                    mid = self.plan.add_field([int(sbuf.data_ptr())], mfn.full3)
                    variant = R.VARIANT_M_IS_SCALE
                    self.keep.append(sbuf)
                tab = R.coeff_table(coeffs, R.SDMP_NCOEF)
                self.kparams[id(k)] = (list(tab.ravel()) + [A, B, C], mid, variant)
            elif isinstance(k, CP.VarStarKernel):
                if dt is None:
                    raise ValueError("this operator needs dt")
                nd = len(spacing)
                coeffs = [[_f32(float(w) / (spacing[a] * spacing[a])) for w in k.weights[a]]
                          if a < nd else [0.0] for a in range(3)]
                ufn = op.fields[k.u]
                names = ("A", "B", "S") if k.has_prev else ("A", "S")
                bufs = {n: torch.zeros_like(ufn.storage[0]) for n in names}
                ids = {n: self.plan.add_field([int(b.data_ptr())], ufn.full3) for n, b in bufs.items()}
                self.keep.extend(bufs.values())
                self.var_bufs.append((k, ufn, bufs))
                tab = R.coeff_table(coeffs, R.SDMP_NCOEF)
                self.kparams[id(k)] = (list(tab.ravel()), ids["A"], ids.get("B", -1), ids["S"])
            elif isinstance(k, CP.RotatedKernel):
                r = k.so // 2
                w1 = [float(c) for c in S.fd_coefficients(1, k.so)]
                d1 = [[0.0] + [_f32(w1[r + j] / h) for j in range(1, r + 1)] for h in spacing]
                dt2 = _f32(float(dt) * float(dt))
                self.kparams[id(k)] = (list(R.coeff_table(d1, R.SDMP_NCOEF).ravel()) + [dt2],
                                       self._bound_scale(op.fields[k.m], dt2))
            elif isinstance(k, CP.TTIKernel):
                lap, d1, dt2 = tti_binding(k, spacing, dt)
                fl = list(R.coeff_table(lap, R.SDMP_NCOEF).ravel()) + \
                    list(R.coeff_table(d1, R.SDMP_NCOEF).ravel()) + [dt2]
                self.kparams[id(k)] = (fl, self._bound_scale(op.fields[k.m], dt2))
            elif isinstance(k, CP.StaggeredPhase):
                sc, dtf = staggered_binding(k, spacing, dt)
                self.kparams[id(k)] = (list(R.coeff_table(sc, R.SDMP_MAX_RADIUS).ravel()) + [dtf],)

        # -- sparse tables --------------------------------------------------
        self.sparse_sets = {}
        for t in op.sparse_terms:
            self._add_sparse(t, decomp, rank)

        # -- actions --------------------------------------------------------
        self.native_index = []
        for a in ep.actions:
            self._encode(a, decomp, rank)
        if need_static:
            self._encode_static(ep, decomp, rank)
        # CUDA-graph replay of whole buffer-rotation periods (SDMP_GRAPH=0
        # disables); removes per-step launch overhead on small grids
        self.plan.set_graph(os.environ.get("SDMP_GRAPH", "1") != "0")

    # ------------------------------------------------------------------
    def _bound_scale(self, mfn, dt2):
        """S = fp32(dt^2) / m bound once per static-field version (the
        kernels read S instead of dividing per point; __fdiv_rn in both
        places, so the bits are unchanged).  Returns S's plan field id."""
        torch = __import__("torch")
        sbuf = torch.zeros_like(mfn.storage[0])
        self.scale_bufs.append((sbuf, mfn, dt2))
        self.keep.append(sbuf)
        return self.plan.add_field([int(sbuf.data_ptr())], mfn.full3)

    def _full_box(self, spec, box):
        fn = self.op.fields[spec]
        nd = len(box[0])
        lo = [l + h for l, h in zip(box[0], fn.halo3)] + [0] * (3 - nd)
        hi = [u + h for u, h in zip(box[1], fn.halo3)] + [1] * (3 - nd)
        return lo, hi

    def _encode(self, a: CP.Action, decomp, rank):
        P = self.plan
        # ExecPlan action -> index of its native action (-1: nothing to do)
        self.native_index.append(self.plan.nact)
        if a.kind == "compute":
            ints, fl = self._compute_ints(a.kernel, a.box, a.stream)
            P.add_action(ints + self._push_ints(a), fl)
        elif a.kind == "post":
            if not a.messages:
                self.native_index[-1] = -1
                return
            P.add_action(self._post_ints(a, self.fid, self.pfid, self.pflag, decomp, rank))
        elif a.kind == "wait":
            slots = sorted({direction_slot(m.direction) for m in a.messages})
            if not slots:
                self.native_index[-1] = -1
                return
            P.add_action([R.ACT["WAIT"], a.stream, a.phase, len(slots)] + slots)
        elif a.kind == "record":
            P.add_action([R.ACT["RECORD"], a.stream, a.event])
        elif a.kind == "streamwait":
            P.add_action([R.ACT["STREAMWAIT"], a.stream, a.event])
        elif a.kind == "inject":
            sid, mid, C = self.sparse_sets[id(a.sparse)][:3]
            P.add_action([R.ACT["INJECT"], a.stream, self.fid[a.sparse.field], 1, mid, sid]
                         + self._push_ints(a), [C])
        elif a.kind == "interp":
            sid = self.sparse_sets[id(a.sparse)][0]
            P.add_action([R.ACT["INTERP"], a.stream, self.fid[a.sparse.field], 0, sid])

    PUSH_MAGIC = -77

    def _push_ints(self, a) -> list:
        """Fused-push block (csrc/plan.cu parse_push): each output value of
        the action inside a send box is also stored into the neighbour's
        HALO (same buffer rotation, tshift +1)."""
        if a.push is None:
            return []
        outs, msgs, sends = a.push
        # directions no output crosses are dropped (per-field halo radii)
        keep = [d for d in range(len(msgs)) if any(fs[d] for fs in sends)]
        msgs = [msgs[d] for d in keep]
        sends = [[fs[d] for d in keep] for fs in sends]
        if not msgs:
            return []
        fn = self.op.fields[outs[0]]
        h = fn.halo3
        nd = len(msgs[0].send[0])
        ints = [self.PUSH_MAGIC, len(msgs), len(outs), 1]
        for m in msgs:
            lo = [l + hh for l, hh in zip(m.send[0], h)] + [0] * (3 - nd)
            hi = [u + hh for u, hh in zip(m.send[1], h)] + [1] * (3 - nd)
            off = [r - s_ for r, s_ in zip(m.recv[0], m.send[0])] + [0] * (3 - nd)
            ints += lo + hi + off
        for f, fs in zip(outs, sends):
            for m, s_ in zip(msgs, fs):
                # -1: the neighbour never reads f across this face (no store)
                ints.append(self.pfid[(m.peer, f)] if s_ else -1)
        return ints

    def _post_ints(self, a, fid, pfid, pflag, decomp, rank):
        # halo copies of diagonal / basic posts: one SM kernel storing every
        # box of the post over NVLink (default, "batch"; r04 A/B on 2 GPUs:
        # elastic diagonal 572 vs 517 GB/s, exposed 2.5% vs 2.9-4.4%), copy
        # engines ("ce", cudaMemcpy3DAsync on 4 streams) or one SM kernel per
        # box ("sm")
        eng = {"ce": 0, "sm": 1, "batch": 2}[os.environ.get("SDMP_COPY_ENGINE", "batch")]
        ints = [R.ACT["POST"], a.stream, a.phase, 0, (16 if a.pushed else 0) | eng]
        # z is never split: its halo (and padding) is exterior on every rank,
        # zero on sender and receiver alike, so each message ships whole
        # FULL-z rows -- an x-face becomes R contiguous (ny x full_z) blocks
        # and a y-face nx contiguous (R x full_z) blocks instead of R*ny or
        # nx*R separate nz-float rows (fewer, larger copy-engine bursts);
        # the receiver's z halo is rewritten with the zeros it holds
        whole_z = (decomp.ndims == 3 and decomp.topology.dims[2] == 1
                   and os.environ.get("SDMP_WHOLE_Z", "1") != "0")
        n = 0
        for m in a.messages:
            for f, t in a.spot.fields:
                if not a.spot.sends(f, t, m.direction):
                    continue  # f is not read across this face (HaloSpot.field_radius)
                fn = self.op.fields[f]
                slo = [l + h for l, h in zip(m.send[0], fn.halo3)] + [0] * (3 - len(m.send[0]))
                ext = [u - l for l, u in zip(*m.send)] + [1] * (3 - len(m.send[0]))
                dlo = [l + h for l, h in zip(m.recv[0], fn.halo3)] + [0] * (3 - len(m.recv[0]))
                if whole_z and ext[2] == fn.local3[2]:
                    slo[2], dlo[2], ext[2] = 0, 0, fn.full3[2]
                ints += [fid[f], t, pfid[(m.peer, f)]] + slo + dlo + ext
                n += 1
        ints[3] = n
        sigs = []
        for m in a.messages:
            sigs.append((pflag[m.peer], m.slot))
        ints += [len(sigs)]
        for fl, slot in sigs:
            ints += [fl, slot]
        return ints

    def _compute_ints(self, k, box, stream):
        ints = []
        fid = self.fid
        if isinstance(k, CP.StarKernel):
            fl, mid, variant = self.kparams[id(k)]
            lo, hi = self._full_box(k.u, box)
            u2 = fid[k.u] if k.B != 0 else -1
            r = list(k.radius) + [0] * (3 - len(k.radius))
            ints = [R.ACT["STAR"], stream, fid[k.u], 0, u2, -1, mid, fid[k.u], 1] + lo + hi + r + [variant]
            return ints, fl
        if isinstance(k, CP.VarStarKernel):
            fl, fa, fb, fs = self.kparams[id(k)]
            lo, hi = self._full_box(k.u, box)
            u2 = fid[k.u] if k.has_prev else -1
            r = list(k.radius) + [0] * (3 - len(k.radius))
            ints = [R.ACT["VSTAR"], stream, fid[k.u], 0, u2, -1, fa, fb, fs, fid[k.u], 1] + \
                lo + hi + r + [0]
            return ints, fl
        if isinstance(k, CP.RotatedKernel):
            fl, sid = self.kparams[id(k)]
            lo, hi = self._full_box(k.u, box)
            refs = [(k.u, 0), (k.u, -1), (k.m, 0), (k.a[0], 0), (k.a[1], 0), (k.a[2], 0),
                    (k.u, 1)]
            ints = [R.ACT["ROT"], stream]
            for f, t in refs:
                ints += [sid if f == k.m else fid[f], t]
            # radius | M_IS_SCALE: the m slot carries the bound dt^2/m
            return ints + lo + hi + [(k.so // 2) | R.VARIANT_M_IS_SCALE], fl
        if isinstance(k, CP.TTIKernel):
            fl, sid = self.kparams[id(k)]
            lo, hi = self._full_box(k.p, box)
            refs = [(k.p, 0), (k.p, -1), (k.r, 0), (k.r, -1), (k.m, 0), (k.epsp, 0),
                    (k.delp, 0), (k.a[0], 0), (k.a[1], 0), (k.a[2], 0), (k.p, 1), (k.r, 1)]
            ints = [R.ACT["TTI"], stream]
            for f, t in refs:
                ints += [sid if f == k.m else fid[f], t]
            return ints + lo + hi + [(k.so // 2) | R.VARIANT_M_IS_SCALE], fl
        if isinstance(k, CP.StaggeredPhase):
            (fl,) = self.kparams[id(k)]
            lo, hi = self._full_box(k.v[0], box)
            if k.kind == "v":
                refs = [(f, 0) for f in k.v] + [(f, 0) for f in k.tau] + [(k.params[0], 0)] + \
                       [(f, 1) for f in k.v]
                kind = R.ACT["EL_V"]
            elif k.kind == "t":
                refs = [(f, 1) for f in k.v] + [(f, 0) for f in k.tau] + \
                       [(k.params[0], 0), (k.params[1], 0)] + [(f, 1) for f in k.tau]
                kind = R.ACT["EL_T"]
            else:
                refs = [(f, 1) for f in k.v] + [(f, 0) for f in k.tau] + [(f, 0) for f in k.mem] + \
                       [(f, 0) for f in k.params] + [(f, 1) for f in k.tau] + [(f, 1) for f in k.mem]
                kind = R.ACT["VISCO_T"]
            ints = [kind, stream]
            for f, t in refs:
                ints += [fid[f], t]
            # radius | collocated << 8
            return ints + lo + hi + [k.so // 2 | (256 if k.collocated else 0)], fl
        raise CP.CompilerError(f"no native encoding for {type(k).__name__}")

    def _encode_static(self, ep, decomp, rank):
        spot = ep.hoisted
        a = CP.Action("post", 2, phase=0, spot=spot, messages=ep.hoisted_messages)
        self.static.add_action(self._post_ints(a, self.static_fid, self.spfid, self.spflag,
                                               decomp, rank))
        slots = sorted({direction_slot(m.direction) for m in ep.hoisted_messages})
        if slots:
            self.static.add_action([R.ACT["WAIT"], 2, 0, len(slots)] + slots)

    def _add_sparse(self, t, decomp, rank):
        torch = __import__("torch")
        fn = self.op.fields[t.field]
        grid = self.op.grid.spec
        dev = fn.storage.device
        sp = t.sparse
        if t.kind == "inject":
            node, ptr, pid, w = SP.injection_table(sp.coordinates, grid, decomp, rank,
                                                   fn.halo3, fn.full3)
            c, p, q, mspec = t.scale
            if p > 0 and self.dt is None:
                raise ValueError("injection expression needs dt")
            C = _f32(float(c) * (float(self.dt) ** p if p else 1.0))
            if q not in (0, -1):
                raise CP.CompilerError("injection scale m^q supports q in {0, -1}")
            mid = self.fid[mspec] if q == -1 else -1
            tens = [torch.from_numpy(a).to(dev) for a in (node, ptr, pid, w)]
            amps = torch.zeros((sp.nt, sp.npoint), dtype=torch.float32, device=dev)
            self.keep += tens + [amps]
            sid = self.plan.add_sparse(0, sp.npoint, len(node), 0,
                                       *[int(x.data_ptr()) for x in tens], int(amps.data_ptr()),
                                       sp.npoint, 0)
            self.sparse_sets[id(t)] = (sid, mid, C, amps, sp)
        else:
            pids, idx, w = SP.interpolation_table(sp.coordinates, grid, decomp, rank,
                                                  fn.halo3, fn.full3)
            nc = 1 << grid.ndims
            dti = torch.from_numpy(idx).to(dev)
            dtw = torch.from_numpy(w).to(dev)
            traces = torch.zeros((sp.nt, max(len(pids), 1)), dtype=torch.float32, device=dev)
            self.keep += [dti, dtw, traces]
            sid = self.plan.add_sparse(1, len(pids), 0, nc, int(dti.data_ptr()), 0, 0,
                                       int(dtw.data_ptr()), int(traces.data_ptr()),
                                       max(len(pids), 1), 0)
            self.sparse_sets[id(t)] = (sid, pids, traces, sp)

    # ------------------------------------------------------------------
    def run(self, time_m: int, time_M: int):
        torch = __import__("torch")
        for t in self.op.sparse_terms:
            if time_M >= t.sparse.nt or time_m < 0:
                raise ValueError(f"time range {time_m}..{time_M} outside sparse data nt={t.sparse.nt}")
            entry = self.sparse_sets[id(t)]
            if t.kind == "inject":
                entry[3].copy_(torch.from_numpy(np.ascontiguousarray(t.sparse.data, np.float32)))
            else:
                entry[2].zero_()
        # bound dt^2/m buffers and the hoisted exchange of static fields are
        # redone only when a static field changed (Data writes bump _version)
        for sbuf, mfn, C in self.scale_bufs:
            if self._seen.get(id(sbuf)) != mfn._version:
                R.bind_scale(sbuf, mfn.storage[0], C)
                self._seen[id(sbuf)] = mfn._version
        for k, ufn, bufs in self.var_bufs:
            ver = tuple(self.op.fields[f]._version for f in k.statics)
            if self._seen.get(id(k)) != ver:
                self._bind_var(k, ufn, bufs)
                self._seen[id(k)] = ver
        if self.static is not None:
            ver = tuple(self.op.fields[f]._version for f, _t in self.eplan.hoisted.fields)
            if self._seen.get("static") != ver:
                self.static.run(0, 0)
                self.static.sync()
                self._seen["static"] = ver
        self.plan.run(time_m, time_M)
        self.plan.sync()

    def check_cfl(self):
        """Collective (every rank calls it from Operator.apply): re-check the
        acoustic CFL guard whenever m changed."""
        for k, mfn in self.cfl:
            if self._seen.get(("cfl", id(k))) != mfn._version:
                self._check_cfl(k, mfn)
                self._seen[("cfl", id(k))] = mfn._version

    def _check_cfl(self, k, mfn):
        """Acoustic CFL guard: refuse a dt above the
        leapfrog stability limit of this stencil, dt_max = 2 / (v_max
        sqrt(lambda_max)) with lambda_max = sum_a |w_0 + 2 sum_k (-1)^k w_k| /
        h_a^2 (the stencil's symbol at the Nyquist wavenumber) and
        v_max = 1 / sqrt(min m) over the global domain."""
        c = float(k.c)
        if self.dt is None or c <= 0:
            return
        m_min = float(mfn._domain_view(0).min())
        m_min = -self.ctx.allreduce_max(-m_min)
        if m_min <= 0:
            raise ValueError("acoustic model has m <= 0 (m = 1/vp^2 must be positive)")
        lam = 0.0
        for w, h in zip(k.weights, self.op.grid.spacing):
            sym = float(w[0]) + 2.0 * sum(float(w[j]) * (-1) ** j for j in range(1, len(w)))
            lam += abs(sym) / (h * h)
        dt_max = 2.0 / (math.sqrt(c * lam / m_min))
        if float(self.dt) > dt_max * (1.0 + 1e-6):
            raise ValueError(
                f"dt = {float(self.dt):.6g} exceeds the CFL stability limit {dt_max:.6g} of "
                f"this SO-{k.u.space_order} acoustic stencil (v_max = {1 / math.sqrt(m_min):.4g}); "
                "reduce dt (kernels.critical_dt gives a conservative choice)")

    def _bind_var(self, k, ufn, bufs, max_points: int = 1 << 26):
        """A, B, S of a variable-coefficient star from its static fields:
        evaluated in fp64 on the device (x-slabs), stored as fp32."""
        torch = __import__("torch")
        dom = tuple(slice(h, h + n) for h, n in zip(ufn.halo3, ufn.local3))
        views = {f: self.op.fields[f]._domain_view(0) for f in k.statics}
        outs = {n: b[dom] for n, b in bufs.items()}
        nx = ufn.local3[0]
        plane = max(1, math.prod(ufn.local3[1:]))
        step = max(1, max_points // plane)
        for x0 in range(0, nx, step):
            x1 = min(nx, x0 + step)
            vals = {f: v[x0:x1].double() for f, v in views.items()}
            A, B, Sv = k.coefficients(vals, self.dt, self.op.grid.spacing)
            for n, val in (("A", A), ("B", B), ("S", Sv)):
                if n in outs:
                    o = outs[n][x0:x1]
                    if torch.is_tensor(val):
                        o.copy_(val.to(o.dtype))
                    else:
                        o.fill_(float(val))
        torch.cuda.synchronize()

    def collect_sparse(self, time_m, time_M):
        """Assemble receiver traces into ``rec.data`` on every rank."""
        for t in self.op.sparse_terms:
            if t.kind != "interp":
                continue
            sid, pids, traces, sp = self.sparse_sets[id(t)]
            local = traces[time_m:time_M + 1, :len(pids)].cpu().numpy()
            parts = self.ctx.allgather((pids, local))
            for pp, vals in parts:
                if len(pp):
                    sp.data[time_m:time_M + 1, pp] = vals

    def trace(self):
        return self.plan.trace()
