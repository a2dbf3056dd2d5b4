"""User-facing API: Grid, Function, TimeFunction, SparseTimeFunction, Eq,
solve, Operator — the drop-in surface of the paper's Listing 1
 over the reference's symbolic types
(symbolics.py:39-149) and the SPEC's distributed data model
(SPEC.md:202-284, 485-558).

* ``Grid(shape, extent, topology=None)`` decomposes over the torchrun world
  (one process per GPU; PAPER.md:222-249 topology override).
* ``Function`` / ``TimeFunction`` own a device tensor
  ``(time_buffers, *FULL)`` per rank (FULL = owned + 2*halo, exterior halo
  permanently zero); 2D grids are stored as 3D with a
  unit z axis.
* ``.data`` is logically global (``global_to_local`` writes and reads,
  SPEC.md:158-166, 232-250; Listing 3).
* ``Operator(eqs).apply(time_m=0, time_M=..., dt=..., mpi="basic|diagonal|
  full")`` runs time_m..time_M inclusive (Listing 4) on the GPU
  through libsdmp.  Unsupported equations raise; there is no CPU path.
"""
from __future__ import annotations

import math
import os
import time as _time
import weakref
from fractions import Fraction
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import compiler as CP
from . import decomposition as DC
from . import dist
from . import symbolics as S
from .symbolics import Eq, StencilEquation, solve_forward  # re-exported

_FUNCS: "weakref.WeakValueDictionary" = weakref.WeakValueDictionary()
GUARD_WORD = 0x7FC0DEAD  # NaN canary of SDMP_GUARD allocations


def torch_module():
    import torch
    return torch


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2312_13094_b200 needs a CUDA device (B200); "
                           "there is no CPU execution path")
    return torch


# ---------------------------------------------------------------------------
# Grid


class Grid:
    """Structured grid + domain decomposition."""

    def __init__(self, shape, extent=None, topology=None, origin=None, comm=None):
        shape = tuple(int(n) for n in shape)
        if extent is None:
            extent = tuple(float(n - 1) for n in shape)
        self.spec = S.GridSpec(shape, tuple(float(e) for e in extent))
        self.origin = tuple(origin) if origin is not None else (0.0,) * len(shape)
        ctx = dist.SelfContext(dist.context().device) if comm == "self" else dist.context()
        self.ctx = ctx
        self.decomposition = DC.Decomposition.create(shape, ctx.size, topology)
        self.rank = ctx.rank

    shape = property(lambda self: self.spec.shape)
    extent = property(lambda self: self.spec.extent)
    spacing = property(lambda self: self.spec.spacing)
    ndims = property(lambda self: self.spec.ndims)
    topology = property(lambda self: self.decomposition.topology.dims)

    @property
    def spacing_map(self) -> Dict[S.Symbol, float]:
        return {S.Symbol("h_" + S.AXIS_NAMES[a]): h for a, h in enumerate(self.spacing)}

    @property
    def local_extent(self):
        return self.decomposition.extent(self.rank)

    @property
    def local_shape(self):
        return self.decomposition.local_shape(self.rank)


# ---------------------------------------------------------------------------
# Distributed data


class Data:
    """Logically global view of a field's DOMAIN (Listing 3).

    ``data[key] = value`` writes the local intersection of the global region
    on every rank (collective in the SPEC sense: all ranks call it with the
    same arguments).  ``data[key]`` returns this rank's part of the global
    region as a numpy array (the per-rank view Listings 3/4 print).
    ``gather()`` assembles the global array (row-major) on every rank.
    For a TimeFunction, a key with one entry per spatial axis addresses all
    time buffers on write and the most recent buffer on read; an extra
    leading entry selects time buffers explicitly.
    """

    def __init__(self, fn: "Function"):
        self.fn = fn

    @property
    def shape(self):
        return self.fn.grid.shape

    def _split(self, key):
        fn = self.fn
        nd = fn.grid.ndims
        if not isinstance(key, tuple):
            key = (key,)
        if key == (Ellipsis,):
            key = ()
        tsel = None
        if fn.is_time and len(key) == nd + 1:
            tsel, key = key[0], key[1:]
        if len(key) > nd:
            raise IndexError(f"too many indices for a {nd}D field")
        key = key + (slice(None),) * (nd - len(key))
        region = tuple(DC.normalise_slice(k, n) for k, n in zip(key, fn.grid.shape))
        squeeze = tuple(a for a, k in enumerate(key) if not isinstance(k, slice))
        return tsel, region, squeeze

    def _buffers(self, tsel, write):
        fn = self.fn
        nb = fn.time_buffers
        if tsel is None:
            return list(range(nb)) if write else [fn._latest]
        if isinstance(tsel, slice):
            return list(range(nb))[tsel]
        return [int(tsel) % nb]

    def __setitem__(self, key, value):
        import torch
        fn = self.fn
        tsel, region, _sq = self._split(key)
        ext = fn.grid.local_extent
        loc = DC.global_to_local(ext, region)
        # the write is collective: every rank bumps the
        # version, including ranks the region misses, so the plans' "static
        # field changed" decisions (collective CFL check, static halo
        # re-exchange) agree across ranks
        fn._version += 1
        if loc is None:
            return
        val = value
        if not np.isscalar(value):
            rshape = tuple(b - a for a, b in region)
            try:
                val = np.broadcast_to(np.asarray(value, dtype=np.float32), rshape)
            except ValueError:
                raise ValueError(f"value of shape {np.shape(value)} does not match "
                                 f"region {rshape}") from None
            # the part of the value that lands on this rank
            sub = tuple(slice(l + e0 - r0, h + e0 - r0) for (l, h), (e0, _e1), (r0, _r1)
                        in zip(loc, ext, region))
            val = torch.from_numpy(np.array(val[sub], dtype=np.float32, order="C")).to(
                fn.storage.device)
            if fn.grid.ndims == 2:
                val = val.unsqueeze(-1)
        for b in self._buffers(tsel, True):
            view = fn._domain_view(b)
            sl = tuple(slice(l, h) for l, h in loc)
            if isinstance(val, (int, float, np.floating, np.integer)):
                view[sl] = float(val)
            else:
                view[sl] = val
        if fn.storage.is_cuda:
            torch.cuda.synchronize()

    def __getitem__(self, key):
        fn = self.fn
        tsel, region, squeeze = self._split(key)
        loc = DC.global_to_local(fn.grid.local_extent, region)
        bufs = self._buffers(tsel, False)
        outs = []
        for b in bufs:
            if loc is None:
                outs.append(np.zeros((0,) * fn.grid.ndims, dtype=np.float32))
                continue
            view = fn._domain_view(b)
            arr = view[tuple(slice(l, h) for l, h in loc)].cpu().numpy()
            if fn.grid.ndims == 2:
                arr = arr[..., 0]
            outs.append(arr)
        if tsel is None or not isinstance(tsel, slice):
            out = outs[0]
            if loc is not None and squeeze:
                out = out.reshape([s for a, s in enumerate(out.shape) if a not in squeeze])
            return out
        return np.stack(outs)

    @property
    def local(self) -> np.ndarray:
        """This rank's full DOMAIN block (latest buffer)."""
        return self[...]

    def gather(self, buffer: Optional[int] = None) -> np.ndarray:
        """Global row-major array assembled from every rank (all ranks
        receive it; SPEC.md:242-250 gathers to root)."""
        fn = self.fn
        b = fn._latest if buffer is None else buffer % fn.time_buffers
        arr = fn._domain_view(b).cpu().numpy()
        if fn.grid.ndims == 2:
            arr = arr[..., 0]
        parts = fn.grid.ctx.allgather((fn.grid.local_extent, arr))
        out = np.zeros(fn.grid.shape, dtype=np.float32)
        for ext, a in parts:
            out[tuple(slice(x, y) for x, y in ext)] = a
        return out

    def dump(self, path: str, buffer: Optional[int] = None) -> None:
        """Gather and write the global field: one text header
        line ``field=<name> shape=<n0>,<n1>[,<n2>] dtype=float64 order=C``,
        then the values as row-major 64-bit floats.  Collective; rank 0
        writes."""
        out = self.gather(buffer)
        if self.fn.grid.ctx.rank == 0:
            with open(path, "wb") as f:
                shape = ",".join(str(n) for n in out.shape)
                f.write(f"field={self.fn.name} shape={shape} dtype=float64 order=C\n".encode())
                f.write(np.ascontiguousarray(out, dtype="<f8").tobytes())

    def __array__(self, dtype=None):
        a = self[...]
        return a.astype(dtype) if dtype is not None else a

    def __repr__(self):
        return repr(self[...])


# ---------------------------------------------------------------------------
# Functions


class Function:
    """Static (coefficient) field: one buffer (time_order 0)."""

    is_time = False

    def __init__(self, name, grid: Grid, space_order=2, halo=None, time_order=0):
        import torch
        self.name = name
        self.grid = grid
        self.spec = S.FieldSpec(name=name, grid=grid.spec, space_order=space_order,
                                time_order=time_order, halo=halo)
        # Devito-style re-definition: a new field with the same name and spec
        # (e.g. a script that rebuilds its Grid / TimeFunction) replaces the
        # registry entry; Operators built earlier keep the Function objects
        # they resolved, equations built afterwards bind to the newest one.
        _FUNCS[self.spec] = self
        nd = grid.ndims
        # device layout: halo per side = FieldSpec.halo, except that the z
        # halo of 3D fields is padded up to a multiple of 8 (the paper's
        # "padding" region): keeps rows 32 B-aligned for TMA and
        # every TMA box start non-negative.  Padding is zero like the exterior
        # halo; exchange radii and all DOMAIN-relative boxes are unchanged.
        h = tuple(self.spec.halo)
        if nd == 3:
            h = h[:2] + ((h[2] + 7) // 8 * 8,)
        self.halo3 = h + (0,) * (3 - nd)
        loc = tuple(grid.local_shape) + (1,) * (3 - nd)
        self.local3 = loc
        self.full3 = tuple(n + 2 * h for n, h in zip(loc, self.halo3))
        # Storage lives on this rank's GPU.  Without a GPU (host-logic tests)
        # the arrays are allocated on the CPU, but apply() refuses to run.
        dev = (torch.device("cuda", grid.ctx.device or 0) if torch.cuda.is_available()
               else torch.device("cpu"))
        shape = (self.time_buffers,) + self.full3
        self._guard = None
        if os.environ.get("SDMP_GUARD", "0") != "0":
            # debug: the buffers sit between two guard zones of at least one
            # x-plane filled with a NaN canary; check_guard() verifies no
            # kernel or copy wrote past either end of the allocation
            # (memory checking without compute-sanitizer)
            n = math.prod(shape)
            g = max(16384, self.full3[1] * self.full3[2])
            g = (g + 255) // 256 * 256
            flat = torch.full((g + n + g,), float("nan"), dtype=torch.float32, device=dev)
            flat.view(torch.int32).fill_(GUARD_WORD)
            self.storage = flat[g:g + n].view(shape)
            self.storage.zero_()
            self._guard = (flat, g, n)
        else:
            self.storage = torch.zeros(shape, dtype=torch.float32, device=dev)
        self._latest = 0
        # bumped by every Data write: plans re-bind derived buffers (dt^2/m)
        # and re-exchange static halos only when a static field changed
        self._version = 0

    # -- storage helpers ---------------------------------------------------
    def check_guard(self) -> bool:
        """SDMP_GUARD=1 allocations: both guard zones still hold the canary."""
        if self._guard is None:
            return True
        flat, g, n = self._guard
        w = flat.view(torch_module().int32)
        return bool((w[:g] == GUARD_WORD).all()) and bool((w[g + n:] == GUARD_WORD).all())

    @property
    def time_buffers(self) -> int:
        return self.spec.time_buffers

    @property
    def space_order(self):
        return self.spec.space_order

    def _domain_view(self, b: int):
        h = self.halo3
        return self.storage[b][tuple(slice(hh, hh + n) for hh, n in zip(h, self.local3))]

    def buffer_ptrs(self) -> List[int]:
        return [int(self.storage[b].data_ptr()) for b in range(self.time_buffers)]

    @property
    def data(self) -> Data:
        return Data(self)

    def data_gather(self, buffer=None) -> np.ndarray:
        return Data(self).gather(buffer)

    # -- symbolic sugar (delegates to the reference-compatible FieldSpec) --
    def at(self, tshift=0, offsets=None):
        return self.spec.at(tshift, offsets)

    def _e(self):
        return self.spec.at()

    def __add__(self, o): return self._e() + (o._e() if isinstance(o, Function) else o)
    def __radd__(self, o): return (o._e() if isinstance(o, Function) else o) + self._e()
    def __sub__(self, o): return self._e() - (o._e() if isinstance(o, Function) else o)
    def __rsub__(self, o): return (o._e() if isinstance(o, Function) else o) - self._e()
    def __mul__(self, o): return self._e() * (o._e() if isinstance(o, Function) else o)
    def __rmul__(self, o): return (o._e() if isinstance(o, Function) else o) * self._e()
    def __truediv__(self, o): return self._e() / (o._e() if isinstance(o, Function) else o)
    def __rtruediv__(self, o): return (o._e() if isinstance(o, Function) else o) / self._e()
    def __neg__(self): return -self._e()

    forward = property(lambda self: self.spec.forward)
    backward = property(lambda self: self.spec.backward)
    dt = property(lambda self: self.spec.dt)
    dt2 = property(lambda self: self.spec.dt2)
    dx = property(lambda self: self.spec.dx)
    dy = property(lambda self: self.spec.dy)
    dz = property(lambda self: self.spec.dz)
    laplace = property(lambda self: self.spec.laplace)

    def d(self, axis, order=1):
        return self.spec.d(axis, order)

    def __repr__(self):
        return f"{type(self).__name__}({self.name!r}, shape={self.grid.shape})"


class TimeFunction(Function):
    """Evolving field with time_order + 1 rotating buffers."""

    is_time = True

    def __init__(self, name, grid: Grid, space_order=2, time_order=1, halo=None):
        if time_order not in (1, 2):
            raise ValueError("TimeFunction time_order must be 1 or 2")
        super().__init__(name, grid, space_order=space_order, halo=halo,
                         time_order=time_order)


def load_dump(path: str):
    """Read a :meth:`Data.dump` file -> (field name, float64 array)."""
    with open(path, "rb") as f:
        header = f.readline().decode().split()
        meta = dict(kv.split("=", 1) for kv in header)
        shape = tuple(int(n) for n in meta["shape"].split(","))
        data = np.frombuffer(f.read(), dtype="<f8").reshape(shape)
    return meta["field"], data


def field_of(spec: S.FieldSpec) -> Function:
    fn = _FUNCS.get(spec)
    if fn is None:
        raise CP.CompilerError(f"no live Function/TimeFunction for field {spec.name!r}")
    return fn


# ---------------------------------------------------------------------------
# Sparse functions


def ricker(f0: float, t, t0: Optional[float] = None) -> np.ndarray:
    """Ricker wavelet; t0 defaults to 1/f0."""
    t0 = 1.0 / f0 if t0 is None else t0
    a = (math.pi * f0 * (np.asarray(t, dtype=np.float64) - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


class SparseTerm:
    def __init__(self, kind, sparse, field: S.FieldSpec, tshift: int, scale=None):
        self.kind = kind
        self.sparse = sparse
        self.field = field
        self.tshift = tshift
        self.scale = scale  # (c, p, q, m_spec) for inject


class SparseTimeFunction:
    """Off-grid points with a time series each (sources / receivers).

    ``coordinates``: (npoint, ndims) physical positions;
    ``data``: (nt, npoint) fp32 host array.  Used in expressions as the
    symbol ``<name>`` (e.g. ``src * dt**2 / m``)."""

    def __init__(self, name, grid: Grid, npoint: int, nt: int, coordinates=None):
        self.name = name
        self.grid = grid
        self.npoint = int(npoint)
        self.nt = int(nt)
        self.coordinates = (np.zeros((npoint, grid.ndims)) if coordinates is None
                            else np.asarray(coordinates, dtype=np.float64).reshape(npoint, grid.ndims))
        self.data = np.zeros((nt, npoint), dtype=np.float32)
        self.symbol = S.Symbol(name)

    def _e(self):
        return self.symbol

    def __mul__(self, o): return self.symbol * (o._e() if isinstance(o, Function) else o)
    def __rmul__(self, o): return (o._e() if isinstance(o, Function) else o) * self.symbol
    def __truediv__(self, o): return self.symbol / (o._e() if isinstance(o, Function) else o)

    def inject(self, field, expr=None) -> SparseTerm:
        """Add ``expr`` (linear in this function: ``src * c * dt^p * m^q``)
        into ``field`` (normally ``u.forward``) at the points."""
        if isinstance(field, Function):
            field = field.forward
        if not isinstance(field, S.FieldAccess) or field.tshift != 1:
            raise CP.CompilerError("inject target must be a forward access, e.g. u.forward")
        expr = self.symbol if expr is None else expr
        return SparseTerm("inject", self, field.spec, 1, _injection_scale(expr, self.symbol))

    def interpolate(self, expr) -> SparseTerm:
        """Sample ``expr`` (a field, read at the current time buffer) at the
        points into ``data[time]``."""
        if isinstance(expr, Function):
            expr = expr.spec.at()
        if not isinstance(expr, S.FieldAccess) or expr.tshift != 0 or any(expr.offsets):
            raise CP.CompilerError("interpolate supports a plain field (current time buffer)")
        return SparseTerm("interp", self, expr.spec, 0)


def _injection_scale(expr: S.Expr, sym: S.Symbol):
    """expr = sym * c * dt^p * m^q  ->  (c, p, q, m_spec) by exact probing."""
    leaves = {n for n in S.walk(expr) if isinstance(n, (S.Symbol, S.FieldAccess))}
    ms = {n.spec for n in leaves if isinstance(n, S.FieldAccess)}
    if any(isinstance(n, S.FieldAccess) and (not n.spec.is_static or any(n.offsets))
           for n in leaves) or len(ms) > 1:
        raise CP.CompilerError("injection expression may only scale by dt powers and one "
                               "static field")
    m = next(iter(ms)) if ms else None
    import random
    rng = random.Random(3)
    samples = []
    for _ in range(3):
        dt = Fraction(rng.randint(2, 40), rng.randint(2, 9))
        mv = Fraction(rng.randint(2, 40), rng.randint(2, 9))
        bind = {}
        for n in leaves:
            if n == sym:
                bind[n] = Fraction(1)
            elif isinstance(n, S.Symbol) and n.name == "dt":
                bind[n] = dt
            elif isinstance(n, S.FieldAccess):
                bind[n] = mv
            else:
                raise CP.CompilerError(f"unsupported symbol {n} in injection expression")
        val = S.eval_exact(expr, bind)
        b0 = dict(bind)
        b0[sym] = Fraction(0)
        if S.eval_exact(expr, b0) != 0:
            raise CP.CompilerError("injection expression must be linear in the source")
        samples.append((dt, mv, val))
    for p in (0, 1, 2):
        for q in ((0, -1, 1) if m is not None else (0,)):
            cs = {v / (d ** p * x ** q) for d, x, v in samples}
            if len(cs) == 1:
                return (cs.pop(), p, q, m)
    raise CP.CompilerError("injection scale is not of the form c * dt^p * m^q")


# ---------------------------------------------------------------------------
# Equations


def solve(eq, target) -> S.Expr:
    """Devito-style ``solve(eq, u.forward)`` -> rhs expression
    (reference solve_forward, symbolics.py:629-674)."""
    if isinstance(target, Function):
        target = target.forward
    if isinstance(eq, S.Expr):
        eq = S.Eq(eq)
    return S.solve_forward(eq, target).rhs


def _as_update(eq) -> S.StencilEquation:
    if isinstance(eq, S.StencilEquation):
        return eq
    if isinstance(eq, S.Eq):
        lhs = eq.lhs
        if isinstance(lhs, S.FieldAccess) and lhs.tshift == 1 and not any(lhs.offsets):
            rhs = S.discretize_expr(eq.rhs)
            if not any(n == lhs for n in S.walk(rhs)):
                return S.StencilEquation(lhs, rhs)
        # implicit form: solve for the forward access of the evolving field
        evolving = [a for a in S.accesses(S.discretize_expr(eq.lhs)) +
                    S.accesses(S.discretize_expr(eq.rhs)) if not a.spec.is_static]
        if not evolving:
            raise CP.CompilerError("equation has no evolving field")
        return S.solve_forward(eq, evolving[0].spec.forward)
    raise CP.CompilerError(f"unsupported equation type {type(eq).__name__}")


# ---------------------------------------------------------------------------
# Operator


def _env_mode():
    for var in ("STENCIL_DMP_MODE", "DEVITO_MPI"):
        v = os.environ.get(var)
        if v:
            return v
    return "diagonal"


class Operator:
    """Compile equations + sparse terms once; ``apply`` runs them on the GPU
    (SPEC.md:643-651)."""

    def __init__(self, expressions, name="Kernel"):
        if not isinstance(expressions, (list, tuple)):
            expressions = [expressions]
        flat = []
        for e in expressions:
            if isinstance(e, (list, tuple)):
                flat.extend(e)
            else:
                flat.append(e)
        self.name = name
        self.sparse_terms = [e for e in flat if isinstance(e, SparseTerm)]
        kernel_like = []
        for e in flat:
            if isinstance(e, SparseTerm):
                continue
            if hasattr(e, "kernels"):  # KernelDef from paper_2312_13094_b200.kernels
                kernel_like.extend(e.kernels)
                kernel_like.extend(_as_update(q) for q in getattr(e, "equations", []))
            elif isinstance(e, (CP.StarKernel, CP.VarStarKernel, CP.RotatedKernel, CP.TTIKernel,
                                CP.StaggeredPhase)):
                kernel_like.append(e)
            else:
                kernel_like.append(_as_update(e))
        self.updates = [e for e in kernel_like if isinstance(e, S.StencilEquation)]
        self.kernels = CP.recognise(kernel_like)
        self.fields: Dict[S.FieldSpec, Function] = {}
        for k in self.kernels:
            for f, _t, _r in k.reads():
                self.fields[f] = field_of(f)
            for f, _t in k.writes():
                self.fields[f] = field_of(f)
        for t in self.sparse_terms:
            self.fields[t.field] = field_of(t.field)
            if t.scale is not None and t.scale[3] is not None:
                self.fields[t.scale[3]] = field_of(t.scale[3])
        grids = {id(f.grid) for f in self.fields.values()}
        if len(grids) != 1:
            raise CP.CompilerError("all fields of an Operator must live on one Grid")
        self.grid = next(iter(self.fields.values())).grid
        self._plans = {}
        self.last_summary = None

    # ------------------------------------------------------------------
    def plan(self, mode=None, dt=None, exchange=True):
        """The per-rank ExecPlan (host description; used by tests)."""
        mode = CP.normalise_mode(mode or _env_mode())
        an = CP.halo_phases(self.kernels, self.grid.decomposition.nranks)
        fused = os.environ.get("SDMP_FUSED", "1") != "0"
        return CP.lower_mode(an, self.grid.decomposition, self.grid.rank, mode,
                             self.sparse_terms, exchange=exchange, fused=fused)

    def dump(self, mode=None) -> str:
        """Listing 6/7-style plan text (HaloSpots, or the mode's update /
        wait calls around the CORE / REMAINDER loop nests)."""
        return CP.dump_plan(self.kernels, self.grid.decomposition.nranks, mode, self.updates)

    def _native(self, mode, dt, exchange=True):
        key = (mode, None if dt is None else float(np.float32(dt)), exchange)
        if key not in self._plans:
            from .runtime_plan import NativeOperatorPlan
            self._plans[key] = NativeOperatorPlan(self, mode, dt, exchange=exchange)
        return self._plans[key]

    def apply(self, time_m: int = 0, time_M: Optional[int] = None, dt=None, mpi=None,
              time=None, **kwargs):
        """Run timesteps time_m..time_M inclusive."""
        torch = _torch()
        if time_M is None:
            time_M = time
        if time_M is None:
            nts = [t.sparse.nt for t in self.sparse_terms]
            if not nts:
                raise ValueError("apply() needs time_M (or sparse functions to infer it)")
            time_M = min(nts) - 1
        mode = CP.normalise_mode(mpi or kwargs.get("mode") or _env_mode())
        plan = self._native(mode, dt)
        plan.check_cfl()  # collective: apply is called by every rank
        t0 = _time.perf_counter()
        plan.run(int(time_m), int(time_M))
        torch.cuda.synchronize()
        wall = _time.perf_counter() - t0
        for f in self.fields.values():
            if f.is_time:
                f._latest = (int(time_M) + 1) % f.time_buffers
        plan.collect_sparse(int(time_m), int(time_M))
        npts = math.prod(self.grid.shape)
        steps = int(time_M) - int(time_m) + 1
        self.last_summary = {"mode": mode, "steps": steps, "wall_s": wall,
                             "gpts_s": npts * steps / wall / 1e9 if wall > 0 else float("nan")}
        return self.last_summary


__all__ = ["Grid", "Function", "TimeFunction", "SparseTimeFunction", "Operator", "Eq",
           "solve", "ricker", "Data", "StencilEquation", "solve_forward", "load_dump"]
