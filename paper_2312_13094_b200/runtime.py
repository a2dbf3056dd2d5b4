"""ctypes binding of libsdmp.so (include/sdmp.h) + thin typed wrappers.

This module is the only place the product touches the native library.  There
is no CPU fallback: if libsdmp.so is missing or a CUDA device is absent, the
calls raise.  Device memory is owned by torch tensors; the library borrows
raw pointers (SURVEY.md §8b ownership rule).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDMP_LIB") or os.path.join(HERE, "libsdmp.so")  # SDMP_LIB: A/B builds

SDMP_MAX_RADIUS = 8
SDMP_NCOEF = SDMP_MAX_RADIUS + 1

ACT = dict(STAR=1, VSTAR=8, ROT=9, TTI=2, EL_V=3, EL_T=4, VISCO_T=5, INJECT=6, INTERP=7, POST=10, WAIT=11,
           RECORD=12, STREAMWAIT=13)

_lib = None
_lock = threading.Lock()

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class NativeError(RuntimeError):
    """A libsdmp call failed; the message carries sdmp_last_error()."""


def _declare(lib):
    sig = {
        "sdmp_last_error": (C.c_char_p, []),
        "sdmp_version": (C.c_int, []),
        "sdmp_device_count": (C.c_int, [i32p]),
        "sdmp_device_info": (C.c_int, [C.c_int, i32p, i64p, i32p, i32p]),
        "sdmp_star_update": (C.c_int, [vp, vp, vp, vp, vp, i64p, i64p, i64p, i32p, f32p,
                                       C.c_float, C.c_float, C.c_float, C.c_int32]),
        "sdmp_var_star_update": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64p, i64p, i64p, i32p,
                                           f32p, C.c_int32]),
        "sdmp_rot_update": (C.c_int, [vp, C.POINTER(vp), vp, i64p, i64p, i64p, C.c_int32, f32p,
                                      C.c_float]),
        "sdmp_tti_update": (C.c_int, [vp, C.POINTER(vp), vp, vp, i64p, i64p, i64p, C.c_int32,
                                      f32p, f32p, C.c_float, C.c_int32]),
        "sdmp_elastic_velocity": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), vp, C.POINTER(vp),
                                            i64p, i64p, i64p, C.c_int32, f32p, C.c_float]),
        "sdmp_elastic_stress": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), vp, vp,
                                          C.POINTER(vp), i64p, i64p, i64p, C.c_int32, f32p,
                                          C.c_float]),
        "sdmp_elastic_colloc_velocity": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), vp,
                                                   C.POINTER(vp), i64p, i64p, i64p, C.c_int32,
                                                   f32p, C.c_float]),
        "sdmp_elastic_colloc_stress": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), vp, vp,
                                                 C.POINTER(vp), i64p, i64p, i64p, C.c_int32,
                                                 f32p, C.c_float]),
        "sdmp_visco_stress": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                        C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), i64p, i64p,
                                        i64p, C.c_int32, f32p, C.c_float]),
        "sdmp_bind_scale": (C.c_int, [vp, vp, vp, C.c_int64, C.c_float]),
        "sdmp_inject": (C.c_int, [vp, vp, vp, vp, C.c_int32, vp, vp, vp, C.c_float, vp]),
        "sdmp_interpolate": (C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp]),
        "sdmp_pack": (C.c_int, [vp, vp, i64p, i64p, i64p, vp]),
        "sdmp_unpack": (C.c_int, [vp, vp, i64p, i64p, i64p, vp]),
        "sdmp_copy_box": (C.c_int, [vp, vp, i64p, i64p, vp, i64p, i64p, i64p, C.c_int32]),
        "sdmp_ipc_export": (C.c_int, [vp, C.POINTER(C.c_ubyte), C.POINTER(C.c_uint64)]),
        "sdmp_ipc_import": (C.c_int, [C.POINTER(C.c_ubyte), C.c_uint64, C.POINTER(vp)]),
        "sdmp_flags_alloc": (C.c_int, [C.c_int32, C.POINTER(vp)]),
        "sdmp_flags_free": (C.c_int, [vp]),
        "sdmp_enable_peer": (C.c_int, [C.c_int]),
        "sdmp_plan_create": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(vp)]),
        "sdmp_plan_destroy": (C.c_int, [vp]),
        "sdmp_plan_add_field": (C.c_int, [vp, C.c_int32, u64p, i64p, i32p]),
        "sdmp_plan_add_flags": (C.c_int, [vp, vp, i32p]),
        "sdmp_plan_set_local_flags": (C.c_int, [vp, vp]),
        "sdmp_plan_add_sparse": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp,
                                           vp, vp, vp, vp, C.c_int64, C.c_int64, i32p]),
        "sdmp_plan_add_action": (C.c_int, [vp, i64p, C.c_int32, f32p, C.c_int32]),
        "sdmp_plan_run": (C.c_int, [vp, C.c_int64, C.c_int64, vp]),
        "sdmp_plan_step": (C.c_int, [vp, C.c_int64, vp]),
        "sdmp_plan_sync": (C.c_int, [vp]),
        "sdmp_plan_set_tracing": (C.c_int, [vp, C.c_int32]),
        "sdmp_plan_trace": (C.c_int, [vp, C.POINTER(C.c_double), C.c_int32, i32p]),
        "sdmp_plan_set_timeout": (C.c_int, [vp, C.c_int64]),
        "sdmp_plan_set_graph": (C.c_int, [vp, C.c_int32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return sig


EXPORTED = None


def lib():
    """Load libsdmp.so once (raises if it was not built)."""
    global _lib, EXPORTED
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"{LIB_PATH} not found: build it with "
                    "`python -m paper_2312_13094_b200.build` (no CPU fallback exists)")
            handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
            EXPORTED = sorted(_declare(handle))
            _lib = handle
    return _lib


def check(rc: int, what: str = "", rank: Optional[int] = None):
    if rc != 0:
        msg = lib().sdmp_last_error().decode(errors="replace")
        where = f" [rank {rank}]" if rank is not None else ""
        raise NativeError(f"{what}{where} failed ({rc}): {msg}")


# ---------------------------------------------------------------------------
# small marshalling helpers


def arr_i64(vals) -> C.Array:
    vals = [int(v) for v in vals]
    return (C.c_int64 * len(vals))(*vals)


def arr_i32(vals) -> C.Array:
    vals = [int(v) for v in vals]
    return (C.c_int32 * len(vals))(*vals)


def arr_f32(vals) -> C.Array:
    vals = np.asarray(vals, dtype=np.float32).ravel()
    return (C.c_float * len(vals)).from_buffer_copy(vals.tobytes())


def arr_ptr(ptrs) -> C.Array:
    return (vp * len(ptrs))(*[C.c_void_p(int(p)) if p else None for p in ptrs])


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (0 for None)."""
    if t is None:
        return 0
    return int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def coeff_table(per_axis: Sequence[Sequence[float]], width: int) -> np.ndarray:
    """Pack per-axis coefficient lists into the 3 x width fp32 table."""
    t = np.zeros((3, width), dtype=np.float32)
    for a, c in enumerate(per_axis):
        c = np.asarray(c, dtype=np.float32)
        t[a, :len(c)] = c
    return t


# ---------------------------------------------------------------------------
# typed kernel entry points (stream-ordered, asynchronous)


def star_update(u0, u2, m, u1, full, lo, hi, radius, coeffs, A, B, Cc, variant=0, stream=None):
    tab = coeff_table(coeffs, SDMP_NCOEF)
    check(lib().sdmp_star_update(stream_handle(stream), ptr(u0), ptr(u2), ptr(m), ptr(u1),
                                 arr_i64(full), arr_i64(lo), arr_i64(hi), arr_i32(radius),
                                 arr_f32(tab), float(A), float(B), float(Cc), int(variant)),
          "sdmp_star_update")


VARIANT_M_IS_SCALE = 0x100


def bind_scale(out, inp, Cc, stream=None):
    """out = C / inp elementwise (0 where inp == 0), fp32, on the device."""
    check(lib().sdmp_bind_scale(stream_handle(stream), ptr(out), ptr(inp), int(inp.numel()),
                                float(Cc)), "sdmp_bind_scale")


def pack(field, full, lo, hi, buf, stream=None):
    check(lib().sdmp_pack(stream_handle(stream), ptr(field), arr_i64(full), arr_i64(lo),
                          arr_i64(hi), ptr(buf)), "sdmp_pack")


def unpack(field, full, lo, hi, buf, stream=None):
    check(lib().sdmp_unpack(stream_handle(stream), ptr(field), arr_i64(full), arr_i64(lo),
                            arr_i64(hi), ptr(buf)), "sdmp_unpack")


def copy_box(src, src_full, src_lo, dst, dst_full, dst_lo, extent, engine=0, stream=None):
    check(lib().sdmp_copy_box(stream_handle(stream), ptr(src) if not isinstance(src, int) else src,
                              arr_i64(src_full), arr_i64(src_lo),
                              ptr(dst) if not isinstance(dst, int) else dst, arr_i64(dst_full),
                              arr_i64(dst_lo), arr_i64(extent), int(engine)), "sdmp_copy_box")


def ipc_export(dev_ptr: int):
    h = (C.c_ubyte * 64)()
    off = C.c_uint64(0)
    check(lib().sdmp_ipc_export(C.c_void_p(dev_ptr), h, C.byref(off)), "sdmp_ipc_export")
    return bytes(h), int(off.value)


def ipc_import(handle: bytes, offset: int) -> int:
    h = (C.c_ubyte * 64).from_buffer_copy(handle)
    out = C.c_void_p(0)
    check(lib().sdmp_ipc_import(h, C.c_uint64(offset), C.byref(out)), "sdmp_ipc_import")
    return int(out.value)


def flags_alloc(n: int) -> int:
    out = C.c_void_p(0)
    check(lib().sdmp_flags_alloc(int(n), C.byref(out)), "sdmp_flags_alloc")
    return int(out.value)


class NativePlan:
    """Owner of one sdmp_plan (per rank / device)."""

    def __init__(self, device: int, phases: int, rank: Optional[int] = None):
        self.rank = rank
        h = C.c_void_p(0)
        check(lib().sdmp_plan_create(int(device), int(phases), C.byref(h)),
              "sdmp_plan_create", rank)
        self.h = h
        self._keep = []  # keep device arrays referenced for the plan lifetime
        self.nact = 0
        ms = os.environ.get("SDMP_TIMEOUT_MS")
        if ms:
            self.set_timeout(int(ms))

    def add_field(self, ptrs: Sequence[int], full: Sequence[int]) -> int:
        fid = C.c_int32(0)
        arr = (C.c_uint64 * len(ptrs))(*[int(p) for p in ptrs])
        check(lib().sdmp_plan_add_field(self.h, len(ptrs), arr, arr_i64(full), C.byref(fid)),
              "sdmp_plan_add_field", self.rank)
        return fid.value

    def add_flags(self, dev_ptr: int) -> int:
        fid = C.c_int32(0)
        check(lib().sdmp_plan_add_flags(self.h, C.c_void_p(dev_ptr), C.byref(fid)),
              "sdmp_plan_add_flags", self.rank)
        return fid.value

    def set_local_flags(self, dev_ptr: int):
        check(lib().sdmp_plan_set_local_flags(self.h, C.c_void_p(dev_ptr)),
              "sdmp_plan_set_local_flags", self.rank)

    def add_sparse(self, kind, npts, nnodes, ncorner, node, ptr_, pid, w, series, stride, t0,
                   keep=()) -> int:
        sid = C.c_int32(0)
        self._keep.extend(keep)
        check(lib().sdmp_plan_add_sparse(self.h, int(kind), int(npts), int(nnodes), int(ncorner),
                                         C.c_void_p(node), C.c_void_p(ptr_), C.c_void_p(pid),
                                         C.c_void_p(w), C.c_void_p(series), int(stride), int(t0),
                                         C.byref(sid)), "sdmp_plan_add_sparse", self.rank)
        return sid.value

    def add_action(self, ints: Sequence[int], floats: Sequence[float] = ()):
        fl = arr_f32(floats) if len(floats) else None
        check(lib().sdmp_plan_add_action(self.h, arr_i64(ints), len(ints), fl, len(floats)),
              "sdmp_plan_add_action", self.rank)
        self.nact += 1

    def run(self, time_m: int, time_M: int, stream=None):
        check(lib().sdmp_plan_run(self.h, int(time_m), int(time_M), C.c_void_p(stream_handle(stream))),
              "sdmp_plan_run", self.rank)

    def sync(self):
        check(lib().sdmp_plan_sync(self.h), "sdmp_plan_sync", self.rank)

    def set_tracing(self, on: bool):
        check(lib().sdmp_plan_set_tracing(self.h, int(on)), "sdmp_plan_set_tracing", self.rank)

    def set_graph(self, on: bool):
        """Replay buffer-rotation periods as captured CUDA graphs (after the
        first run of the plan)."""
        check(lib().sdmp_plan_set_graph(self.h, int(on)), "sdmp_plan_set_graph", self.rank)

    def set_timeout(self, ms: int):
        check(lib().sdmp_plan_set_timeout(self.h, int(ms)), "sdmp_plan_set_timeout", self.rank)

    def trace(self, max_rows: int = 512):
        """Per-action rows (index, stream, kind, mean start ms, mean duration
        ms, kernel launches per step) averaged over the last traced run."""
        rows = (C.c_double * (6 * max_rows))()
        n = C.c_int32(0)
        check(lib().sdmp_plan_trace(self.h, rows, max_rows, C.byref(n)), "sdmp_plan_trace",
              self.rank)
        return [tuple(rows[6 * i: 6 * i + 6]) for i in range(n.value)]

    def close(self):
        if self.h:
            lib().sdmp_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
