"""Every exported compute entry point of include/sdmp.h called directly
through ctypes (plain device pointers and int64/float arrays, as a reference
maintainer would bind them) and checked against the CPU
oracle on the same fp32 inputs: var-star, TTI, elastic velocity / stress,
viscoelastic stress, inject, interpolate.  Tolerance: rel-L2 <= 1e-5."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import stencils as K  # noqa: E402
from paper_2312_13094_b200 import runtime as R  # noqa: E402
from paper_2312_13094_b200 import symbolics as S  # noqa: E402

REL = 1e-5
NC = R.SDMP_NCOEF
MR = R.SDMP_MAX_RADIUS


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def arr(ctype, vals):
    return (ctype * len(vals))(*vals)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()


def ptrs(ts):
    return arr(C.c_void_p, [t.data_ptr() for t in ts])


def call(name, *args):
    fn = getattr(R.lib(), name)
    rc = fn(*args)
    torch.cuda.synchronize()
    assert rc == 0, R.lib().sdmp_last_error().decode()


def setup(full, h):
    rng = np.random.default_rng(11)
    return rng, tuple(h for _ in range(3))


@pytest.mark.parametrize("so", [4, 8, 16])
def test_var_star_update(so):
    r = so // 2
    full = (20 + 2 * so, 22 + 2 * so, 32 + 2 * so)
    lo, hi = (so,) * 3, tuple(n - so for n in full)
    rng = np.random.default_rng(so)
    u0, u2 = (np.float32(rng.standard_normal(full)) for _ in range(2))
    A = np.float32(2.0 - 0.1 * rng.random(full))
    B = np.float32(-1.0 + 0.1 * rng.random(full))
    Sv = np.float32(0.01 + 0.01 * rng.random(full))
    w = [float(c) for c in S.fd_coefficients(2, so)]
    coeffs = [np.float32([w[r + k] / (10.0 ** 2) for k in range(r + 1)]) for _ in range(3)]
    tab = R.coeff_table(coeffs, NC)
    t = [dev(x) for x in (u0, u2, A, B, Sv)]
    u1 = torch.zeros_like(t[0])
    call("sdmp_var_star_update", None, *[C.c_void_p(x.data_ptr()) for x in t[:5]],
         C.c_void_p(u1.data_ptr()), arr(C.c_int64, full), arr(C.c_int64, lo),
         arr(C.c_int64, hi), arr(C.c_int32, [r] * 3),
         tab.ctypes.data_as(C.POINTER(C.c_float)), 0)
    want = np.zeros(full)
    K.var_star_update(u0.astype(np.float64), u2.astype(np.float64), A.astype(np.float64),
                      B.astype(np.float64), Sv.astype(np.float64),
                      [c.astype(np.float64) for c in coeffs], (lo, hi), want)
    s = tuple(slice(a, b) for a, b in zip(lo, hi))
    assert rel_l2(u1.cpu().numpy()[s], want[s]) <= REL


@pytest.mark.parametrize("so", [4, 8])
def test_tti_update(so):
    r = so // 2
    full = (16 + 4 * so, 16 + 4 * so, 24 + 4 * so)
    lo, hi = (2 * so,) * 3, tuple(n - 2 * so for n in full)
    rng = np.random.default_rng(so + 1)
    p0, p2, r0, r2 = (np.float32(rng.standard_normal(full)) for _ in range(4))
    m = np.float32(0.2 + 0.2 * rng.random(full))
    epsp = np.float32(1.0 + 0.3 * rng.random(full))
    delp = np.float32(1.0 + 0.1 * rng.random(full))
    th, ph = rng.random(full) * 0.6, rng.random(full) * 0.6
    a = [np.float32(np.sin(th) * np.cos(ph)), np.float32(np.sin(th) * np.sin(ph)),
         np.float32(np.cos(th))]
    h = 10.0
    w2 = [float(c) for c in S.fd_coefficients(2, so)]
    w1 = [float(c) for c in S.fd_coefficients(1, so)]
    lap = [np.float32([w2[r + k] / h ** 2 for k in range(r + 1)]) for _ in range(3)]
    d1 = [np.float32([0.0] + [w1[r + k] / h for k in range(1, r + 1)]) for _ in range(3)]
    dt2 = float(np.float32(0.5 ** 2))
    ins = [dev(x) for x in (p0, p2, r0, r2, m, epsp, delp, *a)]
    p1, r1 = torch.zeros_like(ins[0]), torch.zeros_like(ins[0])
    call("sdmp_tti_update", None, ptrs(ins), C.c_void_p(p1.data_ptr()), C.c_void_p(r1.data_ptr()),
         arr(C.c_int64, full), arr(C.c_int64, lo), arr(C.c_int64, hi), r,
         R.coeff_table(lap, NC).ctypes.data_as(C.POINTER(C.c_float)),
         R.coeff_table(d1, NC).ctypes.data_as(C.POINTER(C.c_float)), C.c_float(dt2), 0)
    f64 = lambda x: x.astype(np.float64)
    wp, wr = np.zeros(full), np.zeros(full)
    K.tti_update(f64(p0), f64(p2), f64(r0), f64(r2), f64(m), f64(epsp), f64(delp),
                 [f64(x) for x in a], [f64(c) for c in lap], [f64(c) for c in d1], dt2,
                 (lo, hi), wp, wr)
    s = tuple(slice(x, y) for x, y in zip(lo, hi))
    assert rel_l2(p1.cpu().numpy()[s], wp[s]) <= REL
    assert rel_l2(r1.cpu().numpy()[s], wr[s]) <= REL


@pytest.mark.parametrize("so", [4, 8, 16])
def test_staggered_entry_points(so):
    r = so // 2
    full = (16 + 2 * so, 18 + 2 * so, 24 + 2 * so)
    lo, hi = (so,) * 3, tuple(n - so for n in full)
    rng = np.random.default_rng(so + 2)
    rnd = lambda: np.float32(rng.standard_normal(full))
    v0 = [rnd() for _ in range(3)]
    t0 = [rnd() for _ in range(6)]
    r0 = [rnd() for _ in range(6)]
    b = np.float32(0.5 + rng.random(full))
    lam, mu = np.float32(1.0 + rng.random(full)), np.float32(0.5 + rng.random(full))
    l2m, mus = np.float32(2.0 + rng.random(full)), np.float32(0.5 + rng.random(full))
    its = np.float32(np.full(full, 0.3))
    h, dt = 10.0, float(np.float32(0.4))
    sc = [np.float32([float(c) / h for c in S.staggered_coefficients(so)]) for _ in range(3)]
    sct = R.coeff_table(sc, MR).ctypes.data_as(C.POINTER(C.c_float))
    f64 = lambda x: x.astype(np.float64)
    box = (lo, hi)
    s = tuple(slice(x, y) for x, y in zip(lo, hi))
    geo = (arr(C.c_int64, full), arr(C.c_int64, lo), arr(C.c_int64, hi), r)
    # velocity
    dv0, dt0, db = [dev(x) for x in v0], [dev(x) for x in t0], dev(b)
    dv1 = [torch.zeros_like(db) for _ in range(3)]
    call("sdmp_elastic_velocity", None, ptrs(dv0), ptrs(dt0), C.c_void_p(db.data_ptr()),
         ptrs(dv1), *geo, sct, C.c_float(dt))
    wv = [np.zeros(full) for _ in range(3)]
    K.velocity_update([f64(x) for x in v0], [f64(x) for x in t0], f64(b), [f64(c) for c in sc],
                      dt, box, wv)
    for g, w in zip(dv1, wv):
        assert rel_l2(g.cpu().numpy()[s], w[s]) <= REL
    # elastic stress (reads the new velocities)
    v1 = [np.float32(w) for w in wv]
    dv1 = [dev(x) for x in v1]
    dt1 = [torch.zeros_like(db) for _ in range(6)]
    dlam, dmu = dev(lam), dev(mu)  # keep the tensors alive across the call
    call("sdmp_elastic_stress", None, ptrs(dv1), ptrs(dt0), C.c_void_p(dlam.data_ptr()),
         C.c_void_p(dmu.data_ptr()), ptrs(dt1), *geo, sct, C.c_float(dt))
    wt = [np.zeros(full) for _ in range(6)]
    K.stress_update([f64(x) for x in v1], [f64(x) for x in t0], f64(lam), f64(mu),
                    [f64(c) for c in sc], dt, box, wt)
    for g, w in zip(dt1, wt):
        assert rel_l2(g.cpu().numpy()[s], w[s]) <= REL
    # viscoelastic stress + memory variables
    dr0 = [dev(x) for x in r0]
    prm = [dev(x) for x in (l2m, mus, its)]
    ds1 = [torch.zeros_like(db) for _ in range(6)]
    dr1 = [torch.zeros_like(db) for _ in range(6)]
    call("sdmp_visco_stress", None, ptrs(dv1), ptrs(dt0), ptrs(dr0), ptrs(prm), ptrs(ds1),
         ptrs(dr1), *geo, sct, C.c_float(dt))
    ws, wr = [np.zeros(full) for _ in range(6)], [np.zeros(full) for _ in range(6)]
    K.visco_stress_update([f64(x) for x in v1], [f64(x) for x in t0], [f64(x) for x in r0],
                          f64(l2m), f64(mus), f64(its), [f64(c) for c in sc], dt, box, ws, wr)
    for g, w in zip(ds1 + dr1, ws + wr):
        assert rel_l2(g.cpu().numpy()[s], w[s]) <= REL


def test_inject_interpolate_entry_points():
    full = (12, 10, 16)
    rng = np.random.default_rng(5)
    field = torch.zeros(full, device="cuda")
    n = field.numel()
    node = torch.tensor([17, 200, 1503], dtype=torch.int64, device="cuda")
    ptr = torch.tensor([0, 2, 3, 5], dtype=torch.int32, device="cuda")
    pid = torch.tensor([0, 1, 1, 0, 1], dtype=torch.int32, device="cuda")
    w = torch.tensor([0.25, 0.5, 1.0, 0.125, 0.375], device="cuda")
    amps = torch.tensor([2.0, -4.0], device="cuda")
    m = torch.full(full, 0.5, device="cuda")
    call("sdmp_inject", None, C.c_void_p(field.data_ptr()), C.c_void_p(node.data_ptr()),
         C.c_void_p(ptr.data_ptr()), 3, C.c_void_p(pid.data_ptr()), C.c_void_p(w.data_ptr()),
         C.c_void_p(amps.data_ptr()), C.c_float(3.0), C.c_void_p(m.data_ptr()))
    flat = field.reshape(-1).cpu().numpy()
    want = {17: (0.25 * 2 + 0.5 * -4) * 3 / 0.5, 200: (1.0 * -4) * 3 / 0.5,
            1503: (0.125 * 2 + 0.375 * -4) * 3 / 0.5}
    for k, v in want.items():
        assert abs(flat[k] - v) < 1e-5
    assert np.count_nonzero(flat) == 3 and n == flat.size
    # interpolate two points with 2 corners each
    src = torch.from_numpy(np.float32(rng.standard_normal(full))).cuda()
    idx = torch.tensor([5, 6, 400, 401], dtype=torch.int64, device="cuda")
    ww = torch.tensor([0.3, 0.7, 0.9, 0.1], device="cuda")
    out = torch.zeros(2, device="cuda")
    call("sdmp_interpolate", None, C.c_void_p(src.data_ptr()), C.c_void_p(idx.data_ptr()),
         C.c_void_p(ww.data_ptr()), 2, 2, C.c_void_p(out.data_ptr()))
    sf = src.reshape(-1).cpu().numpy().astype(np.float64)
    got = out.cpu().numpy()
    assert abs(got[0] - (0.3 * sf[5] + 0.7 * sf[6])) < 1e-5
    assert abs(got[1] - (0.9 * sf[400] + 0.1 * sf[401])) < 1e-5


@pytest.mark.parametrize("so", [4, 8])
def test_collocated_elastic_entry_points(so):
    r = so // 2
    full = (16 + 2 * so, 18 + 2 * so, 24 + 2 * so)
    lo, hi = (so,) * 3, tuple(n - so for n in full)
    rng = np.random.default_rng(so + 7)
    rnd = lambda: np.float32(rng.standard_normal(full))
    v0, t0 = [rnd() for _ in range(3)], [rnd() for _ in range(6)]
    b = np.float32(0.5 + rng.random(full))
    lam, mu = np.float32(1.0 + rng.random(full)), np.float32(0.5 + rng.random(full))
    h, dt = 10.0, float(np.float32(0.4))
    w1 = [float(c) for c in S.fd_coefficients(1, so)]
    c1 = [np.float32([w1[r + k] / h for k in range(1, r + 1)]) for _ in range(3)]
    c1t = R.coeff_table(c1, MR).ctypes.data_as(C.POINTER(C.c_float))
    f64 = lambda x: x.astype(np.float64)
    box, s = (lo, hi), tuple(slice(x, y) for x, y in zip(lo, hi))
    geo = (arr(C.c_int64, full), arr(C.c_int64, lo), arr(C.c_int64, hi), r)
    dv0, dt0, db = [dev(x) for x in v0], [dev(x) for x in t0], dev(b)
    dv1 = [torch.zeros_like(db) for _ in range(3)]
    call("sdmp_elastic_colloc_velocity", None, ptrs(dv0), ptrs(dt0), C.c_void_p(db.data_ptr()),
         ptrs(dv1), *geo, c1t, C.c_float(dt))
    wv = [np.zeros(full) for _ in range(3)]
    K.velocity_update([f64(x) for x in v0], [f64(x) for x in t0], f64(b), [f64(c) for c in c1],
                      dt, box, wv, col=True)
    for g, w in zip(dv1, wv):
        assert rel_l2(g.cpu().numpy()[s], w[s]) <= REL
    v1 = [np.float32(w) for w in wv]
    dv1 = [dev(x) for x in v1]
    dlam, dmu = dev(lam), dev(mu)
    dt1 = [torch.zeros_like(db) for _ in range(6)]
    call("sdmp_elastic_colloc_stress", None, ptrs(dv1), ptrs(dt0), C.c_void_p(dlam.data_ptr()),
         C.c_void_p(dmu.data_ptr()), ptrs(dt1), *geo, c1t, C.c_float(dt))
    wt = [np.zeros(full) for _ in range(6)]
    K.stress_update([f64(x) for x in v1], [f64(x) for x in t0], f64(lam), f64(mu),
                    [f64(c) for c in c1], dt, box, wt, col=True)
    for g, w in zip(dt1, wt):
        assert rel_l2(g.cpu().numpy()[s], w[s]) <= REL


def test_rot_update_entry_point():
    so = 8
    r = so // 2
    full = (16 + 4 * so, 16 + 4 * so, 24 + 4 * so)
    lo, hi = (2 * so,) * 3, tuple(n - 2 * so for n in full)
    rng = np.random.default_rng(21)
    u0, u2 = (np.float32(rng.standard_normal(full)) for _ in range(2))
    m = np.float32(0.2 + 0.2 * rng.random(full))
    th, ph = rng.random(full) * 0.6, rng.random(full) * 0.6
    a = [np.float32(np.sin(th) * np.cos(ph)), np.float32(np.sin(th) * np.sin(ph)),
         np.float32(np.cos(th))]
    w1 = [float(c) for c in S.fd_coefficients(1, so)]
    d1 = [np.float32([0.0] + [w1[r + k] / 10.0 for k in range(1, r + 1)]) for _ in range(3)]
    dt2 = float(np.float32(0.25))
    ins = [dev(x) for x in (u0, u2, m, *a)]
    u1 = torch.zeros_like(ins[0])
    call("sdmp_rot_update", None, ptrs(ins), C.c_void_p(u1.data_ptr()), arr(C.c_int64, full),
         arr(C.c_int64, lo), arr(C.c_int64, hi), r,
         R.coeff_table(d1, NC).ctypes.data_as(C.POINTER(C.c_float)), C.c_float(dt2))
    f64 = lambda x: x.astype(np.float64)
    want = np.zeros(full)
    K.rot_update(f64(u0), f64(u2), f64(m), [f64(x) for x in a], [f64(c) for c in d1], dt2,
                 (lo, hi), want)
    s = tuple(slice(x, y) for x, y in zip(lo, hi))
    assert rel_l2(u1.cpu().numpy()[s], want[s]) <= REL


@pytest.mark.parametrize("so", [4, 8])
def test_tti_and_rot_bound_scale_flag(so):
    """radius | SDMP_VARIANT_M_IS_SCALE: the m operand holds the bound
    RN(dt2 / m) (what the plan passes) -- bit-identical to dividing per
    point, for the single-pass (SO-4 TTI, both rotated) and two-pass (SO-8
    TTI) kernels."""
    r = so // 2
    full = (16 + 4 * so, 16 + 4 * so, 24 + 4 * so)
    lo, hi = (2 * so,) * 3, tuple(n - 2 * so for n in full)
    rng = np.random.default_rng(so + 7)
    p0, p2, r0, r2 = (np.float32(rng.standard_normal(full)) for _ in range(4))
    m = np.float32(0.2 + 0.2 * rng.random(full))
    epsp = np.float32(1.0 + 0.3 * rng.random(full))
    delp = np.float32(1.0 + 0.1 * rng.random(full))
    th, ph = rng.random(full) * 0.6, rng.random(full) * 0.6
    a = [np.float32(np.sin(th) * np.cos(ph)), np.float32(np.sin(th) * np.sin(ph)),
         np.float32(np.cos(th))]
    w2 = [float(c) for c in S.fd_coefficients(2, so)]
    w1 = [float(c) for c in S.fd_coefficients(1, so)]
    lap = R.coeff_table([np.float32([w2[r + k] / 100.0 for k in range(r + 1)])] * 3, NC)
    d1 = R.coeff_table([np.float32([0.0] + [w1[r + k] / 10.0 for k in range(1, r + 1)])] * 3, NC)
    dt2 = np.float32(0.25)
    scale = np.float32(dt2 / m)   # IEEE round-to-nearest fp32 division
    fp = lambda t: t.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
    outs = []
    for mm, rad in ((m, r), (scale, r | R.VARIANT_M_IS_SCALE)):
        ins = [dev(x) for x in (p0, p2, r0, r2, mm, epsp, delp, *a)]
        p1, r1 = torch.zeros_like(ins[0]), torch.zeros_like(ins[0])
        call("sdmp_tti_update", None, ptrs(ins), C.c_void_p(p1.data_ptr()),
             C.c_void_p(r1.data_ptr()), arr(C.c_int64, full), arr(C.c_int64, lo),
             arr(C.c_int64, hi), rad, fp(lap), fp(d1), C.c_float(float(dt2)), 0)
        rins = [dev(x) for x in (p0, p2, mm, *a)]
        u1 = torch.zeros_like(rins[0])
        call("sdmp_rot_update", None, ptrs(rins), C.c_void_p(u1.data_ptr()),
             arr(C.c_int64, full), arr(C.c_int64, lo), arr(C.c_int64, hi), rad, fp(d1),
             C.c_float(float(dt2)))
        outs.append([t.cpu().numpy() for t in (p1, r1, u1)])
    for x, y in zip(*outs):
        assert np.array_equal(x, y)
        assert np.abs(x).max() > 0


def test_copy_box_engines_identical():
    """sdmp_copy_box engine 0 (copy engine), 1 (SM, one kernel per box) and 2
    (the batched post kernel) move the same box bit for bit, including
    rows that are not 16-byte aligned (scalar path)."""
    full = (20, 18, 40)
    rng = np.random.default_rng(3)
    src = dev(rng.standard_normal(full))
    for slo, dlo, ext in (((2, 3, 8), (1, 0, 8), (4, 5, 24)), ((2, 3, 1), (1, 0, 3), (4, 5, 30)),
                          ((0, 0, 0), (0, 0, 0), (20, 18, 40))):
        res = []
        for engine in (0, 1, 2):
            dst = torch.zeros_like(src)
            call("sdmp_copy_box", None, C.c_void_p(src.data_ptr()), arr(C.c_int64, full),
                 arr(C.c_int64, slo), C.c_void_p(dst.data_ptr()), arr(C.c_int64, full),
                 arr(C.c_int64, dlo), arr(C.c_int64, ext), engine)
            res.append(dst.cpu().numpy())
        want = np.zeros(full, np.float32)
        sv = src.cpu().numpy()
        want[tuple(slice(d, d + e) for d, e in zip(dlo, ext))] = \
            sv[tuple(slice(s_, s_ + e) for s_, e in zip(slo, ext))]
        for r_ in res:
            assert np.array_equal(r_, want)
