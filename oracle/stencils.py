"""ORACLE (test infrastructure) — per-point updates in fp64 numpy.

Every function works on FULL arrays (DOMAIN + halo, the layout of
SPEC.md:214-217) and updates the cells of a box given in FULL coordinates,
leaving everything else untouched; the exterior halo stays zero
(SPEC.md:269).  Coefficients are passed in already bound to fp32
(SURVEY.md §8c parity rule) and evaluated here in fp64.
"""
import math

import numpy as np


def _sl(box, shift=None):
    lo, hi = box
    shift = shift or (0,) * len(lo)
    return tuple(slice(l + s, h + s) for l, h, s in zip(lo, hi, shift))


def _unit(a, k, nd):
    v = [0] * nd
    v[a] = k
    return v


def star_laplacian(u, box, coeffs):
    """sum_a [c_a0 u + sum_k c_ak (u[-k e_a] + u[+k e_a])]; ``coeffs[a]`` are
    the centre-out weights w_k / h_a^2 (reference discretize of
    ``u.laplace``, symbolics.py:148-149, 494-566)."""
    nd = u.ndim
    out = np.zeros(tuple(h - l for l, h in zip(*box)), dtype=np.float64)
    for a in range(nd):
        c = coeffs[a]
        acc = c[0] * u[_sl(box)]
        for k in range(1, len(c)):
            acc = acc + c[k] * (u[_sl(box, _unit(a, -k, nd))] + u[_sl(box, _unit(a, k, nd))])
        out += acc
    return out


def star_update(u0, u2, m, coeffs, A, B, C, box, out):
    """u1 = A u0 + B u2 + (C / m) L(u0)   (m=None -> C L(u0)).

    Acoustic (A,B,C) = (2, -1, dt^2): the reference's solved
    ``m*u.dt2 - u.laplace`` (symbolics.py:629-674);
    diffusion (1, 0, dt): ``Eq(u.dt, u.laplace)``."""
    s = _sl(box)
    lap = star_laplacian(u0, box, coeffs)
    scale = C if m is None else C / m[s]
    val = A * u0[s] + scale * lap
    if B != 0.0:
        val = val + B * u2[s]
    out[s] = val


def var_star_update(u0, u2, A, B, S, coeffs, box, out):
    """u1 = A u0 + B u2 + S L(u0) with pointwise coefficient arrays: the
    reference's solved ``m*u.dt2 - u.laplace + damp*u.dt`` (forward
    first-order time difference, symbolics.py:530-546, solved by
    solve_forward, symbolics.py:591-674) gives A = (2m + d dt)/(m + d dt),
    B = -m/(m + d dt), S = dt^2/(m + d dt).  B None -> no u2 term."""
    s = _sl(box)
    lap = star_laplacian(u0, box, coeffs)
    val = A[s] * u0[s] + S[s] * lap
    if B is not None:
        val = val + B[s] * u2[s]
    out[s] = val


def first_derivative(f, box, a, w1):
    """Central first derivative along a with weights w1[k], k=1..R (already
    divided by h): sum_k w_k (f[+k] - f[-k])."""
    nd = f.ndim
    acc = np.zeros(tuple(h - l for l, h in zip(*box)))
    for k in range(1, len(w1)):
        acc += w1[k] * (f[_sl(box, _unit(a, k, nd))] - f[_sl(box, _unit(a, -k, nd))])
    return acc


def grow(box, r):
    return (tuple(l - r for l in box[0]), tuple(h + r for h in box[1]))


def tti_update(p0, p2, r0, r2, m, epsp, delp, dirc, lap_c, d1_c, dt2, box, p1, r1):
    """Pseudo-acoustic TTI, two coupled fields (PAPER.md:999-1018,
    Devito's centred kernel form):

        Gzz f = sum_i d_i( a_i * sum_j a_j d_j f )   (nested, radius SO)
        H0 f  = lap f - Gzz f
        p1 = 2 p0 - p2 + dt2/m (eps' H0 p0 + del' Gzz r0)
        r1 = 2 r0 - r2 + dt2/m (del' H0 p0 + Gzz r0)

    ``dirc`` = (a_x, a_y, a_z) = (sin t cos f, sin t sin f, cos t) arrays,
    ``epsp`` = 1 + 2 eps, ``delp`` = sqrt(1 + 2 delta), ``d1_c[a]`` first
    derivative weights w_k/h_a (k = 0..R, entry 0 unused)."""
    R = len(d1_c[0]) - 1
    gbox = grow(box, R)

    def gzz(f):
        g = np.zeros(tuple(h - l for l, h in zip(*gbox)))
        for j in range(3):
            g += dirc[j][_sl(gbox)] * first_derivative(f, gbox, j, d1_c[j])
        out = np.zeros(tuple(h - l for l, h in zip(*box)))
        for i in range(3):
            # a_i * g on gbox, then centred derivative evaluated on box
            ag = dirc[i][_sl(gbox)] * g
            tmp = np.zeros(p0.shape)
            tmp[_sl(gbox)] = ag
            out += first_derivative(tmp, box, i, d1_c[i])
        return out

    s = _sl(box)
    gp = gzz(p0)
    gr = gzz(r0)
    h0p = star_laplacian(p0, box, lap_c) - gp
    sc = dt2 / m[s]
    p1[s] = 2.0 * p0[s] - p2[s] + sc * (epsp[s] * h0p + delp[s] * gr)
    r1[s] = 2.0 * r0[s] - r2[s] + sc * (delp[s] * h0p + gr)


def rot_update(u0, u2, m, dirc, d1_c, dt2, box, u1):
    """Single-field rotated operator (tti_gxx_kernel):
    m u_tt = G u with G u = sum_i d_i(a_i sum_j a_j d_j u) (nested centred
    first derivatives); u1 = 2 u0 - u2 + dt2/m G u0."""
    R = len(d1_c[0]) - 1
    gbox = grow(box, R)
    g = np.zeros(tuple(h - l for l, h in zip(*gbox)))
    for j in range(3):
        g += dirc[j][_sl(gbox)] * first_derivative(u0, gbox, j, d1_c[j])
    G = np.zeros(tuple(h - l for l, h in zip(*box)))
    for i in range(3):
        tmp = np.zeros(u0.shape)
        tmp[_sl(gbox)] = dirc[i][_sl(gbox)] * g
        G += first_derivative(tmp, box, i, d1_c[i])
    s = _sl(box)
    u1[s] = 2.0 * u0[s] - u2[s] + dt2 / m[s] * G


# --- staggered first derivatives (Virieux 1986) --------------------------------

def dplus(f, box, a, c, col=False):
    """Derivative at i+1/2: sum_k c_k (f[i+k] - f[i-k+1]); c already / h.
    ``col``: the collocated centred derivative sum_k c_k (f[i+k] - f[i-k])."""
    if col:
        return first_derivative(f, box, a, [0.0] + list(c))
    nd = f.ndim
    acc = np.zeros(tuple(h - l for l, h in zip(*box)))
    for k in range(1, len(c) + 1):
        acc += c[k - 1] * (f[_sl(box, _unit(a, k, nd))] - f[_sl(box, _unit(a, 1 - k, nd))])
    return acc


def dminus(f, box, a, c, col=False):
    """Derivative at i-1/2: sum_k c_k (f[i+k-1] - f[i-k]) (``col``: centred)."""
    if col:
        return first_derivative(f, box, a, [0.0] + list(c))
    nd = f.ndim
    acc = np.zeros(tuple(h - l for l, h in zip(*box)))
    for k in range(1, len(c) + 1):
        acc += c[k - 1] * (f[_sl(box, _unit(a, k - 1, nd))] - f[_sl(box, _unit(a, -k, nd))])
    return acc


# v-components (x,y,z) and stress components in the order
# xx, yy, zz, xy, xz, yz.
def velocity_update(v0, t0, b, sc, dt, box, v1, col=False):
    """Phase 1 of elastic/viscoelastic: v1 = v0 + dt * b * div(tau0)
    (PAPER.md:1045-1051, 1066).  ``sc[a]`` staggered weights / h_a."""
    s = _sl(box)
    txx, tyy, tzz, txy, txz, tyz = t0
    dvx = (dplus(txx, box, 0, sc[0], col) + dminus(txy, box, 1, sc[1], col)
           + dminus(txz, box, 2, sc[2], col))
    dvy = (dminus(txy, box, 0, sc[0], col) + dplus(tyy, box, 1, sc[1], col)
           + dminus(tyz, box, 2, sc[2], col))
    dvz = (dminus(txz, box, 0, sc[0], col) + dminus(tyz, box, 1, sc[1], col)
           + dplus(tzz, box, 2, sc[2], col))
    bdt = dt * b[s]
    v1[0][s] = v0[0][s] + bdt * dvx
    v1[1][s] = v0[1][s] + bdt * dvy
    v1[2][s] = v0[2][s] + bdt * dvz


def _strains(v, box, sc, col=False):
    vx, vy, vz = v
    exx = dminus(vx, box, 0, sc[0], col)
    eyy = dminus(vy, box, 1, sc[1], col)
    ezz = dminus(vz, box, 2, sc[2], col)
    exy = dplus(vx, box, 1, sc[1], col) + dplus(vy, box, 0, sc[0], col)
    exz = dplus(vx, box, 2, sc[2], col) + dplus(vz, box, 0, sc[0], col)
    eyz = dplus(vy, box, 2, sc[2], col) + dplus(vz, box, 1, sc[1], col)
    return exx, eyy, ezz, exy, exz, eyz


def stress_update(v1, t0, lam, mu, sc, dt, box, t1, col=False):
    """Phase 2 elastic: tau1 = tau0 + dt (lam tr(grad v) I + mu (grad v + grad v^T))."""
    s = _sl(box)
    exx, eyy, ezz, exy, exz, eyz = _strains(v1, box, sc, col)
    l, m = lam[s], mu[s]
    tr = exx + eyy + ezz
    t1[0][s] = t0[0][s] + dt * (l * tr + 2.0 * m * exx)
    t1[1][s] = t0[1][s] + dt * (l * tr + 2.0 * m * eyy)
    t1[2][s] = t0[2][s] + dt * (l * tr + 2.0 * m * ezz)
    t1[3][s] = t0[3][s] + dt * (m * exy)
    t1[4][s] = t0[4][s] + dt * (m * exz)
    t1[5][s] = t0[5][s] + dt * (m * eyz)


def visco_stress_update(v1, s0, r0, l2m, mus, its, sc, dt, box, s1, r1):
    """Phase 2 viscoelastic, single relaxation:

        A_ii = (pi tp/ts - 2 mu ts_s/ts) div v + 2 mu ts_s/ts d_i v_i
        A_ij = mu ts_s/ts (d_i v_j + d_j v_i)
        r1   = r0 - dt/tau_sigma (r0 + A)
        s1   = s0 + dt (A + r1)

    with ``l2m`` = pi*tau_eps_p/tau_sigma, ``mus`` = mu*tau_eps_s/tau_sigma,
    ``its`` = 1/tau_sigma per point."""
    s = _sl(box)
    exx, eyy, ezz, exy, exz, eyz = _strains(v1, box, sc)
    L, M, I = l2m[s], mus[s], its[s]
    div = exx + eyy + ezz
    base = (L - 2.0 * M) * div
    A = [base + 2.0 * M * exx, base + 2.0 * M * eyy, base + 2.0 * M * ezz,
         M * exy, M * exz, M * eyz]
    for c in range(6):
        rn = r0[c][s] - dt * I * (r0[c][s] + A[c])
        r1[c][s] = rn
        s1[c][s] = s0[c][s] + dt * (A[c] + rn)


# --- sparse --------------------------------------------------

def ricker(f0, t, t0):
    """SPEC.md:527-535."""
    a = (math.pi * f0 * (np.asarray(t, dtype=np.float64) - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def trilinear(coords, spacing, shape):
    """Enclosing cell (clamped to n-2) + 2^nd weights, corners row-major
    ((0.25,0.75) -> (0.1875, 0.5625, 0.0625, 0.1875))."""
    nd = len(shape)
    cell, frac = [], []
    for x, h, n in zip(coords, spacing, shape):
        q = x / h
        i = min(max(int(math.floor(q)), 0), n - 2)
        cell.append(i)
        frac.append(q - i)
    corners, weights = [], []
    for bits in np.ndindex(*(2,) * nd):
        w = 1.0
        for b, f in zip(bits, frac):
            w *= f if b else 1.0 - f
        corners.append(tuple(c + b for c, b in zip(cell, bits)))
        weights.append(w)
    return corners, weights


def inject(field, halo, origin, nodes_w, amps, scale=None):
    """Per owned node, sum w*amp in point-id order then add (deterministic;
    SPEC.md:507-515).  ``scale`` = None | (C, None) | (C, m): the sum is
    multiplied by C or C/m[node].  ``nodes_w``: {global node: [(pid, w), ...]} already
    restricted to this rank's DOMAIN; ``origin`` = owned start per axis."""
    for node in sorted(nodes_w):
        acc = 0.0
        for pid, w in sorted(nodes_w[node]):
            acc += w * amps[pid]
        idx = tuple(g - o + h for g, o, h in zip(node, origin, halo))
        if scale is None:
            field[idx] += acc
        elif scale[1] is None:
            field[idx] += acc * scale[0]
        else:  # C / m[node]
            field[idx] += acc * (scale[0] / scale[1][idx])


def interpolate(field, halo, origin, corners, weights):
    acc = 0.0
    for c, w in zip(corners, weights):
        acc += w * field[tuple(g - o + h for g, o, h in zip(c, origin, halo))]
    return acc
