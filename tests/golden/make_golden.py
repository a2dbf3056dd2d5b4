"""Generate golden fixtures from the *reference* symbolic front end.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/symbolics_golden.json: exact FD tables, the printed
solved/CSE'd update equations (Appendix-B form) for every kernel family and
space order the B200 path supports, and exact-rational evaluation probes.
The product's own symbolics (paper_2312_13094_b200/symbolics.py) is checked
against this file by tests/test_symbolics_golden.py.
"""
import hashlib
import json
import os
import sys
from fractions import Fraction

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "symbolics_golden.json")


def case_equations(S, kind, ndims, so):
    """Build the family's symbolic equation with module ``S`` (reference or
    product: both expose the same API). Returns (eq, unknown)."""
    shape = (4,) * ndims if kind == "diffusion" else (16,) * ndims
    g = S.GridSpec(shape=shape, extent=(2.0,) * ndims)
    if kind == "diffusion":
        u = S.FieldSpec(name="u", grid=g, space_order=so, time_order=1)
        return S.Eq(u.dt, u.laplace), u.forward
    if kind == "acoustic":
        u = S.FieldSpec(name="u", grid=g, space_order=so, time_order=2)
        m = S.FieldSpec(name="m", grid=g, space_order=so, time_order=0)
        return S.Eq(m.at() * u.dt2 - u.laplace), u.forward
    if kind == "tti_gxx":
        # G = D^T D with D = a_x d/dx + a_y d/dy + a_z d/dz,
        # nested first derivatives; a_* are static direction-cosine fields.
        u = S.FieldSpec(name="u", grid=g, space_order=so, time_order=2)
        m = S.FieldSpec(name="m", grid=g, space_order=so, time_order=0)
        a = [S.FieldSpec(name=f"a{S.AXIS_NAMES[i]}", grid=g, space_order=so,
                         time_order=0) for i in range(3)]
        inner = S.add(*(S.mul(a[j].at(), u.d(j)) for j in range(3)))
        gxx = S.add(*(S.Deriv(S.mul(a[i].at(), inner), i, 1) for i in range(3)))
        return S.Eq(m.at() * u.dt2 - gxx), u.forward
    if kind in ("tti_p", "tti_r"):
        # the paper's two-field TTI (the same construction
        # as compiler.tti_updates): Gzz f = sum_i D_i(a_i sum_j a_j D_j f),
        # H0 = laplace - Gzz, m p.dt2 = epsp H0 p + delp Gzz r,
        # m r.dt2 = delp H0 p + Gzz r
        F = lambda n, to: S.FieldSpec(name=n, grid=g, space_order=so, time_order=to)
        p, r, m, epsp, delp = F("p", 2), F("r", 2), F("m", 0), F("epsp", 0), F("delp", 0)
        a = [F(f"a{S.AXIS_NAMES[i]}", 0) for i in range(3)]

        def gzz(f):
            inner = S.add(*(S.mul(a[j].at(), f.d(j)) for j in range(3)))
            return S.add(*(S.Deriv(S.mul(a[i].at(), inner), i, 1) for i in range(3)))

        h0p = S.add(p.laplace, S.neg(gzz(p)))
        gr = gzz(r)
        if kind == "tti_p":
            return (S.Eq(S.mul(m.at(), p.dt2), S.add(S.mul(epsp.at(), h0p), S.mul(delp.at(), gr))),
                    p.forward)
        return S.Eq(S.mul(m.at(), r.dt2), S.add(S.mul(delp.at(), h0p), gr)), r.forward
    if kind.startswith("elastic_"):
        # the SPEC's collocated elastic_kernel (the same
        # construction as compiler.elastic_updates): one velocity, one normal
        # and one shear stress update
        F = lambda n, to: S.FieldSpec(name=n, grid=g, space_order=so, time_order=to)
        v = [F(n, 1) for n in ("vx", "vy", "vz")]
        t = [F(n, 1) for n in ("txx", "tyy", "tzz", "txy", "txz", "tyz")]
        b, lam, mu = F("b", 0), F("lam", 0), F("mu", 0)
        T = {(0, 0): 0, (1, 1): 1, (2, 2): 2, (0, 1): 3, (0, 2): 4, (1, 2): 5}
        tau = lambda i, j: t[T[(min(i, j), max(i, j))]]
        dv = lambda i, j: S.Deriv(v[i].forward, j, 1)
        if kind == "elastic_vx":
            div = S.add(*(tau(0, j).d(j) for j in range(3)))
            return S.Eq(v[0].dt, S.mul(b.at(), div)), v[0].forward
        if kind == "elastic_txx":
            tr = S.add(*(dv(k, k) for k in range(3)))
            rhs = S.add(S.mul(lam.at(), tr), S.mul(S.Const(Fraction(2)), mu.at(), dv(0, 0)))
            return S.Eq(t[0].dt, rhs), t[0].forward
        if kind == "elastic_txy":
            return S.Eq(t[3].dt, S.mul(mu.at(), S.add(dv(0, 1), dv(1, 0)))), t[3].forward
    raise ValueError(kind)


CASES = (
    [("diffusion", 2, so) for so in (2, 4, 8)]
    + [("diffusion", 3, so) for so in (2, 4)]
    + [("acoustic", nd, so) for nd in (2, 3) for so in (2, 4, 8, 12, 16)]
    + [("tti_gxx", 3, so) for so in (2, 4, 8)]
    + [(k, 3, so) for k in ("tti_p", "tti_r") for so in (4, 8)]
    + [(k, 3, so) for k in ("elastic_vx", "elastic_txx", "elastic_txy") for so in (4, 8, 16)]
)


def probe(S, expr, seed):
    """Exact evaluation on seeded rational bindings keyed by leaf text."""
    import random
    rng = random.Random(seed)
    leaves = sorted({S.format_expr(n) for n in S.walk(expr)
                     if isinstance(n, (S.Symbol, S.FieldAccess))})
    vals = {k: Fraction(rng.randint(1, 40), rng.randint(1, 12)) for k in leaves}
    bind = {n: vals[S.format_expr(n)] for n in S.walk(expr)
            if isinstance(n, (S.Symbol, S.FieldAccess))}
    return str(S.eval_exact(expr, bind))


def describe(S, kind, nd, so):
    eq, unknown = case_equations(S, kind, nd, so)
    solved = S.solve_forward(eq, unknown)
    cse = S.apply_cse(solved)
    lines = S.format_equation(solved)
    cse_lines = S.format_equation(cse)
    offs = sorted({a.offsets for a in S.accesses(solved.rhs)})
    text = "\n".join(lines)
    cse_text = "\n".join(cse_lines)
    rec = {
        "kind": kind, "ndims": nd, "so": so,
        "sha256": hashlib.sha256(text.encode()).hexdigest(),
        "cse_sha256": hashlib.sha256(cse_text.encode()).hexdigest(),
        "n_accesses": len(S.accesses(solved.rhs)),
        "unique_offsets": len(offs),
        "radius": max(abs(o) for off in offs for o in off),
        "n_temporaries": len(cse.temporaries),
        "probe": [probe(S, solved.rhs, s) for s in range(3)],
    }
    if len(text) < 4000:
        rec["lines"] = lines
        rec["cse_lines"] = cse_lines
    return rec


def main():
    sys.path.insert(0, REF)
    from stencil_dmp import symbolics as S
    data = {
        "generator": "tests/golden/make_golden.py (reference symbolics.py)",
        "fd": {f"{d},{acc}": [str(c) for c in S.fd_coefficients(d, acc)]
               for d in (1, 2) for acc in range(2, 18, 2)},
        "cases": [describe(S, *c) for c in CASES],
    }
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
    print("wrote", OUT, len(data["cases"]), "cases")


if __name__ == "__main__":
    main()
