"""Product symbolics vs golden fixtures generated from the reference
symbolics (tests/golden/make_golden.py; reference symbolics.py:452-720)."""
import json
import os
from fractions import Fraction

import pytest

from paper_2312_13094_b200 import symbolics as S
from tests.golden.make_golden import CASES, describe

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "symbolics_golden.json")))


@pytest.mark.parametrize("key", sorted(GOLD["fd"]))
def test_fd_table_matches_reference(key):
    d, acc = map(int, key.split(","))
    assert [str(c) for c in S.fd_coefficients(d, acc)] == GOLD["fd"][key]


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_solved_equation_matches_reference(idx):
    want = GOLD["cases"][idx]
    got = describe(S, *CASES[idx])
    assert (got["kind"], got["ndims"], got["so"]) == (want["kind"], want["ndims"], want["so"])
    if "lines" in want:
        assert got["lines"] == want["lines"]
        assert got["cse_lines"] == want["cse_lines"]
    for k in ("sha256", "cse_sha256", "n_accesses", "unique_offsets", "radius",
              "n_temporaries", "probe"):
        assert got[k] == want[k], k


def test_paper_appendix_b_form():
    # u[t1] = dt*(r0*u[t0] + r1*r3 + r1*u[x-1] ...)
    g = S.GridSpec(shape=(4, 4), extent=(2.0, 2.0))
    u = S.FieldSpec(name="u", grid=g, space_order=2)
    out = S.apply_cse(S.solve_forward(S.Eq(u.dt, u.laplace), u.forward))
    bodies = dict(out.temporaries)
    assert S.mul(Fraction(-2), u.at()) in bodies.values()
    assert isinstance(out.rhs, S.Product) and out.rhs.factors[0] == S.DT


def test_staggered_weights():
    assert S.staggered_coefficients(4) == [Fraction(9, 8), Fraction(-1, 24)]
    assert S.staggered_coefficients(8) == [Fraction(1225, 1024), Fraction(-245, 3072),
                                           Fraction(49, 5120), Fraction(-5, 7168)]
    for so in (2, 4, 6, 8, 12, 16):
        c = S.staggered_coefficients(so)
        # exact on odd monomials x^(2j+1): sum c_k 2(k-1/2)^(2j+1) = delta_j0
        for j in range(len(c)):
            tot = sum(ck * 2 * (Fraction(2 * k + 1, 2)) ** (2 * j + 1)
                      for k, ck in enumerate(c))
            assert tot == (1 if j == 0 else 0)


def test_pow_extension():
    assert S.DT ** 2 == S.mul(S.DT, S.DT)
    with pytest.raises(TypeError):
        S.DT ** 0.5


def _case(kind, so):
    return next(c for c in GOLD["cases"] if (c["kind"], c["so"]) == (kind, so))


@pytest.mark.parametrize("so", [4, 8])
def test_tti_family_template_is_the_reference_discretization(so):
    """compiler.tti_updates (the template the Operator recognises TTI by)
    prints exactly the solved updates the REFERENCE symbolics produce for
    the paper's two-field TTI system (golden from make_golden.py)."""
    import hashlib
    from paper_2312_13094_b200 import compiler as CP
    g = S.GridSpec(shape=(16,) * 3, extent=(2.0,) * 3)
    F = lambda n, to: S.FieldSpec(name=n, grid=g, space_order=so, time_order=to)
    eq_p, eq_r = CP.tti_updates(F("p", 2), F("r", 2), F("m", 0), F("epsp", 0), F("delp", 0),
                                [F(f"a{c}", 0) for c in "xyz"])
    for eq, kind in ((eq_p, "tti_p"), (eq_r, "tti_r")):
        text = "\n".join(S.format_equation(eq))
        assert hashlib.sha256(text.encode()).hexdigest() == _case(kind, so)["sha256"], kind


@pytest.mark.parametrize("so", [4, 8, 16])
def test_collocated_elastic_template_is_the_reference_discretization(so):
    import hashlib
    from paper_2312_13094_b200 import compiler as CP
    g = S.GridSpec(shape=(16,) * 3, extent=(2.0,) * 3)
    F = lambda n, to: S.FieldSpec(name=n, grid=g, space_order=so, time_order=to)
    v = [F(n, 1) for n in ("vx", "vy", "vz")]
    t = [F(n, 1) for n in ("txx", "tyy", "tzz", "txy", "txz", "tyz")]
    eqs = CP.elastic_updates(v, t, F("b", 0), F("lam", 0), F("mu", 0))
    by = {e.lhs.spec.name: e for e in eqs}
    for name, kind in (("vx", "elastic_vx"), ("txx", "elastic_txx"), ("txy", "elastic_txy")):
        text = "\n".join(S.format_equation(by[name]))
        assert hashlib.sha256(text.encode()).hexdigest() == _case(kind, so)["sha256"], kind
