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
