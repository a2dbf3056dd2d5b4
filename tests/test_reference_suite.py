"""Runs the reference's OWN symbolic test-suite
(/root/reference/pkg/tests/test_symbolics.py) against the product module by
aliasing ``stencil_dmp.symbolics`` to ``paper_2312_13094_b200.symbolics``.

Only possible in the build container (the reference is not on the GPU box).
The reference itself passes 24/25 of these tests: test_cse_extracts_shared_
center_term (test_symbolics.py:248) contradicts the reference's own
apply_cse; the product reproduces the reference's behaviour exactly, so the
same single test fails in both and is deselected here.
"""
import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests/test_symbolics.py"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHIM = r"""
import sys, types
sys.path.insert(0, %r)
import paper_2312_13094_b200.symbolics as s
pkg = types.ModuleType('stencil_dmp'); pkg.__path__ = []; pkg.symbolics = s
sys.modules['stencil_dmp'] = pkg; sys.modules['stencil_dmp.symbolics'] = s
import pytest
sys.exit(pytest.main(['-q', '-p', 'no:cacheprovider', '--rootdir', '/tmp',
                      %r, '-k', 'not test_cse_extracts_shared_center_term']))
"""


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference not mounted")
def test_reference_suite_runs_against_product():
    code = SHIM % (ROOT, REF_TESTS)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True,
                         text=True, cwd="/tmp", timeout=300)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert "24 passed, 1 deselected" in res.stdout, res.stdout[-2000:]
