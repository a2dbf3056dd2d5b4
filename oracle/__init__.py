"""ORACLE — CPU restatement of the reference's FD-propagator path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker (or the timed CPU reference arm), never as
the thing measured or shipped.  The product package
``paper_2312_13094_b200`` never imports it and has no CPU fallback.

What it restates (numpy, fp64 arithmetic):

* ``decomp``   — SPEC.md:118-200 (topology, axis split, neighbours,
  global->local, owners) and SPEC.md:252-260 / 358-366 / 440-448 (regions,
  messages per mode), written brute-force (per-cell classification) so it
  checks the product's box algebra independently.
* ``stencils`` — the per-point updates: acoustic / diffusion from the
  reference's own solved equations (symbolics.py:591-674; PAPER.md:964-990,
  1111-1131), TTI rotated Laplacian,
  staggered elastic, viscoelastic;
  sparse trilinear inject/interpolate + Ricker.
* ``runtime``  — simulated SPMD ranks executing basic / diagonal / full
   over per-rank FULL buffers.

Parity status:

* symbolic stage (FD weights, solved acoustic/diffusion updates) — PINNED to
  the reference: golden fixtures generated from the reference symbolics
  (tests/golden/make_golden.py) plus the reference's own test-suite run
  against the product (tests/test_reference_suite.py);
* Listing 3 / Listing 4 values and SPEC worked examples — PINNED (hand
  constants from PAPER.md / SPEC.md);
* runtime / exchange / sparse — restated from SPEC prose (no executable
  reference exists: the reference implements only ``symbolics``);
* TTI (full two-field), staggered elastic, viscoelastic — PARITY UNPINNED:
  the reference has no implementation or fixture for them; the oracle
  restates the paper's equations.
"""
