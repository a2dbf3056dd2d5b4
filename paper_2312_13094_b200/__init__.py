"""B200-native finite-difference propagators with automated halo exchange
(arXiv 2312.13094 hot path).

Drop-in surfaces:

* ``paper_2312_13094_b200.symbolics`` — the reference ``stencil_dmp.symbolics``
  API (GridSpec, FieldSpec, Eq, solve_forward, fd_coefficients, apply_cse, ...);
* ``Grid / Function / TimeFunction / SparseTimeFunction / Operator / solve``
  — the paper's Listing 1 API, executed by hand-written sm_100a kernels in
  ``libsdmp.so`` (include/sdmp.h) with basic / diagonal / full halo exchange
  over NVLink between one process per GPU.
"""
from . import symbolics
from .symbolics import (Eq, FieldSpec, GridSpec, StencilEquation, apply_cse, discretize,
                        fd_coefficients, solve_forward)
from .api import (Data, Function, Grid, Operator, SparseTimeFunction, TimeFunction, load_dump,
                  ricker, solve)
from .decomposition import Decomposition, Topology, default_topology, decompose_axis
from .distfield import RegionName, region_boxes

__version__ = "0.1.0"
