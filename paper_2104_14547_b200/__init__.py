"""paper_2104_14547_b200 — B200-native hot path of NURBS-Diff (arXiv 2104.14547).

Batched NURBS curve/surface evaluation (forward, Eq.3 P:110 / Alg.1) and its
deterministic backward (Eq.8-10 P:214-251 / Alg.2) as hand-written sm_100a CUDA
behind the C ABI of include/nurbs.h. This package is the thin Python binding: it only
marshals torch tensors (device pointers, the current CUDA stream) into those calls.
"""
from ._abi import NURBS_MAX_DEGREE, NurbsError, nurbs_shape  # noqa: F401
from .api import (  # noqa: F401
    Tables,
    curve_bwd,
    curve_fwd,
    nurbs_curve_bwd,
    nurbs_curve_fwd,
    nurbs_surface_bwd,
    nurbs_surface_fwd,
    nurbs_tables,
    nurbs_validate,
    surface_bwd,
    surface_fwd,
    surface_shape,
    curve_shape,
    bwd_workspace_bytes,
    grid_plan,
    path_flags,
    nurbs_sum_partials,
    fit_workspace_bytes,
    nurbs_surface_fit_step,
    SurfaceFitter,
    nurbs_surface_derivs,
    surface_derivs,
    points_shape,
    points_workspace_bytes,
    nurbs_surface_points_fwd,
    nurbs_surface_points_bwd,
    nurbs_validate_points,
    surface_points_fwd,
    surface_points_bwd,
    knots_workspace_bytes,
    nurbs_surface_bwd_knots,
    nurbs_curve_bwd_knots,
    surface_bwd_knots,
    curve_bwd_knots,
)
from .pipeline import HostBatchPipeline  # noqa: F401,E402
