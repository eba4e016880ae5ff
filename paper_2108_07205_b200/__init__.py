"""B200-native refined-wall Stokes solver (arXiv 2108.07205 per-time-step path).

Public API mirrors the reference C++ solver (proj/include/stokesbie): see
``api.py``.  Everything numerical runs in ``_lib/libsbx.so`` (sm_100a CUDA
kernels behind the C-ABI of ``include/sbx.h``).
"""
from .api import (  # noqa: F401
    CHANNEL, CIRCLE, ELLIPSE, EXTERIOR_COMBINED, FOURIER, INTERIOR_DIRICHLET, MIXED, STAR, SVD_OPTIMAL, TWO_STEP_ID,
    AppBlockSolver, UpdateCache, CurveParams, Discretization, ElsSolver, HbsOperator, HbsOptions, LowRankUpdate,
    RefinementPlan, add_holes, app_build, boundary_data, circle, coarsen, compress_update, density_on_refined,
    channel, ellipse, els_apply_forward, els_build, els_conditioning, els_gmres, els_solve, els_solve_into, els_solve_raw,
    evaluate_solution,
    gather_kept_added, hbs_apply, hbs_compress, hbs_invert, hbs_load, hbs_save, hbs_solve, init, kernel_launches, panelize, refine, row_id, dense_inverse, matmul,
    star, submatrix, update_from_factors, update_dump, update_load, dump_matrix, load_matrix,
)
from ._sbx import (  # noqa: F401
    ConvergenceError, CudaError, GeometryError, ProxyViolationError, SbxError, SingularMatrixError,
)
