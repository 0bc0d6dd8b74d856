"""B200-native hot path of ctkrylov's hybrid AB-/BA-GMRES.

Names mirror the reference package (ctkrylov/__init__.py:4-17) for the
operators, the Arnoldi / projected-solve layer, lambda selection and the
GMRES drivers, so a reference script ports by swapping its import.  The
projectors and Krylov vector work run in libctk.so (hand-written sm_100a
CUDA behind the C ABI in include/ctk.h); there is no CPU fallback.
"""

from .linop import (LinearOperator, OperatorShapeError, compose, dense_operator, op_norm_estimate,
                    transpose_of)
from .ct import (BUILTIN_PROBLEMS, CtProblem, DeviceGeometry, GeometryError, GpuAdjoint, GpuBack,
                 GpuForward, ImageGrid, ParallelGeometry, back_pixel_driven, build_test_problem,
                 forward_ray_driven, make_ct_problem, matched_back, shepp_logan, write_csv_image,
                 write_pgm)
from .arnoldi import (ArnoldiState, Breakdown, DeviceBasis, ProjectedSolution, arnoldi_step,
                      solve_projected_ls, solve_projected_tikhonov)
from .regparam import (DegenerateCurveError, gcv_minimize, lambda_grid, lcurve_corner,
                       select_lambda, svd_of_hessenberg, tikhonov_curve_points)
from .gmres import (ConfigError, IterationRecord, KernelTimer, SolveResult, SolverConfig,
                    run_ab_gmres, run_ba_gmres, run_gmres)
from .gk import run_lsmr, run_lsqr
from .problems import CONFIGS, add_noise, random_ellipse_phantom
from .metrics import dp_should_stop, ncp_distance, ncp_should_stop, rns_should_stop, rre, ssim

__version__ = "0.1.0"
