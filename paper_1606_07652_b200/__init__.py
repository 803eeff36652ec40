"""B200-native band-limited FMM RBF matvec (arXiv 1606.07652 path).

The product is the sm_100a CUDA library ``libblfmm_gpu.so`` behind the C ABI
of ``include/blfmm_gpu.h``; this package is the host-side mirror of the
reference library's interface (see ``api``) plus the seeded input generators
(``inputs``) used by tests and the benchmark.
"""
from .api import *  # noqa: F401,F403
from .api import (AccuracyError, BlfmmError, BoundingBox, BoxTree, CudaError,  # noqa: F401
                  DomainError, GridMode, InvalidArgument, KernelType, LengthError, LevelGrids,
                  LowRankFactors, Plan, PointSet, QuadratureGrid, RadialKernel, SumRequest,
                  SumResult, SumStats, bandlimited_radial_table, build_tree, choose_truncation,
                  couple, direct_matvec, direct_matvec_hybrid, eval_bandlimited,
                  fmm_matvec_single, make_level_grids, make_quadrature, mlfmm_matvec,
                  parse_kernel_spec, translation_coefficients, upsweep)

__all__ = [n for n in dir() if not n.startswith("_")]
