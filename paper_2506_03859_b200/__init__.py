"""B200-native (sm_100a) farPCA blocked adaptive QB loop.

Drop-in for the hot path of the reference's rsvd library (run_fixed_precision /
run_fixed_rank with Gaussian, standardized-Bernoulli, sparse-sign and
sparse-Gaussian test matrices).  The compute path is libfarqb.so
(paper_2506_03859_b200/csrc, C-ABI in include/farqb.h); this package is the
host-side mirror of the reference interface.
"""
from .rsvd import (  # noqa: F401
    AllocError, BlockDegenerate, BlockSource, CallbackError, ConfigError, ConvergenceFailure,
    CudaError, DimensionError, Engine, FarpcaConfig, InvalidArgument, QBResult, RsvdError,
    ShiftConvention, SketchBlock, SketchKind, SketchSpec, ToleranceNotReached, default_block,
    default_density, default_engine, default_max_iters, estimate_cost, gen_sketch,
    relative_error, run_fixed_precision, run_fixed_rank, sketch_kind_from_name, sketch_kind_name, truncate_to_tolerance)

from . import dist  # noqa: F401,E402  (row-sharded multi-GPU helpers)
from .matrix_io import (  # noqa: F401,E402
    FormatError, dumps_mm, dumps_ppm, dumps_raw, load_matrix, load_raw, loads_mm, loads_ppm, loads_raw,
    matrix_format_from_name, matrix_format_name, save_matrix, save_raw)

__all__ = [n for n in dir() if not n.startswith("_")]
from . import experiment  # noqa: F401,E402
