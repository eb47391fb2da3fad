"""B200-native FFT field iteration for two-phase periodic conductors.

Drop-in for the solver path of the reference package ``fftcond``
(arXiv 2001.08289): same public names for the solver surface, with the
fixed-point loops running as fused sm_100a CUDA sweeps behind a C ABI
(``include/fftcond_b200.h``).  d = 2 (reference) and d = 3 (extension).
"""

from .analysis import MisestimationReport, MisestimationRun, misestimation_report, misestimation_reports
from .cell import (
    PhaseMap,
    build_cube_array,
    build_disk_array,
    build_random_medium,
    build_square_array,
    build_uniform,
    load_chi_bits,
    load_raster,
    save_chi_bits,
    save_raster,
    volume_fraction,
)
from .exceptions import (
    BackendError,
    BranchCutError,
    ConfigError,
    ContractError,
    DegenerateParamError,
    IntervalError,
    PoleError,
    RasterParseError,
    SupportError,
)
from .fields import AugmentedField, VectorField
from .scalars import (
    SchemeKind,
    SpectralInterval,
    SubstitutionParams,
    aux_constants,
    inverse_map_t,
    map_t,
    map_z,
    solve_p,
    verify_sigma1,
)
from .solver import (
    ConvergenceHistory,
    HistoryRecord,
    SolveResult,
    SolverConfig,
    TerminationStatus,
    estimate_rate,
    solve,
    solve_basic,
    solve_basic_sub,
    solve_em,
    solve_em_sub,
)

from .spectral import (
    apply_chi_aug,
    apply_local_A,
    equilibrium_residual,
    equilibrium_residual_aug,
    extract_sigma_star,
    extract_sigma_star_aug,
    gamma0,
    gamma0_aug,
    gamma1,
    gamma1_aug,
    inner,
    inner_aug,
    invert_shifted_A,
    norm,
    norm_aug,
    recover_physical_fields,
)

__version__ = "0.1.0"

__all__ = [
    "AugmentedField", "BackendError", "BranchCutError", "ConfigError", "ContractError",
    "ConvergenceHistory", "DegenerateParamError", "HistoryRecord", "IntervalError", "PhaseMap",
    "PoleError", "RasterParseError", "SchemeKind", "SolveResult", "SolverConfig", "SpectralInterval",
    "SubstitutionParams", "SupportError", "TerminationStatus", "VectorField", "build_cube_array",
    "MisestimationReport", "MisestimationRun", "misestimation_report", "misestimation_reports",
    "build_disk_array", "build_random_medium", "build_square_array", "build_uniform", "estimate_rate",
    "map_t", "map_z", "solve", "solve_basic", "solve_basic_sub", "solve_em", "solve_em_sub", "solve_p",
    "volume_fraction", "aux_constants", "inverse_map_t", "verify_sigma1", "apply_chi_aug", "apply_local_A",
    "equilibrium_residual", "equilibrium_residual_aug", "extract_sigma_star", "extract_sigma_star_aug", "gamma0",
    "gamma0_aug", "gamma1", "gamma1_aug", "inner", "inner_aug", "invert_shifted_A", "norm", "norm_aug",
    "recover_physical_fields", "load_chi_bits", "load_raster", "save_chi_bits", "save_raster",
]
