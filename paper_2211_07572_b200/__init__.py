"""B200-native SlabLU engine (arXiv 2211.07572) — dense-mode factorize/solve.

Drop-in for the reference's C++ solver API (assemble_fd5 -> factorize ->
solve); compute runs in hand-written sm_100a kernels behind the C ABI in
include/slablu_gpu.h (libslablu_gpu.so, built in-tree).
"""
from .slablu import (  # noqa: F401
    BlockTridiagonal, CompressionChoice, CompressionError, CompressOptions, CompressStats, ConfigError, Error, ErrorReport, Factorization, GridStrip, ProblemSpec,
    SingularMatrixError, SlabPartition, SweepFactorization, sweep_build, load, import_sweep, SolverConfig, SparseSystem, UnsupportedError, assemble_fd5,
    assemble_canned_device, bessel_j0, choose_b, device_count, error_report, error_report_device, factorize, factorize_device, gaussian_matrix,
    hbs_compress, hbs_compress_adaptive, helmholtz_bump_problem, helmholtz_problem, kappa_from_ppw, partition, poisson_log_problem,
    run_problem, sample_field, sample_solution, sample_solution_device, solve, solve_device, true_solution_helmholtz,
    true_solution_poisson,
)
from ._lib import LIB_PATH, EXPORTS  # noqa: F401
