"""B200-native hot path of the randomized minimal-norm solver (arXiv 0905.4745).

The package is a thin Python mirror of the reference's interface
(include/minnorm/*.hpp) over the C ABI of ``libminnorm_b200.so``
(include/minnorm_b200.h): sm_100a CUDA kernels for the SRFT sketch, the
fused preconditioned-CG pass and the adjoint transform, cuSOLVER for the
small QR, NCCL for column-sharded multi-GPU runs.
"""
from .api import (apply_adjoint_matrix, ConfigError, Context, DeviceError, DimensionError, LsqConfig, LsqSolution, ProblemInstance,
                  RankDeficiencyError, Sampling, SolveReport, SolverConfig, SrftOperator, UnsupportedError,
                  build_srft, default_context, derive_seed, dft, idft, redistribute_plan, shard_columns, solve_classical,
                  solve_least_squares, solve_randomized, srft_from_fields, ClassicalReport, ParseError,
                  read_matrix_market, read_vector_market, write_matrix_market, generate_instance,
                  GeneratedInstance)

__all__ = [
    "apply_adjoint_matrix", "ConfigError", "Context", "DeviceError", "DimensionError", "LsqConfig", "LsqSolution", "ProblemInstance",
    "RankDeficiencyError", "Sampling", "SolveReport", "SolverConfig", "SrftOperator", "UnsupportedError",
    "build_srft", "default_context", "derive_seed", "dft", "idft", "redistribute_plan", "shard_columns", "solve_classical",
    "solve_least_squares", "solve_randomized", "srft_from_fields", "ClassicalReport", "ParseError",
    "read_matrix_market", "read_vector_market", "write_matrix_market", "generate_instance", "GeneratedInstance",
]
