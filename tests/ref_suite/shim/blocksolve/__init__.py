"""`blocksolve` shim: the reference package's import surface mapped onto
paper_2309_11488_b200, so the reference's own test suite
(/root/reference/pkg/tests, staged by tests/ref_suite/stage.py) runs
unmodified against the B200 build.  Mirrors bs/__init__.py:3-24.
Test infrastructure only."""

from paper_2309_11488_b200 import (  # noqa: F401
    Backend, BlockingError, BlockMatrix, BlockSolveError, BlockVector, BlockView,
    BundleMeta, CopyPlan, DuplicateEntry, GeneratorSpec, Ilu0Factorization,
    IndexOutOfRange, LaneUsage, Layout, MatrixOperator, MissingDiagonal,
    MultisegmentWell, ParallelPlan, ParseError, Partitioning, PlanInvalidated,
    ShapeError, SingularPivot, SingularWellMatrix, SolveFailed, SolveReport,
    SolverConfig, SparsityPattern, StandardWell, StoppingCriteria, Strategy,
    SystemBundle, TooManyPartitions, WellAugmentedOperator, WellMode, WellSet,
    apply_multisegment, apply_permutation, apply_permutation_vec, apply_standard,
    bicgstab, convert_layout, decompose, dot, drop_cross_blocks, extract_pattern,
    fold_into_matrix, generate, graph_color, lane_usage, level_schedule, norm,
    partition, read_system, refresh_values, residual, sequential_plan,
    solve_with_fallback, spmv, transmissibility_weights, write_system)
from paper_2309_11488_b200 import __version__  # noqa: F401
