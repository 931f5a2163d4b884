"""flowmatch on B200: lock-free push-relabel grid max-flow / min-cut and cost-scaling
dense assignment, as hand-written sm_100a CUDA behind a C ABI (libfm_b200.so).

The public names mirror the reference package ``flowmatch`` for the hot path
(``hybrid_solve``, ``solve_assignment``, ``SolveReport``, ``FlowNetwork``,
``build_network``, ``AssignmentInstance``, ``InfeasibleInstanceError``, ...) so
that callers switch by changing the import.  Grid graphs enter as
:class:`GridNetwork` (structure-of-arrays capacities).
"""

from __future__ import annotations

from . import generators
from .assign import (
    DEFAULT_ALPHA,
    DEFAULT_ASSIGN_CYCLE,
    AssignmentInstance,
    AssignmentSolver,
    InfeasibleInstanceError,
    OpCounters,
    ScalingState,
    arc_fix,
    begin_refine,
    extract_matching,
    make_scaling_state,
    min_cost_loop,
    price_update_heuristic,
    reduce_to_mincost,
    refine_par,
    refine_seq,
    solve_assignment,
)
from .cli import cli_main
from .dimacs import (
    InstanceFile,
    ParseError,
    detect_kind,
    generate,
    load_max,
    parse_dimacs_asn,
    parse_dimacs_max,
    serialize_instance,
    serialize_network,
)
from .graph import (
    FlowNetwork,
    GridNetwork,
    NetworkError,
    ResidualState,
    SolveReport,
    build_grid_network,
    build_network,
    is_epsilon_optimal,
    part_reduced_cost,
    reduced_cost,
)
from .maxflow import DEFAULT_CYCLE_BUDGET, GridSolver, hybrid_solve, hybrid_solve_batch, min_cut

__version__ = "0.1.0"

__all__ = [
    "OpCounters",
    "ResidualState",
    "ScalingState",
    "arc_fix",
    "begin_refine",
    "extract_matching",
    "is_epsilon_optimal",
    "make_scaling_state",
    "min_cost_loop",
    "part_reduced_cost",
    "price_update_heuristic",
    "reduce_to_mincost",
    "reduced_cost",
    "refine_par",
    "refine_seq",
    "AssignmentInstance",
    "AssignmentSolver",
    "DEFAULT_ALPHA",
    "DEFAULT_ASSIGN_CYCLE",
    "DEFAULT_CYCLE_BUDGET",
    "FlowNetwork",
    "GridNetwork",
    "GridSolver",
    "InfeasibleInstanceError",
    "InstanceFile",
    "ParseError",
    "NetworkError",
    "SolveReport",
    "build_grid_network",
    "build_network",
    "cli_main",
    "detect_kind",
    "generate",
    "load_max",
    "parse_dimacs_asn",
    "parse_dimacs_max",
    "serialize_instance",
    "serialize_network",
    "generators",
    "hybrid_solve",
    "hybrid_solve_batch",
    "min_cut",
    "solve_assignment",
    "__version__",
]
