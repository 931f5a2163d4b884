"""Every kernel variant the grid solver can be switched to (options passed to
fm_grid_set_option) stays bit-exact: same flow value and same minimal cut as the
pinned CPU oracle.  Guards the A/B paths (v1/v2 push kernels, sweep-based and
Jacobi BFS, the persistent ring push round, multi-step / fused operations, solo
thresholds, tile pass counts) against rotting behind the defaults."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

pytestmark = pytest.mark.gpu

VARIANTS = {
    "default": {},
    "pr_tile_v2": {"pr_kernel": 0},
    "bfs_sweeps_bits": {"bfs_bits": 1},
    "bfs_jacobi_v1": {"bfs_bits": 0},
    "pr_ring": {"pr_ring": 1},
    "steps2": {"op_steps": 2},
    "fused": {"op_fused": 1},
    "steps2_fused": {"op_steps": 2, "op_fused": 1},
    "solo_never": {"solo_max": 0},
    "solo_always": {"solo_max": 1024},
    "k4": {"k_local_list": 4},
    "k64": {"k_local_list": 64},
    "batch1": {"pr_batch": 1},
    "no_local_relabel": {"local_div": 0},
    "br_rerun": {"br_rerun": 1, "br_cap": 2},
    "no_two_hop": {"two_hop": 0},
    "three_hop": {"two_hop": 2},
    "pr_graph": {"pr_graph": 1},
    "unpacked": {"packed": 0},
    "bfs_from_scratch": {"bfs_incr": 0},
    "bfs_incremental_rerun": {"bfs_incr": 1, "br_rerun": 1},
    "bfs_incremental_no_local": {"bfs_incr": 1, "local_div": 0},
    "pr_graph_b1": {"pr_graph": 1, "pr_batch": 1},
    "pr_graph_b2": {"pr_graph": 1, "pr_batch": 2},
    "no_tma": {"tma": 0},
    "unpacked_no_tma": {"packed": 0, "tma": 0},
    "no_ring_tail": {"ring_tail": 0},
    "ring_tail_every_round": {"ring_tail": 1},
    "bfs_ring_queue": {"bfs_owner": 0},
    "bfs_owner_few_warps": {"br_cap": 1},
}

# the last two are whole-tile grids (H % 32 == 0, W % 128 == 0): the vectorised relabel
# preparation / cut seeding and the inbox fold take their fast paths there
CASES = [("G", 96, 160, 11), ("G", 257, 130, 12), ("S", 200, 256, 2048), ("G", 31, 33, 13),
         ("G", 64, 256, 14), ("S", 128, 384, 2048)]


@pytest.fixture(scope="module")
def expected():
    out = {}
    for kind, H, W, seed in CASES:
        caps = G.grid_random(H, W, seed) if kind == "G" else G.grid_segmentation(H, W, seed)
        want = oracle.grid_maxflow(*caps, solver="seq")
        out[(kind, H, W, seed)] = (caps, want["value"], want["cut"])
    return out


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_bit_exact(name, expected):
    for key, (caps, value, cut) in expected.items():
        H, W = caps[0].shape
        solver = fmb.GridSolver(H, W, options=VARIANTS[name])
        try:
            flow, got_cut, _ = solver.solve_host(caps)
        finally:
            solver.close()
        assert flow == value, (name, key)
        assert (got_cut == cut).all(), (name, key)
