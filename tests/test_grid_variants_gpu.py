"""Every kernel variant the grid solver can be switched to (env knobs read when a
GridSolver is created) stays bit-exact: same flow value and same minimal cut as the
pinned CPU oracle.  Guards the A/B paths (v1/v2 push kernels, sweep-based and
Jacobi BFS, the persistent ring push round, multi-step / fused operations, solo
thresholds, tile pass counts) against rotting behind the defaults."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

pytestmark = pytest.mark.gpu

VARIANTS = {
    "default": {},
    "pr_tile_v2": {"FM_PR_KERNEL": "0"},
    "bfs_sweeps_bits": {"FM_BFS_BITS": "1"},
    "bfs_jacobi_v1": {"FM_BFS_BITS": "0"},
    "pr_ring": {"FM_PR_RING": "1"},
    "steps2": {"FM_OP_STEPS": "2"},
    "fused": {"FM_OP_FUSED": "1"},
    "steps2_fused": {"FM_OP_STEPS": "2", "FM_OP_FUSED": "1"},
    "solo_never": {"FM_SOLO_MAX": "0"},
    "solo_always": {"FM_SOLO_MAX": "1024"},
    "k4": {"FM_K_LOCAL_LIST": "4"},
    "k64": {"FM_K_LOCAL_LIST": "64"},
    "batch1": {"FM_PR_BATCH": "1"},
    "no_local_relabel": {"FM_LOCAL_DIV": "0"},
    "br_rerun": {"FM_BR_RERUN": "1", "FM_BR_CAP": "2"},
    "no_two_hop": {"FM_TWO_HOP": "0"},
    "three_hop": {"FM_TWO_HOP": "2"},
    "pr_graph": {"FM_PR_GRAPH": "1"},
    "unpacked": {"FM_PACKED": "0"},
    "bfs_from_scratch": {"FM_BFS_INCR": "0"},
    "bfs_incremental_rerun": {"FM_BFS_INCR": "1", "FM_BR_RERUN": "1"},
    "bfs_incremental_no_local": {"FM_BFS_INCR": "1", "FM_LOCAL_DIV": "0"},
    "pr_graph_b1": {"FM_PR_GRAPH": "1", "FM_PR_BATCH": "1"},
}

CASES = [("G", 96, 160, 11), ("G", 257, 130, 12), ("S", 200, 256, 2048), ("G", 31, 33, 13)]


@pytest.fixture(scope="module")
def expected():
    out = {}
    for kind, H, W, seed in CASES:
        caps = G.grid_random(H, W, seed) if kind == "G" else G.grid_segmentation(H, W, seed)
        want = oracle.grid_maxflow(*caps, solver="seq")
        out[(kind, H, W, seed)] = (caps, want["value"], want["cut"])
    return out


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_bit_exact(name, expected, monkeypatch):
    for k, v in VARIANTS[name].items():
        monkeypatch.setenv(k, v)
    for key, (caps, value, cut) in expected.items():
        H, W = caps[0].shape
        solver = fmb.GridSolver(H, W)   # knobs are read here
        try:
            flow, got_cut, _ = solver.solve_host(caps)
        finally:
            solver.close()
        assert flow == value, (name, key)
        assert (got_cut == cut).all(), (name, key)
