"""GPU generic-graph path (fm_csr.cu): hybrid_solve on arbitrary FlowNetworks.
Mirrors the reference's own batteries: known answers and fixtures
(test_maxflow_par.py, test_io_cli.py), the hypothesis oracle test shape
(test_maxflow_par.py:152-164), the acceptance battery's random graphs and its
1000-repetition stability criterion (test_acceptance.py:269-273)."""

from __future__ import annotations

import random

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from conftest import unpack_cut

pytestmark = pytest.mark.gpu


def test_known_answers_and_fixtures_with_cuts(golden):
    for case in golden["maxflow"]:
        net = fmb.build_network([tuple(e) for e in case["edges"]], case["n"], case["s"], case["t"])
        rep = fmb.hybrid_solve(net, worker_count=2)
        assert rep.objective == case["value"], case["name"]
        assert (rep.cut == unpack_cut(case["cut"], case["n"])).all(), case["name"]


def test_reference_generic_battery_vs_edmonds_karp():
    # test_maxflow_par.py:152-164 shape (n 2..8, m 1..16, caps 0..10), plus the
    # acceptance battery's sizes (n <= 100, m <= 1000, caps <= 100)
    for seed in range(300):
        rng = random.Random(seed)
        if seed < 200:
            n, m, hi = rng.randint(2, 8), rng.randint(1, 16), 10
        else:
            n, m, hi = rng.randint(2, 100), rng.randint(1, 1000), 100
        edges = [(rng.randrange(n), rng.randrange(n), rng.randint(0, hi)) for _ in range(m)]
        net = fmb.build_network(edges, n, 0, n - 1)
        want = oracle.edmonds_karp(n, 0, n - 1, edges)
        rep = fmb.hybrid_solve(net)
        assert rep.objective == want, seed
        d = oracle.maxflow_seq(n, 0, n - 1, edges, want_state=True)
        cut = oracle.reach_cut(n, 0, n - 1, edges, d["residual"], d["excess"]).astype(bool)
        assert (rep.cut == cut).all(), seed


def test_repeated_runs_are_stable(golden):
    case = next(c for c in golden["maxflow"] if c["name"] == "fixture maxflow_fixed.max")
    net = fmb.build_network([tuple(e) for e in case["edges"]], case["n"], case["s"], case["t"])
    values = {fmb.hybrid_solve(net, worker_count=8).objective for _ in range(1000)}
    assert values == {62}


def test_small_cycle_budget_and_trapped_excess():
    net = fmb.build_network([(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)], 4, 0, 3)
    assert fmb.hybrid_solve(net, cycle_budget=1).objective == 5
    net = fmb.build_network([(0, 1, 1), (1, 3, 1), (0, 2, 5)], 4, 0, 3)
    rep = fmb.hybrid_solve(net)
    assert rep.objective == 1 and rep.cut.tolist() == [True, False, True, False]


def test_grid_as_generic_network_agrees_with_grid_kernel():
    from paper_1110_6231_b200 import generators as G

    caps = G.grid_random(40, 30, 4)
    grid = fmb.build_grid_network(*caps)
    rep_grid = fmb.hybrid_solve(grid)
    generic = fmb.FlowNetwork(grid.node_count, grid.source, grid.sink)
    for a, b, c in zip(*[x.tolist() for x in grid.arc_arrays()]):
        generic.add_arc_pair(a, b, c)
    rep = fmb.hybrid_solve(generic)
    assert rep.objective == rep_grid.objective
    assert (rep.cut[: 40 * 30].reshape(40, 30) == rep_grid.cut).all()
