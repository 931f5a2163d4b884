"""Hypothesis batteries on the GPU paths, in the shape of the reference's own
property tests (test_maxflow_par.py:152-164 oracle agreement on random small
networks; test_assign_seq.py brute-force agreement): grid max-flow value and minimal
cut against the pinned sequential oracle, generic networks against Edmonds-Karp and
the seeded-reach cut, dense assignment against brute force."""

from __future__ import annotations

import itertools

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_1110_6231_b200 as fmb

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def grids(draw):
    H = draw(st.integers(1, 70))
    W = draw(st.integers(1, 70))
    hi = draw(st.sampled_from([1, 2, 9, 100, 40000]))
    seed = draw(st.integers(0, 2**31 - 1))
    p_src = draw(st.sampled_from([0.0, 0.05, 0.5, 1.0]))
    p_snk = draw(st.sampled_from([0.0, 0.05, 0.5, 1.0]))
    rng = np.random.default_rng(seed)
    caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
    caps[0][:, -1] = 0
    caps[1][:, 0] = 0
    caps[2][-1, :] = 0
    caps[3][0, :] = 0
    capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < p_src)).astype(np.int32)
    capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < p_snk)).astype(np.int32)
    return caps + [capS, capT]


@SETTINGS
@given(grids())
def test_grid_matches_oracle(caps):
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    assert rep.objective == want["value"]
    assert (rep.cut == want["cut"]).all()


@st.composite
def networks(draw):
    n = draw(st.integers(2, 12))
    m = draw(st.integers(0, 30))
    edges = draw(st.lists(st.tuples(st.integers(0, n - 1), st.integers(0, n - 1), st.integers(0, 20)),
                          min_size=m, max_size=m))
    return n, edges


@SETTINGS
@given(networks())
def test_generic_network_matches_edmonds_karp(case):
    n, edges = case
    want = oracle.edmonds_karp(n, 0, n - 1, edges)
    rep = fmb.hybrid_solve(fmb.build_network(edges, n, 0, n - 1))
    assert rep.objective == want
    d = oracle.maxflow_seq(n, 0, n - 1, edges, want_state=True)
    cut = oracle.reach_cut(n, 0, n - 1, edges, d["residual"], d["excess"]).astype(bool)
    assert (rep.cut == cut).all()


@SETTINGS
@given(st.integers(1, 7).flatmap(lambda n: st.lists(st.lists(st.integers(0, 60), min_size=n, max_size=n),
                                                    min_size=n, max_size=n)))
def test_assignment_matches_brute_force(rows):
    w = np.array(rows, dtype=np.int32)
    n = w.shape[0]
    best = max(sum(int(w[x, p[x]]) for x in range(n)) for p in itertools.permutations(range(n)))
    rep, m = fmb.solve_assignment(w)
    assert rep.objective == best
    assert sorted(m) == list(range(n)) and sum(int(w[x, y]) for x, y in enumerate(m)) == best
