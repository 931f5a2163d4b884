"""Sparse assignment instances (complete=False) in compressed form (fm_assign_sparse_solve,
SURVEY.md 8f-2): the same optimal objective as the reference's golden vectors, scipy's
exact solvers and the dense path, a valid perfect matching over present arcs, and the
reference's infeasibility behaviour."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
from conftest import assign_matrix

pytestmark = pytest.mark.gpu

ABSENT = -(2**31)


def _inst_from_dense(w):
    xs, ys = np.nonzero(w != ABSENT)
    return fmb.AssignmentInstance.build(w.shape[0], [(int(x), int(y), int(w[x, y])) for x, y in zip(xs, ys)])


def _check(inst, rep, m):
    n = inst.n
    assert sorted(m) == list(range(n))
    wmap = {(x, y): w for x, y, w in inst.edges}
    assert all((x, y) in wmap for x, y in enumerate(m))
    assert rep.objective == sum(wmap[(x, y)] for x, y in enumerate(m))


def _scipy_opt(w):
    from scipy.optimize import linear_sum_assignment

    big = np.where(w == ABSENT, -(10**12), w.astype(np.int64))
    r, c = linear_sum_assignment(big, maximize=True)
    return int(big[r, c].sum())


def test_golden_cases_in_compressed_form(golden):
    for case in golden["assignment"]:
        w = assign_matrix(case)
        inst = _inst_from_dense(w)
        if case["par"] == "infeasible":
            with pytest.raises(fmb.InfeasibleInstanceError):
                fmb.solve_assignment(inst, layout="sparse")
            continue
        rep, m = fmb.solve_assignment(inst, layout="sparse")
        assert rep.objective == case["par"]["objective"], case["name"]
        assert rep.stats["layout"] == "sparse"
        _check(inst, rep, m)


@pytest.mark.parametrize("n,M,density,seed", [(20, 100, 0.3, 1), (64, 10000, 0.1, 2), (300, 1000, 0.05, 7),
                                              (1000, 100, 0.01, 3), (1500, 10000, 0.02, 4)])
def test_random_sparse_vs_scipy_and_dense(n, M, density, seed):
    w = G.assignment_reference(n, M, seed, density=density)
    inst = _inst_from_dense(w)
    want = _scipy_opt(w)
    rep, m = fmb.solve_assignment(inst, layout="sparse")
    assert rep.objective == want
    _check(inst, rep, m)
    rep2, _ = fmb.solve_assignment(inst, layout="dense")
    assert rep2.objective == want
    for pu, af in ((False, False), (True, False), (False, True)):
        rep3, m3 = fmb.solve_assignment(inst, layout="sparse", use_price_update=pu, use_arc_fix=af)
        assert rep3.objective == want
        _check(inst, rep3, m3)


def test_auto_layout_picks_compressed_for_sparse():
    w = G.assignment_reference(200, 100, 11, density=0.02)
    inst = _inst_from_dense(w)
    rep, _ = fmb.solve_assignment(inst)           # 2% present: compressed form
    assert rep.stats.get("layout") == "sparse" and rep.objective == _scipy_opt(w)
    full = G.assignment_reference(50, 100, 12)
    rep2, _ = fmb.solve_assignment(fmb.AssignmentInstance.from_matrix(full.tolist()))
    assert rep2.stats.get("layout") != "sparse"  # complete: dense kernels


def test_large_sparse_instance_linear_memory():
    """n = 50,000 with ~6 arcs per node: the dense matrix would be 10 GB; the compressed
    solve needs O(n + m).  Checked against scipy's sparse exact solver."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import min_weight_full_bipartite_matching

    rng = np.random.default_rng(5)
    n, deg = 50_000, 5
    perm = rng.permutation(n)
    xs = np.concatenate([np.arange(n), rng.integers(0, n, n * deg)])
    ys = np.concatenate([perm, rng.integers(0, n, n * deg)])
    keys = np.unique(xs.astype(np.int64) * n + ys)
    xs, ys = (keys // n).astype(np.int64), (keys % n).astype(np.int64)
    ws = rng.integers(0, 10_000, len(xs))
    inst = fmb.AssignmentInstance(n=n, edges=tuple(zip(xs.tolist(), ys.tolist(), ws.tolist())), complete=False)
    rep, m = fmb.solve_assignment(inst)
    assert rep.stats["layout"] == "sparse"
    # scipy minimises: weights w' = C - w (positive) give the same optimal matching
    C = 20_000
    g = csr_matrix(((C - ws).astype(np.float64), (xs, ys)), shape=(n, n))
    r, c = min_weight_full_bipartite_matching(g)
    want = int(n * C - (C - ws)[np.searchsorted(keys, r.astype(np.int64) * n + c)].sum())
    assert rep.objective == want
    assert len(set(m)) == n


def test_infeasible_sparse_instances():
    # a y without arcs
    inst = fmb.AssignmentInstance.build(3, [(0, 0, 1), (1, 0, 2), (2, 1, 3)])
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.solve_assignment(inst, layout="sparse")
    # Hall violation with every node incident to an arc: x0 and x1 both only reach y0
    inst = fmb.AssignmentInstance.build(3, [(0, 0, 1), (1, 0, 2), (2, 1, 3), (2, 2, 4)])
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.solve_assignment(inst, layout="sparse")
