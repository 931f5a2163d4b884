"""GPU parity of the dense cost-scaling assignment path against the reference's
golden vectors, scipy's exact solver and the epsilon-optimality certificate."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
from conftest import assign_matrix

pytestmark = pytest.mark.gpu


def _objective(w, m):
    return int(sum(int(w[x, y]) for x, y in enumerate(m)))


def _is_perm(m, n):
    return sorted(m) == list(range(n))


def test_golden_assignment(golden):
    for case in golden["assignment"]:
        w = assign_matrix(case)
        n = case["n"]
        if case["seq"] == "infeasible":
            with pytest.raises(fmb.InfeasibleInstanceError):
                fmb.solve_assignment(w)
            continue
        rep, m = fmb.solve_assignment(w)
        assert rep.objective == case["seq"]["objective"], case["name"]
        assert _is_perm(m, n) and _objective(w, m) == rep.objective
        assert all(w[x, y] != -(2**31) for x, y in enumerate(m))


def test_instance_api_and_modes(golden):
    inst = fmb.AssignmentInstance.from_matrix([[3, 8, 2], [6, 4, 9], [5, 7, 1]])
    for mode in ("seq", "par"):
        rep, m = fmb.solve_assignment(inst, mode=mode)
        assert rep.objective == 22 and m == [1, 2, 0]
    for alpha in (2, 5, 100):
        assert fmb.solve_assignment(inst, alpha=alpha)[0].objective == 22
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.solve_assignment(fmb.AssignmentInstance.build(2, [(0, 0, 5), (1, 0, 3)]))


def test_random_small_vs_brute_force():
    rng = np.random.default_rng(11)
    for it in range(200):
        n = int(rng.integers(1, 8))
        hi = int(rng.choice([1, 3, 50, 100]))
        w = rng.integers(0, hi + 1, size=(n, n)).astype(np.int32)
        best = max(sum(int(w[x, p[x]]) for x in range(n)) for p in itertools.permutations(range(n)))
        for fix in (True, False):
            rep, m = fmb.solve_assignment(w, use_arc_fix=fix)
            assert rep.objective == best, (it, n, hi)
            assert _is_perm(m, n) and _objective(w, m) == best


@pytest.mark.parametrize("n,M", [(512, 100), (512, 10000), (1024, 100), (1024, 10000), (1000, 1000)])
def test_vs_scipy_and_certificate(n, M):
    from scipy.optimize import linear_sum_assignment

    w = G.assignment_reference(n, M, n)
    solver = fmb.AssignmentSolver(n)
    obj, m, prices, st = solver.solve_host(w, want_prices=True)
    solver.close()
    r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
    assert obj == int(w[r, c].sum())
    code, cobj = oracle.assign_certify_dense(w, m, prices)
    assert code == 0 and cobj == obj


def test_oracle_port_parity_mid_size():
    w = G.assignment_reference(256, 10000, 256)
    want = oracle.assign(256, matrix=w, mode="seq")
    rep, m = fmb.solve_assignment(w)
    assert rep.objective == want["objective"]


def test_optical_flow_style():
    from scipy.optimize import linear_sum_assignment

    w = G.assignment_optical_flow(1024, 1024)
    rep, m = fmb.solve_assignment(w)
    r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
    assert rep.objective == int(w[r, c].sum())


def test_sparse_feasible_and_infeasible():
    w = G.assignment_reference(40, 100, 3, density=0.1)
    from scipy.optimize import linear_sum_assignment

    big = np.where(w == -(2**31), -10**9, w).astype(np.int64)
    r, c = linear_sum_assignment(big, maximize=True)
    rep, m = fmb.solve_assignment(w)
    assert rep.objective == int(big[r, c].sum())
    bad = np.full((5, 5), -(2**31), np.int32)
    bad[:, 0] = 1
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.solve_assignment(bad)


def test_device_tensor_input():
    torch = pytest.importorskip("torch")
    w = G.assignment_reference(300, 100, 3)
    rep_h, _ = fmb.solve_assignment(w)
    rep_d, m = fmb.solve_assignment(torch.from_numpy(w).cuda())
    assert rep_d.objective == rep_h.objective


def _eps_optimal(view):
    """graph.py:167-186 is_epsilon_optimal on the reference-shaped view."""
    net, st = view.net, view.state
    for a in range(net.arc_count):
        if st.residual[a] <= 0 or view.fixed[a]:
            continue
        rc = net.cost[a] + st.price[net.tail[a]] - st.price[net.head[a]]
        if rc < -view.epsilon:
            return False
    return True


def test_epsilon_optimal_after_every_refine():
    """test_assign_seq.py:210-229 on the GPU refine: the state handed to
    on_refine_end is epsilon-optimal, the last refine runs at epsilon 1."""
    import random

    rng = random.Random(13)
    for _ in range(12):
        n = rng.randint(1, 9)
        matrix = [[rng.randint(0, 100) for _ in range(n)] for _ in range(n)]
        seen = []

        def check(view):
            seen.append(view.epsilon)
            assert _eps_optimal(view)

        rep, m = fmb.solve_assignment(fmb.AssignmentInstance.from_matrix(matrix), on_refine_end=check)
        best = max(sum(matrix[x][p[x]] for x in range(n)) for p in itertools.permutations(range(n)))
        assert seen and seen[-1] == 1 and rep.objective == best


def test_on_refine_end_larger_and_heuristics_off():
    w = G.assignment_reference(64, 10000, 64)
    for pu, af in ((True, True), (False, False)):
        eps = []
        rep, m = fmb.solve_assignment(w, use_price_update=pu, use_arc_fix=af,
                                      on_refine_end=lambda v: (eps.append(v.epsilon), _eps_optimal(v) or pytest.fail("not eps-optimal")))
        want = oracle.assign(64, matrix=w)["objective"]
        assert rep.objective == want and eps[-1] == 1 and eps == sorted(eps, reverse=True)


@pytest.mark.parametrize("n,M", [(999, 100), (1023, 10000), (2048, 10000)])
def test_scalar_path_and_n2048_vs_scipy(n, M):
    """n not a multiple of 4 takes the scalar row-scan path; n = 2048 a mid size."""
    from scipy.optimize import linear_sum_assignment

    w = G.assignment_reference(n, M, n)
    solver = fmb.AssignmentSolver(n)
    obj, m, prices, _ = solver.solve_host(w, want_prices=True)
    solver.close()
    r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
    assert obj == int(w[r, c].sum())
    assert oracle.assign_certify_dense(w, m, prices)[0] == 0


def test_sparse_mid_size_vs_scipy():
    from scipy.optimize import linear_sum_assignment

    w = G.assignment_reference(300, 1000, 7, density=0.05)
    w64 = w.astype(np.int64)
    big = np.where(w64 == -(2**31), -10**12, w64)
    r, c = linear_sum_assignment(big, maximize=True)
    rep, m = fmb.solve_assignment(w)
    assert rep.objective == int(big[r, c].sum())
    assert all(w[x, y] != -(2**31) for x, y in enumerate(m))


@pytest.mark.parametrize("ybatch_min", [1, 1000000])
def test_y_batch_threshold_variants(ybatch_min):
    """The gathered Y op pushes its excess back either unit by unit (an argmin per
    unit) or, from ybatch_min units on, as one rank-ordered batch; both orders are
    the same sequence of reference operations, so objective and matching agree with
    scipy's exact solver either way (option ybatch_min)."""
    from scipy.optimize import linear_sum_assignment
    rng = np.random.default_rng(int(ybatch_min) % 97)
    for n, M in ((300, 10000), (700, 100), (1024, 10)):
        w = rng.integers(0, M + 1, size=(n, n)).astype(np.int32)
        r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
        solver = fmb.AssignmentSolver(n, options={"ybatch_min": ybatch_min})
        try:
            obj, m, _, _ = solver.solve_host(w)
        finally:
            solver.close()
        m = list(m)
        assert obj == int(w[r, c].sum()) and _is_perm(m, n) and _objective(w, m) == obj


@pytest.mark.parametrize("filt", [0, 1])
@pytest.mark.parametrize("ring", [0, 1])
def test_price_update_barrier_and_queue_variants(ring, filt):
    """The price update's label relaxation runs either as barrier-separated waves or
    queue-driven without barriers (option pu_ring), with the full or the filtered
    column scan (option pu_filter); all reach the same
    labels (a fixpoint of min-updates over path lengths), so the optimum and the
    epsilon-optimality certificate hold either way, including sparse instances."""
    from scipy.optimize import linear_sum_assignment
    for n, M in ((1, 5), (7, 3), (64, 10000), (333, 100), (1024, 10000)):
        w = G.assignment_reference(n, M, n + 7)
        solver = fmb.AssignmentSolver(n, options={"pu_ring": ring, "pu_filter": filt})
        try:
            obj, m, prices, _ = solver.solve_host(w, want_prices=True)
        finally:
            solver.close()
        r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
        assert obj == int(w[r, c].sum())
        code, cobj = oracle.assign_certify_dense(w, m, prices)
        assert code == 0 and cobj == obj
    rng = np.random.default_rng(int(ring) + 5)
    n = 400
    w = rng.integers(0, 1000, size=(n, n)).astype(np.int32)
    keep = rng.random((n, n)) < 0.1
    keep[np.arange(n), rng.permutation(n)] = True
    w = np.where(keep, w, -(2**31)).astype(np.int32)
    cost = np.where(w == -(2**31), -1e15, w.astype(np.float64))
    r, c = linear_sum_assignment(cost, maximize=True)
    solver = fmb.AssignmentSolver(n, options={"pu_ring": ring, "pu_filter": filt})
    try:
        obj, m, _, _ = solver.solve_host(w)
    finally:
        solver.close()
    assert obj == int(w[r, c].astype(np.int64).sum()) and sorted(m) == list(range(n))


@pytest.mark.parametrize("opts", [{"round_ctas": 16}, {"round_ctas": 64}, {"pu_groups": 1}, {"pu_groups": 8},
                                  {"pu_groups": 4, "pu_filter": 0}, {"tail_threshold": 8}, {"cta_x": 1, "cta_y": 1}])
def test_refine_launch_shape_variants(opts):
    """Fewer cooperative CTAs, other price-update group counts, a longer single-CTA tail
    (shared-memory lists past TL_CAP spill to the global list) and warp ops for every
    list: the same optimum (scipy) and a valid certificate."""
    from scipy.optimize import linear_sum_assignment
    for n, M in ((64, 10000), (333, 100), (1024, 10000), (1024, 3)):
        w = G.assignment_reference(n, M, n + 11)
        solver = fmb.AssignmentSolver(n, options=opts)
        try:
            obj, m, prices, _ = solver.solve_host(w, want_prices=True)
        finally:
            solver.close()
        r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
        assert obj == int(w[r, c].sum()), (opts, n, M)
        code, cobj = oracle.assign_certify_dense(w, m, prices)
        assert code == 0 and cobj == obj
