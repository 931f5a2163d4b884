"""The reference's assignment API beyond solve_assignment, on the GPU path:
make_scaling_state / ScalingState / begin_refine / refine_par / refine_seq /
price_update_heuristic / arc_fix / min_cost_loop / extract_matching, the
per-round observer, validate=True device checks and heuristic_every_k.

The tests are the shapes of the reference's own tests (test_assign_par.py,
test_assign_seq.py), run against paper_1110_6231_b200 instead of flowmatch,
plus n = 4096 parity against scipy and the exact certificate."""

from __future__ import annotations

import itertools
import random

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

pytestmark = pytest.mark.gpu


def _brute(inst):
    n = inst.n
    w = {(x, y): v for x, y, v in inst.edges}
    best = None
    for p in itertools.permutations(range(n)):
        if all((x, p[x]) in w for x in range(n)):
            v = sum(w[(x, p[x])] for x in range(n))
            best = v if best is None else max(best, v)
    return best


# ---- test_assign_seq.py shapes

def test_begin_refine_frozen_single_cell():
    """test_assign_seq.py:65-72."""
    scaling = fmb.make_scaling_state(fmb.AssignmentInstance.from_matrix([[3]]))
    assert scaling.epsilon == 6
    fmb.begin_refine(scaling)
    assert scaling.epsilon == 1
    assert scaling.state.price == [5, 0]
    assert scaling.state.excess == [1, -1]
    assert scaling.state.residual == [1, 0]


def test_begin_refine_epsilon_never_below_one():
    scaling = fmb.make_scaling_state(fmb.AssignmentInstance.from_matrix([[0]]))
    fmb.begin_refine(scaling)
    assert scaling.epsilon == 1
    fmb.begin_refine(scaling)
    assert scaling.epsilon == 1


def _manual(net, inst, supplies, eps, bound):
    state = fmb.ResidualState.fresh(net)
    return fmb.ScalingState(net=net, instance=inst, state=state, supplies=supplies, epsilon=eps, alpha=10,
                            scaled_cost_bound=bound), state


def test_price_update_single_hop_frozen():
    """test_assign_seq.py:99-108 (a caller-built network: costs not multiples of n+1)."""
    net = fmb.FlowNetwork(2, None, None)
    net.add_arc_pair(0, 1, 1, 5)
    scaling, state = _manual(net, fmb.AssignmentInstance.from_matrix([[0]]), [1, -1], 2, 6)
    state.excess = [1, -1]
    assert fmb.is_epsilon_optimal(net, state, 2)
    fmb.price_update_heuristic(scaling)
    assert state.price == [-6, 0]
    assert fmb.is_epsilon_optimal(net, state, 2)


def test_price_update_accumulates_along_multi_hop_paths():
    """test_assign_seq.py:111-128."""
    net = fmb.FlowNetwork(4, None, None)
    net.add_arc_pair(0, 2, 1, 1)
    placed = net.add_arc_pair(0, 3, 1, 0)
    net.add_arc_pair(1, 3, 1, 1)
    scaling, state = _manual(net, fmb.AssignmentInstance.from_matrix([[0, 0], [0, 0]]), [1, 1, -1, -1], 2, 10)
    state.residual[placed] -= 1
    state.residual[placed ^ 1] += 1
    state.excess = [0, 1, -1, 0]
    assert fmb.is_epsilon_optimal(net, state, 2)
    fmb.price_update_heuristic(scaling)
    assert state.price == [-2, -6, 0, -4]
    assert fmb.is_epsilon_optimal(net, state, 2)


def test_price_update_noop_without_deficit_or_active():
    net = fmb.FlowNetwork(2, None, None)
    net.add_arc_pair(0, 1, 1, 5)
    scaling, state = _manual(net, fmb.AssignmentInstance.from_matrix([[0]]), [0, 0], 2, 6)
    fmb.price_update_heuristic(scaling)
    assert state.price == [0, 0]
    state.excess = [1, 0]
    fmb.price_update_heuristic(scaling)
    assert state.price == [0, 0]


def test_arc_fix_threshold_is_strict():
    """test_assign_seq.py:143-152 on a reduce_to_mincost network: the threshold is
    2 n eps and only reduced costs strictly above it freeze."""
    inst = fmb.AssignmentInstance.from_matrix([[0, 0], [0, 0]])
    scaling = fmb.make_scaling_state(inst)
    scaling.epsilon = 2   # threshold 2 * 2 * 2 = 8
    # forward reduced costs 0 + p(x) - p(y): 9 for x0's arcs, 8 for x1's
    scaling.state.price[:] = [9, 8, 0, 0]
    assert fmb.arc_fix(scaling) == 2        # (0,0) and (0,1) at 9 > 8; (1,*) at 8 stay
    assert scaling.fixed == [True] * 4 + [False] * 4
    assert fmb.arc_fix(scaling) == 0


def test_refine_seq_single_cell_frozen():
    scaling = fmb.make_scaling_state(fmb.AssignmentInstance.from_matrix([[3]]))
    counters = fmb.OpCounters()
    fmb.refine_seq(scaling, counters)
    assert scaling.epsilon == 1
    assert scaling.state.excess == [0, 0]
    assert counters.pushes == 1 and counters.relabels == 0
    assert fmb.extract_matching(scaling) == [0]


def test_solve_frozen_values_and_rounds():
    """test_assign_seq.py:166-181: rounds = refines (two at max weight 9, n = 3)."""
    rep, m = fmb.solve_assignment(fmb.AssignmentInstance.from_matrix([[7]]))
    assert (rep.objective, m) == (7, [0])
    rep, m = fmb.solve_assignment(fmb.AssignmentInstance.from_matrix([[1, 2], [3, 5]]))
    assert (rep.objective, m) == (6, [0, 1])
    for mode in ("seq", "par"):
        rep, m = fmb.solve_assignment(fmb.AssignmentInstance.from_matrix([[3, 8, 2], [6, 4, 9], [5, 7, 1]]),
                                      mode=mode)
        assert rep.objective == 22 and m == [1, 2, 0] and rep.rounds == 2


def test_epsilon_optimal_after_every_refine_validate():
    """test_assign_seq.py:210-229 with validate=True (device invariant checks on)."""
    rng = random.Random(13)
    for _ in range(8):
        n = rng.randint(1, 6)
        matrix = [[rng.randint(0, 100) for _ in range(n)] for _ in range(n)]
        checked = []

        def check(scaling):
            checked.append(scaling.epsilon)
            assert fmb.is_epsilon_optimal(scaling.net, scaling.state, scaling.epsilon, scaling.fixed)

        for mode in ("seq", "par"):
            checked.clear()
            rep, _ = fmb.solve_assignment(fmb.AssignmentInstance.from_matrix(matrix), mode=mode, validate=True,
                                          on_refine_end=check)
            assert checked and checked[-1] == 1
            assert checked == sorted(checked, reverse=True)
            assert rep.objective == _brute(fmb.AssignmentInstance.from_matrix(matrix))


# ---- test_assign_par.py shapes

def test_refine_par_noop_when_already_matched():
    scaling = fmb.make_scaling_state(fmb.AssignmentInstance.from_matrix([[2, 7], [6, 1]]))
    while True:
        fmb.refine_seq(scaling)
        if scaling.epsilon == 1:
            break
    price = list(scaling.state.price)
    residual = list(scaling.state.residual)
    fixed = list(scaling.fixed)
    counters = fmb.OpCounters()
    fmb.refine_par(scaling, counters=counters)
    assert counters.rounds == 0
    assert scaling.state.price == price
    assert scaling.state.residual == residual
    assert scaling.fixed == fixed


def test_refine_par_completes_single_refine():
    scaling = fmb.make_scaling_state(fmb.AssignmentInstance.from_matrix([[3]]))
    fmb.begin_refine(scaling)
    counters = fmb.OpCounters()
    fmb.refine_par(scaling, worker_count=2, counters=counters)
    assert counters.rounds >= 1
    assert scaling.state.excess == [0, 0]
    assert fmb.extract_matching(scaling) == [0]


def test_par_matches_seq_objective():
    rng = random.Random(23)
    for _ in range(10):
        n = rng.randint(1, 7)
        matrix = [[rng.randint(0, 100) for _ in range(n)] for _ in range(n)]
        inst = fmb.AssignmentInstance.from_matrix(matrix)
        want = fmb.solve_assignment(inst)[0].objective
        assert want == _brute(inst)
        for wc in (1, 2, 4):
            assert fmb.solve_assignment(inst, mode="par", worker_count=wc)[0].objective == want


@pytest.mark.parametrize("every_k", [None, 1, 2])
def test_forced_multi_round_schedules_stay_exact(every_k):
    """cycle_budget=1: one Y/X phase pair per coordinator round, so the price update
    fires mid-refine on states with placed flow (test_assign_par.py:83-101), through
    min_cost_loop's coordinator loop with a per-round observer."""
    rng = random.Random(29)
    for _ in range(12):
        n = rng.randint(1, 6)
        matrix = [[rng.randint(0, 100) for _ in range(n)] for _ in range(n)]
        inst = fmb.AssignmentInstance.from_matrix(matrix)
        want = _brute(inst)
        rounds = []
        rep, m = fmb.solve_assignment(inst, mode="par", worker_count=1, cycle_budget=1,
                                      heuristic_every_k=every_k, observer=lambda s: rounds.append(s.epsilon))
        assert rep.objective == want and sorted(m) == list(range(n))
        assert rounds and rounds[-1] == 1 and rep.rounds >= len(set(rounds))
        # the fused path with the same every-k schedule
        assert fmb.solve_assignment(inst, mode="par", cycle_budget=1, heuristic_every_k=every_k)[0].objective == want


def test_forced_multi_round_larger_instances_vs_scipy():
    from scipy.optimize import linear_sum_assignment

    for n, M, k in ((48, 10000, 1), (96, 100, 3), (130, 1000, None)):
        w = G.assignment_reference(n, M, n)
        inst = fmb.AssignmentInstance.from_matrix(w.tolist())
        seen = []
        rep, m = fmb.solve_assignment(inst, mode="par", cycle_budget=2, heuristic_every_k=k, validate=True,
                                      observer=lambda s: seen.append(s.epsilon))
        r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
        assert rep.objective == int(w[r, c].sum()) and len(seen) > 1


def test_par_epsilon_optimal_at_refine_ends():
    rng = random.Random(31)
    for _ in range(6):
        n = rng.randint(1, 6)
        matrix = [[rng.randint(0, 100) for _ in range(n)] for _ in range(n)]

        def check(scaling):
            assert fmb.is_epsilon_optimal(scaling.net, scaling.state, scaling.epsilon, scaling.fixed)

        fmb.solve_assignment(fmb.AssignmentInstance.from_matrix(matrix), mode="par", worker_count=2,
                             validate=True, on_refine_end=check)


def test_par_infeasible_instance_raises():
    inst = fmb.AssignmentInstance.build(2, [(0, 0, 5), (1, 0, 3)])
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.solve_assignment(inst, mode="par", worker_count=2)
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.solve_assignment(inst, mode="par", observer=lambda s: None)
    scaling = fmb.make_scaling_state(inst)
    with pytest.raises(fmb.InfeasibleInstanceError):
        fmb.min_cost_loop(scaling, mode="par")


def test_par_sparse_feasible_instance():
    inst = fmb.AssignmentInstance.build(3, [(0, 1, 4), (1, 0, 2), (1, 2, 7), (2, 2, 5), (2, 0, 1)])
    want = _brute(inst)
    for wc in (1, 2, 4):
        got, matching = fmb.solve_assignment(inst, mode="par", worker_count=wc)
        assert got.objective == want and sorted(matching) == [0, 1, 2]
        got, matching = fmb.solve_assignment(inst, mode="par", worker_count=wc, observer=lambda s: None)
        assert got.objective == want and sorted(matching) == [0, 1, 2]


def test_par_observer_fires_each_round():
    rounds = []
    fmb.solve_assignment(fmb.AssignmentInstance.from_matrix([[3, 8, 2], [6, 4, 9], [5, 7, 1]]), mode="par",
                         worker_count=2, observer=lambda scaling: rounds.append(scaling.epsilon))
    assert rounds and rounds[-1] == 1


def test_min_cost_loop_modes_and_counters():
    """min_cost_loop (assign_scaling.py:400-467): seq counts one round per refine,
    par counts coordinator rounds; both reach the brute-force optimum, and the
    caller's ScalingState ends at epsilon 1 holding the matching."""
    rng = random.Random(41)
    for _ in range(6):
        n = rng.randint(2, 7)
        matrix = [[rng.randint(0, 1000) for _ in range(n)] for _ in range(n)]
        inst = fmb.AssignmentInstance.from_matrix(matrix)
        want = _brute(inst)
        ends = []
        sc = fmb.make_scaling_state(inst)
        rep, m = fmb.min_cost_loop(sc, mode="seq", on_refine_end=lambda s: ends.append(s.epsilon))
        assert rep.objective == want and rep.rounds == len(ends) and sc.epsilon == 1
        assert fmb.extract_matching(sc) == m
        sc = fmb.make_scaling_state(inst)
        rep, m = fmb.min_cost_loop(sc, mode="par", cycle_budget=1)
        assert rep.objective == want and rep.rounds >= len(ends)


def test_stepwise_matches_fused_path():
    """begin_refine + refine_par driven from the host refine by refine reaches the
    same optimum as the fused device solve."""
    w = G.assignment_reference(200, 10000, 7)
    inst = fmb.AssignmentInstance.from_matrix(w.tolist())
    sc = fmb.make_scaling_state(inst)
    counters = fmb.OpCounters()
    while True:
        fmb.begin_refine(sc)
        fmb.refine_par(sc, counters=counters)
        assert fmb.is_epsilon_optimal(sc.net, sc.state, sc.epsilon, sc.fixed)
        if sc.epsilon == 1:
            break
    m = fmb.extract_matching(sc)
    obj = int(sum(w[x, m[x]] for x in range(200)))
    assert obj == fmb.solve_assignment(w)[0].objective


# ---- config 5 (n = 4096) parity and the exact certificate

@pytest.mark.parametrize("case", ["optical_flow", "generate_M100", "generate_M10000"])
def test_n4096_vs_scipy_and_exact_certificate(case):
    """BASELINE.json config 5 at its full size: the objective equals scipy's exact
    linear_sum_assignment, the matching is a permutation of present pairs, and the
    GPU certificate (no negative residual cycle) proves it optimal."""
    from scipy.optimize import linear_sum_assignment

    n = 4096
    w = {"optical_flow": lambda: G.assignment_optical_flow(n, n),
         "generate_M100": lambda: G.assignment_reference(n, 100, n),
         "generate_M10000": lambda: G.assignment_reference(n, 10000, n)}[case]()
    solver = fmb.AssignmentSolver(n)
    try:
        obj, m, prices, _ = solver.solve_host(w, want_prices=True)
        status, cobj, passes = solver.certify(w, m, prices)
    finally:
        solver.close()
    r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
    assert obj == int(w[r, c].astype(np.int64).sum())
    assert sorted(m.tolist()) == list(range(n))
    assert status == 1 and cobj == obj, (status, passes)
    want = {"optical_flow": 40790923, "generate_M100": 409600, "generate_M10000": 40945732}[case]
    assert obj == want


def test_certificate_rejects_suboptimal_and_non_matchings():
    """The certificate is exact: on small instances it agrees with brute force for
    EVERY permutation, and it flags non-matchings."""
    rng = np.random.default_rng(3)
    solver = fmb.AssignmentSolver(5)
    try:
        for _ in range(20):
            w = rng.integers(0, 30, (5, 5)).astype(np.int32)
            best = max(sum(int(w[x, p[x]]) for x in range(5)) for p in itertools.permutations(range(5)))
            for p in itertools.permutations(range(5)):
                status, obj, _ = solver.certify(w, list(p))
                assert (status == 1) == (obj == best)
        assert solver.certify(w, [0, 0, 1, 2, 3])[0] == -1
        w2 = w.copy()
        w2[0, 0] = -(2**31)
        assert solver.certify(w2, [0, 1, 2, 3, 4])[0] == -1
    finally:
        solver.close()


def test_oracle_certificate_matches_gpu_certificate():
    rng = np.random.default_rng(11)
    for n in (7, 33, 130):
        w = rng.integers(0, 50, (n, n)).astype(np.int32)
        rep, m = fmb.solve_assignment(w)
        solver = fmb.AssignmentSolver(n)
        try:
            status, obj, _ = solver.certify(w, m)
            perm = rng.permutation(n)
            s2, o2, _ = solver.certify(w, perm)
        finally:
            solver.close()
        assert status == 1 and obj == rep.objective and oracle.assign_certify_dense(w, m)[0] == 0
        assert (s2 == 1) == (oracle.assign_certify_dense(w, perm)[0] == 0)


def test_device_weight_tensor_validated():
    import torch

    w = G.assignment_reference(64, 100, 3)
    want = fmb.solve_assignment(w)[0].objective
    assert fmb.solve_assignment(torch.from_numpy(w.astype(np.int64)).cuda())[0].objective == want
    with pytest.raises(ValueError, match="square"):
        fmb.solve_assignment(torch.zeros((4, 5), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="integers"):
        fmb.solve_assignment(torch.zeros((4, 4), dtype=torch.float32, device="cuda"))
    big = torch.zeros((4, 4), dtype=torch.int64, device="cuda")
    big[0, 0] = 2**40
    with pytest.raises(ValueError, match="int32"):
        fmb.solve_assignment(big)
    with pytest.raises(ValueError, match="device=1"):
        fmb.solve_assignment(torch.from_numpy(w).cuda(), device=1)
    nc = torch.from_numpy(np.ascontiguousarray(w.T)).cuda().t()   # non-contiguous view of w
    assert fmb.solve_assignment(nc)[0].objective == want


def test_concurrent_threads_share_cache_safely():
    """Two threads solving the same shapes at once (ctypes releases the GIL): each
    solve holds its workspace, a busy one is never shared."""
    import threading

    caps = G.grid_random(96, 128, 5)
    want = oracle.grid_maxflow(*caps, solver="seq")["value"]
    w = G.assignment_reference(128, 1000, 5)
    wantw = fmb.solve_assignment(w)[0].objective
    errors = []

    def work():
        try:
            for _ in range(6):
                assert fmb.hybrid_solve(fmb.build_grid_network(*caps)).objective == want
                assert fmb.solve_assignment(w)[0].objective == wantw
        except BaseException as exc:   # noqa: BLE001
            errors.append(exc)

    th = [threading.Thread(target=work) for _ in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
