"""GPU parity of the grid max-flow / min-cut path (libfm_b200.so) against the
reference's golden vectors and the pinned CPU oracle.  Bit-exact: identical flow
value and identical minimal source-side cut."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
from conftest import grid_caps, unpack_cut

pytestmark = pytest.mark.gpu


def _solve(caps, **kw):
    return fmb.hybrid_solve(fmb.build_grid_network(*caps), **kw)


def test_golden_grids(golden):
    for case in golden["grids"]:
        caps = grid_caps(case)
        rep = _solve(caps)
        assert rep.objective == case["value"], case["name"]
        H, W = case["H"], case["W"]
        if "cut" in case:
            assert (rep.cut.reshape(-1) == unpack_cut(case["cut"], H * W)).all(), case["name"]


def test_edge_cases_match_reference_behaviour(golden):
    by = {c["name"]: c for c in golden["grids"]}
    rep = _solve(grid_caps(by["edge capS=0 8x8"]))
    assert rep.objective == 0 and rep.rounds == 0 and not rep.cut.any()
    rep = _solve(grid_caps(by["edge capT=0 8x8"]))
    assert rep.objective == 0 and rep.cut.all()
    caps = grid_caps(by["edge neighbours=0 8x8"])
    assert _solve(caps).objective == int(np.minimum(caps[4], caps[5]).sum())


def test_random_small_grids_vs_oracle():
    rng = np.random.default_rng(7)
    for it in range(150):
        H, W = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        hi = int(rng.choice([1, 3, 10, 100]))
        caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(6)]
        caps[0][:, -1] = 0
        caps[1][:, 0] = 0
        caps[2][-1, :] = 0
        caps[3][0, :] = 0
        want = oracle.grid_maxflow(*caps, solver="seq")
        rep = _solve(caps)
        assert rep.objective == want["value"], (it, H, W)
        assert (rep.cut == want["cut"]).all(), (it, H, W)


@pytest.mark.parametrize("budget", [1, 3, 7000])
def test_cycle_budget_terminates(budget):
    caps = G.grid_random(24, 40, 2440)
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = _solve(caps, cycle_budget=budget)
    assert rep.objective == want["value"]
    assert (rep.cut == want["cut"]).all()


@pytest.mark.parametrize("shape,seed", [((32, 32), 32), ((61, 47), 5), ((128, 96), 9)])
def test_cancel_violations_flag_same_answer(shape, seed):
    """maxflow_par.py:132-154 as the opt-in pass: same flow AND same minimal cut."""
    caps = G.grid_random(*shape, seed)
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = _solve(caps, cancel_violations=True)
    assert rep.objective == want["value"]
    assert (rep.cut == want["cut"]).all()
    seg = G.grid_segmentation(*shape, seed)
    want = oracle.grid_maxflow(*seg, solver="seq")
    rep = _solve(seg, cancel_violations=True)
    assert rep.objective == want["value"] and (rep.cut == want["cut"]).all()


def test_device_planes_validated_like_host_planes():
    """build_grid_network on CUDA tensors applies the host path's checks (negative
    capacity, arcs leaving the grid), narrows wider integer dtypes after a range
    check, rejects float planes, and solves on the planes' own device."""
    import torch

    caps = [torch.from_numpy(c).cuda() for c in G.grid_random(40, 56, 3)]
    want = oracle.grid_maxflow(*[c.cpu().numpy() for c in caps], solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*[c.to(torch.int64) for c in caps]))
    assert rep.objective == want["value"] and (rep.cut.cpu().numpy() == want["cut"]).all()
    bad = [c.clone() for c in caps]
    bad[0][:, -1] = 2
    with pytest.raises(fmb.NetworkError, match="capR: last column"):
        fmb.build_grid_network(*bad)
    bad = [c.clone() for c in caps]
    bad[3][0, 5] = 1
    with pytest.raises(fmb.NetworkError, match="capU: first row"):
        fmb.build_grid_network(*bad)
    bad = [c.clone() for c in caps]
    bad[5][3, 3] = -4
    with pytest.raises(fmb.NetworkError, match="negative capacity"):
        fmb.build_grid_network(*bad)
    with pytest.raises(fmb.NetworkError, match="must be integers"):
        fmb.build_grid_network(*[c.float() for c in caps])
    big = [c.to(torch.int64) for c in caps]
    big[4][0, 0] = 2**33
    with pytest.raises(fmb.NetworkError, match="does not fit"):
        fmb.build_grid_network(*big)
    with pytest.raises(ValueError, match="device=1"):
        fmb.hybrid_solve(fmb.build_grid_network(*caps), device=1)


def test_observer_invariants():
    """Coordinator-point invariants of the reference's tests
    (test_maxflow_par.py:94-149, test_acceptance.py:71-95) on the GPU state."""
    caps = G.grid_random(12, 10, 5)
    net = fmb.build_grid_network(*caps).materialise()
    seen = []

    def observer(net_, hybrid, scanned):
        res = hybrid.state.residual
        for a in range(0, net_.arc_count, 2):
            assert res[a] + res[a ^ 1] == net_.capacity[a] + net_.capacity[a ^ 1]
        h = hybrid.state.height
        V = net_.node_count
        for a in range(net_.arc_count):
            if res[a] > 0 and scanned[net_.tail[a]] and scanned[net_.head[a]]:
                x, y = net_.tail[a], net_.head[a]
                if x != net_.source and h[x] < V:
                    assert h[x] <= h[y] + 1
        ex = hybrid.state.excess
        live = sum(ex[x] for x in range(V) if x not in (net_.source, net_.sink) and not hybrid.marked[x])
        assert min(ex[: V - 2]) >= 0
        seen.append((ex[net_.sink] + live, hybrid.excess_total))

    rep = fmb.hybrid_solve(net, observer=observer)
    want = oracle.grid_maxflow(*caps, solver="seq")
    assert rep.objective == want["value"]
    assert seen and seen[-1][0] == seen[-1][1]
    assert (rep.cut == want["cut"]).all()


def test_device_tensor_path_matches_host_path():
    torch = pytest.importorskip("torch")
    caps = G.grid_random(100, 130, 9)
    host = _solve(caps)
    dev = [torch.from_numpy(c).cuda() for c in caps]
    rep = fmb.hybrid_solve(fmb.build_grid_network(*dev))
    assert rep.objective == host.objective
    assert (rep.cut.cpu().numpy() == host.cut).all()


@pytest.mark.parametrize("shape,kind", [((512, 512), "G"), ((1024, 1024), "G"), ((512, 768), "S")])
def test_larger_grids_vs_oracle(shape, kind):
    H, W = shape
    caps = G.grid_random(H, W, H) if kind == "G" else G.grid_segmentation(H, W, 2048)
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = _solve(caps)
    assert rep.objective == want["value"]
    assert (rep.cut == want["cut"]).all()


@pytest.mark.parametrize("shape,kind", [((2048, 2048), "S"), ((2048, 2048), "G")])
def test_certificate_at_config_sizes(shape, kind):
    """Sizes where the oracle is slow: certify the GPU's final state (valid
    preflow, cut = seeded residual reach, cut capacity == flow)."""
    H, W = shape
    caps = G.grid_segmentation(H, W, 2048) if kind == "S" else G.grid_random(H, W, H)
    solver = fmb.GridSolver(H, W)
    flow, cut, _ = solver.solve_host(caps)
    st = solver.export()
    code, fl, cc, ns = oracle.grid_certify(caps, st, cut)
    solver.close()
    assert code == 0, code
    assert fl == cc == flow


def test_segmentation_1024_vs_oracle():
    caps = G.grid_segmentation(1024, 1024, 2048)
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = _solve(caps)
    assert rep.objective == want["value"]
    assert (rep.cut == want["cut"]).all()


def test_certificate_at_4096():
    caps = G.grid_random(4096, 4096, 4096)
    solver = fmb.GridSolver(4096, 4096)
    flow, cut, st = solver.solve_host(caps)
    state = solver.export()
    code, fl, cc, ns = oracle.grid_certify(caps, state, cut)
    solver.close()
    assert code == 0 and fl == cc == flow


@pytest.mark.parametrize("H,W", [(1, 1), (1, 5), (7, 1), (33, 65)])
def test_degenerate_shapes(H, W):
    caps = G.grid_random(H, W, H * 100 + W)
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = _solve(caps)
    assert rep.objective == want["value"] and (rep.cut == want["cut"]).all()


def test_certificate_at_8192():
    """Config 3's grid on one GPU: certified maximum flow and minimal cut."""
    caps = G.grid_random(8192, 8192, 8192)
    solver = fmb.GridSolver(8192, 8192)
    flow, cut, st = solver.solve_host(caps)
    state = solver.export()
    code, fl, cc, ns = oracle.grid_certify(caps, state, cut)
    solver.close()
    assert code == 0 and fl == cc == flow
