"""Randomised grid parity beyond the fixed cases: random shapes (odd, non-multiple-of-32,
tall/wide strips), capacity ranges from {0,1} to wide int32 values, sparse sink /
source arcs.  Small instances are compared bit-exactly with the pinned CPU oracle
(flow value and minimal cut); larger ones are certified (valid preflow, cut = seeded
residual reach, cut capacity == flow)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb

pytestmark = pytest.mark.gpu


def _random_caps(rng, H, W, hi, p_src, p_snk):
    caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
    capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < p_src)).astype(np.int32)
    capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < p_snk)).astype(np.int32)
    caps[0][:, -1] = 0
    caps[1][:, 0] = 0
    caps[2][-1, :] = 0
    caps[3][0, :] = 0
    return caps + [capS, capT]


@pytest.mark.parametrize("seed", range(12))
def test_random_shapes_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    H, W = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    hi = int(rng.choice([1, 7, 100, 100000]))
    caps = _random_caps(rng, H, W, hi, float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.05, 1.0)))
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    assert rep.objective == want["value"], (seed, H, W, hi)
    assert (rep.cut == want["cut"]).all(), (seed, H, W, hi)


@pytest.mark.parametrize("seed", range(6))
def test_random_medium_certified(seed):
    rng = np.random.default_rng(2000 + seed)
    H, W = int(rng.integers(300, 1100)), int(rng.integers(300, 1100))
    hi = int(rng.choice([3, 100, 1000000]))
    caps = _random_caps(rng, H, W, hi, float(rng.uniform(0.1, 1.0)), float(rng.uniform(0.1, 1.0)))
    solver = fmb.GridSolver(H, W)
    try:
        flow, cut, _ = solver.solve_host(caps)
        state = solver.export()
    finally:
        solver.close()
    code, fl, cc, _ = oracle.grid_certify(caps, state, cut)
    assert code == 0, (seed, H, W, hi, code)
    assert fl == cc == flow


@pytest.mark.parametrize("shape", [(1, 4097), (4097, 1), (2, 3000), (3000, 3), (33, 1025)])
def test_strips_vs_oracle(shape):
    rng = np.random.default_rng(shape[0] * 7919 + shape[1])
    caps = _random_caps(rng, shape[0], shape[1], 50, 0.5, 0.5)
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    assert rep.objective == want["value"] and (rep.cut == want["cut"]).all()


def _stress_case(seed, k):
    """Case k of scripts/stress_grid.py's generator (same draw order)."""
    rng = np.random.default_rng(seed)
    for _ in range(k + 1):
        H, W = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        hi = int(rng.choice([1, 2, 5, 30, 100, 5000]))
        caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
        ps, pt = rng.uniform(0.02, 1.0, 2)
        capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < ps)).astype(np.int32)
        capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < pt)).astype(np.int32)
        caps[0][:, -1] = 0
        caps[1][:, 0] = 0
        caps[2][-1, :] = 0
        caps[3][0, :] = 0
        caps = caps + [capS, capT]
    return caps


def test_regression_sparse_sink_borders():
    """scripts/stress_grid.py seed 7 case 270 (392 x 353, unit capacities, sparse sink
    arcs): a BFS that queued only the tiles holding a sink arc never revisited a tile
    whose only link to the sink is a sink pixel on its neighbour's border (that value is
    1 from the start, so no change is ever signalled) -- flow 31076 instead of 31077."""
    caps = _stress_case(7, 270)
    want = oracle.grid_maxflow(*caps, solver="seq")
    assert want["value"] == 31077
    for _ in range(3):
        rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
        assert rep.objective == 31077 and (rep.cut == want["cut"]).all()


@pytest.mark.parametrize("seed", range(8))
def test_sparse_sink_grids(seed):
    rng = np.random.default_rng(3000 + seed)
    H, W = int(rng.integers(200, 420)), int(rng.integers(200, 420))
    caps = _random_caps(rng, H, W, int(rng.choice([1, 3])), 0.5, float(rng.choice([0.005, 0.02, 0.05])))
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    assert rep.objective == want["value"] and (rep.cut == want["cut"]).all()


def test_int32_capacity_limits():
    """The device state is int32: capacities whose sums could overflow it (excess of a
    pixel = capS + the capacities into it; a merged pair's residual = its two
    capacities) are refused by the grid kernel with ValueError instead of being wrapped
    silently (hybrid_solve then runs the int64 kernel); below the limit the answer is exact."""
    rng = np.random.default_rng(5)
    H, W = 60, 70

    def caps_upto(hi):
        caps = [rng.integers(0, hi, size=(H, W), dtype=np.int64).astype(np.int32) for _ in range(6)]
        caps[0][:, -1] = 0
        caps[1][:, 0] = 0
        caps[2][-1, :] = 0
        caps[3][0, :] = 0
        return caps

    ok = caps_upto(2**28)
    want = oracle.grid_maxflow(*ok, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*ok))
    assert rep.objective == want["value"] and (rep.cut == want["cut"]).all()
    big = caps_upto(2**31 - 1)
    solver = fmb.GridSolver(H, W)
    try:
        with pytest.raises(ValueError, match="int32 device state"):
            solver.solve_host(big)
    finally:
        solver.close()
    # hybrid_solve moves such grids to the int64 generic kernel (tests/test_wide_caps_gpu.py)
    from paper_1110_6231_b200.cli import _cut_capacity

    net = fmb.build_grid_network(*big)
    rep = fmb.hybrid_solve(net)
    assert rep.stats["layout"] == "csr64" and _cut_capacity(net, rep.cut) == rep.objective


@pytest.mark.parametrize("hi", [32767, 32768, 65535])
def test_packed_residual_boundary(hi):
    """The push kernel packs a pixel's four residuals into 16-bit fields when every
    neighbour pair's two capacities sum to <= 65535 and keeps int32 residuals
    otherwise: capacities at and just past that limit (with pairs saturated at the
    maximum) stay bit-exact on both sides of the switch."""
    rng = np.random.default_rng(hi)
    H, W = 150, 170
    caps = _random_caps(rng, H, W, hi, 0.6, 0.6)
    caps[0][::3, :-1] = hi      # pairs at the maximum sum
    caps[1][::3, 1:] = hi
    caps[2][:-1, ::5] = hi
    caps[3][1:, ::5] = hi
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    assert rep.objective == want["value"] and (rep.cut == want["cut"]).all()


@pytest.mark.parametrize("seed", range(10))
def test_random_whole_tile_grids_vs_oracle(seed):
    """Whole-tile shapes (H % 32 == 0, W % 128 == 0) take the vectorised relabel
    preparation, the inbox fold and the vectorised cut seeding; sparse sink / source
    arcs make long BFS distances and tail rounds (owner BFS, ring tail)."""
    rng = np.random.default_rng(5000 + seed)
    H, W = 32 * int(rng.integers(1, 5)), 128 * int(rng.integers(1, 3))
    hi = int(rng.choice([1, 7, 100, 40000]))
    caps = _random_caps(rng, H, W, hi, float(rng.uniform(0.01, 0.5)), float(rng.uniform(0.01, 0.5)))
    want = oracle.grid_maxflow(*caps, solver="seq")
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    assert rep.objective == want["value"]
    assert (rep.cut == want["cut"]).all()
