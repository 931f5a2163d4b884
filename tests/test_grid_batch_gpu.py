"""Pipelined batch solve (fm_grid_solve_host_batch / hybrid_solve_batch): every
instance's flow and minimal cut equal the single-call solve's and the oracle's,
whatever the batch length, shape or cut request."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

pytestmark = pytest.mark.gpu


def _nets(H, W, seeds, gen=G.grid_random):
    return [fmb.build_grid_network(*gen(H, W, s)) for s in seeds]


@pytest.mark.parametrize("H,W,count", [(64, 96, 1), (48, 64, 3), (100, 70, 4), (33, 1, 2), (256, 256, 5)])
def test_batch_matches_oracle_and_single_solves(H, W, count):
    seeds = [H * 1000 + W + k for k in range(count)]
    reps = fmb.hybrid_solve_batch(_nets(H, W, seeds))
    assert len(reps) == count
    for k, s in enumerate(seeds):
        caps = G.grid_random(H, W, s)
        want = oracle.grid_maxflow(*caps, solver="seq")
        assert reps[k].objective == want["value"], (k, s)
        assert (reps[k].cut == want["cut"]).all(), (k, s)
        single = fmb.hybrid_solve(fmb.build_grid_network(*caps))
        assert single.objective == reps[k].objective and (single.cut == reps[k].cut).all()


def test_batch_large_grids_match_single_solves():
    """Whole-tile grids on the fast paths (TMA push kernel, owner BFS, ring cut):
    same flow and cut as one call per grid, for a mixed stream (G and S energies)."""
    H = W = 1024
    caps = [G.grid_random(H, W, 11), G.grid_segmentation(H, W, 2048), G.grid_random(H, W, 12)]
    reps = fmb.hybrid_solve_batch([fmb.build_grid_network(*c) for c in caps])
    for c, r in zip(caps, reps):
        single = fmb.hybrid_solve(fmb.build_grid_network(*c))
        assert r.objective == single.objective
        assert (r.cut == single.cut).all()


def test_batch_without_cut_and_empty_batch():
    nets = _nets(40, 40, [1, 2])
    reps = fmb.hybrid_solve_batch(nets, want_cut=False)
    assert all(r.cut is None for r in reps)
    assert [r.objective for r in reps] == [fmb.hybrid_solve(n).objective for n in nets]
    assert fmb.hybrid_solve_batch([]) == []


def test_batch_rejects_mixed_shapes_and_bad_arguments():
    with pytest.raises(ValueError):
        fmb.hybrid_solve_batch(_nets(32, 32, [1]) + _nets(32, 64, [2]))
    with pytest.raises(ValueError):
        fmb.hybrid_solve_batch(_nets(32, 32, [1]), cycle_budget=0)
    solver = fmb.GridSolver(32, 32)
    try:
        with pytest.raises(ValueError):
            solver.solve_host_batch([G.grid_random(32, 32, 1)[:5]])
        with pytest.raises(ValueError):
            solver.solve_host_batch([G.grid_random(16, 32, 1)])
    finally:
        solver.close()


def test_batch_reuses_solver_across_calls():
    """Repeated batch calls on the cached workspace (second input set, cut stages and
    copy streams reused) stay exact."""
    nets = _nets(128, 160, [5, 6, 7])
    first = fmb.hybrid_solve_batch(nets)
    second = fmb.hybrid_solve_batch(nets[::-1])
    for a, b in zip(first, second[::-1]):
        assert a.objective == b.objective and (a.cut == b.cut).all()


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
@pytest.mark.parametrize("H,W", [(33, 7), (64, 96), (512, 512)])
def test_narrow_planes_match_int32(dtype, H, W):
    """uint8 / uint16 host planes cross PCIe narrow and are widened on the device
    (vector body + scalar tail): same flow and cut as the int32 planes, single call and
    batch."""
    caps = [G.grid_random(H, W, 100 + k) for k in range(3)]
    want = [fmb.hybrid_solve(fmb.build_grid_network(*c)) for c in caps]
    nets = [fmb.build_grid_network(*[a.astype(dtype) for a in c]) for c in caps]
    assert all(n.narrow_bytes == np.dtype(dtype).itemsize for n in nets)
    single = fmb.hybrid_solve(nets[0])
    assert single.objective == want[0].objective and (single.cut == want[0].cut).all()
    for r, w in zip(fmb.hybrid_solve_batch(nets), want):
        assert r.objective == w.objective and (r.cut == w.cut).all()


def test_narrow_planes_large_values_uint16():
    """uint16 capacities up to 65535 (packed-residual limits exercised by the int32 path's
    checks) give the int32 planes' result."""
    rng = np.random.default_rng(5)
    H, W = 96, 128
    caps = [rng.integers(0, 65536, size=(H, W)).astype(np.int32) for _ in range(6)]
    caps[0][:, -1] = 0
    caps[1][:, 0] = 0
    caps[2][-1, :] = 0
    caps[3][0, :] = 0
    want = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    got = fmb.hybrid_solve(fmb.build_grid_network(*[a.astype(np.uint16) for a in caps]))
    assert got.objective == want.objective and (got.cut == want.cut).all()
