"""Capacities past the int32 range (the reference's capacities are unbounded Python
ints, graph.py:87-125): grids and generic networks run on the int64 generic kernel
(fm_csr_solve64).  Scaling every capacity by K scales the max flow by K and keeps the
minimal cut, so the int32 solve of the unscaled network (itself pinned to the oracle)
is the exact answer; the returned cut's capacity equals the flow (a certificate)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
from paper_1110_6231_b200.cli import _cut_capacity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W,K", [(64, 48, 2**33), (128, 96, 2**40 + 7), (33, 1, 2**35), (1, 70, 3 * 2**31)])
def test_wide_grid_is_the_scaled_int32_solve(H, W, K):
    caps = G.grid_random(H, W, H * W)
    want = oracle.grid_maxflow(*caps, solver="seq")
    wide = [c.astype(np.int64) * K for c in caps]
    net = fmb.build_grid_network(*wide)
    assert net.wide
    rep = fmb.hybrid_solve(net)
    assert rep.stats["layout"] == "csr64" and rep.stats["residual_bits"] == 64
    assert rep.objective == want["value"] * K
    assert (rep.cut == want["cut"]).all()
    assert _cut_capacity(net, rep.cut) == rep.objective


def test_int32_planes_whose_sums_overflow():
    """Every capacity fits int32 but a pixel's in-flow sum does not: the grid kernel
    refuses its int32 state and the solve moves to the int64 kernel."""
    caps = G.grid_random(96, 80, 3)
    want = oracle.grid_maxflow(*caps, solver="seq")
    K = 2**23
    scaled = [(c.astype(np.int64) * K).astype(np.int32) for c in caps]
    net = fmb.build_grid_network(*scaled)
    assert not net.wide
    rep = fmb.hybrid_solve(net)
    assert rep.stats["layout"] == "csr64"
    assert rep.objective == want["value"] * K and (rep.cut == want["cut"]).all()


def test_wide_grid_mixed_values_certificate():
    rng = np.random.default_rng(9)
    H, W = 80, 64
    caps = [rng.integers(0, 2**40, size=(H, W), dtype=np.int64) for _ in range(6)]
    caps[0][:, -1] = 0
    caps[1][:, 0] = 0
    caps[2][-1, :] = 0
    caps[3][0, :] = 0
    net = fmb.build_grid_network(*caps)
    rep = fmb.hybrid_solve(net)
    assert rep.objective > 2**40
    assert _cut_capacity(net, rep.cut) == rep.objective
    # python-int planes (object arrays) give the same answer
    obj = [np.array(c.tolist(), dtype=object) for c in caps]
    rep2 = fmb.hybrid_solve(fmb.build_grid_network(*obj))
    assert rep2.objective == rep.objective and (rep2.cut == rep.cut).all()


def test_wide_generic_network():
    big = 2**45
    edges = [(0, 1, 3 * big), (0, 2, 2 * big), (1, 2, big), (1, 3, 2 * big + 5), (2, 3, 3 * big), (3, 4, 10 * big)]
    net = fmb.build_network(edges, 5, 0, 4)
    rep = fmb.hybrid_solve(net)
    assert rep.objective == 5 * big
    assert rep.stats["residual_bits"] == 64
    assert rep.cut.tolist() == [True, False, False, False, False]
    small = fmb.build_network([(a, b, c // big) for a, b, c in edges], 5, 0, 4)
    assert fmb.hybrid_solve(small).stats["residual_bits"] == 32


def test_capacities_beyond_the_device_range_raise():
    with pytest.raises(ValueError, match="2\\^62"):
        fmb.hybrid_solve(fmb.build_network([(0, 1, 2**62)], 2, 0, 1))
    with pytest.raises(ValueError, match="2\\^63"):
        fmb.hybrid_solve(fmb.build_network([(0, 1, 2**64)], 2, 0, 1))
    with pytest.raises(ValueError, match="2\\^63"):
        fmb.hybrid_solve(fmb.build_network([(0, 1, 2**61)] * 4 + [(1, 2, 1)], 3, 0, 2))


def test_wide_grid_through_dimacs():
    from paper_1110_6231_b200 import dimacs

    caps = G.grid_random(20, 30, 4)
    K = 2**37
    net = fmb.build_grid_network(*[c.astype(np.int64) * K for c in caps])
    text = dimacs.serialize_network(net)
    g, extra = dimacs.load_max(text)
    assert isinstance(g, fmb.GridNetwork) and g.wide and extra == 0
    want = oracle.grid_maxflow(*caps, solver="seq")["value"] * K
    assert fmb.hybrid_solve(g).objective == want
    assert fmb.hybrid_solve(dimacs.parse_dimacs_max(text)).objective == want
