"""CPU-side checks of the drop-in boundary: names and signatures mirror the
reference, validation behaves like the reference, the grid adapter matches the
oracle's, and libfm_b200.so loads and exports every symbol the header declares.
No compute call is made here (no GPU in this container)."""

from __future__ import annotations

import inspect
import os
import re

import numpy as np
import pytest

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import _lib
from conftest import ROOT, has_gpu


def test_reference_signatures_kept():
    sig = inspect.signature(fmb.hybrid_solve)
    params = list(sig.parameters.values())
    assert [p.name for p in params[:4]] == ["net", "worker_count", "cycle_budget", "observer"]
    assert params[1].default == 4 and params[2].default == 7000 and params[3].default is None
    sig = inspect.signature(fmb.solve_assignment)
    want = dict(mode="seq", worker_count=1, cycle_budget=500000, alpha=10, use_price_update=True,
                use_arc_fix=True, heuristic_every_k=None, validate=False, on_refine_end=None,
                observer=None)
    for k, v in want.items():
        assert sig.parameters[k].default == v, k
        assert sig.parameters[k].kind is inspect.Parameter.KEYWORD_ONLY
    rep = fmb.SolveReport(5)
    assert (rep.objective, rep.pushes, rep.relabels, rep.rounds, rep.elapsed) == (5, 0, 0, 0, 0.0)
    assert issubclass(fmb.NetworkError, ValueError)


def test_build_network_messages():
    with pytest.raises(fmb.NetworkError, match="node_count must be at least 2"):
        fmb.build_network([], 1, 0, 0)
    with pytest.raises(fmb.NetworkError, match="source and sink must differ"):
        fmb.build_network([], 3, 1, 1)
    with pytest.raises(fmb.NetworkError, match="arc 0: negative capacity"):
        fmb.build_network([(0, 1, -1)], 3, 0, 2)
    net = fmb.build_network([(0, 1, 3), (1, 2, 4)], 3, 0, 2)
    assert net.arc_count == 4 and net.out_arcs[1] == [1, 2] and net.reverse_of(2) == 3


def test_grid_network_validation():
    from paper_1110_6231_b200.generators import grid_random

    caps = list(grid_random(4, 5, 1))
    net = fmb.build_grid_network(*caps)
    assert (net.node_count, net.source, net.sink) == (22, 20, 21)
    bad = [c.copy() for c in caps]
    bad[0][:, -1] = 3
    with pytest.raises(fmb.NetworkError, match="capR: last column"):
        fmb.build_grid_network(*bad)
    bad = [c.copy() for c in caps]
    bad[4][0, 0] = -1
    with pytest.raises(fmb.NetworkError, match="negative capacity"):
        fmb.build_grid_network(*bad)
    with pytest.raises(fmb.NetworkError, match="shape"):
        fmb.build_grid_network(caps[0][:3], *caps[1:])


def test_grid_adapter_matches_oracle_and_reference_layout():
    import oracle
    from paper_1110_6231_b200.generators import grid_random

    caps = grid_random(7, 9, 3)
    net = fmb.build_grid_network(*caps)
    mine = net.arc_arrays()
    ref = oracle.grid_arcs(*caps)
    for a, b in zip(mine, ref):
        assert np.array_equal(a, b)
    net.materialise()
    assert net.arc_count == 2 * len(ref[0])
    # arc 2k forward, 2k+1 reverse, as graph.py:71-84
    assert net.capacity[1] == 0 and net.head[1] == net.tail[0]


def test_non_grid_network_needs_the_device():
    net = fmb.build_network([(0, 1, 3), (1, 2, 4)], 3, 0, 2)
    with pytest.raises(ValueError, match="worker_count"):
        fmb.hybrid_solve(net, worker_count=0)
    from paper_1110_6231_b200.maxflow import csr_arrays

    ostart, oarc, head, cap = csr_arrays(net)
    assert ostart.tolist() == [0, 1, 3, 4] and oarc.tolist() == [0, 1, 2, 3]
    assert head.tolist() == [1, 0, 2, 1] and cap.tolist() == [3, 0, 4, 0]
    if not has_gpu() and os.path.exists(_lib.LIB_PATH):
        with pytest.raises(RuntimeError, match="no CUDA device"):
            fmb.hybrid_solve(net)


def test_assignment_instance_validation():
    with pytest.raises(ValueError, match="n must be"):
        fmb.AssignmentInstance.build(0, [])
    with pytest.raises(ValueError, match="x out of range"):
        fmb.AssignmentInstance.build(2, [(5, 0, 1)])
    with pytest.raises(ValueError, match="duplicate edge"):
        fmb.AssignmentInstance.build(2, [(0, 0, 1), (0, 0, 2)])
    inst = fmb.AssignmentInstance.from_matrix([[1, 2], [3, 4]])
    assert inst.complete
    sparse = fmb.AssignmentInstance.build(2, [(0, 0, 1)])
    assert not sparse.complete
    d = sparse.dense()
    assert d[0, 0] == 1 and d[1, 1] == _lib.FM_ABSENT_WEIGHT
    with pytest.raises(ValueError, match="unknown mode"):
        fmb.solve_assignment(inst, mode="fast")


def _header_functions():
    text = open(os.path.join(ROOT, "include", "flowmatch_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z0-9_]+)\s*\(", text)))


def test_capi_exports_every_header_symbol():
    names = _header_functions()
    assert "fm_grid_solve" in names and "fm_assign_solve" in names
    assert sorted(_lib.SIGNATURES) == names
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libfm_b200.so not built (run __graft_entry__.build())")
    L = _lib.load()
    for n in names:
        assert hasattr(L, n), n
    assert b"sm_100a" in L.fm_version()


def test_no_device_is_a_loud_error():
    if has_gpu() or not os.path.exists(_lib.LIB_PATH):
        pytest.skip("a GPU is visible or the library is not built")
    assert _lib.device_count() == 0
    from paper_1110_6231_b200.generators import grid_random

    net = fmb.build_grid_network(*grid_random(4, 4, 1))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        fmb.hybrid_solve(net)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        fmb.solve_assignment(fmb.AssignmentInstance.from_matrix([[1]]))


def test_generators_deterministic():
    from paper_1110_6231_b200 import generators as G

    a = G.grid_random(16, 8, 5)
    b = G.grid_random(16, 8, 5)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert a[0][:, -1].sum() == 0 and a[3][0].sum() == 0
    s = G.grid_segmentation(64, 48, 7)
    assert s[4].min() >= 0 and s[0][:, :-1].min() >= 1
    w = G.assignment_optical_flow(64, 3)
    assert w.shape == (64, 64) and w.dtype == np.int32 and w.max() <= 10000


def test_wide_grid_planes_are_kept_not_wrapped():
    from paper_1110_6231_b200 import generators as G

    caps = [c.astype(np.int64) for c in G.grid_random(8, 6, 1)]
    net = fmb.build_grid_network(*caps)
    assert not net.wide and net.caps[0].dtype == np.int32
    caps[4] = caps[4] * 2**32 + 1
    net = fmb.build_grid_network(*caps)
    assert net.wide and net.caps[4].dtype == np.int64
    with pytest.raises(fmb.NetworkError, match="does not fit in int32"):
        net.host_caps()
    tl, hd, cp = net.arc_arrays()
    assert cp.dtype == np.int64 and int(cp.max()) >= 2**32
    with pytest.raises(fmb.NetworkError, match="integers"):
        fmb.build_grid_network(*[c.astype(np.float64) for c in caps])
    big = [np.array(c.tolist(), dtype=object) for c in caps]
    big[5][0, 0] = 2**70
    with pytest.raises(fmb.NetworkError, match="2\\^63"):
        fmb.build_grid_network(*big)


def test_forward_star_matches_materialised_arc_lists():
    from paper_1110_6231_b200 import generators as G
    from paper_1110_6231_b200.maxflow import _forward_star, csr_arrays

    net = fmb.build_grid_network(*G.grid_random(5, 7, 2))
    tl, hd, cp = net.arc_arrays()
    ostart, oarc, head, cap = _forward_star(net.node_count, tl.astype(np.int64), hd.astype(np.int64), cp)
    net.materialise()
    want = [a for l in net.out_arcs for a in l]
    assert oarc.tolist() == want
    assert head.tolist() == net.head and cap.tolist() == net.capacity
    o2, a2, h2, c2 = csr_arrays(net)
    assert (o2 == ostart).all() and (a2 == oarc).all()


def test_dimacs_max_keeps_wide_capacities():
    from paper_1110_6231_b200 import dimacs

    n, s, t, tl, hd, cp = dimacs.parse_max_arrays("p max 3 2\nn 1 s\nn 3 t\na 1 2 1099511627776\na 2 3 5\n")
    assert cp.dtype == np.int64 and cp.tolist() == [2**40, 5]
    net = dimacs.parse_dimacs_max("p max 3 1\nn 1 s\nn 3 t\na 1 3 9223372036854775807\n")
    assert net.capacity[0] == 2**63 - 1


def test_narrow_host_planes_kept_and_validated():
    """Six uint8 (or uint16) host planes of one dtype are kept narrow (they cross PCIe
    narrow); mixed dtypes are widened to int32; edge checks apply either way."""
    import numpy as np
    import paper_1110_6231_b200 as fmb
    from paper_1110_6231_b200 import generators as G
    from paper_1110_6231_b200.graph import NetworkError
    c = G.grid_random(20, 30, 1)
    n8 = fmb.build_grid_network(*[a.astype(np.uint8) for a in c])
    assert n8.narrow_bytes == 1 and n8.caps[4].dtype == np.uint8
    assert all((a == b).all() for a, b in zip(n8.host_caps(), c))
    assert fmb.build_grid_network(*[a.astype(np.uint16) for a in c]).narrow_bytes == 2
    mixed = fmb.build_grid_network(*([c[0].astype(np.uint8)] + list(c[1:])))
    assert mixed.narrow_bytes == 0 and all(a.dtype == np.int32 for a in mixed.caps)
    bad = [a.astype(np.uint8) for a in c]
    bad[2][-1, 3] = 1
    with pytest.raises(NetworkError):
        fmb.build_grid_network(*bad)
