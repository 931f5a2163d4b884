"""Pin the CPU oracle (oracle/fm_oracle.c) against the reference's own outputs.

Golden values come from the reference package (tests/golden/make_golden.py).
The deterministic oracle entry points must reproduce not only the answers but
the reference's push / relabel / round counters exactly."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import assign_matrix, grid_caps, unpack_cut


def _checksum(*arrays):
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int32).tobytes())
    return h.hexdigest()[:16]


def test_known_maxflow_answers(golden):
    for case in golden["maxflow"]:
        n, s, t = case["n"], case["s"], case["t"]
        arcs = [tuple(e) for e in case["edges"]]
        seq = oracle.maxflow_seq(n, s, t, arcs)
        assert seq["value"] == case["value"], case["name"]
        assert {k: seq[k] for k in ("pushes", "relabels", "rounds")} == case["seq"], case["name"]
        hy = oracle.hybrid(n, s, t, arcs, 1, 7000, want_state=True)
        assert hy["value"] == case["value"]
        assert {k: hy[k] for k in ("pushes", "relabels", "rounds")} == case["hybrid1"], case["name"]
        cut = oracle.reach_cut(n, s, t, arcs, hy["residual"], hy["excess"])
        assert (cut.astype(bool) == unpack_cut(case["cut"], n)).all(), case["name"]
        assert oracle.edmonds_karp(n, s, t, arcs) == case["edmonds_karp"] == case["value"]


def test_known_values_match_reference_tests(golden):
    by = {c["name"].split()[0]: c["value"] for c in golden["maxflow"]}
    assert by["diamond"] == 5 and by["six-arc"] == 8 and by["trapped"] == 1
    assert by["antiparallel"] == 2 and by["disconnected"] == 0
    fx = {c["name"]: c["value"] for c in golden["maxflow"] if c["name"].startswith("fixture")}
    assert fx["fixture maxflow_small.max"] == 14 and fx["fixture maxflow_fixed.max"] == 62


@pytest.mark.parametrize("idx", range(14))
def test_grid_golden(golden, idx):
    if idx >= len(golden["grids"]):
        pytest.skip("no such case")
    case = golden["grids"][idx]
    caps = grid_caps(case)
    assert _checksum(*caps) == case["checksum"], "generator drifted from the golden instance"
    H, W = case["H"], case["W"]
    arcs = oracle.grid_arcs(*caps)
    n, s, t = H * W + 2, H * W, H * W + 1
    seq = oracle.maxflow_seq(n, s, t, arcs)
    assert seq["value"] == case["value"]
    assert {k: seq[k] for k in ("pushes", "relabels", "rounds")} == case["seq"]
    if "hybrid1" in case and H * W <= 128 * 128:
        hy = oracle.hybrid(n, s, t, arcs, 1, 7000, want_state=True)
        assert {k: hy[k] for k in ("pushes", "relabels", "rounds")} == case["hybrid1"]
        cut = oracle.reach_cut(n, s, t, arcs, hy["residual"], hy["excess"])[: H * W].astype(bool)
        assert (cut == unpack_cut(case["cut"], H * W)).all()
    if "cut" in case:
        # the seq solver ends in a true flow; its reach-from-s is the same minimal cut
        d = oracle.grid_maxflow(*caps, solver="seq")
        assert (d["cut"].reshape(-1) == unpack_cut(case["cut"], H * W)).all()


def test_grid_hybrid_threads_agree(golden):
    """Real-thread lock-free rounds (the CPU baseline) give the same value and cut."""
    case = next(c for c in golden["grids"] if c["name"].startswith("G 64x64"))
    caps = grid_caps(case)
    for wc in (2, 4, 8):
        d = oracle.grid_maxflow(*caps, solver="hybrid", worker_count=wc)
        assert d["value"] == case["value"]
        assert (d["cut"].reshape(-1) == unpack_cut(case["cut"], 64 * 64)).all()


def test_assignment_golden(golden):
    from scipy.optimize import linear_sum_assignment

    for case in golden["assignment"]:
        w = assign_matrix(case)
        if "checksum" in case:
            assert _checksum(w) == case["checksum"], case["name"]
        n = case["n"]
        present = w != -(2**31)
        e = np.argwhere(present)
        edges = [(int(x), int(y), int(w[x, y])) for x, y in e] if "edges" not in case else case["edges"]
        for mode in ("seq", "par"):
            want = case[mode]
            if want == "infeasible":
                with pytest.raises(ValueError):
                    oracle.assign(n, edges=edges, mode=mode)
                continue
            got = oracle.assign(n, edges=edges, mode=mode)
            for k in ("objective", "pushes", "relabels", "rounds", "matching"):
                assert got[k] == want[k], (case["name"], mode, k)
        if case["seq"] != "infeasible" and present.all():
            r, c = linear_sum_assignment(w.astype(np.int64), maximize=True)
            assert int(w[r, c].sum()) == case["seq"]["objective"]
        if case.get("brute_force") is not None:
            assert case["brute_force"] == case["seq"]["objective"]


def test_assignment_known_answers(golden):
    by = {c["name"]: c for c in golden["assignment"]}
    assert by["single test_assign_seq.py:167"]["seq"]["objective"] == 7
    assert by["2x2 test_assign_seq.py:170-173"]["seq"]["objective"] == 6
    c3 = by["3x3 test_assign_seq.py:175-181"]["seq"]
    assert c3["objective"] == 22 and c3["matching"] == [1, 2, 0] and c3["rounds"] == 2
    assert by["fixture assign_complete_n5.asn"]["seq"]["objective"] == 410
    assert by["fixture assign_sparse_n6.asn"]["seq"]["objective"] == 366
    assert by["fixture assign_fixed_n8.asn"]["seq"]["objective"] == 695


def test_grid_certificate_accepts_oracle_and_rejects_tampering(golden):
    """The certificate used at sizes the oracle cannot solve: build a merged-pair
    final state from the oracle's separate-pair residuals, certify it, then break it."""
    case = next(c for c in golden["grids"] if c["name"].startswith("G 32x32"))
    caps = grid_caps(case)
    H, W = 32, 32
    arcs = oracle.grid_arcs(*caps)
    n, s, t = H * W + 2, H * W, H * W + 1
    d = oracle.maxflow_seq(n, s, t, arcs, want_state=True)
    tl, hd, cp = arcs
    res = d["residual"]
    flow = cp - res[0::2]   # flow on each input arc
    capR, capL, capD, capU, capS, capT = caps
    st = {k: np.zeros(H * W, np.int64) for k in ("rR", "rL", "rD", "rU", "rT", "rS")}
    for (a, b, c), f in zip(zip(tl, hd, cp), flow):
        if a == s:
            st["rS"][b] += f
        elif b == t:
            st["rT"][a] += c - f
        elif b == a + 1:
            st["rR"][a] += c - f
            st["rL"][b] += f
        elif b == a - 1:
            st["rL"][a] += c - f
            st["rR"][b] += f
        elif b == a + W:
            st["rD"][a] += c - f
            st["rU"][b] += f
        else:
            st["rU"][a] += c - f
            st["rD"][b] += f
    st["e"] = d["excess"][: H * W]
    st = {k: v.reshape(H, W) for k, v in st.items()}
    cut = unpack_cut(case["cut"], H * W)
    code, fl, cc, ns = oracle.grid_certify(caps, st, cut)
    assert code == 0 and fl == cc == case["value"]
    bad = cut.copy()
    bad[np.argmax(~cut)] = True
    assert oracle.grid_certify(caps, st, bad)[0] != 0
    st2 = dict(st)
    st2["rT"] = st["rT"].copy()
    st2["rT"].reshape(-1)[0] += 1
    assert oracle.grid_certify(caps, st2, cut)[0] != 0
