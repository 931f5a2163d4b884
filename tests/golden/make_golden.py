"""Generate the golden vectors in tests/golden/*.json from the REFERENCE package.

Run here (the container that has /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every value below is produced by the reference itself (imported read-only from
/root/reference/pkg/src): flow values and push/relabel/round counters of
solve_maxflow_seq and hybrid_solve(worker_count=1), objectives / counters /
matchings of solve_assignment(mode="seq"|"par"), and the minimal source-side
cut read off the reference's final hybrid_solve state through its observer
hook (maxflow_par.py:228-229) with the seeded-reach rule of SURVEY.md 8a-A10.
Instances are stored as generator parameters (+ a checksum of the generated
arrays) or, for hand-written / fixture instances, explicitly.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from collections import deque

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import flowmatch as fm  # noqa: E402  (the reference)
from paper_1110_6231_b200 import generators as G  # noqa: E402


def checksum(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int32).tobytes())
    return h.hexdigest()[:16]


def grid_edges(caps):
    """SURVEY.md 8d adapter, written out plainly (per pixel, row-major)."""
    capR, capL, capD, capU, capS, capT = caps
    H, W = capS.shape
    s, t = H * W, H * W + 1
    edges = []
    for r in range(H):
        for c in range(W):
            p = r * W + c
            if capS[r, c] > 0:
                edges.append((s, p, int(capS[r, c])))
            if capT[r, c] > 0:
                edges.append((p, t, int(capT[r, c])))
            if c + 1 < W:
                edges.append((p, p + 1, int(capR[r, c])))
                edges.append((p + 1, p, int(capL[r, c + 1])))
            if r + 1 < H:
                edges.append((p, p + W, int(capD[r, c])))
                edges.append((p + W, p, int(capU[r + 1, c])))
    return edges, H * W + 2, s, t


def seeded_reach(net, residual, excess):
    """S = residual reach from {s} U {v != t : excess(v) > 0}."""
    n = net.node_count
    ins = [False] * n
    q = deque()
    for v in range(n):
        if v == net.source or (v != net.sink and excess[v] > 0):
            ins[v] = True
            q.append(v)
    while q:
        x = q.popleft()
        for a in net.out_arcs[x]:
            if residual[a] > 0 and not ins[net.head[a]]:
                ins[net.head[a]] = True
                q.append(net.head[a])
    return ins


def ref_hybrid_with_cut(net, wc=1):
    final = {}

    def obs(net_, hybrid, scanned):
        final["residual"] = list(hybrid.state.residual)
        final["excess"] = list(hybrid.state.excess)
        final["excess_total"] = hybrid.excess_total

    rep = fm.hybrid_solve(net, worker_count=wc, observer=obs)
    if "residual" not in final:  # no round ran: the initial preflow is final
        st = fm.ResidualState.fresh(net)
        fm.init_preflow(net, st)
        final["residual"], final["excess"] = st.residual, st.excess
    return rep, seeded_reach(net, final["residual"], final["excess"])


def pack(bits) -> str:
    return np.packbits(np.asarray(bits, dtype=np.uint8)).tobytes().hex()


def maxflow_case(name, edges, n, s, t, hybrid=True):
    net = fm.build_network(edges, n, s, t)
    seq = fm.solve_maxflow_seq(net)
    d = dict(name=name, n=n, s=s, t=t, edges=[list(e) for e in edges], value=seq.objective,
             seq=dict(pushes=seq.pushes, relabels=seq.relabels, rounds=seq.rounds))
    if hybrid:
        hy, cut = ref_hybrid_with_cut(net)
        assert hy.objective == seq.objective
        d["hybrid1"] = dict(pushes=hy.pushes, relabels=hy.relabels, rounds=hy.rounds)
        d["cut"] = pack(cut)
    d["edmonds_karp"] = fm.edmonds_karp(net)
    return d


def main():
    t0 = time.time()
    out = {"generated_by": "tests/golden/make_golden.py", "reference": REF}

    # ---- known answers from the reference's own tests (file:line in the name)
    mf = []
    mf.append(maxflow_case("diamond test_maxflow_par.py:73-77",
                           [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)], 4, 0, 3))
    mf.append(maxflow_case("six-arc test_maxflow_par.py:116-142",
                           [(0, 1, 5), (0, 2, 3), (1, 2, 2), (2, 1, 2), (1, 3, 4), (2, 3, 4)], 4, 0, 3))
    mf.append(maxflow_case("trapped test_maxflow_par.py:80-91", [(0, 1, 1), (1, 3, 1), (0, 2, 5)], 4, 0, 3))
    mf.append(maxflow_case("antiparallel test_maxflow_seq.py:158-160",
                           [(0, 1, 2), (1, 0, 3), (1, 2, 5)], 3, 0, 2))
    mf.append(maxflow_case("disconnected", [(1, 2, 4)], 3, 0, 2))
    fixdir = "/root/reference/pkg/tests/fixtures"
    for fname in ("maxflow_small.max", "maxflow_medium.max", "maxflow_fixed.max"):
        net = fm.parse_dimacs_max(open(os.path.join(fixdir, fname)).read())
        edges = [(net.tail[a], net.head[a], net.capacity[a]) for a in range(0, net.arc_count, 2)]
        mf.append(maxflow_case(f"fixture {fname}", edges, net.node_count, net.source, net.sink))
    out["maxflow"] = mf
    print("maxflow known answers", [c["value"] for c in mf], f"{time.time() - t0:.1f}s")

    # ---- grids (generator G, plus edge cases and a small segmentation instance)
    grids = []
    specs = [("G", 4, 4, 4), ("G", 8, 8, 8), ("G", 16, 16, 16), ("G", 1, 32, 132), ("G", 32, 1, 133),
             ("G", 32, 32, 32), ("G", 24, 40, 2440), ("G", 64, 64, 64), ("S", 64, 64, 2048),
             ("G", 128, 128, 128), ("G", 256, 256, 256)]
    for kind, H, W, seed in specs:
        caps = G.grid_random(H, W, seed) if kind == "G" else G.grid_segmentation(H, W, seed)
        grids.append(grid_case(f"{kind} {H}x{W} seed {seed}", kind, H, W, seed, caps,
                               hybrid=H * W <= 256 * 256))
        print("grid", grids[-1]["name"], grids[-1]["value"], f"{time.time() - t0:.1f}s")
    # edge cases: all capS = 0, all capT = 0, zero neighbour caps
    caps = list(G.grid_random(8, 8, 80))
    caps[4] = np.zeros_like(caps[4])
    grids.append(grid_case("edge capS=0 8x8", "G", 8, 8, 80, caps, mutate="capS=0"))
    caps = list(G.grid_random(8, 8, 81))
    caps[5] = np.zeros_like(caps[5])
    grids.append(grid_case("edge capT=0 8x8", "G", 8, 8, 81, caps, mutate="capT=0"))
    caps = list(G.grid_random(8, 8, 82))
    for k in range(4):
        caps[k] = np.zeros_like(caps[k])
    grids.append(grid_case("edge neighbours=0 8x8", "G", 8, 8, 82, caps, mutate="nbr=0"))
    out["grids"] = grids

    # ---- assignment
    asg = []

    def assign_case(name, matrix=None, inst=None, extra=None):
        if inst is None:
            inst = fm.AssignmentInstance.from_matrix(matrix)
        d = dict(name=name, n=inst.n)
        if extra:
            d.update(extra)
        else:
            d["edges"] = [list(e) for e in inst.edges]
        for mode in ("seq", "par"):
            try:
                rep, m = fm.solve_assignment(inst, mode=mode)
                d[mode] = dict(objective=rep.objective, pushes=rep.pushes, relabels=rep.relabels,
                               rounds=rep.rounds, matching=m)
            except fm.InfeasibleInstanceError:
                d[mode] = "infeasible"
        if inst.n <= fm.ORACLE_SIZE_LIMIT:
            bf = fm.brute_force_assignment(inst)
            d["brute_force"] = None if bf is None else bf[0]
        asg.append(d)
        print("assign", name, d["seq"] if d["seq"] == "infeasible" else d["seq"]["objective"],
              f"{time.time() - t0:.1f}s")

    assign_case("single test_assign_seq.py:167", [[7]])
    assign_case("2x2 test_assign_seq.py:170-173", [[1, 2], [3, 5]])
    assign_case("3x3 test_assign_seq.py:175-181", [[3, 8, 2], [6, 4, 9], [5, 7, 1]])
    assign_case("permutation test_assign_seq.py:199-202", [[9, 1], [1, 9]])
    assign_case("all-equal 4x4", [[5] * 4 for _ in range(4)])
    assign_case("all-zero 3x3", [[0] * 3 for _ in range(3)])
    assign_case("infeasible test_assign_seq.py:205-208", inst=fm.AssignmentInstance.build(2, [(0, 0, 5), (1, 0, 3)]))
    for fname in ("assign_complete_n5.asn", "assign_sparse_n6.asn", "assign_fixed_n8.asn"):
        inst = fm.parse_dimacs_asn(open(os.path.join(fixdir, fname)).read())
        assign_case(f"fixture {fname}", inst=inst)
    for n, M in [(8, 100), (30, 100), (64, 100), (64, 10000), (128, 100), (128, 10000), (256, 100), (256, 10000)]:
        W = G.assignment_reference(n, M, n)
        rec = fm.generate("assignment", n, None, max_value=M, rng_seed=n)
        ref = np.zeros((n, n), np.int64)
        for x, y, w in rec.records:
            ref[x, y] = w
        assert (ref == W).all()
        inst = fm.AssignmentInstance.from_matrix(W.tolist())
        assign_case(f"generate assignment n={n} M={M} seed={n}", inst=inst,
                    extra=dict(generator="assignment_reference", max_value=M, seed=n, checksum=checksum(W)))
    Ws = G.assignment_reference(12, 50, 5, density=0.3)
    rec = fm.generate("assignment", 12, 0.3, max_value=50, rng_seed=5)
    assign_case("generate sparse n=12 d=0.3 seed=5", inst=fm.AssignmentInstance.build(12, rec.records),
                extra=dict(generator="assignment_reference", max_value=50, seed=5, density=0.3,
                           checksum=checksum(Ws)))
    out["assignment"] = asg
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote golden.json in {time.time() - t0:.1f}s")


def grid_case(name, kind, H, W, seed, caps, hybrid=True, mutate=None):
    caps = [np.ascontiguousarray(a, dtype=np.int32) for a in caps]
    edges, n, s, t = grid_edges(caps)
    net = fm.build_network(edges, n, s, t)
    seq = fm.solve_maxflow_seq(net)
    d = dict(name=name, kind=kind, H=H, W=W, seed=seed, mutate=mutate, checksum=checksum(*caps),
             value=seq.objective, seq=dict(pushes=seq.pushes, relabels=seq.relabels, rounds=seq.rounds))
    if hybrid:
        hy, cut = ref_hybrid_with_cut(net)
        assert hy.objective == seq.objective
        d["hybrid1"] = dict(pushes=hy.pushes, relabels=hy.relabels, rounds=hy.rounds)
        d["cut"] = pack(cut[: H * W])
        d["cut_size"] = int(sum(cut[: H * W]))
    return d


if __name__ == "__main__":
    main()
