"""CPU oracle for the grid max-flow / assignment hot path -- TEST INFRASTRUCTURE.

This package is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  ``paper_1110_6231_b200`` never imports it
and has no CPU fallback.

``fm_oracle.c`` restates the reference algorithms (file:line cited there):
``solve_maxflow_seq`` (maxflow_seq.py:163-239), ``hybrid_solve``
(maxflow_par.py:157-238, real threads + C11 atomics), ``edmonds_karp``
(oracles.py:20-65), ``solve_assignment`` seq / par
(assign_scaling.py:400-497, assign_par.py:115-237), plus the grid adapter of
SURVEY.md 8d and a cut / optimality certificate.  Parity of the restatement is
pinned against the reference's own outputs in ``tests/golden``
(``tests/test_oracle_golden.py``): values and push/relabel/round counters.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_c = ctypes


def build() -> str:
    """Compile liboracle.so in place (gcc); returns its path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or (
        os.path.exists(os.path.join(_HERE, "fm_oracle.c"))
        and os.path.getmtime(os.path.join(_HERE, "fm_oracle.c")) > os.path.getmtime(_LIB_PATH)
    ):
        build()
    L = ctypes.CDLL(_LIB_PATH)
    L.fmo_maxflow_seq.argtypes = [_c.c_int32, _c.c_int32, _c.c_int32, _c.c_int64,
                                  _i32p, _i32p, _i32p, _c.c_int64, _i64p,
                                  _c.c_void_p, _c.c_void_p]
    L.fmo_maxflow_seq.restype = _c.c_int
    L.fmo_hybrid.argtypes = [_c.c_int32, _c.c_int32, _c.c_int32, _c.c_int64,
                             _i32p, _i32p, _i32p, _c.c_int32, _c.c_int32, _i64p,
                             _c.c_void_p, _c.c_void_p, _c.c_void_p]
    L.fmo_hybrid.restype = _c.c_int
    L.fmo_reach_cut.argtypes = [_c.c_int32, _c.c_int32, _c.c_int32, _c.c_int64,
                                _i32p, _i32p, _i32p, _i64p, _u8p]
    L.fmo_reach_cut.restype = _c.c_int
    L.fmo_edmonds_karp.argtypes = [_c.c_int32, _c.c_int32, _c.c_int32, _c.c_int64,
                                   _i32p, _i32p, _i32p]
    L.fmo_edmonds_karp.restype = _c.c_int64
    L.fmo_grid_arc_count.argtypes = [_c.c_int32, _c.c_int32, _i32p, _i32p]
    L.fmo_grid_arc_count.restype = _c.c_int64
    L.fmo_grid_build_arcs.argtypes = [_c.c_int32, _c.c_int32] + [_i32p] * 9
    L.fmo_grid_build_arcs.restype = _c.c_int64
    L.fmo_grid_certify.argtypes = [_c.c_int32, _c.c_int32] + [_i32p] * 13 + [_u8p, _i64p]
    L.fmo_grid_certify.restype = _c.c_int
    L.fmo_assign.argtypes = [_c.c_int32, _c.c_int64, _i32p, _i32p, _i64p, _c.c_int32,
                             _c.c_int64, _c.c_int64, _c.c_int32, _c.c_int64, _i64p,
                             _i32p, _c.c_void_p]
    L.fmo_assign.restype = _c.c_int
    L.fmo_assign_certify_dense.argtypes = [_c.c_int32, _i32p, _i32p, _c.c_void_p, _i64p]
    L.fmo_assign_certify_dense.restype = _c.c_int
    _lib = L
    return L


def _edges(edges):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 3) if len(edges) else np.zeros((0, 3), np.int64)
    return (np.ascontiguousarray(e[:, 0], dtype=np.int32),
            np.ascontiguousarray(e[:, 1], dtype=np.int32),
            np.ascontiguousarray(e[:, 2], dtype=np.int32))


def _arcs(arcs):
    if isinstance(arcs, tuple):
        return tuple(np.ascontiguousarray(a, dtype=np.int32) for a in arcs)
    return _edges(arcs)


# --------------------------------------------------------------------- max-flow

def maxflow_seq(n, s, t, arcs, heuristic_period=None, want_state=False):
    """solve_maxflow_seq restated.  arcs = list of (tail, head, cap) or a
    (tails, heads, caps) array tuple.  Returns dict(value, pushes, relabels,
    rounds[, residual, excess])."""
    tl, hd, cp = _arcs(arcs)
    m = len(tl)
    out = np.zeros(8, np.int64)
    res = np.zeros(max(1, 2 * m), np.int32) if want_state else None
    ex = np.zeros(n, np.int64) if want_state else None
    rc = lib().fmo_maxflow_seq(n, s, t, m, tl, hd, cp, int(heuristic_period or 0), out,
                               res.ctypes.data if want_state else None,
                               ex.ctypes.data if want_state else None)
    if rc:
        raise RuntimeError(f"oracle maxflow_seq failed rc={rc}")
    d = dict(value=int(out[0]), pushes=int(out[1]), relabels=int(out[2]), rounds=int(out[3]))
    if want_state:
        d["residual"] = res[: 2 * m]
        d["excess"] = ex
    return d


def hybrid(n, s, t, arcs, worker_count=1, cycle_budget=7000, want_state=False):
    """hybrid_solve restated (real threads for worker_count > 1)."""
    tl, hd, cp = _arcs(arcs)
    m = len(tl)
    out = np.zeros(8, np.int64)
    res = np.zeros(max(1, 2 * m), np.int32)
    ex = np.zeros(n, np.int64)
    marked = np.zeros(n, np.uint8)
    rc = lib().fmo_hybrid(n, s, t, m, tl, hd, cp, int(worker_count), int(cycle_budget), out,
                          res.ctypes.data, ex.ctypes.data, marked.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle hybrid failed rc={rc}")
    d = dict(value=int(out[0]), pushes=int(out[1]), relabels=int(out[2]), rounds=int(out[3]),
             excess_total=int(out[4]), cancelled=int(out[5]))
    if want_state:
        d.update(residual=res[: 2 * m], excess=ex, marked=marked)
    return d


def reach_cut(n, s, t, arcs, residual, excess):
    """Seeded residual reach {s} U {e>0}: uint8[n] source side."""
    tl, hd, _ = _arcs(arcs)
    out = np.zeros(n, np.uint8)
    rc = lib().fmo_reach_cut(n, s, t, len(tl), tl, hd,
                             np.ascontiguousarray(residual, dtype=np.int32),
                             np.ascontiguousarray(excess, dtype=np.int64), out)
    if rc:
        raise RuntimeError("oracle reach_cut failed")
    return out


def edmonds_karp(n, s, t, arcs):
    tl, hd, cp = _arcs(arcs)
    return int(lib().fmo_edmonds_karp(n, s, t, len(tl), tl, hd, cp))


# ------------------------------------------------------------------------- grid

def grid_arcs(capR, capL, capD, capU, capS, capT):
    """The SURVEY.md 8d adapter: grid SoA capacities -> reference arc list
    (tails, heads, caps) with s = H*W, t = H*W + 1."""
    H, W = capS.shape
    a = [np.ascontiguousarray(x, dtype=np.int32).reshape(-1) for x in (capR, capL, capD, capU, capS, capT)]
    m = int(lib().fmo_grid_arc_count(H, W, a[4], a[5]))
    tl = np.zeros(max(1, m), np.int32)
    hd = np.zeros(max(1, m), np.int32)
    cp = np.zeros(max(1, m), np.int32)
    k = int(lib().fmo_grid_build_arcs(H, W, *a, tl, hd, cp))
    assert k == m
    return tl[:m], hd[:m], cp[:m]


def grid_maxflow(capR, capL, capD, capU, capS, capT, solver="seq", worker_count=1,
                 cycle_budget=7000):
    """Solve a grid with the restated reference solver.  Returns dict(value,
    cut[H,W] bool, pushes, relabels, rounds)."""
    H, W = capS.shape
    arcs = grid_arcs(capR, capL, capD, capU, capS, capT)
    n, s, t = H * W + 2, H * W, H * W + 1
    if solver == "seq":
        d = maxflow_seq(n, s, t, arcs, want_state=True)
    else:
        d = hybrid(n, s, t, arcs, worker_count, cycle_budget, want_state=True)
    cut = reach_cut(n, s, t, arcs, d["residual"], d["excess"])
    d["cut"] = cut[: H * W].reshape(H, W).astype(bool)
    del d["residual"], d["excess"]
    d.pop("marked", None)
    return d


def grid_certify(caps, state, cut):
    """Check a merged-pair final grid state (dict rR,rL,rD,rU,rT,rS,e) against the
    original capacities and a claimed cut.  Returns (code, flow, cutcap, |S|);
    code 0 = certified maximum flow and minimal source-side cut."""
    capR, capL, capD, capU, capS, capT = caps
    H, W = capS.shape
    f = lambda x: np.ascontiguousarray(x, dtype=np.int32).reshape(-1)
    out = np.zeros(4, np.int64)
    code = lib().fmo_grid_certify(H, W, f(capR), f(capL), f(capD), f(capU), f(capS), f(capT),
                                  f(state["rR"]), f(state["rL"]), f(state["rD"]), f(state["rU"]),
                                  f(state["rT"]), f(state["rS"]), f(state["e"]),
                                  np.ascontiguousarray(cut, dtype=np.uint8).reshape(-1), out)
    return int(code), int(out[0]), int(out[1]), int(out[2])


# ------------------------------------------------------------------- assignment

def assign(n, edges=None, matrix=None, mode="seq", alpha=10, cycle_budget=500000,
           use_price_update=True, use_arc_fix=True, heuristic_every_k=None):
    """solve_assignment restated; mode "par" is the one-worker lock-free refine
    (deterministic).  Returns dict(objective, pushes, relabels, rounds, matching,
    prices) or raises ValueError('infeasible')."""
    if matrix is not None:
        w = np.ascontiguousarray(matrix, dtype=np.int64)
        n = w.shape[0]
        xs = np.repeat(np.arange(n, dtype=np.int32), n)
        ys = np.tile(np.arange(n, dtype=np.int32), n)
        ws = w.reshape(-1).copy()
    else:
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 3)
        xs = np.ascontiguousarray(e[:, 0], dtype=np.int32)
        ys = np.ascontiguousarray(e[:, 1], dtype=np.int32)
        ws = np.ascontiguousarray(e[:, 2], dtype=np.int64)
    out = np.zeros(4, np.int64)
    match = np.zeros(n, np.int32)
    price = np.zeros(2 * n, np.int64)
    flags = (1 if use_price_update else 0) | (2 if use_arc_fix else 0)
    rc = lib().fmo_assign(n, len(xs), xs, ys, ws, 0 if mode == "seq" else 1, alpha,
                          cycle_budget, flags, int(heuristic_every_k or 0), out, match,
                          price.ctypes.data)
    if rc == 1:
        raise ValueError("infeasible")
    if rc:
        raise RuntimeError(f"oracle assign failed rc={rc}")
    return dict(objective=int(out[0]), pushes=int(out[1]), relabels=int(out[2]),
                rounds=int(out[3]), matching=match.tolist(), prices=price)


def assign_certify_dense(w, matching, prices=None):
    """EXACT certificate: 0 = perfect matching with no negative residual cycle (proven
    maximum weight), 1 = not a perfect matching of present pairs, 2 = a negative cycle
    (suboptimal).  prices (2n, scale n + 1) only speed up the Bellman-Ford passes."""
    w = np.ascontiguousarray(w, dtype=np.int32)
    n = w.shape[0]
    out = np.zeros(2, np.int64)
    p = None if prices is None else np.ascontiguousarray(prices, dtype=np.int64)
    code = lib().fmo_assign_certify_dense(n, w, np.ascontiguousarray(matching, dtype=np.int32),
                                          p.ctypes.data if p is not None else None, out)
    return int(code), int(out[0])
