"""Sparse assignment (fm_assign_sparse_solve) timings: median of REPS solves per case.
usage: python scripts/sparse_bench.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1110_6231_b200 as fmb

REPS = int(os.environ.get("REPS", "3"))


def case(n, deg, wmax, seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    xs = np.concatenate([np.arange(n), rng.integers(0, n, n * deg)])
    ys = np.concatenate([perm, rng.integers(0, n, n * deg)])
    keys = np.unique(xs.astype(np.int64) * n + ys)
    xs, ys = (keys // n), (keys % n)
    ws = rng.integers(0, wmax + 1, len(xs))
    return fmb.AssignmentInstance(n=n, edges=tuple(zip(xs.tolist(), ys.tolist(), ws.tolist())), complete=False)


for n, deg, wmax in [(4096, 8, 10000), (4096, 64, 10000), (50000, 5, 10000), (200000, 5, 10000), (20000, 20, 100)]:
    inst = case(n, deg, wmax, n + deg)
    ts, devs = [], []
    for _ in range(REPS + 1):
        t0 = time.perf_counter()
        rep, m = fmb.solve_assignment(inst, layout="sparse")
        ts.append(1000 * (time.perf_counter() - t0))
        devs.append(rep.stats.get("ms_total", 0.0))
    st = rep.stats
    print(f"n={n} m={len(inst.edges)} wmax={wmax}: wall {statistics.median(ts[1:]):8.2f} ms, device "
          f"{statistics.median(devs[1:]):8.2f} ms, rounds {st.get('rounds')}, launches {st.get('launches')}, "
          f"objective {rep.objective}", flush=True)
