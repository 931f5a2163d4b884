"""Race hunting for the assignment path (GPU box): random dense and sparse instances of
random size / weight range, each solved twice; the objective must equal scipy's exact
maximum-weight perfect matching and the matching must be a permutation with that weight."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy.optimize import linear_sum_assignment
import paper_1110_6231_b200 as fmb

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ABS = -(2 ** 31)
bad = 0
t0 = time.time()
for case in range(n_cases):
    n = int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 700))]))
    hi = int(rng.choice([1, 3, 100, 10000, 1000000]))
    w = rng.integers(0, hi + 1, size=(n, n)).astype(np.int32)
    sparse = rng.random() < 0.3
    if sparse:   # drop arcs but keep a random perfect matching present
        keep = rng.random((n, n)) < rng.uniform(0.05, 0.5)
        perm = rng.permutation(n)
        keep[np.arange(n), perm] = True
        w = np.where(keep, w, ABS).astype(np.int32)
    cost = np.where(w == ABS, -1e15, w.astype(np.float64))
    r, c = linear_sum_assignment(cost, maximize=True)
    want = int(w[r, c].astype(np.int64).sum())
    for rep_i in range(2):
        tc = time.time()
        rep, m = fmb.solve_assignment(w)
        if time.time() - tc > 2.0:
            print(f"SLOW case {case} rep {rep_i}: n {n} hi {hi} sparse {sparse} {time.time() - tc:.1f} s", flush=True)
        got = int(sum(int(w[x, y]) for x, y in enumerate(m)))
        if rep.objective != want or got != want or sorted(m) != list(range(n)):
            bad += 1
            print(f"MISMATCH case {case} rep {rep_i}: n {n} hi {hi} sparse {sparse} obj {rep.objective} want {want}", flush=True)
print(f"{n_cases} assignment cases: {bad} mismatches, {time.time() - t0:.1f} s", flush=True)
