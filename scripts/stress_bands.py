"""Race hunting for the row-band path on one GPU (virtual bands): random grids split in
2-4 bands, flow and cut checked against the CPU oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1110_6231_b200 import bands as B

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
t0 = time.time()
for case in range(n_cases):
    nb = int(rng.integers(2, 5))
    H, W = int(rng.integers(66 * nb, 300)), int(rng.integers(1, 300))
    hi = int(rng.choice([1, 3, 30, 100]))
    caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
    ps, pt = rng.uniform(0.02, 1.0, 2)
    capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < ps)).astype(np.int32)
    capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < pt)).astype(np.int32)
    caps[0][:, -1] = 0; caps[1][:, 0] = 0; caps[2][-1, :] = 0; caps[3][0, :] = 0
    caps += [capS, capT]
    want = oracle.grid_maxflow(*caps, solver="seq")
    flow, cut, _ = B.solve_virtual_bands(caps, nb)
    if flow != want["value"] or not (cut == want["cut"]).all():
        bad += 1
        print(f"MISMATCH case {case}: {H}x{W} bands {nb} hi {hi} flow {flow} want {want['value']}", flush=True)
print(f"{n_cases} banded cases: {bad} mismatches, {time.time() - t0:.1f} s", flush=True)
