"""Where does the banded cut differ from the oracle's minimal cut? (stress_bands case)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1110_6231_b200 import bands as B

seed, K = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
for case in range(K + 1):
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
flow, cut, st = B.solve_virtual_bands(caps, nb)
spans = B.band_rows(H, nb)
print("case", K, H, W, "bands", nb, spans, "flow", flow, want["value"])
diff = cut != want["cut"]
rows = np.nonzero(diff.any(axis=1))[0]
print("cut sizes", int(cut.sum()), int(want["cut"].sum()), "differing pixels", int(diff.sum()), "rows", rows[:40].tolist())
print("extra in ours", int((cut & ~want["cut"]).sum()), "missing in ours", int((~cut & want["cut"]).sum()))
