"""Larger random grids (400-1600 px per side) certified on the GPU box: valid preflow,
cut == seeded residual reach, cut capacity == flow (the oracle solve would be slow)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1110_6231_b200 as fmb

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
# argv[3] = "graph": force the device-side round loop (while-graph, triggers every 2 launches)
# that grids >= 2^23 px use by default
opts = {"pr_graph": 1, "pr_batch": 2} if len(sys.argv) > 3 and sys.argv[3] == "graph" else {}
bad = 0
t0 = time.time()
for case in range(n_cases):
    H, W = int(rng.integers(400, 1600)), int(rng.integers(400, 1600))
    hi = int(rng.choice([1, 3, 30, 100, 100000]))
    caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
    ps, pt = rng.uniform(0.005, 1.0, 2)
    capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < ps)).astype(np.int32)
    capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < pt)).astype(np.int32)
    caps[0][:, -1] = 0; caps[1][:, 0] = 0; caps[2][-1, :] = 0; caps[3][0, :] = 0
    caps += [capS, capT]
    solver = fmb.GridSolver(H, W, options=opts)
    flow, cut, _ = solver.solve_host(caps)
    state = solver.export()
    solver.close()
    code, fl, cc, _ = oracle.grid_certify(caps, state, cut)
    if code != 0 or not (fl == cc == flow):
        bad += 1
        print(f"FAIL case {case}: {H}x{W} hi {hi} code {code} flow {flow} cert {fl} cutcap {cc}", flush=True)
print(f"{n_cases} large grids: {bad} failures, {time.time() - t0:.1f} s", flush=True)
