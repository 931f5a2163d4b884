"""Regenerate case K of scripts/stress_grid.py (same seed) and solve it N times with the
current env knobs, certifying each final state."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1110_6231_b200 as fmb

seed, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(seed)
for case in range(K + 1):
    H, W = int(rng.integers(1, 400)), int(rng.integers(1, 400))
    hi = int(rng.choice([1, 2, 5, 30, 100, 5000]))
    caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
    ps, pt = rng.uniform(0.02, 1.0, 2)
    capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < ps)).astype(np.int32)
    capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < pt)).astype(np.int32)
    caps[0][:, -1] = 0; caps[1][:, 0] = 0; caps[2][-1, :] = 0; caps[3][0, :] = 0
    caps += [capS, capT]
want = oracle.grid_maxflow(*caps, solver="seq")
print("case", K, H, W, "hi", hi, "want", want["value"], flush=True)
bad = 0
solver = fmb.GridSolver(H, W)
for r in range(N):
    flow, cut, st = solver.solve_host(caps)
    state = solver.export()
    code, fl, cc, _ = oracle.grid_certify(caps, state, cut)
    ok = flow == want["value"] and (cut == want["cut"]).all()
    if not ok or code != 0:
        bad += 1
        print(f"rep {r}: flow {flow} cert code {code} cert flow {fl} cut cap {cc} rounds {st['rounds']}", flush=True)
print(f"{N} reps: {bad} bad", flush=True)
np.savez_compressed(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", f"case_{seed}_{K}.npz"), *caps)
