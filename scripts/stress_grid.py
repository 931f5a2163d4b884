"""Race hunting on the GPU box: many random grids (random shapes / capacity ranges /
terminal densities), each solved several times, every answer checked against the CPU
oracle (flow value and minimal cut).  Prints the number of mismatches (must be 0)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1110_6231_b200 as fmb

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rng = np.random.default_rng(int(sys.argv[3]) if len(sys.argv) > 3 else 1)
bad = 0
t0 = time.time()
for case in range(n_cases):
    H, W = int(rng.integers(1, 400)), int(rng.integers(1, 400))
    hi = int(rng.choice([1, 2, 5, 30, 100, 5000]))
    caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
    ps, pt = rng.uniform(0.02, 1.0, 2)
    capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < ps)).astype(np.int32)
    capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < pt)).astype(np.int32)
    caps[0][:, -1] = 0; caps[1][:, 0] = 0; caps[2][-1, :] = 0; caps[3][0, :] = 0
    caps += [capS, capT]
    want = oracle.grid_maxflow(*caps, solver="seq")
    solver = fmb.GridSolver(H, W)
    for r in range(reps):
        flow, cut, _ = solver.solve_host(caps)
        if flow != want["value"] or not (cut == want["cut"]).all():
            bad += 1
            print(f"MISMATCH case {case} rep {r}: {H}x{W} hi {hi} flow {flow} want {want['value']}", flush=True)
    solver.close()
print(f"{n_cases} cases x {reps} reps: {bad} mismatches, {time.time() - t0:.1f} s", flush=True)
