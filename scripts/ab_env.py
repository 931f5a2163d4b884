"""Assignment A/B over one env knob (solver re-created per value): mean phase times per case."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
n, reps, knob = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
cases = {"optical_flow": G.assignment_optical_flow(n, n), "M100": G.assignment_reference(n, 100, n),
         "M10000": G.assignment_reference(n, 10000, n)}
wds = {k: torch.from_numpy(w).cuda() for k, w in cases.items()}
for val in sys.argv[4:]:
    os.environ[knob] = val
    solver = fmb.AssignmentSolver(n)
    out = []
    for name, wd in wds.items():
        solver.solve_device(wd)
        sts = [solver.solve_device(wd)[3] for _ in range(reps)]
        out.append(f"{name} {statistics.mean(s['ms_total'] for s in sts):.2f} (Y {statistics.mean(s['ms_pr_kern'] for s in sts):.2f} "
                   f"sync {statistics.mean(s['bytes_bfs'] for s in sts)*1e-6:.2f} tail {statistics.mean(s['ms_cut'] for s in sts):.2f})")
    solver.close()
    print(f"n={n} {knob}={val}: " + " | ".join(out), flush=True)
