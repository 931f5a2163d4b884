"""Option sweep of the assignment solver at n = N: median device time of REPS solves.
usage: python scripts/assign_sweep.py N "name=v,name=v" ["..."]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

n = int(sys.argv[1])
cases = {"optical": G.assignment_optical_flow(n, n), "M100": G.assignment_reference(n, 100, n),
         "M10000": G.assignment_reference(n, 10000, n)}
REPS = int(os.environ.get("REPS", "3"))
dev = {k: torch.from_numpy(w).cuda() for k, w in cases.items()}
want = {}
for spec in sys.argv[2:] or [""]:
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in spec.split(",") if kv}
    s = fmb.AssignmentSolver(n, options=opts)
    out = []
    for k, wd in dev.items():
        s.solve_device(wd)
        ts = []
        for _ in range(REPS):
            obj, m, _, st = s.solve_device(wd)
            ts.append(st["ms_total"])
        want.setdefault(k, obj)
        assert obj == want[k], (k, obj, want[k])
        out.append(f"{k} {statistics.median(ts):7.2f} ms (pu {st['ms_bfs']:5.2f}, rounds {st['rounds']})")
    s.close()
    print(f"{spec or 'default':36s} " + " | ".join(out), flush=True)
