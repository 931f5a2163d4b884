"""Assignment timing/stats sweep: python scripts/bench_assign.py N [pu|nopu]..."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
n = int(sys.argv[1]); modes = sys.argv[2:] or ["pu"]
ws = {"optical_flow": G.assignment_optical_flow(n, n) if int(round(n ** .5)) ** 2 == n else None,
      "M100": G.assignment_reference(n, 100, n), "M10000": G.assignment_reference(n, 10000, n)}
solver = fmb.AssignmentSolver(n)
for name, w in ws.items():
    if w is None:
        continue
    wd = torch.from_numpy(w).cuda()
    for mode in modes:
        pu = mode == "pu"
        t0 = time.time()
        obj, m, _, st = solver.solve_device(wd, use_price_update=pu)
        torch.cuda.synchronize()
        r = st["reserved"]
        print(f"{name:14s} {mode:5s} obj {obj} ms {st['ms_total']:.2f} wall {1000*(time.time()-t0):.1f} pushes {st['pushes']} "
              f"relabels {st['relabels']} rounds {st['rounds']} tail_rounds {st['pr_sweeps']} tail_ops {r[3]} "
              f"pu {r[1]} pu_iters {r[2]} fixed {r[0]} refines {st['refines']} launches {st['launches']}", flush=True)
