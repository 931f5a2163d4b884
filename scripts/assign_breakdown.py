"""Where the n=4096 assignment solve time goes (GPU box): per case, total / price
updates / grid-wide rounds (Y phase, X phase, barriers) / single-CTA tail."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cases = {"optical_flow": G.assignment_optical_flow(n, n), "M100": G.assignment_reference(n, 100, n),
         "M10000": G.assignment_reference(n, 10000, n)}
solver = fmb.AssignmentSolver(n)
for name, w in cases.items():
    wd = torch.from_numpy(w).cuda()
    solver.solve_device(wd)
    obj, m, _, st = solver.solve_device(wd)
    r = st["reserved"]
    print(f"{name:12s} total {st['ms_total']:7.2f} ms | price-update {st['ms_bfs']:6.2f} | grid rounds {st['ms_d2h']:6.2f} "
          f"(Y {st['ms_pr_kern']:5.2f} X {st['ms_bfs_kern']:5.2f} sync {st['bytes_bfs']*1e-6:5.2f}) | tail {st['ms_cut']:6.2f} "
          f"| rounds {st['rounds']} tail_rounds {st['pr_sweeps']} refines {st['refines']} pu {r[1]} pu_iters {r[2]} "
          f"pushes {st['pushes']} relabels {st['relabels']} tail_ops {r[3]} launches {st['launches']} "
          f"| pu frontier Y visits {st['cut_sweeps']} pu iteration ms {st['pr_tiles']*1e-6:.2f}", flush=True)
