"""Option sweep of the grid solver: median solve time of REPS solves per option set.
usage: python scripts/grid_sweep.py SIZE KIND "name=v,name=v" ["..."]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

S = int(sys.argv[1])
kind = sys.argv[2]
caps = G.grid_random(S, S, S) if kind == "G" else G.grid_segmentation(S, S, 2048)
dev = [torch.from_numpy(c).cuda() for c in caps]
cut = torch.empty((S, S), dtype=torch.uint8, device="cuda")
REPS = int(os.environ.get("REPS", "5"))
# certified flows (tests/test_grid_gpu.py certificates): every option set must reproduce them
KNOWN = {("G", 4096): 829367847, ("G", 8192): 3318000345, ("G", 2048): None, ("S", 2048): 19312601}
flow0 = KNOWN.get((kind, S))
for spec in sys.argv[3:] or [""]:
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in spec.split(",") if kv}
    solver = fmb.GridSolver(S, S, options=opts)
    solver.solve_device(dev, cut_out=cut)
    sts = []
    for _ in range(REPS):
        f, st = solver.solve_device(dev, cut_out=cut)
        sts.append(st)
        flow0 = f if flow0 is None else flow0
        assert f == flow0, (f, flow0)
    solver.close()
    med = lambda k: statistics.median(s[k] for s in sts)
    print(f"{kind} {S} {spec or 'default':40s} total {med('ms_total'):7.2f} push {med('ms_push'):6.2f} "
          f"(kern {med('ms_pr_kern'):6.2f}) bfs {med('ms_bfs'):6.2f} (kern {med('ms_bfs_kern'):5.2f}) cut {med('ms_cut'):5.2f} "
          f"rounds {med('rounds'):4.0f} ops {(med('pushes') + med('relabels')) / 1e6:6.1f}M launches {med('pr_launches'):4.0f}",
          flush=True)
