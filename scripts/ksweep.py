"""Repeated solves per setting (env knobs read at solver creation): mean / min of ms_total."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
S, kind, reps = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
knob = sys.argv[4]
caps = G.grid_random(S, S, S) if kind == "G" else G.grid_segmentation(S, S, 2048)
dev = [torch.from_numpy(c).cuda() for c in caps]
cut = torch.empty((S, S), dtype=torch.uint8, device="cuda")
for val in sys.argv[5:]:
    os.environ[knob] = val
    sv = fmb.GridSolver(S, S)
    sv.solve_device(dev, cut_out=cut)
    t = [sv.solve_device(dev, cut_out=cut)[1]["ms_total"] for _ in range(reps)]
    sv.close()
    print(f"{kind} {S} {knob}={val}: mean {statistics.mean(t):.2f} min {min(t):.2f} max {max(t):.2f}", flush=True)
