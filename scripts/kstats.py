"""Per-setting mean of the solve's phase timers (env knob values, solver re-created per value)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
S, kind, reps, knob = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), sys.argv[4]
caps = G.grid_random(S, S, S) if kind == "G" else G.grid_segmentation(S, S, 2048)
dev = [torch.from_numpy(c).cuda() for c in caps]
cut = torch.empty((S, S), dtype=torch.uint8, device="cuda")
keys = ["ms_total", "ms_push", "ms_pr_kern", "ms_bfs", "ms_bfs_kern", "rounds", "pr_launches", "pushes", "relabels"]
for val in sys.argv[5:]:
    os.environ[knob] = val
    sv = fmb.GridSolver(S, S)
    sv.solve_device(dev, cut_out=cut)
    sts = [sv.solve_device(dev, cut_out=cut)[1] for _ in range(reps)]
    sv.close()
    print(f"{kind} {S} {knob}={val}: " + " ".join(f"{k} {statistics.mean(st[k] for st in sts):.4g}" for k in keys if k in sts[0]), flush=True)
