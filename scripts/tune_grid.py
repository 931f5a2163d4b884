"""Tuning sweep for the grid solver (K_LOCAL / BFS_INTERVAL env overrides).
usage: python scripts/tune_grid.py SIZE KIND [KL:BI ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

S = int(sys.argv[1]); kind = sys.argv[2]
cfgs = sys.argv[3:] or ["0:0"]
caps = G.grid_random(S, S, S) if kind == "G" else G.grid_segmentation(S, S, 2048)
dev = [torch.from_numpy(c).cuda() for c in caps]
cut = torch.empty((S, S), dtype=torch.uint8, device="cuda")
keys = ("ms_total", "ms_push", "ms_bfs", "ms_cut", "ms_pr_kern", "ms_bfs_kern", "rounds", "pr_sweeps",
        "pr_tiles", "bfs_sweeps", "bfs_levels", "pushes", "relabels", "cut_sweeps")
for cfg in cfgs:
    kl, bi = cfg.split(":")
    os.environ["FM_K_LOCAL"], os.environ["FM_BFS_INTERVAL"] = kl, bi
    solver = fmb.GridSolver(S, S)
    gs = kl == "global"
    for i in range(int(os.environ.get("REPS", "3"))):
        f, st = solver.solve_device(dev, cut_out=cut, global_sweep=gs)
    print(kind, S, cfg, "flow", f, {k: (round(st[k], 2) if isinstance(st[k], float) else st[k]) for k in keys},
          "bfs_tile_visits_changed", st["reserved"][0], "list_passes", st["reserved"][2], "list_items", st["reserved"][3], flush=True)
    solver.close()
