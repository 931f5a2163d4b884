"""Per-round trace of one grid solve (library option trace=1 prints a stderr line per
round).  usage: python scripts/grid_trace.py SIZE KIND [name=value ...]
KIND: G (generator G, seed SIZE) or S (segmentation, seed 2048)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

S = int(sys.argv[1])
kind = sys.argv[2]
opts = dict(kv.split("=") for kv in sys.argv[3:])
opts = {k: int(v) for k, v in opts.items()}
caps = G.grid_random(S, S, S) if kind == "G" else G.grid_segmentation(S, S, 2048)
dev = [torch.from_numpy(c).cuda() for c in caps]
cut = torch.empty((S, S), dtype=torch.uint8, device="cuda")
solver = fmb.GridSolver(S, S, options={k: v for k, v in opts.items() if k != "trace"})
for i in range(int(os.environ.get("REPS", "3"))):
    f, st = solver.solve_device(dev, cut_out=cut)
print(kind, S, opts, "flow", f, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()}, flush=True)
solver.set_option("trace", opts.get("trace", 1))
f, st = solver.solve_device(dev, cut_out=cut)
print("traced", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()}, flush=True)
