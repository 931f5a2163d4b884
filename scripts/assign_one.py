"""One n x n assignment solve on the device (profiling target).
usage: python scripts/assign_one.py N KIND [name=value ...]   (KIND: M100 | M10000 | optical)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

n = int(sys.argv[1])
kind = sys.argv[2] if len(sys.argv) > 2 else "M10000"
w = G.assignment_optical_flow(n, n) if kind == "optical" else G.assignment_reference(n, int(kind[1:]), n)
wd = torch.from_numpy(w).cuda()
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[3:]}
s = fmb.AssignmentSolver(n, options=opts)
for _ in range(int(os.environ.get("REPS", "1"))):
    obj, m, _, st = s.solve_device(wd)
print(kind, n, "objective", obj, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()}, flush=True)
