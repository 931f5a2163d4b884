#!/bin/bash
for lib in ${LIBS:-paper_1110_6231_b200/libfm_b200.so}; do
  echo "LIB=$lib"
  FM_LIB_PATH=$lib timeout 200 python - <<'PY'
import sys; sys.path.insert(0, ".")
import paper_1110_6231_b200 as f, torch
from paper_1110_6231_b200 import generators as G
s = f.AssignmentSolver(4096)
for name, w in (("opt", G.assignment_optical_flow(4096, 4096)), ("m100", G.assignment_reference(4096, 100, 4096)), ("m1e4", G.assignment_reference(4096, 10000, 4096))):
    w = torch.from_numpy(w).cuda(); s.solve_device(w); o, m, _, st = s.solve_device(w)
    print(name, "obj", o, "total", round(st["ms_total"], 2), "pu", round(st["ms_bfs"], 2), "tail", round(st["ms_cut"], 2), "multi", round(st["ms_d2h"], 2), "rounds", st["rounds"], "tail_rounds", st["pr_sweeps"], "Yph", round(st["ms_pr_kern"], 2), "Xph", round(st["ms_bfs_kern"], 2), "syncs", round(st["bytes_bfs"] * 1e-6, 2), flush=True)
PY
done
