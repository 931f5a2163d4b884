"""Small grid / segmentation / assignment / generic solves for compute-sanitizer runs
(memcheck, initcheck, synccheck) on the GPU box: scripts/sanitize_smoke.py under
`compute-sanitizer --tool <tool> python scripts/sanitize_smoke.py`."""
import os, sys; sys.path.insert(0, os.getcwd())
import numpy as np, paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
for (H, W) in ((200, 256), (33, 70), (1, 97)):
    caps = G.grid_random(H, W, 7)
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps)); print("grid", H, W, rep.objective)
for (H, W) in ((100, 128),):
    caps = G.grid_segmentation(H, W, 3)
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps)); print("seg", rep.objective)
w = G.assignment_reference(96, 100, 5); rep, m = fmb.solve_assignment(w); print("assign", rep.objective)
net = fmb.build_network([(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)], 4, 0, 3); print("csr", fmb.hybrid_solve(net).objective)
from paper_1110_6231_b200 import bands as B
flow, cut, st = B.solve_virtual_bands(G.grid_random(100, 70, 9), 3); print("bands", flow)
# sparse assignment (cooperative rounds + price update), int64 generic kernel, wide grid
xs, ys = np.nonzero(G.assignment_reference(300, 1000, 7, density=0.05) != -(2**31))
ws = np.random.default_rng(1).integers(0, 1000, len(xs))
inst = fmb.AssignmentInstance.build(300, list(zip(xs.tolist(), ys.tolist(), ws.tolist())))
rep, m = fmb.solve_assignment(inst, layout="sparse"); print("sparse", rep.objective)
net = fmb.build_network([(0, 1, 3 * 2**40), (0, 2, 2**41), (1, 3, 2**41), (2, 3, 3 * 2**40), (1, 2, 2**40)], 4, 0, 3)
print("csr64", fmb.hybrid_solve(net).objective)
caps = [c.astype(np.int64) * 2**33 for c in G.grid_random(40, 50, 3)]
print("wide grid", fmb.hybrid_solve(fmb.build_grid_network(*caps)).objective)
caps = G.grid_random(120, 96, 5)
s = fmb.GridSolver(120, 96, options={"ring_tail": 1}); print("ring_tail grid", s.solve_host(caps)[0]); s.close()
# pipelined batch from host planes (int32 and uint8: narrow H2D + device widening)
nets = [fmb.build_grid_network(*G.grid_random(64, 96, s)) for s in (1, 2, 3)]
print("batch", [r.objective for r in fmb.hybrid_solve_batch(nets)])
nets8 = [fmb.build_grid_network(*[a.astype(np.uint8) for a in G.grid_random(33, 7, s)]) for s in (4, 5)]
print("batch u8", [r.objective for r in fmb.hybrid_solve_batch(nets8)])
# assignment with a large-candidate gather (n = 1024, narrow weight range) and the filtered price update
w = G.assignment_reference(1024, 3, 9); rep, m = fmb.solve_assignment(w); print("assign 1024", rep.objective)
