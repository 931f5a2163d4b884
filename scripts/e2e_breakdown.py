"""Where the end-to-end grid solve time goes (GPU box): pinned host planes ->
hybrid_solve -> bool cut, vs the device-resident solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
caps = [np.ascontiguousarray(c) for c in G.grid_random(S, S, S)]
pinned = [torch.from_numpy(c).pin_memory().numpy() for c in caps]
net = fmb.build_grid_network(*pinned)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = fmb.hybrid_solve(net)
    t1 = time.perf_counter()
    st = rep.stats
    print(f"e2e {1000*(t1-t0):.2f} ms (cut {rep.cut.dtype}) | solve {st['ms_total']:.2f} h2d {st['ms_h2d']:.2f} d2h {st['ms_d2h']:.2f} "
          f"rest {1000*(t1-t0)-st['ms_total']-st['ms_h2d']-st['ms_d2h']:.2f}", flush=True)
