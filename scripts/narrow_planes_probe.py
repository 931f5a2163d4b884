"""Host-plane dtype probe (GPU box): raw pinned H2D of int32 vs uint8 planes, then
hybrid_solve / hybrid_solve_batch end to end on each at 4096^2."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import generators as G
S = 4096
caps = G.grid_random(S, S, S)
p32 = [torch.from_numpy(c).pin_memory() for c in caps]
p8 = [torch.from_numpy(c.astype(np.uint8)).pin_memory() for c in caps]
for name, ps in (("int32", p32), ("uint8", p8)):
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d = [p.cuda(non_blocking=True) for p in ps]
        torch.cuda.synchronize(); print(name, "raw H2D ms", round(1000 * (time.perf_counter() - t0), 2), ps[0].is_pinned())
n32 = fmb.build_grid_network(*[p.numpy() for p in p32]); n8 = fmb.build_grid_network(*[p.numpy() for p in p8])
print("narrow", n8.narrow_bytes, n8.caps[0].ctypes.data == p8[0].data_ptr())
for name, net in (("int32", n32), ("uint8", n8)):
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = fmb.hybrid_solve(net)
        torch.cuda.synchronize(); print(name, "single ms", round(1000 * (time.perf_counter() - t0), 2), r.stats["ms_total"])
    for K in (3, 6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rs = fmb.hybrid_solve_batch([net] * K)
        torch.cuda.synchronize(); print(name, "batch", K, "ms/step", round(1000 * (time.perf_counter() - t0) / K, 2), [round(x.stats["ms_total"], 2) for x in rs])
