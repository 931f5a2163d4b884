"""Banded-solve coordination cost on one GPU: N virtual bands (one host thread each,
neighbours through device memory) vs the plain single-band solve of the same grid.
Usage: python scripts/bands_overhead.py [size] [reps]"""

import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import bands as B
from paper_1110_6231_b200 import generators as G

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 5
for kind, caps in (("G", G.grid_random(S, S, S)), ("S", G.grid_segmentation(S, S, S))):
    dcaps = [torch.from_numpy(c).cuda() for c in caps]
    cut = torch.empty((S, S), dtype=torch.uint8, device="cuda")
    sv = fmb.GridSolver(S, S)
    sv.solve_device(dcaps, cut_out=cut)
    ts = []
    for _ in range(REPS):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f1, st1 = sv.solve_device(dcaps, cut_out=cut)
        torch.cuda.synchronize()
        ts.append(1000 * (time.perf_counter() - t0))
    sv.close()
    base = statistics.median(ts)
    print(f"{kind} {S}^2 plain: {base:.2f} ms (device {st1['ms_total']:.2f}), rounds {st1['rounds']}", flush=True)
    for nb in (2, 4, 8):
        grp = B.BandGroup(S, S, nb, [0] * nb)
        grp.solve(dcaps, cut_out=cut)
        ts, dev = [], []
        for _ in range(REPS):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f, _, st = grp.solve(dcaps, cut_out=cut)
            ts.append(1000 * (time.perf_counter() - t0))
            dev.append(st["ms_total"])
            assert f == f1, (f, f1)
        grp.close()
        m = statistics.median(ts)
        print(f"  {nb} virtual bands: {m:.2f} ms wall ({m / base:.2f}x plain), device max {statistics.median(dev):.2f} ms, "
              f"rounds {st['rounds']} push launches {st['pr_launches']} ring visits {st['reserved'][0]}", flush=True)
