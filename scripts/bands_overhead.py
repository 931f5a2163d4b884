"""Banded-solve coordination cost on one GPU: virtual bands (LocalTransport) vs the
plain solve of the same grid (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import bands as B
from paper_1110_6231_b200 import generators as G

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
caps = G.grid_random(S, S, S)
net = fmb.build_grid_network(*caps)
for _ in range(2):
    rep = fmb.hybrid_solve(net)
print(f"plain: flow {rep.objective} {1000 * rep.elapsed:.1f} ms (device {rep.stats['ms_total']:.1f} ms, rounds {rep.rounds})")
for nb in (2, 4):
    for _ in range(2):
        flow, cut, st = B.solve_virtual_bands(caps, nb)
    assert flow == rep.objective and (cut == rep.cut).all()
    print(f"{nb} virtual bands: {1000 * st['elapsed']:.1f} ms, rounds {st['rounds']} exchanges {st['exchanges']} "
          f"bfs_exchanges {st['bfs_exchanges']} pushes {st['pushes']} relabels {st['relabels']}")
