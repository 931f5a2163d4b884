"""Host-side logic of the row-band path (CPU): band partition, ghost-row capacity
slicing, and the multi-process coordinator's collectives over gloo (world size 2)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1110_6231_b200 import bands as B
from paper_1110_6231_b200 import generators as G


def test_band_rows_cover_and_align():
    for H, nb in [(4096, 8), (8192, 4), (100, 3), (33, 2), (5, 5), (64, 1)]:
        spans = B.band_rows(H, nb)
        assert spans[0][0] == 0 and spans[-1][1] == H and len(spans) == nb
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c and b > a
        if H >= 32 * nb:
            assert all(r0 % 32 == 0 for r0, _ in spans)
    with pytest.raises(ValueError):
        B.band_rows(3, 4)


def test_band_caps_ghost_rows():
    caps = G.grid_random(70, 9, 3)
    spans = B.band_rows(70, 3)
    total_s = 0
    for k, (r0, r1) in enumerate(spans):
        gt, gb = k > 0, k + 1 < len(spans)
        bc = B.band_caps(caps, r0, r1, gt, gb)
        assert bc[0].shape == (r1 - r0 + gt + gb, 9)
        lo = 1 if gt else 0
        for a, g in zip(bc, caps):
            assert np.array_equal(a[lo:lo + r1 - r0], g[r0:r1])
        if gt:  # ghost above: only its arc into the band
            assert np.array_equal(bc[2][0], caps[2][r0 - 1])
            for j in (0, 1, 3, 4, 5):
                assert not bc[j][0].any()
        if gb:
            assert np.array_equal(bc[3][-1], caps[3][r1])
            for j in (0, 1, 2, 4, 5):
                assert not bc[j][-1].any()
        total_s += int(bc[4].sum())
    assert total_s == int(caps[4].sum())


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class FakeBand:
        """Stands in for a GPU band: counts what crosses each border."""

        def __init__(self, rank):
            self.rank = rank
            self.ghost_top, self.ghost_bot = rank > 0, rank + 1 < world
            self.caps = [torch.zeros(1)]
            self.buf = {s: torch.zeros(4, dtype=torch.int32) for s in (B.TOP, B.BOTTOM)}
            self.rbuf = {s: torch.zeros(4, dtype=torch.int32) for s in (B.TOP, B.BOTTOM)}
            self.got = {}

        def sides(self):
            return ([B.TOP] if self.ghost_top else []) + ([B.BOTTOM] if self.ghost_bot else [])

        def rows_out(self, side, kind):
            self.buf[side][:] = torch.tensor([self.rank, side, kind, 7], dtype=torch.int32)
            return self.buf[side]

        def rows_in(self, side, kind, src):
            self.got[side] = src.tolist()
            return 1

    b = FakeBand(rank)
    tr = B.DistTransport.__new__(B.DistTransport)
    tr.band, tr.rank, tr.world = b, rank, world

    # exchange without CUDA: patch the stream sync used on GPUs
    import torch.cuda

    orig = torch.cuda.current_stream
    torch.cuda.current_stream = lambda: type("S", (), {"synchronize": lambda self: None})()
    try:
        changed = tr.exchange(B.ROW_DIST)
    finally:
        torch.cuda.current_stream = orig
    t = torch.tensor([changed, rank + 1], dtype=torch.int64)
    dist.all_reduce(t)
    q.put((rank, b.got, t.tolist()))
    dist.destroy_process_group()


def test_dist_transport_gloo_world2():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        rank, got, tot = q.get(timeout=120)
        res[rank] = (got, tot)
    for p in ps:
        p.join(timeout=60)
    # rank 0's bottom neighbour is rank 1, which sent from its TOP side, and vice versa
    assert res[0][0][B.BOTTOM] == [1, B.TOP, B.ROW_DIST, 7]
    assert res[1][0][B.TOP] == [0, B.BOTTOM, B.ROW_DIST, 7]
    assert res[0][1] == [2, 3] and res[1][1] == [2, 3]
