"""Host-side logic of the row-band path (CPU, no GPU): the band partition (Python and
the library's fm_band_split agree), the band inputs, and the shared-memory collective
the bands agree through -- threads of one process, and two processes (world size 2,
the shared segment's name exchanged over gloo as the torchrun path does)."""

from __future__ import annotations

import ctypes
import os
import threading
import uuid

import numpy as np
import pytest

from paper_1110_6231_b200 import _lib
from paper_1110_6231_b200 import bands as B
from paper_1110_6231_b200 import generators as G


def test_band_rows_cover_and_align():
    for H, nb in [(4096, 8), (8192, 4), (8192, 8), (100, 3), (33, 2), (64, 1), (1000, 7), (32, 1)]:
        spans = B.band_rows(H, nb)
        assert spans[0][0] == 0 and spans[-1][1] == H and len(spans) == nb
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c and b > a
        assert all(r0 % 32 == 0 for r0, _ in spans)
        assert all((r1 - r0) % 32 == 0 for r0, r1 in spans[:-1])
    with pytest.raises(ValueError):
        B.band_rows(40, 3)          # 2 tile rows, 3 bands
    assert B.band_rows(8192, 8) == [(k * 1024, (k + 1) * 1024) for k in range(8)]


def test_band_split_matches_library():
    L = _lib.load()
    for H, nb in [(4096, 8), (8192, 3), (100, 3), (1000, 7), (33, 2), (8191, 5)]:
        edges = (ctypes.c_int32 * (nb + 1))()
        assert L.fm_band_split(H, nb, edges) == 0
        spans = B.band_rows(H, nb)
        assert list(edges) == [r0 for r0, _ in spans] + [H]
    edges = (ctypes.c_int32 * 4)()
    assert L.fm_band_split(40, 3, edges) == _lib.FM_INVALID_ARG


def test_band_planes_slices_and_halo_rows():
    caps = G.grid_random(70, 9, 3)
    spans = B.band_rows(70, 2)
    total_s = 0
    for k, (r0, r1) in enumerate(spans):
        rows, above, below = B.band_planes(caps, r0, r1)
        for a, g in zip(rows, caps):
            assert a.shape == (r1 - r0, 9) and a.dtype == np.int32 and np.array_equal(a, g[r0:r1])
        assert (above is None) == (r0 == 0) and (below is None) == (r1 == 70)
        if above is not None:
            assert np.array_equal(above, caps[2][r0 - 1])
        if below is not None:
            assert np.array_equal(below, caps[3][r1])
        total_s += int(rows[4].sum())
    assert total_s == int(caps[4].sum())


def test_coll_threads_allgather_many_rounds():
    """Process-local segment (the in-process group's), 4 threads x 200 rounds: every
    rank sees every rank's values of that round (slot sets alternate by parity)."""
    n = 4
    L = _lib.load()
    views = []
    name = f"/fm_coll_test_{uuid.uuid4().hex[:12]}"
    for r in range(n):   # rank 0 creates the segment, the others open it
        c = ctypes.c_void_p()
        assert L.fm_coll_create(name.encode(), n, r, ctypes.byref(c)) == 0
        views.append(c)
    errors = []

    def worker(r):
        v = (ctypes.c_int64 * 3)()
        out = (ctypes.c_int64 * (3 * n))()
        for k in range(200):
            v[0], v[1], v[2] = r, k, r * 1000 + k
            if L.fm_coll_allgather(views[r], v, 3, out) != 0:
                errors.append("rc")
                return
            got = [list(out[q * 3:(q + 1) * 3]) for q in range(n)]
            if got != [[q, k, q * 1000 + k] for q in range(n)]:
                errors.append((r, k, got))
                return

    th = [threading.Thread(target=worker, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    for c in reversed(views):
        L.fm_coll_destroy(c)
    assert not errors, errors[:3]


def test_coll_rejects_bad_arguments():
    L = _lib.load()
    c = ctypes.c_void_p()
    assert L.fm_coll_create(None, 0, 0, ctypes.byref(c)) == _lib.FM_INVALID_ARG
    assert L.fm_coll_create(None, 2, 2, ctypes.byref(c)) == _lib.FM_INVALID_ARG
    assert L.fm_coll_create(None, 1, 0, ctypes.byref(c)) == 0
    v = (ctypes.c_int64 * 9)()
    assert L.fm_coll_allgather(c, v, 9, v) == _lib.FM_INVALID_ARG
    one = B.Coll(None, 1, 0)
    assert one.allgather([5, 6]) == [[5, 6]]
    one.close()
    L.fm_coll_destroy(c)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the torchrun path's set-up: rank 0 names (and creates) the segment, the name
    # travels through torch.distributed, the others open it after a barrier
    name = [f"/fm_coll_t_{uuid.uuid4().hex[:12]}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    c0 = B.Coll(name[0], world, 0) if rank == 0 else None
    dist.barrier()
    c = c0 if rank == 0 else B.Coll(name[0], world, rank)
    dist.barrier()
    seen = []
    for k in range(50):
        # the values a band contributes per push batch: {idle, raised, consumed, relabels}
        seen.append(c.allgather([rank, k, 10 * rank + k, -k]))
    dist.barrier()
    c.close()
    q.put((rank, seen))
    dist.destroy_process_group()


def test_coll_two_processes_gloo_world2():
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
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    for k in range(50):
        want = [[r, k, 10 * r + k, -k] for r in range(2)]
        assert res[0][k] == want and res[1][k] == want
