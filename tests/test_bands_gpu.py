"""Row-band sharding (multi-GPU grid path) exercised as virtual bands on one GPU:
flow and minimal cut must be bit-identical to the single-band solve and the oracle."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1110_6231_b200 as fmb
from paper_1110_6231_b200 import bands as B
from paper_1110_6231_b200 import generators as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W,nb,kind", [(64, 48, 2, "G"), (100, 70, 3, "G"), (256, 256, 4, "G"),
                                         (96, 64, 3, "S"), (512, 512, 8, "G"), (40, 33, 2, "G")])
def test_virtual_bands_match_oracle(H, W, nb, kind):
    caps = G.grid_random(H, W, H + W) if kind == "G" else G.grid_segmentation(H, W, 7)
    want = oracle.grid_maxflow(*caps, solver="seq")
    flow, cut, st = B.solve_virtual_bands(caps, nb)
    assert flow == want["value"]
    assert (cut == want["cut"]).all()
    assert st["rounds"] >= 1 or want["value"] == 0


def test_virtual_bands_match_single_band_at_1024():
    caps = G.grid_random(1024, 1024, 11)
    rep = fmb.hybrid_solve(fmb.build_grid_network(*caps))
    for nb in (2, 4):
        flow, cut, _ = B.solve_virtual_bands(caps, nb)
        assert flow == rep.objective
        assert (cut == rep.cut).all()


def _dist_band_worker(rank, world, port, H, W, seed, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    caps = G.grid_random(H, W, seed)
    spans = B.band_rows(H, world)
    r0, r1 = spans[rank]
    gt, gb = rank > 0, rank + 1 < world
    flow, band, st = B.solve_distributed(B.band_caps(caps, r0, r1, gt, gb), gt, gb, H * W, rank, world, 0)
    cut = band.cut_host()[(1 if gt else 0):(1 if gt else 0) + (r1 - r0)]
    q.put((rank, flow, r0, r1, cut))
    band.close()
    dist.destroy_process_group()


def test_multiprocess_bands_gloo_on_one_gpu():
    """The one-process-per-GPU coordinator (DistTransport) with 2 ranks sharing the
    single test GPU; gloo stages the boundary rows through host memory."""
    import multiprocessing as mp
    import socket

    H, W, seed = 200, 96, 5
    caps = G.grid_random(H, W, seed)
    want = oracle.grid_maxflow(*caps, solver="seq")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dist_band_worker, args=(r, 2, port, H, W, seed, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    cut = np.zeros((H, W), bool)
    for rank, flow, r0, r1, c in got:
        assert flow == want["value"]
        cut[r0:r1] = c.astype(bool)
    assert (cut == want["cut"]).all()


@pytest.mark.parametrize("nb", [3, 8])
def test_bands_segmentation_and_many_bands(nb):
    caps = G.grid_segmentation(512, 384, 11)
    want = oracle.grid_maxflow(*caps, solver="seq")
    flow, cut, _ = B.solve_virtual_bands(caps, nb)
    assert flow == want["value"] and (cut == want["cut"]).all()


def test_bands_blocked_generator_rows():
    # the multi-GPU bench builds each band from its own rows of the blocked generator
    H, W = 600, 200
    full = G.grid_random_blocked(H, W, 3)
    want = oracle.grid_maxflow(*full, solver="seq")
    spans = B.band_rows(H, 3)
    bands = []
    for k, (r0, r1) in enumerate(spans):
        gt, gb = k > 0, k + 1 < len(spans)
        rows = G.grid_random_rows(H, W, 3, r0 - gt, r1 + gb)
        bc = B.band_caps_from_rows(rows, gt, gb)
        assert all(np.array_equal(a, b) for a, b in zip(bc, B.band_caps(full, r0, r1, gt, gb)))
        bands.append(B.Band(bc, gt, gb, H * W + 2))
    co = B.BandedSolve(B.LocalTransport(bands), total_pixels=H * W)
    assert co.run() == want["value"]
    for b in bands:
        b.close()


def _stress_band_case(seed, k):
    """Case k of scripts/stress_bands.py's generator (same draw order)."""
    rng = np.random.default_rng(seed)
    for _ in range(k + 1):
        nb = int(rng.integers(2, 5))
        H, W = int(rng.integers(66 * nb, 300)), int(rng.integers(1, 300))
        hi = int(rng.choice([1, 3, 30, 100]))
        caps = [rng.integers(0, hi + 1, size=(H, W)).astype(np.int32) for _ in range(4)]
        ps, pt = rng.uniform(0.02, 1.0, 2)
        capS = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < ps)).astype(np.int32)
        capT = (rng.integers(0, hi + 1, size=(H, W)) * (rng.random((H, W)) < pt)).astype(np.int32)
        caps[0][:, -1] = 0
        caps[1][:, 0] = 0
        caps[2][-1, :] = 0
        caps[3][0, :] = 0
        caps = caps + [capS, capT]
    return caps, nb


@pytest.mark.parametrize("k", [132, 149])
def test_regression_band_cut_ghost_residuals(k):
    """scripts/stress_bands.py seed 5: the cut came out short of the minimal one next to
    band borders (flow correct) because the ghost rows' residuals toward the band were
    those exported before the last push exchange folded its flow in."""
    caps, nb = _stress_band_case(5, k)
    want = oracle.grid_maxflow(*caps, solver="seq")
    flow, cut, _ = B.solve_virtual_bands(caps, nb)
    assert flow == want["value"] and (cut == want["cut"]).all()


@pytest.mark.parametrize("seed", range(12))
def test_random_band_cases(seed):
    caps, nb = _stress_band_case(100 + seed, 0)
    want = oracle.grid_maxflow(*caps, solver="seq")
    flow, cut, _ = B.solve_virtual_bands(caps, nb)
    assert flow == want["value"] and (cut == want["cut"]).all()
