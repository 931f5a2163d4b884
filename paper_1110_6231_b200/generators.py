"""Seeded synthetic instances of the benchmark shapes.

* :func:`grid_random` -- generator G: random integer capacities on an H x W grid.
* :func:`grid_segmentation` -- generator S: a synthetic-image graph-cut energy.
* :func:`assignment_reference` -- bit-identical to the reference's
  ``generate("assignment", n, density, max_value, rng_seed)`` (dimacs.py:271-344),
  vectorised: the planted shuffle runs on Python's ``random.Random(seed)`` and the
  weight stream continues on numpy's MT19937 from the very same state.
* :func:`assignment_optical_flow` -- the n = 4096 optical-flow-style dense matrix.
"""

from __future__ import annotations

import random

import numpy as np


def grid_random(H: int, W: int, seed: int):
    """Generator G.  numpy Generator(PCG64(seed)); draws (int32) in this order:
    capS in [0,100], capT in [0,100], capR/capL/capD/capU in [1,100] with the
    arcs that would leave the grid zeroed.  Returns (capR, capL, capD, capU, capS, capT)."""
    g = np.random.Generator(np.random.PCG64(seed))
    capS = g.integers(0, 101, size=(H, W), dtype=np.int32)
    capT = g.integers(0, 101, size=(H, W), dtype=np.int32)
    capR = g.integers(1, 101, size=(H, W), dtype=np.int32)
    capL = g.integers(1, 101, size=(H, W), dtype=np.int32)
    capD = g.integers(1, 101, size=(H, W), dtype=np.int32)
    capU = g.integers(1, 101, size=(H, W), dtype=np.int32)
    capR[:, -1] = 0
    capL[:, 0] = 0
    capD[-1, :] = 0
    capU[0, :] = 0
    return capR, capL, capD, capU, capS, capT


def segmentation_image(H: int, W: int, seed: int, disks: int = 48) -> np.ndarray:
    """Synthetic uint8 image: background 60, `disks` random disks (radius 30-250 px
    scaled to the image) at 180, plus N(0, 30^2) noise, clipped."""
    g = np.random.Generator(np.random.PCG64(seed))
    img = np.full((H, W), 60.0, np.float32)
    yy = np.arange(H, dtype=np.float32)[:, None]
    xx = np.arange(W, dtype=np.float32)[None, :]
    scale = min(H, W) / 2048.0
    for _ in range(disks):
        cy, cx = g.uniform(0, H), g.uniform(0, W)
        rad = g.uniform(30, 250) * scale
        y0, y1 = int(max(0, cy - rad)), int(min(H, cy + rad + 1))
        x0, x1 = int(max(0, cx - rad)), int(min(W, cx + rad + 1))
        if y0 >= y1 or x0 >= x1:
            continue
        sub = (yy[y0:y1] - cy) ** 2 + (xx[:, x0:x1] - cx) ** 2 <= rad * rad
        img[y0:y1, x0:x1][sub] = 180.0
    img += g.normal(0.0, 30.0, size=(H, W)).astype(np.float32)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def grid_segmentation(H: int, W: int, seed: int):
    """Generator S (config 2): unaries D_p(l) = round(10 (I_p - mu_l)^2 / (2 * 30^2)),
    mu_fg = 180, mu_bg = 60; capS = D_p(bg), capT = D_p(fg); pairwise both
    directions lambda_pq = 1 + round(50 exp(-(I_p - I_q)^2 / (2 * 10^2)))."""
    img = segmentation_image(H, W, seed).astype(np.float64)
    d_bg = np.rint(10.0 * (img - 60.0) ** 2 / (2 * 30.0 ** 2)).astype(np.int32)
    d_fg = np.rint(10.0 * (img - 180.0) ** 2 / (2 * 30.0 ** 2)).astype(np.int32)
    capS, capT = d_bg, d_fg
    capR = np.zeros((H, W), np.int32)
    capD = np.zeros((H, W), np.int32)
    lam_h = 1 + np.rint(50.0 * np.exp(-((img[:, 1:] - img[:, :-1]) ** 2) / (2 * 10.0 ** 2))).astype(np.int32)
    lam_v = 1 + np.rint(50.0 * np.exp(-((img[1:, :] - img[:-1, :]) ** 2) / (2 * 10.0 ** 2))).astype(np.int32)
    capR[:, :-1] = lam_h
    capL = np.zeros((H, W), np.int32)
    capL[:, 1:] = lam_h
    capD[:-1, :] = lam_v
    capU = np.zeros((H, W), np.int32)
    capU[1:, :] = lam_v
    return capR, capL, capD, capU, capS, capT


# ------------------------------------------------------------------ assignment

def _randbelow_words(words: np.ndarray, bound: int) -> np.ndarray:
    """Python's Random._randbelow_with_getrandbits(bound) applied to a stream of
    32-bit MT outputs (bound <= 2^32): k = bound.bit_length(); each word yields
    the candidate word >> (32 - k); candidates >= bound are rejected."""
    k = int(bound).bit_length()
    cand = (words >> np.uint64(32 - k)).astype(np.int64)
    return cand[cand < bound]


def assignment_reference(n: int, max_value: int = 100, seed: int = 0, density=None) -> np.ndarray:
    """The reference generator's assignment instance as a dense int32 matrix
    (dimacs.py:271-344); absent arcs (density given) are INT32_MIN."""
    if n < 1:
        raise ValueError(f"assignment generation needs n >= 1, got {n}")
    if max_value < 0:
        raise ValueError(f"max_value must be nonnegative, got {max_value}")
    rng = random.Random(seed)
    planted = list(range(n))
    rng.shuffle(planted)
    if density is not None:
        density = float(density)
        if not (0.0 < density <= 1.0):
            raise ValueError(f"density must be in (0, 1], got {density}")
        w = np.full((n, n), -(2**31), np.int64)
        for x in range(n):
            for y in range(n):
                if planted[x] == y or rng.random() < density:
                    w[x, y] = rng.randint(0, max_value)
        return w.astype(np.int32)
    # complete: n*n calls rng.randint(0, max_value), row-major; continue the same
    # MT19937 stream in numpy
    version, internal, _ = rng.getstate()
    bg = np.random.MT19937()
    bg.state = {"bit_generator": "MT19937",
                "state": {"key": np.asarray(internal[:624], dtype=np.uint32), "pos": int(internal[624])}}
    bound = max_value + 1
    need = n * n
    out = []
    got = 0
    accept = bound / float(1 << int(bound).bit_length())
    while got < need:
        draw = int((need - got) / accept * 1.02) + 1024
        vals = _randbelow_words(bg.random_raw(draw).astype(np.uint64), bound)
        out.append(vals)
        got += len(vals)
    # the rejection stream is consumed strictly in order, so overshooting is harmless
    return np.concatenate(out)[:need].reshape(n, n).astype(np.int32)


def assignment_optical_flow(n: int = 4096, seed: int = 4096) -> np.ndarray:
    """Optical-flow-style dense matching.  X = s x s lattice points
    (s = sqrt(n)) with 8-dim int8 descriptors of a smooth random field; Y = the same
    points moved by a smooth flow (rotation 2 deg about the centre + translation
    (3, -2) px + N(0, 0.5^2)), descriptor noise N(0, 4^2), then shuffled.
    w(x, y) = max(0, 10^4 - |d_x - d_y|_1 - 20 |p_x + f(p_x) - p_y|_1) (int32)."""
    s = int(round(n ** 0.5))
    if s * s != n:
        raise ValueError("n must be a perfect square")
    g = np.random.Generator(np.random.PCG64(seed))
    noise = g.normal(size=(8, s, s))
    # smooth field: Gaussian low-pass in the Fourier domain (sigma ~ 3 px)
    fy = np.fft.fftfreq(s)[:, None]
    fx = np.fft.fftfreq(s)[None, :]
    filt = np.exp(-2 * (np.pi * 3.0) ** 2 * (fx ** 2 + fy ** 2))
    field = np.real(np.fft.ifft2(np.fft.fft2(noise) * filt))
    field /= np.abs(field).max() + 1e-12
    desc_x = np.rint(field * 100).astype(np.int16).reshape(8, -1).T  # n x 8
    ii, jj = np.meshgrid(np.arange(s, dtype=np.float64), np.arange(s, dtype=np.float64), indexing="ij")
    px = np.stack([ii.reshape(-1), jj.reshape(-1)], 1)
    c = (s - 1) / 2.0
    th = np.deg2rad(2.0)
    rot = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    moved = (px - c) @ rot.T + c + np.array([3.0, -2.0])
    flow = moved - px
    py = moved + g.normal(0.0, 0.5, size=moved.shape)
    desc_y = np.clip(desc_x + np.rint(g.normal(0.0, 4.0, size=desc_x.shape)), -127, 127).astype(np.int16)
    perm = g.permutation(n)
    py, desc_y = py[perm], desc_y[perm]
    pred = px + flow
    w = np.empty((n, n), np.int32)
    step = 256
    for a in range(0, n, step):
        b = min(n, a + step)
        dd = np.abs(desc_x[a:b, None, :].astype(np.int32) - desc_y[None, :, :].astype(np.int32)).sum(-1)
        dp = np.abs(pred[a:b, None, :] - py[None, :, :]).sum(-1)
        w[a:b] = np.maximum(0, 10000 - dd - np.rint(20.0 * dp).astype(np.int64)).astype(np.int32)
    return w


BLOCK_ROWS = 512


def grid_random_rows(H: int, W: int, seed: int, r0: int, r1: int):
    """Rows [r0, r1) of the *blocked* generator G_b used for multi-GPU grids: rows
    come in blocks of 512, block b drawn like generator G from PCG64([seed, b]) (same
    ranges and plane order), so every rank builds its band without the whole grid.
    Returns the six planes restricted to those rows (arcs leaving the grid zeroed)."""
    if not (0 <= r0 < r1 <= H):
        raise ValueError("bad row range")
    planes = [[] for _ in range(6)]
    for b in range(r0 // BLOCK_ROWS, (r1 - 1) // BLOCK_ROWS + 1):
        lo, hi = b * BLOCK_ROWS, min(H, (b + 1) * BLOCK_ROWS)
        g = np.random.Generator(np.random.PCG64([seed, b]))
        n = hi - lo
        blk = [g.integers(0, 101, size=(n, W), dtype=np.int32),
               g.integers(0, 101, size=(n, W), dtype=np.int32)]
        blk += [g.integers(1, 101, size=(n, W), dtype=np.int32) for _ in range(4)]
        a, z = max(lo, r0), min(hi, r1)
        # order of the returned planes: R, L, D, U, S, T (drawn as S, T, R, L, D, U)
        for k, src in enumerate((2, 3, 4, 5, 0, 1)):
            planes[k].append(blk[src][a - lo:z - lo])
    capR, capL, capD, capU, capS, capT = [np.ascontiguousarray(np.concatenate(p)) for p in planes]
    capR[:, -1] = 0
    capL[:, 0] = 0
    if r1 == H:
        capD[-1, :] = 0
    if r0 == 0:
        capU[0, :] = 0
    return capR, capL, capD, capU, capS, capT


def grid_random_blocked(H: int, W: int, seed: int):
    """The whole grid of the blocked generator (tests / single-GPU reference)."""
    return grid_random_rows(H, W, seed, 0, H)
