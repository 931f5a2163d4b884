"""Row-band sharding of the grid max-flow / min-cut across GPUs.

The H x W grid is cut into horizontal bands whose borders sit on 32-row tile
boundaries.  Each band is an ``fm_grid`` (one per GPU, one process per GPU) holding
its own rows plus a *ghost row* per neighbour: a frozen copy of the neighbour's
boundary row.  The lock-free kernel already parks every push that crosses a tile
border in the receiver's inbox; a push into a ghost pixel is exactly such a parked
push, so a band step is

    push launches -> ship ghost-row flow, boundary heights and residuals to the
    neighbours -> repeat until idle or the round's budget -> global relabel

where the global relabel (backward BFS from t) is a band-local frontier fixpoint
plus an exchange of boundary distances, repeated until no band changes (a
distributed min-relaxation; distances are monotone).  Termination and flow are
int64 sums over bands.  Transport: ``LocalTransport`` runs all bands on one device
in one process (virtual bands, used by the single-GPU tests), ``DistTransport``
moves the 4 B x W boundary rows with ``torch.distributed`` send/recv (NCCL over
NVLink) between neighbouring ranks and all-reduces the scalars.

Reference semantics kept: the same coordinator structure as hybrid_solve
(maxflow_par.py:195-229): rounds of lock-free work, then global relabel + gap +
marking, until no unmarked pixel holds excess.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .graph import SolveReport

ROW_FLOW, ROW_H, ROW_RES, ROW_DIST, ROW_CUT, ROW_PUSH_STATE = 0, 1, 2, 3, 4, 5
TOP, BOTTOM = 0, 1
TILE = 32


def band_rows(H: int, nbands: int) -> list[tuple[int, int]]:
    """Split H rows into nbands contiguous bands on 32-row tile boundaries
    (the last band takes the remainder).  Every band gets at least one row."""
    if nbands < 1:
        raise ValueError("nbands must be >= 1")
    if nbands > max(1, H):
        raise ValueError(f"cannot split {H} rows into {nbands} bands")
    tiles = (H + TILE - 1) // TILE
    if nbands > tiles:
        # fewer tile rows than bands: fall back to plain row counts
        edges = [round(k * H / nbands) for k in range(nbands + 1)]
    else:
        edges = [min(H, round(k * tiles / nbands) * TILE) for k in range(nbands + 1)]
        edges[-1] = H
    out = [(edges[k], edges[k + 1]) for k in range(nbands)]
    if any(r1 <= r0 for r0, r1 in out):
        raise ValueError(f"empty band in split of {H} rows into {nbands}")
    return out


def band_caps(caps, r0: int, r1: int, ghost_top: bool, ghost_bot: bool):
    """The six capacity planes of band rows [r0, r1) plus ghost rows.  A ghost row
    carries only the capacity of its arc INTO the band (capD above, capU below):
    the rest of that pixel belongs to the neighbour band."""
    capR, capL, capD, capU, capS, capT = [np.asarray(a) for a in caps]
    W = capS.shape[1]
    rows = [np.ascontiguousarray(a[r0:r1], dtype=np.int32) for a in (capR, capL, capD, capU, capS, capT)]
    if ghost_top:
        g = [np.zeros((1, W), np.int32) for _ in range(6)]
        g[2][0] = capD[r0 - 1]
        rows = [np.concatenate([gg, a]) for gg, a in zip(g, rows)]
    if ghost_bot:
        g = [np.zeros((1, W), np.int32) for _ in range(6)]
        g[3][0] = capU[r1]
        rows = [np.concatenate([a, gg]) for gg, a in zip(g, rows)]
    return [np.ascontiguousarray(a) for a in rows]


def band_caps_from_rows(rows, ghost_top: bool, ghost_bot: bool):
    """Band planes from the rows [r0 - ghost_top, r1 + ghost_bot) of a grid: ghost rows
    keep only their arc into the band (capD above, capU below)."""
    out = [np.array(a, dtype=np.int32, copy=True) for a in rows]
    if ghost_top:
        for k in (0, 1, 3, 4, 5):
            out[k][0] = 0
    if ghost_bot:
        for k in (0, 1, 2, 4, 5):
            out[k][-1] = 0
    return [np.ascontiguousarray(a) for a in out]


class Band:
    """One band: an fm_grid handle in band mode plus its device inputs."""

    def __init__(self, caps_band, ghost_top: bool, ghost_bot: bool, global_nodes: int, device: int = 0):
        import torch

        L = _lib.load()
        _lib.require_device()
        self.ghost_top, self.ghost_bot = bool(ghost_top), bool(ghost_bot)
        self.Hb, self.W = caps_band[0].shape
        h = ctypes.c_void_p()
        _lib.check(L.fm_grid_create(int(self.Hb), int(self.W), int(device), ctypes.byref(h)), "fm_grid_create")
        self._h = h
        _lib.check(L.fm_grid_band_config(h, int(self.ghost_top), int(self.ghost_bot), int(global_nodes)),
                   "fm_grid_band_config")
        self.device = device
        dev = torch.device("cuda", device)
        # band steps on torch's current stream: row exports are then ordered before the
        # NCCL sends that read them without a host synchronisation
        _lib.check(L.fm_grid_band_stream(h, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)),
                   "fm_grid_band_stream")
        self.caps = [torch.from_numpy(np.ascontiguousarray(c)).to(dev) for c in caps_band]
        # row buffers sized for the widest message (ROW_PUSH_STATE: 3 rows)
        self.buf = {s: torch.empty(3 * self.W, dtype=torch.int32, device=dev) for s in (TOP, BOTTOM)}
        self.rbuf = {s: torch.empty(3 * self.W, dtype=torch.int32, device=dev) for s in (TOP, BOTTOM)}

    def sides(self):
        return ([TOP] if self.ghost_top else []) + ([BOTTOM] if self.ghost_bot else [])

    def load_caps(self, caps_band) -> None:
        """Copy new host planes (same shape) into the band's device inputs."""
        for d, h in zip(self.caps, caps_band):
            d.copy_(h if hasattr(h, "device") else __import__("torch").from_numpy(np.ascontiguousarray(h)),
                    non_blocking=True)

    def close(self):
        if self._h:
            _lib.load().fm_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- thin C-ABI wrappers
    def init(self, flags=0) -> int:
        out = ctypes.c_int64()
        _lib.check(_lib.load().fm_grid_band_init(self._h, *[_lib.ptr(c) for c in self.caps], int(flags),
                                                 ctypes.byref(out)), "fm_grid_band_init")
        return int(out.value)

    def bfs(self, phase: int) -> int:
        out = ctypes.c_int64()
        _lib.check(_lib.load().fm_grid_band_bfs(self._h, int(phase), ctypes.byref(out)), "fm_grid_band_bfs")
        return int(out.value)

    def finalize(self):
        out = (ctypes.c_int64 * 3)()
        _lib.check(_lib.load().fm_grid_band_finalize(self._h, out), "fm_grid_band_finalize")
        return int(out[0]), int(out[1]), int(out[2])

    def push(self, launches: int, cycle_budget: int):
        out = (ctypes.c_int64 * 4)()
        _lib.check(_lib.load().fm_grid_band_push(self._h, int(launches), int(cycle_budget), out),
                   "fm_grid_band_push")
        return int(out[0]), int(out[1]), int(out[2]), bool(out[3])

    def cut(self, phase: int) -> int:
        out = ctypes.c_int64()
        _lib.check(_lib.load().fm_grid_band_cut(self._h, int(phase), ctypes.byref(out)), "fm_grid_band_cut")
        return int(out.value)

    def rows_out(self, side: int, kind: int):
        b = self.buf[side][: (3 if kind == ROW_PUSH_STATE else 1) * self.W]
        _lib.check(_lib.load().fm_grid_band_rows(self._h, 0, int(side), int(kind), _lib.ptr(b), None),
                   "fm_grid_band_rows")
        return b

    def rows_in(self, side: int, kind: int, src) -> int:
        out = ctypes.c_int64()
        _lib.check(_lib.load().fm_grid_band_rows(self._h, 1, int(side), int(kind), _lib.ptr(src),
                                                 ctypes.byref(out)), "fm_grid_band_rows")
        return int(out.value)

    def flow(self) -> int:
        out = ctypes.c_int64()
        _lib.check(_lib.load().fm_grid_band_flow(self._h, ctypes.byref(out)), "fm_grid_band_flow")
        return int(out.value)

    def stats(self) -> dict:
        st = _lib.FmStats()
        _lib.check(_lib.load().fm_grid_stats(self._h, ctypes.byref(st)), "fm_grid_stats")
        return st.as_dict()

    def cut_host(self) -> np.ndarray:
        """The current cut plane of this band (ghost rows included), no recompute."""
        cut = np.zeros((self.Hb, self.W), np.uint8)
        _lib.check(_lib.load().fm_grid_cut_plane(self._h, _lib.ptr(cut), 1), "fm_grid_cut_plane")
        return cut

    def export_state(self) -> dict:
        names = ("rR", "rL", "rD", "rU", "rT", "rS", "e", "h")
        out = {k: np.zeros((self.Hb, self.W), np.int32) for k in names}
        marked = np.zeros((self.Hb, self.W), np.uint8)
        _lib.check(_lib.load().fm_grid_export(self._h, *[_lib.ptr(out[k]) for k in names],
                                              _lib.ptr(marked), None, None), "fm_grid_export")
        out["marked"] = marked
        return out


class LocalTransport:
    """All bands in this process (virtual bands; any devices)."""

    def __init__(self, bands: list[Band]):
        self.bands = bands

    def local(self):
        return self.bands

    def exchange(self, kind: int) -> int:
        """Ship row `kind` across every band border; returns imported cells changed."""
        import torch

        changed = 0
        bs = self.bands
        outs = {}
        for k, b in enumerate(bs):
            for side in b.sides():
                outs[(k, side)] = b.rows_out(side, kind).clone()
        torch.cuda.synchronize()
        for k, b in enumerate(bs):
            if b.ghost_top:
                changed += b.rows_in(TOP, kind, outs[(k - 1, BOTTOM)])
            if b.ghost_bot:
                changed += b.rows_in(BOTTOM, kind, outs[(k + 1, TOP)])
        return changed

    def sum(self, values) -> list[int]:
        return [int(v) for v in values]

    def max(self, values) -> list[int]:
        return [int(v) for v in values]


class DistTransport:
    """One band per rank; boundary rows move between neighbouring ranks with
    torch.distributed send/recv (NCCL over NVLink), scalars by all-reduce."""

    def __init__(self, band: Band, rank: int, world: int):
        import torch.distributed as dist

        self.band, self.rank, self.world = band, rank, world
        # gloo moves host tensors only: stage boundary rows through host memory
        self.host_staging = dist.get_backend() == "gloo"

    def local(self):
        return [self.band]

    def exchange(self, kind: int) -> int:
        import torch
        import torch.distributed as dist

        b = self.band
        ops, recv = [], {}
        for side in b.sides():
            peer = self.rank - 1 if side == TOP else self.rank + 1
            out = b.rows_out(side, kind)
            rb = b.rbuf[side][: out.numel()]
            if getattr(self, "host_staging", False):
                out, rb = out.cpu(), torch.empty(rb.shape, dtype=rb.dtype)
            recv[side] = rb
            ops.append(dist.P2POp(dist.isend, out, peer))
            ops.append(dist.P2POp(dist.irecv, rb, peer))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()   # NCCL: the current stream (the bands' stream) waits for the transfers
        if getattr(self, "host_staging", False) and torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        changed = 0
        for side in b.sides():
            src = recv[side]
            if src.device.type == "cpu" and b.rbuf[side].device.type == "cuda":
                dst = b.rbuf[side][: src.numel()]
                dst.copy_(src)
                torch.cuda.current_stream().synchronize()
                src = dst
            changed += b.rows_in(side, kind, src)
        return changed

    def _reduce(self, values, op):
        import torch
        import torch.distributed as dist

        dev = "cpu" if getattr(self, "host_staging", False) else self.band.caps[0].device
        t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=op)
        return [int(v) for v in t.tolist()]

    def sum(self, values):
        import torch.distributed as dist

        return self._reduce(values, dist.ReduceOp.SUM)

    def max(self, values):
        import torch.distributed as dist

        return self._reduce(values, dist.ReduceOp.MAX)


def _total(tr, per_band_values) -> int:
    """Sum of one scalar over all bands (local and, when distributed, remote)."""
    return tr.sum([sum(per_band_values)])[0]


class BandedSolve:
    """Coordinator of a banded solve (identical on every rank / for every transport)."""

    def __init__(self, transport, cycle_budget: int = 7000, launches_per_exchange: int = 4,
                 max_launches: int = 16, relabel_div: int = 16, total_pixels: int | None = None):
        self.tr = transport
        self.cycle_budget = cycle_budget
        self.lpe = launches_per_exchange
        self.max_launches = max_launches
        self.relabel_div = relabel_div
        self.total_pixels = total_pixels
        self.stats = dict(rounds=0, exchanges=0, bfs_exchanges=0, pushes=0, relabels=0)

    def global_relabel(self) -> int:
        bands = self.tr.local()
        for b in bands:
            b.bfs(0)
        while True:
            changed = self.tr.exchange(ROW_DIST)
            self.stats["bfs_exchanges"] += 1
            if _total(self.tr, [changed]) == 0:
                break
            for b in bands:
                b.bfs(1)
        active = 0
        for b in bands:
            a, _, _ = b.finalize()
            active += a
        self.tr.exchange(ROW_H)      # exact heights of the neighbours' boundary rows
        return _total(self.tr, [active])

    def run(self):
        bands = self.tr.local()
        for b in bands:
            b.init()
        self.tr.exchange(ROW_RES)
        active = self.global_relabel()
        budget = max(1024, (self.total_pixels or 1) // self.relabel_div)
        while active > 0:
            batches = relabels = 0
            while True:
                # every decision below uses all-reduced values or the batch count, so
                # all ranks take the same branch (their collectives stay matched)
                idle_all = True
                for b in bands:
                    p, r, _, idle = b.push(self.lpe, self.cycle_budget)
                    self.stats["pushes"] += p
                    self.stats["relabels"] += r
                    relabels += r
                    idle_all &= idle
                batches += 1
                moved = self.tr.exchange(ROW_PUSH_STATE)
                self.stats["exchanges"] += 1
                tot = self.tr.sum([moved, 0 if idle_all else 1, relabels])
                if tot[0] == 0 and tot[1] == 0:
                    break
                if tot[2] >= budget or batches * self.lpe >= self.max_launches:
                    break
            active = self.global_relabel()
            self.stats["rounds"] += 1
        # minimal source-side cut: seeded reach, then boundary exchange to a fixpoint.
        # The ghost rows' residuals toward us must be current first: the RES rows of the
        # last push exchange were exported before that exchange's flow was folded in, so a
        # ghost arc opened by it would be missing from the reach (stress-found: cut short of
        # the minimal one next to band borders, flow correct)
        self.tr.exchange(ROW_RES)
        for b in bands:
            b.cut(0)
        while True:
            changed = self.tr.exchange(ROW_CUT)
            if _total(self.tr, [changed]) == 0:
                break
            for b in bands:
                b.cut(1)
        return _total(self.tr, [sum(b.flow() for b in bands)])


def solve_virtual_bands(caps, nbands: int, device: int = 0, cycle_budget: int = 7000):
    """Solve a host grid split into `nbands` bands on one device (tests / A-B).
    Returns (flow, cut bool[H, W], coordinator stats)."""
    caps = [np.ascontiguousarray(c, dtype=np.int32) for c in caps]
    H, W = caps[4].shape
    spans = band_rows(H, nbands)
    bands = []
    for k, (r0, r1) in enumerate(spans):
        gt, gb = k > 0, k + 1 < len(spans)
        bands.append(Band(band_caps(caps, r0, r1, gt, gb), gt, gb, H * W + 2, device))
    started = time.perf_counter()
    co = BandedSolve(LocalTransport(bands), cycle_budget=cycle_budget, total_pixels=H * W)
    flow = co.run()
    elapsed = time.perf_counter() - started
    cut = np.zeros((H, W), bool)
    for (r0, r1), b in zip(spans, bands):
        c = b.cut_host()
        lo = 1 if b.ghost_top else 0
        cut[r0:r1] = c[lo:lo + (r1 - r0)].astype(bool)
    for b in bands:
        b.close()
    co.stats["elapsed"] = elapsed
    return flow, cut, co.stats


def banded_report(flow, cut, stats) -> SolveReport:
    return SolveReport(objective=flow, pushes=stats.get("pushes", 0), relabels=stats.get("relabels", 0),
                       rounds=stats.get("rounds", 0), elapsed=stats.get("elapsed", 0.0), cut=cut,
                       stats=stats)


def solve_distributed(caps_band, ghost_top: bool, ghost_bot: bool, global_hw: int, rank: int, world: int,
                      device: int, cycle_budget: int = 7000, band=None):
    """This rank's share of a banded solve (torch.distributed must be initialised).
    Returns (flow over all bands, this band, coordinator stats)."""
    if band is None:
        band = Band(caps_band, ghost_top, ghost_bot, global_hw + 2, device)
    started = time.perf_counter()
    co = BandedSolve(DistTransport(band, rank, world), cycle_budget=cycle_budget, total_pixels=global_hw)
    flow = co.run()
    co.stats["elapsed"] = time.perf_counter() - started
    return flow, band, co.stats
