"""Row-band sharding of the grid max-flow / min-cut across GPUs.

The H x W grid is cut into horizontal bands whose borders sit on 32-row tile
boundaries; band k lives on its own device (or several bands share one: virtual
bands).  Nothing moves by message.  A band's kernels read the neighbour bands'
boundary rows -- heights when choosing a push, BFS distances in the global relabel,
cut bits in the min-cut reach -- directly from the neighbours' memory, push flow
into their inboxes with remote atomics and raise their external-push flags, and
queue their ring-BFS tiles; the bands' persistent ring launches all end on one
shared pending counter.  The host side of each band runs the reference's
coordinator loop (maxflow_par.py:195-229) in C++ (fm_grid_band_solve) and agrees
with the other bands through an fm_coll: a shared-memory barrier + all-gather of a
few int64 per push batch (idle / flow in flight / relabel budget) and per relabel
(active pixels).

Two ways to run it:

* :class:`BandGroup` -- one process drives every band, one host thread per band
  (``hybrid_solve(net, devices=N)``; virtual bands on one GPU in the tests).
* :class:`DistBand` -- one process per GPU (torchrun): the bands exchange CUDA IPC
  handles of their buffers and the name of the shared-memory segment through
  ``torch.distributed`` once, at set-up; the solve itself uses no collective.
"""

from __future__ import annotations

import ctypes
import os
import time
import uuid

import numpy as np

from . import _lib
from .graph import SolveReport

TILE = 32
EXPORT_BYTES = 1024   # FM_BAND_EXPORT_BYTES


def band_rows(H: int, nbands: int) -> list[tuple[int, int]]:
    """Split H rows into nbands contiguous bands on 32-row tile boundaries (the last
    band takes the remainder); the same split as the library's fm_band_split."""
    if nbands < 1 or H < 1:
        raise ValueError("nbands and H must be >= 1")
    tiles = (H + TILE - 1) // TILE
    if nbands > tiles:
        raise ValueError(f"cannot split {H} rows ({tiles} tile rows) into {nbands} bands")
    edges = [min(H, ((k * tiles + nbands // 2) // nbands) * TILE) for k in range(nbands + 1)]
    edges[-1] = H
    out = [(edges[k], edges[k + 1]) for k in range(nbands)]
    if any(r1 <= r0 for r0, r1 in out):
        raise ValueError(f"empty band in split of {H} rows into {nbands}")
    return out


def band_planes(caps, r0: int, r1: int):
    """Inputs of band [r0, r1): the six planes' rows, capD of the row above the band
    and capU of the row below it (None at the grid's top / bottom)."""
    caps = [np.asarray(a) for a in caps]
    rows = [np.ascontiguousarray(a[r0:r1], dtype=np.int32) for a in caps]
    H = caps[0].shape[0]
    above = np.ascontiguousarray(caps[2][r0 - 1], dtype=np.int32) if r0 > 0 else None
    below = np.ascontiguousarray(caps[3][r1], dtype=np.int32) if r1 < H else None
    return rows, above, below


def _stats(st: _lib.FmStats) -> dict:
    return st.as_dict()


class BandGroup:
    """Every band of an H x W grid in this process (fm_group): band k on devices[k]."""

    def __init__(self, H: int, W: int, nbands: int, devices=None):
        L = _lib.load()
        _lib.require_device()
        ndev = _lib.device_count()
        if devices is None:
            devices = [k % ndev for k in range(nbands)]
        devices = [int(d) for d in devices]
        if len(devices) != nbands or any(d < 0 or d >= ndev for d in devices):
            raise ValueError(f"devices {devices} do not name {nbands} visible devices (have {ndev})")
        self.H, self.W, self.nbands, self.devices = int(H), int(W), int(nbands), devices
        self.spans = band_rows(self.H, self.nbands)
        h = ctypes.c_void_p()
        arr = (ctypes.c_int32 * nbands)(*devices)
        _lib.check(L.fm_group_create(self.H, self.W, self.nbands, arr, ctypes.byref(h)), "fm_group_create")
        self._h = h

    def set_option(self, name: str, value: int) -> None:
        L = _lib.load()
        for k in range(self.nbands):
            b = ctypes.c_void_p()
            _lib.check(L.fm_group_band(self._h, k, ctypes.byref(b), None, None), "fm_group_band")
            _lib.check(L.fm_grid_set_option(b, name.encode(), int(value)), "fm_grid_set_option")

    def solve(self, caps, cycle_budget: int = 7000, want_cut: bool = True, precancel: bool = True,
              cut_out=None):
        """caps: six H x W int32 planes (numpy, or torch tensors on any device).
        Returns (flow, cut bool[H, W] or the filled cut_out, stats)."""
        L = _lib.load()
        planes = [c if hasattr(c, "data_ptr") else np.ascontiguousarray(c, dtype=np.int32) for c in caps]
        for c in planes:
            if tuple(c.shape) != (self.H, self.W):
                raise ValueError(f"capacity plane of shape {tuple(c.shape)}, expected {(self.H, self.W)}")
        cut = None
        if want_cut:
            cut = cut_out if cut_out is not None else np.zeros((self.H, self.W), np.uint8)
        flags = (0 if want_cut else _lib.FM_GRID_NO_CUT) | (0 if precancel else _lib.FM_GRID_NO_PRECANCEL)
        flow = ctypes.c_int64()
        st = _lib.FmStats()
        rc = L.fm_group_solve(self._h, *[_lib.ptr(c) for c in planes], int(cycle_budget), flags,
                              ctypes.byref(flow), _lib.ptr(cut) if cut is not None else None, ctypes.byref(st))
        _lib.check(rc, "fm_group_solve")
        if cut is not None and cut_out is None:
            cut = cut.astype(bool)
        return int(flow.value), cut, _stats(st)

    def band_stats(self, k: int) -> dict:
        st = _lib.FmStats()
        _lib.check(_lib.load().fm_group_band_stats(self._h, int(k), ctypes.byref(st)), "fm_group_band_stats")
        return _stats(st)

    def close(self) -> None:
        if self._h:
            _lib.load().fm_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_virtual_bands(caps, nbands: int, device: int = 0, cycle_budget: int = 7000):
    """Solve a host grid split into `nbands` bands that all live on one device (tests,
    A/B).  Returns (flow, cut bool[H, W], stats)."""
    caps = [np.ascontiguousarray(c, dtype=np.int32) for c in caps]
    H, W = caps[4].shape
    started = time.perf_counter()
    grp = BandGroup(H, W, nbands, [device] * nbands)
    try:
        flow, cut, st = grp.solve(caps, cycle_budget)
    finally:
        grp.close()
    st["elapsed"] = time.perf_counter() - started
    return flow, cut, st


def banded_report(flow, cut, stats) -> SolveReport:
    return SolveReport(objective=flow, pushes=stats.get("pushes", 0), relabels=stats.get("relabels", 0),
                       rounds=stats.get("rounds", 0), elapsed=stats.get("elapsed", 0.0), cut=cut,
                       stats=stats)


class DistBand:
    """This rank's band of a grid cut into `world` bands, one process per GPU
    (torch.distributed must be initialised; any backend).  Set-up exchanges the CUDA
    IPC handles of every band's buffers and the shared-memory segment's name; the
    solve needs no collective of torch.distributed."""

    def __init__(self, H: int, W: int, rank: int, world: int, device: int, colocated: int = 1):
        import torch.distributed as dist

        L = _lib.load()
        _lib.require_device()
        self.H, self.W, self.rank, self.world, self.device = int(H), int(W), int(rank), int(world), int(device)
        self.spans = band_rows(self.H, self.world)
        self.r0, self.r1 = self.spans[self.rank]
        h = ctypes.c_void_p()
        _lib.check(L.fm_grid_create(self.r1 - self.r0, self.W, self.device, ctypes.byref(h)), "fm_grid_create")
        self._h = h
        self._coll = None
        _lib.check(L.fm_grid_band_setup(h, self.rank, self.world, self.H, int(colocated)), "fm_grid_band_setup")
        blob = ctypes.create_string_buffer(EXPORT_BYTES)
        _lib.check(L.fm_grid_band_export(h, blob), "fm_grid_band_export")
        name = f"/fm_coll_{uuid.uuid4().hex[:16]}" if self.rank == 0 else None
        got = [None] * self.world
        dist.all_gather_object(got, (blob.raw, name))
        blobs = [g[0] for g in got]
        self.shm_name = got[0][1]
        up = blobs[self.rank - 1] if self.rank > 0 else None
        dn = blobs[self.rank + 1] if self.rank + 1 < self.world else None
        _lib.check(L.fm_grid_band_link(h, up, dn, blobs[0]), "fm_grid_band_link")
        c = ctypes.c_void_p()
        if self.rank == 0:
            _lib.check(L.fm_coll_create(self.shm_name.encode(), self.world, 0, ctypes.byref(c)), "fm_coll_create")
        dist.barrier()
        if self.rank != 0:
            _lib.check(L.fm_coll_create(self.shm_name.encode(), self.world, self.rank, ctypes.byref(c)),
                       "fm_coll_create")
        self._coll = c
        dist.barrier()   # every rank has the segment open (rank 0 may unlink it on close)

    def set_option(self, name: str, value: int) -> None:
        _lib.check(_lib.load().fm_grid_set_option(self._h, name.encode(), int(value)), "fm_grid_set_option")

    def solve(self, rows, above=None, below=None, cycle_budget: int = 7000, want_cut: bool = True,
              cut_out=None):
        """rows: the six planes of this band's rows (numpy or torch, any device);
        above / below: capD of the row above, capU of the row below (W).  Every rank
        calls it at once.  Returns (flow of the whole grid, cut rows of this band, stats)."""
        L = _lib.load()
        planes = [c if hasattr(c, "data_ptr") else np.ascontiguousarray(c, dtype=np.int32) for c in rows]
        Hb = self.r1 - self.r0
        for c in planes:
            if tuple(c.shape) != (Hb, self.W):
                raise ValueError(f"band plane of shape {tuple(c.shape)}, expected {(Hb, self.W)}")
        if (self.rank > 0) != (above is not None) or (self.rank + 1 < self.world) != (below is not None):
            raise ValueError("above / below rows must be given exactly where the band has a neighbour")
        conv = lambda a: None if a is None else (a if hasattr(a, "data_ptr") else np.ascontiguousarray(a, dtype=np.int32))
        above, below = conv(above), conv(below)
        cut = None
        if want_cut:
            cut = cut_out if cut_out is not None else np.zeros((Hb, self.W), np.uint8)
        flow = ctypes.c_int64()
        st = _lib.FmStats()
        rc = L.fm_grid_band_solve(self._h, self._coll, *[_lib.ptr(c) for c in planes],
                                  _lib.ptr(above) if above is not None else None,
                                  _lib.ptr(below) if below is not None else None, int(cycle_budget),
                                  0 if want_cut else _lib.FM_GRID_NO_CUT, ctypes.byref(flow),
                                  _lib.ptr(cut) if cut is not None else None, ctypes.byref(st))
        _lib.check(rc, "fm_grid_band_solve")
        return int(flow.value), cut, _stats(st)

    def close(self) -> None:
        L = _lib.load()
        if self._coll:
            L.fm_coll_destroy(self._coll)
            self._coll = None
        if self._h:
            L.fm_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Coll:
    """The shared-memory barrier + all-gather on its own (host logic; no GPU)."""

    def __init__(self, name: str | None, nranks: int, rank: int):
        c = ctypes.c_void_p()
        _lib.check(_lib.load().fm_coll_create(name.encode() if name else None, int(nranks), int(rank),
                                              ctypes.byref(c)), "fm_coll_create")
        self._c, self.nranks = c, int(nranks)

    def allgather(self, vals) -> list[list[int]]:
        v = (ctypes.c_int64 * len(vals))(*[int(x) for x in vals])
        out = (ctypes.c_int64 * (len(vals) * self.nranks))()
        _lib.check(_lib.load().fm_coll_allgather(self._c, v, len(vals), out), "fm_coll_allgather")
        n = len(vals)
        return [list(out[r * n:(r + 1) * n]) for r in range(self.nranks)]

    def close(self) -> None:
        if self._c:
            _lib.load().fm_coll_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
