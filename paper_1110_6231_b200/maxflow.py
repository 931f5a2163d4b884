"""Grid max-flow / min-cut: drop-in for the reference's ``hybrid_solve``.

``hybrid_solve(net, worker_count=4, cycle_budget=7000, observer=None)`` keeps the
reference signature, defaults and return type (maxflow_par.py:157-238).  On a
:class:`GridNetwork` it runs the CUDA path in libfm_b200.so; the result carries the
flow value in ``objective`` (= excess at t, maxflow_par.py:233) plus the minimal
source-side cut in ``report.cut``.  Any other ``FlowNetwork`` runs the generic
CSR lock-free kernel (fm_csr.cu).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import FlowNetwork, GridNetwork, SolveReport, _device_planes

DEFAULT_CYCLE_BUDGET = 7000  # maxflow_par.py:28
DEFAULT_BFS_INTERVAL = 0     # 0 = library default sweeps between global relabels


class GridSolver:
    """Reusable device workspace for H x W grids (owns the C handle).

    The SoA state (9 int32 planes + 3 byte planes, ~40 B/pixel) is allocated once
    and reused across solves of the same shape.  options: kernel-variant / tuning
    switches passed to fm_grid_set_option (the library reads no environment).
    """

    def __init__(self, H: int, W: int, device: int = 0, options: dict | None = None):
        L = _lib.load()
        _lib.require_device()
        h = ctypes.c_void_p()
        _lib.check(L.fm_grid_create(int(H), int(W), int(device), ctypes.byref(h)), "fm_grid_create")
        self.H, self.W, self.device = int(H), int(W), int(device)
        self._h = h
        self.last_stats: dict = {}
        for k, v in (options or {}).items():
            self.set_option(k, v)

    def set_option(self, name: str, value: int) -> None:
        """Kernel-variant / tuning switch, from the next solve."""
        _lib.check(_lib.load().fm_grid_set_option(self._h, name.encode(), int(value)), "fm_grid_set_option")

    def close(self) -> None:
        if self._h:
            _lib.load().fm_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _flags(self, cancel_violations=False, want_cut=True, precancel=True, global_sweep=False) -> int:
        f = _lib.FM_GRID_GLOBAL_SWEEP if global_sweep else 0
        if cancel_violations:
            f |= _lib.FM_GRID_CANCEL_VIOLATIONS
        if not want_cut:
            f |= _lib.FM_GRID_NO_CUT
        if not precancel:
            f |= _lib.FM_GRID_NO_PRECANCEL
        return f

    def solve_host(self, caps, cycle_budget=DEFAULT_CYCLE_BUDGET, bfs_interval=DEFAULT_BFS_INTERVAL,
                   want_cut=True, cancel_violations=False, precancel=True, global_sweep=False):
        """Host int32 planes in, (flow, cut bool[H,W] or None, stats) out; the
        host<->device copies are part of the call."""
        caps = [np.ascontiguousarray(a, dtype=np.int32) for a in caps]
        flow = ctypes.c_int64()
        # bool and uint8 share the 0/1 byte layout: the cut lands in its final array
        cut = np.empty((self.H, self.W), np.bool_) if want_cut else None
        st = _lib.FmStats()
        rc = _lib.load().fm_grid_solve_host(
            self._h, *[_lib.ptr(a) for a in caps], int(cycle_budget), int(bfs_interval),
            self._flags(cancel_violations, want_cut, precancel, global_sweep), ctypes.byref(flow),
            _lib.ptr(cut) if want_cut else None, ctypes.byref(st))
        _lib.check(rc, "fm_grid_solve_host")
        self.last_stats = st.as_dict()
        return int(flow.value), cut, self.last_stats

    def solve_host_batch(self, caps_list, cycle_budget=DEFAULT_CYCLE_BUDGET, bfs_interval=DEFAULT_BFS_INTERVAL,
                         want_cut=True, cancel_violations=False, precancel=True):
        """Several same-shape instances from host planes in one pipelined call
        (fm_grid_solve_host_batch: the H2D of instance k+1 and the cut D2H of instance
        k-1 overlap the solve of instance k).  Returns [(flow, cut, stats)], each equal
        to solve_host's result for that instance."""
        planes = []
        caps_list = list(caps_list)
        # uint8 / uint16 planes (all of one dtype) cross PCIe narrow, widened on the device
        dts = {getattr(a, "dtype", None) for caps in caps_list for a in caps}
        narrow = next(iter(dts)) if len(dts) == 1 and next(iter(dts)) in (np.uint8, np.uint16) else None
        for caps in caps_list:
            if len(caps) != 6:
                raise ValueError("each instance needs the six planes capR, capL, capD, capU, capS, capT")
            cs = [np.ascontiguousarray(a, dtype=narrow or np.int32) for a in caps]
            for a in cs:
                if a.shape != (self.H, self.W):
                    raise ValueError(f"plane shape {a.shape} does not match the solver's {(self.H, self.W)}")
            planes.append(cs)
        n = len(planes)
        eb = np.dtype(narrow).itemsize if narrow is not None else 4
        ptrs = (ctypes.c_void_p * max(1, 6 * n))(*[_lib.ptr(a) for cs in planes for a in cs])
        flows = np.zeros(max(1, n), np.int64)
        cuts = [np.empty((self.H, self.W), np.bool_) for _ in range(n)] if want_cut else None
        cptr = (ctypes.c_void_p * max(1, n))(*[_lib.ptr(c) for c in cuts]) if want_cut else None
        sts = (_lib.FmStats * max(1, n))()
        rc = _lib.load().fm_grid_solve_host_batch(
            self._h, n, ptrs, int(eb), int(cycle_budget), int(bfs_interval),
            self._flags(cancel_violations, want_cut, precancel), _lib.ptr(flows), cptr, sts)
        _lib.check(rc, "fm_grid_solve_host_batch")
        out = [(int(flows[k]), cuts[k] if want_cut else None, sts[k].as_dict()) for k in range(n)]
        if out:
            self.last_stats = out[-1][2]
        return out

    def solve_device(self, caps, cycle_budget=DEFAULT_CYCLE_BUDGET, bfs_interval=DEFAULT_BFS_INTERVAL,
                     cut_out=None, cancel_violations=False, precancel=True, stream=None,
                     global_sweep=False):
        """Device int32 tensors in (borrowed); cut_out = uint8 CUDA tensor or None.
        Runs on `stream` (a torch.cuda.Stream or raw handle; default: the
        library's own stream)."""
        flow = ctypes.c_int64()
        st = _lib.FmStats()
        s = None
        if stream is not None:
            s = int(getattr(stream, "cuda_stream", stream))
        rc = _lib.load().fm_grid_solve(
            self._h, *[_lib.ptr(a) for a in caps], int(cycle_budget), int(bfs_interval),
            self._flags(cancel_violations, cut_out is not None, precancel, global_sweep), ctypes.byref(flow),
            _lib.ptr(cut_out) if cut_out is not None else None, ctypes.byref(st), s)
        _lib.check(rc, "fm_grid_solve")
        self.last_stats = st.as_dict()
        return int(flow.value), self.last_stats

    # ---- stepwise (observer) API
    def begin(self, caps, cancel_violations=False, precancel=True):
        caps = [np.ascontiguousarray(a, dtype=np.int32) for a in caps]
        self._keep = caps
        _lib.check(_lib.load().fm_grid_begin(self._h, *[_lib.ptr(a) for a in caps],
                                             self._flags(cancel_violations, True, precancel)),
                   "fm_grid_begin")

    def round(self, cycle_budget=DEFAULT_CYCLE_BUDGET, bfs_interval=DEFAULT_BFS_INTERVAL) -> bool:
        done = ctypes.c_int32()
        st = _lib.FmStats()
        _lib.check(_lib.load().fm_grid_round(self._h, int(cycle_budget), int(bfs_interval),
                                             ctypes.byref(done), ctypes.byref(st)), "fm_grid_round")
        self.last_stats = st.as_dict()
        return bool(done.value)

    def export(self) -> dict:
        H, W = self.H, self.W
        names = ("rR", "rL", "rD", "rU", "rT", "rS", "e", "h")
        out = {k: np.zeros((H, W), np.int32) for k in names}
        marked = np.zeros((H, W), np.uint8)
        flow = ctypes.c_int64()
        et = ctypes.c_int64()
        _lib.check(_lib.load().fm_grid_export(self._h, *[_lib.ptr(out[k]) for k in names],
                                              _lib.ptr(marked), ctypes.byref(flow), ctypes.byref(et)),
                   "fm_grid_export")
        out["marked"] = marked
        out["flow"] = int(flow.value)
        out["excess_total"] = int(et.value)
        return out

    def cut_host(self) -> np.ndarray:
        cut = np.zeros((self.H, self.W), np.uint8)
        st = _lib.FmStats()
        _lib.check(_lib.load().fm_grid_cut_host(self._h, _lib.ptr(cut), ctypes.byref(st)), "fm_grid_cut_host")
        self.last_stats = st.as_dict()
        return cut


_solvers = _lib.SolverCache(per_device=1)   # grids are large: one cached workspace per device


# ---------------------------------------------------------------- observer mirror

@dataclass
class _StateView:
    """Reference-shaped ResidualState view (graph.py:128-154) of a grid state."""

    residual: list
    excess: list
    height: list
    price: list


@dataclass
class GridHybridState:
    """Reference-shaped HybridState (maxflow_par.py:31-41) at a coordinator point."""

    state: _StateView
    excess_total: int
    cycle_budget: int = DEFAULT_CYCLE_BUDGET
    worker_count: int = 1
    marked: list = field(default_factory=list)


def _slot_residuals(net: GridNetwork, st: dict) -> np.ndarray:
    """Map the merged-pair device state onto the reference arc slots (adapter order).

    A merged pair (p->q cap a, q->p cap b) with net flow phi = a - r(p->q) is
    decomposed as flow max(phi, 0) on p->q and max(-phi, 0) on q->p."""
    capR, capL, capD, capU, capS, capT = net.host_caps()
    H, W = net.H, net.W
    HW = H * W
    p = np.arange(HW)
    r, c = p // W, p % W
    cols = np.zeros((HW, 12), np.int64)
    keep = np.zeros((HW, 12), bool)
    fS, fT = capS.reshape(-1), capT.reshape(-1)
    rS, rT = st["rS"].reshape(-1), st["rT"].reshape(-1)
    keep[:, 0:2] = (fS > 0)[:, None]
    cols[:, 0], cols[:, 1] = fS - rS, rS
    keep[:, 2:4] = (fT > 0)[:, None]
    cols[:, 2], cols[:, 3] = rT, fT - rT
    hasR = c + 1 < W
    keep[:, 4:8] = hasR[:, None]
    q = np.minimum(p + 1, HW - 1)
    a, b = capR.reshape(-1), capL.reshape(-1)[q]
    phi = a - st["rR"].reshape(-1)
    f1, f2 = np.maximum(phi, 0), np.maximum(-phi, 0)
    cols[:, 4], cols[:, 5], cols[:, 6], cols[:, 7] = a - f1, f1, b - f2, f2
    hasD = r + 1 < H
    keep[:, 8:12] = hasD[:, None]
    q = np.minimum(p + W, HW - 1)
    a, b = capD.reshape(-1), capU.reshape(-1)[q]
    phi = a - st["rD"].reshape(-1)
    f1, f2 = np.maximum(phi, 0), np.maximum(-phi, 0)
    cols[:, 8], cols[:, 9], cols[:, 10], cols[:, 11] = a - f1, f1, b - f2, f2
    return cols.reshape(-1)[keep.reshape(-1)]


def _observe(net: GridNetwork, solver: GridSolver, observer, cycle_budget, worker_count):
    st = solver.export()
    HW = net.H * net.W
    V = HW + 2
    excess = st["e"].reshape(-1).astype(np.int64).tolist() + [0, st["flow"]]
    height = st["h"].reshape(-1).astype(np.int64).tolist() + [V, 0]
    marked = st["marked"].reshape(-1).astype(bool).tolist() + [False, False]
    residual = _slot_residuals(net, st).tolist() if net._materialised else None
    hybrid = GridHybridState(
        state=_StateView(residual=residual, excess=excess, height=height, price=[0] * V),
        excess_total=st["excess_total"], cycle_budget=cycle_budget, worker_count=worker_count,
        marked=marked)
    scanned = [not m for m in marked]
    scanned[HW] = True
    observer(net, hybrid, scanned)


def hybrid_solve(net: FlowNetwork, worker_count: int = 4, cycle_budget: int = DEFAULT_CYCLE_BUDGET,
                 observer=None, *, device: int | None = None, bfs_interval: int = DEFAULT_BFS_INTERVAL,
                 cancel_violations: bool = False, want_cut: bool = True, devices=None) -> SolveReport:
    """Coordinated lock-free push-relabel rounds until all live excess is at t
    (maxflow_par.py:157-238), on the GPU.

    worker_count keeps its validation but has no effect on the device (one CUDA
    thread owns each pixel).  cycle_budget = max lock-free sweeps per round.
    observer(net, hybrid, scanned) is called at every coordinator point with
    reference-shaped state (slow: state is copied to the host; tests only).
    devices: shard a grid in row bands -- an int N (N bands over the
    visible GPUs, round-robin) or a list of device ids, one band each (a device may
    repeat: virtual bands).  Same flow and minimal cut as the single-GPU solve.
    """
    if net.source is None or net.sink is None:
        raise ValueError("network has no source/sink")
    if worker_count < 1:
        raise ValueError(f"worker_count must be at least 1, got {worker_count}")
    if cycle_budget < 1:
        raise ValueError(f"cycle_budget must be at least 1, got {cycle_budget}")
    if devices is not None:
        devs = _band_devices(devices)
        if len(devs) > 1:
            return _banded_solve(net, devs, cycle_budget, observer, cancel_violations, want_cut)
        device = devs[0] if device is None else device
    if not isinstance(net, GridNetwork):
        if observer is not None:
            raise NotImplementedError("observer hooks are supported on GridNetwork solves")
        return csr_solve(net, cycle_budget)
    if net.wide:
        return _wide_grid_solve(net, cycle_budget, observer, cancel_violations, want_cut, device)
    started = time.perf_counter()
    caps = net.caps
    if net.on_device:
        caps = _device_planes(caps)
        dev = caps[0].device.index or 0
        if device is not None and int(device) != dev:
            raise ValueError(f"device={device} but the capacity planes are on cuda:{dev}")
        device = dev
    elif device is None:
        device = 0
    with _solvers.use((net.H, net.W, device), device, lambda: GridSolver(net.H, net.W, device)) as solver:
        if observer is None:
            if net.on_device:
                import torch

                cut_t = torch.empty((net.H, net.W), dtype=torch.uint8, device=caps[0].device) if want_cut else None
                flow, stats = solver.solve_device(caps, cycle_budget, bfs_interval, cut_out=cut_t,
                                                  cancel_violations=cancel_violations,
                                                  stream=torch.cuda.current_stream(caps[0].device))
                cut = cut_t.bool() if cut_t is not None else None
            elif net.narrow_bytes:
                # uint8 / uint16 planes: narrow H2D + device widening (one-instance batch)
                flow, cut, stats = solver.solve_host_batch([net.caps], cycle_budget, bfs_interval, want_cut=want_cut,
                                                           cancel_violations=cancel_violations)[0]
            else:
                try:
                    flow, cut, stats = solver.solve_host(net.host_caps(), cycle_budget, bfs_interval,
                                                         want_cut=want_cut, cancel_violations=cancel_violations)
                except ValueError as exc:
                    if _INT32_STATE_MSG not in str(exc):
                        raise
                    # int32 planes whose per-pixel sums leave the grid kernel's int32 state
                    return _wide_grid_solve(net, cycle_budget, None, cancel_violations, want_cut, device)
        else:
            solver.begin(net.host_caps(), cancel_violations=cancel_violations)
            while True:
                st = solver.export()
                if int(((st["e"] > 0) & (st["marked"] == 0)).sum()) == 0:
                    break
                done = solver.round(cycle_budget, bfs_interval)
                _observe(net, solver, observer, cycle_budget, worker_count)
                if done:
                    break
            st = solver.export()
            flow = st["flow"]
            stats = dict(solver.last_stats)
            cut = solver.cut_host().astype(bool) if want_cut else None
    elapsed = time.perf_counter() - started
    return SolveReport(objective=int(flow), pushes=int(stats.get("pushes", 0)),
                       relabels=int(stats.get("relabels", 0)), rounds=int(stats.get("rounds", 0)),
                       elapsed=elapsed, cut=cut, stats=stats)


def hybrid_solve_batch(nets, worker_count: int = 4, cycle_budget: int = DEFAULT_CYCLE_BUDGET, *,
                       device: int | None = None, bfs_interval: int = DEFAULT_BFS_INTERVAL,
                       cancel_violations: bool = False, want_cut: bool = True) -> list[SolveReport]:
    """hybrid_solve over a sequence of same-shape host GridNetworks (a stream of images):
    one pipelined device call in which the host->device copy of network k+1 and the
    cut copy-back of network k-1 overlap the solve of network k.  Returns one
    SolveReport per network, each equal to hybrid_solve(net)'s; `elapsed` of each is
    the whole call's time divided by the count."""
    nets = list(nets)
    if worker_count < 1:
        raise ValueError(f"worker_count must be at least 1, got {worker_count}")
    if cycle_budget < 1:
        raise ValueError(f"cycle_budget must be at least 1, got {cycle_budget}")
    if not nets:
        return []
    for net in nets:
        if not isinstance(net, GridNetwork):
            raise ValueError("hybrid_solve_batch takes GridNetworks")
        if net.source is None or net.sink is None:
            raise ValueError("network has no source/sink")
        if net.on_device or net.wide:
            raise ValueError("hybrid_solve_batch takes host int32 grids (use hybrid_solve for device or wide ones)")
        if (net.H, net.W) != (nets[0].H, nets[0].W):
            raise ValueError("hybrid_solve_batch needs networks of one shape")
    H, W = nets[0].H, nets[0].W
    device = 0 if device is None else int(device)
    started = time.perf_counter()
    with _solvers.use((H, W, device), device, lambda: GridSolver(H, W, device)) as solver:
        narrow = all(net.narrow_bytes for net in nets) and len({net.caps[0].dtype for net in nets}) == 1
        res = solver.solve_host_batch([net.caps if narrow else net.host_caps() for net in nets], cycle_budget, bfs_interval,
                                      want_cut=want_cut, cancel_violations=cancel_violations)
    per = (time.perf_counter() - started) / len(nets)
    return [SolveReport(objective=int(f), pushes=int(st.get("pushes", 0)), relabels=int(st.get("relabels", 0)),
                        rounds=int(st.get("rounds", 0)), elapsed=per, cut=cut, stats=st) for f, cut, st in res]


_groups = _lib.SolverCache(per_device=1)

# fm_grid's refusal of inputs past its int32 state (fm_grid.cu, grid_init_kernel)
_INT32_STATE_MSG = "too large for the int32 device state"


def _wide_grid_solve(net: GridNetwork, cycle_budget, observer, cancel_violations, want_cut, device) -> SolveReport:
    """A grid whose capacities (or per-pixel sums) leave int32: the reference's
    capacities are unbounded ints (graph.py:87-125), so the grid's arc-pair network
    runs on the int64 generic kernel (fm_csr_solve64); the cut maps back to H x W."""
    if observer is not None:
        raise NotImplementedError("observer hooks need int32 grid capacities")
    if cancel_violations:
        raise ValueError("cancel_violations needs int32 grid capacities")
    tl, hd, cp = net.arc_arrays()
    rep = _csr_run(net.node_count, net.source, net.sink, tl, hd, cp, cycle_budget, False, device or 0)
    cut = rep.cut[: net.H * net.W].reshape(net.H, net.W) if want_cut else None
    rep.stats["layout"] = "csr64"
    return SolveReport(objective=rep.objective, pushes=rep.pushes, relabels=rep.relabels, rounds=rep.rounds,
                       elapsed=rep.elapsed, cut=cut, stats=rep.stats)


def _band_devices(devices) -> list[int]:
    if isinstance(devices, (int, np.integer)):
        n = int(devices)
        if n < 1:
            raise ValueError(f"devices must be at least 1, got {n}")
        ndev = max(1, _lib.device_count())
        return [k % ndev for k in range(n)]
    devs = [int(d) for d in devices]
    if not devs:
        raise ValueError("devices must name at least one device")
    return devs


def _banded_solve(net, devs, cycle_budget, observer, cancel_violations, want_cut) -> SolveReport:
    """hybrid_solve over row bands (one per entry of devs), paper_1110_6231_b200.bands."""
    from .bands import BandGroup

    if not isinstance(net, GridNetwork):
        raise ValueError("devices > 1 shards grid networks in row bands; this network is not a GridNetwork")
    if observer is not None:
        raise NotImplementedError("observer hooks run on single-device solves (devices=None)")
    if cancel_violations:
        raise ValueError("cancel_violations is a single-device option")
    started = time.perf_counter()
    caps = _device_planes(net.caps) if net.on_device else net.host_caps()
    key = (net.H, net.W, tuple(devs))
    with _groups.use(key, -1, lambda: BandGroup(net.H, net.W, len(devs), devs)) as grp:
        flow, cut, stats = grp.solve(caps, cycle_budget, want_cut=want_cut)
    stats["devices"] = list(devs)
    return SolveReport(objective=int(flow), pushes=int(stats.get("pushes", 0)),
                       relabels=int(stats.get("relabels", 0)), rounds=int(stats.get("rounds", 0)),
                       elapsed=time.perf_counter() - started, cut=cut, stats=stats)


def csr_arrays(net: FlowNetwork):
    """(ostart, oarc, head, cap) of a FlowNetwork's arc-pair forward star
    (graph.py:43-84): out-arc lists keep input order; cap is int64."""
    tails = np.asarray(net.tail, dtype=np.int64)[0::2]
    heads = np.asarray(net.head, dtype=np.int64)[0::2]
    try:
        cap = np.asarray(net.capacity[0::2], dtype=np.int64)
    except OverflowError:
        raise ValueError("capacity beyond 2^63 is not supported on the device") from None
    return _forward_star(net.node_count, tails, heads, cap)


def _forward_star(n, tails, heads, cap):
    """CSR of the arc pairs (tails[k] -> heads[k], cap[k]): slot 2k forward, 2k+1 its
    reverse (capacity 0); each node's out-slots in slot order (graph.py:64-73)."""
    m = len(tails)
    slot_tail = np.empty(2 * m, np.int64)
    slot_tail[0::2], slot_tail[1::2] = tails, heads
    head = np.empty(2 * m, np.int32)
    head[0::2], head[1::2] = heads, tails
    cap2 = np.zeros(2 * m, np.int64)
    cap2[0::2] = cap
    oarc = np.argsort(slot_tail, kind="stable").astype(np.int32)
    ostart = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(slot_tail, minlength=n), out=ostart[1:])
    return ostart, oarc, head, cap2


def csr_solve(net: FlowNetwork, cycle_budget: int = DEFAULT_CYCLE_BUDGET, want_state: bool = False):
    """Generic-graph lock-free push-relabel on the GPU (fm_csr.cu).  Returns a
    SolveReport whose cut is a bool[node_count] (True = source side).  Capacities
    past int32 run with int64 residuals (fm_csr_solve64)."""
    if net.source is None or net.sink is None:
        raise ValueError("network has no source/sink")
    tails = np.asarray(net.tail, dtype=np.int64)[0::2]
    heads = np.asarray(net.head, dtype=np.int64)[0::2]
    try:
        cap = np.asarray(net.capacity[0::2], dtype=np.int64)
    except OverflowError:
        raise ValueError("capacity beyond 2^63 is not supported on the device") from None
    return _csr_run(net.node_count, net.source, net.sink, tails, heads, cap, cycle_budget, want_state, 0)


def _csr_run(n, source, sink, tails, heads, cap, cycle_budget, want_state, device):
    L = _lib.load()
    _lib.require_device()
    started = time.perf_counter()
    ostart, oarc, head, cap2 = _forward_star(n, np.asarray(tails, np.int64), np.asarray(heads, np.int64),
                                             np.asarray(cap, np.int64))
    m2 = len(head)
    wide = bool(m2) and int(cap2.max()) >= 2**31
    if wide:
        if int(cap2.max()) >= 2**62:
            raise ValueError("capacity beyond 2^62 is not supported on the device")
        if sum(int(c) for c in cap2[oarc[ostart[source]:ostart[source + 1]]]) >= 2**63:
            raise ValueError("total capacity out of the source beyond 2^63-1 is not supported on the device")
    else:
        cap2 = cap2.astype(np.int32)
    rdt = np.int64 if wide else np.int32
    flow = ctypes.c_int64()
    cut = np.zeros(n, np.uint8)
    res = np.zeros(max(1, m2), rdt) if want_state else None
    ex = np.zeros(n, np.int64) if want_state else None
    st = _lib.FmStats()
    p = lambda a: _lib.ptr(a) if a is not None and a.size else None
    fn = L.fm_csr_solve64 if wide else L.fm_csr_solve
    if device:
        raise NotImplementedError("the generic (CSR) kernel runs on device 0")
    rc = fn(n, int(source), int(sink), m2, _lib.ptr(ostart), p(oarc), p(head), p(cap2),
            int(cycle_budget), 0, ctypes.byref(flow), _lib.ptr(cut), p(res), p(ex), ctypes.byref(st))
    _lib.check(rc, "fm_csr_solve64" if wide else "fm_csr_solve")
    stats = st.as_dict()
    stats["residual_bits"] = 64 if wide else 32
    if want_state:
        stats["residual"], stats["excess"] = res[:m2], ex
    return SolveReport(objective=int(flow.value), pushes=int(st.pushes), relabels=int(st.relabels),
                       rounds=int(st.rounds), elapsed=time.perf_counter() - started, cut=cut.astype(bool),
                       stats=stats)


def min_cut(net: GridNetwork, report: SolveReport | None = None, **kw):
    """Minimal source side of a minimum cut (bool H x W; True = source side)."""
    if report is None or report.cut is None:
        report = hybrid_solve(net, **kw)
    return report.cut
