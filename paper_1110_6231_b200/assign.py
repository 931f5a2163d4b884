"""Dense assignment by cost scaling: drop-in for the reference's ``solve_assignment``.

Same names, keyword arguments, defaults, return value ``(SolveReport, matching)``
and exceptions as assign_scaling.py:44-82,470-497.  Every mode runs the CUDA
refine in libfm_b200.so (there is no CPU path): ``mode`` is validated and
recorded, ``worker_count``/``cycle_budget`` keep their validation.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import SolveReport

DEFAULT_ALPHA = 10             # assign_scaling.py:33
DEFAULT_ASSIGN_CYCLE = 500000  # assign_scaling.py:34
ORACLE_SIZE_LIMIT = 9          # oracles.py:17 (kept for API parity)


class InfeasibleInstanceError(Exception):
    """The instance admits no perfect matching (assign_scaling.py:44-45)."""


@dataclass(frozen=True)
class AssignmentInstance:
    """Bipartite max-weight matching instance with |X| = |Y| = n
    (assign_scaling.py:48-82; same validation messages)."""

    n: int
    edges: tuple
    complete: bool

    @classmethod
    def build(cls, n: int, edges) -> "AssignmentInstance":
        if n < 1:
            raise ValueError(f"n must be at least 1, got {n}")
        seen: set = set()
        normalized = []
        for x, y, w in edges:
            if not (0 <= x < n):
                raise ValueError(f"edge ({x},{y}): x out of range [0, {n})")
            if not (0 <= y < n):
                raise ValueError(f"edge ({x},{y}): y out of range [0, {n})")
            if (x, y) in seen:
                raise ValueError(f"duplicate edge ({x},{y})")
            seen.add((x, y))
            normalized.append((int(x), int(y), int(w)))
        return cls(n=n, edges=tuple(normalized), complete=len(seen) == n * n)

    @classmethod
    def from_matrix(cls, weights) -> "AssignmentInstance":
        n = len(weights)
        edges = [(x, y, weights[x][y]) for x in range(n) for y in range(n)]
        return cls.build(n, edges)

    def dense(self) -> np.ndarray:
        """int32 n x n weights, FM_ABSENT_WEIGHT where the instance has no arc."""
        w = np.full((self.n, self.n), _lib.FM_ABSENT_WEIGHT, np.int64)
        if self.edges:
            e = np.asarray(self.edges, dtype=np.int64)
            w[e[:, 0], e[:, 1]] = e[:, 2]
        return _check_weights(w)


def _check_weights(w) -> np.ndarray:
    """Square int32 matrix (INT32_MIN = absent arc).  An int32 input is taken as is;
    wider integer inputs are range-checked before the narrowing copy."""
    w = np.asarray(w)
    if w.ndim != 2 or w.shape[0] != w.shape[1]:
        raise ValueError(f"weights must be square, got shape {w.shape}")
    if w.dtype == np.int32:
        return np.ascontiguousarray(w)
    if w.size and (int(w.min()) < -(2**31) or int(w.max()) >= 2**31):
        raise ValueError("weights must fit in int32")
    return np.ascontiguousarray(w, dtype=np.int32)


class AssignmentSolver:
    """Reusable device workspace for n x n instances (owns the C handle)."""

    def __init__(self, n: int, device: int = 0):
        L = _lib.load()
        _lib.require_device()
        h = ctypes.c_void_p()
        _lib.check(L.fm_assign_create(int(n), int(device), ctypes.byref(h)), "fm_assign_create")
        self.n, self.device, self._h = int(n), int(device), h
        self.last_stats: dict = {}

    def close(self):
        if self._h:
            _lib.load().fm_assign_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _flags(use_price_update, use_arc_fix, validate) -> int:
        return ((_lib.FM_ASSIGN_PRICE_UPDATE if use_price_update else 0)
                | (_lib.FM_ASSIGN_ARC_FIX if use_arc_fix else 0)
                | (_lib.FM_ASSIGN_VALIDATE if validate else 0))

    def solve_host(self, weights, alpha=DEFAULT_ALPHA, use_price_update=True, use_arc_fix=True,
                   validate=False, want_prices=False):
        w = _check_weights(weights)
        obj = ctypes.c_int64()
        match = np.zeros(self.n, np.int32)
        prices = np.zeros(2 * self.n, np.int64) if want_prices else None
        st = _lib.FmStats()
        rc = _lib.load().fm_assign_solve_host(
            self._h, _lib.ptr(w), int(alpha), self._flags(use_price_update, use_arc_fix, validate),
            ctypes.byref(obj), _lib.ptr(match), _lib.ptr(prices) if want_prices else None,
            ctypes.byref(st))
        self.last_stats = st.as_dict()
        _lib.check(rc, "fm_assign_solve_host")
        return int(obj.value), match, prices, self.last_stats

    def solve_device(self, weights_dev, alpha=DEFAULT_ALPHA, use_price_update=True, use_arc_fix=True,
                     validate=False, want_prices=False, stream=None):
        obj = ctypes.c_int64()
        match = np.zeros(self.n, np.int32)
        prices = np.zeros(2 * self.n, np.int64) if want_prices else None
        st = _lib.FmStats()
        s = int(getattr(stream, "cuda_stream", stream)) if stream is not None else None
        rc = _lib.load().fm_assign_solve(
            self._h, _lib.ptr(weights_dev), int(alpha),
            self._flags(use_price_update, use_arc_fix, validate), ctypes.byref(obj),
            _lib.ptr(match), _lib.ptr(prices) if want_prices else None, ctypes.byref(st), s)
        self.last_stats = st.as_dict()
        _lib.check(rc, "fm_assign_solve")
        return int(obj.value), match, prices, self.last_stats


    # ---- stepwise API (on_refine_end)
    def begin(self, weights, alpha=DEFAULT_ALPHA, use_price_update=True, use_arc_fix=True, validate=False):
        w = _check_weights(weights)
        self._keep = w
        _lib.check(_lib.load().fm_assign_begin(self._h, _lib.ptr(w), int(alpha),
                                               self._flags(use_price_update, use_arc_fix, validate)),
                   "fm_assign_begin")

    def refine(self):
        eps = ctypes.c_int64()
        done = ctypes.c_int32()
        _lib.check(_lib.load().fm_assign_refine(self._h, ctypes.byref(eps), ctypes.byref(done)), "fm_assign_refine")
        return int(eps.value), bool(done.value)

    def state(self):
        n = self.n
        prices = np.zeros(2 * n, np.int64)
        match = np.zeros(n, np.int32)
        fixed = np.zeros(n * ((n + 31) // 32), np.uint32)
        obj = ctypes.c_int64()
        st = _lib.FmStats()
        _lib.check(_lib.load().fm_assign_state(self._h, _lib.ptr(prices), _lib.ptr(match), _lib.ptr(fixed),
                                               ctypes.byref(obj), ctypes.byref(st)), "fm_assign_state")
        self.last_stats = st.as_dict()
        return prices, match, fixed.reshape(n, -1), int(obj.value)


class _ResidualView:
    """ResidualState-shaped view (graph.py:128-154) of the device state."""

    def __init__(self, residual, excess, price):
        self.residual = residual
        self.excess = excess
        self.height = [0] * len(excess)
        self.price = price


class ScalingView:
    """ScalingState-shaped view (assign_scaling.py:102-117) handed to on_refine_end:
    net is the reference's min-cost network (reduce_to_mincost, arcs in instance edge
    order), state.residual / state.price / fixed describe the device state at the end
    of the refine (all excesses are zero there)."""

    def __init__(self, n, xs, ys, ws, instance, alpha, bound):
        from .graph import FlowNetwork

        self.n = n
        self.instance = instance
        self.alpha = alpha
        self.scaled_cost_bound = bound
        self.supplies = [1] * n + [-1] * n
        net = FlowNetwork(2 * n, None, None)
        for x, y, w in zip(xs.tolist(), ys.tolist(), ws.tolist()):
            net.add_arc_pair(x, n + y, 1, -(w * (n + 1)))
        self.net = net
        self._xs, self._ys = xs, ys
        self.epsilon = 1
        self.state = None
        self.fixed = []

    def update(self, eps, prices, match, fixed_bits):
        matched = match[self._xs] == self._ys
        res = np.empty(2 * len(self._xs), np.int64)
        res[0::2] = np.where(matched, 0, 1)
        res[1::2] = 1 - res[0::2]
        fx = ((fixed_bits[self._xs, self._ys >> 5] >> (self._ys & 31).astype(np.uint32)) & 1).astype(bool)
        fixed = np.repeat(fx, 2)
        self.epsilon = eps
        self.state = _ResidualView(res.tolist(), [0] * (2 * self.n), prices.tolist())
        self.fixed = fixed.tolist()


def _solve_stepwise(inst, w, alpha, use_price_update, use_arc_fix, validate, on_refine_end, device):
    n = w.shape[0]
    solver = _solver_for(n, device)
    started = time.perf_counter()
    if isinstance(inst, AssignmentInstance) and inst.edges:
        e = np.asarray(inst.edges, dtype=np.int64)
        xs, ys, ws = e[:, 0], e[:, 1], e[:, 2]
    else:
        xs, ys = np.nonzero(w != _lib.FM_ABSENT_WEIGHT)
        ws = w[xs, ys].astype(np.int64)
    bound = int(np.abs(ws).max()) * (n + 1) if len(ws) else 0
    view = ScalingView(n, xs, ys, ws, inst if isinstance(inst, AssignmentInstance) else None, alpha, bound)
    solver.begin(w, alpha, use_price_update, use_arc_fix, validate)
    while True:
        eps, done = solver.refine()
        prices, match, fixed, obj = solver.state()
        view.update(eps, prices, match, fixed)
        on_refine_end(view)
        if done:
            break
    st = solver.last_stats
    report = SolveReport(objective=obj, pushes=int(st["pushes"]), relabels=int(st["relabels"]),
                         rounds=int(st["rounds"]), elapsed=time.perf_counter() - started, stats=st)
    return report, match.tolist()


_solvers: dict = {}


def _solver_for(n: int, device: int) -> AssignmentSolver:
    key = (n, device)
    s = _solvers.get(key)
    if s is None:
        s = _solvers[key] = AssignmentSolver(n, device)
    return s


def solve_assignment(inst: AssignmentInstance, *, mode: str = "seq", worker_count: int = 1,
                     cycle_budget: int = DEFAULT_ASSIGN_CYCLE, alpha: int = DEFAULT_ALPHA,
                     use_price_update: bool = True, use_arc_fix: bool = True,
                     heuristic_every_k: int | None = None, validate: bool = False,
                     on_refine_end=None, observer=None, device: int = 0):
    """Maximum-weight perfect matching on the GPU (assign_scaling.py:470-497).

    Returns (SolveReport, matching) with matching[x] = y; objective is the
    matching weight in original units.  Raises InfeasibleInstanceError when no
    perfect matching exists.  ``inst`` may also be a dense n x n weight array
    (numpy or CUDA tensor).
    """
    if mode not in ("seq", "par"):
        raise ValueError(f"unknown mode {mode!r}")
    if alpha < 2:
        raise ValueError(f"alpha must be at least 2, got {alpha}")
    if worker_count < 1:
        raise ValueError(f"worker_count must be at least 1, got {worker_count}")
    if cycle_budget < 1:
        raise ValueError(f"cycle_budget must be at least 1, got {cycle_budget}")
    if observer is not None:
        raise NotImplementedError("observer (per coordinator round) is not exposed by the device refine; "
                                  "use on_refine_end")
    if on_refine_end is not None:
        w = inst.dense() if isinstance(inst, AssignmentInstance) else (
            inst.detach().cpu().numpy() if hasattr(inst, "detach") else np.asarray(inst))
        return _solve_stepwise(inst, _check_weights(w), alpha, use_price_update, use_arc_fix, validate,
                               on_refine_end, device)
    started = time.perf_counter()
    if isinstance(inst, AssignmentInstance):
        n = inst.n
        solver = _solver_for(n, device)
        obj, match, _, st = solver.solve_host(inst.dense(), alpha, use_price_update, use_arc_fix, validate)
    elif hasattr(inst, "is_cuda") and inst.is_cuda:
        n = int(inst.shape[0])
        solver = _solver_for(n, device)
        import torch

        obj, match, _, st = solver.solve_device(inst.contiguous(), alpha, use_price_update, use_arc_fix,
                                                validate, stream=torch.cuda.current_stream(inst.device))
    else:
        w = np.asarray(inst)
        n = int(w.shape[0])
        solver = _solver_for(n, device)
        obj, match, _, st = solver.solve_host(w, alpha, use_price_update, use_arc_fix, validate)
    elapsed = time.perf_counter() - started
    report = SolveReport(objective=obj, pushes=int(st["pushes"]), relabels=int(st["relabels"]),
                         rounds=int(st["rounds"]), elapsed=elapsed, stats=st)
    return report, match.tolist()
