"""Dense assignment by cost scaling: drop-in for the reference's assignment API.

Same names, keyword arguments, defaults, return values and exceptions as
assign_scaling.py:44-497 and assign_par.py:115-237:

* ``solve_assignment(inst, *, mode, worker_count, cycle_budget, alpha,
  use_price_update, use_arc_fix, heuristic_every_k, validate, on_refine_end,
  observer) -> (SolveReport, matching)``.  Without hooks it runs the fused device
  solve (fm_assign_solve: every refine on the GPU, one host sync per refine);
  with hooks it builds the reference-shaped :class:`ScalingState` and runs
  :func:`min_cost_loop`.
* ``make_scaling_state`` / ``ScalingState`` / ``reduce_to_mincost`` /
  ``OpCounters``: the reference's types, same fields.
* ``begin_refine``, ``refine_par``, ``refine_seq``, ``price_update_heuristic``,
  ``arc_fix``, ``min_cost_loop``, ``extract_matching``: each loads the caller's
  ScalingState onto the device (fm_assign_load), runs the step there
  (fm_assign_begin_refine / _round / _price_update / _arc_fix) and writes the
  result back into the caller's lists in place, as the reference mutates them.

Every mode runs on the GPU (there is no CPU path): ``mode`` is validated and
selects the reference's schedule (seq: price update right after the preamble; par:
after the first coordinator round and every ``heuristic_every_k`` rounds).
``worker_count`` keeps its validation (one CUDA warp or CTA owns each node).
"""

from __future__ import annotations

import ctypes
import itertools
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import FlowNetwork, ResidualState, SolveReport

DEFAULT_ALPHA = 10             # assign_scaling.py:33
DEFAULT_ASSIGN_CYCLE = 500000  # assign_scaling.py:34
OPS_BUDGET_FACTOR = 40         # assign_scaling.py:38
OPS_BUDGET_FLOOR = 10000       # assign_scaling.py:39
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


# sparse instances run in compressed form (fm_assign_sparse_solve) when the dense n x n
# matrix would be large or mostly absent: more than 2^24 cells, or under 1/8 of them present
SPARSE_DENSE_CELLS = 1 << 24
SPARSE_MAX_DENSITY = 0.125


def _use_sparse(inst, layout: str) -> bool:
    if layout not in ("auto", "dense", "sparse"):
        raise ValueError(f"layout must be 'auto', 'dense' or 'sparse', got {layout!r}")
    if not isinstance(inst, AssignmentInstance) or inst.complete:
        if layout == "sparse" and isinstance(inst, AssignmentInstance):
            return True
        return False
    if layout != "auto":
        return layout == "sparse"
    cells = inst.n * inst.n
    return cells > SPARSE_DENSE_CELLS or len(inst.edges) < SPARSE_MAX_DENSITY * cells


def solve_sparse(inst: "AssignmentInstance", alpha: int = DEFAULT_ALPHA, use_price_update: bool = True,
                 use_arc_fix: bool = True, device: int = 0, want_prices: bool = False):
    """Sparse instance on the GPU in compressed form (O(n + m) memory).
    Returns (objective, matching[x] = y, prices (2n) or None, stats)."""
    L = _lib.load()
    _lib.require_device()
    n = inst.n
    try:   # flat iteration: ~2.5x faster than np.asarray over the tuple of tuples
        e = np.fromiter(itertools.chain.from_iterable(inst.edges), dtype=np.int64,
                        count=3 * len(inst.edges)).reshape(-1, 3)
    except (ValueError, OverflowError):
        e = np.asarray(inst.edges, dtype=np.int64).reshape(-1, 3)   # ragged / odd input: numpy's error
    if e.size and (int(e[:, 2].min()) < -(2**31) + 1 or int(e[:, 2].max()) >= 2**31):
        raise ValueError("weights must fit in int32")
    xs = np.ascontiguousarray(e[:, 0], dtype=np.int32)
    ys = np.ascontiguousarray(e[:, 1], dtype=np.int32)
    ws = np.ascontiguousarray(e[:, 2], dtype=np.int32)
    obj = ctypes.c_int64()
    match = np.zeros(n, np.int32)
    prices = np.zeros(2 * n, np.int64) if want_prices else None
    st = _lib.FmStats()
    flags = (_lib.FM_ASSIGN_PRICE_UPDATE if use_price_update else 0) | (_lib.FM_ASSIGN_ARC_FIX if use_arc_fix else 0)
    p = lambda a: _lib.ptr(a) if a.size else None
    rc = L.fm_assign_sparse_solve(n, len(xs), p(xs), p(ys), p(ws), int(alpha), flags, int(device),
                                  ctypes.byref(obj), _lib.ptr(match), _lib.ptr(prices) if want_prices else None,
                                  ctypes.byref(st))
    _lib.check(rc, "fm_assign_sparse_solve")
    return int(obj.value), match, prices, st.as_dict()


def _check_weights(w) -> np.ndarray:
    """Square int32 matrix (INT32_MIN = absent arc).  An int32 input is taken as is;
    wider integer inputs are range-checked before the narrowing copy."""
    w = np.asarray(w)
    if w.ndim != 2 or w.shape[0] != w.shape[1]:
        raise ValueError(f"weights must be square, got shape {w.shape}")
    if w.shape[0] < 1:
        raise ValueError("n must be at least 1, got 0")
    if w.dtype == np.int32:
        return np.ascontiguousarray(w)
    if not np.issubdtype(w.dtype, np.integer):
        raise ValueError(f"weights must be integers, got {w.dtype}")
    if w.size and (int(w.min()) < -(2**31) or int(w.max()) >= 2**31):
        raise ValueError("weights must fit in int32")
    return np.ascontiguousarray(w, dtype=np.int32)


def _check_weights_device(w):
    """CUDA weight tensor -> contiguous square int32 tensor on its own device."""
    import torch

    if w.dim() != 2 or w.shape[0] != w.shape[1]:
        raise ValueError(f"weights must be square, got shape {tuple(w.shape)}")
    if w.shape[0] < 1:
        raise ValueError("n must be at least 1, got 0")
    if w.dtype != torch.int32:
        if w.dtype.is_floating_point or w.dtype.is_complex or w.dtype == torch.bool:
            raise ValueError(f"weights must be integers, got {w.dtype}")
        if w.numel() and (int(w.min()) < -(2**31) or int(w.max()) >= 2**31):
            raise ValueError("weights must fit in int32")
        w = w.to(torch.int32)
    return w.contiguous()


@dataclass
class OpCounters:
    """assign_scaling.py:120-124."""

    pushes: int = 0
    relabels: int = 0
    rounds: int = 0


def reduce_to_mincost(inst: AssignmentInstance):
    """Unit-capacity min-cost network plus supplies (assign_scaling.py:85-99): X nodes
    0..n-1, Y nodes n..2n-1, forward arc 2k = edge k with cost -(w (n+1))."""
    n = inst.n
    scale = n + 1
    net = FlowNetwork(2 * n, None, None)
    m = len(inst.edges)
    if m:
        e = np.asarray(inst.edges, dtype=object if _wide(inst.edges) else np.int64)
        xs = e[:, 0].astype(np.int64)
        ys = e[:, 1].astype(np.int64) + n
        tail = np.empty(2 * m, np.int64)
        tail[0::2], tail[1::2] = xs, ys
        head = np.empty(2 * m, np.int64)
        head[0::2], head[1::2] = ys, xs
        net.tail = tail.tolist()
        net.head = head.tolist()
        net.capacity = [1, 0] * m
        cost = [0] * (2 * m)
        c = [-(int(w) * scale) for w in e[:, 2].tolist()]
        cost[0::2] = c
        cost[1::2] = [-v for v in c]
        net.cost = cost
        # out-arc lists in arc order (add_arc_pair appends per node)
        order = np.argsort(tail, kind="stable")
        bounds = np.searchsorted(tail[order], np.arange(2 * n + 1))
        ol = order.tolist()
        net.out_arcs = [ol[bounds[v]:bounds[v + 1]] for v in range(2 * n)]
    supplies = [1] * n + [-1] * n
    return net, supplies


def _wide(edges) -> bool:
    return any(abs(int(w)) >= 2**62 for _, _, w in edges)


@dataclass
class ScalingState:
    """Everything one cost-scaling solve mutates (assign_scaling.py:102-117)."""

    net: FlowNetwork
    instance: AssignmentInstance
    state: ResidualState
    supplies: list
    epsilon: int
    alpha: int
    scaled_cost_bound: int
    fixed: list = field(default_factory=list)

    def __post_init__(self) -> None:
        if not self.fixed:
            self.fixed = [False] * self.net.arc_count


def make_scaling_state(inst: AssignmentInstance, alpha: int = DEFAULT_ALPHA) -> ScalingState:
    """assign_scaling.py:127-142: prices 0, excess = supplies, eps0 = max(1, max|cost|)."""
    if alpha < 2:
        raise ValueError(f"alpha must be at least 2, got {alpha}")
    net, supplies = reduce_to_mincost(inst)
    state = ResidualState.fresh(net)
    state.excess = list(supplies)
    bound = max((abs(c) for c in net.cost), default=0)
    return ScalingState(net=net, instance=inst, state=state, supplies=supplies, epsilon=max(1, bound),
                        alpha=alpha, scaled_cost_bound=bound)


class AssignmentSolver:
    """Reusable device workspace for n x n instances (owns the C handle).

    options: tuning switches passed to fm_assign_set_option."""

    def __init__(self, n: int, device: int = 0, options: dict | None = None):
        L = _lib.load()
        _lib.require_device()
        h = ctypes.c_void_p()
        _lib.check(L.fm_assign_create(int(n), int(device), ctypes.byref(h)), "fm_assign_create")
        self.n, self.device, self._h = int(n), int(device), h
        self.last_stats: dict = {}
        for k, v in (options or {}).items():
            self.set_option(k, v)

    def set_option(self, name: str, value: int) -> None:
        _lib.check(_lib.load().fm_assign_set_option(self._h, name.encode(), int(value)), "fm_assign_set_option")

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
        if w.shape[0] != self.n:
            raise ValueError(f"solver is sized for n={self.n}, got {w.shape[0]}")
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
        weights_dev = _check_weights_device(weights_dev)
        if weights_dev.shape[0] != self.n:
            raise ValueError(f"solver is sized for n={self.n}, got {weights_dev.shape[0]}")
        if (weights_dev.device.index or 0) != self.device:
            raise ValueError(f"weights are on {weights_dev.device}, solver on cuda:{self.device}")
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

    # ---- stateful API (ScalingState on the device)
    def load(self, weights, alpha, flags, eps, prices, match, fixed_bits, scale=0, bound=-1) -> None:
        w = None if weights is None else _check_weights(weights)
        self._keep = (w, prices, match, fixed_bits)
        _lib.check(_lib.load().fm_assign_load(self._h, _lib.ptr(w) if w is not None else None, int(alpha),
                                              int(flags), int(eps), int(scale), int(bound), _lib.ptr(prices),
                                              _lib.ptr(match), _lib.ptr(fixed_bits)), "fm_assign_load")

    def begin_refine(self) -> int:
        eps = ctypes.c_int64()
        _lib.check(_lib.load().fm_assign_begin_refine(self._h, ctypes.byref(eps)), "fm_assign_begin_refine")
        return int(eps.value)

    def round(self, cycle_budget: int):
        out = (ctypes.c_int64 * 4)()
        _lib.check(_lib.load().fm_assign_round(self._h, int(min(cycle_budget, 2**31 - 1)), out), "fm_assign_round")
        return int(out[0]), int(out[1]), int(out[2]), int(out[3])

    def price_update(self) -> None:
        _lib.check(_lib.load().fm_assign_price_update(self._h), "fm_assign_price_update")

    def arc_fix(self) -> int:
        out = ctypes.c_int64()
        _lib.check(_lib.load().fm_assign_arc_fix(self._h, ctypes.byref(out)), "fm_assign_arc_fix")
        return int(out.value)

    def export(self):
        n = self.n
        prices = np.zeros(2 * n, np.int64)
        match = np.zeros(n, np.int32)
        fixed = np.zeros(n * ((n + 31) // 32), np.uint32)
        ey = np.zeros(n, np.int32)
        eps = ctypes.c_int64()
        _lib.check(_lib.load().fm_assign_export(self._h, _lib.ptr(prices), _lib.ptr(match), _lib.ptr(fixed),
                                                _lib.ptr(ey), ctypes.byref(eps)), "fm_assign_export")
        return prices, match, fixed.reshape(n, -1), ey, int(eps.value)


    def certify(self, weights, match, prices=None, scale: int = 0):
        """Exact optimality certificate (fm_assign_certify): (status, objective,
        passes), status 1 = proven maximum weight, 0 = a negative residual cycle
        exists, -1 = not a perfect matching of present pairs.  weights: host array
        or CUDA tensor.  Overwrites this workspace's solve state."""
        on_dev = hasattr(weights, "is_cuda") and weights.is_cuda
        w = _check_weights_device(weights) if on_dev else _check_weights(weights)
        m = np.ascontiguousarray(match, dtype=np.int32)
        p = None if prices is None else np.ascontiguousarray(prices, dtype=np.int64)
        cert, obj, passes = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
        _lib.check(_lib.load().fm_assign_certify(self._h, _lib.ptr(w), int(on_dev), _lib.ptr(m),
                                                 _lib.ptr(p) if p is not None else None, int(scale),
                                                 ctypes.byref(cert), ctypes.byref(obj), ctypes.byref(passes)),
                   "fm_assign_certify")
        return int(cert.value), int(obj.value), int(passes.value)


_solvers = _lib.SolverCache(per_device=2)


def _solver_ctx(n: int, device: int):
    return _solvers.use((n, device), device, lambda: AssignmentSolver(n, device))


# --------------------------------------------------------------- ScalingState <-> device

class _Session:
    """A ScalingState loaded onto a device workspace.  upload() reads the caller's
    lists (the reference mutates them in place, so they are the source of truth
    between calls); download() writes the device state back into the same list
    objects."""

    def __init__(self, scaling: ScalingState, solver: AssignmentSolver, use_price_update=True,
                 use_arc_fix=True, validate=False):
        self.sc = scaling
        self.solver = solver
        self.flags = AssignmentSolver._flags(use_price_update, use_arc_fix, validate)
        net, n = scaling.net, scaling.instance.n
        self.n = n
        m2 = len(net.tail)
        if m2 % 2:
            raise ValueError("network arcs must come in pairs")
        tail = np.asarray(net.tail[0::2], dtype=np.int64)
        head = np.asarray(net.head[0::2], dtype=np.int64)
        if m2 and (tail.min() < 0 or tail.max() >= n or head.min() < n or head.max() >= 2 * n):
            raise ValueError("not an assignment network: forward arcs must run X (0..n-1) -> Y (n..2n-1)")
        self.xs, self.ys = tail, head - n
        # device arc cost = -scale * w: the reduce_to_mincost scale n + 1 when every
        # forward cost is a multiple of it, else scale 1 with w = -cost
        cost = [-int(c) for c in net.cost[0::2]]
        self.scale = n + 1 if not any(c % (n + 1) for c in cost) else 1
        w = np.fromiter((c // self.scale for c in cost), dtype=object, count=len(cost))
        if len(w) and (min(w) <= -(2**31) or max(w) >= 2**31):
            raise ValueError("arc costs / (n + 1) must fit in int32")
        W = np.full((n, n), _lib.FM_ABSENT_WEIGHT, np.int32)
        if len(w):
            key = self.xs * n + self.ys
            if len(np.unique(key)) != len(key):
                raise ValueError("duplicate (x, y) arc pair")
            W[self.xs, self.ys] = w.astype(np.int64)
        self.W = W

    def upload(self) -> None:
        sc, n = self.sc, self.n
        res = np.asarray(sc.state.residual[0::2], dtype=np.int64)
        cap = np.asarray(sc.net.capacity[0::2], dtype=np.int64)
        flow = cap - res
        if len(flow) and (flow.min() < 0 or flow.max() > 1):
            raise ValueError("forward arc flow must be 0 or 1")
        match = np.full(n, -1, np.int32)
        fx, fy = self.xs[flow == 1], self.ys[flow == 1]
        if len(np.unique(fx)) != len(fx):
            raise ValueError("an X node carries more than one unit of flow")
        match[fx] = fy
        nw = (n + 31) // 32
        bits = np.zeros((n, nw), np.uint32)
        fixed = np.asarray(sc.fixed[0::2], dtype=bool) if len(sc.fixed) else np.zeros(0, bool)
        if fixed.any():
            x, y = self.xs[fixed], self.ys[fixed]
            np.bitwise_or.at(bits, (x, y >> 5), (np.uint32(1) << (y & 31).astype(np.uint32)))
        prices = np.asarray(sc.state.price, dtype=np.int64)
        # the device derives excesses from the flow and the unit supplies; a state
        # that disagrees (caller-built supplies) cannot be represented
        want = np.concatenate([(match < 0).astype(np.int64),
                               np.bincount(match[match >= 0], minlength=n).astype(np.int64) - 1])
        if list(sc.supplies) != [1] * n + [-1] * n or not np.array_equal(
                np.asarray(sc.state.excess, dtype=np.int64), want):
            raise ValueError("state excesses must be the unit supplies (+1 per X, -1 per Y) net of the flow")
        self.solver.load(self.W, sc.alpha, self.flags, max(1, int(sc.epsilon)), prices, match, bits,
                         scale=self.scale, bound=int(sc.scaled_cost_bound))

    def active(self) -> bool:
        """Any node holding excess (unmatched X or Y with excess > 0), read on the device."""
        n = self.n
        match = np.zeros(n, np.int32)
        ey = np.zeros(n, np.int32)
        s = self.solver
        _lib.check(_lib.load().fm_assign_export(s._h, None, _lib.ptr(match), None, _lib.ptr(ey), None),
                   "fm_assign_export")
        return bool((match < 0).any() or (ey > 0).any())

    def download(self) -> None:
        sc, n = self.sc, self.n
        prices, match, bits, ey, eps = self.solver.export()
        flow = (match[self.xs] == self.ys).astype(np.int64)
        res = np.empty(2 * len(flow), np.int64)
        res[0::2], res[1::2] = 1 - flow, flow
        sc.state.residual[:] = res.tolist()
        ex = np.concatenate([(match < 0).astype(np.int64), ey.astype(np.int64)])
        sc.state.excess[:] = ex.tolist()
        sc.state.price[:] = prices.tolist()
        fx = ((bits[self.xs, self.ys >> 5] >> (self.ys & 31).astype(np.uint32)) & 1).astype(bool)
        sc.fixed[:] = np.repeat(fx, 2).tolist()
        sc.epsilon = eps


def _ops_budget(scaling: ScalingState) -> int:
    """assign_scaling.py:374-377."""
    n = scaling.instance.n
    m = max(1, len(scaling.instance.edges))
    return max(OPS_BUDGET_FLOOR, OPS_BUDGET_FACTOR * n * n * m)


def _with_session(scaling, use_price_update, use_arc_fix, validate, body):
    n = scaling.instance.n
    dev = 0
    with _solver_ctx(n, dev) as solver:
        sess = _Session(scaling, solver, use_price_update, use_arc_fix, validate)
        sess.upload()
        out = body(sess)
        sess.download()
        return out


def begin_refine(scaling: ScalingState) -> None:
    """Refine preamble on the device (assign_scaling.py:145-182): epsilon <-
    max(1, ceil(epsilon / alpha)), unfrozen flow dropped, X prices reset so each X's
    best unfixed arc sits at reduced cost -epsilon."""
    _with_session(scaling, False, False, False, lambda s: s.solver.begin_refine())


def arc_fix(scaling: ScalingState) -> int:
    """Freeze arc pairs whose reduced cost exceeds 2 n epsilon (assign_scaling.py:185-205)."""
    return _with_session(scaling, False, True, False, lambda s: s.solver.arc_fix())


def price_update_heuristic(scaling: ScalingState, validate: bool = False) -> None:
    """Dial-bucket price update (assign_scaling.py:208-276) as a device label
    relaxation; a no-op without an active or without a deficit node (:230-232)."""
    ex = scaling.state.excess
    if not any(e > 0 for e in ex) or not any(e < 0 for e in ex):
        return
    _with_session(scaling, True, False, validate, lambda s: s.solver.price_update())


def _refine_rounds(sess: _Session, scaling: ScalingState, cycle_budget, counters, use_price_update,
                   use_arc_fix, heuristic_every_k, observer, pu_after_first=True):
    """refine_par's coordinator loop (assign_par.py:162-236) over device rounds."""
    ops_budget = _ops_budget(scaling)
    ops_used = 0
    round_index = 0
    active = sess.active()
    while True:
        if not active:
            if round_index > 0:
                if use_arc_fix:
                    sess.solver.arc_fix()
                if observer is not None:
                    sess.download()
                    observer(scaling)
            break
        round_index += 1
        pushes, relabels, _, left = sess.solver.round(cycle_budget)
        counters.pushes += pushes
        counters.relabels += relabels
        counters.rounds += 1
        round_ops = pushes + relabels
        if round_ops == 0:
            raise InfeasibleInstanceError("active nodes stalled with no usable residual arcs")
        ops_used += round_ops
        if ops_used > ops_budget:
            raise InfeasibleInstanceError("operation budget exceeded; prices diverge, "
                                          "instance admits no perfect matching")
        run_pu = (pu_after_first and round_index == 1) or (
            heuristic_every_k is not None and heuristic_every_k > 0 and round_index % heuristic_every_k == 0)
        if run_pu and use_price_update:
            sess.solver.price_update()
        if observer is not None:
            sess.download()
            observer(scaling)
        active = left > 0


def refine_par(scaling: ScalingState, worker_count: int = 1, cycle_budget: int = DEFAULT_ASSIGN_CYCLE, *,
               counters: OpCounters | None = None, use_price_update: bool = True, use_arc_fix: bool = True,
               heuristic_every_k: int | None = None, validate: bool = False, observer=None) -> ScalingState:
    """Parallel refine (assign_par.py:115-237) on the GPU: coordinator rounds of
    device push/relabel phases until no node holds excess.  Expects begin_refine to
    have run.  Price update after the first round (and every heuristic_every_k
    rounds), arc fixing at completion, observer(scaling) at every coordinator point.
    Raises InfeasibleInstanceError when active nodes stall or the operation budget is
    exhausted; AssertionError from the device checks when validate=True."""
    if worker_count < 1:
        raise ValueError(f"worker_count must be at least 1, got {worker_count}")
    if cycle_budget < 1:
        raise ValueError(f"cycle_budget must be at least 1, got {cycle_budget}")
    if counters is None:
        counters = OpCounters()
    _with_session(scaling, use_price_update, use_arc_fix, validate,
                  lambda s: _refine_rounds(s, scaling, cycle_budget, counters, use_price_update, use_arc_fix,
                                           heuristic_every_k, observer))
    return scaling


def refine_seq(scaling: ScalingState, counters: OpCounters | None = None, *, use_price_update: bool = True,
               use_arc_fix: bool = True, validate: bool = False) -> ScalingState:
    """One scaling phase in the sequential schedule (assign_scaling.py:339-371):
    preamble, price update right after it, push/relabel to completion, arc fixing."""
    if counters is None:
        counters = OpCounters()

    def body(s):
        s.solver.begin_refine()
        if use_price_update:
            s.solver.price_update()
        scratch = OpCounters()
        _refine_rounds(s, scaling, DEFAULT_ASSIGN_CYCLE, scratch, use_price_update, use_arc_fix, None, None,
                       pu_after_first=False)
        counters.pushes += scratch.pushes
        counters.relabels += scratch.relabels

    _with_session(scaling, use_price_update, use_arc_fix, validate, body)
    return scaling


def extract_matching(scaling: ScalingState) -> list:
    """The perfect matching read off saturated forward arcs (assign_scaling.py:380-397)."""
    net, n = scaling.net, scaling.instance.n
    res = np.asarray(scaling.state.residual[0::2], dtype=np.int64)
    cap = np.asarray(net.capacity[0::2], dtype=np.int64)
    sat = (res == 0) & (cap == 1)
    xs = np.asarray(net.tail[0::2], dtype=np.int64)[sat]
    ys = np.asarray(net.head[0::2], dtype=np.int64)[sat] - n
    if len(np.unique(xs)) != len(xs) or len(np.unique(ys)) != len(ys):
        raise AssertionError("flow does not encode a matching")
    if len(xs) != n:
        raise AssertionError("flow does not cover every node")
    matching = np.full(n, -1, np.int64)
    matching[xs] = ys
    return matching.tolist()


def min_cost_loop(scaling: ScalingState, *, mode: str = "seq", worker_count: int = 1,
                  cycle_budget: int = DEFAULT_ASSIGN_CYCLE, use_price_update: bool = True,
                  use_arc_fix: bool = True, heuristic_every_k: int | None = None, validate: bool = False,
                  on_refine_end=None, observer=None):
    """Refines at epsilon, epsilon/alpha, ... down to and including 1
    (assign_scaling.py:400-467), every step on the device.  The state stays on the
    device between refines unless a hook needs it on the host.  Returns
    (SolveReport, matching); objective in original weight units."""
    if mode not in ("seq", "par"):
        raise ValueError(f"unknown mode {mode!r}")
    if worker_count < 1:
        raise ValueError(f"worker_count must be at least 1, got {worker_count}")
    if cycle_budget < 1:
        raise ValueError(f"cycle_budget must be at least 1, got {cycle_budget}")
    counters = OpCounters()
    started = time.perf_counter()

    def body(s):
        while True:
            eps = s.solver.begin_refine()
            if mode == "seq":
                if use_price_update:
                    s.solver.price_update()
                scratch = OpCounters()
                _refine_rounds(s, scaling, DEFAULT_ASSIGN_CYCLE, scratch, use_price_update, use_arc_fix, None,
                               None, pu_after_first=False)
                counters.pushes += scratch.pushes
                counters.relabels += scratch.relabels
                counters.rounds += 1
            else:
                _refine_rounds(s, scaling, cycle_budget, counters, use_price_update, use_arc_fix,
                               heuristic_every_k, observer)
            if on_refine_end is not None:
                s.download()
                on_refine_end(scaling)
            if eps == 1:
                break

    _with_session(scaling, use_price_update, use_arc_fix, validate, body)
    matching = extract_matching(scaling)
    objective = _objective(scaling.instance, matching)
    report = SolveReport(objective=objective, pushes=counters.pushes, relabels=counters.relabels,
                         rounds=counters.rounds, elapsed=time.perf_counter() - started)
    return report, matching


def _objective(inst: AssignmentInstance, matching) -> int:
    """Sum of original weights over the matching (assign_scaling.py:456-458)."""
    n = inst.n
    if not inst.edges:
        return 0
    e = np.asarray(inst.edges, dtype=object)
    key = e[:, 0].astype(np.int64) * n + e[:, 1].astype(np.int64)
    order = np.argsort(key)
    want = np.arange(n, dtype=np.int64) * n + np.asarray(matching, dtype=np.int64)
    pos = order[np.searchsorted(key[order], want)]
    return int(sum(e[pos, 2].tolist()))


def _as_instance(inst) -> AssignmentInstance:
    if isinstance(inst, AssignmentInstance):
        return inst
    w = inst.detach().cpu().numpy() if hasattr(inst, "detach") else np.asarray(inst)
    w = _check_weights(w)
    xs, ys = np.nonzero(w != _lib.FM_ABSENT_WEIGHT)
    edges = tuple(zip(xs.tolist(), ys.tolist(), w[xs, ys].tolist()))
    return AssignmentInstance(n=w.shape[0], edges=edges, complete=len(edges) == w.shape[0] ** 2)


def solve_assignment(inst, *, mode: str = "seq", worker_count: int = 1,
                     cycle_budget: int = DEFAULT_ASSIGN_CYCLE, alpha: int = DEFAULT_ALPHA,
                     use_price_update: bool = True, use_arc_fix: bool = True,
                     heuristic_every_k: int | None = None, validate: bool = False,
                     on_refine_end=None, observer=None, device: int | None = None, layout: str = "auto"):
    """Maximum-weight perfect matching on the GPU (assign_scaling.py:470-497).

    Returns (SolveReport, matching) with matching[x] = y; objective is the matching
    weight in original units.  Raises InfeasibleInstanceError when no perfect
    matching exists.  ``inst`` may also be a dense n x n weight array (numpy, or a
    CUDA tensor that then never leaves the GPU).  Without hooks the whole solve is
    one fused device call; rounds = refines (one coordinator round per refine, as
    the reference's default cycle budget gives).  layout: a sparse instance
    (complete=False) runs in compressed form when its dense matrix would be large or
    mostly absent ("auto"), or as asked ("dense" / "sparse")."""
    if mode not in ("seq", "par"):
        raise ValueError(f"unknown mode {mode!r}")
    if alpha < 2:
        raise ValueError(f"alpha must be at least 2, got {alpha}")
    if worker_count < 1:
        raise ValueError(f"worker_count must be at least 1, got {worker_count}")
    if cycle_budget < 1:
        raise ValueError(f"cycle_budget must be at least 1, got {cycle_budget}")
    if on_refine_end is not None or observer is not None:
        scaling = make_scaling_state(_as_instance(inst), alpha=alpha)
        return min_cost_loop(scaling, mode=mode, worker_count=worker_count, cycle_budget=cycle_budget,
                             use_price_update=use_price_update, use_arc_fix=use_arc_fix,
                             heuristic_every_k=heuristic_every_k, validate=validate,
                             on_refine_end=on_refine_end, observer=observer)
    started = time.perf_counter()
    every_k = int(heuristic_every_k) if heuristic_every_k else 0
    if _use_sparse(inst, layout) and not validate and not every_k:
        obj, match, _, st = solve_sparse(inst, alpha, use_price_update, use_arc_fix,
                                         0 if device is None else int(device))
        st = dict(st)
        st["layout"] = "sparse"
        report = SolveReport(objective=obj, pushes=int(st["pushes"]), relabels=int(st["relabels"]),
                             rounds=int(st["refines"]), elapsed=time.perf_counter() - started, stats=st)
        return report, match.tolist()
    if hasattr(inst, "is_cuda") and inst.is_cuda:
        import torch

        w = _check_weights_device(inst)
        dev = w.device.index or 0
        if device is not None and int(device) != dev:
            raise ValueError(f"device={device} but the weights are on cuda:{dev}")
        n = int(w.shape[0])
        with _solver_ctx(n, dev) as solver:
            solver.set_option("heuristic_every_k", every_k)
            obj, match, _, st = solver.solve_device(w, alpha, use_price_update, use_arc_fix, validate,
                                                    stream=torch.cuda.current_stream(w.device))
    else:
        w = inst.dense() if isinstance(inst, AssignmentInstance) else _check_weights(inst)
        dev = 0 if device is None else int(device)
        n = int(w.shape[0])
        with _solver_ctx(n, dev) as solver:
            solver.set_option("heuristic_every_k", every_k)
            obj, match, _, st = solver.solve_host(w, alpha, use_price_update, use_arc_fix, validate)
    st = dict(st)
    st["device_rounds"] = st["rounds"]
    report = SolveReport(objective=obj, pushes=int(st["pushes"]), relabels=int(st["relabels"]),
                         rounds=int(st["refines"]), elapsed=time.perf_counter() - started, stats=st)
    return report, match.tolist()
