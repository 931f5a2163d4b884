"""Network types crossing the drop-in boundary.

Mirrors the reference's core types (graph.py:23-186) with the same names,
fields and validation messages, and adds :class:`GridNetwork`, the
structure-of-arrays form of a 4-connected grid graph that the CUDA path consumes.
A ``GridNetwork`` *is a* ``FlowNetwork``: its arc-pair lists are materialised
lazily, in the SURVEY.md 8d adapter order, only when code asks for them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class NetworkError(ValueError):
    """Invalid network construction input (graph.py:23-24)."""


@dataclass(frozen=True, slots=True)
class SolveReport:
    """Outcome of one solver run (graph.py:27-40).

    objective is the flow value (max-flow) or matching weight (assignment).
    rounds counts coordinator rounds.  elapsed is wall seconds.  The fields
    after elapsed are additions (defaults keep the reference's positional
    order): cut = minimal source side of the min cut (bool H x W array) for
    grid solves, stats = device counters and CUDA-event timings.
    """

    objective: int
    pushes: int = 0
    relabels: int = 0
    rounds: int = 0
    elapsed: float = 0.0
    cut: object = None
    stats: object = None


class FlowNetwork:
    """Immutable directed graph with unit-indexed arc pairs (graph.py:43-84)."""

    __slots__ = ("node_count", "source", "sink", "tail", "head", "capacity", "cost", "out_arcs")

    def __init__(self, node_count: int, source: int | None, sink: int | None):
        self.node_count = node_count
        self.source = source
        self.sink = sink
        self.tail: list[int] = []
        self.head: list[int] = []
        self.capacity: list[int] = []
        self.cost: list[int] = []
        self.out_arcs: list[list[int]] = [[] for _ in range(node_count)]

    @property
    def arc_count(self) -> int:
        return len(self.tail)

    def reverse_of(self, a: int) -> int:
        return a ^ 1

    def add_arc_pair(self, tail: int, head: int, capacity: int, cost: int = 0) -> int:
        a = len(self.tail)
        self.tail += (tail, head)
        self.head += (head, tail)
        self.capacity += (capacity, 0)
        self.cost += (cost, -cost)
        self.out_arcs[tail].append(a)
        self.out_arcs[head].append(a + 1)
        return a


@dataclass(slots=True)
class ResidualState:
    """Mutable solver state (graph.py:128-154): residual[a] per arc, excess[x]
    (negative = deficit), height (max-flow), price (assignment)."""

    residual: list
    excess: list
    height: list
    price: list

    @classmethod
    def fresh(cls, net: "FlowNetwork") -> "ResidualState":
        n = net.node_count
        return cls(residual=list(net.capacity), excess=[0] * n, height=[0] * n, price=[0] * n)

    def flow_on(self, net: "FlowNetwork", a: int) -> int:
        return net.capacity[a] - self.residual[a]


def reduced_cost(net: "FlowNetwork", state: ResidualState, a: int) -> int:
    """cost(a) + price(tail) - price(head) (graph.py:157-159)."""
    return net.cost[a] + state.price[net.tail[a]] - state.price[net.head[a]]


def part_reduced_cost(net: "FlowNetwork", state: ResidualState, a: int) -> int:
    """cost(a) - price(head) (graph.py:162-164)."""
    return net.cost[a] - state.price[net.head[a]]


def is_epsilon_optimal(net: "FlowNetwork", state: ResidualState, epsilon: int, fixed=None) -> bool:
    """True iff every residual, non-fixed arc has reduced cost >= -epsilon
    (graph.py:167-186), evaluated over all arcs at once with numpy (object dtype
    when the values leave int64)."""
    m = len(net.tail)
    if m == 0:
        return True
    try:
        cost = np.asarray(net.cost, dtype=np.int64)
        price = np.asarray(state.price, dtype=np.int64)
        big = int(np.abs(cost).max()) + 2 * int(np.abs(price).max()) >= 2**62
    except OverflowError:
        big = True
    if big:
        cost = np.asarray(net.cost, dtype=object)
        price = np.asarray(state.price, dtype=object)
    tail = np.asarray(net.tail, dtype=np.int64)
    head = np.asarray(net.head, dtype=np.int64)
    live = np.asarray(state.residual, dtype=np.int64) > 0
    if fixed is not None:
        live &= ~np.asarray(fixed, dtype=bool)
    rc = cost[live] + price[tail[live]] - price[head[live]]
    return bool((rc >= -epsilon).all()) if len(rc) else True


def build_network(edge_list, node_count: int, source: int, sink: int) -> FlowNetwork:
    """Validated FlowNetwork from (tail, head, capacity[, cost]) tuples
    (graph.py:87-125; same error messages)."""
    if node_count < 2:
        raise NetworkError(f"node_count must be at least 2, got {node_count}")
    if not (0 <= source < node_count):
        raise NetworkError(f"source id {source} out of range [0, {node_count})")
    if not (0 <= sink < node_count):
        raise NetworkError(f"sink id {sink} out of range [0, {node_count})")
    if source == sink:
        raise NetworkError(f"source and sink must differ, both are {source}")
    net = FlowNetwork(node_count, source, sink)
    for i, edge in enumerate(edge_list):
        if len(edge) == 3:
            tail, head, capacity = edge
            cost = 0
        else:
            tail, head, capacity, cost = edge
        if not (0 <= tail < node_count):
            raise NetworkError(f"arc {i}: tail id {tail} out of range [0, {node_count})")
        if not (0 <= head < node_count):
            raise NetworkError(f"arc {i}: head id {head} out of range [0, {node_count})")
        if capacity < 0:
            raise NetworkError(f"arc {i}: negative capacity {capacity}")
        net.add_arc_pair(tail, head, capacity, cost)
    return net


_PLANES = ("capR", "capL", "capD", "capU", "capS", "capT")


class GridNetwork(FlowNetwork):
    """4-connected H x W grid network in structure-of-arrays form.

    Pixel p = r * W + c; source s = H*W, sink t = H*W + 1.
    capR/capL/capD/capU[p] are the capacities of p->p+1, p->p-1, p->p+W, p->p-W;
    capS[p] of s->p and capT[p] of p->t.  Arrays are int32 numpy arrays (host)
    or int32 CUDA tensors (device; the solve then never leaves the GPU).  Capacities
    past the int32 range (the reference's are unbounded Python ints) are kept as int64
    host planes and solved through the int64 generic kernel (fm_csr_solve64).
    """

    __slots__ = ("H", "W", "caps", "_materialised")

    def __init__(self, capR, capL, capD, capU, capS, capT):
        shape = tuple(capS.shape)
        if len(shape) != 2:
            raise NetworkError(f"grid planes must be 2-D, got shape {shape}")
        H, W = int(shape[0]), int(shape[1])
        caps = (capR, capL, capD, capU, capS, capT)
        for name, a in zip(_PLANES, caps):
            if tuple(a.shape) != shape:
                raise NetworkError(f"{name} has shape {tuple(a.shape)}, expected {shape}")
        # FlowNetwork's fields without its per-node list allocation (H*W + 2 empty lists
        # would take seconds): the adjacency lists are built on demand by materialise()
        self.node_count, self.source, self.sink = H * W + 2, H * W, H * W + 1
        self.tail, self.head, self.capacity, self.cost = [], [], [], []
        self.out_arcs = None
        self.H, self.W = H, W
        self.caps = caps
        self._materialised = False

    @property
    def on_device(self) -> bool:
        return hasattr(self.caps[0], "is_cuda") and bool(self.caps[0].is_cuda)

    def host_caps(self):
        """The six planes as C-contiguous int32 numpy arrays (NetworkError if a value
        does not fit: nothing is wrapped)."""
        out = []
        for name, a in zip(_PLANES, self.caps):
            if isinstance(a, np.ndarray) and a.dtype == np.int32:
                out.append(np.ascontiguousarray(a))    # the common case: no copy, no scan
                continue
            a = _host_plane(name, a)
            if a.size and (int(a.max()) >= 2**31 or int(a.min()) < -(2**31)):
                raise NetworkError(f"{name}: capacity {int(a.max())} does not fit in int32")
            out.append(a.astype(np.int32))
        return tuple(out)

    @property
    def narrow_bytes(self) -> int:
        """1 or 2 when the six host planes are C-contiguous uint8 / uint16 arrays of one
        dtype (they then cross PCIe narrow and are widened on the device), else 0."""
        if self.on_device:
            return 0
        dt = getattr(self.caps[0], "dtype", None)
        if dt not in (np.uint8, np.uint16):
            return 0
        ok = all(isinstance(a, np.ndarray) and a.dtype == dt and a.flags.c_contiguous for a in self.caps)
        return int(np.dtype(dt).itemsize) if ok else 0

    def wide_caps(self):
        """The six planes as C-contiguous int64 numpy arrays."""
        return tuple(_host_plane(name, a) for name, a in zip(_PLANES, self.caps))

    @property
    def wide(self) -> bool:
        """True when a capacity leaves the int32 range (host planes only)."""
        return not self.on_device and any(
            _may_leave_int32(a.dtype) and a.size and int(np.asarray(a).max()) >= 2**31 for a in self.caps)

    def arc_arrays(self):
        """(tails, heads, caps) of the reference network in adapter order:
        per pixel, row-major: (s,p,capS) if >0, (p,t,capT) if >0, (p,p+1,capR),
        (p+1,p,capL[p+1]), (p,p+W,capD), (p+W,p,capU[p+W])."""
        capR, capL, capD, capU, capS, capT = self.wide_caps()
        H, W = self.H, self.W
        HW = H * W
        p = np.arange(HW, dtype=np.int64)
        r, c = p // W, p % W
        s, t = HW, HW + 1
        tl = np.full((HW, 6), -1, np.int64)
        hd = np.full((HW, 6), -1, np.int64)
        cp = np.zeros((HW, 6), np.int64)
        keep = np.zeros((HW, 6), bool)
        fS, fT = capS.reshape(-1), capT.reshape(-1)
        keep[:, 0] = fS > 0
        tl[:, 0], hd[:, 0], cp[:, 0] = s, p, fS
        keep[:, 1] = fT > 0
        tl[:, 1], hd[:, 1], cp[:, 1] = p, t, fT
        hasR = c + 1 < W
        keep[:, 2] = hasR
        keep[:, 3] = hasR
        tl[:, 2], hd[:, 2], cp[:, 2] = p, p + 1, capR.reshape(-1)
        q = np.minimum(p + 1, HW - 1)
        tl[:, 3], hd[:, 3], cp[:, 3] = p + 1, p, capL.reshape(-1)[q]
        hasD = r + 1 < H
        keep[:, 4] = hasD
        keep[:, 5] = hasD
        tl[:, 4], hd[:, 4], cp[:, 4] = p, p + W, capD.reshape(-1)
        q = np.minimum(p + W, HW - 1)
        tl[:, 5], hd[:, 5], cp[:, 5] = p + W, p, capU.reshape(-1)[q]
        k = keep.reshape(-1)
        return tl.reshape(-1)[k].astype(np.int32), hd.reshape(-1)[k].astype(np.int32), cp.reshape(-1)[k]

    def materialise(self) -> "GridNetwork":
        """Fill the FlowNetwork arc-pair lists (slow; tests and small grids only)."""
        if self._materialised:
            return self
        tl, hd, cp = self.arc_arrays()
        self.tail, self.head, self.capacity, self.cost = [], [], [], []
        self.out_arcs = [[] for _ in range(self.node_count)]
        for a, b, c in zip(tl.tolist(), hd.tolist(), cp.tolist()):
            self.add_arc_pair(a, b, c)
        self._materialised = True
        return self

    @property
    def arc_count(self) -> int:
        if not self._materialised:
            self.materialise()
        return len(self.tail)


def _may_leave_int32(dt) -> bool:
    """Whether values of this dtype can leave the int32 range (narrow integer planes
    never can: no scan needed)."""
    dt = np.dtype(dt)
    return not (dt == np.int32 or dt == np.bool_ or (np.issubdtype(dt, np.integer) and dt.itemsize < 4))


def _host_plane(name, a):
    """One capacity plane as a C-contiguous int64 numpy array; non-integer input or a
    value beyond int64 raises NetworkError."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = np.asarray(a)
    if a.dtype == object:
        try:
            a = a.astype(np.int64)
        except (OverflowError, TypeError) as exc:
            raise NetworkError(f"{name}: capacities must be integers below 2^63 ({exc})") from None
    if not (np.issubdtype(a.dtype, np.integer) or a.dtype == bool):
        raise NetworkError(f"{name}: capacities must be integers, got {a.dtype}")
    if a.dtype == np.uint64 and a.size and int(a.max()) >= 2**63:
        raise NetworkError(f"{name}: capacity {int(a.max())} does not fit in int64")
    return np.ascontiguousarray(a, dtype=np.int64)


def _device_planes(planes):
    """Six CUDA planes as contiguous int32 tensors on one device.  Wider integer
    inputs are range-checked before the narrowing copy; anything else raises."""
    import torch

    dev = planes[0].device
    out = []
    for name, a in zip(_PLANES, planes):
        if not hasattr(a, "is_cuda") or not a.is_cuda:
            raise NetworkError(f"{name}: mixed host and device planes")
        if a.device != dev:
            raise NetworkError(f"{name} is on {a.device}, expected {dev}")
        if a.dtype != torch.int32:
            if a.dtype.is_floating_point or a.dtype.is_complex or a.dtype == torch.bool:
                raise NetworkError(f"{name}: capacities must be integers, got {a.dtype}")
            if a.numel() and int(a.max()) >= 2**31:
                raise NetworkError(f"{name}: capacity {int(a.max())} does not fit in int32")
            a = a.to(torch.int32)
        out.append(a.contiguous())
    return out


def build_grid_network(capR, capL, capD, capU, capS, capT) -> GridNetwork:
    """Validated GridNetwork from six H x W capacity planes (int32 numpy arrays or
    CUDA tensors; other integer dtypes are range-checked and narrowed).

    Raises NetworkError for a shape mismatch, a negative capacity, or a
    non-zero capacity on an arc that would leave the grid (last column of
    capR, first column of capL, last row of capD, first row of capU).  Device
    planes get the same checks (a few reductions on their device)."""
    net = GridNetwork(capR, capL, capD, capU, capS, capT)
    if net.on_device:
        import torch

        planes = _device_planes(net.caps)
        mins = torch.stack([a.min() for a in planes]).cpu().tolist() if planes[0].numel() else [0] * 6
        for name, m in zip(_PLANES, mins):
            if m < 0:
                raise NetworkError(f"{name}: negative capacity {m}")
        capR, capL, capD, capU = planes[:4]
        edge = torch.stack([capR[:, -1].any(), capL[:, 0].any(), capD[-1, :].any(), capU[0, :].any()]).cpu().tolist()
    else:
        # int32 planes are kept as given (no copy: pinned caller buffers stay pinned), so
        # are six uint8 / uint16 planes of one dtype (they cross PCIe narrow); other
        # integer planes are range-checked and stay int64 only when a value needs it
        dt = getattr(net.caps[0], "dtype", None)
        keep = (np.int32,) + ((dt,) if dt in (np.uint8, np.uint16) and
                              all(getattr(a, "dtype", None) == dt for a in net.caps) else ())
        planes = tuple(np.ascontiguousarray(a) if isinstance(a, np.ndarray) and a.dtype in keep else _host_plane(name, a)
                       for name, a in zip(_PLANES, net.caps))
        for name, a in zip(_PLANES, planes):
            if a.size and a.dtype.kind != "u" and int(a.min()) < 0:   # unsigned planes need no scan
                raise NetworkError(f"{name}: negative capacity {int(a.min())}")
        if not any(a.dtype not in keep and a.size and int(a.max()) >= 2**31 for a in planes):
            planes = tuple(a if a.dtype in keep else a.astype(np.int32) for a in planes)
        capR, capL, capD, capU = planes[:4]
        edge = [capR[:, -1].any(), capL[:, 0].any(), capD[-1, :].any(), capU[0, :].any()]
    if edge[0]:
        raise NetworkError("capR: last column must be 0 (arc leaves the grid)")
    if edge[1]:
        raise NetworkError("capL: first column must be 0 (arc leaves the grid)")
    if edge[2]:
        raise NetworkError("capD: last row must be 0 (arc leaves the grid)")
    if edge[3]:
        raise NetworkError("capU: first row must be 0 (arc leaves the grid)")
    net.caps = tuple(planes)
    return net
