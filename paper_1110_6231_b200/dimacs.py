"""DIMACS max-flow / assignment files.

``parse_dimacs_max`` / ``parse_dimacs_asn`` keep the reference's signatures and
error messages (dimacs.py:123-248) but parse in C++ (``fm_dimacs_parse_*`` in
libfm_b200.so).  ``load_max`` goes one step further for big files: it detects the
SURVEY.md 8d grid layout (s = H*W, t = H*W + 1, arcs only between 4-neighbours
and to the terminals) and returns a :class:`GridNetwork` built straight from the
arrays, so a grid file never materialises Python arc lists.  ``generate`` and the
serializers reproduce the reference's seeded instances byte for byte
(dimacs.py:59-74,271-344).
"""

from __future__ import annotations

import ctypes
import random
from dataclasses import dataclass

import numpy as np

from . import _lib
from .assign import AssignmentInstance
from .graph import FlowNetwork, GridNetwork, build_network


class ParseError(ValueError):
    """Malformed instance file; the message carries a line number if known."""


def _bytes(text) -> bytes:
    return text.encode("utf-8") if isinstance(text, str) else bytes(text)


def parse_max_arrays(text):
    """(node_count, source, sink, tails, heads, caps) of a DIMACS max file."""
    L = _lib.load()
    b = _bytes(text)
    nst = (ctypes.c_int32 * 3)()
    m = ctypes.c_int64()
    rc = L.fm_dimacs_parse_max(b, len(b), nst, ctypes.byref(m), None, None, None, 0)
    if rc:
        raise ParseError(_lib.last_error())
    k = int(m.value)
    tl, hd = (np.zeros(max(1, k), np.int32) for _ in range(2))
    cp = np.zeros(max(1, k), np.int64)
    rc = L.fm_dimacs_parse_max(b, len(b), nst, ctypes.byref(m), _lib.ptr(tl), _lib.ptr(hd), _lib.ptr(cp), k)
    if rc:
        raise ParseError(_lib.last_error())
    return int(nst[0]), int(nst[1]), int(nst[2]), tl[:k], hd[:k], cp[:k]


def parse_dimacs_max(text) -> FlowNetwork:
    """DIMACS max-flow text -> FlowNetwork, arcs in file order (dimacs.py:123-184)."""
    n, s, t, tl, hd, cp = parse_max_arrays(text)
    if n < 2 or s == t:
        build_network([], n, s, t)  # raises the reference's NetworkError
    net = FlowNetwork(n, s, t)
    k = len(tl)
    tail = np.empty(2 * k, np.int64)
    head = np.empty(2 * k, np.int64)
    cap = np.zeros(2 * k, np.int64)
    tail[0::2], tail[1::2] = tl, hd
    head[0::2], head[1::2] = hd, tl
    cap[0::2] = cp
    net.tail, net.head, net.capacity = tail.tolist(), head.tolist(), cap.tolist()
    net.cost = [0] * (2 * k)
    order = np.argsort(tail, kind="stable")
    starts = np.searchsorted(tail[order], np.arange(n + 1))
    net.out_arcs = [order[starts[v]:starts[v + 1]].tolist() for v in range(n)]
    return net


def parse_dimacs_asn(text) -> AssignmentInstance:
    """DIMACS assignment text -> AssignmentInstance (dimacs.py:187-248)."""
    L = _lib.load()
    b = _bytes(text)
    n = ctypes.c_int32()
    m = ctypes.c_int64()
    if L.fm_dimacs_parse_asn(b, len(b), ctypes.byref(n), ctypes.byref(m), None, None, None, 0):
        raise ParseError(_lib.last_error())
    k = int(m.value)
    xs, ys = np.zeros(max(1, k), np.int32), np.zeros(max(1, k), np.int32)
    ws = np.zeros(max(1, k), np.int64)
    if L.fm_dimacs_parse_asn(b, len(b), ctypes.byref(n), ctypes.byref(m), _lib.ptr(xs), _lib.ptr(ys),
                             _lib.ptr(ws), k):
        raise ParseError(_lib.last_error())
    edges = tuple(zip(xs[:k].tolist(), ys[:k].tolist(), ws[:k].tolist()))
    return AssignmentInstance(n=int(n.value), edges=edges, complete=k == int(n.value) ** 2)


def grid_from_arrays(n, s, t, tails, heads, caps):
    """Recognise the SURVEY.md 8d grid layout: pixels 0..HW-1, s = HW, t = HW + 1,
    arcs s->p, p->t and between 4-neighbours (parallel arcs are summed, arcs into s
    or out of t and self-loops never carry flow and are dropped).  Returns
    (GridNetwork, extra) with extra = capacity of direct s->t arcs (added to the
    flow), or None when the network is not such a grid."""
    HW = n - 2
    if HW < 1 or s != HW or t != HW + 1:
        return None
    tl = tails.astype(np.int64)
    hd = heads.astype(np.int64)
    cp = caps.astype(np.int64)
    keep = (tl != hd) & (hd != s) & (tl != t)
    tl, hd, cp = tl[keep], hd[keep], cp[keep]
    extra = int(cp[(tl == s) & (hd == t)].sum())
    inner = (tl < HW) & (hd < HW)
    d = np.abs(hd[inner] - tl[inner])
    far = d[d > 1]
    W = int(far[0]) if far.size else HW
    if far.size and not (far == W).all():
        return None
    if HW % W:
        return None
    H = HW // W
    capS = np.zeros(HW, np.int64)
    capT = np.zeros(HW, np.int64)
    planes = [np.zeros(HW, np.int64) for _ in range(4)]
    m_s = (tl == s) & (hd < HW)
    np.add.at(capS, hd[m_s], cp[m_s])
    m_t = (hd == t) & (tl < HW)
    np.add.at(capT, tl[m_t], cp[m_t])
    a, b, c = tl[inner], hd[inner], cp[inner]
    right = (b == a + 1) & (a % W != W - 1)
    left = (b == a - 1) & (a % W != 0)
    down = b == a + W
    up = b == a - W
    if not (right | left | down | up).all():
        return None
    for k, msk in enumerate((right, left, down, up)):
        np.add.at(planes[k], a[msk], c[msk])
    # past int32 the planes stay int64 (hybrid_solve runs them on the int64 kernel)
    wide = max(int(p.max()) if p.size else 0 for p in planes + [capS, capT]) >= 2 ** 31
    sh = lambda x: np.ascontiguousarray(x.reshape(H, W), dtype=np.int64 if wide else np.int32)
    return GridNetwork(*[sh(p) for p in planes], sh(capS), sh(capT)), extra


def load_max(text):
    """Parse a max-flow file for solving: a GridNetwork when the file is a grid in the
    adapter layout (plus the s->t capacity to add), else a FlowNetwork."""
    n, s, t, tl, hd, cp = parse_max_arrays(text)
    g = grid_from_arrays(n, s, t, tl, hd, cp)
    if g is not None:
        return g
    return parse_dimacs_max(text), 0


# ------------------------------------------------------------------ generation

@dataclass(frozen=True)
class InstanceFile:
    """A generated instance (dimacs.py:26-56): records in file order."""

    kind: str
    node_count: int
    records: tuple
    source: int | None = None
    sink: int | None = None

    def to_text(self) -> str:
        if self.kind == "maxflow":
            return serialize_max(self.node_count, self.records, self.source, self.sink)
        return serialize_asn(self.node_count // 2, self.records)

    def to_network(self) -> FlowNetwork:
        if self.kind != "maxflow":
            raise ValueError(f"not a maxflow instance: kind={self.kind!r}")
        return build_network(self.records, self.node_count, self.source, self.sink)

    def to_instance(self) -> AssignmentInstance:
        if self.kind != "assignment":
            raise ValueError(f"not an assignment instance: kind={self.kind!r}")
        return AssignmentInstance.build(self.node_count // 2, self.records)


def serialize_max(node_count, arcs, source, sink) -> str:
    lines = [f"p max {node_count} {len(arcs)}", f"n {source + 1} s", f"n {sink + 1} t"]
    lines += [f"a {a + 1} {b + 1} {c}" for a, b, c in arcs]
    return "\n".join(lines) + "\n"


def serialize_asn(n, edges) -> str:
    lines = [f"p asn {2 * n} {len(edges)}"] + [f"n {x + 1}" for x in range(n)]
    lines += [f"a {x + 1} {n + y + 1} {w}" for x, y, w in edges]
    return "\n".join(lines) + "\n"


def serialize_network(net: FlowNetwork) -> str:
    """Canonical text of a FlowNetwork: forward arcs in index order (dimacs.py:77-83)."""
    if isinstance(net, GridNetwork):
        tl, hd, cp = net.arc_arrays()
        return serialize_max(net.node_count, list(zip(tl.tolist(), hd.tolist(), cp.tolist())),
                             net.source, net.sink)
    arcs = [(net.tail[a], net.head[a], net.capacity[a]) for a in range(0, net.arc_count, 2)]
    return serialize_max(net.node_count, arcs, net.source, net.sink)


def serialize_instance(inst: AssignmentInstance) -> str:
    """Canonical text of an AssignmentInstance, edges in stored order (dimacs.py:86-88)."""
    return serialize_asn(inst.n, inst.edges)


def generate(kind: str, n: int, m_or_density=None, max_value: int = 100, rng_seed: int = 0) -> InstanceFile:
    """The reference's seeded generator (dimacs.py:271-344), same random stream."""
    rng = random.Random(rng_seed)
    if kind == "maxflow":
        if n < 2:
            raise ValueError(f"maxflow generation needs n >= 2, got {n}")
        if m_or_density is None or int(m_or_density) < 1:
            raise ValueError("maxflow generation needs an arc count m >= 1")
        if max_value < 1:
            raise ValueError(f"max_value must be at least 1, got {max_value}")
        m = int(m_or_density)
        source, sink = 0, n - 1
        hops = rng.randint(0, min(n - 2, m - 1))
        path = [source] + rng.sample(range(1, n - 1), hops) + [sink]
        arcs = [(path[i], path[i + 1], rng.randint(1, max_value)) for i in range(len(path) - 1)]
        while len(arcs) < m:
            tail, head = rng.randrange(n), rng.randrange(n)
            if tail == head:
                continue
            arcs.append((tail, head, rng.randint(0, max_value)))
        return InstanceFile("maxflow", n, tuple(arcs), source, sink)
    if kind == "assignment":
        if n < 1:
            raise ValueError(f"assignment generation needs n >= 1, got {n}")
        if max_value < 0:
            raise ValueError(f"max_value must be nonnegative, got {max_value}")
        if m_or_density is None:
            keep_all, density = True, 1.0
        else:
            keep_all, density = False, float(m_or_density)
            if not (0.0 < density <= 1.0):
                raise ValueError(f"density must be in (0, 1], got {density}")
        planted = list(range(n))
        rng.shuffle(planted)
        wanted = {(x, planted[x]) for x in range(n)}
        edges = []
        for x in range(n):
            for y in range(n):
                if keep_all or (x, y) in wanted or rng.random() < density:
                    edges.append((x, y, rng.randint(0, max_value)))
        return InstanceFile("assignment", 2 * n, tuple(edges))
    raise ValueError(f"unknown kind {kind!r}")


def detect_kind(text) -> str:
    """'maxflow' or 'assignment' from the problem line (dimacs.py:251-268)."""
    for lineno, raw in enumerate(_bytes(text).decode("utf-8").splitlines(), start=1):
        parts = raw.split()
        if not parts or parts[0] == "c":
            continue
        if parts[0] == "p":
            if len(parts) < 2:
                raise ParseError(f"line {lineno}: malformed problem line")
            if parts[1] == "max":
                return "maxflow"
            if parts[1] == "asn":
                return "assignment"
            raise ParseError(f"line {lineno}: unknown problem type {parts[1]!r}")
        break
    raise ParseError("missing problem line")
