"""ctypes binding of libfm_b200.so (the C ABI declared in include/flowmatch_b200.h).

The CUDA library is the only compute path: if it is missing or no CUDA device is
visible, calls raise instead of falling back to anything on the CPU.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import subprocess
import threading
from collections import OrderedDict

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfm_b200.so")

FM_OK = 0
FM_INFEASIBLE = 1
FM_INVALID_ARG = 2
FM_CUDA_ERROR = 3
FM_NO_DEVICE = 4
FM_VALIDATION = 5

FM_GRID_CANCEL_VIOLATIONS = 0x1
FM_GRID_NO_PRECANCEL = 0x2
FM_GRID_NO_CUT = 0x4
FM_GRID_GLOBAL_SWEEP = 0x8

FM_ASSIGN_PRICE_UPDATE = 0x1
FM_ASSIGN_ARC_FIX = 0x2
FM_ASSIGN_VALIDATE = 0x4

FM_ABSENT_WEIGHT = -(2**31)


class FmStats(ctypes.Structure):
    _fields_ = [
        ("pushes", ctypes.c_int64),
        ("relabels", ctypes.c_int64),
        ("rounds", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("pr_sweeps", ctypes.c_int64),
        ("bfs_sweeps", ctypes.c_int64),
        ("bfs_levels", ctypes.c_int64),
        ("cut_sweeps", ctypes.c_int64),
        ("refines", ctypes.c_int64),
        ("bytes_push", ctypes.c_int64),
        ("bytes_bfs", ctypes.c_int64),
        ("pr_tiles", ctypes.c_int64),
        ("ms_total", ctypes.c_double),
        ("ms_push", ctypes.c_double),
        ("ms_bfs", ctypes.c_double),
        ("ms_cut", ctypes.c_double),
        ("ms_h2d", ctypes.c_double),
        ("ms_d2h", ctypes.c_double),
        ("ms_pr_kern", ctypes.c_double),
        ("ms_bfs_kern", ctypes.c_double),
        ("pr_launches", ctypes.c_int64),
        ("bfs_launches", ctypes.c_int64),
        ("reserved", ctypes.c_int64 * 4),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}
        d["reserved"] = list(self.reserved)
        return d


# exported symbol -> (restype, argtypes); the tests check this list against the header
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
SIGNATURES = {
    "fm_last_error": (ctypes.c_char_p, []),
    "fm_device_count": (ctypes.c_int, []),
    "fm_version": (ctypes.c_char_p, []),
    "fm_grid_create": (ctypes.c_int, [_i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "fm_grid_destroy": (None, [_vp]),
    "fm_grid_solve": (ctypes.c_int, [_vp] + [_vp] * 6 + [_i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "fm_grid_solve_host": (ctypes.c_int, [_vp] + [_vp] * 6 + [_i32, _i32, _i32, _vp, _vp, _vp]),
    "fm_grid_solve_host_batch": (ctypes.c_int, [_vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "fm_grid_begin": (ctypes.c_int, [_vp] + [_vp] * 6 + [_i32]),
    "fm_grid_round": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "fm_grid_export": (ctypes.c_int, [_vp] + [_vp] * 11),
    "fm_grid_cut_host": (ctypes.c_int, [_vp, _vp, _vp]),
    "fm_grid_cut_plane": (ctypes.c_int, [_vp, _vp, _i32]),
    "fm_grid_stats": (ctypes.c_int, [_vp, _vp]),
    "fm_coll_create": (ctypes.c_int, [ctypes.c_char_p, _i32, _i32, ctypes.POINTER(_vp)]),
    "fm_coll_destroy": (None, [_vp]),
    "fm_coll_allgather": (ctypes.c_int, [_vp, _vp, _i32, _vp]),
    "fm_band_split": (ctypes.c_int, [_i32, _i32, _vp]),
    "fm_grid_band_setup": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i32]),
    "fm_grid_band_export": (ctypes.c_int, [_vp, _vp]),
    "fm_grid_band_link": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "fm_grid_band_link_local": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "fm_grid_band_solve": (ctypes.c_int, [_vp, _vp] + [_vp] * 8 + [_i32, _i32, _vp, _vp, _vp]),
    "fm_group_create": (ctypes.c_int, [_i32, _i32, _i32, _vp, ctypes.POINTER(_vp)]),
    "fm_group_destroy": (None, [_vp]),
    "fm_group_band": (ctypes.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "fm_group_solve": (ctypes.c_int, [_vp] + [_vp] * 6 + [_i32, _i32, _vp, _vp, _vp]),
    "fm_group_band_stats": (ctypes.c_int, [_vp, _i32, _vp]),
    "fm_dimacs_parse_max": (ctypes.c_int, [ctypes.c_char_p, _i64, _vp, _vp, _vp, _vp, _vp, _i64]),
    "fm_dimacs_parse_asn": (ctypes.c_int, [ctypes.c_char_p, _i64, _vp, _vp, _vp, _vp, _vp, _i64]),
    "fm_csr_solve": (ctypes.c_int, [_i32, _i32, _i32, _i64] + [_vp] * 4 + [_i32, _i32] + [_vp] * 5),
    "fm_csr_solve64": (ctypes.c_int, [_i32, _i32, _i32, _i64] + [_vp] * 4 + [_i32, _i32] + [_vp] * 5),
    "fm_assign_create": (ctypes.c_int, [_i32, _i32, ctypes.POINTER(_vp)]),
    "fm_assign_destroy": (None, [_vp]),
    "fm_assign_solve": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "fm_assign_solve_host": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "fm_assign_begin": (ctypes.c_int, [_vp, _vp, _i64, _i32]),
    "fm_assign_refine": (ctypes.c_int, [_vp, _vp, _vp]),
    "fm_assign_state": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "fm_grid_set_option": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64]),
    "fm_assign_set_option": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64]),
    "fm_assign_load": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i64, _i64, _i64, _vp, _vp, _vp]),
    "fm_assign_begin_refine": (ctypes.c_int, [_vp, _vp]),
    "fm_assign_round": (ctypes.c_int, [_vp, _i32, _vp]),
    "fm_assign_price_update": (ctypes.c_int, [_vp]),
    "fm_assign_arc_fix": (ctypes.c_int, [_vp, _vp]),
    "fm_assign_export": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "fm_assign_certify": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _i64, _vp, _vp, _vp]),
    "fm_assign_sparse_solve": (ctypes.c_int, [_i32, _i64, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp]),
}

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile libfm_b200.so in place with nvcc for sm_100a."""
    cmd = ["make", "-s", "-C", _HERE]
    if force:
        subprocess.run(["make", "-s", "-C", _HERE, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load():
    """Load the library (never builds implicitly on a GPU box)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("FM_LIB_PATH", LIB_PATH)  # A/B builds of the same ABI
        if not os.path.exists(path):
            raise RuntimeError(
                f"CUDA extension {path} is missing; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().fm_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map C status codes onto the reference's exception types."""
    if rc == FM_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == FM_INFEASIBLE:
        from .assign import InfeasibleInstanceError

        raise InfeasibleInstanceError(msg)
    if rc == FM_INVALID_ARG:
        raise ValueError(msg)
    if rc == FM_VALIDATION:
        raise AssertionError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    return int(load().fm_device_count())


def require_device() -> None:
    if device_count() < 1:
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")


def ptr(a) -> int:
    """Address of a numpy array or torch tensor (borrowed for the call)."""
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    return int(a.ctypes.data)


class SolverCache:
    """Device workspaces reused across calls, keyed by (shape..., device).

    Each workspace carries a lock held for the whole solve: ctypes releases the
    GIL during the foreign call, so two threads must never drive one handle at
    once; a caller that finds it held gets a private workspace instead.  At most `per_device` workspaces stay cached per device; an evicted
    workspace is only dropped from the cache, never closed here -- a thread still
    solving on it holds a reference, and the handle is freed (its __del__) when
    the last reference goes.
    """

    def __init__(self, per_device: int = 1):
        self.per_device = per_device
        self._d: OrderedDict = OrderedDict()
        self._lock = threading.Lock()

    @contextlib.contextmanager
    def use(self, key, device: int, factory):
        with self._lock:
            ent = self._d.get(key)
            if ent is None:
                same = [k for k, v in self._d.items() if v[2] == device]
                for k in same[: max(0, len(same) - self.per_device + 1)]:
                    self._d.pop(k)
                ent = self._d[key] = (factory(), threading.Lock(), device)
            else:
                self._d.move_to_end(key)
            solver, lk, _ = ent
        if not lk.acquire(blocking=False):
            # busy (another thread, or a hook of this thread's own solve that calls back
            # in): a private workspace keeps the two solves apart, like the reference's
            # fresh state per call
            yield factory()
            return
        try:
            yield solver
        finally:
            lk.release()

    def clear(self) -> None:
        with self._lock:
            self._d.clear()
