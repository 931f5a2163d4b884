"""Shared fixtures.  `-m gpu` tests need a CUDA device and libfm_b200.so; everything
else runs on CPU (the oracle, host logic, the C ABI's symbol table)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfm_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def grid_caps(case):
    """Regenerate the capacities of a golden grid case."""
    from paper_1110_6231_b200 import generators as G

    H, W, seed = case["H"], case["W"], case["seed"]
    caps = list(G.grid_random(H, W, seed) if case["kind"] == "G" else G.grid_segmentation(H, W, seed))
    m = case.get("mutate")
    if m == "capS=0":
        caps[4] = np.zeros_like(caps[4])
    elif m == "capT=0":
        caps[5] = np.zeros_like(caps[5])
    elif m == "nbr=0":
        for k in range(4):
            caps[k] = np.zeros_like(caps[k])
    return [np.ascontiguousarray(a, dtype=np.int32) for a in caps]


def unpack_cut(hexstr, count):
    bits = np.unpackbits(np.frombuffer(bytes.fromhex(hexstr), dtype=np.uint8))
    return bits[:count].astype(bool)


def assign_matrix(case):
    """Dense weights of a golden assignment case (INT32_MIN = absent arc)."""
    from paper_1110_6231_b200 import generators as G

    n = case["n"]
    if case.get("generator") == "assignment_reference":
        return G.assignment_reference(n, case["max_value"], case["seed"], density=case.get("density"))
    w = np.full((n, n), -(2**31), np.int64)
    for x, y, wt in case["edges"]:
        w[x, y] = wt
    return w.astype(np.int32)


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
