import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# fp64 tolerance of the north star (BASELINE.json): |Δ| <= 1e-9 * Σ_{y⪯x}|f(y)|
FP64_RTOL = 1e-9


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def load_matrix(name):
    """Integer matrix fixture from tests/golden (first line = citation)."""
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([(-1 if t == "inf" else int(t)) for t in line.split()])
    return np.array(rows, dtype=np.int64)


def load_facts():
    out = {}
    with open(os.path.join(GOLDEN, "example_facts.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            parts = line.split()
            out[parts[0]] = parts[1]
    return out


def assert_fp64_close(got, want, scale, rtol=FP64_RTOL):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = np.asarray(scale, dtype=np.float64)
    err = np.abs(got - want)
    bound = rtol * scale + 1e-300
    bad = ~(err <= bound)
    if bad.any():
        idx = np.argwhere(bad)[0]
        raise AssertionError(f"fp64 mismatch at {tuple(idx)}: got {got[tuple(idx)]!r} "
                             f"want {want[tuple(idx)]!r} bound {bound[tuple(idx)]!r} "
                             f"({int(bad.sum())} bad of {bad.size})")


@pytest.fixture(scope="session")
def paper_example():
    from workloads import paper_example_edges
    src, dst = paper_example_edges()
    return 12, src, dst
