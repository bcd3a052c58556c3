import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 via gpurun)")


def unpack(flat, idx, k):
    return flat[idx[k]:idx[k + 1]]


class Golden:
    """Lazy view of the committed reference fixtures (tests/golden/*.npz)."""

    def __init__(self):
        self._cache = {}

    def __getitem__(self, name):
        if name not in self._cache:
            self._cache[name] = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
        return self._cache[name]

    def tile_sets(self):
        g = self["schedules"]
        return [unpack(g["sets"], g["sets_idx"], k).astype(np.int64)
                for k in range(len(g["sets_idx"]) - 1)]

    def spmv_cases(self):
        """Yield (k, off, col, val, x, rows, cols) for every golden matrix."""
        g = self["spmv"]
        for k in range(len(g["rows"])):
            yield (k, unpack(g["off"], g["off_idx"], k), unpack(g["col"], g["col_idx"], k),
                   unpack(g["val"], g["col_idx"], k), unpack(g["x"], g["x_idx"], k),
                   int(g["rows"][k]), int(g["cols"][k]))

    def spmm_cases(self):
        """Yield (k, off, col, val, B, rows, cols) for every golden SpMM matrix."""
        g = self["spmm"]
        for k in range(len(g["rows"])):
            n = int(g["n"][k])
            yield (k, unpack(g["off"], g["off_idx"], k), unpack(g["col"], g["col_idx"], k),
                   unpack(g["val"], g["col_idx"], k), unpack(g["B"], g["B_idx"], k).reshape(-1, n),
                   int(g["rows"][k]), int(g["cols"][k]))


@pytest.fixture(scope="session")
def golden():
    return Golden()


SCHEDULE_NAMES = ["thread-mapped", "merge-path", "group-mapped"]


def integer_csr(rng, rows, cols, nnz):
    """Random CSR with small integer values (bit-exact territory in fp32 and fp64)."""
    from paper_2301_04792_b200 import generate_random_csr

    m = generate_random_csr(rows, cols, nnz, seed=int(rng.integers(1 << 30)))
    m.values = rng.integers(-4, 5, size=m.nnz).astype(np.float64)
    return m
