"""Host logic of the N-GPU input distribution (paper_1706_05151_b200/comm.py
split_rows, the Python twin of csrc/comm.cu k_volume_split): rows split into
equal ORIENTATION COST (adjacency entries + 32 per row), whole 32-vertex tiles,
covering [0, n) in order.  CPU only."""
import numpy as np
import pytest

from paper_1706_05151_b200 import comm as M


def csr_offsets(deg):
    off = np.zeros(len(deg) + 1, dtype=np.uint64)
    np.cumsum(deg, out=off[1:])
    return off


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_split_rows_tiles_and_balance(parts):
    rng = np.random.default_rng(parts)
    n = 200_000
    # PA-like: early rows heavy, late rows light
    deg = (20 + 4000 / np.sqrt(1 + np.arange(n))).astype(np.uint64) + rng.integers(0, 3, n).astype(np.uint64)
    off = csr_offsets(deg)
    b = M.split_rows(off, parts)
    assert b.dtype == np.uint32 and len(b) == parts + 1
    assert b[0] == 0 and b[-1] == n
    assert np.all(np.diff(b.astype(np.int64)) >= 0)
    assert np.all(b[1:-1] % 32 == 0)
    cost = off.astype(np.float64) + 32.0 * np.arange(n + 1)
    per = np.diff(cost[b])
    # each part within one tile's cost of the mean
    tile = (deg.max() + 32.0) * 32
    assert np.all(np.abs(per - cost[-1] / parts) <= tile + 1)


def test_split_rows_degenerate():
    off = csr_offsets(np.zeros(10, dtype=np.uint64))  # no edges: rows alone carry the cost
    b = M.split_rows(off, 4)
    assert b[0] == 0 and b[-1] == 10 and np.all(np.diff(b.astype(np.int64)) >= 0)
    b = M.split_rows(csr_offsets(np.array([5], dtype=np.uint64)), 3)
    assert b.tolist() == [0, 0, 0, 1] or (b[0] == 0 and b[-1] == 1)
