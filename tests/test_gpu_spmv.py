"""GPU parity of the TMA-fed CSR SpMV (k_spmv_bt, spmv.cu) against a numpy restatement of the
reduction contract (TPR lanes per row, lane l sums entries l, l + TPR, ... in order,
then the xor butterfly), on matrices long enough to dispatch it (rows >= 262144), with empty rows,
rows beyond one batch, tiles beyond the stage capacity (read directly from global memory) and array
ends at every 16-byte alignment."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def _lane_contract(ptr, col, val, x, tpr):
    rows = len(ptr) - 1
    lens = np.diff(ptr)
    steps = int(-(-lens.max() // tpr))
    prod = np.zeros((rows, steps * tpr))
    idx = np.arange(len(col)) - np.repeat(ptr[:-1], lens)
    prod[np.repeat(np.arange(rows), lens), idx] = val * x[col]  # one rounding per product
    prod = prod.reshape(rows, steps, tpr)
    acc = np.zeros((rows, tpr))
    for s in range(steps):  # lane l: entries l, l + TPR, ... in order (padding adds +0.0)
        acc = acc + prod[:, s, :]
    lanes = np.arange(tpr)
    o = tpr // 2
    while o > 0:
        acc = acc + acc[:, lanes ^ o]
        o //= 2
    return acc[:, 0]


@pytest.mark.parametrize("tpr,lo,hi,tail", [(8, 20, 34, 0), (8, 20, 34, 1), (4, 10, 18, 2), (4, 10, 18, 3)])
def test_spmv_bt_lane_contract(cf, tpr, lo, hi, tail):
    rng = np.random.default_rng(100 + tail)
    rows, cols = 300_000 + 7 * tail, 50_000
    lens = rng.integers(lo, hi, rows)
    lens[rng.integers(0, rows, 2000)] = 0                      # empty rows
    lens[1000:1064] = rng.integers(60, 100, 64)                # a tile beyond the stage capacity
    lens[70_001:70_020] = rng.integers(100, 140, 19)           # rows of several batches
    lens[-1] += tail                                           # array end at each alignment
    ptr = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    nnz = int(ptr[-1])
    col = rng.integers(0, cols, nnz).astype(np.int32)
    val = rng.uniform(-1, 1, nnz)
    x = rng.uniform(-1, 1, cols)
    mean = nnz / rows
    assert (24 < mean <= 64) if tpr == 8 else (12 < mean <= 24)  # the dispatch under test
    A = cf.CsrMatrix(rows, cols, ptr, col, val)
    y = A @ x
    assert np.array_equal(y, _lane_contract(ptr, col, val, x, tpr))
