"""Host-side positives CSR of the drop-in (anns.positives_csr, trainer._csr):
the vectorised segmented sort / dedupe equals the per-row np.sort / np.unique
it replaced, for empty rows, unsorted rows, duplicates and both int widths."""

import numpy as np

from paper_2409_20156_b200.anns import positives_csr
from paper_2409_20156_b200.trainer import _csr


def _per_row(positives, unique):
    f = (lambda p: np.unique(np.asarray(p, np.int64))) if unique else (lambda p: np.sort(np.asarray(p, np.int64)))
    lists = [f(p) for p in positives]
    indptr = np.zeros(len(lists) + 1, np.int64)
    np.cumsum([len(x) for x in lists], out=indptr[1:])
    ids = np.concatenate(lists).astype(np.int32) if indptr[-1] else np.zeros(0, np.int32)
    return indptr, ids


def test_positives_csr_matches_per_row_sort_and_unique():
    rng = np.random.default_rng(7)
    for _ in range(400):
        n = int(rng.integers(0, 30))
        pos = []
        for _ in range(n):
            a = rng.integers(0, 15, size=int(rng.integers(0, 7)))
            if rng.random() < 0.5:
                a = np.sort(a)
            pos.append(a.astype(np.int32 if rng.random() < 0.5 else np.int64))
        for unique in (False, True):
            want = _per_row(pos, unique)
            got = positives_csr(pos, unique=unique)
            np.testing.assert_array_equal(got[0], want[0])
            np.testing.assert_array_equal(got[1], want[1])
            assert got[1].dtype == np.int32 and got[0].dtype == np.int64
        got = _csr(pos)
        want = _per_row(pos, True)
        np.testing.assert_array_equal(got[0], want[0])
        np.testing.assert_array_equal(got[1], want[1])


def test_positives_csr_rows_argument():
    pos = [np.array([5, 1]), np.array([], np.int64), np.array([3, 3, 2])]
    indptr, ids = positives_csr(pos, rows=[2, 0])
    np.testing.assert_array_equal(indptr, [0, 3, 5])
    np.testing.assert_array_equal(ids, [2, 3, 3, 1, 5])
