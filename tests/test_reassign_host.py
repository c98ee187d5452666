"""Host logic of the code reassignment extension (no GPU): mutual nearest
pairs within tau."""

import numpy as np

from paper_2509_03775_b200.reassign import mutual_pairs


def test_mutual_pairs():
    nn = np.array([1, 0, 3, 4, 3, -1, 5], np.int32)
    d2 = np.array([0.5, 0.5, 2.0, 0.1, 0.1, 0.0, 9.0])
    assert mutual_pairs(nn, d2, 1.0) == [(0, 1), (3, 4)]
    assert mutual_pairs(nn, d2, 0.2) == [(3, 4)]
    assert mutual_pairs(nn, d2, 0.0) == []
    # a one-directional nearest is never merged
    assert mutual_pairs(np.array([1, 2, 1], np.int32), np.zeros(3), 1.0) == [(1, 2)]
