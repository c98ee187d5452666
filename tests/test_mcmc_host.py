"""CPU tests of the library's MCMC host loop (cgs_host_split_decide,
cgs_host_split_eligible): it must consume the caller's numpy Generator
exactly as the reference's Python loop (sampler.py:339-364) does and take the
same decisions, so MCMC chains stay bit-identical."""

import math

import numpy as np
import pytest

from paper_2509_03775_b200 import _native as nat
from paper_2509_03775_b200 import sampler as S


def _python_loop(rows, refcount, dim, lam, es, em, corr_flag, rng):
    """The reference's per-candidate loop, verbatim float expressions
    (sampler.py:349-364 with acceptance_probability, :138-164)."""
    out = []
    for row in rows.tolist():
        if refcount[row] < 2:
            out.append(None)
            continue
        u = rng.normal(0.0, es, size=dim)
        prob = S.acceptance_probability("split", u, lam, es, em, corr_flag)
        coin = rng.random()
        acc = coin < prob
        if acc:
            refcount[row] -= 1
        out.append((u, prob, acc))
    return out


@pytest.mark.parametrize("dim,lam,es,em,corr", [(7, 0.0, 0.02, 0.02, False),
                                                (48, 0.0, 0.05, 0.05, True),
                                                (7, 2.3, 0.01, 0.005, False),
                                                (12, 0.5, 0.03, 0.03, False)])
def test_split_decide_matches_python_loop(dim, lam, es, em, corr):
    if nat.numpy_ddot_ptr() is None:
        pytest.skip("numpy BLAS ddot not resolvable")
    base = np.random.default_rng(7)
    k = 300
    rc0 = base.integers(0, 5, size=k).astype(np.int64)
    rows = base.integers(0, k, size=2000).astype(np.int64)
    r1, r2 = np.random.default_rng(11), np.random.default_rng(11)
    rc_py = rc0.copy()
    ref = _python_loop(rows, rc_py, dim, lam, es, em, corr, r1)
    rc_c = rc0.copy()
    n = len(rows)
    u = np.empty((n, dim))
    log_a, coin = np.empty(n), np.empty(n)
    dec = np.empty(n, np.int8)
    att = nat.I64(0)
    c_q = 1.0 / es ** 2 - 1.0 / em ** 2
    cv = dim * math.log(em / es) if corr else 0.0
    nat.call("cgs_host_split_decide", nat.bitgen_ptr(r2), nat.numpy_ddot_ptr(), n, rows.ctypes.data,
             rc_c.ctypes.data, k, dim, lam, es, c_q, 1 if corr else 0, cv, u.ctypes.data,
             log_a.ctypes.data, coin.ctypes.data, dec.ctypes.data, nat.ctypes.byref(att))
    assert np.array_equal(rc_c, rc_py)
    assert att.value == sum(r is not None for r in ref)
    assert (dec == 1).sum() > 0  # accepts (and their refcount effect) exercised
    if not (lam == 0.0 and es == em):  # A == 1 there
        assert (dec == 0).sum() > 0
    for c, r in enumerate(ref):
        if r is None:
            assert dec[c] == -1
            continue
        assert np.array_equal(u[c], r[0])
        assert float(np.exp(min(0.0, log_a[c]))) == r[1]  # bit-identical probability
        assert (dec[c] == 1) == r[2]
    assert np.array_equal(r1.random(8), r2.random(8))  # same stream position afterwards


def test_host_eligible_matches_numpy():
    rng = np.random.default_rng(3)
    k = 5000
    rc = rng.integers(0, 4, size=k).astype(np.int64)
    idx = rng.integers(0, k, size=1_000_003).astype(np.int32)
    assert np.array_equal(S._eligible(idx, rc), np.flatnonzero(rc[idx] >= 2))
    assert len(S._eligible(idx[:0], rc)) == 0


def test_settle_split_matches_sequential_loop():
    """sampler.settle_split (the device-proposal split's host bookkeeping)
    equals the reference loop's sequential refcount skips (sampler.py:349-364)."""
    from paper_2509_03775_b200.sampler import settle_split
    rng = np.random.default_rng(5)
    for trial in range(20):
        k = int(rng.integers(1, 40))
        rc0 = rng.integers(0, 6, size=k).astype(np.int64)
        n = int(rng.integers(0, 300))
        rows = rng.integers(0, k, size=n).astype(np.int64)
        acc = rng.random(n) < rng.uniform(0.1, 0.9)
        tried, dec = settle_split(rows, acc, rc0)
        rc = rc0.copy()
        for c in range(n):
            exp_tried = rc[rows[c]] >= 2
            assert tried[c] == exp_tried, (trial, c)
            assert dec[c] == (exp_tried and acc[c])
            if exp_tried and acc[c]:
                rc[rows[c]] -= 1
