"""GPU: the nearest-code search behind the code reassignment extension
(cgs_code_nn: tcgen05 tf32 distance GEMM + exact fp64 certification) against
an fp64 brute force of the same definition (no reference oracle exists: the
reference never recomputes assignments by distance)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_03775_b200 as m
    m._native.library()
    return m


def brute_nn(rows: np.ndarray, live: np.ndarray):
    """fp64, sum over k in order of fl(fl(x - y)^2) (the definition in
    include/cgs_b200.h), ties -> smaller index."""
    x = rows[live].astype(np.float64)
    d2 = np.zeros((len(live), len(live)))
    for k in range(rows.shape[1]):
        t = x[:, k, None] - x[None, :, k]
        d2 += t * t
    np.fill_diagonal(d2, np.inf)
    j = np.argmin(d2, axis=1)  # first minimum = smallest index (live is ascending)
    idx = np.full(rows.shape[0], -1, np.int32)
    dist = np.zeros(rows.shape[0])
    idx[live] = live[j]
    dist[live] = d2[np.arange(len(live)), j]
    return idx, dist


def _state(cg, n_sh, n_sr, degree, seed, dead=(), dupes=()):
    rng = np.random.default_rng(seed)
    D = 3 * (degree + 1) ** 2
    sh = rng.normal(0, 0.2, (n_sh, D)).astype(np.float32)
    sr = np.concatenate([rng.normal(-4, 0.5, (n_sr, 3)), rng.normal(0, 1, (n_sr, 4))], 1)
    sr[:, 3:] /= np.linalg.norm(sr[:, 3:], axis=1, keepdims=True)
    sr = sr.astype(np.float32)
    for a, b in dupes:
        sh[b] = sh[a]
        sr[b] = sr[a]
    n = 4 * max(n_sh, n_sr)
    g2sh = np.arange(n, dtype=np.int32) % n_sh
    g2sr = np.arange(n, dtype=np.int32) % n_sr
    keep = ~np.isin(g2sh, np.asarray(dead, np.int32))
    g2sh = g2sh[keep]
    g2sr = g2sr[keep]
    pos = rng.normal(0, 1, (len(g2sh), 3)).astype(np.float32)
    logit = rng.normal(0, 1, len(g2sh)).astype(np.float32)
    return cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)


@pytest.mark.parametrize("which,n_rows,degree", [("sh", 3000, 3), ("sh", 700, 1), ("sr", 2500, 3)])
def test_nearest_codes_exact(cg, which, n_rows, degree):
    dead = list(range(5, n_rows, 53))
    st = _state(cg, n_rows, n_rows, degree, seed=n_rows + degree, dead=dead,
                dupes=[(11, 400), (12, 401), (401, 650)])
    book = st.sh if which == "sh" else st.sr
    live = book.live_indices()
    assert len(live) == n_rows - len(dead)
    idx, dist = cg.nearest_codes(st, which)
    rows = book.rows.cpu().numpy()
    want_i, want_d = brute_nn(rows, live)
    got_i, got_d = idx.cpu().numpy(), dist.cpu().numpy()
    assert np.array_equal(got_i[: len(want_i)], want_i)
    assert np.array_equal(got_d[: len(want_d)], want_d)
    assert got_i[400] == 11 and got_d[400] == 0.0  # exact duplicate, smaller index wins


def test_nearest_codes_edge_cases(cg):
    st = _state(cg, 300, 300, 3, seed=3, dead=list(range(1, 300)))  # a single live row
    idx, _ = cg.nearest_codes(st, "sh")
    assert (idx.cpu().numpy() == -1).all()
    st = _state(cg, 300, 300, 3, seed=4, dead=list(range(2, 300)))  # two live rows
    idx, dist = cg.nearest_codes(st, "sh")
    i = idx.cpu().numpy()
    assert i[0] == 1 and i[1] == 0 and (i[2:] == -1).all()


def test_reassign_codes_merges_mutual_pairs(cg):
    """Planted near-duplicates are merged (child -> parent), refcounts and the
    free list follow the merge rule, and the state stays valid."""
    st = _state(cg, 1200, 600, 3, seed=9)
    rows = st.sh.rows.cpu().numpy().copy()
    rng = np.random.default_rng(0)
    planted = [(20, 900), (33, 34), (500, 1100)]
    for p, c in planted:
        rows[c] = rows[p] + rng.normal(0, 1e-4, rows.shape[1]).astype(np.float32)
    st.sh.rows.copy_(torch.as_tensor(rows))
    before = st.sh.refcount.copy()
    g2sh_before = st.gaussians.g2sh.cpu().numpy().copy()
    live = st.sh.live_indices()
    want_i, want_d = brute_nn(rows, live)
    tau = 1e-5
    pairs = cg.mutual_pairs(want_i, want_d, tau)
    assert sorted(pairs) == sorted(planted)
    freed = cg.reassign_codes(st, "sh", tau)
    assert freed == len(planted)
    g2sh = st.gaussians.g2sh.cpu().numpy()
    remap = {c: p for p, c in planted}
    assert np.array_equal(g2sh, np.array([remap.get(int(v), int(v)) for v in g2sh_before]))
    for p, c in planted:
        assert not st.sh.is_live(c)
        assert st.sh.refcount[p] == before[p] + before[c]
    cg.validate_state(st)
    assert cg.reassign_codes(st, "sh", tau) == 0  # nothing left within tau
