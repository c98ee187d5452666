"""CPU oracle for the ContraGS training hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2509_03775_b200``) never imports, links or executes anything under
``oracle/`` and fails loudly when its CUDA extension is missing.

It restates, in float64 numpy, the reference package ``contrags`` 0.1.0
(`/root/reference/pkg/src/contrags/`), which is pure Python and therefore
cannot travel to the GPU box.  Each function cites the reference
``file:line`` it follows.  Parity is PINNED: ``tests/test_oracle_golden.py``
checks every function here against fixtures produced by running the
unmodified reference (``tests/golden/make_golden.py``) and against the
reference's own known-answer tests (`pkg/tests/test_render.py`,
`test_sh.py`, `test_model.py`).

Deliberate restatement choices (results are the reference's, the loop
structure is not): tile binning is vectorised with a stable argsort instead
of the reference's per-splat Python loop (`render.py:240-254`), and the tile
raster walks each tile's list in chunks, carrying the transmittance through
a sequential cumulative product, and stops once every pixel has terminated.
Both are exact restatements: same pair order, same sequential products,
inactive terms contribute exact zeros.
"""

from __future__ import annotations

import heapq
import math
from types import SimpleNamespace

import numpy as np

# render.py:26-34
NEAR = 0.01
BLUR = 0.3
A_CLAMP = 0.99
A_SKIP = 1.0 / 255.0
T_STOP = 1e-4
TILE = 16
FOOT = math.sqrt(2.0 * math.log(255.0))
COLOR_OFFSET = 0.5          # sh.py:20
SR_DIM = 7                  # model.py:16

# ---------------------------------------------------------------------------
# spherical harmonics (sh.py:12-100); constants from their closed forms
_Y0 = 0.5 / math.sqrt(math.pi)
_Y1 = math.sqrt(3.0 / (4.0 * math.pi))
_Y2a = 0.5 * math.sqrt(15.0 / math.pi)
_Y2b = 0.25 * math.sqrt(5.0 / math.pi)
_Y2c = 0.25 * math.sqrt(15.0 / math.pi)
_Y3a = 0.25 * math.sqrt(35.0 / (2.0 * math.pi))
_Y3b = 0.5 * math.sqrt(105.0 / math.pi)
_Y3c = 0.25 * math.sqrt(21.0 / (2.0 * math.pi))
_Y3d = 0.25 * math.sqrt(7.0 / math.pi)
_Y3e = 0.25 * math.sqrt(105.0 / math.pi)


def sh_dim(degree: int) -> int:
    """model.py:19-23"""
    if degree not in (0, 1, 2, 3):
        raise ValueError(f"sh_degree must be in 0..3, got {degree}")
    return 3 * (degree + 1) ** 2


def sh_degree_of(dim: int) -> int:
    """model.py:26-30"""
    for d in range(4):
        if 3 * (d + 1) ** 2 == dim:
            return d
    raise ValueError(f"SH codebook dim {dim} does not match any degree 0..3")


def sh_basis(v: np.ndarray, degree: int) -> np.ndarray:
    """Real SH basis at unit directions, reference sign convention (sh.py:27-53)."""
    v = np.asarray(v, dtype=np.float64)
    x, y, z = v[..., 0], v[..., 1], v[..., 2]
    cols = [np.full(x.shape, _Y0)]
    if degree >= 1:
        cols += [-_Y1 * y, _Y1 * z, -_Y1 * x]
    if degree >= 2:
        x2, y2, z2 = x * x, y * y, z * z
        cols += [_Y2a * x * y, -_Y2a * y * z, _Y2b * (2.0 * z2 - x2 - y2),
                 -_Y2a * x * z, _Y2c * (x2 - y2)]
    if degree >= 3:
        x2, y2, z2 = x * x, y * y, z * z
        cols += [-_Y3a * y * (3.0 * x2 - y2), _Y3b * x * y * z,
                 -_Y3c * y * (4.0 * z2 - x2 - y2),
                 _Y3d * z * (2.0 * z2 - 3.0 * x2 - 3.0 * y2),
                 -_Y3c * x * (4.0 * z2 - x2 - y2), _Y3e * z * (x2 - y2),
                 -_Y3a * x * (x2 - 3.0 * y2)]
    return np.stack(cols, axis=-1)


def sh_basis_grad(v: np.ndarray, degree: int) -> np.ndarray:
    """d basis / d direction, (..., B, 3) (sh.py:56-100)."""
    v = np.asarray(v, dtype=np.float64)
    x, y, z = v[..., 0], v[..., 1], v[..., 2]
    nb = (degree + 1) ** 2
    G = np.zeros(v.shape[:-1] + (nb, 3))
    if degree >= 1:
        G[..., 1, 1] = -_Y1
        G[..., 2, 2] = _Y1
        G[..., 3, 0] = -_Y1
    if degree >= 2:
        G[..., 4, :] = np.stack([_Y2a * y, _Y2a * x, 0 * x], -1)
        G[..., 5, :] = np.stack([0 * x, -_Y2a * z, -_Y2a * y], -1)
        G[..., 6, :] = np.stack([-2 * _Y2b * x, -2 * _Y2b * y, 4 * _Y2b * z], -1)
        G[..., 7, :] = np.stack([-_Y2a * z, 0 * x, -_Y2a * x], -1)
        G[..., 8, :] = np.stack([2 * _Y2c * x, -2 * _Y2c * y, 0 * x], -1)
    if degree >= 3:
        x2, y2, z2 = x * x, y * y, z * z
        G[..., 9, :] = np.stack([-_Y3a * 6 * x * y, -_Y3a * (3 * x2 - 3 * y2), 0 * x], -1)
        G[..., 10, :] = np.stack([_Y3b * y * z, _Y3b * x * z, _Y3b * x * y], -1)
        G[..., 11, :] = np.stack([2 * _Y3c * x * y, -_Y3c * (4 * z2 - x2 - 3 * y2),
                                  -8 * _Y3c * y * z], -1)
        G[..., 12, :] = np.stack([-6 * _Y3d * x * z, -6 * _Y3d * y * z,
                                  _Y3d * (6 * z2 - 3 * x2 - 3 * y2)], -1)
        G[..., 13, :] = np.stack([-_Y3c * (4 * z2 - 3 * x2 - y2), 2 * _Y3c * x * y,
                                  -8 * _Y3c * x * z], -1)
        G[..., 14, :] = np.stack([2 * _Y3e * x * z, -2 * _Y3e * y * z, _Y3e * (x2 - y2)], -1)
        G[..., 15, :] = np.stack([-_Y3a * (3 * x2 - 3 * y2), 6 * _Y3a * x * y, 0 * x], -1)
    return G


# ---------------------------------------------------------------------------
# quaternion / covariance helpers (render.py:37-91)
def quat_unit(q: np.ndarray) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    nrm = np.sqrt(np.sum(q * q, axis=-1, keepdims=True))
    if np.any(nrm == 0.0):
        raise ValueError("zero quaternion")
    return q / nrm


def quat_matrix(q: np.ndarray) -> np.ndarray:
    """Rotation of unit quaternions (w,x,y,z) (render.py:45-58)."""
    w, x, y, z = (q[..., i] for i in range(4))
    r0 = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1)
    r1 = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1)
    r2 = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)
    return np.stack([r0, r1, r2], -2)


def quat_matrix_jac(q: np.ndarray) -> np.ndarray:
    """dR/dq_k of quat_matrix's polynomial, (..., 4, 3, 3) (render.py:61-82)."""
    w, x, y, z = (q[..., i] for i in range(4))
    o = np.zeros_like(w)

    def m(*rows):
        return 2.0 * np.stack([np.stack(r, -1) for r in rows], -2)

    return np.stack([
        m((o, -z, y), (z, o, -x), (-y, x, o)),
        m((o, y, z), (y, -2 * x, -w), (z, w, -2 * x)),
        m((-2 * y, x, w), (x, o, z), (-w, z, -2 * y)),
        m((-2 * z, -w, x), (w, -2 * z, y), (x, y, o)),
    ], axis=-3)


def sr_covariance(rows: np.ndarray) -> np.ndarray:
    """Sigma3 = R diag(exp(2 ls)) R^T for SR rows (..., 7) (render.py:85-91)."""
    rows = np.asarray(rows, dtype=np.float64)
    R = quat_matrix(quat_unit(rows[..., 3:7]))
    s2 = np.exp(2.0 * rows[..., 0:3])
    return (R * s2[..., None, :]) @ np.swapaxes(R, -1, -2)


# ---------------------------------------------------------------------------
# state container (model.py:33-154), numpy only
class OCodebook:
    """Row store with refcounts, lineage parents and a min-heap free list (model.py:33-118)."""

    def __init__(self, rows, refcount=None, parent=None, free=None):
        self.rows = np.ascontiguousarray(rows, dtype=np.float32).copy()
        cap = self.rows.shape[0]
        self.refcount = (np.zeros(cap, np.int64) if refcount is None
                         else np.asarray(refcount, np.int64).copy())
        self.parent = (np.full(cap, -1, np.int32) if parent is None
                       else np.asarray(parent, np.int32).copy())
        if free is None:
            free = np.flatnonzero(self.refcount == 0)
        self.free = [int(r) for r in free]
        heapq.heapify(self.free)

    @property
    def dim(self):
        return self.rows.shape[1]

    @property
    def capacity(self):
        return self.rows.shape[0]

    @property
    def live_count(self):
        return self.capacity - len(self.free)

    def live(self):
        return np.flatnonzero(self.refcount > 0)

    def alloc(self, value, parent=-1):
        """model.py:78-95: lowest free slot first, else append."""
        value = np.asarray(value, dtype=np.float32)
        if self.free:
            r = heapq.heappop(self.free)
            self.rows[r] = value
        else:
            r = self.capacity
            self.rows = np.vstack([self.rows, value[None, :]])
            self.refcount = np.append(self.refcount, 0)
            self.parent = np.append(self.parent, np.int32(-1)).astype(np.int32)
        self.refcount[r] = 1
        self.parent[r] = parent
        return r

    def incref(self, r):
        if self.refcount[r] <= 0:
            raise ValueError(f"cannot reference dead row {r}")
        self.refcount[r] += 1

    def decref(self, r):
        """model.py:102-113: freeing a row clears its parent and breaks lineage into it."""
        if self.refcount[r] <= 0:
            raise ValueError(f"cannot release dead row {r}")
        self.refcount[r] -= 1
        if self.refcount[r] == 0:
            self.parent[r] = -1
            self.parent[self.parent == r] = -1
            heapq.heappush(self.free, int(r))
            return True
        return False

    def pairs(self):
        """model.py:115-118"""
        ch = np.flatnonzero((self.parent >= 0) & (self.refcount > 0))
        if len(ch) == 0:
            return np.zeros((0, 2), dtype=np.int64)
        return np.stack([ch, self.parent[ch]], axis=1)


class OState:
    """Scene state S = {G, C} (model.py:121-154)."""

    def __init__(self, positions, logits, g2sh, g2sr, sh: OCodebook, sr: OCodebook,
                 iteration=0):
        self.positions = np.asarray(positions, np.float32).copy()
        self.logits = np.asarray(logits, np.float32).copy()
        self.g2sh = np.asarray(g2sh, np.int32).copy()
        self.g2sr = np.asarray(g2sr, np.int32).copy()
        self.sh = sh
        self.sr = sr
        self.iteration = int(iteration)

    @property
    def n(self):
        return len(self.positions)

    @property
    def degree(self):
        return sh_degree_of(self.sh.dim)

    @classmethod
    def from_arrays(cls, positions, logits, g2sh, g2sr, sh_rows, sr_rows):
        sh = OCodebook(sh_rows, np.bincount(g2sh, minlength=len(sh_rows)))
        sr = OCodebook(sr_rows, np.bincount(g2sr, minlength=len(sr_rows)))
        return cls(positions, logits, g2sh, g2sr, sh, sr)

    @classmethod
    def from_fixture(cls, d, prefix):
        sh = OCodebook(d[prefix + "sh_rows"], d[prefix + "sh_refcount"],
                       d[prefix + "sh_parent"], d[prefix + "sh_free"])
        sr = OCodebook(d[prefix + "sr_rows"], d[prefix + "sr_refcount"],
                       d[prefix + "sr_parent"], d[prefix + "sr_free"])
        return cls(d[prefix + "positions"], d[prefix + "opacity_logits"], d[prefix + "g2sh"],
                   d[prefix + "g2sr"], sh, sr, int(d[prefix + "iteration"]))

    def copy(self):
        def cb(b):
            return OCodebook(b.rows, b.refcount, b.parent, list(b.free))
        return OState(self.positions, self.logits, self.g2sh, self.g2sr, cb(self.sh),
                      cb(self.sr), self.iteration)


def validate(st: OState):
    """model.py:286-316 invariants."""
    n = st.n
    for name, book, idx in (("sh", st.sh, st.g2sh), ("sr", st.sr, st.g2sr)):
        if n and (idx.min() < 0 or idx.max() >= book.capacity):
            raise ValueError(f"{name} index out of range")
        if not np.array_equal(np.bincount(idx, minlength=book.capacity), book.refcount):
            raise ValueError(f"{name} refcounts disagree with the index arrays")
        if set(book.free) != set(np.flatnonzero(book.refcount == 0).tolist()):
            raise ValueError(f"{name} free list disagrees with zero refcounts")
        lp = book.parent[book.refcount > 0]
        lp = lp[lp >= 0]
        if len(lp) and np.any(book.refcount[lp] == 0):
            raise ValueError(f"{name} has a live row whose parent is dead")


# ---------------------------------------------------------------------------
# camera (camera.py:29-36)
class OCam(SimpleNamespace):
    """R (3,3) world->camera, t (3,), fx, fy, cx, cy, width, height."""

    def to_cam(self, p):
        return np.asarray(p, np.float64) @ self.R.T + self.t

    def center(self):
        return -self.R.T @ self.t


def cam_from_fixture(d, prefix) -> OCam:
    fx, fy, cx, cy = (float(v) for v in d[prefix + "intr"])
    w, h = (int(v) for v in d[prefix + "size"])
    return OCam(R=np.asarray(d[prefix + "R"], np.float64), t=np.asarray(d[prefix + "t"], np.float64),
                fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)


def cam_from_any(c) -> OCam:
    return OCam(R=np.asarray(c.rotation, np.float64), t=np.asarray(c.translation, np.float64),
                fx=float(c.fx), fy=float(c.fy), cx=float(c.cx), cy=float(c.cy),
                width=int(c.width), height=int(c.height))


# ---------------------------------------------------------------------------
# projection (render.py:145-203, _pixel_rect :110-115)
def project(st: OState, cam: OCam) -> dict:
    """Per visible splat geometry in ascending Gaussian index, plus depth order."""
    p = st.positions.astype(np.float64)
    tc = cam.to_cam(p)
    vis = np.flatnonzero(tc[:, 2] > NEAR)
    t = tc[vis]
    x, y, z = t[:, 0], t[:, 1], t[:, 2]
    fx, fy = cam.fx, cam.fy
    mean = np.stack([fx * x / z + cam.cx, fy * y / z + cam.cy], 1)
    J = np.zeros((len(vis), 2, 3))
    J[:, 0, 0] = fx / z
    J[:, 0, 2] = -fx * x / (z * z)
    J[:, 1, 1] = fy / z
    J[:, 1, 2] = -fy * y / (z * z)
    M = J @ cam.R
    S3 = sr_covariance(st.sr.rows[st.g2sr[vis]])
    S2 = M @ S3 @ np.swapaxes(M, 1, 2)
    S2[:, 0, 0] += BLUR
    S2[:, 1, 1] += BLUR
    a, b, c = S2[:, 0, 0], S2[:, 0, 1], S2[:, 1, 1]
    det = a * c - b * b
    conic = np.stack([np.stack([c / det, -b / det], -1), np.stack([-b / det, a / det], -1)], -2)
    lam = 0.5 * (a + c) + np.sqrt(0.25 * (a - c) ** 2 + b * b)
    radius = FOOT * np.sqrt(lam) + 1e-9
    off = p[vis] - cam.center()
    vlen = np.sqrt(np.sum(off * off, axis=1))
    vdir = off / vlen[:, None]
    deg = st.degree
    nb = (deg + 1) ** 2
    coeffs = st.sh.rows[st.g2sh[vis]].astype(np.float64).reshape(-1, nb, 3)
    Bv = sh_basis(vdir, deg)
    raw = np.sum(Bv[:, :, None] * coeffs, axis=1) + COLOR_OFFSET
    opac = 1.0 / (1.0 + np.exp(-st.logits[vis].astype(np.float64)))
    order = np.lexsort((vis, z))
    return dict(idx=vis, t=t, mean2d=mean, M=M, cov3d=S3, cov2d=S2, conic=conic,
                radius=radius, viewdir=vdir, viewlen=vlen, color_raw=raw,
                colors=np.maximum(raw, 0.0), opac=opac, order=order, coeffs=coeffs)


def pixel_rects(mean2d, radius, width, height):
    """Inclusive pixel rect on pixel centres (render.py:110-115), vectorised."""
    x0 = np.maximum(0.0, np.ceil(mean2d[:, 0] - radius - 0.5))
    x1 = np.minimum(width - 1.0, np.floor(mean2d[:, 0] + radius - 0.5))
    y0 = np.maximum(0.0, np.ceil(mean2d[:, 1] - radius - 0.5))
    y1 = np.minimum(height - 1.0, np.floor(mean2d[:, 1] + radius - 0.5))
    return (x0.astype(np.int64), x1.astype(np.int64), y0.astype(np.int64), y1.astype(np.int64))


def bin_tiles(proj: dict, cam: OCam):
    """Stable tile binning (render.py:240-254).

    Returns (tile_offsets (T+1,), members) where members are positions into
    ``proj['order']``; tile t = ty*ntx + tx in row-major order.  Pairs are
    emitted in depth order and a stable sort by tile keeps that order inside
    each tile, which is exactly the reference's per-tile append order.
    """
    ntx = (cam.width + TILE - 1) // TILE
    nty = (cam.height + TILE - 1) // TILE
    order = proj["order"]
    x0, x1, y0, y1 = pixel_rects(proj["mean2d"][order], proj["radius"][order],
                                 cam.width, cam.height)
    ok = (x0 <= x1) & (y0 <= y1)
    tx0, tx1, ty0, ty1 = x0 // TILE, x1 // TILE, y0 // TILE, y1 // TILE
    span = np.where(ok, tx1 - tx0 + 1, 0)
    cnt = np.where(ok, (ty1 - ty0 + 1) * span, 0)
    total = int(cnt.sum())
    src = np.repeat(np.arange(len(order)), cnt)
    start = np.repeat(np.cumsum(cnt) - cnt, cnt)
    local = np.arange(total) - start
    sp = np.repeat(span, cnt)
    tile = (np.repeat(ty0, cnt) + local // np.maximum(sp, 1)) * ntx + np.repeat(tx0, cnt) + local % np.maximum(sp, 1)
    perm = np.argsort(tile, kind="stable")
    members = src[perm]
    offs = np.searchsorted(tile[perm], np.arange(ntx * nty + 1))
    return offs.astype(np.int64), members.astype(np.int64)


def _tile_px(t, cam):
    ntx = (cam.width + TILE - 1) // TILE
    ty, tx = divmod(t, ntx)
    y0, x0 = ty * TILE, tx * TILE
    y1, x1 = min(y0 + TILE, cam.height), min(x0 + TILE, cam.width)
    ys, xs = np.mgrid[y0:y1, x0:x1]
    return (y0, y1, x0, x1), xs.ravel() + 0.5, ys.ravel() + 0.5


def _alphas(proj, sel, px, py):
    """One chunk of compositing terms (render.py:265-280): alpha (K,P) zeroed when skipped."""
    m = proj["mean2d"][sel]
    Q = proj["conic"][sel]
    dx = px[None, :] - m[:, 0:1]
    dy = py[None, :] - m[:, 1:2]
    pw = -0.5 * (Q[:, 0, 0, None] * dx * dx + Q[:, 1, 1, None] * dy * dy) - Q[:, 0, 1, None] * dx * dy
    al = np.minimum(proj["opac"][sel, None] * np.exp(pw), A_CLAMP)
    keep = al >= A_SKIP
    return np.where(keep, al, 0.0), keep, dx, dy


def _walk_tile(proj, sel, px, py, chunk=64):
    """Composite a tile's list front to back, stopping once every pixel is done.

    Yields per chunk (rows, alpha, keep, active, t_before, dx, dy); the
    transmittance is a single sequential product across chunks exactly as
    the reference's cumprod over the whole list (render.py:281-283).
    """
    T = np.ones(px.shape[0])
    k = 0
    while k < len(sel):
        rows = sel[k:k + chunk]
        al, keep, dx, dy = _alphas(proj, rows, px, py)
        prod = np.cumprod(np.vstack([T[None, :], 1.0 - al]), axis=0)
        t_before = prod[:-1]
        active = t_before >= T_STOP
        yield rows, al, keep, active, t_before, dx, dy
        T = prod[-1]
        k += chunk
        if np.all(T < T_STOP):
            break


def raster_forward(st: OState, cam: OCam) -> dict:
    """rasterize_forward (render.py:287-315): image, T, contrib counts, tile lists."""
    proj = project(st, cam)
    offs, members = bin_tiles(proj, cam)
    H, W = cam.height, cam.width
    img = np.zeros((H, W, 3))
    T = np.ones((H, W))
    cnt = np.zeros((H, W), np.int32)
    order = proj["order"]
    ids = proj["idx"][order][members]
    for t in range(len(offs) - 1):
        if offs[t] == offs[t + 1]:
            continue
        (y0, y1, x0, x1), px, py = _tile_px(t, cam)
        sel = order[members[offs[t]:offs[t + 1]]]
        acc = np.zeros((px.shape[0], 3))
        tf = np.ones(px.shape[0])
        kc = np.zeros(px.shape[0], np.int64)
        for rows, al, keep, active, tb, _, _ in _walk_tile(proj, sel, px, py):
            w = al * tb * active
            acc += w.T @ proj["colors"][rows]
            kc += np.sum(keep & active, axis=0)
            # final T: sequential product of the active factors (render.py:310)
            tf = np.prod(np.vstack([tf[None, :], np.where(active, 1.0 - al, 1.0)]), axis=0)
        shape = (y1 - y0, x1 - x0)
        img[y0:y1, x0:x1] = acc.reshape(shape + (3,))
        T[y0:y1, x0:x1] = tf.reshape(shape)
        cnt[y0:y1, x0:x1] = kc.reshape(shape)
    return dict(image=img, final_T=T, counts=cnt, tile_offsets=offs, tile_ids=ids, proj=proj)


def raster_backward(st: OState, cam: OCam, dL: np.ndarray, screen: bool = False,
                    perturb=None) -> dict:
    """rasterize_backward + _pull_back (render.py:318-459), float64.

    Diagnostics (defaults reproduce the reference): ``screen=True`` also
    returns the screen-space sums (d_color, d_opac, d_mean2d, d_conic) per
    visible splat; ``perturb(name, array)`` may replace the per-pixel terms
    alpha / t_before / suffix (precision-sensitivity studies)."""
    dL = np.asarray(dL, np.float64)
    if dL.shape != (cam.height, cam.width, 3):
        raise ValueError("dL_dimage shape mismatch")
    proj = project(st, cam)
    offs, members = bin_tiles(proj, cam)
    order = proj["order"]
    V = len(proj["idx"])
    g_col = np.zeros((V, 3))
    g_op = np.zeros(V)
    g_mean = np.zeros((V, 2))
    g_con = np.zeros((V, 3))
    for t in range(len(offs) - 1):
        if offs[t] == offs[t + 1]:
            continue
        (y0, y1, x0, x1), px, py = _tile_px(t, cam)
        sel = order[members[offs[t]:offs[t + 1]]]
        gp = dL[y0:y1, x0:x1].reshape(-1, 3)
        chunks = list(_walk_tile(proj, sel, px, py))
        # suffix sums run back to front across chunks (render.py:354-355)
        tail = np.zeros((px.shape[0], 3))
        for rows, al, keep, active, tb, dx, dy in reversed(chunks):
            if perturb is not None:
                al, tb = perturb("alpha", al), perturb("t_before", tb)
            w = al * tb * active
            col = proj["colors"][rows]
            contrib = w[:, :, None] * col[:, None, :]
            csum = np.cumsum(contrib[::-1], axis=0)[::-1]
            suffix = csum - contrib + tail[None]
            if perturb is not None:
                suffix = perturb("suffix", suffix)
            tail = tail + csum[0] if len(rows) else tail
            pt = (lambda n, x: perturb(n, x)) if perturb is not None else (lambda n, x: x)
            np.add.at(g_col, rows, pt("tile_sum", w @ gp))
            dCda = col[:, None, :] * tb[:, :, None] - suffix / (1.0 - al)[:, :, None]
            da = np.sum(dCda * gp[None], axis=2)
            da = np.where(keep & active & (al < A_CLAMP), da, 0.0)
            np.add.at(g_op, rows, pt("tile_sum", np.sum(da * al, axis=1) / proj["opac"][rows]))
            dp = da * al
            Q = proj["conic"][rows]
            qx = Q[:, 0, 0, None] * dx + Q[:, 0, 1, None] * dy
            qy = Q[:, 0, 1, None] * dx + Q[:, 1, 1, None] * dy
            if perturb is not None and perturb("local_moments", None) is not None:
                # moments about the tile's first pixel centre, perturbed, then
                # shifted to the splat centre in fp64 (GPU representation study)
                lx = px - px[0]
                ly = py - py[0]
                mom = np.stack([dp.sum(1), (dp * lx).sum(1), (dp * ly).sum(1), (dp * lx * lx).sum(1),
                                (dp * lx * ly).sum(1), (dp * ly * ly).sum(1)], 1)
                mom = perturb("local_moments", mom)
                ox = (px[0] - proj["mean2d"][rows, 0])
                oy = (py[0] - proj["mean2d"][rows, 1])
                m0, mx, my, mxx, mxy, myy = mom.T
                sx = ox * m0 + mx
                sy = oy * m0 + my
                sxx = ox * ox * m0 + 2 * ox * mx + mxx
                sxy = ox * oy * m0 + ox * my + oy * mx + mxy
                syy = oy * oy * m0 + 2 * oy * my + myy
                A, B, C = Q[:, 0, 0], Q[:, 0, 1], Q[:, 1, 1]
                np.add.at(g_mean, rows, np.stack([A * sx + B * sy, B * sx + C * sy], 1))
                np.add.at(g_con, rows, np.stack([-0.5 * sxx, -sxy, -0.5 * syy], 1))
                continue
            np.add.at(g_mean, rows, pt("tile_sum", np.stack([np.sum(dp * qx, 1), np.sum(dp * qy, 1)], 1)))
            np.add.at(g_con, rows, pt("tile_sum", np.stack([np.sum(dp * (-0.5 * dx * dx), 1),
                                                            np.sum(dp * (-dx * dy), 1),
                                                            np.sum(dp * (-0.5 * dy * dy), 1)], 1)))
    # rows index the visible arrays directly (sel values are visible positions)
    out = pull_back(st, cam, proj, g_col, g_op, g_mean, g_con, perturb=perturb)
    if screen:
        return out, dict(g_col=g_col, g_op=g_op, g_mean=g_mean, g_con=g_con, proj=proj)
    return out


def pull_back(st: OState, cam: OCam, proj: dict, g_col, g_op, g_mean, g_con, perturb=None) -> dict:
    """Chain screen-space gradients to model parameters (render.py:382-459).
    ``perturb`` (diagnostics only) may replace dSigma3 and the view term."""
    pt = (lambda n, x: perturb(n, x)) if perturb is not None else (lambda n, x: x)
    idx = proj["idx"]
    t = proj["t"]
    x, y, z = t[:, 0], t[:, 1], t[:, 2]
    fx, fy = cam.fx, cam.fy
    Q = proj["conic"]
    dQ = np.empty((len(idx), 2, 2))
    dQ[:, 0, 0] = g_con[:, 0]
    dQ[:, 1, 1] = g_con[:, 2]
    dQ[:, 0, 1] = dQ[:, 1, 0] = 0.5 * g_con[:, 1]
    dS2 = -(Q @ dQ @ Q)
    M = proj["M"]
    Mt = np.swapaxes(M, 1, 2)
    dS3 = pt("dS3", Mt @ dS2 @ M)
    dM = 2.0 * (dS2 @ M @ proj["cov3d"])
    dJ = dM @ cam.R.T
    z2, z3 = z * z, z * z * z
    dt = np.stack([
        g_mean[:, 0] * fx / z - dJ[:, 0, 2] * fx / z2,
        g_mean[:, 1] * fy / z - dJ[:, 1, 2] * fy / z2,
        -g_mean[:, 0] * fx * x / z2 - g_mean[:, 1] * fy * y / z2
        - dJ[:, 0, 0] * fx / z2 - dJ[:, 1, 1] * fy / z2
        + dJ[:, 0, 2] * 2 * fx * x / z3 + dJ[:, 1, 2] * 2 * fy * y / z3], 1)
    dpos = dt @ cam.R
    deg = st.degree
    draw = g_col * (proj["color_raw"] > 0.0)
    Bv = sh_basis(proj["viewdir"], deg)
    dcoef = Bv[:, :, None] * draw[:, None, :]
    if deg >= 1:
        Bg = sh_basis_grad(proj["viewdir"], deg)
        dview = np.sum(np.sum(draw[:, None, :, None] * proj["coeffs"][:, :, :, None]
                              * Bg[:, :, None, :], axis=2), axis=1)
        v = proj["viewdir"]
        dpos = dpos + pt("dview", (dview - v * np.sum(v * dview, axis=1, keepdims=True)) / proj["viewlen"][:, None])
    rows = st.sr.rows[st.g2sr[idx]].astype(np.float64)
    qr = rows[:, 3:7]
    qn = quat_unit(qr)
    R = quat_matrix(qn)
    s2 = np.exp(2.0 * rows[:, 0:3])
    Rt = np.swapaxes(R, 1, 2)
    dD = Rt @ dS3 @ R
    dls = np.stack([dD[:, 0, 0], dD[:, 1, 1], dD[:, 2, 2]], 1) * 2.0 * s2
    dR = 2.0 * (dS3 @ R) * s2[:, None, :]
    dqn = np.sum(dR[:, None] * quat_matrix_jac(qn), axis=(2, 3))
    qnorm = np.sqrt(np.sum(qr * qr, axis=1))
    dq = (dqn - qn * np.sum(qn * dqn, axis=1, keepdims=True)) / qnorm[:, None]
    o = proj["opac"]
    out = dict(positions=np.zeros((st.n, 3)), opacity_logits=np.zeros(st.n),
               sh_rows=np.zeros((st.sh.capacity, st.sh.dim)),
               sr_rows=np.zeros((st.sr.capacity, SR_DIM)))
    out["positions"][idx] = dpos
    out["opacity_logits"][idx] = g_op * o * (1.0 - o)
    np.add.at(out["sh_rows"], st.g2sh[idx], dcoef.reshape(len(idx), -1))
    np.add.at(out["sr_rows"], st.g2sr[idx], np.concatenate([dls, dq], axis=1))
    return out


# ---------------------------------------------------------------------------
# loss (metrics.py:17-172)
_SSIM_K = np.exp(-0.5 * ((np.arange(11) - 5.0) / 1.5) ** 2)
_SSIM_K = _SSIM_K / _SSIM_K.sum()
C1 = 0.01 ** 2
C2 = 0.03 ** 2


def _valid_filter(x):
    """Separable 11x11 Gaussian correlation, valid positions only (metrics.py:33-37)."""
    H, W = x.shape
    rows = sum(_SSIM_K[j] * x[j:H - 10 + j, :] for j in range(11))
    return sum(_SSIM_K[j] * rows[:, j:W - 10 + j] for j in range(11))


def _valid_filter_T(g, shape):
    """Adjoint of _valid_filter (metrics.py:40-45)."""
    pad = np.zeros((shape[0] + 10, shape[1] + 10))
    pad[10:-10, 10:-10] = g
    return _valid_filter(pad)


def _pair(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"image shapes differ: {a.shape} vs {b.shape}")
    if a.ndim == 2:
        a, b = a[:, :, None], b[:, :, None]
    return a, b


def _ssim_terms(x, y):
    mx, my = _valid_filter(x), _valid_filter(y)
    sx = _valid_filter(x * x) - mx * mx
    sy = _valid_filter(y * y) - my * my
    sxy = _valid_filter(x * y) - mx * my
    A1, A2 = 2 * mx * my + C1, 2 * sxy + C2
    B1, B2 = mx * mx + my * my + C1, sx + sy + C2
    return mx, my, A1, A2, B1, B2


def ssim(a, b) -> float:
    """metrics.py:67-84"""
    a, b = _pair(a, b)
    if a.shape[0] < 11 or a.shape[1] < 11:
        raise ValueError("images must be at least 11x11 for SSIM")
    tot, n = 0.0, 0
    for c in range(a.shape[2]):
        _, _, A1, A2, B1, B2 = _ssim_terms(a[:, :, c], b[:, :, c])
        s = A1 * A2 / (B1 * B2)
        tot += s.sum()
        n += s.size
    return tot / n


def ssim_grad(a, b):
    """metrics.py:87-114"""
    a, b = _pair(a, b)
    g = np.zeros_like(a)
    n = 0
    for c in range(a.shape[2]):
        x, y = a[:, :, c], b[:, :, c]
        mx, my, A1, A2, B1, B2 = _ssim_terms(x, y)
        F = 1.0 / (B1 * B2)
        s = A1 * A2 * F
        d_mx = 2 * my * F * (A2 - A1) - 2 * mx * s * (1.0 / B1 - 1.0 / B2)
        d_ex2 = -s / B2
        d_exy = 2 * A1 * F
        g[:, :, c] = (_valid_filter_T(d_mx, x.shape) + 2 * x * _valid_filter_T(d_ex2, x.shape)
                      + y * _valid_filter_T(d_exy, x.shape))
        n += s.size
    return g / n


def recon_loss(img, gt, lam):
    """metrics.py:122-130 -> (l1, ssim, recon)"""
    a, b = _pair(img, gt)
    l1v = float(np.mean(np.abs(a - b)))
    if lam == 0.0:
        sv = ssim(a, b) if min(a.shape[:2]) >= 11 else float("nan")
        return l1v, sv, l1v
    sv = ssim(a, b)
    return l1v, sv, (1.0 - lam) * l1v + lam * (1.0 - sv)


def recon_loss_grad(img, gt, lam):
    """metrics.py:133-140"""
    a, b = _pair(img, gt)
    g = (1.0 - lam) * np.sign(a - b) / a.size
    if lam != 0.0:
        g = g - lam * ssim_grad(a, b)
    return g.reshape(np.shape(img))


def psnr(a, b, cap=100.0):
    """metrics.py:165-172"""
    a, b = _pair(a, b)
    mse = float(np.mean((a - b) ** 2))
    return cap if mse == 0.0 else -10.0 * math.log10(mse)


# ---------------------------------------------------------------------------
# sampler (sampler.py)
class SamplerError(RuntimeError):
    pass


def config(**kw) -> SimpleNamespace:
    """SamplerConfig defaults (sampler.py:29-65)."""
    base = dict(p_update=0.98, p_split=0.01, p_merge=0.01, eps_split_sh=0.1,
                eps_merge_sh=0.05, eps_split_sr=0.1, eps_merge_sr=0.05, lambda_sh=2.3,
                lambda_sr=3.0, lambda_ssim=0.2, step_pos=0.5, step_opacity=10.0,
                step_sh=20.0, step_sr=2.0, noise_pos=1.0, noise_opacity=0.0, noise_sh=0.0,
                noise_sr=0.0, split_fraction=0.01, densify_every=100, densify_growth=0.05,
                densify_jitter=0.02, gaussian_cap=2_000_000, normalization_correction=False,
                exact_ratio=False, seed=0)
    base.update(kw)
    return SimpleNamespace(**base)


def sgld_update(st: OState, grads: dict, cfg, rng):
    """sampler.py:262-300 (numpy float64 then cast to float32)."""
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        if not np.all(np.isfinite(grads[k])):
            raise SamplerError(f"non-finite gradients at iteration {st.iteration}")

    def move(val, grad, eps, mult, shape):
        nxt = val - 0.5 * eps * grad
        if mult != 0.0 and eps > 0.0:
            nxt = nxt + mult * math.sqrt(eps) * rng.standard_normal(shape)
        return nxt

    if cfg.step_pos > 0.0:
        st.positions = move(st.positions.astype(np.float64), grads["positions"], cfg.step_pos,
                            cfg.noise_pos, st.positions.shape).astype(np.float32)
    if cfg.step_opacity > 0.0:
        st.logits = move(st.logits.astype(np.float64), grads["opacity_logits"],
                         cfg.step_opacity, cfg.noise_opacity, st.logits.shape).astype(np.float32)
    if cfg.step_sh > 0.0:
        lv = st.sh.live()
        st.sh.rows[lv] = move(st.sh.rows[lv].astype(np.float64), grads["sh_rows"][lv],
                              cfg.step_sh, cfg.noise_sh, (len(lv), st.sh.dim)).astype(np.float32)
    if cfg.step_sr > 0.0:
        lv = st.sr.live()
        r = move(st.sr.rows[lv].astype(np.float64), grads["sr_rows"][lv], cfg.step_sr,
                 cfg.noise_sr, (len(lv), SR_DIM))
        q = r[:, 3:7]
        # sequential ((q0^2+q1^2)+q2^2)+q3^2, as numpy's axis-1 reduce of a (n,4) view
        nq = np.sqrt(((q[:, 0] * q[:, 0] + q[:, 1] * q[:, 1]) + q[:, 2] * q[:, 2]) + q[:, 3] * q[:, 3])
        r[:, 3:7] = q / nq[:, None]
        st.sr.rows[lv] = r.astype(np.float32)


def log_q_sm(u, eps_s, eps_m, correction=False):
    """sampler.py:138-144"""
    u = np.atleast_1d(np.asarray(u, np.float64))
    lq = -0.5 * float(u @ u) * (1.0 / eps_s ** 2 - 1.0 / eps_m ** 2)
    if correction:
        lq += u.size * math.log(eps_m / eps_s)
    return lq


def q_sm(u, eps_s, eps_m, correction=False):
    """sampler.py:122-135"""
    with np.errstate(over="ignore"):
        return float(np.exp(log_q_sm(u, eps_s, eps_m, correction)))


def accept_prob(kind, u, lam, eps_s, eps_m, correction=False, extra=0.0):
    """sampler.py:147-164"""
    lq = log_q_sm(u, eps_s, eps_m, correction)
    if kind == "split":
        la = -lam - lq + extra
    elif kind == "merge":
        la = lam + lq + extra
    else:
        raise ValueError(f"unknown transition kind {kind!r}")
    return float(np.exp(min(0.0, la)))


def _book(st, which):
    return (st.sh, st.g2sh) if which == "sh" else (st.sr, st.g2sr)


def _eps(cfg, which):
    return ((cfg.eps_split_sh, cfg.eps_merge_sh) if which == "sh"
            else (cfg.eps_split_sr, cfg.eps_merge_sr))


def split_step(st: OState, cfg, rng) -> dict:
    """Split branch of train_step (sampler.py:339-364, 184-221)."""
    which = "sh" if rng.random() < 0.5 else "sr"
    book, idx = _book(st, which)
    elig = np.flatnonzero(book.refcount[idx] >= 2)
    n_c = 0 if st.n <= 0 else max(1, int(round(cfg.split_fraction * st.n)))
    n_c = min(n_c, len(elig))
    rec = dict(codebook=which, attempts=0, accepts=0, probs=[])
    if n_c <= 0:
        return rec
    cands = rng.choice(elig, size=n_c, replace=False)
    lam = cfg.lambda_sh if which == "sh" else cfg.lambda_sr
    es, em = _eps(cfg, which)
    for i in cands:
        row = int(idx[i])
        if book.refcount[row] < 2:
            continue
        u = rng.normal(0.0, es, size=book.dim)
        prob = accept_prob("split", u, lam, es, em, cfg.normalization_correction)
        rec["probs"].append(prob)
        rec["attempts"] += 1
        if rng.random() < prob:
            new = book.alloc((book.rows[row].astype(np.float64) + u).astype(np.float32), parent=row)
            idx[i] = new
            book.decref(row)
            rec["accepts"] += 1
    return rec


def merge_step(st: OState, cfg, rng) -> dict:
    """Merge branch of train_step (sampler.py:365-385, 224-259)."""
    which = "sh" if rng.random() < 0.5 else "sr"
    book, idx = _book(st, which)
    lam = cfg.lambda_sh if which == "sh" else cfg.lambda_sr
    es, em = _eps(cfg, which)
    npairs = len(book.pairs())
    n_c = 0 if npairs <= 0 else max(1, int(round(cfg.split_fraction * npairs)))
    rec = dict(codebook=which, attempts=0, accepts=0, probs=[])
    for _ in range(n_c):
        pr = book.pairs()
        if len(pr) == 0:
            break
        d = book.rows[pr[:, 1]].astype(np.float64) - book.rows[pr[:, 0]].astype(np.float64)
        lw = -0.5 * np.einsum("nd,nd->n", d, d) / em ** 2
        w = np.exp(lw - lw.max())
        k = int(rng.choice(len(pr), p=w / w.sum()))
        child, parent, u = int(pr[k, 0]), int(pr[k, 1]), d[k]
        prob = accept_prob("merge", u, lam, es, em, cfg.normalization_correction)
        rec["probs"].append(prob)
        rec["attempts"] += 1
        if rng.random() < prob:
            members = np.flatnonzero(idx == child)
            for i in members:
                book.incref(parent)
                idx[i] = parent
                book.decref(child)
            rec["accepts"] += 1
    return rec


def densify(st: OState, growth, cap, rng, jitter=0.02) -> int:
    """model.py:235-267"""
    if growth <= 0:
        raise ValueError("growth_rate must be positive")
    n = st.n
    if cap < n:
        raise ValueError(f"cap {cap} is below current count {n}")
    k = min(int(growth * n), cap - n)
    if k <= 0:
        return 0
    op = 1.0 / (1.0 + np.exp(-st.logits.astype(np.float64)))
    src = rng.choice(n, size=k, replace=True, p=op / op.sum())
    jit = rng.normal(0.0, jitter, size=(k, 3))
    st.positions = np.concatenate([st.positions, (st.positions[src].astype(np.float64) + jit).astype(np.float32)])
    st.logits = np.concatenate([st.logits, st.logits[src]])
    st.g2sh = np.concatenate([st.g2sh, st.g2sh[src]])
    st.g2sr = np.concatenate([st.g2sr, st.g2sr[src]])
    np.add.at(st.sh.refcount, st.g2sh[n:], 1)
    np.add.at(st.sr.refcount, st.g2sr[n:], 1)
    return k


def train_step(st: OState, views, cfg, rng) -> dict:
    """One MH transition plus densify schedule (sampler.py:320-399).

    ``views`` is a list of (OCam, gt image) pairs.
    """
    if not views:
        raise ValueError("at least one view is required")
    r = rng.random()
    kind = ("update" if r < cfg.p_update else
            "split" if r < cfg.p_update + cfg.p_split else "merge")
    sh0, sr0 = st.sh.live_count, st.sr.live_count
    rec = dict(kind=kind, codebook="-", attempts=0, accepts=0, probs=[], recon=float("nan"))
    if kind == "update":
        cam, gt = views[int(rng.integers(len(views)))]
        fw = raster_forward(st, cam)
        _, _, recon = recon_loss(fw["image"], gt, cfg.lambda_ssim)
        g = raster_backward(st, cam, recon_loss_grad(fw["image"], gt, cfg.lambda_ssim))
        sgld_update(st, g, cfg, rng)
        rec.update(attempts=1, accepts=1, probs=[1.0], recon=recon)
    elif kind == "split":
        rec.update(split_step(st, cfg, rng))
    else:
        rec.update(merge_step(st, cfg, rng))
    st.iteration += 1
    if cfg.densify_every > 0 and st.iteration % cfg.densify_every == 0:
        densify(st, cfg.densify_growth, cfg.gaussian_cap, rng, cfg.densify_jitter)
    rec["live_sh"], rec["live_sr"] = st.sh.live_count, st.sr.live_count
    rec["delta_sh"], rec["delta_sr"] = rec["live_sh"] - sh0, rec["live_sr"] - sr0
    return rec
