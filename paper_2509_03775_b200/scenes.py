"""Seeded synthetic scenes for BASELINE.json configs 0-4.

The reference measures on no public dataset; the paper's datasets are not in
this container, so these host-side generators stand in for them with the
shapes, sizes and value distributions BASELINE.json names.  Everything is
drawn in float64 with ``np.random.default_rng(seed)`` and cast to float32
the way the reference stores it (`pkg/src/contrags/model.py:176`,
`modelio.py:261`).  Layout follows the reference exactly: SR rows are
``[log-scale(3); quaternion(4) w,x,y,z]`` (`model.py:16`), SH rows are
coefficient-major ``row[b*3 + ch]`` (`sh.py:3-5`), opacity is per Gaussian
(`model.py:126`).  Configs 0/1 keep opacity in a codebook column; that column
is gathered by index into the per-Gaussian logit at build time.

A scene is returned as plain numpy arrays (``SceneArrays``) so the same
arrays can seed the device state, the CPU oracle and golden fixtures.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .camera import hemisphere_cameras, orbit_cameras, ring_cameras


@dataclass
class SceneArrays:
    positions: np.ndarray        # (N,3) f32
    opacity_logits: np.ndarray   # (N,) f32
    g2sh: np.ndarray             # (N,) i32
    g2sr: np.ndarray             # (N,) i32
    sh_rows: np.ndarray          # (K_sh, 3(d+1)^2) f32
    sr_rows: np.ndarray          # (K_sr, 7) f32
    sh_degree: int
    cameras: list = field(default_factory=list)
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.positions.shape[0])


def _unit_quats(rng, k):
    q = rng.normal(0.0, 1.0, size=(k, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _sr_table(rng, k, ls_mean, ls_std):
    sr = np.empty((k, 7), dtype=np.float32)
    sr[:, 0:3] = rng.normal(ls_mean, ls_std, size=(k, 3))
    sr[:, 3:7] = _unit_quats(rng, k)
    return sr


def config0(seed: int = 0) -> SceneArrays:
    """N=4096, one K=256 table [ls3; q4; opacity; SH-1 (12)], 64x64 view at radius 3."""
    rng = np.random.default_rng(seed)
    n, k = 4096, 256
    pos = rng.uniform(-1.0, 1.0, size=(n, 3)).astype(np.float32)
    table = np.empty((k, 20), dtype=np.float32)
    table[:, 0:3] = rng.normal(-4.0, 0.5, size=(k, 3))
    table[:, 3:7] = _unit_quats(rng, k)
    table[:, 7] = rng.normal(0.0, 1.0, size=k)
    table[:, 8:20] = rng.normal(0.0, 0.2, size=(k, 12))
    idx = rng.integers(0, k, size=n).astype(np.int32)
    cams = ring_cameras(1, (0.0, 0.0, 0.0), 3.0, 0.0, 64, 64, 64)
    return SceneArrays(positions=pos, opacity_logits=table[idx, 7].copy(),
                       g2sh=idx.copy(), g2sr=idx.copy(),
                       sh_rows=np.ascontiguousarray(table[:, 8:20]),
                       sr_rows=np.ascontiguousarray(table[:, 0:7]),
                       sh_degree=1, cameras=cams, name="config0")


def config1(seed: int = 0, n: int = 100_000, k: int = 4096, views: int = 4,
            size: int = 256) -> SceneArrays:
    """N=100k, SR K=4096, [opacity; SH-3] K=4096, 4 views 256^2 on a radius-4 ring."""
    rng = np.random.default_rng(seed)
    pos = rng.normal(0.0, 1.0, size=(n, 3)).astype(np.float32)
    sr = _sr_table(rng, k, -4.0, 0.5)
    table2 = np.empty((k, 49), dtype=np.float32)
    table2[:, 0] = rng.normal(0.0, 1.0, size=k)
    table2[:, 1:49] = rng.normal(0.0, 0.2, size=(k, 48))
    g2sr = rng.integers(0, k, size=n).astype(np.int32)
    g2sh = rng.integers(0, k, size=n).astype(np.int32)
    cams = ring_cameras(views, (0.0, 0.0, 0.0), 4.0, 0.0, float(size), size, size)
    return SceneArrays(positions=pos, opacity_logits=table2[g2sh, 0].copy(),
                       g2sh=g2sh, g2sr=g2sr,
                       sh_rows=np.ascontiguousarray(table2[:, 1:49]), sr_rows=sr,
                       sh_degree=3, cameras=cams, name="config1")


def config2(seed: int = 0, n: int = 1_000_000, views: int = 8) -> SceneArrays:
    """N=1M clustered scene, SR K=8192, SH-3 K=16384, 1280x720 hemisphere views."""
    rng = np.random.default_rng(seed)
    n_bg = n // 10
    n_cl = n - n_bg
    centres = rng.uniform(-6.0, 6.0, size=(32, 3))
    rots = _unit_quats(rng, 32)
    sig = rng.uniform(0.2, 1.5, size=(32, 3))
    which = rng.integers(0, 32, size=n_cl)
    local = rng.normal(0.0, 1.0, size=(n_cl, 3)) * sig[which]
    w, x, y, z = rots[:, 0], rots[:, 1], rots[:, 2], rots[:, 3]
    R = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], -2)
    clustered = np.einsum("nij,nj->ni", R[which], local) + centres[which]
    bg = rng.uniform(-10.0, 10.0, size=(n_bg, 3))
    pos = np.concatenate([clustered, bg]).astype(np.float32)
    sr = _sr_table(rng, 8192, -4.0, 0.5)
    sh = rng.normal(0.0, 0.2, size=(16384, 48)).astype(np.float32)
    logits = rng.normal(0.0, 1.0, size=n).astype(np.float32)
    g2sr = rng.integers(0, 8192, size=n).astype(np.int32)
    g2sh = rng.integers(0, 16384, size=n).astype(np.int32)
    cams = hemisphere_cameras(views, 12.0, 1000.0, 1280, 720)
    return SceneArrays(positions=pos, opacity_logits=logits, g2sh=g2sh, g2sr=g2sr,
                       sh_rows=sh, sr_rows=sr, sh_degree=3, cameras=cams, name="config2")


def _outdoor_positions(rng, n):
    n_ground = (7 * n) // 10
    ground = np.empty((n_ground, 3))
    ground[:, 0:2] = rng.normal(0.0, 8.0, size=(n_ground, 2))
    ground[:, 2] = rng.normal(0.0, 0.3, size=n_ground)
    shell = rng.normal(0.0, 8.0, size=(n - n_ground, 3))
    return np.concatenate([ground, shell]).astype(np.float32)


def config3(seed: int = 0, n: int = 4_000_000, views: int = 8, k_sr: int = 16384,
            k_sh: int = 65536, width: int = 1960, height: int = 1088) -> SceneArrays:
    """N=4M outdoor-shaped scene, SR K=16384, SH-3 K=65536, 1960x1088 orbit views."""
    rng = np.random.default_rng(seed)
    pos = _outdoor_positions(rng, n)
    sr = _sr_table(rng, k_sr, -5.0, 0.7)
    sh = rng.normal(0.0, 0.2, size=(k_sh, 48)).astype(np.float32)
    logits = rng.normal(0.0, 1.0, size=n).astype(np.float32)
    g2sr = rng.integers(0, k_sr, size=n).astype(np.int32)
    g2sh = rng.integers(0, k_sh, size=n).astype(np.int32)
    cams = orbit_cameras(views, 15.0, 0.3, 1000.0, width, height, cx=width / 2.0, cy=height / 2.0)
    return SceneArrays(positions=pos, opacity_logits=logits, g2sh=g2sh, g2sr=g2sr,
                       sh_rows=sh, sr_rows=sr, sh_degree=3, cameras=cams, name="config3")


def config4(seed: int = 0, n: int = 6_000_000, views: int = 64) -> SceneArrays:
    """N=6M render-only scene, K=65536 both, 64 poses 1920x1080 on a radius-15 orbit."""
    s = config3(seed, n=n, views=views, k_sr=65536, k_sh=65536, width=1920, height=1080)
    s.name = "config4"
    return s


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def build(config: int, seed: int = 0, **kw) -> SceneArrays:
    return CONFIGS[int(config)](seed, **kw)


def refcounts(idx: np.ndarray, capacity: int) -> np.ndarray:
    return np.bincount(idx, minlength=capacity).astype(np.int64)
