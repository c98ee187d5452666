"""Differentiable tile rasterizer on the B200 (reference `pkg/src/contrags/render.py`).

``rasterize_forward`` / ``rasterize_backward`` keep the reference's names,
arguments, return types and error behaviour; underneath, one call renders a
*frame* of up to 16 views at once through the C ABI (``cgs_render_forward``,
``cgs_render_backward``), so batched training steps launch each kernel once
per step instead of once per view.  Images, transmittance and gradients are
float32 CUDA tensors; discrete outputs (tile lists, depth order, contribution
counts) follow the reference's float64 decisions.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .camera import Camera
from .model import ModelState

# reference render.py:26-34
NEAR_PLANE = 0.01
BLUR_PX2 = 0.3
ALPHA_CLAMP = 0.99
ALPHA_SKIP = 1.0 / 255.0
TMIN = 1e-4
TILE = 16
FOOTPRINT_SIGMAS = float(np.sqrt(2.0 * np.log(255.0)))


def scene_struct(state: ModelState) -> nat.CScene:
    g = state.gaussians
    s = nat.CScene()
    s.n = g.count
    s.positions = nat.ptr(g.positions)
    s.opacity_logits = nat.ptr(g.opacity_logits)
    s.g2sh = nat.ptr(g.g2sh)
    s.g2sr = nat.ptr(g.g2sr)
    s.sh_rows = nat.ptr(state.sh.rows)
    s.sh_capacity = state.sh.capacity
    s.sh_degree = state.sh_degree
    s.sr_rows = nat.ptr(state.sr.rows)
    s.sr_capacity = state.sr.capacity
    return s


_pair_hint: dict = {}


def _initial_pair_capacity(n: int, cams) -> int:
    key = (n, tuple((c.width, c.height) for c in cams))
    if key in _pair_hint:
        return _pair_hint[key]
    return max(1 << 16, 8 * n * len(cams))


class Frame:
    """One batched forward render of ``cams`` (<= 16 views) and its workspace."""

    def __init__(self, state: ModelState, cams, pair_capacity: Optional[int] = None,
                 ws: Optional[torch.Tensor] = None):
        if not 1 <= len(cams) <= nat.MAX_VIEWS:
            raise ValueError(f"a frame holds 1..{nat.MAX_VIEWS} views")
        self.state = state
        self.cams = list(cams)
        self.device = state.device
        self.n = state.num_gaussians
        self.sr_cap = state.sr.capacity
        self.c_cams = nat.cams_array(self.cams)
        self.pair_cap = int(pair_capacity or _initial_pair_capacity(self.n, self.cams))
        self.pixels = sum(c.width * c.height for c in self.cams)
        self.image = torch.empty((self.pixels * 3,), dtype=torch.float32, device=self.device)
        self.final_T = torch.empty((self.pixels,), dtype=torch.float32, device=self.device)
        self.counts = torch.empty((self.pixels,), dtype=torch.int32, device=self.device)
        self._alloc_ws(ws)
        self.token = None
        self._stats = None

    def _alloc_ws(self, ws: Optional[torch.Tensor] = None):
        """Frame workspace; a caller buffer that is large enough is used in place
        (the trainer sizes one for the Gaussian capacity, so densify does not
        reallocate)."""
        nb = nat.library().cgs_frame_workspace_bytes(self.n, self.c_cams, len(self.cams),
                                                     self.pair_cap, self.sr_cap)
        if nb == 0:
            raise ValueError(nat.last_error())
        if ws is not None and ws.numel() >= nb:
            self.ws = ws[:nb]
        else:
            self.ws = torch.empty((nb,), dtype=torch.uint8, device=self.device)

    def run(self):
        self.scene = scene_struct(self.state)
        nat.call("cgs_render_forward", ctypes.byref(self.scene), self.c_cams, len(self.cams),
                 nat.ptr(self.ws), self.ws.numel(), self.pair_cap, nat.ptr(self.image),
                 nat.ptr(self.final_T), nat.ptr(self.counts), nat.stream_handle(self.device))
        self.token = self.state.token()
        self._stats = None
        return self

    FORWARD_STAGES = ("cgs_project", "cgs_sort_depth", "cgs_duplicate_tiles", "cgs_sort_pairs")

    def run_staged(self):
        """``run`` through the staged ABI, one entry point per stage (same results)."""
        self.scene = scene_struct(self.state)
        args = (ctypes.byref(self.scene), self.c_cams, len(self.cams), nat.ptr(self.ws),
                self.ws.numel(), self.pair_cap)
        h = nat.stream_handle(self.device)
        for fn in self.FORWARD_STAGES:
            nat.call(fn, *args, h)
        nat.call("cgs_raster_fwd", *args, nat.ptr(self.image), nat.ptr(self.final_T),
                 nat.ptr(self.counts), h)
        self.token = self.state.token()
        self._stats = None
        return self

    def stats(self) -> nat.CFrameStats:
        if self._stats is None:
            st = nat.CFrameStats()
            nat.call("cgs_frame_stats", nat.ptr(self.ws), ctypes.byref(st),
                     nat.stream_handle(self.device))
            self._stats = st
        return self._stats

    def run_checked(self):
        """Forward, then grow the pair capacity and re-run if it overflowed (synchronizes)."""
        self.run()
        st = self.stats()
        if st.overflow:
            self.pair_cap = int(math.ceil(st.n_pairs * 1.25)) + 1024
            self._alloc_ws()
            self.run()
            st = self.stats()
        key = (self.n, tuple((c.width, c.height) for c in self.cams))
        _pair_hint[key] = max(_pair_hint.get(key, 0), int(st.n_pairs * 1.25) + 1024)
        if st.zero_quaternion:
            raise ValueError("zero quaternion")
        return self

    # -- per-view views of the outputs --------------------------------------
    def _pix_slices(self):
        out, base = [], 0
        for c in self.cams:
            out.append((base, c.height, c.width))
            base += c.width * c.height
        return out

    def view_image(self, v: int) -> torch.Tensor:
        b, h, w = self._pix_slices()[v]
        return self.image[3 * b: 3 * (b + h * w)].view(h, w, 3)

    def view_T(self, v: int) -> torch.Tensor:
        b, h, w = self._pix_slices()[v]
        return self.final_T[b: b + h * w].view(h, w)

    def view_counts(self, v: int) -> torch.Tensor:
        b, h, w = self._pix_slices()[v]
        return self.counts[b: b + h * w].view(h, w)

    def tile_lists(self):
        """(offsets over all views' tiles, Gaussian ids) as host arrays."""
        tiles = sum(c.num_tiles for c in self.cams)
        offs = torch.empty((tiles + 1,), dtype=torch.int64, device=self.device)
        ids = torch.empty((max(self.pair_cap, 1),), dtype=torch.int32, device=self.device)
        nat.call("cgs_frame_tile_lists", self.c_cams, len(self.cams), self.n, self.pair_cap,
                 self.sr_cap, nat.ptr(self.ws), self.ws.numel(), nat.ptr(offs), nat.ptr(ids),
                 nat.stream_handle(self.device))
        o = offs.cpu().numpy()
        return o, ids[: int(o[-1])].cpu().numpy().astype(np.int64)

    def splats(self, v: int = 0) -> dict:
        """Projection records of view v (stage parity with render.py:145-203)."""
        n = max(self.n, 1)
        dev = self.device
        mean = torch.empty((n, 2), dtype=torch.float64, device=dev)
        conic = torch.empty((n, 3), dtype=torch.float64, device=dev)
        opac = torch.empty((n,), dtype=torch.float64, device=dev)
        col = torch.empty((n, 3), dtype=torch.float32, device=dev)
        nt = torch.empty((n,), dtype=torch.int32, device=dev)
        nat.call("cgs_frame_splats", self.c_cams, len(self.cams), self.n, self.pair_cap,
                 self.sr_cap, nat.ptr(self.ws), self.ws.numel(), v, nat.ptr(mean), nat.ptr(conic),
                 nat.ptr(opac), nat.ptr(col), nat.ptr(nt), nat.stream_handle(dev))
        return dict(mean2d=mean.cpu().numpy()[: self.n], conic=conic.cpu().numpy()[: self.n],
                    opac=opac.cpu().numpy()[: self.n], colors=col.cpu().numpy()[: self.n],
                    n_tiles=nt.cpu().numpy()[: self.n].astype(np.int64))

    # -- backward -------------------------------------------------------------
    def backward(self, dL: torch.Tensor, scale: float = 1.0, grads: "GradientSet" = None,
                 ws: torch.Tensor = None, after_gaussians=None) -> "GradientSet":
        """Gradients of sum_v <dL_v, image_v> (scaled) for every parameter group.

        ``after_gaussians``, when given, is called once the per-Gaussian
        gradients (positions, logits) are enqueued and before the codebook
        reduce (the staged ABI), so a caller can start reducing them across
        ranks on another stream while the codebook kernels run."""
        st = self.state
        dev = self.device
        if grads is None:
            grads = GradientSet.empty(st)
        nb = backward_workspace_bytes(st, self)
        if ws is None or ws.numel() < nb:
            ws = torch.empty((nb,), dtype=torch.uint8, device=dev)
        self.scene = scene_struct(st)
        sh_off, sh_mem = st.code_csr("sh")
        sr_off, sr_mem = st.code_csr("sr")
        if after_gaussians is not None:
            args = (ctypes.byref(self.scene), self.c_cams, len(self.cams), nat.ptr(self.ws),
                    self.ws.numel(), self.pair_cap)
            h = nat.stream_handle(dev)
            nat.call("cgs_raster_bwd", *args, nat.ptr(self.final_T), nat.ptr(dL), nat.ptr(ws),
                     ws.numel(), h)
            nat.call("cgs_gaussian_reduce_pullback", *args, float(scale), nat.ptr(ws), ws.numel(),
                     nat.ptr(grads.positions), nat.ptr(grads.opacity_logits), h)
            after_gaussians(grads)
            nat.call("cgs_codebook_reduce", *args, float(scale), nat.ptr(sh_off), nat.ptr(sh_mem),
                     nat.ptr(sr_off), nat.ptr(sr_mem), nat.ptr(ws), ws.numel(),
                     nat.ptr(grads.sh_rows), nat.ptr(grads.sr_rows), h)
            return grads
        nat.call("cgs_render_backward", ctypes.byref(self.scene), self.c_cams, len(self.cams),
                 nat.ptr(self.ws), self.ws.numel(), self.pair_cap, nat.ptr(self.final_T),
                 nat.ptr(dL), float(scale), nat.ptr(sh_off), nat.ptr(sh_mem), nat.ptr(sr_off),
                 nat.ptr(sr_mem), nat.ptr(ws), ws.numel(), nat.ptr(grads.positions),
                 nat.ptr(grads.opacity_logits), nat.ptr(grads.sh_rows), nat.ptr(grads.sr_rows),
                 nat.stream_handle(dev))
        return grads


    def backward_staged(self, dL: torch.Tensor, scale: float = 1.0) -> "GradientSet":
        """``backward`` through the staged ABI (raster, per-Gaussian reduce +
        pull-back, codebook reduce; same results)."""
        st = self.state
        dev = self.device
        grads = GradientSet.empty(st)
        nb = backward_workspace_bytes(st, self)
        ws = torch.empty((nb,), dtype=torch.uint8, device=dev)
        self.scene = scene_struct(st)
        sh_off, sh_mem = st.code_csr("sh")
        sr_off, sr_mem = st.code_csr("sr")
        args = (ctypes.byref(self.scene), self.c_cams, len(self.cams), nat.ptr(self.ws),
                self.ws.numel(), self.pair_cap)
        h = nat.stream_handle(dev)
        nat.call("cgs_raster_bwd", *args, nat.ptr(self.final_T), nat.ptr(dL), nat.ptr(ws),
                 ws.numel(), h)
        nat.call("cgs_gaussian_reduce_pullback", *args, float(scale), nat.ptr(ws), ws.numel(),
                 nat.ptr(grads.positions), nat.ptr(grads.opacity_logits), h)
        nat.call("cgs_codebook_reduce", *args, float(scale), nat.ptr(sh_off), nat.ptr(sh_mem),
                 nat.ptr(sr_off), nat.ptr(sr_mem), nat.ptr(ws), ws.numel(),
                 nat.ptr(grads.sh_rows), nat.ptr(grads.sr_rows), h)
        return grads


def backward_workspace_bytes(state: ModelState, frame: "Frame") -> int:
    return nat.library().cgs_backward_workspace_bytes(frame.n, frame.c_cams, len(frame.cams),
                                                      frame.pair_cap, state.sh.capacity,
                                                      state.sr.capacity)


@dataclass
class GradientSet:
    """Gradients per parameter group (reference render.py:215-224), float32 on device."""

    positions: torch.Tensor       # (N, 3)
    opacity_logits: torch.Tensor  # (N,)
    sh_rows: torch.Tensor         # (sh capacity, sh dim)
    sr_rows: torch.Tensor         # (sr capacity, 7)
    flat: Optional[torch.Tensor] = field(default=None, repr=False)

    @classmethod
    def empty(cls, state: ModelState, buf: Optional[torch.Tensor] = None) -> "GradientSet":
        """One flat buffer [pos | logit | sh | sr] (a single allreduce over NVLink),
        carved from ``buf`` when it is large enough."""
        n, ksh, d, ksr = state.num_gaussians, state.sh.capacity, state.sh.dim, state.sr.capacity
        sizes = [3 * n, n, ksh * d, 7 * ksr]
        if buf is not None and buf.numel() >= sum(sizes):
            flat = buf[: sum(sizes)]
        else:
            flat = torch.empty((sum(sizes),), dtype=torch.float32, device=state.device)
        parts = torch.split(flat, sizes)
        return cls(positions=parts[0].view(n, 3), opacity_logits=parts[1],
                   sh_rows=parts[2].view(ksh, d), sr_rows=parts[3].view(ksr, 7), flat=flat)

    def all_finite(self) -> bool:
        ts = [self.flat] if self.flat is not None else [self.positions, self.opacity_logits,
                                                         self.sh_rows, self.sr_rows]
        return all(bool(torch.isfinite(t).all()) for t in ts)

    def numpy(self) -> dict:
        return dict(positions=self.positions.cpu().numpy(),
                    opacity_logits=self.opacity_logits.cpu().numpy(),
                    sh_rows=self.sh_rows.cpu().numpy(), sr_rows=self.sr_rows.cpu().numpy())


class _TileDict(dict):
    """RenderArtifacts.tile_splats materialized lazily from the device CSR."""


@dataclass
class RenderArtifacts:
    image: torch.Tensor                 # (H, W, 3) float32
    final_transmittance: torch.Tensor   # (H, W)
    contrib_counts: torch.Tensor        # (H, W) int32
    state_token: tuple
    frame: Frame = field(repr=False, default=None)
    view: int = 0
    _tiles: Optional[dict] = field(default=None, repr=False)

    @property
    def tile_splats(self) -> dict:
        """(ty, tx) -> Gaussian indices in depth order; every tile key present."""
        if self._tiles is None:
            offs, ids = self.frame.tile_lists()
            cam = self.frame.cams[self.view]
            base = sum(c.num_tiles for c in self.frame.cams[: self.view])
            ntx = (cam.width + TILE - 1) // TILE
            nty = (cam.height + TILE - 1) // TILE
            d = _TileDict()
            for ty in range(nty):
                for tx in range(ntx):
                    t = base + ty * ntx + tx
                    d[(ty, tx)] = ids[offs[t]:offs[t + 1]]
            self._tiles = d
        return self._tiles


def state_camera_token(state: ModelState, cam: Camera) -> tuple:
    return (state.token(), cam.key())


def render_frame(state: ModelState, cams) -> Frame:
    """Batched forward of up to 16 views (synchronizes once to size the pair buffers)."""
    return Frame(state, cams).run_checked()


def render_u8(state: ModelState, cams) -> list:
    """The rendered views as 8-bit HxWx3 host arrays -- the PNG bytes the
    reference's ``contrags render`` writes per view (cli.py:209-220:
    rasterize_forward + save_png).  Views go through batched frames of up to
    16; each frame's images are quantized on the device (cgs_quantize8) and
    copied to the host as bytes."""
    from .modelio import image_to_u8
    cams = list(cams)
    out = []
    for i in range(0, len(cams), nat.MAX_VIEWS):
        fr = Frame(state, cams[i:i + nat.MAX_VIEWS]).run_checked()
        u8 = image_to_u8(fr.image).cpu().numpy()
        for b, h, w in fr._pix_slices():
            out.append(u8[3 * b: 3 * (b + h * w)].reshape(h, w, 3))
    return out


def rasterize_forward(state: ModelState, cam: Camera) -> RenderArtifacts:
    """Front-to-back compositing over 16x16 tiles, black background (render.py:287-315)."""
    fr = render_frame(state, [cam])
    return RenderArtifacts(image=fr.view_image(0), final_transmittance=fr.view_T(0),
                           contrib_counts=fr.view_counts(0),
                           state_token=state_camera_token(state, cam), frame=fr, view=0)


def _as_device_image(x, shape, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.detach().to(device=device, dtype=torch.float32)
    else:
        t = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).to(device)
    if tuple(t.shape) != tuple(shape):
        raise ValueError("dL_dimage shape mismatch")
    return t.contiguous()


def rasterize_backward(state: ModelState, cam: Camera, artifacts: RenderArtifacts,
                       dL_dimage) -> GradientSet:
    """Adjoint of rasterize_forward (render.py:318-379 + _pull_back :382-459)."""
    if artifacts.state_token != state_camera_token(state, cam):
        raise ValueError("stale artifacts: state or camera changed since the forward pass")
    dL = _as_device_image(dL_dimage, (cam.height, cam.width, 3), state.device)
    return artifacts.frame.backward(dL.reshape(-1))


@dataclass
class ProjectedSplat:
    mean2d: np.ndarray
    conic: np.ndarray
    depth: float
    tile_span: tuple
    color: Optional[np.ndarray] = None
    opacity: Optional[float] = None


def build_covariances(sr_rows) -> np.ndarray:
    """R(q) S S^T R(q)^T for SR rows (render.py:85-91); host helper."""
    rows = np.asarray(sr_rows, dtype=np.float64)
    q = rows[..., 3:7]
    nq = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(nq == 0.0):
        raise ValueError("zero quaternion")
    w, x, y, z = np.moveaxis(q / nq, -1, 0)
    R = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], -2)
    s2 = np.exp(2.0 * rows[..., 0:3])
    return (R * s2[..., None, :]) @ np.swapaxes(R, -1, -2)


def build_covariance(sr_row) -> np.ndarray:
    return build_covariances(np.asarray(sr_row, dtype=np.float64).reshape(7))


def project_gaussian(mu, cov3d, cam: Camera, near: float = NEAR_PLANE) -> Optional[ProjectedSplat]:
    """Single-Gaussian projection (render.py:118-136); host helper for tests/tools."""
    mu = np.asarray(mu, dtype=np.float64).reshape(3)
    t = cam.world_to_camera(mu)
    if t[2] <= near:
        return None
    tx, ty, tz = t
    mean2d = np.array([cam.fx * tx / tz + cam.cx, cam.fy * ty / tz + cam.cy])
    J = np.array([[cam.fx / tz, 0.0, -cam.fx * tx / tz ** 2], [0.0, cam.fy / tz, -cam.fy * ty / tz ** 2]])
    M = J @ cam.rotation
    cov2d = M @ np.asarray(cov3d, dtype=np.float64) @ M.T + BLUR_PX2 * np.eye(2)
    conic = np.linalg.inv(cov2d)
    lam = 0.5 * (cov2d[0, 0] + cov2d[1, 1]) + np.sqrt(0.25 * (cov2d[0, 0] - cov2d[1, 1]) ** 2
                                                       + cov2d[0, 1] ** 2)
    r = FOOTPRINT_SIGMAS * np.sqrt(lam) + 1e-9
    x0 = max(0, int(np.ceil(mean2d[0] - r - 0.5)))
    x1 = min(cam.width - 1, int(np.floor(mean2d[0] + r - 0.5)))
    y0 = max(0, int(np.ceil(mean2d[1] - r - 0.5)))
    y1 = min(cam.height - 1, int(np.floor(mean2d[1] + r - 0.5)))
    return ProjectedSplat(mean2d=mean2d, conic=conic, depth=float(tz), tile_span=(x0, x1, y0, y1))
