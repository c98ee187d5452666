"""Pinhole camera (host-side input type of the render path).

Mirrors the reference camera contract (`pkg/src/contrags/camera.py:10-73`):
``rotation`` is the row-major world->camera rotation, ``translation`` the
world->camera translation, +x right, +y down, +z forward.  A camera is 16
doubles plus two ints; it crosses the C ABI as ``cgs_camera_t``
(include/cgs_b200.h) by value, never as a device buffer.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np


class CCamera(ctypes.Structure):
    """ctypes mirror of ``cgs_camera_t`` (include/cgs_b200.h)."""

    _fields_ = [
        ("R", ctypes.c_double * 9),
        ("t", ctypes.c_double * 3),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class Camera:
    """World->camera pose plus intrinsics (reference `camera.py:10-36`)."""

    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        rot = np.array(self.rotation, dtype=np.float64).reshape(3, 3)
        trans = np.array(self.translation, dtype=np.float64).reshape(3)
        object.__setattr__(self, "rotation", rot)
        object.__setattr__(self, "translation", trans)
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        if int(self.width) < 1 or int(self.height) < 1:
            raise ValueError("image dimensions must be >= 1")
        object.__setattr__(self, "width", int(self.width))
        object.__setattr__(self, "height", int(self.height))

    # -- host helpers (reference camera.py:29-36) -------------------------
    def world_to_camera(self, points: np.ndarray) -> np.ndarray:
        pts = np.asarray(points, dtype=np.float64)
        return pts @ self.rotation.T + self.translation

    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    # -- ABI ----------------------------------------------------------------
    def to_c(self) -> CCamera:
        c = CCamera()
        c.R[:] = [float(v) for v in self.rotation.reshape(-1)]
        c.t[:] = [float(v) for v in self.translation]
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        return c

    def key(self) -> bytes:
        """Byte identity of the camera (used by the staleness token)."""
        return (self.rotation.tobytes() + self.translation.tobytes()
                + np.float64([self.fx, self.fy, self.cx, self.cy]).tobytes()
                + np.int64([self.width, self.height]).tobytes())

    @property
    def num_tiles(self) -> int:
        return ((self.width + 15) // 16) * ((self.height + 15) // 16)


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """(rotation, translation) looking from ``eye`` at ``target``.

    Same axis convention as reference `camera.py:39-58` (+x right, +y down,
    +z forward); a forward vector parallel to ``up`` falls back to x-up.
    """
    eye = np.asarray(eye, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    forward = target - eye
    forward = forward / np.linalg.norm(forward)
    up_vec = np.asarray(up, dtype=np.float64)
    right = np.cross(forward, up_vec)
    rn = np.linalg.norm(right)
    if rn < 1e-9:
        up_vec = np.array([1.0, 0.0, 0.0])
        right = np.cross(forward, up_vec)
        rn = np.linalg.norm(right)
    right = right / rn
    down = np.cross(forward, right)
    rot = np.stack([right, down, forward], axis=0)
    return rot, -rot @ eye


def ring_cameras(num_views: int, center, radius: float, height: float,
                 fx: float, width: int, height_px: int) -> list:
    """Cameras evenly spaced on a horizontal ring (reference `camera.py:61-73`)."""
    center = np.asarray(center, dtype=np.float64)
    out = []
    for k in range(num_views):
        ang = 2.0 * np.pi * k / num_views
        eye = center + np.array([radius * np.cos(ang), radius * np.sin(ang), height])
        rot, trans = look_at(eye, center)
        out.append(Camera(rotation=rot, translation=trans, fx=fx, fy=fx,
                          cx=width / 2.0, cy=height_px / 2.0,
                          width=width, height=height_px))
    return out


def orbit_cameras(num_views: int, radius: float, elevation: float, fx: float,
                  width: int, height: int, cx=None, cy=None) -> list:
    """Cameras on an inclined orbit looking at the origin (configs 3-4)."""
    out = []
    for k in range(num_views):
        az = 2.0 * np.pi * k / num_views
        eye = np.array([radius * np.cos(elevation) * np.cos(az),
                        radius * np.cos(elevation) * np.sin(az),
                        radius * np.sin(elevation)])
        rot, trans = look_at(eye, (0.0, 0.0, 0.0))
        out.append(Camera(rotation=rot, translation=trans, fx=fx, fy=fx,
                          cx=width / 2.0 if cx is None else cx,
                          cy=height / 2.0 if cy is None else cy,
                          width=width, height=height))
    return out


def hemisphere_cameras(num_views: int, radius: float, fx: float, width: int,
                       height: int) -> list:
    """Fibonacci directions on the upper hemisphere looking at the origin (config 2)."""
    out = []
    golden = np.pi * (3.0 - np.sqrt(5.0))
    for k in range(num_views):
        z = 1.0 - (k + 0.5) / num_views          # (0, 1): upper hemisphere
        r = np.sqrt(max(0.0, 1.0 - z * z))
        phi = golden * k
        eye = radius * np.array([r * np.cos(phi), r * np.sin(phi), z])
        rot, trans = look_at(eye, (0.0, 0.0, 0.0))
        out.append(Camera(rotation=rot, translation=trans, fx=fx, fy=fx,
                          cx=width / 2.0, cy=height / 2.0, width=width, height=height))
    return out
