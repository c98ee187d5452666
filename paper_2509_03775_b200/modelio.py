"""CGS1 model files and the metrics CSV for device-resident state
(reference `pkg/src/contrags/modelio.py:1-24`, `:58-132`, `:306-321`).

The byte layout is the reference's, little-endian:

    magic "CGS1" | u32 version=1 | u32 sh_degree | u64 N | u32 live_sh | u32 live_sr
    f32 positions[N*3] | f32 opacity[N] | i32 g2sh[N] | i32 g2sr[N]
    f32 sh_rows[live_sh*dim] | f32 sr_rows[live_sr*7]

with only live codebook rows stored, in ascending original index order, and
the assignments re-indexed against the packed rows (`modelio.py:47-53`).
`serialize_model` of a device state is byte-identical to the reference's
serialisation of the same state (tests/test_modelio.py).  The packing runs
on the device (one gather per table, one remap per index array); one D2H copy
of the packed buffers feeds the byte string.  Lineage, the iteration counter
and the RNG state are not persisted, as in the reference (`modelio.py:19-20`).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .model import ModelState, sh_dim

MAGIC = b"CGS1"
VERSION = 1
CSV_HEADER = "iteration,kind,codebook,attempts,accepts,live_sh,live_sr,recon,total,psnr"
_HDR = "<IIQII"


class ModelFormatError(ValueError):
    """modelio.py:46-47"""


def _packed(book, idx: torch.Tensor):
    """(live rows (ascending), remapped assignments) on the device."""
    live = book.device_live().long()
    remap = torch.full((book.capacity,), -1, dtype=torch.int32, device=idx.device)
    remap[live] = torch.arange(live.numel(), dtype=torch.int32, device=idx.device)
    return book.rows.index_select(0, live), remap[idx.long()]


def serialize_model(state: ModelState) -> bytes:
    """Canonical byte serialisation; freed rows are compacted out (modelio.py:58-74)."""
    g = state.gaussians
    n = g.count
    sh_rows, g2sh = _packed(state.sh, g.g2sh)
    sr_rows, g2sr = _packed(state.sr, g.g2sr)
    parts = [t.contiguous().view(torch.uint8).reshape(-1) for t in
             (g.positions.float(), g.opacity_logits.float(), g2sh, g2sr, sh_rows.float(),
              sr_rows.float())]
    body = torch.cat(parts).cpu().numpy().tobytes() if n or parts else b""
    head = MAGIC + struct.pack(_HDR, VERSION, state.sh_degree, n, sh_rows.shape[0],
                               sr_rows.shape[0])
    return head + body


def save_model(state: ModelState, path) -> None:
    with open(path, "wb") as f:
        f.write(serialize_model(state))


def _take(data: bytes, offset: int, nbytes: int, section: str):
    if offset + nbytes > len(data):
        raise ModelFormatError(
            f"truncated model file in section '{section}' at byte {offset}: "
            f"need {nbytes} bytes, have {len(data) - offset}")
    return data[offset:offset + nbytes], offset + nbytes


def deserialize_model(data: bytes, device=None, **kw) -> ModelState:
    """modelio.py:86-127: same checks and error messages; state on ``device``."""
    chunk, off = _take(data, 0, 4, "magic")
    if chunk != MAGIC:
        raise ModelFormatError(f"bad magic {chunk!r} at byte 0, expected {MAGIC!r}")
    chunk, off = _take(data, off, struct.calcsize(_HDR), "header")
    version, degree, n, live_sh, live_sr = struct.unpack(_HDR, chunk)
    if version != VERSION:
        raise ModelFormatError(f"unsupported version {version} at byte 4")
    dim = sh_dim(degree)

    def read_array(off, dtype, count, shape, section):
        nbytes = np.dtype(dtype).itemsize * count
        chunk, off2 = _take(data, off, nbytes, section)
        return np.frombuffer(chunk, dtype=dtype).reshape(shape).copy(), off2

    positions, off = read_array(off, "<f4", n * 3, (n, 3), "positions")
    logits, off = read_array(off, "<f4", n, (n,), "opacity")
    g2sh, off = read_array(off, "<i4", n, (n,), "g2sh")
    g2sr, off = read_array(off, "<i4", n, (n,), "g2sr")
    sh_rows, off = read_array(off, "<f4", live_sh * dim, (live_sh, dim), "sh_rows")
    sr_rows, off = read_array(off, "<f4", live_sr * 7, (live_sr, 7), "sr_rows")
    if off != len(data):
        raise ModelFormatError(f"{len(data) - off} trailing bytes at byte {off}")
    if n and (live_sh == 0 or live_sr == 0):
        raise ModelFormatError("nonzero N with an empty codebook")
    for name, idx, count in (("g2sh", g2sh, live_sh), ("g2sr", g2sr, live_sr)):
        if n and (idx.min() < 0 or idx.max() >= count):
            raise ModelFormatError(f"{name} index out of range")
    sh_rc = np.bincount(g2sh, minlength=live_sh).astype(np.int64)
    sr_rc = np.bincount(g2sr, minlength=live_sr).astype(np.int64)
    if np.any(sh_rc == 0) or np.any(sr_rc == 0):
        raise ModelFormatError("stored codebook contains unreferenced rows")
    return ModelState.from_arrays(positions, logits, g2sh, g2sr, sh_rows, sr_rows,
                                  sh_refcount=sh_rc, sr_refcount=sr_rc, device=device, **kw)


def load_model(path, device=None, **kw) -> ModelState:
    with open(path, "rb") as f:
        return deserialize_model(f.read(), device=device, **kw)


def _csv_float(v) -> str:
    v = float(v)
    return repr(v) if np.isfinite(v) else "nan"


def write_metrics_csv(records, path) -> None:
    """Fixed-schema CSV, one row per TransitionRecord (modelio.py:306-321)."""
    with open(path, "w") as f:
        f.write(CSV_HEADER + "\n")
        for r in records:
            f.write(",".join([
                str(r.iteration), r.kind, r.codebook,
                str(r.attempts), str(r.accepts),
                str(r.live_sh), str(r.live_sr),
                _csv_float(r.recon), _csv_float(r.total), _csv_float(r.psnr),
            ]) + "\n")


# ---------------------------------------------------------------------------
# 8-bit images (reference modelio.py:137-153)

def image_to_u8(image: torch.Tensor) -> torch.Tensor:
    """Device HxWx3 (or flat) float image -> uint8 on the same device: the
    bytes the reference's save_png writes, clip(rint(x * 255), 0, 255) in
    float64 (the cgs_quantize8 kernel)."""
    from . import _native as nat
    if not (isinstance(image, torch.Tensor) and image.is_cuda):
        raise TypeError("image_to_u8 takes a CUDA tensor (numpy images: quantize8)")
    x = image.detach().to(torch.float32).contiguous()
    out = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    nat.call("cgs_quantize8", nat.ptr(x), x.numel(), nat.ptr(out), nat.stream_handle(x.device))
    return out


_GRID8 = {}


def _grid8(device) -> torch.Tensor:
    """k / 255 for k = 0..255 as numpy divides (a scalar division on the device
    may multiply by the reciprocal instead)."""
    g = _GRID8.get(device)
    if g is None:
        g = _GRID8[device] = torch.as_tensor(np.arange(256, dtype=np.float64) / 255.0).to(device)
    return g


def quantize8(image):
    """Round a float image onto the 8-bit grid (modelio.py:151-153).  A CUDA
    tensor is quantized on the device (float64 result on the device); an array
    is rounded on the host exactly as the reference does."""
    if isinstance(image, torch.Tensor) and image.is_cuda:
        return _grid8(image.device)[image_to_u8(image).long()]
    return np.clip(np.rint(np.asarray(image, dtype=np.float64) * 255.0), 0, 255) / 255.0

