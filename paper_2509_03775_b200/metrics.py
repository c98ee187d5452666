"""Reconstruction loss, codebook penalty and image metrics (reference `metrics.py`).

``recon_loss`` / ``recon_loss_grad`` run the fused L1 + SSIM kernels
(``cgs_recon_loss``); the scalar helpers (``total_loss``, ``LossTerms``) are
host arithmetic exactly as in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
PSNR_CAP_DB = 100.0


def _dev_img(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        dev = device or (x.device if x.is_cuda else torch.device("cuda"))
        return x.detach().to(device=dev, dtype=torch.float32).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).to(device or "cuda")


def _pair(a, b):
    A = _dev_img(a)
    B = _dev_img(b, A.device)
    if tuple(A.shape) != tuple(B.shape):
        raise ValueError(f"image shapes differ: {tuple(A.shape)} vs {tuple(B.shape)}")
    if A.dim() == 2:
        raise ValueError("HxW images: pass HxWx3 (single-channel loss is not on the hot path)")
    if A.dim() != 3 or A.shape[2] != 3:
        raise ValueError("images must be HxWx3")
    return A, B


class LossWorkspace:
    """Reusable workspace + outputs for the batched loss kernels."""

    def __init__(self, n_views: int, height: int, width: int, device):
        nb = nat.library().cgs_loss_workspace_bytes(n_views, height, width)
        self.ws = torch.empty((nb,), dtype=torch.uint8, device=device)
        self.losses = torch.empty((3 * n_views,), dtype=torch.float64, device=device)
        self.shape = (n_views, height, width)

    def run(self, img: torch.Tensor, gt: torch.Tensor, lam: float, dL=None, grad_scale=1.0,
            want_ssim=False):
        v, h, w = self.shape
        nat.call("cgs_recon_loss", nat.ptr(img), nat.ptr(gt), v, h, w, float(lam),
                 1 if want_ssim else 0, float(grad_scale), nat.ptr(dL), nat.ptr(self.losses),
                 nat.ptr(self.ws), self.ws.numel(), nat.stream_handle(img.device))
        return self.losses


def _loss(a, b, lam, want_grad, want_ssim):
    A, B = _pair(a, b)
    h, w, _ = A.shape
    ws = LossWorkspace(1, h, w, A.device)
    dL = torch.empty_like(A) if want_grad else None
    vals = ws.run(A, B, lam, dL, 1.0, want_ssim)
    return vals, dL


def recon_loss(rendered, ground_truth, lambda_ssim: float):
    """(l1, ssim, recon) with recon = (1-lam) L1 + lam (1-SSIM) (metrics.py:122-130)."""
    h, w = (rendered.shape[0], rendered.shape[1])
    want = min(h, w) >= SSIM_WINDOW
    vals, _ = _loss(rendered, ground_truth, lambda_ssim, False, want)
    l1v, sv, rec = (float(x) for x in vals.cpu().numpy())
    return l1v, sv, rec


def recon_loss_grad(rendered, ground_truth, lambda_ssim: float) -> torch.Tensor:
    """d recon / d rendered (metrics.py:133-140), float32 on device."""
    _, dL = _loss(rendered, ground_truth, lambda_ssim, True, False)
    return dL


def l1(a, b) -> float:
    vals, _ = _loss(a, b, 0.0, False, False)
    return float(vals[0].item())


def ssim(a, b) -> float:
    A, _ = _pair(a, b)
    if A.shape[0] < SSIM_WINDOW or A.shape[1] < SSIM_WINDOW:
        raise ValueError(f"images must be at least {SSIM_WINDOW}x{SSIM_WINDOW} for SSIM")
    vals, _ = _loss(a, b, 0.0, False, True)
    return float(vals[1].item())


@dataclass
class LossTerms:
    l1: float
    ssim: float
    recon: float
    codebook_penalty: float
    total: float
    log_posterior_unnorm: float


def total_loss(recon: float, live_sh: int, live_sr: int, lambda_sh: float, lambda_sr: float,
               l1: float = float("nan"), ssim: float = float("nan")) -> LossTerms:
    """metrics.py:153-162"""
    if live_sh < 0 or live_sr < 0:
        raise ValueError("codebook sizes must be non-negative")
    penalty = lambda_sr * live_sr + lambda_sh * live_sh
    total = recon + penalty
    return LossTerms(l1=l1, ssim=ssim, recon=recon, codebook_penalty=penalty, total=total,
                     log_posterior_unnorm=-total)


def psnr(rendered, ground_truth, cap: float = PSNR_CAP_DB) -> float:
    """metrics.py:165-172 (device mean of squared error, fp64 accumulate)."""
    A, B = _pair(rendered, ground_truth)
    mse = float(((A.double() - B.double()) ** 2).mean().item())
    if mse == 0.0:
        return cap
    return -10.0 * math.log10(mse)


def evaluate(state, views) -> dict:
    """``contrags eval`` (cli.py:223-237) on the device: for each (camera,
    ground truth) view, PSNR and SSIM of the 8-bit-quantized render
    (quantize8) against the ground truth; returns the per-view lists and their
    means."""
    from .modelio import quantize8
    from .render import Frame
    psnrs, ssims = [], []
    for cam, gt in views:
        fr = Frame(state, [cam]).run_checked()
        rendered = quantize8(fr.view_image(0))
        psnrs.append(psnr(rendered, gt))
        ssims.append(ssim(rendered, gt))
    return {"psnr": psnrs, "ssim": ssims, "mean_psnr": float(np.mean(psnrs)),
            "mean_ssim": float(np.mean(ssims))}

