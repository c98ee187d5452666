"""Precision sensitivity of the config-2/3 strip gradients (CPU, oracle only).

Which fp32 stage can explain the GPU's error on view-covering / near-plane
splats?  Runs the fp64 oracle backward on a full-scene strip, then re-runs
(a) the pull-back with the screen-space sums rounded to fp32, and (b) the
tile backward with the per-pixel alpha / T_before / suffix perturbed by a
relative error eps, and reports the resulting group-relative gradient error
on the near set and on the rest."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import _strip_cam  # noqa: E402
from oracle import cgs_oracle as O  # noqa: E402
from paper_2509_03775_b200 import scenes  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rows = (528, 560) if config == 3 else (344, 376)
a = scenes.build(config, 0)
ocam = _strip_cam(O.cam_from_any(a.cameras[0]), *rows)
ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
t0 = time.time()
fw = O.raster_forward(ost, ocam)
dL = np.random.default_rng(0).normal(0, 1e-4, fw["image"].shape)
ref, scr = O.raster_backward(ost, ocam, dL, screen=True)
print("oracle fwd+bwd", time.time() - t0, "s")
proj = scr["proj"]
tz = (a.positions.astype(np.float64) @ ocam.R.T + ocam.t)[:, 2]
offs = fw["tile_offsets"]
ntile = len(offs) - 1
# tiles per visible splat
x0, x1, y0, y1 = O.pixel_rects(proj["mean2d"], proj["radius"], ocam.width, ocam.height)
ok = (x0 <= x1) & (y0 <= y1)
nt = np.where(ok, (x1 // 16 - x0 // 16 + 1) * (y1 // 16 - y0 // 16 + 1), 0)
ntiles = np.zeros(len(a.positions), np.int64)
ntiles[proj["idx"]] = nt
near = ((tz > 0.01) & (tz < 0.02)) | (ntiles == ntile)
print("near set", near.sum(), "covering", (ntiles == ntile).sum(), "tz<0.02", ((tz > 0.01) & (tz < 0.02)).sum())


def masks():
    far = {"positions": ~near, "opacity_logits": ~near}
    for k, idx in (("sh_rows", a.g2sh), ("sr_rows", a.g2sr)):
        t = np.zeros(ref[k].shape[0], bool)
        t[np.unique(idx[near])] = True
        far[k] = ~t
    return far


far = masks()


def report(tag, g):
    out = [tag]
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        m = far[k]
        scale = max(np.abs(ref[k]).max(), 1e-30)
        e_far = np.abs(g[k][m] - ref[k][m]).max() / scale
        e_near = np.abs(g[k][~m] - ref[k][~m]).max() / scale if (~m).any() else 0.0
        bad = ~np.isclose(g[k], ref[k], rtol=1e-4, atol=1e-6)
        out.append(f"{k}: far {e_far:.1e} near {e_near:.1e} n_bad {bad.sum()}")
    print(" | ".join(out))


f32 = lambda x: x.astype(np.float32).astype(np.float64)
g = O.pull_back(ost, ocam, proj, f32(scr["g_col"]), f32(scr["g_op"]), f32(scr["g_mean"]), f32(scr["g_con"]))
report("screen sums fp32", g)
rng = np.random.default_rng(5)
for eps in ():
    for which in ("alpha", "t_before", "suffix"):
        def pert(name, x, which=which, eps=eps):
            return x * (1.0 + eps * rng.standard_normal(x.shape)) if name == which else x
        g = O.raster_backward(ost, ocam, dL, perturb=pert)
        report(f"{which} eps={eps:g}", g)
for which, eps in (("local_moments", 1e-7), ("local_moments", 1e-6), ("dS3", 6e-8), ("dview", 6e-8)):
    def pert(name, x, which=which, eps=eps):
        if name != which:
            return x
        return True if x is None else x * (1.0 + eps * rng.standard_normal(x.shape))
    report(f"{which} eps={eps:g}", O.raster_backward(ost, ocam, dL, perturb=pert))
