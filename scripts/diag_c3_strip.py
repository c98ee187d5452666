"""Diagnostic: config-3 strip, GPU vs oracle per-pixel comparison."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_03775_b200 as cg
from bench import _strip_cam
from oracle import cgs_oracle as O
from paper_2509_03775_b200 import scenes
CFG = int(os.environ.get("CFG", "3")); ROWS = tuple(int(x) for x in os.environ.get("ROWS", "528,560").split(","))
a = scenes.build(CFG, 0)
ocam = _strip_cam(O.cam_from_any(a.cameras[0]), *ROWS)
cam = cg.Camera(rotation=ocam.R, translation=ocam.t, fx=ocam.fx, fy=ocam.fy, cx=ocam.cx,
                cy=ocam.cy, width=ocam.width, height=ocam.height)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
art = cg.rasterize_forward(st, cam)
ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
fw = O.raster_forward(ost, ocam)
cnt = art.contrib_counts.cpu().numpy(); rc = fw["counts"]
d = cnt.astype(int) - rc
print("count diff hist", np.unique(d, return_counts=True))
img = art.image.cpu().numpy()
print("img max abs diff", np.abs(img - fw["image"]).max(), "at matching counts", np.abs(img - fw["image"])[d == 0].max())
T = art.final_transmittance.cpu().numpy()
ys, xs = np.nonzero(d != 0)
for y, x in list(zip(ys, xs))[:8]:
    print("px", y, x, "cnt", cnt[y, x], rc[y, x], "T", T[y, x], fw["final_T"][y, x], "img", img[y, x], fw["image"][y, x])
proj = O.project(ost, ocam)
sp = art.frame.splats(0)
idx = proj["idx"]
on = sp["n_tiles"][idx] > 0
print("mean2d max diff", np.abs(sp["mean2d"][idx][on] - proj["mean2d"][on]).max())
con = proj["conic"]; ref_con = np.stack([con[:, 0, 0], con[:, 0, 1], con[:, 1, 1]], 1)
rel = np.abs(sp["conic"][idx][on] - ref_con[on]) / np.maximum(np.abs(ref_con[on]), 1e-300)
print("conic max rel diff", rel.max())
print("opac max diff", np.abs(sp["opac"][idx][on] - proj["opac"][on]).max())
print("colors max diff", np.abs(sp["colors"][idx][on] - proj["colors"][on]).max())
dL = np.random.default_rng(0).normal(0, 1e-4, img.shape)
g = cg.rasterize_backward(st, cam, art, dL).numpy()
og = O.raster_backward(ost, ocam, dL)
tz = (a.positions.astype(np.float64) @ ocam.R.T + ocam.t)[:, 2]
for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
    diff = np.abs(g[k] - og[k])
    bad = ~np.isclose(g[k], og[k], rtol=1e-4, atol=1e-6)
    rows = np.unique(np.nonzero(bad)[0]) if bad.ndim > 1 else np.nonzero(bad)[0]
    print(k, "violations", int(bad.sum()), "rows", len(rows), "max diff", diff.max(), "max ref", np.abs(og[k]).max())
    for r in rows[:6]:
        extra = f" tz {tz[r]:.4f} ntiles {sp['n_tiles'][r]}" if k in ("positions", "opacity_logits") else ""
        print("   row", r, "ours", g[k][r], "ref", og[k][r], extra)
