"""Diagnostic: config-1 view 0 at full size (100k Gaussians, 256x256) vs the
numpy oracle -- image, T, contribution counts and gradients."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_03775_b200 as cg
from oracle import cgs_oracle as O
from paper_2509_03775_b200 import scenes

a, g = scenes.config1(0), scenes.config1(1)
cam = a.cameras[0]
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
art = cg.rasterize_forward(st, cam)
gt = cg.rasterize_forward(gst, cam).image.cpu().numpy()
img = art.image.cpu().numpy()
ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
ocam = O.cam_from_any(cam)
t0 = time.time()
fw = O.raster_forward(ost, ocam)
print("oracle fwd", round(time.time() - t0, 1), "s")
d = np.abs(img - fw["image"])
print("image max abs", d.max(), "violations", int((~np.isclose(img, fw["image"], rtol=1e-4, atol=1e-6)).sum()))
cnt = art.contrib_counts.cpu().numpy()
print("counts mismatching pixels", int((cnt != fw["counts"]).sum()))
dL = O.recon_loss_grad(fw["image"], gt.astype(np.float64), 0.2)
t0 = time.time()
og = O.raster_backward(ost, ocam, dL)
print("oracle bwd", round(time.time() - t0, 1), "s")
gr = cg.rasterize_backward(st, cam, art, dL).numpy()
for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
    r = og[k]
    v = gr[k]
    rel = np.abs(v - r).max() / max(np.abs(r).max(), 1e-30)
    bad = ~np.isclose(v, r, rtol=1e-4, atol=1e-6)
    print(k, "group-rel", rel, "elementwise violations", int(bad.sum()), "of", r.size,
          "max |ref|", np.abs(r).max())
