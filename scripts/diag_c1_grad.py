"""Diagnostic: config-1 views 1-2 gradients vs the oracle (the full-size
parity test), printing the worst tolerance ratios per gradient array."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_03775_b200 as cg
from oracle import cgs_oracle as O
from paper_2509_03775_b200 import scenes

RTOL, ATOL = 1e-4, 1e-6
a, g = scenes.config1(0), scenes.config1(1)
cams = a.cameras[1:3]
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
fr = cg.render_frame(st, cams)
gfr = cg.render_frame(gst, cams)
ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
dls, refs = [], []
for v, cam in enumerate(cams):
    ocam = O.cam_from_any(cam)
    fw = O.raster_forward(ost, ocam)
    cnt = fr.view_counts(v).cpu().numpy()
    knife = cnt != fw["counts"]
    dL = O.recon_loss_grad(fw["image"], gfr.view_image(v).cpu().numpy().astype(np.float64), 0.2)
    dL[knife] = 0.0
    dls.append(dL)
    refs.append(O.raster_backward(ost, ocam, dL))
dl = torch.as_tensor(np.concatenate([x.reshape(-1) for x in dls]).astype(np.float32)).cuda()
gr = fr.backward(dl).numpy()
for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
    ref = refs[0][k] + refs[1][k]
    ratio = np.abs(gr[k] - ref) / (ATOL + RTOL * np.abs(ref))
    flat = np.argsort(-ratio.reshape(-1))[:5]
    print(k, "max ratio", ratio.max(), "violations", int((ratio > 1).sum()))
    for f in flat:
        idx = np.unravel_index(f, ref.shape)
        print("   ", idx, "gpu", gr[k][idx], "ref", ref[idx], "ratio", ratio[idx])
