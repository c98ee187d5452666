import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2509_03775_b200 as cg
from oracle import cgs_oracle as O
from paper_2509_03775_b200 import scenes
a = scenes.config1(0)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
for v in range(4):
    cam = a.cameras[v]
    fr = cg.render_frame(st, [cam])
    fw = O.raster_forward(ost, O.cam_from_any(cam))
    T = fr.view_T(0).cpu().numpy(); img = fr.view_image(0).cpu().numpy(); cnt = fr.view_counts(0).cpu().numpy()
    bad = ~np.isclose(T, fw["final_T"], rtol=1e-4, atol=1e-6)
    badi = ~np.isclose(img, fw["image"], rtol=1e-4, atol=1e-6)
    print("view", v, "T viol", bad.sum(), "img viol", badi.sum(), "count mismatch", (cnt != fw["counts"]).sum())
    for y, x in zip(*np.nonzero(bad))[:5] if False else list(zip(*np.nonzero(bad)))[:5]:
        print("  px", y, x, "T", T[y, x], "ref", fw["final_T"][y, x], "cnt", cnt[y, x], fw["counts"][y, x])
