"""Diagnostic: config-3 tile lists vs the oracle's binning, and backward stats."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_03775_b200 as cg
from paper_2509_03775_b200 import scenes
from oracle import cgs_oracle as O

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
a = scenes.build(cfg, 0)
cam = a.cameras[0]
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
fr = cg.render_frame(st, [cam])
s = fr.stats()
print("pairs", s.n_pairs, "onscreen", s.n_onscreen, "overflow", s.overflow)
offs, ids = fr.tile_lists()
t0 = time.time()
ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
ocam = O.cam_from_any(cam)
proj = O.project(ost, ocam)
roffs, members = O.bin_tiles(proj, ocam)
rids = proj["idx"][proj["order"][members]]
print("oracle binning", time.time() - t0, "s")
print("offsets equal", np.array_equal(offs, roffs), "ids equal", np.array_equal(ids, rids))
if not np.array_equal(ids, rids):
    bad = np.flatnonzero(ids != rids)
    print("mismatches", len(bad), "first", bad[:10])
dL = torch.full_like(fr.image, 1e-3)
g = fr.backward(dL)
torch.cuda.synchronize()
s = fr.stats()
print("processed", s.n_processed, "touched", s.n_touched)
gp = g.positions.abs().sum(1)
print("nonzero position grads", int((gp > 0).sum()))
