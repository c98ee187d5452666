"""cProfile of the drop-in cg.train() loop at config 1 (reference semantics;
GPU diagnostic)."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_03775_b200 as cg  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
a, g, cams = bench.make_scene(cfgn, 0, 0, 1)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows,
                               gaussian_headroom=0.25)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
views = [(c, cg.rasterize_forward(gst, c).image.cpu().numpy()) for c in cams]
cfg = cg.SamplerConfig(lambda_ssim=0.0 if cfgn == 0 else 0.2, noise_pos=0.01)
rng = np.random.default_rng(0)
cg.train(st, views, cfg, 5, rng)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
cg.train(st, views, cfg, 60, rng)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
