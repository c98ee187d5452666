"""Diagnostic: run the config-1 trainer without per-step synchronisation (as
the bench does) with torch's sync debug mode on, so any synchronising torch
call inside MCMC / densify / re-capture is reported with its stack; host time
of each step printed for the slow ones."""
import os
import sys
import time
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_03775_b200 as cg  # noqa: E402
from paper_2509_03775_b200 import scenes  # noqa: E402
from paper_2509_03775_b200.engine import Trainer  # noqa: E402

a, g = scenes.config1(0), scenes.config1(1)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows,
                               gaussian_headroom=0.25)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
gts = cg.render_frame(gst, a.cameras).image.view(4, 256, 256, 3).clone()
cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, noise_pos=0.01)
tr = Trainer(st, a.cameras, gts, cfg, np.random.default_rng(0), use_graphs=True)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
warnings.simplefilter("always")
torch.cuda.set_sync_debug_mode("warn")
for k in range(120):
    t0 = time.perf_counter()
    it0 = st.iteration
    if k == 94:
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
        tr.step()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
    else:
        tr.step()
    dt = 1000 * (time.perf_counter() - t0)
    if dt > 2.0:
        print(f"update {k}: iteration {it0} -> {st.iteration}: host {dt:.2f} ms", flush=True)
torch.cuda.set_sync_debug_mode(0)
torch.cuda.synchronize()
print("mcmc_ms", [round(x, 2) for x in tr.mcmc_ms], "densify_ms", tr.densify_ms, "capture_ms",
      tr.capture_ms)
