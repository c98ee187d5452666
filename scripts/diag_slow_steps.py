"""Diagnostic: host wall time of every training step at config 1 (graphs on,
bench settings) over 130 updates (MCMC every 25, densify at iteration 100);
cProfile of the slowest step."""
import cProfile
import os
import pstats
import sys
import time

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
times = []
for k in range(130):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it0 = st.iteration
    if k in (74, 99):  # the updates that trigger MCMC / densify
        pr = cProfile.Profile()
        pr.enable()
        tr.step()
        torch.cuda.synchronize()
        pr.disable()
        print(f"--- profile of update {k} (iteration {it0} -> {st.iteration})")
        pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
    else:
        tr.step()
        torch.cuda.synchronize()
    times.append((1000 * (time.perf_counter() - t0), it0, st.iteration))
slow = sorted(times, reverse=True)[:8]
print("slowest steps (ms, iteration before, after):", [(round(t, 2), a_, b_) for t, a_, b_ in slow])
print("median ms", np.median([t for t, _, _ in times]))
print("mcmc_ms", tr.mcmc_ms, "densify_ms", tr.densify_ms, "capture_ms", tr.capture_ms)
