"""Per-step GPU time of the config-3 trainer (bench settings) with the
transition events marked: how much of each densify / reassignment / MCMC
event shows up as device time (GPU diagnostic)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_03775_b200 as cg  # noqa: E402
from paper_2509_03775_b200.engine import Trainer  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
a, g, cams = bench.make_scene(cfgn, 0, 0, 1)
dev = torch.device("cuda", 0)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows,
                               device=dev, gaussian_headroom=0.25)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows,
                                device=dev)
fr = cg.render_frame(gst, cams)
H, W = cams[0].height, cams[0].width
gts = (fr.image.view(len(cams), H, W, 3).clamp(0, 1) * 255).round() / 255
del fr, gst
extra = {"reassign_every": 100, "reassign_tau": 1e-8} if cfgn == 3 else {}
if st.num_gaussians >= 2_000_000:
    extra["gaussian_cap"] = int(st.num_gaussians * 1.25)
cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, seed=0, noise_pos=0.01, **extra)
tr = Trainer(st, cams, gts, cfg, np.random.default_rng(0), mcmc_every=100, use_graphs=True)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
s_ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
e_ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
marks = []
for k in range(steps):
    c0 = (tr.mcmc_events, len(tr.densify_ms), len(tr.reassign_ms), tr.captures)
    s_ev[k].record()
    h0 = time.perf_counter()
    tr.step()
    h1 = time.perf_counter()
    e_ev[k].record()
    c1 = (tr.mcmc_events, len(tr.densify_ms), len(tr.reassign_ms), tr.captures)
    marks.append((c1[0] - c0[0], c1[1] - c0[1], c1[2] - c0[2], c1[3] - c0[3], 1000 * (h1 - h0)))
torch.cuda.synchronize()
ms = [s.elapsed_time(e) for s, e in zip(s_ev, e_ev)]
p50 = float(np.median(ms))
print(f"config {cfgn}: {steps} steps, total {sum(ms):.1f} ms, p50 {p50:.3f} ms, excess over p50 "
      f"{sum(ms) - steps * p50:.1f} ms")
for k, (m, (mc, dn, ra, cp, hms)) in enumerate(zip(ms, marks)):
    if mc or dn or ra or cp or m > 1.5 * p50:
        print(f"  step {k:4d}: {m:8.2f} ms (excess {m - p50:7.2f})  host {hms:7.2f} ms  "
              f"mcmc {mc} densify {dn} reassign {ra} recapture {cp}")
print("mcmc_ms", [round(x, 1) for x in tr.mcmc_ms], "densify_ms", [round(x, 1) for x in tr.densify_ms],
      "reassign_ms", [round(x, 1) for x in tr.reassign_ms], "capture_ms", [round(x, 1) for x in tr.capture_ms])
