"""Diagnostic: per-CTA timeline of raster_fwd / raster_bwd at config 1
(cgs_trace_tiles).  Prints the kernel span, the CTA duration distribution and
how much of the span runs with fewer resident CTAs than SMs (the tail).

    python scripts/diag_tile_trace.py [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2509_03775_b200 as cg
from paper_2509_03775_b200 import _native as nat
from paper_2509_03775_b200.engine import Trainer

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
a, g, cams = bench.make_scene(cfgn, 0, 0, 1)
dev = torch.device("cuda", 0)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                               a.sr_rows, device=dev, gaussian_headroom=0.25)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                g.sr_rows, device=dev)
gt = cg.render_frame(gst, cams).image.view(len(cams), cams[0].height, cams[0].width, 3)
cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, seed=0, noise_pos=0.01)
tr = Trainer(st, cams, gt.clone(), cfg, np.random.default_rng(0), mcmc_every=10 ** 9,
             use_graphs=False)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
T = tr.frame.desc_total_tiles if hasattr(tr.frame, "desc_total_tiles") else sum(
    ((c.width + 15) // 16) * ((c.height + 15) // 16) for c in cams)
buf = torch.zeros(8 * T + 33, dtype=torch.int64, device=dev)
lib = nat.library()
for rep in range(3):
    buf.zero_()
    lib.cgs_trace_tiles(buf.data_ptr())
    tr.step()
    torch.cuda.synchronize()
    lib.cgs_trace_tiles(None)
    allb = buf.cpu().numpy().astype(np.int64)
    rec = allb[:8 * T].reshape(2, T, 4)
    hist = allb[8 * T:]
    tot = hist.sum()
    print(f"[{rep}] bwd warp hits {tot}: no contribution {hist[0] / tot:.1%}, "
          f"1-4 lanes {hist[1:5].sum() / tot:.1%}, 5-16 {hist[5:17].sum() / tot:.1%}, "
          f"17-31 {hist[17:32].sum() / tot:.1%}, 32 {hist[32] / tot:.1%}")
    print("   per-lane-count fractions 0..32:", " ".join(f"{x / tot:.3f}" for x in hist))
    for name, r in (("fwd", rec[0]), ("bwd", rec[1])):
        r = r[r[:, 1] > 0]
        t0 = r[:, 0].min()
        s, e = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3  # us
        d = e - s
        span = e.max()
        grid = np.linspace(0, span, 400)
        active = np.array([np.sum((s <= x) & (e > x)) for x in grid])
        nsm = len(np.unique(r[:, 2]))
        tail = grid[active < nsm]
        tail_start = tail[tail > span * 0.2].min() if np.any(tail > span * 0.2) else span
        order = np.argsort(-d)
        print(f"[{rep}] {name}: CTAs {len(r)} span {span:.1f} us, CTA us p50 {np.median(d):.1f} "
              f"p90 {np.percentile(d, 90):.1f} max {d.max():.1f}; SMs {nsm}; "
              f"active<SMs from {tail_start:.1f} us ({100 * (span - tail_start) / span:.0f}% of span); "
              f"last start {s.max():.1f} us; sum CTA us / (SMs*span) {d.sum() / (nsm * span):.2f}")
        print("   longest CTAs (start, dur, tile):",
              [(round(s[i], 1), round(d[i], 1), int(r[i, 3])) for i in order[:6]])
        print("   active CTAs at 10%..100% of span:",
              [int(active[min(399, int(399 * f))]) for f in np.linspace(0.1, 1.0, 10)])
