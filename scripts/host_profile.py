"""cProfile of the bench's training steps (host side) on the GPU box."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_03775_b200 as cg  # noqa: E402
from paper_2509_03775_b200 import scenes  # noqa: E402
from paper_2509_03775_b200.engine import Trainer  # noqa: E402

graphs = "--graphs" in sys.argv
a, g = scenes.config1(0), scenes.config1(1)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
fr = cg.render_frame(gst, a.cameras)
gts = fr.image.view(4, 256, 256, 3).clone()
cfg = cg.SamplerConfig(device_noise=True, noise_pos=0.01)
tr = Trainer(st, a.cameras, gts, cfg, np.random.default_rng(0), use_graphs=graphs)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    tr.step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

# device timeline via CUPTI (torch.profiler): kernel time vs step time
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(20):
        tr.step()
    torch.cuda.synchronize()
ka = [e for e in prof.events() if e.device_type.name == "CUDA"]
tot = sum(e.device_time_total for e in ka) if ka else 0
print(f"CUDA kernel time total over 20 steps: {tot/1000:.2f} ms")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))

# gaps in the device timeline
kev = sorted([(e.time_range.start, e.time_range.end, e.name) for e in prof.events()
              if e.device_type.name == "CUDA"])
span = kev[-1][1] - kev[0][0]
busy = sum(b - a for a, b, _ in kev)
print(f"span {span/1000:.2f} ms  busy {busy/1000:.2f} ms  over 20 steps")
gaps = []
for (a0, b0, n0), (a1, b1, n1) in zip(kev, kev[1:]):
    gaps.append((a1 - b0, n0[:40], n1[:40]))
gaps.sort(reverse=True)
for gp in gaps[:25]:
    print(f"gap {gp[0]:9.1f} us  after {gp[1]:40s} before {gp[2]}")
import collections
agg = collections.defaultdict(float)
for gp, a, b in gaps:
    if gp > 0:
        agg[b] += gp
print("gap time by next kernel:")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"  {v/1000:8.3f} ms  before {k}")
