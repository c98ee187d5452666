"""Config-3 (or CGS_CFG) host costs of the MCMC-side operations (split, merge, densify,
code reassignment), each timed from a drained device queue, plus a cProfile
of the slowest (GPU diagnostic)."""
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
from paper_2509_03775_b200.sampler import TransitionRecord, merge_step, split_step  # noqa: E402
from paper_2509_03775_b200.reassign import reassign_codes  # noqa: E402
from paper_2509_03775_b200.model import densify  # noqa: E402

CFG = int(os.environ.get("CGS_CFG", "3"))
a, g = scenes.build(CFG, 0), scenes.build(CFG, 1)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows,
                               gaussian_headroom=0.25)
gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
cams = a.cameras[:1]
fr = cg.render_frame(gst, cams)
gts = fr.image.view(1, cams[0].height, cams[0].width, 3).clone()
del fr, gst
cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, noise_pos=0.01, reassign_every=0,
                       gaussian_cap=int(st.num_gaussians * 1.25))
rng = np.random.default_rng(0)
tr = Trainer(st, cams, gts, cfg, rng, mcmc_every=0, use_graphs=True)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()


def timed(name, fn, reps=3, prof=False):
    out = []
    first = "first" in sys.argv  # profile the first call (one-time costs) instead of the last
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if prof and r == (0 if first else reps - 1):
            pr = cProfile.Profile()
            pr.enable()
            fn()
            torch.cuda.synchronize()
            pr.disable()
        else:
            fn()
            torch.cuda.synchronize()
        out.append(1000 * (time.perf_counter() - t0))
        tr.step()
    print(f"{name:10s} " + " ".join(f"{x:8.2f}" for x in out) + " ms", flush=True)
    if prof:
        pstats.Stats(pr).sort_stats("cumtime").print_stats(18)


def split():
    split_step(st, None, cfg, rng, TransitionRecord(iteration=st.iteration + 1, kind="split", codebook="-"))


def merge():
    merge_step(st, None, cfg, rng, TransitionRecord(iteration=st.iteration + 1, kind="merge", codebook="-"))


def dens():
    densify(st, cfg.densify_growth, cfg.gaussian_cap, rng, jitter_sigma=cfg.densify_jitter,
            device_select=True)


def reas():
    for w in ("sh", "sr"):
        reassign_codes(st, w, 1e-8)


def step():
    tr.step()


timed("step", step, reps=5)
timed("split", split, prof="split" in sys.argv)
timed("merge", merge, prof="merge" in sys.argv)
timed("densify", dens, reps=2, prof="densify" in sys.argv)
timed("reassign", reas, prof=True)
timed("step", step, reps=5)
