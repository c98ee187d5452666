import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2509_03775_b200 as cg
from paper_2509_03775_b200 import scenes, model
a = scenes.config1(0)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows, gaussian_headroom=0.25)
rng = np.random.default_rng(0)
st.prefetch_host_index()
torch.cuda.synchronize()
import cProfile, pstats
for it in range(3):
    t0 = time.perf_counter()
    pr = cProfile.Profile(); pr.enable()
    k = cg.densify(st, 0.05, 10**9, rng)
    torch.cuda.synchronize()
    pr.disable()
    print("densify", it, k, round(1000*(time.perf_counter()-t0), 2), "ms")
    if it == 0:
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
