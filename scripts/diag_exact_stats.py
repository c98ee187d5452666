"""Exactness counters per frame and per-stage CUDA-event times at configs
1-3 (GPU diagnostic).  With a CGS_REFINE_ALL=1 build (CGS_LIB_PATH) every
pixel is re-walked in float64 and the counters report where the fp32 path
alone would have decided differently and its largest T error."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_03775_b200 as cg  # noqa: E402
from paper_2509_03775_b200 import scenes  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for config in [int(c) for c in (sys.argv[1:] or ["1", "2", "3"])]:
    a = scenes.build(config, 0)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    views = range(4) if config == 1 else range(min(4, len(a.cameras)))
    for v in views:
        fr = cg.render_frame(st, [a.cameras[v]])
        s = fr.stats()
        tiles = fr.fd_total_tiles if hasattr(fr, "fd_total_tiles") else None
        print(f"config {config} view {v}: pairs {s.n_pairs} refined tiles {s.n_refined_tiles} px {s.n_refined_pixels} "
              f"(of {tiles}) fp32-vs-f64: last differs {s.diag_last_mismatch} count differs "
              f"{s.diag_count_mismatch} max T rel err {s.diag_max_T_err:.3e} max alpha rel err {s.diag_max_alpha_err:.3e}", flush=True)
    fr = cg.render_frame(st, a.cameras[:4] if config == 1 else a.cameras[:1])
    dL = torch.randn_like(fr.image) * 1e-4
    t_f = timed(lambda: fr.run())
    t_b = timed(lambda: fr.backward(dL))
    print(f"  forward {t_f:.3f} ms  backward {t_b:.3f} ms", flush=True)
