"""Live per-kernel launch times (CUDA events on the launch stream) of the
config-4 render-only frames, for 1 and 16 views per frame (GPU diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_03775_b200 as cg  # noqa: E402
from paper_2509_03775_b200 import _native as nat  # noqa: E402
from paper_2509_03775_b200 import scenes  # noqa: E402

a = scenes.config4(0)
st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
lib = nat.library()
KERNELS = ["project_kernel", "onesweep_kernel", "scan_kernel", "depth_tie_fix_kernel",
           "emit_pairs_kernel", "tile_count_kernel", "tile_scatter_kernel", "raster_fwd_kernel",
           "refine_fwd_kernel"]
for B in [int(x) for x in (sys.argv[1:] or ["1", "16"])]:
    frames = [cg.Frame(st, a.cameras[i:i + B]).run_checked() for i in range(0, 16, B)]
    for f in frames:
        f.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in frames:
        f.run()
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    s = frames[0].stats()
    print(f"views/frame {B}: 16 poses {total:.2f} ms ({16 * 1920 * 1080 / total / 1e3:.0f} Mpix/s); "
          f"frame 0: onscreen {s.n_onscreen} pairs {s.n_pairs} refined tiles {s.n_refined_tiles}", flush=True)
    for k in KERNELS:
        lib.cgs_profile_kernel(k.encode())
        for f in frames:
            f.run()
        torch.cuda.synchronize()
        ms, n = nat.F64(0.0), nat.I64(0)
        lib.cgs_profile_read(ms, n)
        print(f"   {k:22s} {ms.value:9.3f} ms over {n.value} launches", flush=True)
    lib.cgs_profile_kernel(b"")
    del frames
    torch.cuda.empty_cache()
