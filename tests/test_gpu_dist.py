"""GPU: the data-parallel update path with its NCCL allreduce in the loop.
Only one GPU is available here, so the process group has one rank (NCCL
still runs the collective); the multi-rank host logic is covered by
tests/test_dist_gloo.py.  With one rank the allreduced trainer must match
the plain one bit for bit."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_allreduce_trainer_matches_single_process():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.distributed as dist
    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import dist as D
    from paper_2509_03775_b200 import scenes
    from paper_2509_03775_b200.engine import Trainer

    a, g = scenes.config0(0), scenes.config0(1)
    cams = a.cameras
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                    g.sr_rows)
    H, W = cams[0].height, cams[0].width
    gts = cg.render_frame(gst, cams).image.view(len(cams), H, W, 3).clone()
    cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, seed=3, noise_pos=0.01)

    def run(allreduce):
        st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                       a.sr_rows)
        tr = Trainer(st, cams, gts, cfg, np.random.default_rng(5), mcmc_every=3, world=1,
                     allreduce=allreduce, use_graphs=True)
        for _ in range(7):
            tr.step()
        torch.cuda.synchronize()
        tr.check()
        return st

    plain = run(None)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        reduced = run(D.make_allreduce())
    finally:
        dist.destroy_process_group()
    assert torch.equal(plain.gaussians.positions, reduced.gaussians.positions)
    assert torch.equal(plain.gaussians.opacity_logits, reduced.gaussians.opacity_logits)
    assert torch.equal(plain.sh.rows, reduced.sh.rows) and torch.equal(plain.sr.rows, reduced.sr.rows)
    assert torch.equal(plain.gaussians.g2sh, reduced.gaussians.g2sh)
