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


# ---------------------------------------------------------------------------
# Two ranks on one GPU.  Each rank is a process on cuda:0 running the real
# engine.Trainer over its shard of the config-1 views, with the flat gradient
# buffer summed by a gloo allreduce (host-mediated: no kernel of one rank waits
# on the other's, so sharing the GPU is safe).  This is the multi-GPU path
# minus NCCL: sharding, 1 / total_views pre-scaling, the allreduce operand
# layout, and replica identity through SGLD, MCMC and densify.

def _snapshot(st):
    h = st.to_host()
    out = {k: np.asarray(v) for k, v in h.items()}
    out["sh_free"] = np.array(sorted(st.sh._free), dtype=np.int64)
    out["sr_free"] = np.array(sorted(st.sr._free), dtype=np.int64)
    return out


def _dp_run(rank, world, port, steps, mcmc_every, q):
    import torch.distributed as dist
    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import dist as D
    from paper_2509_03775_b200 import scenes
    from paper_2509_03775_b200.engine import Trainer
    try:
        torch.cuda.set_device(0)
        if world > 1:
            dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                    world_size=world)
        a, g = scenes.config1(0, n=20_000), scenes.config1(1, n=20_000)
        cams = D.shard_views(a.cameras, rank, world)
        st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                       a.sr_rows, gaussian_headroom=0.25)
        gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                        g.sr_rows)
        H, W = cams[0].height, cams[0].width
        gts = cg.render_frame(gst, cams).image.view(len(cams), H, W, 3).clone()
        cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, seed=3, noise_pos=0.01,
                               densify_every=25)
        tr = Trainer(st, cams, gts, cfg, np.random.default_rng(5), mcmc_every=mcmc_every,
                     world=world, allreduce=D.make_allreduce() if world > 1 else None,
                     use_graphs=True, total_views=len(a.cameras))
        for _ in range(steps):
            tr.step()
        torch.cuda.synchronize()
        tr.check()
        q.put((rank, _snapshot(st), tr.mcmc_events, len(tr.densify_ms)))
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, traceback.format_exc(), 0, 0))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _spawn(world, steps, mcmc_every):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_dp_run, args=(r, world, port, steps, mcmc_every, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert not isinstance(r[1], str), r[1]
    assert all(p.exitcode == 0 for p in procs)
    return res


def test_two_rank_trainer_replicas_stay_identical():
    """30 steps on 2 ranks x 2 views (MCMC split + merge every 10 steps, densify
    at iteration 25): both replicas end bit-identical -- positions, logits,
    assignments, both codebooks' rows, refcounts, lineage and free heaps."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    res = _spawn(2, 30, 10)
    (_, s0, ev0, dn0), (_, s1, ev1, dn1) = res
    assert ev0 == ev1 == 3 and dn0 == dn1 >= 1
    for k in s0:
        assert np.array_equal(s0[k], s1[k]), k
    assert len(s0["positions"]) > 20_000  # densify grew N


def test_two_rank_step_equals_one_rank_batch():
    """One update: 2 ranks x 2 views with the allreduce equal the 1-rank update
    over all 4 views (same mean gradient up to the fp32 summation order)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    (_, two, _, _), _ = _spawn(2, 1, 0)
    ((_, one, _, _),) = _spawn(1, 1, 0)
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        a, b = two[k].astype(np.float64), one[k].astype(np.float64)
        assert np.allclose(a, b, rtol=1e-6, atol=1e-7), (k, np.abs(a - b).max())
    for k in ("g2sh", "g2sr", "sh_refcount", "sr_refcount"):
        assert np.array_equal(two[k], one[k]), k


def test_trainer_rejects_nonfinite_gradients_without_a_pass():
    """The one-rank trainer takes the gradients' finiteness from the backward's
    own flag (cgs_backward_nonfinite_flag) instead of a second pass: a NaN in
    a target still rejects the update (no state change) and check() raises
    SamplerError (sampler.py:270-271)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import scenes
    from paper_2509_03775_b200.engine import Trainer
    a, g = scenes.config0(0), scenes.config0(1)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                    g.sr_rows)
    cams = a.cameras
    H, W = cams[0].height, cams[0].width
    gts = cg.render_frame(gst, cams).image.view(len(cams), H, W, 3).clone()
    cfg = cg.SamplerConfig(device_noise=True, noise_pos=0.01)
    tr = Trainer(st, cams, gts, cfg, np.random.default_rng(0), mcmc_every=0, use_graphs=True)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    tr.check()
    before = st.gaussians.positions.clone()
    gts[0, H // 2, W // 2, 0] = float("nan")
    tr.step()
    torch.cuda.synchronize()
    assert torch.equal(before, st.gaussians.positions)
    with pytest.raises(cg.SamplerError):
        tr.check()
