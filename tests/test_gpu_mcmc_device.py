"""GPU: the throughput trainer's device split proposals (cgs_split_propose):
proposals and acceptance probabilities follow the reference formulas
(sampler.py:138-164) on the drawn u, the coins are consistent with them,
draws are a pure function of (seed, counter, candidate), and a device-noise
trainer with forced split / merge keeps the scene's invariants."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _propose(n, dim, es, em, lam, seed, ctr, corr_on=True):
    from paper_2509_03775_b200 import _native as nat
    dev = torch.device("cuda", 0)
    u = torch.empty((n, dim), dtype=torch.float64, device=dev)
    prob = torch.empty((n,), dtype=torch.float64, device=dev)
    acc = torch.empty((n,), dtype=torch.int8, device=dev)
    c_q = 1.0 / es ** 2 - 1.0 / em ** 2
    corr = dim * math.log(em / es) if corr_on else 0.0
    nat.call("cgs_split_propose", n, dim, es, c_q, 1 if corr_on else 0, corr, lam, seed, ctr,
             nat.ptr(u), nat.ptr(prob), nat.ptr(acc), nat.stream_handle(dev))
    return u.cpu().numpy(), prob.cpu().numpy(), acc.cpu().numpy().astype(bool)


def test_split_proposals_follow_the_reference_formulas():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    n, dim, es, em, lam = 200000, 7, 0.05, 0.2, 1.5
    u, prob, acc = _propose(n, dim, es, em, lam, 1234, 77)
    # u ~ N(0, es^2 I): moments
    assert abs(u.mean()) < 3e-4 and abs(u.std() / es - 1.0) < 5e-3
    # prob = exp(min(0, -lam - log q)), log q = -0.5 |u|^2 (1/es^2 - 1/em^2) + d ln(em/es)
    log_q = -0.5 * np.einsum("nd,nd->n", u, u) * (1.0 / es ** 2 - 1.0 / em ** 2) + dim * math.log(em / es)
    ref = np.exp(np.minimum(0.0, -lam - log_q))
    assert np.allclose(prob, ref, rtol=1e-12, atol=0.0)
    # coins uniform: the accept rate matches the mean probability
    assert abs(acc.mean() - prob.mean()) < 4 * math.sqrt(prob.mean() * (1 - prob.mean()) / n) + 1e-4
    # a pure function of (seed, counter, candidate): same inputs, same draws;
    # a prefix of the candidates draws the same values
    u2, prob2, acc2 = _propose(1000, dim, es, em, lam, 1234, 77)
    assert np.array_equal(u2, u[:1000]) and np.array_equal(acc2, acc[:1000])
    u3, _, _ = _propose(1000, dim, es, em, lam, 1234, 78)
    assert not np.array_equal(u3, u2)


def test_device_noise_trainer_mcmc_keeps_invariants():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import scenes
    from paper_2509_03775_b200.engine import Trainer
    from paper_2509_03775_b200.model import validate_state
    a, g = scenes.config0(0), scenes.config0(1)
    cams = a.cameras
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                    g.sr_rows)
    H, W = cams[0].height, cams[0].width
    gts = cg.render_frame(gst, cams).image.view(len(cams), H, W, 3).clone()
    cfg = cg.SamplerConfig(lambda_ssim=0.2, device_noise=True, seed=3, noise_pos=0.01,
                           split_fraction=0.2)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    tr = Trainer(st, cams, gts, cfg, np.random.default_rng(5), mcmc_every=2, use_graphs=True)
    for _ in range(12):
        tr.step()
    torch.cuda.synchronize()
    tr.check()
    assert tr.mcmc_events == 6
    validate_state(st)  # refcounts match the device indices, lineage consistent
