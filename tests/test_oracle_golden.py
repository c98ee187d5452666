"""Pin the CPU oracle (oracle/cgs_oracle.py) to the unmodified reference.

Fixtures come from tests/golden/make_golden.py (reference run in the build
container); known answers are the reference's own tests
(pkg/tests/test_render.py, test_sh.py, test_model.py).  No GPU needed.
"""

import math
import os

import numpy as np
import pytest

from conftest import golden
from oracle import cgs_oracle as O


def ostate(d, p):
    return O.OState.from_fixture(d, p)


def render_names():
    return [str(n) for n in golden("render_cases")["names"]]


# -- known answers from the reference's tests --------------------------------
def test_covariance_known_answers():
    # tests/test_render.py:34-50
    row = np.array([0.0, np.log(2.0), np.log(3.0), 1.0, 0.0, 0.0, 0.0])
    assert np.allclose(O.sr_covariance(row), np.diag([1.0, 4.0, 9.0]), atol=1e-12)
    a = np.pi / 2
    row = np.concatenate([[np.log(2.0), 0.0, 0.0], [np.cos(a / 2), 0.0, 0.0, np.sin(a / 2)]])
    assert np.allclose(O.sr_covariance(row), np.diag([1.0, 4.0, 1.0]), atol=1e-12)
    with pytest.raises(ValueError):
        O.sr_covariance(np.zeros(7))


def _front_cam(w=32, h=32, fx=None):
    fx = fx or w
    return O.OCam(R=np.eye(3), t=np.zeros(3), fx=fx, fy=fx, cx=w / 2.0, cy=h / 2.0, width=w, height=h)


def _single(pos, opac, dc, ls=-1.5, n=1):
    sh = O.OCodebook(np.zeros((n, 3)), np.ones(n, np.int64))
    sr = O.OCodebook(np.tile([ls, ls, ls, 1.0, 0, 0, 0], (n, 1)), np.ones(n, np.int64))
    st = O.OState(np.zeros((n, 3)), np.zeros(n), np.arange(n), np.arange(n), sh, sr)
    st.positions[0] = pos
    st.logits[0] = np.log(opac / (1 - opac))
    st.sh.rows[0] = (np.asarray(dc) - 0.5) / 0.28209479177387814
    return st


def test_projection_known_answer():
    # tests/test_render.py:65-71: on-axis z=2, fx=100, Sigma=I -> 2500 I + 0.3 I
    st = _single((0.0, 0.0, 2.0), 0.5, (0.5, 0.5, 0.5), ls=0.0)
    p = O.project(st, _front_cam(64, 64, 100.0))
    assert np.allclose(p["cov2d"][0], 2500.0 * np.eye(2) + 0.3 * np.eye(2), rtol=1e-12)
    st.positions[0] = (0, 0, 0.005)                     # near-plane cull (:73-76)
    assert len(O.project(st, _front_cam())["idx"]) == 0


def test_forward_known_pixels():
    # tests/test_render.py:90-114
    cam = _front_cam(32, 32)
    z = 2.0
    off = 0.5 * z / cam.fx
    st = _single((off, off, z), 0.5, (1.0, 0.0, 0.0), ls=-1.0)
    img = O.raster_forward(st, cam)["image"]
    assert np.allclose(img[16, 16], [0.5, 0.0, 0.0], atol=1e-9)
    st2 = _single((0.5 * 2 / 32, 0.5 * 2 / 32, 2.0), 0.5, (1.0, 0.0, 0.0), ls=-1.0, n=2)
    st2.positions[1] = (0.5 * 3 / 32, 0.5 * 3 / 32, 3.0)
    st2.logits[:] = 0.0
    st2.sh.rows[1] = (np.array([0.0, 1.0, 0.0]) - 0.5) / 0.28209479177387814
    img = O.raster_forward(st2, cam)["image"]
    assert np.allclose(img[16, 16], [0.5, 0.25, 0.0], atol=1e-9)
    # behind camera (:116-123)
    st3 = _single((0.0, 0.0, -3.0), 0.9, (1.0, 1.0, 1.0))
    fw = O.raster_forward(st3, cam)
    assert np.all(fw["image"] == 0) and np.all(fw["final_T"] == 1) and np.all(fw["counts"] == 0)


def test_sh_known_answers(gold):
    # tests/test_sh.py:7-22 and golden basis values / gradients
    d = gold("loss_sh")
    assert abs(O.sh_basis(np.array([0.0, 0.0, 1.0]), 0)[0] - 0.2820948) < 1e-7
    for deg in range(4):
        assert np.allclose(O.sh_basis(d["sh_dirs"], deg), d[f"sh_basis{deg}"], rtol=1e-14, atol=1e-15)
        assert np.allclose(O.sh_basis_grad(d["sh_dirs"], deg), d[f"sh_grad{deg}"], rtol=1e-14, atol=1e-15)


# -- golden render cases -----------------------------------------------------
@pytest.mark.parametrize("name", render_names())
def test_projection_and_binning_match_reference(name):
    d = golden("render_cases")
    p = name + "_"
    st = ostate(d, p + "in_")
    cam = O.cam_from_fixture(d, p + "cam_")
    pr = O.project(st, cam)
    assert np.array_equal(pr["idx"], d[p + "proj_idx"])
    assert np.array_equal(pr["order"], d[p + "proj_order"])         # bit-exact depth order
    for k in ("mean2d", "conic", "radius", "colors", "color_raw", "opac", "t"):
        assert np.allclose(pr[k], d[p + "proj_" + k], rtol=1e-12, atol=1e-12), k
    fw = O.raster_forward(st, cam)
    assert np.array_equal(fw["tile_offsets"], d[p + "tile_offsets"])  # tile lists bit-exact
    assert np.array_equal(fw["tile_ids"], d[p + "tile_ids"])
    assert np.array_equal(fw["counts"], d[p + "counts"])
    assert np.allclose(fw["image"], d[p + "image"], rtol=1e-12, atol=1e-13)
    assert np.allclose(fw["final_T"], d[p + "final_T"], rtol=1e-12, atol=1e-13)
    if p + "naive_image" in d:
        assert np.abs(fw["image"] - d[p + "naive_image"]).max() <= 1e-5   # test_render.py:125-132


@pytest.mark.parametrize("name", [n for n in render_names() if n != "behind"])
def test_loss_and_backward_match_reference(name):
    d = golden("render_cases")
    p = name + "_"
    st = ostate(d, p + "in_")
    cam = O.cam_from_fixture(d, p + "cam_")
    lam = float(d[p + "lambda"])
    img = d[p + "image"]
    l1v, sv, rec = O.recon_loss(img, d[p + "gt"], lam)
    assert np.allclose([l1v, sv, rec], d[p + "loss"], rtol=1e-12, atol=1e-14, equal_nan=True)
    dL = O.recon_loss_grad(img, d[p + "gt"], lam)
    assert np.allclose(dL, d[p + "dL"], rtol=1e-10, atol=1e-15)
    g = O.raster_backward(st, cam, d[p + "dL"])
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        ref = d[p + "g_" + k]
        scale = max(np.abs(ref).max(), 1e-30)
        assert np.abs(g[k] - ref).max() <= 1e-10 * scale, k


def test_gradcheck_cases_match_fd_and_reference():
    # tests/test_render.py:171-182: analytic vs central differences, group-rel <= 1e-4
    d = golden("gradcheck")
    for name in d["names"]:
        p = str(name) + "_"
        st = ostate(d, p + "in_")
        cam = O.cam_from_fixture(d, p + "cam_")
        g = O.raster_backward(st, cam, d[p + "dL"])
        for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
            fd = d[p + "fd_" + k]
            err = np.abs(g[k] - fd).max() / max(np.abs(fd).max(), 1e-8)
            assert err <= 1e-4, (name, k, err)
            assert np.allclose(g[k], d[p + "g_" + k], rtol=1e-9, atol=1e-15)


def test_behind_camera_case():
    d = golden("render_cases")
    st = ostate(d, "behind_in_")
    cam = O.cam_from_fixture(d, "behind_cam_")
    fw = O.raster_forward(st, cam)
    assert np.all(fw["image"] == 0) and np.all(fw["final_T"] == 1) and len(fw["tile_ids"]) == 0


def test_loss_fixtures():
    d = golden("loss_sh")
    for k in range(4):
        a, b, lam = d[f"loss{k}_a"], d[f"loss{k}_b"], float(d[f"loss{k}_lam"])
        assert np.allclose(O.recon_loss(a, b, lam), d[f"loss{k}_vals"], rtol=1e-12, atol=1e-15)
        assert np.allclose(O.recon_loss_grad(a, b, lam), d[f"loss{k}_grad"], rtol=1e-9, atol=1e-16)
        assert math.isclose(O.psnr(a, b), float(d[f"loss{k}_psnr"]), rel_tol=1e-13)


# -- sampler -------------------------------------------------------------------
def _cfg(d, prefix):
    kw = {}
    for k, v in d.items():
        if k.startswith(prefix):
            name = k[len(prefix):]
            kw[name] = v.item() if v.shape == () else v
    return O.config(**kw)


def _assert_state(st, d, p):
    assert np.array_equal(st.positions, d[p + "positions"])
    assert np.array_equal(st.logits, d[p + "opacity_logits"])
    assert np.array_equal(st.g2sh, d[p + "g2sh"])
    assert np.array_equal(st.g2sr, d[p + "g2sr"])
    for b, name in ((st.sh, "sh"), (st.sr, "sr")):
        assert np.array_equal(b.rows, d[p + name + "_rows"]), name
        assert np.array_equal(b.refcount, d[p + name + "_refcount"])
        assert np.array_equal(b.parent, d[p + name + "_parent"])
        assert sorted(b.free) == d[p + name + "_free"].tolist()


def test_sgld_bit_exact():
    d = golden("sgld")
    g = {k: d["g_" + k] for k in ("positions", "opacity_logits", "sh_rows", "sr_rows")}
    for name in d["names"]:
        st = ostate(d, "in_")
        cfg = _cfg(d, f"{name}_cfg_")
        rng = np.random.default_rng(1234)
        O.sgld_update(st, g, cfg, rng)
        _assert_state(st, d, f"{name}_out_")
        assert np.array_equal(rng.random(4), d[f"{name}_rng_after"])


def test_sgld_rejects_nonfinite():
    d = golden("sgld")
    st = ostate(d, "in_")
    g = {k: d["g_" + k].copy() for k in ("positions", "opacity_logits", "sh_rows", "sr_rows")}
    g["sr_rows"][0, 0] = np.nan
    before = st.positions.copy()
    with pytest.raises(O.SamplerError):
        O.sgld_update(st, g, O.config(), np.random.default_rng(0))
    assert np.array_equal(st.positions, before)


@pytest.mark.parametrize("chain", ["defaults", "always", "corrected"])
def test_mcmc_chain_bit_exact(chain):
    d = golden("mcmc")
    st = ostate(d, f"{chain}_s0_")
    cfg = _cfg(d, f"{chain}_cfg_")
    rng = np.random.default_rng(int(d[f"{chain}_seed"]))
    for step in range(1, int(d[f"{chain}_steps"]) + 1):
        p = f"{chain}_s{step}_"
        kind = str(d[p + "kind"])
        cfg.p_update, cfg.p_split, cfg.p_merge = (0.0, 1.0, 0.0) if kind == "split" else (0.0, 0.0, 1.0)
        rec = O.train_step(st, [(None, None)], cfg, rng)
        O.validate(st)
        _assert_state(st, d, p)
        want = d[p + "rec"].tolist()
        assert [rec["attempts"], rec["accepts"], rec["delta_sh"], rec["delta_sr"],
                rec["live_sh"], rec["live_sr"]] == want
        assert rec["codebook"] == str(d[p + "rec_codebook"])
        assert np.array_equal(np.array(rec["probs"]), d[p + "accept_probs"])
    assert np.array_equal(rng.random(4), d[f"{chain}_rng_after"])


def test_densify_bit_exact():
    d = golden("mcmc")
    st = ostate(d, "defaults_s0_")
    rng = np.random.default_rng(7)
    assert O.densify(st, 0.05, 2_000_000, rng, 0.02) == int(d["densify_added"])
    _assert_state(st, d, "densify_out_")
    assert np.array_equal(rng.random(4), d["densify_rng_after"])


def test_acceptance_known_answers():
    # SPEC.md:291,308,326
    u = np.array([0.1])
    assert math.isclose(O.q_sm(u, 0.1, 0.05), math.exp(1.5), rel_tol=1e-12)
    assert math.isclose(O.accept_prob("split", np.zeros(3), 2.3, 0.1, 0.05), math.exp(-2.3), rel_tol=1e-12)
    assert O.accept_prob("merge", np.zeros(3), 2.3, 0.1, 0.05) == 1.0


def test_row_strips_compose_to_the_view():
    """bench.py's CPU baseline splits each view into row strips (one camera each,
    principal point shifted): images concatenate and gradients sum to the
    full view's, since every pixel's compositing depends only on that pixel."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import _strip_cam
    from paper_2509_03775_b200 import scenes
    a = scenes.config0(0)
    st = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    cam = O.cam_from_any(a.cameras[0])
    full = O.raster_forward(st, cam)
    dL = np.random.default_rng(0).normal(0, 1e-3, full["image"].shape)
    gfull = O.raster_backward(st, cam, dL)
    imgs, gsum = [], None
    for y0 in range(0, cam.height, 16):
        c = _strip_cam(cam, y0, min(cam.height, y0 + 16))
        imgs.append(O.raster_forward(st, c)["image"])
        g = O.raster_backward(st, c, dL[y0:y0 + 16])
        gsum = g if gsum is None else {k: gsum[k] + g[k] for k in g}
    assert np.allclose(np.concatenate(imgs, 0), full["image"], rtol=1e-12, atol=1e-15)
    for k in gfull:
        assert np.allclose(gsum[k], gfull[k], rtol=1e-9, atol=1e-15), k
