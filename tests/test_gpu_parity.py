"""GPU parity: the sm_100a path (through the C ABI) vs the reference goldens and
the CPU oracle.  Tolerance (BASELINE.json north_star): images and gradients
within rtol 1e-4 / atol 1e-6 (fp32 device math vs the reference's fp64);
tile lists, depth orders, code assignments and MCMC decisions bit-exact."""

import numpy as np
import pytest

from conftest import golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-6


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_03775_b200 as m
    m._native.library()
    return m


def render_names():
    return [str(n) for n in golden("render_cases")["names"]]


@pytest.mark.parametrize("name", render_names())
def test_forward_matches_reference(cg, name):
    from gpu_helpers import cam_from, state_from
    d = golden("render_cases")
    p = name + "_"
    st = state_from(d, p + "in_")
    cam = cam_from(d, p + "cam_")
    art = cg.rasterize_forward(st, cam)
    img = art.image.cpu().numpy()
    T = art.final_transmittance.cpu().numpy()
    assert np.allclose(img, d[p + "image"], rtol=RTOL, atol=ATOL), np.abs(img - d[p + "image"]).max()
    assert np.allclose(T, d[p + "final_T"], rtol=RTOL, atol=ATOL)
    # discrete outputs: bit-exact
    offs, ids = art.frame.tile_lists()
    assert np.array_equal(offs, d[p + "tile_offsets"])
    assert np.array_equal(ids, d[p + "tile_ids"])
    assert np.array_equal(art.contrib_counts.cpu().numpy(), d[p + "counts"])
    tiles = art.tile_splats
    ntx = (cam.width + 15) // 16
    for (ty, tx), lst in tiles.items():
        t = ty * ntx + tx
        assert np.array_equal(lst, d[p + "tile_ids"][d[p + "tile_offsets"][t]:d[p + "tile_offsets"][t + 1]])
    # projection stage (render.py:145-203) on the visible splats that have tiles
    sp = art.frame.splats(0)
    idx = d[p + "proj_idx"]
    on = sp["n_tiles"][idx] > 0
    assert np.allclose(sp["mean2d"][idx][on], d[p + "proj_mean2d"][on], rtol=1e-12, atol=1e-9)
    con = d[p + "proj_conic"]
    ref_con = np.stack([con[:, 0, 0], con[:, 0, 1], con[:, 1, 1]], 1)
    assert np.allclose(sp["conic"][idx][on], ref_con[on], rtol=1e-10, atol=1e-14)
    assert np.allclose(sp["opac"][idx][on], d[p + "proj_opac"][on], rtol=1e-7)
    assert np.allclose(sp["colors"][idx][on], d[p + "proj_colors"][on], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("name", [n for n in render_names() if n != "behind"])
def test_loss_and_backward_match_reference(cg, name):
    from gpu_helpers import cam_from, group_rel, state_from
    d = golden("render_cases")
    p = name + "_"
    st = state_from(d, p + "in_")
    cam = cam_from(d, p + "cam_")
    lam = float(d[p + "lambda"])
    art = cg.rasterize_forward(st, cam)
    # loss on the reference image (isolates the loss kernels)
    vals = cg.recon_loss(d[p + "image"], d[p + "gt"], lam)
    assert np.allclose(vals, d[p + "loss"], rtol=1e-6, atol=1e-9, equal_nan=True)
    g = cg.rasterize_backward(st, cam, art, d[p + "dL"]).numpy()
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        ref = d[p + "g_" + k]
        assert group_rel(g[k], ref) <= 1e-4, (k, group_rel(g[k], ref))
        assert np.allclose(g[k], ref, rtol=RTOL, atol=ATOL), (k, np.abs(g[k] - ref).max())


def test_loss_grad_matches_reference(cg):
    d = golden("loss_sh")
    for k in range(4):
        a, b, lam = d[f"loss{k}_a"], d[f"loss{k}_b"], float(d[f"loss{k}_lam"])
        vals = cg.recon_loss(a, b, lam)
        assert np.allclose(vals, d[f"loss{k}_vals"], rtol=1e-6, atol=1e-9)
        g = cg.recon_loss_grad(a, b, lam).cpu().numpy()
        ref = d[f"loss{k}_grad"]
        assert np.allclose(g, ref, rtol=1e-4, atol=1e-3 * np.abs(ref).max()), np.abs(g - ref).max()


def test_gradcheck_against_finite_differences(cg):
    """tests/test_render.py:171-182 on the device path: group-rel <= 1e-4 vs FD."""
    from gpu_helpers import cam_from, group_rel, state_from
    d = golden("gradcheck")
    for name in d["names"]:
        p = str(name) + "_"
        st = state_from(d, p + "in_")
        cam = cam_from(d, p + "cam_")
        art = cg.rasterize_forward(st, cam)
        g = cg.rasterize_backward(st, cam, art, d[p + "dL"]).numpy()
        for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
            assert group_rel(g[k], d[p + "fd_" + k]) <= 1e-4, (name, k)


def test_known_pixels(cg):
    """tests/test_render.py:90-123 known answers."""
    cam = cg.Camera(rotation=np.eye(3), translation=np.zeros(3), fx=32.0, fy=32.0, cx=16.0,
                    cy=16.0, width=32, height=32)
    st = cg.init_one_to_one(2, 0, seed=0)
    off_f, off_b = 0.5 * 2.0 / 32, 0.5 * 3.0 / 32
    st.gaussians.positions = np.array([[off_f, off_f, 2.0], [off_b, off_b, 3.0]], np.float32)
    st.gaussians.opacity_logits = np.zeros(2, np.float32)
    rows = np.stack([(np.array([1.0, 0, 0]) - 0.5) / 0.28209479177387814,
                     (np.array([0, 1.0, 0]) - 0.5) / 0.28209479177387814]).astype(np.float32)
    st.sh.rows = rows
    sr = np.zeros((2, 7), np.float32)
    sr[:, 0:3] = -1.0
    sr[:, 3] = 1.0
    st.sr.rows = sr
    img = cg.rasterize_forward(st, cam).image.cpu().numpy()
    assert np.allclose(img[16, 16], [0.5, 0.25, 0.0], atol=1e-6)
    st.gaussians.positions = np.array([[0, 0, -3.0], [0, 0, -1.0]], np.float32)
    art = cg.rasterize_forward(st, cam)
    assert float(art.image.abs().max()) == 0.0
    assert bool((art.final_transmittance == 1).all()) and int(art.contrib_counts.max()) == 0
    g = cg.rasterize_backward(st, cam, art, np.ones((32, 32, 3)))
    assert float(g.flat.abs().max()) == 0.0


def test_zero_upstream_and_stale_artifacts(cg):
    from gpu_helpers import cam_from, state_from
    d = golden("render_cases")
    st = state_from(d, "synth1_in_")
    cam = cam_from(d, "synth1_cam_")
    art = cg.rasterize_forward(st, cam)
    g = cg.rasterize_backward(st, cam, art, np.zeros((cam.height, cam.width, 3)))
    assert float(g.flat.abs().max()) == 0.0
    st.gaussians.positions[0, 0] += 0.25
    with pytest.raises(ValueError):
        cg.rasterize_backward(st, cam, art, np.zeros((cam.height, cam.width, 3)))
    art = cg.rasterize_forward(st, cam)
    with pytest.raises(ValueError):
        cg.rasterize_backward(st, cam, art, np.zeros((cam.height + 1, cam.width, 3)))


def test_deterministic_and_batched_frame_equals_single_views(cg):
    from gpu_helpers import cam_from, state_from
    d = golden("render_cases")
    st = state_from(d, "cfg1s_v0_in_")
    c0, c1 = cam_from(d, "cfg1s_v0_cam_"), cam_from(d, "cfg1s_v1_cam_")
    f = cg.render_frame(st, [c0, c1])
    a0 = cg.rasterize_forward(st, c0)
    a1 = cg.rasterize_forward(st, c1)
    assert torch.equal(f.view_image(0), a0.image) and torch.equal(f.view_image(1), a1.image)
    dl = torch.as_tensor(np.random.default_rng(0).normal(size=(2 * 96 * 96 * 3,)).astype(np.float32),
                         device="cuda") * 1e-4
    g_b = f.backward(dl).numpy()
    g_b2 = f.backward(dl).numpy()
    for k in g_b:
        assert np.array_equal(g_b[k], g_b2[k]), "backward must be bit-deterministic"
    g0 = a0.frame.backward(dl[: 96 * 96 * 3].contiguous()).numpy()
    g1 = a1.frame.backward(dl[96 * 96 * 3:].contiguous()).numpy()
    for k in g_b:
        assert np.allclose(g_b[k], g0[k] + g1[k], rtol=1e-5, atol=1e-9), k


def test_sgld_bit_exact(cg):
    from gpu_helpers import assert_state_equal, state_from
    d = golden("sgld")
    for name in d["names"]:
        st = state_from(d, "in_")
        grads = cg.GradientSet.empty(st)
        for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
            getattr(grads, k).copy_(torch.as_tensor(d["g_" + k].astype(np.float32)))
        kw = {}
        for key, v in d.items():
            pre = f"{name}_cfg_"
            if key.startswith(pre):
                kw[key[len(pre):]] = v.item() if v.shape == () else v
        cfg = cg.SamplerConfig(**kw)
        rng = np.random.default_rng(1234)
        cg.sgld_update(st, grads, cfg, rng)
        assert_state_equal(st, d, f"{name}_out_")
        assert np.array_equal(rng.random(4), d[f"{name}_rng_after"])


def test_sgld_rejects_nonfinite(cg):
    from gpu_helpers import state_from
    d = golden("sgld")
    st = state_from(d, "in_")
    grads = cg.GradientSet.empty(st)
    grads.flat.zero_()
    grads.sr_rows[3, 2] = float("nan")
    before = st.gaussians.positions.clone()
    with pytest.raises(cg.SamplerError):
        cg.sgld_update(st, grads, cg.SamplerConfig(), np.random.default_rng(0))
    assert torch.equal(before, st.gaussians.positions)


@pytest.mark.parametrize("chain", ["defaults", "always", "corrected"])
def test_mcmc_chain_bit_exact(cg, chain):
    """train_step split/merge branches + densify vs the reference, step by step."""
    from gpu_helpers import assert_state_equal, state_from
    d = golden("mcmc")
    st = state_from(d, f"{chain}_s0_")
    kw = {}
    for key, v in d.items():
        pre = f"{chain}_cfg_"
        if key.startswith(pre):
            kw[key[len(pre):]] = v.item() if v.shape == () else v
    rng = np.random.default_rng(int(d[f"{chain}_seed"]))
    cam = cg.ring_cameras(1, (0, 0, 0), 3.0, 0.0, 64, 64, 64)[0]
    for step in range(1, int(d[f"{chain}_steps"]) + 1):
        p = f"{chain}_s{step}_"
        kind = str(d[p + "kind"])
        mix = (0.0, 1.0, 0.0) if kind == "split" else (0.0, 0.0, 1.0)
        cfg = cg.SamplerConfig(**{**kw, "p_update": mix[0], "p_split": mix[1], "p_merge": mix[2]})
        rec = cg.train_step(st, [(cam, None)], cfg, rng)
        cg.validate_state(st)
        assert_state_equal(st, d, p)
        assert [rec.attempts, rec.accepts, rec.delta_sh, rec.delta_sr, rec.live_sh,
                rec.live_sr] == d[p + "rec"].tolist()
        assert rec.codebook == str(d[p + "rec_codebook"])
        assert np.array_equal(np.array(rec.accept_probs), d[p + "accept_probs"])
    assert np.array_equal(rng.random(4), d[f"{chain}_rng_after"])


def test_train_loop_matches_reference(cg):
    """train() (sampler.py:402-420) for 16 iterations on config 0 against the
    reference's own run (tests/golden/train.npz): a mixed schedule of updates,
    splits and merges drawn by choose_transition, densify every 5 and PSNR
    every 4.  Discrete outcomes (transition kinds, codebooks, attempts,
    accepts, live counts, final assignments / refcounts / lineage / free
    lists) are bit-exact; recon and PSNR, and the final float state after
    ten fp32-gradient SGLD updates, within tolerance."""
    from gpu_helpers import state_from
    d = golden("train")
    st = state_from(d, "s0_")
    kw = {k[len("cfg_"):]: (v.item() if v.shape == () else v) for k, v in d.items()
          if k.startswith("cfg_")}
    cfg = cg.SamplerConfig(**kw)
    cam = cg.ring_cameras(1, (0, 0, 0), 3.0, 0.0, 64, 64, 64)[0]
    recs = cg.train(st, [(cam, d["gt"])], cfg, 16, rng=np.random.default_rng(11), eval_every=4,
                    check_invariants=True)
    assert [r.kind for r in recs] == [str(k) for k in d["kinds"]]
    assert [r.codebook for r in recs] == [str(k) for k in d["codebooks"]]
    assert np.array_equal(np.array([[r.iteration, r.attempts, r.accepts, r.live_sh, r.live_sr]
                                    for r in recs]), d["ints"])
    got = np.array([[r.recon, r.psnr] for r in recs], dtype=np.float64)
    want = d["floats"]
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.allclose(got[:, 0][ok[:, 0]], want[:, 0][ok[:, 0]], rtol=1e-4, atol=1e-7)
    assert np.allclose(got[:, 1][ok[:, 1]], want[:, 1][ok[:, 1]], rtol=0, atol=2e-3)  # dB
    h = st.to_host()
    for k in ("g2sh", "g2sr", "sh_refcount", "sr_refcount", "sh_parent", "sr_parent", "sh_free",
              "sr_free"):
        assert np.array_equal(h[k], d["s1_" + k]), k
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        assert np.allclose(h[k], d["s1_" + k], rtol=1e-4, atol=1e-5), (
            k, np.abs(h[k] - d["s1_" + k]).max())


def test_densify_bit_exact(cg):
    from gpu_helpers import assert_state_equal, state_from
    d = golden("mcmc")
    st = state_from(d, "defaults_s0_")
    rng = np.random.default_rng(7)
    assert cg.densify(st, 0.05, 2_000_000, rng, jitter_sigma=0.02) == int(d["densify_added"])
    assert_state_equal(st, d, "densify_out_")
    cg.validate_state(st)


def test_update_step_matches_oracle(cg):
    """One full reference update transition (forward, L1+SSIM loss, backward,
    SGLD with host noise) vs the oracle from identical inputs."""
    from oracle import cgs_oracle as O
    from paper_2509_03775_b200 import scenes
    a = scenes.config1(3, n=3000, k=256, views=2, size=96)
    g = scenes.config1(4, n=3000, k=256, views=2, size=96)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
    views = [(c, cg.rasterize_forward(gst, c).image.cpu().numpy()) for c in a.cameras]
    cfg = cg.SamplerConfig(p_update=1.0, p_split=0.0, p_merge=0.0, noise_pos=0.0)
    ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    oviews = [(O.cam_from_any(c), im.astype(np.float64)) for c, im in views]
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    rec = cg.train_step(st, views, cfg, r1)
    orec = O.train_step(ost, oviews, O.config(p_update=1.0, p_split=0.0, p_merge=0.0, noise_pos=0.0), r2)
    assert abs(rec.recon - orec["recon"]) <= 1e-5 * abs(orec["recon"])
    h = st.to_host()
    # one SGLD step moves parameters by 0.5*eps*grad; compare the motion
    for k, ok, base in (("positions", "positions", a.positions),
                        ("opacity_logits", "logits", a.opacity_logits)):
        mine = h[k].astype(np.float64) - base
        ref = getattr(ost, ok).astype(np.float64) - base
        assert np.abs(mine - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-12) + 2e-7, k
    assert np.array_equal(r1.random(3), r2.random(3))


@pytest.mark.parametrize("key_bytes,bits", [(2, 14), (4, 22), (8, 64), (4, 32)])
def test_onesweep_sort_is_stable(cg, key_bytes, bits):
    nat = cg._native
    rng = np.random.default_rng(key_bytes * 100 + bits)
    for n in (0, 1, 1000, 4097, 300_000):
        dt = {2: np.uint16, 4: np.uint32, 8: np.uint64}[key_bytes]
        hi = min(2 ** bits, 2 ** 63) if bits < 64 else 2 ** 63
        keys = rng.integers(0, min(hi, 1000 if n > 1000 else hi), size=n).astype(dt)
        if key_bytes == 8 and n:
            keys = (keys.astype(np.uint64) << np.uint64(40)) | rng.integers(0, 2 ** 40, n).astype(np.uint64)
        vals = np.arange(n, dtype=np.uint32)
        kt = torch.as_tensor(keys.view(np.int16 if key_bytes == 2 else np.int32 if key_bytes == 4 else np.int64)).cuda()
        vt = torch.as_tensor(vals.view(np.int32)).cuda()
        ws = torch.empty(nat.library().cgs_sort_workspace_bytes(max(n, 1), key_bytes), dtype=torch.uint8, device="cuda")
        nat.call("cgs_radix_sort_pairs", nat.ptr(kt), nat.ptr(vt), n, key_bytes, bits, nat.ptr(ws),
                 ws.numel(), nat.stream_handle())
        order = np.argsort(keys, kind="stable")
        got_v = vt.cpu().numpy().view(np.uint32)
        assert np.array_equal(got_v, vals[order])
        assert np.array_equal(kt.cpu().numpy().view(dt), keys[order])


def test_scan(cg):
    nat = cg._native
    rng = np.random.default_rng(3)
    for n in (0, 1, 2047, 2048, 2049, 1_000_003):
        x = rng.integers(0, 50, size=n).astype(np.uint32)
        xt = torch.as_tensor(x.view(np.int32)).cuda()
        out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        tot = torch.zeros(1, dtype=torch.int64, device="cuda")
        ws = torch.empty(nat.library().cgs_scan_workspace_bytes(max(n, 1)), dtype=torch.uint8, device="cuda")
        nat.call("cgs_exclusive_scan_u32", nat.ptr(xt), nat.ptr(out), n, nat.ptr(tot), nat.ptr(ws),
                 ws.numel(), nat.stream_handle())
        ref = np.cumsum(x, dtype=np.uint64) - x
        assert np.array_equal(out.cpu().numpy()[:n].view(np.uint32), ref.astype(np.uint32))
        assert int(tot.item()) == int(x.sum())


def _crowded_scene(seed=3, n=30000):
    """Gaussians packed in front of a 64x64 camera: tile lists of 2k-20k splats,
    so every tile-sort class (<=2048 bitonic, <=4096 bitonic, radix) runs."""
    from paper_2509_03775_b200 import scenes
    a = scenes.config0(seed)
    rng = np.random.default_rng(seed)
    pos = np.empty((n, 3), np.float32)
    pos[:, 0] = rng.uniform(-0.5, 0.5, n)
    pos[:, 1:] = rng.normal(0.0, 0.6, (n, 2))
    k = a.sr_rows.shape[0]
    idx = rng.integers(0, k, n).astype(np.int32)
    return (pos, rng.normal(0.0, 1.0, n).astype(np.float32), idx, idx, a.sh_rows, a.sr_rows,
            a.cameras[0])


def _config1_view0():
    from paper_2509_03775_b200 import scenes
    a = scenes.config1(0)
    return (a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows, a.cameras[0])


def _plane_scene(n, seed=5):
    """n splats on the plane z = 0 seen by an axis-aligned camera: every splat
    has exactly the same fp64 depth, so the depth order inside each tile is
    the Gaussian index alone -- one run of n equal depth keys (the long-run
    path of the depth tie fix: shared-memory bitonic sort up to 8192, the
    per-element rank beyond)."""
    from paper_2509_03775_b200 import camera, scenes
    a = scenes.config0(seed)
    rng = np.random.default_rng(seed)
    side = 96
    cam = camera.Camera(rotation=np.eye(3), translation=np.array([0.0, 0.0, 4.0]), fx=96.0,
                        fy=96.0, cx=side / 2, cy=side / 2, width=side, height=side)
    pos = np.zeros((n, 3), np.float32)
    pos[:, :2] = rng.uniform(-1.6, 1.6, size=(n, 2))
    perm = rng.permutation(n)  # index order unrelated to position
    pos = pos[perm]
    idx = rng.integers(0, a.sr_rows.shape[0], n).astype(np.int32)
    logit = rng.normal(-2.0, 0.5, n).astype(np.float32)
    return pos, logit, idx, idx, a.sh_rows, a.sr_rows, cam


@pytest.mark.parametrize("n", [2000, 12000])
def test_equal_depth_plane_order_bit_exact(cg, n):
    """A run of n splats at one exact depth (longer than the per-element tie
    fix handles): tile lists and per-tile order equal the oracle's (index
    order), and the image matches."""
    from oracle import cgs_oracle as O
    pos, logit, g2sh, g2sr, sh, sr, cam = _plane_scene(n)
    st = cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    fr = cg.render_frame(st, [cam])
    offs, ids = fr.tile_lists()
    ost = O.OState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    ocam = O.cam_from_any(cam)
    proj = O.project(ost, ocam)
    assert len(np.unique(proj["t"][:, 2])) == 1  # one exact depth
    roffs, members = O.bin_tiles(proj, ocam)
    rids = proj["idx"][proj["order"][members]]
    assert np.array_equal(offs, roffs)
    assert np.array_equal(ids, rids)
    ref = O.raster_forward(ost, ocam)
    img = fr.image.view(cam.height, cam.width, 3).cpu().numpy()
    assert np.allclose(img, ref["image"], rtol=RTOL, atol=ATOL)
    assert np.array_equal(fr.counts.view(cam.height, cam.width).cpu().numpy(), ref["counts"])


@pytest.mark.parametrize("make", [_crowded_scene, _config1_view0], ids=["crowded", "config1"])
def test_full_size_tile_lists_bit_exact(cg, make):
    """Tile lists (binning + per-tile fp64 depth order) at full size vs the oracle's
    vectorised _bin_tiles restatement (render.py:203, 240-254)."""
    from oracle import cgs_oracle as O
    pos, logit, g2sh, g2sr, sh, sr, cam = make()
    st = cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    fr = cg.render_frame(st, [cam])
    offs, ids = fr.tile_lists()
    ost = O.OState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    ocam = O.cam_from_any(cam)
    proj = O.project(ost, ocam)
    roffs, members = O.bin_tiles(proj, ocam)
    rids = proj["idx"][proj["order"][members]]
    lens = np.diff(roffs)
    assert np.array_equal(offs, roffs)
    assert np.array_equal(ids, rids)
    if make is _crowded_scene:  # the three sort classes were exercised
        assert lens.max() > 4096 and np.any((lens > 2048) & (lens <= 4096)) and np.any(lens <= 2048)


def _multi_plane_scene(seed=9, planes=48):
    """Splats on 48 planes z = const seen by an axis-aligned camera: each
    plane is one run of equal depth keys, 1-300 splats long, so the sorted
    keys hold runs inside one tie-fix window, across window edges and longer
    than the window's halo or the per-element limit."""
    from paper_2509_03775_b200 import camera, scenes
    a = scenes.config0(seed)
    rng = np.random.default_rng(seed)
    side = 96
    cam = camera.Camera(rotation=np.eye(3), translation=np.array([0.0, 0.0, 4.0]), fx=96.0,
                        fy=96.0, cx=side / 2, cy=side / 2, width=side, height=side)
    lens = rng.integers(1, 300, planes)
    z = np.repeat(np.linspace(-1.0, 1.4, planes), lens).astype(np.float32)
    n = len(z)
    pos = np.zeros((n, 3), np.float32)
    pos[:, :2] = rng.uniform(-1.3, 1.3, size=(n, 2))
    pos[:, 2] = z
    pos = pos[rng.permutation(n)]
    idx = rng.integers(0, a.sr_rows.shape[0], n).astype(np.int32)
    logit = rng.normal(-2.0, 0.5, n).astype(np.float32)
    return pos, logit, idx, idx, a.sh_rows, a.sr_rows, cam


def test_equal_depth_runs_order_bit_exact(cg):
    """Many runs of equal depth keys of lengths 1-300 (depth tie fix: window
    ranks, window-crossing and long runs): tile lists equal the oracle's."""
    from oracle import cgs_oracle as O
    pos, logit, g2sh, g2sr, sh, sr, cam = _multi_plane_scene()
    st = cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    fr = cg.render_frame(st, [cam])
    offs, ids = fr.tile_lists()
    ost = O.OState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    ocam = O.cam_from_any(cam)
    proj = O.project(ost, ocam)
    roffs, members = O.bin_tiles(proj, ocam)
    rids = proj["idx"][proj["order"][members]]
    assert np.array_equal(offs, roffs)
    assert np.array_equal(ids, rids)
    ref = O.raster_forward(ost, ocam)
    assert np.array_equal(fr.counts.view(cam.height, cam.width).cpu().numpy(), ref["counts"])


def _wide_scene(w, h):
    """Config-0 Gaussians seen by one large view: 7500 tiles (counting tile
    sort, 32768-pair chunks) or 12288 tiles (above kCountMaxTiles: the
    two-pass onesweep tile sort)."""
    from paper_2509_03775_b200 import camera, scenes
    a = scenes.config0(11)
    cam = camera.ring_cameras(1, (0.0, 0.0, 0.0), 3.0, 0.0, float(w) / 2, w, h)[0]
    return a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows, cam


@pytest.mark.parametrize("wh", [(1600, 1200), (2048, 1536)], ids=["counting", "onesweep"])
def test_large_view_tile_lists_bit_exact(cg, wh):
    """Both tile-sort paths (render_fwd.cu) give _bin_tiles' lists (render.py:240-254)."""
    from oracle import cgs_oracle as O
    pos, logit, g2sh, g2sr, sh, sr, cam = _wide_scene(*wh)
    st = cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    fr = cg.render_frame(st, [cam])
    offs, ids = fr.tile_lists()
    ost = O.OState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    ocam = O.cam_from_any(cam)
    proj = O.project(ost, ocam)
    roffs, members = O.bin_tiles(proj, ocam)
    assert np.array_equal(offs, roffs)
    assert np.array_equal(ids, proj["idx"][proj["order"][members]])
    assert roffs[-1] > 40000  # several chunks


def _giant_scene(seed=5, n=240, giants=6, size=320):
    """A few near-plane Gaussians covering every one of 400 tiles (> kLongSplat
    pairs: CTA-per-splat emission and reduction) among ordinary ones."""
    from paper_2509_03775_b200 import camera, scenes
    a = scenes.config0(seed)
    rng = np.random.default_rng(seed)
    cam = camera.ring_cameras(1, (0.0, 0.0, 0.0), 3.0, 0.0, float(size), size, size)[0]
    pos = rng.uniform(-0.8, 0.8, size=(n, 3)).astype(np.float32)
    eye = -cam.rotation.T @ cam.translation
    fwd = cam.rotation[2]
    for k in range(giants):  # just beyond the near plane, in front of the eye
        pos[k] = (eye + fwd * (0.05 + 0.02 * k) + rng.normal(0, 0.01, 3)).astype(np.float32)
    idx = rng.integers(0, a.sr_rows.shape[0], n).astype(np.int32)
    sr = a.sr_rows.copy()
    sr[idx[:giants], 0:3] = -1.0  # large scales for the giants' rows
    logit = rng.normal(-1.0, 0.5, n).astype(np.float32)
    return pos, logit, idx, idx, a.sh_rows, sr, cam


def test_near_plane_giants_match_oracle(cg):
    from gpu_helpers import group_rel
    from oracle import cgs_oracle as O
    pos, logit, g2sh, g2sr, sh, sr, cam = _giant_scene()
    st = cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    art = cg.rasterize_forward(st, cam)
    ost = O.OState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    ocam = O.cam_from_any(cam)
    fw = O.raster_forward(ost, ocam)
    offs, ids = art.frame.tile_lists()
    assert np.array_equal(offs, fw["tile_offsets"]) and np.array_equal(ids, fw["tile_ids"])
    assert np.diff(offs).min() > 0 and (np.bincount(ids) > 256).sum() >= 3  # giants in every tile
    img = art.image.cpu().numpy()
    assert np.allclose(img, fw["image"], rtol=RTOL, atol=ATOL), np.abs(img - fw["image"]).max()
    dL = np.random.default_rng(1).normal(0, 1e-3, img.shape)
    g = cg.rasterize_backward(st, cam, art, dL).numpy()
    og = O.raster_backward(ost, ocam, dL)
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        assert group_rel(g[k], og[k]) <= 1e-4, (k, group_rel(g[k], og[k]))
        assert np.allclose(g[k], og[k], rtol=RTOL, atol=ATOL), (k, np.abs(g[k] - og[k]).max())


def _deep_stack_scene(seed=7, n=2400, size=48):
    """Thousands of faint, wide Gaussians stacked in depth over 9 tiles: the
    processed prefixes span several backward chunks (kChunk = 256 splats),
    pixels terminate inside and across chunks, some never do."""
    from paper_2509_03775_b200 import camera, scenes
    a = scenes.config0(seed)
    rng = np.random.default_rng(seed)
    cam = camera.ring_cameras(1, (0.0, 0.0, 0.0), 3.0, 0.0, float(size), size, size)[0]
    pos = np.empty((n, 3), np.float32)
    pos[:, :2] = rng.uniform(-0.3, 0.3, size=(n, 2))
    pos[:, 2] = rng.uniform(-1.0, 1.0, size=n)
    pos = pos @ cam.rotation.astype(np.float32)  # x, y across the view, z along it
    idx = rng.integers(0, a.sr_rows.shape[0], n).astype(np.int32)
    sr = a.sr_rows.copy()
    sr[:, 0:3] = rng.uniform(-0.8, -0.4, size=(sr.shape[0], 3))
    logit = rng.normal(-4.5, 0.5, n).astype(np.float32)
    return pos, logit, idx, idx, a.sh_rows, sr, cam


def test_staged_abi_equals_fused(cg):
    """The staged entry points (cgs_project ... cgs_raster_fwd, cgs_raster_bwd
    ... cgs_codebook_reduce) reproduce cgs_render_forward / _backward bit for
    bit on a config-1 frame (2 views, 256x256)."""
    from paper_2509_03775_b200 import scenes
    a = scenes.config1(0)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    cams = a.cameras[:2]
    fused = cg.Frame(st, cams).run_checked()
    staged = cg.Frame(st, cams, pair_capacity=fused.pair_cap).run_staged()
    for x in ("image", "final_T", "counts"):
        assert torch.equal(getattr(fused, x), getattr(staged, x)), x
    o1, i1 = fused.tile_lists()
    o2, i2 = staged.tile_lists()
    assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
    dL = torch.randn_like(fused.image) * 1e-3
    g1 = fused.backward(dL, scale=0.5)
    g2 = staged.backward_staged(dL, scale=0.5)
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        assert torch.equal(getattr(g1, k), getattr(g2, k)), k
    # the split form the multi-GPU trainer uses (per-Gaussian gradients
    # handed to a callback before the codebook reduce) gives the same bits,
    # and the callback sees the per-Gaussian part already final
    seen = {}

    def after(g):
        torch.cuda.current_stream().synchronize()
        seen["pos"] = g.positions.clone()

    g3 = fused.backward(dL, scale=0.5, after_gaussians=after)
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        assert torch.equal(getattr(g1, k), getattr(g3, k)), k
    assert torch.equal(seen["pos"], g1.positions)


def test_deep_stack_chunked_backward_matches_oracle(cg):
    """Backward work units split a tile's processed prefix into 256-splat
    chunks started from the forward's per-pixel checkpoints (T and colour
    suffix): image, T, counts and gradients match the oracle."""
    from gpu_helpers import group_rel
    from oracle import cgs_oracle as O
    pos, logit, g2sh, g2sr, sh, sr, cam = _deep_stack_scene()
    st = cg.ModelState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    art = cg.rasterize_forward(st, cam)
    ost = O.OState.from_arrays(pos, logit, g2sh, g2sr, sh, sr)
    ocam = O.cam_from_any(cam)
    fw = O.raster_forward(ost, ocam)
    offs, ids = art.frame.tile_lists()
    assert np.array_equal(offs, fw["tile_offsets"]) and np.array_equal(ids, fw["tile_ids"])
    cnt = art.contrib_counts.cpu().numpy()
    assert cnt.max() > 1024 and np.diff(offs).min() > 1600  # >= 3 chunks per tile
    assert np.array_equal(cnt, fw["counts"])
    img = art.image.cpu().numpy()
    assert np.allclose(img, fw["image"], rtol=RTOL, atol=ATOL)
    assert np.allclose(art.final_transmittance.cpu().numpy(), fw["final_T"], rtol=RTOL, atol=ATOL)
    dL = np.random.default_rng(2).normal(0, 1e-3, img.shape)
    g = cg.rasterize_backward(st, cam, art, dL).numpy()
    og = O.raster_backward(ost, ocam, dL)
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        assert group_rel(g[k], og[k]) <= 1e-4, (k, group_rel(g[k], og[k]))
        assert np.allclose(g[k], og[k], rtol=RTOL, atol=ATOL), (k, np.abs(g[k] - og[k]).max())


def test_sgld_device_noise_statistics(cg):
    """Throughput mode (device Philox noise): with zero gradients the update is
    exactly k * eta per coordinate, eta ~ N(0, 1) i.i.d.; fresh draws per
    update, deterministic for a given (seed, offset)."""
    n = 200_003  # not a multiple of 4: exercises the ragged last chunk
    rng = np.random.default_rng(0)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    logit = np.zeros(n, np.float32)
    idx = np.zeros(n, np.int32)
    sh = np.zeros((1, 12), np.float32)
    sr = np.array([[-3, -3, -3, 1, 0, 0, 0]], np.float32)

    def run(seed, updates):
        st = cg.ModelState.from_arrays(pos, logit, idx, idx, sh, sr)
        grads = cg.GradientSet.empty(st)
        grads.flat.zero_()
        cfg = cg.SamplerConfig(device_noise=True, seed=seed, noise_pos=1.0, noise_opacity=1.0,
                               step_pos=0.25, step_opacity=0.04)
        ctr = torch.zeros((1,), dtype=torch.int64, device=st.device)
        outs = []
        for _ in range(updates):
            cg.sgld_update(st, grads, cfg, rng, offset_dev=ctr)
            outs.append((st.gaussians.positions.double().cpu().numpy(),
                         st.gaussians.opacity_logits.double().cpu().numpy()))
        return outs

    a = run(7, 2)
    b = run(7, 2)
    for (pa, la), (pb, lb) in zip(a, b):
        assert np.array_equal(pa, pb) and np.array_equal(la, lb)  # deterministic
    eta_p = (a[0][0] - pos.astype(np.float64)) / (1.0 * np.sqrt(0.25))
    eta_l = (a[0][1] - 0.0) / (1.0 * np.sqrt(0.04))
    eta_p2 = (a[1][0] - a[0][0]) / np.sqrt(0.25)
    for e in (eta_p.ravel(), eta_l, eta_p2.ravel()):
        m = e.size
        assert abs(e.mean()) < 5.0 / np.sqrt(m)
        assert abs(e.std() - 1.0) < 0.01
        assert abs(np.mean(e ** 4) - 3.0) < 0.1  # Gaussian kurtosis
    assert abs(np.corrcoef(eta_p.ravel(), eta_p2.ravel())[0, 1]) < 0.01  # fresh per update


def test_exact_ratio_chain_matches_reference(cg):
    """train_step with exact_ratio=True (sampler.py:309-317): each candidate's
    acceptance uses the rendered loss before/after the trial move; decisions,
    states and the Generator stream match the reference, probabilities to 1e-6."""
    from gpu_helpers import assert_state_equal, cam_from, state_from
    d = golden("exact")
    st = state_from(d, "s0_")
    cam = cam_from(d, "cam_")
    kw = {k[4:]: (v.item() if v.shape == () else v) for k, v in d.items() if k.startswith("cfg_")}
    rng = np.random.default_rng(2024)
    for step in range(1, int(d["steps"]) + 1):
        p = f"s{step}_"
        kind = str(d[p + "kind"])
        mix = (0.0, 1.0, 0.0) if kind == "split" else (0.0, 0.0, 1.0)
        cfg = cg.SamplerConfig(**{**kw, "p_update": mix[0], "p_split": mix[1], "p_merge": mix[2]})
        rec = cg.train_step(st, [(cam, d["gt"])], cfg, rng)
        cg.validate_state(st)
        assert [rec.attempts, rec.accepts, rec.live_sh, rec.live_sr] == d[p + "rec"].tolist()
        assert np.allclose(rec.accept_probs, d[p + "accept_probs"], rtol=1e-6, atol=0)
        assert_state_equal(st, d, p)
    assert np.array_equal(rng.random(4), d["rng_after"])


@pytest.mark.parametrize("views", [(0, 1), (2, 3)])
def test_config1_full_size_matches_oracle(cg, views):
    """BASELINE config 1 at full size (100k Gaussians, SH-3, 256x256), all four
    views (two batched frames of two) against the oracle (~6 s of numpy per
    view): contribution counts bit-exact, images / transmittance within rtol
    1e-4, atol 1e-6, every gradient entry within the same tolerance.

    The raster computes alpha and T in fp32 and the reference in fp64; the
    discrete decisions are nevertheless the reference's: alphas within 2e-5
    of 1/255 or 0.99 are recomputed in float64, and pixels whose fp32
    transmittance comes within 2e-3 of the 1e-4 termination threshold are
    re-walked in float64 (frame stats n_exact_alpha / n_refined; views 1-2
    hold pixels that an fp32-only raster decides differently)."""
    from oracle import cgs_oracle as O
    from paper_2509_03775_b200 import scenes
    a, g = scenes.config1(0), scenes.config1(1)
    cams = [a.cameras[v] for v in views]
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                    g.sr_rows)
    fr = cg.render_frame(st, cams)
    gfr = cg.render_frame(gst, cams)
    ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    dls, refs = [], []
    for v, cam in enumerate(cams):
        ocam = O.cam_from_any(cam)
        fw = O.raster_forward(ost, ocam)
        cnt = fr.view_counts(v).cpu().numpy()
        assert np.array_equal(cnt, fw["counts"]), int((cnt != fw["counts"]).sum())
        img = fr.view_image(v).cpu().numpy()
        T = fr.view_T(v).cpu().numpy()
        assert np.allclose(img, fw["image"], rtol=RTOL, atol=ATOL)
        assert np.allclose(T, fw["final_T"], rtol=RTOL, atol=ATOL)
        dL = O.recon_loss_grad(fw["image"], gfr.view_image(v).cpu().numpy().astype(np.float64), 0.2)
        dls.append(dL)
        refs.append(O.raster_backward(ost, ocam, dL))
    st_ = fr.stats()
    assert st_.n_refined_tiles > 0  # the float64 re-walk ran (and decided like the oracle above)
    dl = torch.as_tensor(np.concatenate([x.reshape(-1) for x in dls]).astype(np.float32)).cuda()
    gr = fr.backward(dl).numpy()
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        ref = refs[0][k] + refs[1][k]
        assert np.allclose(gr[k], ref, rtol=RTOL, atol=ATOL), (k, np.abs(gr[k] - ref).max())


def test_device_densify_matches_host_densify(cg):
    """Throughput-mode densify (device opacity-weighted selection from the same
    host uniforms, deferred refcounts) reproduces the parity-mode densify
    (numpy choice with p, model.py:256) on identical inputs."""
    from gpu_helpers import state_from
    d = golden("mcmc")
    a = state_from(d, "defaults_s0_")
    b = state_from(d, "defaults_s0_")
    ra, rb = np.random.default_rng(99), np.random.default_rng(99)
    for _ in range(3):  # repeated: the second and third read deferred refcounts
        ka = cg.densify(a, 0.05, 10 ** 6, ra)
        kb = cg.densify(b, 0.05, 10 ** 6, rb, device_select=True)
        assert ka == kb
    ha, hb = a.to_host(), b.to_host()
    for k in ("positions", "opacity_logits", "g2sh", "g2sr", "sh_refcount", "sr_refcount"):
        assert np.array_equal(ha[k], hb[k]), k
    cg.validate_state(b)
    assert np.array_equal(ra.random(4), rb.random(4))


@pytest.mark.parametrize("config,pose,rows", [(2, 0, (344, 376)), (3, 0, (528, 560)),
                                              (2, 5, (688, 720)), (3, 3, (96, 128))])
def test_full_scene_strip_matches_oracle(cg, config, pose, rows):
    """BASELINE config 2 / 3 scenes at full size (config 3: 4M Gaussians, SH-3
    K=65536, near-plane giants), rendered through a 32-row strip of a pose (the
    strip is a camera of its own: principal point shifted) so the numpy oracle
    finishes in about a minute: tile lists and contribution counts bit-exact;
    images, T and every gradient entry within rtol 1e-4 / atol 1e-6.

    The strips hold view-covering and near-plane splats (camera z within a
    few times the 0.01 cull distance).  Their d_mean2d and d_conic are large
    sums over every pixel that cancel in the pull-back through J ~ 1/z^3;
    the backward keeps its per-tile moments in tile-local coordinates and
    shifts and sums them in float64, so the cancellation is exact enough for
    the tolerance (the earlier fp32 centre-frame partials missed it by up to
    10%, scripts/diag_sensitivity.py)."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import _strip_cam
    from oracle import cgs_oracle as O
    from paper_2509_03775_b200 import scenes
    a = scenes.build(config, 0)
    ocam = _strip_cam(O.cam_from_any(a.cameras[pose]), *rows)
    cam = cg.Camera(rotation=ocam.R, translation=ocam.t, fx=ocam.fx, fy=ocam.fy, cx=ocam.cx,
                    cy=ocam.cy, width=ocam.width, height=ocam.height)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    art = cg.rasterize_forward(st, cam)
    ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    fw = O.raster_forward(ost, ocam)
    offs, ids = art.frame.tile_lists()
    assert np.array_equal(offs, fw["tile_offsets"]) and np.array_equal(ids, fw["tile_ids"])
    assert np.array_equal(art.contrib_counts.cpu().numpy(), fw["counts"])
    img = art.image.cpu().numpy()
    assert np.allclose(img, fw["image"], rtol=RTOL, atol=ATOL)
    assert np.allclose(art.final_transmittance.cpu().numpy(), fw["final_T"], rtol=RTOL, atol=ATOL)
    dL = np.random.default_rng(0).normal(0, 1e-4, img.shape)
    g = cg.rasterize_backward(st, cam, art, dL).numpy()
    og = O.raster_backward(ost, ocam, dL)
    ntiles = art.frame.splats(0)["n_tiles"]
    tz = (a.positions.astype(np.float64) @ ocam.R.T + ocam.t)[:, 2]
    giants = ((tz > 0.01) & (tz < 0.02)) | (ntiles == len(offs) - 1)
    assert giants.any()  # the strip exercises the cancelling case
    for k in ("positions", "opacity_logits", "sh_rows", "sr_rows"):
        assert np.allclose(g[k], og[k], rtol=RTOL, atol=ATOL), (k, np.abs(g[k] - og[k]).max())
        assert group_rel_np(g[k], og[k]) <= 1e-4, k


def group_rel_np(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def test_split_eligible_abi_matches_host_rule(cg):
    """cgs_split_eligible (device compaction of sampler.py:344's eligibility, kept
    in the ABI for callers without a host assignment mirror) agrees with the
    host rule the sampler uses."""
    from gpu_helpers import state_from
    from paper_2509_03775_b200 import _native as nat
    d = golden("mcmc")
    st = state_from(d, "always_s6_")
    for which, book, idx in (("sh", st.sh, st.gaussians.g2sh), ("sr", st.sr, st.gaussians.g2sr)):
        n = st.num_gaussians
        out = torch.empty((n,), dtype=torch.int32, device=st.device)
        cnt = torch.zeros((1,), dtype=torch.int64, device=st.device)
        ws = torch.empty((nat.library().cgs_scan_workspace_bytes(n) + 1024,), dtype=torch.uint8,
                         device=st.device)
        nat.call("cgs_split_eligible", nat.ptr(idx), n, nat.ptr(book.device_refcount()),
                 nat.ptr(out), nat.ptr(cnt), nat.ptr(ws), ws.numel(), nat.stream_handle(st.device))
        k = int(cnt.item())
        ref = np.flatnonzero(book.refcount[st.host_index(which)] >= 2)
        assert np.array_equal(out[:k].cpu().numpy(), ref), which


def test_config4_batched_strips_match_oracle(cg):
    """BASELINE config 4 (render only, N=6M, K=65536 both) through a batched
    frame of two views -- a 1920x32 strip of pose 0 (rows 524-556, the
    horizon) and one of pose 21 (rows 0-32) -- as bench.py --config 4 renders
    poses in multi-view frames: per view, tile lists and contribution counts
    bit-exact against the oracle (render.py:240-254, 287-315), image and T
    within rtol 1e-4 / atol 1e-6."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import _strip_cam
    from oracle import cgs_oracle as O
    from paper_2509_03775_b200 import scenes
    a = scenes.build(4, 0)
    ocams = [_strip_cam(O.cam_from_any(a.cameras[0]), 524, 556),
             _strip_cam(O.cam_from_any(a.cameras[21]), 0, 32)]
    cams = [cg.Camera(rotation=c.R, translation=c.t, fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy,
                      width=c.width, height=c.height) for c in ocams]
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    fr = cg.render_frame(st, cams)
    offs, ids = fr.tile_lists()
    ost = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    tile0 = 0
    for v, oc in enumerate(ocams):
        fw = O.raster_forward(ost, oc)
        nt = len(fw["tile_offsets"]) - 1
        vo = offs[tile0: tile0 + nt + 1]
        vo = vo - vo[0]
        vids = ids[offs[tile0]: offs[tile0 + nt]]
        assert np.array_equal(vo, fw["tile_offsets"]), v
        assert np.array_equal(vids, fw["tile_ids"]), v
        tile0 += nt
        assert np.array_equal(fr.view_counts(v).cpu().numpy(), fw["counts"]), v
        assert np.allclose(fr.view_image(v).cpu().numpy(), fw["image"], rtol=RTOL, atol=ATOL), v
        assert np.allclose(fr.view_T(v).cpu().numpy(), fw["final_T"], rtol=RTOL, atol=ATOL), v


def test_colour_gate_knife_edge_matches_oracle(cg):
    """SH rows whose float64 colour max(raw + 0.5, 0) sits within a few fp32
    ulps of the gate raw = 0 (render.py:198, 418-419): the projection's fp32
    colour path must hand them to its float64 recompute, so every gate and the
    gated SH gradients equal the oracle's."""
    from gpu_helpers import group_rel
    from oracle import cgs_oracle as O
    from paper_2509_03775_b200 import scenes
    a = scenes.config0(11)
    sh = a.sh_rows.copy()
    c0 = np.float32(-0.5 / O.sh_basis(np.array([[0.0, 0.0, 1.0]]), 0)[0, 0])
    for r in range(96):  # rows 0..95: DC terms k ulps from the gate, no view dependence
        for ch in range(3):
            k = (r + 7 * ch) % 41 - 20
            v = c0
            for _ in range(abs(k)):
                v = np.nextafter(v, np.float32(np.inf) if k > 0 else np.float32(-np.inf))
            sh[r, ch] = v
        sh[r, 3:] = 0.0
    g2sh = (np.arange(a.positions.shape[0]) % 128).astype(np.int32)  # most splats on knife-edge rows
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, g2sh, a.g2sr, sh, a.sr_rows)
    cam = a.cameras[0]
    art = cg.rasterize_forward(st, cam)
    ost = O.OState.from_arrays(a.positions, a.opacity_logits, g2sh, a.g2sr, sh, a.sr_rows)
    ocam = O.cam_from_any(cam)
    proj = O.project(ost, ocam)
    sp = art.frame.splats(0)
    idx = proj["idx"]
    on = sp["n_tiles"][idx] > 0
    knife = np.isin(g2sh[idx], np.arange(96)) & on
    assert knife.sum() > 500
    raw = proj["color_raw"]
    assert ((np.abs(raw[knife]) < 1e-6).sum()) > 500  # really on the edge
    assert np.array_equal(sp["colors"][idx][on] > 0, raw[on] > 0)
    img = art.image.cpu().numpy()
    fw = O.raster_forward(ost, ocam)
    assert np.allclose(img, fw["image"], rtol=RTOL, atol=ATOL)
    dL = np.random.default_rng(2).normal(0, 1e-3, img.shape)
    g = cg.rasterize_backward(st, cam, art, dL).numpy()
    og = O.raster_backward(ost, ocam, dL)
    for k in ("sh_rows", "positions"):
        assert group_rel(g[k], og[k]) <= 1e-4, (k, group_rel(g[k], og[k]))
        assert np.allclose(g[k], og[k], rtol=RTOL, atol=ATOL), (k, np.abs(g[k] - og[k]).max())
