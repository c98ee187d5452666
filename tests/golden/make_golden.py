"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (the reference does not exist on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. \
        python tests/golden/make_golden.py

Every fixture stores its inputs (so nothing has to be regenerated on the GPU
box) and the reference outputs.  Fixtures are small (configs reduced where
noted) and compressed.  The reference functions called are cited next to
each case.
"""

from __future__ import annotations

import copy
import heapq
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import contrags  # noqa: E402
from contrags import metrics as rmetrics  # noqa: E402
from contrags import modelio as rmodelio  # noqa: E402
from contrags import oracles as roracles  # noqa: E402
from contrags import render as rrender  # noqa: E402
from contrags import sampler as rsampler  # noqa: E402
from contrags import sh as rsh  # noqa: E402
from contrags.camera import Camera as RCamera  # noqa: E402
from contrags.model import Codebook, GaussianArrays, ModelState  # noqa: E402

from paper_2509_03775_b200 import scenes  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
def ref_state(a: scenes.SceneArrays) -> ModelState:
    """Reference ModelState from scene arrays; zero-refcount rows go to the free heap."""
    sh = Codebook(a.sh_rows.copy())
    sr = Codebook(a.sr_rows.copy())
    sh.refcount[:] = np.bincount(a.g2sh, minlength=sh.capacity)
    sr.refcount[:] = np.bincount(a.g2sr, minlength=sr.capacity)
    for book in (sh, sr):
        book._free = [int(r) for r in np.flatnonzero(book.refcount == 0)]
        heapq.heapify(book._free)
    g = GaussianArrays(positions=a.positions.copy(), opacity_logits=a.opacity_logits.copy(),
                       g2sh=a.g2sh.copy(), g2sr=a.g2sr.copy())
    st = ModelState(gaussians=g, sh=sh, sr=sr)
    contrags.validate_state(st)
    return st


def state_arrays(st: ModelState, prefix: str, out: dict):
    """Snapshot (copies: the reference mutates index arrays and rows in place)."""
    g = st.gaussians
    out[prefix + "positions"] = g.positions.copy()
    out[prefix + "opacity_logits"] = g.opacity_logits.copy()
    out[prefix + "g2sh"] = g.g2sh.copy()
    out[prefix + "g2sr"] = g.g2sr.copy()
    for name, book in (("sh", st.sh), ("sr", st.sr)):
        out[prefix + name + "_rows"] = book.rows.copy()
        out[prefix + name + "_refcount"] = book.refcount.copy()
        out[prefix + name + "_parent"] = book.parent.copy()
        out[prefix + name + "_free"] = np.array(sorted(book._free), dtype=np.int64)
    out[prefix + "iteration"] = np.int64(st.iteration)


def cam_arrays(cam, prefix, out):
    out[prefix + "R"] = cam.rotation
    out[prefix + "t"] = cam.translation
    out[prefix + "intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy])
    out[prefix + "size"] = np.array([cam.width, cam.height], dtype=np.int64)


def to_rcam(c) -> RCamera:
    return RCamera(rotation=c.rotation, translation=c.translation, fx=c.fx, fy=c.fy,
                   cx=c.cx, cy=c.cy, width=c.width, height=c.height)


def tile_csr(tile_splats: dict, cam):
    ntx = (cam.width + 15) // 16
    nty = (cam.height + 15) // 16
    offs = [0]
    ids = []
    for ty in range(nty):
        for tx in range(ntx):
            lst = tile_splats[(ty, tx)]
            ids.extend(int(v) for v in lst)
            offs.append(len(ids))
    return np.array(offs, dtype=np.int64), np.array(ids, dtype=np.int64)


def render_case(st: ModelState, cam, gt_img, lam, prefix, out, with_naive=False,
                with_proj=True, backward=True):
    """rasterize_forward / recon_loss(_grad) / rasterize_backward (render.py:287,318)."""
    cam_arrays(cam, prefix + "cam_", out)
    state_arrays(st, prefix + "in_", out)
    art = rrender.rasterize_forward(st, cam)
    out[prefix + "image"] = art.image
    out[prefix + "final_T"] = art.final_transmittance
    out[prefix + "counts"] = art.contrib_counts
    offs, ids = tile_csr(art.tile_splats, cam)
    out[prefix + "tile_offsets"] = offs
    out[prefix + "tile_ids"] = ids
    if with_proj:
        proj = rrender._Projection(st, cam)
        out[prefix + "proj_idx"] = proj.idx
        out[prefix + "proj_t"] = proj.t
        out[prefix + "proj_mean2d"] = proj.mean2d
        out[prefix + "proj_conic"] = proj.conic
        out[prefix + "proj_radius"] = proj.radius
        out[prefix + "proj_colors"] = proj.colors
        out[prefix + "proj_color_raw"] = proj.color_raw
        out[prefix + "proj_opac"] = proj.opac
        out[prefix + "proj_order"] = proj.order
    if with_naive:
        out[prefix + "naive_image"] = roracles.naive_render(st, cam)
    if gt_img is not None:
        out[prefix + "gt"] = gt_img
        out[prefix + "lambda"] = np.float64(lam)
        l1v, sv, recon = rmetrics.recon_loss(art.image, gt_img, lam)
        out[prefix + "loss"] = np.array([l1v, sv, recon])
        dL = rmetrics.recon_loss_grad(art.image, gt_img, lam)
        out[prefix + "dL"] = dL
        if not backward:
            # the reference cannot pull back with zero visible splats
            # (render.py:456 reshapes an empty array) -> no gradient golden
            return art
        gr = rrender.rasterize_backward(st, cam, art, dL)
        out[prefix + "g_positions"] = gr.positions
        out[prefix + "g_opacity_logits"] = gr.opacity_logits
        out[prefix + "g_sh_rows"] = gr.sh_rows
        out[prefix + "g_sr_rows"] = gr.sr_rows
    return art


def make_render():
    out = {}
    names = []
    # (1) config 0, GT from seed 1, L1 loss (lambda 0)
    a = scenes.config0(0)
    g = scenes.config0(1)
    cam = to_rcam(a.cameras[0])
    gt = rrender.rasterize_forward(ref_state(g), cam).image
    render_case(ref_state(a), cam, gt, 0.0, "cfg0_", out)
    names.append("cfg0")
    # (2) reduced config-1 layout: separate SR / [op; SH-3] tables, 2 views, lambda 0.2
    a = scenes.config1(3, n=3000, k=256, views=2, size=96)
    g = scenes.config1(4, n=3000, k=256, views=2, size=96)
    for v, c in enumerate(a.cameras):
        cam = to_rcam(c)
        gt = rrender.rasterize_forward(ref_state(g), cam).image
        render_case(ref_state(a), cam, gt, 0.2, f"cfg1s_v{v}_", out)
        names.append(f"cfg1s_v{v}")
    # (3) reference synth scenes, SH deg 0..3 (tests/test_render.py:125-132)
    for seed in range(6):
        st, man, imgs = rmodelio.synth_scene(40, 1, 48, seed % 4, 10, seed)
        gst, _, _ = rmodelio.synth_scene(40, 1, 48, seed % 4, 10, seed + 100)
        cam = man.views[0].camera
        gt = rrender.rasterize_forward(gst, cam).image
        render_case(st, cam, gt, 0.2, f"synth{seed}_", out, with_naive=True)
        names.append(f"synth{seed}")
    # (4) ragged image (partial tiles on both axes) and a near-plane giant
    a = scenes.config0(5)
    c = a.cameras[0]
    cam = RCamera(rotation=c.rotation, translation=c.translation, fx=40.0, fy=44.0,
                  cx=25.3, cy=18.9, width=50, height=37)
    st = ref_state(a)
    st.gaussians.positions[0] = cam.center() + 0.0101 * cam.rotation[2] + 0.003 * cam.rotation[0]
    st.gaussians.positions[1] = cam.center() + 0.02 * cam.rotation[2]
    g = scenes.config0(6)
    gst = ref_state(g)
    gt = rrender.rasterize_forward(gst, cam).image
    render_case(st, cam, gt, 0.2, "ragged_", out)
    names.append("ragged")
    # (5) everything behind the camera (tests/test_render.py:116-123)
    a = scenes.config0(7)
    st = ref_state(a)
    c = a.cameras[0]
    st.gaussians.positions[:] = (c.center() - 2.0 * c.rotation[2]).astype(np.float32)
    render_case(st, to_rcam(c), np.full((64, 64, 3), 0.25), 0.0, "behind_", out,
                backward=False)
    names.append("behind")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "render_cases.npz"), **out)
    print("render_cases:", names)


def make_gradcheck():
    """make_gradcheck_case + fd_gradient (tests/conftest.py:67-86, oracles.py:178-217)."""
    from conftest import make_gradcheck_case
    out = {}
    names = []
    for degree in (0, 1, 3):
        st, cam, gt, fd = make_gradcheck_case(base_seed=degree * 17 + 1, n=6, size=16,
                                              degree=degree, shared=3, lambda_ssim=0.2)
        p = f"gc{degree}_"
        render_case(st, cam, gt, 0.2, p, out)
        out[p + "fd_positions"] = fd.positions
        out[p + "fd_opacity_logits"] = fd.opacity_logits
        out[p + "fd_sh_rows"] = fd.sh_rows
        out[p + "fd_sr_rows"] = fd.sr_rows
        names.append(f"gc{degree}")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "gradcheck.npz"), **out)
    print("gradcheck:", names)


def make_loss_sh():
    out = {}
    rng = np.random.default_rng(11)
    for k, (h, w, lam) in enumerate([(32, 40, 0.2), (64, 64, 0.0), (23, 17, 0.5), (11, 11, 0.2)]):
        a = rng.uniform(0, 1, size=(h, w, 3))
        b = np.clip(a + rng.normal(0, 0.1, size=a.shape), 0, 1)
        l1v, sv, rec = rmetrics.recon_loss(a, b, lam)
        out[f"loss{k}_a"] = a
        out[f"loss{k}_b"] = b
        out[f"loss{k}_lam"] = np.float64(lam)
        out[f"loss{k}_vals"] = np.array([l1v, sv, rec])
        out[f"loss{k}_grad"] = rmetrics.recon_loss_grad(a, b, lam)
        out[f"loss{k}_psnr"] = np.float64(rmetrics.psnr(a, b))
    dirs = rng.normal(size=(64, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    out["sh_dirs"] = dirs
    for d in range(4):
        out[f"sh_basis{d}"] = rsh.basis(dirs, d)
        out[f"sh_grad{d}"] = rsh.basis_grad(dirs, d)
    np.savez_compressed(os.path.join(OUT, "loss_sh.npz"), **out)
    print("loss_sh written")


def _cfg_arrays(cfg: rsampler.SamplerConfig):
    import dataclasses
    return {f.name: getattr(cfg, f.name) for f in dataclasses.fields(cfg)}


def make_sgld():
    """sgld_update (sampler.py:262-300) on config-0 grads, several configs."""
    out = {}
    a = scenes.config0(0)
    st = ref_state(a)
    # kill a few rows so the live-row masking is exercised
    for i in np.flatnonzero(st.gaussians.g2sh == st.gaussians.g2sh[0]):
        contrags.remap_gaussian(st, int(i), "sh", int(st.gaussians.g2sh[1]))
    cam = to_rcam(a.cameras[0])
    gt = rrender.rasterize_forward(ref_state(scenes.config0(1)), cam).image
    art = rrender.rasterize_forward(st, cam)
    dL = rmetrics.recon_loss_grad(art.image, gt, 0.0)
    gr = rrender.rasterize_backward(st, cam, art, dL)
    # fp32-representable gradients so a fp32-gradient device path is bit comparable
    g32 = rrender.GradientSet(positions=gr.positions.astype(np.float32).astype(np.float64),
                              opacity_logits=gr.opacity_logits.astype(np.float32).astype(np.float64),
                              sh_rows=gr.sh_rows.astype(np.float32).astype(np.float64),
                              sr_rows=gr.sr_rows.astype(np.float32).astype(np.float64))
    state_arrays(st, "in_", out)
    out["g_positions"] = g32.positions
    out["g_opacity_logits"] = g32.opacity_logits
    out["g_sh_rows"] = g32.sh_rows
    out["g_sr_rows"] = g32.sr_rows
    cfgs = {
        "default": rsampler.SamplerConfig(),
        "nonoise": rsampler.SamplerConfig(noise_pos=0.0),
        "allnoise": rsampler.SamplerConfig(noise_opacity=0.5, noise_sh=0.1, noise_sr=0.2),
        "fixture": rsampler.SamplerConfig.for_synthetic_fixture(),
        "zerosteps": rsampler.SamplerConfig(step_pos=0.0, step_sh=0.0),
    }
    names = []
    for name, cfg in cfgs.items():
        s2 = copy.deepcopy(st)
        rng = np.random.default_rng(1234)
        rsampler.sgld_update(s2, g32, cfg, rng)
        state_arrays(s2, f"{name}_out_", out)
        for k, v in _cfg_arrays(cfg).items():
            out[f"{name}_cfg_{k}"] = np.asarray(v)
        out[f"{name}_rng_after"] = np.asarray(rng.random(4))
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "sgld.npz"), **out)
    print("sgld:", names)


def make_mcmc():
    """train_step split/merge branches (sampler.py:339-385) + densify (model.py:235-267).

    Each chain runs forced-mixture steps from a seeded Generator and records
    the full state after every step plus the TransitionRecord.
    """
    out = {}
    chains = {
        # acceptance ~0 at paper defaults: exercises proposals + rejects
        "defaults": (rsampler.SamplerConfig(), 0),
        # lambda 0, eps_s == eps_m -> A == 1: every move accepted
        "always": (rsampler.SamplerConfig(lambda_sh=0.0, lambda_sr=0.0, eps_split_sh=0.05,
                                          eps_merge_sh=0.05, eps_split_sr=0.05,
                                          eps_merge_sr=0.05, split_fraction=0.05,
                                          densify_every=7, gaussian_cap=5000), 1),
        "corrected": (rsampler.SamplerConfig(lambda_sh=-10.0, lambda_sr=-5.5,
                                             normalization_correction=True,
                                             split_fraction=0.03, densify_every=5,
                                             densify_growth=0.02, gaussian_cap=4600), 2),
    }
    names = []
    a = scenes.config0(0)
    schedule = ["split", "split", "merge", "split", "merge", "merge", "split", "merge",
                "split", "split", "merge", "merge"]
    for name, (cfg, seed) in chains.items():
        st = ref_state(a)
        rng = np.random.default_rng(100 + seed)
        state_arrays(st, f"{name}_s0_", out)
        for k, v in _cfg_arrays(cfg).items():
            out[f"{name}_cfg_{k}"] = np.asarray(v)
        out[f"{name}_seed"] = np.int64(100 + seed)
        for step, kind in enumerate(schedule):
            c = copy.deepcopy(cfg)
            c.p_update, c.p_split, c.p_merge = ((0.0, 1.0, 0.0) if kind == "split" else (0.0, 0.0, 1.0))
            rec = rsampler.train_step(st, [(to_rcam(a.cameras[0]), None)], c, rng)
            contrags.validate_state(st)
            p = f"{name}_s{step + 1}_"
            state_arrays(st, p, out)
            out[p + "kind"] = np.array(kind)
            out[p + "rec"] = np.array([rec.attempts, rec.accepts, rec.delta_sh, rec.delta_sr,
                                       rec.live_sh, rec.live_sr])
            out[p + "rec_codebook"] = np.array(rec.codebook)
            out[p + "accept_probs"] = np.array(rec.accept_probs, dtype=np.float64)
        out[f"{name}_steps"] = np.int64(len(schedule))
        out[f"{name}_rng_after"] = np.asarray(rng.random(4))
        names.append(name)
    # stand-alone densify (tests/test_model.py:85-109 shapes, config-0 state)
    st = ref_state(a)
    rng = np.random.default_rng(7)
    added = contrags.densify(st, 0.05, 2_000_000, rng, jitter_sigma=0.02)
    state_arrays(st, "densify_out_", out)
    out["densify_added"] = np.int64(added)
    out["densify_rng_after"] = np.asarray(rng.random(4))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "mcmc.npz"), **out)
    print("mcmc:", names)


def ref_state_from(d, p) -> ModelState:
    """Reference ModelState from a state_arrays snapshot."""
    sh = Codebook(d[p + "sh_rows"].copy())
    sr = Codebook(d[p + "sr_rows"].copy())
    for book, name in ((sh, "sh"), (sr, "sr")):
        book.refcount[:] = d[p + name + "_refcount"]
        book.parent[:] = d[p + name + "_parent"]
        book._free = [int(r) for r in d[p + name + "_free"]]
        heapq.heapify(book._free)
    g = GaussianArrays(positions=d[p + "positions"].copy(),
                       opacity_logits=d[p + "opacity_logits"].copy(),
                       g2sh=d[p + "g2sh"].copy(), g2sr=d[p + "g2sr"].copy())
    st = ModelState(gaussians=g, sh=sh, sr=sr)
    contrags.validate_state(st)
    return st


def make_modelio():
    """serialize_model / deserialize_model (modelio.py:58-127) on MCMC-chain states
    with freed and appended rows, plus the reference's errors on corrupt files."""
    d = dict(np.load(os.path.join(OUT, "mcmc.npz"), allow_pickle=False))
    out = {}
    cases = []
    for chain in [str(n) for n in d["names"]]:
        for step in (0, 6, 12):
            p = f"{chain}_s{step}_"
            data = rmodelio.serialize_model(ref_state_from(d, p))
            out[f"{chain}_s{step}_bytes"] = np.frombuffer(data, dtype=np.uint8).copy()
            cases.append(f"{chain}_s{step}")
    good = rmodelio.serialize_model(ref_state_from(d, "always_s12_"))
    bad = {"truncated": good[:-5], "magic": b"CGSX" + good[4:], "trailing": good + b"\0\0",
           "version": good[:4] + (2).to_bytes(4, "little") + good[8:]}
    for name, blob in bad.items():
        try:
            rmodelio.deserialize_model(blob)
            msg = ""
        except rmodelio.ModelFormatError as e:
            msg = str(e)
        out[f"bad_{name}_bytes"] = np.frombuffer(blob, dtype=np.uint8).copy()
        out[f"bad_{name}_msg"] = np.array(msg)
    out["cases"] = np.array(cases)
    out["bad"] = np.array(list(bad))
    np.savez_compressed(os.path.join(OUT, "modelio.npz"), **out)
    print("modelio:", cases)


def make_exact():
    """train_step with exact_ratio=True (sampler.py:309-317): every split/merge
    candidate renders the view before and after the trial move.  Small scene
    (600 Gaussians sharing 48 rows, 48x48 view) so the reference finishes in
    seconds; lambda small enough that the rendered ratio decides acceptance."""
    rng0 = np.random.default_rng(11)
    n, k = 600, 48
    a = scenes.config0(3)
    pos = rng0.uniform(-0.8, 0.8, (n, 3)).astype(np.float32)
    idx = rng0.integers(0, k, n).astype(np.int32)
    sr = a.sr_rows[:k].copy()
    sr[:, 0:3] += 2.0  # larger splats so moves change the image
    sh = a.sh_rows[:k].copy()
    logit = rng0.normal(0.5, 1.0, n).astype(np.float32)
    arrays = scenes.SceneArrays(pos, logit, idx, idx, sh, sr, 1)
    gt_arrays = scenes.SceneArrays(rng0.uniform(-0.8, 0.8, (n, 3)).astype(np.float32), logit, idx,
                                   idx, sh, sr, 1)
    cam = scenes.ring_cameras(1, (0.0, 0.0, 0.0), 3.0, 0.0, 48.0, 48, 48)[0]
    rcam = to_rcam(cam)
    gt = rrender.rasterize_forward(ref_state(gt_arrays), rcam).image
    cfg = rsampler.SamplerConfig(lambda_sh=1e-3, lambda_sr=1e-3, eps_split_sh=0.05,
                                 eps_merge_sh=0.05, eps_split_sr=0.05, eps_merge_sr=0.05,
                                 split_fraction=0.02, exact_ratio=True, lambda_ssim=0.0,
                                 densify_every=0)
    st = ref_state(arrays)
    out = {}
    state_arrays(st, "s0_", out)
    cam_arrays(cam, "cam_", out)
    out["gt"] = gt
    for kk, v in _cfg_arrays(cfg).items():
        out[f"cfg_{kk}"] = np.asarray(v)
    rng = np.random.default_rng(2024)
    schedule = ["split", "split", "merge", "split", "merge"]
    for step, kind in enumerate(schedule):
        c = copy.deepcopy(cfg)
        c.p_update, c.p_split, c.p_merge = ((0.0, 1.0, 0.0) if kind == "split" else (0.0, 0.0, 1.0))
        rec = rsampler.train_step(st, [(rcam, gt)], c, rng)
        contrags.validate_state(st)
        p = f"s{step + 1}_"
        state_arrays(st, p, out)
        out[p + "kind"] = np.array(kind)
        out[p + "rec"] = np.array([rec.attempts, rec.accepts, rec.live_sh, rec.live_sr])
        out[p + "accept_probs"] = np.array(rec.accept_probs, dtype=np.float64)
    out["steps"] = np.int64(len(schedule))
    out["rng_after"] = np.asarray(rng.random(4))
    np.savez_compressed(os.path.join(OUT, "exact.npz"), **out)
    print("exact: accepts", [int(out[f"s{i + 1}_rec"][1]) for i in range(len(schedule))],
          "attempts", [int(out[f"s{i + 1}_rec"][0]) for i in range(len(schedule))])


def make_train():
    """train() (sampler.py:402-420) end to end on config 0: the reference's own
    loop with a mixed transition schedule (updates, splits, merges drawn by
    choose_transition), densify every 5 iterations and PSNR evaluation every
    4; records every TransitionRecord and the final state."""
    out = {}
    a, g = scenes.config0(0), scenes.config0(1)
    cam = to_rcam(a.cameras[0])
    gt = rrender.rasterize_forward(ref_state(g), cam).image
    cfg = rsampler.SamplerConfig.for_synthetic_fixture(seed=7)
    cfg.p_update, cfg.p_split, cfg.p_merge = 0.6, 0.2, 0.2
    cfg.lambda_sh = cfg.lambda_sr = 0.0   # with eps_s == eps_m: every move accepted
    cfg.eps_merge_sh, cfg.eps_merge_sr = cfg.eps_split_sh, cfg.eps_split_sr
    cfg.densify_every, cfg.gaussian_cap = 5, 4400
    st = ref_state(a)
    state_arrays(st, "s0_", out)
    out["gt"] = gt
    for k, v in _cfg_arrays(cfg).items():
        out[f"cfg_{k}"] = np.asarray(v)
    recs = rsampler.train(st, [(cam, gt)], cfg, 16, rng=np.random.default_rng(11), eval_every=4,
                          check_invariants=True)
    out["kinds"] = np.array([r.kind for r in recs])
    out["codebooks"] = np.array([r.codebook for r in recs])
    out["ints"] = np.array([[r.iteration, r.attempts, r.accepts, r.live_sh, r.live_sr]
                            for r in recs], dtype=np.int64)
    out["floats"] = np.array([[r.recon, r.psnr] for r in recs], dtype=np.float64)
    state_arrays(st, "s1_", out)
    np.savez_compressed(os.path.join(OUT, "train.npz"), **out)
    print("train written", list(out["kinds"]))


MAKERS = {"loss_sh": make_loss_sh, "sgld": make_sgld, "mcmc": make_mcmc, "render": make_render,
          "gradcheck": make_gradcheck, "modelio": make_modelio, "exact": make_exact,
          "train": make_train}

if __name__ == "__main__":
    print("numpy", np.__version__)
    for name in (sys.argv[1:] or list(MAKERS)):
        MAKERS[name]()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
