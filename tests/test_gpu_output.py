"""GPU parity of the render-output path (reference cli.py:209-237 cmd_render /
cmd_eval, modelio.py:137-153 save_png / quantize8): the 8-bit bytes of a
rendered view and the PSNR / SSIM of its quantized image, through the
cgs_quantize8 kernel."""

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


def _ref_u8(x):
    """save_png's bytes (modelio.py:139-142) for a float image."""
    return np.clip(np.rint(np.asarray(x, dtype=np.float64) * 255.0), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("n", [0, 1, 3, 5, 4096 * 3 + 7])
def test_quantize8_bit_exact(cg, n):
    """The kernel's bytes equal numpy's float64 rounding of the same fp32 values,
    including exact half steps (round half to even), values outside [0, 1] and
    unaligned sizes (scalar tail)."""
    rng = np.random.default_rng(n)
    x = rng.uniform(-0.2, 1.2, n).astype(np.float32)
    k = rng.integers(0, 255, n)
    half = (k + 0.5) / 255.0
    x[::3] = half[::3].astype(np.float32)  # at (or an ulp from) a rounding boundary
    x[1::7] = (k[1::7] / 255.0).astype(np.float32)
    got = cg.image_to_u8(torch.as_tensor(x).cuda()).cpu().numpy()
    assert np.array_equal(got, _ref_u8(x))
    # unaligned source (scalar path)
    if n > 4:
        xt = torch.as_tensor(x).cuda()[1:]
        assert np.array_equal(cg.image_to_u8(xt).cpu().numpy(), _ref_u8(x[1:]))


def test_quantize8_device_matches_host(cg):
    x = np.random.default_rng(3).uniform(0, 1, (17, 19, 3))
    dev = cg.quantize8(torch.as_tensor(x, dtype=torch.float32).cuda()).cpu().numpy()
    assert np.array_equal(dev, cg.quantize8(x.astype(np.float32)))


def test_render_u8_matches_reference_png_bytes(cg):
    """render_u8 over the golden render cases (one batched frame) vs the bytes
    the reference's cmd_render writes for its own image (save_png of the golden
    image).  The rendered floats match within rtol 1e-4 / atol 1e-6, so a byte
    may differ only where the reference value lies within that tolerance of a
    rounding boundary -- and then by one step."""
    from gpu_helpers import cam_from, state_from
    d = golden("render_cases")
    for name in [str(n) for n in d["names"]]:
        p = name + "_"
        st = state_from(d, p + "in_")
        cam = cam_from(d, p + "cam_")
        (got,) = cg.render_u8(st, [cam])
        ref = d[p + "image"]
        want = _ref_u8(ref)
        assert got.shape == want.shape and got.dtype == np.uint8
        diff = got.astype(int) - want.astype(int)
        y = ref * 255.0
        knife = np.abs(y - np.floor(y) - 0.5) <= 255.0 * (RTOL * np.abs(ref) + ATOL)
        assert np.all(np.abs(diff) <= 1), name
        assert np.all(knife[diff != 0]), name


def test_evaluate_matches_oracle(cg):
    """evaluate (cmd_eval) on two golden views against the oracle's PSNR / SSIM of
    the quantized reference image (metrics.py:67-84, 165-172)."""
    from gpu_helpers import cam_from, state_from
    from oracle import cgs_oracle as O
    d = golden("render_cases")
    st = state_from(d, "cfg0_in_")
    cam = cam_from(d, "cfg0_cam_")
    gt = np.random.default_rng(1).integers(0, 256, d["cfg0_image"].shape) / 255.0
    r = cg.evaluate(st, [(cam, gt), (cam, d["cfg0_image"])])
    q = np.clip(np.rint(d["cfg0_image"] * 255.0), 0, 255) / 255.0
    # (a byte may flip where the reference value sits on a rounding boundary)
    assert np.isclose(r["psnr"][0], O.psnr(q, gt), rtol=1e-4)
    assert np.isclose(r["ssim"][0], O.ssim(q, gt), rtol=1e-4, atol=1e-5)
    assert np.isclose(r["mean_psnr"], np.mean(r["psnr"]))
    assert r["psnr"][1] > 40.0  # quantization noise only


def test_frames_on_concurrent_streams_equal_serial(cg):
    """Frames (own workspaces) rendered concurrently on several streams, as
    the config-4 batch path does, give the serial renders bit for bit."""
    from paper_2509_03775_b200 import scenes
    a = scenes.config1(3, n=20000, views=6, size=96)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows)
    frames = [cg.Frame(st, [c]).run_checked() for c in a.cameras]
    ref = [f.image.clone() for f in frames]
    for f in frames:
        f.image.zero_()
    main = torch.cuda.current_stream()
    streams = [main, torch.cuda.Stream(), torch.cuda.Stream()]
    fork = torch.cuda.Event()
    fork.record(main)
    for s in streams[1:]:
        s.wait_event(fork)
    for i, f in enumerate(frames):
        with torch.cuda.stream(streams[i % 3]):
            f.run()
    for s in streams[1:]:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)
    torch.cuda.synchronize()
    for f, r in zip(frames, ref):
        assert torch.equal(f.image, r)
