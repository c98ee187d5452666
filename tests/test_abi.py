"""CPU-side checks of the C ABI: the in-tree library loads (no GPU needed to
dlopen it) and exports every function include/cgs_b200.h declares, and the
ctypes signatures cover exactly that set.  No compute calls here."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "cgs_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"CGS_API\s+[\w\s\*]*?\b(cgs_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2509_03775_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_expected_surface():
    names = declared()
    assert len(names) >= 20
    for must in ("cgs_render_forward", "cgs_render_backward", "cgs_recon_loss", "cgs_sgld_update",
                 "cgs_apply_splits", "cgs_apply_remap", "cgs_densify_append", "cgs_radix_sort_pairs"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_ctypes_signatures_match_header():
    from paper_2509_03775_b200 import _native
    assert sorted(_native.SIGNATURES) == declared()


def test_abi_version_and_error_channel(lib):
    lib.cgs_abi_version.restype = ctypes.c_int
    assert lib.cgs_abi_version() == 1
    lib.cgs_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.cgs_last_error(), bytes)


def test_invalid_arguments_rejected_without_gpu(lib):
    """Argument validation happens before any CUDA call (ValueError path)."""
    from paper_2509_03775_b200 import _native
    from paper_2509_03775_b200.camera import ring_cameras
    _native.library()
    cams = _native.cams_array(ring_cameras(1, (0, 0, 0), 3.0, 0.0, 64, 64, 64))
    # too many views -> 0 bytes + error message
    assert _native.library().cgs_frame_workspace_bytes(10, cams, 17, 1000, 4) == 0
    assert "n_views" in _native.last_error()
    assert _native.library().cgs_frame_workspace_bytes(10, cams, 1, 1000, 4) > 0
    sc = _native.CScene()
    sc.sh_degree = 7
    rc = _native.library().cgs_render_forward(ctypes.byref(sc), cams, 1, None, 0, 1000, None,
                                              None, None, None)
    assert rc == _native.CGS_EINVAL
    with pytest.raises(ValueError):
        _native.check(rc)


def test_staged_and_code_nn_validation_without_gpu(lib):
    """The staged entry points and cgs_code_nn validate before any CUDA call."""
    from paper_2509_03775_b200 import _native
    from paper_2509_03775_b200.camera import ring_cameras
    L = _native.library()
    cams = _native.cams_array(ring_cameras(1, (0, 0, 0), 3.0, 0.0, 64, 64, 64))
    bad = _native.CScene()
    bad.sh_degree = 7
    for fn in ("cgs_project", "cgs_sort_depth", "cgs_duplicate_tiles", "cgs_sort_pairs"):
        assert getattr(L, fn)(ctypes.byref(bad), cams, 1, None, 0, 1000, None) == _native.CGS_EINVAL
    assert L.cgs_raster_fwd(ctypes.byref(bad), cams, 1, None, 0, 1000, None, None, None,
                            None) == _native.CGS_EINVAL
    assert L.cgs_raster_bwd(ctypes.byref(bad), cams, 1, None, 0, 1000, None, None, None, 0,
                            None) == _native.CGS_EINVAL
    assert L.cgs_gaussian_reduce_pullback(ctypes.byref(bad), cams, 1, None, 0, 1000, 1.0, None,
                                          0, None, None, None) == _native.CGS_EINVAL
    assert L.cgs_codebook_reduce(ctypes.byref(bad), cams, 1, None, 0, 1000, 1.0, None, None,
                                 None, None, None, 0, None, None, None) == _native.CGS_EINVAL
    assert L.cgs_project(ctypes.byref(bad), cams, 17, None, 0, 1000, None) == _native.CGS_EINVAL
    # code_nn: widths 1..48 (SH degree 3), non-null arrays
    assert L.cgs_code_nn_workspace_bytes(1000, 48) > 0
    assert L.cgs_code_nn_workspace_bytes(1000, 49) == 0
    assert L.cgs_code_nn_workspace_bytes(1000, 0) == 0
    assert L.cgs_code_nn(None, 48, 10, None, 5, None, None, None, 0, None) == _native.CGS_EINVAL
    assert "code_nn" in _native.last_error()
