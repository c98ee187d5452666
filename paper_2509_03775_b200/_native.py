"""ctypes binding of ``libcgs_b200.so`` (C ABI: include/cgs_b200.h).

The product path has no CPU fallback: if the library is missing or a CUDA
device is absent, every compute entry point raises.  Pointers passed here
are raw device addresses of torch tensors; every call is enqueued on the
caller's current torch CUDA stream.
"""

from __future__ import annotations

import ctypes

import numpy as np
import os

from .camera import CCamera

LIB_PATH = os.environ.get("CGS_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libcgs_b200.so")  # override: tuning variants

CGS_OK, CGS_EINVAL, CGS_ECUDA, CGS_EWORKSPACE, CGS_ENONFINITE = 0, 1, 2, 3, 4
MAX_VIEWS = 16


class CScene(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("positions", ctypes.c_void_p),
        ("opacity_logits", ctypes.c_void_p),
        ("g2sh", ctypes.c_void_p),
        ("g2sr", ctypes.c_void_p),
        ("sh_rows", ctypes.c_void_p),
        ("sh_capacity", ctypes.c_int64),
        ("sh_degree", ctypes.c_int32),
        ("sr_rows", ctypes.c_void_p),
        ("sr_capacity", ctypes.c_int64),
    ]


class CFrameStats(ctypes.Structure):
    _fields_ = [
        ("n_onscreen", ctypes.c_int64),
        ("n_pairs", ctypes.c_int64),
        ("n_processed", ctypes.c_int64),
        ("n_touched", ctypes.c_int64),
        ("pair_capacity", ctypes.c_int64),
        ("overflow", ctypes.c_int32),
        ("n_views", ctypes.c_int32),
        ("zero_quaternion", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("n_refined_tiles", ctypes.c_int64),
        ("n_refined_pixels", ctypes.c_int64),
        ("diag_last_mismatch", ctypes.c_int64),
        ("diag_count_mismatch", ctypes.c_int64),
        ("diag_max_T_err", ctypes.c_float),
        ("diag_max_alpha_err", ctypes.c_float),
    ]


class CSgldParams(ctypes.Structure):
    _fields_ = [
        ("step_pos", ctypes.c_double), ("step_opacity", ctypes.c_double),
        ("step_sh", ctypes.c_double), ("step_sr", ctypes.c_double),
        ("noise_pos", ctypes.c_double), ("noise_opacity", ctypes.c_double),
        ("noise_sh", ctypes.c_double), ("noise_sr", ctypes.c_double),
        ("grad_scale", ctypes.c_double),
        ("seed", ctypes.c_uint64), ("offset", ctypes.c_uint64),
        ("noise_source", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("offset_dev", ctypes.c_void_p),
        ("skip_if", ctypes.c_void_p),
        ("sticky", ctypes.c_void_p),
        ("grads_nonfinite", ctypes.c_void_p),
    ]


P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
SZ = ctypes.c_size_t
F32 = ctypes.c_float
F64 = ctypes.c_double
U64 = ctypes.c_uint64
CAMP = ctypes.POINTER(CCamera)
SCNP = ctypes.POINTER(CScene)

# name -> (restype, argtypes); must match include/cgs_b200.h
SIGNATURES = {
    "cgs_abi_version": (I32, []),
    "cgs_last_error": (ctypes.c_char_p, []),
    "cgs_launch_count": (ctypes.c_uint64, []),
    "cgs_profile_kernel": (I32, [ctypes.c_char_p]),
    "cgs_profile_read": (I32, [ctypes.POINTER(F64), ctypes.POINTER(I64)]),
    "cgs_trace_tiles": (I32, [ctypes.c_void_p]),
    "cgs_frame_workspace_bytes": (SZ, [I64, CAMP, I32, I64, I64]),
    "cgs_render_forward": (I32, [SCNP, CAMP, I32, P, SZ, I64, P, P, P, P]),
    "cgs_frame_stats": (I32, [P, ctypes.POINTER(CFrameStats), P]),
    "cgs_code_nn_workspace_bytes": (SZ, [I64, I32]),
    "cgs_code_nn": (I32, [P, I32, I64, P, I64, P, P, P, SZ, P]),
    "cgs_project": (I32, [SCNP, CAMP, I32, P, SZ, I64, P]),
    "cgs_sort_depth": (I32, [SCNP, CAMP, I32, P, SZ, I64, P]),
    "cgs_duplicate_tiles": (I32, [SCNP, CAMP, I32, P, SZ, I64, P]),
    "cgs_sort_pairs": (I32, [SCNP, CAMP, I32, P, SZ, I64, P]),
    "cgs_raster_fwd": (I32, [SCNP, CAMP, I32, P, SZ, I64, P, P, P, P]),
    "cgs_raster_bwd": (I32, [SCNP, CAMP, I32, P, SZ, I64, P, P, P, SZ, P]),
    "cgs_gaussian_reduce_pullback": (I32, [SCNP, CAMP, I32, P, SZ, I64, F32, P, SZ, P, P, P]),
    "cgs_codebook_reduce": (I32, [SCNP, CAMP, I32, P, SZ, I64, F32, P, P, P, P, P, SZ, P, P, P]),
    "cgs_frame_tile_lists": (I32, [CAMP, I32, I64, I64, I64, P, SZ, P, P, P]),
    "cgs_frame_splats": (I32, [CAMP, I32, I64, I64, I64, P, SZ, I32, P, P, P, P, P, P]),
    "cgs_backward_workspace_bytes": (SZ, [I64, CAMP, I32, I64, I64, I64]),
    "cgs_render_backward": (I32, [SCNP, CAMP, I32, P, SZ, I64, P, P, F32, P, P, P, P, P, SZ, P, P,
                                  P, P, P]),
    "cgs_code_csr_workspace_bytes": (SZ, [I64, I64]),
    "cgs_code_csr": (I32, [P, I64, I64, P, P, P, SZ, P]),
    "cgs_loss_workspace_bytes": (SZ, [I32, I32, I32]),
    "cgs_recon_loss": (I32, [P, P, I32, I32, I32, F64, I32, F32, P, P, P, SZ, P]),
    "cgs_sgld_update": (I32, [P, P, I64, P, I32, P, I64, P, P, I64, I64, I64, P, P, P, P,
                              ctypes.POINTER(CSgldParams), P, P, P, P, P, P]),
    "cgs_split_eligible": (I32, [P, I64, P, P, P, P, SZ, P]),
    "cgs_quantize8": (I32, [P, I64, P, P]),
    "cgs_host_split_eligible": (I32, [P, I64, P, I64, P, P, I32]),
    "cgs_backward_nonfinite_flag": (P, [P]),
    "cgs_host_split_decide": (I32, [P, P, I64, P, P, I64, I32, F64, F64, F64, I32, F64, P, P, P, P,
                                    P]),
    "cgs_apply_splits": (I32, [P, I32, P, P, P, P, P, I64, P]),
    "cgs_split_propose": (I32, [I64, I32, F64, F64, I32, F64, F64, U64, U64, P, P, P, P]),
    "cgs_apply_remap": (I32, [P, I64, P, I64, P]),
    "cgs_densify_append": (I32, [P, P, P, P, I64, P, P, I64, P]),
    "cgs_densify_select_workspace_bytes": (SZ, [I64]),
    "cgs_densify_select": (I32, [P, I64, P, I64, P, P, SZ, P]),
    "cgs_refcount_histogram": (I32, [P, I64, P, I64, P]),
    "cgs_scan_workspace_bytes": (SZ, [I64]),
    "cgs_exclusive_scan_u32": (I32, [P, P, I64, P, P, SZ, P]),
    "cgs_sort_workspace_bytes": (SZ, [I64, I32]),
    "cgs_radix_sort_pairs": (I32, [P, P, I64, I32, I32, P, SZ, P]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def library() -> ctypes.CDLL:
    """Load (once) the CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return library().cgs_last_error().decode(errors="replace")


def check(rc: int, what: str = ""):
    if rc == CGS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == CGS_EINVAL:
        raise ValueError(msg)
    if rc == CGS_ENONFINITE:
        from .sampler import SamplerError
        raise SamplerError(msg)
    raise NativeError(f"cgs error {rc}: {msg}")


def call(name: str, *args):
    """Invoke an ABI function and raise the reference's exception type on failure."""
    rc = getattr(library(), name)(*args)
    check(rc, name)


def cams_array(cams) -> ctypes.Array:
    arr = (CCamera * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = c.to_c()
    return arr


def ptr(t) -> int:
    """Device address of a torch tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def upload(a, device, dtype=None):
    """Host array -> device tensor through pinned memory, enqueued on the current
    stream without blocking the host (a pageable copy would wait for the
    stream's queued work).  The caching host allocator keeps the pinned block
    alive until the copy has completed."""
    import numpy as np
    import torch
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    host = torch.from_numpy(arr)
    if host.numel() == 0:
        return torch.empty(host.shape, dtype=host.dtype, device=device)
    return host.pin_memory().to(device, non_blocking=True)


# ---------------------------------------------------------------------------
# numpy internals the MCMC host loop (cgs_host_split_decide) runs on
def bitgen_ptr(rng) -> int:
    """Address of the bitgen_t behind a numpy Generator (its PyCapsule): the
    C loop draws from the caller's own stream."""
    cap = rng.bit_generator.capsule
    get = ctypes.pythonapi.PyCapsule_GetPointer
    get.restype = ctypes.c_void_p
    get.argtypes = [ctypes.py_object, ctypes.c_char_p]
    return get(cap, b"BitGenerator")


_DDOT = []


def numpy_ddot_ptr():
    """numpy's BLAS ddot (what ``u @ u`` runs for float64 vectors), resolved
    from the OpenBLAS numpy ships and checked against ``u @ u`` bit for bit;
    None if it cannot be found (callers then keep the Python loop)."""
    if _DDOT:
        return _DDOT[0]
    import glob
    import os
    fn = None
    libdir = os.path.join(os.path.dirname(os.path.dirname(np.__file__)), "numpy.libs")
    for path in sorted(glob.glob(os.path.join(libdir, "*openblas*.so*"))):
        try:
            lib = ctypes.CDLL(path)
        except OSError:
            continue
        for name in ("scipy_cblas_ddot64_", "cblas_ddot64_", "cblas_ddot"):
            f = getattr(lib, name, None)
            if f is None:
                continue
            f.restype = ctypes.c_double
            f.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                          ctypes.c_int64]
            rng = np.random.default_rng(12345)
            ok = True
            for d in (1, 3, 7, 12, 48, 100):
                for _ in range(8):
                    u = rng.normal(0.0, 0.1, d)
                    if f(d, u.ctypes.data, 1, u.ctypes.data, 1) != float(u @ u):
                        ok = False
            if ok:
                fn = ctypes.cast(f, ctypes.c_void_p).value
                break
        if fn:
            break
    _DDOT.append(fn)
    return fn
