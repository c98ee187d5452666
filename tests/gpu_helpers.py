"""Build device states / cameras from golden fixtures (GPU tests only)."""

import numpy as np

from paper_2509_03775_b200 import Camera, ModelState


def state_from(d, p, device="cuda"):
    st = ModelState.from_arrays(d[p + "positions"], d[p + "opacity_logits"], d[p + "g2sh"],
                                d[p + "g2sr"], d[p + "sh_rows"], d[p + "sr_rows"],
                                sh_refcount=d[p + "sh_refcount"], sr_refcount=d[p + "sr_refcount"],
                                sh_parent=d[p + "sh_parent"], sr_parent=d[p + "sr_parent"],
                                device=device, iteration=int(d[p + "iteration"]))
    for book, name in ((st.sh, "sh"), (st.sr, "sr")):
        import heapq
        book._free = [int(r) for r in d[p + name + "_free"]]
        heapq.heapify(book._free)
    return st


def cam_from(d, p):
    fx, fy, cx, cy = (float(v) for v in d[p + "intr"])
    w, h = (int(v) for v in d[p + "size"])
    return Camera(rotation=d[p + "R"], translation=d[p + "t"], fx=fx, fy=fy, cx=cx, cy=cy,
                  width=w, height=h)


def host_state(st):
    return st.to_host()


def assert_state_equal(st, d, p):
    h = st.to_host()
    assert np.array_equal(h["positions"], d[p + "positions"]), "positions"
    assert np.array_equal(h["opacity_logits"], d[p + "opacity_logits"]), "logits"
    assert np.array_equal(h["g2sh"], d[p + "g2sh"]), "g2sh"
    assert np.array_equal(h["g2sr"], d[p + "g2sr"]), "g2sr"
    for name in ("sh", "sr"):
        assert np.array_equal(h[name + "_rows"], d[p + name + "_rows"]), name + "_rows"
        assert np.array_equal(h[name + "_refcount"], d[p + name + "_refcount"]), name + "_refcount"
        assert np.array_equal(h[name + "_parent"], d[p + name + "_parent"]), name + "_parent"
        assert np.array_equal(h[name + "_free"], d[p + name + "_free"]), name + "_free"


def group_rel(a, r):
    a = np.asarray(a, np.float64)
    r = np.asarray(r, np.float64)
    return float(np.abs(a - r).max()) / max(float(np.abs(r).max()), 1e-30) if r.size else 0.0
