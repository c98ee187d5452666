"""Code reassignment extension (BASELINE.json config 3
"code reassignment every 100 iters").

The reference never recomputes assignments by distance: its
only assignment changes are split, merge and densify.  This module is the
build's own, opt-in extension and has no reference oracle; its tests check
it against an fp64 brute force of the same definition.

* ``nearest_codes(state, which)``: for every live row of the codebook, the
  nearest other live row (squared L2 in fp64, ties -> smaller index), from
  the tensor-core distance GEMM behind ``cgs_code_nn``.
* ``reassign_codes(state, which, tau)``: deterministic deduplication of
  near-identical codes: every *mutual* nearest pair (i, j), i < j, with
  distance <= tau is merged -- the Gaussians on j move to i and j is freed,
  with the same bookkeeping as an accepted merge (sampler.py:240-247,
  lineage into j broken).  Mutual pairs are disjoint, so the result does not
  depend on processing order.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .model import ModelState, _book_of


def nearest_codes(state: ModelState, which: str):
    """(nn_index (cap,) int32, nn_dist2 (cap,) float64) as device tensors;
    -1 / 0 for rows that are not live."""
    book, _ = _book_of(state, which)
    dev = book.device
    live = book.device_live()
    n_live = int(live.numel())
    cap = book.capacity
    idx = torch.empty((cap,), dtype=torch.int32, device=dev)
    dist = torch.empty((cap,), dtype=torch.float64, device=dev)
    nb = nat.library().cgs_code_nn_workspace_bytes(n_live, book.dim)
    if nb == 0:
        raise ValueError(nat.last_error() or "code_nn: unsupported codebook width")
    ws = torch.empty((nb,), dtype=torch.uint8, device=dev)
    nat.call("cgs_code_nn", nat.ptr(book.rows), book.dim, cap, nat.ptr(live), n_live,
             nat.ptr(idx), nat.ptr(dist), nat.ptr(ws), nb, nat.stream_handle(dev))
    return idx, dist


def mutual_pairs(nn_index: np.ndarray, nn_dist2: np.ndarray, tau: float) -> list:
    """(parent i, child j) for every mutual nearest pair i < j with d <= tau."""
    nn = np.asarray(nn_index)
    i = np.arange(nn.shape[0])
    j = np.where(nn >= 0, nn, 0)
    keep = (nn > i) & (nn[j] == i) & (np.asarray(nn_dist2) <= tau)
    return [(int(a), int(b)) for a, b in zip(i[keep], nn[keep])]


def reassign_codes(state: ModelState, which: str, tau: float) -> int:
    """Merge every mutual nearest pair of live rows within squared distance
    tau (child -> parent, see module doc).  Returns the number of rows freed."""
    from .sampler import _apply_remap, _merge_bookkeeping
    if tau < 0:
        raise ValueError("tau must be >= 0")
    idx, dist = nearest_codes(state, which)
    pairs = mutual_pairs(idx.cpu().numpy(), dist.cpu().numpy(), tau)
    if not pairs:
        return 0
    book, _ = _book_of(state, which)
    for parent, child in pairs:
        _merge_bookkeeping(book, child, parent)
    _apply_remap(state, which, {c: p for p, c in pairs})
    return len(pairs)
