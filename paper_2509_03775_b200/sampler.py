"""Markov-chain training engine (reference `pkg/src/contrags/sampler.py`).

Same API, same transition semantics and the same consumption of the
caller's ``np.random.Generator``, so split / merge /
densify decisions are bit-identical to the reference.  The continuous work
runs on the device: rendering and gradients through the C ABI, SGLD through
``cgs_sgld_update``, split/merge/densify applies through the MCMC kernels.
Host work is only the inherently sequential accept/reject bookkeeping on the
refcount / lineage / free-list mirrors.

Noise: by default (parity mode) SGLD noise is drawn from the caller's
Generator in the reference's order and uploaded.  With
``SamplerConfig.device_noise=True`` (throughput mode) it is drawn on the
device from Philox(seed, iteration) and the host stream no longer matches
the reference after the first noisy update (documented in DESIGN.md).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .metrics import LossWorkspace, total_loss
from .model import ModelState, _book_of, densify, validate_state
from .render import Frame, GradientSet, backward_workspace_bytes, rasterize_forward


class SamplerError(RuntimeError):
    pass


@dataclass
class SamplerConfig:
    """sampler.py:29-93 (same fields and defaults) + device_noise."""

    p_update: float = 0.98
    p_split: float = 0.01
    p_merge: float = 0.01
    eps_split_sh: float = 0.1
    eps_merge_sh: float = 0.05
    eps_split_sr: float = 0.1
    eps_merge_sr: float = 0.05
    lambda_sh: float = 2.3
    lambda_sr: float = 3.0
    lambda_ssim: float = 0.2
    step_pos: float = 0.5
    step_opacity: float = 10.0
    step_sh: float = 20.0
    step_sr: float = 2.0
    noise_pos: float = 1.0
    noise_opacity: float = 0.0
    noise_sh: float = 0.0
    noise_sr: float = 0.0
    split_fraction: float = 0.01
    densify_every: int = 100
    densify_growth: float = 0.05
    densify_jitter: float = 0.02
    gaussian_cap: int = 2_000_000
    normalization_correction: bool = False
    exact_ratio: bool = False
    seed: int = 0
    device_noise: bool = False
    # code reassignment extension (reassign.py; not in the reference): every
    # reassign_every iterations merge mutual nearest code rows within
    # squared distance reassign_tau.  0 = off (the reference's behaviour).
    reassign_every: int = 0
    reassign_tau: float = 0.0

    def validate(self) -> None:
        if abs(self.p_update + self.p_split + self.p_merge - 1.0) > 1e-12:
            raise ValueError("mixture probabilities must sum to 1")
        for name in ("eps_split_sh", "eps_merge_sh", "eps_split_sr", "eps_merge_sr"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    @classmethod
    def for_synthetic_fixture(cls, seed: int = 0) -> "SamplerConfig":
        return cls(step_pos=4.0, step_opacity=80.0, step_sh=150.0, step_sr=15.0,
                   noise_pos=0.0, gaussian_cap=256, seed=seed)

    def eps_for(self, which: str):
        if which == "sh":
            return self.eps_split_sh, self.eps_merge_sh
        if which == "sr":
            return self.eps_split_sr, self.eps_merge_sr
        raise ValueError(f"unknown codebook {which!r}")

    def lambda_for(self, which: str) -> float:
        return self.lambda_sh if which == "sh" else self.lambda_sr


class TransitionRecord:
    """sampler.py:96-110; ``recon`` may be a device scalar read on first access."""

    def __init__(self, iteration: int, kind: str, codebook: str, attempts: int = 0,
                 accepts: int = 0, delta_sh: int = 0, delta_sr: int = 0, live_sh: int = 0,
                 live_sr: int = 0, recon=float("nan"), psnr: float = float("nan"),
                 accept_probs=None, lambdas=(2.3, 3.0)):
        self.iteration = iteration
        self.kind = kind
        self.codebook = codebook
        self.attempts = attempts
        self.accepts = accepts
        self.delta_sh = delta_sh
        self.delta_sr = delta_sr
        self.live_sh = live_sh
        self.live_sr = live_sr
        self._recon = recon
        self.psnr = psnr
        self.accept_probs = [] if accept_probs is None else accept_probs
        self._lambdas = lambdas

    @property
    def recon(self) -> float:
        if isinstance(self._recon, torch.Tensor):
            self._recon = float(self._recon.item())
        return self._recon

    @recon.setter
    def recon(self, v):
        self._recon = v

    @property
    def total(self) -> float:
        r = self.recon
        if not np.isfinite(r):
            return float("nan")
        return total_loss(r, self.live_sh, self.live_sr, *self._lambdas).total

    def __repr__(self):
        return (f"TransitionRecord(iteration={self.iteration}, kind={self.kind!r}, "
                f"codebook={self.codebook!r}, attempts={self.attempts}, accepts={self.accepts}, "
                f"live_sh={self.live_sh}, live_sr={self.live_sr})")


def choose_transition(config: SamplerConfig, rng: np.random.Generator) -> str:
    """sampler.py:113-119"""
    r = rng.random()
    if r < config.p_update:
        return "update"
    if r < config.p_update + config.p_split:
        return "split"
    return "merge"


def _log_q_sm(u, eps_split, eps_merge, correction):
    u = np.atleast_1d(np.asarray(u, dtype=np.float64))
    u2 = float(u @ u)
    log_q = -0.5 * u2 * (1.0 / eps_split ** 2 - 1.0 / eps_merge ** 2)
    if correction:
        log_q += u.size * math.log(eps_merge / eps_split)
    return log_q


def q_sm(u, eps_split: float, eps_merge: float, correction: bool = False) -> float:
    """sampler.py:122-135"""
    with np.errstate(over="ignore"):
        return float(np.exp(_log_q_sm(u, eps_split, eps_merge, correction)))


def acceptance_probability(kind: str, u, lam: float, eps_split: float, eps_merge: float,
                           correction: bool = False, extra_log_ratio: float = 0.0) -> float:
    """sampler.py:147-164"""
    log_q = _log_q_sm(u, eps_split, eps_merge, correction)
    if kind == "split":
        log_a = -lam - log_q + extra_log_ratio
    elif kind == "merge":
        log_a = lam + log_q + extra_log_ratio
    else:
        raise ValueError(f"unknown transition kind {kind!r}")
    return float(np.exp(min(0.0, log_a)))


@dataclass
class SplitProposal:
    which: str
    gaussian: int
    row: int
    u: np.ndarray
    new_value: np.ndarray


@dataclass
class MergeProposal:
    which: str
    child: int
    parent: int
    u: np.ndarray


# ---------------------------------------------------------------------------
# single-move API (per-call device round trips; train_step batches instead)
def propose_split(state: ModelState, which: str, i: int, config: SamplerConfig,
                  rng: np.random.Generator) -> Optional[SplitProposal]:
    """sampler.py:184-199"""
    book, idx = _book_of(state, which)
    row = int(idx[i])
    if book.refcount[row] < 2:
        return None
    eps_split, _ = config.eps_for(which)
    u = rng.normal(0.0, eps_split, size=book.dim)
    return SplitProposal(which=which, gaussian=int(i), row=row, u=u,
                         new_value=book.row(row).astype(np.float64) + u)


def _apply_split_batch(state: ModelState, which: str, moves):
    """Device apply of accepted splits: moves = [(gaussian, old_row, new_row, u)]."""
    if not moves:
        return
    book, idx = _book_of(state, which)
    dev = book.device
    g = nat.upload(np.array([m[0] for m in moves], np.int64), dev)
    o = nat.upload(np.array([m[1] for m in moves], np.int32), dev)
    nw = nat.upload(np.array([m[2] for m in moves], np.int32), dev)
    u = nat.upload(np.stack([m[3] for m in moves]), dev, np.float64)
    nat.call("cgs_apply_splits", nat.ptr(book.rows), book.dim, nat.ptr(idx), nat.ptr(g), nat.ptr(o),
             nat.ptr(nw), nat.ptr(u), len(moves), nat.stream_handle(dev))
    book.mutations += 1
    state.touch(assignments=True)
    state.prefetch_host_index(which)


def apply_split(state: ModelState, proposal: SplitProposal) -> int:
    """sampler.py:202-209"""
    book, _ = _book_of(state, proposal.which)
    new_row = book.alloc_index(parent=proposal.row)
    book.decref(proposal.row)
    _apply_split_batch(state, proposal.which,
                       [(proposal.gaussian, proposal.row, new_row, np.asarray(proposal.u, np.float64))])
    return new_row


def accept_split(state: ModelState, proposal: SplitProposal, lam: float, config: SamplerConfig,
                 rng: np.random.Generator, extra_log_ratio: float = 0.0) -> bool:
    """sampler.py:212-221"""
    es, em = config.eps_for(proposal.which)
    prob = acceptance_probability("split", proposal.u, lam, es, em,
                                  config.normalization_correction, extra_log_ratio)
    if rng.random() < prob:
        apply_split(state, proposal)
        return True
    return False


_WARM = set()


def warm_host_paths(device) -> None:
    """Pay the one-time costs of the MCMC host path up front (once per device):
    numpy's lazily imported submodule behind np.unique and the lazily loaded
    CUDA module of the row gather, ~70 ms together on the first merge
    otherwise."""
    key = str(device)
    if key in _WARM:
        return
    import numpy.ma  # noqa: F401  (np.unique imports it on first use)
    np.unique(np.zeros(2, np.int64))
    if torch.device(device).type == "cuda":
        z = torch.zeros((2, 7), dtype=torch.float32, device=device)
        z.index_select(0, torch.zeros((1,), dtype=torch.int64, device=device)).cpu()
    _WARM.add(key)


def _rows_host(book, rows: np.ndarray) -> np.ndarray:
    if len(rows) == 0:
        return np.zeros((0, book.dim), np.float32)
    t = nat.upload(rows, book.device, np.int64)
    return book.rows.index_select(0, t).cpu().numpy()


class _RowCache:
    """Host copy of the codebook rows a merge step can touch (values are fixed within it)."""

    def __init__(self, book, pairs):
        self.idx = np.unique(pairs.reshape(-1)) if len(pairs) else np.zeros(0, np.int64)
        self.vals = _rows_host(book, self.idx)
        self.pos = {int(r): k for k, r in enumerate(self.idx)}

    def get(self, rows):
        return self.vals[[self.pos[int(r)] for r in rows]]


def _pick_merge(book, which, config, rng, cache: _RowCache) -> Optional[MergeProposal]:
    pairs = book.lineage_pairs()
    if len(pairs) == 0:
        return None
    _, eps_merge = config.eps_for(which)
    diffs = cache.get(pairs[:, 1]).astype(np.float64) - cache.get(pairs[:, 0]).astype(np.float64)
    log_w = -0.5 * np.einsum("nd,nd->n", diffs, diffs) / eps_merge ** 2
    w = np.exp(log_w - log_w.max())
    k = int(rng.choice(len(pairs), p=w / w.sum()))
    return MergeProposal(which=which, child=int(pairs[k, 0]), parent=int(pairs[k, 1]), u=diffs[k])


def propose_merge(state: ModelState, which: str, config: SamplerConfig,
                  rng: np.random.Generator) -> Optional[MergeProposal]:
    """sampler.py:224-237"""
    book, _ = _book_of(state, which)
    return _pick_merge(book, which, config, rng, _RowCache(book, book.lineage_pairs()))


def _merge_bookkeeping(book, child: int, parent: int):
    """Refcount effect of remapping every member of child to parent (sampler.py:244-247)."""
    members = int(book.refcount[child])
    book.refcount[parent] += members
    book.refcount[child] = 1
    book.decref(child)


def _apply_remap(state: ModelState, which: str, remap: dict):
    if not remap:
        return
    book, idx = _book_of(state, which)
    table = np.full(book.capacity, -1, np.int32)
    for c, p in remap.items():
        table[c] = p
    t = nat.upload(table, book.device)
    nat.call("cgs_apply_remap", nat.ptr(idx), state.num_gaussians, nat.ptr(t), len(table),
             nat.stream_handle(book.device))
    state.touch(assignments=True)
    state.prefetch_host_index(which)


def apply_merge(state: ModelState, proposal: MergeProposal) -> None:
    """sampler.py:240-247"""
    book, _ = _book_of(state, proposal.which)
    _merge_bookkeeping(book, proposal.child, proposal.parent)
    _apply_remap(state, proposal.which, {proposal.child: proposal.parent})


def accept_merge(state: ModelState, proposal: MergeProposal, lam: float, config: SamplerConfig,
                 rng: np.random.Generator, extra_log_ratio: float = 0.0) -> bool:
    """sampler.py:250-259"""
    es, em = config.eps_for(proposal.which)
    prob = acceptance_probability("merge", proposal.u, lam, es, em,
                                  config.normalization_correction, extra_log_ratio)
    if rng.random() < prob:
        apply_merge(state, proposal)
        return True
    return False


# ---------------------------------------------------------------------------
def _sgld_params(config: SamplerConfig, grad_scale: float, seed: int, offset: int,
                 source: int) -> nat.CSgldParams:
    p = nat.CSgldParams()
    p.step_pos, p.step_opacity = config.step_pos, config.step_opacity
    p.step_sh, p.step_sr = config.step_sh, config.step_sr
    p.noise_pos, p.noise_opacity = config.noise_pos, config.noise_opacity
    p.noise_sh, p.noise_sr = config.noise_sh, config.noise_sr
    p.grad_scale = grad_scale
    p.seed, p.offset = seed & (2 ** 64 - 1), offset & (2 ** 64 - 1)
    p.noise_source = source
    return p


def _host_noise(state: ModelState, config: SamplerConfig, rng, n_sh_live, n_sr_live):
    """The reference's noise draws, in group order (sampler.py:276-297)."""
    out = [None, None, None, None]
    specs = [(config.step_pos, config.noise_pos, (state.num_gaussians, 3)),
             (config.step_opacity, config.noise_opacity, (state.num_gaussians,)),
             (config.step_sh, config.noise_sh, (n_sh_live, state.sh.dim)),
             (config.step_sr, config.noise_sr, (n_sr_live, 7))]
    dev = state.device
    for k, (eps, mult, shape) in enumerate(specs):
        if eps > 0.0 and mult != 0.0:
            out[k] = torch.as_tensor(rng.standard_normal(shape)).to(dev)
    return out


def sgld_update(state: ModelState, grads: GradientSet, config: SamplerConfig,
                rng: np.random.Generator, flags: torch.Tensor = None, check: bool = True,
                offset_dev: torch.Tensor = None, skip_if: torch.Tensor = None,
                sticky: torch.Tensor = None, grads_nonfinite: torch.Tensor = None) -> None:
    """SGLD step per group (sampler.py:262-300) on the device.

    ``offset_dev`` (int64 device counter) makes device-noise draws advance on
    the device, so a captured CUDA graph of the update draws fresh noise on
    every replay.  ``skip_if`` (device int32, e.g. the frame's overflow flag)
    makes the update write nothing when set; ``sticky`` (device int32)
    accumulates the flags (1 non-finite, 2 skipped) for a check at the end;
    ``grads_nonfinite`` (the backward's flag, render.Frame.backward) replaces
    the update's own finiteness pass over the gradients."""
    noise = _draw_noise(state, config, rng)
    _sgld_launch(state, grads, config, noise, flags if flags is not None else None, offset_dev,
                 skip_if, sticky, check, grads_nonfinite)


def _draw_noise(state: ModelState, config: SamplerConfig, rng) -> list:
    """Parity mode: the reference's host draws for this update (None in
    device-noise mode, where the kernel draws Philox normals)."""
    if config.device_noise:
        return [None] * 4
    return _host_noise(state, config, rng, state.sh.device_live().numel(),
                       state.sr.device_live().numel())


def _sgld_launch(state: ModelState, grads: GradientSet, config: SamplerConfig, noise: list,
                 flags, offset_dev, skip_if, sticky, check: bool,
                 grads_nonfinite=None) -> None:
    dev = state.device
    g = state.gaussians
    sh_live = state.sh.device_live()
    sr_live = state.sr.device_live()
    if config.device_noise:
        params = _sgld_params(config, 1.0, config.seed, state.iteration, 0)
        params.offset_dev = nat.ptr(offset_dev)
    else:
        params = _sgld_params(config, 1.0, 0, 0, 1)
    params.skip_if = nat.ptr(skip_if)
    params.sticky = nat.ptr(sticky)
    params.grads_nonfinite = nat.ptr(grads_nonfinite)
    if flags is None:
        flags = torch.zeros((1,), dtype=torch.int32, device=dev)
    nat.call("cgs_sgld_update", nat.ptr(g.positions), nat.ptr(g.opacity_logits), g.count,
             nat.ptr(state.sh.rows), state.sh.dim, nat.ptr(sh_live), sh_live.numel(),
             nat.ptr(state.sr.rows), nat.ptr(sr_live), sr_live.numel(), state.sh.capacity,
             state.sr.capacity, nat.ptr(grads.positions), nat.ptr(grads.opacity_logits),
             nat.ptr(grads.sh_rows), nat.ptr(grads.sr_rows), ctypes.byref(params),
             nat.ptr(noise[0]), nat.ptr(noise[1]), nat.ptr(noise[2]), nat.ptr(noise[3]),
             nat.ptr(flags), nat.stream_handle(dev))
    state.touch()
    state.sh.mutations += 1
    state.sr.mutations += 1
    if check:
        f = int(flags[0].item())
        if f & 1:
            raise SamplerError(f"non-finite gradients at iteration {state.iteration}")
        if f & 2:
            raise RuntimeError("update skipped: the frame overflowed its pair capacity")


def _candidate_count(fraction: float, population: int) -> int:
    """sampler.py:303-306"""
    if population <= 0:
        return 0
    return max(1, int(round(fraction * population)))


def _exact_log_ratio(state, views, config, rng, trial):
    """log p(S')/p(S) from one rendered view by trial-applying the move
    (sampler.py:309-317).  The reference deep-copies the state per candidate;
    here the move is applied to the device arrays only, rendered and
    reverted (``trial`` is a context manager: _split_trial / _merge_trial),
    and the "before" loss is reused while the state and view are unchanged."""
    from .metrics import recon_loss
    cam, gt = views[int(rng.integers(len(views)))]
    cache = state.__dict__.setdefault("_exact_before", {})
    key = (state.token(), cam.key(), id(gt), config.lambda_ssim)
    before = cache.get(key)
    if before is None:
        before = recon_loss(rasterize_forward(state, cam).image, gt, config.lambda_ssim)[2]
        cache.clear()
        cache[key] = before
    with trial:
        after = recon_loss(rasterize_forward(state, cam).image, gt, config.lambda_ssim)[2]
    # the reverted state renders as before (only its version counters moved)
    cache.clear()
    cache[(state.token(), cam.key(), id(gt), config.lambda_ssim)] = before
    return before - after


class _split_trial:
    """Gaussian i on a new row of value f32(f64(row) + u) (apply_split,
    sampler.py:202-209) for one render: the value goes to the spare row past
    the codebook's capacity, g2sh/g2sr[i] points at it; all reverted on exit
    (no host bookkeeping is touched)."""

    def __init__(self, state, which, i, row, u):
        self.state, self.which, self.i, self.row = state, which, int(i), int(row)
        self.u = np.asarray(u, np.float64)

    def __enter__(self):
        from .model import _grow
        book, idx = _book_of(self.state, self.which)
        r = book.capacity
        book._buf = _grow(book._buf, r + 1)
        uu = torch.as_tensor(self.u, dtype=torch.float64, device=book.device)
        book._buf[r] = (book._buf[self.row].double() + uu).float()
        self.old = idx[self.i].clone()
        idx[self.i] = r
        book._cap += 1  # the render sees the spare row (rows / capacity)
        self.state.touch(assignments=True)
        book.mutations += 1
        return self

    def __exit__(self, *exc):
        book, idx = _book_of(self.state, self.which)
        idx[self.i] = self.old
        book._cap -= 1
        self.state.touch(assignments=True)
        book.mutations += 1
        return False


class _merge_trial:
    """Every Gaussian on `child` on `parent` instead (apply_merge,
    sampler.py:240-247) for one render; reverted on exit."""

    def __init__(self, state, which, child, parent):
        self.state, self.which = state, which
        self.child, self.parent = int(child), int(parent)

    def __enter__(self):
        _, idx = _book_of(self.state, self.which)
        self.members = idx == self.child
        idx.masked_fill_(self.members, self.parent)
        self.state.touch(assignments=True)
        return self

    def __exit__(self, *exc):
        _, idx = _book_of(self.state, self.which)
        idx.masked_fill_(self.members, self.child)
        self.state.touch(assignments=True)
        return False


def clone_state(state: ModelState) -> ModelState:
    """Deep copy (device arrays cloned, host mirrors copied)."""
    h = state.to_host()
    st = ModelState.from_arrays(h["positions"], h["opacity_logits"], h["g2sh"], h["g2sr"],
                                h["sh_rows"], h["sr_rows"], h["sh_refcount"], h["sr_refcount"],
                                h["sh_parent"], h["sr_parent"], device=state.device,
                                iteration=state.iteration, rng_seed=state.rng_seed)
    for src, dst in ((state.sh, st.sh), (state.sr, st.sr)):
        dst._free = list(src._free)
        dst._live_version += 1
    return st


def split_step(state: ModelState, views, config: SamplerConfig, rng, rec: TransitionRecord):
    """Split branch of train_step (sampler.py:339-364): eligibility and the accept
    loop on the host mirrors (assignments, refcounts) with the caller's
    Generator, then one batched device apply -- no device synchronisation."""
    which = "sh" if rng.random() < 0.5 else "sr"
    rec.codebook = which
    book, _ = _book_of(state, which)
    n = state.num_gaussians
    # eligible = Gaussians whose row is shared (sampler.py:344), from the host
    # mirrors of the assignments and refcounts: no device round trip
    hidx = state.host_index(which)
    elig = _eligible(hidx, book.refcount)
    n_elig = len(elig)
    n_cand = min(_candidate_count(config.split_fraction, n), n_elig)
    if n_cand <= 0:
        return
    # rng.choice(eligible, ...) == eligible[rng.choice(len(eligible), ...)]
    cand = elig[rng.choice(n_elig, size=n_cand, replace=False)]
    rows = hidx[cand]
    lam = config.lambda_for(which)
    es, em = config.eps_for(which)
    if not config.exact_ratio:
        if config.device_noise and book.device.type == "cuda":
            _split_device(state, which, book, cand, rows, config, rec, lam, es, em)
            return
        moves = _split_loop_native(book, cand, rows, config, rng, rec, lam, es, em)
        if moves is not None:
            _apply_split_batch(state, which, moves)
            return
    moves = []
    # The sequential accept loop is the host's only per-candidate work; the
    # acceptance arithmetic is inlined with exactly the float expressions of
    # acceptance_probability / _log_q_sm (sampler.py:138-164).
    dim = book.dim
    c_q = 1.0 / es ** 2 - 1.0 / em ** 2
    corr = dim * math.log(em / es) if config.normalization_correction else None
    refcount = book.refcount
    normal, uniform, npexp = rng.normal, rng.random, np.exp
    probs = rec.accept_probs
    for i, row in zip(cand.tolist(), rows.tolist()):
        if refcount[row] < 2:
            continue
        u = normal(0.0, es, size=dim)
        extra = 0.0
        if config.exact_ratio:
            # flush pending applies so the trial render sees the current state
            _apply_split_batch(state, which, moves)
            moves = []
            extra = _exact_log_ratio(state, views, config, rng, _split_trial(state, which, i, row, u))
        log_q = -0.5 * float(u @ u) * c_q
        if corr is not None:
            log_q += corr
        prob = float(npexp(min(0.0, -lam - log_q + extra)))
        probs.append(prob)
        rec.attempts += 1
        if uniform() < prob:
            new_row = book.alloc_index(parent=row)
            book.decref(row)
            refcount = book.refcount  # alloc may have grown the array
            moves.append((i, row, new_row, u))
            rec.accepts += 1
    _apply_split_batch(state, which, moves)


def settle_split(rows: np.ndarray, accept: np.ndarray, refcount: np.ndarray):
    """The reference loop's refcount skips (sampler.py:349-364) for candidates
    whose accept coins are already drawn: candidate c is tried iff its row's
    refcount, lowered by the accepts of the earlier candidates of that row, is
    still >= 2; it is executed iff tried and accepted.  Vectorised: counting
    the raw accept flags of earlier same-row candidates is exact, since once a
    row reaches refcount 1 all its later candidates are skipped anyway.
    Returns (tried, executed) boolean arrays in candidate order."""
    rows = np.asarray(rows, dtype=np.int64)
    acc = np.asarray(accept, dtype=bool)
    n = len(rows)
    if n == 0:
        return np.zeros(0, bool), np.zeros(0, bool)
    order = np.argsort(rows, kind="stable")
    r_sorted, a_sorted = rows[order], acc[order].astype(np.int64)
    cum = np.cumsum(a_sorted) - a_sorted
    starts = np.flatnonzero(np.r_[True, r_sorted[1:] != r_sorted[:-1]])
    before = cum - np.repeat(cum[starts], np.diff(np.r_[starts, n]))
    tried = np.empty(n, dtype=bool)
    tried[order] = before < np.asarray(refcount)[r_sorted] - 1
    return tried, tried & acc


def _split_device(state: ModelState, which: str, book, cand, rows, config: SamplerConfig,
                  rec: TransitionRecord, lam: float, es: float, em: float) -> None:
    """Throughput (device-noise) mode: the split proposals and coins of all
    candidates drawn on the device at once (cgs_split_propose, Philox keyed by
    (seed, iteration, candidate)) instead of one numpy draw after another;
    the refcount skips of the reference loop (sampler.py:350-351) are then
    settled on the host in candidate order: a row's candidates are tried while
    its refcount is >= 2, and each accepted one lowers it.  Same proposal
    distribution and acceptance rule as the reference; a different random
    stream (like the device SGLD noise)."""
    n_cand, dim = len(cand), book.dim
    dev = book.device
    u = torch.empty((n_cand, dim), dtype=torch.float64, device=dev)
    prob = torch.empty((n_cand,), dtype=torch.float64, device=dev)
    acc = torch.empty((n_cand,), dtype=torch.int8, device=dev)
    c_q = 1.0 / es ** 2 - 1.0 / em ** 2
    use_corr = 1 if config.normalization_correction else 0
    corr = dim * math.log(em / es) if use_corr else 0.0
    ctr = (int(state.iteration) << 1) | (0 if which == "sh" else 1)
    nat.call("cgs_split_propose", n_cand, dim, float(es), float(c_q), use_corr, float(corr),
             float(lam), int(config.seed) & 0xFFFFFFFFFFFFFFFF, ctr, nat.ptr(u), nat.ptr(prob),
             nat.ptr(acc), nat.stream_handle(dev))
    acc_h = acc.cpu().numpy().astype(bool)
    prob_h = prob.cpu().numpy()
    rows64 = np.ascontiguousarray(rows, dtype=np.int64)
    tried, dec = settle_split(rows64, acc_h, book.refcount)
    rec.accept_probs.extend(prob_h[tried].tolist())
    rec.attempts += int(tried.sum())
    take = np.flatnonzero(dec)
    if len(take) == 0:
        return
    new_rows = np.empty(len(take), dtype=np.int32)
    for j, c in enumerate(take.tolist()):
        row = int(rows64[c])
        rc = book.refcount
        rc[row] -= 1  # decref of the old row (it stays >= 1)
        new_rows[j] = book.alloc_index(parent=row)  # lowest free row
        book.mutations += 1
        rec.accepts += 1
    _, idx = _book_of(state, which)
    g = nat.upload(np.asarray(cand, np.int64)[take], dev)
    o = nat.upload(rows64[take].astype(np.int32), dev)
    nw = nat.upload(new_rows, dev)
    ut = u.index_select(0, nat.upload(take.astype(np.int64), dev)).contiguous()
    nat.call("cgs_apply_splits", nat.ptr(book.rows), book.dim, nat.ptr(idx), nat.ptr(g), nat.ptr(o),
             nat.ptr(nw), nat.ptr(ut), len(take), nat.stream_handle(dev))
    book.mutations += 1
    state.touch(assignments=True)
    state.prefetch_host_index(which)


def _eligible(hidx: np.ndarray, refcount: np.ndarray) -> np.ndarray:
    """np.flatnonzero(refcount[hidx] >= 2) (sampler.py:344), by the library's
    threaded host scan."""
    import os
    n = len(hidx)
    out = np.empty(max(n, 1), dtype=np.int32)
    cnt = nat.I64(0)
    h = np.ascontiguousarray(hidx, dtype=np.int32)
    rc = np.ascontiguousarray(refcount, dtype=np.int64)
    nat.call("cgs_host_split_eligible", h.ctypes.data, n, rc.ctypes.data, len(rc), out.ctypes.data,
             ctypes.byref(cnt), min(16, os.cpu_count() or 1))
    return out[: cnt.value]


def _split_loop_native(book, cand, rows, config: SamplerConfig, rng, rec: TransitionRecord,
                       lam: float, es: float, em: float):
    """The split accept loop (sampler.py:349-364) in the library
    (cgs_host_split_decide) on the caller's Generator stream; returns the
    accepted moves, or None (nothing consumed) when the native path is
    unavailable or its exp-based decisions disagree with numpy's exp (then
    the Generator and refcounts are restored and the Python loop runs)."""
    ddot = nat.numpy_ddot_ptr()
    rc = book.refcount
    if ddot is None or rc.dtype != np.int64 or not rc.flags.c_contiguous:
        return None
    n_cand, dim = len(cand), book.dim
    rows64 = np.ascontiguousarray(rows, dtype=np.int64)
    saved_state = rng.bit_generator.state
    saved_rc = rc[rows64].copy()
    u = np.empty((n_cand, dim), dtype=np.float64)
    log_a = np.empty(n_cand, dtype=np.float64)
    coin = np.empty(n_cand, dtype=np.float64)
    dec = np.empty(n_cand, dtype=np.int8)
    att = nat.I64(0)
    c_q = 1.0 / es ** 2 - 1.0 / em ** 2
    use_corr = 1 if config.normalization_correction else 0
    corr = dim * math.log(em / es) if use_corr else 0.0
    nat.call("cgs_host_split_decide", nat.bitgen_ptr(rng), ddot, n_cand, rows64.ctypes.data,
             rc.ctypes.data, len(rc), dim, float(lam), float(es), float(c_q), use_corr, float(corr),
             u.ctypes.data, log_a.ctypes.data, coin.ctypes.data, dec.ctypes.data, ctypes.byref(att))
    tried = dec >= 0
    probs = np.exp(np.minimum(0.0, log_a[tried]))  # numpy's exp, as acceptance_probability
    if not np.array_equal(coin[tried] < probs, dec[tried] == 1):
        rc[rows64] = saved_rc
        rng.bit_generator.state = saved_state
        return None
    rec.accept_probs.extend(probs.tolist())
    rec.attempts += int(att.value)
    moves = []
    for c in np.flatnonzero(dec == 1).tolist():
        row = int(rows64[c])
        new_row = book.alloc_index(parent=row)  # lowest free row (the old row's decref is done)
        book.mutations += 1
        moves.append((int(cand[c]), row, new_row, u[c]))
        rec.accepts += 1
    return moves


def merge_step(state: ModelState, views, config: SamplerConfig, rng, rec: TransitionRecord):
    """Merge branch of train_step (sampler.py:365-385)."""
    which = "sh" if rng.random() < 0.5 else "sr"
    rec.codebook = which
    book, _ = _book_of(state, which)
    lam = config.lambda_for(which)
    pairs0 = book.lineage_pairs()
    n_cand = _candidate_count(config.split_fraction, len(pairs0))
    cache = _RowCache(book, pairs0)
    remap: dict = {}
    es, em = config.eps_for(which)
    for _ in range(n_cand):
        prop = _pick_merge(book, which, config, rng, cache)
        if prop is None:
            break
        extra = 0.0
        if config.exact_ratio:
            _apply_remap(state, which, remap)
            remap = {}
            extra = _exact_log_ratio(state, views, config, rng,
                                     _merge_trial(state, which, prop.child, prop.parent))
        prob = acceptance_probability("merge", prop.u, lam, es, em, config.normalization_correction,
                                      extra)
        rec.accept_probs.append(prob)
        rec.attempts += 1
        if rng.random() < prob:
            _merge_bookkeeping(book, prop.child, prop.parent)
            for c in list(remap):
                if remap[c] == prop.child:
                    remap[c] = prop.parent
            remap[prop.child] = prop.parent
            rec.accepts += 1
    _apply_remap(state, which, remap)


class _StepEngine:
    """Buffers of the drop-in update path, cached on the state per camera
    batch shape: frame / backward / gradient workspaces sized for the current
    Gaussian count and codebook capacities, the loss workspace, a pinned
    staging buffer for the host target image, and the pair capacity (probed
    once, then scaled with N).  An update then needs one host synchronisation
    (reading the recon loss and the flags together)."""

    def __init__(self, state: ModelState, cams):
        self.dev = state.device
        self.shape = tuple((c.width, c.height) for c in cams)
        v, h, w = len(cams), cams[0].height, cams[0].width
        self.loss = LossWorkspace(v, h, w, self.dev)
        self.dL = None
        self.flags = torch.zeros((1,), dtype=torch.int32, device=self.dev)
        self.host = torch.zeros((2,), dtype=torch.float64).pin_memory()
        self.gt_stage = None
        self.gt_dev = None
        self.pair_cap = None
        self.pairs_per_gaussian = None
        self.key = None
        self.frames = {}

    def prepare(self, state: ModelState, cams):
        if self.pairs_per_gaussian is None:
            probe = Frame(state, cams).run_checked()
            self.pairs_per_gaussian = probe.stats().n_pairs / max(state.num_gaussians, 1)
        cap = int(self.pairs_per_gaussian * state.num_gaussians * 1.5) + 4096
        self.pair_cap = max(self.pair_cap or 0, cap)
        key = (state.num_gaussians, state.sh.capacity, state.sr.capacity, self.pair_cap)
        if key != self.key:
            self.key = key
            self.frames = {}
            self.frame_ws = None
            self.bws = None
            self.grads = GradientSet.empty(state)
        ck = tuple(c.key() for c in cams)
        fr = self.frames.get(ck)
        if fr is None:
            fr = Frame(state, cams, pair_capacity=self.pair_cap, ws=self.frame_ws)
            self.frame_ws = fr.ws
            if len(self.frames) > 64:
                self.frames = {}
            self.frames[ck] = fr
        if self.dL is None or self.dL.shape != fr.image.shape:
            self.dL = torch.empty_like(fr.image)
        nb = backward_workspace_bytes(state, fr)
        if self.bws is None or self.bws.numel() < nb:
            self.bws = torch.empty((nb,), dtype=torch.uint8, device=self.dev)
        return fr

    def grow(self, state: ModelState, fr: Frame):
        """The frame overflowed: size the pairs from its count and start over."""
        n_pairs = fr.stats().n_pairs
        self.pair_cap = max(self.pair_cap, int(n_pairs * 1.25) + 1024)
        self.pairs_per_gaussian = max(self.pairs_per_gaussian, n_pairs / max(state.num_gaussians, 1))
        self.key = None

    def target(self, gt) -> torch.Tensor:
        """The step's target image on the device (uploaded every call, through a
        pinned staging buffer: a caller may edit or replace its arrays)."""
        if isinstance(gt, torch.Tensor) and gt.is_cuda:
            return gt.to(torch.float32).contiguous()
        a = np.asarray(gt)
        if self.gt_stage is None or tuple(self.gt_stage.shape) != a.shape:
            self.gt_stage = torch.empty(a.shape, dtype=torch.float32).pin_memory()
            self.gt_dev = torch.empty(a.shape, dtype=torch.float32, device=self.dev)
        np.copyto(self.gt_stage.numpy(), a, casting="unsafe")
        self.gt_dev.copy_(self.gt_stage, non_blocking=True)
        return self.gt_dev


def _engine(state: ModelState, cams) -> _StepEngine:
    cache = state.__dict__.setdefault("_step_engines", {})
    key = tuple((c.width, c.height) for c in cams)
    eng = cache.get(key)
    if eng is None:
        eng = cache[key] = _StepEngine(state, cams)
    return eng


def update_step(state: ModelState, cams, gts, config: SamplerConfig, rng, check: bool = True):
    """Batched SGLD update over views (mean of per-view gradients; reduces to the
    reference's single-view update when len(cams) == 1).  Returns the recon
    loss (mean over views) as a float; one host synchronisation, which also
    reads the update's flags.  A frame that overflowed its pair capacity
    skips the update on the device; it is then re-run with the same noise."""
    v = len(cams)
    h, w = cams[0].height, cams[0].width
    if any((c.height, c.width) != (h, w) for c in cams):
        raise ValueError("a batched update needs equal image sizes")
    eng = _engine(state, cams)
    gt_d = eng.target(gts)
    if tuple(gt_d.shape[-3:]) != (h, w, 3):
        raise ValueError("ground-truth image shape mismatch")
    state.code_csr("sh")
    state.code_csr("sr")
    noise = _draw_noise(state, config, rng)
    for _ in range(3):
        fr = eng.prepare(state, cams)
        fr.run()
        losses = eng.loss.run(fr.image, gt_d, config.lambda_ssim, eng.dL, 1.0)
        fr.backward(eng.dL, scale=1.0 / v, grads=eng.grads, ws=eng.bws)
        ov = fr.ws[40:44].view(torch.int32)  # cgs_frame_stats_t.overflow
        _sgld_launch(state, eng.grads, config, noise, eng.flags, None, ov, None, False,
                     eng.bws[16:20].view(torch.int32))  # the backward's non-finite flag
        eng.host[0].copy_(losses.view(v, 3)[:, 2].mean(), non_blocking=True)
        eng.host[1].copy_(eng.flags[0], non_blocking=True)
        torch.cuda.current_stream(state.device).synchronize()
        f = int(eng.host[1].item())
        if f & 2:  # overflow: nothing was written; grow and redo
            eng.grow(state, fr)
            continue
        if f & 1 and check:
            raise SamplerError(f"non-finite gradients at iteration {state.iteration}")
        if fr.stats().zero_quaternion:
            raise ValueError("zero quaternion")
        return float(eng.host[0].item())
    raise RuntimeError("pair capacity overflow persisted")


def train_step(state: ModelState, views: list, config: SamplerConfig,
               rng: np.random.Generator) -> TransitionRecord:
    """One MH transition plus the densification schedule (sampler.py:320-399)."""
    if not views:
        raise ValueError("at least one view is required")
    kind = choose_transition(config, rng)
    sh_before, sr_before = state.sh.live_count, state.sr.live_count
    rec = TransitionRecord(iteration=state.iteration + 1, kind=kind, codebook="-",
                           lambdas=(config.lambda_sh, config.lambda_sr))
    if kind == "update":
        cam, gt = views[int(rng.integers(len(views)))]
        rec.recon = update_step(state, [cam], gt, config, rng)
        rec.attempts, rec.accepts = 1, 1
        rec.accept_probs.append(1.0)
    elif kind == "split":
        split_step(state, views, config, rng, rec)
    else:
        merge_step(state, views, config, rng, rec)
    state.iteration += 1
    if config.densify_every > 0 and state.iteration % config.densify_every == 0:
        densify(state, config.densify_growth, config.gaussian_cap, rng,
                jitter_sigma=config.densify_jitter)
    rec.live_sh = state.sh.live_count
    rec.live_sr = state.sr.live_count
    rec.delta_sh = rec.live_sh - sh_before
    rec.delta_sr = rec.live_sr - sr_before
    return rec


def train(state: ModelState, views: list, config: SamplerConfig, iters: int,
          rng: Optional[np.random.Generator] = None, eval_every: int = 0,
          eval_views: Optional[list] = None, check_invariants: bool = False) -> list:
    """sampler.py:402-420"""
    from .metrics import psnr as psnr_fn
    if rng is None:
        rng = np.random.default_rng(config.seed)
    warm_host_paths(state.device)
    records = []
    for _ in range(iters):
        rec = train_step(state, views, config, rng)
        if check_invariants:
            validate_state(state)
        if eval_every > 0 and state.iteration % eval_every == 0:
            targets = eval_views if eval_views else views
            vals = [psnr_fn(rasterize_forward(state, cam).image, gt) for cam, gt in targets]
            rec.psnr = float(np.mean(vals))
        records.append(rec)
    return records
