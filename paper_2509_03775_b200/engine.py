"""Batched, device-resident training loop (the bench's "step").

One iteration = one SGLD update transition over a batch of views rendered as
one frame (mean of per-view gradients -- the batch extension of
`sampler.py:329-338`; with one view it is exactly the reference update),
followed, on the schedule, by one forced split and one forced merge
transition (`sampler.py:339-385`) and densify when due (`sampler.py:387-390`).

No host synchronisation inside an update: the frame's pair buffers are sized
from a warm-up render (pairs per Gaussian x the current N x headroom, so they
grow with densify); an overflowing frame makes the SGLD kernels skip the
update (no state change), as non-finite gradients do, and both latch a sticky
device flag that is checked when the caller reads results.  Across GPUs, views are
sharded by rank and the flat gradient buffer is summed by NCCL allreduce
(``torch.distributed``; the per-Gaussian part on a side stream overlapping the
codebook reduce, the codebook part after it); MCMC decisions use the same host
Generator seed on every rank, so replicas stay identical with no broadcast.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as nat
from .metrics import LossWorkspace
from .model import ModelState, densify, densify_prepare
from .render import Frame, GradientSet, backward_workspace_bytes
from .sampler import (SamplerConfig, SamplerError, TransitionRecord, merge_step, sgld_update,
                      split_step)


def _host_noise_groups(config: SamplerConfig) -> bool:
    """Whether the reference's update draws noise (sampler.py:276-297)."""
    return any(eps > 0.0 and mult != 0.0 for eps, mult in (
        (config.step_pos, config.noise_pos), (config.step_opacity, config.noise_opacity),
        (config.step_sh, config.noise_sh), (config.step_sr, config.noise_sr)))


class Trainer:
    def __init__(self, state: ModelState, cams, gts: torch.Tensor, config: SamplerConfig,
                 rng: np.random.Generator, mcmc_every: int = 25, world: int = 1,
                 pair_headroom: float = 1.5, allreduce=None, use_graphs: bool = False,
                 total_views: int = None):
        if use_graphs and not config.device_noise and _host_noise_groups(config):
            # a captured graph would replay the noise drawn once at capture
            raise ValueError("use_graphs needs config.device_noise=True when the SGLD update draws "
                             "noise (host-drawn noise cannot be replayed from a CUDA graph)")
        self.state = state
        self.cams = list(cams)
        self.config = config
        self.rng = rng
        self.mcmc_every = mcmc_every
        self.world = world
        self.allreduce = allreduce
        self._ar_stream = None
        from .sampler import warm_host_paths
        warm_host_paths(state.device)
        self.headroom = pair_headroom
        h, w = self.cams[0].height, self.cams[0].width
        if any((c.height, c.width) != (h, w) for c in self.cams):
            raise ValueError("batched views need equal sizes")
        self.V = len(self.cams)
        # gradients are summed over every view of the step on every rank, then
        # divided by their total: the mean even when shards are unequal
        self.total_views = total_views if total_views is not None else self.V * world
        if self.total_views < self.V:
            raise ValueError("total_views must count every rank's views")
        self.dev = state.device
        self.gts = gts
        self.loss_ws = LossWorkspace(self.V, h, w, self.dev)
        self.flags = torch.zeros((1,), dtype=torch.int32, device=self.dev)
        self.sticky = torch.zeros((1,), dtype=torch.int32, device=self.dev)
        self.frame = None
        self.grads = None
        self.bws = None
        self.dL = None
        self.pair_cap = None
        self._pairs_per_gaussian = None
        self.updates = 0
        self.mcmc_events = 0
        self.mcmc_ms = []
        self.densify_ms = []
        self.reassign_ms = []
        self.reassigned = {"sh": 0, "sr": 0}
        self.capture_ms = []
        self.last_loss = None
        self.use_graphs = use_graphs
        self.noise_ctr = torch.zeros((1,), dtype=torch.int64, device=self.dev)
        self._gkey = None
        self._g_fwd = self._g_sgld = None
        # kernel accounting: the C ABI counts every launch call, including the
        # ones recorded while capturing (not executed); replays execute the
        # recorded kernels without calling the ABI
        self._g_kernels = {}
        self.capture_counted = 0
        self.replayed_kernels = 0
        self._pool = None
        self._cap_stream = None
        self.captures = 0
        state.prefetch_host_index()  # the MCMC loop reads the assignments from the host
        if config.densify_every > 0 and config.device_noise:  # its buffers outside any timed window
            ncap = max(state.gaussians.capacity, state.num_gaussians)
            densify_prepare(state, ncap, int(config.densify_growth * ncap) + 1)

    # -- buffers ---------------------------------------------------------------
    def _capacity_buffers(self):
        """Frame, backward and gradient buffers sized for the Gaussian capacity
        (densify grows N inside it without a reallocation; only the graphs are
        re-captured)."""
        st = self.state
        lib = nat.library()
        ncap = max(st.gaussians.capacity, st.num_gaussians)
        key = (ncap, st.sh.capacity, st.sr.capacity, self.pair_cap)
        if getattr(self, "_cap_key", None) == key:
            return
        cams = nat.cams_array(self.cams)
        fb = lib.cgs_frame_workspace_bytes(ncap, cams, self.V, self.pair_cap, st.sr.capacity)
        bb = lib.cgs_backward_workspace_bytes(ncap, cams, self.V, self.pair_cap, st.sh.capacity,
                                              st.sr.capacity)
        self._frame_ws = torch.empty((fb,), dtype=torch.uint8, device=self.dev)
        self.bws = torch.empty((bb,), dtype=torch.uint8, device=self.dev)
        self._grad_buf = torch.empty((4 * ncap + st.sh.capacity * st.sh.dim + 7 * st.sr.capacity,),
                                     dtype=torch.float32, device=self.dev)
        self._cap_key = key

    def _prepare(self):
        st = self.state
        fr = self.frame
        if fr is None or fr.n != st.num_gaussians or fr.sr_cap != st.sr.capacity:
            if self._pairs_per_gaussian is None:
                probe = Frame(st, self.cams).run_checked()
                self._pairs_per_gaussian = probe.stats().n_pairs / max(st.num_gaussians, 1)
            # pairs grow with N (densify): sized for the Gaussian capacity, so
            # densify inside it keeps every buffer (a GB-scale reallocation
            # costs tens of milliseconds); never shrinks
            ncap = max(st.gaussians.capacity, st.num_gaussians)
            cap = int(self._pairs_per_gaussian * ncap * self.headroom) + 4096
            self.pair_cap = max(self.pair_cap or 0, cap)
            self._capacity_buffers()
            self.frame = Frame(st, self.cams, pair_capacity=self.pair_cap, ws=self._frame_ws)
            if self.dL is None or self.dL.shape != self.frame.image.shape:
                self.dL = torch.empty_like(self.frame.image)
        nb = backward_workspace_bytes(st, self.frame)
        if self.bws is None or self.bws.numel() < nb:
            self.bws = torch.empty((nb,), dtype=torch.uint8, device=self.dev)
        g = self.grads
        if (g is None or g.positions.shape[0] != st.num_gaussians
                or g.sh_rows.shape[0] != st.sh.capacity or g.sr_rows.shape[0] != st.sr.capacity):
            self._capacity_buffers()
            self.grads = GradientSet.empty(st, self._grad_buf)

    # -- transitions -------------------------------------------------------------
    # The update is enqueued in three parts: forward + loss, backward, SGLD.
    # With graphs on, the forward and SGLD parts are replayed from CUDA graphs
    # (re-captured whenever a buffer address or size they baked in changes);
    # the backward stays an eager C-ABI call so the profiled raster kernel
    # is bracketed by live CUDA events on its launch stream.
    def _enqueue_forward(self):
        fr = self.frame
        fr.run()
        self.loss_ws.run(fr.image, self.gts, self.config.lambda_ssim, self.dL, 1.0)

    def _enqueue_backward(self):
        scale = 1.0 / self.total_views
        if self.allreduce is None:
            self.frame.backward(self.dL, scale=scale, grads=self.grads, ws=self.bws)
            return
        # two allreduces: [d_pos | d_logit] on a side stream as soon as the
        # per-Gaussian gradients are written, overlapping the codebook
        # reduce kernels; [d_SH | d_SR] after them.  Element-wise sums, so the
        # result equals one allreduce of the flat buffer.
        cur = torch.cuda.current_stream(self.dev)
        if self._ar_stream is None:
            self._ar_stream = torch.cuda.Stream(self.dev)
        ar = self._ar_stream

        def head(g):
            ar.wait_stream(cur)
            with torch.cuda.stream(ar):
                self.allreduce(g.flat[: 4 * g.opacity_logits.numel()])

        g = self.frame.backward(self.dL, scale=scale, grads=self.grads, ws=self.bws,
                                after_gaussians=head)
        self.allreduce(g.flat[4 * g.opacity_logits.numel():])
        cur.wait_stream(ar)

    def _enqueue_sgld(self):
        # cgs_frame_stats_t.overflow (byte 40 of the frame workspace): an
        # overflowing frame skips the update; flags latch into self.sticky
        ov = self.frame.ws[40:44].view(torch.int32)
        # one rank: the backward's own non-finite flag covers the gradients
        # (cgs_backward_nonfinite_flag, byte 16); after an allreduce a rank's
        # flag does not see the other ranks' values, so the update checks
        nf = self.bws[16:20].view(torch.int32) if self.allreduce is None else None
        sgld_update(self.state, self.grads, self.config, self.rng, flags=self.flags, check=False,
                    offset_dev=self.noise_ctr, skip_if=ov, sticky=self.sticky,
                    grads_nonfinite=nf)

    def _graph_key(self):
        st = self.state
        g = st.gaussians
        sl, rl = st.sh.device_live(), st.sr.device_live()
        return (id(self.frame), id(self.grads), self.bws.data_ptr(), g.positions.data_ptr(), g.count,
                g.g2sh.data_ptr(), g.g2sr.data_ptr(), st.sh.rows.data_ptr(), st.sr.rows.data_ptr(),
                st.sh.capacity, st.sr.capacity, sl.data_ptr(), sl.numel(), rl.data_ptr(), rl.numel())

    def _capture(self, fn):
        """Capture fn into a CUDA graph on a side stream.  Unlike the
        ``torch.cuda.graph`` context this skips the device synchronisation,
        ``gc.collect()`` and ``empty_cache()`` (the latter forces fresh
        cudaMallocs afterwards); all graphs share one memory pool."""
        if self._pool is None:
            self._pool = torch.cuda.graph_pool_handle()
            self._cap_stream = torch.cuda.Stream(self.dev)
        g = torch.cuda.CUDAGraph()
        c0 = nat.library().cgs_launch_count()
        cur = torch.cuda.current_stream(self.dev)
        self._cap_stream.wait_stream(cur)
        with torch.cuda.stream(self._cap_stream):
            g.capture_begin(pool=self._pool)
            try:
                fn()
            finally:
                g.capture_end()
        cur.wait_stream(self._cap_stream)
        k = int(nat.library().cgs_launch_count() - c0)
        self.capture_counted += k
        self._g_kernels[id(g)] = k
        return g

    def _replay(self, g):
        g.replay()
        self.replayed_kernels += self._g_kernels.get(id(g), 0)

    def update(self):
        """SGLD update over the view batch (device only, no host synchronisation)."""
        self._prepare()
        self.state.code_csr("sh")
        self.state.code_csr("sr")
        if self.use_graphs:
            key = self._graph_key()
            if key != self._gkey:
                import time
                t0 = time.perf_counter()
                self._enqueue_forward()
                self._enqueue_backward()
                self._enqueue_sgld()
                self._g_fwd = self._capture(self._enqueue_forward)
                self._g_sgld = self._capture(self._enqueue_sgld)
                self._gkey = key
                self.captures += 1
                self.capture_ms.append(1000.0 * (time.perf_counter() - t0))
            else:
                self._replay(self._g_fwd)
                self._enqueue_backward()
                self._replay(self._g_sgld)
        else:
            self._enqueue_forward()
            self._enqueue_backward()
            self._enqueue_sgld()
        self.last_loss = self.loss_ws.losses
        self.updates += 1
        self._advance()

    def _advance(self):
        st = self.state
        st.iteration += 1
        c = self.config
        if c.densify_every > 0 and st.iteration % c.densify_every == 0:
            import time
            t0 = time.perf_counter()
            densify(st, c.densify_growth, c.gaussian_cap, self.rng, jitter_sigma=c.densify_jitter,
                    device_select=c.device_noise)
            self.densify_ms.append(1000.0 * (time.perf_counter() - t0))
        if c.reassign_every > 0 and st.iteration % c.reassign_every == 0:
            import time
            from .reassign import reassign_codes
            t0 = time.perf_counter()
            for which in ("sh", "sr"):
                self.reassigned[which] += reassign_codes(st, which, c.reassign_tau)
            self.reassign_ms.append(1000.0 * (time.perf_counter() - t0))

    def mcmc(self):
        """One forced split and one forced merge transition (reference rules)."""
        import time
        t0 = time.perf_counter()
        for fn in (split_step, merge_step):
            rec = TransitionRecord(iteration=self.state.iteration + 1, kind="mcmc", codebook="-")
            fn(self.state, None, self.config, self.rng, rec)
            self._advance()
        self.mcmc_events += 1
        self.mcmc_ms.append(1000.0 * (time.perf_counter() - t0))

    def step(self):
        self.update()
        if self.mcmc_every and self.updates % self.mcmc_every == 0:
            self.mcmc()

    # -- results -----------------------------------------------------------------
    def check(self):
        """Raise if any update overflowed its pair buffers or saw non-finite gradients."""
        v = int(self.sticky.item())
        if v & 2:
            raise RuntimeError("pair capacity overflow during the run (raise pair_headroom); "
                               "the overflowing updates were skipped")
        if v & 1:
            raise SamplerError("non-finite gradients during the run (those updates were skipped)")

    def recon(self) -> float:
        return float(self.last_loss.view(self.V, 3)[:, 2].mean().item())
