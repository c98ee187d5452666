"""Benchmark: ContraGS training iterations on B200 (BASELINE.json metric
"train iters/s & rendered Mpix/s ... HBM roofline fraction").

Workload (default ``--config 1``, BASELINE.json configs[1]): N=100k Gaussians,
SR K=4096, [opacity; SH-3] K=4096, a batch of 4 views at 256x256 per GPU per
iteration, L1+SSIM (lambda 0.2) loss, SGLD update, forced split + merge MCMC
transitions every 25 iterations, densify every 100 (reference defaults).
Synthetic seeded scene; targets are renders of the seed+1
scene.  At N GPUs each rank renders its own 4 views of a 4N-view ring
(weak scaling) and the flat gradient buffer is summed with one NCCL
allreduce; `value` counts config-1 iterations (4 views) of the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

VIEWS_PER_GPU = {0: 1, 1: 4, 2: 1, 3: 1}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--mcmc-every", type=int, default=25)
    ap.add_argument("--noise-pos", type=float, default=0.01)
    ap.add_argument("--profile-kernel", default="raster_bwd_kernel")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--workload", default="train", choices=["train", "codenn"],
                    help="codenn: the code reassignment extension's nearest-code search "
                         "(tcgen05 distance GEMM) on a config-3 SH codebook")
    ap.add_argument("--codenn-rows", type=int, default=65536)
    ap.add_argument("--views-per-frame", type=int, default=1,
                    help="config 4: poses rendered per batched frame")
    ap.add_argument("--render-streams", type=int, default=2,
                    help="config 4: CUDA streams the frames are rendered on (frames are "
                         "independent: one frame's latency-bound sort / scan phases overlap "
                         "another's raster)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def make_scene(config, seed, rank, world):
    from paper_2509_03775_b200 import camera, scenes
    if config == 1:
        a = scenes.config1(seed, views=4 * world)
        g = scenes.config1(seed + 1, views=4 * world)
        cams = a.cameras[4 * rank: 4 * rank + 4]
    else:
        a = scenes.build(config, seed)
        g = scenes.build(config, seed + 1)
        nv = VIEWS_PER_GPU.get(config, 1)
        cams = [a.cameras[(rank * nv + k) % len(a.cameras)] for k in range(nv)]
    return a, g, cams


def workload_name(config):
    return {0: "config0: N=4096 SH-1 K=256, 1x64^2 view, L1",
            1: "config1: N=100k, SR K=4096, SH-3 K=4096, 4x256^2 views/GPU, L1+SSIM, MCMC every 25",
            2: "config2: N=1M clustered, SR 8192, SH-3 16384, 1x1280x720 view/GPU",
            3: "config3: N=4M outdoor, SR 16384, SH-3 65536, 1x1960x1088 view/GPU, "
               "code reassignment (extension) every 100 iters",
            4: "config4: render-only, N=6M, K=65536 both, 64 poses 1920x1080 sharded over GPUs"}[config]


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons through NVML during the
    timed region (same fields as the recipe's nvidia-smi clocks line): one
    sample when the region starts and one when it stops (synchronously, so
    even a 10 ms region has a record), and every `period` seconds between."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index, period=0.002):
        import threading
        self.gpu = gpu_index
        self.period = period
        self.samples = []
        self.stop_ev = threading.Event()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.err = None
        self.h = None
        self.max_sm = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # NVML missing: report it instead of inventing clocks
            self.err = repr(e)

    def _sample(self):
        nv, h = self.nv, self.h
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(h),
                             nv.nvmlDeviceGetUtilizationRates(h).gpu))

    def _run(self):
        try:
            while not self.stop_ev.wait(self.period):
                self._sample()
        except Exception as e:
            self.err = repr(e)

    def start(self):
        if self.h is None:
            return
        self._sample()
        self.thread.start()

    def stop(self):
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        self.stop_ev.set()
        self.thread.join(timeout=5)
        self._sample()
        busy = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = set()
        for _, rs, _ in busy:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": self.max_sm,
                "reasons": sorted(reasons), "samples": len(self.samples),
                "samples_under_load": len(busy), "period_ms": 1000.0 * self.period}


# ---------------------------------------------------------------------------
_W = {}


def _worker_init(arrays):
    """Pool initializer: each worker builds the oracle state once."""
    from oracle import cgs_oracle as O
    _W["st"] = O.OState.from_arrays(*arrays)


def _strip_cam(cam, y0, y1):
    """Rows [y0, y1) of a view as a camera of its own (principal point shifted).
    Every pixel's compositing and gradient depend only on that pixel, so the
    strips' images concatenate to the view's image and their gradients sum to
    the view's gradient."""
    from oracle import cgs_oracle as O
    return O.OCam(R=cam.R, t=cam.t, fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy - y0,
                  width=cam.width, height=y1 - y0)


def _job_fwd(cam):
    from oracle import cgs_oracle as O
    return O.raster_forward(_W["st"], cam)["image"]


def _job_loss(args):
    from oracle import cgs_oracle as O
    img, gt, lam = args
    return O.recon_loss_grad(img, gt, lam)


def _job_bwd(args):
    from oracle import cgs_oracle as O
    cam, dL = args
    return O.raster_backward(_W["st"], cam, dL)


def _oracle_iteration(a, gts, cams, lam, pool, strips):
    """One full reference update iteration on host cores: forward, L1/SSIM loss
    gradient and backward of every view, split into row strips so all worker
    processes are busy, then the mean gradient and the SGLD update (reference
    sampler.py:320-338, 262-300)."""
    from oracle import cgs_oracle as O
    ocams = [O.cam_from_any(c) for c in cams]
    parts = []
    for v, c in enumerate(ocams):
        rows = max(16, ((c.height + strips - 1) // strips + 15) // 16 * 16)
        for y0 in range(0, c.height, rows):
            parts.append((v, y0, min(c.height, y0 + rows)))
    t0 = time.perf_counter()
    imgs = pool.map(_job_fwd, [_strip_cam(ocams[v], y0, y1) for v, y0, y1 in parts])
    full = [np.concatenate([im for (v2, _, _), im in zip(parts, imgs) if v2 == v], axis=0)
            for v in range(len(ocams))]
    dls = pool.map(_job_loss, [(full[v], gts[v], lam) for v in range(len(ocams))])
    res = pool.map(_job_bwd, [(_strip_cam(ocams[v], y0, y1), dls[v][y0:y1]) for v, y0, y1 in parts])
    grads = {k: sum(r[k] for r in res) / len(ocams) for k in res[0]}
    st = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    O.sgld_update(st, grads, O.config(), np.random.default_rng(0))
    return time.perf_counter() - t0


def _oracle_gts(g, cams):
    from oracle import cgs_oracle as O
    gst = O.OState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
    return [np.round(np.clip(O.raster_forward(gst, O.cam_from_any(c))["image"], 0.0, 1.0) * 255.0)
            / 255.0 for c in cams]  # 8-bit targets, as in the GPU arm


def cpu_iteration_timer(config, seed):
    """Returns (fn() -> seconds per iteration, cores, sample description, pool)."""
    a, g, cams = make_scene(config, seed, 0, 1)
    gts = _oracle_gts(g, cams)
    cores = max(1, os.cpu_count() or 1)
    strips = max(1, cores // len(cams))
    arrays = (a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    pool = mp.get_context("fork").Pool(cores, initializer=_worker_init, initargs=(arrays,))
    lam = 0.0 if config == 0 else 0.2

    def run():
        return _oracle_iteration(a, gts, cams, lam, pool, strips)

    sample = (f"one full {workload_name(config).split(':')[0]} update iteration "
              f"({len(cams)} views x {strips} row strips fwd + L1/SSIM grad + bwd in {cores} "
              "worker processes, mean grad, SGLD) through the numpy oracle port "
              "(oracle/cgs_oracle.py) of the reference")
    return run, cores, sample, pool


def api_train_rate(config, seed, noise_pos, iters=60):
    """The drop-in API as a user of the reference calls it: cg.train (reference
    sampler.py:402-420) over (Camera, host numpy image) views with reference
    semantics -- one randomly chosen view per update, split / merge by the
    reference mixture, host-drawn (parity-mode) SGLD noise, the TransitionRecord
    read back every step.  Returns (it/s, description)."""
    import torch
    import paper_2509_03775_b200 as cg
    a, g, cams = make_scene(config, seed, 0, 1)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows, gaussian_headroom=0.25)
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                    g.sr_rows)
    views = [(c, cg.rasterize_forward(gst, c).image.cpu().numpy()) for c in cams]
    del gst
    cfg = cg.SamplerConfig(lambda_ssim=0.0 if config == 0 else 0.2, noise_pos=noise_pos)
    rng = np.random.default_rng(seed)
    cg.train(st, views, cfg, 5, rng)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs = cg.train(st, views, cfg, iters, rng)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    kinds = {k: sum(r.kind == k for r in recs) for k in ("update", "split", "merge")}
    return iters / secs, (f"cg.train({iters} iterations) on config {config}: reference semantics "
                          f"(one view per update, {kinds}), host numpy targets uploaded per step, "
                          f"host-drawn SGLD noise (noise_pos={noise_pos}), TransitionRecord per step")


def cpu_one_core(config, seed):
    """The reference algorithm (numpy oracle port) on ONE core: forward, L1/SSIM
    gradient and backward of view 0 in this process with BLAS limited to one
    thread (SURVEY.md §8(d) asks for a 1-core figure beside the all-cores one).
    Config 0/1: the whole view, scaled by the step's view count; larger
    configs: a 32-row strip of it, scaled by its share of the step's pixels.
    Returns (it/s estimate, seconds measured, description)."""
    from threadpoolctl import threadpool_limits
    from oracle import cgs_oracle as O
    a, g, cams = make_scene(config, seed, 0, 1)
    cam = O.cam_from_any(cams[0])
    rows = cam.height if config <= 1 else 32
    strip = _strip_cam(cam, 0, rows)
    gst = O.OState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows, g.sr_rows)
    gt = np.round(np.clip(O.raster_forward(gst, strip)["image"], 0.0, 1.0) * 255.0) / 255.0
    st = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    lam = 0.0 if config == 0 or rows < 11 else 0.2
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        img = O.raster_forward(st, strip)["image"]
        dL = O.recon_loss_grad(img, gt, lam)
        O.raster_backward(st, strip, dL)
        secs = time.perf_counter() - t0
    share = (rows * cam.width) / float(sum(c.width * c.height for c in cams))
    per_iter = secs / share
    return (1.0 / per_iter, secs,
            f"view 0 {'rows 0-31 ' if rows != cam.height else ''}fwd + loss grad + bwd through the "
            f"numpy oracle port in 1 process, BLAS 1 thread: {secs:.1f} s for {share:.3g} of the "
            f"step's pixels, scaled to one iteration ({per_iter:.1f} s)")


def run_reference(args):
    """--impl reference: the reference's algorithm (oracle port) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    run, cores, sample, pool = cpu_iteration_timer(args.config, args.seed)
    first = run()  # warm-up: the requested W (>= 1), bounded to ~30 s of CPU work
    n_warm = 1
    while n_warm < args.warmup and first * (n_warm + 1) <= 30.0:
        run()
        n_warm += 1
    budget = 150.0
    k_eff = max(2, min(args.steps, int(budget / max(first, 1e-3))))
    times = [run() for _ in range(k_eff)]
    pool.close()
    total = sum(times)
    value = k_eff / total
    out = {"impl": "reference", "metric": "train iters/s", "value": value, "unit": "it/s",
           "n_gpus": args.gpus, "steps": k_eff, "warmup": n_warm, "ms_per_step": 1000 * total / k_eff,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded scene, SURVEY.md §8(d))",
           "config": {"workload": workload_name(args.config), "seed": args.seed},
           "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "kind": "port",
                            "sample": sample + f"; {k_eff} timed iterations (bounded to ~{budget:.0f} s)"},
           "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------------------
def _oracle_render_mpix(a, cam, crop=(480, 270)):
    """Reference forward (numpy oracle port) of a crop window of one pose: the
    full scene is projected and the crop's pixels rasterized.  Returns
    (Mpix/s, seconds, sample description)."""
    from oracle import cgs_oracle as O
    cw, ch = crop
    c = O.cam_from_any(cam)
    c = O.OCam(R=c.R, t=c.t, fx=c.fx, fy=c.fy, cx=c.cx - (c.width - cw) / 2.0,
               cy=c.cy - (c.height - ch) / 2.0, width=cw, height=ch)
    st = O.OState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows, a.sr_rows)
    t0 = time.perf_counter()
    O.raster_forward(st, c)
    secs = time.perf_counter() - t0
    return (cw * ch / secs / 1e6, secs,
            f"oracle forward of the central {cw}x{ch} window of pose 0 (all {a.n} Gaussians "
            "projected), 1 process")


def run_codenn(args, world, rank, local):
    """--workload codenn: nearest live code row for every live row of an SH-3
    codebook of --codenn-rows rows (config 3/4 K_sh = 65536), the search behind
    reassign_codes (extension, no reference counterpart).  A step is one
    cgs_code_nn call (pack, tcgen05 tf32 distance GEMM with candidate epilogue,
    exact fp64 certification).  value = rows searched per second; roofline =
    the GEMM kernel's tensor FLOP/s.  N > 1 runs replicas (the search is not
    sharded)."""
    import torch
    torch.cuda.set_device(local)
    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import _native as nat
    dev = torch.device("cuda", local)
    K, D = args.codenn_rows, 48
    rng = np.random.default_rng(args.seed)
    rows = rng.normal(0.0, 0.2, (K, D)).astype(np.float32)
    n = K
    st = cg.ModelState.from_arrays(np.zeros((n, 3), np.float32), np.zeros(n, np.float32),
                                   np.arange(n, dtype=np.int32), np.zeros(n, np.int32), rows,
                                   np.array([[-4, -4, -4, 1, 0, 0, 0]], np.float32), device=dev)
    lib = nat.library()
    flush = torch.empty((64 * 1024 * 1024,), dtype=torch.float32, device=dev)
    for _ in range(max(3, args.warmup)):
        cg.nearest_codes(st, "sh")
    torch.cuda.synchronize()
    lib.cgs_profile_kernel(b"codenn_gemm_kernel")
    clocks = ClockSampler(local)
    l0 = lib.cgs_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record()
        idx, dist2 = cg.nearest_codes(st, "sh")
        ev[k][1].record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = int(lib.cgs_launch_count() - l0)
    tot = sum(s.elapsed_time(e) for s, e in ev)
    prof_ms, prof_n = nat.F64(0.0), nat.I64(0)
    lib.cgs_profile_read(prof_ms, prof_n)
    lib.cgs_profile_kernel(b"")
    avg_s = prof_ms.value / max(prof_n.value, 1) / 1000.0
    mpad = (K + 127) // 128 * 128
    flops_exec = 3 * 2.0 * mpad * mpad * 48  # 3xTF32: three tensor products per K step
    flops_alg = 2.0 * K * K * D
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    bf16 = float(peaks.get("bf16_tflops", 2250.0))
    peak = bf16 / 2.0
    # e2e: the same search from host rows: H2D of the rows, search, D2H of index + distance
    host_rows = torch.as_tensor(rows).pin_memory()
    host_idx = torch.empty((st.sh.capacity,), dtype=torch.int32).pin_memory()
    host_d = torch.empty((st.sh.capacity,), dtype=torch.float64).pin_memory()
    e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        e_ev[k][0].record()
        st.sh.rows[:K].copy_(host_rows, non_blocking=True)
        idx, dist2 = cg.nearest_codes(st, "sh")
        host_idx.copy_(idx, non_blocking=True)
        host_d.copy_(dist2, non_blocking=True)
        e_ev[k][1].record()
    torch.cuda.synchronize()
    e_tot = sum(s.elapsed_time(e) for s, e in e_ev)
    got = host_idx.numpy()[:K]
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # fp64 brute force (the definition) for a bounded sample of rows
        import time
        sample = 64
        x = rows.astype(np.float64)
        t0 = time.perf_counter()
        for i in range(sample):
            t = x - x[i]
            d2 = np.einsum("ij,ij->i", t, t)
            d2[i] = np.inf
            j = int(np.argmin(d2))
            assert j == got[i] or d2[j] == d2[got[i]], (i, j, got[i])
        secs = time.perf_counter() - t0
        cpu = {"value": sample / secs, "unit": "rows/s", "cores": 1, "kind": "port",
               "sample": f"{sample} rows against all {K} (numpy fp64 brute force, the "
                         "extension's definition; no reference counterpart)", "seconds": secs}
    if rank == 0:
        out = {"metric": "code-NN rows/s", "value": world * args.steps * K / (tot / 1000.0),
               "unit": "rows/s", "n_gpus": world, "steps": args.steps,
               "warmup": max(3, args.warmup), "ms_per_step": tot / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "tf32 tensor GEMM (candidates) + fp64 certification",
               "data": f"synthetic SH-3 codebook, {K} rows N(0, 0.2) (config 3/4 K_sh)",
               "config": {"workload": f"code reassignment nearest-code search, K={K}, D={D}",
                          "l2": "flushed (256 MB write) between timed iterations",
                          "parallelism": f"replicas x{world} (not sharded)"},
               "gpu_launches": launches, "clocks": clk,
               "roofline": {"bound": "tensor", "kernel": "codenn_gemm_kernel",
                            "achieved": flops_alg / avg_s / 1e12 if avg_s > 0 else 0.0,
                            "peak": peak, "unit": "TFLOP/s",
                            "peak_source": "tf32 dense = half the measured bf16 GEMM burst rate "
                                           "(MEASURED_PEAKS.json bf16_tflops); nominal 1.1 PF",
                            "frac": (flops_alg / avg_s / 1e12) / peak if avg_s > 0 else 0.0,
                            "avg_launch_ms": avg_s * 1000.0, "flops_algorithmic": flops_alg,
                            "tensor_flops_executed": flops_exec,
                            "tensor_tflops_executed": flops_exec / avg_s / 1e12 if avg_s > 0 else 0.0,
                            "note": "achieved = algorithmic 2 K^2 D flops; the 3xTF32 split "
                                    "executes 3x that on the tensor pipe (tensor_tflops_executed)",
                            "traffic": None},
               "e2e": {"value": world * args.steps * K / (e_tot / 1000.0), "unit": "rows/s",
                       "h2d_bytes_per_step": K * D * 4,
                       "d2h_bytes_per_step": int(host_idx.numel() * 4 + host_d.numel() * 8)},
               "cpu_baseline": cpu}
        print(json.dumps(out))


def run_render(args, world, rank, local):
    """--config 4: render-only throughput.  A step renders all 64 poses of the
    job (strong scaling: poses sharded round-robin over ranks), forward only,
    in batched frames of --views-per-frame poses; value = rendered Mpix/s of
    the whole job.  e2e adds the D2H copy of every image to pinned memory."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import _native as nat
    from paper_2509_03775_b200 import scenes
    a = scenes.config4(args.seed)
    dev = torch.device("cuda", local)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows, device=dev)
    mine = a.cameras[rank::world]
    B = max(1, min(args.views_per_frame, nat.MAX_VIEWS))
    groups = [mine[i:i + B] for i in range(0, len(mine), B)]
    frames = [cg.Frame(st, g).run_checked() for g in groups]  # sizes the pair buffers
    flush = torch.empty((64 * 1024 * 1024,), dtype=torch.float32, device=dev)
    lib = nat.library()
    # frames (own workspaces) round-robin over S streams, forked from and
    # joined back into the current stream, so the events around a step on the
    # current stream time all of it
    S = max(1, args.render_streams)
    main_s = torch.cuda.current_stream(dev)
    streams = [main_s] + [torch.cuda.Stream(device=dev) for _ in range(S - 1)]

    def fan(work):
        fork = torch.cuda.Event()
        fork.record(main_s)
        for s in streams[1:]:
            s.wait_event(fork)
        for i, f in enumerate(frames):
            with torch.cuda.stream(streams[i % S]):
                work(i, f)
        for s in streams[1:]:
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)

    def step():
        fan(lambda i, f: f.run())

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if any(f.stats().overflow for f in frames):
        raise RuntimeError("pair capacity overflow")
    clocks = ClockSampler(local)
    l0 = lib.cgs_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record()
        step()
        ev[k][1].record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = int(lib.cgs_launch_count() - l0)
    ms = [s.elapsed_time(e) for s, e in ev]
    tot = sum(ms)
    if world > 1:
        t = torch.tensor([tot], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    px_job = sum(c.width * c.height for c in a.cameras)
    value = args.steps * px_job / (tot / 1000.0) / 1e6
    # e2e: the same renders as the reference's `contrags render` delivers them
    # (cli.py:209-220: 8-bit RGB, save_png's bytes): each frame quantized on the
    # device (cgs_quantize8) and its bytes copied into pinned host memory
    u8s = [torch.empty(f.image.shape, dtype=torch.uint8, device=dev) for f in frames]
    hosts = [torch.empty(f.image.shape, dtype=torch.uint8).pin_memory() for f in frames]
    e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    def deliver(i, f):
        f.run()
        nat.call("cgs_quantize8", nat.ptr(f.image), f.image.numel(), nat.ptr(u8s[i]),
                 nat.stream_handle(dev))
        hosts[i].copy_(u8s[i], non_blocking=True)

    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        e_ev[k][0].record()
        fan(deliver)
        e_ev[k][1].record()
    torch.cuda.synchronize()
    e_tot = sum(s.elapsed_time(e) for s, e in e_ev)
    if world > 1:
        t = torch.tensor([e_tot], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_tot = float(t.item())
    stats = [f.stats() for f in frames]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, secs, sample = _oracle_render_mpix(a, a.cameras[0])
        cpu = {"value": v, "unit": "Mpix/s", "cores": 1, "kind": "port", "sample": sample,
               "seconds": secs}
    if rank == 0:
        out = {"metric": "rendered Mpix/s", "value": value, "unit": "Mpix/s", "n_gpus": world,
               "steps": args.steps, "warmup": max(3, args.warmup),
               "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f32 (fp64 projection geometry)",
               "data": "synthetic (seeded scene, SURVEY.md §8(d)); random-init codebooks",
               "config": {"workload": workload_name(4), "views_per_frame": B,
                          "streams": S,
                          "poses_per_gpu": len(mine), "gaussians": a.n,
                          "l2": "flushed (256 MB write) between timed iterations",
                          "parallelism": f"dp{world} (poses sharded, no collective)"},
               "gpu_launches": launches, "clocks": clk,
               "e2e": {"value": args.steps * px_job / (e_tot / 1000.0) / 1e6, "unit": "Mpix/s",
                       "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": int(sum(h.numel() for h in hosts)) * world,
                       "note": "8-bit RGB images as cmd_render writes them (device quantize8, "
                               "then D2H of the bytes)"},
               "cpu_baseline": cpu,
               "frame": {"pairs": int(sum(x.n_pairs for x in stats)),
                         "onscreen": int(sum(x.n_onscreen for x in stats))}}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "codenn":
        return run_codenn(args, world, rank, local)
    if args.config == 4:
        return run_render(args, world, rank, local)

    import torch
    import torch.distributed as dist

    # CGS_DIST_BACKEND=gloo (tests, one-GPU boxes): every rank may share a GPU
    # (device = local rank mod the visible devices); the default is NCCL, one
    # rank per GPU
    backend = os.environ.get("CGS_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2509_03775_b200 as cg
    from paper_2509_03775_b200 import _native as nat
    from paper_2509_03775_b200.engine import Trainer

    a, g, cams = make_scene(args.config, args.seed, rank, world)
    dev = torch.device("cuda", local)
    st = cg.ModelState.from_arrays(a.positions, a.opacity_logits, a.g2sh, a.g2sr, a.sh_rows,
                                   a.sr_rows, device=dev, gaussian_headroom=0.25)
    gst = cg.ModelState.from_arrays(g.positions, g.opacity_logits, g.g2sh, g.g2sr, g.sh_rows,
                                    g.sr_rows, device=dev)
    gt_frame = cg.render_frame(gst, cams)
    H, W = cams[0].height, cams[0].width
    # targets are 8-bit RGB, like the reference's PNG inputs (modelio.py:138-153):
    # the GT renders quantised to k/255; the e2e path uploads the uint8 bytes
    gts = (gt_frame.image.view(len(cams), H, W, 3).clamp(0.0, 1.0) * 255.0).round() * (1.0 / 255.0)
    del gt_frame, gst
    lam = 0.0 if args.config == 0 else 0.2
    # Reference defaults except the position Langevin noise: the default
    # noise_pos=1.0 with step_pos=0.5 adds N(0, 0.5) per coordinate per update,
    # which diffuses this scene out of the views within ~10 iterations (the
    # raster work then collapses).  noise_pos=0.01 keeps the noise draw (device
    # Philox) in every update while the scene stays in view, so the GPU step and
    # the CPU baseline (initial scene) measure the same workload.
    # config 3 names "code reassignment every 100 iters" (an extension: the
    # reference has none): merge mutual nearest code rows
    # within 1e-8 squared distance (near-identical rows only)
    reassign = {"reassign_every": 100, "reassign_tau": 1e-8} if args.config == 3 else {}
    if st.num_gaussians >= 2_000_000:  # the reference default cap (2M) is below N here
        reassign["gaussian_cap"] = int(st.num_gaussians * 1.25)
    cfg = cg.SamplerConfig(lambda_ssim=lam, device_noise=True, seed=args.seed,
                           noise_pos=args.noise_pos, **reassign)
    from paper_2509_03775_b200 import dist as cdist
    allreduce = cdist.make_allreduce() if world > 1 else None
    rng = np.random.default_rng(args.seed)
    tr = Trainer(st, cams, gts, cfg, rng, mcmc_every=args.mcmc_every, world=world,
                 allreduce=allreduce, use_graphs=not args.no_graphs,
                 total_views=len(cams) * world)

    flush = torch.empty((64 * 1024 * 1024,), dtype=torch.float32, device=dev)  # 256 MB > L2

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        tr.step()
    torch.cuda.synchronize()
    tr.check()

    lib = nat.library()
    lib.cgs_profile_kernel(args.profile_kernel.encode())
    clocks = ClockSampler(local)
    launches0 = lib.cgs_launch_count()
    cap0, rep0 = tr.capture_counted, tr.replayed_kernels
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    views_done = 0
    # Python's cyclic GC is paused inside the timed loops (collected just
    # before), as timeit does: a generation-2 pass is a host stall unrelated
    # to the workload.  The trainer itself allocates no Python cycles.
    import gc
    gc.collect()
    gc.disable()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    host_s = 0.0
    for k in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        starts[k].record()
        h0 = time.perf_counter()
        tr.step()
        host_s += time.perf_counter() - h0
        ends[k].record()
        views_done += len(cams)
    torch.cuda.synchronize()
    barrier()
    gc.enable()
    clk = clocks.stop()
    # ABI launch calls + kernels executed by graph replays - calls recorded
    # (not executed) while capturing
    launches = int(lib.cgs_launch_count() - launches0) + (tr.replayed_kernels - rep0) - (
        tr.capture_counted - cap0)
    tr.check()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    prof_ms, prof_n = nat.F64(0.0), nat.I64(0)
    lib.cgs_profile_read(prof_ms, prof_n)
    lib.cgs_profile_kernel(b"")
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    iters_value = (args.steps * world) / (total_ms / 1000.0)  # config-1 iterations, whole job
    mpix = views_done * world * H * W / (total_ms / 1000.0) / 1e6
    stats = tr.frame.stats()

    # roofline of the profiled kernel (algorithmic bytes)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        try:
            peak = float(json.load(open(peaks_path))["hbm_gbs"])
            peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    px = sum(c.width * c.height for c in cams)
    P_x = int(stats.n_processed)
    name = args.profile_kernel
    if name == "raster_bwd_kernel":
        alg = 44 * P_x + 36 * P_x + 32 * px
    elif name == "raster_fwd_kernel":
        alg = 44 * P_x + 24 * px
    elif name == "project_kernel":
        n = st.num_gaussians
        alg = 24 * n * len(cams) + 4 * (7 * st.sr.capacity + st.sh.dim * st.sh.capacity) + 52 * int(stats.n_onscreen)
    else:
        alg = 0
    avg_s = (prof_ms.value / max(prof_n.value, 1)) / 1000.0
    achieved = alg / avg_s / 1e9 if avg_s > 0 else 0.0
    # DRAM bytes per launch of the same kernel from the committed ncu --set full
    # capture (profiles/ncu_traffic.json, written by scripts/ncu_summary.py)
    traffic, traffic_src, issue_pct, compute = None, None, None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(name)
            if t:
                traffic = float(t["bytes_per_launch"])
                traffic_src = f"profiles/ncu_traffic.json ({t.get('source')}, ncu --set full)"
                issue_pct = t.get("issue_active_pct")
                # the compute side of the same launch: the raster kernels are
                # bound by instruction issue, not by HBM or FP32 throughput
                pct = lambda k: (t[k] / 100.0) if t.get(k) is not None else None
                compute = {"bound": "issue", "issue_active_frac": pct("issue_active_pct"),
                           "fp32_frac_of_peak": t.get("fp32_frac_of_peak"),
                           "fp32_peak": "148 SMs x 128 lanes x 2 FLOP per cycle",
                           "fma_pipe_frac": pct("fma_pipe_pct"), "alu_pipe_frac": pct("alu_pipe_pct"),
                           "xu_pipe_frac": pct("xu_pipe_pct"),
                           "lane_efficiency": t.get("lane_efficiency"),
                           "source": traffic_src}
        except Exception:
            pass
    roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "avg_launch_ms": avg_s * 1000.0, "launches": int(prof_n.value),
                "alg_bytes_per_launch": alg, "P_x": P_x, "pixels": px,
                "issue_active_frac": issue_pct / 100.0 if issue_pct else None,
                "compute": compute,
                "note": "the raster kernels are instruction-issue bound (ncu: ~75% issue slots "
                        "busy, ALU + FMA pipes, see profiles/r2_ncu_raster_config1.txt), not "
                        "HBM bound; achieved uses processed-prefix algorithmic bytes only "
                        "(SURVEY.md §8(d)), traffic is the ncu DRAM bytes of one launch"}

    # e2e: same step through the public API with host buffers (pinned H2D of the
    # step's target images, D2H of the recon loss) inside the timed region
    e2e = None
    if not args.no_e2e:
        # config 1: BASELINE.json's run definition -- 100 iterations, forced
        # split + merge every 25, densify when the transition count crosses
        # 100 -- whatever --steps is; graph re-captures fall inside the window.
        # Other configs: at least one MCMC period, so the window holds the
        # events in their natural proportion
        n_e2e = (max(args.steps, 100) if args.config == 1
                 else max(args.steps, min(max(args.mcmc_every, 1), 1000)))
        ev0, dn0, cp0 = tr.mcmc_events, len(tr.densify_ms), tr.captures
        host_gt = (gts * 255.0).round().to(torch.uint8).cpu().pin_memory()
        # double-buffered device targets: step k+1's upload runs on a copy
        # stream while step k computes (the first upload is inside step 0's
        # interval, every later one inside the previous step's)
        dev_gt = [torch.empty(host_gt.shape, dtype=torch.uint8, device=dev) for _ in range(2)]
        copy_st = torch.cuda.Stream(dev)
        up_done = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]
        host_loss = torch.empty((3 * len(cams),), dtype=torch.float64).pin_memory()
        e_s = [torch.cuda.Event(enable_timing=True) for _ in range(n_e2e)]
        e_e = [torch.cuda.Event(enable_timing=True) for _ in range(n_e2e)]
        cur = torch.cuda.current_stream(dev)

        def upload(b):
            copy_st.wait_event(used[b])
            with torch.cuda.stream(copy_st):
                dev_gt[b].copy_(host_gt, non_blocking=True)
                up_done[b].record(copy_st)

        gc.collect()
        gc.disable()
        barrier()
        torch.cuda.synchronize()
        for k in range(n_e2e):
            if not args.no_flush:
                flush.zero_()
            e_s[k].record()
            b = k & 1
            if k == 0:
                upload(b)
            cur.wait_event(up_done[b])
            torch.mul(dev_gt[b], 1.0 / 255.0, out=tr.gts)  # uint8 -> [0, 1] on the device
            used[b].record(cur)
            if k + 1 < n_e2e:
                upload(b ^ 1)
            tr.step()
            host_loss.copy_(tr.last_loss, non_blocking=True)
            e_e[k].record()
        torch.cuda.synchronize()
        barrier()
        gc.enable()
        tr.check()
        e_ms = sum(s.elapsed_time(e) for s, e in zip(e_s, e_e))
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": (n_e2e * world) / (e_ms / 1000.0), "unit": "it/s",
               "h2d_bytes_per_step": int(host_gt.numel()),
               "d2h_bytes_per_step": int(host_loss.numel() * 8),
               "iterations": n_e2e, "mcmc_events": tr.mcmc_events - ev0,
               "densify": len(tr.densify_ms) - dn0, "graph_recaptures": tr.captures - cp0,
               "note": "engine.Trainer with host (pinned) 8-bit targets uploaded every step and "
                       "the losses read back; per-step CUDA events"
                       + ("; BASELINE config-1 run: 100 iterations, MCMC every 25, densify"
                          if args.config == 1 else "")}

    api = None
    if rank == 0 and world == 1 and not args.no_e2e and args.config in (0, 1):
        api = {}
        for c in sorted({args.config, 0}, reverse=True):
            v, d = api_train_rate(c, args.seed, args.noise_pos)
            api[f"config{c}"] = {"value": v,
                                 "unit": "train iters/s (reference semantics: 1 view per update)",
                                 "description": d}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        run, cores, sample, pool = cpu_iteration_timer(args.config, args.seed)
        secs = run()
        pool.close()
        cpu = {"value": 1.0 / secs, "unit": "it/s", "cores": cores, "kind": "port",
               "sample": sample, "seconds": secs}
        v1, s1, d1 = cpu_one_core(args.config, args.seed)
        cpu["one_core"] = {"value": v1, "unit": "it/s", "cores": 1, "kind": "port",
                           "seconds_measured": s1, "sample": d1}

    if rank == 0:
        out = {"metric": "train iters/s", "value": iters_value, "unit": "it/s", "n_gpus": world,
               "steps": args.steps, "warmup": max(3, args.warmup),
               "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f32 (fp64 projection geometry)",
               "data": "synthetic (seeded scene, SURVEY.md §8(d)); random-init codebooks",
               "config": {"workload": workload_name(args.config), "views_per_gpu": len(cams),
                          "image": f"{W}x{H}", "gaussians": st.num_gaussians,
                          "l2": "flushed (256 MB write) between timed iterations"
                          if not args.no_flush else "not flushed",
                          "targets": "8-bit RGB (the reference's PNG inputs), uint8 upload in e2e",
                          "python_gc": "cyclic GC collected before and paused inside the timed loops",
                          "mcmc_every": args.mcmc_every,
                          "sgld_noise": f"device Philox, noise_pos={args.noise_pos} (reference default 1.0 "
                                        "diffuses the scene out of view; see DESIGN.md)",
                          "parallelism": f"dp{world} (views sharded, {backend} allreduce)"},
               "mpix_per_s": mpix, "gpu_launches": launches,
               "step_ms": {"min": min(step_ms), "p50": statistics.median(step_ms),
                           "max": max(step_ms)}, "roofline": roofline,
               "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "drop_in_train": api,
               "frame": {"pairs": int(stats.n_pairs), "processed_pairs": P_x,
                         "touched": int(stats.n_touched), "onscreen": int(stats.n_onscreen)},
               "recon": tr.recon(), "mcmc_events": tr.mcmc_events,
               "mcmc_ms": tr.mcmc_ms, "densify_ms": tr.densify_ms, "capture_ms": tr.capture_ms,
               "reassign_ms": tr.reassign_ms, "reassigned_rows": tr.reassigned,
               "host_enqueue_ms_per_step": 1000.0 * host_s / args.steps,
               "cuda_graphs": tr.use_graphs, "graph_captures": tr.captures}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
