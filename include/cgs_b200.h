/*
 * cgs_b200.h -- C ABI of the B200-native ContraGS training hot path.
 *
 * The reference (`contrags` 0.1.0, /root/reference/pkg/src/contrags) is pure
 * Python with no FFI, so there is no C interface to replace; the entry points
 * below are what a host binding of that package's hot path binds (see
 * INTEGRATION.md for the ctypes stub).  Each function names the reference
 * Python function(s) whose semantics it implements.
 *
 * Conventions
 *   - all array arguments are DEVICE pointers unless marked "host";
 *   - every call is asynchronous on `stream` (a cudaStream_t) unless marked
 *     "synchronizes";
 *   - all buffers, including workspaces, are caller-allocated; besides a
 *     thread-local last-error string and the diagnostics switches below, the
 *     library keeps only per-device caches of launch configuration (kernel
 *     shared-memory attributes, occupancy-sized grids), indexed by the
 *     current device ordinal, so one process may drive several GPUs;
 *   - functions return 0 on success and a nonzero CGS_E* code otherwise,
 *     never throwing across the ABI; cgs_last_error() describes the failure.
 *
 * Layouts follow the reference exactly (pkg/src/contrags/model.py:121-154):
 *   positions (N,3) f32, opacity_logits (N,) f32, g2sh/g2sr (N,) i32,
 *   SH rows (cap_sh, 3(d+1)^2) f32 coefficient-major row[b*3+ch] (sh.py:3-5),
 *   SR rows (cap_sr, 7) f32 = [log-scale(3); quaternion w,x,y,z (4)].
 * Images are (views, H, W, 3) f32, row-major, views concatenated.
 */
#ifndef CGS_B200_H
#define CGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGS_ABI_VERSION 1
#define CGS_MAX_VIEWS 16

#define CGS_OK 0
#define CGS_EINVAL 1     /* invalid argument (reference: ValueError)          */
#define CGS_ECUDA 2      /* CUDA runtime error                                */
#define CGS_EWORKSPACE 3 /* workspace too small                               */
#define CGS_ENONFINITE 4 /* non-finite gradients (reference: SamplerError)    */
#define CGS_EINTERNAL 5  /* internal invariant violated (a bug, not an input) */

#if defined(__GNUC__)
#define CGS_API __attribute__((visibility("default")))
#else
#define CGS_API
#endif

typedef void* cgs_stream_t; /* cudaStream_t */

/* Pinhole camera, reference camera.py:10-36: R is the row-major
 * world->camera rotation, t the world->camera translation. */
typedef struct cgs_camera {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  int32_t width, height;
} cgs_camera_t;

/* Scene state S = {G, C}, reference model.py:121-154 (device pointers). */
typedef struct cgs_scene {
  int64_t n;
  const float* positions;
  const float* opacity_logits;
  const int32_t* g2sh;
  const int32_t* g2sr;
  const float* sh_rows;
  int64_t sh_capacity;
  int32_t sh_degree; /* 0..3 */
  const float* sr_rows;
  int64_t sr_capacity;
} cgs_scene_t;

/* Counters a frame writes into its workspace header (device); read them
 * with cgs_frame_stats. */
typedef struct cgs_frame_stats {
  int64_t n_onscreen;   /* splats with a non-empty pixel rect, all views       */
  int64_t n_pairs;      /* (tile, splat) pairs P                               */
  int64_t n_processed;  /* pairs inside each tile's processed prefix, P_x      */
  int64_t n_touched;    /* (view, gaussian) pull-back entries U                */
  int64_t pair_capacity;
  int32_t overflow;     /* P exceeded pair_capacity: raster skipped            */
  int32_t n_views;
  int32_t zero_quaternion; /* a visible splat uses a zero quaternion (ValueError,
                              render.py:40-41); its splat is dropped           */
  int32_t pad_;
  int64_t n_refined_tiles; /* tiles whose flagged pixels were re-walked in
                              float64 (an fp32 alpha within 2e-5 of 1/255 or
                              0.99, or fp32 T within 5e-5 of 1e-4)           */
  int64_t n_refined_pixels; /* those pixels                                  */
  int64_t diag_last_mismatch;  /* pixels flagged by the T band (by default); */
  int64_t diag_count_mismatch; /* by an alpha band.  Diagnostics builds        */
                               /* (CGS_REFINE_ALL, every pixel re-walked):     */
                               /* pixels where the fp32 path alone decides the */
                               /* last index / the count differently           */
  float diag_max_T_err;        /* CGS_REFINE_ALL: largest fp32 T and alpha     */
  float diag_max_alpha_err;    /* relative errors against float64              */
} cgs_frame_stats_t;

/* SGLD parameters, reference sampler.py:262-300 + SamplerConfig :45-55. */
typedef struct cgs_sgld_params {
  double step_pos, step_opacity, step_sh, step_sr;
  double noise_pos, noise_opacity, noise_sh, noise_sr;
  double grad_scale;     /* multiplies every gradient (1/views for a mean)   */
  uint64_t seed;         /* device Philox stream (noise_source == 0)         */
  uint64_t offset;
  int32_t noise_source;  /* 0: device Philox, 1: caller arrays (parity)      */
  int32_t pad_;
  uint64_t* offset_dev;  /* optional device counter: incremented by the update
                            and used as the Philox offset instead of `offset`
                            (CUDA-graph replays then draw fresh noise)       */
  const int32_t* skip_if; /* optional device flag (e.g. the frame's
                            stats.overflow): when nonzero the update writes
                            nothing and sets flags[0] |= 2                   */
  int32_t* sticky;       /* optional device accumulator: sticky |= flags[0]
                            (so a run can be checked once, at its end)       */
  const int32_t* grads_nonfinite; /* optional device flag that already covers
                            every gradient entry (cgs_backward_nonfinite_flag
                            of the backward that wrote them): replaces the
                            update's own finiteness pass                    */
} cgs_sgld_params_t;

/* ---- library --------------------------------------------------------- */
CGS_API int cgs_abi_version(void);
CGS_API const char* cgs_last_error(void); /* thread-local, host */

/* ---- instrumentation (host; used by bench.py) ------------------------ */
/* Number of kernels this library has launched since load. */
CGS_API uint64_t cgs_launch_count(void);
/* Bracket every launch of the kernel called `name` (e.g. "raster_bwd_kernel")
 * with CUDA events on its launch stream; "" or NULL disables.  Resets the
 * accumulated events. */
CGS_API int cgs_profile_kernel(const char* name);
/* Sum of the recorded launches' durations (synchronizes those events). */
CGS_API int cgs_profile_read(double* total_ms, int64_t* launches);
/* Diagnostics: with a zeroed device buffer of >= 8 * total_tiles + 33
 * uint64 set, the raster kernels record {start ns, end ns, SM id, tile} per
 * CTA (forward at [4 b], backward persistent CTA b at [4 (total_tiles + b)])
 * and the backward adds a histogram of contributing lanes per warp hit at
 * [8 total_tiles + 0..32]; NULL disables. */
CGS_API int cgs_trace_tiles(void* dev_buf);

/* ---- render: rasterize_forward / rasterize_backward ------------------- */
/* Workspace for one batched frame of n_views cameras (host cams).
 * pair_capacity bounds the (tile, splat) pairs P (render.py:240-254). */
CGS_API size_t cgs_frame_workspace_bytes(int64_t n, const cgs_camera_t* cams, int32_t n_views,
                                 int64_t pair_capacity, int64_t sr_capacity);

/* rasterize_forward (render.py:287-315) for n_views cameras at once:
 * fused projection + codebook gather + SH (render.py:145-203), onesweep
 * depth sort (render.py:203), tile duplication + stable tile sort
 * (render.py:240-254), per-tile front-to-back blend (render.py:265-311).
 * If P > pair_capacity the raster is skipped and stats.overflow is set. */
CGS_API int cgs_render_forward(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                       void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                       float* image, float* final_T, int32_t* contrib_counts,
                       cgs_stream_t stream);

/* Device counters -> host struct. Synchronizes the stream. */
CGS_API int cgs_frame_stats(const void* workspace, cgs_frame_stats_t* out_host, cgs_stream_t stream);

/* The frame accessors below re-derive the workspace layout from the same
 * (cams, n_views, n, pair_capacity, sr_capacity) the forward was given. */

/* RenderArtifacts.tile_splats (render.py:296-302) as CSR: for view v and
 * row-major tile t, ids[offsets[v*T+t] .. offsets[v*T+t+1]) are Gaussian
 * indices in compositing order.  offsets: total_tiles+1 int64, ids: P int32. */
CGS_API int cgs_frame_tile_lists(const cgs_camera_t* cams, int32_t n_views, int64_t n,
                         int64_t pair_capacity, int64_t sr_capacity, const void* workspace,
                         size_t workspace_bytes, int64_t* offsets, int32_t* ids,
                         cgs_stream_t stream);

/* Per-splat projection records for view v (for stage parity): mean2d (N,2)
 * f64, conic (N,3) f64 [A,B,C], opacity (N) f64, color (N,3) f32, n_tiles (N)
 * u32 (0 = culled or empty rect); only splats with n_tiles > 0 are defined. */
CGS_API int cgs_frame_splats(const cgs_camera_t* cams, int32_t n_views, int64_t n, int64_t pair_capacity,
                     int64_t sr_capacity, const void* workspace, size_t workspace_bytes,
                     int32_t view, double* mean2d, double* conic, double* opacity, float* color,
                     uint32_t* n_tiles, cgs_stream_t stream);

CGS_API size_t cgs_backward_workspace_bytes(int64_t n, const cgs_camera_t* cams, int32_t n_views,
                                    int64_t pair_capacity, int64_t sh_capacity,
                                    int64_t sr_capacity);

/* rasterize_backward + _pull_back (render.py:318-459), reusing the frame's
 * (tile, depth)-sorted pairs: reverse-order tile blend with in-CTA warp
 * reductions (one 9-float partial per processed pair); per splat a
 * fixed-order walk of its pairs (row-major tile order) through the inverse
 * pair map + fp64 chain rule; per codebook row a segmented reduction over
 * its members (render.py:456-458) -- no atomics, no per-step sorts.
 * The code -> members CSRs (cgs_code_csr) are optional: pass NULL to have
 * them built in the workspace (two extra sorts).  All four gradient arrays
 * are fully written (zeros where the reference writes zeros), multiplied by
 * `scale`.  final_T is the forward's output.  Deterministic. */
CGS_API int cgs_render_backward(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                        const void* frame_ws, size_t frame_ws_bytes, int64_t pair_capacity,
                        const float* final_T, const float* dL_dimage, float scale,
                        const int32_t* sh_csr_offsets, const int32_t* sh_csr_members,
                        const int32_t* sr_csr_offsets, const int32_t* sr_csr_members,
                        void* workspace, size_t workspace_bytes,
                        float* grad_positions, float* grad_logits,
                        float* grad_sh_rows, float* grad_sr_rows, cgs_stream_t stream);

/* ---- staged entry points (SURVEY.md 8(b) proposed exports) ----------- */
/* cgs_render_forward = cgs_project -> cgs_sort_depth -> cgs_duplicate_tiles
 * -> cgs_sort_pairs -> cgs_raster_fwd on the same frame workspace and
 * arguments, in that order on one stream (bit-identical results); likewise
 * cgs_render_backward = cgs_raster_bwd -> cgs_gaussian_reduce_pullback ->
 * cgs_codebook_reduce on the same backward workspace.  Stages read only what
 * the earlier stages left in the workspaces.
 *   project        render.py:145-203  fp64 projection, SH colour, pixel rect,
 *                  contribution box, depth keys (+ depth-key histograms)
 *   sort_depth     render.py:203      stable depth order (lexsort (idx, tz)),
 *                  per-splat pair offsets, pair count / overflow stats
 *   duplicate      render.py:240-254  (tile, splat) pairs in depth order
 *   sort_pairs     render.py:240-254  stable tile sort, tile ranges
 *   raster_fwd     render.py:287-315  blend, T, counts (+ chunk checkpoints)
 *   raster_bwd     render.py:318-379  per processed pair 9-float partials
 *   gaussian_reduce_pullback render.py:382-455 per splat sums + fp64 chain
 *                  rule; grad_positions / grad_logits fully written (x scale)
 *   codebook_reduce render.py:456-458 per code row segmented sums (CSRs
 *                  optional, NULL = build in the workspace); grads x scale */
CGS_API int cgs_project(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                        void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                        cgs_stream_t stream);
CGS_API int cgs_sort_depth(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                           void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                           cgs_stream_t stream);
CGS_API int cgs_duplicate_tiles(const cgs_scene_t* scene, const cgs_camera_t* cams,
                                int32_t n_views, void* workspace, size_t workspace_bytes,
                                int64_t pair_capacity, cgs_stream_t stream);
CGS_API int cgs_sort_pairs(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                           void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                           cgs_stream_t stream);
CGS_API int cgs_raster_fwd(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                           void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                           float* image, float* final_T, int32_t* contrib_counts,
                           cgs_stream_t stream);
CGS_API int cgs_raster_bwd(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                           const void* frame_ws, size_t frame_ws_bytes, int64_t pair_capacity,
                           const float* final_T, const float* dL_dimage, void* workspace,
                           size_t workspace_bytes, cgs_stream_t stream);
CGS_API int cgs_gaussian_reduce_pullback(const cgs_scene_t* scene, const cgs_camera_t* cams,
                                         int32_t n_views, const void* frame_ws,
                                         size_t frame_ws_bytes, int64_t pair_capacity,
                                         float scale, void* workspace, size_t workspace_bytes,
                                         float* grad_positions, float* grad_logits,
                                         cgs_stream_t stream);
CGS_API int cgs_codebook_reduce(const cgs_scene_t* scene, const cgs_camera_t* cams,
                                int32_t n_views, const void* frame_ws, size_t frame_ws_bytes,
                                int64_t pair_capacity, float scale,
                                const int32_t* sh_csr_offsets, const int32_t* sh_csr_members,
                                const int32_t* sr_csr_offsets, const int32_t* sr_csr_members,
                                void* workspace, size_t workspace_bytes, float* grad_sh_rows,
                                float* grad_sr_rows, cgs_stream_t stream);

/* code -> members CSR of an index array (g2sh or g2sr): offsets (capacity+1)
 * and members (n, ascending Gaussian index within each row).  Rebuild only
 * when assignments change (split / merge / densify). */
CGS_API size_t cgs_code_csr_workspace_bytes(int64_t n, int64_t capacity);
CGS_API int cgs_code_csr(const int32_t* idx, int64_t n, int64_t capacity, int32_t* offsets,
                         int32_t* members, void* workspace, size_t workspace_bytes,
                         cgs_stream_t stream);

/* ---- loss: recon_loss / recon_loss_grad (metrics.py:122-140) --------- */
CGS_API size_t cgs_loss_workspace_bytes(int32_t n_views, int32_t height, int32_t width);

/* Per view v: losses[3v..3v+2] = (l1, ssim, recon) as f64.  SSIM is computed
 * when lambda != 0 or want_ssim != 0 and both sides are >= 11 (else NaN,
 * metrics.py:126-128); if dL_dimage is non-null it receives d recon / d image
 * scaled by grad_scale.  lambda != 0 with a side < 11 is CGS_EINVAL. */
CGS_API int cgs_recon_loss(const float* image, const float* gt, int32_t n_views, int32_t height,
                   int32_t width, double lambda_ssim, int32_t want_ssim, float grad_scale,
                   float* dL_dimage, double* losses, void* workspace, size_t workspace_bytes,
                   cgs_stream_t stream);

/* 8-bit image output: out[i] = clip(rint(values[i] * 255), 0, 255) with the
 * product and rounding in float64 (round half to even) -- the bytes the
 * reference's save_png writes for a rendered image and the grid of its
 * quantize8 (modelio.py:137-153; cli.py:209-237 cmd_render / cmd_eval).
 * values, out: device, n entries (an HxWx3 image: n = 3 H W). */
CGS_API int cgs_quantize8(const float* values, int64_t n, uint8_t* out, cgs_stream_t stream);

/* Device address of the backward workspace's non-finite flag: nonzero when
 * any gradient entry cgs_render_backward (or the staged backward) wrote was
 * non-finite.  Pure address arithmetic on the workspace pointer. */
CGS_API const int32_t* cgs_backward_nonfinite_flag(const void* backward_workspace);

/* ---- SGLD update (sampler.py:262-300) --------------------------------- */
/* Checks every gradient for finiteness first; if any is non-finite nothing
 * is written and flags[0] |= 1 (host raises SamplerError); params.skip_if
 * set likewise writes nothing (flags[0] |= 2).  Live rows are
 * given as index lists; the finiteness check covers all sh_capacity /
 * sr_capacity gradient rows (GradientSet.all_finite, render.py:222-224).
 * Parity noise arrays (noise_source 1) hold the reference's standard
 * normals: (N,3), (N,), (live_sh, D), (live_sr, 7). */
CGS_API int cgs_sgld_update(float* positions, float* opacity_logits, int64_t n,
                    float* sh_rows, int32_t sh_dim, const int32_t* sh_live, int64_t n_sh_live,
                    float* sr_rows, const int32_t* sr_live, int64_t n_sr_live,
                    int64_t sh_capacity, int64_t sr_capacity,
                    const float* grad_positions, const float* grad_logits,
                    const float* grad_sh_rows, const float* grad_sr_rows,
                    const cgs_sgld_params_t* params_host,
                    const double* noise_pos, const double* noise_logit,
                    const double* noise_sh, const double* noise_sr,
                    int32_t* flags, cgs_stream_t stream);

/* ---- MCMC host helpers (sampler.py:339-364), host memory, no CUDA ------ */
/* Ascending ids i < n with refcount[idx[i]] >= 2 (sampler.py:344) into out
 * (capacity n); count in *n_out.  `threads` host threads. */
CGS_API int cgs_host_split_eligible(const int32_t* idx, int64_t n, const int64_t* refcount,
                                    int64_t k, int32_t* out, int64_t* n_out, int32_t threads);
/* The split accept loop over n_cand candidates in order (sampler.py:349-364):
 * a candidate whose row has refcount < 2 is skipped with no draws
 * (decision -1); otherwise u = rng.normal(0, eps_split, dim) (numpy's own
 * random_normal on `bitgen`, the bitgen_t of rng.bit_generator.capsule),
 * log A = -lam - (-0.5 |u|^2 c_q [+ corr]) with |u|^2 from `ddot` (numpy's
 * BLAS ddot, as `u @ u`), coin = rng.random(); accepted (decision 1) when
 * coin < exp(min(0, log A)), and then refcount[row] -= 1.  u (n_cand x dim),
 * log A and the coins are returned per candidate; *n_attempts counts the
 * non-skipped ones.  The caller allocates rows (lowest free index) after. */
CGS_API int cgs_host_split_decide(void* bitgen, void* ddot, int64_t n_cand, const int64_t* rows,
                                  int64_t* refcount, int64_t k, int32_t dim, double lam,
                                  double eps_split, double c_q, int32_t use_corr, double corr,
                                  double* u_out, double* log_a_out, double* uniform_out,
                                  int8_t* decision_out, int64_t* n_attempts);

/* ---- MCMC / densify device helpers (sampler.py:184-259, model.py:235-267) */
/* Ascending Gaussian ids i with refcount[idx[i]] >= 2 (sampler.py:344);
 * count written to *count (device int64).  Workspace from
 * cgs_scan_workspace_bytes(n). */
CGS_API int cgs_split_eligible(const int32_t* idx, int64_t n, const int32_t* refcount,
                       int32_t* eligible, int64_t* count, void* workspace,
                       size_t workspace_bytes, cgs_stream_t stream);

/* Split proposals on the device (throughput trainer, device-noise mode; the
 * reference-parity path draws on the host, cgs_host_split_decide): for each
 * candidate c, u[c] = eps_split * N(0, I_dim) and a uniform from Philox
 * (seed, counter, c); prob[c] = exp(min(0, -lam - log q)), log q =
 * -0.5 |u|^2 c_q [+ corr] (sampler.py:138-164); accept[c] = uniform <
 * prob[c].  Refcount skips (sampler.py:350-351) are the caller's.  u: (n_cand,
 * dim) f64, prob f64, accept i8, all device. */
CGS_API int cgs_split_propose(int64_t n_cand, int32_t dim, double eps_split, double c_q,
                              int32_t use_corr, double corr, double lam, uint64_t seed,
                              uint64_t counter, double* u, double* prob, int8_t* accept,
                              cgs_stream_t stream);

/* Accepted splits in proposal order (sampler.py:202-209): for each j,
 * rows[new_row[j]] = f32(f64(rows[old_row[j]]) + u[j]) and idx[gauss[j]] =
 * new_row[j].  u: (k, dim) f64. */
CGS_API int cgs_apply_splits(float* rows, int32_t dim, int32_t* idx, const int64_t* gauss,
                     const int32_t* old_row, const int32_t* new_row, const double* u,
                     int64_t k, cgs_stream_t stream);

/* Accepted merges composed into one row remap (sampler.py:240-247):
 * idx[i] = remap[idx[i]] where remap[r] >= 0. */
CGS_API int cgs_apply_remap(int32_t* idx, int64_t n, const int32_t* remap, int64_t remap_len,
                    cgs_stream_t stream);

/* densify clones (model.py:256-266): Gaussian n+j copies src[j] with
 * position f32(f64(pos[src[j]]) + jitter[j]). */
CGS_API int cgs_densify_append(float* positions, float* opacity_logits, int32_t* g2sh, int32_t* g2sr,
                       int64_t n, const int64_t* src, const double* jitter, int64_t k,
                       cgs_stream_t stream);

/* densify sources on the device (throughput mode; replaces the host
 * rng.choice(n, k, p=sigmoid(logit)/sum) of model.py:256 with the same
 * host-drawn uniforms, see update.cu): src[j] = first i with
 * cumsum(sigmoid(logit))[i] > uniforms[j] * total (fixed point 2^-40). */
CGS_API size_t cgs_densify_select_workspace_bytes(int64_t n);
CGS_API int cgs_densify_select(const float* opacity_logits, int64_t n, const double* uniforms,
                               int64_t k, int64_t* src, void* ws, size_t ws_bytes,
                               cgs_stream_t stream);

/* ---- nearest code rows (code reassignment extension) ------------------ */
/* No reference counterpart: the reference never recomputes assignments by
 * distance.  For every live row i (indices
 * `live`, n_live of them) of rows (capacity x dim, dim <= 48 = SH degree 3):
 *   nn_index[i] = argmin over live j != i of sum_k fl(fl(r_ik - r_jk)^2)
 *   (fp64, sequential in k, ties -> smaller j), nn_dist2[i] = that sum;
 * -1 / 0 for rows that are not live (or when n_live < 2).  Candidates come
 * from a tcgen05 3xTF32 distance GEMM; an fp64 check with a rounding bound
 * (and an fp64 brute force for any row it cannot certify) makes the result
 * exact. */
CGS_API size_t cgs_code_nn_workspace_bytes(int64_t n_live, int32_t dim);
CGS_API int cgs_code_nn(const float* rows, int32_t dim, int64_t capacity, const int32_t* live,
                        int64_t n_live, int32_t* nn_index, double* nn_dist2, void* workspace,
                        size_t workspace_bytes, cgs_stream_t stream);

/* counts[r] = #{i : idx[i] == r} (validate_state, model.py:297). */
CGS_API int cgs_refcount_histogram(const int32_t* idx, int64_t n, int32_t* counts, int64_t capacity,
                           cgs_stream_t stream);

/* ---- primitives (exported for unit tests) ---------------------------- */
CGS_API size_t cgs_scan_workspace_bytes(int64_t n);
/* exclusive prefix sum of u32 into u32; total into *total (device u64). */
CGS_API int cgs_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint64_t* total,
                           void* workspace, size_t workspace_bytes, cgs_stream_t stream);

CGS_API size_t cgs_sort_workspace_bytes(int64_t n, int32_t key_bytes);
/* Stable LSD onesweep radix sort of (key, value) pairs on the low key_bits.
 * key_bytes in {2,4,8}.  keys/vals are sorted in place (alt buffers of the
 * same size are carved from the workspace). */
CGS_API int cgs_radix_sort_pairs(void* keys, uint32_t* vals, int64_t n, int32_t key_bytes,
                         int32_t key_bits, void* workspace, size_t workspace_bytes,
                         cgs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CGS_B200_H */
