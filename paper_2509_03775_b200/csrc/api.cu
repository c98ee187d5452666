// C ABI (include/cgs_b200.h): argument checking, workspace planning and the
// error channel.  No C++ exception crosses this boundary.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "frame.cuh"

namespace cgs {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

// ---- instrumentation -----------------------------------------------------
static std::atomic<unsigned long long> g_launches{0};
static std::mutex g_prof_mu;
static std::string g_prof_name;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_events;
static std::vector<cudaEvent_t> g_prof_pool;
static unsigned long long* g_tile_trace = nullptr;

unsigned long long* tile_trace_buffer() { return g_tile_trace; }

static std::mutex g_side_mu[kMaxDevices];
static cudaStream_t g_side[kMaxDevices] = {};
static cudaEvent_t g_side_ev[kMaxDevices][2] = {};

SideFork::SideFork(cudaStream_t st) : main(st) {
  if ((rc = current_device(&dev)) != 0) return;
  g_side_mu[dev].lock();
  cudaError_t e = cudaSuccess;
  if (!g_side[dev]) {
    e = cudaStreamCreateWithFlags(&g_side[dev], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_side_ev[dev][0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_side_ev[dev][1], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventRecord(g_side_ev[dev][0], st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(g_side[dev], g_side_ev[dev][0], 0);
  if (e != cudaSuccess) {
    rc = cuda_status(e, "side stream fork");
    return;
  }
  side = g_side[dev];
}

int SideFork::join() {
  if (!side) return rc;
  cudaError_t e = cudaEventRecord(g_side_ev[dev][1], side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(main, g_side_ev[dev][1], 0);
  side = nullptr;
  if (e != cudaSuccess) rc = cuda_status(e, "side stream join");
  return rc;
}

SideFork::~SideFork() {
  join();
  if (dev >= 0) g_side_mu[dev].unlock();
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int current_device(int* dev) {
  int d = 0;
  CGS_CUDA(cudaGetDevice(&d));
  if (d < 0 || d >= kMaxDevices) {
    set_error("device ordinal out of range");
    return CGS_EINTERNAL;
  }
  *dev = d;
  return CGS_OK;
}

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(const char* name, cudaStream_t s) : on(false), st(s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_name.empty() && g_prof_name == name) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) return;  // events are not re-armed per replay
    on = true;
    cudaEvent_t a = prof_event(), b = prof_event();
    cudaEventRecord(a, st);
    g_prof_events.emplace_back(a, b);
  }
}

ProfScope::~ProfScope() {
  if (!on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEventRecord(g_prof_events.back().second, st);
}

int cuda_status(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return CGS_ECUDA;
}

// defined in the kernel translation units
int frame_forward(const cgs_scene_t* sc, const FrameDesc& fd, FrameLayout& L, float* image,
                  float* final_T, int32_t* counts, double* sr_cov, cudaStream_t st);
int frame_stage_project(const cgs_scene_t* sc, const FrameDesc& fd, FrameLayout& L,
                        double* sr_cov, cudaStream_t st);
int frame_stage_sort_depth(const FrameDesc& fd, FrameLayout& L, cudaStream_t st);
int frame_stage_duplicate(const FrameDesc& fd, FrameLayout& L, cudaStream_t st);
int frame_stage_sort_pairs(const FrameDesc& fd, FrameLayout& L, cudaStream_t st);
int frame_stage_raster(const FrameDesc& fd, FrameLayout& L, const float* logits, float* image,
                       float* final_T,
                       int32_t* counts, cudaStream_t st);
struct BwdLayout;
int bwd_stage_entry(int stage, const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                    void* ws, size_t ws_bytes, const float* dL, const float* final_T, float scale,
                    float* gpos, float* glogit, float* gsh, float* gsr,
                    const int32_t* const csr_off[2], const int32_t* const csr_mem[2],
                    cudaStream_t st);
size_t bwd_ws_bytes(int64_t n, int n_views, int total_tiles, int64_t pair_cap, int64_t sh_cap,
                    int64_t sr_cap);
int frame_backward_entry(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                         void* ws, size_t ws_bytes, const float* dL, const float* final_T,
                         float scale, float* gpos, float* glogit, float* gsh, float* gsr,
                         const int32_t* const csr_off[2], const int32_t* const csr_mem[2],
                         cudaStream_t st);
size_t code_csr_ws_bytes(int64_t n, int64_t cap);
int build_code_csr(const int32_t* idx, int64_t n, int64_t cap, int32_t* off, int32_t* mem,
                   void* ws, size_t ws_bytes, cudaStream_t st);
size_t loss_ws_bytes(int nv, int h, int w);
int recon_loss(const float* img, const float* gt, int nv, int H, int W, double lam, float gscale,
               float* dL, double* losses, int want_ssim, void* ws, size_t ws_bytes,
               cudaStream_t st);
int sgld_update(float* pos, float* logit, int64_t n, float* sh, int D, const int32_t* sh_live,
                int64_t n_sh, float* sr, const int32_t* sr_live, int64_t n_sr, const float* gpos,
                const float* glogit, const float* gsh, const float* gsr, int64_t sh_cap,
                int64_t sr_cap, const cgs_sgld_params_t* hp, const double* npos,
                const double* nlog, const double* nsh, const double* nsr, int32_t* flags,
                cudaStream_t st);
int quantize8(const float* x, int64_t n, uint8_t* out, cudaStream_t st);
int split_eligible(const int32_t* idx, int64_t n, const int32_t* rc, int32_t* out, int64_t* count,
                   void* ws, size_t ws_bytes, cudaStream_t st);
int apply_splits(float* rows, int dim, int32_t* idx, const int64_t* gauss, const int32_t* old_row,
                 const int32_t* new_row, const double* u, int64_t k, cudaStream_t st);
int split_propose(int64_t n_cand, int dim, double es, double c_q, int use_corr, double corr,
                  double lam, uint64_t seed, uint64_t ctr, double* u, double* prob, int8_t* accept,
                  cudaStream_t st);
int apply_remap(int32_t* idx, int64_t n, const int32_t* remap, int64_t len, cudaStream_t st);
int densify_append(float* pos, float* logit, int32_t* g2sh, int32_t* g2sr, int64_t n,
                   const int64_t* src, const double* jit, int64_t k, cudaStream_t st);
size_t densify_select_ws_bytes(int64_t n);
int densify_select(const float* logit, int64_t n, const double* u, int64_t k, int64_t* src,
                   void* ws, size_t ws_bytes, cudaStream_t st);
int refcount_histogram(const int32_t* idx, int64_t n, int32_t* counts, int64_t cap,
                       cudaStream_t st);

static int check_cams(const cgs_camera_t* cams, int nv) {
  if (nv < 1 || nv > CGS_MAX_VIEWS) {
    set_error("n_views must be in 1.." + std::to_string(CGS_MAX_VIEWS));
    return CGS_EINVAL;
  }
  if (!cams) {
    set_error("cams is null");
    return CGS_EINVAL;
  }
  for (int v = 0; v < nv; ++v) {
    if (!(cams[v].fx > 0 && cams[v].fy > 0)) {
      set_error("focal lengths must be positive");
      return CGS_EINVAL;
    }
    if (cams[v].width < 1 || cams[v].height < 1 || cams[v].width > 65535 * 16 ||
        cams[v].height > 65535 * 16) {
      set_error("image dimensions out of range");
      return CGS_EINVAL;
    }
  }
  return CGS_OK;
}

static int check_scene(const cgs_scene_t* sc) {
  if (!sc) {
    set_error("scene is null");
    return CGS_EINVAL;
  }
  if (sc->sh_degree < 0 || sc->sh_degree > 3) {
    set_error("sh_degree must be in 0..3");
    return CGS_EINVAL;
  }
  if (sc->n < 0) {
    set_error("negative Gaussian count");
    return CGS_EINVAL;
  }
  return CGS_OK;
}

}  // namespace cgs

using namespace cgs;

extern "C" {

int cgs_abi_version(void) { return CGS_ABI_VERSION; }

const char* cgs_last_error(void) { return g_err.c_str(); }

uint64_t cgs_launch_count(void) { return g_launches.load(); }

int cgs_profile_kernel(const char* name) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& pr : g_prof_events) {
    g_prof_pool.push_back(pr.first);
    g_prof_pool.push_back(pr.second);
  }
  g_prof_events.clear();
  g_prof_name = name ? name : "";
  return CGS_OK;
}

int cgs_trace_tiles(void* dev_buf) {
  g_tile_trace = static_cast<unsigned long long*>(dev_buf);
  return CGS_OK;
}

int cgs_profile_read(double* total_ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double tot = 0.0;
  for (auto& pr : g_prof_events) {
    CGS_CUDA(cudaEventSynchronize(pr.second));
    float ms = 0.0f;
    CGS_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = static_cast<int64_t>(g_prof_events.size());
  return CGS_OK;
}

size_t cgs_frame_workspace_bytes(int64_t n, const cgs_camera_t* cams, int32_t n_views,
                                 int64_t pair_capacity, int64_t sr_capacity) {
  if (check_cams(cams, n_views)) return 0;
  FrameDesc fd = make_frame_desc(cams, n_views);
  return plan_frame(nullptr, 0, n, fd, pair_capacity, sr_capacity).bytes;
}

int cgs_render_forward(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                       void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                       float* image, float* final_T, int32_t* contrib_counts,
                       cgs_stream_t stream) {
  int rc = check_scene(scene);
  if (rc) return rc;
  rc = check_cams(cams, n_views);
  if (rc) return rc;
  FrameDesc fd = make_frame_desc(cams, n_views);
  FrameLayout L = plan_frame(workspace, workspace_bytes, scene->n, fd, pair_capacity,
                             scene->sr_capacity);
  if (L.bytes > workspace_bytes || !workspace) {
    set_error("frame workspace too small: need " + std::to_string(L.bytes));
    return CGS_EWORKSPACE;
  }
  if (scene->n * n_views >= (1LL << 32) - 1) {
    set_error("views * Gaussians must be < 2^32");
    return CGS_EINVAL;
  }
  return frame_forward(scene, fd, L, image, final_T, contrib_counts, L.sr_cov,
                       static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// validated scene, frame descriptor and layout for the staged entry points
static int staged_frame(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                        const void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                        FrameDesc* fd, FrameLayout* L) {
  int rc = check_scene(scene);
  if (rc) return rc;
  rc = check_cams(cams, n_views);
  if (rc) return rc;
  *fd = make_frame_desc(cams, n_views);
  *L = plan_frame(const_cast<void*>(workspace), workspace_bytes, scene->n, *fd, pair_capacity,
                  scene->sr_capacity);
  if (L->bytes > workspace_bytes || !workspace) {
    set_error("frame workspace too small: need " + std::to_string(L->bytes));
    return CGS_EWORKSPACE;
  }
  if (scene->n * n_views >= (1LL << 32) - 1) {
    set_error("views * Gaussians must be < 2^32");
    return CGS_EINVAL;
  }
  return CGS_OK;
}

extern "C" {

#define CGS_STAGE_PROLOGUE                                                                   \
  FrameDesc fd;                                                                              \
  FrameLayout L;                                                                             \
  int rc = staged_frame(scene, cams, n_views, workspace, workspace_bytes, pair_capacity, &fd, \
                        &L);                                                                 \
  if (rc) return rc;                                                                         \
  cudaStream_t st = static_cast<cudaStream_t>(stream)

int cgs_project(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                cgs_stream_t stream) {
  CGS_STAGE_PROLOGUE;
  return frame_stage_project(scene, fd, L, L.sr_cov, st);
}

int cgs_sort_depth(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                   void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                   cgs_stream_t stream) {
  CGS_STAGE_PROLOGUE;
  return frame_stage_sort_depth(fd, L, st);
}

int cgs_duplicate_tiles(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                        void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                        cgs_stream_t stream) {
  CGS_STAGE_PROLOGUE;
  return frame_stage_duplicate(fd, L, st);
}

int cgs_sort_pairs(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                   void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                   cgs_stream_t stream) {
  CGS_STAGE_PROLOGUE;
  return frame_stage_sort_pairs(fd, L, st);
}

int cgs_raster_fwd(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                   void* workspace, size_t workspace_bytes, int64_t pair_capacity, float* image,
                   float* final_T, int32_t* contrib_counts, cgs_stream_t stream) {
  CGS_STAGE_PROLOGUE;
  return frame_stage_raster(fd, L, scene->opacity_logits, image, final_T, contrib_counts, st);
}

const int32_t* cgs_backward_nonfinite_flag(const void* backward_workspace) {
  // BwdHeader.nonfinite (render_bwd.cu) sits at byte 16 of the workspace
  return backward_workspace
             ? reinterpret_cast<const int32_t*>(static_cast<const char*>(backward_workspace) + 16)
             : nullptr;
}

int cgs_frame_stats(const void* workspace, cgs_frame_stats_t* out, cgs_stream_t stream) {
  if (!workspace || !out) {
    set_error("null argument");
    return CGS_EINVAL;
  }
  const FrameHeader* h = static_cast<const FrameHeader*>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FrameHeader hh;
  CGS_CUDA(cudaMemcpyAsync(&hh, h, sizeof(FrameHeader), cudaMemcpyDeviceToHost, st));
  CGS_CUDA(cudaStreamSynchronize(st));
  *out = hh.stats;
  // the float64 re-walk's counters, kept where the refine kernels count them
  // (no publishing kernel in the step)
  out->n_refined_tiles = static_cast<int64_t>(hh.scratch[3]);
  out->n_refined_pixels = static_cast<int64_t>(hh.scratch[4]);
  out->diag_last_mismatch = static_cast<int64_t>(hh.scratch[5]);
  out->diag_count_mismatch = static_cast<int64_t>(hh.scratch[6]);
  const uint32_t te = static_cast<uint32_t>(hh.scratch[7]), ae = static_cast<uint32_t>(hh.scratch[7] >> 32);
  std::memcpy(&out->diag_max_T_err, &te, sizeof(float));
  std::memcpy(&out->diag_max_alpha_err, &ae, sizeof(float));
  return CGS_OK;
}

}  // extern "C"

namespace cgs {

// tile lists: offsets from ranges, ids = splat id mod n
__global__ void tile_offsets_kernel(const uint2* ranges, int total_tiles, const FrameHeader* h,
                                    int64_t* offsets) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < total_tiles) {
    const uint2 r = ranges[t];
    offsets[t] = r.x < r.y ? static_cast<int64_t>(r.x) : -1;
  }
  if (t == 0) offsets[total_tiles] = static_cast<int64_t>(h->n_pairs);
}

// empty tiles get the next non-empty start (backward fill, sequential)
__global__ void tile_offsets_fill_kernel(int64_t* offsets, int total_tiles) {
  for (int t = total_tiles - 1; t >= 0; --t)
    if (offsets[t] < 0) offsets[t] = offsets[t + 1];
}

__global__ void tile_ids_kernel(const uint32_t* vals, const FrameHeader* h, int64_t n,
                                int32_t* ids) {
  const int64_t np = static_cast<int64_t>(h->n_pairs);
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < np;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ids[p] = static_cast<int32_t>(vals[p] % static_cast<uint32_t>(n));
}

__global__ void splats_kernel(const SplatRec* recs, const uint32_t* ntl, int64_t n, int view,
                              double* mean2d, double* conic, double* opac, float* color,
                              uint32_t* nt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = static_cast<int64_t>(view) * n + i;
    const uint32_t k = ntl[s];
    nt[i] = k;
    if (k == 0) continue;
    const SplatRec r = recs[s];
    mean2d[2 * i] = r.mx;
    mean2d[2 * i + 1] = r.my;
    conic[3 * i] = r.ca;
    conic[3 * i + 1] = r.cb;
    conic[3 * i + 2] = r.cc;
    opac[i] = r.opac;
    color[3 * i] = r.r;
    color[3 * i + 1] = r.g;
    color[3 * i + 2] = r.b;
  }
}

}  // namespace cgs

extern "C" {

int cgs_frame_tile_lists(const cgs_camera_t* cams, int32_t n_views, int64_t n,
                         int64_t pair_capacity, int64_t sr_capacity, const void* workspace,
                         size_t workspace_bytes, int64_t* offsets, int32_t* ids,
                         cgs_stream_t stream) {
  int rc = check_cams(cams, n_views);
  if (rc) return rc;
  FrameDesc fd = make_frame_desc(cams, n_views);
  FrameLayout L = plan_frame(const_cast<void*>(workspace), workspace_bytes, n, fd, pair_capacity,
                             sr_capacity);
  if (L.bytes > workspace_bytes) {
    set_error("frame workspace too small");
    return CGS_EWORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tile_offsets_kernel<<<(fd.total_tiles + 255) / 256 + 1, 256, 0, st>>>(L.ranges, fd.total_tiles,
                                                                        L.hdr, offsets);
  CGS_CHECK_LAUNCH("tile_offsets_kernel");
  tile_offsets_fill_kernel<<<1, 1, 0, st>>>(offsets, fd.total_tiles);
  CGS_CHECK_LAUNCH("tile_offsets_fill_kernel");
  if (n > 0) {
    tile_ids_kernel<<<grid_for(pair_capacity, 256, 8), 256, 0, st>>>(sorted_pair_vals(L), L.hdr, n,
                                                                     ids);
    CGS_CHECK_LAUNCH("tile_ids_kernel");
  }
  return CGS_OK;
}

int cgs_frame_splats(const cgs_camera_t* cams, int32_t n_views, int64_t n, int64_t pair_capacity,
                     int64_t sr_capacity, const void* workspace, size_t workspace_bytes,
                     int32_t view, double* mean2d, double* conic, double* opacity, float* color,
                     uint32_t* n_tiles, cgs_stream_t stream) {
  int rc = check_cams(cams, n_views);
  if (rc) return rc;
  if (view < 0 || view >= n_views) {
    set_error("view out of range");
    return CGS_EINVAL;
  }
  FrameDesc fd = make_frame_desc(cams, n_views);
  FrameLayout L = plan_frame(const_cast<void*>(workspace), workspace_bytes, n, fd, pair_capacity,
                             sr_capacity);
  if (L.bytes > workspace_bytes) {
    set_error("frame workspace too small");
    return CGS_EWORKSPACE;
  }
  if (n <= 0) return CGS_OK;
  splats_kernel<<<grid_for(n, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      L.recs, L.n_tiles, n, view, mean2d, conic, opacity, color, n_tiles);
  CGS_CHECK_LAUNCH("splats_kernel");
  return CGS_OK;
}

size_t cgs_backward_workspace_bytes(int64_t n, const cgs_camera_t* cams, int32_t n_views,
                                    int64_t pair_capacity, int64_t sh_capacity,
                                    int64_t sr_capacity) {
  if (check_cams(cams, n_views)) return 0;
  FrameDesc fd = make_frame_desc(cams, n_views);
  return bwd_ws_bytes(n, n_views, fd.total_tiles, pair_capacity, sh_capacity, sr_capacity);
}

size_t cgs_code_csr_workspace_bytes(int64_t n, int64_t capacity) {
  return code_csr_ws_bytes(n, capacity);
}

int cgs_code_csr(const int32_t* idx, int64_t n, int64_t capacity, int32_t* offsets,
                 int32_t* members, void* workspace, size_t workspace_bytes, cgs_stream_t stream) {
  if (n < 0 || capacity < 0 || !offsets || (n > 0 && (!idx || !members))) {
    set_error("code_csr: invalid arguments");
    return CGS_EINVAL;
  }
  return build_code_csr(idx, n, capacity, offsets, members, workspace, workspace_bytes,
                        static_cast<cudaStream_t>(stream));
}

int cgs_render_backward(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                        const void* frame_ws, size_t frame_ws_bytes, int64_t pair_capacity,
                        const float* final_T, const float* dL_dimage, float scale,
                        const int32_t* sh_csr_offsets, const int32_t* sh_csr_members,
                        const int32_t* sr_csr_offsets, const int32_t* sr_csr_members,
                        void* workspace, size_t workspace_bytes, float* grad_positions,
                        float* grad_logits, float* grad_sh_rows, float* grad_sr_rows,
                        cgs_stream_t stream) {
  int rc = check_scene(scene);
  if (rc) return rc;
  rc = check_cams(cams, n_views);
  if (rc) return rc;
  FrameDesc fd = make_frame_desc(cams, n_views);
  FrameLayout L = plan_frame(const_cast<void*>(frame_ws), frame_ws_bytes, scene->n, fd,
                             pair_capacity, scene->sr_capacity);
  if (L.bytes > frame_ws_bytes) {
    set_error("frame workspace too small");
    return CGS_EWORKSPACE;
  }
  const int32_t* const off[2] = {sh_csr_offsets, sr_csr_offsets};
  const int32_t* const mem[2] = {sh_csr_members, sr_csr_members};
  return frame_backward_entry(scene, fd, L, workspace, workspace_bytes, dL_dimage, final_T, scale,
                              grad_positions, grad_logits, grad_sh_rows, grad_sr_rows, off, mem,
                              static_cast<cudaStream_t>(stream));
}

static int bwd_stage(int stage, const cgs_scene_t* scene, const cgs_camera_t* cams,
                     int32_t n_views, const void* frame_ws, size_t frame_ws_bytes,
                     int64_t pair_capacity, void* workspace, size_t workspace_bytes,
                     const float* final_T, const float* dL, float scale, float* gpos,
                     float* glogit, float* gsh, float* gsr, const int32_t* const off[2],
                     const int32_t* const mem[2], cgs_stream_t stream) {
  FrameDesc fd;
  FrameLayout L;
  int rc = staged_frame(scene, cams, n_views, frame_ws, frame_ws_bytes, pair_capacity, &fd, &L);
  if (rc) return rc;
  return bwd_stage_entry(stage, scene, fd, L, workspace, workspace_bytes, dL, final_T, scale, gpos,
                         glogit, gsh, gsr, off, mem, static_cast<cudaStream_t>(stream));
}

int cgs_raster_bwd(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                   const void* frame_ws, size_t frame_ws_bytes, int64_t pair_capacity,
                   const float* final_T, const float* dL_dimage, void* workspace,
                   size_t workspace_bytes, cgs_stream_t stream) {
  return bwd_stage(0, scene, cams, n_views, frame_ws, frame_ws_bytes, pair_capacity, workspace,
                   workspace_bytes, final_T, dL_dimage, 1.0f, nullptr, nullptr, nullptr, nullptr,
                   nullptr, nullptr, stream);
}

int cgs_gaussian_reduce_pullback(const cgs_scene_t* scene, const cgs_camera_t* cams,
                                 int32_t n_views, const void* frame_ws, size_t frame_ws_bytes,
                                 int64_t pair_capacity, float scale, void* workspace,
                                 size_t workspace_bytes, float* grad_positions,
                                 float* grad_logits, cgs_stream_t stream) {
  return bwd_stage(1, scene, cams, n_views, frame_ws, frame_ws_bytes, pair_capacity, workspace,
                   workspace_bytes, nullptr, nullptr, scale, grad_positions, grad_logits, nullptr,
                   nullptr, nullptr, nullptr, stream);
}

int cgs_codebook_reduce(const cgs_scene_t* scene, const cgs_camera_t* cams, int32_t n_views,
                        const void* frame_ws, size_t frame_ws_bytes, int64_t pair_capacity,
                        float scale, const int32_t* sh_csr_offsets,
                        const int32_t* sh_csr_members, const int32_t* sr_csr_offsets,
                        const int32_t* sr_csr_members, void* workspace, size_t workspace_bytes,
                        float* grad_sh_rows, float* grad_sr_rows, cgs_stream_t stream) {
  const int32_t* const off[2] = {sh_csr_offsets, sr_csr_offsets};
  const int32_t* const mem[2] = {sh_csr_members, sr_csr_members};
  return bwd_stage(2, scene, cams, n_views, frame_ws, frame_ws_bytes, pair_capacity, workspace,
                   workspace_bytes, nullptr, nullptr, scale, nullptr, nullptr, grad_sh_rows,
                   grad_sr_rows, off, mem, stream);
}

size_t cgs_loss_workspace_bytes(int32_t n_views, int32_t height, int32_t width) {
  return loss_ws_bytes(n_views, height, width);
}

int cgs_recon_loss(const float* image, const float* gt, int32_t n_views, int32_t height,
                   int32_t width, double lambda_ssim, int32_t want_ssim, float grad_scale,
                   float* dL_dimage, double* losses, void* workspace, size_t workspace_bytes,
                   cgs_stream_t stream) {
  if (n_views < 1 || height < 1 || width < 1 || !image || !gt || !losses) {
    set_error("recon_loss: invalid arguments");
    return CGS_EINVAL;
  }
  return recon_loss(image, gt, n_views, height, width, lambda_ssim, grad_scale, dL_dimage, losses,
                    want_ssim, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

int cgs_sgld_update(float* positions, float* opacity_logits, int64_t n, float* sh_rows,
                    int32_t sh_dim, const int32_t* sh_live, int64_t n_sh_live, float* sr_rows,
                    const int32_t* sr_live, int64_t n_sr_live, int64_t sh_capacity,
                    int64_t sr_capacity, const float* grad_positions, const float* grad_logits,
                    const float* grad_sh_rows, const float* grad_sr_rows,
                    const cgs_sgld_params_t* params_host, const double* noise_pos,
                    const double* noise_logit, const double* noise_sh, const double* noise_sr,
                    int32_t* flags, cgs_stream_t stream) {
  if (!params_host || !flags || n < 0 || sh_dim < 1) {
    set_error("sgld_update: invalid arguments");
    return CGS_EINVAL;
  }
  return sgld_update(positions, opacity_logits, n, sh_rows, sh_dim, sh_live, n_sh_live, sr_rows,
                     sr_live, n_sr_live, grad_positions, grad_logits, grad_sh_rows, grad_sr_rows,
                     sh_capacity, sr_capacity, params_host, noise_pos, noise_logit, noise_sh,
                     noise_sr, flags, static_cast<cudaStream_t>(stream));
}

int cgs_quantize8(const float* values, int64_t n, uint8_t* out, cgs_stream_t stream) {
  if (n < 0 || (n > 0 && (!values || !out))) {
    set_error("quantize8: invalid arguments");
    return CGS_EINVAL;
  }
  return quantize8(values, n, out, static_cast<cudaStream_t>(stream));
}

int cgs_split_eligible(const int32_t* idx, int64_t n, const int32_t* refcount, int32_t* eligible,
                       int64_t* count, void* workspace, size_t workspace_bytes,
                       cgs_stream_t stream) {
  return split_eligible(idx, n, refcount, eligible, count, workspace, workspace_bytes,
                        static_cast<cudaStream_t>(stream));
}

int cgs_split_propose(int64_t n_cand, int32_t dim, double eps_split, double c_q, int32_t use_corr,
                      double corr, double lam, uint64_t seed, uint64_t counter, double* u,
                      double* prob, int8_t* accept, cgs_stream_t stream) {
  if (n_cand < 0 || dim < 1 || (n_cand > 0 && (!u || !prob || !accept))) {
    set_error("split_propose: invalid arguments");
    return CGS_EINVAL;
  }
  return split_propose(n_cand, dim, eps_split, c_q, use_corr, corr, lam, seed, counter, u, prob,
                       accept, static_cast<cudaStream_t>(stream));
}

int cgs_apply_splits(float* rows, int32_t dim, int32_t* idx, const int64_t* gauss,
                     const int32_t* old_row, const int32_t* new_row, const double* u, int64_t k,
                     cgs_stream_t stream) {
  return apply_splits(rows, dim, idx, gauss, old_row, new_row, u, k,
                      static_cast<cudaStream_t>(stream));
}

int cgs_apply_remap(int32_t* idx, int64_t n, const int32_t* remap, int64_t remap_len,
                    cgs_stream_t stream) {
  return apply_remap(idx, n, remap, remap_len, static_cast<cudaStream_t>(stream));
}

int cgs_densify_append(float* positions, float* opacity_logits, int32_t* g2sh, int32_t* g2sr,
                       int64_t n, const int64_t* src, const double* jitter, int64_t k,
                       cgs_stream_t stream) {
  return densify_append(positions, opacity_logits, g2sh, g2sr, n, src, jitter, k,
                        static_cast<cudaStream_t>(stream));
}

size_t cgs_densify_select_workspace_bytes(int64_t n) { return densify_select_ws_bytes(n); }

int cgs_densify_select(const float* opacity_logits, int64_t n, const double* uniforms, int64_t k,
                       int64_t* src, void* ws, size_t ws_bytes, cgs_stream_t stream) {
  return densify_select(opacity_logits, n, uniforms, k, src, ws, ws_bytes,
                        static_cast<cudaStream_t>(stream));
}

int cgs_refcount_histogram(const int32_t* idx, int64_t n, int32_t* counts, int64_t capacity,
                           cgs_stream_t stream) {
  return refcount_histogram(idx, n, counts, capacity, static_cast<cudaStream_t>(stream));
}

size_t cgs_scan_workspace_bytes(int64_t n) { return scan_ws_bytes(n) + 512; }

}  // extern "C"

namespace cgs {

struct CopyScanOp {
  const uint32_t* in;
  uint32_t* out;
  __device__ uint64_t load(int64_t i) const { return in[i]; }
  __device__ void store(int64_t i, uint64_t ex, uint64_t) const { out[i] = static_cast<uint32_t>(ex); }
  __device__ void finish(uint64_t) const {}
};

template <typename K>
static int sort_impl(void* keys, uint32_t* vals, int64_t n, int bits, void* ws, size_t wsb,
                     cudaStream_t st) {
  Carver c(ws, wsb);
  SortWs<K> w = carve_sort<K>(c, n);
  if (!c.fits()) {
    set_error("sort workspace too small");
    return CGS_EWORKSPACE;
  }
  if (n <= 0) return CGS_OK;
  K* ko;
  uint32_t* vo;
  int rc = launch_radix_sort<K>(static_cast<K*>(keys), vals, nullptr, n, n, bits, w, &ko, &vo, st);
  if (rc) return rc;
  if (ko != keys) {
    CGS_CUDA(cudaMemcpyAsync(keys, ko, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    CGS_CUDA(cudaMemcpyAsync(vals, vo, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  return CGS_OK;
}

}  // namespace cgs

extern "C" {

int cgs_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint64_t* total,
                           void* workspace, size_t workspace_bytes, cgs_stream_t stream) {
  Carver c(workspace, workspace_bytes);
  ScanWs w = carve_scan(c, n);
  if (!c.fits()) {
    set_error("scan workspace too small");
    return CGS_EWORKSPACE;
  }
  return launch_scan(CopyScanOp{in, out}, nullptr, n, n, w,
                     reinterpret_cast<unsigned long long*>(total),
                     static_cast<cudaStream_t>(stream));
}

size_t cgs_sort_workspace_bytes(int64_t n, int32_t key_bytes) {
  switch (key_bytes) {
    case 2: return sort_ws_bytes<uint16_t>(n) + 1024;
    case 4: return sort_ws_bytes<uint32_t>(n) + 1024;
    case 8: return sort_ws_bytes<uint64_t>(n) + 1024;
    default: return 0;
  }
}

int cgs_radix_sort_pairs(void* keys, uint32_t* vals, int64_t n, int32_t key_bytes,
                         int32_t key_bits, void* workspace, size_t workspace_bytes,
                         cgs_stream_t stream) {
  if (key_bits < 1 || key_bits > 8 * key_bytes) {
    set_error("key_bits out of range");
    return CGS_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (key_bytes) {
    case 2: return sort_impl<uint16_t>(keys, vals, n, key_bits, workspace, workspace_bytes, st);
    case 4: return sort_impl<uint32_t>(keys, vals, n, key_bits, workspace, workspace_bytes, st);
    case 8: return sort_impl<uint64_t>(keys, vals, n, key_bits, workspace, workspace_bytes, st);
    default:
      set_error("key_bytes must be 2, 4 or 8");
      return CGS_EINVAL;
  }
}

}  // extern "C"
