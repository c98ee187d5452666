// Shared definitions for the sm_100a kernels of the ContraGS hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/cgs_b200.h"

namespace cgs {

// reference render.py:26-34
constexpr double kNear = 0.01;
constexpr double kBlur = 0.3;
constexpr double kFootprint = 3.3290429691304455;  // sqrt(2 ln 255)
constexpr int kTile = 16;
constexpr int kTilePixels = kTile * kTile;

// The reference compares float64 values against 1/255, 0.99 and 1e-4
// (render.py:278-283).  The raster computes alpha and T in fp32; these are
// the smallest floats >= each threshold, so `x >= kF` on a float x is
// exactly the reference's float64 comparison of that value.
constexpr float kAlphaSkipF = 0x1.010102p-8f;   // >= 1/255
constexpr float kAlphaClampF = 0x1.fae148p-1f;  // >= 0.99
constexpr float kTMinF = 0x1.a36e3p-14f;        // >= 1e-4
constexpr float kAlphaClampVal = 0.99f;

// SH constants, reference sh.py:12-18
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_0 = 1.0925484305920792, kC2_1 = -1.0925484305920792,
                 kC2_2 = 0.31539156525252005, kC2_3 = -1.0925484305920792,
                 kC2_4 = 0.5462742152960396;
constexpr double kC3_0 = -0.5900435899266435, kC3_1 = 2.890611442640554,
                 kC3_2 = -0.4570457994644658, kC3_3 = 0.3731763325901154,
                 kC3_4 = -0.4570457994644658, kC3_5 = 1.445305721320277,
                 kC3_6 = -0.5900435899266435;

// Camera as passed to kernels (by value, inside FrameDesc).
struct CamDev {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  double center[3];  // -R^T t (camera.py:34-36)
  int width, height;
  int ntx, nty;
  int tile_base;    // first global tile id of this view
  int64_t pix_base;  // first pixel of this view in the concatenated images
};

struct FrameDesc {
  int n_views;
  int total_tiles;
  int64_t total_pixels;
  CamDev cam[CGS_MAX_VIEWS];
};

// 64-byte per-splat record written by projection, gathered by the raster.
struct __align__(16) SplatRec {
  double mx, my;        // mean2d (f64, render.py:157-158)
  double ca, cb, cc;    // conic [[A,B],[B,C]] (f64, render.py:176-181)
  float opac;           // sigmoid(logit) (computed in f64, render.py:200)
  float r, g, b;        // clamped colour (render.py:196-198)
  uint16_t px0, px1, py0, py1;  // inclusive contribution box, inside the pixel rect of
                                // render.py:110-115 (px0 = py0 = 0xffff when empty)
};
static_assert(sizeof(SplatRec) == 64, "SplatRec must be 64 bytes");

// Workspace header (first bytes of a frame workspace), device-resident.
struct FrameHeader {
  cgs_frame_stats_t stats;
  unsigned long long n_onscreen;   // scan totals (u64 for the scan kernel)
  unsigned long long n_pairs_raw;  // P as counted
  unsigned long long n_pairs;      // P if it fits the pair capacity, else 0
  unsigned long long scratch[8];
};

// -------------------------------------------------------------------------
void set_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* where);

// Lazily initialised per-device values (function attributes, occupancy-sized
// grids) are kept in arrays indexed by the current device ordinal: one
// process may drive several GPUs.
constexpr int kMaxDevices = 64;
int current_device(int* dev);

// Fork-join onto a second stream of the current device, for independent
// kernels of one stage (captured into a CUDA graph as parallel branches when
// the caller's stream is capturing).  The fork records an event on `st` that
// the side stream waits on; the join makes `st` wait for the side stream.
// The SideFork object holds the device's fork lock from fork to join, so
// concurrent host threads cannot interleave their event pairs.
struct SideFork {
  cudaStream_t side = nullptr;
  int dev = -1;
  int rc = 0;
  cudaStream_t main = nullptr;
  explicit SideFork(cudaStream_t st);
  int join();
  ~SideFork();
};

#define CGS_CUDA(call)                                      \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cgs::cuda_status(e_, #call); \
  } while (0)

// Instrumentation: every launch bumps a counter (cgs_launch_count); the one
// kernel named by cgs_profile_kernel is bracketed by CUDA events recorded on
// its own launch stream (cgs_profile_read).
void note_launch();
// Diagnostics: when set (cgs_trace_tiles), the raster kernels write one
// {start ns, end ns, SM id, tile} record per CTA: forward at [4 b], backward
// at [4 (total_tiles + b)].
unsigned long long* tile_trace_buffer();
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
struct ProfScope {
  bool on;
  cudaStream_t st;
  ProfScope(const char* name, cudaStream_t s);
  ~ProfScope();
};

#define CGS_CHECK_LAUNCH(name)                                              \
  do {                                                                      \
    cgs::note_launch();                                                     \
    cudaError_t e_ = cudaGetLastError();                                    \
    if (e_ != cudaSuccess) return cgs::cuda_status(e_, name);               \
  } while (0)

// Launch a kernel inside an optional profiling scope.
#define CGS_PROFILED(name, st, ...) \
  do {                              \
    cgs::ProfScope p_(name, st);    \
    __VA_ARGS__;                    \
  } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace.
struct Carver {
  char* base;
  size_t off = 0;
  size_t cap;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    off = align_up(off);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
  bool fits() const { return off <= cap; }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid size for grid-stride kernels: a multiple of the 148 SMs.
inline int grid_for(int64_t n, int block, int per_sm = 8) {
  int64_t g = ceil_div(n, block);
  int64_t cap = 148LL * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace cgs
