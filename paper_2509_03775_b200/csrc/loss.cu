// Reconstruction loss and its image gradient (reference metrics.py:17-140).
//
// L = (1-lam) mean|a-b| + lam (1 - SSIM), SSIM over an 11x11 Gaussian window
// (sigma 1.5), valid positions only, mean over channels.  Two tiled kernels:
//   ssim_stats  32x32 valid positions per CTA from a 42x42 smem halo: the five
//               windowed moments (separable, fp64), SSIM map partial sums, and
//               the three adjoint seeds d_mx, d_ex2, d_exy (metrics.py:96-109)
//   ssim_grad   32x32 pixels per CTA: adjoint filtering of the seeds
//               (metrics.py:40-45) fused with the L1 sign term -> dL/dimage
// Per-CTA partial sums are reduced in fixed order (deterministic).
#include <atomic>
#include <cmath>

#include "common.cuh"

namespace cgs {

// 11-tap Gaussian window (sigma 1.5, metrics.py:20-30), passed by value so
// that it lives in each launch's parameter bank: no per-device state.
struct SsimWin {
  double k[11];
};

struct LossLayout {
  float* seeds;      // V * 3 * 3 * (H-10)*(W-10)  [view][chan][map][pos]
  double* part_s;    // V * blocks_per_view (ssim sums)
  double* part_l1;   // V * blocks_per_view (|a-b| sums)
  size_t bytes;
};

static inline int64_t valid_n(int h, int w) {
  return (h >= 11 && w >= 11) ? static_cast<int64_t>(h - 10) * (w - 10) : 0;
}

static inline int blocks_x(int w) { return (w + 31) / 32; }
static inline int blocks_y(int h) { return (h + 31) / 32; }

static LossLayout plan_loss(void* base, size_t cap, int nv, int h, int w) {
  LossLayout L{};
  Carver c(base, cap);
  const int64_t vn = valid_n(h, w);
  L.seeds = c.take<float>(static_cast<size_t>(nv) * 9 * (vn > 0 ? vn : 1));
  const int64_t nb = static_cast<int64_t>(blocks_x(w)) * blocks_y(h) * 3;
  L.part_s = c.take<double>(nv * nb);
  L.part_l1 = c.take<double>(nv * nb);
  L.bytes = c.off + 256;
  return L;
}

// Both kernels tile 32x32 outputs per CTA (256 threads) and run the separable
// 11-tap window as two register-blocked passes: each thread slides the window
// over 4 adjacent outputs (14 loads feed 44 taps per moment), so the passes
// are fp64-FMA bound rather than shared-memory bound.
constexpr int kLT = 32;            // outputs per CTA side
constexpr int kLH = kLT + 10;      // halo side (42)
constexpr int kLP = kLH + 1;       // padded smem row (floats)

// The five windowed moments are filtered in fp32 on values shifted by 0.5:
// x' = x - 0.5 keeps |x'| <= ~0.5, so the variance m2 - m0^2 and covariance
// m4 - m0 m1 carry an absolute fp32 error of ~1e-8, far below C2 = 9e-4 that
// every SSIM denominator adds (the SSIM value moves by ~1e-9 relative; the
// per-window SSIM and its seeds are then formed in fp64).  The seeds are the
// derivatives with respect to the shifted moments (m0, m2, m4): the adjoint
// sum  F(d0) + 2 x' F(d2) + y' F(d4)  then has less cancellation than the
// unshifted form.  Max elementwise deviation of the SSIM image gradient from
// the float64 reference on the golden cases: 3.8e-5 relative (3.1e-5 with
// fp64 moments and fp32 unshifted seeds).
constexpr float kSsimShift = 0.5f;
struct StatsSmem {
  float sa[kLH][kLP];
  float sb[kLH][kLP];
  float hm[5][kLH][kLT + 1];
  double red_s[8], red_l[8];
};

struct GradSmem {
  float sd[3][kLH][kLP];
  double hv[3][kLH][kLT];
};

// grid: (ceil(W/32), ceil(H/32), view*3 + channel); block 256.
#ifndef CGS_SSIM_MINB
#define CGS_SSIM_MINB 4
#endif
__global__ void __launch_bounds__(256, CGS_SSIM_MINB) ssim_stats_kernel(const float* __restrict__ img,
                                                         const float* __restrict__ gt, int H, int W,
                                                         int do_ssim, LossLayout L, SsimWin win) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StatsSmem& S = *reinterpret_cast<StatsSmem*>(smem_raw);
  const int vc = blockIdx.z;
  const int v = vc / 3, ch = vc - 3 * (vc / 3);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT;
  const float* A = img + static_cast<int64_t>(v) * H * W * 3;
  const float* Bm = gt + static_cast<int64_t>(v) * H * W * 3;
  // L1 partial over this block's 32x32 pixels of channel ch (4 per thread)
  double l1 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int px = x0 + (tid & 31), py = y0 + (tid >> 5) + 8 * k;
    if (px < W && py < H) {
      const int64_t o = (static_cast<int64_t>(py) * W + px) * 3 + ch;
      l1 += fabs(static_cast<double>(A[o]) - static_cast<double>(Bm[o]));
    }
  }
  double s_acc = 0.0;
  const int Hv = H - 10, Wv = W - 10;
  if (do_ssim && Hv > 0 && Wv > 0 && x0 < Wv && y0 < Hv) {
    // all of a thread's halo loads are issued before any is stored (7 per
    // array in flight instead of one)
    constexpr int kPer = (kLH * kLH + 255) / 256;
    float la[kPer], lb[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = tid + 256 * q;
      const int yy = e / kLH, xx = e - yy * kLH;
      const int gx = x0 + xx, gy = y0 + yy;
      la[q] = lb[q] = 0.0f;
      if (e < kLH * kLH && gx < W && gy < H) {
        const int64_t o = (static_cast<int64_t>(gy) * W + gx) * 3 + ch;
        la[q] = __ldg(A + o) - kSsimShift;
        lb[q] = __ldg(Bm + o) - kSsimShift;
      }
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = tid + 256 * q;
      if (e < kLH * kLH) {
        const int yy = e / kLH, xx = e - yy * kLH;
        S.sa[yy][xx] = la[q];
        S.sb[yy][xx] = lb[q];
      }
    }
    __syncthreads();
    // horizontal: 42 rows x 8 segments of 4 outputs
    for (int it = tid; it < kLH * 8; it += 256) {
      const int row = it >> 3, c0 = (it & 7) * 4;
      float av[14], bv[14];
#pragma unroll
      for (int i = 0; i < 14; ++i) {
        av[i] = S.sa[row][c0 + i];
        bv[i] = S.sb[row][c0 + i];
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        float m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
        for (int j = 0; j < 11; ++j) {
          const float a = av[o + j], b = bv[o + j], k = static_cast<float>(win.k[j]);
          const float ka = k * a, kb = k * b;
          m0 += ka; m1 += kb; m2 = fmaf(ka, a, m2); m3 = fmaf(kb, b, m3); m4 = fmaf(ka, b, m4);
        }
        S.hm[0][row][c0 + o] = m0; S.hm[1][row][c0 + o] = m1; S.hm[2][row][c0 + o] = m2;
        S.hm[3][row][c0 + o] = m3; S.hm[4][row][c0 + o] = m4;
      }
    }
    __syncthreads();
    // vertical: 32 columns x 8 segments of 4 outputs (one item per thread)
    const int col = tid & 31, r0 = (tid >> 5) * 4;
    float m[5][4];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      float hv[14];
#pragma unroll
      for (int i = 0; i < 14; ++i) hv[i] = S.hm[q][r0 + i][col];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < 11; ++j) acc = fmaf(static_cast<float>(win.k[j]), hv[o + j], acc);
        m[q][o] = acc;
      }
    }
    const int ux = x0 + col;
    const int64_t vn = static_cast<int64_t>(Hv) * Wv;
    float* sd = L.seeds + (static_cast<int64_t>(v) * 3 + ch) * 3 * vn;
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int uy = y0 + r0 + o;
      if (ux >= Wv || uy >= Hv) continue;
      // shifted moments m0..m4 -> means, (co)variances (shift-invariant)
      const double m0 = m[0][o], m1 = m[1][o];
      const double vx = m[2][o] - m0 * m0, vy = m[3][o] - m1 * m1, cxy = m[4][o] - m0 * m1;
      const double mx = m0 + kSsimShift, my = m1 + kSsimShift;
      const double C1 = 1e-4, C2 = 9e-4;
      const double A1 = 2 * mx * my + C1, A2 = 2 * cxy + C2;
      const double B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
      const double F = 1.0 / (B1 * B2);
      const double sv = A1 * A2 * F;
      s_acc += sv;
      // seeds: dS/dm0, dS/dm2, dS/dm4 (metrics.py:96-109 in the shifted
      // variables: dS/dmu_x - 2 m0 dS/dvar_x - m1 dS/dcov, dS/dvar_x, dS/dcov)
      const double d_var = -sv / B2;
      const double d_cov = 2 * A1 * F;
      const double d_mx = sv * (2 * my / A1 - 2 * mx / B1) - 2 * m0 * d_var - m1 * d_cov;
      const double d_ex2 = d_var;
      const double d_exy = d_cov;
      const int64_t pos = static_cast<int64_t>(uy) * Wv + ux;
      sd[pos] = static_cast<float>(d_mx);
      sd[vn + pos] = static_cast<float>(d_ex2);
      sd[2 * vn + pos] = static_cast<float>(d_exy);
    }
  }
  // fixed-order block reduction
  double a = s_acc, b = l1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((tid & 31) == 0) {
    S.red_s[tid >> 5] = a;
    S.red_l[tid >> 5] = b;
  }
  __syncthreads();
  if (tid == 0) {
    double ts = 0, tl = 0;
    for (int w = 0; w < 8; ++w) { ts += S.red_s[w]; tl += S.red_l[w]; }
    const int64_t nb = static_cast<int64_t>(gridDim.x) * gridDim.y * 3;
    const int64_t bi = (static_cast<int64_t>(ch) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    L.part_s[v * nb + bi] = ts;
    L.part_l1[v * nb + bi] = tl;
  }
}

// dL/dimage: adjoint filtering of the three seed maps (metrics.py:40-45, the
// window is symmetric) fused with the L1 sign term; 32x32 pixels per CTA.
#ifndef CGS_SSIMG_MINB
#define CGS_SSIMG_MINB 4
#endif
__global__ void __launch_bounds__(256, CGS_SSIMG_MINB) ssim_grad_kernel(const float* __restrict__ img,
                                                        const float* __restrict__ gt, int H, int W,
                                                        double lam, double inv_size,
                                                        double inv_count, float grad_scale,
                                                        int do_ssim, LossLayout L,
                                                        float* __restrict__ dL, SsimWin win) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GradSmem& S = *reinterpret_cast<GradSmem*>(smem_raw);
  const int vc = blockIdx.z;
  const int v = vc / 3, ch = vc - 3 * (vc / 3);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT;
  const int Hv = H - 10, Wv = W - 10;
  const bool ssim_on = do_ssim && Hv > 0 && Wv > 0;
  const int col = tid & 31, r0 = (tid >> 5) * 4;
  double r[3][4] = {};
  if (ssim_on) {
    const int64_t vn = static_cast<int64_t>(Hv) * Wv;
    const float* seeds = L.seeds + (static_cast<int64_t>(v) * 3 + ch) * 3 * vn;
    // seed window rows/cols [y0-10, y0+31], zero outside the valid range
    constexpr int kPer = (kLH * kLH + 255) / 256;
    float ls[3][kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = tid + 256 * i;
      const int yy = e / kLH, xx = e - yy * kLH;
      const int uy = y0 - 10 + yy, ux = x0 - 10 + xx;
      const bool ok = e < kLH * kLH && uy >= 0 && uy < Hv && ux >= 0 && ux < Wv;
      const int64_t pos = static_cast<int64_t>(uy) * Wv + ux;
#pragma unroll
      for (int q = 0; q < 3; ++q) ls[q][i] = ok ? __ldg(seeds + q * vn + pos) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = tid + 256 * i;
      if (e < kLH * kLH) {
        const int yy = e / kLH, xx = e - yy * kLH;
#pragma unroll
        for (int q = 0; q < 3; ++q) S.sd[q][yy][xx] = ls[q][i];
      }
    }
    __syncthreads();
    for (int it = tid; it < kLH * 8; it += 256) {
      const int row = it >> 3, c0 = (it & 7) * 4;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double sv[14];
#pragma unroll
        for (int i = 0; i < 14; ++i) sv[i] = S.sd[q][row][c0 + i];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < 11; ++j) acc += win.k[j] * sv[o + j];
          S.hv[q][row][c0 + o] = acc;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double hv[14];
#pragma unroll
      for (int i = 0; i < 14; ++i) hv[i] = S.hv[q][r0 + i][col];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 11; ++j) acc += win.k[j] * hv[o + j];
        r[q][o] = acc;
      }
    }
  }
  const float* A = img + static_cast<int64_t>(v) * H * W * 3;
  const float* Bm = gt + static_cast<int64_t>(v) * H * W * 3;
  const int px = x0 + col;
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const int py = y0 + r0 + o;
    if (px >= W || py >= H) continue;
    const int64_t off = (static_cast<int64_t>(py) * W + px) * 3 + ch;
    const double a = A[off], b = Bm[off];
    double gs = 0.0;
    if (ssim_on)  // adjoint in the shifted variables (the stats kernel's seeds)
      gs = (r[0][o] + 2.0 * (a - kSsimShift) * r[1][o] + (b - kSsimShift) * r[2][o]) * inv_count;
    const double sgn = a > b ? 1.0 : (a < b ? -1.0 : 0.0);
    double g = (1.0 - lam) * sgn * inv_size;
    if (lam != 0.0) g -= lam * gs;
    dL[static_cast<int64_t>(v) * H * W * 3 + off] = static_cast<float>(g * grad_scale);
  }
}

// One CTA per view: strided fixed-order partial sums, then a fixed tree.
__global__ void __launch_bounds__(256) loss_final_kernel(LossLayout L, int64_t nb, double lam,
                                                         double inv_size, double inv_count,
                                                         int has_ssim, double* losses) {
  __shared__ double rs[256], rl[256];
  const int v = blockIdx.x, tid = threadIdx.x;
  double s = 0, l = 0;
  for (int64_t i = tid; i < nb; i += 256) {
    s += L.part_s[v * nb + i];
    l += L.part_l1[v * nb + i];
  }
  rs[tid] = s;
  rl[tid] = l;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) {
      rs[tid] += rs[tid + o];
      rl[tid] += rl[tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    const double l1 = rl[0] * inv_size;
    const double ss = has_ssim ? rs[0] * inv_count : nan("");
    losses[3 * v + 0] = l1;
    losses[3 * v + 1] = ss;
    losses[3 * v + 2] = lam == 0.0 ? l1 : (1.0 - lam) * l1 + lam * (1.0 - ss);
  }
}

static SsimWin make_window() {
  SsimWin w;
  double s = 0;
  for (int j = 0; j < 11; ++j) {
    const double r = (j - 5.0) / 1.5;
    w.k[j] = exp(-0.5 * r * r);
    s += w.k[j];
  }
  for (int j = 0; j < 11; ++j) w.k[j] /= s;
  return w;
}

size_t loss_ws_bytes(int nv, int h, int w) {
  return plan_loss(nullptr, 0, nv, h, w).bytes;
}

int recon_loss(const float* img, const float* gt, int nv, int H, int W, double lam, float gscale,
               float* dL, double* losses, int want_ssim, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  static const SsimWin win = make_window();
  LossLayout L = plan_loss(ws, ws_bytes, nv, H, W);
  if (L.bytes > ws_bytes) {
    set_error("loss workspace too small");
    return CGS_EWORKSPACE;
  }
  if (lam != 0.0 && (H < 11 || W < 11)) {
    set_error("images must be at least 11x11 for SSIM");
    return CGS_EINVAL;
  }
  const bool has_ssim = (H >= 11 && W >= 11) && (lam != 0.0 || want_ssim);
  const dim3 grid(blocks_x(W), blocks_y(H), 3 * nv);
  static std::atomic<bool> attr[kMaxDevices] = {};  // per device ordinal
  int dev = 0;
  if (int rc = current_device(&dev)) return rc;
  if (!attr[dev].load()) {
    CGS_CUDA(cudaFuncSetAttribute(ssim_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(StatsSmem))));
    CGS_CUDA(cudaFuncSetAttribute(ssim_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(GradSmem))));
    attr[dev].store(true);
  }
  CGS_PROFILED("ssim_stats_kernel", st, ssim_stats_kernel<<<grid, 256, sizeof(StatsSmem), st>>>(img, gt, H, W, has_ssim ? 1 : 0, L, win));
  CGS_CHECK_LAUNCH("ssim_stats_kernel");
  const double inv_size = 1.0 / (3.0 * H * W);
  const double inv_count = has_ssim ? 1.0 / (3.0 * (H - 10.0) * (W - 10.0)) : 0.0;
  const int64_t nb = static_cast<int64_t>(blocks_x(W)) * blocks_y(H) * 3;
  if (!dL) {
    loss_final_kernel<<<nv, 256, 0, st>>>(L, nb, lam, inv_size, inv_count, has_ssim ? 1 : 0,
                                          losses);
    CGS_CHECK_LAUNCH("loss_final_kernel");
    return CGS_OK;
  }
  // the loss values (reporting only) beside the image gradient, on a side
  // stream: both read only ssim_stats' output
  SideFork fork(st);
  if (fork.rc) return fork.rc;
  loss_final_kernel<<<nv, 256, 0, fork.side>>>(L, nb, lam, inv_size, inv_count, has_ssim ? 1 : 0,
                                               losses);
  CGS_CHECK_LAUNCH("loss_final_kernel");
  CGS_PROFILED("ssim_grad_kernel", st, ssim_grad_kernel<<<grid, 256, sizeof(GradSmem), st>>>(img, gt, H, W, lam, inv_size, inv_count, gscale,
                                         (has_ssim && lam != 0.0) ? 1 : 0, L, dL, win));
  CGS_CHECK_LAUNCH("ssim_grad_kernel");
  return fork.join();
}


// 8-bit image output (reference modelio.py:137-153: save_png's bytes and
// quantize8's grid): clip(rint(x * 255), 0, 255) evaluated in float64 on the
// fp32 values, as numpy does on the image (rint: round half to even).  Four
// values per thread, 16-byte loads when the buffer allows.
__global__ void __launch_bounds__(256) quantize8_kernel(const float* __restrict__ x, int64_t n,
                                                        uint8_t* __restrict__ out) {
  auto q = [](float v) -> uint32_t {
    double r = rint(static_cast<double>(v) * 255.0);
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);  // NaN -> 0 like numpy's clip + cast
    return r == r ? static_cast<uint32_t>(r) : 0u;
  };
  const int64_t n4 = n / 4;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (reinterpret_cast<uintptr_t>(out) & 3u) == 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (vec) {
      const float4 v = reinterpret_cast<const float4*>(x)[i];
      reinterpret_cast<uint32_t*>(out)[i] = q(v.x) | (q(v.y) << 8) | (q(v.z) << 16) | (q(v.w) << 24);
    } else {
      for (int k = 0; k < 4; ++k) out[4 * i + k] = static_cast<uint8_t>(q(x[4 * i + k]));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t j = 4 * n4 + threadIdx.x;
    out[j] = static_cast<uint8_t>(q(x[j]));
  }
}

int quantize8(const float* x, int64_t n, uint8_t* out, cudaStream_t st) {
  if (n <= 0) return CGS_OK;
  const int64_t n4 = (n + 3) / 4;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n4 + 255) / 256, 148 * 8));
  CGS_PROFILED("quantize8_kernel", st, quantize8_kernel<<<grid, 256, 0, st>>>(x, n, out));
  CGS_CHECK_LAUNCH("quantize8_kernel");
  return CGS_OK;
}
}  // namespace cgs
