// Reconstruction loss and its image gradient (reference metrics.py:17-140).
//
// L = (1-lam) mean|a-b| + lam (1 - SSIM), SSIM over an 11x11 Gaussian window
// (sigma 1.5), valid positions only, mean over channels.  Two tiled kernels:
//   ssim_stats  16x16 valid positions per CTA from a 26x26 smem halo: the five
//               windowed moments (separable, fp64), SSIM map partial sums, and
//               the three adjoint seeds d_mx, d_ex2, d_exy (metrics.py:96-109)
//   ssim_grad   16x16 pixels per CTA: adjoint filtering of the seeds
//               (metrics.py:40-45) fused with the L1 sign term -> dL/dimage
// Per-CTA partial sums are reduced in fixed order (deterministic).
#include <cmath>

#include "common.cuh"

namespace cgs {

__constant__ double c_win[11];

struct LossLayout {
  float* seeds;      // V * 3 * 3 * (H-10)*(W-10)  [view][chan][map][pos]
  double* part_s;    // V * blocks_per_view (ssim sums)
  double* part_l1;   // V * blocks_per_view (|a-b| sums)
  size_t bytes;
};

static inline int64_t valid_n(int h, int w) {
  return (h >= 11 && w >= 11) ? static_cast<int64_t>(h - 10) * (w - 10) : 0;
}

static inline int blocks_x(int w) { return (w + 15) / 16; }
static inline int blocks_y(int h) { return (h + 15) / 16; }

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

// grid: (bx, by, view*3 + channel); block 256.
__global__ void __launch_bounds__(256) ssim_stats_kernel(const float* __restrict__ img,
                                                         const float* __restrict__ gt, int H, int W,
                                                         int do_ssim, LossLayout L) {
  __shared__ double sx[26][26], sy[26][26];
  __shared__ double hm[5][26][16];
  __shared__ double red_s[8], red_l[8];
  const int vc = blockIdx.z;
  const int v = vc / 3, ch = vc - 3 * (vc / 3);
  const int tid = threadIdx.x, lx = tid & 15, ly = tid >> 4;
  const int x0 = blockIdx.x * 16, y0 = blockIdx.y * 16;
  const float* A = img + static_cast<int64_t>(v) * H * W * 3;
  const float* Bm = gt + static_cast<int64_t>(v) * H * W * 3;
  // L1 partial over this block's 16x16 pixels of channel ch
  double l1 = 0.0;
  {
    const int px = x0 + lx, py = y0 + ly;
    if (px < W && py < H) {
      const int64_t o = (static_cast<int64_t>(py) * W + px) * 3 + ch;
      l1 = fabs(static_cast<double>(A[o]) - static_cast<double>(Bm[o]));
    }
  }
  double s_acc = 0.0;
  const int Hv = H - 10, Wv = W - 10;
  if (do_ssim && Hv > 0 && Wv > 0 && x0 < Wv && y0 < Hv) {
    for (int e = tid; e < 26 * 26; e += 256) {
      const int yy = e / 26, xx = e - yy * 26;
      const int gx = x0 + xx, gy = y0 + yy;
      double a = 0.0, b = 0.0;
      if (gx < W && gy < H) {
        const int64_t o = (static_cast<int64_t>(gy) * W + gx) * 3 + ch;
        a = A[o];
        b = Bm[o];
      }
      sx[yy][xx] = a;
      sy[yy][xx] = b;
    }
    __syncthreads();
    for (int e = tid; e < 26 * 16; e += 256) {
      const int yy = e / 16, xx = e - yy * 16;
      double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
      for (int j = 0; j < 11; ++j) {
        const double a = sx[yy][xx + j], b = sy[yy][xx + j], k = c_win[j];
        m0 += k * a; m1 += k * b; m2 += k * a * a; m3 += k * b * b; m4 += k * a * b;
      }
      hm[0][yy][xx] = m0; hm[1][yy][xx] = m1; hm[2][yy][xx] = m2; hm[3][yy][xx] = m3; hm[4][yy][xx] = m4;
    }
    __syncthreads();
    const int ux = x0 + lx, uy = y0 + ly;
    if (ux < Wv && uy < Hv) {
      double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 11; ++j) {
        const double k = c_win[j];
#pragma unroll
        for (int q = 0; q < 5; ++q) m[q] += k * hm[q][ly + j][lx];
      }
      const double mx = m[0], my = m[1];
      const double vx = m[2] - mx * mx, vy = m[3] - my * my, cxy = m[4] - mx * my;
      const double C1 = 1e-4, C2 = 9e-4;
      const double A1 = 2 * mx * my + C1, A2 = 2 * cxy + C2;
      const double B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
      const double F = 1.0 / (B1 * B2);
      const double s = A1 * A2 * F;
      s_acc = s;
      const double d_mx = 2 * my * F * (A2 - A1) - 2 * mx * s * (1.0 / B1 - 1.0 / B2);
      const double d_ex2 = -s / B2;
      const double d_exy = 2 * A1 * F;
      const int64_t vn = static_cast<int64_t>(Hv) * Wv;
      float* sd = L.seeds + (static_cast<int64_t>(v) * 3 + ch) * 3 * vn;
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
    red_s[tid >> 5] = a;
    red_l[tid >> 5] = b;
  }
  __syncthreads();
  if (tid == 0) {
    double ts = 0, tl = 0;
    for (int w = 0; w < 8; ++w) { ts += red_s[w]; tl += red_l[w]; }
    const int64_t nb = static_cast<int64_t>(gridDim.x) * gridDim.y * 3;
    const int64_t bi = (static_cast<int64_t>(ch) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    L.part_s[v * nb + bi] = ts;
    L.part_l1[v * nb + bi] = tl;
  }
}

__global__ void __launch_bounds__(256) ssim_grad_kernel(const float* __restrict__ img,
                                                        const float* __restrict__ gt, int H, int W,
                                                        double lam, double inv_size,
                                                        double inv_count, float grad_scale,
                                                        int do_ssim, LossLayout L,
                                                        float* __restrict__ dL) {
  __shared__ float sd[3][26][26];
  __shared__ double hv[3][26][16];
  const int vc = blockIdx.z;
  const int v = vc / 3, ch = vc - 3 * (vc / 3);
  const int tid = threadIdx.x, lx = tid & 15, ly = tid >> 4;
  const int x0 = blockIdx.x * 16, y0 = blockIdx.y * 16;
  const int Hv = H - 10, Wv = W - 10;
  double gs = 0.0;
  const bool ssim_on = do_ssim && Hv > 0 && Wv > 0;
  if (ssim_on) {
    const int64_t vn = static_cast<int64_t>(Hv) * Wv;
    const float* seeds = L.seeds + (static_cast<int64_t>(v) * 3 + ch) * 3 * vn;
    // window rows/cols [y0-10, y0+15], zero outside the valid seed range
    for (int e = tid; e < 26 * 26; e += 256) {
      const int yy = e / 26, xx = e - yy * 26;
      const int uy = y0 - 10 + yy, ux = x0 - 10 + xx;
      const bool ok = uy >= 0 && uy < Hv && ux >= 0 && ux < Wv;
      const int64_t pos = static_cast<int64_t>(uy) * Wv + ux;
#pragma unroll
      for (int q = 0; q < 3; ++q) sd[q][yy][xx] = ok ? seeds[q * vn + pos] : 0.0f;
    }
    __syncthreads();
    for (int e = tid; e < 26 * 16; e += 256) {
      const int yy = e / 16, xx = e - yy * 16;
      double a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
      for (int j = 0; j < 11; ++j) {
        const double k = c_win[j];
        a0 += k * sd[0][yy][xx + j];
        a1 += k * sd[1][yy][xx + j];
        a2 += k * sd[2][yy][xx + j];
      }
      hv[0][yy][xx] = a0; hv[1][yy][xx] = a1; hv[2][yy][xx] = a2;
    }
    __syncthreads();
  }
  const int px = x0 + lx, py = y0 + ly;
  if (px >= W || py >= H) return;
  const float* A = img + static_cast<int64_t>(v) * H * W * 3;
  const float* Bm = gt + static_cast<int64_t>(v) * H * W * 3;
  const int64_t o = (static_cast<int64_t>(py) * W + px) * 3 + ch;
  const double a = A[o], b = Bm[o];
  if (ssim_on) {
    double r0 = 0, r1 = 0, r2 = 0;
#pragma unroll
    for (int j = 0; j < 11; ++j) {
      const double k = c_win[j];
      r0 += k * hv[0][ly + j][lx];
      r1 += k * hv[1][ly + j][lx];
      r2 += k * hv[2][ly + j][lx];
    }
    gs = (r0 + 2.0 * a * r1 + b * r2) * inv_count;
  }
  const double sgn = a > b ? 1.0 : (a < b ? -1.0 : 0.0);
  double g = (1.0 - lam) * sgn * inv_size;
  if (lam != 0.0) g -= lam * gs;
  dL[static_cast<int64_t>(v) * H * W * 3 + o] = static_cast<float>(g * grad_scale);
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

static bool g_win_ready = false;

static int ensure_window() {
  if (g_win_ready) return CGS_OK;
  double k[11], s = 0;
  for (int j = 0; j < 11; ++j) {
    const double r = (j - 5.0) / 1.5;
    k[j] = exp(-0.5 * r * r);
    s += k[j];
  }
  for (int j = 0; j < 11; ++j) k[j] /= s;
  CGS_CUDA(cudaMemcpyToSymbol(c_win, k, sizeof(k)));
  g_win_ready = true;
  return CGS_OK;
}

size_t loss_ws_bytes(int nv, int h, int w) {
  return plan_loss(nullptr, 0, nv, h, w).bytes;
}

int recon_loss(const float* img, const float* gt, int nv, int H, int W, double lam, float gscale,
               float* dL, double* losses, int want_ssim, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  int rc = ensure_window();
  if (rc) return rc;
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
  CGS_PROFILED("ssim_stats_kernel", st, ssim_stats_kernel<<<grid, 256, 0, st>>>(img, gt, H, W, has_ssim ? 1 : 0, L));
  CGS_CHECK_LAUNCH("ssim_stats_kernel");
  const double inv_size = 1.0 / (3.0 * H * W);
  const double inv_count = has_ssim ? 1.0 / (3.0 * (H - 10.0) * (W - 10.0)) : 0.0;
  if (dL) {
    CGS_PROFILED("ssim_grad_kernel", st, ssim_grad_kernel<<<grid, 256, 0, st>>>(img, gt, H, W, lam, inv_size, inv_count, gscale,
                                           (has_ssim && lam != 0.0) ? 1 : 0, L, dL));
    CGS_CHECK_LAUNCH("ssim_grad_kernel");
  }
  const int64_t nb = static_cast<int64_t>(blocks_x(W)) * blocks_y(H) * 3;
  loss_final_kernel<<<nv, 256, 0, st>>>(L, nb, lam, inv_size, inv_count, has_ssim ? 1 : 0,
                                        losses);
  CGS_CHECK_LAUNCH("loss_final_kernel");
  return CGS_OK;
}

}  // namespace cgs
