// Device helpers shared by the forward and backward render kernels.
#pragma once

#include "common.cuh"

namespace cgs {

constexpr double kLog2e = 1.4426950408889634;

// Unit quaternion (w,x,y,z) -> rotation, reference render.py:45-58.
__device__ __forceinline__ void quat_to_rot(double w, double x, double y, double z, double* R) {
  R[0] = 1 - 2 * (y * y + z * z);
  R[1] = 2 * (x * y - w * z);
  R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);
  R[4] = 1 - 2 * (x * x + z * z);
  R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);
  R[7] = 2 * (y * z + w * x);
  R[8] = 1 - 2 * (x * x + y * y);
}

// Real SH basis, reference sh.py:27-53 (same constants and sign convention).
template <int DEG>
__device__ __forceinline__ void sh_basis(double x, double y, double z, double* o) {
  o[0] = kC0;
  if constexpr (DEG >= 1) {
    o[1] = -kC1 * y;
    o[2] = kC1 * z;
    o[3] = -kC1 * x;
  }
  if constexpr (DEG >= 2) {
    const double xx = x * x, yy = y * y, zz = z * z;
    o[4] = kC2_0 * x * y;
    o[5] = kC2_1 * y * z;
    o[6] = kC2_2 * (2.0 * zz - xx - yy);
    o[7] = kC2_3 * x * z;
    o[8] = kC2_4 * (xx - yy);
  }
  if constexpr (DEG >= 3) {
    const double xx = x * x, yy = y * y, zz = z * z;
    o[9] = kC3_0 * y * (3.0 * xx - yy);
    o[10] = kC3_1 * x * y * z;
    o[11] = kC3_2 * y * (4.0 * zz - xx - yy);
    o[12] = kC3_3 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    o[13] = kC3_4 * x * (4.0 * zz - xx - yy);
    o[14] = kC3_5 * z * (xx - yy);
    o[15] = kC3_6 * x * (xx - 3.0 * yy);
  }
}

// fp32 twin of sh_basis (codebook-gradient reduction, where the inputs are
// fp32 already and the sum is accumulated in fp64).
template <int DEG>
__device__ __forceinline__ void sh_basis_f(float x, float y, float z, float* o) {
  o[0] = static_cast<float>(kC0);
  if constexpr (DEG >= 1) {
    o[1] = static_cast<float>(-kC1) * y;
    o[2] = static_cast<float>(kC1) * z;
    o[3] = static_cast<float>(-kC1) * x;
  }
  if constexpr (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    o[4] = static_cast<float>(kC2_0) * x * y;
    o[5] = static_cast<float>(kC2_1) * y * z;
    o[6] = static_cast<float>(kC2_2) * (2.0f * zz - xx - yy);
    o[7] = static_cast<float>(kC2_3) * x * z;
    o[8] = static_cast<float>(kC2_4) * (xx - yy);
  }
  if constexpr (DEG >= 3) {
    const float xx = x * x, yy = y * y, zz = z * z;
    o[9] = static_cast<float>(kC3_0) * y * (3.0f * xx - yy);
    o[10] = static_cast<float>(kC3_1) * x * y * z;
    o[11] = static_cast<float>(kC3_2) * y * (4.0f * zz - xx - yy);
    o[12] = static_cast<float>(kC3_3) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    o[13] = static_cast<float>(kC3_4) * x * (4.0f * zz - xx - yy);
    o[14] = static_cast<float>(kC3_5) * z * (xx - yy);
    o[15] = static_cast<float>(kC3_6) * x * (xx - 3.0f * yy);
  }
}

// Single SH basis function b at direction (x,y,z) (runtime index).
__device__ __forceinline__ double sh_basis_one(int b, double x, double y, double z) {
  const double xx = x * x, yy = y * y, zz = z * z;
  switch (b) {
    case 0: return kC0;
    case 1: return -kC1 * y;
    case 2: return kC1 * z;
    case 3: return -kC1 * x;
    case 4: return kC2_0 * x * y;
    case 5: return kC2_1 * y * z;
    case 6: return kC2_2 * (2.0 * zz - xx - yy);
    case 7: return kC2_3 * x * z;
    case 8: return kC2_4 * (xx - yy);
    case 9: return kC3_0 * y * (3.0 * xx - yy);
    case 10: return kC3_1 * x * y * z;
    case 11: return kC3_2 * y * (4.0 * zz - xx - yy);
    case 12: return kC3_3 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    case 13: return kC3_4 * x * (4.0 * zz - xx - yy);
    case 14: return kC3_5 * z * (xx - yy);
    default: return kC3_6 * x * (xx - 3.0 * yy);
  }
}

// d basis_b / d dir accumulated against weights: g += sum_b w[b] * dB_b/d(x,y,z)
// (reference sh.py:56-100).
template <int DEG, typename T = double>
__device__ __forceinline__ void sh_basis_grad_dot(T x, T y, T z, const T* w, T* g) {
  g[0] = g[1] = g[2] = T(0);
  if constexpr (DEG >= 1) {
    g[1] += -T(kC1) * w[1];
    g[2] += T(kC1) * w[2];
    g[0] += -T(kC1) * w[3];
  }
  if constexpr (DEG >= 2) {
    g[0] += T(kC2_0) * y * w[4];
    g[1] += T(kC2_0) * x * w[4];
    g[1] += T(kC2_1) * z * w[5];
    g[2] += T(kC2_1) * y * w[5];
    g[0] += -T(2.0) * T(kC2_2) * x * w[6];
    g[1] += -T(2.0) * T(kC2_2) * y * w[6];
    g[2] += T(4.0) * T(kC2_2) * z * w[6];
    g[0] += T(kC2_3) * z * w[7];
    g[2] += T(kC2_3) * x * w[7];
    g[0] += T(2.0) * T(kC2_4) * x * w[8];
    g[1] += -T(2.0) * T(kC2_4) * y * w[8];
  }
  if constexpr (DEG >= 3) {
    const T xx = x * x, yy = y * y, zz = z * z;
    g[0] += T(kC3_0) * T(6.0) * x * y * w[9];
    g[1] += T(kC3_0) * (T(3.0) * xx - T(3.0) * yy) * w[9];
    g[0] += T(kC3_1) * y * z * w[10];
    g[1] += T(kC3_1) * x * z * w[10];
    g[2] += T(kC3_1) * x * y * w[10];
    g[0] += -T(2.0) * T(kC3_2) * x * y * w[11];
    g[1] += T(kC3_2) * (T(4.0) * zz - xx - T(3.0) * yy) * w[11];
    g[2] += T(8.0) * T(kC3_2) * y * z * w[11];
    g[0] += -T(6.0) * T(kC3_3) * x * z * w[12];
    g[1] += -T(6.0) * T(kC3_3) * y * z * w[12];
    g[2] += T(kC3_3) * (T(6.0) * zz - T(3.0) * xx - T(3.0) * yy) * w[12];
    g[0] += T(kC3_4) * (T(4.0) * zz - T(3.0) * xx - yy) * w[13];
    g[1] += -T(2.0) * T(kC3_4) * x * y * w[13];
    g[2] += T(8.0) * T(kC3_4) * x * z * w[13];
    g[0] += T(2.0) * T(kC3_5) * x * z * w[14];
    g[1] += -T(2.0) * T(kC3_5) * y * z * w[14];
    g[2] += T(kC3_5) * (xx - yy) * w[14];
    g[0] += T(kC3_6) * (T(3.0) * xx - T(3.0) * yy) * w[15];
    g[1] += -T(6.0) * T(kC3_6) * x * y * w[15];
  }
}

// Transposed (reduce-scatter) warp sum of 9 values in 12 shuffles instead of
// 9 x 5 = 45: at each butterfly level a lane keeps the half of its values its
// partner does not and adds the partner's copy of them.  Lanes
// 0,2,4,8,10,16,18,20,24 return the sums of values 0..8 (reduce9_slot); the
// order of additions is fixed, so the result is deterministic.
__device__ __forceinline__ float warp_reduce9(const float (&o)[9]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  float v5[5];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const float lo = o[j], hi = j < 4 ? o[5 + j] : 0.0f;
      v5[j] = (up ? hi : lo) + __shfl_xor_sync(full, up ? lo : hi, 16);
    }
  }
  float v3[3];
  {
    const bool up = lane & 8;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float lo = v5[j], hi = j < 2 ? v5[3 + j] : 0.0f;
      v3[j] = (up ? hi : lo) + __shfl_xor_sync(full, up ? lo : hi, 8);
    }
  }
  float v2[2];
  {
    const bool up = lane & 4;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float lo = v3[j], hi = j < 1 ? v3[2 + j] : 0.0f;
      v2[j] = (up ? hi : lo) + __shfl_xor_sync(full, up ? lo : hi, 4);
    }
  }
  float v1;
  {
    const bool up = lane & 2;
    v1 = (up ? v2[1] : v2[0]) + __shfl_xor_sync(full, up ? v2[0] : v2[1], 2);
  }
  return v1 + __shfl_xor_sync(full, v1, 1);
}

// The same transposed reduction for N values (N <= 32): at each butterfly
// level (16, 8, 4, 2, 1) a lane keeps the lower or upper half of its list
// (padded with a zero when odd) and adds its partner's copy of it; 20
// shuffles for N = 18 (two splats' 9 values) against 2 x 12.
template <int N, int H>
__device__ __forceinline__ void reduce_level(const float* in, float* out, int lane) {
  constexpr int LO = (N + 1) / 2;
  const bool up = lane & H;
#pragma unroll
  for (int j = 0; j < LO; ++j) {
    const float lo = in[j], hi = j + LO < N ? in[j + LO] : 0.0f;
    out[j] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, H);
  }
}

template <int N>
__device__ __forceinline__ float warp_reduce_t(const float (&o)[N]) {
  const int lane = threadIdx.x & 31;
  constexpr int N1 = (N + 1) / 2, N2 = (N1 + 1) / 2, N3 = (N2 + 1) / 2, N4 = (N3 + 1) / 2;
  float a[N1], b[N2], c[N3], d[N4], e[1];
  reduce_level<N, 16>(o, a, lane);
  reduce_level<N1, 8>(a, b, lane);
  reduce_level<N2, 4>(b, c, lane);
  reduce_level<N3, 2>(c, d, lane);
  reduce_level<N4, 1>(d, e, lane);
  return e[0];
}

// Value index held by `lane` after warp_reduce_t<N>, or -1 (a padding zero).
__host__ __device__ constexpr int reduce_slot(int n, int lane) {
  // the lane's list: len entries (padded), the first `real` of them original
  // indices base, base + 1, ...
  int base = 0, len = n, real = n;
  for (int h = 16; h >= 1; h >>= 1) {
    const int lo = (len + 1) / 2;
    if (lane & h) {
      base += lo;
      real = real > lo ? real - lo : 0;
    } else {
      real = real < lo ? real : lo;
    }
    len = lo;
  }
  return real == 1 ? base : -1;
}
static_assert(reduce_slot(9, 10) == 4 && reduce_slot(9, 24) == 8 && reduce_slot(9, 1) == -1,
              "warp_reduce_t<9> holds warp_reduce9's values on its even lanes");

// Value index held by `lane` after warp_reduce9, or -1.
__device__ __forceinline__ int reduce9_slot(int lane) {
  constexpr unsigned kMask = (1u << 0) | (1u << 2) | (1u << 4) | (1u << 8) | (1u << 10) |
                             (1u << 16) | (1u << 18) | (1u << 20) | (1u << 24);
  return ((kMask >> lane) & 1u) ? __popc(kMask & ((1u << lane) - 1u)) : -1;
}

// ---- bulk-copy (TMA engine) staging helpers, sm_90+/sm_100a PTX ------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Order earlier generic-proxy accesses of shared memory before later
// async-proxy (bulk copy) writes to it.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 1-D bulk copy global -> shared (UBLKCP), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Copy records [first, first + nb) of a tile list into s_raw (all threads of
// the CTA call it).  Default: each thread copies its own records with four
// 16-byte cp.async (no per-lane serialisation: a bulk copy per record is
// issued one lane at a time through the uniform datapath) and waits for them
// itself (records_wait) -- the callers stage record k on thread k.  With
// CGS_REC_CPASYNC=0: one bulk copy per record, completion on the mbarrier
// (thread 0 posts the expected byte count).
#ifndef CGS_REC_CPASYNC
#define CGS_REC_CPASYNC 1
#endif
static_assert(sizeof(SplatRec) == 64, "records move as four 16-byte pieces");
__device__ __forceinline__ void issue_records(SplatRec* s_raw, uint64_t* bar,
                                              const uint32_t* __restrict__ pair_vals,
                                              const SplatRec* __restrict__ recs, uint32_t first,
                                              int nb, int tid, int nthreads) {
#if CGS_REC_CPASYNC
  (void)bar;
  for (int k = tid; k < nb; k += nthreads) {
    const char* src = reinterpret_cast<const char*>(&recs[pair_vals[first + k]]);
    const uint32_t dst = smem_u32(&s_raw[k]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q), "l"(src + 16 * q)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
#else
  if (tid == 0) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nb) * sizeof(SplatRec));
  for (int k = tid; k < nb; k += nthreads)
    bulk_g2s(&s_raw[k], &recs[pair_vals[first + k]], sizeof(SplatRec), bar);
#endif
}

// Completion of the last issue_records (this thread's copies, or the batch on
// the mbarrier); flips the phase.
__device__ __forceinline__ void records_wait(uint64_t* bar, uint32_t& phase) {
#if CGS_REC_CPASYNC
  (void)bar;
  asm volatile("cp.async.wait_all;" ::: "memory");
#else
  mbar_wait(bar, phase);
#endif
  phase ^= 1;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// fp64 record -> fp32 shared-memory form for one tile, in the eigenbasis of
// the conic.  With conic Q = lambda1 e1 e1^T + lambda2 e2 e2^T (e2 = e1
// rotated by 90 deg), d^T Q d = lambda1 u^2 + lambda2 v^2, u = e1 . d,
// v = e2 . d.  The offsets (u0, v0) of the tile centre (cx, cy) = tile origin
// + (8, 8) from the mean are formed in fp64, so per pixel u = u0 + e1 . (lx,
// ly), v = v0 + e2 . (lx, ly) with tile-centred pixel coordinates lx, ly in
// [-7.5, 7.5] are small, well-conditioned fp32 numbers even for elongated
// near-plane splats centred far off screen (evaluating A dx^2 + 2B dx dy +
// C dy^2 directly in fp32 cancels catastrophically there).
//
// The raster works with the log-domain alpha
//   t = log2(255 alpha) = log2(255 o) - log2(e)/2 (lambda1 u^2 + lambda2 v^2)
// (render.py:274-277): keep is t >= 0 (alpha >= 1/255), the clamp is
// t >= log2(0.99 * 255), and alpha = 2^t / 255 is formed only for kept
// splats.
//   a = (u0, v0, e1x, e1y)   b = (k1, k2, log2(255 o), red)   c = (green, blue)
// with k = -log2(e)/2 lambda.
struct Staged {
  float4 a, b;
  float2 c;
};

__device__ __forceinline__ Staged stage_splat(const SplatRec& r, double cx, double cy) {
  const double A = r.ca, B = r.cb, C = r.cc;
  const double m = 0.5 * (A + C), h = 0.5 * (A - C);
  const double rr = sqrt(h * h + B * B);
  const double l1 = m + rr;                              // larger eigenvalue
  const double l2 = l1 > 0.0 ? (A * C - B * B) / l1 : 0.0;  // det / l1 (no cancellation in m - rr)
  // eigenvector of l1: the better conditioned of (l1 - C, B) and (B, l1 - A)
  double ex = l1 - C, ey = B;
  const double fx = B, fy = l1 - A;
  if (fx * fx + fy * fy > ex * ex + ey * ey) {
    ex = fx;
    ey = fy;
  }
  const double nn = sqrt(ex * ex + ey * ey);
  if (nn > 0.0) {
    ex /= nn;
    ey /= nn;
  } else {
    ex = 1.0;
    ey = 0.0;
  }
  const double dx = cx - r.mx, dy = cy - r.my;
  Staged st;
  st.a = make_float4(static_cast<float>(ex * dx + ey * dy), static_cast<float>(-ey * dx + ex * dy),
                     static_cast<float>(ex), static_cast<float>(ey));
  st.b = make_float4(static_cast<float>(-0.5 * kLog2e * l1), static_cast<float>(-0.5 * kLog2e * l2),
                     __log2f(255.0f * r.opac), r.r);
  st.c = make_float2(r.g, r.b);
  return st;
}

// Pixel of lane `lane` of forward warp `w` (tile-local; raster_fwd_kernel and
// the order refine.cu reads its flag masks in).  Warp w owns the 8x4 block
// ((w & 1) * 8, (w >> 1) * 4).  With CGS_FWD_HALF each half-warp h = lane >> 4
// owns the 4x4 half (4 h, 0) of it and walks its own hit list; otherwise the
// lanes cover the block row by row.
#ifndef CGS_FWD_HALF
#define CGS_FWD_HALF 1
#endif
__host__ __device__ constexpr int fwd_px_x(int w, int lane) {
  return CGS_FWD_HALF ? (w & 1) * 8 + (lane >> 4) * 4 + (lane & 3) : (w & 1) * 8 + (lane & 7);
}
__host__ __device__ constexpr int fwd_px_y(int w, int lane) {
  return CGS_FWD_HALF ? (w >> 1) * 4 + ((lane >> 2) & 3) : (w >> 1) * 4 + (lane >> 3);
}

// Centre of tile column / row t in pixel coordinates (stage_splat's origin);
// pixel x of the tile sits at centre + (x - 7.5).
__device__ __forceinline__ double tile_centre(int t) { return static_cast<double>(t * kTile + kTile / 2); }
constexpr float kTileHalf = 0.5f * (kTile - 1);  // 7.5

// t = log2(255 alpha_unclamped) at tile-centred pixel (lx, ly), fp32.
__device__ __forceinline__ float staged_t(const float4& a, const float4& b, float lx, float ly) {
  const float u = fmaf(a.w, ly, fmaf(a.z, lx, a.x));
  const float v = fmaf(a.z, ly, fmaf(-a.w, lx, a.y));
  return fmaf(b.x * u, u, fmaf(b.y * v, v, b.z));
}

// alpha = min(2^t / 255, 0.99) (render.py:278) for a kept t.
__device__ __forceinline__ float alpha_of_t(float t) {
  return fminf(fast_exp2(t) * static_cast<float>(1.0 / 255.0), kAlphaClampVal);
}

// ---- exact decisions ------------------------------------------------------
// The fp32 alpha above is within ~1e-5 relative of the reference's float64
// alpha (fp32 eigenbasis offsets, ex2.approx; measured with CGS_REFINE_ALL).
// Every discrete decision the reference takes -- keep (alpha >= 1/255,
// render.py:279), gradient flow through the clamp (alpha < 0.99,
// render.py:361) and termination (T_before >= 1e-4, render.py:283) -- is
// taken on the fp32 values only when they lie outside a relative band around
// the threshold (kAlphaBand on alpha, i.e. kAlphaBand / ln 2 on t; kTBand on
// T).  A pixel that meets a value inside a band is flagged by the forward and
// re-walked entirely in float64, exactly as the reference computes it
// (refine.cu, exact_alpha_raw).
constexpr double kAlphaBand = 4e-5;
constexpr double kTBand = 5e-5;
constexpr double kLn2 = 0.6931471805599453;
constexpr float kTSkipLo = static_cast<float>(-kAlphaBand / kLn2);  // keep band on t
constexpr float kTSkipHi = static_cast<float>(kAlphaBand / kLn2);
constexpr double kTClamp = 7.979853867163743;  // log2(0.99 * 255)
constexpr float kTClampLo = static_cast<float>(kTClamp - kAlphaBand / kLn2);
constexpr float kTClampHi = static_cast<float>(kTClamp + kAlphaBand / kLn2);
constexpr float kTHalfClamp = static_cast<float>(0.5 * kTClamp);  // the bands' symmetry point
constexpr float kTBandLo = static_cast<float>(1e-4 * (1.0 - kTBand));
constexpr float kTBandHi = static_cast<float>(1e-4 * (1.0 + kTBand));

// Whether any pixel centre of the tile-centred rectangle [x0, x1] x [y0, y1]
// can have t >= -margin: an upper bound of t over the rectangle from its
// projections onto the eigen axes (the rectangle lies inside the (u, v) box
// of those projections, and t decreases with |u| and |v|).  Exact for
// rectangles aligned with the eigen axes, conservative otherwise; it cuts
// the blocks that the axis-aligned contribution box keeps for a rotated,
// elongated ellipse.
__device__ __forceinline__ bool staged_may_hit(const float4& a, const float4& b, float x0, float x1,
                                               float y0, float y1) {
  const float ex = a.z, ey = a.w;
  const float ulo = a.x + fminf(ex * x0, ex * x1) + fminf(ey * y0, ey * y1);
  const float uhi = a.x + fmaxf(ex * x0, ex * x1) + fmaxf(ey * y0, ey * y1);
  const float vlo = a.y + fminf(-ey * x0, -ey * x1) + fminf(ex * y0, ex * y1);
  const float vhi = a.y + fmaxf(-ey * x0, -ey * x1) + fmaxf(ex * y0, ex * y1);
  const float du = fmaxf(0.0f, fmaxf(ulo, -uhi));
  const float dv = fmaxf(0.0f, fmaxf(vlo, -vhi));
  // t <= log2(255 o) + k1 du^2 + k2 dv^2 (k1, k2 <= 0); margin 1e-3 (log2
  // units) >> the fp32 error of t, and below the keep band's lower edge
  return fmaf(b.x * du, du, fmaf(b.y * dv, dv, b.z)) >= kTSkipLo - 1e-3f;
}

// Reference float64 alpha of splat record r at pixel (px, py) of its view
// (render.py:261, 274-280): d = centre - mean, power = -1/2 (A dx^2 + C dy^2)
// - B dx dy, alpha = min(o exp(power), 0.99) with o = sigmoid(logit) in f64
// (render.py:200).  Round-to-nearest intrinsics keep numpy's operation order
// (no FMA contraction).  Returns the unclamped o exp(power).
__device__ __forceinline__ double exact_alpha_raw(const SplatRec& r, float logit, int px, int py) {
  const double dx = __dsub_rn(static_cast<double>(px) + 0.5, r.mx);
  const double dy = __dsub_rn(static_cast<double>(py) + 0.5, r.my);
  const double q = __dadd_rn(__dmul_rn(r.ca, __dmul_rn(dx, dx)), __dmul_rn(r.cc, __dmul_rn(dy, dy)));
  const double power = __dsub_rn(__dmul_rn(-0.5, q), __dmul_rn(__dmul_rn(r.cb, dx), dy));
  const double o = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-static_cast<double>(logit))));
  return __dmul_rn(o, exp(power));
}

}  // namespace cgs
