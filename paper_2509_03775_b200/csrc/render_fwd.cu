// Forward render path (reference render.py:145-315) for sm_100a.
//
//   sr_precompute   Sigma3 per SR codebook row (render.py:85-91, 168-169)
//   project         per (view, Gaussian): fp64 EWA projection, codebook gather,
//                   SH colour, pixel/tile rect, depth keys (render.py:145-203,110-115)
//   depth order     the splats with tiles (compacted by the projection), one
//                   3-pass LSD onesweep on a 24-bit key (fp32 depth bits above
//                   the near plane, monotone in the fp64 depth); runs of equal
//                   keys are re-ordered by (fp64 depth, splat id)
//                   = np.lexsort((idx, tz)) (render.py:203), per view
//   pair offsets    one decoupled-lookback scan over the splats' tile counts in
//                   depth order (per splat and per depth rank; the last
//                   partition writes the frame counts)
//   emit + sort     (tile, splat) pairs in depth order, stable sort by tile
//                   id: the per-tile append order of _bin_tiles
//                   (render.py:240-254) -- a one-pass counting sort (count
//                   per chunk, matrix scan, ranked scatter) for frames of at
//                   most kCountMaxTiles tiles, else a 2-pass onesweep
//   raster_fwd      raster.cu
#include <atomic>
#include <cmath>

#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

// ---------------------------------------------------------------------------
// Sigma3 = R(q/|q|) diag(exp(2 ls)) R^T per SR row; slot 6 flags |q| == 0.
struct ZeroSpans {  // word ranges sr_precompute zeroes for the rest of the frame
  uint32_t* p[5];
  int64_t n[5];
};
__global__ void __launch_bounds__(256) sr_precompute_kernel(const float* __restrict__ rows,
                                                            int64_t cap, double* __restrict__ out,
                                                            ZeroSpans z) {
  {  // the frame header, depth-sort histogram and the sort / scan states (no memset nodes)
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
#pragma unroll
    for (int q = 0; q < 5; ++q)
      for (int64_t k = t0; k < z.n[q]; k += nt) z.p[q][k] = 0u;
  }
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < cap;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float* row = rows + r * 7;
    double q[4] = {row[3], row[4], row[5], row[6]};
    double nq = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    double* o = out + r * 8;
    if (nq == 0.0) {
      for (int k = 0; k < 6; ++k) o[k] = 0.0;
      o[6] = 1.0;
      o[7] = 0.0;
      continue;
    }
    const double w = q[0] / nq, x = q[1] / nq, y = q[2] / nq, z = q[3] / nq;
    double R[9];
    quat_to_rot(w, x, y, z, R);
    const double s0 = exp(2.0 * static_cast<double>(row[0]));
    const double s1 = exp(2.0 * static_cast<double>(row[1]));
    const double s2 = exp(2.0 * static_cast<double>(row[2]));
    // Sigma_ij = sum_k R_ik s_k R_jk
    auto S = [&](int i, int j) {
      return R[i * 3 + 0] * s0 * R[j * 3 + 0] + R[i * 3 + 1] * s1 * R[j * 3 + 1] +
             R[i * 3 + 2] * s2 * R[j * 3 + 2];
    };
    o[0] = S(0, 0); o[1] = S(0, 1); o[2] = S(0, 2);
    o[3] = S(1, 1); o[4] = S(1, 2); o[5] = S(2, 2);
    o[6] = 0.0;
    o[7] = 0.0;
  }
}

struct ProjIn {
  int64_t n;
  const float* pos;
  const float* logit;
  const int32_t* g2sh;
  const int32_t* g2sr;
  const float* sh_rows;
  const double* sr_cov;  // 8 doubles per SR row
};

struct ProjOut {
  SplatRec* recs;
  uint64_t* depth_key;
  uint32_t* dkey;  // 32-bit depth sort keys of the splats with tiles, compacted
  uint32_t* dval;  // their splat ids (sort payload)
  uint32_t* hist;  // 4 x 256 digit histogram of dkey (depth sort)
  uint32_t* n_tiles;
  uint64_t* rect;
  FrameHeader* hdr;
};

// A splat's per-Gaussian inputs.
struct ProjPre {
  float px, py, pz, logit;
  int32_t sh, sr;
};

__device__ __forceinline__ ProjPre load_pre(const ProjIn& in, int64_t i) {
  ProjPre p;
  p.px = in.pos[3 * i + 0];
  p.py = in.pos[3 * i + 1];
  p.pz = in.pos[3 * i + 2];
  p.logit = in.logit[i];
  p.sh = in.g2sh[i];
  p.sr = in.g2sr[i];
  return p;
}

#ifndef CGS_PROJECT_SH32
#define CGS_PROJECT_SH32 1
#endif
constexpr float kShGateRel = 4e-6f;  // >= 4x the fp32 colour error bound per sum|c|

// Float64 colour max(raw + 0.5, 0) of one SH row at unit direction (x, y, z)
// in the reference's order (render.py:187-198), rounded to fp32.
template <int DEG>
__device__ __noinline__ void sh_colour64(const float* __restrict__ row, double x, double y,
                                         double z, float* rgb) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  double B[NB];
  sh_basis<DEG>(x, y, z, B);
  double col[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < 3 * NB; ++e) col[e % 3] += B[e / 3] * static_cast<double>(__ldg(row + e));
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) rgb[ch] = static_cast<float>(fmax(col[ch] + 0.5, 0.0));
}

// One (view, Gaussian) splat; returns its 32-bit depth sort key (~0: no tiles).
// Quotients by the same divisor (1/tz, 1/det, 1/|view|) multiply by one
// reciprocal: within an ulp of the reference's divisions, far inside the
// decision bands (raster_common.cuh), like the reference's own einsum order.
template <int DEG>
__device__ __forceinline__ uint32_t project_one(const ProjIn& in, const FrameDesc& fd,
                                                const ProjOut& out, int64_t s, int v,
                                                const ProjPre& pre) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  constexpr int D = 3 * NB;
  const CamDev& cam = fd.cam[v];
  const double px = pre.px, py = pre.py, pz = pre.pz;
  // camera coordinates t = R p + trans (camera.py:29-32)
  const double tx = cam.R[0] * px + cam.R[1] * py + cam.R[2] * pz + cam.t[0];
  const double ty = cam.R[3] * px + cam.R[4] * py + cam.R[5] * pz + cam.t[1];
  const double tz = cam.R[6] * px + cam.R[7] * py + cam.R[8] * pz + cam.t[2];
  if (!(tz > kNear)) {  // near-plane cull, render.py:149
    out.n_tiles[s] = 0;
    return 0xffffffffu;
  }
  const double2* cv2 = reinterpret_cast<const double2*>(in.sr_cov + static_cast<int64_t>(pre.sr) * 8);
  const double2 c01 = cv2[0], c23 = cv2[1], c45 = cv2[2], c67 = cv2[3];
  const double cv[7] = {c01.x, c01.y, c23.x, c23.y, c45.x, c45.y, c67.x};
  if (cv[6] != 0.0) {  // zero quaternion: reference raises ValueError
    out.n_tiles[s] = 0;
    out.hdr->stats.zero_quaternion = 1;
    return 0xffffffffu;
  }
  const double rz = 1.0 / tz;
  const double mx = cam.fx * tx * rz + cam.cx;
  const double my = cam.fy * ty * rz + cam.cy;
  // J (render.py:160-164) and M = J R (render.py:165)
  const double j00 = cam.fx * rz, j02 = -cam.fx * tx * (rz * rz);
  const double j11 = cam.fy * rz, j12 = -cam.fy * ty * (rz * rz);
  double m0[3], m1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    m0[k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
    m1[k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
  }
  const double S[9] = {cv[0], cv[1], cv[2], cv[1], cv[3], cv[4], cv[2], cv[4], cv[5]};
  double sm0[3], sm1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    sm0[k] = S[k * 3 + 0] * m0[0] + S[k * 3 + 1] * m0[1] + S[k * 3 + 2] * m0[2];
    sm1[k] = S[k * 3 + 0] * m1[0] + S[k * 3 + 1] * m1[1] + S[k * 3 + 2] * m1[2];
  }
  // Sigma2 = M Sigma3 M^T + 0.3 I (render.py:171-174)
  const double a = m0[0] * sm0[0] + m0[1] * sm0[1] + m0[2] * sm0[2] + kBlur;
  const double b = m0[0] * sm1[0] + m0[1] * sm1[1] + m0[2] * sm1[2];
  const double c = m1[0] * sm1[0] + m1[1] * sm1[1] + m1[2] * sm1[2] + kBlur;
  const double det = a * c - b * b;
  const double lam = 0.5 * (a + c) + sqrt(0.25 * (a - c) * (a - c) + b * b);
  const double rad = kFootprint * sqrt(lam) + 1e-9;
  // inclusive pixel rect on pixel centres (render.py:110-115)
  const double x0 = fmax(0.0, ceil(mx - rad - 0.5));
  const double x1 = fmin(cam.width - 1.0, floor(mx + rad - 0.5));
  const double y0 = fmax(0.0, ceil(my - rad - 0.5));
  const double y1 = fmin(cam.height - 1.0, floor(my + rad - 0.5));
  if (!(x0 <= x1 && y0 <= y1)) {
    out.n_tiles[s] = 0;
    return 0xffffffffu;
  }
  const int tx0 = static_cast<int>(x0) / kTile, tx1 = static_cast<int>(x1) / kTile;
  const int ty0 = static_cast<int>(y0) / kTile, ty1 = static_cast<int>(y1) / kTile;
  // view direction and SH colour (render.py:187-198)
  double ox = px - cam.center[0], oy = py - cam.center[1], oz = pz - cam.center[2];
  const double rlen = 1.0 / sqrt((ox * ox + oy * oy) + oz * oz);
  ox *= rlen;
  oy *= rlen;
  oz *= rlen;
  const float* row = in.sh_rows + static_cast<int64_t>(pre.sh) * D;
  float rgb[3];
#if CGS_PROJECT_SH32
  {
    // fp32 basis and sum (no float->double conversions: 3(d+1)^2 of them per
    // splat ran at the conversion pipe's quarter rate).  The only discrete
    // decision on the colour is the gate raw > 0 of max(raw + 0.5, 0)
    // (render.py:198, 418-419); the fp32 raw is within 9e-7 sum|c| of the
    // float64 one (basis error <= 1.8e-7 absolute with |B| <= 0.75, 16-term
    // FMA chain), so a raw within kShGateRel sum|c| of the gate is
    // recomputed in float64 (sh_colour64, out of line: rare).  Elsewhere the
    // value differs from the float64 one by that bound (far inside the image
    // tolerance).
    float Bf[NB];
    sh_basis_f<DEG>(static_cast<float>(ox), static_cast<float>(oy), static_cast<float>(oz), Bf);
    float c3[3] = {0.0f, 0.0f, 0.0f}, a3[3] = {0.0f, 0.0f, 0.0f};
    auto acc = [&](int e, float v) {
      c3[e % 3] = fmaf(Bf[e / 3], v, c3[e % 3]);
      a3[e % 3] += fabsf(v);
    };
    if constexpr (D % 4 == 0) {
      const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
      for (int q = 0; q < D / 4; ++q) {
        const float4 v = __ldg(r4 + q);
        acc(4 * q + 0, v.x);
        acc(4 * q + 1, v.y);
        acc(4 * q + 2, v.z);
        acc(4 * q + 3, v.w);
      }
    } else {
#pragma unroll
      for (int e = 0; e < D; ++e) acc(e, __ldg(row + e));
    }
    bool near = false;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float raw = c3[ch] + 0.5f;
      near |= fabsf(raw) <= fmaf(kShGateRel, a3[ch], 1e-7f);
      rgb[ch] = fmaxf(raw, 0.0f);
    }
    if (near) sh_colour64<DEG>(row, ox, oy, oz, rgb);
  }
#else
  sh_colour64<DEG>(row, ox, oy, oz, rgb);
#endif
  SplatRec rec;
  rec.mx = mx;
  rec.my = my;
  const double idet = 1.0 / det;
  rec.ca = c * idet;  // conic = adj(Sigma2) / det (render.py:176-181)
  rec.cb = -b * idet;
  rec.cc = a * idet;
  const double opac = 1.0 / (1.0 + exp(-static_cast<double>(pre.logit)));
  rec.opac = static_cast<float>(opac);
  rec.r = rgb[0];
  rec.g = rgb[1];
  rec.b = rgb[2];
  // Contribution box for the raster's warp-level skip: pixels whose centre
  // lies outside the bounding box of {d : o exp(-d^T conic d / 2) >= 1/255}
  // have alpha < 1/255 in the reference's float64 arithmetic (render.py:
  // 274-280), so they are never kept there and skipping them is exact.  The
  // box half-widths are sqrt(t Sigma2_xx), sqrt(t Sigma2_yy) with
  // t = 2 ln(255 o), widened by a relative 1e-7 for rounding; it lies inside
  // the pixel rect (o < 1, Sigma2_xx <= lambda_max).  o < 1/255: no pixel.
  {
    const double t = 2.0 * log(255.0 * opac) * (1.0 + 1e-7) + 1e-12;
    uint16_t bx0 = 0xffff, bx1 = 0, by0 = 0xffff, by1 = 0;
    if (t > 0.0) {
      const double hx = sqrt(t * a) * (1.0 + 1e-7) + 1e-7;
      const double hy = sqrt(t * c) * (1.0 + 1e-7) + 1e-7;
      const double cx0 = fmax(x0, ceil(mx - hx - 0.5)), cx1 = fmin(x1, floor(mx + hx - 0.5));
      const double cy0 = fmax(y0, ceil(my - hy - 0.5)), cy1 = fmin(y1, floor(my + hy - 0.5));
      if (cx0 <= cx1 && cy0 <= cy1) {
        bx0 = static_cast<uint16_t>(cx0);
        bx1 = static_cast<uint16_t>(cx1);
        by0 = static_cast<uint16_t>(cy0);
        by1 = static_cast<uint16_t>(cy1);
      }
    }
    rec.px0 = bx0;  // empty box: px0 = py0 = 0xffff
    rec.px1 = bx1;
    rec.py0 = by0;
    rec.py1 = by1;
  }
  out.recs[s] = rec;
  out.depth_key[s] = static_cast<uint64_t>(__double_as_longlong(tz));
  // 24-bit depth key: the fp32 bits of tz rounded toward zero (monotone for
  // tz > 0), offset from the near plane's and dropping kDepthKeyShift low
  // bits (relative resolution 2^-19; deeper than ~4e7 clamps) -- 3 sort passes
  // instead of 4; equal keys are ordered by (fp64 depth, id) afterwards
  const uint32_t kb = __float_as_uint(__double2float_rz(tz)) - kDepthKeyBase;
  const uint32_t key = min(kb >> kDepthKeyShift, kDepthKeyMax);
  out.n_tiles[s] = static_cast<uint32_t>((ty1 - ty0 + 1) * (tx1 - tx0 + 1));
  out.rect[s] = static_cast<uint64_t>(tx0) | (static_cast<uint64_t>(tx1) << 16) |
                (static_cast<uint64_t>(ty0) << 32) | (static_cast<uint64_t>(ty1) << 48);
  return key;
}

// Grid-stride over all splats of the frame; also builds the depth sort's
// 4-pass digit histogram (warp-aggregated shared counters, one global
// atomic per non-zero bin per CTA) so the sort skips its histogram pass.
template <int DEG>
#ifndef CGS_PROJECT_HIST_DIRECT
#define CGS_PROJECT_HIST_DIRECT 1
#endif
// 4 CTAs per SM (64 registers, a few spilled): the projection is latency
// bound on its gathers; occupancy beats the spills (config 3: 345 -> 277 us;
// loading the next iteration's inputs ahead measured no better)
#ifndef CGS_PROJECT_MINB
#define CGS_PROJECT_MINB 4
#endif
__global__ void __launch_bounds__(256, CGS_PROJECT_MINB) project_kernel(ProjIn in, FrameDesc fd, ProjOut out) {
  __shared__ uint32_t s_h[4 * 256];
  __shared__ uint32_t s_wc[8];
  __shared__ unsigned long long s_base;
  for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) s_h[k] = 0;
  __syncthreads();
  const int64_t vn = in.n * fd.n_views;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // consecutive threads take the views of one Gaussian: its gathers
  // (position, logit, indices, SR / SH rows) coalesce across the views
  const int nv = fd.n_views;
  auto gauss_of = [nv, vn](int64_t t) -> int64_t {
    if (nv == 1) return t;
    return vn < (int64_t{1} << 32) ? static_cast<uint32_t>(t) / static_cast<uint32_t>(nv) : t / nv;
  };
  int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x);
  for (; b < vn; b += stride) {
    const int64_t t = b + threadIdx.x;
    const bool ok = t < vn;
    const int64_t gi = gauss_of(t);
    const int v = static_cast<int>(t - gi * fd.n_views);
    const int64_t s = static_cast<int64_t>(v) * in.n + gi;
    const uint32_t key = ok ? project_one<DEG>(in, fd, out, s, v, load_pre(in, gi)) : 0xffffffffu;
    // the depth sort takes only the splats with tiles: (key, splat id)
    // appended in any order (its ties are ordered by (fp64 depth, id)
    // afterwards, depth_tie_fix_kernel), one global atomic per CTA iteration
    const bool on = key != 0xffffffffu;
    const unsigned bal = __ballot_sync(kFull, on);
    if (lane == 0) s_wc[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < 8; ++w) tot += s_wc[w];
      s_base = tot ? atomicAdd(&out.hdr->n_onscreen, static_cast<unsigned long long>(tot)) : 0ull;
    }
    __syncthreads();
    if (on) {
      uint32_t pos = __popc(bal & lanemask_lt());
      for (int w = 0; w < warp; ++w) pos += s_wc[w];
      out.dkey[s_base + pos] = key;
      out.dval[s_base + pos] = static_cast<uint32_t>(s);
    }
#if CGS_PROJECT_HIST_DIRECT
    // low two bytes of a depth key are spread over the digits: one shared
    // atomic per lane is cheaper than eight ballots; the top byte (high
    // exponent bits) takes few values, so it is warp-aggregated
#pragma unroll
    for (int p = 0; p < kDepthPasses - 1; ++p)
      if (on) atomicAdd(&s_h[p * 256 + ((key >> (8 * p)) & 255u)], 1u);
    {
      const unsigned d = (key >> (8 * (kDepthPasses - 1))) & 255u;
      const unsigned peers = warp_peers8(d) & bal;
      if (on && lane == __ffs(peers) - 1)
        atomicAdd(&s_h[(kDepthPasses - 1) * 256 + d], __popc(peers));
    }
#else
#pragma unroll
    for (int p = 0; p < kDepthPasses; ++p) {
      const unsigned d = (key >> (8 * p)) & 255u;
      const unsigned peers = warp_peers8(d) & bal;
      if (on && lane == __ffs(peers) - 1) atomicAdd(&s_h[p * 256 + d], __popc(peers));
    }
#endif
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x)
    if (s_h[k]) atomicAdd(&out.hist[k], s_h[k]);
}

// ---------------------------------------------------------------------------
// Exact order inside runs of equal depth keys, into a second buffer: each
// element of a run is placed at the run start + its rank by (fp64 depth bits,
// splat id) among the run -- positive doubles order as integers, and within
// one view the splat id orders as the Gaussian index -- so the order is the
// reference's lexsort((idx, tz)) (render.py:203) whatever order the keys were
// appended in; every other element is copied.  Runs are short (a few splats:
// the 24-bit key resolves depth to 2^-19 relative), and one thread per
// element keeps a run parallel.  An element never scans further than
// kTieDirect either way: a longer run (many splats at one depth, e.g. a
// fronto-parallel plane) is listed by its first element and sorted by
// depth_tie_long_kernel instead.
constexpr int kTieDirect = 256;
constexpr int kTieSmem = 8192;  // longest run sorted in shared memory (bitonic)
__global__ void __launch_bounds__(256) depth_tie_fix_kernel(const uint32_t* __restrict__ key,
                                                            const uint32_t* __restrict__ val,
                                                            uint32_t* __restrict__ out,
                                                            const uint64_t* __restrict__ depth_key,
                                                            const unsigned long long* __restrict__ n_dev,
                                                            uint32_t* __restrict__ long_runs,
                                                            unsigned long long* __restrict__ n_long) {
  const int64_t vn = static_cast<int64_t>(*n_dev);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < vn;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = key[i];
    const uint32_t vi = val[i];
    const bool left = i > 0 && key[i - 1] == k, right = i + 1 < vn && key[i + 1] == k;
    if (!left && !right) {
      out[i] = vi;
      continue;
    }
    int64_t s = i, e = i + 1;
    while (s > 0 && key[s - 1] == k && i - s <= kTieDirect) --s;
    while (e < vn && key[e] == k && e - i <= kTieDirect) ++e;
    if (e - s > kTieDirect) {  // a long run: its first element lists it
      if (!left) long_runs[atomicAdd(n_long, 1ull)] = static_cast<uint32_t>(i);
      continue;
    }
    const uint64_t di = depth_key[vi];
    int64_t r = 0;
    for (int64_t j = s; j < e; ++j) {
      const uint32_t vj = val[j];
      const uint64_t dj = depth_key[vj];
      r += (dj < di || (dj == di && vj < vi)) ? 1 : 0;
    }
    out[s + r] = vi;
  }
}

// One CTA per long run (depth_tie_fix_kernel's list): (fp64 depth bits, id)
// pairs bitonic-sorted in shared memory for runs up to kTieSmem; a longer run
// falls back to the per-element rank (quadratic in its length, but correct).
__global__ void __launch_bounds__(1024) depth_tie_long_kernel(const uint32_t* __restrict__ key,
                                                              const uint32_t* __restrict__ val,
                                                              uint32_t* __restrict__ out,
                                                              const uint64_t* __restrict__ depth_key,
                                                              const unsigned long long* __restrict__ n_dev,
                                                              const uint32_t* __restrict__ long_runs,
                                                              const unsigned long long* __restrict__ n_long) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kTieSmem);
  __shared__ int s_more;
  const int64_t vn = static_cast<int64_t>(*n_dev);
  const int64_t nl = static_cast<int64_t>(*n_long);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t q = blockIdx.x; q < nl; q += gridDim.x) {
    const int64_t s = long_runs[q];
    const uint32_t k = key[s];
    // run end: advance a CTA-wide window until an element differs
    int64_t e = s;
    for (;;) {
      const int64_t j = e + tid;
      const bool same = j < vn && key[j] == k;
      const int all = __syncthreads_and(same);
      if (all) {
        e += nt;
        continue;
      }
      // first differing position in this window
      if (tid == 0) s_more = nt;
      __syncthreads();
      if (!same) atomicMin(&s_more, tid);
      __syncthreads();
      e += s_more;
      __syncthreads();
      break;
    }
    const int64_t L = e - s;
    if (L <= kTieSmem) {
      int P = 1;
      while (P < L) P <<= 1;
      for (int t = tid; t < P; t += nt) {
        if (t < L) {
          const uint32_t v = val[s + t];
          sv[t] = v;
          sk[t] = depth_key[v];
        } else {
          sv[t] = 0xffffffffu;
          sk[t] = ~0ull;
        }
      }
      __syncthreads();
      for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int t = tid; t < P; t += nt) {
            const int o = t ^ stride;
            if (o > t) {
              const bool up = (t & size) == 0;
              const bool gt = sk[t] > sk[o] || (sk[t] == sk[o] && sv[t] > sv[o]);
              if (gt == up) {
                const uint64_t tk = sk[t];
                sk[t] = sk[o];
                sk[o] = tk;
                const uint32_t tv = sv[t];
                sv[t] = sv[o];
                sv[o] = tv;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int t = tid; t < L; t += nt) out[s + t] = sv[t];
      __syncthreads();
    } else {
      for (int64_t i = s + tid; i < e; i += nt) {
        const uint32_t vi = val[i];
        const uint64_t di = depth_key[vi];
        int64_t r = 0;
        for (int64_t j = s; j < e; ++j) {
          const uint32_t vj = val[j];
          const uint64_t dj = depth_key[vj];
          r += (dj < di || (dj == di && vj < vi)) ? 1 : 0;
        }
        out[s + r] = vi;
      }
    }
  }
}

// Pair offsets in depth order (perm = depth rank -> splat), stored per splat.
struct PairOffsets {
  const uint32_t* perm;
  const uint32_t* n_tiles;
  uint64_t* off;
  uint64_t* off_rank;
  FrameHeader* hdr;
  int64_t pair_cap;
  int n_views;
  __device__ uint64_t load(int64_t r) const { return n_tiles[perm[r]]; }
  __device__ void store(int64_t r, uint64_t ex, uint64_t v) const {
    off_rank[r] = ex;
    if (v) off[perm[r]] = ex;
  }
  // pair total -> frame counts and the overflow flag (the rest of the
  // frame reads these)
  __device__ void finish(uint64_t raw) const {
    const bool over = raw > static_cast<unsigned long long>(pair_cap);
    hdr->n_pairs_raw = raw;
    hdr->n_pairs = over ? 0ULL : raw;
    hdr->stats.n_onscreen = static_cast<int64_t>(hdr->n_onscreen);
    hdr->stats.n_pairs = static_cast<int64_t>(raw);
    hdr->stats.overflow = over ? 1 : 0;
    hdr->stats.pair_capacity = pair_cap;
    hdr->stats.n_views = n_views;
    hdr->stats.n_processed = 0;  // the backward's counters (pull_back_kernel publishes them)
    hdr->stats.n_touched = 0;
  }
};


// Warp-cooperative pair emission in depth order: a warp takes 32
// consecutive depth ranks and writes the pairs of those with at most
// kLongSplat tiles with all 32 lanes (warp-local offsets from a shuffle scan).
// Longer splats -- near-plane giants covering every tile sit together at the
// front of the depth order -- are appended to long_list and emitted by
// emit_long_pairs_kernel, one CTA per splat, so no warp serialises on them.
// Within one splat, tiles are emitted row-major over its tile rect.
template <typename KT>
__device__ __forceinline__ uint32_t emit_one(uint64_t p, int k, uint64_t rc, int ntx, int tbase,
                                             uint32_t s, KT* keys, uint32_t* vals) {
  const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
  const int ty0 = static_cast<int>((rc >> 32) & 0xffff);
  const int span = tx1 - tx0 + 1;
  const uint32_t t = static_cast<uint32_t>(tbase + (ty0 + k / span) * ntx + tx0 + k % span);
  keys[p] = static_cast<KT>(t);
  vals[p] = s;
  return t;
}

// Adds the tile keys of the warp's live lanes to the shared digit histogram.
template <typename KT>
__device__ __forceinline__ void hist_keys(uint32_t* s_h, int passes, int key_bits, uint32_t key,
                                          bool live, int lane) {
  const unsigned valid = __ballot_sync(kFull, live);
  if (!valid) return;
  for (int p = 0; p < passes; ++p) {
    const unsigned d = (key >> (8 * p)) & 255u;
    const unsigned peers = warp_peers_bits(d, key_bits - 8 * p) & valid;
    if (live && lane == __ffs(peers) - 1) atomicAdd(&s_h[p * 256 + d], __popc(peers));
  }
}

// Tile-sort digit histogram of one splat's tiles, per row of its rect
// instead of per pair: a row is a contiguous range [a, b] of tile ids, so the
// low digit (t & 255) gets a wrapped range increment (difference array d0 +
// a count base0 added to every digit) and each higher digit (t >> 8p) is
// constant over whole 256^p-aligned segments (one add per segment).
__device__ __forceinline__ void hist_rect(uint32_t* s_h, int* d0, int* base0, int passes,
                                          uint64_t rc, int ntx, int tbase) {
  const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
  const int ty0 = static_cast<int>((rc >> 32) & 0xffff), ty1 = static_cast<int>((rc >> 48) & 0xffff);
  for (int ty = ty0; ty <= ty1; ++ty) {
    const uint32_t a = static_cast<uint32_t>(tbase + ty * ntx + tx0);
    const uint32_t b = a + static_cast<uint32_t>(tx1 - tx0);
    const uint32_t len = b - a + 1u;
    if (len >> 8) atomicAdd(base0, static_cast<int>(len >> 8));
    const uint32_t rem = len & 255u;
    if (rem) {
      const uint32_t st = a & 255u, en = st + rem;  // digits [st, en) mod 256
      atomicAdd(&d0[st], 1);
      if (en <= 256u) {
        atomicAdd(&d0[en], -1);
      } else {
        atomicAdd(&d0[256], -1);
        atomicAdd(&d0[0], 1);
        atomicAdd(&d0[en - 256u], -1);
      }
    }
    for (int p = 1; p < passes; ++p) {
      const int sh = 8 * p;
      for (uint32_t seg = a >> sh; seg <= (b >> sh); ++seg) {
        const uint32_t lo = max(a, seg << sh), hi = min(b, ((seg + 1u) << sh) - 1u);
        atomicAdd(&s_h[p * 256 + (seg & 255u)], hi - lo + 1u);
      }
    }
  }
}

template <typename KT>
__device__ __forceinline__ void emit_warps(
    const uint32_t* __restrict__ perm, const uint64_t* __restrict__ off_rank,
    const uint64_t* __restrict__ rect,
    FrameHeader* __restrict__ hdr, const FrameDesc& fd, int64_t n, uint32_t* __restrict__ long_list,
    KT* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* s_h, int* d0, int* base0,
    int key_bits) {
  const int passes = (key_bits + 7) / 8;
  if (hdr->stats.overflow) return;
  const int lane = threadIdx.x & 31;
  const int64_t ns = static_cast<int64_t>(hdr->n_onscreen);  // ranks with tiles come first
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w * 32 < ns;
       w += warps) {
    const int64_t r = w * 32 + lane;
    const bool ok = r < ns;
    const uint32_t s = ok ? perm[r] : 0u;
    // offset and tile count from the rank-ordered offsets (coalesced): the
    // count is the next rank's offset minus this one's, the last rank's runs
    // to the pair total (hdr->scratch[0], the scan's total)
    const uint64_t o_r = ok ? off_rank[r] : 0ull;
    uint64_t o_nx = __shfl_down_sync(kFull, o_r, 1);
    if (ok && (lane == 31 || r + 1 >= ns))
      o_nx = r + 1 < ns ? off_rank[r + 1] : static_cast<uint64_t>(hdr->scratch[0]);
    const uint32_t cnt = ok ? static_cast<uint32_t>(o_nx - o_r) : 0u;
    const bool lng = cnt > kLongSplat;
    if (lng) long_list[atomicAdd(&hdr->scratch[2], 1ULL)] = s;
    const uint32_t c = lng ? 0u : cnt;  // pairs this warp emits for lane's splat
    const uint32_t inc = warp_incl_scan(c);
    const uint32_t loc = inc - c;        // warp-local offset of lane's pairs
    const uint32_t total = __shfl_sync(kFull, inc, 31);
    if (total == 0) continue;
    const uint64_t o = o_r;
    const uint64_t rc = c ? rect[s] : 0ULL;
    const int v = ok ? static_cast<int>(s / static_cast<uint32_t>(n)) : 0;
    const int ntx = fd.cam[v].ntx;
    const int tbase = fd.cam[v].tile_base;
    if (c && passes) hist_rect(s_h, d0, base0, passes, rc, ntx, tbase);
    for (uint32_t q0 = 0; q0 < total; q0 += 32) {
      const uint32_t q = q0 + lane;
      const uint32_t end = loc + c;
      int own = 0;  // first lane whose pair range ends after q (ends are nondecreasing)
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int cand = own + step;
        if (__shfl_sync(kFull, end, (cand - 1) & 31) <= q && cand < 32) own = cand;
      }
      const uint64_t oo = __shfl_sync(kFull, o, own);
      const uint32_t lo2 = __shfl_sync(kFull, loc, own);
      const uint64_t rco = __shfl_sync(kFull, rc, own);
      const int nt = __shfl_sync(kFull, ntx, own);
      const int tb = __shfl_sync(kFull, tbase, own);
      const uint32_t so = __shfl_sync(kFull, s, own);
      if (q < total) {
        const int k = static_cast<int>(q - lo2);
        emit_one<KT>(oo + k, k, rco, nt, tb, so, keys, vals);
      }
    }
  }
}

template <typename KT>
__global__ void __launch_bounds__(256) emit_pairs_kernel(
    const uint32_t* __restrict__ perm, const uint64_t* __restrict__ off_rank,
    const uint64_t* __restrict__ rect,
    FrameHeader* __restrict__ hdr, FrameDesc fd, int64_t n, uint32_t* __restrict__ long_list,
    KT* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ hist, int key_bits) {
  const int passes = (key_bits + 7) / 8;
  __shared__ uint32_t s_h[4 * 256];  // tile sort digit histogram (this CTA's pairs)
  __shared__ int s_d0[257];          // low digit as a difference array
  __shared__ int s_base0;
  for (int k = threadIdx.x; k < passes * 256; k += blockDim.x) s_h[k] = 0;
  for (int k = threadIdx.x; k < 257; k += blockDim.x) s_d0[k] = 0;
  if (threadIdx.x == 0) s_base0 = 0;
  __syncthreads();
  emit_warps<KT>(perm, off_rank, rect, hdr, fd, n, long_list, keys, vals, s_h, s_d0, &s_base0,
                 key_bits);
  __syncthreads();
  if (threadIdx.x < 32) {  // low digit: prefix sum of the difference array (8 per lane)
    const int lane = threadIdx.x;
    int v8[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v8[k] = s_d0[lane * 8 + k];
      sum += v8[k];
    }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - sum + s_base0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      run += v8[k];
      s_h[lane * 8 + k] += static_cast<uint32_t>(run);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < passes * 256; k += blockDim.x)
    if (s_h[k]) atomicAdd(&hist[k], s_h[k]);
}


// One CTA per long splat (near-plane giants): its pair range is contiguous.
template <typename KT>
__global__ void __launch_bounds__(256) emit_long_pairs_kernel(
    const uint32_t* __restrict__ long_list, const uint64_t* __restrict__ off,
    const uint32_t* __restrict__ n_tiles, const uint64_t* __restrict__ rect,
    const FrameHeader* __restrict__ hdr, FrameDesc fd, int64_t n, KT* __restrict__ keys,
    uint32_t* __restrict__ vals, uint32_t* __restrict__ hist, int key_bits) {
  const int passes = (key_bits + 7) / 8;
  __shared__ uint32_t s_h[4 * 256];
  if (hdr->stats.overflow) return;
  const int64_t nl = static_cast<int64_t>(hdr->scratch[2]);
  if (blockIdx.x >= nl) return;
  for (int k = threadIdx.x; k < passes * 256; k += blockDim.x) s_h[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t e = blockIdx.x; e < nl; e += gridDim.x) {
    const uint32_t s = long_list[e];
    const uint64_t o = off[s];
    const int cnt = static_cast<int>(n_tiles[s]);
    const uint64_t rc = rect[s];
    const int v = static_cast<int>(s / static_cast<uint32_t>(n));
    for (int k0 = 0; k0 < cnt; k0 += blockDim.x) {
      const int k = k0 + threadIdx.x;
      uint32_t key = 0;
      if (k < cnt) key = emit_one<KT>(o + k, k, rc, fd.cam[v].ntx, fd.cam[v].tile_base, s, keys, vals);
      hist_keys<KT>(s_h, passes, key_bits, key, k < cnt, lane);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < passes * 256; k += blockDim.x)
    if (s_h[k]) atomicAdd(&hist[k], s_h[k]);
}

template <typename KT>
__global__ void __launch_bounds__(256) tile_ranges_kernel(const KT* __restrict__ keys,
                                                          const FrameHeader* __restrict__ hdr,
                                                          uint2* __restrict__ ranges) {
  const int64_t np = static_cast<int64_t>(hdr->n_pairs);
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < np;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const KT t = keys[p];
    if (p == 0 || keys[p - 1] != t) ranges[t].x = static_cast<uint32_t>(p);
    if (p == np - 1 || keys[p + 1] != t) ranges[t].y = static_cast<uint32_t>(p + 1);
  }
}

// ---------------------------------------------------------------------------
// One-pass counting tile sort (frames of <= kCountMaxTiles tiles).  The
// emission order is (depth rank, tile row-major in the splat's rect) and a
// splat meets each tile once, so a stable sort by tile only has to keep the
// emission order among the pairs of one tile (render.py:240-254).  Pairs are
// cut into chunks of 2^count_log2 consecutive emission indices:
//   tile_count   per chunk, the count of each tile -> tcount[t * C + c]
//   scan_kernel  exclusive scan of the flattened tile-major matrix: entry
//                (t, c) becomes the first output position of chunk c's pairs
//                of tile t (all chunks of earlier tiles come first)
//   tile_scatter per chunk, 8 warps over 8 consecutive slices: each warp
//                counts its slice per tile (u16 counters in shared memory),
//                an exclusive sum over the warps places the slices, then each
//                warp walks its slice in order, 32 pairs at a time ranked by
//                match.any peers, and writes each splat id at its position.
// One read of the keys to count, one read of keys + ids and one write of the
// ids to scatter, against 2 onesweep passes (keys and ids read and written
// twice, plus the per-digit lookback) -- and the tile ranges come out of the
// scan (no tile_ranges pass).
// Loads are batched ahead of their use (the counting is shared-memory
// atomics and ordered shared updates, so without it every iteration waits a
// full memory latency).
constexpr int kCountLoadBatch = 8;

__global__ void __launch_bounds__(256) tile_count_kernel(const uint16_t* __restrict__ keys,
                                                         const FrameHeader* __restrict__ hdr,
                                                         int tiles, int log2cp,
                                                         uint32_t* __restrict__ tcount,
                                                         unsigned long long* __restrict__ scan_n,
                                                         uint2* __restrict__ ranges) {
  extern __shared__ uint32_t s_cnt[];  // tiles
  const int64_t np = static_cast<int64_t>(hdr->n_pairs);  // 0 on overflow
  const int64_t C = (np + (1LL << log2cp) - 1) >> log2cp;
  if (blockIdx.x == 0 && threadIdx.x == 0) *scan_n = static_cast<unsigned long long>(tiles) * C;
  if (C == 0 && blockIdx.x == 0)  // no pairs: empty ranges (else tile_scatter's chunk 0 writes them)
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) ranges[t] = make_uint2(0u, 0u);
  const int64_t c = blockIdx.x;
  if (c >= C) return;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) s_cnt[t] = 0u;
  __syncthreads();
  const int64_t b = c << log2cp;
  const int64_t e = min(b + static_cast<int64_t>(1LL << log2cp), np);
  // chunk starts are 8 KB aligned: 16-byte loads of 8 keys, kCountLoadBatch
  // of them in flight per thread
  constexpr int64_t kStep = 8 * 256;
  for (int64_t i0 = b + 8 * threadIdx.x; i0 < e; i0 += kCountLoadBatch * kStep) {
    uint4 q[kCountLoadBatch];
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      const int64_t i = i0 + u * kStep;
      q[u] = i + 8 <= e ? *reinterpret_cast<const uint4*>(keys + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      const int64_t i = i0 + u * kStep;
      if (i + 8 <= e) {
        const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          atomicAdd(&s_cnt[w[k] & 0xffffu], 1u);
          atomicAdd(&s_cnt[w[k] >> 16], 1u);
        }
      } else {
        for (int64_t j = i; j < e; ++j) atomicAdd(&s_cnt[keys[j]], 1u);
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) tcount[t * C + c] = s_cnt[t];
}

// In-place exclusive scan of the tile-major count matrix, each result also
// written to the chunk-major matrix the scatter reads one row of (the
// scattered transposing stores are fire-and-forget here; as loads in the
// scatter they would stall it).
struct TileCountScan {
  uint32_t* m;           // tiles x C, tile-major
  uint32_t* mt;          // C x tiles, chunk-major
  const unsigned long long* n;  // tiles * C
  uint32_t tiles;
  __device__ uint64_t load(int64_t i) const { return m[i]; }
  __device__ void store(int64_t i, uint64_t ex, uint64_t) const {
    // tiles x C < 2^32 (kCountMaxTiles x the chunk count); __ldg lets the
    // compiler load the count once per thread, not once per element
    const uint32_t C = static_cast<uint32_t>(__ldg(n)) / tiles;
    const uint32_t t = static_cast<uint32_t>(i) / C, c = static_cast<uint32_t>(i) - t * C;
    mt[static_cast<int64_t>(c) * tiles + t] = static_cast<uint32_t>(ex);
  }
  __device__ void finish(uint64_t) const {}
};

// Timing experiments only (wrong results): 1 no stores, 2 no ranking pass,
// 3 prologue only, 4 no duplicate test, 5 also no counter atomics, 6 also no
// stores.  Config 3 (12.2 M pairs): 184 / 144 / 35 / 12 / 137 / 124 / 66 us
// -- the scattered id stores (~58 us) and the phase-c loads (~31 us) at 8
// warps per SM (the per-warp counter rows) are the floor of this design.
#ifndef CGS_SCATTER_DIAG
#define CGS_SCATTER_DIAG 0
#endif
constexpr int kCountKeyLoads = 16;
constexpr int kTagSlots = 2048;  // per-warp duplicate test slots (u8 lane ids)  // phase a: a 4096-key slice in one round of loads

__global__ void __launch_bounds__(kCountWarps * 32) tile_scatter_kernel(
    const uint16_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    const FrameHeader* __restrict__ hdr, int tiles, int log2cp, int key_bits,
    const uint32_t* __restrict__ toff, uint32_t* __restrict__ out, uint2* __restrict__ ranges) {
  extern __shared__ uint32_t s_dyn[];
  const int tpad = (tiles + 1) & ~1;  // u16 rows of whole words
  uint32_t* s_off = s_dyn;                                          // tiles
  uint16_t* s_pre = reinterpret_cast<uint16_t*>(s_dyn + tpad);      // kCountWarps x tpad
  const int64_t np = static_cast<int64_t>(hdr->n_pairs);
  const int64_t C = (np + (1LL << log2cp) - 1) >> log2cp;
  const int64_t c = blockIdx.x;
  if (c >= C) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = kCountWarps * 32;
  const uint32_t* row = toff + c * tiles;  // this chunk's first position per tile
  for (int t = tid; t < tiles; t += NT) s_off[t] = row[t];
  uint32_t* s_pre32 = reinterpret_cast<uint32_t*>(s_pre);
  for (int k = tid; k < kCountWarps * tpad / 2; k += NT) s_pre32[k] = 0u;
  __syncthreads();
  if (c == 0)  // chunk 0's entries are the tile starts
    for (int t = tid; t < tiles; t += NT)
      ranges[t] = make_uint2(s_off[t], t + 1 < tiles ? s_off[t + 1] : static_cast<uint32_t>(np));
  const int64_t b = c << log2cp;
  const int64_t e = min(b + static_cast<int64_t>(1LL << log2cp), np);
  const int64_t slice = (1LL << log2cp) / kCountWarps;  // 512 .. 4096, a multiple of 256
  const int64_t wb = min(b + warp * slice, e), we = min(wb + slice, e);
  uint16_t* my = s_pre + warp * tpad;
  uint32_t* my32 = reinterpret_cast<uint32_t*>(my);
  uint8_t* tag = reinterpret_cast<uint8_t*>(s_pre + kCountWarps * tpad) + warp * kTagSlots;
  if (CGS_SCATTER_DIAG == 3) return;
  {  // the warp's slice per tile: 16-byte loads of 8 keys (slices are 1 KB aligned), all at once
    uint4 q[kCountKeyLoads];
#pragma unroll
    for (int u = 0; u < kCountKeyLoads; ++u) {
      const int64_t i = wb + 8 * lane + u * 256;
      q[u] = i + 8 <= we ? *reinterpret_cast<const uint4*>(keys + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kCountKeyLoads; ++u) {
      const int64_t i = wb + 8 * lane + u * 256;
      if (i + 8 <= we) {
        const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          atomicAdd(&my32[(w[k] & 0xffffu) >> 1], 1u << ((w[k] & 1u) << 4));
          atomicAdd(&my32[w[k] >> 17], 1u << (((w[k] >> 16) & 1u) << 4));
        }
      } else {
        for (int64_t j = i; j < we && j < i + 8; ++j) {
          const uint32_t t = keys[j];
          atomicAdd(&my32[t >> 1], 1u << ((t & 1u) << 4));
        }
      }
    }
  }
  __syncthreads();
  for (int t = tid; t < tiles; t += NT) {  // slices placed in warp order
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kCountWarps; ++w) {
      const uint32_t x = s_pre[w * tpad + t];
      s_pre[w * tpad + t] = static_cast<uint16_t>(run);
      run += x;
    }
  }
  __syncthreads();
  // In order, 32 pairs at a time; the next kCountLoadBatch groups load while
  // this batch is ranked.  Per group the leader of each peer set (ballots
  // over the key bits) takes its range with one shared atomic that returns
  // the counter; a warp's atomics on one word execute in program order, so
  // the ranges follow the emission order.
  if (CGS_SCATTER_DIAG == 2) return;
  uint32_t tk[kCountLoadBatch], sv[kCountLoadBatch];
  auto load_batch = [&](int64_t g0, uint32_t (&k)[kCountLoadBatch], uint32_t (&v)[kCountLoadBatch]) {
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      const int64_t i = g0 + u * 32 + lane;
      k[u] = i < we ? static_cast<uint32_t>(keys[i]) : 0xffffffffu;
      v[u] = i < we ? vals[i] : 0u;
    }
  };
  load_batch(wb, tk, sv);
  for (int64_t g0 = wb; g0 < we; g0 += kCountLoadBatch * 32) {
    uint32_t nk[kCountLoadBatch], nv[kCountLoadBatch];
    load_batch(g0 + kCountLoadBatch * 32, nk, nv);
    // Peers (lanes with the same tile): most groups have none.  Each lane
    // writes its id into a per-warp tag slot of its tile (t mod kTagSlots)
    // and reads it back; if no lane lost its slot the 32 tiles are distinct.
    // Otherwise one ballot per key bit.
    unsigned peers[kCountLoadBatch];
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      const uint32_t t = tk[u];
      const bool ok = t != 0xffffffffu;
      bool lost = false;
      if (CGS_SCATTER_DIAG < 4) {
        if (ok) tag[t & (kTagSlots - 1)] = static_cast<uint8_t>(lane);
        __syncwarp();
        lost = ok && tag[t & (kTagSlots - 1)] != lane;
        __syncwarp();
      }
      peers[u] = 1u << lane;
      if (CGS_SCATTER_DIAG < 4 && __any_sync(kFull, lost)) {
        unsigned pm = kFull;
        for (int bit = 0; bit < key_bits; ++bit) {
          const bool on = (t >> bit) & 1u;
          const unsigned bal = __ballot_sync(kFull, on);
          pm &= on ? bal : ~bal;
        }
        if (ok) peers[u] = pm;
      }
    }
    uint32_t old[kCountLoadBatch];
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      const uint32_t t = tk[u];
      old[u] = 0u;
      if (CGS_SCATTER_DIAG < 5 && t != 0xffffffffu && (peers[u] & lanemask_lt()) == 0u)
        old[u] = atomicAdd(&my32[t >> 1], static_cast<uint32_t>(__popc(peers[u])) << ((t & 1u) << 4)) >>
                 ((t & 1u) << 4);
    }
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      const uint32_t t = tk[u];
      const uint32_t base = __shfl_sync(kFull, old[u], __ffs(peers[u]) - 1) & 0xffffu;
      if (t != 0xffffffffu && ((CGS_SCATTER_DIAG != 1 && CGS_SCATTER_DIAG < 6) || sv[u] == 0xfffffffu))
        out[s_off[t] + base + __popc(peers[u] & lanemask_lt())] = sv[u];
    }
#pragma unroll
    for (int u = 0; u < kCountLoadBatch; ++u) {
      tk[u] = nk[u];
      sv[u] = nv[u];
    }
  }
}

static int count_sort_pairs(FrameLayout& L, const FrameDesc& fd, cudaStream_t st) {
  const int T = fd.total_tiles;
  const size_t smem_count = static_cast<size_t>(T) * sizeof(uint32_t);
  const int tpad = (T + 1) & ~1;
  const size_t smem_scatter = static_cast<size_t>(tpad) * 4 + static_cast<size_t>(kCountWarps) * tpad * 2 +
                              static_cast<size_t>(kCountWarps) * kTagSlots;
  static std::atomic<bool> attr[kMaxDevices] = {};
  int dev = 0;
  if (int e = current_device(&dev)) return e;
  if (!attr[dev].load()) {
    constexpr int kMaxCount = kCountMaxTiles * 4;
    constexpr int kMaxScatter = (kCountMaxTiles + 1) * 4 + kCountWarps * (kCountMaxTiles + 1) * 2 +
                                kCountWarps * kTagSlots;
    CGS_CUDA(cudaFuncSetAttribute(tile_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxCount));
    CGS_CUDA(cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxScatter));
    attr[dev].store(true);
  }
  const unsigned grid = static_cast<unsigned>(L.count_chunks_cap > 0 ? L.count_chunks_cap : 1);
  const uint16_t* keys = static_cast<const uint16_t*>(L.pkeys);
  CGS_PROFILED("tile_count_kernel", st,
               tile_count_kernel<<<grid, 256, smem_count, st>>>(keys, L.hdr, T, L.count_log2,
                                                                L.tcount, L.tcount_n, L.ranges));
  CGS_CHECK_LAUNCH("tile_count_kernel");
  int rc = launch_scan<TileCountScan, 24>(TileCountScan{L.tcount, L.toff, L.tcount_n, static_cast<uint32_t>(T)}, L.tcount_n, 0,
                       static_cast<int64_t>(T) * L.count_chunks_cap, L.tscan, nullptr, st,
                       /*state_ready=*/L.states_zeroed);
  if (rc) return rc;
  CGS_PROFILED("tile_scatter_kernel", st,
               tile_scatter_kernel<<<grid, kCountWarps * 32, smem_scatter, st>>>(
                   keys, L.pvals, L.hdr, T, L.count_log2, bits_for(T), L.toff, sorted_pair_vals(L), L.ranges));
  CGS_CHECK_LAUNCH("tile_scatter_kernel");
  return CGS_OK;
}

// ---------------------------------------------------------------------------
template <int DEG>
static void launch_project(const ProjIn& in, const FrameDesc& fd, const ProjOut& out,
                           int64_t vn, cudaStream_t st) {
  CGS_PROFILED("project_kernel", st,
               project_kernel<DEG><<<grid_for(vn, 256, 16), 256, 0, st>>>(in, fd, out));
}

template <typename KT>
static int emit_pairs_stage(FrameLayout& L, const FrameDesc& fd, SortWs<KT>& ws,
                            const uint32_t* perm, cudaStream_t st) {
  const int eg = grid_for(L.vn, 256, 16);
  // the emission kernels also build the onesweep tile sort's digit histogram
  // (key_bits 0: none, the counting tile sort counts for itself)
  const int key_bits = L.count_sort ? 0 : L.tile_key_bits;
  const int passes = (key_bits + 7) / 8;
  if (passes) CGS_CUDA(cudaMemsetAsync(ws.hist, 0, passes * 256 * sizeof(uint32_t), st));
  CGS_PROFILED("emit_pairs_kernel", st,
               emit_pairs_kernel<KT><<<eg, 256, 0, st>>>(perm, L.off_rank, L.rect, L.hdr,
                                                          fd, L.n, L.long_list,
                                                          static_cast<KT*>(L.pkeys), L.pvals,
                                                          ws.hist, key_bits));
  CGS_CHECK_LAUNCH("emit_pairs_kernel");
  emit_long_pairs_kernel<KT><<<148 * 4, 256, 0, st>>>(L.long_list, L.pair_off, L.n_tiles, L.rect,
                                                       L.hdr, fd, L.n, static_cast<KT*>(L.pkeys),
                                                       L.pvals, ws.hist, key_bits);
  CGS_CHECK_LAUNCH("emit_long_pairs_kernel");
  return CGS_OK;
}

template <typename KT>
static int sort_pairs_stage(FrameLayout& L, const FrameDesc& fd, SortWs<KT>& ws, cudaStream_t st) {
  KT* kres;
  uint32_t* vres;
  int rc = launch_radix_sort<KT>(static_cast<KT*>(L.pkeys), L.pvals, &L.hdr->n_pairs, 0,
                                 L.pair_cap, L.tile_key_bits, ws, &kres, &vres, st,
                                 /*hist_ready=*/true);
  if (rc) return rc;
  if (vres != sorted_pair_vals(L)) {
    set_error("tile sort: unexpected result buffer");
    return CGS_EINTERNAL;
  }
  CGS_CUDA(cudaMemsetAsync(L.ranges, 0, sizeof(uint2) * (fd.total_tiles > 0 ? fd.total_tiles : 1), st));
  tile_ranges_kernel<KT><<<grid_for(L.pair_cap, 256, 8), 256, 0, st>>>(kres, L.hdr, L.ranges);
  CGS_CHECK_LAUNCH("tile_ranges_kernel");
  return CGS_OK;
}

// The frame forward in five stages (exported one by one as cgs_project,
// cgs_sort_depth, cgs_duplicate_tiles, cgs_sort_pairs, cgs_raster_fwd; each
// reads only what the earlier stages left in the frame workspace).
int frame_stage_project(const cgs_scene_t* sc, const FrameDesc& fd, FrameLayout& L,
                        double* sr_cov, cudaStream_t st) {
  const int64_t vn = L.vn;
  static_assert(sizeof(FrameHeader) % sizeof(uint32_t) == 0, "header zeroed as words");
  L.states_zeroed = false;
  if (sc->sr_capacity > 0) {
    // it also zeroes the frame header, the depth-sort histogram and the
    // depth sort's / the two scans' states (the later launches skip their memsets)
    ZeroSpans z{};
    auto put = [&](int q, void* p, size_t bytes) {
      z.p[q] = static_cast<uint32_t*>(p);
      z.n[q] = static_cast<int64_t>(bytes / sizeof(uint32_t));
    };
    put(0, L.hdr, sizeof(FrameHeader));
    put(1, L.dsort.hist, 4 * 256 * sizeof(uint32_t));
    const ZeroSpan a = sort_state_span(L.dsort), b = scan_state_span(L.scan);
    put(2, a.p, a.bytes);
    put(3, b.p, b.bytes);
    if (L.count_sort) {
      const ZeroSpan c = scan_state_span(L.tscan);
      put(4, c.p, c.bytes);
    }
    CGS_PROFILED("sr_precompute_kernel", st,
                 sr_precompute_kernel<<<grid_for(sc->sr_capacity, 256, 4), 256, 0, st>>>(
                     sc->sr_rows, sc->sr_capacity, sr_cov, z));
    CGS_CHECK_LAUNCH("sr_precompute_kernel");
    L.states_zeroed = true;
  } else {
    CGS_CUDA(cudaMemsetAsync(L.hdr, 0, sizeof(FrameHeader), st));
    CGS_CUDA(cudaMemsetAsync(L.dsort.hist, 0, 4 * 256 * sizeof(uint32_t), st));
  }
  if (vn > 0) {
    ProjIn in{sc->n, sc->positions, sc->opacity_logits, sc->g2sh, sc->g2sr, sc->sh_rows, sr_cov};
    ProjOut out{L.recs, L.depth_key, L.dkey, L.dval, L.dsort.hist, L.n_tiles, L.rect, L.hdr};
    switch (sc->sh_degree) {
      case 0: launch_project<0>(in, fd, out, vn, st); break;
      case 1: launch_project<1>(in, fd, out, vn, st); break;
      case 2: launch_project<2>(in, fd, out, vn, st); break;
      default: launch_project<3>(in, fd, out, vn, st); break;
    }
    CGS_CHECK_LAUNCH("project_kernel");
  }
  return CGS_OK;
}

// Depth order of every splat of the frame (all views; the tile sort
// separates the views again), then per-splat pair offsets in that order.
// 3 passes over the 24-bit keys: the permutation ends in the sort's
// alternate value buffer (depth_perm).
int frame_stage_sort_depth(const FrameDesc& fd, FrameLayout& L, cudaStream_t st) {
  const int64_t vn = L.vn;
  uint32_t* perm = depth_perm(L);
  if (vn > 0) {
    uint32_t* kres;
    // the projection appended the splats with tiles (count: hdr->n_onscreen)
    int rc = launch_radix_sort<uint32_t>(L.dkey, L.dval, &L.hdr->n_onscreen, vn, vn,
                                         8 * kDepthPasses, L.dsort, &kres, &perm, st,
                                         /*hist_ready=*/true, /*state_ready=*/L.states_zeroed);
    if (rc) return rc;
    if (perm != L.dsort.vals_alt) {
      set_error("depth sort: unexpected result buffer");
      return CGS_EINTERNAL;
    }
    CGS_PROFILED("depth_tie_fix_kernel", st,
                 depth_tie_fix_kernel<<<grid_for(vn, 256, 8), 256, 0, st>>>(
                     kres, perm, L.dval, L.depth_key, &L.hdr->n_onscreen, L.tie_runs,
                     &L.hdr->scratch[1]));
    CGS_CHECK_LAUNCH("depth_tie_fix_kernel");
    {  // long runs (none in a typical frame: the kernel returns at once)
      constexpr size_t smem = kTieSmem * (sizeof(uint64_t) + sizeof(uint32_t));
      static std::atomic<bool> attr[kMaxDevices] = {};
      int dev = 0;
      if (int e = current_device(&dev)) return e;
      if (!attr[dev].load()) {
        CGS_CUDA(cudaFuncSetAttribute(depth_tie_long_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr[dev].store(true);
      }
      depth_tie_long_kernel<<<148, 1024, smem, st>>>(kres, perm, L.dval, L.depth_key,
                                                     &L.hdr->n_onscreen, L.tie_runs,
                                                     &L.hdr->scratch[1]);
      CGS_CHECK_LAUNCH("depth_tie_long_kernel");
    }
    perm = depth_perm(L);
  }
  int rc = launch_scan(PairOffsets{perm, L.n_tiles, L.pair_off, L.off_rank, L.hdr, L.pair_cap, fd.n_views}, &L.hdr->n_onscreen, vn,
                       vn, L.scan, &L.hdr->scratch[0], st, /*state_ready=*/L.states_zeroed);
  if (rc) return rc;
  return CGS_OK;
}

int frame_stage_duplicate(const FrameDesc& fd, FrameLayout& L, cudaStream_t st) {
  return L.tile_key_bytes == 2 ? emit_pairs_stage<uint16_t>(L, fd, L.psort16, depth_perm(L), st)
                               : emit_pairs_stage<uint32_t>(L, fd, L.psort32, depth_perm(L), st);
}

int frame_stage_sort_pairs(const FrameDesc& fd, FrameLayout& L, cudaStream_t st) {
  if (L.count_sort) return count_sort_pairs(L, fd, st);
  return L.tile_key_bytes == 2 ? sort_pairs_stage<uint16_t>(L, fd, L.psort16, st)
                               : sort_pairs_stage<uint32_t>(L, fd, L.psort32, st);
}

int frame_stage_raster(const FrameDesc& fd, FrameLayout& L, const float* logits, float* image,
                       float* final_T, int32_t* counts, cudaStream_t st) {
  if (fd.total_tiles > 0) {
    int rc = launch_tile_order(fd, L, nullptr, st);
    if (rc) return rc;
    rc = launch_raster_fwd(fd, L, sorted_pair_vals(L), logits, image, final_T, counts, st);
    if (rc) return rc;
  }
  return CGS_OK;
}

int frame_forward(const cgs_scene_t* sc, const FrameDesc& fd, FrameLayout& L, float* image,
                  float* final_T, int32_t* counts, double* sr_cov, cudaStream_t st) {
  int rc = frame_stage_project(sc, fd, L, sr_cov, st);
  if (!rc) rc = frame_stage_sort_depth(fd, L, st);
  if (!rc) rc = frame_stage_duplicate(fd, L, st);
  if (!rc) rc = frame_stage_sort_pairs(fd, L, st);
  if (!rc) rc = frame_stage_raster(fd, L, sc->opacity_logits, image, final_T, counts, st);
  return rc;
}

}  // namespace cgs
