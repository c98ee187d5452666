// Backward render path (reference render.py:318-459) for sm_100a.
//
//   raster_bwd      raster.cu: one CTA per tile, reverse traversal, one
//                   9-float partial per processed pair, stored at the pair's
//                   emission index (render.py:343-377)
//   splat_reduce    per (view, Gaussian) splat: walk its pairs in emission
//                   order (= row-major tile order, the order of np.add.at over
//                   the reference's tile dict) -- contiguous partials -- keep
//                   those inside each tile's processed prefix (depth rank <
//                   the tile's last processed rank), sum them in fp64 and
//                   apply the chain rule to model space (render.py:382-446)
//   gauss_write     per Gaussian: sum over views -> position / logit gradients
//   code reduces    per codebook row through a code -> members CSR (rebuilt
//                   only when assignments change): SH rows = sum basis (x)
//                   d_raw, SR rows = sum dSigma3 then the per-row chain
//                   (render.py:431-458).  No atomics, no per-step sorts.
#include <cmath>
#include <cstddef>

#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

struct BwdHeader {
  unsigned long long n_processed;
  unsigned long long n_touched;
  int nonfinite;  // byte 16: a written gradient entry was non-finite (cgs_backward_nonfinite_flag)
  int pad;
  unsigned long long scratch[5];
};
static_assert(offsetof(BwdHeader, nonfinite) == 16, "ABI: cgs_backward_nonfinite_flag");

struct BwdLayout {
  BwdHeader* hdr;
  float* partials;     // pair_cap * 9, indexed by emission index
  uint8_t* touched;    // V*N
  float4* s_posl;      // V*N: d_pos xyz, d_logit
  float4* s_view;      // V*N: view direction
  float4* s_draw;      // V*N: gated d colour
  float4* s_s3a;       // V*N: dSigma3 00 01 02 11
  float2* s_s3b;       // V*N: dSigma3 12 22
  float4* acc0;        // V*N: summed d_color(3), sum dp (= d_opac * opacity)
  double2* accm;       // V*N: sum dp d (centre-frame first moments, f64)
  double2* accq;       // V*N: sum dp dx^2, sum dp dx dy (second moments, f64)
  double* accr;        // V*N: sum dp dy^2
  uint8_t* code_hit[2];  // sh_cap, sr_cap: the row has a touched member (pull_back_kernel)
  int32_t* csr_off[2];  // internal code CSR (sh, sr) when the caller passes none
  int32_t* csr_mem[2];
  void* csr_ws;
  size_t csr_ws_bytes;
  ScanWs scan;
  size_t bytes;
};

size_t code_csr_ws_bytes(int64_t n, int64_t cap);

// Few touched splats (under 1/8 of the frame's, e.g. config 3 where a hundred
// near-plane splats end every pixel): the pull-back flags the codebook rows
// with a touched member and the codebook reduces skip the other rows' member
// lists.  Dense frames skip the flags (their scattered writes cost more than
// they save).  n_touched is final once the splat reduce kernels ran.
__device__ __forceinline__ bool code_sparse(const BwdLayout& B, int64_t vn) {
  return B.hdr->n_touched * 8ull < static_cast<unsigned long long>(vn);
}

inline BwdLayout plan_bwd(void* base, size_t cap, int64_t n, int n_views, int total_tiles,
                          int64_t pair_cap, int64_t sh_cap, int64_t sr_cap) {
  BwdLayout B{};
  Carver c(base, cap);
  const int64_t pc = pair_cap > 0 ? pair_cap : 1;
  const int64_t vn = n * n_views > 0 ? n * n_views : 1;
  B.hdr = c.take<BwdHeader>(1);
  B.partials = c.take<float>(pc * 9);  // [pc x 8 | pc]: values 0-7 as float4 pairs, value 8
  B.touched = c.take<uint8_t>(vn);
  B.s_posl = c.take<float4>(vn);
  B.s_view = c.take<float4>(vn);
  B.s_draw = c.take<float4>(vn);
  B.s_s3a = c.take<float4>(vn);
  B.s_s3b = c.take<float2>(vn);
  B.acc0 = c.take<float4>(vn);
  B.accm = c.take<double2>(vn);
  B.accq = c.take<double2>(vn);
  B.accr = c.take<double>(vn);
  B.code_hit[0] = c.take<uint8_t>(sh_cap > 0 ? sh_cap : 1);
  B.code_hit[1] = c.take<uint8_t>(sr_cap > 0 ? sr_cap : 1);
  const int64_t n1 = n > 0 ? n : 1;
  B.csr_off[0] = c.take<int32_t>(sh_cap + 1);
  B.csr_mem[0] = c.take<int32_t>(n1);
  B.csr_off[1] = c.take<int32_t>(sr_cap + 1);
  B.csr_mem[1] = c.take<int32_t>(n1);
  B.csr_ws_bytes = code_csr_ws_bytes(n1, sh_cap > sr_cap ? sh_cap : sr_cap);
  B.csr_ws = c.take<unsigned char>(B.csr_ws_bytes);
  B.scan = carve_scan(c, total_tiles > 0 ? total_tiles : 1);
  B.bytes = c.off + 256;
  return B;
}

// ---------------------------------------------------------------------------

struct GaussIn {
  const SplatRec* recs;  // projection records of the frame (conic, clamped colour)
  const float* pos;
  const float* logit;
  const int32_t* g2sh;
  const int32_t* g2sr;
  const float* sh_rows;
  const double* sr_cov;
};

// Chain rule from screen space to model space for one (view, Gaussian)
// splat (render.py:382-446).  acc = [d_color(3), sum dp, d_mean2d(2),
// d_conic(A, B, C)] (dp = d_alpha * alpha, so d_opac = sum dp / o,
// render.py:364-365).  Writes the per-splat pull-back record s.
#ifndef CGS_PULLBACK_SH_F32
#define CGS_PULLBACK_SH_F32 1
#endif
template <int DEG>
__device__ void pull_back_splat(const double* acc, int64_t s, uint32_t gi, const CamDev& cam,
                                const GaussIn& g, const BwdLayout& B) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  constexpr int D = 3 * NB;
  const double px = g.pos[3 * gi + 0], py = g.pos[3 * gi + 1], pz = g.pos[3 * gi + 2];
  // colour path first (render.py:415-429), so its registers are free before
  // the geometric chain.
  // quotients by one divisor multiply by its reciprocal (ulp-level, as the
  // projection)
  double ox = px - cam.center[0], oy = py - cam.center[1], oz = pz - cam.center[2];
  const double len = sqrt((ox * ox + oy * oy) + oz * oz);
  const double rlen = 1.0 / len;
  ox *= rlen;
  oy *= rlen;
  oz *= rlen;
  const SplatRec& rec = g.recs[s];
  // colour gate raw > 0 (render.py:418-419): the projection stored
  // max(raw, 0) in fp32, which is > 0 exactly when raw > 0 (fp64 decision)
  const double draw[3] = {rec.r > 0.0f ? acc[0] : 0.0, rec.g > 0.0f ? acc[1] : 0.0,
                          rec.b > 0.0f ? acc[2] : 0.0};
  double dpc[3] = {0.0, 0.0, 0.0};
  if constexpr (DEG >= 1) {
    const float* row = g.sh_rows + static_cast<int64_t>(g.g2sh[gi]) * D;
#if CGS_PULLBACK_SH_F32
    // view-direction term in fp32 (it enters d_pos additively and the result
    // is stored in fp32): half the registers of the fp64 form
    const float d0 = static_cast<float>(draw[0]), d1 = static_cast<float>(draw[1]),
                d2 = static_cast<float>(draw[2]);
    float wb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b)
      wb[b] = fmaf(d2, __ldg(row + 3 * b + 2), fmaf(d1, __ldg(row + 3 * b + 1),
                                                     d0 * __ldg(row + 3 * b + 0)));
    const float fx = static_cast<float>(ox), fy = static_cast<float>(oy),
                fz = static_cast<float>(oz);
    float dv[3];
    sh_basis_grad_dot<DEG, float>(fx, fy, fz, wb, dv);
    const float vd = fx * dv[0] + fy * dv[1] + fz * dv[2];
    const float il = static_cast<float>(rlen);
    dpc[0] = (dv[0] - fx * vd) * il;
    dpc[1] = (dv[1] - fy * vd) * il;
    dpc[2] = (dv[2] - fz * vd) * il;
#else
    double wb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b)
      wb[b] = draw[0] * static_cast<double>(__ldg(row + 3 * b + 0)) +
              draw[1] * static_cast<double>(__ldg(row + 3 * b + 1)) +
              draw[2] * static_cast<double>(__ldg(row + 3 * b + 2));
    double dv[3];
    sh_basis_grad_dot<DEG>(ox, oy, oz, wb, dv);
    const double vd = ox * dv[0] + oy * dv[1] + oz * dv[2];
    dpc[0] = (dv[0] - ox * vd) / len;
    dpc[1] = (dv[1] - oy * vd) / len;
    dpc[2] = (dv[2] - oz * vd) / len;
#endif
  }
  const double tx = cam.R[0] * px + cam.R[1] * py + cam.R[2] * pz + cam.t[0];
  const double ty = cam.R[3] * px + cam.R[4] * py + cam.R[5] * pz + cam.t[1];
  const double tz = cam.R[6] * px + cam.R[7] * py + cam.R[8] * pz + cam.t[2];
  const double fx = cam.fx, fy = cam.fy;
  const double rz = 1.0 / tz, rz2 = rz * rz, rz3 = rz2 * rz;
  const double j00 = fx * rz, j02 = -fx * tx * rz2;
  const double j11 = fy * rz, j12 = -fy * ty * rz2;
  double M[2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    M[0][k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
    M[1][k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
  }
  const double* cv = g.sr_cov + static_cast<int64_t>(g.g2sr[gi]) * 8;
  const double S[3][3] = {{cv[0], cv[1], cv[2]}, {cv[1], cv[3], cv[4]}, {cv[2], cv[4], cv[5]}};
  // the forward's conic (render.py:176-181; the reference's pull-back reuses
  // _Projection's conic the same way)
  const double Q[2][2] = {{rec.ca, rec.cb}, {rec.cb, rec.cc}};
  // dConic (render.py:391-394) and dSigma2 = -Q dQ Q (render.py:396-397)
  const double dQ[2][2] = {{acc[6], 0.5 * acc[7]}, {0.5 * acc[7], acc[8]}};
  double QdQ[2][2], dS2[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) QdQ[a][b] = Q[a][0] * dQ[0][b] + Q[a][1] * dQ[1][b];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) dS2[a][b] = -(QdQ[a][0] * Q[0][b] + QdQ[a][1] * Q[1][b]);
  // dSigma3 = M^T dS2 M, dM = 2 dS2 M Sigma3 (render.py:400-401)
  double dS2M[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) dS2M[a][k] = dS2[a][0] * M[0][k] + dS2[a][1] * M[1][k];
  double dS3[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) dS3[a][k] = M[0][a] * dS2M[0][k] + M[1][a] * dS2M[1][k];
  double dM[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dM[a][k] = 2.0 * (dS2M[a][0] * S[0][k] + dS2M[a][1] * S[1][k] + dS2M[a][2] * S[2][k]);
  // dJ = dM R^T (render.py:402)
  double dJ[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      dJ[a][c] = dM[a][0] * cam.R[c * 3 + 0] + dM[a][1] * cam.R[c * 3 + 1] + dM[a][2] * cam.R[c * 3 + 2];
  // d_t (render.py:404-412) and d_pos = d_t R (render.py:413)
  const double dmx = acc[4], dmy = acc[5];
  double dt[3];
  dt[0] = dmx * fx * rz + dJ[0][2] * (-fx * rz2);
  dt[1] = dmy * fy * rz + dJ[1][2] * (-fy * rz2);
  dt[2] = dmx * (-fx * tx * rz2) + dmy * (-fy * ty * rz2) + dJ[0][0] * (-fx * rz2) +
          dJ[1][1] * (-fy * rz2) + dJ[0][2] * (2 * fx * tx * rz3) + dJ[1][2] * (2 * fy * ty * rz3);
  double dp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) dp[k] = dt[0] * cam.R[0 + k] + dt[1] * cam.R[3 + k] + dt[2] * cam.R[6 + k];
  if constexpr (DEG >= 1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) dp[k] += dpc[k];
  }
  const double o = 1.0 / (1.0 + exp(-static_cast<double>(g.logit[gi])));
  const double dlogit = (acc[3] / o) * o * (1.0 - o);  // render.py:364-365, 446
  B.s_posl[s] = make_float4(static_cast<float>(dp[0]), static_cast<float>(dp[1]),
                            static_cast<float>(dp[2]), static_cast<float>(dlogit));
  B.s_view[s] = make_float4(static_cast<float>(ox), static_cast<float>(oy), static_cast<float>(oz), 0.0f);
  B.s_draw[s] = make_float4(static_cast<float>(draw[0]), static_cast<float>(draw[1]),
                            static_cast<float>(draw[2]), 0.0f);
  B.s_s3a[s] = make_float4(static_cast<float>(dS3[0][0]), static_cast<float>(0.5 * (dS3[0][1] + dS3[1][0])),
                           static_cast<float>(0.5 * (dS3[0][2] + dS3[2][0])), static_cast<float>(dS3[1][1]));
  B.s_s3b[s] = make_float2(static_cast<float>(0.5 * (dS3[1][2] + dS3[2][1])), static_cast<float>(dS3[2][2]));
}

struct PairWalk {
  const SplatRec* recs;  // mean2d of each splat (tile moments -> splat centre)
  const uint64_t* pair_off;
  const uint32_t* n_tiles;
  const uint64_t* rect;
  const uint64_t* depth_key;
  const uint64_t* tile_last_dk;
  const uint32_t* tile_last_sid;
  const unsigned long long* view_last_dk;
  const float* partials;  // by emission index: [pair_cap x 8 | pair_cap]
  int64_t p9;             // offset of value 8 (8 * pair_cap)
};

// Adds the tile sums of splat s's processed pairs k = k0, k0+kstep, ... (in
// emission order) into acc; returns whether any pair was processed.  A tile
// sum holds [d_color(3), m0, m1x, m1y, m2xx, m2xy, m2yy]: moments of
// dp = d_alpha * alpha over the tile's pixels in coordinates (lx, ly)
// centred on the tile (raster_bwd_kernel).  They are shifted here, in
// float64, to the splat centre: with o = tile centre - mean2d and
// d = o + (lx, ly), acc = [d_color(3), sum dp, sum dp dx, sum dp dy,
// sum dp dx^2, sum dp dx dy, sum dp dy^2] (render.py:364-377).
__device__ __forceinline__ bool walk_pairs(const PairWalk& w, const FrameDesc& fd, int64_t n,
                                           int64_t s, uint32_t cnt, uint32_t k0, uint32_t kstep,
                                           double* acc) {
  const uint64_t o = w.pair_off[s];
  const uint64_t rc = w.rect[s];
  const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
  const int ty0 = static_cast<int>((rc >> 32) & 0xffff);
  const int span = tx1 - tx0 + 1;
  // splat ids are 32-bit: 32-bit division for the view
  const int v = fd.n_views == 1 ? 0 : static_cast<int>(static_cast<uint32_t>(s) / static_cast<uint32_t>(n));
  const int tb = fd.cam[v].tile_base, ntx = fd.cam[v].ntx;
  const uint64_t dk = w.depth_key[s];
  if (dk > w.view_last_dk[v]) return false;  // behind every tile's processed prefix
  const double mx = w.recs[s].mx, my = w.recs[s].my;
  bool any = false;
  // tile (tx, ty) of pair k: stepped incrementally for kstep = 1
  int ty = ty0 + static_cast<int>(k0) / span, tx = tx0 + static_cast<int>(k0) % span;
  for (uint32_t k = k0; k < cnt; k += kstep) {
    if (kstep != 1) {
      ty = ty0 + static_cast<int>(k) / span;
      tx = tx0 + static_cast<int>(k) % span;
    }
    const int t = tb + ty * ntx + tx;
    const uint64_t tk = w.tile_last_dk[t];
    if (dk < tk || (dk == tk && static_cast<uint32_t>(s) <= w.tile_last_sid[t])) {  // in the processed prefix
      any = true;
      const int64_t e = static_cast<int64_t>(o + k);
      const float4* p4 = reinterpret_cast<const float4*>(w.partials) + 2 * e;
      const float4 x = p4[0], y = p4[1];
      const double m0 = x.w, m1x = y.x, m1y = y.y;
      const double ox = tile_centre(tx) - mx, oy = tile_centre(ty) - my;  // tile centre offset
      acc[0] += x.x; acc[1] += x.y; acc[2] += x.z; acc[3] += m0;
      acc[4] += ox * m0 + m1x;
      acc[5] += oy * m0 + m1y;
      acc[6] += (ox * ox * m0 + 2.0 * ox * m1x) + static_cast<double>(y.z);
      acc[7] += (ox * oy * m0 + (ox * m1y + oy * m1x)) + static_cast<double>(y.w);
      acc[8] += (oy * oy * m0 + 2.0 * oy * m1y) + static_cast<double>(w.partials[w.p9 + e]);
    }
    if (kstep == 1 && ++tx > tx1) {
      tx = tx0;
      ++ty;
    }
  }
  return any;
}

// Summed moments -> the per-splat record the pull-back reads.
__device__ __forceinline__ void store_splat_acc(const BwdLayout& B, int64_t s, const double* t) {
  B.acc0[s] = make_float4(static_cast<float>(t[0]), static_cast<float>(t[1]),
                          static_cast<float>(t[2]), static_cast<float>(t[3]));
  B.accm[s] = make_double2(t[4], t[5]);
  B.accq[s] = make_double2(t[6], t[7]);
  B.accr[s] = t[8];
}

// One thread per splat; splats with more than 32 pairs (e.g. near-plane
// splats processed in every tile) are walked by the whole warp.  The sum
// order is fixed, so the result is deterministic.
template <int DEG>
#ifndef CGS_SR_MINB
#define CGS_SR_MINB 3
#endif
__global__ void __launch_bounds__(256, CGS_SR_MINB) splat_reduce_kernel(PairWalk pw, const FrameHeader* __restrict__ fh,
                                                           FrameDesc fd, int64_t n, int64_t vn,
                                                           GaussIn g, BwdLayout B) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (fh->stats.overflow) {  // touched is written here for every splat (no memset before)
    for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < vn; s += stride)
      B.touched[s] = 0;
    return;
  }
  for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x); base < vn; base += stride) {
    const int64_t s = base + threadIdx.x;
    const bool ok = s < vn;
    const uint32_t cnt = ok ? pw.n_tiles[s] : 0u;
    double acc[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) acc[u] = 0.0;
    bool touched = false;
    const bool huge = cnt > kLongSplat;  // splat_reduce_long_kernel's (one CTA each)
    const bool lng = cnt > 32 && !huge;
    if (cnt > 0 && !lng && !huge) touched = walk_pairs(pw, fd, n, s, cnt, 0, 1, acc);
    unsigned mask = __ballot_sync(kFull, lng);
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const int64_t sl = __shfl_sync(kFull, s, l);
      const uint32_t cl = __shfl_sync(kFull, cnt, l);
      double loc[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) loc[u] = 0.0;
      const bool any = walk_pairs(pw, fd, n, sl, cl, lane, 32, loc);
      const bool wany = __any_sync(kFull, any);
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const double t = warp_sum(loc[u]);
        if (lane == l) acc[u] = t;
      }
      if (lane == l) touched = wany;
    }
    const unsigned tm = __ballot_sync(kFull, ok && touched);
    if (lane == 0 && tm) atomicAdd(&B.hdr->n_touched, static_cast<unsigned long long>(__popc(tm)));
    if (!ok) continue;
    B.touched[s] = touched ? 1 : 0;  // huge: 0 here, splat_reduce_long_kernel (next) sets 1
    if (huge) continue;
    if (!touched) continue;
    store_splat_acc(B, s, acc);
  }
}

// Splats with more than kLongSplat pairs (listed during emission): one CTA
// each walks the pairs with a 256 stride, then a fixed-order block reduction.
__global__ void __launch_bounds__(256) splat_reduce_long_kernel(PairWalk pw,
                                                                const FrameHeader* __restrict__ fh,
                                                                const uint32_t* __restrict__ list,
                                                                FrameDesc fd, int64_t n,
                                                                BwdLayout B) {
  __shared__ double s_w[8][9];
  if (fh->stats.overflow) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nl = static_cast<int64_t>(fh->scratch[2]);
  for (int64_t e = blockIdx.x; e < nl; e += gridDim.x) {
    const uint32_t s = list[e];
    double acc[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) acc[u] = 0.0;
    const bool any = walk_pairs(pw, fd, n, s, pw.n_tiles[s], tid, 256, acc);
#pragma unroll
    for (int u = 0; u < 9; ++u) acc[u] = warp_sum(acc[u]);
    if (lane == 0)
#pragma unroll
      for (int u = 0; u < 9; ++u) s_w[warp][u] = acc[u];
    const bool touched = __syncthreads_or(any);
    if (tid == 0 && touched) {
      double t[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        t[u] = s_w[0][u];
        for (int w = 1; w < 8; ++w) t[u] += s_w[w][u];
      }
      B.touched[s] = 1;
      store_splat_acc(B, s, t);
      atomicAdd(&B.hdr->n_touched, 1ULL);
    }
    __syncthreads();
  }
}

// Chain rule per touched splat (kept apart from the gather walk so the
// latency-bound walk runs at full occupancy).
template <int DEG>
#ifndef CGS_PULLBACK_VIEW_INNER
#define CGS_PULLBACK_VIEW_INNER 1
#endif
#ifndef CGS_PB_MINB
#define CGS_PB_MINB 4
#endif
__global__ void __launch_bounds__(128, CGS_PB_MINB) pull_back_kernel(const FrameHeader* __restrict__ fh,
                                                        FrameDesc fd, int64_t n, int64_t vn,
                                                        GaussIn g, BwdLayout B) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the backward's counters are final here (cgs_frame_stats)
    FrameHeader* h = const_cast<FrameHeader*>(fh);
    h->stats.n_processed = static_cast<int64_t>(B.hdr->n_processed);
    h->stats.n_touched = static_cast<int64_t>(B.hdr->n_touched);
  }
  if (fh->stats.overflow) return;
  const bool sparse = code_sparse(B, vn);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < vn;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
#if CGS_PULLBACK_VIEW_INNER
    // consecutive threads take the views of one Gaussian (its gathers coalesce)
    const int64_t gi = fd.n_views == 1 ? t
                       : (vn < (int64_t{1} << 31) ? static_cast<int64_t>(static_cast<uint32_t>(t) /
                                                                         static_cast<uint32_t>(fd.n_views))
                                                  : t / fd.n_views);
    const int v = static_cast<int>(t - gi * fd.n_views);
    const int64_t s = static_cast<int64_t>(v) * n + gi;
#else
    const int64_t s = t;
    const int v = static_cast<int>(s / n);
    const int64_t gi = s - static_cast<int64_t>(v) * n;
#endif
    if (!B.touched[s]) continue;
    if (sparse) {  // the codebook reduces skip rows without a touched member
      B.code_hit[0][g.g2sh[gi]] = 1;
      B.code_hit[1][g.g2sr[gi]] = 1;
    }
    const float4 a0 = B.acc0[s];
    const double2 am = B.accm[s], aq = B.accq[s];
    const double ar = B.accr[s];
    // d_mean2d = Q sum dp d, d_conic = -(1/2 sum dp dx^2, sum dp dx dy,
    // 1/2 sum dp dy^2) (render.py:368-377), Q the forward's conic
    const SplatRec& rq = g.recs[s];
    const double acc[9] = {a0.x, a0.y, a0.z, a0.w,
                           rq.ca * am.x + rq.cb * am.y, rq.cb * am.x + rq.cc * am.y,
                           -0.5 * aq.x, -aq.y, -0.5 * ar};
    pull_back_splat<DEG>(acc, s, static_cast<uint32_t>(gi), fd.cam[v], g, B);
  }
}

// Per-Gaussian sums over views (render.py:454-455); writes every entry.
__global__ void __launch_bounds__(256) gauss_write_kernel(BwdLayout B, int64_t n, int n_views,
                                                          float scale, float* __restrict__ gpos,
                                                          float* __restrict__ glogit) {
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int v = 0; v < n_views; ++v) {
      const int64_t s = static_cast<int64_t>(v) * n + i;
      if (B.touched[s]) {
        const float4 e = B.s_posl[s];
        s0 += e.x; s1 += e.y; s2 += e.z; s3 += e.w;
      }
    }
    const float g0 = static_cast<float>(s0 * scale), g1 = static_cast<float>(s1 * scale),
                g2 = static_cast<float>(s2 * scale), g3 = static_cast<float>(s3 * scale);
    gpos[3 * i + 0] = g0;
    gpos[3 * i + 1] = g1;
    gpos[3 * i + 2] = g2;
    glogit[i] = g3;
    bad |= !isfinite(g0) || !isfinite(g1) || !isfinite(g2) || !isfinite(g3);
  }
  // the SGLD update's finiteness check (sampler.py:270-271), done here on
  // the values as they are written instead of by a second pass
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&B.hdr->nonfinite, 1);
}

// SH row gradient = sum over members of basis(view) (x) d_raw (render.py:421,
// 456).  One warp per SH row: lane t takes (member, view) items t, t + 32, ... and
// accumulates all D coefficient products in registers; the 32 lane partials
// then go through shared memory and each lane sums whole columns over the
// lanes in fixed order (deterministic; fp32 partials of a few items each).
template <int DEG>
__global__ void __launch_bounds__(128) sh_code_reduce_kernel(
    const int32_t* __restrict__ off, const int32_t* __restrict__ mem, int64_t cap, int64_t n,
    int n_views, BwdLayout B, float scale, float* __restrict__ gsh) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  constexpr int D = 3 * NB;
  __shared__ float s_part[4][32][D + 1];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool sparse = code_sparse(B, n * n_views);
  bool bad = false;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < cap;
       r += warps) {
    float* out = gsh + r * D;
    if (sparse && !B.code_hit[0][r]) {  // no touched member: the row's gradient is zero
      for (int c = lane; c < D; c += 32) out[c] = 0.0f;
      continue;
    }
    const int m0 = off[r], m1 = off[r + 1];
    const int items = (m1 - m0) * n_views;
    float acc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] = 0.0f;
    bool any = false;
    for (int t = lane; t < items; t += 32) {
      const int mi = n_views == 1 ? t : t / n_views, v = t - mi * n_views;
      const int64_t sp = static_cast<int64_t>(v) * n + mem[m0 + mi];
      if (!B.touched[sp]) continue;
      any = true;
      const float4 vd = B.s_view[sp];
      const float4 dr = B.s_draw[sp];
      float Bv[NB];
      sh_basis_f<DEG>(vd.x, vd.y, vd.z, Bv);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        acc[3 * b + 0] = fmaf(Bv[b], dr.x, acc[3 * b + 0]);
        acc[3 * b + 1] = fmaf(Bv[b], dr.y, acc[3 * b + 1]);
        acc[3 * b + 2] = fmaf(Bv[b], dr.z, acc[3 * b + 2]);
      }
    }
    if (!__any_sync(kFull, any)) {  // no member contributed: the row's gradient is zero
      for (int c = lane; c < D; c += 32) out[c] = 0.0f;
      continue;
    }
#pragma unroll
    for (int c = 0; c < D; ++c) s_part[wl][lane][c] = acc[c];
    __syncwarp();
    for (int c = lane; c < D; c += 32) {
      float sum = 0.0f;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) sum += s_part[wl][l][c];
      out[c] = sum * scale;
      bad |= !isfinite(sum * scale);
    }
    __syncwarp();
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&B.hdr->nonfinite, 1);
}

// SR row gradient: sum dSigma3 over members, then the per-row chain through
// Sigma3 = R diag(s^2) R^T, quaternion normalisation and exp
// (render.py:431-444).  One warp per row; writes every row.
__global__ void __launch_bounds__(256) sr_code_reduce_kernel(
    const int32_t* __restrict__ off, const int32_t* __restrict__ mem, int64_t cap, int64_t n,
    int n_views, BwdLayout B, const float* __restrict__ sr_rows, float scale,
    float* __restrict__ gsr) {
  const int lane = threadIdx.x & 31;
  const bool sparse = code_sparse(B, n * n_views);
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < cap;
       r += warps) {
    if (sparse && !B.code_hit[1][r]) {  // no touched member: the row's gradient is zero
      if (lane == 0)
        for (int k = 0; k < 7; ++k) gsr[r * 7 + k] = 0.0f;
      continue;
    }
    const int m0 = off[r], m1 = off[r + 1];
    double s[6] = {0, 0, 0, 0, 0, 0};
    bool any = false;
    for (int m = m0 + lane; m < m1; m += 32) {
      const int64_t i = mem[m];
      for (int v = 0; v < n_views; ++v) {
        const int64_t sp = static_cast<int64_t>(v) * n + i;
        if (!B.touched[sp]) continue;
        any = true;
        const float4 a = B.s_s3a[sp];
        const float2 b = B.s_s3b[sp];
        s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w; s[4] += b.x; s[5] += b.y;
      }
    }
#pragma unroll
    for (int u = 0; u < 6; ++u) s[u] = warp_sum(s[u]);
    any = __any_sync(kFull, any);
    if (lane != 0) continue;
    float* out = gsr + r * 7;
    if (!any) {
      for (int k = 0; k < 7; ++k) out[k] = 0.0f;
      continue;
    }
    const float* rr = sr_rows + r * 7;
    const double qr[4] = {rr[3], rr[4], rr[5], rr[6]};
    const double qn = sqrt(((qr[0] * qr[0] + qr[1] * qr[1]) + qr[2] * qr[2]) + qr[3] * qr[3]);
    const double w_ = qr[0] / qn, x = qr[1] / qn, y = qr[2] / qn, z = qr[3] / qn;
    double R[9];
    quat_to_rot(w_, x, y, z, R);
    const double s2[3] = {exp(2.0 * static_cast<double>(rr[0])), exp(2.0 * static_cast<double>(rr[1])),
                          exp(2.0 * static_cast<double>(rr[2]))};
    const double dS[3][3] = {{s[0], s[1], s[2]}, {s[1], s[3], s[4]}, {s[2], s[4], s[5]}};
    double dSR[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c)
        dSR[a][c] = dS[a][0] * R[0 * 3 + c] + dS[a][1] * R[1 * 3 + c] + dS[a][2] * R[2 * 3 + c];
    // d_ls_k = (R^T dS R)_kk * 2 s2_k (render.py:436-437)
    double dls[3];
    for (int k = 0; k < 3; ++k)
      dls[k] = (R[0 * 3 + k] * dSR[0][k] + R[1 * 3 + k] * dSR[1][k] + R[2 * 3 + k] * dSR[2][k]) * 2.0 * s2[k];
    // dR = 2 dS R diag(s2) (render.py:438); d qn_k = sum_ab dR_ab dR_ab/dq_k (render.py:61-82)
    double dR[9];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) dR[a * 3 + c] = 2.0 * dSR[a][c] * s2[c];
    const double P0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    const double P1[9] = {0, y, z, y, -2 * x, -w_, z, w_, -2 * x};
    const double P2[9] = {-2 * y, x, w_, x, 0, z, -w_, z, -2 * y};
    const double P3[9] = {-2 * z, -w_, x, w_, -2 * z, y, x, y, 0};
    double dq[4] = {0, 0, 0, 0};
    for (int e = 0; e < 9; ++e) {
      dq[0] += dR[e] * 2.0 * P0[e];
      dq[1] += dR[e] * 2.0 * P1[e];
      dq[2] += dR[e] * 2.0 * P2[e];
      dq[3] += dR[e] * 2.0 * P3[e];
    }
    // through normalisation (render.py:441-444)
    const double qd = w_ * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
    const double qv[4] = {w_, x, y, z};
    bool bad = false;
    for (int k = 0; k < 3; ++k) {
      out[k] = static_cast<float>(dls[k] * scale);
      bad |= !isfinite(out[k]);
    }
    for (int k = 0; k < 4; ++k) {
      out[3 + k] = static_cast<float>((dq[k] - qv[k] * qd) / qn * scale);
      bad |= !isfinite(out[3 + k]);
    }
    if (bad) atomicOr(&B.hdr->nonfinite, 1);
  }
}


// ---------------------------------------------------------------------------
// code -> members CSR: stable onesweep of (code, gaussian) pairs + offsets.
struct CsrLayout {
  uint32_t* keys;
  uint32_t* vals;
  SortWs<uint32_t> sort;
  uint32_t* counts;  // cap + 1
  ScanWs scan;
  size_t bytes;
};

static CsrLayout plan_csr(void* base, size_t cap_bytes, int64_t n, int64_t cap) {
  CsrLayout C{};
  Carver c(base, cap_bytes);
  const int64_t n1 = n > 0 ? n : 1;
  C.keys = c.take<uint32_t>(n1);
  C.vals = c.take<uint32_t>(n1);
  C.sort = carve_sort<uint32_t>(c, n1);
  C.counts = c.take<uint32_t>(cap + 1);
  C.scan = carve_scan(c, cap + 1);
  C.bytes = c.off + 256;
  return C;
}

size_t code_csr_ws_bytes(int64_t n, int64_t cap) { return plan_csr(nullptr, 0, n, cap).bytes; }

__global__ void csr_init_kernel(const int32_t* __restrict__ idx, int64_t n, int64_t cap,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                uint32_t* __restrict__ counts) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = idx[i];
    keys[i] = static_cast<uint32_t>(r);
    vals[i] = static_cast<uint32_t>(i);
    if (r >= 0 && r < cap) atomicAdd(&counts[r], 1u);  // integer counts: order-independent
  }
}

struct CsrOffsets {
  const uint32_t* counts;
  int32_t* off;
  __device__ uint64_t load(int64_t r) const { return counts[r]; }
  __device__ void store(int64_t r, uint64_t ex, uint64_t) const { off[r] = static_cast<int32_t>(ex); }
  __device__ void finish(uint64_t) const {}
};

int build_code_csr(const int32_t* idx, int64_t n, int64_t cap, int32_t* off, int32_t* mem,
                   void* ws, size_t ws_bytes, cudaStream_t st) {
  CsrLayout C = plan_csr(ws, ws_bytes, n, cap);
  if (C.bytes > ws_bytes || !ws) {
    set_error("code CSR workspace too small");
    return CGS_EWORKSPACE;
  }
  CGS_CUDA(cudaMemsetAsync(C.counts, 0, sizeof(uint32_t) * (cap + 1), st));
  if (n > 0) {
    csr_init_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(idx, n, cap, C.keys, C.vals, C.counts);
    CGS_CHECK_LAUNCH("csr_init_kernel");
    uint32_t *ko, *vo;
    int rc = launch_radix_sort<uint32_t>(C.keys, C.vals, nullptr, n, n, bits_for(cap + 1), C.sort,
                                         &ko, &vo, st);
    if (rc) return rc;
    CGS_CUDA(cudaMemcpyAsync(mem, vo, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  return launch_scan(CsrOffsets{C.counts, off}, nullptr, cap + 1, cap + 1, C.scan, nullptr, st);
}

// ---------------------------------------------------------------------------
template <int DEG>
static void launch_splat_reduce(const PairWalk& pw, const FrameLayout& L, const FrameDesc& fd,
                                const GaussIn& gi, const BwdLayout& B, cudaStream_t st) {
  CGS_PROFILED("splat_reduce_kernel", st,
               splat_reduce_kernel<DEG><<<grid_for(L.vn, 256, 8), 256, 0, st>>>(pw, L.hdr, fd, L.n,
                                                                                 L.vn, gi, B));
  note_launch();
  splat_reduce_long_kernel<<<148 * 4, 256, 0, st>>>(pw, L.hdr, L.long_list, fd, L.n, B);
  note_launch();
  CGS_PROFILED("pull_back_kernel", st,
               pull_back_kernel<DEG><<<grid_for(L.vn, 128, 8), 128, 0, st>>>(L.hdr, fd, L.n, L.vn,
                                                                              gi, B));
}

template <int DEG>
static void launch_sh_reduce(const int32_t* off, const int32_t* mem, int64_t cap, int64_t n,
                             int nv, const BwdLayout& B, float scale, float* gsh, cudaStream_t st) {
  CGS_PROFILED("sh_code_reduce_kernel", st,
               sh_code_reduce_kernel<DEG><<<grid_for(cap * 32, 128, 16), 128, 0, st>>>(
                   off, mem, cap, n, nv, B, scale, gsh));
}

// The frame backward in three stages (exported as cgs_raster_bwd,
// cgs_gaussian_reduce_pullback, cgs_codebook_reduce; each reads what the
// earlier stages left in the backward workspace).
int bwd_stage_raster(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                     BwdLayout& B, const float* dL, const float* final_T, cudaStream_t st) {
  // both codebooks' row flags, carved back to back (whole words: the
  // carver aligns every region)
  const size_t hit_bytes =
      align_up(static_cast<size_t>((B.code_hit[1] + (sc->sr_capacity > 0 ? sc->sr_capacity : 1)) - B.code_hit[0]), 4);
  if (fd.total_tiles > 0 && L.vn > 0)  // unit_order_kernel zeroes B.hdr and the row flags, splat_reduce writes every touched flag
    return launch_raster_bwd(fd, L, final_T, dL, B.partials, &B.hdr->n_processed,
                             sc->opacity_logits, st, B.hdr, sizeof(BwdHeader), B.code_hit[0], hit_bytes);
  CGS_CUDA(cudaMemsetAsync(B.code_hit[0], 0, hit_bytes, st));
  CGS_CUDA(cudaMemsetAsync(B.hdr, 0, sizeof(BwdHeader), st));
  if (L.vn > 0) CGS_CUDA(cudaMemsetAsync(B.touched, 0, L.vn, st));
  return CGS_OK;
}

static int launch_gauss_write(const cgs_scene_t* sc, const FrameDesc& fd, BwdLayout& B,
                              float scale, float* gpos, float* glogit, cudaStream_t st) {
  if (sc->n > 0) {
    CGS_PROFILED("gauss_write_kernel", st,
                 gauss_write_kernel<<<grid_for(sc->n, 256, 8), 256, 0, st>>>(B, sc->n, fd.n_views,
                                                                             scale, gpos, glogit));
    CGS_CHECK_LAUNCH("gauss_write_kernel");
  }
  return CGS_OK;
}

// write_gauss = false leaves the per-Gaussian gradient write to the codebook
// stage (frame_backward runs it there beside the codebook reduce).
int bwd_stage_pullback(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                       BwdLayout& B, float scale, float* gpos, float* glogit, cudaStream_t st,
                       bool write_gauss = true) {
  if (fd.total_tiles > 0 && L.vn > 0) {
    PairWalk pw{L.recs, L.pair_off, L.n_tiles, L.rect, L.depth_key, L.tile_last_dk, L.tile_last_sid, L.view_last_dk, B.partials,
                8 * (L.pair_cap > 0 ? L.pair_cap : 1)};
    GaussIn gi{L.recs, sc->positions, sc->opacity_logits, sc->g2sh, sc->g2sr, sc->sh_rows, L.sr_cov};
    switch (sc->sh_degree) {
      case 0: launch_splat_reduce<0>(pw, L, fd, gi, B, st); break;
      case 1: launch_splat_reduce<1>(pw, L, fd, gi, B, st); break;
      case 2: launch_splat_reduce<2>(pw, L, fd, gi, B, st); break;
      default: launch_splat_reduce<3>(pw, L, fd, gi, B, st); break;
    }
    CGS_CHECK_LAUNCH("splat_reduce_kernel");
  }
  return write_gauss ? launch_gauss_write(sc, fd, B, scale, gpos, glogit, st) : CGS_OK;
}

// The SH and SR codebook reduces (and, from frame_backward, the per-Gaussian
// gradient write) are independent: SR (after the gradient write) runs on a
// side stream beside SH.
int bwd_stage_codebook(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                       BwdLayout& B, float scale, float* gsh, float* gsr,
                       const int32_t* const csr_off_in[2], const int32_t* const csr_mem_in[2],
                       cudaStream_t st, float* gpos = nullptr, float* glogit = nullptr) {
  const int32_t* off[2];
  const int32_t* mem[2];
  const int32_t* idx[2] = {sc->g2sh, sc->g2sr};
  const int64_t caps[2] = {sc->sh_capacity, sc->sr_capacity};
  for (int b = 0; b < 2; ++b) {
    if (csr_off_in && csr_off_in[b] && csr_mem_in && csr_mem_in[b]) {
      off[b] = csr_off_in[b];
      mem[b] = csr_mem_in[b];
    } else {
      int rc = build_code_csr(idx[b], sc->n, caps[b], B.csr_off[b], B.csr_mem[b], B.csr_ws,
                              B.csr_ws_bytes, st);
      if (rc) return rc;
      off[b] = B.csr_off[b];
      mem[b] = B.csr_mem[b];
    }
  }
  SideFork fork(st);
  if (fork.rc) return fork.rc;
  if (gpos) {
    const int rc = launch_gauss_write(sc, fd, B, scale, gpos, glogit, fork.side);
    if (rc) return rc;
  }
  if (sc->sr_capacity > 0) {
    CGS_PROFILED("sr_code_reduce_kernel", fork.side,
                 sr_code_reduce_kernel<<<grid_for(sc->sr_capacity * 32, 256, 16), 256, 0, fork.side>>>(
                     off[1], mem[1], sc->sr_capacity, sc->n, fd.n_views, B, sc->sr_rows, scale, gsr));
    CGS_CHECK_LAUNCH("sr_code_reduce_kernel");
  }
  if (sc->sh_capacity > 0) {
    switch (sc->sh_degree) {
      case 0: launch_sh_reduce<0>(off[0], mem[0], sc->sh_capacity, sc->n, fd.n_views, B, scale, gsh, st); break;
      case 1: launch_sh_reduce<1>(off[0], mem[0], sc->sh_capacity, sc->n, fd.n_views, B, scale, gsh, st); break;
      case 2: launch_sh_reduce<2>(off[0], mem[0], sc->sh_capacity, sc->n, fd.n_views, B, scale, gsh, st); break;
      default: launch_sh_reduce<3>(off[0], mem[0], sc->sh_capacity, sc->n, fd.n_views, B, scale, gsh, st); break;
    }
    CGS_CHECK_LAUNCH("sh_code_reduce_kernel");
  }
  if (int rc = fork.join()) return rc;
  return CGS_OK;
}

int frame_backward(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L, BwdLayout& B,
                   const float* dL, const float* final_T, float scale, float* gpos, float* glogit,
                   float* gsh, float* gsr, const int32_t* const csr_off_in[2],
                   const int32_t* const csr_mem_in[2], cudaStream_t st) {
  int rc = bwd_stage_raster(sc, fd, L, B, dL, final_T, st);
  if (!rc) rc = bwd_stage_pullback(sc, fd, L, B, scale, gpos, glogit, st, false);
  if (!rc) rc = bwd_stage_codebook(sc, fd, L, B, scale, gsh, gsr, csr_off_in, csr_mem_in, st, gpos,
                                   glogit);
  return rc;
}

size_t bwd_ws_bytes(int64_t n, int n_views, int total_tiles, int64_t pair_cap, int64_t sh_cap,
                    int64_t sr_cap) {
  return plan_bwd(nullptr, 0, n, n_views, total_tiles, pair_cap, sh_cap, sr_cap).bytes;
}

int plan_bwd_checked(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L, void* ws,
                     size_t ws_bytes, BwdLayout* out) {
  *out = plan_bwd(ws, ws_bytes, sc->n, fd.n_views, fd.total_tiles, L.pair_cap, sc->sh_capacity,
                  sc->sr_capacity);
  if (out->bytes > ws_bytes || !ws) {
    set_error("backward workspace too small: need " + std::to_string(out->bytes));
    return CGS_EWORKSPACE;
  }
  return CGS_OK;
}

// One backward stage (0 raster, 1 per-Gaussian reduce + pull-back,
// 2 codebook reduce) on caller workspaces (the staged C ABI).
int bwd_stage_entry(int stage, const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                    void* ws, size_t ws_bytes, const float* dL, const float* final_T, float scale,
                    float* gpos, float* glogit, float* gsh, float* gsr,
                    const int32_t* const csr_off[2], const int32_t* const csr_mem[2],
                    cudaStream_t st) {
  BwdLayout B;
  int rc = plan_bwd_checked(sc, fd, L, ws, ws_bytes, &B);
  if (rc) return rc;
  switch (stage) {
    case 0: return bwd_stage_raster(sc, fd, L, B, dL, final_T, st);
    case 1: return bwd_stage_pullback(sc, fd, L, B, scale, gpos, glogit, st);
    default: return bwd_stage_codebook(sc, fd, L, B, scale, gsh, gsr, csr_off, csr_mem, st);
  }
}

int frame_backward_entry(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                         void* ws, size_t ws_bytes, const float* dL, const float* final_T,
                         float scale, float* gpos, float* glogit, float* gsh, float* gsr,
                         const int32_t* const csr_off[2], const int32_t* const csr_mem[2],
                         cudaStream_t st) {
  BwdLayout B = plan_bwd(ws, ws_bytes, sc->n, fd.n_views, fd.total_tiles, L.pair_cap,
                         sc->sh_capacity, sc->sr_capacity);
  if (B.bytes > ws_bytes || !ws) {
    set_error("backward workspace too small: need " + std::to_string(B.bytes));
    return CGS_EWORKSPACE;
  }
  return frame_backward(sc, fd, L, B, dL, final_T, scale, gpos, glogit, gsh, gsr, csr_off, csr_mem, st);
}

}  // namespace cgs
