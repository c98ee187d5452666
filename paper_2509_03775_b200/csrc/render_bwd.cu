// Backward render path (reference render.py:318-459) for sm_100a.
//
//   proc scan        offsets of each tile's processed prefix (P_x pairs)
//   raster_bwd       one CTA per tile, reverse traversal from each pixel's last
//                    processed splat; per splat the 256 pixel contributions are
//                    reduced in fixed order (warp shuffles, then 8 warps in
//                    smem) into one 9-float partial per processed pair
//                    (render.py:343-377)
//   pair sort        stable onesweep of processed pairs by (gaussian, view)
//   gauss_reduce     fixed-order segmented sum per (gaussian, view) and the fp64
//                    chain rule to model space (render.py:382-446)
//   code reduces     stable sort of pull-back entries by SH / SR row and a
//                    segmented reduction per row (render.py:456-458), no atomics
#include <cmath>

#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

struct BwdHeader {
  unsigned long long n_processed;
  unsigned long long n_runs;      // (gaussian, view) entries
  unsigned long long n_sh_runs;
  unsigned long long n_sr_runs;
  unsigned long long scratch[4];
};

struct BwdLayout {
  BwdHeader* hdr;
  unsigned long long* proc_off;  // total_tiles
  float* partials;               // pair_cap * 9
  uint32_t* pkeys;               // pair_cap
  uint32_t* pvals;
  SortWs<uint32_t> psort;
  uint32_t* run_start;           // pair_cap + 1
  uint32_t* e_gauss;             // entries (<= min(pair_cap, V*N))
  float4* e_posl;                // d_pos xyz, d_logit
  float4* e_view;                // view direction
  float4* e_draw;                // gated d colour
  float4* e_s3a;                 // dSigma3 00 01 02 11
  float2* e_s3b;                 // dSigma3 12 22
  uint32_t* ckeys;               // entry code keys
  uint32_t* cvals;
  SortWs<uint32_t> csort;
  uint32_t* crun;                // entries + 1
  ScanWs scan;
  size_t bytes;
  int64_t ecap;
};

inline BwdLayout plan_bwd(void* base, size_t cap, int64_t n, int n_views, int total_tiles,
                          int64_t pair_cap) {
  BwdLayout B{};
  Carver c(base, cap);
  const int64_t pc = pair_cap > 0 ? pair_cap : 1;
  int64_t ecap = n * n_views;
  if (ecap > pc) ecap = pc;
  if (ecap < 1) ecap = 1;
  B.ecap = ecap;
  B.hdr = c.take<BwdHeader>(1);
  B.proc_off = c.take<unsigned long long>(total_tiles > 0 ? total_tiles : 1);
  B.partials = c.take<float>(pc * 9);
  B.pkeys = c.take<uint32_t>(pc);
  B.pvals = c.take<uint32_t>(pc);
  B.psort = carve_sort<uint32_t>(c, pc);
  B.run_start = c.take<uint32_t>(pc + 1);
  B.e_gauss = c.take<uint32_t>(ecap);
  B.e_posl = c.take<float4>(ecap);
  B.e_view = c.take<float4>(ecap);
  B.e_draw = c.take<float4>(ecap);
  B.e_s3a = c.take<float4>(ecap);
  B.e_s3b = c.take<float2>(ecap);
  B.ckeys = c.take<uint32_t>(ecap);
  B.cvals = c.take<uint32_t>(ecap);
  B.csort = carve_sort<uint32_t>(c, ecap);
  B.crun = c.take<uint32_t>(ecap + 1);
  B.scan = carve_scan(c, pc > total_tiles ? pc : total_tiles);
  B.bytes = c.off + 256;
  return B;
}

// ---------------------------------------------------------------------------
struct TileProcScan {
  const uint32_t* nproc;
  unsigned long long* off;
  __device__ uint64_t load(int64_t t) const { return nproc[t]; }
  __device__ void store(int64_t t, uint64_t ex, uint64_t) const { off[t] = ex; }
};

// Reverse traversal (render.py:343-377).  For pixel p and splat k < last_p,
// T is the transmittance after k, T_before = T / (1 - alpha_k) and the
// running suffix holds sum_{j>k} alpha_j T_j c_j.  Alpha is recomputed with
// exactly the forward's fp32 code, so skip/clamp/termination decisions match.
__global__ void __launch_bounds__(256) raster_bwd_kernel(
    FrameDesc fd, const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_vals,
    const SplatRec* __restrict__ recs, const FrameHeader* __restrict__ fh,
    const uint32_t* __restrict__ px_last, const uint32_t* __restrict__ tile_nproc,
    const float* __restrict__ final_T, const float* __restrict__ dL,
    const unsigned long long* __restrict__ proc_off, int n_views, int64_t n,
    float* __restrict__ partials, uint32_t* __restrict__ pkeys, uint32_t* __restrict__ pvals) {
  __shared__ float4 s_a[256];
  __shared__ float4 s_b[256];
  __shared__ float4 s_n[256];  // natural conic A, B, C and blue
  __shared__ float s_io[256];  // 1 / opacity
  __shared__ float s_red[8][32][9];
  if (fh->stats.overflow) return;
  const int tile = blockIdx.x;
  const int nproc = static_cast<int>(tile_nproc[tile]);
  if (nproc == 0) return;
  int v = 0;
  while (v + 1 < fd.n_views && fd.cam[v + 1].tile_base <= tile) ++v;
  const CamDev& cam = fd.cam[v];
  const int lt = tile - cam.tile_base;
  const int ty = lt / cam.ntx, tx = lt - ty * cam.ntx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lx = tid & 15, ly = tid >> 4;
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < cam.width && py < cam.height;
  const uint2 rg = ranges[tile];
  const unsigned long long qbase = proc_off[tile];
  const double ox = static_cast<double>(tx * kTile), oy = static_cast<double>(ty * kTile);
  const float flx = static_cast<float>(lx), fly = static_cast<float>(ly);

  float T = 1.0f, gr = 0.0f, gg = 0.0f, gb = 0.0f;
  uint32_t last = 0;
  if (inside) {
    const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
    T = final_T[pix];
    last = px_last[pix];
    gr = dL[3 * pix + 0];
    gg = dL[3 * pix + 1];
    gb = dL[3 * pix + 2];
  }
  float sr = 0.0f, sg = 0.0f, sb = 0.0f;  // suffix sums

  for (int b0 = ((nproc - 1) / 256) * 256; b0 >= 0; b0 -= 256) {
    const int nb = min(256, nproc - b0);
    __syncthreads();
    if (tid < nb) {
      const uint32_t sid = pair_vals[rg.x + b0 + tid];
      const SplatRec r = recs[sid];
      float4 a, b;
      float c;
      stage_splat(r, ox, oy, a, b, c);
      s_a[tid] = a;
      s_b[tid] = b;
      s_n[tid] = make_float4(static_cast<float>(r.ca), static_cast<float>(r.cb),
                             static_cast<float>(r.cc), c);
      s_io[tid] = static_cast<float>(1.0 / r.opac);
      const unsigned long long q = qbase + b0 + tid;
      const uint32_t vv = sid / static_cast<uint32_t>(n);
      const uint32_t gi = sid - vv * static_cast<uint32_t>(n);
      pkeys[q] = gi * static_cast<uint32_t>(n_views) + vv;  // gaussian-major key
      pvals[q] = static_cast<uint32_t>(q);
    }
    __syncthreads();
    for (int se = nb; se > 0; se -= 32) {
      const int ss = se > 32 ? se - 32 : 0;
      for (int j = se - 1; j >= ss; --j) {
        const int k = b0 + j;
        float o[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) o[u] = 0.0f;
        bool any = false;
        if (static_cast<uint32_t>(k) < last) {
          const float4 a = s_a[j];
          const float4 b = s_b[j];
          const float dx = a.x + flx, dy = a.y + fly;
          const float al = splat_alpha(a, b, dx, dy);
          if (al >= kAlphaSkipF) {
            const float4 nc = s_n[j];
            const float iom = __frcp_rn(1.0f - al);
            const float Tb = T * iom;
            const float w = al * Tb;
            o[0] = w * gr;
            o[1] = w * gg;
            o[2] = w * gb;
            const float dCr = fmaf(b.z, Tb, -sr * iom);
            const float dCg = fmaf(b.w, Tb, -sg * iom);
            const float dCb = fmaf(nc.w, Tb, -sb * iom);
            const float da = dCr * gr + dCg * gg + dCb * gb;
            sr = fmaf(w, b.z, sr);
            sg = fmaf(w, b.w, sg);
            sb = fmaf(w, nc.w, sb);
            T = Tb;
            if (al < kAlphaClampVal) {
              const float dp = da * al;
              o[3] = dp * s_io[j];
              o[4] = dp * fmaf(nc.x, dx, nc.y * dy);
              o[5] = dp * fmaf(nc.y, dx, nc.z * dy);
              o[6] = dp * (-0.5f * dx * dx);
              o[7] = dp * (-dx * dy);
              o[8] = dp * (-0.5f * dy * dy);
            }
            any = true;
          }
        }
        // 12-shuffle transposed reduction; lanes 0,2,4,8,10,16,18,20,24 end
        // up holding the warp sums of values 0..8 and store them in one STS.
        float red = 0.0f;
        if (__any_sync(kFull, any)) red = warp_reduce9(o);
        const int slot = reduce9_slot(lane);
        if (slot >= 0) s_red[warp][j - ss][slot] = red;
      }
      __syncthreads();
      const int cnt = (se - ss) * 9;
      for (int e = tid; e < cnt; e += 256) {
        const int jj = e / 9, u = e - jj * 9;
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < 8; ++w) acc += s_red[w][jj][u];
        partials[(qbase + b0 + ss + jj) * 9 + u] = acc;
      }
      __syncthreads();
    }
  }
}

struct RunStarts {
  const uint32_t* keys;
  uint32_t* starts;
  __device__ uint64_t load(int64_t i) const {
    return (i == 0 || keys[i] != keys[i - 1]) ? 1ULL : 0ULL;
  }
  __device__ void store(int64_t i, uint64_t ex, uint64_t v) const {
    if (v) starts[ex] = static_cast<uint32_t>(i);
  }
};

__global__ void run_sentinel_kernel(uint32_t* starts, const unsigned long long* n_runs,
                                    const unsigned long long* n_items) {
  starts[*n_runs] = static_cast<uint32_t>(*n_items);
}

// Publish the backward's counters in the frame header (cgs_frame_stats).
__global__ void bwd_stats_kernel(FrameHeader* fh, const BwdHeader* bh) {
  fh->stats.n_processed = static_cast<int64_t>(bh->n_processed);
  fh->stats.n_touched = static_cast<int64_t>(bh->n_runs);
}

struct GaussIn {
  const float* pos;
  const float* logit;
  const int32_t* g2sh;
  const int32_t* g2sr;
  const float* sh_rows;
  const double* sr_cov;
};

// Segmented sum of a (gaussian, view) run's partials + chain rule
// (render.py:382-446).  One thread per run; runs longer than 64 pairs (e.g. a
// near-plane splat processed in every tile) are summed by the whole warp.
template <int DEG>
__global__ void __launch_bounds__(256) gauss_reduce_kernel(
    const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ sq,
    const uint32_t* __restrict__ run_start, const BwdHeader* __restrict__ bh,
    const float* __restrict__ partials, int n_views, GaussIn g, FrameDesc fd, BwdLayout B) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  constexpr int D = 3 * NB;
  const int64_t nruns = static_cast<int64_t>(bh->n_runs);
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x); base < nruns; base += stride) {
    const int64_t r = base + threadIdx.x;
    const bool ok = r < nruns;
    uint32_t rs = 0, re = 0;
    if (ok) {
      rs = run_start[r];
      re = run_start[r + 1];
    }
    double acc[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) acc[u] = 0.0;
    const bool lng = ok && (re - rs) > 64;
    if (ok && !lng) {
      for (uint32_t p = rs; p < re; ++p) {
        const float* pp = partials + static_cast<int64_t>(sq[p]) * 9;
#pragma unroll
        for (int u = 0; u < 9; ++u) acc[u] += static_cast<double>(pp[u]);
      }
    }
    unsigned mask = __ballot_sync(kFull, lng);
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t a0 = __shfl_sync(kFull, rs, l), a1 = __shfl_sync(kFull, re, l);
      double loc[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) loc[u] = 0.0;
      for (uint32_t p = a0 + lane; p < a1; p += 32) {
        const float* pp = partials + static_cast<int64_t>(sq[p]) * 9;
#pragma unroll
        for (int u = 0; u < 9; ++u) loc[u] += static_cast<double>(pp[u]);
      }
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const double t = warp_sum(loc[u]);
        if (lane == l) acc[u] = t;
      }
    }
    if (!ok) continue;
    const uint32_t key = skeys[rs];
    const uint32_t gi = key / static_cast<uint32_t>(n_views);
    const int v = static_cast<int>(key - gi * static_cast<uint32_t>(n_views));
    const CamDev& cam = fd.cam[v];
    const double px = g.pos[3 * gi + 0], py = g.pos[3 * gi + 1], pz = g.pos[3 * gi + 2];
    const double tx = cam.R[0] * px + cam.R[1] * py + cam.R[2] * pz + cam.t[0];
    const double ty = cam.R[3] * px + cam.R[4] * py + cam.R[5] * pz + cam.t[1];
    const double tz = cam.R[6] * px + cam.R[7] * py + cam.R[8] * pz + cam.t[2];
    const double fx = cam.fx, fy = cam.fy;
    const double j00 = fx / tz, j02 = -fx * tx / (tz * tz);
    const double j11 = fy / tz, j12 = -fy * ty / (tz * tz);
    double M[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      M[0][k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
      M[1][k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
    }
    const double* cv = g.sr_cov + static_cast<int64_t>(g.g2sr[gi]) * 8;
    const double S[3][3] = {{cv[0], cv[1], cv[2]}, {cv[1], cv[3], cv[4]}, {cv[2], cv[4], cv[5]}};
    double SM[3][2];  // S M^T
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) SM[a][b] = S[a][0] * M[b][0] + S[a][1] * M[b][1] + S[a][2] * M[b][2];
    const double c00 = M[0][0] * SM[0][0] + M[0][1] * SM[1][0] + M[0][2] * SM[2][0] + kBlur;
    const double c01 = M[0][0] * SM[0][1] + M[0][1] * SM[1][1] + M[0][2] * SM[2][1];
    const double c11 = M[1][0] * SM[0][1] + M[1][1] * SM[1][1] + M[1][2] * SM[2][1] + kBlur;
    const double det = c00 * c11 - c01 * c01;
    const double Q[2][2] = {{c11 / det, -c01 / det}, {-c01 / det, c00 / det}};
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
    const double z2 = tz * tz, z3 = z2 * tz;
    const double dmx = acc[4], dmy = acc[5];
    double dt[3];
    dt[0] = dmx * fx / tz + dJ[0][2] * (-fx / z2);
    dt[1] = dmy * fy / tz + dJ[1][2] * (-fy / z2);
    dt[2] = dmx * (-fx * tx / z2) + dmy * (-fy * ty / z2) + dJ[0][0] * (-fx / z2) +
            dJ[1][1] * (-fy / z2) + dJ[0][2] * (2 * fx * tx / z3) + dJ[1][2] * (2 * fy * ty / z3);
    double dp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) dp[k] = dt[0] * cam.R[0 + k] + dt[1] * cam.R[3 + k] + dt[2] * cam.R[6 + k];
    // colour path (render.py:415-429)
    double ox = px - cam.center[0], oy = py - cam.center[1], oz = pz - cam.center[2];
    const double len = sqrt((ox * ox + oy * oy) + oz * oz);
    ox /= len; oy /= len; oz /= len;
    double Bv[NB];
    sh_basis<DEG>(ox, oy, oz, Bv);
    const float* row = g.sh_rows + static_cast<int64_t>(g.g2sh[gi]) * D;
    double raw[3] = {0.5, 0.5, 0.5};
    double cf[D];
#pragma unroll
    for (int e = 0; e < D; ++e) {
      cf[e] = static_cast<double>(__ldg(row + e));
    }
    {
      double col[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int e = 0; e < D; ++e) col[e % 3] += Bv[e / 3] * cf[e];
      raw[0] += col[0]; raw[1] += col[1]; raw[2] += col[2];
    }
    const double draw[3] = {raw[0] > 0.0 ? acc[0] : 0.0, raw[1] > 0.0 ? acc[1] : 0.0,
                            raw[2] > 0.0 ? acc[2] : 0.0};
    if constexpr (DEG >= 1) {
      double wb[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b)
        wb[b] = draw[0] * cf[3 * b + 0] + draw[1] * cf[3 * b + 1] + draw[2] * cf[3 * b + 2];
      double dv[3];
      sh_basis_grad_dot<DEG>(ox, oy, oz, wb, dv);
      const double vd = ox * dv[0] + oy * dv[1] + oz * dv[2];
      dp[0] += (dv[0] - ox * vd) / len;
      dp[1] += (dv[1] - oy * vd) / len;
      dp[2] += (dv[2] - oz * vd) / len;
    }
    const double o = 1.0 / (1.0 + exp(-static_cast<double>(g.logit[gi])));
    const double dlogit = acc[3] * o * (1.0 - o);
    B.e_gauss[r] = gi;
    B.e_posl[r] = make_float4(static_cast<float>(dp[0]), static_cast<float>(dp[1]),
                              static_cast<float>(dp[2]), static_cast<float>(dlogit));
    B.e_view[r] = make_float4(static_cast<float>(ox), static_cast<float>(oy),
                              static_cast<float>(oz), 0.0f);
    B.e_draw[r] = make_float4(static_cast<float>(draw[0]), static_cast<float>(draw[1]),
                              static_cast<float>(draw[2]), 0.0f);
    B.e_s3a[r] = make_float4(static_cast<float>(dS3[0][0]), static_cast<float>(0.5 * (dS3[0][1] + dS3[1][0])),
                             static_cast<float>(0.5 * (dS3[0][2] + dS3[2][0])), static_cast<float>(dS3[1][1]));
    B.e_s3b[r] = make_float2(static_cast<float>(0.5 * (dS3[1][2] + dS3[2][1])), static_cast<float>(dS3[2][2]));
  }
}

// Per-Gaussian sums over its view entries (adjacent: keys are gaussian-major).
__global__ void __launch_bounds__(256) gauss_write_kernel(const BwdHeader* __restrict__ bh,
                                                          BwdLayout B, float scale,
                                                          float* __restrict__ gpos,
                                                          float* __restrict__ glogit) {
  const int64_t nr = static_cast<int64_t>(bh->n_runs);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < nr;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t gi = B.e_gauss[r];
    if (r > 0 && B.e_gauss[r - 1] == gi) continue;
    double s[4] = {0, 0, 0, 0};
    for (int64_t q = r; q < nr && B.e_gauss[q] == gi; ++q) {
      const float4 e = B.e_posl[q];
      s[0] += e.x; s[1] += e.y; s[2] += e.z; s[3] += e.w;
    }
    gpos[3 * static_cast<int64_t>(gi) + 0] = static_cast<float>(s[0] * scale);
    gpos[3 * static_cast<int64_t>(gi) + 1] = static_cast<float>(s[1] * scale);
    gpos[3 * static_cast<int64_t>(gi) + 2] = static_cast<float>(s[2] * scale);
    glogit[gi] = static_cast<float>(s[3] * scale);
  }
}

__global__ void __launch_bounds__(256) code_keys_kernel(const BwdHeader* __restrict__ bh,
                                                        const uint32_t* __restrict__ e_gauss,
                                                        const int32_t* __restrict__ g2x,
                                                        uint32_t* __restrict__ keys,
                                                        uint32_t* __restrict__ vals) {
  const int64_t nr = static_cast<int64_t>(bh->n_runs);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < nr;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    keys[r] = static_cast<uint32_t>(g2x[e_gauss[r]]);
    vals[r] = static_cast<uint32_t>(r);
  }
}

// SH row gradient = sum over members of basis(view) (x) d_raw (render.py:421,456).
// One warp per code row; lane owns columns lane and lane + 32.
template <int DEG>
__global__ void __launch_bounds__(256) sh_code_reduce_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ crun, const unsigned long long* __restrict__ n_code_runs,
    const float4* __restrict__ e_view, const float4* __restrict__ e_draw, float scale,
    float* __restrict__ gsh) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  constexpr int D = 3 * NB;
  const int lane = threadIdx.x & 31;
  const int64_t nrun = static_cast<int64_t>(*n_code_runs);
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int c0 = lane, c1 = lane + 32;
  const int b0 = c0 / 3, ch0 = c0 % 3, b1 = c1 / 3, ch1 = c1 % 3;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < nrun;
       w += warps) {
    const uint32_t rs = crun[w], re = crun[w + 1];
    const uint32_t row = keys[rs];
    double a0 = 0.0, a1 = 0.0;
    for (uint32_t m = rs; m < re; ++m) {
      const uint32_t e = vals[m];
      const float4 vd = e_view[e];
      const float4 dr = e_draw[e];
      double Bv[NB];
      sh_basis<DEG>(vd.x, vd.y, vd.z, Bv);
      double bv0 = 0.0, bv1 = 0.0;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (b == b0) bv0 = Bv[b];
        if (b == b1) bv1 = Bv[b];
      }
      const float d0 = ch0 == 0 ? dr.x : (ch0 == 1 ? dr.y : dr.z);
      const float d1 = ch1 == 0 ? dr.x : (ch1 == 1 ? dr.y : dr.z);
      a0 += bv0 * static_cast<double>(d0);
      a1 += bv1 * static_cast<double>(d1);
    }
    if (c0 < D) gsh[static_cast<int64_t>(row) * D + c0] = static_cast<float>(a0 * scale);
    if (c1 < D) gsh[static_cast<int64_t>(row) * D + c1] = static_cast<float>(a1 * scale);
  }
}

// SR row gradient: sum dSigma3 over members, then the per-row chain through
// Sigma3 = R diag(s^2) R^T, quaternion normalisation and exp (render.py:431-444).
__global__ void __launch_bounds__(256) sr_code_reduce_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ crun, const unsigned long long* __restrict__ n_code_runs,
    const float4* __restrict__ e_s3a, const float2* __restrict__ e_s3b,
    const float* __restrict__ sr_rows, float scale, float* __restrict__ gsr) {
  const int lane = threadIdx.x & 31;
  const int64_t nrun = static_cast<int64_t>(*n_code_runs);
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < nrun;
       w += warps) {
    const uint32_t rs = crun[w], re = crun[w + 1];
    double s[6] = {0, 0, 0, 0, 0, 0};
    for (uint32_t m = rs + lane; m < re; m += 32) {
      const uint32_t e = vals[m];
      const float4 a = e_s3a[e];
      const float2 b = e_s3b[e];
      s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w; s[4] += b.x; s[5] += b.y;
    }
#pragma unroll
    for (int u = 0; u < 6; ++u) s[u] = warp_sum(s[u]);
    if (lane != 0) continue;
    const uint32_t row = keys[rs];
    const float* rr = sr_rows + static_cast<int64_t>(row) * 7;
    const double qr[4] = {rr[3], rr[4], rr[5], rr[6]};
    const double qn = sqrt(((qr[0] * qr[0] + qr[1] * qr[1]) + qr[2] * qr[2]) + qr[3] * qr[3]);
    const double w_ = qr[0] / qn, x = qr[1] / qn, y = qr[2] / qn, z = qr[3] / qn;
    double R[9];
    quat_to_rot(w_, x, y, z, R);
    const double s2[3] = {exp(2.0 * static_cast<double>(rr[0])), exp(2.0 * static_cast<double>(rr[1])),
                          exp(2.0 * static_cast<double>(rr[2]))};
    const double dS[3][3] = {{s[0], s[1], s[2]}, {s[1], s[3], s[4]}, {s[2], s[4], s[5]}};
    // dS R
    double dSR[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c)
        dSR[a][c] = dS[a][0] * R[0 * 3 + c] + dS[a][1] * R[1 * 3 + c] + dS[a][2] * R[2 * 3 + c];
    // d_ls_k = (R^T dS R)_kk * 2 s2_k
    double dls[3];
    for (int k = 0; k < 3; ++k)
      dls[k] = (R[0 * 3 + k] * dSR[0][k] + R[1 * 3 + k] * dSR[1][k] + R[2 * 3 + k] * dSR[2][k]) * 2.0 * s2[k];
    // dR = 2 dS R diag(s2)
    double dR[9];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) dR[a * 3 + c] = 2.0 * dSR[a][c] * s2[c];
    // d qn_k = sum_ab dR_ab dR_ab/dq_k (render.py:61-82)
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
    const double qd = w_ * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
    const double qv[4] = {w_, x, y, z};
    float* out = gsr + static_cast<int64_t>(row) * 7;
    for (int k = 0; k < 3; ++k) out[k] = static_cast<float>(dls[k] * scale);
    for (int k = 0; k < 4; ++k) out[3 + k] = static_cast<float>((dq[k] - qv[k] * qd) / qn * scale);
  }
}

// ---------------------------------------------------------------------------
template <int DEG>
static void launch_gauss(const BwdLayout& B, const uint32_t* sk, const uint32_t* sv, int nv,
                         const GaussIn& gi, const FrameDesc& fd, cudaStream_t st) {
  CGS_PROFILED("gauss_reduce_kernel", st, gauss_reduce_kernel<DEG><<<148 * 4, 256, 0, st>>>(sk, sv, B.run_start, B.hdr, B.partials, nv, gi,
                                                    fd, B));
}

template <int DEG>
static void launch_sh_reduce(const BwdLayout& B, const uint32_t* k, const uint32_t* v, float scale,
                             float* gsh, cudaStream_t st) {
  CGS_PROFILED("sh_code_reduce_kernel", st, sh_code_reduce_kernel<DEG><<<148 * 8, 256, 0, st>>>(k, v, B.crun, &B.hdr->n_sh_runs, B.e_view,
                                                      B.e_draw, scale, gsh));
}

static int code_pass(BwdLayout& B, const int32_t* g2x, int64_t cap_rows,
                     unsigned long long* n_code_runs, uint32_t** ko, uint32_t** vo,
                     cudaStream_t st) {
  code_keys_kernel<<<grid_for(B.ecap, 256, 8), 256, 0, st>>>(B.hdr, B.e_gauss, g2x, B.ckeys, B.cvals);
  CGS_CHECK_LAUNCH("code_keys_kernel");
  int rc = launch_radix_sort<uint32_t>(B.ckeys, B.cvals, &B.hdr->n_runs, 0, B.ecap,
                                       bits_for(cap_rows + 1), B.csort, ko, vo, st);
  if (rc) return rc;
  rc = launch_scan(RunStarts{*ko, B.crun}, &B.hdr->n_runs, 0, B.ecap, B.scan, n_code_runs, st);
  if (rc) return rc;
  run_sentinel_kernel<<<1, 1, 0, st>>>(B.crun, n_code_runs, &B.hdr->n_runs);
  CGS_CHECK_LAUNCH("run_sentinel_kernel");
  return CGS_OK;
}

int frame_backward(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L, BwdLayout& B,
                   const float* dL, const float* final_T, float scale, float* gpos, float* glogit,
                   float* gsh, float* gsr, cudaStream_t st) {
  const int D = 3 * (sc->sh_degree + 1) * (sc->sh_degree + 1);
  CGS_CUDA(cudaMemsetAsync(B.hdr, 0, sizeof(BwdHeader), st));
  if (sc->n > 0) {
    CGS_CUDA(cudaMemsetAsync(gpos, 0, sizeof(float) * 3 * sc->n, st));
    CGS_CUDA(cudaMemsetAsync(glogit, 0, sizeof(float) * sc->n, st));
  }
  if (sc->sh_capacity > 0) CGS_CUDA(cudaMemsetAsync(gsh, 0, sizeof(float) * D * sc->sh_capacity, st));
  if (sc->sr_capacity > 0) CGS_CUDA(cudaMemsetAsync(gsr, 0, sizeof(float) * 7 * sc->sr_capacity, st));
  if (fd.total_tiles == 0 || L.vn == 0) return CGS_OK;
  int rc = launch_scan(TileProcScan{L.tile_nproc, B.proc_off}, nullptr, fd.total_tiles,
                       fd.total_tiles, B.scan, &B.hdr->n_processed, st);
  if (rc) return rc;
  CGS_PROFILED("raster_bwd_kernel", st, raster_bwd_kernel<<<fd.total_tiles, 256, 0, st>>>(fd, L.ranges, sorted_pair_vals(L), L.recs, L.hdr,
                                                    L.px_last, L.tile_nproc, final_T, dL, B.proc_off,
                                                    fd.n_views, L.n, B.partials, B.pkeys, B.pvals));
  CGS_CHECK_LAUNCH("raster_bwd_kernel");
  uint32_t *sk, *sv;
  rc = launch_radix_sort<uint32_t>(B.pkeys, B.pvals, &B.hdr->n_processed, 0, L.pair_cap,
                                   bits_for(L.vn + 1), B.psort, &sk, &sv, st);
  if (rc) return rc;
  rc = launch_scan(RunStarts{sk, B.run_start}, &B.hdr->n_processed, 0, L.pair_cap, B.scan,
                   &B.hdr->n_runs, st);
  if (rc) return rc;
  run_sentinel_kernel<<<1, 1, 0, st>>>(B.run_start, &B.hdr->n_runs, &B.hdr->n_processed);
  CGS_CHECK_LAUNCH("run_sentinel_kernel");
  GaussIn gi{sc->positions, sc->opacity_logits, sc->g2sh, sc->g2sr, sc->sh_rows, L.sr_cov};
  switch (sc->sh_degree) {
    case 0: launch_gauss<0>(B, sk, sv, fd.n_views, gi, fd, st); break;
    case 1: launch_gauss<1>(B, sk, sv, fd.n_views, gi, fd, st); break;
    case 2: launch_gauss<2>(B, sk, sv, fd.n_views, gi, fd, st); break;
    default: launch_gauss<3>(B, sk, sv, fd.n_views, gi, fd, st); break;
  }
  CGS_CHECK_LAUNCH("gauss_reduce_kernel");
  CGS_PROFILED("gauss_write_kernel", st, gauss_write_kernel<<<grid_for(B.ecap, 256, 8), 256, 0, st>>>(B.hdr, B, scale, gpos, glogit));
  CGS_CHECK_LAUNCH("gauss_write_kernel");
  // SH codebook rows
  uint32_t *ck, *cv;
  rc = code_pass(B, sc->g2sh, sc->sh_capacity, &B.hdr->n_sh_runs, &ck, &cv, st);
  if (rc) return rc;
  switch (sc->sh_degree) {
    case 0: launch_sh_reduce<0>(B, ck, cv, scale, gsh, st); break;
    case 1: launch_sh_reduce<1>(B, ck, cv, scale, gsh, st); break;
    case 2: launch_sh_reduce<2>(B, ck, cv, scale, gsh, st); break;
    default: launch_sh_reduce<3>(B, ck, cv, scale, gsh, st); break;
  }
  CGS_CHECK_LAUNCH("sh_code_reduce_kernel");
  // SR codebook rows
  rc = code_pass(B, sc->g2sr, sc->sr_capacity, &B.hdr->n_sr_runs, &ck, &cv, st);
  if (rc) return rc;
  CGS_PROFILED("sr_code_reduce_kernel", st, sr_code_reduce_kernel<<<148 * 8, 256, 0, st>>>(ck, cv, B.crun, &B.hdr->n_sr_runs, B.e_s3a, B.e_s3b,
                                                 sc->sr_rows, scale, gsr));
  CGS_CHECK_LAUNCH("sr_code_reduce_kernel");
  bwd_stats_kernel<<<1, 1, 0, st>>>(const_cast<FrameHeader*>(L.hdr), B.hdr);
  CGS_CHECK_LAUNCH("bwd_stats_kernel");
  return CGS_OK;
}

}  // namespace cgs

namespace cgs {

size_t bwd_ws_bytes(int64_t n, int n_views, int total_tiles, int64_t pair_cap) {
  return plan_bwd(nullptr, 0, n, n_views, total_tiles, pair_cap).bytes;
}

int frame_backward_entry(const cgs_scene_t* sc, const FrameDesc& fd, const FrameLayout& L,
                         void* ws, size_t ws_bytes, const float* dL, const float* final_T,
                         float scale, float* gpos, float* glogit, float* gsh, float* gsr,
                         cudaStream_t st) {
  BwdLayout B = plan_bwd(ws, ws_bytes, sc->n, fd.n_views, fd.total_tiles, L.pair_cap);
  if (B.bytes > ws_bytes || !ws) {
    set_error("backward workspace too small: need " + std::to_string(B.bytes));
    return CGS_EWORKSPACE;
  }
  return frame_backward(sc, fd, L, B, dL, final_T, scale, gpos, glogit, gsh, gsr, st);
}

}  // namespace cgs
