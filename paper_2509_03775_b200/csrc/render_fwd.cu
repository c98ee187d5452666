// Forward render path (reference render.py:145-315) for sm_100a.
//
//   sr_precompute   Sigma3 per SR codebook row (render.py:85-91, 168-169)
//   project         per (view, Gaussian): fp64 EWA projection, codebook gather,
//                   SH colour, pixel/tile rect, depth key (render.py:145-203,110-115)
//   compact + sort  on-screen splats, stable onesweep on fp64 depth bits
//                   (= np.lexsort((idx, tz)), render.py:203)
//   emit + sort     (tile, splat) pairs in depth order, stable sort by tile id
//                   (= per-tile append order of _bin_tiles, render.py:240-254)
//   raster_fwd      one 256-thread CTA per 16x16 tile, front-to-back blend with
//                   tile-level early exit (render.py:265-311)
#include <cmath>

#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

// ---------------------------------------------------------------------------
// Sigma3 = R(q/|q|) diag(exp(2 ls)) R^T per SR row; slot 6 flags |q| == 0.
__global__ void __launch_bounds__(256) sr_precompute_kernel(const float* __restrict__ rows,
                                                            int64_t cap, double* __restrict__ out) {
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
  uint32_t* n_tiles;
  uint64_t* rect;
  FrameHeader* hdr;
};

template <int DEG>
__global__ void __launch_bounds__(256) project_kernel(ProjIn in, FrameDesc fd, ProjOut out) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  constexpr int D = 3 * NB;
  const int64_t vn = in.n * fd.n_views;
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < vn;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = static_cast<int>(s / in.n);
    const int64_t i = s - static_cast<int64_t>(v) * in.n;
    const CamDev& cam = fd.cam[v];
    const double px = in.pos[3 * i + 0], py = in.pos[3 * i + 1], pz = in.pos[3 * i + 2];
    // camera coordinates t = R p + trans (camera.py:29-32)
    const double tx = cam.R[0] * px + cam.R[1] * py + cam.R[2] * pz + cam.t[0];
    const double ty = cam.R[3] * px + cam.R[4] * py + cam.R[5] * pz + cam.t[1];
    const double tz = cam.R[6] * px + cam.R[7] * py + cam.R[8] * pz + cam.t[2];
    if (!(tz > kNear)) {  // near-plane cull, render.py:149
      out.n_tiles[s] = 0;
      continue;
    }
    const double* cv = in.sr_cov + static_cast<int64_t>(in.g2sr[i]) * 8;
    if (cv[6] != 0.0) {  // zero quaternion: reference raises ValueError
      out.n_tiles[s] = 0;
      out.hdr->stats.zero_quaternion = 1;
      continue;
    }
    const double mx = cam.fx * tx / tz + cam.cx;
    const double my = cam.fy * ty / tz + cam.cy;
    // J (render.py:160-164) and M = J R (render.py:165)
    const double j00 = cam.fx / tz, j02 = -cam.fx * tx / (tz * tz);
    const double j11 = cam.fy / tz, j12 = -cam.fy * ty / (tz * tz);
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
      continue;
    }
    const int tx0 = static_cast<int>(x0) / kTile, tx1 = static_cast<int>(x1) / kTile;
    const int ty0 = static_cast<int>(y0) / kTile, ty1 = static_cast<int>(y1) / kTile;
    // view direction and SH colour (render.py:187-198)
    double ox = px - cam.center[0], oy = py - cam.center[1], oz = pz - cam.center[2];
    const double len = sqrt((ox * ox + oy * oy) + oz * oz);
    ox /= len; oy /= len; oz /= len;
    double B[NB];
    sh_basis<DEG>(ox, oy, oz, B);
    const float* row = in.sh_rows + static_cast<int64_t>(in.g2sh[i]) * D;
    double col[3] = {0.0, 0.0, 0.0};
    if constexpr (D % 4 == 0) {
      const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
      for (int q = 0; q < D / 4; ++q) {
        const float4 f = __ldg(r4 + q);
        const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = 4 * q + u;
          col[e % 3] += B[e / 3] * static_cast<double>(fv[u]);
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < D; ++e) col[e % 3] += B[e / 3] * static_cast<double>(__ldg(row + e));
    }
    SplatRec rec;
    rec.mx = mx;
    rec.my = my;
    rec.ca = c / det;
    rec.cb = -b / det;
    rec.cc = a / det;
    rec.opac = 1.0 / (1.0 + exp(-static_cast<double>(in.logit[i])));
    rec.r = static_cast<float>(fmax(col[0] + 0.5, 0.0));
    rec.g = static_cast<float>(fmax(col[1] + 0.5, 0.0));
    rec.b = static_cast<float>(fmax(col[2] + 0.5, 0.0));
    rec.rect = 0u;
    out.recs[s] = rec;
    out.depth_key[s] = static_cast<uint64_t>(__double_as_longlong(tz));
    out.n_tiles[s] = static_cast<uint32_t>((ty1 - ty0 + 1) * (tx1 - tx0 + 1));
    out.rect[s] = static_cast<uint64_t>(tx0) | (static_cast<uint64_t>(tx1) << 16) |
                  (static_cast<uint64_t>(ty0) << 32) | (static_cast<uint64_t>(ty1) << 48);
  }
}

// ---------------------------------------------------------------------------
struct CompactOnscreen {
  const uint32_t* n_tiles;
  const uint64_t* depth;
  uint64_t* keys;
  uint32_t* vals;
  __device__ uint64_t load(int64_t i) const { return n_tiles[i] > 0 ? 1ULL : 0ULL; }
  __device__ void store(int64_t i, uint64_t ex, uint64_t v) const {
    if (v) {
      keys[ex] = depth[i];
      vals[ex] = static_cast<uint32_t>(i);
    }
  }
};

struct PairOffsets {
  const uint32_t* sorted;
  const uint32_t* n_tiles;
  uint64_t* off;
  __device__ uint64_t load(int64_t j) const { return n_tiles[sorted[j]]; }
  __device__ void store(int64_t j, uint64_t ex, uint64_t) const { off[j] = ex; }
};

__global__ void finalize_counts_kernel(FrameHeader* hdr, int64_t pair_cap, int n_views) {
  const unsigned long long raw = hdr->n_pairs_raw;
  const bool over = raw > static_cast<unsigned long long>(pair_cap);
  hdr->n_pairs = over ? 0ULL : raw;
  hdr->stats.n_onscreen = static_cast<int64_t>(hdr->n_onscreen);
  hdr->stats.n_pairs = static_cast<int64_t>(raw);
  hdr->stats.overflow = over ? 1 : 0;
  hdr->stats.pair_capacity = pair_cap;
  hdr->stats.n_views = n_views;
}

// Warp-cooperative pair emission: a warp takes 32 consecutive splats in depth
// order and writes their concatenated pair range with all 32 lanes, so a
// near-plane splat covering every tile does not serialise one thread.
template <typename KT>
__global__ void __launch_bounds__(256) emit_pairs_kernel(
    const uint32_t* __restrict__ sorted, const uint64_t* __restrict__ off,
    const uint32_t* __restrict__ n_tiles, const uint64_t* __restrict__ rect,
    const FrameHeader* __restrict__ hdr, FrameDesc fd, int64_t n, KT* __restrict__ keys,
    uint32_t* __restrict__ vals) {
  if (hdr->stats.overflow) return;
  const int64_t ns = static_cast<int64_t>(hdr->n_onscreen);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       w * 32 < ns; w += warps) {
    const int64_t j = w * 32 + lane;
    const bool ok = j < ns;
    const uint32_t s = ok ? sorted[j] : 0u;
    const uint64_t cnt = ok ? n_tiles[s] : 0ULL;
    uint64_t o = ok ? off[j] : ~0ULL;
    uint64_t e = ok ? o + cnt : 0ULL;
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) {
      const uint64_t t = __shfl_xor_sync(kFull, e, k);
      e = t > e ? t : e;
    }
    const uint64_t start = __shfl_sync(kFull, o, 0);
    const uint64_t rc = ok ? rect[s] : 0ULL;
    const int v = ok ? static_cast<int>(s / n) : 0;
    const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
    const int ty0 = static_cast<int>((rc >> 32) & 0xffff);
    const int span = tx1 - tx0 + 1;
    const int ntx = fd.cam[v].ntx;
    const int tbase = fd.cam[v].tile_base;
    for (uint64_t p0 = start; p0 < e; p0 += 32) {
      const uint64_t p = p0 + lane;
      int owner = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int cand = owner + step;
        const uint64_t oc = __shfl_sync(kFull, o, cand & 31);
        if (cand < 32 && oc <= p) owner = cand;
      }
      const uint64_t oo = __shfl_sync(kFull, o, owner);
      const int sp = __shfl_sync(kFull, span, owner);
      const int bx = __shfl_sync(kFull, tx0, owner);
      const int by = __shfl_sync(kFull, ty0, owner);
      const int nt = __shfl_sync(kFull, ntx, owner);
      const int tb = __shfl_sync(kFull, tbase, owner);
      const uint32_t sid = __shfl_sync(kFull, s, owner);
      if (p < e) {
        const int k = static_cast<int>(p - oo);
        const int ty = by + k / sp, tx = bx + k % sp;
        keys[p] = static_cast<KT>(tb + ty * nt + tx);
        vals[p] = sid;
      }
    }
  }
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
// Forward raster: 256 threads = 16x16 pixels of one tile.  Splats are staged
// 256 at a time into shared memory (fp64 record -> tile-relative fp32
// offsets), the next batch's records are prefetched into registers while
// the current batch is blended, and the CTA exits as soon as every pixel's
// transmittance is below 1e-4.
__global__ void __launch_bounds__(256) raster_fwd_kernel(
    FrameDesc fd, const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_vals,
    const SplatRec* __restrict__ recs, const FrameHeader* __restrict__ hdr,
    float* __restrict__ image, float* __restrict__ final_T, int32_t* __restrict__ counts,
    uint32_t* __restrict__ px_last, uint32_t* __restrict__ tile_nproc) {
  __shared__ float4 s_a[256];
  __shared__ float4 s_b[256];
  __shared__ float s_c[256];
  __shared__ uint32_t s_max[8];
  if (hdr->stats.overflow) return;
  const int tile = blockIdx.x;
  int v = 0;
  while (v + 1 < fd.n_views && fd.cam[v + 1].tile_base <= tile) ++v;
  const CamDev& cam = fd.cam[v];
  const int lt = tile - cam.tile_base;
  const int ty = lt / cam.ntx, tx = lt - ty * cam.ntx;
  const int tid = threadIdx.x;
  const int lx = tid & 15, ly = tid >> 4;
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < cam.width && py < cam.height;
  const uint2 rg = ranges[tile];
  const int n = static_cast<int>(rg.y - rg.x);
  const double ox = static_cast<double>(tx * kTile), oy = static_cast<double>(ty * kTile);
  const float flx = static_cast<float>(lx), fly = static_cast<float>(ly);

  float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
  int cnt = 0;
  uint32_t last = 0;
  bool done = !inside;
  bool terminated = false;

  SplatRec nxt;
  if (tid < n) nxt = recs[pair_vals[rg.x + tid]];
  for (int b0 = 0; b0 < n; b0 += 256) {
    const int nb = min(256, n - b0);
    if (tid < nb) {
      float4 a, b;
      float c;
      stage_splat(nxt, ox, oy, a, b, c);
      s_a[tid] = a;
      s_b[tid] = b;
      s_c[tid] = c;
    }
    __syncthreads();
    if (b0 + 256 + tid < n) nxt = recs[pair_vals[rg.x + b0 + 256 + tid]];
    if (!done) {
      for (int j = 0; j < nb; ++j) {
        const float4 a = s_a[j];
        const float4 b = s_b[j];
        const float dx = a.x + flx, dy = a.y + fly;
        const float al = splat_alpha(a, b, dx, dy);
        if (al >= kAlphaSkipF) {
          const float w = al * T;
          cr = fmaf(w, b.z, cr);
          cg = fmaf(w, b.w, cg);
          cb = fmaf(w, s_c[j], cb);
          T = T * (1.0f - al);
          ++cnt;
          if (!(T >= kTMinF)) {
            done = true;
            terminated = true;
            last = static_cast<uint32_t>(b0 + j + 1);
            break;
          }
        }
      }
    }
    if (__syncthreads_count(done) == 256) break;
  }
  if (inside && !terminated) last = static_cast<uint32_t>(n);
  if (inside) {
    const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
    image[3 * pix + 0] = cr;
    image[3 * pix + 1] = cg;
    image[3 * pix + 2] = cb;
    final_T[pix] = T;
    counts[pix] = cnt;
    px_last[pix] = last;
  }
  uint32_t m = last;
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) m = max(m, __shfl_xor_sync(kFull, m, k));
  if ((tid & 31) == 0) s_max[tid >> 5] = m;
  __syncthreads();
  if (tid == 0) {
    uint32_t mm = 0;
    for (int w = 0; w < 8; ++w) mm = max(mm, s_max[w]);
    tile_nproc[tile] = mm;
  }
}

// ---------------------------------------------------------------------------
template <int DEG>
static void launch_project(const ProjIn& in, const FrameDesc& fd, const ProjOut& out,
                           int64_t vn, cudaStream_t st) {
  CGS_PROFILED("project_kernel", st, project_kernel<DEG><<<grid_for(vn, 256, 16), 256, 0, st>>>(in, fd, out));
}

template <typename KT>
static int sort_and_range(FrameLayout& L, const FrameDesc& fd, SortWs<KT>& ws,
                          cudaStream_t st) {
  KT* kres;
  uint32_t* vres;
  int rc = launch_radix_sort<KT>(static_cast<KT*>(L.pkeys), L.pvals, &L.hdr->n_pairs, 0,
                                 L.pair_cap, L.tile_key_bits, ws, &kres, &vres, st);
  if (rc) return rc;
  CGS_CUDA(cudaMemsetAsync(L.ranges, 0, sizeof(uint2) * (fd.total_tiles > 0 ? fd.total_tiles : 1), st));
  tile_ranges_kernel<KT><<<grid_for(L.pair_cap, 256, 8), 256, 0, st>>>(kres, L.hdr, L.ranges);
  CGS_CHECK_LAUNCH("tile_ranges_kernel");
  return CGS_OK;
}

int frame_forward(const cgs_scene_t* sc, const FrameDesc& fd, FrameLayout& L, float* image,
                  float* final_T, int32_t* counts, double* sr_cov, cudaStream_t st) {
  const int64_t vn = L.vn;
  CGS_CUDA(cudaMemsetAsync(L.hdr, 0, sizeof(FrameHeader), st));
  if (sc->sr_capacity > 0) {
    CGS_PROFILED("sr_precompute_kernel", st, sr_precompute_kernel<<<grid_for(sc->sr_capacity, 256, 4), 256, 0, st>>>(sc->sr_rows,
                                                                            sc->sr_capacity, sr_cov));
    CGS_CHECK_LAUNCH("sr_precompute_kernel");
  }
  if (vn > 0) {
    ProjIn in{sc->n, sc->positions, sc->opacity_logits, sc->g2sh, sc->g2sr, sc->sh_rows, sr_cov};
    ProjOut out{L.recs, L.depth_key, L.n_tiles, L.rect, L.hdr};
    switch (sc->sh_degree) {
      case 0: launch_project<0>(in, fd, out, vn, st); break;
      case 1: launch_project<1>(in, fd, out, vn, st); break;
      case 2: launch_project<2>(in, fd, out, vn, st); break;
      default: launch_project<3>(in, fd, out, vn, st); break;
    }
    CGS_CHECK_LAUNCH("project_kernel");
  }
  int rc = launch_scan(CompactOnscreen{L.n_tiles, L.depth_key, L.skeys, L.svals}, nullptr, vn, vn,
                       L.scan, &L.hdr->n_onscreen, st);
  if (rc) return rc;
  uint64_t* dk;
  uint32_t* dv;
  rc = launch_radix_sort<uint64_t>(L.skeys, L.svals, &L.hdr->n_onscreen, 0, vn, 64, L.dsort, &dk,
                                   &dv, st);
  if (rc) return rc;
  rc = launch_scan(PairOffsets{dv, L.n_tiles, L.pair_off}, &L.hdr->n_onscreen, 0, vn, L.scan,
                   &L.hdr->n_pairs_raw, st);
  if (rc) return rc;
  finalize_counts_kernel<<<1, 1, 0, st>>>(L.hdr, L.pair_cap, fd.n_views);
  CGS_CHECK_LAUNCH("finalize_counts_kernel");
  const int eg = grid_for(vn, 256, 16);
  if (L.tile_key_bytes == 2) {
    CGS_PROFILED("emit_pairs_kernel", st, emit_pairs_kernel<uint16_t><<<eg, 256, 0, st>>>(dv, L.pair_off, L.n_tiles, L.rect, L.hdr, fd,
                                                    L.n, static_cast<uint16_t*>(L.pkeys), L.pvals));
    CGS_CHECK_LAUNCH("emit_pairs_kernel");
    rc = sort_and_range<uint16_t>(L, fd, L.psort16, st);
  } else {
    CGS_PROFILED("emit_pairs_kernel", st, emit_pairs_kernel<uint32_t><<<eg, 256, 0, st>>>(dv, L.pair_off, L.n_tiles, L.rect, L.hdr, fd,
                                                    L.n, static_cast<uint32_t*>(L.pkeys), L.pvals));
    CGS_CHECK_LAUNCH("emit_pairs_kernel");
    rc = sort_and_range<uint32_t>(L, fd, L.psort32, st);
  }
  if (rc) return rc;
  if (fd.total_tiles > 0) {
    CGS_PROFILED("raster_fwd_kernel", st, raster_fwd_kernel<<<fd.total_tiles, 256, 0, st>>>(fd, L.ranges, sorted_pair_vals(L), L.recs,
                                                      L.hdr, image, final_T, counts, L.px_last,
                                                      L.tile_nproc));
    CGS_CHECK_LAUNCH("raster_fwd_kernel");
  }
  return CGS_OK;
}

}  // namespace cgs
