// Tile rasterizer kernels, forward and backward (reference render.py:265-377).
//
// Forward: one CTA per 16x16 tile, 256 threads, one pixel each, warp w on
// the 8x4 block ((w & 1) * 8, (w >> 1) * 4), each half-warp on one 4x4 half
// of it with its own hit list (fwd_px_x / fwd_px_y).  Backward: persistent CTAs of
// 128 threads over (tile, 256-splat chunk) work units; warp w on the 8x8
// quadrant ((w & 1) * 8, (w >> 1) * 8), each lane on pixels (x, y) and
// (x, y + 4) (two pixels per lane amortise its per-splat warp reduction); a
// unit starts from the per-pixel state the forward left at its chunk end.
// A splat whose contribution box (projection: the bounding box of its
// alpha >= 1/255 ellipse, inside the pixel rect of render.py:110-115) misses
// a warp's pixel block is skipped by that warp without evaluating it:
// outside the box the reference's float64 alpha is < 1/255, so the skip
// changes no result.
//
// Work is taken longest-first (tile_order_kernel for the forward's tiles,
// unit_order_kernel for the backward's units): greedy longest-processing-time
// scheduling of the uneven lists, so the last wave is made of short ones.
// Tiles and units are independent, so the order changes no result.
//
// Splat records are gathered by the bulk-copy engine (cp.async.bulk, one
// 64-byte record per copy, completion on an mbarrier) one batch ahead of the
// blending, and converted once per batch to tile-relative fp32 form in shared
// memory.
#include <atomic>

#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

#ifndef CGS_BWD_EIGEN_CULL
#define CGS_BWD_EIGEN_CULL 1
#endif
#ifndef CGS_FWD_EIGEN_CULL
#define CGS_FWD_EIGEN_CULL 0
#endif
#ifndef CGS_FWD_NOBAND  // timing experiments only: no flagging (not exact)
#define CGS_FWD_NOBAND 0
#endif

// Tile-local inclusive contribution box of a splat as 4 signed bytes
// (x0, x1, y0, y1), clamped to [-1, 16] (an empty box has x0 = 16: no hit).
__device__ __forceinline__ uint32_t local_rect(const SplatRec& r, int tx0, int ty0) {
  auto c = [](int v) { return static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(v < -1 ? -1 : (v > 16 ? 16 : v)))); };
  return c(r.px0 - tx0) | (c(r.px1 - tx0) << 8) | (c(r.py0 - ty0) << 16) | (c(r.py1 - ty0) << 24);
}

__device__ __forceinline__ bool quad_hit(uint32_t rc, int qx, int qy) {
  const int x0 = static_cast<int8_t>(rc & 0xff), x1 = static_cast<int8_t>((rc >> 8) & 0xff);
  const int y0 = static_cast<int8_t>((rc >> 16) & 0xff), y1 = static_cast<int8_t>(rc >> 24);
  return x1 >= qx && x0 <= qx + 7 && y1 >= qy && y0 <= qy + 7;
}

// Counting sort of tiles by descending work (work / 16 in 256 buckets) in one
// CTA.  work = list length (forward) or processed prefix (backward).  The
// order inside a bucket is whatever the shared atomics give: scheduling only.
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2* __restrict__ ranges,
                                                          const uint32_t* __restrict__ nproc,
                                                          int total_tiles,
                                                          uint32_t* __restrict__ order,
                                                          uint32_t* __restrict__ zero_a,
                                                          uint64_t* __restrict__ zero_b,
                                                          unsigned long long* __restrict__ zero_v,
                                                          int n_views) {
  __shared__ uint32_t cnt[256];
  const int tid = threadIdx.x;
  auto bucket = [&](int t) -> uint32_t {
    const uint32_t w = nproc ? nproc[t] : ranges[t].y - ranges[t].x;
    return 255u - min(255u, w >> 4);
  };
  if (tid < 256) cnt[tid] = 0;
  __syncthreads();
  for (int t = tid; t < total_tiles; t += blockDim.x) atomicAdd(&cnt[bucket(t)], 1u);
  __syncthreads();
  if (tid < 32) {  // exclusive scan of 256 counts, 8 per lane
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c[k] = cnt[tid * 8 + k];
      sum += c[k];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (tid >= o) inc += y;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cnt[tid * 8 + k] = run;
      run += c[k];
    }
  }
  __syncthreads();
  for (int t = tid; t < total_tiles; t += blockDim.x) order[atomicAdd(&cnt[bucket(t)], 1u)] = t;
  if (zero_a)  // the forward's per-tile maxima start from 0 (split tiles combine with atomicMax)
    for (int t = tid; t < total_tiles; t += blockDim.x) {
      zero_a[t] = 0u;
      zero_b[t] = 0ull;
    }
  if (zero_v)  // and its per-view maxima of the last processed depth keys
    for (int v = tid; v < n_views; v += blockDim.x) zero_v[v] = 0ull;
}

// Per-pixel forward state.  `last` doubles as the done flag (last index + 1
// once the pixel terminated; pixels outside the image start done with
// last = 1); `refine` flags the pixel for the float64 re-walk (T came within
// kTBand of 1e-4, or an alpha within kAlphaBand of 1/255 or 0.99: refine.cu).
struct PixState {
  float T, r, g, b;
  int cnt;
  uint32_t last;
  bool refine;
  __device__ __forceinline__ bool done() const { return last != 0u; }
};

// Front-to-back blend of one splat into one pixel (render.py:274-283, 302-311).
__device__ __forceinline__ void blend(PixState& p, float al, float cr, float cg, float cb,
                                      uint32_t idx) {
  if (p.done() || !(al >= kAlphaSkipF)) return;
  const float w = al * p.T;
  p.r = fmaf(w, cr, p.r);
  p.g = fmaf(w, cg, p.g);
  p.b = fmaf(w, cb, p.b);
  p.T = p.T * (1.0f - al);
  ++p.cnt;
  if (p.T < kTBandHi) {  // rare: near or past the termination threshold
#if !CGS_FWD_NOBAND
    p.refine |= p.T >= kTBandLo;  // the float64 chain may fall on either side
#endif
    if (!(p.T >= kTMinF)) p.last = idx + 1;  // every later splat is inactive (T_before < 1e-4)
  }
}

// 4-bit mask of the tile quadrants a tile-local contribution box overlaps
// (bit w = quadrant ((w & 1) * 8, (w >> 1) * 8), the pixels of warp w).
__device__ __forceinline__ uint32_t quad_mask(uint32_t rc) {
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w)
    if (quad_hit(rc, (w & 1) * 8, (w >> 1) * 8)) m |= 1u << w;
  return m;
}

// Per-warp ordered list of the batch entries j < nb whose mask has bit
// `warp`; returns the count.  (8 ballots per 256 entries instead of a
// per-entry skip test in the blend loop.)
template <int NB>
__device__ __forceinline__ int warp_hit_list(const uint8_t* s_mask, int nb, int warp, int lane,
                                             uint8_t* list) {
  int cnt = 0;
#pragma unroll
  for (int c = 0; c < NB / 32; ++c) {
    const int j = c * 32 + lane;
    const bool hit = j < nb && ((s_mask[j] >> warp) & 1u);
    const unsigned bal = __ballot_sync(kFull, hit);
    if (hit) list[cnt + __popc(bal & lanemask_lt())] = static_cast<uint8_t>(j);
    cnt += __popc(bal);
  }
  __syncwarp();
  return cnt;
}

// Forward: 256 threads, one pixel each; warp w owns the 8x4 block
// ((w & 1) * 8, (w >> 1) * 4) of the tile and walks only the splats whose
// contribution box meets it (8-bit block masks, per-warp hit lists).  Finer
// blocks than the backward's quadrants skip more splats, and 8 warps per tile
// hide more latency (no per-splat reduction here to amortise).
__device__ __forceinline__ uint32_t block8x4_mask(uint32_t rc) {
  const int x0 = static_cast<int8_t>(rc & 0xff), x1 = static_cast<int8_t>((rc >> 8) & 0xff);
  const int y0 = static_cast<int8_t>((rc >> 16) & 0xff), y1 = static_cast<int8_t>(rc >> 24);
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const int bx = (w & 1) * 8, by = (w >> 1) * 4;
    if (x1 >= bx && x0 <= bx + 7 && y1 >= by && y0 <= by + 3) m |= 1u << w;
  }
  return m;
}

// CGS_FWD_HALF: 16-bit mask of the 4x4 blocks a contribution box meets, bit
// 4 qy + qx for the block (4 qx, 4 qy) -- the half (lane >> 4) of warp w is
// bit 2 w + (lane >> 4) (fwd_px_x / fwd_px_y).
__device__ __forceinline__ uint32_t block4x4_mask(uint32_t rc) {
  const int x0 = static_cast<int8_t>(rc & 0xff), x1 = static_cast<int8_t>((rc >> 8) & 0xff);
  const int y0 = static_cast<int8_t>((rc >> 16) & 0xff), y1 = static_cast<int8_t>(rc >> 24);
  uint32_t cm = 0, m = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (x1 >= 4 * q && x0 <= 4 * q + 3) cm |= 1u << q;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (y1 >= 4 * q && y0 <= 4 * q + 3) m |= cm << (4 * q);
  return m;
}

// Two ordered hit lists per warp, one per half-warp (bits 2 warp and
// 2 warp + 1 of the 16-bit masks); returns this lane's half's count.
template <int NB>
__device__ __forceinline__ int warp_hit_lists2(const uint16_t* s_mask, int nb, int warp, int lane,
                                               uint8_t* list0, uint8_t* list1) {
  int c0 = 0, c1 = 0;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int c = 0; c < NB / 32; ++c) {
    const int j = c * 32 + lane;
    const uint32_t m = j < nb ? (s_mask[j] >> (2 * warp)) & 3u : 0u;
    const unsigned b0 = __ballot_sync(kFull, m & 1u), b1 = __ballot_sync(kFull, m & 2u);
    if (m & 1u) list0[c0 + __popc(b0 & lt)] = static_cast<uint8_t>(j);
    if (m & 2u) list1[c1 + __popc(b1 & lt)] = static_cast<uint8_t>(j);
    c0 += __popc(b0);
    c1 += __popc(b1);
  }
  __syncwarp();
  return (lane >> 4) ? c1 : c0;
}

#ifndef CGS_FWD_PAIRS
#define CGS_FWD_PAIRS 1
#endif
#ifndef CGS_FWD_MINB
#define CGS_FWD_MINB 6
#endif
// Diagnostics: CGS_REFINE_ALL=1 flags every pixel for the float64 re-walk
// (the refine kernels then also record how far the fp32 path was from it).
#ifndef CGS_REFINE_ALL
#define CGS_REFINE_ALL 0
#endif
constexpr int kFwdThreads = 256;  // one pixel per thread
constexpr int kFwdBatch = 256;
constexpr int kFwdWarps = kFwdThreads / 32;
#ifndef CGS_FWD_FIRST
#define CGS_FWD_FIRST 128
#endif
constexpr int kFwdFirst = CGS_FWD_FIRST;  // first batch
static_assert(kChunk % kFwdBatch == 0, "checkpoints sit on batch boundaries");
static_assert(kFwdFirst > 0 && kFwdFirst <= kFwdBatch && kFwdFirst % 32 == 0, "first batch");
__global__ void __launch_bounds__(kFwdThreads, CGS_FWD_MINB) raster_fwd_kernel(
    FrameDesc fd, const uint32_t* __restrict__ order, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ pair_vals, const SplatRec* __restrict__ recs,
    FrameHeader* __restrict__ hdr, float* __restrict__ image,
    float* __restrict__ final_T, int32_t* __restrict__ counts, uint32_t* __restrict__ px_last,
    uint32_t* __restrict__ tile_nproc, const uint64_t* __restrict__ depth_key,
    uint64_t* __restrict__ tile_last_dk, uint32_t* __restrict__ tile_last_sid,
    unsigned long long* __restrict__ view_last_dk, float4* __restrict__ ckpt,
    uint32_t* __restrict__ refine_tiles, uint32_t* __restrict__ refine_mask,
    unsigned long long* __restrict__ trace) {
  constexpr int B = kFwdBatch, NT = kFwdThreads;
  const unsigned long long t_start = trace ? global_ns() : 0ull;
  __shared__ __align__(128) SplatRec s_raw[B];
  // staged splats, one 48-byte entry each (a, b, colour): one address per hit
  __shared__ float4 s_st[B][3];
#if CGS_FWD_HALF
  __shared__ uint16_t s_mask[B];
  __shared__ uint8_t s_list[kFwdWarps][2][B];
#else
  __shared__ uint8_t s_mask[B];
  __shared__ uint8_t s_list[kFwdWarps][B];
#endif
  __shared__ uint32_t s_max[kFwdWarps];
  __shared__ __align__(8) uint64_t s_bar;
  if (hdr->stats.overflow) return;
  const int tile = static_cast<int>(order[blockIdx.x]);
  int v = 0;
  while (v + 1 < fd.n_views && fd.cam[v + 1].tile_base <= tile) ++v;
  const CamDev& cam = fd.cam[v];
  const int lt = tile - cam.tile_base;
  const int ty = lt / cam.ntx, tx = lt - ty * cam.ntx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lx = fwd_px_x(warp, lane), ly = fwd_px_y(warp, lane);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool in = px < cam.width && py < cam.height;
  const uint2 rg = ranges[tile];
  const int n = static_cast<int>(rg.y - rg.x);
  const double cx = tile_centre(tx), cy = tile_centre(ty);
  const float flx = static_cast<float>(lx) - kTileHalf, fly = static_cast<float>(ly) - kTileHalf;
#if CGS_FWD_HALF
  uint8_t* my_list = s_list[warp][lane >> 4];
#else
  uint8_t* my_list = s_list[warp];
#endif
  PixState p{1.0f, 0.0f, 0.0f, 0.0f, 0, in ? 0u : 1u, CGS_REFINE_ALL != 0};
  int n_ckpt = 0;
  // fp32 alpha to blend (render.py:274-279); the caller keeps it when it is
  // >= kAlphaSkipF.  A pixel that meets a t within a decision band of
  // raster_common.cuh is flagged for the float64 re-walk (refine.cu), which
  // overwrites it.  The keep band (|t| < band) and the clamp band
  // (|t - kTClamp| < band) are symmetric about kTClamp / 2, so one test
  // catches both: ||t - kTClamp/2| - kTClamp/2| < band.
  auto eval = [&](const float4& a, const float4& b) -> float {
    const float t = staged_t(a, b, flx, fly);
#if !CGS_FWD_NOBAND
    p.refine |= fabsf(fabsf(t - kTHalfClamp) - kTHalfClamp) < kTSkipHi;
#endif
    return alpha_of_t(t);
  };
  if (tid == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  bool pending = false;
  // batch ends: kFwdFirst, then the multiples of B (a tile whose pixels all
  // terminate early stages only the first few splats of its list)
  auto batch_end = [&](int b) { return min(b == 0 ? kFwdFirst : (b / B + 1) * B, n); };
  if (n > 0) {
    issue_records(s_raw, &s_bar, pair_vals, recs, rg.x, batch_end(0), tid, NT);
    pending = true;
  }
  for (int b0 = 0, bend = batch_end(0); b0 < n; b0 = bend, bend = batch_end(bend)) {
    const int nb = bend - b0;
    records_wait(&s_bar, phase);
    pending = false;
    if (tid < nb) {
      const Staged sg = stage_splat(s_raw[tid], cx, cy);
      s_st[tid][0] = sg.a;
      s_st[tid][1] = sg.b;
      s_st[tid][2] = make_float4(sg.c.x, sg.c.y, 0.0f, 0.0f);
#if CGS_FWD_HALF
      uint32_t m8 = block4x4_mask(local_rect(s_raw[tid], tx * kTile, ty * kTile));
#if CGS_FWD_EIGEN_CULL
#pragma unroll
      for (int w = 0; w < 16; ++w) {  // 4x4 blocks the ellipse cannot reach
        const float x0 = (w & 3) * 4 - kTileHalf, y0 = (w >> 2) * 4 - kTileHalf;
        if ((m8 >> w) & 1u)
          if (!staged_may_hit(sg.a, sg.b, x0, x0 + 3.0f, y0, y0 + 3.0f)) m8 &= ~(1u << w);
      }
#endif
      s_mask[tid] = static_cast<uint16_t>(m8);
#else
      uint32_t m8 = block8x4_mask(local_rect(s_raw[tid], tx * kTile, ty * kTile));
#if CGS_FWD_EIGEN_CULL
#pragma unroll
      for (int w = 0; w < 8; ++w) {  // 8x4 blocks the ellipse cannot reach
        const float x0 = (w & 1) * 8 - kTileHalf, y0 = (w >> 1) * 4 - kTileHalf;
        if ((m8 >> w) & 1u)
          if (!staged_may_hit(sg.a, sg.b, x0, x0 + 7.0f, y0, y0 + 3.0f)) m8 &= ~(1u << w);
      }
#endif
      s_mask[tid] = static_cast<uint8_t>(m8);
#endif
    }
    __syncthreads();
    if (bend < n) {
      fence_proxy_async_smem();
      issue_records(s_raw, &s_bar, pair_vals, recs, rg.x + bend, batch_end(bend) - bend, tid, NT);
      pending = true;
    }
#if CGS_FWD_HALF
    const int hits = warp_hit_lists2<B>(s_mask, nb, warp, lane, s_list[warp][0], s_list[warp][1]);
#else
    const int hits = warp_hit_list<B>(s_mask, nb, warp, lane, my_list);
#endif
    if (!p.done()) {
#if CGS_FWD_PAIRS
      // two hits per iteration: both alphas are independent of the blend
      // state, so they issue together; the blends stay in list order
      int i = 0;
      for (; i + 1 < hits; i += 2) {
        const int j0 = my_list[i], j1 = my_list[i + 1];
        const float4 a0 = s_st[j0][0], b0v = s_st[j0][1];
        const float4 a1 = s_st[j1][0], b1v = s_st[j1][1];
        const float al0 = eval(a0, b0v);
        const float al1 = eval(a1, b1v);
        if (al0 >= kAlphaSkipF) {
          const float4 c = s_st[j0][2];
          blend(p, al0, b0v.w, c.x, c.y, static_cast<uint32_t>(b0 + j0));
          if (p.done()) break;
        }
        if (al1 >= kAlphaSkipF) {
          const float4 c = s_st[j1][2];
          blend(p, al1, b1v.w, c.x, c.y, static_cast<uint32_t>(b0 + j1));
          if (p.done()) break;
        }
      }
      if (!p.done() && i < hits) {
        const int j = my_list[i];
        const float4 a = s_st[j][0], b = s_st[j][1];
        const float al = eval(a, b);
        if (al >= kAlphaSkipF) {
          const float4 c = s_st[j][2];
          blend(p, al, b.w, c.x, c.y, static_cast<uint32_t>(b0 + j));
        }
      }
#else
      for (int i = 0; i < hits; ++i) {
        const int j = my_list[i];
        const float4 a = s_st[j][0], b = s_st[j][1];
        const float al = eval(a, b);
        if (al >= kAlphaSkipF) {
          const float4 c = s_st[j][2];
          blend(p, al, b.w, c.x, c.y, static_cast<uint32_t>(b0 + j));
          if (p.done()) break;
        }
      }
#endif
    }
    if (__syncthreads_count(p.done()) == NT) break;
    if (bend < n && (bend % kChunk) == 0) {  // chunk boundary for the backward
      // T after the chunk and the chunk's own colour sum; colour restarts at 0
      ckpt[ckpt_slot(rg.x, tile, bend / kChunk) * kTilePixels + ly * kTile + lx] =
          make_float4(p.T, p.r, p.g, p.b);
      p.r = p.g = p.b = 0.0f;
      ++n_ckpt;
    }
  }
  if (pending) records_wait(&s_bar, phase);
  // Chunk sums -> suffix at each boundary (sum of the later chunks, so it
  // carries rounding relative to itself, like a back-to-front running sum)
  // and the pixel colour = sum of all chunks.  Only this thread's own writes.
  for (int j = n_ckpt; j >= 1; --j) {
    float4& c = ckpt[ckpt_slot(rg.x, tile, j) * kTilePixels + ly * kTile + lx];
    const float4 q = c;
    c = make_float4(q.x, p.r, p.g, p.b);
    p.r += q.y;
    p.g += q.z;
    p.b += q.w;
  }
  if (in && !p.done()) p.last = static_cast<uint32_t>(n);
  if (in) {
    const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
    image[3 * pix + 0] = p.r;
    image[3 * pix + 1] = p.g;
    image[3 * pix + 2] = p.b;
    final_T[pix] = p.T;
    counts[pix] = p.cnt;
    px_last[pix] = p.last;
  }
  {  // flagged pixels: per-warp masks and the tile in the re-walk list
    const unsigned bal = __ballot_sync(kFull, in && p.refine);
    if (__syncthreads_or(bal != 0u)) {
      if (lane == 0) refine_mask[static_cast<int64_t>(tile) * kFwdWarps + warp] = bal;
      if (tid == 0) refine_tiles[atomicAdd(&hdr->scratch[3], 1ull)] = static_cast<uint32_t>(tile);
    }
  }
  uint32_t m = in ? p.last : 0u;
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) m = max(m, __shfl_xor_sync(kFull, m, k));
  if (lane == 0) s_max[warp] = m;
  __syncthreads();
  if (tid == 0) {
    uint32_t np = 0;
#pragma unroll
    for (int w = 0; w < kFwdWarps; ++w) np = max(np, s_max[w]);
    const uint32_t ls = np ? pair_vals[rg.x + np - 1] : 0u;
    tile_nproc[tile] = np;
    const uint64_t ldk = np ? depth_key[ls] : 0ull;
    tile_last_dk[tile] = ldk;
    tile_last_sid[tile] = ls;
    if (np) atomicMax(&view_last_dk[v], static_cast<unsigned long long>(ldk));
    if (trace) {
      unsigned long long* t = trace + 4 * static_cast<int64_t>(blockIdx.x);
      t[0] = t_start;
      t[1] = global_ns();
      t[2] = smid();
      t[3] = static_cast<unsigned long long>(tile);
    }
  }
}

// ---------------------------------------------------------------------------
// Reverse traversal (render.py:343-377).  For pixel p and splat k < last_p,
// T is the transmittance after k, T_before = T / (1 - alpha_k) and the
// running suffix holds sum_{j>k} alpha_j T_j c_j.  Alpha is recomputed with
// exactly the forward's fp32 code, so skip/clamp/termination decisions match.
// Per splat the 9 gradient values (d_colour 3, d_opacity, d_mean2d 2,
// d_conic 3) are summed over the tile's pixels in fixed order: per warp a
// 12-shuffle transposed reduction, then the 4 warps in shared memory.
struct PixBwd {
  float T, gr, gg, gb;
  float sdot;  // suffix colour . dL/dC: only this dot product enters dL/dalpha
  uint32_t last;
};

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Adds pixel p's contribution of splat k to o[9]; returns whether it had one.
// o = [sum w g (3), sum dp, sum dp lx, sum dp ly, sum dp lx^2, sum dp lx ly,
// sum dp ly^2] with dp = dL/dalpha * alpha and (lx, ly) the pixel's offset
// from the tile centre.  The moments stay in these small local coordinates:
// splat_reduce shifts them to the splat centre in float64 (render.py:364-377's
// d_mean2d = sum dp Q d, d_conic = -1/2 sum dp d d^T with d = tile centre
// offset + (lx, ly)).  For splats centred far from the tile (near-plane
// giants) d_mean2d and d_conic are large and cancel in the pull-back; local
// moments keep every rounding error consistent between the two, so the
// cancellation survives.
// t = the fp32 log2(255 alpha) (raster_common.cuh).  Refined pixels
// (kRefinedBit) are skipped here (refine.cu adds them); on every other pixel
// the forward met no value inside the decision bands (it flags the pixel when
// it does), so t outside the bands decides exactly as the reference's float64
// alpha -- and t inside the keep band can only come from a pixel outside the
// splat's contribution box, which the forward's finer block lists never
// evaluated: there the float64 alpha is < 1/255 (not kept).
__device__ __forceinline__ bool bwd_pixel(PixBwd& p, uint32_t k, float t, float cr, float cg,
                                          float cb, float lx, float ly, float* o) {
  if (!(k < p.last) || !(t >= kTSkipHi)) return false;
  const float al = alpha_of_t(t);
  const bool flow = t < kTClampLo;  // no gradient through the clamp (render.py:361)
  const float iom = fast_rcp(1.0f - al);  // 1 - alpha >= 0.01
  const float Tb = p.T * iom;
  const float w = al * Tb;
  o[0] = fmaf(w, p.gr, o[0]);  // d colour += weight * dL (render.py:351-352)
  o[1] = fmaf(w, p.gg, o[1]);
  o[2] = fmaf(w, p.gb, o[2]);
  // dC/dalpha = c T_before - suffix / (1 - alpha) (render.py:357-359); dotted
  // with dL/dC: T_before (c . g) - (suffix . g) / (1 - alpha), the suffix kept
  // as its running dot product with g (suffix += w c  =>  sdot += w (c . g))
  const float cdot = fmaf(cr, p.gr, fmaf(cg, p.gg, cb * p.gb));
  const float da = fmaf(Tb, cdot, -p.sdot * iom);
  p.sdot = fmaf(w, cdot, p.sdot);
  p.T = Tb;
  if (flow) {
    const float dp = da * al;
    const float tx = dp * lx, ty = dp * ly;
    o[3] += dp;
    o[4] += tx;
    o[5] += ty;
    o[6] = fmaf(tx, lx, o[6]);
    o[7] = fmaf(tx, ly, o[7]);
    o[8] = fmaf(ty, ly, o[8]);
  }
  return true;
}

// Batches of kBwdBatch splats, last batch first.  Staging writes, per
// splat, the mask of warps that will process it (box meets the warp's
// quadrant and k < the warp's last index); each warp walks its ordered hit
// list backwards and stores its 9 reduced values per hit in its own s_red
// slice; the combine sums the present warps in fixed order.
#ifndef CGS_BWD_BATCH
#define CGS_BWD_BATCH 64
#endif
constexpr int kBwdBatch = CGS_BWD_BATCH;
#ifndef CGS_BWD_PAIR_REDUCE
#define CGS_BWD_PAIR_REDUCE 1
#endif
constexpr bool kBwdPairReduce = CGS_BWD_PAIR_REDUCE != 0;
static_assert(kBwdBatch % 32 == 0 && kChunk % kBwdBatch == 0 && kBwdBatch <= 256,
              "batch: whole ballots, whole batches per chunk, u8 hit-list entries");

// Backward work units: chunk c of tile t covers splats [c kChunk, min((c+1)
// kChunk, nproc_t)).  Sorted by length, longest first (counting sort in one
// CTA, as tile_order_kernel); ctl[0] = unit count, ctl[1] = fetch counter.
__global__ void __launch_bounds__(1024) unit_order_kernel(const uint32_t* __restrict__ nproc,
                                                          int total_tiles,
                                                          uint2* __restrict__ units,
                                                          uint32_t* __restrict__ ctl,
                                                          uint32_t* __restrict__ zero,
                                                          int n_zero,
                                                          uint32_t* __restrict__ zero2,
                                                          int n_zero2) {
  // Full chunks (length kChunk, the longest) first, in tile order, placed by
  // a block scan of per-tile counts (no shared-atomic contention on one
  // bucket); then the partial last chunks by length, longest first, through
  // 256 length buckets.
  __shared__ uint32_t cnt[256];
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_full;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto bucket = [](uint32_t w) -> uint32_t {  // w in [1, kChunk)
    return 255u - min(255u, ((w - 1u) * 256u) / kChunk);
  };
  if (tid < 256) cnt[tid] = 0;
  if (tid == 0) s_full = 0;
  for (int k = tid; k < n_zero; k += blockDim.x) zero[k] = 0u;  // the caller's spans (no memset nodes)
  for (int k = tid; k < n_zero2; k += blockDim.x) zero2[k] = 0u;
  __syncthreads();
  uint32_t full = 0;
  for (int t = tid; t < total_tiles; t += blockDim.x) {
    const uint32_t np = nproc[t];
    full += np / kChunk;
    if (np % kChunk) atomicAdd(&cnt[bucket(np % kChunk)], 1u);
  }
  full = warp_incl_scan(full);
  if (lane == 31 && full) atomicAdd(&s_full, full);
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the 256 partial buckets, after the full chunks
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c[k] = cnt[tid * 8 + k];
      sum += c[k];
    }
    uint32_t inc = warp_incl_scan(sum);
    uint32_t run = inc - sum + s_full;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cnt[tid * 8 + k] = run;
      run += c[k];
    }
    if (tid == 31) {
      ctl[0] = run;  // all units
      ctl[1] = 0u;
    }
  }
  __syncthreads();
  uint32_t base = 0;
  for (int t0 = 0; t0 < total_tiles; t0 += blockDim.x) {
    const int t = t0 + tid;
    const uint32_t np = t < total_tiles ? nproc[t] : 0u;
    const uint32_t nf = np / kChunk;
    const uint32_t inc = warp_incl_scan(nf);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      const uint32_t x = s_warp[w];
      if (w < warp) wpre += x;
      tot += x;
    }
    const uint32_t off = base + wpre + inc - nf;
    for (uint32_t c = 0; c < nf; ++c) units[off + c] = make_uint2(static_cast<uint32_t>(t), c);
    if (np % kChunk)
      units[atomicAdd(&cnt[bucket(np % kChunk)], 1u)] = make_uint2(static_cast<uint32_t>(t), nf);
    base += tot;
    __syncthreads();
  }
}

// Persistent CTAs fetch work units (unit_order_kernel) from a global
// counter.  A unit starts from the pixel state the forward left at its chunk
// end (ckpt: T and the colour suffix of the later splats; the tile's last
// chunk starts from final_T and an empty suffix), so the chunks of one tile
// run on different SMs at once and no tile's list length bounds the kernel.
template <bool TRACE>
__global__ void __launch_bounds__(128) raster_bwd_kernel(
    FrameDesc fd, const uint2* __restrict__ units, uint32_t* __restrict__ unit_ctl,
    const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ pair_vals, const SplatRec* __restrict__ recs,
    const FrameHeader* __restrict__ fh,
    const uint32_t* __restrict__ px_last, const uint32_t* __restrict__ tile_nproc,
    const float* __restrict__ final_T, const float* __restrict__ dL,
    const float4* __restrict__ ckpt,
    const uint64_t* __restrict__ pair_off, const uint64_t* __restrict__ rect, int64_t n,
    float* __restrict__ partials, int64_t partial9_offset,
    unsigned long long* __restrict__ n_processed,
    unsigned long long* __restrict__ trace) {
  constexpr int B = kBwdBatch;
  const unsigned long long t_start = trace ? global_ns() : 0ull;
  __shared__ __align__(128) SplatRec s_raw[B];
  static_assert(2 * B == 128, "staging and combine each take half of the CTA");
  __shared__ float4 s_a[2][B];
  __shared__ float4 s_b[2][B];
  __shared__ float2 s_n[2][B];  // green, blue
  __shared__ uint8_t s_mask[2][B];
  __shared__ uint8_t s_list[4][B];
  __shared__ uint32_t s_eidx[2][B];  // emission index of each staged pair
  __shared__ float s_red[2][4][B][9];
  __shared__ uint32_t s_wlast[4];
  __shared__ uint32_t s_unit;
  __shared__ __align__(8) uint64_t s_bar;
  if (fh->stats.overflow) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qx = (warp & 1) * 8, qy = (warp >> 1) * 8;
  const int lx = qx + (lane & 7), ly = qy + (lane >> 3);
  // tile-centred pixel coordinates (stage_splat); also the moments' coordinates
  const float flx = static_cast<float>(lx) - kTileHalf, fly = static_cast<float>(ly) - kTileHalf;
  const int slot = reduce9_slot(lane);
  const int slot18 = reduce_slot(18, lane);
  uint8_t* my_list = s_list[warp];
  const uint32_t n_units = unit_ctl[0];
  // splat jj of buffer cb: sum the present warps in fixed order and store
  // the 9 tile sums at the pair's emission index (values 0-7 as two aligned
  // float4, value 8 in the separate array after them)
  auto combine_splat = [&](int cb, int jj) {
    const uint32_t m = s_mask[cb][jj];
    float g[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const float r0 = (m & 1u) ? s_red[cb][0][jj][u] : 0.0f;
      const float r1 = (m & 2u) ? s_red[cb][1][jj][u] : 0.0f;
      const float r2 = (m & 4u) ? s_red[cb][2][jj][u] : 0.0f;
      const float r3 = (m & 8u) ? s_red[cb][3][jj][u] : 0.0f;
      g[u] = (r0 + r1) + (r2 + r3);
    }
    const int64_t e = s_eidx[cb][jj];
    float4* o4 = reinterpret_cast<float4*>(partials) + 2 * e;
    o4[0] = make_float4(g[0], g[1], g[2], g[3]);
    o4[1] = make_float4(g[4], g[5], g[6], g[7]);
    partials[partial9_offset + e] = g[8];
  };
  if (tid == 0) mbar_init(&s_bar, 1);
  uint32_t phase = 0;
  for (;;) {
    if (tid == 0) s_unit = atomicAdd(&unit_ctl[1], 1u);
    __syncthreads();
    const uint32_t ui = s_unit;
    if (ui >= n_units) break;
    const uint2 un = units[ui];
    const int tile = static_cast<int>(un.x);
    const int nproc = static_cast<int>(tile_nproc[tile]);
    const int k0 = static_cast<int>(un.y) * kChunk;
    const int k_end = min(k0 + kChunk, nproc);
    if (tid == 0) atomicAdd(n_processed, static_cast<unsigned long long>(k_end - k0));  // P_x
    int v = 0;
    while (v + 1 < fd.n_views && fd.cam[v + 1].tile_base <= tile) ++v;
    const CamDev& cam = fd.cam[v];
    const int lt = tile - cam.tile_base;
    const int ty = lt / cam.ntx, tx = lt - ty * cam.ntx;
    const int px = tx * kTile + lx, py0 = ty * kTile + ly, py1 = py0 + 4;
    const uint2 rg = ranges[tile];
    const double cx = tile_centre(tx), cy = tile_centre(ty);
    const bool last_chunk = k_end == nproc;
    const float4* ck = last_chunk ? nullptr
                                  : ckpt + ckpt_slot(rg.x, tile, k_end / kChunk) * kTilePixels;

    PixBwd q0{1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0u};
    PixBwd q1 = q0;
    auto load_px = [&](PixBwd& q, int py, int lyy) {
      if (px < cam.width && py < cam.height) {
        const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
        q.last = px_last[pix];
        if (q.last & kRefinedBit) return;  // raster_refine_kernel<true> takes this pixel
        q.gr = dL[3 * pix + 0];
        q.gg = dL[3 * pix + 1];
        q.gb = dL[3 * pix + 2];
        if (last_chunk || q.last <= static_cast<uint32_t>(k_end)) {
          // done before this chunk ends: final state, nothing behind it (a
          // split forward tile may not have written this boundary)
          q.T = final_T[pix];
        } else {
          const float4 c = ck[lyy * kTile + lx];
          q.T = c.x;
          q.sdot = fmaf(c.y, q.gr, fmaf(c.z, q.gg, c.w * q.gb));
        }
      }
    };
    load_px(q0, py0, ly);
    load_px(q1, py1, ly + 4);
    uint32_t wlast = max(q0.last, q1.last);  // warp-uniform upper bound of k
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) wlast = max(wlast, __shfl_xor_sync(kFull, wlast, k));
    if (lane == 0) s_wlast[warp] = wlast;
    __syncthreads();
    int b0 = k0 + ((k_end - 1 - k0) / B) * B;
    fence_proxy_async_smem();  // s_raw was read by the previous unit's staging
    issue_records(s_raw, &s_bar, pair_vals, recs, rg.x + b0, min(B, k_end - b0), tid, 128);
    // the staging thread of record k also needs the splat's rect and first
    // pair index (its emission index): loaded one batch ahead, with the records
    uint32_t pre_s = 0;
    uint64_t pre_rc = 0, pre_po = 0;
    auto prefetch_eidx = [&](int first, int cnt) {
      if (tid < cnt) {
        pre_s = pair_vals[rg.x + first + tid];
        pre_rc = rect[pre_s];
        pre_po = pair_off[pre_s];
      }
    };
    prefetch_eidx(b0, min(B, k_end - b0));
    // Two-buffer pipeline: threads [0, B) stage batch i while threads
    // [B, 2B) combine batch i-1 (its staged values and warp sums live in the
    // other buffer), so a batch costs two barriers instead of three.
    int buf = 0, cnb = 0;
    for (; b0 >= k0; b0 -= B) {
      const int nb = min(B, k_end - b0);
      records_wait(&s_bar, phase);
      if (tid < B) {
        const int k = tid;
        if (k < nb) {
          const SplatRec& r = s_raw[k];
          const Staged sg = stage_splat(r, cx, cy);
          s_a[buf][k] = sg.a;
          s_b[buf][k] = sg.b;
          s_n[buf][k] = sg.c;
          s_eidx[buf][k] = static_cast<uint32_t>(emission_index_of(pre_po, pre_rc, fd, n, pre_s, tile));
          uint32_t m = quad_mask(local_rect(r, tx * kTile, ty * kTile));
#if CGS_BWD_EIGEN_CULL
#pragma unroll
          for (int w = 0; w < 4; ++w) {  // quadrants the ellipse cannot reach
            const float x0 = (w & 1) * 8 - kTileHalf, y0 = (w >> 1) * 8 - kTileHalf;
            if ((m >> w) & 1u)
              if (!staged_may_hit(sg.a, sg.b, x0, x0 + 7.0f, y0, y0 + 7.0f)) m &= ~(1u << w);
          }
#endif
#pragma unroll
          for (int w = 0; w < 4; ++w)
            if (!(static_cast<uint32_t>(b0 + k) < s_wlast[w])) m &= ~(1u << w);
          s_mask[buf][k] = static_cast<uint8_t>(m);
        }
      } else if (tid - B < cnb) {
        combine_splat(buf ^ 1, tid - B);
      }
      __syncthreads();
      if (b0 > k0) {
        fence_proxy_async_smem();
        issue_records(s_raw, &s_bar, pair_vals, recs, rg.x + b0 - B, B, tid, 128);
        prefetch_eidx(b0 - B, B);
      }
      const int hits = warp_hit_list<B>(s_mask[buf], nb, warp, lane, my_list);
      // Hits in reverse order; two at a time (CGS_BWD_PAIR_REDUCE) the 18
      // values of both splats go through one transposed warp reduction (20
      // shuffles instead of 24).  The pixel updates stay sequential.
      auto hit_values = [&](int j, float* o) -> bool {
        const uint32_t k = static_cast<uint32_t>(b0 + j);
        const float4 a = s_a[buf][j];
        const float4 b = s_b[buf][j];
        const float2 nc = s_n[buf][j];
        const float t0 = staged_t(a, b, flx, fly);
        const float t1 = staged_t(a, b, flx, fly + 4.0f);
        const bool any = bwd_pixel(q0, k, t0, b.w, nc.x, nc.y, flx, fly, o);
        return bwd_pixel(q1, k, t1, b.w, nc.x, nc.y, flx, fly + 4.0f, o) || any;
      };
      int i = hits - 1;
      if (kBwdPairReduce && !TRACE) {
        for (; i >= 1; i -= 2) {
          const int ja = my_list[i], jb = my_list[i - 1];
          float o[18];
#pragma unroll
          for (int u = 0; u < 18; ++u) o[u] = 0.0f;
          bool any = hit_values(ja, o);
          any = hit_values(jb, o + 9) || any;
          float red = 0.0f;
          if (__any_sync(kFull, any)) red = warp_reduce_t<18>(o);
          if (slot18 >= 0) s_red[buf][warp][slot18 < 9 ? ja : jb][slot18 < 9 ? slot18 : slot18 - 9] = red;
        }
      }
      for (; i >= 0; --i) {
        const int j = my_list[i];
        float o[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) o[u] = 0.0f;
        const bool any = hit_values(j, o);
        if (TRACE && lane == 0)  // diagnostics: lanes with a contribution per warp hit
          atomicAdd(trace + 8 * static_cast<int64_t>(fd.total_tiles) + __popc(__ballot_sync(kFull, any)), 1ull);
        else if (TRACE) __ballot_sync(kFull, any);
        // lanes 0,2,4,8,10,16,18,20,24 end up holding the warp sums of values 0..8
        float red = 0.0f;
        if (__any_sync(kFull, any)) red = warp_reduce9(o);
        if (slot >= 0) s_red[buf][warp][j][slot] = red;
      }
      __syncthreads();
      cnb = nb;
      buf ^= 1;
    }
    if (tid >= B && tid - B < cnb) combine_splat(buf ^ 1, tid - B);  // the unit's last batch
  }
  if (TRACE && tid == 0) {
    unsigned long long* t = trace + 4 * (static_cast<int64_t>(fd.total_tiles) + blockIdx.x);
    t[0] = t_start;
    t[1] = global_ns();
    t[2] = smid();
    t[3] = static_cast<unsigned long long>(blockIdx.x);
  }
}


// ---------------------------------------------------------------------------
int launch_tile_order(const FrameDesc& fd, const FrameLayout& L, const uint32_t* nproc,
                      cudaStream_t st) {
  tile_order_kernel<<<1, 1024, 0, st>>>(L.ranges, nproc, fd.total_tiles, L.tile_order,
                                        nproc ? nullptr : L.tile_nproc,
                                        nproc ? nullptr : L.tile_last_dk,
                                        nproc ? nullptr : L.view_last_dk,
                                        fd.n_views > 0 ? fd.n_views : 1);
  CGS_CHECK_LAUNCH("tile_order_kernel");
  return CGS_OK;
}

int launch_raster_fwd(const FrameDesc& fd, const FrameLayout& L, const uint32_t* vals,
                      const float* logits, float* image, float* final_T, int32_t* counts,
                      cudaStream_t st) {
  // L.tile_order was computed from the list lengths before the depth sort
  // (tile_order_kernel also zeroed the per-tile and per-view maxima)
  CGS_PROFILED("raster_fwd_kernel", st,
               raster_fwd_kernel<<<fd.total_tiles, kFwdThreads, 0, st>>>(
                   fd, L.tile_order, L.ranges, vals, L.recs, L.hdr, image, final_T, counts,
                   L.px_last, L.tile_nproc, L.depth_key, L.tile_last_dk, L.tile_last_sid, L.view_last_dk, L.ckpt, L.refine_tiles,
                   L.refine_mask, tile_trace_buffer()));
  CGS_CHECK_LAUNCH("raster_fwd_kernel");
  {
    const int rc = launch_refine(false, fd, L, vals, logits, image, final_T, counts, nullptr,
                                 nullptr, st);
    if (rc) return rc;
  }
  return CGS_OK;
}

int launch_raster_bwd(const FrameDesc& fd, const FrameLayout& L, const float* final_T,
                      const float* dL, float* partials, unsigned long long* n_processed,
                      const float* logits, cudaStream_t st, void* zero_first, size_t zero_bytes,
                      void* zero_second, size_t zero_bytes2) {
  unit_order_kernel<<<1, 1024, 0, st>>>(L.tile_nproc, fd.total_tiles, L.units, L.unit_ctl,
                                        static_cast<uint32_t*>(zero_first),
                                        static_cast<int>(zero_bytes / sizeof(uint32_t)),
                                        static_cast<uint32_t*>(zero_second),
                                        static_cast<int>(zero_bytes2 / sizeof(uint32_t)));
  CGS_CHECK_LAUNCH("unit_order_kernel");
  // persistent grid: every resident CTA slot (per device ordinal)
  static std::atomic<int> resident_dev[kMaxDevices] = {};
  int dev = 0;
  if (int rc = current_device(&dev)) return rc;
  int resident = resident_dev[dev].load();
  if (resident == 0) {
    int sms = 0, per_sm = 0;
    CGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_bwd_kernel<false>, 128, 0));
    resident = sms * (per_sm > 0 ? per_sm : 1);
    resident_dev[dev].store(resident);
  }
  const int grid = static_cast<int>(L.n_ckpt < resident ? L.n_ckpt : resident);
  unsigned long long* trace = tile_trace_buffer();
  auto kern = trace ? raster_bwd_kernel<true> : raster_bwd_kernel<false>;
  CGS_PROFILED("raster_bwd_kernel", st,
               kern<<<grid, 128, 0, st>>>(fd, L.units, L.unit_ctl, L.ranges, sorted_pair_vals(L),
                                          L.recs, L.hdr, L.px_last, L.tile_nproc, final_T, dL,
                                          L.ckpt, L.pair_off, L.rect, L.n, partials,
                                          8 * (L.pair_cap > 0 ? L.pair_cap : 1), n_processed,
                                          trace));
  CGS_CHECK_LAUNCH("raster_bwd_kernel");
  return launch_refine(true, fd, L, sorted_pair_vals(L), logits, nullptr, nullptr, nullptr, dL,
                       partials, st);
}
}  // namespace cgs
