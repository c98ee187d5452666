// Tile rasterizer kernels, forward and backward (reference render.py:265-377).
//
// Forward: one CTA per 16x16 tile, 256 threads, one pixel each, warp w on
// the 8x4 block ((w & 1) * 8, (w >> 1) * 4).  Backward: persistent CTAs of
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
#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

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
                                                          uint32_t* __restrict__ zero_b) {
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
    for (int t = tid; t < total_tiles; t += blockDim.x) zero_a[t] = zero_b[t] = 0u;
}

struct PixState {
  float T, r, g, b;
  int cnt;
  uint32_t last;
  bool done;
};

// Front-to-back blend of one splat into one pixel (render.py:274-283, 302-311).
__device__ __forceinline__ void blend(PixState& p, float al, float cr, float cg, float cb,
                                      uint32_t idx) {
  if (p.done || !(al >= kAlphaSkipF)) return;
  const float w = al * p.T;
  p.r = fmaf(w, cr, p.r);
  p.g = fmaf(w, cg, p.g);
  p.b = fmaf(w, cb, p.b);
  p.T = p.T * (1.0f - al);
  ++p.cnt;
  if (!(p.T >= kTMinF)) {  // every later splat is inactive (T_before < 1e-4)
    p.done = true;
    p.last = idx + 1;
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

// HALVES = 2 splits every tile over two CTAs of 128 threads (rows 0-7 and
// 8-15, batches of 128 splats): a tile's blend is sequential in its list, so
// one CTA per tile makes the longest list the kernel's floor; two CTAs halve
// it for the price of staging each record twice.  Per-tile results (processed
// count, last rank) are combined with atomicMax (zeroed by tile_order_kernel).
#ifndef CGS_FWD_PAIRS
#define CGS_FWD_PAIRS 1
#endif
#ifndef CGS_FWD_HALVES
#define CGS_FWD_HALVES 1
#endif
#ifndef CGS_FWD_MINB
#define CGS_FWD_MINB (CGS_FWD_HALVES == 2 ? 12 : 6)
#endif
constexpr int kFwdHalves = CGS_FWD_HALVES;
constexpr int kFwdThreads = 256 / kFwdHalves;  // one pixel per thread
constexpr int kFwdBatch = 256 / kFwdHalves;
constexpr int kFwdWarps = kFwdThreads / 32;
static_assert(kChunk % kFwdBatch == 0, "checkpoints sit on batch boundaries");

__global__ void __launch_bounds__(kFwdThreads, CGS_FWD_MINB) raster_fwd_kernel(
    FrameDesc fd, const uint32_t* __restrict__ order, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ pair_vals, const SplatRec* __restrict__ recs,
    const FrameHeader* __restrict__ hdr, float* __restrict__ image,
    float* __restrict__ final_T, int32_t* __restrict__ counts, uint32_t* __restrict__ px_last,
    uint32_t* __restrict__ tile_nproc, const uint32_t* __restrict__ rank_of,
    uint32_t* __restrict__ last_rank, float4* __restrict__ ckpt,
    unsigned long long* __restrict__ trace) {
  constexpr int B = kFwdBatch, NT = kFwdThreads;
  const unsigned long long t_start = trace ? global_ns() : 0ull;
  __shared__ __align__(128) SplatRec s_raw[B];
  __shared__ float4 s_a[B];
  __shared__ float4 s_b[B];
  __shared__ float2 s_c[B];
  __shared__ uint8_t s_mask[B];
  __shared__ uint8_t s_list[kFwdWarps][B];
  __shared__ uint32_t s_max[kFwdWarps];
  __shared__ __align__(8) uint64_t s_bar;
  if (hdr->stats.overflow) return;
  const int half = kFwdHalves == 2 ? static_cast<int>(blockIdx.x & 1u) : 0;
  const int tile = static_cast<int>(order[blockIdx.x / kFwdHalves]);
  int v = 0;
  while (v + 1 < fd.n_views && fd.cam[v + 1].tile_base <= tile) ++v;
  const CamDev& cam = fd.cam[v];
  const int lt = tile - cam.tile_base;
  const int ty = lt / cam.ntx, tx = lt - ty * cam.ntx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wb = warp + half * kFwdWarps;  // 8x4 block index within the tile
  const int lx = (wb & 1) * 8 + (lane & 7), ly = (wb >> 1) * 4 + (lane >> 3);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool in = px < cam.width && py < cam.height;
  const uint2 rg = ranges[tile];
  const int n = static_cast<int>(rg.y - rg.x);
  const double ox = static_cast<double>(tx * kTile), oy = static_cast<double>(ty * kTile);
  const float flx = static_cast<float>(lx), fly = static_cast<float>(ly);
  uint8_t* my_list = s_list[warp];
  PixState p{1.0f, 0.0f, 0.0f, 0.0f, 0, 0u, !in};
  int n_ckpt = 0;

  if (tid == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  bool pending = false;
  if (n > 0) {
    issue_records(s_raw, &s_bar, pair_vals, recs, rg.x, min(B, n), tid, NT);
    pending = true;
  }
  for (int b0 = 0; b0 < n; b0 += B) {
    const int nb = min(B, n - b0);
    mbar_wait(&s_bar, phase);
    phase ^= 1;
    pending = false;
    if (tid < nb) {
      const Staged sg = stage_splat(s_raw[tid], ox, oy);
      s_a[tid] = sg.a;
      s_b[tid] = sg.b;
      s_c[tid] = sg.c;
      const uint32_t m8 = block8x4_mask(local_rect(s_raw[tid], tx * kTile, ty * kTile));
      s_mask[tid] = static_cast<uint8_t>(m8 >> (half * kFwdWarps));
    }
    __syncthreads();
    if (b0 + B < n) {
      fence_proxy_async_smem();
      issue_records(s_raw, &s_bar, pair_vals, recs, rg.x + b0 + B, min(B, n - b0 - B), tid, NT);
      pending = true;
    }
    const int hits = warp_hit_list<B>(s_mask, nb, warp, lane, my_list);
    if (!p.done) {
#if CGS_FWD_PAIRS
      // two hits per iteration: both alphas are independent of the blend
      // state, so they issue together; the blends stay in list order
      int i = 0;
      for (; i + 1 < hits; i += 2) {
        const int j0 = my_list[i], j1 = my_list[i + 1];
        const float4 a0 = s_a[j0], b0v = s_b[j0];
        const float4 a1 = s_a[j1], b1v = s_b[j1];
        float u, v;
        const float al0 = staged_alpha(a0, b0v, flx, fly, u, v);
        const float al1 = staged_alpha(a1, b1v, flx, fly, u, v);
        if (al0 >= kAlphaSkipF) {
          const float2 c = s_c[j0];
          blend(p, al0, b0v.w, c.x, c.y, static_cast<uint32_t>(b0 + j0));
          if (p.done) break;
        }
        if (al1 >= kAlphaSkipF) {
          const float2 c = s_c[j1];
          blend(p, al1, b1v.w, c.x, c.y, static_cast<uint32_t>(b0 + j1));
          if (p.done) break;
        }
      }
      if (!p.done && i < hits) {
        const int j = my_list[i];
        const float4 a = s_a[j];
        const float4 b = s_b[j];
        float u, v;
        const float al = staged_alpha(a, b, flx, fly, u, v);
        if (al >= kAlphaSkipF) {
          const float2 c = s_c[j];
          blend(p, al, b.w, c.x, c.y, static_cast<uint32_t>(b0 + j));
        }
      }
#else
      for (int i = 0; i < hits; ++i) {
        const int j = my_list[i];
        const float4 a = s_a[j];
        const float4 b = s_b[j];
        float u, v;
        const float al = staged_alpha(a, b, flx, fly, u, v);
        if (al >= kAlphaSkipF) {
          const float2 c = s_c[j];
          blend(p, al, b.w, c.x, c.y, static_cast<uint32_t>(b0 + j));
          if (p.done) break;
        }
      }
#endif
    }
    if (__syncthreads_count(p.done) == NT) break;
    if (b0 + B < n && ((b0 + B) % kChunk) == 0) {  // chunk boundary for the backward
      // T after the chunk and the chunk's own colour sum; colour restarts at 0
      ckpt[ckpt_slot(rg.x, tile, (b0 + B) / kChunk) * kTilePixels + ly * kTile + lx] =
          make_float4(p.T, p.r, p.g, p.b);
      p.r = p.g = p.b = 0.0f;
      ++n_ckpt;
    }
  }
  if (pending) mbar_wait(&s_bar, phase);
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
  if (in && !p.done) p.last = static_cast<uint32_t>(n);
  if (in) {
    const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
    image[3 * pix + 0] = p.r;
    image[3 * pix + 1] = p.g;
    image[3 * pix + 2] = p.b;
    final_T[pix] = p.T;
    counts[pix] = p.cnt;
    px_last[pix] = p.last;
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
    const uint32_t lr = np ? rank_of[pair_vals[rg.x + np - 1]] + 1 : 0u;  // ranks grow along the list
    if (kFwdHalves == 1) {
      tile_nproc[tile] = np;
      last_rank[tile] = lr;
    } else {
      atomicMax(&tile_nproc[tile], np);
      atomicMax(&last_rank[tile], lr);
    }
    if (trace) {
      unsigned long long* t = trace + 4 * static_cast<int64_t>(blockIdx.x / kFwdHalves);
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
  float T, gr, gg, gb, sr, sg, sb;
  uint32_t last;
};

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Adds pixel p's contribution of splat k to o[9]; returns whether it had one.
// o = [sum w g (3), sum dp, sum dp u, sum dp v, sum dp u^2, sum dp u v,
// sum dp v^2] with dp = dL/dalpha * alpha and (u, v) the pixel offset in the
// conic's eigenbasis (passed as dx, dy): the per-splat gradient is a linear
// map of these moments (moments_to_grad), applied once per splat after the
// pixel sums instead of per pixel.
__device__ __forceinline__ bool bwd_pixel(PixBwd& p, uint32_t k, float al, float cr, float cg,
                                          float cb, float dx, float dy, float* o) {
  if (!(k < p.last) || !(al >= kAlphaSkipF)) return false;
  const float iom = fast_rcp(1.0f - al);  // 1 - alpha >= 0.01
  const float Tb = p.T * iom;
  const float w = al * Tb;
  o[0] = fmaf(w, p.gr, o[0]);  // d colour += weight * dL (render.py:351-352)
  o[1] = fmaf(w, p.gg, o[1]);
  o[2] = fmaf(w, p.gb, o[2]);
  // dC/dalpha = c T_before - suffix / (1 - alpha) (render.py:357-359)
  const float dCr = fmaf(cr, Tb, -p.sr * iom);
  const float dCg = fmaf(cg, Tb, -p.sg * iom);
  const float dCb = fmaf(cb, Tb, -p.sb * iom);
  const float da = dCr * p.gr + dCg * p.gg + dCb * p.gb;
  p.sr = fmaf(w, cr, p.sr);
  p.sg = fmaf(w, cg, p.sg);
  p.sb = fmaf(w, cb, p.sb);
  p.T = Tb;
  if (al < kAlphaClampVal) {  // no gradient through the clamp (render.py:361)
    const float dp = da * al;
    const float tx = dp * dx, ty = dp * dy;
    o[3] += dp;
    o[4] += tx;
    o[5] += ty;
    o[6] = fmaf(tx, dx, o[6]);
    o[7] = fmaf(tx, dy, o[7]);
    o[8] = fmaf(ty, dy, o[8]);
  }
  return true;
}

// Moments -> [d colour (3), d opacity, d mean2d (2), d conic (A, B, C)]
// (render.py:364-377: d_opac = sum dp / o, d_mean = sum dp Q d,
// d_conic = -(1/2 dx^2, dx dy, 1/2 dy^2) summed with weight dp), with
// d = u e1 + v e2 and Q d = lambda1 u e1 + lambda2 v e2; in fp64.
__device__ __forceinline__ void moments_to_grad(const float* m, float e1x, float e1y, float l1,
                                                float l2, float io, float* g) {
  const double ex = e1x, ey = e1y;
  g[0] = m[0];
  g[1] = m[1];
  g[2] = m[2];
  g[3] = m[3] * io;
  const double a = static_cast<double>(l1) * m[4], b = static_cast<double>(l2) * m[5];
  g[4] = static_cast<float>(a * ex - b * ey);
  g[5] = static_cast<float>(a * ey + b * ex);
  const double uu = m[6], uv = m[7], vv = m[8];
  const double xx = ex * ex * uu - 2.0 * ex * ey * uv + ey * ey * vv;
  const double xy = ex * ey * uu + (ex * ex - ey * ey) * uv - ex * ey * vv;
  const double yy = ey * ey * uu + 2.0 * ex * ey * uv + ex * ex * vv;
  g[6] = static_cast<float>(-0.5 * xx);
  g[7] = static_cast<float>(-xy);
  g[8] = static_cast<float>(-0.5 * yy);
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
static_assert(kBwdBatch % 32 == 0 && kChunk % kBwdBatch == 0 && kBwdBatch <= 256,
              "batch: whole ballots, whole batches per chunk, u8 hit-list entries");

// Backward work units: chunk c of tile t covers splats [c kChunk, min((c+1)
// kChunk, nproc_t)).  Sorted by length, longest first (counting sort in one
// CTA, as tile_order_kernel); ctl[0] = unit count, ctl[1] = fetch counter.
__global__ void __launch_bounds__(1024) unit_order_kernel(const uint32_t* __restrict__ nproc,
                                                          int total_tiles,
                                                          uint2* __restrict__ units,
                                                          uint32_t* __restrict__ ctl) {
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
  __shared__ float4 s_n[2][B];  // green, blue, lambda1, lambda2
  __shared__ float s_io[2][B];  // 1 / opacity
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
  const float flx = static_cast<float>(lx), fly = static_cast<float>(ly);
  const int slot = reduce9_slot(lane);
  uint8_t* my_list = s_list[warp];
  const uint32_t n_units = unit_ctl[0];
  // splat jj of buffer cb: sum the present warps in fixed order, chain to the
  // 9 gradients, store at the pair's emission index (values 0-7 as two
  // aligned float4, value 8 in the separate array after them)
  auto combine_splat = [&](int cb, int jj) {
    const uint32_t m = s_mask[cb][jj];
    float mom[9], g[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const float r0 = (m & 1u) ? s_red[cb][0][jj][u] : 0.0f;
      const float r1 = (m & 2u) ? s_red[cb][1][jj][u] : 0.0f;
      const float r2 = (m & 4u) ? s_red[cb][2][jj][u] : 0.0f;
      const float r3 = (m & 8u) ? s_red[cb][3][jj][u] : 0.0f;
      mom[u] = (r0 + r1) + (r2 + r3);
    }
    const float4 aa = s_a[cb][jj];
    const float4 nn = s_n[cb][jj];
    moments_to_grad(mom, aa.z, aa.w, nn.z, nn.w, s_io[cb][jj], g);
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
    const double ox = static_cast<double>(tx * kTile), oy = static_cast<double>(ty * kTile);
    const bool last_chunk = k_end == nproc;
    const float4* ck = last_chunk ? nullptr
                                  : ckpt + ckpt_slot(rg.x, tile, k_end / kChunk) * kTilePixels;

    PixBwd q0{1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0u};
    PixBwd q1 = q0;
    auto load_px = [&](PixBwd& q, int py, int lyy) {
      if (px < cam.width && py < cam.height) {
        const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
        q.last = px_last[pix];
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
          q.sr = c.y;
          q.sg = c.z;
          q.sb = c.w;
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
    // Two-buffer pipeline: threads [0, B) stage batch i while threads
    // [B, 2B) combine batch i-1 (its staged values and warp sums live in the
    // other buffer), so a batch costs two barriers instead of three.
    int buf = 0, cnb = 0;
    for (; b0 >= k0; b0 -= B) {
      const int nb = min(B, k_end - b0);
      mbar_wait(&s_bar, phase);
      phase ^= 1;
      if (tid < B) {
        const int k = tid;
        if (k < nb) {
          const SplatRec& r = s_raw[k];
          const Staged sg = stage_splat(r, ox, oy);
          s_a[buf][k] = sg.a;
          s_b[buf][k] = sg.b;
          s_n[buf][k] = make_float4(sg.c.x, sg.c.y, sg.lam1, sg.lam2);
          s_io[buf][k] = 1.0f / r.opac;
          s_eidx[buf][k] = static_cast<uint32_t>(
              emission_index(pair_off, rect, fd, n, pair_vals[rg.x + b0 + k], tile));
          uint32_t m = quad_mask(local_rect(r, tx * kTile, ty * kTile));
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
      }
      const int hits = warp_hit_list<B>(s_mask[buf], nb, warp, lane, my_list);
      for (int i = hits - 1; i >= 0; --i) {
        const int j = my_list[i];
        const uint32_t k = static_cast<uint32_t>(b0 + j);
        float o[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) o[u] = 0.0f;
        const float4 a = s_a[buf][j];
        const float4 b = s_b[buf][j];
        const float4 nc = s_n[buf][j];
        float u0, v0, u1, v1;
        const float al0 = staged_alpha(a, b, flx, fly, u0, v0);
        const float al1 = staged_alpha(a, b, flx, fly + 4.0f, u1, v1);
        bool any = bwd_pixel(q0, k, al0, b.w, nc.x, nc.y, u0, v0, o);
        any = bwd_pixel(q1, k, al1, b.w, nc.x, nc.y, u1, v1, o) || any;
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
                                        nproc ? nullptr : L.last_rank);
  CGS_CHECK_LAUNCH("tile_order_kernel");
  return CGS_OK;
}

int launch_raster_fwd(const FrameDesc& fd, const FrameLayout& L, const uint32_t* vals,
                      float* image, float* final_T, int32_t* counts, cudaStream_t st) {
  // L.tile_order was computed from the list lengths before the depth sort
  CGS_PROFILED("raster_fwd_kernel", st,
               raster_fwd_kernel<<<fd.total_tiles * kFwdHalves, kFwdThreads, 0, st>>>(
                   fd, L.tile_order, L.ranges, vals,
                                                                 L.recs, L.hdr,
                                                                 image, final_T, counts, L.px_last,
                                                                 L.tile_nproc, L.rank_of,
                                                                 L.last_rank, L.ckpt,
                                                                 tile_trace_buffer()));
  CGS_CHECK_LAUNCH("raster_fwd_kernel");
  return CGS_OK;
}

int launch_raster_bwd(const FrameDesc& fd, const FrameLayout& L, const float* final_T,
                      const float* dL, float* partials, unsigned long long* n_processed,
                      cudaStream_t st) {
  unit_order_kernel<<<1, 1024, 0, st>>>(L.tile_nproc, fd.total_tiles, L.units, L.unit_ctl);
  CGS_CHECK_LAUNCH("unit_order_kernel");
  static int resident = 0;  // persistent grid: every resident CTA slot
  if (resident == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    CGS_CUDA(cudaGetDevice(&dev));
    CGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_bwd_kernel<false>, 128, 0));
    resident = sms * (per_sm > 0 ? per_sm : 1);
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
  return CGS_OK;
}
}  // namespace cgs
