// Frame workspace layout shared by the forward and backward render paths.
#pragma once

#include "common.cuh"
#include "sort_scan.cuh"

namespace cgs {

// Pixels the fp32 raster flags (a value inside a decision band, see
// raster_common.cuh) are re-walked in float64 (refine.cu); px_last of such a
// pixel carries kRefinedBit.
constexpr uint32_t kRefinedBit = 0x80000000u;
struct RefinePx {  // float64 result of a re-walked pixel (forward -> backward)
  double C[3];
  double T;
  uint32_t last;
  uint32_t pad;
};

// Splats with more tile pairs than this (near-plane giants cover every tile)
// are emitted and reduced by a whole CTA each, from a list built during
// emission, instead of by the warp that owns their depth rank.
constexpr uint32_t kLongSplat = 256;

// The backward splits a tile's processed prefix into chunks of kChunk splats
// (independent CTAs); the forward leaves each pixel's transmittance and
// colour suffix at every chunk boundary it passes (ckpt).  kChunk is a
// multiple of the forward's 256-splat batch.
#ifndef CGS_CHUNK
#define CGS_CHUNK 256
#endif
constexpr int kChunk = CGS_CHUNK;

// Checkpoint slot of boundary j >= 1 (splat index j * kChunk) of a tile whose
// list starts at pair position `start`: distinct over all (tile, j) with
// j * kChunk < list length, and < total_tiles + pair_cap / kChunk + 1.
__host__ __device__ __forceinline__ int64_t ckpt_slot(uint32_t start, int tile, int j) {
  return static_cast<int64_t>(start / kChunk) + tile + (j - 1);
}

#ifndef CGS_ONESWEEP_TILE_SORT  // 1: always the two-pass onesweep tile sort (comparisons)
#define CGS_ONESWEEP_TILE_SORT 0
#endif
constexpr bool kForceOnesweepTileSort = CGS_ONESWEEP_TILE_SORT != 0;

struct FrameLayout {
  FrameHeader* hdr;
  SplatRec* recs;          // V*N
  uint64_t* depth_key;     // V*N (f64 bits of camera z)
  uint32_t* dkey;          // V*N 32-bit depth sort keys
  uint32_t* dval;          // V*N depth sort payload (splat ids); depth rank -> splat
  SortWs<uint32_t> dsort;  // depth sort (result: depth_perm)
  uint32_t* n_tiles;       // V*N
  uint64_t* rect;          // V*N packed tile rect
  uint64_t* pair_off;      // V*N per splat: first emission index of its pairs
  uint64_t* off_rank;      // the same by depth rank (N_s; the emission reads it coalesced)
  uint32_t* tie_runs;      // starts of equal-depth-key runs longer than 256 (count: hdr->scratch[1])
  void* pkeys;             // pair_cap tile keys (u16 or u32)
  uint32_t* pvals;         // pair_cap splat ids
  SortWs<uint16_t> psort16;
  SortWs<uint32_t> psort32;
  // total_tiles: (fp64 depth bits, splat id) of the tile's last processed
  // splat -- the depth order's key, so splat s is in the tile's processed
  // prefix iff (depth_key[s], s) <= it; (0, 0): none processed
  uint64_t* tile_last_dk;
  uint32_t* tile_last_sid;
  // n_views: the largest tile_last_dk of the view -- a splat deeper than it
  // is in no tile's processed prefix (the pair walk skips it)
  unsigned long long* view_last_dk;
  uint32_t* long_list;     // V*N: splats with more than kLongSplat pairs (count: hdr->scratch[2])
  uint2* ranges;           // total_tiles [start, end)
  uint32_t* px_last;       // total_pixels
  uint32_t* tile_nproc;    // total_tiles
  uint32_t* tile_order;    // total_tiles: raster CTA -> tile, longest work first
  float4* ckpt;            // n_ckpt x 256: per-pixel (T, colour suffix) at chunk boundaries
  uint32_t* refine_tiles;  // total_tiles: tiles with pixels to re-walk in float64 (count: hdr->scratch[3])
  uint32_t* refine_mask;   // 8 x total_tiles: per-warp masks of those pixels
  uint32_t* refine_off;    // total_tiles: first RefinePx entry of each listed tile
  RefinePx* refine_px;     // refine_px_cap float64 results of re-walked pixels
  int64_t refine_px_cap;
  uint2* units;            // n_ckpt: backward work units (tile, chunk), longest first
  uint32_t* unit_ctl;      // [0] unit count, [1] fetch counter
  int64_t n_ckpt;
  ScanWs scan;
  double* sr_cov;          // sr_cap * 8 (Sigma3 + zero-quaternion flag)
  size_t bytes;
  int64_t n, vn, pair_cap;
  int tile_key_bytes;      // 2 or 4
  int tile_key_bits;
  int pair_result_alt;     // 1 if the tile-sorted pairs live in the sort's alt buffers
  // One-pass counting tile sort (tile_count / matrix scan / tile_scatter,
  // render_fwd.cu) for frames of at most kCountMaxTiles tiles: chunk c of
  // 2^count_log2 pairs, tile t -> tcount[t * C + c], C = live chunks.
  int count_sort;
  int count_log2;
  int64_t count_chunks_cap;
  uint32_t* tcount;            // total_tiles x count_chunks_cap
  uint32_t* toff;              // count_chunks_cap x total_tiles (scan result, chunk-major)
  unsigned long long* tcount_n;  // total_tiles x live chunks (the matrix scan's length)
  ScanWs tscan;
  // set by frame_stage_project when sr_precompute zeroed the depth sort's and
  // the scans' states (host-side flag: the stages run in order on one stream)
  bool states_zeroed = false;
};

// Counting tile sort limits: the scatter keeps a u16 counter per (warp,
// tile) plus a u32 offset per tile in shared memory (20 B per tile, and 2 KB
// of duplicate-test tags per warp), and its
// chunk prefix over 8 warps must fit u16 (chunks <= 32768 pairs).
constexpr int kCountWarps = 8;
constexpr int kCountMaxTiles = 10496;  // (20 B per tile + 16 KB) <= 227 KB
constexpr int kCountMaxLog2 = 15;
inline int count_chunk_log2(int tiles) {  // >= 4 pairs per tile and chunk, 4096 .. 32768
  int l = 12;
  while (l < kCountMaxLog2 && (1LL << l) < 4LL * tiles) ++l;
  return l;
}

// Depth sort keys (project_kernel): 24 bits, 3 onesweep passes (an odd pass
// count leaves the sorted splat ids in the sort's alternate value buffer);
// depth_tie_fix_kernel writes the final order back into dval.
constexpr int kDepthPasses = 3;
constexpr uint32_t kDepthKeyBase = 0x3C23D70Au;  // fp32 bits of kNear = 0.01 rounded toward zero
constexpr int kDepthKeyShift = 4;
constexpr uint32_t kDepthKeyMax = (1u << (8 * kDepthPasses)) - 1u;
inline uint32_t* depth_perm(const FrameLayout& L) { return L.dval; }

inline int bits_for(int64_t v) {
  int b = 1;
  while ((1LL << b) < v) ++b;
  return b;
}

inline FrameDesc make_frame_desc(const cgs_camera_t* cams, int n_views) {
  FrameDesc fd{};
  fd.n_views = n_views;
  int tiles = 0;
  int64_t pix = 0;
  for (int v = 0; v < n_views; ++v) {
    CamDev& c = fd.cam[v];
    for (int k = 0; k < 9; ++k) c.R[k] = cams[v].R[k];
    for (int k = 0; k < 3; ++k) c.t[k] = cams[v].t[k];
    c.fx = cams[v].fx; c.fy = cams[v].fy; c.cx = cams[v].cx; c.cy = cams[v].cy;
    // center = -R^T t (camera.py:34-36)
    for (int j = 0; j < 3; ++j)
      c.center[j] = -(c.R[0 * 3 + j] * c.t[0] + c.R[1 * 3 + j] * c.t[1] + c.R[2 * 3 + j] * c.t[2]);
    c.width = cams[v].width;
    c.height = cams[v].height;
    c.ntx = (c.width + kTile - 1) / kTile;
    c.nty = (c.height + kTile - 1) / kTile;
    c.tile_base = tiles;
    c.pix_base = pix;
    tiles += c.ntx * c.nty;
    pix += static_cast<int64_t>(c.width) * c.height;
  }
  fd.total_tiles = tiles;
  fd.total_pixels = pix;
  return fd;
}

inline FrameLayout plan_frame(void* base, size_t cap_bytes, int64_t n, const FrameDesc& fd,
                              int64_t pair_cap, int64_t sr_cap) {
  FrameLayout L{};
  Carver c(base, cap_bytes);
  const int64_t vn = n * fd.n_views;
  const int64_t vn1 = vn > 0 ? vn : 1;
  const int64_t pc = pair_cap > 0 ? pair_cap : 1;
  L.n = n;
  L.vn = vn;
  L.pair_cap = pair_cap;
  L.tile_key_bytes = fd.total_tiles <= 65535 ? 2 : 4;
  L.tile_key_bits = bits_for(fd.total_tiles + 1);
  L.hdr = c.take<FrameHeader>(1);
  L.recs = c.take<SplatRec>(vn1);
  L.depth_key = c.take<uint64_t>(vn1);
  L.dkey = c.take<uint32_t>(vn1);
  L.dval = c.take<uint32_t>(vn1);
  L.dsort = carve_sort<uint32_t>(c, vn1);
  L.n_tiles = c.take<uint32_t>(vn1);
  L.rect = c.take<uint64_t>(vn1);
  L.pair_off = c.take<uint64_t>(vn1);
  L.off_rank = c.take<uint64_t>(vn1);
  L.tie_runs = c.take<uint32_t>(vn1 / 256 + 16);
  if (L.tile_key_bytes == 2) {
    L.pkeys = c.take<uint16_t>(pc);
    L.psort16 = carve_sort<uint16_t>(c, pc);
  } else {
    L.pkeys = c.take<uint32_t>(pc);
    L.psort32 = carve_sort<uint32_t>(c, pc);
  }
  L.pvals = c.take<uint32_t>(pc);
  L.count_sort = (L.tile_key_bytes == 2 && fd.total_tiles > 0 && fd.total_tiles <= kCountMaxTiles &&
                  !kForceOnesweepTileSort) ? 1 : 0;
  if (L.count_sort) {
    L.count_log2 = count_chunk_log2(fd.total_tiles);
    L.count_chunks_cap = (pc + (1LL << L.count_log2) - 1) >> L.count_log2;
    L.tcount = c.take<uint32_t>(static_cast<size_t>(fd.total_tiles) * L.count_chunks_cap);
    L.toff = c.take<uint32_t>(static_cast<size_t>(fd.total_tiles) * L.count_chunks_cap);
    L.tcount_n = c.take<unsigned long long>(1);
    L.tscan = carve_scan(c, static_cast<int64_t>(fd.total_tiles) * L.count_chunks_cap);
  }
  L.long_list = c.take<uint32_t>(vn1);
  L.ranges = c.take<uint2>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.px_last = c.take<uint32_t>(fd.total_pixels > 0 ? fd.total_pixels : 1);
  L.tile_nproc = c.take<uint32_t>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.tile_last_dk = c.take<uint64_t>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.tile_last_sid = c.take<uint32_t>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.view_last_dk = c.take<unsigned long long>(fd.n_views > 0 ? fd.n_views : 1);
  L.tile_order = c.take<uint32_t>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.n_ckpt = fd.total_tiles + pc / kChunk + 2;
  L.ckpt = c.take<float4>(L.n_ckpt * 256);
  L.refine_tiles = c.take<uint32_t>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.refine_mask = c.take<uint32_t>(8 * static_cast<int64_t>(fd.total_tiles > 0 ? fd.total_tiles : 1));
  L.refine_off = c.take<uint32_t>(fd.total_tiles > 0 ? fd.total_tiles : 1);
  L.refine_px_cap = fd.total_pixels / 64 + 16384;
  L.refine_px = c.take<RefinePx>(L.refine_px_cap);
  L.units = c.take<uint2>(L.n_ckpt);
  L.unit_ctl = c.take<uint32_t>(2);
  L.scan = carve_scan(c, vn1 > fd.total_tiles ? vn1 : fd.total_tiles);
  L.sr_cov = c.take<double>((sr_cap > 0 ? sr_cap : 1) * 8);
  L.bytes = c.off + 256;
  const int ppasses = (L.tile_key_bits + 7) / 8;
  L.pair_result_alt = L.count_sort ? 1 : (ppasses % 2) == 1;  // the scatter writes vals_alt
  return L;
}

// Final (tile, depth)-ordered splat ids of the pairs.
inline uint32_t* sorted_pair_vals(const FrameLayout& L) {
  if (!L.pair_result_alt) return L.pvals;
  return L.tile_key_bytes == 2 ? L.psort16.vals_alt : L.psort32.vals_alt;
}

// Raster launches (raster.cu).  tile_order: CTA -> tile, longest work first
// (work = list length when nproc is null, else the processed prefix).
int launch_tile_order(const FrameDesc& fd, const FrameLayout& L, const uint32_t* nproc,
                      cudaStream_t st);
int launch_raster_fwd(const FrameDesc& fd, const FrameLayout& L, const uint32_t* vals,
                      const float* logits, float* image, float* final_T, int32_t* counts,
                      cudaStream_t st);
// Float64 re-walk of the flagged pixels (refine.cu): bwd = false rewrites
// their forward outputs; bwd = true adds their gradient terms to the pairs'
// partials after raster_bwd (which skips them).
int launch_refine(bool bwd, const FrameDesc& fd, const FrameLayout& L, const uint32_t* vals,
                  const float* logits, float* image, float* final_T, int32_t* counts,
                  const float* dL, float* partials, cudaStream_t st);
int launch_raster_bwd(const FrameDesc& fd, const FrameLayout& L, const float* final_T,
                      const float* dL, float* partials, unsigned long long* n_processed,
                      const float* logits, cudaStream_t st, void* zero_first = nullptr,
                      size_t zero_bytes = 0, void* zero_second = nullptr,
                      size_t zero_bytes2 = 0);

// Emission index of pair (splat s, tile t): pairs of a splat are emitted in
// row-major order over its tile rect starting at pair_off[s].
__device__ __forceinline__ uint64_t emission_index_of(uint64_t po, uint64_t rc, const FrameDesc& fd,
                                                      int64_t n, uint32_t s, int tile) {
  const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
  const int ty0 = static_cast<int>((rc >> 32) & 0xffff);
  const int v = static_cast<int>(s / static_cast<uint32_t>(n));
  const int lt = tile - fd.cam[v].tile_base;
  const int ty = lt / fd.cam[v].ntx, tx = lt - ty * fd.cam[v].ntx;
  return po + static_cast<uint64_t>((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
}
__device__ __forceinline__ uint64_t emission_index(const uint64_t* pair_off, const uint64_t* rect,
                                                   const FrameDesc& fd, int64_t n, uint32_t s,
                                                   int tile) {
  const uint64_t rc = rect[s];
  const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
  const int ty0 = static_cast<int>((rc >> 32) & 0xffff);
  const int v = static_cast<int>(s / static_cast<uint32_t>(n));
  const int lt = tile - fd.cam[v].tile_base;
  const int ty = lt / fd.cam[v].ntx, tx = lt - ty * fd.cam[v].ntx;
  return pair_off[s] + static_cast<uint64_t>((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
}

}  // namespace cgs
