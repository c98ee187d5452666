// Float64 re-walk of the pixels the fp32 raster cannot decide exactly.
//
// raster_fwd_kernel flags a pixel whose fp32 transmittance came within kTBand
// (relative) of the 1e-4 termination threshold, or that met an fp32 alpha
// within kAlphaBand of 1/255 or 0.99 (raster_common.cuh).  Those pixels are
// recomputed here exactly as the reference computes them (render.py:265-311,
// float64): alpha from the float64 mean / conic / sigmoid(logit) in numpy's
// operation order, kept at 1/255, composited while T_before >= 1e-4.
//
// One CTA per listed tile; the tile's flagged pixels are walked one after the
// other, each by the whole CTA, over the tile list in chunks of kRefChunk
// records.  Per chunk the records whose contribution box holds the pixel are
// compacted in list order (outside its box a record's float64 alpha is below
// 1/255, so it is never kept -- projection builds the boxes for exactly that);
// only those -- typically a tenth of the list -- are evaluated: their alphas
// do not depend on the pixel's state, so they are computed in parallel, the
// transmittance before each is the product of the earlier factors (a block
// scan in list order), and the first record after which T < 1e-4 is the last
// one the pixel composites.  A pixel's state between chunks (T, colour,
// count, last) lives in shared memory.
//
//   forward  (refine_kernel<false>, after raster_fwd_kernel): rewrites the
//            pixel's image, final T, contribution count and last index
//            (px_last | kRefinedBit), raises the tile's processed prefix if
//            the pixel goes further, and stores its float64 colour
//            (RefinePx) for the backward.
//   backward (refine_kernel<true>, after raster_bwd_kernel, which skips
//            refined pixels): the same walk with suffix = C - prefix
//            (render.py:354-359) gives each (pixel, record) term of
//            raster_bwd_kernel's 9 tile sums (local moments), added to the
//            pair's partial by the thread that owns the record; pixels are
//            walked in a fixed order with barriers in between, so the
//            backward stays deterministic.
#include <atomic>

#include "frame.cuh"
#include "raster_common.cuh"

namespace cgs {

namespace {

// 128 threads x 6 records (768-record chunks; 4 CTAs per SM): config 3
// (short walks -- its pixels end after ~60 splats -- in ~1500 tiles) 149 ->
// 115 us for both kernels, config 1 (walks of ~1000) unchanged; 256 x 4 and
// 128 x 4 / 128 x 8 measured worse on one or the other
#ifndef CGS_REF_THREADS
#define CGS_REF_THREADS 128
#endif
constexpr int kThreads = CGS_REF_THREADS;
constexpr int kWarps = kThreads / 32;
static_assert(kThreads % 32 == 0 && 8 % kWarps == 0, "the forward's 8 warp masks split evenly");
#ifndef CGS_REF_EPT
#define CGS_REF_EPT 6
#endif
constexpr int kEpt = CGS_REF_EPT;           // records per thread per chunk
constexpr int kRefChunk = kThreads * kEpt;  // 768
#ifndef CGS_REF_FIRST
#define CGS_REF_FIRST (CGS_REF_THREADS * CGS_REF_EPT)
#endif
constexpr int kRefFirst = CGS_REF_FIRST;
static_assert(kRefFirst > 0 && kRefFirst <= kRefChunk, "first chunk");

struct Carry {  // one flagged pixel, between chunks
  double T, P[3], C[3];
  int cnt;
  uint32_t last;
  int done;
};

}  // namespace

template <bool BWD>
#ifdef CGS_REF_MINB
#define CGS_REF_BOUNDS __launch_bounds__(kThreads, CGS_REF_MINB)
#else
#define CGS_REF_BOUNDS __launch_bounds__(kThreads)
#endif
__global__ void CGS_REF_BOUNDS refine_kernel(
    FrameDesc fd, const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_vals,
    const SplatRec* __restrict__ recs, const float* __restrict__ logits, int64_t n_gauss,
    FrameHeader* __restrict__ hdr, const uint32_t* __restrict__ refine_tiles,
    const uint32_t* __restrict__ refine_mask, uint32_t* __restrict__ refine_off,
    RefinePx* __restrict__ refine_px, int64_t refine_px_cap, float* __restrict__ image,
    float* __restrict__ final_T, int32_t* __restrict__ counts, uint32_t* __restrict__ px_last,
    uint32_t* __restrict__ tile_nproc, const uint64_t* __restrict__ depth_key,
    uint64_t* __restrict__ tile_last_dk, uint32_t* __restrict__ tile_last_sid,
    unsigned long long* __restrict__ view_last_dk, const float* __restrict__ dL,
    const uint64_t* __restrict__ pair_off, const uint64_t* __restrict__ rect,
    float* __restrict__ partials, int64_t partial9_offset) {
  __shared__ uint2 s_ck[kRefChunk];  // compacted in-box records of the chunk: (chunk index, splat id)
  __shared__ uint16_t s_pix[256];
  __shared__ Carry s_car[256];
  __shared__ double s_wp[kWarps];      // warp products
  __shared__ double s_wc[kWarps][3];   // warp colour sums (up to the warp's first end)
  __shared__ int s_wk[kWarps];         // warp contribution counts
  __shared__ int s_wt[kWarps];         // warp's first terminating index or kThreads
  __shared__ double s_wta[kWarps];     // T after that record
  __shared__ int s_cnt[kWarps];
  __shared__ int s_npx, s_alive, s_m;
  __shared__ uint32_t s_off;
  if (hdr->stats.overflow) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_list = static_cast<int64_t>(hdr->scratch[3]);
  for (int64_t ti = blockIdx.x; ti < n_list; ti += gridDim.x) {
    const int tile = static_cast<int>(refine_tiles[ti]);
    int v = 0;
    while (v + 1 < fd.n_views && fd.cam[v + 1].tile_base <= tile) ++v;
    const CamDev& cam = fd.cam[v];
    const int lt = tile - cam.tile_base;
    const int ty = lt / cam.ntx, tx = lt - ty * cam.ntx;
    const uint2 rg = ranges[tile];
    const int n = static_cast<int>(rg.y - rg.x);
    {  // flagged pixels, in the forward's warp / lane order (8 warps of 8x4 blocks)
      int tot = 0;
      for (int fw0 = 0; fw0 < 8; fw0 += kWarps) {
        const int fw = fw0 + warp;
        const int lx = fwd_px_x(fw, lane), ly = fwd_px_y(fw, lane);
        const bool in = tx * kTile + lx < cam.width && ty * kTile + ly < cam.height;
        const uint32_t wm = refine_mask[static_cast<int64_t>(tile) * 8 + fw];
        const bool f = in && ((wm >> lane) & 1u);
        const unsigned bal = __ballot_sync(kFull, f);
        if (lane == 0) s_cnt[warp] = __popc(bal);
        __syncthreads();
        int base = tot, t_r = 0;
        for (int w = 0; w < kWarps; ++w) {
          if (w < warp) base += s_cnt[w];
          t_r += s_cnt[w];
        }
        if (f) s_pix[base + __popc(bal & lanemask_lt())] = static_cast<uint16_t>(ly * kTile + lx);
        tot += t_r;
        __syncthreads();
      }
      if (tid == 0) {
        s_npx = tot;
        if (!BWD) {
          const unsigned long long o = atomicAdd(&hdr->scratch[4], static_cast<unsigned long long>(tot));
          s_off = o + tot <= static_cast<unsigned long long>(refine_px_cap) ? static_cast<uint32_t>(o)
                                                                          : 0xffffffffu;
          refine_off[ti] = s_off;
        } else {
          s_off = refine_off[ti];
        }
      }
      __syncthreads();
    }
    const int npx = s_npx;
    const bool have_c = BWD && s_off != 0xffffffffu;
    const int np = BWD ? static_cast<int>(tile_nproc[tile]) : n;
    const int n_walk = BWD ? np : n;  // the backward needs no pair past the prefix
    // backward without stored colours: pass 0 walks for C first
    for (int pass = (BWD && have_c) ? 1 : 0; pass < (BWD ? 2 : 1); ++pass) {
      const bool grads = BWD && pass == 1;
      for (int q = tid; q < npx; q += kThreads) {
        Carry& c = s_car[q];
        if (grads && have_c) {
          const RefinePx& e = refine_px[s_off + q];
          c.C[0] = e.C[0];
          c.C[1] = e.C[1];
          c.C[2] = e.C[2];
        }  // pass 1 without stored colours: C was left by pass 0
        c.T = 1.0;
        c.P[0] = c.P[1] = c.P[2] = 0.0;
        c.cnt = 0;
        c.last = static_cast<uint32_t>(n);
        c.done = 0;
      }
      if (tid == 0) s_alive = npx;
      __syncthreads();
      // this thread's records of a chunk: id and contribution box; the next
      // chunk's are loaded while the current one is walked
      uint32_t sid[kEpt], nsid[kEpt];
      uint2 box[kEpt], nbox[kEpt];
      // the first chunk is kRefFirst records (a flagged pixel usually
      // terminates early in the list), later ones kRefChunk
      auto chunk_len = [&](int c0) { return min(c0 == 0 ? kRefFirst : kRefChunk, n_walk - c0); };
      auto load_chunk = [&](int c0, uint32_t (&si)[kEpt], uint2 (&bx)[kEpt]) {
        const int nb = chunk_len(c0);
#pragma unroll
        for (int i = 0; i < kEpt; ++i) {
          const int e = kEpt * tid + i;
          si[i] = e < nb ? pair_vals[rg.x + c0 + e] : 0u;
        }
#pragma unroll
        for (int i = 0; i < kEpt; ++i) {
          const int e = kEpt * tid + i;
          bx[i] = e < nb ? *reinterpret_cast<const uint2*>(&recs[si[i]].px0) : make_uint2(0xffffu, 0u);
        }
      };
      if (n_walk > 0) load_chunk(0, nsid, nbox);
      for (int c0 = 0; c0 < n_walk && s_alive > 0; c0 += chunk_len(c0)) {
        const int nb = chunk_len(c0);
#pragma unroll
        for (int i = 0; i < kEpt; ++i) {
          sid[i] = nsid[i];
          box[i] = nbox[i];
        }
        if (c0 + nb < n_walk) load_chunk(c0 + nb, nsid, nbox);
        (void)nb;
        for (int q = 0; q < npx; ++q) {
          if (s_car[q].done) continue;  // block-uniform
          const int lpix = s_pix[q];
          const int lx = lpix & 15, ly = lpix >> 4;
          const int px = tx * kTile + lx, py = ty * kTile + ly;
          // compact the records whose box holds the pixel, in list order
          int mine = 0;
          bool inb[kEpt];
#pragma unroll
          for (int i = 0; i < kEpt; ++i) {
            const int x0 = box[i].x & 0xffff, x1 = box[i].x >> 16, y0 = box[i].y & 0xffff, y1 = box[i].y >> 16;
            inb[i] = x0 != 0xffff && px >= x0 && px <= x1 && py >= y0 && py <= y1;
            mine += inb[i];
          }
          int incl = mine;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane == 31) s_cnt[warp] = incl;
          __syncthreads();
          int pos = incl - mine, m = 0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            if (w < warp) pos += s_cnt[w];
            m += s_cnt[w];
          }
#pragma unroll
          for (int i = 0; i < kEpt; ++i)
            if (inb[i]) s_ck[pos++] = make_uint2(static_cast<uint32_t>(kEpt * tid + i), sid[i]);
          __syncthreads();
          double g[3] = {0.0, 0.0, 0.0};
          if (grads) {
            const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
            g[0] = dL[3 * pix + 0];
            g[1] = dL[3 * pix + 1];
            g[2] = dL[3 * pix + 2];
          }
          // rounds of kThreads compacted records, one per thread
          for (int r0 = 0; r0 < m; r0 += kThreads) {
            const Carry& car = s_car[q];
            const double T0 = car.T;
            const int j = r0 + tid;
            double a = 0.0, cr = 0.0, cg = 0.0, cb = 0.0;
            bool flow = false;
            uint32_t k = 0, s = 0;
            if (j < m) {
              const uint2 ck = s_ck[j];
              k = ck.x;
              s = ck.y;
              const SplatRec rr = recs[s];
              const double o = 1.0 / (1.0 + exp(-static_cast<double>(logits[s % static_cast<uint64_t>(n_gauss)])));
              // render.py:274-280 in the reference's operation order
              const double dx = __dsub_rn(static_cast<double>(px) + 0.5, rr.mx);
              const double dy = __dsub_rn(static_cast<double>(py) + 0.5, rr.my);
              const double qf = __dadd_rn(__dmul_rn(rr.ca, __dmul_rn(dx, dx)), __dmul_rn(rr.cc, __dmul_rn(dy, dy)));
              const double pw = __dsub_rn(__dmul_rn(-0.5, qf), __dmul_rn(__dmul_rn(rr.cb, dx), dy));
              const double x = __dmul_rn(o, exp(pw));
              const double al = x < 0.99 ? x : 0.99;
              if (al >= 1.0 / 255.0) {  // kept (render.py:279)
                a = al;
                flow = x < 0.99;
              }
              cr = rr.r;
              cg = rr.g;
              cb = rr.b;
#if CGS_REFINE_ALL
              if (!BWD && x >= 0.5 / 255.0) {  // diagnostics: the fp32 raster's alpha error
                const Staged sg = stage_splat(rr, tile_centre(tx), tile_centre(ty));
                const float x32 = exp2f(staged_t(sg.a, sg.b, static_cast<float>(lx) - kTileHalf,
                                                 static_cast<float>(ly) - kTileHalf)) / 255.0f;
                const float er = fabsf(static_cast<float>(static_cast<double>(x32) / x - 1.0));
                atomicMax(reinterpret_cast<unsigned int*>(&hdr->scratch[7]) + 1, __float_as_uint(er));
              }
#endif
            }
            const double f = 1.0 - a;
            // T before this record: warp scan of the factors, then the warps before
            double inc = f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(kFull, inc, o);
              if (lane >= o) inc *= y;
            }
            double ex = __shfl_up_sync(kFull, inc, 1);
            if (lane == 0) ex = 1.0;
            if (lane == 31) s_wp[warp] = inc;
            __syncthreads();
            double pre = T0;
            for (int w = 0; w < warp; ++w) pre *= s_wp[w];
            const double tb = pre * ex, ta = pre * inc;
            // the first record after which T < 1e-4 is the last active one
            // (render.py:281-283); only a kept record lowers T
            const unsigned tm = __ballot_sync(kFull, j < m && ta < 1e-4);
            const int wfirst = tm ? __ffs(tm) - 1 : 32;
            const bool act = a > 0.0 && lane <= wfirst;  // within this warp
            const double w = act ? a * tb : 0.0;
            double c3[3] = {w * cr, w * cg, w * cb};
            double e3[3] = {c3[0], c3[1], c3[2]};  // inclusive warp scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                const double y = __shfl_up_sync(kFull, e3[c], o);
                if (lane >= o) e3[c] += y;
              }
            }
            const int kc = __popc(__ballot_sync(kFull, act));
            if (lane == 31) {
              s_wc[warp][0] = e3[0];
              s_wc[warp][1] = e3[1];
              s_wc[warp][2] = e3[2];
              s_wk[warp] = kc;
            }
            const double ta_first = __shfl_sync(kFull, ta, tm ? wfirst : 0);
            if (lane == 0) {
              s_wt[warp] = tm ? r0 + warp * 32 + wfirst : 0x7fffffff;
              s_wta[warp] = ta_first;
            }
            __syncthreads();
            // the block's first terminating warp ends the pixel
            int tw = kWarps;
            for (int ww = 0; ww < kWarps; ++ww)
              if (tw == kWarps && s_wt[ww] != 0x7fffffff) tw = ww;
            if (grads && act && warp <= tw) {
              double P[3] = {car.P[0], car.P[1], car.P[2]};
              for (int ww = 0; ww < warp; ++ww)
#pragma unroll
                for (int c = 0; c < 3; ++c) P[c] += s_wc[ww][c];
              // suffix = C - prefix through this record (render.py:354-359)
              const double iom = 1.0 / (1.0 - a);
              const double da = (cr * tb - (car.C[0] - (P[0] + e3[0])) * iom) * g[0] +
                                (cg * tb - (car.C[1] - (P[1] + e3[1])) * iom) * g[1] +
                                (cb * tb - (car.C[2] - (P[2] + e3[2])) * iom) * g[2];
              if (c0 + static_cast<int>(k) < np) {  // the pair's partial (raster_bwd layout)
                float o9[9] = {static_cast<float>(w * g[0]), static_cast<float>(w * g[1]),
                               static_cast<float>(w * g[2]), 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
                if (flow) {  // render.py:361-377, moments local to the tile
                  const double dp = da * a, fx = lx - 7.5, fy = ly - 7.5;  // tile-centred
                  o9[3] = static_cast<float>(dp);
                  o9[4] = static_cast<float>(dp * fx);
                  o9[5] = static_cast<float>(dp * fy);
                  o9[6] = static_cast<float>(dp * fx * fx);
                  o9[7] = static_cast<float>(dp * fx * fy);
                  o9[8] = static_cast<float>(dp * fy * fy);
                }
                const int64_t ei = static_cast<int64_t>(pair_off[s]) + [&] {
                  const uint64_t rc = rect[s];
                  const int tx0 = static_cast<int>(rc & 0xffff), tx1 = static_cast<int>((rc >> 16) & 0xffff);
                  const int ty0 = static_cast<int>((rc >> 32) & 0xffff);
                  return static_cast<int64_t>((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
                }();
                float4* p4 = reinterpret_cast<float4*>(partials) + 2 * ei;
                float4 xv = p4[0], yv = p4[1];
                xv.x += o9[0]; xv.y += o9[1]; xv.z += o9[2]; xv.w += o9[3];
                yv.x += o9[4]; yv.y += o9[5]; yv.z += o9[6]; yv.w += o9[7];
                p4[0] = xv;
                p4[1] = yv;
                partials[partial9_offset + ei] += o9[8];
              }
            }
            if (tid == 0) {  // pixel state after the round
              Carry& c = s_car[q];
              double tot = T0;
              for (int ww = 0; ww < kWarps && ww <= tw; ++ww) {
                c.P[0] += s_wc[ww][0];
                c.P[1] += s_wc[ww][1];
                c.P[2] += s_wc[ww][2];
                c.cnt += s_wk[ww];
                if (ww < tw) tot *= s_wp[ww];
              }
              if (tw < kWarps) {
                c.T = s_wta[tw];
                c.last = static_cast<uint32_t>(c0 + s_ck[s_wt[tw]].x + 1);
                c.done = 1;
                --s_alive;
              } else {
                c.T = tot;
              }
            }
            __syncthreads();
            if (s_car[q].done) break;
          }
        }
      }
      if (pass == 0) {  // per flagged pixel results
        for (int q = tid; q < npx; q += kThreads) {
          Carry& c = s_car[q];
          c.C[0] = c.P[0];
          c.C[1] = c.P[1];
          c.C[2] = c.P[2];
          if (BWD) continue;
          const int lpix = s_pix[q];
          const int px = tx * kTile + (lpix & 15), py = ty * kTile + (lpix >> 4);
          const int64_t pix = cam.pix_base + static_cast<int64_t>(py) * cam.width + px;
#if CGS_REFINE_ALL
          {  // diagnostics: the fp32 path's decisions against the float64 ones
            const uint32_t l32 = px_last[pix];
            if (l32 != c.last) atomicAdd(&hdr->scratch[5], 1ull);
            else if (counts[pix] != c.cnt) atomicAdd(&hdr->scratch[6], 1ull);
            else {
              const float er = fabsf(static_cast<float>(final_T[pix] / c.T - 1.0));
              atomicMax(reinterpret_cast<unsigned int*>(&hdr->scratch[7]), __float_as_uint(er));
            }
          }
#endif
          image[3 * pix + 0] = static_cast<float>(c.P[0]);
          image[3 * pix + 1] = static_cast<float>(c.P[1]);
          image[3 * pix + 2] = static_cast<float>(c.P[2]);
          final_T[pix] = static_cast<float>(c.T);
          counts[pix] = c.cnt;
          px_last[pix] = c.last | kRefinedBit;
          if (c.last > 0) atomicMax(&tile_nproc[tile], c.last);
          if (s_off != 0xffffffffu) {
            RefinePx r;
            r.C[0] = c.P[0];
            r.C[1] = c.P[1];
            r.C[2] = c.P[2];
            r.T = c.T;
            r.last = c.last;
            r.pad = 0;
            refine_px[s_off + q] = r;
          }
        }
        __syncthreads();
      }
    }
    if (!BWD && tid == 0) {  // the tile's last processed splat after the re-walk
      const uint32_t np = atomicOr(&tile_nproc[tile], 0u);  // this CTA's atomicMax results
      if (np > 0) {
        const uint32_t ls = pair_vals[rg.x + np - 1];
        tile_last_dk[tile] = depth_key[ls];
        tile_last_sid[tile] = ls;
        atomicMax(&view_last_dk[v], static_cast<unsigned long long>(depth_key[ls]));
      }
    }
    __syncthreads();
  }
}

int launch_refine(bool bwd, const FrameDesc& fd, const FrameLayout& L, const uint32_t* vals,
                  const float* logits, float* image, float* final_T, int32_t* counts,
                  const float* dL, float* partials, cudaStream_t st) {
  const int64_t p9 = 8 * (L.pair_cap > 0 ? L.pair_cap : 1);
  // one wave of resident CTAs (per device ordinal: a process may drive several GPUs)
  static std::atomic<int> resident[2][kMaxDevices] = {};
  int dev = 0;
  if (int rc = current_device(&dev)) return rc;
  if (resident[bwd][dev].load() == 0) {
    int sms = 0, per_sm = 0;
    CGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (bwd)
      CGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_kernel<true>, kThreads, 0));
    else
      CGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_kernel<false>, kThreads, 0));
    resident[bwd][dev].store(sms * (per_sm > 0 ? per_sm : 1));
  }
  const int grid = resident[bwd][dev].load();
  if (bwd) {
    CGS_PROFILED("refine_bwd_kernel", st,
                 (refine_kernel<true><<<grid, kThreads, 0, st>>>(
                     fd, L.ranges, vals, L.recs, logits, L.n, L.hdr, L.refine_tiles, L.refine_mask,
                     L.refine_off, L.refine_px, L.refine_px_cap, nullptr, nullptr, nullptr,
                     L.px_last, L.tile_nproc, L.depth_key, L.tile_last_dk, L.tile_last_sid, L.view_last_dk, dL, L.pair_off, L.rect,
                     partials, p9)));
    CGS_CHECK_LAUNCH("refine_bwd_kernel");
  } else {
    CGS_PROFILED("refine_fwd_kernel", st,
                 (refine_kernel<false><<<grid, kThreads, 0, st>>>(
                     fd, L.ranges, vals, L.recs, logits, L.n, L.hdr, L.refine_tiles, L.refine_mask,
                     L.refine_off, L.refine_px, L.refine_px_cap, image, final_T, counts,
                     L.px_last, L.tile_nproc, L.depth_key, L.tile_last_dk, L.tile_last_sid, L.view_last_dk, nullptr, nullptr, nullptr,
                     nullptr, 0)));
    CGS_CHECK_LAUNCH("refine_fwd_kernel");
  }
  return CGS_OK;
}

}  // namespace cgs
