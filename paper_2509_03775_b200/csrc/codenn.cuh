// Nearest live code row per live code row: the "distance GEMM" of the code
// reassignment extension (BASELINE.json north_star
// item 5).  The reference never recomputes assignments by distance
// (SURVEY.md section 0.1), so there is no reference oracle: the definition
// is this build's, and tests/ check it against an fp64 brute force.
//
//   nn(i) = argmin_{j live, j != i} || r_i - r_j ||^2   (fp64 of the fp32
//   rows, ties -> smaller row index), for every live row i.
//
// Three kernels:
//  1. codenn_pack: live rows -> fp32 tiles in the tcgen05 K-major
//     no-swizzle "core matrix" order (8 rows x 16 B per core matrix), row
//     norms; padding rows get norm +inf.
//  2. codenn_gemm: S = R R^T on the 5th-gen tensor cores (tcgen05.mma
//     kind::tf32 as 3xTF32 -- head/tail split, three MMAs per K step -- for
//     ~fp32 accuracy; M=128 x N=128 per instruction, accumulators in TMEM,
//     double-buffered), operand tiles brought in by the bulk-copy engine
//     (one cp.async.bulk per 128-row tile and part: the packed order makes a
//     tile contiguous).  Warp roles: 8 epilogue warps (TMEM lane quarter
//     w % 4, column half w / 4), one producer, one MMA issuer.  The epilogue
//     turns S into approximate distances n_i + n_j - 2 s_ij and keeps each
//     row's kNnCand best.
//  3. codenn_refine: exact fp64 distances of the candidates; accepted when
//     the best exact distance is strictly below (kCand-th approximate
//     distance - error bound), which no row outside the candidate set can
//     beat; otherwise a warp brute-forces the row in fp64.  The result is
//     therefore exact whatever the tf32 rounding did.
#pragma once
#include <cstdint>

#include "raster_common.cuh"

namespace cgs {

constexpr int kNnM = 128;       // rows per CTA (UMMA M)
constexpr int kNnN = 128;       // columns per B tile (UMMA N)
constexpr int kNnCand = 4;      // candidates kept per row
constexpr int kNnStages = 2;    // B-tile smem stages
constexpr int kNnThreads = 320; // 8 epilogue warps + producer + MMA

__host__ __device__ __forceinline__ int nn_dpad(int d) { return (d + 7) / 8 * 8; }

// byte offset of element (r, k) in the packed core-matrix order
__host__ __device__ __forceinline__ int64_t nn_packed_off(int64_t r, int k, int dp) {
  return ((r >> 3) * (dp >> 2) + (k >> 2)) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

// ---- tcgen05 / TMEM PTX wrappers (sm_100a) ---------------------------------
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  // K-major, SWIZZLE_NONE: start >> 4 in [0,14), LBO >> 4 in [16,30), SBO >> 4
  // in [32,46), version 1 in [46,48), base offset 0, layout type 0 in [61,64)
  return static_cast<uint64_t>((saddr >> 4) & 0x3fff) |
         (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3fff) << 16) |
         (static_cast<uint64_t>((sbo_bytes >> 4) & 0x3fff) << 32) | (1ull << 46);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane into v[o, o + 32)
// (no wait: call tmem_ld_wait before using them)
template <int N>
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, float (&v)[N], int o) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 32; ++k) v[o + k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- 1. pack -----------------------------------------------------------------
// live rows (indices `live`, n_live of them) of rows (cap x d, row stride d)
// -> packed: two (mpad x dp) arrays in core-matrix order, the tf32 head
// hi = rna_tf32(x) and the tail lo = x - hi (exact in fp32), for the 3xTF32
// product hi hi' + hi lo' + lo hi' (error ~2^-20 |x||x'| instead of tf32's
// 2^-10); norms (fp32 of the fp64 sum); rows >= n_live are zero with norm +inf.
__global__ void codenn_pack_kernel(const float* __restrict__ rows, int d,
                                   const int32_t* __restrict__ live, int64_t n_live, int64_t mpad,
                                   int dp, float* __restrict__ packed, float* __restrict__ norms,
                                   unsigned* __restrict__ max_norm_bits) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < mpad;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float* src = r < n_live ? rows + static_cast<int64_t>(live[r]) * d : nullptr;
    double nn = 0.0;
    char* base = reinterpret_cast<char*>(packed);
    for (int k = 0; k < dp; ++k) {
      const float x = (src && k < d) ? src[k] : 0.0f;
      nn += static_cast<double>(x) * x;
      uint32_t hb;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
      const float hi = __uint_as_float(hb);
      *reinterpret_cast<float*>(base + nn_packed_off(r, k, dp)) = hi;
      *reinterpret_cast<float*>(base + mpad * dp * 4 + nn_packed_off(r, k, dp)) = x - hi;
    }
    norms[r] = r < n_live ? static_cast<float>(nn) : __int_as_float(0x7f800000);
    // non-negative floats order as their bit patterns
    if (r < n_live) atomicMax(max_norm_bits, __float_as_uint(static_cast<float>(nn)));
  }
}

// ---- 2. tensor-core distance GEMM + per-row candidates ------------------------
constexpr int kNnNormSlots = 4;  // column-norm ring, decoupled from the B stages

struct NnSmem {
  uint64_t full[kNnStages];
  uint64_t empty[kNnStages];
  uint64_t nfull[kNnNormSlots];
  uint64_t nempty[kNnNormSlots];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t afull;
  uint32_t tmem_base;
};

constexpr int kNnEpiWarps = 8;  // warp w: TMEM lanes [32 (w % 4), +32), column half w / 4
constexpr int kNnChunk = 64;    // columns per TMEM read

// Dynamic smem: [NnSmem | pad to 1024 | A tile (hi, lo: 2 x 128 x dp) | B
// stages (hi, lo: 2 x 128 x dp each) | B-stage norms (128 each) | epilogue
// compaction slots (2 x 32 x 256 words) | candidate merge (128 x 4 x 2 words)]: 213 KB at
// dp = 48, the widest row supported (SH degree 3).
inline size_t codenn_gemm_smem(int dp) {
  return 1024 + 2 * static_cast<size_t>(kNnM) * dp * 4 +
         static_cast<size_t>(kNnStages) * 2 * kNnN * dp * 4 + kNnNormSlots * kNnN * 4 +
         2 * static_cast<size_t>(32) * 256 * 4 + static_cast<size_t>(kNnM) * kNnCand * 8;
}

__device__ __forceinline__ void nn_insert(float d, int j, float (&bd)[kNnCand], int (&bj)[kNnCand]) {
  if (!(d < bd[kNnCand - 1])) return;
  bd[kNnCand - 1] = d;
  bj[kNnCand - 1] = j;
#pragma unroll
  for (int k = kNnCand - 1; k > 0; --k) {
    if (bd[k] < bd[k - 1]) {
      const float td = bd[k];
      bd[k] = bd[k - 1];
      bd[k - 1] = td;
      const int tj = bj[k];
      bj[k] = bj[k - 1];
      bj[k - 1] = tj;
    }
  }
}

__device__ __forceinline__ void epi_bar() {  // the 8 epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kNnEpiWarps * 32) : "memory");
}

// grid = mpad / 128 CTAs; cand_d / cand_j: mpad x kNnCand (approximate
// distances ascending, packed-row indices).  debug_s (optional, tests):
// the raw S = R R^T, mpad x mpad.  trace (optional): CTA 0's per-tile
// timeline.
__global__ void __launch_bounds__(kNnThreads, 1) codenn_gemm_kernel(
    const float* __restrict__ packed, const float* __restrict__ norms, int64_t mpad, int dp,
    float* __restrict__ cand_d, int32_t* __restrict__ cand_j, float* __restrict__ debug_s,
    unsigned long long* __restrict__ trace = nullptr) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  NnSmem& S = *reinterpret_cast<NnSmem*>(smem_raw);
  float* sA = reinterpret_cast<float*>(smem_raw + 1024);
  float* sB = sA + 2 * kNnM * dp;                                   // stages x [hi | lo]
  float* sN = sB + static_cast<size_t>(kNnStages) * 2 * kNnN * dp;  // kNnNormSlots x kNnN norms
  float* sV = sN + kNnNormSlots * kNnN;  // 32 x 256 (epilogue threads) compaction slots
  int* sVi = reinterpret_cast<int*>(sV + 32 * 256);       // 32 x 256 column ids
  float* sMd = reinterpret_cast<float*>(sVi + 32 * 256);  // 128 x kNnCand
  int* sMj = reinterpret_cast<int*>(sMd + kNnM * kNnCand);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kNnM;
  const int n_tiles = static_cast<int>(mpad / kNnN);
  const uint32_t a_bytes = static_cast<uint32_t>(kNnM * dp * 4);
  const uint32_t b_bytes = static_cast<uint32_t>(kNnN * dp * 4);
  constexpr int kProducer = kNnEpiWarps, kMma = kNnEpiWarps + 1;

  if (tid == 0) {
    for (int s = 0; s < kNnStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);  // the MMA commit
    }
    for (int s = 0; s < kNnNormSlots; ++s) {
      mbar_init(&S.nfull[s], 1);
      mbar_init(&S.nempty[s], kNnEpiWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&S.tfull[s], 1);
      mbar_init(&S.tempty[s], kNnEpiWarps);  // one arrival per epilogue warp
    }
    mbar_init(&S.afull, 1);
  }
  if (warp == kMma) {  // TMEM: 2 accumulator stages x kNnN fp32 columns (256 allocated)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(&S.tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == kProducer) {
    // ===== producer: A tile once, then B tiles (+ their norms) through the stages =====
    if (lane == 0) {
      const char* lo = reinterpret_cast<const char*>(packed) + mpad * dp * 4;
      mbar_arrive_expect_tx(&S.afull, 2 * a_bytes);
      bulk_g2s(sA, reinterpret_cast<const char*>(packed) + row0 * dp * 4, a_bytes, &S.afull);
      bulk_g2s(sA + kNnM * dp, lo + row0 * dp * 4, a_bytes, &S.afull);
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % kNnStages;
        const uint32_t ph = (t / kNnStages) & 1u;
        mbar_wait(&S.empty[s], ph ^ 1u);
        if (trace && blockIdx.x == 0 && t < 256) trace[4 * t + 3] = global_ns();
        mbar_arrive_expect_tx(&S.full[s], 2 * b_bytes);
        float* dst = sB + static_cast<size_t>(s) * 2 * kNnN * dp;
        const int64_t off = static_cast<int64_t>(t) * kNnN * dp * 4;
        bulk_g2s(dst, reinterpret_cast<const char*>(packed) + off, b_bytes, &S.full[s]);
        bulk_g2s(dst + kNnN * dp, lo + off, b_bytes, &S.full[s]);
        const int ns = t % kNnNormSlots;
        mbar_wait(&S.nempty[ns], ((t / kNnNormSlots) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&S.nfull[ns], kNnN * 4);
        bulk_g2s(sN + ns * kNnN, norms + static_cast<int64_t>(t) * kNnN, kNnN * 4, &S.nfull[ns]);
      }
    }
  } else if (warp == kMma) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(kNnM, kNnN);
      const uint32_t sbo = static_cast<uint32_t>(dp / 4) * 128u;  // next 8-row group
      mbar_wait(&S.afull, 0);
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % kNnStages;
        const uint32_t ph = (t / kNnStages) & 1u;
        const int acc = t & 1;
        mbar_wait(&S.tempty[acc], ((t >> 1) & 1u) ^ 1u);  // epilogue drained this stage
        mbar_wait(&S.full[s], ph);
        tmem_fence_after();
        if (trace && blockIdx.x == 0 && t < 256) trace[4 * t] = global_ns();
        const uint32_t a0 = smem_u32(sA), a1 = smem_u32(sA + kNnM * dp);
        const uint32_t b0 = smem_u32(sB + static_cast<size_t>(s) * 2 * kNnN * dp);
        const uint32_t b1 = b0 + static_cast<uint32_t>(kNnN * dp * 4);
        const uint32_t d = tmem + static_cast<uint32_t>(acc * kNnN);
        for (int ks = 0; ks < dp / 8; ++ks) {  // K step of 8 tf32 = two 16-B core matrices
          const uint64_t ah = umma_desc(a0 + ks * 256u, 128u, sbo);
          const uint64_t al = umma_desc(a1 + ks * 256u, 128u, sbo);
          const uint64_t bh = umma_desc(b0 + ks * 256u, 128u, sbo);
          const uint64_t bl = umma_desc(b1 + ks * 256u, 128u, sbo);
          umma_tf32(d, ah, bh, idesc, ks > 0 ? 1u : 0u);  // 3xTF32: hi hi' + hi lo' + lo hi'
          umma_tf32(d, ah, bl, idesc, 1u);
          umma_tf32(d, al, bh, idesc, 1u);
        }
        umma_commit(&S.empty[s]);    // B operand consumed once these MMAs complete
        umma_commit(&S.tfull[acc]);  // accumulator ready
      }
    }
  } else {
    // ===== epilogue: warp w reads TMEM lanes [32 (w % 4), +32) (its tile rows),
    // columns [kNnN / 2 (w / 4), +kNnN / 2) of each tile =====
    const int quarter = warp & 3, half = warp >> 2;
    const int r = quarter * 32 + lane;
    const int64_t gi = row0 + r;
    const float ni = norms[gi];
    float bd[kNnCand];
    int bj[kNnCand];
#pragma unroll
    for (int k = 0; k < kNnCand; ++k) {
      bd[k] = __int_as_float(0x7f800000);
      bj[k] = -1;
    }
    for (int t = 0; t < n_tiles; ++t) {
      const int acc = t & 1, ns = t % kNnNormSlots;
      mbar_wait(&S.nfull[ns], (t / kNnNormSlots) & 1u);
      mbar_wait(&S.tfull[acc], (t >> 1) & 1u);
      tmem_fence_after();
      if (trace && blockIdx.x == 0 && t < 256 && tid == 0) trace[4 * t + 1] = global_ns();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                             static_cast<uint32_t>(acc * kNnN + half * (kNnN / 2));
#pragma unroll 1
      for (int c0 = 0; c0 < kNnN / 2; c0 += kNnChunk) {
        const int cl = half * (kNnN / 2) + c0;  // column within the tile
        const int64_t j0 = static_cast<int64_t>(t) * kNnN + cl;
        float v[kNnChunk];
#pragma unroll
        for (int q = 0; q < kNnChunk / 32; ++q) tmem_ld32_nowait(tbase + c0 + 32 * q, v, 32 * q);
        tmem_ld_wait();
        if (debug_s) {
#pragma unroll
          for (int k = 0; k < kNnChunk; ++k) debug_s[gi * mpad + j0 + k] = v[k];
        }
        const float4* n4 = reinterpret_cast<const float4*>(sN + ns * kNnN + cl);  // broadcast
        // row-relative distance n_j - 2 s_ij (n_i is the same for the whole row;
        // it is added to the candidates at the end)
#pragma unroll
        for (int q = 0; q < kNnChunk / 4; ++q) {
          const float4 f = n4[q];
          v[4 * q] = fmaf(-2.0f, v[4 * q], f.x);
          v[4 * q + 1] = fmaf(-2.0f, v[4 * q + 1], f.y);
          v[4 * q + 2] = fmaf(-2.0f, v[4 * q + 2], f.z);
          v[4 * q + 3] = fmaf(-2.0f, v[4 * q + 3], f.w);
        }
        if (gi >= j0 && gi < j0 + kNnChunk) {  // the diagonal: never its own neighbour
#pragma unroll
          for (int k = 0; k < kNnChunk; ++k)
            if (j0 + k == gi) v[k] = __int_as_float(0x7f800000);
        }
        // tree minimum, then the (rare) insertions
        float m[kNnChunk / 2];
#pragma unroll
        for (int k = 0; k < kNnChunk / 2; ++k) m[k] = fminf(v[2 * k], v[2 * k + 1]);
#pragma unroll
        for (int w = kNnChunk / 4; w >= 1; w >>= 1)
#pragma unroll
          for (int k = 0; k < w; ++k) m[k] = fminf(m[2 * k], m[2 * k + 1]);
        if (m[0] < bd[kNnCand - 1]) {
          // compact the qualifying columns into this thread's shared-memory
          // slots ([slot][thread], conflict-free), then insert them in order
#pragma unroll
          for (int h = 0; h < kNnChunk / 32; ++h) {  // 32 slots per thread
            const float thr = bd[kNnCand - 1];
            int cnt = 0;
#pragma unroll
            for (int k = 32 * h; k < 32 * h + 32; ++k) {
              if (v[k] < thr) {
                sV[cnt * 256 + tid] = v[k];
                sVi[cnt * 256 + tid] = k;
                ++cnt;
              }
            }
            for (int q = 0; q < cnt; ++q)
              nn_insert(sV[q * 256 + tid], static_cast<int>(j0 + sVi[q * 256 + tid]), bd, bj);
          }
        }
      }
      tmem_fence_before();
      __syncwarp();
      if (trace && blockIdx.x == 0 && t < 256 && tid == 0) trace[4 * t + 2] = global_ns();
      if (lane == 0) {
        mbar_arrive(&S.tempty[acc]);
        mbar_arrive(&S.nempty[ns]);  // done with this tile's norms
      }
    }
    // merge the two column halves of each row
    if (half == 1) {
#pragma unroll
      for (int k = 0; k < kNnCand; ++k) {
        sMd[r * kNnCand + k] = bd[k];
        sMj[r * kNnCand + k] = bj[k];
      }
    }
    epi_bar();
    if (half == 0) {
#pragma unroll
      for (int k = 0; k < kNnCand; ++k) nn_insert(sMd[r * kNnCand + k], sMj[r * kNnCand + k], bd, bj);
#pragma unroll
      for (int k = 0; k < kNnCand; ++k) {  // + n_i: monotone, so the order is kept
        cand_d[gi * kNnCand + k] = bd[k] + ni;
        cand_j[gi * kNnCand + k] = bj[k];
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tmem_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// ---- 3. exact refinement ---------------------------------------------------------
__device__ __forceinline__ double nn_dist64(const float* __restrict__ rows, int d, int32_t a,
                                            int32_t b) {
  const float* x = rows + static_cast<int64_t>(a) * d;
  const float* y = rows + static_cast<int64_t>(b) * d;
  double s = 0.0;  // sequential, no fma contraction: sum_k fl(fl(x_k - y_k)^2)
  for (int k = 0; k < d; ++k) {
    const double t = __dsub_rn(static_cast<double>(x[k]), static_cast<double>(y[k]));
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// One thread per live row: exact distances of the candidates; rows whose
// candidate set is not provably complete are appended to `redo`.
// Error bound of an approximate distance n_i + n_j - 2 s~_ij: the 3xTF32
// product drops lo lo' (<= 2^-22 |ab|) and reads lo truncated to tf32
// (<= 2^-21 |ab| per term), and accumulates 3 x 64 products in fp32
// (<= 2^-16 sum |ab|), so |s~ - s| <= 2^-15 |a| |b|; the fp32 norms and the
// final fma add <= 2^-22 (n_i + n_j + 2 |a| |b|).  With |b| <= M = max |row|
// the bound used, 2e-4 |a| M + 1e-6 (n_i + M^2), is ~3x above both for
// every j (tests/test_gpu_codenn.py measures the product error).
__global__ void codenn_refine_kernel(const float* __restrict__ rows, int d,
                                     const int32_t* __restrict__ live, int64_t n_live,
                                     const float* __restrict__ norms,
                                     const unsigned* __restrict__ max_norm_bits,
                                     const float* __restrict__ cand_d,
                                     const int32_t* __restrict__ cand_j, int32_t* __restrict__ nn_idx,
                                     double* __restrict__ nn_dist, int32_t* __restrict__ redo,
                                     unsigned* __restrict__ n_redo) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_live;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t ri = live[i];
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int32_t bidx = -1;
    for (int k = 0; k < kNnCand; ++k) {
      const int32_t j = cand_j[i * kNnCand + k];
      if (j < 0 || j >= n_live) continue;
      const int32_t rj = live[j];
      const double dd = nn_dist64(rows, d, ri, rj);
      if (dd < best || (dd == best && rj < bidx)) {
        best = dd;
        bidx = rj;
      }
    }
    // every row outside the candidates has approx >= cand_d[last], so exact
    // >= cand_d[last] - bound; complete when that is > best (strict: ties
    // with an outside row would need the index rule)
    const double m2 = static_cast<double>(__uint_as_float(*max_norm_bits));
    const double ni = static_cast<double>(norms[i]);
    const double bound = 2e-4 * sqrt(ni) * sqrt(m2) + 1e-6 * (ni + m2) + 1e-30;
    const float last = cand_d[i * kNnCand + kNnCand - 1];
    const bool full_set = n_live - 1 <= kNnCand;  // every other row is a candidate
    if (bidx >= 0 && (full_set || static_cast<double>(last) - bound > best)) {
      nn_idx[ri] = bidx;
      nn_dist[ri] = best;
    } else if (n_live > 1) {
      redo[atomicAdd(n_redo, 1u)] = static_cast<int32_t>(i);
    }
  }
}

// One warp per row to redo: fp64 brute force over all live rows.
__global__ void codenn_bruteforce_kernel(const float* __restrict__ rows, int d,
                                         const int32_t* __restrict__ live, int64_t n_live,
                                         const int32_t* __restrict__ redo,
                                         const unsigned* __restrict__ n_redo,
                                         int32_t* __restrict__ nn_idx,
                                         double* __restrict__ nn_dist) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nr = *n_redo;
  for (int64_t q = wid; q < nr; q += nw) {
    const int32_t ri = live[redo[q]];
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int32_t bidx = 0x7fffffff;
    for (int64_t j = lane; j < n_live; j += 32) {
      const int32_t rj = live[j];
      if (rj == ri) continue;
      const double dd = nn_dist64(rows, d, ri, rj);
      if (dd < best || (dd == best && rj < bidx)) {
        best = dd;
        bidx = rj;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int32_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob < best || (ob == best && oi < bidx)) {
        best = ob;
        bidx = oi;
      }
    }
    if (lane == 0) {
      nn_idx[ri] = bidx == 0x7fffffff ? -1 : bidx;
      nn_dist[ri] = best;
    }
  }
}

}  // namespace cgs
