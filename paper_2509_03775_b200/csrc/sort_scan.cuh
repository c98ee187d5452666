// Single-pass primitives for sm_100a: decoupled-lookback exclusive scan and
// onesweep (decoupled-lookback) LSD radix sort, both stable and
// deterministic.  Element counts may live in device memory so the whole
// frame can be enqueued (and graph-captured) without host round trips; the
// grid is sized for a capacity and surplus CTAs exit after claiming an
// out-of-range partition id.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace cgs {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T ld_volatile(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}
template <typename T>
__device__ __forceinline__ void st_volatile(T* p, T v) {
  *reinterpret_cast<volatile T*>(p) = v;
}

__device__ __forceinline__ int64_t dev_count(const unsigned long long* n_dev, int64_t n_host) {
  return n_dev ? static_cast<int64_t>(ld_volatile(n_dev)) : n_host;
}

// Lanes of the warp whose 8-bit digit equals this lane's (all 32 lanes must
// call it).  Eight ballots instead of one match.any, which issues far slower.
__device__ __forceinline__ unsigned warp_peers8(unsigned d) {
  unsigned peers = kFull;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(kFull, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

// Same for a digit of `bits` <= 8 significant bits (warp-uniform): the
// ballots of bits every key has zero are skipped (keys narrower than the
// last 8-bit pass, e.g. 11-bit tile keys).
__device__ __forceinline__ unsigned warp_peers_bits(unsigned d, int bits) {
  unsigned peers = kFull;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (b >= bits) break;
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(kFull, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ===========================================================================
// Exclusive scan.  Op provides:
//   __device__ uint64_t load(int64_t i) const;
//   __device__ void store(int64_t i, uint64_t exclusive, uint64_t value) const;
//   __device__ void finish(uint64_t total) const;  (called once, with the total)
// Partitions of 8 warps x 32 lanes x ROUNDS consecutive elements per lane
// (lane-major inside a warp, so the running sum follows index order).  Status words: value in bits 0..61, flag in 62..63.
// ===========================================================================
constexpr int kScanWarps = 8;
#ifndef CGS_SCAN_ROUNDS
#define CGS_SCAN_ROUNDS 8
#endif
constexpr int kScanRounds = CGS_SCAN_ROUNDS;
constexpr int kScanTile = kScanWarps * kScanRounds * 32;  // 2048
constexpr unsigned long long kScanAgg = 1ULL << 62;
constexpr unsigned long long kScanPre = 2ULL << 62;
constexpr unsigned long long kScanVal = (1ULL << 62) - 1;

struct ScanWs {
  unsigned long long* status;  // max_parts
  unsigned* counter;
  int64_t max_parts;
};

inline size_t scan_ws_bytes(int64_t n_cap) {
  int64_t parts = ceil_div(n_cap > 0 ? n_cap : 1, kScanTile);
  return align_up(parts * sizeof(unsigned long long)) + 256;
}

inline ScanWs carve_scan(Carver& c, int64_t n_cap) {
  ScanWs w;
  w.max_parts = ceil_div(n_cap > 0 ? n_cap : 1, kScanTile);
  w.status = c.take<unsigned long long>(w.max_parts);
  w.counter = c.take<unsigned>(64);
  return w;
}

template <class Op, int ROUNDS = kScanRounds>
__global__ void __launch_bounds__(256) scan_kernel(Op op, const unsigned long long* n_dev,
                                                   int64_t n_host, ScanWs ws,
                                                   unsigned long long* total) {
  constexpr int kScanRounds = ROUNDS;  // elements per lane (the partition is 256 x ROUNDS)
  constexpr int kScanTile = kScanWarps * kScanRounds * 32;
  __shared__ unsigned s_part;
  __shared__ unsigned long long s_warp[kScanWarps];
  __shared__ unsigned long long s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_part = atomicAdd(ws.counter, 1u);
  __syncthreads();
  const int64_t part = s_part;
  const int64_t n = dev_count(n_dev, n_host);
  const int64_t nparts = n > 0 ? ceil_div(n, kScanTile) : 1;
  if (part >= nparts) return;
  // lane l of a warp owns the ROUNDS consecutive elements wbase + l ROUNDS
  // + j, so its loads are independent of each other and issue together
  // (a round-per-32-elements layout had ptxas sink them into the shuffle
  // rounds: ~2 loads in flight), its running sum is local and one warp scan
  // of the lane totals places it
  const int64_t wbase = part * kScanTile + static_cast<int64_t>(warp) * kScanRounds * 32;
  const int64_t lbase = wbase + static_cast<int64_t>(lane) * kScanRounds;

  unsigned long long v[kScanRounds], ex[kScanRounds];
#pragma unroll
  for (int j = 0; j < kScanRounds; ++j) {
    const int64_t i = lbase + j;
    v[j] = (i < n) ? op.load(i) : 0ULL;
  }
  unsigned long long lrun = 0;
#pragma unroll
  for (int j = 0; j < kScanRounds; ++j) {
    ex[j] = lrun;
    lrun += v[j];
  }
  const unsigned long long linc = warp_incl_scan(lrun);
  const unsigned long long run = __shfl_sync(kFull, linc, 31);
#pragma unroll
  for (int j = 0; j < kScanRounds; ++j) ex[j] += linc - lrun;
  if (lane == 0) s_warp[warp] = run;
  __syncthreads();
  if (warp == 0) {
    unsigned long long wv = lane < kScanWarps ? s_warp[lane] : 0ULL;
    unsigned long long winc = warp_incl_scan(wv);
    const unsigned long long agg = __shfl_sync(kFull, winc, kScanWarps - 1);
    if (lane < kScanWarps) s_warp[lane] = winc - wv;
    unsigned long long excl = 0;
    if (part == 0) {
      if (lane == 0) st_volatile(&ws.status[0], kScanPre | agg);
    } else {
      if (lane == 0) st_volatile(&ws.status[part], kScanAgg | agg);
      int64_t p = part - 1;
      while (true) {
        const int64_t q = p - lane;
        unsigned long long s = (q >= 0) ? ld_volatile(&ws.status[q]) : kScanPre;
        const unsigned long long flag = s >> 62;
        const unsigned is_pre = __ballot_sync(kFull, flag == 2);
        const unsigned not_ready = __ballot_sync(kFull, flag == 0);
        const int first_pre = is_pre ? __ffs(is_pre) - 1 : 32;
        const unsigned relevant = first_pre >= 31 ? kFull : ((2u << first_pre) - 1u);
        if (not_ready & relevant) continue;  // spin until the window is published
        unsigned long long val = (lane <= first_pre) ? (s & kScanVal) : 0ULL;
        excl += warp_sum(val);
        if (first_pre < 32) break;
        p -= 32;
      }
      if (lane == 0) st_volatile(&ws.status[part], kScanPre | (excl + agg));
    }
    if (lane == 0) {
      s_prefix = excl;
      if (part == nparts - 1) {
        if (total) *total = excl + agg;
        op.finish(excl + agg);  // the scan's total, once (the last partition)
      }
    }
  }
  __syncthreads();
  const unsigned long long base = s_prefix + s_warp[warp];
#pragma unroll
  for (int j = 0; j < kScanRounds; ++j) {
    const int64_t i = lbase + j;
    if (i < n) op.store(i, base + ex[j], v[j]);
  }
}

// The byte range a scan's launch zeroes (status words + counter).
struct ZeroSpan {
  void* p;
  size_t bytes;
};
inline ZeroSpan scan_state_span(const ScanWs& ws) {
  return {ws.status, static_cast<size_t>(reinterpret_cast<const char*>(ws.counter + 1) -
                                         reinterpret_cast<const char*>(ws.status))};
}

template <class Op, int ROUNDS = kScanRounds>
int launch_scan(Op op, const unsigned long long* n_dev, int64_t n_host, int64_t n_cap,
                const ScanWs& ws, unsigned long long* total, cudaStream_t st,
                bool state_ready = false) {
  const int64_t parts = ceil_div(n_cap > 0 ? n_cap : 1, kScanWarps * ROUNDS * 32);
  if (parts > ws.max_parts) {
    set_error("scan: workspace too small");
    return CGS_EINTERNAL;
  }
  // status words and counter are carved back to back: one memset node, none
  // when an earlier kernel zeroed them (state_ready: scan_state_span)
  if (!state_ready)
  CGS_CUDA(cudaMemsetAsync(ws.status, 0,
                           reinterpret_cast<const char*>(ws.counter + 1) -
                               reinterpret_cast<const char*>(ws.status),
                           st));
  CGS_PROFILED("scan_kernel", st, scan_kernel<Op, ROUNDS><<<static_cast<unsigned>(parts), 256, 0, st>>>(op, n_dev, n_host, ws, total));
  CGS_CHECK_LAUNCH("scan_kernel");
  return CGS_OK;
}

// ===========================================================================
// Onesweep LSD radix sort, 8-bit digits.  One histogram kernel for all
// passes, then one kernel per pass: per-warp ballot ranking (stable),
// per-digit decoupled lookback across partitions, smem reorder, coalesced
// scatter.  Status words: 30-bit count, flag in bits 30..31.
// ===========================================================================
// Two partition shapes, chosen from the sort's capacity: 8 warps x 16 keys
// (4096 per partition) for small sorts, 16 warps x 12 keys (6144) for large
// ones (capacity above 4 M) -- twice the resident warps per SM and fewer partitions on the
// decoupled lookback (bench_tools/sort_bench.cu: a 12.2 M-pair tile sort
// 342 -> 311 us, 18.5 M 478 -> 444 us; the small config-1 sorts keep 8 x 16).
#ifndef CGS_SORT_WARPS
#define CGS_SORT_WARPS 8
#endif
#ifndef CGS_SORT_LARGE_WARPS
#define CGS_SORT_LARGE_WARPS 16
#endif
#ifndef CGS_SORT_LARGE_ITEMS
#define CGS_SORT_LARGE_ITEMS 12
#endif
#ifndef CGS_SORT_BACKOFF
#define CGS_SORT_BACKOFF 0  // ns; 0: spin
#endif
#ifndef CGS_SORT_LARGE_N
#define CGS_SORT_LARGE_N (4 << 20)
#endif
constexpr int kSortWarps = CGS_SORT_WARPS;  // >= 8: the first 8 warps own the 256 digits
constexpr int kSortThreads = kSortWarps * 32;
#ifndef CGS_SORT_ITEMS
#define CGS_SORT_ITEMS 16
#endif
constexpr int kSortItems = CGS_SORT_ITEMS;
constexpr int kSortTile = kSortWarps * 32 * kSortItems;  // 4096
constexpr int kSortLargeWarps = CGS_SORT_LARGE_WARPS, kSortLargeItems = CGS_SORT_LARGE_ITEMS;
inline bool sort_large(int64_t n_cap) { return n_cap > CGS_SORT_LARGE_N; }
inline int64_t sort_tile_for(int64_t n_cap) {
  return sort_large(n_cap) ? kSortLargeWarps * 32 * kSortLargeItems : kSortTile;
}
constexpr unsigned kSortAgg = 1u << 30;
constexpr unsigned kSortPre = 2u << 30;
constexpr unsigned kSortVal = (1u << 30) - 1;

template <typename K>
struct SortWs {
  K* keys_alt;
  uint32_t* vals_alt;
  uint32_t* hist;     // passes * 256
  uint32_t* status;   // passes * max_parts * 256
  unsigned* counter;  // passes
  int64_t max_parts;
  int passes_cap;
};

template <typename K>
inline size_t sort_ws_bytes(int64_t n_cap) {
  const int64_t parts = ceil_div(n_cap > 0 ? n_cap : 1, sort_tile_for(n_cap));
  const int passes = static_cast<int>(sizeof(K));
  return align_up(n_cap * sizeof(K)) + align_up(n_cap * sizeof(uint32_t)) +
         align_up(passes * 256 * 4) + align_up(passes * parts * 256 * 4) + 256 + 4 * 256;
}

template <typename K>
inline SortWs<K> carve_sort(Carver& c, int64_t n_cap) {
  SortWs<K> w;
  w.max_parts = ceil_div(n_cap > 0 ? n_cap : 1, sort_tile_for(n_cap));
  w.passes_cap = static_cast<int>(sizeof(K));
  w.keys_alt = c.take<K>(n_cap > 0 ? n_cap : 1);
  w.vals_alt = c.take<uint32_t>(n_cap > 0 ? n_cap : 1);
  w.hist = c.take<uint32_t>(w.passes_cap * 256);
  w.status = c.take<uint32_t>(static_cast<size_t>(w.passes_cap) * w.max_parts * 256);
  w.counter = c.take<unsigned>(64);
  return w;
}

template <typename K>
__global__ void __launch_bounds__(256) sort_hist_kernel(const K* __restrict__ keys,
                                                        const unsigned long long* n_dev,
                                                        int64_t n_host, int key_bits,
                                                        uint32_t* __restrict__ hist) {
  const int passes = (key_bits + 7) / 8;
  __shared__ uint32_t s_h[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const int64_t n = dev_count(n_dev, n_host);
  // warp-aggregated (ballot peers): skewed digits, e.g. the exponent byte of
  // depths, would otherwise serialise 32 lanes on one shared counter
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x); b < n;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = b + threadIdx.x;
    const bool ok = i < n;
    const uint64_t k = ok ? static_cast<uint64_t>(keys[i]) : 0ULL;
    const unsigned valid = __ballot_sync(kFull, ok);
    for (int p = 0; p < passes; ++p) {
      const int db = key_bits - 8 * p < 8 ? key_bits - 8 * p : 8;
      const unsigned d = static_cast<unsigned>((k >> (8 * p)) & ((1u << db) - 1u));
      const unsigned peers = warp_peers8(d) & valid;
      if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&s_h[p * 256 + d], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
    if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
}

#ifdef CGS_SORT_TRACE
__device__ unsigned long long* g_sort_trace;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SORT_TRACE(part, i) \
  if (threadIdx.x == 0 && g_sort_trace) g_sort_trace[(part) * 5 + (i)] = gtimer()
#else
#define SORT_TRACE(part, i)
#endif

template <typename K, int WARPS, int ITEMS>
struct SortSmem {
  uint32_t wcnt[WARPS * 256];
  uint32_t dstart[256];
  int32_t goff[256];
  uint32_t scan_tmp[WARPS];
  unsigned part;
  K keys[WARPS * 32 * ITEMS];
  uint32_t vals[WARPS * 32 * ITEMS];
};

#ifndef CGS_SORT_EARLY_SCATTER
#define CGS_SORT_EARLY_SCATTER 1
#endif
template <typename K, int WARPS, int ITEMS>
__global__ void __launch_bounds__(WARPS * 32, 2) onesweep_kernel(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
    const unsigned long long* n_dev, int64_t n_host, int shift, int digit_bits,
    const uint32_t* __restrict__ hist, uint32_t* status, unsigned* counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  static_assert(WARPS >= 8 && WARPS % 8 == 0, "digit phase: 256 digit-owning threads");
  constexpr int kThreads = WARPS * 32, kTile = kThreads * ITEMS;
  SortSmem<K, WARPS, ITEMS>& S = *reinterpret_cast<SortSmem<K, WARPS, ITEMS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned dmask = (1u << digit_bits) - 1u;  // only the low key_bits are sorted on
  auto digit_of = [&](K k) -> unsigned {
    if constexpr (sizeof(K) <= 4) return (static_cast<uint32_t>(k) >> shift) & dmask;
    else return static_cast<unsigned>((static_cast<uint64_t>(k) >> shift) & dmask);
  };
  if (tid == 0) S.part = atomicAdd(counter, 1u);
  for (int i = tid; i < WARPS * 256; i += kThreads) S.wcnt[i] = 0;
  __syncthreads();
  const int64_t part = S.part;
  const int64_t n = dev_count(n_dev, n_host);
  const int64_t nparts = ceil_div(n, kTile);
  if (part >= nparts) return;
  const int64_t base = part * kTile;
  const int64_t wbase = base + static_cast<int64_t>(warp) * 32 * ITEMS;
  SORT_TRACE(part, 0);

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t rank[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int64_t i = wbase + j * 32 + lane;
    const bool ok = i < n;
    key[j] = ok ? keys_in[i] : static_cast<K>(~static_cast<K>(0));
    val[j] = ok ? vals_in[i] : 0u;
  }
#ifdef CGS_SORT_TRACE
  {
    uint32_t sink = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) sink += static_cast<uint32_t>(key[j]) + val[j];
    if (sink == 0x12345678u) g_sort_trace[0] = 0;
    SORT_TRACE(part, 1);
  }
#endif
  uint32_t* wc = S.wcnt + warp * 256;
  // ranking within the warp, in item order; the full-byte case (every pass
  // but a narrow last one) has its 8 ballots unrolled without the per-bit
  // width test
  auto rank_all = [&](auto peers_of) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const unsigned d = digit_of(key[j]);
      const unsigned peers = peers_of(d);
      const unsigned before = wc[d];
      rank[j] = before + __popc(peers & lanemask_lt());
      __syncwarp();
      if (lane == __ffs(peers) - 1) wc[d] = before + __popc(peers);
      __syncwarp();
    }
  };
  if (digit_bits == 8)
    rank_all([](unsigned d) { return warp_peers8(d); });
  else
    rank_all([&](unsigned d) { return warp_peers_bits(d, digit_bits); });
  __syncthreads();
  SORT_TRACE(part, 2);
  // thread tid < 256 owns digit d = tid: exclusive over warps, then over
  // digits (whole warps 0-7; the others only pass the barriers)
  const bool owner = tid < 256;
  const int d = owner ? tid : 255;
  uint32_t cnt = 0;
  if (owner) {
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = S.wcnt[w * 256 + d];
      S.wcnt[w * 256 + d] = cnt;
      cnt += c;
    }
  }
  {
    const uint32_t inc = owner ? warp_incl_scan(cnt) : 0u;
    if (owner && lane == 31) S.scan_tmp[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < warp && w < 8; ++w) wpre += S.scan_tmp[w];
    if (owner) S.dstart[d] = wpre + inc - cnt;
  }
  // global digit base = exclusive scan of the pass histogram
  const uint32_t h = owner ? hist[d] : 0u;
  uint32_t gbase;
  {
    __syncthreads();
    const uint32_t inc = owner ? warp_incl_scan(h) : 0u;
    if (owner && lane == 31) S.scan_tmp[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < warp && w < 8; ++w) wpre += S.scan_tmp[w];
    gbase = wpre + inc - h;
  }
  // decoupled lookback for digit d over previous partitions: publish this
  // partition's count first, reorder the tile in shared memory (local ranks
  // only; frees the key / value / rank registers before the lookback window
  // is loaded), then walk back
  const int64_t tail = base + kTile - n;
  const uint32_t agg = cnt - ((d == 255 && tail > 0) ? static_cast<uint32_t>(tail) : 0u);
  uint32_t excl = 0;
  uint32_t* st = status + part * 256 + d;
  if (owner) st_volatile(st, (part == 0 ? kSortPre : kSortAgg) | agg);
#if CGS_SORT_EARLY_SCATTER
  __syncthreads();  // dstart complete
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const unsigned dd = digit_of(key[j]);
    const uint32_t pos = S.dstart[dd] + wc[dd] + rank[j];
    S.keys[pos] = key[j];
    S.vals[pos] = val[j];
  }
#endif
  if (owner && part != 0) {
    // Windowed lookback: kLookback independent status loads per round trip,
    // consumed in order until an inclusive prefix is found (an unpublished
    // slot makes the next window start there).  All partitions start
    // together, so partition p typically walks back ~p slots before it meets
    // an inclusive prefix: the window width sets the number of L2 round trips.
#ifndef CGS_SORT_LOOKBACK
#define CGS_SORT_LOOKBACK 16
#endif
    constexpr int kLookback = CGS_SORT_LOOKBACK;
    int64_t p = part - 1;
    bool done = false;
    while (!done) {
      uint32_t s[kLookback];
#pragma unroll
      for (int k = 0; k < kLookback; ++k)
        s[k] = (p - k >= 0) ? ld_volatile(status + (p - k) * 256 + d) : kSortPre;
      int k = 0;
      for (; k < kLookback; ++k) {
        const uint32_t flag = s[k] >> 30;
        if (flag == 0) break;
        excl += s[k] & kSortVal;
        if (flag == 2) {
          done = true;
          break;
        }
      }
      p -= k;
#if CGS_SORT_BACKOFF
      // no progress (the next slot is unpublished): back off before
      // re-polling, so spinning partitions do not steal issue slots and L2
      // bandwidth from the ones they wait for
      if (!done && k == 0) __nanosleep(CGS_SORT_BACKOFF);
#endif
    }
    st_volatile(st, kSortPre | (excl + agg));
  }
  if (owner) S.goff[d] = static_cast<int32_t>(gbase + excl) - static_cast<int32_t>(S.dstart[d]);
  __syncthreads();
  SORT_TRACE(part, 3);
#if !CGS_SORT_EARLY_SCATTER
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const unsigned dd = digit_of(key[j]);
    const uint32_t pos = S.dstart[dd] + wc[dd] + rank[j];
    S.keys[pos] = key[j];
    S.vals[pos] = val[j];
  }
  __syncthreads();
#endif
  const int nvalid = static_cast<int>(n - base < kTile ? n - base : kTile);
  for (int i = tid; i < nvalid; i += kThreads) {
    const K k = S.keys[i];
    const unsigned dd = digit_of(k);
    const int64_t o = static_cast<int64_t>(S.goff[dd]) + i;
    keys_out[o] = k;
    vals_out[o] = S.vals[i];
  }
  SORT_TRACE(part, 4);
}

// Sorts (keys, vals) of length n (device count n_dev if non-null, else
// n_host; n_cap bounds it) on the low key_bits.  Returns, through
// out_keys/out_vals, the buffers holding the result (the inputs or the
// workspace alternates, depending on the pass count).
// The byte range a sort's launch zeroes (status words + counters).
template <typename K>
inline ZeroSpan sort_state_span(const SortWs<K>& ws) {
  return {ws.status, static_cast<size_t>(reinterpret_cast<const char*>(ws.counter + 64) -
                                         reinterpret_cast<const char*>(ws.status))};
}

template <typename K>
int launch_radix_sort(K* keys, uint32_t* vals, const unsigned long long* n_dev, int64_t n_host,
                      int64_t n_cap, int key_bits, const SortWs<K>& ws, K** out_keys,
                      uint32_t** out_vals, cudaStream_t st, bool hist_ready = false,
                      bool state_ready = false) {
  int passes = (key_bits + 7) / 8;
  if (passes < 1) passes = 1;
  if (passes > ws.passes_cap) return CGS_EINVAL;
  if (!hist_ready) CGS_CUDA(cudaMemsetAsync(ws.hist, 0, passes * 256 * sizeof(uint32_t), st));
  // status words and the partition counters are carved back to back: one
  // memset node for both (a graph's memset nodes cost ~2-3 us each), none
  // when an earlier kernel zeroed them (state_ready: sort_state_span)
  if (!state_ready)
  CGS_CUDA(cudaMemsetAsync(ws.status, 0,
                           reinterpret_cast<const char*>(ws.counter + 64) -
                               reinterpret_cast<const char*>(ws.status),
                           st));
  if (!hist_ready) {  // else the producer of the keys already filled ws.hist
    CGS_PROFILED("sort_hist_kernel", st, sort_hist_kernel<K><<<grid_for(n_cap, 256, 4), 256, 0, st>>>(keys, n_dev, n_host, key_bits, ws.hist));
    CGS_CHECK_LAUNCH("sort_hist_kernel");
  }
  static bool attr_set[kMaxDevices] = {};  // per device ordinal
  using SmallSmem = SortSmem<K, kSortWarps, kSortItems>;
  using LargeSmem = SortSmem<K, kSortLargeWarps, kSortLargeItems>;
  const bool large = sort_large(n_cap);
  const size_t smem = large ? sizeof(LargeSmem) : sizeof(SmallSmem);
  int dev = 0;
  if (int rc = current_device(&dev)) return rc;
  if (!attr_set[dev]) {
    CGS_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, kSortWarps, kSortItems>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(SmallSmem))));
    CGS_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, kSortLargeWarps, kSortLargeItems>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(LargeSmem))));
    attr_set[dev] = true;
  }
  K* kin = keys;
  uint32_t* vin = vals;
  K* kout = ws.keys_alt;
  uint32_t* vout = ws.vals_alt;
  const unsigned grid = static_cast<unsigned>(ceil_div(n_cap > 0 ? n_cap : 1, sort_tile_for(n_cap)));
  auto kern = large ? onesweep_kernel<K, kSortLargeWarps, kSortLargeItems>
                    : onesweep_kernel<K, kSortWarps, kSortItems>;
  const int threads = large ? kSortLargeWarps * 32 : kSortThreads;
  for (int p = 0; p < passes; ++p) {
    const int dbits = key_bits - 8 * p < 8 ? key_bits - 8 * p : 8;
    CGS_PROFILED("onesweep_kernel", st, kern<<<grid, threads, smem, st>>>(kin, vin, kout, vout, n_dev, n_host, 8 * p, dbits,
                                                ws.hist + p * 256,
                                                ws.status + static_cast<size_t>(p) * ws.max_parts * 256,
                                                ws.counter + p));
    CGS_CHECK_LAUNCH("onesweep_kernel");
    K* tk = kin; kin = kout; kout = tk;
    uint32_t* tv = vin; vin = vout; vout = tv;
  }
  *out_keys = kin;
  *out_vals = vin;
  return CGS_OK;
}

}  // namespace cgs
