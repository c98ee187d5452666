// Standalone timing of the radix sort / scan primitives (sort_scan.cuh) at
// the sizes of the frame pipeline.  nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -I include bench_tools/sort_bench.cu -o bench_tools/sort_bench
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "../paper_2509_03775_b200/csrc/sort_scan.cuh"

namespace cgs {
void set_error(const std::string& m) { fprintf(stderr, "%s\n", m.c_str()); }
int cuda_status(cudaError_t e, const char* w) {
  fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e));
  return 2;
}
void note_launch() {}
int current_device(int* dev) {
  cudaGetDevice(dev);
  return 0;
}
ProfScope::ProfScope(const char*, cudaStream_t s) : on(false), st(s) {}
ProfScope::~ProfScope() {}
}  // namespace cgs

template <typename K>
static void run(int64_t n, int bits, int reps) {
  using namespace cgs;
  std::vector<K> hk(n);
  std::vector<uint32_t> hv(n);
  uint64_t x = 88172645463325252ULL;
  for (int64_t i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    hk[i] = static_cast<K>(x & ((bits >= 64) ? ~0ULL : ((1ULL << bits) - 1)));
    hv[i] = static_cast<uint32_t>(i);
  }
  K* dk; uint32_t* dv; K* k0; uint32_t* v0;
  cudaMalloc(&dk, n * sizeof(K)); cudaMalloc(&dv, n * 4);
  cudaMalloc(&k0, n * sizeof(K)); cudaMalloc(&v0, n * 4);
  cudaMemcpy(k0, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice);
  cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
  size_t wsb = sort_ws_bytes<K>(n) + 4096;
  void* ws; cudaMalloc(&ws, wsb);
  Carver c(ws, wsb);
  SortWs<K> w = carve_sort<K>(c, n);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  K* ko; uint32_t* vo;
  float best = 1e9;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpyAsync(dk, k0, n * sizeof(K), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(dv, v0, n * 4, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(a, st);
    launch_radix_sort<K>(dk, dv, nullptr, n, n, bits, w, &ko, &vo, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
#ifdef CGS_SORT_TRACE
  {
    const int64_t parts = ceil_div(n, sort_tile_for(n));
    unsigned long long* tr;
    cudaMalloc(&tr, parts * 5 * sizeof(unsigned long long));
    cudaMemset(tr, 0, parts * 5 * sizeof(unsigned long long));
    cudaMemcpyToSymbol(g_sort_trace, &tr, sizeof(tr));
    cudaMemcpyAsync(dk, k0, n * sizeof(K), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(dv, v0, n * 4, cudaMemcpyDeviceToDevice, st);
    launch_radix_sort<K>(dk, dv, nullptr, n, n, bits, w, &ko, &vo, st);  // last pass traced
    cudaStreamSynchronize(st);
    std::vector<unsigned long long> h(parts * 5);
    cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ULL, t4 = 0;
    double ph[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
    for (int64_t p = 0; p < parts; ++p) {
      t0 = std::min(t0, h[p * 5]);
      t4 = std::max(t4, h[p * 5 + 4]);
      for (int q = 0; q < 4; ++q) {
        const double d = double(h[p * 5 + q + 1] - h[p * 5 + q]);
        ph[q] += d / parts;
        mx[q] = std::max(mx[q], d);
      }
    }
    printf("  trace (last pass, ns): span %.0f; load %.0f/%.0f rank %.0f/%.0f scan+lookback %.0f/%.0f "
           "scatter %.0f/%.0f (mean/max)\n", double(t4 - t0), ph[0], mx[0], ph[1], mx[1], ph[2],
           mx[2], ph[3], mx[3]);
    unsigned long long* z = nullptr;
    cudaMemcpyToSymbol(g_sort_trace, &z, sizeof(z));
    cudaFree(tr);
  }
#endif
  // the same without the histogram kernel (the frame pipeline fuses the
  // digit histograms into the projection / emission kernels)
  float nohist = 1e9;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpyAsync(dk, k0, n * sizeof(K), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(dv, v0, n * 4, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(a, st);
    launch_radix_sort<K>(dk, dv, nullptr, n, n, bits, w, &ko, &vo, st, /*hist_ready=*/true);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < nohist) nohist = ms;
  }
  printf("  passes only (histogram precomputed, as in the pipeline): %.1f us\n", nohist * 1000);
  cudaMemcpyAsync(dk, k0, n * sizeof(K), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(dv, v0, n * 4, cudaMemcpyDeviceToDevice, st);
  launch_radix_sort<K>(dk, dv, nullptr, n, n, bits, w, &ko, &vo, st);
  cudaStreamSynchronize(st);
  std::vector<K> rk(n); std::vector<uint32_t> rv(n);
  cudaMemcpy(rk.data(), ko, n * sizeof(K), cudaMemcpyDeviceToHost);
  cudaMemcpy(rv.data(), vo, n * 4, cudaMemcpyDeviceToHost);
  bool ok = true;
  for (int64_t i = 1; i < n; ++i)
    if (rk[i - 1] > rk[i] || (rk[i - 1] == rk[i] && rv[i - 1] > rv[i])) { ok = false; break; }
  // CUB (the CUDA toolkit's DeviceRadixSort::SortPairs, stable LSD onesweep)
  // on the same keys / values and bit range, for comparison
  float cub_best = 1e9;
  {
    K* ck; uint32_t* cv;
    cudaMalloc(&ck, n * sizeof(K)); cudaMalloc(&cv, n * 4);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, ck, v0, cv, static_cast<int>(n), 0, bits, st);
    void* tmp; cudaMalloc(&tmp, tb);
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(a, st);
      cub::DeviceRadixSort::SortPairs(tmp, tb, k0, ck, v0, cv, static_cast<int>(n), 0, bits, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r > 0 && ms < cub_best) cub_best = ms;
    }
    std::vector<K> ck_h(n);
    cudaMemcpy(ck_h.data(), ck, n * sizeof(K), cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < n; ++i)
      if (ck_h[i] != rk[i]) { ok = false; break; }
    cudaFree(ck); cudaFree(cv); cudaFree(tmp);
  }
  const double bytes = 2.0 * n * (sizeof(K) + 4) * ((bits + 7) / 8);  // read + write per pass
  printf("n=%9lld key=%zuB bits=%2d passes=%d  ours %8.1f us (%.1f us/pass, %.2f TB/s)  "
         "CUB %8.1f us (%.2f TB/s)  %s\n", (long long)n, sizeof(K), bits, (bits + 7) / 8,
         best * 1000, best * 1000 / ((bits + 7) / 8), bytes / (best * 1e-3) / 1e12, cub_best * 1000,
         2.0 * n * (sizeof(K) + 4) * ((bits + 7) / 8) / (cub_best * 1e-3) / 1e12,
         ok ? "sorted+stable, same keys as CUB" : "WRONG");
  cudaFree(dk); cudaFree(dv); cudaFree(k0); cudaFree(v0); cudaFree(ws);
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  // the frame pipeline's sorts: depth keys (24 bits) of the on-screen splats
  // and tile keys of the pairs, at configs 1 / 3 / 4
  if (only < 0 || only == 0) run<uint32_t>(350000, 24, 20);     // config 1 depth
  if (only < 0 || only == 1) run<uint16_t>(1070000, 10, 20);    // config 1 tiles
  if (only < 0 || only == 2) run<uint32_t>(2950000, 24, 10);    // config 3 depth
  if (only < 0 || only == 3) run<uint16_t>(12200000, 14, 10);   // config 3 tiles
  if (only < 0 || only == 4) run<uint32_t>(4400000, 24, 10);    // config 4 depth
  if (only < 0 || only == 5) run<uint16_t>(18500000, 13, 10);   // config 4 tiles
  if (only < 0 || only == 6) run<uint32_t>(16000000, 32, 10);   // large, full 32-bit keys
  return 0;
}
