// Launch-overhead probe: back-to-back durations of empty kernels with and
// without a large dynamic shared-memory request, and of the onesweep passes
// one by one, each bracketed by CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        bench_tools/launch_probe.cu -o /tmp/launch_probe
#include <cstdio>
#include <string>
#include <vector>

#include "../paper_2509_03775_b200/csrc/sort_scan.cuh"

namespace cgs {
void set_error(const std::string& m) { fprintf(stderr, "%s\n", m.c_str()); }
int cuda_status(cudaError_t e, const char* w) {
  fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e));
  return 2;
}
void note_launch() {}
ProfScope::ProfScope(const char*, cudaStream_t s) : on(false), st(s) {}
ProfScope::~ProfScope() {}
}  // namespace cgs

__global__ void empty_kernel(int* p) {
  extern __shared__ int sm[];
  if (p && threadIdx.x == 0 && blockIdx.x == 0x7fffffff) p[0] = sm[0];
}

__global__ void marker_kernel(unsigned long long* t, int i) {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  t[i] = g;
}

__global__ void small_smem_kernel(int* p) {
  __shared__ int s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && blockIdx.x == 0x7fffffff) p[0] = s[(threadIdx.x + 1) & 255];
}

template <typename F>
static float time_us(cudaStream_t st, int reps, F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaStreamSynchronize(st);
  cudaEventRecord(a, st);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1000.0f * ms / reps;
}

int main() {
  using namespace cgs;
  cudaStream_t st;
  cudaStreamCreate(&st);
  const int dyn = 41 * 1024;
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  printf("empty 98x256, no smem:            %.2f us/launch\n",
         time_us(st, 200, [&] { empty_kernel<<<98, 256, 0, st>>>(nullptr); }));
  printf("empty 98x256, 41 KB dyn smem:     %.2f us/launch\n",
         time_us(st, 200, [&] { empty_kernel<<<98, 256, dyn, st>>>(nullptr); }));
  printf("alternating 4 KB static / 41 KB:  %.2f us/pair\n", time_us(st, 200, [&] {
           small_smem_kernel<<<1563, 256, 0, st>>>(nullptr);
           empty_kernel<<<98, 256, dyn, st>>>(nullptr);
         }));
  printf("4 KB static alone 1563x256:       %.2f us/launch\n",
         time_us(st, 200, [&] { small_smem_kernel<<<1563, 256, 0, st>>>(nullptr); }));

  // onesweep passes one at a time, n = 400k random 32-bit keys
  const int64_t n = 400000;
  std::vector<uint32_t> hk(n), hv(n);
  uint64_t x = 88172645463325252ULL;
  for (int64_t i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    hk[i] = static_cast<uint32_t>(x);
    hv[i] = static_cast<uint32_t>(i);
  }
  uint32_t *dk, *dv;
  cudaMalloc(&dk, n * 4);
  cudaMalloc(&dv, n * 4);
  cudaMemcpy(dk, hk.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), n * 4, cudaMemcpyHostToDevice);
  size_t wsb = sort_ws_bytes<uint32_t>(n) + 4096;
  void* ws;
  cudaMalloc(&ws, wsb);
  Carver c(ws, wsb);
  SortWs<uint32_t> w = carve_sort<uint32_t>(c, n);
  const size_t smem = sizeof(SortSmem<uint32_t>);
  cudaFuncSetAttribute(onesweep_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaMemsetAsync(w.hist, 0, 4 * 256 * 4, st);
  sort_hist_kernel<uint32_t><<<grid_for(n, 256, 4), 256, 0, st>>>(dk, nullptr, n, 32, w.hist);
  cudaMemsetAsync(w.status, 0, 4 * w.max_parts * 256 * 4, st);
  cudaMemsetAsync(w.counter, 0, 64 * 4, st);
  const unsigned grid = static_cast<unsigned>(ceil_div(n, kSortTile));
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  uint32_t *ki = dk, *vi = dv, *ko = w.keys_alt, *vo = w.vals_alt;
  cudaStreamSynchronize(st);
  cudaEventRecord(ev[0], st);
  for (int p = 0; p < 4; ++p) {
    onesweep_kernel<uint32_t><<<grid, 256, smem, st>>>(ki, vi, ko, vo, nullptr, n, 8 * p, 8,
                                                       w.hist + p * 256,
                                                       w.status + static_cast<size_t>(p) * w.max_parts * 256,
                                                       w.counter + p);
    cudaEventRecord(ev[p + 1], st);
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  cudaEventSynchronize(ev[4]);
  for (int p = 0; p < 4; ++p) {
    float ms;
    cudaEventElapsedTime(&ms, ev[p], ev[p + 1]);
    printf("onesweep pass %d (n=400k, %u CTAs, %zu B smem): %.2f us\n", p, grid, smem, 1000 * ms);
  }
  // the same inside CUDA graphs (no host launch cost)
  auto graph_us = [&](int reps, auto body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < reps; ++r) body();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return 1000.0f * ms / reps;
  };
  printf("graph: empty 98x256 no smem:        %.2f us/kernel\n",
         graph_us(100, [&] { empty_kernel<<<98, 256, 0, st>>>(nullptr); }));
  printf("graph: empty 98x256 41 KB dyn:      %.2f us/kernel\n",
         graph_us(100, [&] { empty_kernel<<<98, 256, dyn, st>>>(nullptr); }));
  printf("graph: alternating 4 KB / 41 KB:    %.2f us/pair\n", graph_us(100, [&] {
           small_smem_kernel<<<1563, 256, 0, st>>>(nullptr);
           empty_kernel<<<98, 256, dyn, st>>>(nullptr);
         }));
  printf("graph: 4-pass onesweep (+2 memsets): %.2f us/sort\n", graph_us(10, [&] {
           cudaMemsetAsync(w.status, 0, 4 * w.max_parts * 256 * 4, st);
           cudaMemsetAsync(w.counter, 0, 64 * 4, st);
           uint32_t *a = dk, *b = dv, *c2 = w.keys_alt, *d2 = w.vals_alt;
           for (int p = 0; p < 4; ++p) {
             onesweep_kernel<uint32_t><<<grid, 256, smem, st>>>(a, b, c2, d2, nullptr, n, 8 * p, 8,
                 w.hist + p * 256, w.status + static_cast<size_t>(p) * w.max_parts * 256,
                 w.counter + p);
             std::swap(a, c2);
             std::swap(b, d2);
           }
         }));
#ifdef CGS_SORT_TRACE
  {  // where does a pass's duration go: marker -> first CTA start, last CTA end -> marker
    const int64_t parts = ceil_div(n, kSortTile);
    unsigned long long *tr, *mk;
    cudaMalloc(&tr, parts * 5 * 8);
    cudaMalloc(&mk, 16);
    cudaMemcpyToSymbol(g_sort_trace, &tr, sizeof(tr));
    for (int rep = 0; rep < 3; ++rep) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      cudaMemsetAsync(w.status, 0, 4 * w.max_parts * 256 * 4, st);
      cudaMemsetAsync(w.counter, 0, 64 * 4, st);
      marker_kernel<<<1, 1, 0, st>>>(mk, 0);
      onesweep_kernel<uint32_t><<<grid, 256, smem, st>>>(dk, dv, w.keys_alt, w.vals_alt, nullptr, n, 0, 8,
                                                         w.hist, w.status, w.counter);
      marker_kernel<<<1, 1, 0, st>>>(mk, 1);
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaStreamSynchronize(st);
      std::vector<unsigned long long> h(parts * 5), m(2);
      cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(m.data(), mk, 16, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ULL, t4 = 0;
      for (int64_t p = 0; p < parts; ++p) {
        t0 = std::min(t0, h[p * 5]);
        t4 = std::max(t4, h[p * 5 + 4]);
      }
      printf("marker->first CTA %.2f us, CTA span %.2f us, last CTA->marker %.2f us\n",
             (t0 - m[0]) / 1e3, (t4 - t0) / 1e3, (m[1] - t4) / 1e3);
    }
  }
#endif
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
