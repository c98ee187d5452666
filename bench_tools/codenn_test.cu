// Standalone check + timing of the tcgen05 distance GEMM (csrc/codenn.cuh):
// S = R R^T against an fp64 host product (tf32 tolerance), nearest rows
// against an fp64 host brute force, and the GEMM's TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        bench_tools/codenn_test.cu -o /tmp/codenn_test && /tmp/codenn_test
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../paper_2509_03775_b200/csrc/codenn.cuh"

namespace cgs {
void set_error(const std::string& m) { fprintf(stderr, "%s\n", m.c_str()); }
int cuda_status(cudaError_t e, const char* w) {
  fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e));
  return 2;
}
void note_launch() {}
}  // namespace cgs

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

using namespace cgs;

static int run(int cap, int d, int n_dead, bool dupes, bool check_s, int reps, bool check_nn = true) {
  std::vector<float> rows(static_cast<size_t>(cap) * d);
  uint64_t x = 0x9E3779B97F4A7C15ull ^ (cap * 131 + d);
  auto nrm = [&]() {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    double u1 = ((x >> 11) + 0.5) / 9007199254740992.0;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    double u2 = ((x >> 11) + 0.5) / 9007199254740992.0;
    return std::sqrt(-2 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  };
  for (auto& v : rows) v = static_cast<float>(0.2 * nrm());
  if (dupes)
    for (int r = 10; r < cap; r += 97) for (int k = 0; k < d; ++k) rows[r * d + k] = rows[(r - 7) * d + k];
  std::vector<int> live;
  for (int r = 0; r < cap; ++r) if (!(n_dead && r % (cap / n_dead + 1) == 3)) live.push_back(r);
  const int64_t n_live = live.size();
  const int dp = nn_dpad(d);
  const int64_t mpad = (n_live + kNnN - 1) / kNnN * kNnN;
  float *d_rows, *packed, *norms, *cand_d, *dbg = nullptr;
  int32_t *d_live, *cand_j, *nn_idx, *redo;
  double* nn_dist;
  unsigned* ctr;
  CK(cudaMalloc(&d_rows, rows.size() * 4));
  CK(cudaMalloc(&d_live, n_live * 4));
  CK(cudaMalloc(&packed, 2 * mpad * dp * 4));
  CK(cudaMalloc(&norms, mpad * 4));
  CK(cudaMalloc(&cand_d, mpad * kNnCand * 4));
  CK(cudaMalloc(&cand_j, mpad * kNnCand * 4));
  CK(cudaMalloc(&nn_idx, cap * 4));
  CK(cudaMalloc(&nn_dist, cap * 8));
  CK(cudaMalloc(&redo, n_live * 4));
  CK(cudaMalloc(&ctr, 8));
  if (check_s) CK(cudaMalloc(&dbg, mpad * mpad * 4));
  CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_live, live.data(), n_live * 4, cudaMemcpyHostToDevice));
  size_t smem = codenn_gemm_smem(dp);
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM (it takes all 512 TMEM columns)
  CK(cudaFuncSetAttribute(codenn_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < reps; ++rep) {
    CK(cudaMemset(ctr, 0, 8));
    CK(cudaMemset(nn_idx, 0xff, cap * 4));
    codenn_pack_kernel<<<256, 256>>>(d_rows, d, d_live, n_live, mpad, dp, packed, norms, ctr + 1);
    CK(cudaGetLastError());
    cudaEventRecord(a);
    codenn_gemm_kernel<<<mpad / kNnM, kNnThreads, smem>>>(packed, norms, mpad, dp, cand_d, cand_j, rep == 0 ? dbg : nullptr);
    cudaEventRecord(b);
    CK(cudaGetLastError());
    codenn_refine_kernel<<<256, 256>>>(d_rows, d, d_live, n_live, norms, ctr + 1, cand_d, cand_j, nn_idx, nn_dist, redo, ctr);
    codenn_bruteforce_kernel<<<592, 256>>>(d_rows, d, d_live, n_live, redo, ctr, nn_idx, nn_dist);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 || reps == 1) best = std::min(best, ms);
  }
  if (reps > 1) {  // per-tile timeline of CTA 0 (last rep)
    unsigned long long* tr;
    CK(cudaMalloc(&tr, 1024 * 8));
    CK(cudaMemset(tr, 0, 1024 * 8));
    codenn_gemm_kernel<<<mpad / kNnM, kNnThreads, smem>>>(packed, norms, mpad, dp, cand_d, cand_j, nullptr, tr);
    CK(cudaDeviceSynchronize());
    unsigned long long h[1024];
    CK(cudaMemcpy(h, tr, 1024 * 8, cudaMemcpyDeviceToHost));
    const unsigned long long t0 = h[3];
    printf("  CTA0 timeline (us from first B issue): tile: producer-issue / mma-start / epi-start / epi-end\n");
    for (int t : {0, 1, 2, 5, 10, 30, 63, 127, 255}) if (t < 256 && h[4 * t])
      printf("   t=%d: %.2f / %.2f / %.2f / %.2f\n", t, (h[4 * t + 3] - t0) / 1e3, (h[4 * t] - t0) / 1e3,
             (h[4 * t + 1] - t0) / 1e3, (h[4 * t + 2] - t0) / 1e3);
    CK(cudaFree(tr));
  }
  unsigned h_ctr[2];
  CK(cudaMemcpy(h_ctr, ctr, 8, cudaMemcpyDeviceToHost));
  int bad_s = 0;
  double max_rel = 0;
  if (check_s) {
    std::vector<float> S(mpad * mpad);
    CK(cudaMemcpy(S.data(), dbg, S.size() * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n_live; i += (n_live > 600 ? 7 : 1))
      for (int64_t j = 0; j < n_live; ++j) {
        double s = 0, sa = 0;
        for (int k = 0; k < d; ++k) {
          s += (double)rows[live[i] * d + k] * rows[live[j] * d + k];
          sa += std::fabs((double)rows[live[i] * d + k] * rows[live[j] * d + k]);
        }
        const double err = std::fabs(S[i * mpad + j] - s);
        max_rel = std::max(max_rel, err / (sa + 1e-30));
        if (err > 1e-4 * sa + 1e-7) { if (bad_s < 5) printf("  S[%lld,%lld] = %g, want %g\n", (long long)i, (long long)j, S[i * mpad + j], s); ++bad_s; }
      }
  }
  std::vector<int32_t> got(cap);
  std::vector<double> gotd(cap);
  CK(cudaMemcpy(got.data(), nn_idx, cap * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(gotd.data(), nn_dist, cap * 8, cudaMemcpyDeviceToHost));
  int bad = 0;
  std::vector<char> is_live(cap, 0);
  for (int r : live) is_live[r] = 1;
  for (int i = 0; i < (check_nn ? cap : 0); ++i) {
    int want = -1;
    double wd = INFINITY;
    if (is_live[i])
      for (int j : live) {
        if (j == i) continue;
        double s = 0;
        for (int k = 0; k < d; ++k) { volatile double t = (double)rows[i * d + k] - rows[j * d + k]; volatile double t2 = t * t; s = s + t2; }
        if (s < wd) { wd = s; want = j; }
      }
    if (got[i] != want || (want >= 0 && gotd[i] != wd)) {
      if (bad < 5) printf("  row %d: got %d (%g), want %d (%g)\n", i, got[i], gotd[i], want, wd);
      ++bad;
    }
  }
  const double flops = 2.0 * mpad * mpad * dp;
  printf("cap=%d d=%d live=%lld dupes=%d: S check %s (max rel %.2e), nn %s (%d bad), redo %u rows; "
         "%s gemm %.1f us, %.1f TFLOP/s (tf32, padded)\n",
         cap, d, (long long)n_live, dupes, check_s ? (bad_s ? "FAIL" : "ok") : "skipped", max_rel,
         check_nn ? (bad ? "FAIL" : "ok") : "unchecked", bad, h_ctr[0], "", best * 1000, flops / (best * 1e-3) / 1e12);
  return bad || bad_s;
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  int fails = 0;
  fails += run(600, 48, 0, false, true, 1);
  fails += run(1000, 48, 37, true, true, 1);
  fails += run(3000, 7, 50, true, true, 1);
  fails += run(2000, 12, 10, false, true, 1);
  fails += run(4096, 48, 0, false, false, 3);
  fails += run(16384, 48, 0, false, false, 3, false);
  fails += run(65536, 48, 0, false, false, 3, false);
  printf(fails ? "FAILURES\n" : "ALL OK\n");
  return fails ? 1 : 0;
}
