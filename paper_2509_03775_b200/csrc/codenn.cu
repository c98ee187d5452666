// Host side of the nearest-code search (codenn.cuh): workspace layout,
// launches and the C ABI entry points cgs_code_nn_workspace_bytes /
// cgs_code_nn.
#include <atomic>
#include "codenn.cuh"

#include <string>

#include "common.cuh"

namespace cgs {

struct NnLayout {
  float* packed;
  float* norms;
  float* cand_d;
  int32_t* cand_j;
  int32_t* redo;
  unsigned* ctr;  // [0] rows to redo, [1] max norm (float bits)
  size_t bytes;
};

static NnLayout plan_nn(void* base, size_t cap_bytes, int64_t n_live, int d) {
  NnLayout L{};
  Carver c(base, cap_bytes);
  const int dp = nn_dpad(d);
  const int64_t mpad = (n_live + kNnN - 1) / kNnN * kNnN;
  const int64_t m1 = mpad > 0 ? mpad : kNnN;
  L.packed = c.take<float>(2 * m1 * dp);  // tf32 heads, then tails
  L.norms = c.take<float>(m1);
  L.cand_d = c.take<float>(m1 * kNnCand);
  L.cand_j = c.take<int32_t>(m1 * kNnCand);
  L.redo = c.take<int32_t>(m1);
  L.ctr = c.take<unsigned>(64);
  L.bytes = c.off + 256;
  return L;
}

static int code_nn(const float* rows, int d, int64_t cap, const int32_t* live, int64_t n_live,
                   int32_t* nn_idx, double* nn_dist, void* ws, size_t ws_bytes, cudaStream_t st) {
  NnLayout L = plan_nn(ws, ws_bytes, n_live, d);
  if (L.bytes > ws_bytes || !ws) {
    set_error("code_nn workspace too small: need " + std::to_string(L.bytes));
    return CGS_EWORKSPACE;
  }
  CGS_CUDA(cudaMemsetAsync(nn_idx, 0xff, sizeof(int32_t) * cap, st));
  CGS_CUDA(cudaMemsetAsync(nn_dist, 0, sizeof(double) * cap, st));
  if (n_live < 2) return CGS_OK;
  const int dp = nn_dpad(d);
  const int64_t mpad = (n_live + kNnN - 1) / kNnN * kNnN;
  CGS_CUDA(cudaMemsetAsync(L.ctr, 0, 64 * sizeof(unsigned), st));
  codenn_pack_kernel<<<grid_for(mpad, 256, 4), 256, 0, st>>>(rows, d, live, n_live, mpad, dp,
                                                               L.packed, L.norms, L.ctr + 1);
  CGS_CHECK_LAUNCH("codenn_pack_kernel");
  // one CTA per SM: the kernel takes all 512 TMEM columns
  size_t smem = codenn_gemm_smem(dp);
  if (smem < 120 * 1024) smem = 120 * 1024;
  static std::atomic<size_t> attr[kMaxDevices] = {};  // per device ordinal
  int dev = 0;
  if (int rc = current_device(&dev)) return rc;
  if (attr[dev].load() < smem) {
    CGS_CUDA(cudaFuncSetAttribute(codenn_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    attr[dev].store(smem);
  }
  CGS_PROFILED("codenn_gemm_kernel", st,
               codenn_gemm_kernel<<<static_cast<unsigned>(mpad / kNnM), kNnThreads, smem, st>>>(
                   L.packed, L.norms, mpad, dp, L.cand_d, L.cand_j, nullptr, nullptr));
  CGS_CHECK_LAUNCH("codenn_gemm_kernel");
  codenn_refine_kernel<<<grid_for(n_live, 256, 4), 256, 0, st>>>(
      rows, d, live, n_live, L.norms, L.ctr + 1, L.cand_d, L.cand_j, nn_idx, nn_dist, L.redo, L.ctr);
  CGS_CHECK_LAUNCH("codenn_refine_kernel");
  codenn_bruteforce_kernel<<<148 * 4, 256, 0, st>>>(rows, d, live, n_live, L.redo, L.ctr, nn_idx,
                                                    nn_dist);
  CGS_CHECK_LAUNCH("codenn_bruteforce_kernel");
  return CGS_OK;
}

}  // namespace cgs

using namespace cgs;

extern "C" {

size_t cgs_code_nn_workspace_bytes(int64_t n_live, int32_t dim) {
  if (n_live < 0 || dim < 1 || dim > 48) return 0;
  return plan_nn(nullptr, 0, n_live, dim).bytes;
}

int cgs_code_nn(const float* rows, int32_t dim, int64_t capacity, const int32_t* live,
                int64_t n_live, int32_t* nn_index, double* nn_dist2, void* workspace,
                size_t workspace_bytes, cgs_stream_t stream) {
  if (!rows || !live || !nn_index || !nn_dist2 || dim < 1 || dim > 48 || n_live < 0 ||
      capacity < n_live || n_live >= (1LL << 31)) {
    set_error("code_nn: invalid arguments");
    return CGS_EINVAL;
  }
  return code_nn(rows, dim, capacity, live, n_live, nn_index, nn_dist2, workspace,
                 workspace_bytes, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
