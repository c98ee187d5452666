// SGLD update (reference sampler.py:262-300) and the MCMC / densify device
// helpers (sampler.py:184-259, model.py:235-267).  Arithmetic mirrors numpy's
// un-fused float64 sequence exactly (explicit _rn intrinsics, no FMA
// contraction), so identical gradients and noise give bit-identical float32
// state.
#include <cmath>

#include "common.cuh"
#include "sort_scan.cuh"

namespace cgs {

// ---- Philox4x32-10 + Box-Muller (device noise, throughput mode) ----------
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

__device__ __forceinline__ double philox_normal(uint64_t seed, uint64_t offset, uint32_t stream,
                                                uint64_t idx) {
  const uint4 c = philox(make_uint4(static_cast<unsigned>(idx), static_cast<unsigned>(idx >> 32),
                                    stream, static_cast<unsigned>(offset)),
                         make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32)));
  const uint64_t a = (static_cast<uint64_t>(c.x) << 21) ^ c.y;
  const uint64_t b = (static_cast<uint64_t>(c.z) << 21) ^ c.w;
  const double u1 = (static_cast<double>(a & ((1ULL << 53) - 1)) + 0.5) * 0x1.0p-53;
  const double u2 = static_cast<double>(b & ((1ULL << 53) - 1)) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// Four normals from one Philox call (two fp32 Box-Muller pairs): normal
// 4c + q of a stream.  Throughput mode only; parity mode takes the host
// Generator's draws.
__device__ __forceinline__ float4 philox_normal4(uint64_t seed, uint64_t offset, uint32_t stream,
                                                 uint64_t chunk) {
  const uint4 c = philox(make_uint4(static_cast<unsigned>(chunk), static_cast<unsigned>(chunk >> 32),
                                    stream | 0x80000000u, static_cast<unsigned>(offset)),
                         make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32)));
  const float k = 0x1.0p-32f;
  const float u0 = (static_cast<float>(c.x) + 0.5f) * k, u1 = static_cast<float>(c.y) * k;
  const float u2 = (static_cast<float>(c.z) + 0.5f) * k, u3 = static_cast<float>(c.w) * k;
  const float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s0, c0, s1, c1;
  sincospif(2.0f * u1, &s0, &c0);
  sincospif(2.0f * u3, &s1, &c1);
  return make_float4(r0 * c0, r0 * s0, r1 * c1, r1 * s1);
}

struct SgldDev {
  double c_pos, c_op, c_sh, c_sr;  // 0.5 * eps per group
  double k_pos, k_op, k_sh, k_sr;  // mult * sqrt(eps) (0 = no noise)
  int on_pos, on_op, on_sh, on_sr;
  double gscale;
  uint64_t seed, offset;
  int noise_src;
  const uint64_t* offset_dev;
  int32_t* sticky;
};

__device__ __forceinline__ float sgld_one(float v, float g, double c, double k, double gscale,
                                          const double* noise_arr, int64_t nidx, int noise_src,
                                          uint64_t seed, uint64_t offset, uint32_t stream) {
  double gg = static_cast<double>(g);
  if (gscale != 1.0) gg = __dmul_rn(gg, gscale);
  double nv = __dsub_rn(static_cast<double>(v), __dmul_rn(c, gg));
  if (k != 0.0) {
    const double eta = noise_src == 1 ? noise_arr[nidx] : philox_normal(seed, offset, stream, nidx);
    nv = __dadd_rn(nv, __dmul_rn(k, eta));
  }
  return __double2float_rn(nv);
}

__global__ void __launch_bounds__(256) finite_check_kernel(const float* __restrict__ a, int64_t na,
                                                           const float* __restrict__ b, int64_t nb,
                                                           const float* __restrict__ c, int64_t nc,
                                                           const float* __restrict__ d, int64_t nd,
                                                           int32_t* flags, uint64_t* ctr,
                                                           const int32_t* __restrict__ skip_if) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (ctr) *ctr += 1;  // noise offset for this update
    if (skip_if && *skip_if) atomicOr(flags, 2);
  }
  const int64_t tot = na + nb + nc + nd;
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < tot;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float x;
    if (i < na) x = a[i];
    else if (i < na + nb) x = b[i - na];
    else if (i < na + nb + nc) x = c[i - na - nb];
    else x = d[i - na - nb - nc];
    if (!isfinite(x)) bad = true;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, 1);
}

// flags for an update whose gradients were checked by their producers
// (cgs_sgld_params_t.grads_nonfinite): one thread, no pass over the data
__global__ void sgld_prologue_kernel(int32_t* flags, uint64_t* ctr, const int32_t* skip_if,
                                     const int32_t* nonfinite) {
  if (ctr) *ctr += 1;  // noise offset for this update
  flags[0] = ((skip_if && *skip_if) ? 2 : 0) | (*nonfinite ? 1 : 0);
}

__global__ void sticky_or_kernel(int32_t* sticky, const int32_t* flags) {
  if (flags[0]) atomicOr(sticky, flags[0]);
}

__global__ void __launch_bounds__(256) sgld_kernel(
    float* __restrict__ pos, float* __restrict__ logit, int64_t n, float* __restrict__ sh,
    int D, const int32_t* __restrict__ sh_live, int64_t n_sh, float* __restrict__ sr,
    const int32_t* __restrict__ sr_live, int64_t n_sr, const float* __restrict__ gpos,
    const float* __restrict__ glogit, const float* __restrict__ gsh,
    const float* __restrict__ gsr, SgldDev p, const double* __restrict__ npos,
    const double* __restrict__ nlog, const double* __restrict__ nsh,
    const double* __restrict__ nsr, const int32_t* __restrict__ flags) {
  if (p.sticky && blockIdx.x == 0 && threadIdx.x == 0 && flags[0]) atomicOr(p.sticky, flags[0]);
  if (flags[0]) return;  // non-finite gradients or skip: reject before any mutation
  const uint64_t offset = p.offset_dev ? *p.offset_dev : p.offset;
  const int64_t a = p.on_pos ? 3 * n : 0;
  const int64_t b = p.on_op ? n : 0;
  const int64_t c = p.on_sh ? n_sh * D : 0;
  const int64_t d = p.on_sr ? n_sr : 0;
  const int64_t tot = a + b + c + d;
  // device noise on positions / logits: 4 elements per Philox call
  const bool chunked = p.noise_src != 1;
  const int64_t ca = chunked ? (a + 3) / 4 : 0, cb = chunked ? (b + 3) / 4 : 0;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ca + cb;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool isp = t < ca;
    const int64_t ch = isp ? t : t - ca;
    float* v = isp ? pos : logit;
    const float* g = isp ? gpos : glogit;
    const int64_t m = isp ? a : b;
    const double cc = isp ? p.c_pos : p.c_op, kk = isp ? p.k_pos : p.k_op;
    float4 eta4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kk != 0.0) eta4 = philox_normal4(p.seed, offset, isp ? 0u : 1u, static_cast<uint64_t>(ch));
    const float eta[4] = {eta4.x, eta4.y, eta4.z, eta4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = 4 * ch + q;
      if (j >= m) break;
      double gg = static_cast<double>(g[j]);
      if (p.gscale != 1.0) gg = __dmul_rn(gg, p.gscale);
      double nv = __dsub_rn(static_cast<double>(v[j]), __dmul_rn(cc, gg));
      if (kk != 0.0) nv = __dadd_rn(nv, __dmul_rn(kk, static_cast<double>(eta[q])));
      v[j] = __double2float_rn(nv);
    }
  }
  for (int64_t i = (chunked ? a + b : 0) + blockIdx.x * static_cast<int64_t>(blockDim.x) +
                   threadIdx.x;
       i < tot; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < a) {
      pos[i] = sgld_one(pos[i], gpos[i], p.c_pos, p.k_pos, p.gscale, npos, i, p.noise_src, p.seed,
                        offset, 0);
    } else if (i < a + b) {
      const int64_t j = i - a;
      logit[j] = sgld_one(logit[j], glogit[j], p.c_op, p.k_op, p.gscale, nlog, j, p.noise_src,
                          p.seed, offset, 1);
    } else if (i < a + b + c) {
      const int64_t j = i - a - b;
      const int64_t li = j / D, col = j - li * D;
      const int64_t e = static_cast<int64_t>(sh_live[li]) * D + col;
      sh[e] = sgld_one(sh[e], gsh[e], p.c_sh, p.k_sh, p.gscale, nsh, j, p.noise_src, p.seed,
                       offset, 2);
    } else {
      const int64_t li = i - a - b - c;
      const int64_t r = sr_live[li];
      double v[7];
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        double gg = static_cast<double>(gsr[r * 7 + k]);
        if (p.gscale != 1.0) gg = __dmul_rn(gg, p.gscale);
        double nv = __dsub_rn(static_cast<double>(sr[r * 7 + k]), __dmul_rn(p.c_sr, gg));
        if (p.k_sr != 0.0) {
          const double eta = p.noise_src == 1 ? nsr[li * 7 + k]
                                              : philox_normal(p.seed, offset, 3, li * 7 + k);
          nv = __dadd_rn(nv, __dmul_rn(p.k_sr, eta));
        }
        v[k] = nv;
      }
      // q / ||q||, numpy's sequential ((q0^2+q1^2)+q2^2)+q3^2 (sampler.py:298-299)
      const double s = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(v[3], v[3]), __dmul_rn(v[4], v[4])),
                                           __dmul_rn(v[5], v[5])),
                                 __dmul_rn(v[6], v[6]));
      const double nq = __dsqrt_rn(s);
#pragma unroll
      for (int k = 0; k < 3; ++k) sr[r * 7 + k] = __double2float_rn(v[k]);
#pragma unroll
      for (int k = 3; k < 7; ++k) sr[r * 7 + k] = __double2float_rn(__ddiv_rn(v[k], nq));
    }
  }
}

int sgld_update(float* pos, float* logit, int64_t n, float* sh, int D, const int32_t* sh_live,
                int64_t n_sh, float* sr, const int32_t* sr_live, int64_t n_sr, const float* gpos,
                const float* glogit, const float* gsh, const float* gsr, int64_t sh_cap,
                int64_t sr_cap, const cgs_sgld_params_t* hp, const double* npos,
                const double* nlog, const double* nsh, const double* nsr, int32_t* flags,
                cudaStream_t st) {
  if (hp->grads_nonfinite) {  // the producers of the gradients checked them
    sgld_prologue_kernel<<<1, 1, 0, st>>>(flags, hp->offset_dev, hp->skip_if, hp->grads_nonfinite);
    CGS_CHECK_LAUNCH("sgld_prologue_kernel");
  } else {
    CGS_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    const int64_t na = 3 * n, nb = n, nc = sh_cap * D, nd = sr_cap * 7;
    CGS_PROFILED("finite_check_kernel", st, finite_check_kernel<<<grid_for(na + nb + nc + nd, 256, 8), 256, 0, st>>>(gpos, na, glogit, nb, gsh,
                                                                            nc, gsr, nd, flags, hp->offset_dev,
                                                                            hp->skip_if));
    CGS_CHECK_LAUNCH("finite_check_kernel");
  }
  SgldDev p{};
  // exactly numpy's scalar sub-expressions: 0.5 * eps and mult * sqrt(eps)
  p.c_pos = 0.5 * hp->step_pos;
  p.c_op = 0.5 * hp->step_opacity;
  p.c_sh = 0.5 * hp->step_sh;
  p.c_sr = 0.5 * hp->step_sr;
  p.k_pos = (hp->noise_pos != 0.0 && hp->step_pos > 0.0) ? hp->noise_pos * std::sqrt(hp->step_pos) : 0.0;
  p.k_op = (hp->noise_opacity != 0.0 && hp->step_opacity > 0.0) ? hp->noise_opacity * std::sqrt(hp->step_opacity) : 0.0;
  p.k_sh = (hp->noise_sh != 0.0 && hp->step_sh > 0.0) ? hp->noise_sh * std::sqrt(hp->step_sh) : 0.0;
  p.k_sr = (hp->noise_sr != 0.0 && hp->step_sr > 0.0) ? hp->noise_sr * std::sqrt(hp->step_sr) : 0.0;
  p.on_pos = hp->step_pos > 0.0;
  p.on_op = hp->step_opacity > 0.0;
  p.on_sh = hp->step_sh > 0.0;
  p.on_sr = hp->step_sr > 0.0;
  p.gscale = hp->grad_scale;
  p.seed = hp->seed;
  p.offset = hp->offset;
  p.noise_src = hp->noise_source;
  p.offset_dev = hp->offset_dev;
  p.sticky = hp->sticky;
  if (p.noise_src == 1) {
    if ((p.k_pos != 0.0 && !npos) || (p.k_op != 0.0 && !nlog) || (p.k_sh != 0.0 && !nsh) ||
        (p.k_sr != 0.0 && !nsr)) {
      set_error("sgld: noise_source=1 needs the noise array of every noisy group");
      return CGS_EINVAL;
    }
  }
  const int64_t tot = (p.on_pos ? 3 * n : 0) + (p.on_op ? n : 0) + (p.on_sh ? n_sh * D : 0) +
                      (p.on_sr ? n_sr : 0);
  if (tot > 0) {
    CGS_PROFILED("sgld_kernel", st, sgld_kernel<<<grid_for(tot, 256, 8), 256, 0, st>>>(pos, logit, n, sh, D, sh_live, n_sh, sr,
                                                       sr_live, n_sr, gpos, glogit, gsh, gsr, p,
                                                       npos, nlog, nsh, nsr, flags));
    CGS_CHECK_LAUNCH("sgld_kernel");
  } else if (p.sticky) {
    sticky_or_kernel<<<1, 1, 0, st>>>(p.sticky, flags);
    CGS_CHECK_LAUNCH("sticky_or_kernel");
  }
  return CGS_OK;
}

// ---- MCMC helpers ---------------------------------------------------------
struct EligibleOp {
  const int32_t* idx;
  const int32_t* rc;
  int32_t* out;
  __device__ uint64_t load(int64_t i) const { return rc[idx[i]] >= 2 ? 1ULL : 0ULL; }
  __device__ void store(int64_t i, uint64_t ex, uint64_t v) const {
    if (v) out[ex] = static_cast<int32_t>(i);
  }
  __device__ void finish(uint64_t) const {}
};

__global__ void copy_count_kernel(const unsigned long long* src, int64_t* dst) {
  *dst = static_cast<int64_t>(*src);
}

int split_eligible(const int32_t* idx, int64_t n, const int32_t* rc, int32_t* out, int64_t* count,
                   void* ws, size_t ws_bytes, cudaStream_t st) {
  Carver c(ws, ws_bytes);
  ScanWs sw = carve_scan(c, n);
  unsigned long long* tot = c.take<unsigned long long>(1);
  if (!c.fits()) {
    set_error("split_eligible: workspace too small");
    return CGS_EWORKSPACE;
  }
  int r = launch_scan(EligibleOp{idx, rc, out}, nullptr, n, n, sw, tot, st);
  if (r) return r;
  copy_count_kernel<<<1, 1, 0, st>>>(tot, count);
  CGS_CHECK_LAUNCH("copy_count_kernel");
  return CGS_OK;
}

__global__ void apply_splits_kernel(float* rows, int dim, int32_t* idx, const int64_t* gauss,
                                    const int32_t* old_row, const int32_t* new_row,
                                    const double* u, int64_t k) {
  const int64_t tot = k * dim;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / dim, c = e - j * dim;
    const double val = __dadd_rn(static_cast<double>(rows[static_cast<int64_t>(old_row[j]) * dim + c]), u[e]);
    rows[static_cast<int64_t>(new_row[j]) * dim + c] = __double2float_rn(val);
    if (c == 0) idx[gauss[j]] = new_row[j];
  }
}

// Split proposals drawn on the device (the throughput trainer's device-noise
// mode; the reference-parity path keeps numpy's stream on the host,
// mcmc_host.cu): per candidate c, u = eps_split * N(0, I_dim) and a uniform
// from counter-based Philox (seed, ctr, c), log A = -lam - log q with log q =
// -0.5 |u|^2 c_q [+ corr] (sampler.py:138-164), accept = uniform < exp(min(0,
// log A)).  The refcount-dependent skips are settled on the host afterwards
// (they do not change the draws here: each candidate has its own counters).
__global__ void __launch_bounds__(256) split_propose_kernel(int64_t n_cand, int dim, double es,
                                                            double c_q, int use_corr, double corr,
                                                            double lam, uint64_t seed,
                                                            uint64_t ctr, double* __restrict__ u,
                                                            double* __restrict__ prob,
                                                            int8_t* __restrict__ accept) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n_cand;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double u2 = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double z = __dmul_rn(es, philox_normal(seed, ctr, 4, static_cast<uint64_t>(c) * dim + j));
      u[c * dim + j] = z;
      u2 = __fma_rn(z, z, u2);
    }
    double log_q = -0.5 * u2 * c_q;
    if (use_corr) log_q += corr;
    const double log_a = -lam - log_q;
    const double p = exp(fmin(0.0, log_a));
    const uint4 r = philox(make_uint4(static_cast<unsigned>(c), static_cast<unsigned>(c >> 32), 5u,
                                      static_cast<unsigned>(ctr)),
                           make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32)));
    const double coin =
        static_cast<double>(((static_cast<uint64_t>(r.x) << 21) ^ r.y) & ((1ULL << 53) - 1)) * 0x1.0p-53;
    prob[c] = p;
    accept[c] = coin < p ? 1 : 0;
  }
}

int split_propose(int64_t n_cand, int dim, double es, double c_q, int use_corr, double corr,
                  double lam, uint64_t seed, uint64_t ctr, double* u, double* prob, int8_t* accept,
                  cudaStream_t st) {
  if (n_cand <= 0) return CGS_OK;
  split_propose_kernel<<<grid_for(n_cand, 256, 4), 256, 0, st>>>(n_cand, dim, es, c_q, use_corr,
                                                                 corr, lam, seed, ctr, u, prob,
                                                                 accept);
  CGS_CHECK_LAUNCH("split_propose_kernel");
  return CGS_OK;
}

int apply_splits(float* rows, int dim, int32_t* idx, const int64_t* gauss, const int32_t* old_row,
                 const int32_t* new_row, const double* u, int64_t k, cudaStream_t st) {
  if (k <= 0) return CGS_OK;
  apply_splits_kernel<<<grid_for(k * dim, 256, 8), 256, 0, st>>>(rows, dim, idx, gauss, old_row,
                                                                 new_row, u, k);
  CGS_CHECK_LAUNCH("apply_splits_kernel");
  return CGS_OK;
}

__global__ void remap_kernel(int32_t* idx, int64_t n, const int32_t* remap, int64_t len) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = idx[i];
    if (r >= 0 && r < len) {
      const int32_t t = remap[r];
      if (t >= 0) idx[i] = t;
    }
  }
}

int apply_remap(int32_t* idx, int64_t n, const int32_t* remap, int64_t len, cudaStream_t st) {
  if (n <= 0) return CGS_OK;
  remap_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(idx, n, remap, len);
  CGS_CHECK_LAUNCH("remap_kernel");
  return CGS_OK;
}

__global__ void densify_kernel(float* pos, float* logit, int32_t* g2sh, int32_t* g2sr, int64_t n,
                               const int64_t* src, const double* jit, int64_t k) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < k;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = src[j], d = n + j;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      pos[3 * d + c] = __double2float_rn(__dadd_rn(static_cast<double>(pos[3 * s + c]), jit[3 * j + c]));
    logit[d] = logit[s];
    g2sh[d] = g2sh[s];
    g2sr[d] = g2sr[s];
  }
}

int densify_append(float* pos, float* logit, int32_t* g2sh, int32_t* g2sr, int64_t n,
                   const int64_t* src, const double* jit, int64_t k, cudaStream_t st) {
  if (k <= 0) return CGS_OK;
  densify_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(pos, logit, g2sh, g2sr, n, src, jit, k);
  CGS_CHECK_LAUNCH("densify_kernel");
  return CGS_OK;
}

// Opacity-weighted selection of densify sources on the device (throughput
// mode).  numpy's choice(n, k, p=o/sum(o)) draws exactly random(k) from the
// Generator and returns searchsorted(cumsum(p)/cumsum(p)[-1], u, 'right')
// (verified against numpy 2.3); the host still draws the same uniforms, the
// device runs the cumulative sum as a fixed-point (2^-40) inclusive scan of
// sigmoid(logit) and a binary search per draw.  Selections can differ from
// numpy's only for a uniform within ~1e-12 relative of a cumulative boundary.
constexpr double kOpacFix = 1099511627776.0;  // 2^40

struct OpacScan {
  const float* logit;
  uint64_t* incl;
  __device__ uint64_t load(int64_t i) const {
    const double o = 1.0 / (1.0 + exp(-static_cast<double>(logit[i])));
    return static_cast<uint64_t>(o * kOpacFix);
  }
  __device__ void store(int64_t i, uint64_t ex, uint64_t v) const { incl[i] = ex + v; }
  __device__ void finish(uint64_t) const {}
};

__global__ void densify_select_kernel(const uint64_t* __restrict__ incl, int64_t n,
                                      const unsigned long long* __restrict__ total,
                                      const double* __restrict__ u, int64_t k,
                                      int64_t* __restrict__ src) {
  const double tot = static_cast<double>(*total);
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < k;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t target = static_cast<uint64_t>(u[j] * tot);
    int64_t lo = 0, hi = n;  // first i with incl[i] > target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (incl[mid] > target) hi = mid;
      else lo = mid + 1;
    }
    src[j] = lo < n ? lo : n - 1;
  }
}

size_t densify_select_ws_bytes(int64_t n) {
  return align_up((n > 0 ? n : 1) * sizeof(uint64_t)) + scan_ws_bytes(n) + 512;
}

int densify_select(const float* logit, int64_t n, const double* u, int64_t k, int64_t* src,
                   void* ws, size_t ws_bytes, cudaStream_t st) {
  if (k <= 0 || n <= 0) return CGS_OK;
  Carver c(ws, ws_bytes);
  uint64_t* incl = c.take<uint64_t>(n);
  ScanWs sw = carve_scan(c, n);
  unsigned long long* tot = c.take<unsigned long long>(1);
  if (!c.fits()) {
    set_error("densify_select: workspace too small");
    return CGS_EWORKSPACE;
  }
  int rc = launch_scan(OpacScan{logit, incl}, nullptr, n, n, sw, tot, st);
  if (rc) return rc;
  densify_select_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(incl, n, tot, u, k, src);
  CGS_CHECK_LAUNCH("densify_select_kernel");
  return CGS_OK;
}

__global__ void histogram_kernel(const int32_t* idx, int64_t n, int32_t* counts, int64_t cap) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = idx[i];
    if (r >= 0 && r < cap) atomicAdd(&counts[r], 1);  // integer: order-independent
  }
}

int refcount_histogram(const int32_t* idx, int64_t n, int32_t* counts, int64_t cap,
                       cudaStream_t st) {
  if (cap > 0) CGS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * cap, st));
  if (n <= 0) return CGS_OK;
  histogram_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(idx, n, counts, cap);
  CGS_CHECK_LAUNCH("histogram_kernel");
  return CGS_OK;
}

}  // namespace cgs
