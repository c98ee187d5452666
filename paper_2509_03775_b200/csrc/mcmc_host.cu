// Host side of the MCMC split transition (reference sampler.py:339-364):
// the per-candidate accept loop and the eligibility scan, in C++ so a
// config-3 split step (N = 4M Gaussians, ~40k candidates) costs milliseconds
// instead of the ~0.3 s of a Python loop.
//
// Bit-identity with the reference.  The loop draws from the caller's own
// numpy Generator: `bitgen` is the `bitgen_t` behind
// `rng.bit_generator.capsule`, and the normals come from numpy's own
// `random_normal` (libnpyrandom.a, linked statically; the same code
// Generator.normal runs), so the stream advances exactly as the reference's
// `rng.normal(0, eps_split, size=dim)` / `rng.random()` calls do.  |u|^2 is
// computed by the caller's BLAS ddot (numpy's `u @ u` calls it; the caller
// passes the function), and log q / log A with the reference's operation
// order (this file is compiled without floating-point contraction).  The
// accept decision uses the C library's exp; the caller recomputes the
// probabilities with numpy's exp and re-runs the Python loop from the saved
// Generator state in the (ulp-level, never observed) case they disagree.
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "../../include/cgs_b200.h"

extern "C" {
// numpy/random/bitgen.h (public numpy C API)
typedef struct bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
} bitgen_t;
// numpy/random/lib/libnpyrandom.a
double random_normal(bitgen_t* bitgen_state, double loc, double scale);
}

namespace {
typedef double (*ddot_fn)(int64_t n, const double* x, int64_t incx, const double* y,
                          int64_t incy);
}

extern "C" {

CGS_API int cgs_host_split_eligible(const int32_t* idx, int64_t n, const int64_t* refcount,
                                    int64_t k, int32_t* out, int64_t* n_out, int32_t threads) {
  if ((n > 0 && (!idx || !out)) || !refcount || !n_out) return CGS_EINVAL;
  const int T = std::max(1, std::min<int>(threads > 0 ? threads : 1, 64));
  const int64_t chunk = (n + T - 1) / T;
  std::vector<int64_t> cnt(T + 1, 0);
  auto shared = [&](int64_t i) {
    const int32_t r = idx[i];
    return r >= 0 && r < k && refcount[r] >= 2;  // sampler.py:344
  };
  auto count = [&](int t) {
    int64_t c = 0;
    for (int64_t i = t * chunk, e = std::min(n, (t + 1) * chunk); i < e; ++i) c += shared(i);
    cnt[t + 1] = c;
  };
  auto write = [&](int t) {
    int64_t o = cnt[t];
    for (int64_t i = t * chunk, e = std::min(n, (t + 1) * chunk); i < e; ++i)
      if (shared(i)) out[o++] = static_cast<int32_t>(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(count, t);
  count(0);
  for (auto& th : pool) th.join();
  pool.clear();
  for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
  for (int t = 1; t < T; ++t) pool.emplace_back(write, t);
  write(0);
  for (auto& th : pool) th.join();
  *n_out = cnt[T];
  return CGS_OK;
}

CGS_API int cgs_host_split_decide(void* bitgen, void* ddot, int64_t n_cand, const int64_t* rows,
                                  int64_t* refcount, int64_t k, int32_t dim, double lam,
                                  double eps_split, double c_q, int32_t use_corr, double corr,
                                  double* u_out, double* log_a_out, double* uniform_out,
                                  int8_t* decision_out, int64_t* n_attempts) {
  if (!bitgen || !ddot || (n_cand > 0 && (!rows || !u_out || !log_a_out || !uniform_out ||
                                          !decision_out)) ||
      !refcount || !n_attempts || dim <= 0)
    return CGS_EINVAL;
  bitgen_t* bg = static_cast<bitgen_t*>(bitgen);
  const ddot_fn dot = reinterpret_cast<ddot_fn>(ddot);
  int64_t att = 0;
  for (int64_t c = 0; c < n_cand; ++c) {
    const int64_t row = rows[c];
    double* u = u_out + c * dim;
    if (row < 0 || row >= k || refcount[row] < 2) {  // sampler.py:350-351: skip, no draws
      decision_out[c] = -1;
      log_a_out[c] = NAN;
      uniform_out[c] = NAN;
      continue;
    }
    for (int j = 0; j < dim; ++j) u[j] = random_normal(bg, 0.0, eps_split);  // rng.normal(0, es, dim)
    // acceptance_probability("split", u, ...) (sampler.py:138-164): log q =
    // -0.5 * (u @ u) * (1/es^2 - 1/em^2) [+ d ln(em/es)], log A = -lam - log q
    const double u2 = dot(dim, u, 1, u, 1);
    double log_q = -0.5 * u2;
    log_q = log_q * c_q;
    if (use_corr) log_q = log_q + corr;
    double log_a = -lam;
    log_a = log_a - log_q;
    log_a = log_a + 0.0;  // extra_log_ratio
    const double prob = std::exp(std::min(0.0, log_a));
    const double coin = bg->next_double(bg->state);  // rng.random()
    log_a_out[c] = log_a;
    uniform_out[c] = coin;
    ++att;
    if (coin < prob) {
      decision_out[c] = 1;
      refcount[row] -= 1;  // decref of the old row (it stays >= 1)
    } else {
      decision_out[c] = 0;
    }
  }
  *n_attempts = att;
  return CGS_OK;
}

}  // extern "C"
