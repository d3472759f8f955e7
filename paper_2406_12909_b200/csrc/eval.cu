// Scoring and ensemble reductions (off the training hot path, but on the
// device and in the reference's float64 operation order so the results are
// bit-identical to numpy):
//   gfm_eval_errors        evaluate's per-batch sums (train.py:178-183)
//   gfm_member_stats       ensemble mean / population sigma (ensemble.py:121-130, 181)
//   gfm_force_sigma_reduce per-structure force spread (ensemble.py:133-148)
#include <cmath>

#include "common.cuh"

namespace gfm {

// one thread: numpy's pairwise sums of |(e - e_true) / n| over the batch's
// graphs and of |f - f_true| over its 3N components, added to the running
// float64 totals [sum_e, n_graphs, sum_f, n_comp] in the reference's order
template <typename T>
__global__ void k_eval_errors(const T* __restrict__ e, const T* __restrict__ et,
                              const int* __restrict__ n_per, int B, const T* __restrict__ f,
                              const T* __restrict__ ft, int N, double* __restrict__ acc) {
  pdl_entry();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  auto ge = [&](long long g) -> double {
    const T d = div_rn(sub_rn(e[g], et[g]), (T)n_per[g]);
    return (double)(d < T(0) ? -d : d);
  };
  auto gf = [&](long long i) -> double {
    const T d = sub_rn(f[i], ft[i]);
    return (double)(d < T(0) ? -d : d);
  };
  const double se = B > 0 ? np_pairwise<double>(ge, 0, B) : 0.0;
  const double sf = N > 0 ? np_pairwise<double>(gf, 0, 3LL * N) : 0.0;
  acc[0] = __dadd_rn(acc[0], se);
  acc[1] = __dadd_rn(acc[1], (double)B);
  acc[2] = __dadd_rn(acc[2], sf);
  acc[3] = __dadd_rn(acc[3], __dmul_rn(3.0, (double)N));
}

// stack [K][n]: mean = (sum over k, in k order) / K; sigma = sqrt((sum of
// (x - mean)^2) / K), exactly 0 where every member agrees bitwise
template <typename T>
__global__ void k_member_stats(const T* __restrict__ x, int K, long long n, T* __restrict__ mean,
                               T* __restrict__ sigma) {
  pdl_entry();
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    T s = x[j], lo = x[j], hi = x[j];
    for (int k = 1; k < K; ++k) {
      const T v = x[(long long)k * n + j];
      s = add_rn(s, v);
      lo = v < lo ? v : lo;
      hi = v > hi ? v : hi;
    }
    const T m = div_rn(s, (T)K);
    T q = T(0);
    for (int k = 0; k < K; ++k) {
      const T d = sub_rn(x[(long long)k * n + j], m);
      q = k == 0 ? mul_rn(d, d) : add_rn(q, mul_rn(d, d));
    }
    if (mean) mean[j] = m;
    if (sigma) sigma[j] = sub_rn(hi, lo) == T(0) ? T(0) : (T)sqrt(div_rn(q, (T)K));
  }
}

// one thread per structure: the (n_g, 3) block of sigma_comp -> max | mean | l2
template <typename T>
__global__ void k_force_sigma_reduce(const T* __restrict__ sc, const int* __restrict__ off, int B,
                                     int how, T* __restrict__ out) {
  pdl_entry();
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < B; g += gridDim.x * blockDim.x) {
    const long long b = 3LL * off[g], n = 3LL * (off[g + 1] - off[g]);
    T r = T(0);
    if (how == 0) {
      r = n > 0 ? sc[b] : T(0);
      for (long long i = 1; i < n; ++i) r = sc[b + i] > r ? sc[b + i] : r;
    } else if (how == 1) {
      r = div_rn(np_pairwise<T>([&](long long i) { return sc[i]; }, b, n), (T)n);
    } else {
      const T ms = div_rn(np_pairwise<T>([&](long long i) { return mul_rn(sc[i], sc[i]); }, b, n),
                          (T)n);
      r = (T)sqrt((double)ms);
    }
    out[g] = r;
  }
}

}  // namespace gfm

using namespace gfm;

#define GFM_TRY(expr)                                                   \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) {                                            \
      gfm::set_error("%s: %s", #expr, cudaGetErrorString(_e));          \
      return (int)_e;                                                   \
    }                                                                   \
  } while (0)

extern "C" {

int gfm_eval_errors(const void* e_pred, const void* e_true, const int* n_per, int n_graphs,
                    const void* f_pred, const void* f_true, int n_nodes, double* acc, int dtype,
                    void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GFM_F64)
    launch_k(k_eval_errors<double>, 1, 32, 0, s, (const double*)e_pred, (const double*)e_true,
             n_per, n_graphs, (const double*)f_pred, (const double*)f_true, n_nodes, acc);
  else
    launch_k(k_eval_errors<float>, 1, 32, 0, s, (const float*)e_pred, (const float*)e_true,
             n_per, n_graphs, (const float*)f_pred, (const float*)f_true, n_nodes, acc);
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_member_stats(const void* stack, int n_members, long long n, void* mean, void* sigma,
                     int dtype, void* stream) {
  if (n_members <= 0 || n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const long long blocks = (n + 255) / 256;
  const int grid = (int)(blocks < 148 * 8 ? blocks : 148 * 8);
  if (dtype == GFM_F64)
    launch_k(k_member_stats<double>, grid, 256, 0, s, (const double*)stack, n_members, n,
             (double*)mean, (double*)sigma);
  else
    launch_k(k_member_stats<float>, grid, 256, 0, s, (const float*)stack, n_members, n,
             (float*)mean, (float*)sigma);
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_force_sigma_reduce(const void* sigma_comp, const int* node_offsets, int n_graphs, int how,
                           void* out, int dtype, void* stream) {
  if (how < 0 || how > 2) {
    set_error("gfm_force_sigma_reduce: how must be 0 (max), 1 (mean) or 2 (l2)");
    return GFM_EINVAL;
  }
  if (n_graphs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = (n_graphs + 127) / 128;
  if (dtype == GFM_F64)
    launch_k(k_force_sigma_reduce<double>, grid, 128, 0, s, (const double*)sigma_comp,
             node_offsets, n_graphs, how, (double*)out);
  else
    launch_k(k_force_sigma_reduce<float>, grid, 128, 0, s, (const float*)sigma_comp,
             node_offsets, n_graphs, how, (float*)out);
  GFM_TRY(cudaGetLastError());
  return 0;
}

}  // extern "C"
