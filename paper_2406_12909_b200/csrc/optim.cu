// Optimiser step over the flat parameter vector and the non-finite guard.
//
// Reference: apply_update (train.py:96-108) and the step-loop guard
// (train.py:262-274).  Master parameters and moments are float64 so the
// update is bit-identical to the reference for identical float64 gradients
// (every operation separately rounded, in the reference's order); the
// float32 working copy used by the kernels is written in the same pass.
#include "common.cuh"

namespace gfm {

template <typename G>
__global__ void k_nonfinite(const G* __restrict__ v, long long n, int* __restrict__ flag) {
  pdl_entry();
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite((double)v[i]);
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

// bc[0] = 1 - b1^t, bc[1] = 1 - b2^t  (device pointer so a captured step can
// advance t without re-recording)
template <typename G>
__global__ void k_adam(const G* __restrict__ grad_sum, long long n, double world,
                       double* __restrict__ master, double* __restrict__ m, double* __restrict__ v,
                       const double* __restrict__ bc, double lr, double b1, double b2,
                       double one_m_b1, double one_m_b2, double eps,
                       const int* __restrict__ skip, float* __restrict__ out32) {
  pdl_entry();
  if (skip && *skip) return;  // train.py:264-274: update discarded
  const double bc1 = bc[0], bc2 = bc[1];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double g = __ddiv_rn((double)grad_sum[i], world);  // total[:n] / comm.size
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(one_m_b1, g));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(one_m_b2, g), g));
    const double mh = __ddiv_rn(mi, bc1);
    const double vh = __ddiv_rn(vi, bc2);
    const double p = __dsub_rn(master[i], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
    m[i] = mi;
    v[i] = vi;
    master[i] = p;
    if (out32) out32[i] = (float)p;
  }
}

template <typename G>
__global__ void k_sgd(const G* __restrict__ grad_sum, long long n, double world,
                      double* __restrict__ master, double lr, const int* __restrict__ skip,
                      float* __restrict__ out32) {
  pdl_entry();
  if (skip && *skip) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double g = __ddiv_rn((double)grad_sum[i], world);
    const double p = __dsub_rn(master[i], __dmul_rn(lr, g));
    master[i] = p;
    if (out32) out32[i] = (float)p;
  }
}

__global__ void k_cast_f64_f32(const double* __restrict__ in, long long n, float* __restrict__ out) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

// bias corrections for step t.  The reference evaluates 1.0 - beta ** t on
// the host (train.py:104-105, libm pow); CUDA's double pow may differ by an
// ulp, so the host precomputes the values into ``table`` ([len][2]) and the
// device only looks them up; pow is the fallback past the table's end.
__device__ __forceinline__ void bias_corr_at(long long tt, double b1, double b2, double* bc,
                                             const double* table, long long table_len) {
  if (table != nullptr && tt < table_len) {
    bc[0] = table[2 * tt];
    bc[1] = table[2 * tt + 1];
  } else {
    bc[0] = 1.0 - pow(b1, (double)tt);
    bc[1] = 1.0 - pow(b2, (double)tt);
  }
}

// t += 1; bc = [1 - b1^t, 1 - b2^t] on the device so a captured step needs
// no host round trip; frozen once the non-finite flag is set.  bc == NULL
// (SGD) advances the applied-step count only.
__global__ void k_adam_advance(long long* t, double b1, double b2, double* bc,
                               const double* table, long long table_len,
                               const int* __restrict__ skip) {
  pdl_entry();
  if (skip && *skip) return;
  const long long tt = *t + 1;
  *t = tt;
  if (bc) bias_corr_at(tt, b1, b2, bc, table, table_len);
}

// Guard and Adam advance in one launch: every block ORs its verdict into
// flag[0]; the last block to finish (ticket in flag[1], reset by that block)
// then advances t / bias_corr exactly as k_adam_advance does unless the
// flag is set.  Saves one dependent launch on the step's critical path.
template <typename G>
__global__ void k_nonfinite_advance(const G* __restrict__ v, long long n, int* flag,
                                    long long* t, double b1, double b2, double* bc,
                                    const double* table, long long table_len) {
  pdl_entry();
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite((double)v[i]);
  bad = __syncthreads_or(bad);
  if (threadIdx.x != 0) return;
  if (bad) atomicOr(flag, 1);
  __threadfence();
  if (atomicAdd(flag + 1, 1) != (int)gridDim.x - 1) return;
  __threadfence();
  flag[1] = 0;
  if (t == nullptr || *(volatile int*)flag) return;
  const long long tt = *t + 1;
  *t = tt;
  if (bc) bias_corr_at(tt, b1, b2, bc, table, table_len);
}

static inline int grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

}  // namespace gfm

using namespace gfm;

extern "C" {

int gfm_nonfinite_flag(const void* v, long long n, int dtype, int* flag, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return 0;
  if (dtype == GFM_F32)
    launch_k(k_nonfinite<float>, grid_for(n), 256, 0, s, (const float*)v, n, flag);
  else if (dtype == GFM_F64)
    launch_k(k_nonfinite<double>, grid_for(n), 256, 0, s, (const double*)v, n, flag);
  else {
    set_error("gfm_nonfinite_flag: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_nonfinite_flag: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_nonfinite_advance(const void* v, long long n, int dtype, int* flag, long long* step,
                          double beta1, double beta2, double* bias_corr, const double* bc_table,
                          long long table_len, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(n > 0 ? n : 1);
  if (dtype == GFM_F32)
    launch_k(k_nonfinite_advance<float>, grid, 256, 0, s, (const float*)v, n, flag, step, beta1,
             beta2, bias_corr, bc_table, table_len);
  else if (dtype == GFM_F64)
    launch_k(k_nonfinite_advance<double>, grid, 256, 0, s, (const double*)v, n, flag, step, beta1,
             beta2, bias_corr, bc_table, table_len);
  else {
    set_error("gfm_nonfinite_advance: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_nonfinite_advance: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_adam_step(const void* grad_sum, int grad_dtype, long long n, double world, double* master,
                  double* m, double* v, const double* bias_corr, double lr, double beta1,
                  double beta2, double eps, const int* skip_flag, float* params32, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return 0;
  const double omb1 = 1.0 - beta1, omb2 = 1.0 - beta2;  // as Python evaluates (1.0 - beta)
  if (grad_dtype == GFM_F32)
    launch_k(k_adam<float>, grid_for(n), 256, 0, s, (const float*)grad_sum, n, world, master, m, v,
                                              bias_corr, lr, beta1, beta2, omb1, omb2, eps,
                                              skip_flag, params32);
  else if (grad_dtype == GFM_F64)
    launch_k(k_adam<double>, grid_for(n), 256, 0, s, (const double*)grad_sum, n, world, master, m, v,
                                               bias_corr, lr, beta1, beta2, omb1, omb2, eps,
                                               skip_flag, params32);
  else {
    set_error("gfm_adam_step: bad grad dtype %d", grad_dtype);
    return GFM_EINVAL;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_adam_step: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_sgd_step(const void* grad_sum, int grad_dtype, long long n, double world, double* master,
                 double lr, const int* skip_flag, float* params32, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return 0;
  if (grad_dtype == GFM_F32)
    launch_k(k_sgd<float>, grid_for(n), 256, 0, s, (const float*)grad_sum, n, world, master, lr,
                                             skip_flag, params32);
  else if (grad_dtype == GFM_F64)
    launch_k(k_sgd<double>, grid_for(n), 256, 0, s, (const double*)grad_sum, n, world, master, lr,
                                              skip_flag, params32);
  else {
    set_error("gfm_sgd_step: bad grad dtype %d", grad_dtype);
    return GFM_EINVAL;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_sgd_step: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_adam_advance(long long* step, double beta1, double beta2, double* bias_corr,
                     const double* bc_table, long long table_len, const int* skip_flag,
                     void* stream) {
  launch_k(k_adam_advance, 1, 1, 0, (cudaStream_t)stream, step, beta1, beta2, bias_corr, bc_table,
           table_len, skip_flag);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_adam_advance: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_cast_f64_to_f32(const double* in, long long n, float* out, void* stream) {
  if (n <= 0) return 0;
  launch_k(k_cast_f64_f32, grid_for(n), 256, 0, (cudaStream_t)stream, in, n, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_cast_f64_to_f32: %s", cudaGetErrorString(e));
  return (int)e;
}

}  // extern "C"
