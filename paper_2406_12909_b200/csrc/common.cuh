// Shared device helpers for the gfm_b200 kernels (sm_100a).
#pragma once

#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gfm_b200.h"

#define GFM_WARP 32

namespace gfm {

// Thread-local last error (set by the C-ABI layer).
void set_error(const char* fmt, ...);

// Process-wide GEMM engine selection for float32 (GFM_GEMM_*).
int gemm_mode();
bool tc_pairs();
extern long long g_pair_launches;

// ---------------------------------------------------------------------------
// Exactly-rounded arithmetic.  nvcc contracts a*b+c into FMA by default; the
// float64 parity paths (neighbour predicate, aggregation, Adam) must match
// numpy's separately rounded operations, so they go through these.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

__device__ __forceinline__ float tanh_t(float x) { return tanhf(x); }
// float32 tanh for the hot gathers / epilogues: 1 - 2 / (2^(2x log2 e) + 1)
// with the SFU ex2 / rcp (5 instructions vs ~16 for tanhf).  Absolute error
// <= ~3e-7 everywhere (saturates exactly to +-1); the consumers are dot
// products and 1 - t^2, where absolute error is what propagates.
__device__ __forceinline__ float tanh_fast(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  return fmaf(-2.0f, r, 1.0f);
}
// Four tanh with one reciprocal: tanh(x) = 1 - 2 / (1 + 2^(2x log2 e)); the
// four 1/y share rcp(ya yb yc yd) (products stay finite because x is clamped
// to 10, where tanh already rounds to 1 in fp32; min.NaN keeps NaN inputs
// NaN).  4 EX2 + 1 RCP instead of 4 + 4 on the SFU, which is what bounds the
// force-head edge kernels; max |error| ~5e-7 (vs 1.9e-7 for tanh_fast).
__device__ __forceinline__ float ex2_approx(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
  return e;
}
__device__ __forceinline__ float min_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float4 tanh4_fast(float4 x) {
  constexpr float k = 2.8853900817779268f;  // 2 log2(e)
  const float ya = ex2_approx(min_nan(x.x, 10.f) * k) + 1.f;
  const float yb = ex2_approx(min_nan(x.y, 10.f) * k) + 1.f;
  const float yc = ex2_approx(min_nan(x.z, 10.f) * k) + 1.f;
  const float yd = ex2_approx(min_nan(x.w, 10.f) * k) + 1.f;
  const float pab = ya * yb, pcd = yc * yd;
  float q;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(q) : "f"(pab * pcd));
  const float rab = q * pcd, rcd = q * pab;
  return make_float4(fmaf(-2.f, rab * yb, 1.f), fmaf(-2.f, rab * ya, 1.f),
                     fmaf(-2.f, rcd * yd, 1.f), fmaf(-2.f, rcd * yc, 1.f));
}

__device__ __forceinline__ double tanh_t(double x) { return tanh(x); }

template <typename T>
__device__ __forceinline__ T sign_t(T x) {
  return x > T(0) ? T(1) : (x < T(0) ? T(-1) : T(0));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v, unsigned mask = 0xffffffffu) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// numpy's pairwise_sum (loops_utils.h.src) over a run of n values produced
// by `get(i)`; used by the float64 instantiations so that add.reduceat
// segments come out bit-identical: seg = x0 + pairwise(x1 .. x_{n}).
template <typename T, typename Get>
__device__ __forceinline__ T np_pairwise_leaf(const Get& get, long long b, long long m) {
  if (m < 8) {
    T r = T(0);
    for (long long i = 0; i < m; ++i) r = add_rn(r, get(b + i));
    return r;
  }
  T r0 = get(b + 0), r1 = get(b + 1), r2 = get(b + 2), r3 = get(b + 3);
  T r4 = get(b + 4), r5 = get(b + 5), r6 = get(b + 6), r7 = get(b + 7);
  long long i = 8;
  for (; i < m - (m % 8); i += 8) {
    r0 = add_rn(r0, get(b + i + 0)); r1 = add_rn(r1, get(b + i + 1));
    r2 = add_rn(r2, get(b + i + 2)); r3 = add_rn(r3, get(b + i + 3));
    r4 = add_rn(r4, get(b + i + 4)); r5 = add_rn(r5, get(b + i + 5));
    r6 = add_rn(r6, get(b + i + 6)); r7 = add_rn(r7, get(b + i + 7));
  }
  T res = add_rn(add_rn(add_rn(r0, r1), add_rn(r2, r3)),
                 add_rn(add_rn(r4, r5), add_rn(r6, r7)));
  for (; i < m; ++i) res = add_rn(res, get(b + i));
  return res;
}

template <typename T, typename Get>
__device__ __noinline__ T np_pairwise_deep(const Get& get, long long base, long long n) {
  // post-order walk of numpy's halving recursion with explicit stacks
  long long sb[64], sn[64];
  int st[64];
  T vals[64];
  int sp = 0, vp = 0;
  sb[0] = base; sn[0] = n; st[0] = 0; sp = 1;
  while (sp > 0) {
    --sp;
    long long b = sb[sp], m = sn[sp];
    if (st[sp] == 1) {
      T r = vals[--vp];
      T l = vals[--vp];
      vals[vp++] = add_rn(l, r);
    } else if (m <= 128) {
      vals[vp++] = np_pairwise_leaf<T>(get, b, m);
    } else {
      long long n2 = m / 2;
      n2 -= n2 % 8;
      st[sp] = 1; ++sp;                                   // combine after both
      sb[sp] = b + n2; sn[sp] = m - n2; st[sp] = 0; ++sp; // right
      sb[sp] = b; sn[sp] = n2; st[sp] = 0; ++sp;          // left first
    }
  }
  return vals[0];
}

template <typename T, typename Get>
__device__ __forceinline__ T np_pairwise(const Get& get, long long base, long long n) {
  if (n <= 128) return np_pairwise_leaf<T>(get, base, n);
  return np_pairwise_deep<T>(get, base, n);
}

// ---- packed fp32x2 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2): one issue slot
// for two lanes of a float4; each half is rounded exactly like the scalar op.
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
#define GFM_F2OP(NAME, PTX)                                                               \
  __device__ __forceinline__ float4 NAME(float4 a, float4 b) {                            \
    unsigned long long lo, hi;                                                            \
    asm(PTX " %0, %1, %2;" : "=l"(lo) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));          \
    asm(PTX " %0, %1, %2;" : "=l"(hi) : "l"(pk2(a.z, a.w)), "l"(pk2(b.z, b.w)));          \
    float4 r;                                                                             \
    upk2(lo, r.x, r.y);                                                                   \
    upk2(hi, r.z, r.w);                                                                   \
    return r;                                                                             \
  }
GFM_F2OP(add4, "add.rn.f32x2")
GFM_F2OP(sub4, "sub.rn.f32x2")
GFM_F2OP(mul4, "mul.rn.f32x2")
#undef GFM_F2OP
// a * b + c, single rounding per element
__device__ __forceinline__ float4 fma4(float4 a, float4 b, float4 c) {
  unsigned long long lo, hi;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(lo)
      : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(hi)
      : "l"(pk2(a.z, a.w)), "l"(pk2(b.z, b.w)), "l"(pk2(c.z, c.w)));
  float4 r;
  upk2(lo, r.x, r.y);
  upk2(hi, r.z, r.w);
  return r;
}
__device__ __forceinline__ float4 bcast4(float s) { return make_float4(s, s, s, s); }
#endif

// ---- programmatic dependent launch (PDL) ------------------------------------
// Kernels launched through launch_k() may start while the previous kernel on
// the stream drains: every such kernel calls pdl_entry() first -- it waits for
// the previous grid's completion and memory flush (griddepcontrol.wait) before
// touching any input, then lets the next kernel launch early.  This hides the
// launch latency and prologue (barrier init, TMEM alloc, descriptor prefetch)
// of the ~70 small kernels of a step behind their predecessors' tails.
// GFM_NO_PDL=1 launches normally (pdl_entry() is then a no-op wait).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef GFM_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
#endif
bool pdl_enabled();

template <typename... KP, typename... A>
inline cudaError_t launch_k(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// launch_k with a thread-block cluster of `cluster` CTAs along x (CTA pairs)
template <typename... KP, typename... A>
inline cudaError_t launch_kc(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             int cluster, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

}  // namespace gfm
