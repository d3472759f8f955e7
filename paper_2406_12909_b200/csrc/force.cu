// Force head, node-factored (forward + backward).
//
// Reference (model.py:377-389, 535-547):
//   pair_e = h[dst] + h[src];  t_e = tanh(pair_e V^T + c);  m_e = t_e . u
//   f[dst] += m_e * dx_e
// The pre-activation is linear in the pair, so with P = h V^T (one N x H x H
// GEMM per step instead of an E x H x H one):
//   pre_e = P[dst] + P[src] + c
// and the edge work becomes a memory-bound gather over the dst-CSR (P[dst]
// held in registers, P[src] gathered from L2), fused with the u-dot and the
// segmented force reduction -- the same kernel shape as the aggregation.
// Backward: dpre_e = dm_e u (1 - t_e^2) with dm_e = df[dst] . dx_e;
//   D_dst[i] = sum_{e in CSR row i} dpre_e,  D_src[j] = sum_{e in CSC row j} dpre_e
//   S = D_dst + D_src      (N x H)
//   grad_V = sum_e dpre_e pair_e^T = S^T h          (node GEMM)
//   dh    += sum_e (dpre_e V) at dst and src = S V  (node GEMM)
//   grad_c = colsum(D_dst),  grad_u = colsum(sum_{e in row i} t_e dm_e)
// Two gather passes (dst-CSR then src-CSC, recomputing t instead of storing
// E x H intermediates); no atomics, fixed summation orders.
#include <type_traits>

#include "common.cuh"

namespace gfm {

// SFU tanh (tanh4_fast, |err| <= 5e-7) in the float32 edge kernels of the
// tensor-core modes; GFM_EXACT_TANH=1 (or the SIMT engine) keeps tanhf.
inline bool fast_tanh_on() {
  static int v = -1;
  if (v < 0) v = getenv("GFM_EXACT_TANH") ? (atoi(getenv("GFM_EXACT_TANH")) == 0) : 1;
  return v && gemm_mode() != GFM_GEMM_SIMT;
}


// choose (NV float4 per lane, LPN lanes per node) for the float32 path
static bool force_vec_shape(int H, int& nv, int& lpn, int* slabs = nullptr) {
  if (H % 4) return false;
  const int h4 = H / 4;
  if (slabs) {  // wide H: 32-lane column slabs (gridDim.y / warps) instead of NV > 1
    *slabs = 1;
    if (h4 > 32 && h4 % 32 == 0 && (h4 / 32 == 2 || h4 / 32 == 4 || h4 / 32 == 8)) {
      nv = 1;
      lpn = 32;
      *slabs = h4 / 32;
      return true;
    }
  }
  for (int v : {1, 2, 4}) {
    if (h4 % v) continue;
    const int l = h4 / v;
    if (l <= 32 && (l & (l - 1)) == 0) {
      nv = v;
      lpn = l;
      return true;
    }
  }
  return false;
}

// sum over the LPN lanes of this node's group (only the group's lanes named,
// so groups of one warp may diverge / exit independently)
template <int LPN>
__device__ __forceinline__ float group_sum(float v) {
  const int lane = threadIdx.x & 31;
  const unsigned mask = LPN == 32 ? 0xffffffffu : (((1u << LPN) - 1u) << (lane / LPN * LPN));
#pragma unroll
  for (int o = LPN / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, LPN);
  return v;
}

template <int LPN>
__device__ __forceinline__ double group_sum_d(double v) {
  const int lane = threadIdx.x & 31;
  const unsigned mask = LPN == 32 ? 0xffffffffu : (((1u << LPN) - 1u) << (lane / LPN * LPN));
#pragma unroll
  for (int o = LPN / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, LPN);
  return v;
}

// c / u are views into the flat parameter vector: not 16-byte aligned
__device__ __forceinline__ float4 ld4u(const float* p, int c4) {
  return make_float4(__ldg(p + 4 * c4), __ldg(p + 4 * c4 + 1), __ldg(p + 4 * c4 + 2),
                     __ldg(p + 4 * c4 + 3));
}

// tanh of the hot gathers: the SFU form in the tensor-core GEMM modes
// (stated 3xTF32 / TF32 bounds), tanhf in the fp32 SIMT mode (1e-4 bound)
template <bool FAST>
__device__ __forceinline__ float th(float x) {
  if constexpr (FAST)
    return tanh_fast(x);
  else
    return tanhf(x);
}

template <bool FAST>
__device__ __forceinline__ float4 th4(float4 x) {
  if constexpr (FAST)
    return tanh4_fast(x);
  else
    return make_float4(tanhf(x.x), tanhf(x.y), tanhf(x.z), tanhf(x.w));
}

__device__ __forceinline__ float dot4(float4 t, float4 u) {
  return t.x * u.x + t.y * u.y + t.z * u.z + t.w * u.w;
}

__device__ __forceinline__ float4 f4add3(float4 a, float4 b, float4 c) {
  return make_float4(a.x + b.x + c.x, a.y + b.y + c.y, a.z + b.z + c.z, a.w + b.w + c.w);
}

// ------------------------------------------------------------------ forward
template <int NV, int LPN, bool FAST>
__global__ void __launch_bounds__(256)
    k_force_fwd_vec(const float* __restrict__ P, int n, int H, const int* __restrict__ rowptr,
                    const int* __restrict__ col_src, const float* __restrict__ dx,
                    const float* __restrict__ c, const float* __restrict__ u,
                    float* __restrict__ f) {
  pdl_entry();
  constexpr int NPW = 32 / LPN;
  const int lane = threadIdx.x & 31, sub = lane % LPN;
  const int i = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NPW + lane / LPN;
  if (i >= n) return;  // whole LPN groups exit together
  const int H4 = H >> 2;
  const float4* P4 = reinterpret_cast<const float4*>(P);
  float4 pi[NV], cu[NV], uu[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int c4 = v * LPN + sub;
    pi[v] = __ldg(P4 + (long long)i * H4 + c4);
    cu[v] = ld4u(c, c4);
    uu[v] = ld4u(u, c4);
  }
  // f = sum_e m_e dx_e = sum_lanes sum_e d_lane(e) dx_e: each lane keeps its
  // partial force in fp64 (one fp32 rounding per edge pair, then one
  // fp32 -> fp64 conversion per pair and component: the conversions share
  // the SFU pipe with the tanh), one group reduction per node
  double fx = 0.0, fy = 0.0, fz = 0.0;
  const int beg = rowptr[i], end = rowptr[i + 1];
  int p = beg;
  for (; p + 2 <= end; p += 2) {  // two edges in flight
    const int s0 = __ldg(col_src + p), s1 = __ldg(col_src + p + 1);
    float4 r0[NV], r1[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      r0[v] = __ldg(P4 + (long long)s0 * H4 + v * LPN + sub);
      r1[v] = __ldg(P4 + (long long)s1 * H4 + v * LPN + sub);
    }
    float d0 = 0.f, d1 = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      d0 += dot4(th4<FAST>(f4add3(pi[v], r0[v], cu[v])), uu[v]);
      d1 += dot4(th4<FAST>(f4add3(pi[v], r1[v], cu[v])), uu[v]);
    }
    fx += (double)fmaf(d1, dx[3LL * p + 3], d0 * dx[3LL * p + 0]);
    fy += (double)fmaf(d1, dx[3LL * p + 4], d0 * dx[3LL * p + 1]);
    fz += (double)fmaf(d1, dx[3LL * p + 5], d0 * dx[3LL * p + 2]);
  }
  for (; p < end; ++p) {
    const int s0 = __ldg(col_src + p);
    float d0 = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      d0 += dot4(th4<FAST>(f4add3(pi[v], __ldg(P4 + (long long)s0 * H4 + v * LPN + sub), cu[v])), uu[v]);
    fx += (double)(d0 * dx[3LL * p + 0]);
    fy += (double)(d0 * dx[3LL * p + 1]);
    fz += (double)(d0 * dx[3LL * p + 2]);
  }
  fx = group_sum_d<LPN>(fx);
  fy = group_sum_d<LPN>(fy);
  fz = group_sum_d<LPN>(fz);
  if (sub == 0) {
    f[3LL * i + 0] = (float)fx;
    f[3LL * i + 1] = (float)fy;
    f[3LL * i + 2] = (float)fz;
  }
}

// wide H (H/4 = 32*SL float4 columns): SL warps per node, one 32-lane column
// slab each.  Per-edge slab partials of m_e meet in shared memory; the slab-0
// warp combines them in slab order and accumulates the force in fp64.
template <int SL, bool FAST>
__global__ void __launch_bounds__(256)
    k_force_fwd_slab(const float* __restrict__ P, int n, int H, const int* __restrict__ rowptr,
                     const int* __restrict__ col_src, const float* __restrict__ dx,
                     const float* __restrict__ c, const float* __restrict__ u,
                     float* __restrict__ f) {
  pdl_entry();
  constexpr int NPB = 8 / SL, CH = 32;  // nodes per block, edges per chunk
  __shared__ float mpart[8][CH];
  __shared__ int degs[NPB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slab = warp % SL, ln = warp / SL;
  const int i = blockIdx.x * NPB + ln;
  const bool live = i < n;
  const int H4 = H >> 2, c4 = slab * 32 + lane;
  const float4* P4 = reinterpret_cast<const float4*>(P);
  float4 pi = make_float4(0.f, 0.f, 0.f, 0.f), cu = pi, uu = pi;
  int beg = 0, end = 0;
  if (live) {
    pi = __ldg(P4 + (long long)i * H4 + c4);
    cu = ld4u(c, c4);
    uu = ld4u(u, c4);
    beg = rowptr[i];
    end = rowptr[i + 1];
  }
  if (slab == 0 && lane == 0) degs[ln] = end - beg;
  __syncthreads();
  int maxdeg = 0;
#pragma unroll
  for (int k = 0; k < NPB; ++k) maxdeg = max(maxdeg, degs[k]);
  double fx = 0.0, fy = 0.0, fz = 0.0;
  for (int p0 = 0; p0 < maxdeg; p0 += CH) {
    // this chunk's sources: one coalesced load, broadcast by shuffles
    const int my_s = beg + p0 + lane < end ? __ldg(col_src + beg + p0 + lane) : 0;
    for (int e = 0; e < CH; e += 2) {
      const int pa = beg + p0 + e, pb = pa + 1;
      if (pa >= end) break;  // warp-uniform
      const bool hb = pb < end;
      const int sa = __shfl_sync(0xffffffffu, my_s, e);
      const int sb = __shfl_sync(0xffffffffu, my_s, hb ? e + 1 : e);
      const float4 ra = __ldg(P4 + (long long)sa * H4 + c4);
      const float4 rb = __ldg(P4 + (long long)sb * H4 + c4);
      const float4 xa = f4add3(pi, ra, cu), xb = f4add3(pi, rb, cu);
      float da = dot4(th4<FAST>(xa), uu);
      float db = dot4(th4<FAST>(xb), uu);
      da = group_sum<32>(da);
      db = group_sum<32>(db);
      if (lane == 0) {
        mpart[warp][e] = da;
        if (hb) mpart[warp][e + 1] = db;
      }
    }
    __syncthreads();
    if (slab == 0) {
      const int p = beg + p0 + lane;
      double gx = 0.0, gy = 0.0, gz = 0.0;
      if (lane < CH && p < end) {
        float m = mpart[warp][lane];
#pragma unroll
        for (int k = 1; k < SL; ++k) m += mpart[warp + k][lane];
        gx = (double)m * dx[3LL * p + 0];
        gy = (double)m * dx[3LL * p + 1];
        gz = (double)m * dx[3LL * p + 2];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gx += __shfl_xor_sync(0xffffffffu, gx, o);
        gy += __shfl_xor_sync(0xffffffffu, gy, o);
        gz += __shfl_xor_sync(0xffffffffu, gz, o);
      }
      fx += gx;
      fy += gy;
      fz += gz;
    }
    __syncthreads();
  }
  if (live && slab == 0 && lane == 0) {
    f[3LL * i + 0] = (float)fx;
    f[3LL * i + 1] = (float)fy;
    f[3LL * i + 2] = (float)fz;
  }
}

// generic: one warp per node, lanes over columns (any H, float or double)
template <typename T>
__global__ void k_force_fwd_warp(const T* __restrict__ P, int n, int H, const int* __restrict__ rowptr,
                                 const int* __restrict__ col_src, const T* __restrict__ dx,
                                 const T* __restrict__ c, const T* __restrict__ u,
                                 T* __restrict__ f) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  double fx = 0.0, fy = 0.0, fz = 0.0;
  for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) {
    const int s = col_src[p];
    T d = T(0);
    for (int k = lane; k < H; k += 32)
      d += tanh_t(P[(long long)i * H + k] + P[(long long)s * H + k] + c[k]) * u[k];
    d = warp_sum(d);
    fx = __dadd_rn(fx, __dmul_rn((double)d, (double)dx[3LL * p + 0]));
    fy = __dadd_rn(fy, __dmul_rn((double)d, (double)dx[3LL * p + 1]));
    fz = __dadd_rn(fz, __dmul_rn((double)d, (double)dx[3LL * p + 2]));
  }
  if (lane == 0) {
    f[3LL * i + 0] = (T)fx;
    f[3LL * i + 1] = (T)fy;
    f[3LL * i + 2] = (T)fz;
  }
}

// ------------------------------------------------------------------ backward
#ifndef GFM_FORCE_BWD_U
#define GFM_FORCE_BWD_U 4
#endif
constexpr int kFU = GFM_FORCE_BWD_U;
// pass 1 (dst rows): D_dst[i] = sum dpre_e, TU[i] = sum t_e dm_e
template <int NV, int LPN, bool FAST>
__global__ void __launch_bounds__(256)
    k_force_bwd_dst_vec(const float* __restrict__ P, int n, int H, const int* __restrict__ rowptr,
                        const int* __restrict__ col_src, const float* __restrict__ dx,
                        const float* __restrict__ df, const float* __restrict__ c,
                        const float* __restrict__ u, float* __restrict__ Ddst,
                        float* __restrict__ TU) {
  pdl_entry();
  constexpr int NPW = 32 / LPN;
  const int lane = threadIdx.x & 31, sub = lane % LPN;
  const int i = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NPW + lane / LPN;
  if (i >= n) return;
  const int H4 = H >> 2;
  const int cb = blockIdx.y * (NV * LPN) + sub;  // column slab (wide H)
  const float4* P4 = reinterpret_cast<const float4*>(P);
  float4 pi[NV], cu[NV], uu[NV], dd[NV], tu[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int c4 = v * LPN + cb;
    pi[v] = __ldg(P4 + (long long)i * H4 + c4);
    cu[v] = ld4u(c, c4);
    uu[v] = ld4u(u, c4);
    dd[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    tu[v] = dd[v];
  }
  const float fx = df[3LL * i + 0], fy = df[3LL * i + 1], fz = df[3LL * i + 2];
  // model.py:537-538 (sum over xyz left to right)
  auto dm_of = [&](int p) {
    return __fadd_rn(__fadd_rn(__fmul_rn(fx, dx[3LL * p]), __fmul_rn(fy, dx[3LL * p + 1])),
                     __fmul_rn(fz, dx[3LL * p + 2]));
  };
  auto edge = [&](float4 (&r)[NV], float dm) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 x = f4add3(pi[v], r[v], cu[v]);
      const float4 t = make_float4(th<FAST>(x.x), th<FAST>(x.y), th<FAST>(x.z), th<FAST>(x.w));
      dd[v].x += dm * uu[v].x * (1.f - t.x * t.x); dd[v].y += dm * uu[v].y * (1.f - t.y * t.y);
      dd[v].z += dm * uu[v].z * (1.f - t.z * t.z); dd[v].w += dm * uu[v].w * (1.f - t.w * t.w);
      tu[v].x += t.x * dm; tu[v].y += t.y * dm; tu[v].z += t.z * dm; tu[v].w += t.w * dm;
    }
  };
  const int beg = rowptr[i], end = rowptr[i + 1];
  if constexpr (LPN >= 8) {
    // lane k of the node's group computes (src, dm) of edge c0 + k once;
    // group shuffles broadcast them; two P rows in flight per lane
    const unsigned gm = LPN == 32 ? 0xffffffffu : (((1u << LPN) - 1u) << (lane - sub));
    for (int c0 = beg; c0 < end; c0 += LPN) {
      const int cnt = min(LPN, end - c0);
      int my_s = 0;
      float my_dm = 0.f;
      if (sub < cnt) {
        my_s = __ldg(col_src + c0 + sub);
        my_dm = dm_of(c0 + sub);
      }
      for (int e = 0; e < cnt; e += kFU) {  // kFU P rows in flight per lane
        int s[kFU];
        float d[kFU];
        float4 r[kFU][NV];
        // row indices first: the P loads issue before the dm shuffles wait
        // on the (dependent) dm loads
#pragma unroll
        for (int q = 0; q < kFU; ++q)
          s[q] = __shfl_sync(gm, my_s, e + q < cnt ? e + q : e, LPN);
#pragma unroll
        for (int q = 0; q < kFU; ++q)
#pragma unroll
          for (int v = 0; v < NV; ++v) r[q][v] = __ldg(P4 + (long long)s[q] * H4 + v * LPN + cb);
#pragma unroll
        for (int q = 0; q < kFU; ++q) d[q] = __shfl_sync(gm, my_dm, e + q < cnt ? e + q : e, LPN);
#pragma unroll
        for (int q = 0; q < kFU; ++q)
          if (e + q < cnt) edge(r[q], d[q]);
      }
    }
  } else {
    for (int p = beg; p < end; ++p) {
      const int s = __ldg(col_src + p);
      float4 r[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = __ldg(P4 + (long long)s * H4 + v * LPN + cb);
      edge(r, dm_of(p));
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const long long o = (long long)i * H4 + v * LPN + cb;
    reinterpret_cast<float4*>(Ddst)[o] = dd[v];
    reinterpret_cast<float4*>(TU)[o] = tu[v];
  }
}

// pass 2 (src rows): S[j] = D_dst[j] + sum over CSC slots of dpre_e
template <int NV, int LPN, bool FAST>
__global__ void __launch_bounds__(256)
    k_force_bwd_src_vec(const float* __restrict__ P, int n, int H, const int* __restrict__ csc_ptr,
                        const int* __restrict__ csc_eid, const int* __restrict__ csc_dst,
                        const float* __restrict__ dx, const float* __restrict__ df,
                        const float* __restrict__ c, const float* __restrict__ u,
                        const float* __restrict__ Ddst, float* __restrict__ S) {
  pdl_entry();
  constexpr int NPW = 32 / LPN;
  const int lane = threadIdx.x & 31, sub = lane % LPN;
  const int j = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NPW + lane / LPN;
  if (j >= n) return;
  const int H4 = H >> 2;
  const int cb = blockIdx.y * (NV * LPN) + sub;  // column slab (wide H)
  const float4* P4 = reinterpret_cast<const float4*>(P);
  float4 pj[NV], cu[NV], uu[NV], acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int c4 = v * LPN + cb;
    pj[v] = __ldg(P4 + (long long)j * H4 + c4);
    cu[v] = ld4u(c, c4);
    uu[v] = ld4u(u, c4);
    acc[v] = reinterpret_cast<const float4*>(Ddst)[(long long)j * H4 + c4];
  }
  auto dm_of = [&](int p, int i) {
    return __fadd_rn(__fadd_rn(__fmul_rn(df[3LL * i], dx[3LL * p]), __fmul_rn(df[3LL * i + 1], dx[3LL * p + 1])),
                     __fmul_rn(df[3LL * i + 2], dx[3LL * p + 2]));
  };
  auto edge = [&](float4 (&r)[NV], float dm) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 x = f4add3(r[v], pj[v], cu[v]);
      const float4 t = make_float4(th<FAST>(x.x), th<FAST>(x.y), th<FAST>(x.z), th<FAST>(x.w));
      acc[v].x += dm * uu[v].x * (1.f - t.x * t.x); acc[v].y += dm * uu[v].y * (1.f - t.y * t.y);
      acc[v].z += dm * uu[v].z * (1.f - t.z * t.z); acc[v].w += dm * uu[v].w * (1.f - t.w * t.w);
    }
  };
  const int qb = csc_ptr[j], qe = csc_ptr[j + 1];
  if constexpr (LPN >= 8) {
    // lane k of the node's group computes (dst, dm) of CSC slot c0 + k once
    const unsigned gm = LPN == 32 ? 0xffffffffu : (((1u << LPN) - 1u) << (lane - sub));
    for (int c0 = qb; c0 < qe; c0 += LPN) {
      const int cnt = min(LPN, qe - c0);
      int my_i = 0;
      float my_dm = 0.f;
      if (sub < cnt) {
        const int p = __ldg(csc_eid + c0 + sub);
        my_i = __ldg(csc_dst + c0 + sub);
        my_dm = dm_of(p, my_i);
      }
      for (int e = 0; e < cnt; e += kFU) {  // kFU P rows in flight per lane
        int i[kFU];
        float d[kFU];
        float4 r[kFU][NV];
        // row indices first: the P loads issue before the dm shuffles wait
        // on the (dependent) dm loads
#pragma unroll
        for (int q = 0; q < kFU; ++q)
          i[q] = __shfl_sync(gm, my_i, e + q < cnt ? e + q : e, LPN);
#pragma unroll
        for (int q = 0; q < kFU; ++q)
#pragma unroll
          for (int v = 0; v < NV; ++v) r[q][v] = __ldg(P4 + (long long)i[q] * H4 + v * LPN + cb);
#pragma unroll
        for (int q = 0; q < kFU; ++q) d[q] = __shfl_sync(gm, my_dm, e + q < cnt ? e + q : e, LPN);
#pragma unroll
        for (int q = 0; q < kFU; ++q)
          if (e + q < cnt) edge(r[q], d[q]);
      }
    }
  } else {
    for (int q = qb; q < qe; ++q) {
      const int p = __ldg(csc_eid + q), i = __ldg(csc_dst + q);
      float4 r[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = __ldg(P4 + (long long)i * H4 + v * LPN + cb);
      edge(r, dm_of(p, i));
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v)
    reinterpret_cast<float4*>(S)[(long long)j * H4 + v * LPN + cb] = acc[v];
}

// generic (any H, float / double): thread per (node, column)
template <typename T>
__global__ void k_force_bwd_dst_scalar(const T* __restrict__ P, int n, int H, const int* __restrict__ rowptr,
                                       const int* __restrict__ col_src, const T* __restrict__ dx,
                                       const T* __restrict__ df, const T* __restrict__ c,
                                       const T* __restrict__ u, T* __restrict__ Ddst,
                                       T* __restrict__ TU) {
  pdl_entry();
  const long long total = (long long)n * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / H), k = (int)(idx % H);
    T dd = T(0), tu = T(0);
    for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const int s = col_src[p];
      const T dm = add_rn(add_rn(mul_rn(df[3LL * i], dx[3LL * p]), mul_rn(df[3LL * i + 1], dx[3LL * p + 1])),
                          mul_rn(df[3LL * i + 2], dx[3LL * p + 2]));
      const T t = tanh_t(P[(long long)i * H + k] + P[(long long)s * H + k] + c[k]);
      dd += mul_rn(mul_rn(dm, u[k]), sub_rn(T(1), mul_rn(t, t)));
      tu += t * dm;
    }
    Ddst[idx] = dd;
    TU[idx] = tu;
  }
}

template <typename T>
__global__ void k_force_bwd_src_scalar(const T* __restrict__ P, int n, int H, const int* __restrict__ csc_ptr,
                                       const int* __restrict__ csc_eid, const int* __restrict__ csc_dst,
                                       const T* __restrict__ dx, const T* __restrict__ df,
                                       const T* __restrict__ c, const T* __restrict__ u,
                                       const T* __restrict__ Ddst, T* __restrict__ S) {
  pdl_entry();
  const long long total = (long long)n * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / H), k = (int)(idx % H);
    T acc = Ddst[idx];
    for (int q = csc_ptr[j]; q < csc_ptr[j + 1]; ++q) {
      const int p = csc_eid[q], i = csc_dst[q];
      const T dm = add_rn(add_rn(mul_rn(df[3LL * i], dx[3LL * p]), mul_rn(df[3LL * i + 1], dx[3LL * p + 1])),
                          mul_rn(df[3LL * i + 2], dx[3LL * p + 2]));
      const T t = tanh_t(P[(long long)i * H + k] + P[(long long)j * H + k] + c[k]);
      acc += mul_rn(mul_rn(dm, u[k]), sub_rn(T(1), mul_rn(t, t)));
    }
    S[idx] = acc;
  }
}

// deterministic column sums of X [n][H] (+ optional second matrix Y):
// pass 1 -- fixed row chunks -> partials; pass 2 -- ordered sum of partials
// Block = 256 threads over a 512-row chunk: thread t owns column
// (blockIdx.y * cw + t % cw) and rows r = t / cw, + 256 / cw, ... of the chunk
// (coalesced row segments); the 256 / cw row-group sums are combined in a
// fixed order in shared memory.
constexpr int kColChunk = 128;
template <typename T>
__global__ void __launch_bounds__(256)
    k_colsum_partial(const T* __restrict__ X1, int n, int H, int chunk, int cw, T* __restrict__ part1,
                     const T* __restrict__ X2, T* __restrict__ part2) {
  pdl_entry();
  // gridDim.z = 2: a second, independent (X, part) pair in the same launch
  const T* __restrict__ X = blockIdx.z ? X2 : X1;
  T* __restrict__ part = blockIdx.z ? part2 : part1;
  // block (ch, cb): rows [ch*chunk, ch*chunk+chunk) x columns [cb*cw, cb*cw+cw);
  // 256/cw row groups stride the rows, then a fixed-order smem combine, so the
  // result depends only on (n, H, chunk, cw) -- deterministic
  __shared__ double red[256];
  const int groups = 256 / cw;
  const int ch = blockIdx.x;
  const long long lo = (long long)ch * chunk;
  const long long hi = min((long long)n, lo + chunk);
  const int c = blockIdx.y * cw + threadIdx.x % cw;
  const int g = threadIdx.x / cw;
  double s = 0.0;
  if (g < groups && c < H) {
#pragma unroll 8  // independent loads in flight; the adds stay in row order
    for (long long i = lo + g; i < hi; i += groups) s += (double)X[i * H + c];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < cw && c < H) {
    double t = 0.0;
    for (int q = 0; q < groups; ++q) t += red[q * cw + threadIdx.x];
    part[(long long)ch * H + c] = (T)t;
  }
}

// column sums of one or two (n x H) arrays (X2 may be null); part holds
// ceil(n / kColChunk) * H partials per array
template <typename T>
cudaError_t colsum2(const T* X1, const T* X2, int n, int H, T* out1, T* out2, T* part,
                    cudaStream_t s) {
  if (H <= 0) return cudaSuccess;
  const int cw = H < 64 ? H : 64;
  const int z = X2 ? 2 : 1;
  if (n <= 0) {
    cudaMemsetAsync(out1, 0, sizeof(T) * H, s);
    if (X2) cudaMemsetAsync(out2, 0, sizeof(T) * H, s);
    return cudaGetLastError();
  }
  const int nch = ceil_div(n, kColChunk);
  T* part2 = part + (size_t)nch * H;
  launch_k(k_colsum_partial<T>, dim3(nch, ceil_div(H, cw), z), 256, 0, s, X1, n, H, kColChunk, cw,
           part, X2, part2);
  // second level: the nch partial rows, one block per column slab
  const int cw2 = H < 32 ? H : 32;
  launch_k(k_colsum_partial<T>, dim3(1, ceil_div(H, cw2), z), 256, 0, s, (const T*)part, nch, H,
           nch, cw2, out1, (const T*)part2, out2);
  return cudaGetLastError();
}

template <typename T>
cudaError_t colsum(const T* X, int n, int H, T* out, T* part, cudaStream_t s) {
  return colsum2<T>(X, nullptr, n, H, out, nullptr, part, s);
}

#define GFM_FVEC_CASES(M) M(1, 1) M(1, 2) M(1, 4) M(1, 8) M(1, 16) M(1, 32) M(2, 32) M(4, 32)

template <typename T>
cudaError_t force_fwd_edges(const T* P, int n, int H, const int* rowptr, const int* col_src,
                            const T* dx, const T* c, const T* u, T* f, int flags, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int nv = 0, lpn = 0;
  if constexpr (std::is_same<T, float>::value) {
    int slabs = 1;
    if (!(flags & GFM_FLAG_SCALAR) && force_vec_shape(H, nv, lpn, &slabs)) {
      if (slabs == 2 || slabs == 4 || slabs == 8) {
        const int grid = ceil_div(n, 8 / slabs);
        const bool fast = fast_tanh_on();
#define GFM_FS(SL_)                                                                                 \
  if (slabs == SL_) {                                                                               \
    if (fast)                                                                                       \
      launch_k(k_force_fwd_slab<SL_, true>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, c, u, f);      \
    else                                                                                            \
      launch_k(k_force_fwd_slab<SL_, false>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, c, u, f);     \
  }
        GFM_FS(2) GFM_FS(4) GFM_FS(8)
#undef GFM_FS
        return cudaGetLastError();
      }
      const int grid = ceil_div(n, 8 * (32 / lpn));
#define GFM_FF(NV_, LPN_)                                                                    \
  if (nv == NV_ && lpn == LPN_) {                                                            \
    if (fast_tanh_on())                                                        \
      launch_k(k_force_fwd_vec<NV_, LPN_, true>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, c, u, f); \
    else                                                                                     \
      launch_k(k_force_fwd_vec<NV_, LPN_, false>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, c, u, f); \
    return cudaGetLastError();                                                               \
  }
      GFM_FVEC_CASES(GFM_FF)
#undef GFM_FF
    }
  }
  launch_k(k_force_fwd_warp<T>, ceil_div(n, 8), 256, 0, s, P, n, H, rowptr, col_src, dx, c, u, f);
  return cudaGetLastError();
}

template <typename T>
cudaError_t force_bwd_edges(const T* P, int n, int H, const int* rowptr, const int* col_src,
                            const int* csc_ptr, const int* csc_eid, const int* csc_dst,
                            const T* dx, const T* df, const T* c, const T* u, T* Ddst, T* TU,
                            T* S, int flags, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int nv = 0, lpn = 0;
  if constexpr (std::is_same<T, float>::value) {
    int slabs = 1;
    if (!(flags & GFM_FLAG_SCALAR) && force_vec_shape(H, nv, lpn, &slabs)) {
      const dim3 grid(ceil_div(n, 8 * (32 / lpn)), slabs);
#define GFM_FB(NV_, LPN_)                                                                         \
  if (nv == NV_ && lpn == LPN_) {                                                                 \
    if (fast_tanh_on()) {                                                           \
      launch_k(k_force_bwd_dst_vec<NV_, LPN_, true>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, df, \
                                                                c, u, Ddst, TU);                  \
      launch_k(k_force_bwd_src_vec<NV_, LPN_, true>, grid, 256, 0, s, P, n, H, csc_ptr, csc_eid,        \
                                                                csc_dst, dx, df, c, u, Ddst, S);  \
    } else {                                                                                      \
      launch_k(k_force_bwd_dst_vec<NV_, LPN_, false>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, df,\
                                                                 c, u, Ddst, TU);                 \
      launch_k(k_force_bwd_src_vec<NV_, LPN_, false>, grid, 256, 0, s, P, n, H, csc_ptr, csc_eid,       \
                                                                 csc_dst, dx, df, c, u, Ddst, S); \
    }                                                                                             \
    return cudaGetLastError();                                                                    \
  }
      GFM_FVEC_CASES(GFM_FB)
#undef GFM_FB
    }
  }
  const long long total = (long long)n * H;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  launch_k(k_force_bwd_dst_scalar<T>, grid, 256, 0, s, P, n, H, rowptr, col_src, dx, df, c, u, Ddst, TU);
  launch_k(k_force_bwd_src_scalar<T>, grid, 256, 0, s, P, n, H, csc_ptr, csc_eid, csc_dst, dx, df, c, u,
                                                 Ddst, S);
  return cudaGetLastError();
}

template cudaError_t force_fwd_edges<float>(const float*, int, int, const int*, const int*,
                                            const float*, const float*, const float*, float*, int,
                                            cudaStream_t);
template cudaError_t force_fwd_edges<double>(const double*, int, int, const int*, const int*,
                                             const double*, const double*, const double*, double*,
                                             int, cudaStream_t);
template cudaError_t force_bwd_edges<float>(const float*, int, int, const int*, const int*,
                                            const int*, const int*, const int*, const float*,
                                            const float*, const float*, const float*, float*,
                                            float*, float*, int, cudaStream_t);
template cudaError_t force_bwd_edges<double>(const double*, int, int, const int*, const int*,
                                             const int*, const int*, const int*, const double*,
                                             const double*, const double*, const double*, double*,
                                             double*, double*, int, cudaStream_t);
template cudaError_t colsum<float>(const float*, int, int, float*, float*, cudaStream_t);
template cudaError_t colsum<double>(const double*, int, int, double*, double*, cudaStream_t);
template cudaError_t colsum2<float>(const float*, const float*, int, int, float*, float*, float*,
                                    cudaStream_t);
template cudaError_t colsum2<double>(const double*, const double*, int, int, double*, double*,
                                     double*, cudaStream_t);

}  // namespace gfm
