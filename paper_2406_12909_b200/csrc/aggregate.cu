// Deterministic segmented aggregation over the dst-sorted CSR (forward) and
// its backward as a src-sorted CSC gather -- no atomics anywhere.
//
// Reference: _aggregate / _aggregate_backward (model.py:293-341), the message
// msg = h[src] * w (model.py:354) and the scatter dh_in[src] += dmsg * w
// (model.py:561).  Extensions (parity unpinned): std (PyG convention) and
// PNA = concat[sum, mean, max, std].
//
// Output row layout for the parts mask (bit order sum, mean, max, std): the
// present parts are concatenated, each H wide.  argmax holds the CSR position
// of the FIRST edge attaining the max per (node, column) (model.py:304-316),
// -1 for an empty neighbourhood.
//
// Two instantiations:
//  * vectorised float32 (H % 4 == 0, H/4 lanes per node up to 32 lanes with
//    1, 2 or 4 float4 per lane): lanes of a node group read the neighbour's
//    row slice with 16-byte coalesced loads, edges unrolled 4 deep for
//    memory-level parallelism.  Accumulation is sequential in CSR order.
//  * scalar (float64, or float32 with odd H): one thread per (node, column);
//    sums follow numpy's reduceat order (x0 + pairwise(x1..)) with separately
//    rounded operations, which makes the float64 result bit-identical to
//    np.add.reduceat / np.maximum.reduceat.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"

// CSC slots batched per iteration (32-lane and narrow rows), with a max part (3-4
// rows per slot) / without: 1 / 2 (C3 pna: 1 is 4% faster than 2; C5 random
// sum at E = 16M: 2 reaches 0.67 of HBM, 1 0.53; tools/agg_knobs3.sh)
#ifndef GFM_AGG_BWD_U
#define GFM_AGG_BWD_U 1
#endif
#ifndef GFM_AGG_BWD_U_DEEP
#define GFM_AGG_BWD_U_DEEP 2
#endif
// 32-lane rows without a max part (one or two gathered rows per slot): 3
// slots (C5 random sum 0.67 -> 0.73 of HBM; narrow rows lose with 3)
// 32-lane rows WITH a max part and scattered (non-local) sources: 2 slots
// (C5 random pna at E = 16M, H >= 128: 0.58-0.60 -> 0.63-0.64 of HBM; the
// L2-local C3 batches keep 1)
#ifndef GFM_AGG_BWD_U_MAXSCAT
#define GFM_AGG_BWD_U_MAXSCAT 2
#endif
#ifndef GFM_AGG_BWD_U_DEEP32
#define GFM_AGG_BWD_U_DEEP32 3
#endif
// dmax rows loaded with G / coef / argmax (1) or after the argmax compare
// (0): the dependent load cost 19% at C3 (tools/agg_knobs3.sh, round 2)
#ifndef GFM_AGG_BWD_PFMAX
#define GFM_AGG_BWD_PFMAX 1
#endif
#ifndef GFM_AGG_FWD_UF
#define GFM_AGG_FWD_UF 4
#endif

namespace gfm {

struct AggLayout {
  int K;                          // number of parts
  int o_sum, o_mean, o_max, o_std;  // column offset of each part (-1 absent)
};

__host__ __device__ inline AggLayout agg_layout(int parts, int H) {
  AggLayout L;
  int k = 0;
  L.o_sum = (parts & GFM_PART_SUM) ? (k++) * H : -1;
  L.o_mean = (parts & GFM_PART_MEAN) ? (k++) * H : -1;
  L.o_max = (parts & GFM_PART_MAX) ? (k++) * H : -1;
  L.o_std = (parts & GFM_PART_STD) ? (k++) * H : -1;
  L.K = k;
  return L;
}

// argmax storage: int32 CSR positions, or (GFM_FLAG_ARGMAX_U8) their low
// byte -- unique within a row of <= 256 edges, which is all the backward's
// "is this edge the row's argmax" test needs (4x fewer gathered bytes)
__device__ __forceinline__ void am_store(int* am, long long idx, int p, bool u8) {
  if (u8)
    reinterpret_cast<unsigned char*>(am)[idx] = (unsigned char)(p & 0xFF);
  else
    am[idx] = p;
}
__device__ __forceinline__ int am_load(const int* am, long long idx, bool u8) {
  return u8 ? (int)reinterpret_cast<const unsigned char*>(am)[idx] : am[idx];
}

// ------------------------------------------------------------ embedding
template <typename T>
__global__ void k_embed(const int* __restrict__ z, int n, const T* __restrict__ emb, int H,
                        T* __restrict__ h) {
  pdl_entry();
  // 2D: blockIdx.y / threadIdx.y over rows, x over columns (no 64-bit divides)
  for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < n; i += gridDim.y * blockDim.y) {
    const T* src = emb + (long long)(z[i] - 1) * H;  // model.py:351
    T* dst = h + (long long)i * H;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < H; c += gridDim.x * blockDim.x)
      dst[c] = src[c];
  }
}

// float4 rows (H % 4 == 0, 16-byte aligned rows)
__global__ void k_embed4(const int* __restrict__ z, int n, const float4* __restrict__ emb, int H4,
                         float4* __restrict__ h) {
  pdl_entry();
  for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < n; i += gridDim.y * blockDim.y) {
    const float4* src = emb + (long long)(z[i] - 1) * H4;
    float4* dst = h + (long long)i * H4;
    for (int c = threadIdx.x; c < H4; c += blockDim.x) dst[c] = __ldg(src + c);
  }
}

// ------------------------------------------------------------ forward, scalar
template <typename T>
__global__ void k_agg_fwd_scalar(const T* __restrict__ h, int n_nodes, int H,
                                 const int* __restrict__ rowptr, const int* __restrict__ col_src,
                                 const T* __restrict__ w, int parts, T* __restrict__ agg,
                                 int* __restrict__ argmax, T* __restrict__ stat_mean, int am_u8) {
  pdl_entry();
  const AggLayout L = agg_layout(parts, H);
  const int ld = L.K * H;
  const long long total = (long long)n_nodes * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / H), c = (int)(idx % H);
    const int beg = rowptr[i], end = rowptr[i + 1];
    const int deg = end - beg;
    T* out = agg + (long long)i * ld;
    if (deg == 0) {
      if (L.o_sum >= 0) out[L.o_sum + c] = T(0);
      if (L.o_mean >= 0) out[L.o_mean + c] = T(0);
      if (L.o_max >= 0) out[L.o_max + c] = T(0);
      if (L.o_std >= 0) out[L.o_std + c] = T(0);
      if (argmax && L.o_max >= 0) am_store(argmax, idx, -1, am_u8);
      if (stat_mean) stat_mean[idx] = T(0);
      continue;
    }
    auto msg = [&](long long p) -> T {
      return mul_rn(h[(long long)col_src[p] * H + c], w[p]);
    };
    if (L.o_sum >= 0 || L.o_mean >= 0 || L.o_std >= 0) {
      const T s1 = add_rn(msg(beg), np_pairwise<T>(msg, beg + 1, deg - 1));
      const T dg = (T)deg;
      const T mean = div_rn(s1, dg);
      if (L.o_sum >= 0) out[L.o_sum + c] = s1;
      if (L.o_mean >= 0) out[L.o_mean + c] = mean;
      if (L.o_std >= 0) {  // moments in float64 (same ops as before for T = double)
        auto md = [&](long long p) -> double { return (double)msg(p); };
        auto sq = [&](long long p) -> double {
          const double m = md(p);
          return __dmul_rn(m, m);
        };
        const double s1d = __dadd_rn(md(beg), np_pairwise<double>(md, beg + 1, deg - 1));
        const double s2d = __dadd_rn(sq(beg), np_pairwise<double>(sq, beg + 1, deg - 1));
        const double mu = __ddiv_rn(s1d, (double)deg);
        const double var = __dsub_rn(__ddiv_rn(s2d, (double)deg), __dmul_rn(mu, mu));
        out[L.o_std + c] = var > 1e-5 ? (T)__dsqrt_rn(var) : T(0);
        if (stat_mean) stat_mean[idx] = (T)mu;
      }
    }
    if (L.o_max >= 0) {
      T best = msg(beg);
      int arg = beg;
      for (int p = beg + 1; p < end; ++p) {
        T m = msg(p);
        if (m > best) {
          best = m;
          arg = p;
        }
      }
      out[L.o_max + c] = best;
      if (argmax) am_store(argmax, idx, arg, am_u8);
    }
  }
}

// ------------------------------------------------------------ forward, float4
// One node's PNA row over the float4 columns v*LPN + cb (v < NV); `ld(sj, v)`
// returns that column slice of source row sj (global or shared-memory staged).
template <int NV, int LPN, typename Ld>
__device__ __forceinline__ void agg_fwd_node(Ld ld, int node, int cb, int H,
                                             const int* __restrict__ rowptr,
                                             const int* __restrict__ col_src,
                                             const float* __restrict__ w, const AggLayout& L,
                                             float* __restrict__ agg, int* __restrict__ argmax,
                                             float* __restrict__ stat_mean, bool am_u8) {
  const bool need_s = L.o_sum >= 0 || L.o_mean >= 0 || L.o_std >= 0;
  const bool need_q = L.o_std >= 0;
  const bool need_m = L.o_max >= 0;
  const int beg = rowptr[node], end = rowptr[node + 1];
  // std accumulates around the first message (x - x0) to avoid the
  // E[x^2] - E[x]^2 cancellation in float32
  float4 s[NV], d1[NV], q[NV], x0[NV], mx[NV];
  int4 am[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    s[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    q[v] = s[v];
    d1[v] = s[v];
    x0[v] = s[v];
    mx[v] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    am[v] = make_int4(-1, -1, -1, -1);
  }
  // packed f32x2 updates (add4/mul4/fma4); `first` (a literal at each call)
  // peels the x0 capture out of the edge loop
  auto consume = [&](const float4 (&r)[NV], float ww, int p, bool first) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 m = mul4(r[v], bcast4(ww));
      if (need_s) s[v] = add4(s[v], m);
      if (need_q) {
        if (first) x0[v] = m;
        const float4 d = sub4(m, x0[v]);
        d1[v] = add4(d1[v], d);
        q[v] = fma4(d, d, q[v]);
      }
      if (need_m) {
        if (m.x > mx[v].x) { mx[v].x = m.x; am[v].x = p; }
        if (m.y > mx[v].y) { mx[v].y = m.y; am[v].y = p; }
        if (m.z > mx[v].z) { mx[v].z = m.z; am[v].z = p; }
        if (m.w > mx[v].w) { mx[v].w = m.w; am[v].w = p; }
      }
    }
  };
  int p = beg;
  if (p < end) {
    const int sj = __ldg(col_src + p);
    const float ww = __ldg(w + p);
    float4 r[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) r[v] = ld(sj, v);
    consume(r, ww, p, true);
    ++p;
  }
  if constexpr (LPN == 32) {
    // the node's LPN lanes load LPN (src, w) pairs at once (one coalesced load
    // each) and broadcast them with shuffles, instead of every lane loading
    // every index
    const int gl = (threadIdx.x & 31) % LPN;
    const unsigned gmask =
        LPN == 32 ? 0xffffffffu : (((1u << LPN) - 1u) << ((threadIdx.x & 31) - gl));
    for (int c0 = p; c0 < end; c0 += LPN) {
      const int cnt = min(LPN, end - c0);
      int my_s = 0;
      float my_w = 0.f;
      if (gl < cnt) {
        my_s = __ldg(col_src + c0 + gl);
        my_w = __ldg(w + c0 + gl);
      }
      int e = 0;
      constexpr int UF = GFM_AGG_FWD_UF;  // rows in flight per lane
      for (; e + UF <= cnt; e += UF) {
        int sj[UF];
        float ww[UF];
#pragma unroll
        for (int u = 0; u < UF; ++u) {
          sj[u] = __shfl_sync(gmask, my_s, e + u, LPN);
          ww[u] = __shfl_sync(gmask, my_w, e + u, LPN);
        }
        float4 r[UF][NV];
#pragma unroll
        for (int u = 0; u < UF; ++u)
#pragma unroll
          for (int v = 0; v < NV; ++v) r[u][v] = ld(sj[u], v);
#pragma unroll
        for (int u = 0; u < UF; ++u) consume(r[u], ww[u], c0 + e + u, false);
      }
      for (; e < cnt; ++e) {
        const int sj = __shfl_sync(gmask, my_s, e, LPN);
        const float ww = __shfl_sync(gmask, my_w, e, LPN);
        float4 r[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) r[v] = ld(sj, v);
        consume(r, ww, c0 + e, false);
      }
    }
  } else {  // narrow rows: the node's whole CSR row fits in a few unrolled loads
    for (; p + 4 <= end; p += 4) {
      int sj[4];
      float ww[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sj[u] = __ldg(col_src + p + u);
        ww[u] = __ldg(w + p + u);
      }
      float4 r[4][NV];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) r[u][v] = ld(sj[u], v);
#pragma unroll
      for (int u = 0; u < 4; ++u) consume(r[u], ww[u], p + u, false);
    }
    for (; p < end; ++p) {
      const int sj = __ldg(col_src + p);
      const float ww = __ldg(w + p);
      float4 r[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = ld(sj, v);
      consume(r, ww, p, false);
    }
  }
  const int deg = end - beg;
  const float inv = deg > 0 ? 1.f / (float)deg : 0.f;
  float4* out4 = reinterpret_cast<float4*>(agg + (long long)node * L.K * H);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int c4 = v * LPN + cb;
    float4 mean = make_float4(s[v].x * inv, s[v].y * inv, s[v].z * inv, s[v].w * inv);
    if (L.o_sum >= 0) out4[(L.o_sum >> 2) + c4] = s[v];
    if (L.o_mean >= 0) out4[(L.o_mean >> 2) + c4] = mean;
    if (need_m) {
      float4 o = deg > 0 ? mx[v] : make_float4(0.f, 0.f, 0.f, 0.f);
      out4[(L.o_max >> 2) + c4] = o;
      if (argmax) {
        if (am_u8)  // 4 low bytes -> one 32-bit store
          reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(argmax) + (long long)node * H)[c4] =
              (unsigned)(am[v].x & 0xFF) | (unsigned)(am[v].y & 0xFF) << 8 |
              (unsigned)(am[v].z & 0xFF) << 16 | (unsigned)(am[v].w & 0xFF) << 24;
        else
          reinterpret_cast<int4*>(argmax + (long long)node * H)[c4] = am[v];
      }
    }
    if (need_q) {
      auto sd = [&](float sq, float sd1) {
        const float mu = sd1 * inv;
        float var = sq * inv - mu * mu;
        return var > 1e-5f ? sqrtf(var) : 0.f;
      };
      float4 o = make_float4(sd(q[v].x, d1[v].x), sd(q[v].y, d1[v].y), sd(q[v].z, d1[v].z),
                             sd(q[v].w, d1[v].w));
      out4[(L.o_std >> 2) + c4] = o;
      if (stat_mean) reinterpret_cast<float4*>(stat_mean + (long long)node * H)[c4] = mean;
    }
  }
}

// resident 256-thread CTAs per SM the register allocation must allow: the
// gather kernels are latency bound (long-scoreboard stalls, L2 far from its
// throughput cap), so more warps in flight is the lever
#ifndef GFM_AGG_FWD_MINB
#define GFM_AGG_FWD_MINB 4
#endif
#ifndef GFM_AGG_BWD_MINB
#define GFM_AGG_BWD_MINB 5
#endif
template <int NV, int LPN, bool U8>
__global__ void __launch_bounds__(256, NV == 1 ? GFM_AGG_FWD_MINB : 1)
    k_agg_fwd_vec(const float* __restrict__ h, int n_nodes, int H, const int* __restrict__ rowptr,
                  const int* __restrict__ col_src, const float* __restrict__ w, int parts,
                  float* __restrict__ agg, int* __restrict__ argmax, float* __restrict__ stat_mean) {
  pdl_entry();
  constexpr int NPW = 32 / LPN;  // nodes per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane % LPN;
  const int node = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NPW + lane / LPN;
  if (node >= n_nodes) return;
  // blockIdx.y selects a slab of NV*LPN float4 columns (wide H uses several
  // slabs instead of more registers per lane: occupancy hides gather latency)
  const int cb = blockIdx.y * (NV * LPN) + sub;
  const AggLayout L = agg_layout(parts, H);
  const float4* __restrict__ h4 = reinterpret_cast<const float4*>(h);
  const int H4 = H >> 2;
  agg_fwd_node<NV, LPN>(
      [&](int sj, int v) { return __ldg(h4 + (long long)sj * H4 + v * LPN + cb); }, node, cb, H,
      rowptr, col_src, w, L, agg, argmax, stat_mean, U8);
}

// 16-byte global -> shared copy without a register round trip: a block's
// whole staging loop is in flight at once (cp.async.cg, L2-only)
__device__ __forceinline__ void stage16(void* smem, const void* gptr) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gptr) : "memory");
}
__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Block-wide [lo, hi] of idx[e0, e1) (lo > hi when empty).
__device__ __forceinline__ void block_minmax(const int* __restrict__ idx, int e0, int e1, int& lo,
                                             int& hi) {
  __shared__ int s_lo[8], s_hi[8];
  int a = INT_MAX, b = -1;
  for (int e = e0 + (int)threadIdx.x; e < e1; e += blockDim.x) {
    const int v = __ldg(idx + e);
    a = min(a, v);
    b = max(b, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    s_lo[threadIdx.x >> 5] = a;
    s_hi[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  lo = s_lo[0];
  hi = s_hi[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
    lo = min(lo, s_lo[k]);
    hi = max(hi, s_hi[k]);
  }
}

// Shared-memory staged forward.  A block owns `nb` consecutive dst nodes and
// one LPN-float4 column slab.  Batched graphs keep every edge inside its graph,
// so the block's sources span a short row range [lo, hi]: that slab of h is
// staged once with coalesced 16-byte loads and every per-edge gather is then a
// shared-memory read (HBM/L2 see each staged row once per block instead of
// once per edge).  Ranges wider than cap_rows fall back to global gathers.
template <int LPN>
__global__ void __launch_bounds__(256)
    k_agg_fwd_tile(const float* __restrict__ h, int n_nodes, int H, const int* __restrict__ rowptr,
                   const int* __restrict__ col_src, const float* __restrict__ w, int parts,
                   float* __restrict__ agg, int* __restrict__ argmax,
                   float* __restrict__ stat_mean, int nb, int cap_rows) {
  pdl_entry();
  extern __shared__ float4 stage[];  // [cap_rows][LPN]
  const int a = blockIdx.x * nb, b = min(n_nodes, a + nb);
  const int cs = blockIdx.y * LPN;  // slab's first float4 column
  const int H4 = H >> 2;
  const float4* __restrict__ h4 = reinterpret_cast<const float4*>(h);
  int lo, hi;
  block_minmax(col_src, rowptr[a], rowptr[b], lo, hi);
  const bool staged = hi >= lo && hi - lo < cap_rows;
  if (staged) {
    const int total = (hi - lo + 1) * LPN;
    for (int t = threadIdx.x; t < total; t += blockDim.x)
      stage16(stage + t, h4 + (long long)(lo + t / LPN) * H4 + cs + t % LPN);
    stage_wait();
  }
  __syncthreads();
  const AggLayout L = agg_layout(parts, H);
  const int sub = threadIdx.x % LPN, cb = cs + sub;
  const int npp = blockDim.x / LPN;
  for (int node = a + (int)threadIdx.x / LPN; node < b; node += npp) {
    if (staged)
      agg_fwd_node<1, LPN>([&](int sj, int) { return stage[(sj - lo) * LPN + sub]; }, node, cb,
                           H, rowptr, col_src, w, L, agg, argmax, stat_mean, false);
    else
      agg_fwd_node<1, LPN>([&](int sj, int) { return __ldg(h4 + (long long)sj * H4 + cb); },
                           node, cb, H, rowptr, col_src, w, L, agg, argmax, stat_mean, false);
  }
}

// ------------------------------------------------------------ backward prep
// G = dsum + dmean/deg - coef*mean,  coef = dstd / (deg*std)  (std > 0)
template <typename T>
__global__ void k_agg_bwd_prep(const T* __restrict__ dagg, const int* __restrict__ rowptr,
                               int n_nodes, int H, int parts, const T* __restrict__ agg,
                               const T* __restrict__ stat_mean, T* __restrict__ G,
                               T* __restrict__ coef) {
  pdl_entry();
  const AggLayout L = agg_layout(parts, H);
  const int ld = L.K * H;
  const long long total = (long long)n_nodes * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / H), c = (int)(idx % H);
    const int deg = rowptr[i + 1] - rowptr[i];
    const T* d = dagg + (long long)i * ld;
    T g = T(0);
    if (L.o_sum >= 0) g = d[L.o_sum + c];
    if (L.o_mean >= 0 && deg > 0) {
      T m = div_rn(d[L.o_mean + c], (T)deg);  // model.py:333
      g = (L.o_sum >= 0) ? add_rn(g, m) : m;
    }
    T cf = T(0);
    if (L.o_std >= 0 && deg > 0) {
      const T sd = agg[(long long)i * ld + L.o_std + c];
      if (sd > T(0)) {
        cf = d[L.o_std + c] / ((T)deg * sd);
        g = g - cf * stat_mean[idx];
      }
    }
    G[idx] = g;
    if (coef) coef[idx] = cf;
  }
}

// float32, H % 4 == 0: one thread per (node, 4 columns), 16-byte loads
__global__ void __launch_bounds__(256)
    k_agg_bwd_prep_vec(const float* __restrict__ dagg, const int* __restrict__ rowptr, int n_nodes,
                       int H, int parts, const float* __restrict__ agg,
                       const float* __restrict__ stat_mean, float* __restrict__ G,
                       float* __restrict__ coef, int interleave) {
  pdl_entry();
  const AggLayout L = agg_layout(parts, H);
  const int H4 = H >> 2, ld4 = (L.K * H) >> 2;
  const long long total = (long long)n_nodes * H4;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / H4), c4 = (int)(idx % H4);
    const int deg = __ldg(rowptr + i + 1) - __ldg(rowptr + i);
    const float4* d = reinterpret_cast<const float4*>(dagg) + (long long)i * ld4;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (L.o_sum >= 0) g = __ldg(d + (L.o_sum >> 2) + c4);
    if (L.o_mean >= 0 && deg > 0) {
      const float4 m = __ldg(d + (L.o_mean >> 2) + c4);
      const float id = (float)deg;
      g.x += __fdiv_rn(m.x, id); g.y += __fdiv_rn(m.y, id);
      g.z += __fdiv_rn(m.z, id); g.w += __fdiv_rn(m.w, id);
    }
    float4 cf = make_float4(0.f, 0.f, 0.f, 0.f);
    if (L.o_std >= 0 && deg > 0) {
      const float4 sd = __ldg(reinterpret_cast<const float4*>(agg) + (long long)i * ld4 + (L.o_std >> 2) + c4);
      const float4 ds = __ldg(d + (L.o_std >> 2) + c4);
      const float4 mu = __ldg(reinterpret_cast<const float4*>(stat_mean) + idx);
      const float fd = (float)deg;
      auto one = [&](float s, float dd, float m, float& gg) {
        if (s > 0.f) {
          const float k = dd / (fd * s);
          gg -= k * m;
          return k;
        }
        return 0.f;
      };
      cf.x = one(sd.x, ds.x, mu.x, g.x); cf.y = one(sd.y, ds.y, mu.y, g.y);
      cf.z = one(sd.z, ds.z, mu.z, g.z); cf.w = one(sd.w, ds.w, mu.w, g.w);
    }
    if (interleave) {  // [G | coef] per 4 columns: one 32-byte row slice per (node, c4)
      reinterpret_cast<float4*>(G)[2 * idx] = g;
      reinterpret_cast<float4*>(G)[2 * idx + 1] = cf;
    } else {
      reinterpret_cast<float4*>(G)[idx] = g;
      if (coef) reinterpret_cast<float4*>(coef)[idx] = cf;
    }
  }
}

// ------------------------------------------------------------ backward gather
// dh[j] (= dz W on entry) += sum over CSC slots of w * dmsg, in CSC order
// (np.add.at order).  dmsg = G[dst] + coef[dst]*msg + [argmax==p]*dmax[dst].
// Optional epilogue: out = acc * (1 - gate^2) (the previous layer's tanh').
template <typename T>
__global__ void k_agg_bwd_scalar(const T* __restrict__ G, int ldg, const T* __restrict__ coef,
                                 const T* __restrict__ dmax, int ldm, const int* __restrict__ argmax,
                                 const T* __restrict__ h_in, const int* __restrict__ csc_ptr,
                                 const int* __restrict__ csc_eid, const int* __restrict__ csc_dst,
                                 const T* __restrict__ w, int n_nodes, int H, T* __restrict__ dh,
                                 const T* __restrict__ gate, T* __restrict__ out, int am_u8,
                                 int w_csc) {
  pdl_entry();
  const long long total = (long long)n_nodes * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / H), c = (int)(idx % H);
    T acc = dh[idx];
    const T hj = coef ? h_in[idx] : T(0);
    for (int q = csc_ptr[j]; q < csc_ptr[j + 1]; ++q) {
      const int p = csc_eid[q], i = csc_dst[q];
      const T ww = w[w_csc ? q : p];
      T dm = G ? G[(long long)i * ldg + c] : T(0);
      if (coef) dm = dm + coef[(long long)i * H + c] * (hj * ww);
      if (argmax) {
        if (am_load(argmax, (long long)i * H + c, am_u8) == (am_u8 ? (p & 0xFF) : p))
          dm = G || coef ? dm + dmax[(long long)i * ldm + c] : dmax[(long long)i * ldm + c];
      }
      acc = add_rn(acc, mul_rn(dm, ww));
    }
    if (gate) {
      const T g = gate[idx];
      out[idx] = mul_rn(acc, sub_rn(T(1), mul_rn(g, g)));  // model.py:553
    } else {
      out[idx] = acc;
    }
  }
}

// One CSC node j over float4 columns v*LPN + cb: ldG/ldC/ldA(i, v) return the
// dst row i slice of G / coef / argmax (global or staged); hasG/hasC/hasA say
// which are present.
struct f4x2 {
  float4 a, b;
};
// 32-byte load (sm_100 LDG.E.ENL2.256): G and coef of one (node, c4) at once
__device__ __forceinline__ f4x2 ldg256(const float* p) {
  f4x2 r;
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
        "=f"(r.b.z), "=f"(r.b.w)
      : "l"(p));
  return r;
}

// GC: ldG returns f4x2 {G, coef} (interleaved workspace), ldC is unused
template <int NV, int LPN, bool GC = false, int U = 1, typename LG, typename LC, typename LA>
__device__ __forceinline__ void agg_bwd_node(LG ldG, LC ldC, LA ldA, bool hasG, bool hasC,
                                             bool hasA, int j, int cb, int H,
                                             const float* __restrict__ dmax, int ldm,
                                             const float* __restrict__ h_in,
                                             const int* __restrict__ csc_ptr,
                                             const int* __restrict__ csc_eid,
                                             const int* __restrict__ csc_dst,
                                             const float* __restrict__ w,
                                             const float* __restrict__ dh,
                                             const float* __restrict__ gate,
                                             float* __restrict__ out, bool am_u8 = false,
                                             bool w_csc = false) {
  const int H4 = H >> 2;
  float4 acc[NV], hj[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const long long o = (long long)j * H4 + v * LPN + cb;
    acc[v] = reinterpret_cast<const float4*>(dh)[o];
    hj[v] = hasC ? reinterpret_cast<const float4*>(h_in)[o] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int qb = csc_ptr[j], qe = csc_ptr[j + 1];
  // PF: the max part's dmax row is loaded with the others instead of after
  // the argmax compare (no dependent load; +4 B per channel and edge)
  constexpr bool PF = GFM_AGG_BWD_PFMAX != 0;
  struct Rows {
    float4 g[NV], cf[NV], d[NV];
    int4 a[NV];
  };
  auto load = [&](int i, Rows& r) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      r.g[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      r.cf[v] = r.g[v];
      r.d[v] = r.g[v];
      r.a[v] = make_int4(-1, -1, -1, -1);
      if constexpr (GC) {
        const f4x2 t = ldG(i, v);
        r.g[v] = t.a;
        r.cf[v] = t.b;
      } else {
        if (hasG) r.g[v] = ldG(i, v);
        if (hasC) r.cf[v] = ldC(i, v);
      }
      if (hasA) {
        r.a[v] = ldA(i, v);
        if constexpr (PF)
          r.d[v] = __ldg(reinterpret_cast<const float4*>(dmax + (long long)i * ldm) + v * LPN + cb);
      }
    }
  };
  auto consume = [&](int p, int i, float wv, const Rows& r) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c4 = v * LPN + cb;
      float4 dm = r.g[v];
      if (hasC) dm = fma4(r.cf[v], mul4(hj[v], bcast4(wv)), dm);
      if (hasA) {
        const int4 am = r.a[v];
        if (am_u8) {
          // four low-byte argmaxes packed in am.x: one byte-wise compare
          const unsigned eq = __vcmpeq4((unsigned)am.x, (unsigned)(p & 0xFF) * 0x01010101u);
          if (eq) {
            const float4 d = PF ? r.d[v]
                                : __ldg(reinterpret_cast<const float4*>(dmax + (long long)i * ldm) + c4);
            if (eq & 0x000000FFu) dm.x += d.x;
            if (eq & 0x0000FF00u) dm.y += d.y;
            if (eq & 0x00FF0000u) dm.z += d.z;
            if (eq & 0xFF000000u) dm.w += d.w;
          }
        } else if (am.x == p || am.y == p || am.z == p || am.w == p) {
          const float4 d = PF ? r.d[v]
                              : __ldg(reinterpret_cast<const float4*>(dmax + (long long)i * ldm) + c4);
          if (am.x == p) dm.x += d.x;
          if (am.y == p) dm.y += d.y;
          if (am.z == p) dm.z += d.z;
          if (am.w == p) dm.w += d.w;
        }
      }
      acc[v] = fma4(dm, bcast4(wv), acc[v]);
    }
  };
  if constexpr (LPN == 32) {
    // the node's 32 lanes load 32 CSC slots (eid, dst, w) at once and
    // broadcast them with shuffles; U slots per batch: all their row loads
    // issue before the (in-order) accumulation (full batches unpredicated,
    // then a one-slot tail)
    const int gl = threadIdx.x & 31;
    for (int c0 = qb; c0 < qe; c0 += 32) {
      const int cnt = min(32, qe - c0);
      int my_p = 0, my_i = 0;
      float my_w = 0.f;
      if (gl < cnt) {
        my_p = __ldg(csc_eid + c0 + gl);
        my_i = __ldg(csc_dst + c0 + gl);
        my_w = __ldg(w + (w_csc ? c0 + gl : my_p));
      }
      int e = 0;
      for (; e + U <= cnt; e += U) {
        int p[U], i[U];
        float ww[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          p[u] = __shfl_sync(0xffffffffu, my_p, e + u);
          i[u] = __shfl_sync(0xffffffffu, my_i, e + u);
          ww[u] = __shfl_sync(0xffffffffu, my_w, e + u);
        }
        Rows r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) load(i[u], r[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) consume(p[u], i[u], ww[u], r[u]);
      }
      for (; e < cnt; ++e) {
        const int p = __shfl_sync(0xffffffffu, my_p, e);
        const int i = __shfl_sync(0xffffffffu, my_i, e);
        const float wv = __shfl_sync(0xffffffffu, my_w, e);
        Rows r;
        load(i, r);
        consume(p, i, wv, r);
      }
    }
  } else {
    // narrow rows (several nodes per warp): U slots per batch (1 with a max
    // part: 2 measured 5% slower at C2; 2 without: C5 random sum at H = 64
    // 0.54 -> 0.73 of HBM)
    constexpr int UN = U;
    int q = qb;
    // (UN == 1: the plain loop below -- the batched form with one slot
    // measured 10% slower at C2)
    if constexpr (UN > 1) for (; q + UN <= qe; q += UN) {
      int p[UN], i[UN];
      float ww[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        p[u] = __ldg(csc_eid + q + u);
        i[u] = __ldg(csc_dst + q + u);
        ww[u] = __ldg(w + (w_csc ? q + u : p[u]));
      }
      Rows r[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) load(i[u], r[u]);
#pragma unroll
      for (int u = 0; u < UN; ++u) consume(p[u], i[u], ww[u], r[u]);
    }
    for (; q < qe; ++q) {
      const int p = __ldg(csc_eid + q), i = __ldg(csc_dst + q);
      const float wv = __ldg(w + (w_csc ? q : p));
      Rows r;
      load(i, r);
      consume(p, i, wv, r);
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const long long o = (long long)j * H4 + v * LPN + cb;
    float4 r = acc[v];
    if (gate) {
      const float4 g = reinterpret_cast<const float4*>(gate)[o];
      r.x *= 1.f - g.x * g.x; r.y *= 1.f - g.y * g.y; r.z *= 1.f - g.z * g.z; r.w *= 1.f - g.w * g.w;
    }
    reinterpret_cast<float4*>(out)[o] = r;
  }
}

template <int NV, int LPN, bool U8, bool GC = false, int U = 1>
__global__ void __launch_bounds__(256, NV == 1 ? (LPN == 32 ? (GFM_AGG_BWD_MINB > 4 ? 4 : GFM_AGG_BWD_MINB) : GFM_AGG_BWD_MINB) : 1)
    k_agg_bwd_vec(const float* __restrict__ G, int ldg, const float* __restrict__ coef,
                  const float* __restrict__ dmax, int ldm, const int* __restrict__ argmax,
                  const float* __restrict__ h_in, const int* __restrict__ csc_ptr,
                  const int* __restrict__ csc_eid, const int* __restrict__ csc_dst,
                  const float* __restrict__ w, int n_nodes, int H, float* __restrict__ dh,
                  const float* __restrict__ gate, float* __restrict__ out, int w_csc) {
  pdl_entry();
  constexpr int NPW = 32 / LPN;
  const int lane = threadIdx.x & 31;
  const int sub = lane % LPN;
  const int j = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NPW + lane / LPN;
  if (j >= n_nodes) return;
  const int cb = blockIdx.y * (NV * LPN) + sub;  // column slab (see k_agg_fwd_vec)
  agg_bwd_node<NV, LPN, GC, U>(
      [&](int i, int v) {
        if constexpr (GC) {
          return ldg256(G + ((long long)i * (H >> 2) + v * LPN + cb) * 8);
        } else {
          return __ldg(reinterpret_cast<const float4*>(G + (long long)i * ldg) + v * LPN + cb);
        }
      },
      [&](int i, int v) {
        return __ldg(reinterpret_cast<const float4*>(coef + (long long)i * H) + v * LPN + cb);
      },
      [&](int i, int v) {
        if constexpr (U8) {  // 4 low-byte argmaxes in one 32-bit load
          const unsigned b = __ldg(reinterpret_cast<const unsigned*>(
                                       reinterpret_cast<const unsigned char*>(argmax) + (long long)i * H) +
                                   v * LPN + cb);
          return make_int4((int)b, 0, 0, 0);  // packed: compared with __vcmpeq4
        }
        return __ldg(reinterpret_cast<const int4*>(argmax + (long long)i * H) + v * LPN + cb);
      },
      G != nullptr, coef != nullptr, argmax != nullptr, j, cb, H, dmax, ldm, h_in, csc_ptr,
      csc_eid, csc_dst, w, dh, gate, out, U8, w_csc != 0);
}

// Shared-memory staged backward (see k_agg_fwd_tile): a block owns nb
// consecutive CSC (source) nodes and one LPN-float4 column slab, stages the
// dst-row range of G, coef and argmax it touches, then gathers from smem.
template <int LPN>
__global__ void __launch_bounds__(256)
    k_agg_bwd_tile(const float* __restrict__ G, int ldg, const float* __restrict__ coef,
                   const float* __restrict__ dmax, int ldm, const int* __restrict__ argmax,
                   const float* __restrict__ h_in, const int* __restrict__ csc_ptr,
                   const int* __restrict__ csc_eid, const int* __restrict__ csc_dst,
                   const float* __restrict__ w, int n_nodes, int H, float* __restrict__ dh,
                   const float* __restrict__ gate, float* __restrict__ out, int nb,
                   int cap_rows, int w_csc) {
  pdl_entry();
  extern __shared__ float4 stage[];  // [G | coef | argmax] each [cap_rows][LPN]
  const int a0 = blockIdx.x * nb, b0 = min(n_nodes, a0 + nb);
  const int cs = blockIdx.y * LPN;
  const bool hasG = G != nullptr, hasC = coef != nullptr, hasA = argmax != nullptr;
  int lo, hi;
  block_minmax(csc_dst, csc_ptr[a0], csc_ptr[b0], lo, hi);
  const bool staged = hi >= lo && hi - lo < cap_rows;
  float4* sG = stage;
  float4* sC = stage + (size_t)cap_rows * LPN;
  int4* sA = reinterpret_cast<int4*>(stage + 2 * (size_t)cap_rows * LPN);
  if (staged) {
    const int total = (hi - lo + 1) * LPN;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const long long r = lo + t / LPN;
      const int c = cs + t % LPN;
      if (hasG) stage16(sG + t, reinterpret_cast<const float4*>(G + r * ldg) + c);
      if (hasC) stage16(sC + t, reinterpret_cast<const float4*>(coef + r * H) + c);
      if (hasA) stage16(sA + t, reinterpret_cast<const int4*>(argmax + r * H) + c);
    }
    stage_wait();
  }
  __syncthreads();
  const int sub = threadIdx.x % LPN, cb = cs + sub;
  const int npp = blockDim.x / LPN;
  for (int j = a0 + (int)threadIdx.x / LPN; j < b0; j += npp) {
    if (staged)
      agg_bwd_node<1, LPN>([&](int i, int) { return sG[(i - lo) * LPN + sub]; },
                           [&](int i, int) { return sC[(i - lo) * LPN + sub]; },
                           [&](int i, int) { return sA[(i - lo) * LPN + sub]; }, hasG, hasC,
                           hasA, j, cb, H, dmax, ldm, h_in, csc_ptr, csc_eid, csc_dst, w, dh,
                           gate, out, false, w_csc != 0);
    else
      agg_bwd_node<1, LPN>(
          [&](int i, int) {
            return __ldg(reinterpret_cast<const float4*>(G + (long long)i * ldg) + cb);
          },
          [&](int i, int) {
            return __ldg(reinterpret_cast<const float4*>(coef + (long long)i * H) + cb);
          },
          [&](int i, int) {
            return __ldg(reinterpret_cast<const int4*>(argmax + (long long)i * H) + cb);
          },
          hasG, hasC, hasA, j, cb, H, dmax, ldm, h_in, csc_ptr, csc_eid, csc_dst, w, dh, gate,
          out, false, w_csc != 0);
  }
}

// ------------------------------------------------------------ dispatch
static inline int grid_1d(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

// choose (NV, LPN, slabs) for the float4 path; returns false if H does not
// fit.  H/4 > 32 float4 columns are split into 32-lane slabs (gridDim.y)
// rather than held as NV > 1 registers per lane.
static bool vec_shape(int H, int& nv, int& lpn, int* slabs = nullptr, bool wide2 = false) {
  if (H % 4) return false;
  const int h4 = H / 4;
  if (slabs) {
    *slabs = 1;
    if (h4 > 32 && h4 % 32 == 0) {
      // wide2: two float4 per lane (round 1: the forward 5% faster at
      // H = 512, the backward 11% slower; round 2: both faster with one)
      nv = wide2 && h4 % 64 == 0 ? 2 : 1;
      lpn = 32;
      *slabs = h4 / (32 * nv);
      return true;
    }
  }
  for (int v : {1, 2, 4}) {
    if (h4 % v) continue;
    int l = h4 / v;
    if (l <= 32 && (l & (l - 1)) == 0) {
      nv = v;
      lpn = l;
      return true;
    }
  }
  return false;
}

#define GFM_VEC_CASES(MACRO) \
  MACRO(1, 1) MACRO(1, 2) MACRO(1, 4) MACRO(1, 8) MACRO(1, 16) MACRO(1, 32) MACRO(2, 32) MACRO(4, 32)

// The shared-memory staged tiles are opt-in (GFM_AGG_TILE=1): measured on
// B200 they lose to the register gathers at C2 and C3 (the gathers are
// issue-bound, not L2-bound, and staging adds a serial phase per block).
static int tile_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// A/B knob of the backward gather: GFM_AGG_GC=1 interleaved [G | coef]
// workspace read with one 32-byte load per (edge, lane) (default off: equal
// time at C2 / C3).  A node-chunked block mapping (consecutive CSC nodes per
// block, for L1 reuse of their graphs' dst rows) measured 1-25% slower.
static bool gc_env() {
  static int v = -1;
  if (v < 0) v = getenv("GFM_AGG_GC") ? atoi(getenv("GFM_AGG_GC")) : 0;
  return v != 0;
}

static bool no_tile() {
  const char* e = getenv("GFM_AGG_TILE");
  return !(e && e[0] == '1');
}

cudaError_t agg_fwd(int dtype, const void* h, int n, int H, const int* rowptr, const int* col_src,
                    const void* w, int parts, void* agg, int* argmax, void* stat_mean,
                    int force_scalar, int am_u8, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int nv = 0, lpn = 0, slabs = 1;
  if (dtype == GFM_F32 && !force_scalar && !am_u8 && H % 64 == 0 && !no_tile()) {
    // staged tiles: 16-lane (64-column) slabs, 128 dst nodes, <= 384 rows
    constexpr int kLpn = 16;
    const int kNb = tile_env("GFM_AGG_TILE_NB", 128), kCap = tile_env("GFM_AGG_TILE_CAP", 384);
    const size_t smem = (size_t)kCap * kLpn * sizeof(float4);
    cudaFuncSetAttribute(k_agg_fwd_tile<kLpn>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const dim3 grid(ceil_div(n, kNb), H / 64);
    launch_k(k_agg_fwd_tile<kLpn>, grid, 256, smem, s, (const float*)h, n, H, rowptr, col_src,
                                                 (const float*)w, parts, (float*)agg, argmax,
                                                 (float*)stat_mean, kNb, kCap);
    return cudaGetLastError();
  }
  // one float4 per lane and more column slabs (more resident warps): C3
  // forward 392 -> 364 us vs two float4 per lane (GFM_AGG_FWD_WIDE2=1)
  static const bool fwd_wide2 = getenv("GFM_AGG_FWD_WIDE2") != nullptr;
  if (dtype == GFM_F32 && !force_scalar && vec_shape(H, nv, lpn, &slabs, fwd_wide2)) {
    const int nodes_per_block = 8 * (32 / lpn);
    const dim3 grid(ceil_div(n, nodes_per_block), slabs);
#define GFM_FWD_CASE(NV_, LPN_)                                                                \
  if (nv == NV_ && lpn == LPN_) {                                                              \
    if (am_u8)                                                                                 \
      launch_k(k_agg_fwd_vec<NV_, LPN_, true>, grid, 256, 0, s, (const float*)h, n, H, rowptr,   \
               col_src, (const float*)w, parts, (float*)agg, argmax, (float*)stat_mean);      \
    else                                                                                       \
      launch_k(k_agg_fwd_vec<NV_, LPN_, false>, grid, 256, 0, s, (const float*)h, n, H, rowptr,  \
               col_src, (const float*)w, parts, (float*)agg, argmax, (float*)stat_mean);      \
    return cudaGetLastError();                                                                 \
  }
    GFM_VEC_CASES(GFM_FWD_CASE)
#undef GFM_FWD_CASE
  }
  if (dtype == GFM_F32)
    launch_k(k_agg_fwd_scalar<float>, grid_1d((long long)n * H), 256, 0, s,
        (const float*)h, n, H, rowptr, col_src, (const float*)w, parts, (float*)agg, argmax,
        (float*)stat_mean, am_u8);
  else
    launch_k(k_agg_fwd_scalar<double>, grid_1d((long long)n * H), 256, 0, s,
        (const double*)h, n, H, rowptr, col_src, (const double*)w, parts, (double*)agg, argmax,
        (double*)stat_mean, am_u8);
  return cudaGetLastError();
}

cudaError_t agg_bwd(int dtype, const void* dagg, const void* agg, const void* stat_mean,
                    const int* argmax, const void* h_in, const int* rowptr, const int* csc_ptr,
                    const int* csc_eid, const int* csc_dst, const void* w, int n, int H, int parts,
                    void* dh, const void* gate, void* out, void* ws, int force_scalar, int am_u8,
                    cudaStream_t s, int prepped = 0, int w_csc = 0, int local = 0) {
  if (n <= 0) return cudaSuccess;
  const AggLayout L = agg_layout(parts, H);
  int ld = L.K * H;
  const size_t esz = dtype == GFM_F32 ? 4 : 8;
  bool gc = false;  // interleaved [G | coef] workspace, read with 32-byte loads
  // G: dsum alone needs no prep (read dagg in place); mean/std need G/coef
  const void* G = nullptr;
  int ldg = ld;
  const void* coef = nullptr;
  if (prepped) {
    // gfm_layer_bwd_data_agg already wrote G | coef into ws and the max part's
    // gradient as `dagg` [N][H]
    G = ws;
    ldg = H;
    coef = L.o_std >= 0 ? (const void*)((const char*)ws + esz * (size_t)n * H) : nullptr;
  } else if (L.o_mean >= 0 || L.o_std >= 0) {
    int nv0 = 0, lpn0 = 0;
    gc = gc_env() && dtype == GFM_F32 && H % 4 == 0 && !force_scalar && L.o_std >= 0 &&
         vec_shape(H, nv0, lpn0) && no_tile();
    void* Gw = ws;
    void* Cw = L.o_std >= 0 ? (void*)((char*)ws + esz * (size_t)n * H) : nullptr;
    if (dtype == GFM_F32 && H % 4 == 0 && !force_scalar)
      launch_k(k_agg_bwd_prep_vec, grid_1d((long long)n * (H / 4)), 256, 0, s,
          (const float*)dagg, rowptr, n, H, parts, (const float*)agg, (const float*)stat_mean,
          (float*)Gw, (float*)Cw, gc ? 1 : 0);
    else if (dtype == GFM_F32)
      launch_k(k_agg_bwd_prep<float>, grid_1d((long long)n * H), 256, 0, s,
          (const float*)dagg, rowptr, n, H, parts, (const float*)agg, (const float*)stat_mean,
          (float*)Gw, (float*)Cw);
    else
      launch_k(k_agg_bwd_prep<double>, grid_1d((long long)n * H), 256, 0, s,
          (const double*)dagg, rowptr, n, H, parts, (const double*)agg, (const double*)stat_mean,
          (double*)Gw, (double*)Cw);
    G = Gw;
    ldg = H;
    coef = Cw;
  } else if (L.o_sum >= 0) {
    G = (const char*)dagg + esz * L.o_sum;
  }
  const void* dmax =
      L.o_max >= 0 ? (prepped ? dagg : (const void*)((const char*)dagg + esz * L.o_max)) : nullptr;
  if (prepped) ld = H;  // dmax is its own [N][H] buffer
  const int* am = L.o_max >= 0 ? argmax : nullptr;
  int nv = 0, lpn = 0, slabs = 1;
  const bool g_ok = G == nullptr || ldg % 4 == 0;
  if (dtype == GFM_F32 && !force_scalar && !am_u8 && H % 32 == 0 && g_ok && ld % 4 == 0 &&
      !no_tile()) {
    // staged tiles: 8-lane (32-column) slabs, 64 CSC nodes, <= 256 dst rows
    constexpr int kLpn = 8;
    const int kNb = tile_env("GFM_AGG_TILE_NB", 64), kCap = tile_env("GFM_AGG_TILE_CAP", 256);
    const size_t smem = 3 * (size_t)kCap * kLpn * sizeof(float4);
    cudaFuncSetAttribute(k_agg_bwd_tile<kLpn>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const dim3 grid(ceil_div(n, kNb), H / 32);
    launch_k(k_agg_bwd_tile<kLpn>, grid, 256, smem, s,
        (const float*)G, ldg, (const float*)coef, (const float*)dmax, ld, am, (const float*)h_in,
        csc_ptr, csc_eid, csc_dst, (const float*)w, n, H, (float*)dh, (const float*)gate,
        (float*)out, kNb, kCap, w_csc);
    return cudaGetLastError();
  }
  if (dtype == GFM_F32 && !force_scalar && vec_shape(H, nv, lpn, &slabs)) {
    // without a max part (no argmax / dmax rows) the gather carries one or
    // two rows per slot: batch more slots; with one, narrow rows batch two
    // slots unless the caller marks the sources as local (batched small
    // graphs: C2 measured 5% slower with two, C5 random pna at H = 64
    // 0.48 -> 0.59 of HBM)
    const bool deep = am == nullptr || (!local && lpn < 32);
    const int nodes_per_block = 8 * (32 / lpn);
    const dim3 grid(ceil_div(n, nodes_per_block), slabs);
#define GFM_BWD_LAUNCH_U(NV_, LPN_, U8_, GC_, U_)                                            \
  launch_k(k_agg_bwd_vec<NV_, LPN_, U8_, GC_, U_>, grid, 256, 0, s, (const float*)G, ldg,      \
           (const float*)coef, (const float*)dmax, ld, am, (const float*)h_in, csc_ptr,        \
           csc_eid, csc_dst, (const float*)w, n, H, (float*)dh, (const float*)gate,            \
           (float*)out, w_csc)
#define GFM_BWD_LAUNCH(NV_, LPN_, U8_, GC_)                                                  \
  do {                                                                                       \
    if (deep) {                                                                              \
      if constexpr (LPN_ == 32)                                                              \
        GFM_BWD_LAUNCH_U(NV_, LPN_, U8_, GC_, GFM_AGG_BWD_U_DEEP32);                         \
      else                                                                                   \
        GFM_BWD_LAUNCH_U(NV_, LPN_, U8_, GC_, GFM_AGG_BWD_U_DEEP);                           \
      break;                                                                                 \
    }                                                                                        \
    if constexpr (LPN_ == 32 && GFM_AGG_BWD_U_MAXSCAT > 1) {                                  \
      if (!local) {                                                                          \
        GFM_BWD_LAUNCH_U(NV_, LPN_, U8_, GC_, GFM_AGG_BWD_U_MAXSCAT);                        \
        break;                                                                               \
      }                                                                                      \
    }                                                                                        \
    GFM_BWD_LAUNCH_U(NV_, LPN_, U8_, GC_, GFM_AGG_BWD_U);                                    \
  } while (0)
#define GFM_BWD_CASE(NV_, LPN_)                                                              \
  if (nv == NV_ && lpn == LPN_) {                                                            \
    if (gc) {                                                                                \
      if (am_u8) GFM_BWD_LAUNCH(NV_, LPN_, true, true);                                      \
      else GFM_BWD_LAUNCH(NV_, LPN_, false, true);                                           \
    } else {                                                                                 \
      if (am_u8) GFM_BWD_LAUNCH(NV_, LPN_, true, false);                                     \
      else GFM_BWD_LAUNCH(NV_, LPN_, false, false);                                          \
    }                                                                                        \
    return cudaGetLastError();                                                               \
  }
    GFM_VEC_CASES(GFM_BWD_CASE)
#undef GFM_BWD_CASE
#undef GFM_BWD_LAUNCH
#undef GFM_BWD_LAUNCH_U
  }
  if (dtype == GFM_F32)
    launch_k(k_agg_bwd_scalar<float>, grid_1d((long long)n * H), 256, 0, s,
        (const float*)G, ldg, (const float*)coef, (const float*)dmax, ld, am, (const float*)h_in,
        csc_ptr, csc_eid, csc_dst, (const float*)w, n, H, (float*)dh, (const float*)gate,
        (float*)out, am_u8, w_csc);
  else
    launch_k(k_agg_bwd_scalar<double>, grid_1d((long long)n * H), 256, 0, s,
        (const double*)G, ldg, (const double*)coef, (const double*)dmax, ld, am,
        (const double*)h_in, csc_ptr, csc_eid, csc_dst, (const double*)w, n, H, (double*)dh,
        (const double*)gate, (double*)out, am_u8, w_csc);
  return cudaGetLastError();
}

}  // namespace gfm

using namespace gfm;

extern "C" {

int gfm_agg_parts_count(int parts) { return agg_layout(parts, 1).K; }

size_t gfm_agg_bwd_workspace_bytes(int n_nodes, int H, int parts, int dtype) {
  const size_t esz = dtype == GFM_F32 ? 4 : 8;
  return esz * (size_t)n_nodes * H * 2 + 256;
}

int gfm_embed(const int* z, int n, const void* emb, int H, void* h, int dtype, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GFM_F32)
  {
    if (H % 4 == 0 && ((uintptr_t)emb & 15) == 0 && ((uintptr_t)h & 15) == 0) {
      const int tx = std::min(32, H / 4), ty = 256 / tx;
      launch_k(k_embed4, dim3(1, std::min(ceil_div(n, ty), 65535)), dim3(tx, ty), 0, s,
          z, n, (const float4*)emb, H / 4, (float4*)h);
    } else {
      launch_k(k_embed<float>, dim3(1, std::min(ceil_div(n, 8), 65535)), dim3(32, 8), 0, s,
          z, n, (const float*)emb, H, (float*)h);
    }
  }
  else if (dtype == GFM_F64)
    launch_k(k_embed<double>, dim3(1, std::min(ceil_div(n, 8), 65535)), dim3(32, 8), 0, s,
        z, n, (const double*)emb, H, (double*)h);
  else {
    set_error("gfm_embed: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_embed: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_agg_fwd(const void* h, int n_nodes, int H, const int* rowptr, const int* col_src,
                const void* edge_w, int parts, void* agg, int* argmax, void* stat_mean, int dtype,
                int flags, void* stream) {
  if ((dtype != GFM_F32 && dtype != GFM_F64) || parts <= 0 || parts > 15 || H <= 0) {
    set_error("gfm_agg_fwd: bad arguments (dtype %d parts %d H %d)", dtype, parts, H);
    return GFM_EINVAL;
  }
  cudaError_t e = agg_fwd(dtype, h, n_nodes, H, rowptr, col_src, edge_w, parts, agg, argmax,
                          stat_mean, flags & GFM_FLAG_SCALAR,
                          (flags & GFM_FLAG_ARGMAX_U8) != 0, (cudaStream_t)stream);
  if (e != cudaSuccess) set_error("gfm_agg_fwd: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_agg_bwd(const void* dagg, const void* agg, const void* stat_mean, const int* argmax,
                const void* h_in, const int* rowptr, const int* csc_ptr, const int* csc_eid,
                const int* csc_dst, const void* edge_w, int n_nodes, int H, int parts, void* dh,
                const void* gate, void* out, void* workspace, int dtype, int flags, void* stream) {
  if ((dtype != GFM_F32 && dtype != GFM_F64) || parts <= 0 || parts > 15 || H <= 0) {
    set_error("gfm_agg_bwd: bad arguments (dtype %d parts %d H %d)", dtype, parts, H);
    return GFM_EINVAL;
  }
  cudaError_t e = agg_bwd(dtype, dagg, agg, stat_mean, argmax, h_in, rowptr, csc_ptr, csc_eid,
                          csc_dst, edge_w, n_nodes, H, parts, dh, gate, out, workspace,
                          flags & GFM_FLAG_SCALAR, (flags & GFM_FLAG_ARGMAX_U8) != 0,
                          (cudaStream_t)stream, (flags & GFM_FLAG_AGG_PREPPED) != 0,
                          (flags & GFM_FLAG_W_CSC) != 0, (flags & GFM_FLAG_GATHER_LOCAL) != 0);
  if (e != cudaSuccess) set_error("gfm_agg_bwd: %s", cudaGetErrorString(e));
  return (int)e;
}

}  // extern "C"
