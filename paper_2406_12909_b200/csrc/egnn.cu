// EGNN-style variant (BASELINE configs[3], "C4"): E(n)-equivariant message
// passing with coordinate updates and autograd forces F = -dE/dx0.
//
// No reference implementation exists; the
// restated algorithm is oracle/egnn_oracle.py (pinned there by finite
// differences and torch double backward).  Per layer, for an edge e = j -> i
// (CSR row i, dst-sorted like make_batch, model.py:260-266):
//   r = x_j - x_i, d2 = r.r, m = tanh(A_i + B_j + wd d2 + c), s = m.ux
//   agg_i = sum_e m,  x'_i = x_i - (1/max(deg_i,1)) sum_e r s
// with A | B = h [wa; wb]^T one node GEMM; h' = tanh(h w^T + agg u^T + b)
// is a node GEMM + the dual tanh below.
//
// Training differentiates a loss holding F, i.e. second derivatives.  It is
// done as reverse-over-forward: a tangent forward from xdot0 = dL/dF, then
// ONE reverse pass over primal + tangent with seeds (dL/dE, -1).  Linear ops
// (every GEMM) act on primal and tangent rows alike, so the host stacks them
// as [p; pdot] (2N rows) and uses the tensor-core GEMM engine unchanged;
// these kernels are the elementwise / edge parts that mix the two:
//
//   k_egnn_edge_fwd      per dst row (warp): recompute-free edge MLP, sums
//                        agg (and its tangent) and the coordinate update
//   k_egnn_edge_bwd      per dst row: the edge adjoints; dst-side sums (dA,
//                        x) in CSR order, per-edge dpre / dr written for ...
//   k_egnn_edge_bwd_src  per src node: ... the CSC gather (dB, x), so every
//                        sum has a fixed order (no atomics: deterministic)
//   k_egnn_tanh_fwd/bwd  h = tanh(z + b), hdot = (1 - h^2) zdot and adjoints
//   k_egnn_head_out      node energies (and tangents) + per-graph pool
//   k_egnn_head_seed     dL/d node energy (primal de[g], tangent -1) rows
//   k_colsum_part/final  deterministic two-level column sums (bias / vector grads)
#include <cstdio>

#include "common.cuh"

namespace gfm {

// lanes own channels lane, lane + 32, ...: CPL = H / 32 per lane
template <typename T, int CPL, bool DUAL>
__global__ void __launch_bounds__(256)
    k_egnn_edge_fwd(const T* __restrict__ AB, int ldab, const T* __restrict__ ABd,
                    const T* __restrict__ x, const T* __restrict__ xd, int n,
                    const int* __restrict__ rowptr, const int* __restrict__ col_src,
                    const T* __restrict__ wd, const T* __restrict__ c, const T* __restrict__ ux,
                    int coord, T* __restrict__ agg, int ldg, T* __restrict__ aggd,
                    T* __restrict__ xo, T* __restrict__ xdo) {
  pdl_entry();
  constexpr int H = 32 * CPL;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    T a[CPL], w[CPL], cc[CPL], u[CPL], acc[CPL], ad[CPL], accd[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int ch = lane + 32 * k;
      a[k] = AB[(long long)i * ldab + ch];
      w[k] = wd[ch];
      cc[k] = c[ch];
      u[k] = ux[ch];
      acc[k] = T(0);
      accd[k] = T(0);
      ad[k] = DUAL ? ABd[(long long)i * ldab + ch] : T(0);
    }
    const T xi0 = x[3 * i], xi1 = x[3 * i + 1], xi2 = x[3 * i + 2];
    T xdi0 = 0, xdi1 = 0, xdi2 = 0;
    if (DUAL) {
      xdi0 = xd[3 * i];
      xdi1 = xd[3 * i + 1];
      xdi2 = xd[3 * i + 2];
    }
    T up0 = 0, up1 = 0, up2 = 0, ud0 = 0, ud1 = 0, ud2 = 0;
    const int e0 = rowptr[i], e1 = rowptr[i + 1];
    for (int e = e0; e < e1; ++e) {
      const int j = col_src[e];
      const T r0 = x[3 * j] - xi0, r1 = x[3 * j + 1] - xi1, r2 = x[3 * j + 2] - xi2;
      const T d2 = r0 * r0 + r1 * r1 + r2 * r2;
      T rd0 = 0, rd1 = 0, rd2 = 0, d2d = 0;
      if (DUAL) {
        rd0 = xd[3 * j] - xdi0;
        rd1 = xd[3 * j + 1] - xdi1;
        rd2 = xd[3 * j + 2] - xdi2;
        d2d = T(2) * (r0 * rd0 + r1 * rd1 + r2 * rd2);
      }
      T sp = 0, sdp = 0;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int ch = lane + 32 * k;
        const T m = tanh_t(a[k] + AB[(long long)j * ldab + H + ch] + w[k] * d2 + cc[k]);
        acc[k] += m;
        sp += m * u[k];
        if (DUAL) {
          const T pd = ad[k] + ABd[(long long)j * ldab + H + ch] + w[k] * d2d;
          const T md = (T(1) - m * m) * pd;
          accd[k] += md;
          sdp += md * u[k];
        }
      }
      if (coord) {
        // r (and rdot) are uniform over the warp: accumulate this lane's
        // share of sum_e r_e s_e and reduce once per node, not per edge
        up0 += r0 * sp;
        up1 += r1 * sp;
        up2 += r2 * sp;
        if (DUAL) {
          ud0 += rd0 * sp + r0 * sdp;
          ud1 += rd1 * sp + r1 * sdp;
          ud2 += rd2 * sp + r2 * sdp;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int ch = lane + 32 * k;
      if (agg) agg[(long long)i * ldg + ch] = acc[k];
      if (DUAL) aggd[(long long)i * ldg + ch] = accd[k];
    }
    if (coord) {
      up0 = warp_sum(up0);
      up1 = warp_sum(up1);
      up2 = warp_sum(up2);
      if (DUAL) {
        ud0 = warp_sum(ud0);
        ud1 = warp_sum(ud1);
        ud2 = warp_sum(ud2);
      }
    }
    if (coord && lane == 0) {
      const T ci = T(1) / T(e1 - e0 > 1 ? e1 - e0 : 1);
      if (xo) {
        xo[3 * i] = xi0 - ci * up0;
        xo[3 * i + 1] = xi1 - ci * up1;
        xo[3 * i + 2] = xi2 - ci * up2;
      }
      if (DUAL) {
        xdo[3 * i] = xdi0 - ci * ud0;
        xdo[3 * i + 1] = xdi1 - ci * ud1;
        xdo[3 * i + 2] = xdi2 - ci * ud2;
      }
    }
  }
}

// Several warp sums at once by recursive halving: 2 sums with 7 shuffles, 4
// with 10 (instead of 10 / 20 butterflies); every lane gets every sum.
template <typename T>
__device__ __forceinline__ void warp_sum2(T& a, T& b) {
  const int lane = threadIdx.x & 31;
  const bool up = lane & 16;
  T k = up ? b : a;
  k += __shfl_xor_sync(0xffffffffu, up ? a : b, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  a = __shfl_sync(0xffffffffu, k, 0);
  b = __shfl_sync(0xffffffffu, k, 16);
}
template <typename T>
__device__ __forceinline__ void warp_sum4(T& a, T& b, T& c, T& d) {
  const int lane = threadIdx.x & 31;
  bool up = lane & 16;  // lanes 0-15 keep (a, b), 16-31 keep (c, d)
  T k0 = up ? c : a, k1 = up ? d : b;
  k0 += __shfl_xor_sync(0xffffffffu, up ? a : c, 16);
  k1 += __shfl_xor_sync(0xffffffffu, up ? b : d, 16);
  up = lane & 8;  // then the first or second of the pair
  T k = up ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, up ? k0 : k1, 8);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  a = __shfl_sync(0xffffffffu, k, 0);
  b = __shfl_sync(0xffffffffu, k, 8);
  c = __shfl_sync(0xffffffffu, k, 16);
  d = __shfl_sync(0xffffffffu, k, 24);
}

// Edge adjoints, one warp per dst row i.  Inputs: aggb / aggdb = dL/d agg of
// the layer (and of its tangent), xbo / xdbo = dL/d x' (layer output
// coordinates; only read when coord).  Outputs: Ab / Adb (dst part of the
// A | B adjoint, columns of the caller's [dz | dA | dB] buffer), per-edge
// preb / predb (E x H) and rb / rdb (E x 3) for the src gather, xbi / xdbi =
// dL/dx of the layer input minus its src part (added by the gather), and
// per-node parameter partials part = [d wd | d ux] (n x 2H).
// min blocks per SM of the dst-side edge backward: 3 (85 registers, no
// spills) instead of 1 (90 registers, 20% warps active): C4 step -1.9%
#ifndef GFM_EGNN_BWD_MINB
#define GFM_EGNN_BWD_MINB 3
#endif
template <typename T, int CPL, bool DUAL>
__global__ void __launch_bounds__(256, GFM_EGNN_BWD_MINB)
    k_egnn_edge_bwd(const T* __restrict__ AB, int ldab, const T* __restrict__ ABd,
                    const T* __restrict__ x, const T* __restrict__ xd, int n,
                    const int* __restrict__ rowptr, const int* __restrict__ col_src,
                    const T* __restrict__ wd, const T* __restrict__ c, const T* __restrict__ ux,
                    int coord, const T* __restrict__ aggb, int ldgb, const T* __restrict__ aggdb,
                    const T* __restrict__ xbo, const T* __restrict__ xdbo, T* __restrict__ Ab,
                    int lda, T* __restrict__ Adb, T* __restrict__ preb, T* __restrict__ predb,
                    T* __restrict__ rb, T* __restrict__ rdb, T* __restrict__ xbi,
                    T* __restrict__ xdbi, T* __restrict__ part) {
  pdl_entry();
  constexpr int H = 32 * CPL;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    T a[CPL], ad[CPL], w[CPL], cc[CPL], u[CPL], gb[CPL], gdb[CPL];
    T sA[CPL], sAd[CPL], pw[CPL], pu[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int ch = lane + 32 * k;
      a[k] = AB[(long long)i * ldab + ch];
      ad[k] = DUAL ? ABd[(long long)i * ldab + ch] : T(0);
      w[k] = wd[ch];
      cc[k] = c[ch];
      u[k] = ux[ch];
      gb[k] = aggb[(long long)i * ldgb + ch];
      gdb[k] = DUAL ? aggdb[(long long)i * ldgb + ch] : T(0);
      sA[k] = sAd[k] = pw[k] = pu[k] = T(0);
    }
    const T xi0 = x[3 * i], xi1 = x[3 * i + 1], xi2 = x[3 * i + 2];
    T xdi0 = 0, xdi1 = 0, xdi2 = 0;
    if (DUAL) {
      xdi0 = xd[3 * i];
      xdi1 = xd[3 * i + 1];
      xdi2 = xd[3 * i + 2];
    }
    const int e0 = rowptr[i], e1 = rowptr[i + 1];
    const T ci = T(1) / T(e1 - e0 > 1 ? e1 - e0 : 1);
    T xb0 = 0, xb1 = 0, xb2 = 0, xdb0 = 0, xdb1 = 0, xdb2 = 0;  // dL/dx', dL/dxdot' at i
    if (coord) {
      xb0 = xbo[3 * i];
      xb1 = xbo[3 * i + 1];
      xb2 = xbo[3 * i + 2];
      if (DUAL) {
        xdb0 = xdbo[3 * i];
        xdb1 = xdbo[3 * i + 1];
        xdb2 = xdbo[3 * i + 2];
      }
    }
    // dL/dx of the layer input: identity part, minus the dst side of every r
    T oi0 = xb0, oi1 = xb1, oi2 = xb2, odi0 = xdb0, odi1 = xdb1, odi2 = xdb2;
    for (int e = e0; e < e1; ++e) {
      const int j = col_src[e];
      const T r0 = x[3 * j] - xi0, r1 = x[3 * j + 1] - xi1, r2 = x[3 * j + 2] - xi2;
      const T d2 = r0 * r0 + r1 * r1 + r2 * r2;
      T rd0 = 0, rd1 = 0, rd2 = 0, d2d = 0;
      if (DUAL) {
        rd0 = xd[3 * j] - xdi0;
        rd1 = xd[3 * j + 1] - xdi1;
        rd2 = xd[3 * j + 2] - xdi2;
        d2d = T(2) * (r0 * rd0 + r1 * rd1 + r2 * rd2);
      }
      T m[CPL], md[CPL], pd[CPL];
      T sp = 0, sdp = 0;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int ch = lane + 32 * k;
        m[k] = tanh_t(a[k] + AB[(long long)j * ldab + H + ch] + w[k] * d2 + cc[k]);
        sp += m[k] * u[k];
        if (DUAL) {
          pd[k] = ad[k] + ABd[(long long)j * ldab + H + ch] + w[k] * d2d;
          md[k] = (T(1) - m[k] * m[k]) * pd[k];
          sdp += md[k] * u[k];
        }
      }
      // coordinate update adjoints: x' = x - ci sum r s, xdot' = xdot - ci sum (rdot s + r sdot)
      // (sb / sdb are warp-uniform; the four warp sums s, sdot, d2b, d2db
      // are reduced together after the channel loop)
      T sb = 0, sdb = 0, rb0 = 0, rb1 = 0, rb2 = 0, rdb0 = 0, rdb1 = 0, rdb2 = 0;
      if (coord) {
        sb = -ci * (r0 * xb0 + r1 * xb1 + r2 * xb2);
        if (DUAL) {
          sb += -ci * (rd0 * xdb0 + rd1 * xdb1 + rd2 * xdb2);
          sdb = -ci * (r0 * xdb0 + r1 * xdb1 + r2 * xdb2);
        }
      }
      T d2bp = 0, d2dbp = 0;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int ch = lane + 32 * k;
        T mb = gb[k] + sb * u[k];
        pu[k] += sb * m[k];
        const T g = T(1) - m[k] * m[k];
        if (DUAL) {
          const T mdb = gdb[k] + sdb * u[k];
          pu[k] += sdb * md[k];
          const T pdb = g * mdb;  // d predot
          mb -= T(2) * m[k] * pd[k] * mdb;
          sAd[k] += pdb;
          pw[k] += pdb * d2d;
          d2dbp += pdb * w[k];
          predb[(long long)e * H + ch] = pdb;
        }
        const T pb = g * mb;  // d pre
        sA[k] += pb;
        pw[k] += pb * d2;
        d2bp += pb * w[k];
        preb[(long long)e * H + ch] = pb;
      }
      T s = sp, sd = sdp, d2b = d2bp, d2db = d2dbp;
      if (DUAL && coord) {
        warp_sum4(s, sd, d2b, d2db);
      } else if (DUAL) {
        warp_sum2(d2b, d2db);
      } else if (coord) {
        warp_sum2(s, d2b);
      } else {
        d2b = warp_sum(d2b);
      }
      if (coord) {
        rb0 = -ci * s * xb0;
        rb1 = -ci * s * xb1;
        rb2 = -ci * s * xb2;
        if (DUAL) {
          rb0 += -ci * sd * xdb0;
          rb1 += -ci * sd * xdb1;
          rb2 += -ci * sd * xdb2;
          rdb0 = -ci * s * xdb0;
          rdb1 = -ci * s * xdb1;
          rdb2 = -ci * s * xdb2;
        }
      }
      rb0 += T(2) * r0 * d2b;
      rb1 += T(2) * r1 * d2b;
      rb2 += T(2) * r2 * d2b;
      if (DUAL) {
        rb0 += T(2) * rd0 * d2db;
        rb1 += T(2) * rd1 * d2db;
        rb2 += T(2) * rd2 * d2db;
        rdb0 += T(2) * r0 * d2db;
        rdb1 += T(2) * r1 * d2db;
        rdb2 += T(2) * r2 * d2db;
      }
      if (lane == 0) {
        rb[3LL * e] = rb0;
        rb[3LL * e + 1] = rb1;
        rb[3LL * e + 2] = rb2;
        if (DUAL) {
          rdb[3LL * e] = rdb0;
          rdb[3LL * e + 1] = rdb1;
          rdb[3LL * e + 2] = rdb2;
        }
      }
      oi0 -= rb0;
      oi1 -= rb1;
      oi2 -= rb2;
      odi0 -= rdb0;
      odi1 -= rdb1;
      odi2 -= rdb2;
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int ch = lane + 32 * k;
      Ab[(long long)i * lda + ch] = sA[k];
      if (DUAL) Adb[(long long)i * lda + ch] = sAd[k];
      part[(long long)i * 2 * H + ch] = pw[k];
      part[(long long)i * 2 * H + H + ch] = pu[k];
    }
    if (lane == 0) {
      xbi[3 * i] = oi0;
      xbi[3 * i + 1] = oi1;
      xbi[3 * i + 2] = oi2;
      if (DUAL) {
        xdbi[3 * i] = odi0;
        xdbi[3 * i + 1] = odi1;
        xdbi[3 * i + 2] = odi2;
      }
    }
  }
}

// src side, one warp per node j over its CSC edges (ascending dst): dB_j and
// the src part of dL/dx (added to what k_egnn_edge_bwd wrote)
template <typename T, int CPL, bool DUAL>
__global__ void __launch_bounds__(256)
    k_egnn_edge_bwd_src(int n, const int* __restrict__ csc_ptr, const int* __restrict__ csc_eid,
                        const T* __restrict__ preb, const T* __restrict__ predb,
                        const T* __restrict__ rb, const T* __restrict__ rdb, T* __restrict__ Bb,
                        int ldb, T* __restrict__ Bdb, T* __restrict__ xbi, T* __restrict__ xdbi) {
  pdl_entry();
  constexpr int H = 32 * CPL;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
    T sB[CPL], sBd[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) sB[k] = sBd[k] = T(0);
    T o0 = 0, o1 = 0, o2 = 0, od0 = 0, od1 = 0, od2 = 0;
    for (int q = csc_ptr[j]; q < csc_ptr[j + 1]; ++q) {
      const long long e = csc_eid[q];
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        sB[k] += preb[e * H + lane + 32 * k];
        if (DUAL) sBd[k] += predb[e * H + lane + 32 * k];
      }
      o0 += rb[3 * e];
      o1 += rb[3 * e + 1];
      o2 += rb[3 * e + 2];
      if (DUAL) {
        od0 += rdb[3 * e];
        od1 += rdb[3 * e + 1];
        od2 += rdb[3 * e + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      Bb[(long long)j * ldb + lane + 32 * k] = sB[k];
      if (DUAL) Bdb[(long long)j * ldb + lane + 32 * k] = sBd[k];
    }
    if (lane == 0) {
      xbi[3 * j] += o0;
      xbi[3 * j + 1] += o1;
      xbi[3 * j + 2] += o2;
      if (DUAL) {
        xdbi[3 * j] += od0;
        xdbi[3 * j + 1] += od1;
        xdbi[3 * j + 2] += od2;
      }
    }
  }
}

// h = tanh(z + b) on the primal rows; hdot = (1 - h^2) zdot on the tangent
// rows (zd / hd may be null: primal only; z null: tangent only, from h)
template <typename T>
__global__ void k_egnn_tanh_fwd(const T* __restrict__ z, const T* __restrict__ zd, int ldz,
                                const T* __restrict__ b, int n, int H, T* __restrict__ h,
                                T* __restrict__ hd, int ldh) {
  pdl_entry();
  const long long total = (long long)n * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / H;
    const int k = (int)(t - i * H);
    // z == null: h already holds the primal output; only the tangent is new
    const T hv = z ? tanh_t(z[i * ldz + k] + (b ? b[k] : T(0))) : h[i * ldh + k];
    if (z) h[i * ldh + k] = hv;
    if (hd) hd[i * ldh + k] = (T(1) - hv * hv) * zd[i * ldz + k];
  }
}

// adjoints of h = tanh(z), hdot = (1 - h^2) zdot:
//   zb = (1 - h^2)(hb - 2 h zdot hdb),  zdb = (1 - h^2) hdb
template <typename T>
__global__ void k_egnn_tanh_bwd(const T* __restrict__ h, int ldh, const T* __restrict__ zd,
                                int ldzd, const T* __restrict__ hb, const T* __restrict__ hdb,
                                int ldhb, int n, int H, T* __restrict__ zb, T* __restrict__ zdb,
                                int ldzb) {
  pdl_entry();
  const long long total = (long long)n * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / H;
    const int k = (int)(t - i * H);
    const T hv = h[i * ldh + k];
    const T g = T(1) - hv * hv;
    T v = hb[i * ldhb + k];
    if (hdb) {
      const T hd = hdb[i * ldhb + k];
      v -= T(2) * hv * zd[i * ldzd + k] * hd;
      zdb[i * ldzb + k] = g * hd;
    }
    zb[i * ldzb + k] = g * v;
  }
}

// node energy = y . a + c (and tangent ydot . a), warp per node; then one
// warp per graph sums its nodes (lanes strided, fixed-order warp sum)
template <typename T>
__global__ void k_egnn_node_energy(const T* __restrict__ y, const T* __restrict__ yd, int ldy,
                                   int n, int G, const T* __restrict__ a, const T* __restrict__ c,
                                   T* __restrict__ ne, T* __restrict__ ned) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    T s = 0, sd = 0;
    for (int g = lane; g < G; g += 32) {
      s += y[(long long)i * ldy + g] * a[g];
      if (yd) sd += yd[(long long)i * ldy + g] * a[g];
    }
    s = warp_sum(s);
    if (yd) sd = warp_sum(sd);
    if (lane == 0) {
      ne[i] = s + c[0];
      if (yd) ned[i] = sd;
    }
  }
}

template <typename T>
__global__ void k_egnn_pool(const T* __restrict__ ne, const T* __restrict__ ned,
                            const int* __restrict__ off, int B, T* __restrict__ e,
                            T* __restrict__ ed) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += warps) {
    T s = 0, sd = 0;
    for (int i = off[b] + lane; i < off[b + 1]; i += 32) {
      s += ne[i];
      if (ned) sd += ned[i];
    }
    s = warp_sum(s);
    if (ned) sd = warp_sum(sd);
    if (lane == 0) {
      e[b] = s;
      if (ned) ed[b] = sd;
    }
  }
}

// head seeds: rows 0..n-1 (primal) get s_i = de[g(i)] (0 for capacity-tail
// nodes, gnode < 0), rows n..2n-1 (tangent, when edot_seed != 0) get
// edot_seed for every node of a graph.  ds = [s 0 0 0] per row (16-byte rows
// for the weight-gradient GEMM), yb = s a.
template <typename T>
__global__ void k_egnn_head_seed(const T* __restrict__ de, const int* __restrict__ gnode, int n,
                                 int rows, T edot_seed, const T* __restrict__ a, int G,
                                 T* __restrict__ ds, T* __restrict__ yb, int ldyb) {
  pdl_entry();
  const int W = G > 4 ? G : 4;
  const long long total = (long long)rows * W;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / W;
    const int g = (int)(t - r * W);
    const int i = (int)(r < n ? r : r - n);
    const int gi = gnode[i];
    const T s = gi < 0 ? T(0) : (r < n ? de[gi] : edot_seed);
    if (g < G) yb[r * ldyb + g] = s * a[g];
    if (g < 4) ds[r * 4 + g] = g == 0 ? s : T(0);
  }
}

// deterministic column sums of rows [0, rows) of X (ld), two levels in ONE
// launch: block (chunk c, slab s) sums rows [c*kColRows, +kColRows) of 32
// columns (8 row groups, fixed-order combine, double) into part[c][cols];
// the slab's last block to finish (a ticket per slab) sums the chunk
// partials in chunk order and resets the ticket.  The result depends only
// on the shape.
constexpr int kColRows = 64;  // 8 rows per thread: many blocks in flight (latency bound)
template <typename T>
__global__ void k_colsum(const T* __restrict__ X, int rows, int cols, int ld,
                         double* __restrict__ part, unsigned* __restrict__ ticket,
                         T* __restrict__ out, int accumulate) {
  pdl_entry();
  __shared__ double red[8][33];
  __shared__ bool last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.y * 32 + tx;
  const int r0 = blockIdx.x * kColRows, r1 = min(rows, r0 + kColRows);
  double s = 0.0;
  if (c < cols) {
#pragma unroll 4
    for (int r = r0 + ty; r < r1; r += 8) s += (double)X[(long long)r * ld + c];
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && c < cols) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += red[q][tx];
    part[(long long)blockIdx.x * cols + c] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    last = atomicAdd(&ticket[blockIdx.y], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // row group ty sums chunks ty, ty + 8, ... in order; the 8 group sums are
  // combined in group order (fixed for a shape)
  double t = 0.0;
  if (c < cols)
    for (int k = ty; k < (int)gridDim.x; k += 8) t += __ldcg(part + (long long)k * cols + c);
  red[ty][tx] = t;
  __syncthreads();
  if (ty == 0 && c < cols) {
    double u = 0.0;
    for (int q = 0; q < 8; ++q) u += red[q][tx];
    out[c] = accumulate ? (T)((double)out[c] + u) : (T)u;
  }
  if (threadIdx.x == 0) ticket[blockIdx.y] = 0u;  // ready for the next call
}

template <typename T>
__global__ void k_scale(const T* __restrict__ x, long long n, T alpha, T* __restrict__ y) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = alpha * x[i];
}

static inline int grid_warps(long long warps) {
  long long b = (warps * 32 + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}
static inline int grid_elems(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

#define GFM_EGNN_CPL(H_, BODY)                     \
  switch ((H_) / 32) {                             \
    case 1: { constexpr int CPL = 1; BODY; } break; \
    case 2: { constexpr int CPL = 2; BODY; } break; \
    case 4: { constexpr int CPL = 4; BODY; } break; \
    case 8: { constexpr int CPL = 8; BODY; } break; \
    case 16: { constexpr int CPL = 16; BODY; } break; \
    default: return cudaErrorInvalidValue;          \
  }

template <typename T>
cudaError_t egnn_edge_fwd_t(const T* AB, int ldab, const T* ABd, const T* x, const T* xd, int n,
                            int H, const int* rowptr, const int* col_src, const T* wd, const T* c,
                            const T* ux, int coord, T* agg, int ldg, T* aggd, T* xo, T* xdo,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = grid_warps(n);
  GFM_EGNN_CPL(H, (ABd ? launch_k(k_egnn_edge_fwd<T, CPL, true>, grid, 256, 0, s, AB, ldab, ABd, x,
                                  xd, n, rowptr, col_src, wd, c, ux, coord, agg, ldg, aggd, xo,
                                  xdo)
                       : launch_k(k_egnn_edge_fwd<T, CPL, false>, grid, 256, 0, s, AB, ldab, ABd,
                                  x, xd, n, rowptr, col_src, wd, c, ux, coord, agg, ldg, aggd, xo,
                                  xdo)))
  return cudaGetLastError();
}

template <typename T>
cudaError_t egnn_edge_bwd_t(const T* AB, int ldab, const T* ABd, const T* x, const T* xd, int n,
                            int H, const int* rowptr, const int* col_src, const int* csc_ptr,
                            const int* csc_eid, const T* wd, const T* c, const T* ux, int coord,
                            const T* aggb, int ldgb, const T* aggdb, const T* xbo, const T* xdbo,
                            T* dAB, int ldd, T* dABd, T* preb, T* predb, T* rb, T* rdb, T* xbi,
                            T* xdbi, T* part, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = grid_warps(n);
  const bool dual = ABd != nullptr;
  GFM_EGNN_CPL(H, (dual ? launch_k(k_egnn_edge_bwd<T, CPL, true>, grid, 256, 0, s, AB, ldab, ABd,
                                   x, xd, n, rowptr, col_src, wd, c, ux, coord, aggb, ldgb, aggdb,
                                   xbo, xdbo, dAB, ldd, dABd, preb, predb, rb, rdb, xbi, xdbi,
                                   part)
                        : launch_k(k_egnn_edge_bwd<T, CPL, false>, grid, 256, 0, s, AB, ldab,
                                   ABd, x, xd, n, rowptr, col_src, wd, c, ux, coord, aggb, ldgb,
                                   aggdb, xbo, xdbo, dAB, ldd, dABd, preb, predb, rb, rdb, xbi,
                                   xdbi, part)))
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  GFM_EGNN_CPL(H, (dual ? launch_k(k_egnn_edge_bwd_src<T, CPL, true>, grid, 256, 0, s, n, csc_ptr,
                                   csc_eid, preb, predb, rb, rdb, dAB + H, ldd,
                                   dABd ? dABd + H : nullptr, xbi, xdbi)
                        : launch_k(k_egnn_edge_bwd_src<T, CPL, false>, grid, 256, 0, s, n,
                                   csc_ptr, csc_eid, preb, predb, rb, rdb, dAB + H, ldd,
                                   (T*)nullptr, xbi, xdbi)))
  return cudaGetLastError();
}

}  // namespace gfm

using namespace gfm;

#define GFM_EDISPATCH(dtype, NAME, ...)                                    \
  cudaError_t _err;                                                        \
  if (dtype == GFM_F32) {                                                  \
    using T = float;                                                       \
    _err = __VA_ARGS__;                                                    \
  } else if (dtype == GFM_F64) {                                           \
    using T = double;                                                      \
    _err = __VA_ARGS__;                                                    \
  } else {                                                                 \
    set_error("%s: bad dtype %d", NAME, dtype);                            \
    return GFM_EINVAL;                                                     \
  }                                                                        \
  if (_err != cudaSuccess) {                                               \
    set_error("%s: %s", NAME, cudaGetErrorString(_err));                   \
    return (int)_err;                                                      \
  }                                                                        \
  return 0;

extern "C" {

int gfm_egnn_edge_fwd(const void* AB, int ldab, const void* ABd, const void* x, const void* xd,
                      int n_nodes, int H, const int* rowptr, const int* col_src, const void* wd,
                      const void* c, const void* ux, int coord_update, void* agg, int ldg,
                      void* aggd, void* x_out, void* xd_out, int dtype, void* stream) {
  if (H % 32 != 0 || H > 512 || (H / 32) & (H / 32 - 1)) {
    set_error("gfm_egnn_edge_fwd: H must be 32, 64, 128, 256 or 512 (got %d)", H);
    return GFM_EINVAL;
  }
  GFM_EDISPATCH(dtype, "gfm_egnn_edge_fwd",
                egnn_edge_fwd_t<T>((const T*)AB, ldab, (const T*)ABd, (const T*)x, (const T*)xd,
                                   n_nodes, H, rowptr, col_src, (const T*)wd, (const T*)c,
                                   (const T*)ux, coord_update, (T*)agg, ldg, (T*)aggd, (T*)x_out,
                                   (T*)xd_out, (cudaStream_t)stream))
}

int gfm_egnn_edge_bwd(const void* AB, int ldab, const void* ABd, const void* x, const void* xd,
                      int n_nodes, int H, const int* rowptr, const int* col_src,
                      const int* csc_ptr, const int* csc_eid, const void* wd, const void* c,
                      const void* ux, int coord_update, const void* aggb, int ldgb,
                      const void* aggdb, const void* xb_out, const void* xdb_out, void* dAB,
                      int ldd, void* dABd, void* preb, void* predb, void* rb, void* rdb,
                      void* xb_in, void* xdb_in, void* part, int dtype, void* stream) {
  if (H % 32 != 0 || H > 512 || (H / 32) & (H / 32 - 1)) {
    set_error("gfm_egnn_edge_bwd: H must be 32, 64, 128, 256 or 512 (got %d)", H);
    return GFM_EINVAL;
  }
  GFM_EDISPATCH(dtype, "gfm_egnn_edge_bwd",
                egnn_edge_bwd_t<T>((const T*)AB, ldab, (const T*)ABd, (const T*)x, (const T*)xd,
                                   n_nodes, H, rowptr, col_src, csc_ptr, csc_eid, (const T*)wd,
                                   (const T*)c, (const T*)ux, coord_update, (const T*)aggb, ldgb,
                                   (const T*)aggdb, (const T*)xb_out, (const T*)xdb_out, (T*)dAB,
                                   ldd, (T*)dABd, (T*)preb, (T*)predb, (T*)rb, (T*)rdb,
                                   (T*)xb_in, (T*)xdb_in, (T*)part, (cudaStream_t)stream))
}

int gfm_egnn_tanh_fwd(const void* z, const void* zd, int ldz, const void* bias, int n, int H,
                      void* h, void* hd, int ldh, int dtype, void* stream) {
  GFM_EDISPATCH(dtype, "gfm_egnn_tanh_fwd",
                (n > 0 ? launch_k(k_egnn_tanh_fwd<T>, grid_elems((long long)n * H), 256, 0,
                                  (cudaStream_t)stream, (const T*)z, (const T*)zd, ldz,
                                  (const T*)bias, n, H, (T*)h, (T*)hd, ldh)
                       : cudaSuccess))
}

int gfm_egnn_tanh_bwd(const void* h, int ldh, const void* zd, int ldzd, const void* hb,
                      const void* hdb, int ldhb, int n, int H, void* zb, void* zdb, int ldzb,
                      int dtype, void* stream) {
  GFM_EDISPATCH(dtype, "gfm_egnn_tanh_bwd",
                (n > 0 ? launch_k(k_egnn_tanh_bwd<T>, grid_elems((long long)n * H), 256, 0,
                                  (cudaStream_t)stream, (const T*)h, ldh, (const T*)zd, ldzd,
                                  (const T*)hb, (const T*)hdb, ldhb, n, H, (T*)zb, (T*)zdb, ldzb)
                       : cudaSuccess))
}

int gfm_egnn_energy(const void* y, const void* yd, int ldy, int n, int G, const void* a,
                    const void* c, const int* node_offsets, int n_graphs, void* node_e,
                    void* node_ed, void* e_pred, void* e_dot, int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  GFM_EDISPATCH(dtype, "gfm_egnn_energy",
                (launch_k(k_egnn_node_energy<T>, grid_warps(n > 0 ? n : 1), 256, 0, s,
                          (const T*)y, (const T*)yd, ldy, n, G, (const T*)a, (const T*)c,
                          (T*)node_e, (T*)node_ed),
                 launch_k(k_egnn_pool<T>, grid_warps(n_graphs > 0 ? n_graphs : 1), 256, 0, s,
                          (const T*)node_e, (const T*)node_ed, node_offsets, n_graphs, (T*)e_pred,
                          (T*)e_dot)))
}

int gfm_egnn_head_seed(const void* de, const int* gnode, int n, int rows, double edot_seed,
                       const void* a, int G, void* ds, void* yb, int ldyb, int dtype,
                       void* stream) {
  GFM_EDISPATCH(dtype, "gfm_egnn_head_seed",
                launch_k(k_egnn_head_seed<T>, grid_elems((long long)rows * (G > 4 ? G : 4)), 256,
                         0, (cudaStream_t)stream, (const T*)de, gnode, n, rows, (T)edot_seed,
                         (const T*)a, G, (T*)ds, (T*)yb, ldyb))
}

size_t gfm_colsum_workspace_bytes(int rows, int cols) {
  const int chunks = rows > 0 ? (rows + kColRows - 1) / kColRows : 1;
  const size_t slabs = (size_t)((cols > 0 ? cols : 1) + 31) / 32;
  return sizeof(double) * (size_t)chunks * (size_t)(cols > 0 ? cols : 1) + 4 * slabs;
}

int gfm_colsum(const void* X, int rows, int cols, int ld, void* out, int accumulate,
               void* workspace, int dtype, void* stream) {
  if (cols <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int chunks = rows > 0 ? (rows + kColRows - 1) / kColRows : 1;
  double* part = (double*)workspace;
  unsigned* ticket = (unsigned*)(part + (size_t)chunks * cols);
  if (rows <= 0) {  // empty: out = 0 (or unchanged when accumulating)
    if (accumulate) return 0;
    GFM_EDISPATCH(dtype, "gfm_colsum", cudaMemsetAsync(out, 0, sizeof(T) * cols, s))
  } else {
    GFM_EDISPATCH(dtype, "gfm_colsum",
                  launch_k(k_colsum<T>, dim3(chunks, (cols + 31) / 32), 256, 0, s, (const T*)X,
                           rows, cols, ld, part, ticket, (T*)out, accumulate))
  }
  return 0;
}

int gfm_scale(const void* x, long long n, double alpha, void* y, int dtype, void* stream) {
  if (n <= 0) return 0;
  GFM_EDISPATCH(dtype, "gfm_scale",
                launch_k(k_scale<T>, grid_elems(n), 256, 0, (cudaStream_t)stream, (const T*)x, n,
                         (T)alpha, (T*)y))
}

}  // extern "C"
