// Batch geometry on device: radius graph -> dst-sorted CSR, stable CSR/CSC
// construction for arbitrary record edge lists, scans and per-graph maps.
//
// Reference: build_cutoff_edges (preprocess.py:90-104) and make_batch
// (model.py:234-285).  Layout produced for a batch of N nodes / E edges:
//   rowptr[N+1], col_src[E], edge_dst[E], edge_w[E], edge_dx[E][3]
//     -- CSR in (dst, src) order == the reference's stable dst sort
//   csc_ptr[N+1], csc_eid[E] (CSR position of each src-sorted edge),
//   csc_dst[E]   -- the stable src sort used by the backward gathers.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace gfm {

// ---------------------------------------------------------------- helpers
__global__ void k_graph_of_node(const int* __restrict__ off, int n_graphs, int* __restrict__ gnode) {
  pdl_entry();
  for (int g = blockIdx.x; g < n_graphs; g += gridDim.x)
    for (int i = off[g] + threadIdx.x; i < off[g + 1]; i += blockDim.x) gnode[i] = g;
}

// Device sample store gather (replaces DDStore fetch + decode_record +
// make_batch's host concatenation, ddstore.py:316-490 / model.py:237-250):
// output structure b is resident structure idx[b]; its atoms land at
// dst_off[b].  One CTA per output structure (grid-strided), coalesced
// contiguous copies; labels are converted to the compute dtype on the way.
template <typename T>
__global__ void k_gather_structures(const int* __restrict__ idx, int n_out,
                                    const int* __restrict__ src_off, const int* __restrict__ dst_off,
                                    const int* __restrict__ z_in, const double* __restrict__ pos_in,
                                    const double* __restrict__ e_in, const double* __restrict__ f_in,
                                    int* __restrict__ z_out, double* __restrict__ pos_out,
                                    T* __restrict__ e_out, T* __restrict__ f_out) {
  pdl_entry();
  for (int b = blockIdx.x; b < n_out; b += gridDim.x) {
    const int s = idx[b];
    const int so = src_off[s], n = src_off[s + 1] - so, d = dst_off[b];
    for (int i = threadIdx.x; i < n; i += blockDim.x) z_out[d + i] = z_in[so + i];
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) {
      pos_out[3 * d + i] = pos_in[3 * so + i];
      f_out[3 * d + i] = (T)f_in[3 * so + i];
    }
    if (threadIdx.x == 0) e_out[b] = (T)e_in[s];
  }
}

// Batch assembly from a store's per-structure CSR blocks (records keep their
// own edges, as make_batch does: model.py:234-285).  The group was packed
// once at ingest (gfm_csr_build over all its structures, float64 w / dx),
// so structure s owns nodes [so, so + n) and CSR / CSC positions
// [eo, eo + m): output graph b copies both blocks to its node / edge bases
// with the ids shifted -- the batch's stable dst / src sorts are exactly
// the concatenation of the per-structure ones (block-diagonal batches).
// meta = [counts (2) | node offsets (B+1) | n_per (B) | edge offsets (B+1)]
// of the B_true structures (host-computed); the last CTA fills the capacity
// tail (rowptr = csc_ptr = E, gnode = -1).
template <typename T>
__global__ void k_gather_batch(const int* __restrict__ idx, const int* __restrict__ meta,
                               int n_cap_graphs, int n_nodes,
                               const int* __restrict__ s_off, const int* __restrict__ s_z,
                               const double* __restrict__ s_pos, const double* __restrict__ s_e,
                               const double* __restrict__ s_f, const int* __restrict__ s_rowptr,
                               const int* __restrict__ s_col, const double* __restrict__ s_w,
                               const double* __restrict__ s_dx, const int* __restrict__ s_cscptr,
                               const int* __restrict__ s_cscid, const int* __restrict__ s_cscdst,
                               int* __restrict__ z, double* __restrict__ pos, T* __restrict__ e,
                               T* __restrict__ f, int* __restrict__ gnode,
                               int* __restrict__ rowptr, int* __restrict__ col_src,
                               int* __restrict__ edge_dst, T* __restrict__ w, T* __restrict__ dx,
                               int* __restrict__ csc_ptr, int* __restrict__ csc_eid,
                               int* __restrict__ csc_dst) {
  pdl_entry();
  const int B = meta[0];
  const int* noff = meta + 2;
  const int* eoff = meta + 2 + 2 * n_cap_graphs + 1;
  const int b = blockIdx.x;
  if (b < B) {
    const int s = idx[b];
    const int so = s_off[s], n = s_off[s + 1] - so, d = noff[b];
    const int eo = s_rowptr[so], m = s_rowptr[so + n] - eo, eb = eoff[b];
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      z[d + t] = s_z[so + t];
      gnode[d + t] = b;
      rowptr[d + t] = eb + (s_rowptr[so + t] - eo);
      csc_ptr[d + t] = eb + (s_cscptr[so + t] - eo);
    }
    for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) {
      pos[3LL * d + t] = s_pos[3LL * so + t];
      f[3LL * d + t] = (T)s_f[3LL * so + t];
    }
    for (int q = threadIdx.x; q < m; q += blockDim.x) {
      const long long sp = (long long)eo + q, dp = (long long)eb + q;
      col_src[dp] = s_col[sp] - so + d;
      // the edge's dst: the CSR row holding position sp (binary search)
      int lo = so, hi = so + n;  // rows [lo, hi): s_rowptr[lo] <= sp < s_rowptr[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_rowptr[mid] <= sp) lo = mid; else hi = mid;
      }
      edge_dst[dp] = lo - so + d;
      w[dp] = (T)s_w[sp];
      dx[3 * dp] = (T)s_dx[3 * sp];
      dx[3 * dp + 1] = (T)s_dx[3 * sp + 1];
      dx[3 * dp + 2] = (T)s_dx[3 * sp + 2];
      csc_eid[dp] = s_cscid[sp] - eo + eb;
      csc_dst[dp] = s_cscdst[sp] - so + d;
    }
    if (threadIdx.x == 0) e[b] = (T)s_e[s];
  }
  if (b == n_cap_graphs - 1) {  // capacity tail: edge-free, graph-less nodes
    const int N = meta[1], E = eoff[B];
    for (int t = N + threadIdx.x; t <= n_nodes; t += blockDim.x) {
      rowptr[t] = E;
      csc_ptr[t] = E;
      if (t < n_nodes) gnode[t] = -1;
    }
  }
}

// Variable-length row-block gather (the sharded store's pack / unpack for
// the NVLink exchange): output block b = input block idx[b], rows
// [src_off[s], src_off[s+1]) -> rows from dst_off[b], `width` 32-bit words
// per row; add (optional) is added to every word of block b (node-id shift
// of edge lists).  One CTA per output block (grid-strided), coalesced.
__global__ void k_gather_blocks(const int* __restrict__ idx, int n_out,
                                const long long* __restrict__ src_off,
                                const long long* __restrict__ dst_off, int width,
                                const unsigned* __restrict__ in, unsigned* __restrict__ out,
                                const int* __restrict__ add) {
  pdl_entry();
  for (int b = blockIdx.x; b < n_out; b += gridDim.x) {
    const int s = idx ? idx[b] : b;
    const long long so = src_off[s] * width, n = (src_off[s + 1] - src_off[s]) * width;
    const long long d = dst_off[b] * width;
    const unsigned a = add ? (unsigned)add[b] : 0u;
    for (long long t = threadIdx.x; t < n; t += blockDim.x) out[d + t] = in[so + t] + a;
  }
}

// out[q] = in[idx[q]] over q < (n_dev ? *n_dev : n) (4- or 8-byte words)
template <typename T>
__global__ void k_permute(const int* __restrict__ idx, int n, const int* __restrict__ n_dev,
                          const T* __restrict__ in, T* __restrict__ out) {
  pdl_entry();
  const int m = n_dev ? min(n, *n_dev) : n;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m; q += gridDim.x * blockDim.x)
    out[q] = in[idx[q]];
}

__global__ void k_iota(int* __restrict__ out, int n) {
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = i;
}

__global__ void k_zero_i32(int* __restrict__ out, int n) {
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = 0;
}

// count[key]++ over keys[0 .. n) where n = n_dev ? *n_dev : n_cap (int atomics:
// the result is order independent, hence deterministic).
__global__ void k_histogram(const int* __restrict__ keys, int n_cap, const int* __restrict__ n_dev,
                            int* __restrict__ count) {
  pdl_entry();
  const int n = n_dev ? *n_dev : n_cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&count[keys[i]], 1);
}

// ------------------------------------------------------------ exclusive scan
// out[0..n] = exclusive prefix of in[0..n), out[n] = total.  Three passes:
// per-block totals, a single-block scan of the totals, per-block rescans.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_excl_scan(int v, int* tmp, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < (blockDim.x >> 5) ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    tmp[lane] = s;
  }
  __syncthreads();
  total = tmp[(blockDim.x >> 5) - 1];
  int before = wid ? tmp[wid - 1] : 0;
  __syncthreads();
  return before + x - v;
}

__global__ void k_scan_partials(const int* __restrict__ in, int n, int* __restrict__ partial) {
  pdl_entry();
  __shared__ int tmp[32];
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += in[base + k];
  int total;
  block_excl_scan(s, tmp, total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

__global__ void k_scan_totals(int* __restrict__ partial, int nb) {
  pdl_entry();
  __shared__ int tmp[32];
  int carry = 0;
  for (int c = 0; c < nb; c += kScanThreads) {
    int i = c + threadIdx.x;
    int v = i < nb ? partial[i] : 0;
    int total;
    int ex = block_excl_scan(v, tmp, total);
    if (i < nb) partial[i] = carry + ex;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[nb] = carry;
}

__global__ void k_scan_final(const int* __restrict__ in, int n, const int* __restrict__ partial,
                             int* __restrict__ out) {
  pdl_entry();
  __shared__ int tmp[32];
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int total;
  int ex = block_excl_scan(s, tmp, total) + partial[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = partial[gridDim.x];
}

size_t scan_ws_bytes(int n) { return sizeof(int) * ((size_t)ceil_div(n > 0 ? n : 1, kScanTile) + 1); }

cudaError_t exclusive_scan(const int* in, int n, int* out, int* ws, cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(out, 0, sizeof(int), s);
  int nb = ceil_div(n, kScanTile);
  launch_k(k_scan_partials, nb, kScanThreads, 0, s, in, n, ws);
  launch_k(k_scan_totals, 1, kScanThreads, 0, s, ws, nb);
  launch_k(k_scan_final, nb, kScanThreads, 0, s, in, n, ws, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ radius graph
// One warp per destination atom i scans the atoms j of its graph in index
// order; pairs with d(i, j) <= rc (j != i) become edges j -> i.  The float64
// predicate reproduces numpy exactly: d = sqrt((dx*dx + dy*dy) + dz*dz), each
// operation separately rounded (no FMA), so the neighbour list is bit-exact
// against build_cutoff_edges.  Optional minimum image over an orthorhombic
// cell (shift = -L * rint(delta / L)) and a per-destination cap keeping the
// max_nbr nearest sources by (distance, source index).
constexpr int kRadiusWarps = 4, kCapBuf = 256;

struct PairGeom {
  double dx, dy, dz, d;
};

__device__ __forceinline__ PairGeom pair_geom(const double* __restrict__ pos, int src, int dst,
                                              const double* cell) {
  PairGeom g;
  g.dx = __dsub_rn(pos[3 * src + 0], pos[3 * dst + 0]);
  g.dy = __dsub_rn(pos[3 * src + 1], pos[3 * dst + 1]);
  g.dz = __dsub_rn(pos[3 * src + 2], pos[3 * dst + 2]);
  if (cell) {
    g.dx = __dadd_rn(g.dx, __dmul_rn(-cell[0], rint(__ddiv_rn(g.dx, cell[0]))));
    g.dy = __dadd_rn(g.dy, __dmul_rn(-cell[1], rint(__ddiv_rn(g.dy, cell[1]))));
    g.dz = __dadd_rn(g.dz, __dmul_rn(-cell[2], rint(__ddiv_rn(g.dz, cell[2]))));
  }
  g.d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(g.dx, g.dx), __dmul_rn(g.dy, g.dy)),
                             __dmul_rn(g.dz, g.dz)));
  return g;
}

__device__ __forceinline__ bool key_less(double da, int ja, double db, int jb) {
  return da < db || (da == db && ja < jb);
}

template <typename T, bool kFill>
__global__ void __launch_bounds__(kRadiusWarps * 32)
    k_radius(const double* __restrict__ pos, const int* __restrict__ node_off,
             const int* __restrict__ gnode, int n_nodes, const double* __restrict__ cells, double rc,
             int max_nbr, int* __restrict__ deg, const int* __restrict__ rowptr,
             int* __restrict__ col_src, int* __restrict__ edge_dst, T* __restrict__ edge_w,
             T* __restrict__ edge_dx) {
  pdl_entry();
  __shared__ double s_d[kRadiusWarps][kCapBuf];
  __shared__ int s_j[kRadiusWarps][kCapBuf];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int i = blockIdx.x * kRadiusWarps + wib;
  if (i >= n_nodes) return;
  const int g = gnode[i];
  const int lo = node_off[g], hi = node_off[g + 1];
  const double* cell = cells ? cells + 3 * g : nullptr;
  const unsigned lt = (1u << lane) - 1u;

  // pass 1: candidate count (and, when a cap binds, candidate list)
  int c = 0;
  for (int j0 = lo; j0 < hi; j0 += 32) {
    const int j = j0 + lane;
    bool hit = false;
    double d = 0.0;
    if (j < hi && j != i) {
      PairGeom pg = pair_geom(pos, j, i, cell);
      d = pg.d;
      hit = d <= rc;
    }
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (kFill && max_nbr > 0 && hit) {
      const int k = c + __popc(b & lt);
      if (k < kCapBuf) {
        s_d[wib][k] = d;
        s_j[wib][k] = j;
      }
    }
    c += __popc(b);
  }
  const bool capped = max_nbr > 0 && c > max_nbr;
  if (!kFill) {
    if (lane == 0) deg[i] = capped ? max_nbr : c;
    return;
  }
  __syncwarp();
  int out = rowptr[i];
  auto emit = [&](int j, int slot) {
    PairGeom pg = pair_geom(pos, j, i, cell);
    const int p = out + slot;
    col_src[p] = j;
    edge_dst[p] = i;
    edge_dx[3LL * p + 0] = (T)pg.dx;
    edge_dx[3LL * p + 1] = (T)pg.dy;
    edge_dx[3LL * p + 2] = (T)pg.dz;
    // make_batch (model.py:256-258): w = 1 / (1 + |pos[src] - pos[dst]|)
    edge_w[p] = (T)__ddiv_rn(1.0, __dadd_rn(1.0, pg.d));
  };
  if (!capped) {
    int k = 0;
    for (int j0 = lo; j0 < hi; j0 += 32) {
      const int j = j0 + lane;
      bool hit = false;
      if (j < hi && j != i) hit = pair_geom(pos, j, i, cell).d <= rc;
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      if (hit) emit(j, k + __popc(b & lt));
      k += __popc(b);
    }
    return;
  }
  if (c <= kCapBuf) {
    // rank every candidate by (d, j); keep rank < max_nbr, emit in j order
    int k = 0;
    for (int a0 = 0; a0 < c; a0 += 32) {
      const int a = a0 + lane;
      bool keep = false;
      int ja = 0;
      if (a < c) {
        const double da = s_d[wib][a];
        ja = s_j[wib][a];
        int rank = 0;
        for (int q = 0; q < c; ++q) rank += key_less(s_d[wib][q], s_j[wib][q], da, ja);
        keep = rank < max_nbr;
      }
      const unsigned b = __ballot_sync(0xffffffffu, keep);
      if (keep) emit(ja, k + __popc(b & lt));
      k += __popc(b);
    }
    return;
  }
  // large candidate sets: recompute ranks from global memory (O(n * c))
  int k = 0;
  for (int j0 = lo; j0 < hi; j0 += 32) {
    const int j = j0 + lane;
    bool keep = false;
    if (j < hi && j != i) {
      const double dj = pair_geom(pos, j, i, cell).d;
      if (dj <= rc) {
        int rank = 0;
        for (int q = lo; q < hi; ++q) {
          if (q == i) continue;
          const double dq = pair_geom(pos, q, i, cell).d;
          if (dq <= rc && key_less(dq, q, dj, j)) ++rank;
        }
        keep = rank < max_nbr;
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if (keep) emit(j, k + __popc(b & lt));
    k += __popc(b);
  }
}

// ------------------------------------------------- stable bucket placement
// For each segment s (one graph's edges [seg[s], seg[s+1])) a warp walks the
// edges in order, 32 at a time; lanes with equal keys are ranked with
// __match_any_sync so the placement is stable.  cursor[] starts as a copy of
// the bucket pointers.  Graphs own disjoint node ranges, so warps never share
// a cursor.  Output perm[position] = input edge index.
__global__ void k_stable_bucket(const int* __restrict__ keys, const int* __restrict__ seg,
                                int n_segs, int* __restrict__ cursor, int* __restrict__ perm) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= n_segs) return;
  const int lo = seg[s], hi = seg[s + 1];
  const unsigned lt = (1u << lane) - 1u;
  for (int e0 = lo; e0 < hi; e0 += 32) {
    const int e = e0 + lane;
    const bool act = e < hi;
    const int key = act ? keys[e] : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    int base = 0;
    if (act) base = cursor[key];
    __syncwarp();
    if (act) {
      perm[base + __popc(peers & lt)] = e;
      if ((peers & lt) == 0) cursor[key] = base + __popc(peers);
    }
    __syncwarp();
  }
}

__global__ void k_copy_i32(const int* __restrict__ in, int n, int* __restrict__ out) {
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i];
}

__global__ void k_edge_offsets(const int* __restrict__ rowptr, const int* __restrict__ node_off,
                               int n_graphs, int* __restrict__ eoff) {
  pdl_entry();
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g <= n_graphs; g += gridDim.x * blockDim.x)
    eoff[g] = rowptr[node_off[g]];
}

// CSR arrays from record edges through the dst permutation; geometry in
// float64 exactly as make_batch (model.py:256-258), cast to T on store.
template <typename T>
__global__ void k_csr_gather(const int* __restrict__ perm, int n_edges, const int* __restrict__ src,
                             const int* __restrict__ dst, const double* __restrict__ pos,
                             const double* __restrict__ shift, int* __restrict__ col_src,
                             int* __restrict__ edge_dst, T* __restrict__ edge_w,
                             T* __restrict__ edge_dx, int* __restrict__ inv) {
  pdl_entry();
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_edges; p += gridDim.x * blockDim.x) {
    const int e = perm[p];
    const int s = src[e], d = dst[e];
    double dx = __dsub_rn(pos[3 * s + 0], pos[3 * d + 0]);
    double dy = __dsub_rn(pos[3 * s + 1], pos[3 * d + 1]);
    double dz = __dsub_rn(pos[3 * s + 2], pos[3 * d + 2]);
    if (shift) {
      dx = __dadd_rn(dx, shift[3LL * e + 0]);
      dy = __dadd_rn(dy, shift[3LL * e + 1]);
      dz = __dadd_rn(dz, shift[3LL * e + 2]);
    }
    const double dist =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    col_src[p] = s;
    edge_dst[p] = d;
    edge_w[p] = (T)__ddiv_rn(1.0, __dadd_rn(1.0, dist));
    edge_dx[3LL * p + 0] = (T)dx;
    edge_dx[3LL * p + 1] = (T)dy;
    edge_dx[3LL * p + 2] = (T)dz;
    if (inv) inv[e] = p;
  }
}

__global__ void k_csc_finish(const int* __restrict__ perm_csc, int n_cap, const int* __restrict__ n_dev,
                             const int* __restrict__ inv, const int* __restrict__ dst,
                             int* __restrict__ csc_eid, int* __restrict__ csc_dst) {
  pdl_entry();
  const int n = n_dev ? *n_dev : n_cap;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int e = perm_csc[q];
    csc_eid[q] = inv ? inv[e] : e;
    csc_dst[q] = dst[e];
  }
}


// ------------------------------------------- fused per-graph batch assembly
// One CTA per graph builds that graph's whole slice of the batch in one pass:
// neighbour search over the graph's atoms (positions staged in smem, same
// fp64 predicate / cap / minimum image as k_radius), the dst-sorted CSR rows,
// the src-sorted CSC (within a graph, CSC order of src j = ascending dst, so a
// walk over dst rows with per-src cursors is already stable), graph_of_node,
// and graph_of_node.  Three launches replace the 15 of count / scan / fill /
// CSC build: a count pass (per-graph edge totals), one single-block scan of
// those totals, and the fill pass (the neighbour search is cheap enough to
// run twice; a one-pass decoupled look-back measured slower -- with every
// graph CTA resident at once its prefix chain is the critical path).
constexpr int kFusedMaxAtoms = 256, kFusedWarps = 8;

__host__ __device__ inline int fused_stride(int n_max, int max_nbr) {
  const int full = n_max > 1 ? n_max - 1 : 1;
  return max_nbr > 0 && max_nbr < full ? max_nbr : full;
}

// per-CTA buffers are sized by the batch's largest graph (rounded up to 32)
__host__ __device__ inline int fused_rows(int n_max) { return ((n_max > 1 ? n_max : 1) + 31) / 32 * 32; }

__host__ __device__ inline size_t fused_smem_bytes(int n_max, int max_nbr) {
  const size_t a = fused_rows(n_max);
  return a * 3 * sizeof(double)                                  // positions
         + (size_t)kFusedWarps * a * (sizeof(double) + sizeof(int))  // cap candidates
         + (3 * a + 16) * sizeof(int)                             // rowptr, csc start, cursor, base
         + (size_t)n_max * fused_stride(n_max, max_nbr) * sizeof(int);  // neighbour lists
}

__device__ __forceinline__ PairGeom pair_geom_s(const double* __restrict__ sp, int j, int i,
                                                const double* cell) {
  PairGeom g;
  g.dx = __dsub_rn(sp[3 * j + 0], sp[3 * i + 0]);
  g.dy = __dsub_rn(sp[3 * j + 1], sp[3 * i + 1]);
  g.dz = __dsub_rn(sp[3 * j + 2], sp[3 * i + 2]);
  if (cell) {
    g.dx = __dadd_rn(g.dx, __dmul_rn(-cell[0], rint(__ddiv_rn(g.dx, cell[0]))));
    g.dy = __dadd_rn(g.dy, __dmul_rn(-cell[1], rint(__ddiv_rn(g.dy, cell[1]))));
    g.dz = __dadd_rn(g.dz, __dmul_rn(-cell[2], rint(__ddiv_rn(g.dz, cell[2]))));
  }
  g.d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(g.dx, g.dx), __dmul_rn(g.dy, g.dy)),
                             __dmul_rn(g.dz, g.dz)));
  return g;
}

template <typename T, bool kFill>
__global__ void __launch_bounds__(kFusedWarps * 32)
    k_radius_batch(const double* __restrict__ pos, const int* __restrict__ node_off, int n_graphs,
                   int n_nodes, const double* __restrict__ cells, double rc, int max_nbr,
                   int stride, int* __restrict__ gnode, int* __restrict__ rowptr,
                   int* __restrict__ col_src, int* __restrict__ edge_dst, T* __restrict__ edge_w,
                   T* __restrict__ edge_dx, int* __restrict__ csc_ptr, int* __restrict__ csc_eid,
                   int* __restrict__ csc_dst, int* __restrict__ gcount, int A, int e_cap) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char fsm[];
  double* s_pos = reinterpret_cast<double*>(fsm);
  double* s_cd = s_pos + 3 * A;                                  // [warps][A]
  int* s_cj = reinterpret_cast<int*>(s_cd + kFusedWarps * A);    // [warps][A]
  int* s_rp = s_cj + kFusedWarps * A;                            // [A + 1] local rowptr
  int* s_cs = s_rp + A + 1;                                      // [A + 1] local csc start
  int* s_cur = s_cs + A + 1;                                     // [A]
  int* s_base = s_cur + A;                                       // [1] graph edge base
  int* s_nb = s_base + 8;                                        // [n][stride] sources
  const int g = blockIdx.x;
  const int lo = node_off[g], hi = node_off[g + 1], n = hi - lo;
  const double* cell = cells ? cells + 3 * g : nullptr;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) s_pos[t] = pos[3LL * lo + t];
  for (int t = threadIdx.x; t <= n; t += blockDim.x) s_cs[t] = 0;
  if (kFill)
    for (int t = threadIdx.x; t < n; t += blockDim.x) gnode[lo + t] = g;
  __syncthreads();

  // A. per destination (warp-strided): neighbours in src order into s_nb
  for (int i = wib; i < n; i += kFusedWarps) {
    double* cd = s_cd + wib * A;
    int* cj = s_cj + wib * A;
    int c = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      bool hit = false;
      double d = 0.0;
      if (j < n && j != i) {
        d = pair_geom_s(s_pos, j, i, cell).d;
        hit = d <= rc;
      }
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int k = c + __popc(b & lt);
        cd[k] = d;
        cj[k] = j;
      }
      c += __popc(b);
    }
    __syncwarp();
    int deg = c;
    if (max_nbr > 0 && c > max_nbr) {
      // rank by (d, j); keep rank < max_nbr, in j order (same rule as k_radius)
      int k = 0;
      for (int a0 = 0; a0 < c; a0 += 32) {
        const int a = a0 + lane;
        bool keep = false;
        int ja = 0;
        if (a < c) {
          const double da = cd[a];
          ja = cj[a];
          int rank = 0;
          for (int q = 0; q < c; ++q) rank += key_less(cd[q], cj[q], da, ja);
          keep = rank < max_nbr;
        }
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (keep) s_nb[i * stride + k + __popc(b & lt)] = ja;
        k += __popc(b);
      }
      deg = max_nbr;
    } else {
      for (int a = lane; a < c; a += 32) s_nb[i * stride + a] = cj[a];
    }
    if (lane == 0) s_rp[i] = deg;
    __syncwarp();
  }
  __syncthreads();

  // B. local scans: rowptr over dst degrees; csc starts over src counts
  if (wib == 0) {
    int carry = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      int v = i < n ? s_rp[i] : 0, x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < n) s_rp[i] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_rp[n] = carry;
  }
  __syncthreads();
  if (!kFill) {  // count pass: the graph's edge total (scanned between the passes)
    if (threadIdx.x == 0) gcount[g] = s_rp[n];
    if (g == 0 && threadIdx.x == 0) gcount[n_graphs + 1] = 0;  // overflow flag of this call
    return;
  }
  // edge buffers hold e_cap edges: a batch with more raises the overflow flag
  // (read by the host, gfm_radius_batch_overflow) and is emitted edge-free
  // instead of writing out of bounds
  const int total = gcount[n_graphs];
  if (total > e_cap) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      rowptr[lo + t] = 0;
      csc_ptr[lo + t] = 0;
    }
    if (g == n_graphs - 1)
      for (int t = node_off[n_graphs] + threadIdx.x; t <= n_nodes; t += blockDim.x) {
        rowptr[t] = 0;
        csc_ptr[t] = 0;
        if (t < n_nodes) gnode[t] = -1;
      }
    if (g == 0 && threadIdx.x == 0) gcount[n_graphs + 1] = 1;
    return;
  }
  for (int i = wib; i < n; i += kFusedWarps)
    for (int k = lane; k < s_rp[i + 1] - s_rp[i]; k += 32) atomicAdd(&s_cs[s_nb[i * stride + k]], 1);
  __syncthreads();
  if (wib == 0) {
    int carry = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      int v = j < n ? s_cs[j] : 0, x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (j < n) {
        s_cs[j] = carry + x - v;
        s_cur[j] = carry + x - v;
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }

  __syncthreads();
  const int base = gcount[g];  // exclusive prefix of the graph edge counts

  // D. outputs
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    rowptr[lo + t] = base + s_rp[t];
    csc_ptr[lo + t] = base + s_cs[t];
  }
  // capacity tail (ragged batches in a fixed-capacity runner): nodes past the
  // last graph are edge-free and belong to no graph
  if (g == n_graphs - 1)
    for (int t = node_off[n_graphs] + threadIdx.x; t <= n_nodes; t += blockDim.x) {
      rowptr[t] = total;
      csc_ptr[t] = total;
      if (t < n_nodes) gnode[t] = -1;
    }
  for (int i = wib; i < n; i += kFusedWarps) {
    const int r0 = s_rp[i], deg = s_rp[i + 1] - r0;
    for (int k = lane; k < deg; k += 32) {
      const int j = s_nb[i * stride + k];
      const PairGeom pg = pair_geom_s(s_pos, j, i, cell);
      const long long p = (long long)base + r0 + k;
      col_src[p] = lo + j;
      edge_dst[p] = lo + i;
      edge_dx[3 * p + 0] = (T)pg.dx;
      edge_dx[3 * p + 1] = (T)pg.dy;
      edge_dx[3 * p + 2] = (T)pg.dz;
      // make_batch (model.py:256-258): w = 1 / (1 + |pos[src] - pos[dst]|)
      edge_w[p] = (T)__ddiv_rn(1.0, __dadd_rn(1.0, pg.d));
    }
  }
  // CSC slots: walk dst rows in order (sources within a row are distinct)
  if (wib == 0) {
    for (int i = 0; i < n; ++i) {
      const int r0 = s_rp[i], deg = s_rp[i + 1] - r0;
      for (int k = lane; k < deg; k += 32) {
        const int j = s_nb[i * stride + k];
        const int slot = s_cur[j]++;
        csc_eid[base + slot] = base + r0 + k;
        csc_dst[base + slot] = lo + i;
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------ entry points
template <typename T>
cudaError_t radius_fill_t(const double* pos, const int* node_off, const int* gnode, int n_nodes,
                          const double* cells, double rc, int max_nbr, const int* rowptr,
                          int* col_src, int* edge_dst, void* w, void* dx, cudaStream_t s) {
  if (n_nodes <= 0) return cudaSuccess;
  launch_k(k_radius<T, true>, ceil_div(n_nodes, kRadiusWarps), kRadiusWarps * 32, 0, s,
      pos, node_off, gnode, n_nodes, cells, rc, max_nbr, nullptr, rowptr, col_src, edge_dst,
      (T*)w, (T*)dx);
  return cudaGetLastError();
}

}  // namespace gfm

using namespace gfm;

static inline int grid_for(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

#define GFM_TRY(expr)                                                   \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) {                                            \
      gfm::set_error("%s: %s", #expr, cudaGetErrorString(_e));          \
      return (int)_e;                                                   \
    }                                                                   \
  } while (0)

extern "C" {

int gfm_graph_of_node(const int* node_offsets, int n_graphs, int* gnode, void* stream) {
  if (n_graphs <= 0) return 0;
  launch_k(k_graph_of_node, grid_for(n_graphs, 1), 128, 0, (cudaStream_t)stream, node_offsets, n_graphs, gnode);
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_gather_structures(const int* idx, int n_out, const int* src_off, const int* dst_off,
                          const int* z_in, const double* pos_in, const double* energy_in,
                          const double* forces_in, int* z_out, double* pos_out, void* energy_out,
                          void* forces_out, int dtype, void* stream) {
  if (n_out <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = n_out < 148 * 16 ? n_out : 148 * 16;
  if (dtype == GFM_F32)
    launch_k(k_gather_structures<float>, grid, 128, 0, s, idx, n_out, src_off, dst_off, z_in, pos_in,
             energy_in, forces_in, z_out, pos_out, (float*)energy_out, (float*)forces_out);
  else
    launch_k(k_gather_structures<double>, grid, 128, 0, s, idx, n_out, src_off, dst_off, z_in,
             pos_in, energy_in, forces_in, z_out, pos_out, (double*)energy_out,
             (double*)forces_out);
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_gather_batch(const int* idx, const int* meta, int n_cap_graphs, int n_nodes,
                     const int* s_off, const int* s_z, const double* s_pos, const double* s_e,
                     const double* s_f, const int* s_rowptr, const int* s_col, const double* s_w,
                     const double* s_dx, const int* s_cscptr, const int* s_cscid,
                     const int* s_cscdst, int* z, double* pos, void* e, void* f, int* gnode,
                     int* rowptr, int* col_src, int* edge_dst, void* w, void* dx, int* csc_ptr,
                     int* csc_eid, int* csc_dst, int dtype, void* stream) {
  if (n_cap_graphs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GFM_F32)
    launch_k(k_gather_batch<float>, n_cap_graphs, 128, 0, s, idx, meta, n_cap_graphs, n_nodes,
             s_off, s_z, s_pos, s_e, s_f, s_rowptr, s_col, s_w, s_dx, s_cscptr, s_cscid, s_cscdst,
             z, pos, (float*)e, (float*)f, gnode, rowptr, col_src, edge_dst, (float*)w, (float*)dx,
             csc_ptr, csc_eid, csc_dst);
  else if (dtype == GFM_F64)
    launch_k(k_gather_batch<double>, n_cap_graphs, 128, 0, s, idx, meta, n_cap_graphs, n_nodes,
             s_off, s_z, s_pos, s_e, s_f, s_rowptr, s_col, s_w, s_dx, s_cscptr, s_cscid,
             s_cscdst, z, pos, (double*)e, (double*)f, gnode, rowptr, col_src, edge_dst,
             (double*)w, (double*)dx, csc_ptr, csc_eid, csc_dst);
  else {
    set_error("gfm_gather_batch: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_gather_blocks(const int* idx, int n_out, const long long* src_off,
                      const long long* dst_off, int width, const void* in, void* out,
                      const int* add, void* stream) {
  if (n_out <= 0) return 0;
  const int grid = n_out < 148 * 16 ? n_out : 148 * 16;
  launch_k(k_gather_blocks, grid, 128, 0, (cudaStream_t)stream, idx, n_out, src_off, dst_off,
           width, (const unsigned*)in, (unsigned*)out, add);
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_permute(const int* idx, int n, const int* n_dev, const void* in, void* out, int dtype,
                void* stream) {
  if (n <= 0) return 0;
  const int grid = ceil_div(n, 256) < 148 * 8 ? ceil_div(n, 256) : 148 * 8;
  if (dtype == GFM_F64)
    launch_k(k_permute<double>, grid, 256, 0, (cudaStream_t)stream, idx, n, n_dev,
             (const double*)in, (double*)out);
  else
    launch_k(k_permute<float>, grid, 256, 0, (cudaStream_t)stream, idx, n, n_dev,
             (const float*)in, (float*)out);
  GFM_TRY(cudaGetLastError());
  return 0;
}

size_t gfm_scan_workspace_bytes(int n) { return scan_ws_bytes(n); }

int gfm_exclusive_scan(const int* in, int n, int* out, void* workspace, void* stream) {
  GFM_TRY(exclusive_scan(in, n, out, (int*)workspace, (cudaStream_t)stream));
  return 0;
}

int gfm_radius_count(const double* pos, const int* node_offsets, const int* gnode, int n_nodes,
                     const double* cells, double rc, int max_nbr, int* deg, void* stream) {
  if (n_nodes <= 0) return 0;
  launch_k(k_radius<float, false>, ceil_div(n_nodes, kRadiusWarps), kRadiusWarps * 32, 0, (cudaStream_t)stream, pos, node_offsets, gnode, n_nodes, cells, rc,
                                                   max_nbr, deg, nullptr, nullptr, nullptr, nullptr,
                                                   nullptr);
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_radius_fill(const double* pos, const int* node_offsets, const int* gnode, int n_nodes,
                    const double* cells, double rc, int max_nbr, const int* rowptr, int* col_src,
                    int* edge_dst, void* edge_w, void* edge_dx, int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GFM_F32)
    GFM_TRY(radius_fill_t<float>(pos, node_offsets, gnode, n_nodes, cells, rc, max_nbr, rowptr,
                                 col_src, edge_dst, edge_w, edge_dx, s));
  else if (dtype == GFM_F64)
    GFM_TRY(radius_fill_t<double>(pos, node_offsets, gnode, n_nodes, cells, rc, max_nbr, rowptr,
                                  col_src, edge_dst, edge_w, edge_dx, s));
  else {
    set_error("gfm_radius_fill: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  return 0;
}

size_t gfm_csr_workspace_bytes(int n_nodes, int n_edges, int n_graphs) {
  (void)n_graphs;
  size_t b = scan_ws_bytes(n_nodes + 1);
  b += sizeof(int) * (size_t)(n_nodes + 1) * 2;  // degree + cursor
  b += sizeof(int) * (size_t)(n_edges + 1) * 2;  // inv + perm_csc
  b += sizeof(int) * (size_t)(n_graphs + 1);     // per-graph edge offsets
  return b + 256 * 6;
}

static char* carve(char*& p, size_t bytes) {
  char* r = p;
  p += (bytes + 255) & ~(size_t)255;
  return r;
}

int gfm_csr_build(const int* src, const int* dst, const int* edge_offsets, int n_graphs,
                  const double* pos, const double* shift, int n_nodes, int n_edges, int* rowptr,
                  int* col_src, int* edge_dst, void* edge_w, void* edge_dx, int* order, int* csc_ptr,
                  int* csc_eid, int* csc_dst, int dtype, void* workspace, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype != GFM_F32 && dtype != GFM_F64) {
    set_error("gfm_csr_build: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  char* p = (char*)workspace;
  int* scan_ws = (int*)carve(p, scan_ws_bytes(n_nodes + 1));
  int* count = (int*)carve(p, sizeof(int) * (n_nodes + 1));
  int* cursor = (int*)carve(p, sizeof(int) * (n_nodes + 1));
  int* inv = (int*)carve(p, sizeof(int) * (n_edges + 1));
  int* perm_csc = (int*)carve(p, sizeof(int) * (n_edges + 1));
  const int nt = 256;
  // dst-sorted CSR (stable): order[p] = original edge index (model.py:260)
  launch_k(k_zero_i32, grid_for(n_nodes), nt, 0, s, count, n_nodes);
  if (n_edges > 0) launch_k(k_histogram, grid_for(n_edges), nt, 0, s, dst, n_edges, nullptr, count);
  GFM_TRY(exclusive_scan(count, n_nodes, rowptr, scan_ws, s));
  launch_k(k_copy_i32, grid_for(n_nodes), nt, 0, s, rowptr, n_nodes, cursor);
  if (n_edges > 0 && n_graphs > 0)
    launch_k(k_stable_bucket, ceil_div(n_graphs, 4), 128, 0, s, dst, edge_offsets, n_graphs, cursor, order);
  if (n_edges > 0) {
    if (dtype == GFM_F32)
      launch_k(k_csr_gather<float>, grid_for(n_edges), nt, 0, s, order, n_edges, src, dst, pos, shift,
                                                           col_src, edge_dst, (float*)edge_w,
                                                           (float*)edge_dx, inv);
    else
      launch_k(k_csr_gather<double>, grid_for(n_edges), nt, 0, s, order, n_edges, src, dst, pos, shift,
                                                            col_src, edge_dst, (double*)edge_w,
                                                            (double*)edge_dx, inv);
  }
  // src-sorted CSC (stable over original order)
  launch_k(k_zero_i32, grid_for(n_nodes), nt, 0, s, count, n_nodes);
  if (n_edges > 0) launch_k(k_histogram, grid_for(n_edges), nt, 0, s, src, n_edges, nullptr, count);
  GFM_TRY(exclusive_scan(count, n_nodes, csc_ptr, scan_ws, s));
  launch_k(k_copy_i32, grid_for(n_nodes), nt, 0, s, csc_ptr, n_nodes, cursor);
  if (n_edges > 0 && n_graphs > 0) {
    launch_k(k_stable_bucket, ceil_div(n_graphs, 4), 128, 0, s, src, edge_offsets, n_graphs, cursor, perm_csc);
    launch_k(k_csc_finish, grid_for(n_edges), nt, 0, s, perm_csc, n_edges, nullptr, inv, dst, csc_eid, csc_dst);
  }
  GFM_TRY(cudaGetLastError());
  return 0;
}

int gfm_csc_from_csr(const int* rowptr, const int* col_src, const int* edge_dst,
                     const int* node_offsets, int n_graphs, int n_nodes, int e_cap, int* csc_ptr,
                     int* csc_eid, int* csc_dst, void* workspace, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  char* p = (char*)workspace;
  int* scan_ws = (int*)carve(p, scan_ws_bytes(n_nodes + 1));
  int* count = (int*)carve(p, sizeof(int) * (n_nodes + 1));
  int* cursor = (int*)carve(p, sizeof(int) * (n_nodes + 1));
  carve(p, sizeof(int) * (e_cap + 1));
  int* perm_csc = (int*)carve(p, sizeof(int) * (e_cap + 1));
  int* eoff = (int*)carve(p, sizeof(int) * (n_graphs + 1));
  const int nt = 256;
  const int* n_dev = rowptr + n_nodes;
  launch_k(k_zero_i32, grid_for(n_nodes), nt, 0, s, count, n_nodes);
  if (e_cap > 0) launch_k(k_histogram, grid_for(e_cap), nt, 0, s, col_src, e_cap, n_dev, count);
  GFM_TRY(exclusive_scan(count, n_nodes, csc_ptr, scan_ws, s));
  launch_k(k_copy_i32, grid_for(n_nodes), nt, 0, s, csc_ptr, n_nodes, cursor);
  if (n_graphs > 0) {
    launch_k(k_edge_offsets, grid_for(n_graphs + 1), nt, 0, s, rowptr, node_offsets, n_graphs, eoff);
    launch_k(k_stable_bucket, ceil_div(n_graphs, 4), 128, 0, s, col_src, eoff, n_graphs, cursor, perm_csc);
  }
  if (e_cap > 0)
    launch_k(k_csc_finish, grid_for(e_cap), nt, 0, s, perm_csc, e_cap, n_dev, nullptr, edge_dst, csc_eid, csc_dst);
  GFM_TRY(cudaGetLastError());
  return 0;
}

size_t gfm_radius_batch_workspace_bytes(int n_graphs) {
  return sizeof(int) * (size_t)((n_graphs > 0 ? n_graphs : 1) + 2) + 256;
}

int gfm_radius_batch_overflow_index(int n_graphs) { return n_graphs + 1; }

int gfm_radius_batch(const double* pos, const int* node_offsets, int n_graphs, int n_nodes,
                     int max_atoms, const double* cells, double rc, int max_nbr, int* gnode,
                     int* rowptr, int* col_src, int* edge_dst, void* edge_w, void* edge_dx,
                     int* csc_ptr, int* csc_eid, int* csc_dst, int e_cap, void* workspace,
                     int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (max_atoms > kFusedMaxAtoms || max_atoms < 0 || n_graphs <= 0) {
    set_error("gfm_radius_batch: graphs of up to %d atoms (got %d), n_graphs >= 1",
              kFusedMaxAtoms, max_atoms);
    return GFM_EINVAL;
  }
  const int stride = fused_stride(max_atoms, max_nbr);
  const size_t smem = fused_smem_bytes(max_atoms, max_nbr);
  if (smem > 227 * 1024) {
    set_error("gfm_radius_batch: %d atoms x %d neighbours exceed shared memory", max_atoms, stride);
    return GFM_EINVAL;
  }
  int* gcount = (int*)workspace;  // [n_graphs + 1] counts -> exclusive prefix
  const int A = fused_rows(max_atoms);
  auto run = [&](auto t) -> cudaError_t {
    using T = decltype(t);
    cudaError_t e = cudaFuncSetAttribute(k_radius_batch<T, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_radius_batch<T, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    launch_k(k_radius_batch<T, false>, n_graphs, kFusedWarps * 32, smem, s, pos, node_offsets,
             n_graphs, n_nodes, cells, rc, max_nbr, stride, gnode, rowptr, col_src, edge_dst,
             (T*)edge_w, (T*)edge_dx, csc_ptr, csc_eid, csc_dst, gcount, A, e_cap);
    launch_k(k_scan_totals, 1, kScanThreads, 0, s, gcount, n_graphs);
    launch_k(k_radius_batch<T, true>, n_graphs, kFusedWarps * 32, smem, s, pos, node_offsets,
             n_graphs, n_nodes, cells, rc, max_nbr, stride, gnode, rowptr, col_src, edge_dst,
             (T*)edge_w, (T*)edge_dx, csc_ptr, csc_eid, csc_dst, gcount, A, e_cap);
    return cudaGetLastError();
  };
  if (dtype == GFM_F32)
    GFM_TRY(run(float{}));
  else if (dtype == GFM_F64)
    GFM_TRY(run(double{}));
  else {
    set_error("gfm_radius_batch: bad dtype %d", dtype);
    return GFM_EINVAL;
  }
  return 0;
}

}  // extern "C"
