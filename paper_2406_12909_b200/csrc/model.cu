// Dense model pieces on the SIMT engine: node update / head linear layers
// (forward, data-grad, deterministic split-K weight-grad), the fused force
// head (gather-fed GEMM + tanh + u-dot + dst-CSR reduction, and its
// backward with recompute), energy readout + graph pooling, the L1 MTL loss
// with its seeds, and the embedding gradient.
//
// Reference: forward_batch (model.py:344-400), mtl_loss (model.py:437-462),
// loss_and_grad (model.py:483-565).
#include "gemm_simt.cuh"

namespace gfm {

static inline int grid_1d(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

// ------------------------------------------------------------ force epilogues
template <typename T>
struct EpiForceFwd {  // t = tanh(pre + c); partial m = sum_n t*u over this N tile
  const T* c;
  const T* u;
  T* m_part;
  int ntiles;
  __device__ void operator()(T (&acc)[kTM][kTN], int m0, int n0, int M, int N, int, int, int bn,
                             int tx, int) const {
    T part[kTM];
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
      part[i] = T(0);
#pragma unroll
      for (int j = 0; j < kTN; ++j) {
        const int n = n0 + j;
        if (n < N) part[i] += tanh_t(acc[i][j] + c[n]) * u[n];
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) part[i] += __shfl_xor_sync(0xffffffffu, part[i], o);
    }
    if (tx == 0) {
#pragma unroll
      for (int i = 0; i < kTM; ++i)
        if (m0 + i < M) m_part[(long long)(m0 + i) * ntiles + bn] = part[i];
    }
  }
};

template <typename T>
struct EpiForceBwd {  // dm = df[dst].dx; dpre = dm*u*(1-t^2); column partials of t*dm
  const T* c;
  const T* u;
  const T* df;
  const int* edge_dst;
  const T* dx;
  T* dpre;
  int H;
  T* ws_u;
  __device__ void operator()(T (&acc)[kTM][kTN], int m0, int n0, int M, int N, int, int bm, int,
                             int tx, int ty) const {
    __shared__ T red[16][kBN];
    T dm[kTM];
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
      const int m = m0 + i;
      dm[i] = T(0);
      if (m < M) {  // model.py:537-538, sum over xyz left to right
        const T* f = df + 3LL * edge_dst[m];
        const T* d = dx + 3LL * m;
        dm[i] = add_rn(add_rn(mul_rn(f[0], d[0]), mul_rn(f[1], d[1])), mul_rn(f[2], d[2]));
      }
    }
    T colpart[kTN];
#pragma unroll
    for (int j = 0; j < kTN; ++j) {
      colpart[j] = T(0);
      const int n = n0 + j;
      if (n >= N) continue;
#pragma unroll
      for (int i = 0; i < kTM; ++i) {
        const int m = m0 + i;
        if (m >= M) continue;
        const T t = tanh_t(acc[i][j] + c[n]);
        dpre[(long long)m * H + n] = mul_rn(mul_rn(dm[i], u[n]), sub_rn(T(1), mul_rn(t, t)));
        colpart[j] += t * dm[i];
      }
    }
#pragma unroll
    for (int j = 0; j < kTN; ++j) red[ty][tx * kTN + j] = colpart[j];
    __syncthreads();
    if (ty == 0) {
#pragma unroll
      for (int j = 0; j < kTN; ++j) {
        const int n = n0 + j;
        T s = T(0);
        for (int y = 0; y < 16; ++y) s += red[y][tx * kTN + j];
        if (n < N) ws_u[(long long)bm * H + n] = s;
      }
    }
  }
};

// ------------------------------------------------------------ reductions
// out segment mapping for split-K weight grads: result matrix R[N][Kt] with
// Kt = K1 + K2 (+1 bias column) is written to three destinations.
template <typename T>
__global__ void k_splitk_reduce(const T* __restrict__ ws, int splits, int N, int K1, int K2,
                                int with_bias, T* __restrict__ g1, T* __restrict__ g2,
                                T* __restrict__ gb) {
  const int Kt = K1 + K2 + with_bias;
  const long long total = (long long)N * Kt;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    T s = ws[idx];
    for (int k = 1; k < splits; ++k) s += ws[(long long)k * total + idx];
    const int n = (int)(idx / Kt), k = (int)(idx % Kt);
    if (k < K1)
      g1[(long long)n * K1 + k] = s;
    else if (k < K1 + K2)
      g2[(long long)n * K2 + (k - K1)] = s;
    else
      gb[n] = s;
  }
}

template <typename T>
__global__ void k_rows_reduce(const T* __restrict__ ws, const int* __restrict__ n_rows_dev,
                              int rows_per_item, int cols, T* __restrict__ out) {
  // out[c] = sum over tiles r < ceil(E / rows_per_item) of ws[r][c]
  const int E = *n_rows_dev;
  const int tiles = (E + rows_per_item - 1) / rows_per_item;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    T s = T(0);
    for (int r = 0; r < tiles; ++r) s += ws[(long long)r * cols + c];
    out[c] = s;
  }
}

// f[i] = sum over CSR row i of m_e * dx_e, m_e = sum of the N-tile partials
// (np.add.at over edge_dst in edge order, model.py:382-384).
template <typename T>
__global__ void k_force_combine(const T* __restrict__ m_part, int ntiles,
                                const int* __restrict__ rowptr, const T* __restrict__ dx, int n,
                                T* __restrict__ f, T* __restrict__ m_out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // float64 accumulation (identical ops for T = double; for float32 the
    // cancelling pair sum keeps full precision)
    double fx = 0.0, fy = 0.0, fz = 0.0;
    for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      T m = m_part[(long long)p * ntiles];
      for (int t = 1; t < ntiles; ++t) m += m_part[(long long)p * ntiles + t];
      if (m_out) m_out[p] = m;
      fx = __dadd_rn(fx, __dmul_rn((double)m, (double)dx[3LL * p + 0]));
      fy = __dadd_rn(fy, __dmul_rn((double)m, (double)dx[3LL * p + 1]));
      fz = __dadd_rn(fz, __dmul_rn((double)m, (double)dx[3LL * p + 2]));
    }
    f[3LL * i + 0] = (T)fx;
    f[3LL * i + 1] = (T)fy;
    f[3LL * i + 2] = (T)fz;
  }
}

// dh_final[i] = dh_energy[i] + sum_{CSR row i} dpair + sum_{CSC row i} dpair
// (model.py:533, 546-547, in that order); optional gate -> dz of last layer.
template <typename T>
__global__ void k_node_combine(const T* __restrict__ dh_e, const T* __restrict__ dpair,
                               const int* __restrict__ rowptr, const int* __restrict__ csc_ptr,
                               const int* __restrict__ csc_eid, int n, int H,
                               const T* __restrict__ gate, T* __restrict__ dh_out,
                               T* __restrict__ dz_out) {
  const long long total = (long long)n * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / H), c = (int)(idx % H);
    double acc = (double)dh_e[idx];
    for (int p = rowptr[i]; p < rowptr[i + 1]; ++p)
      acc = __dadd_rn(acc, (double)dpair[(long long)p * H + c]);
    for (int q = csc_ptr[i]; q < csc_ptr[i + 1]; ++q)
      acc = __dadd_rn(acc, (double)dpair[(long long)csc_eid[q] * H + c]);
    if (dh_out) dh_out[idx] = (T)acc;
    if (dz_out) {
      const T g = gate[idx];
      dz_out[idx] = mul_rn((T)acc, sub_rn(T(1), mul_rn(g, g)));
    }
  }
}

// node_e[i] = y[i] . a + c   (model.py:372)
template <typename T>
__global__ void k_node_energy(const T* __restrict__ y, int n, int G, const T* __restrict__ a,
                              const T* __restrict__ c, T* __restrict__ node_e) {
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += gridDim.x * (blockDim.x >> 5)) {
    T s = T(0);
    for (int g = lane; g < G; g += 32) s += y[(long long)i * G + g] * a[g];
    s = warp_sum(s);
    if (lane == 0) node_e[i] = s + c[0];
  }
}

// e_pred[b] = add.reduceat(node_e, offsets) (model.py:373): x0 + pairwise(x1..)
template <typename T>
__global__ void k_graph_pool(const T* __restrict__ node_e, const int* __restrict__ off,
                             int n_graphs, T* __restrict__ e_pred) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n_graphs; b += gridDim.x * blockDim.x) {
    const int lo = off[b], hi = off[b + 1];
    auto get = [&](long long i) -> T { return node_e[i]; };
    e_pred[b] = hi > lo ? add_rn(node_e[lo], np_pairwise<T>(get, lo + 1, hi - lo - 1)) : T(0);
  }
}

// L1 MTL loss + backward seeds (model.py:437-462, 510-516), one block.
template <typename T>
__global__ void __launch_bounds__(1024)
    k_loss_seeds(const T* __restrict__ e_pred, const T* __restrict__ e_true,
                 const int* __restrict__ n_per, int B, const T* __restrict__ f_pred,
                 const T* __restrict__ f_true, int N, T aE, T aF, T* __restrict__ loss,
                 T* __restrict__ de, T* __restrict__ df, float* __restrict__ contrib) {
  __shared__ T red[32];
  T se = T(0);
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const T r = div_rn(sub_rn(e_pred[b], e_true[b]), (T)n_per[b]);
    se += fabs(r);
    de[b] = div_rn(mul_rn(aE, sign_t(r)), (T)n_per[b] * (T)B);
  }
  T sf = T(0);
  const T inv3n = T(3) * (T)N;
  for (int k = threadIdx.x; k < 3 * N; k += blockDim.x) {
    const T d = sub_rn(f_pred[k], f_true[k]);
    sf += fabs(d);
    df[k] = div_rn(mul_rn(aF, sign_t(d)), inv3n);
  }
  auto block_sum = [&](T v) -> T {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T s = T(0);
    if (threadIdx.x == 0)
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    return s;
  };
  const T tot_e = block_sum(se);
  const T tot_f = block_sum(sf);
  if (threadIdx.x == 0) {
    const T et = B > 0 ? tot_e / (T)B : T(0);
    const T ft = N > 0 ? tot_f / (T)(3LL * N) : T(0);
    const T total = aE * et + aF * ft;
    loss[0] = total;
    loss[1] = et;
    loss[2] = ft;
    if (contrib) {
      contrib[0] = (float)total;
      contrib[1] = 1.0f;
    }
  }
}

// energy-head seed: ds_i = de[g(i)]; dz[i][g] = (ds_i * a[g]) * (1 - y^2)
template <typename T>
__global__ void k_energy_seed(const T* __restrict__ de, const int* __restrict__ gnode, int n,
                              int G, const T* __restrict__ a, const T* __restrict__ y,
                              T* __restrict__ ds, T* __restrict__ dz) {
  const long long total = (long long)n * G;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / G), g = (int)(idx % G);
    const T s = de[gnode[i]];
    if (g == 0) ds[i] = s;
    const T yy = y[idx];
    dz[idx] = mul_rn(mul_rn(s, a[g]), sub_rn(T(1), mul_rn(yy, yy)));
  }
}

// embedding gradient (model.py:564): per (node chunk, 64-column block) a CTA
// accumulates rows by element sequentially, then partials are summed over
// chunks in order.  Absent elements stay exactly 0.
constexpr int kEmbCols = 64;
template <typename T>
__global__ void k_emb_partial(const int* __restrict__ z, int n, const T* __restrict__ dh, int H,
                              int chunk, T* __restrict__ ws, unsigned char* __restrict__ present) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* acc = reinterpret_cast<T*>(smem_raw);                       // [118][kEmbCols]
  unsigned char* seen = smem_raw + sizeof(T) * 118 * kEmbCols;   // [118]
  const int ch = blockIdx.x, cb = blockIdx.y;
  const int c = cb * kEmbCols + threadIdx.x;
  for (int k = threadIdx.x; k < 118 * kEmbCols; k += blockDim.x) acc[k] = T(0);
  for (int k = threadIdx.x; k < 118; k += blockDim.x) seen[k] = 0;
  __syncthreads();
  const int lo = ch * chunk, hi = min(n, lo + chunk);
  for (int i = lo; i < hi; ++i) {
    const int e = z[i] - 1;
    if (c < H) acc[e * kEmbCols + threadIdx.x] = add_rn(acc[e * kEmbCols + threadIdx.x], dh[(long long)i * H + c]);
    if (threadIdx.x == 0) seen[e] = 1;
  }
  __syncthreads();
  for (int e = 0; e < 118; ++e) {
    if (!seen[e]) continue;
    if (c < H) ws[((long long)ch * 118 + e) * H + c] = acc[e * kEmbCols + threadIdx.x];
  }
  if (cb == 0)
    for (int e = threadIdx.x; e < 118; e += blockDim.x) present[ch * 118 + e] = seen[e];
}

template <typename T>
__global__ void k_emb_reduce(const T* __restrict__ ws, const unsigned char* __restrict__ present,
                             int n_chunks, int H, T* __restrict__ grad) {
  const long long total = 118LL * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(idx / H), c = (int)(idx % H);
    T s = T(0);
    bool any = false;
    for (int ch = 0; ch < n_chunks; ++ch) {
      if (!present[ch * 118 + e]) continue;
      const T v = ws[((long long)ch * 118 + e) * H + c];
      s = any ? add_rn(s, v) : add_rn(T(0), v);
      any = true;
    }
    grad[idx] = s;
  }
}

// ------------------------------------------------------------ typed drivers
template <typename T>
cudaError_t linear_fwd_t(const T* X1, int ld1, int K1, const T* X2, int ld2, int K2, const T* W1,
                         int ldw1, const T* W2, int ldw2, const T* bias, int M, const int* M_dev,
                         int N, int act, T* Y, int ldy, cudaStream_t s) {
  Rows2Ld<T> a{X1, ld1, K1, X2, ld2, K2};
  Rows2Ld<T> b{W1, ldw1, K1, W2, ldw2, K2};
  EpiBiasAct<T> epi{Y, ldy, bias, act};
  return launch_simt_gemm<T>(M, M_dev, N, K1 + K2, nullptr, 1, a, b, epi, s);
}

template <typename T>
cudaError_t linear_bwd_data_t(const T* dY, int ldd, int M, const int* M_dev, int N, const T* W1,
                              int ldw1, int K1, const T* W2, int ldw2, int K2, T* o1, int ldo1,
                              T* o2, int ldo2, const T* gate, int ldg, cudaStream_t s) {
  RowsLd<T> a{dY, ldd};
  Cols2Ld<T> b{W1, ldw1, K1, W2, ldw2, K2};
  EpiSplitCols<T> epi{o1, ldo1, K1, o2, ldo2, gate, ldg};
  return launch_simt_gemm<T>(M, M_dev, K1 + K2, N, nullptr, 1, a, b, epi, s);
}

template <typename T>
size_t linear_bwd_weight_ws(int M, int N, int K1, int K2, int with_bias) {
  const int Kt = K1 + K2 + with_bias;
  const int splits = choose_splits(N, Kt, M);
  return sizeof(T) * (size_t)splits * N * Kt;
}

template <typename T>
cudaError_t linear_bwd_weight_t(const T* dY, int ldd, int M, const int* M_dev, int N, const T* X1,
                                int ld1, int K1, const T* X2, int ld2, int K2, int with_bias,
                                T* g1, T* g2, T* gb, T* ws, cudaStream_t s) {
  const int Kt = K1 + K2 + with_bias;
  const int splits = choose_splits(N, Kt, M);
  ColsLd<T> a{dY, ldd};
  Cols2Ld<T> b{X1, ld1, K1, X2, ld2, K2};
  EpiPartial<T> epi{ws, (long long)N * Kt};
  // rows = output features N, cols = Kt, reduction over the M batch rows
  cudaError_t e = launch_simt_gemm<T>(N, nullptr, Kt, M, M_dev, splits, a, b, epi, s);
  if (e != cudaSuccess) return e;
  int k_chunk = ceil_div(ceil_div(M > 0 ? M : 1, splits), kBK) * kBK;
  int real_splits = ceil_div(M > 0 ? M : 1, k_chunk);
  k_splitk_reduce<T><<<grid_1d((long long)N * Kt), 256, 0, s>>>(ws, real_splits, N, K1, K2,
                                                                 with_bias, g1, g2, gb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t force_fwd_t(const T* h, int H, int n, const int* rowptr, const int* col_src,
                        const int* edge_dst, const T* dx, int e_cap, const T* V, const T* c,
                        const T* u, T* m_part, T* f, T* m_out, cudaStream_t s) {
  const int ntiles = ceil_div(H, kBN);
  PairLd<T> a{h, H, edge_dst, col_src};
  RowsLd<T> b{V, H};
  EpiForceFwd<T> epi{c, u, m_part, ntiles};
  cudaError_t e = launch_simt_gemm<T>(e_cap, rowptr + n, H, H, nullptr, 1, a, b, epi, s);
  if (e != cudaSuccess) return e;
  k_force_combine<T><<<grid_1d(n), 256, 0, s>>>(m_part, ntiles, rowptr, dx, n, f, m_out);
  return cudaGetLastError();
}

template <typename T>
size_t force_bwd_ws(int H, int e_cap) {
  // dpre (E x H) + dpair (E x H) + u partials + split-K partials of [V | c]
  const int splits = choose_splits(H, H + 1, e_cap);
  return sizeof(T) * ((size_t)e_cap * H * 2 + (size_t)(ceil_div(e_cap, kBM) + 1) * H +
                      (size_t)splits * H * (H + 1)) + 1024;
}

template <typename T>
cudaError_t force_bwd_t(const T* h, int H, int n, const int* rowptr, const int* col_src,
                        const int* edge_dst, const T* dx, int e_cap, const int* csc_ptr,
                        const int* csc_eid, const T* V, const T* c, const T* u, const T* df,
                        const T* dh_e, T* gV, T* gc, T* gu, T* dh_out, T* dz_out, void* ws,
                        cudaStream_t s) {
  const int* E_dev = rowptr + n;
  T* dpre = (T*)ws;
  T* dpair = dpre + (size_t)e_cap * H;
  T* wsu = dpair + (size_t)e_cap * H;
  T* wsk = wsu + (size_t)(ceil_div(e_cap, kBM) + 1) * H;
  cudaError_t e;
  {  // recompute t, produce dpre and grad_u partials (model.py:537-542)
    PairLd<T> a{h, H, edge_dst, col_src};
    RowsLd<T> b{V, H};
    EpiForceBwd<T> epi{c, u, df, edge_dst, dx, dpre, H, wsu};
    e = launch_simt_gemm<T>(e_cap, E_dev, H, H, nullptr, 1, a, b, epi, s);
    if (e != cudaSuccess) return e;
    k_rows_reduce<T><<<grid_1d(H), 256, 0, s>>>(wsu, E_dev, kBM, H, gu);
  }
  {  // [grad_V | grad_c] = dpre^T [pair | 1]   (model.py:543-544)
    const int splits = choose_splits(H, H + 1, e_cap);
    ColsLd<T> a{dpre, H};
    PairColsLd<T> b{h, H, edge_dst, col_src};
    EpiPartial<T> epi{wsk, (long long)H * (H + 1)};
    e = launch_simt_gemm<T>(H, nullptr, H + 1, e_cap, E_dev, splits, a, b, epi, s);
    if (e != cudaSuccess) return e;
    int k_chunk = ceil_div(ceil_div(e_cap > 0 ? e_cap : 1, splits), kBK) * kBK;
    int real = ceil_div(e_cap > 0 ? e_cap : 1, k_chunk);
    k_splitk_reduce<T><<<grid_1d((long long)H * (H + 1)), 256, 0, s>>>(wsk, real, H, H, 0, 1, gV,
                                                                         nullptr, gc);
  }
  {  // dpair = dpre V  (model.py:545)
    RowsLd<T> a{dpre, H};
    ColsLd<T> b{V, H};
    EpiSplitCols<T> epi{dpair, H, H, nullptr, 0, nullptr, 0};
    e = launch_simt_gemm<T>(e_cap, E_dev, H, H, nullptr, 1, a, b, epi, s);
    if (e != cudaSuccess) return e;
  }
  k_node_combine<T><<<grid_1d((long long)n * H), 256, 0, s>>>(dh_e, dpair, rowptr, csc_ptr, csc_eid,
                                                              n, H, dz_out ? h : nullptr, dh_out,
                                                              dz_out);
  return cudaGetLastError();
}

template <typename T>
cudaError_t embedding_grad_t(const int* z, int n_nodes, const T* dh, int H, int chunk, T* grad,
                             void* workspace, cudaStream_t s) {
  if (chunk <= 0) chunk = n_nodes > 0 ? n_nodes : 1;
  const int nch = ceil_div(n_nodes > 0 ? n_nodes : 1, chunk);
  unsigned char* present =
      (unsigned char*)workspace + ((sizeof(T) * (size_t)nch * 118 * H + 255) & ~(size_t)255);
  const size_t smem = sizeof(T) * 118 * kEmbCols + 128;
  cudaError_t e = cudaFuncSetAttribute(k_emb_partial<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (n_nodes > 0) {
    dim3 grid(nch, ceil_div(H, kEmbCols));
    k_emb_partial<T><<<grid, kEmbCols, smem, s>>>(z, n_nodes, dh, H, chunk, (T*)workspace, present);
  }
  k_emb_reduce<T><<<grid_1d(118LL * H), 256, 0, s>>>((const T*)workspace, present,
                                                      n_nodes > 0 ? nch : 0, H, grad);
  return cudaGetLastError();
}

}  // namespace gfm

using namespace gfm;

#define GFM_DISPATCH(dtype, NAME, ...)                                     \
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

int gfm_linear_fwd(const void* X1, int ld1, int K1, const void* X2, int ld2, int K2,
                   const void* W1, int ldw1, const void* W2, int ldw2, const void* bias, int M,
                   const int* M_dev, int N, int act, void* Y, int ldy, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_linear_fwd",
               linear_fwd_t<T>((const T*)X1, ld1, K1, (const T*)X2, ld2, K2, (const T*)W1, ldw1,
                               (const T*)W2, ldw2, (const T*)bias, M, M_dev, N, act, (T*)Y, ldy,
                               (cudaStream_t)stream))
}

int gfm_linear_bwd_data(const void* dY, int ldd, int M, const int* M_dev, int N, const void* W1,
                        int ldw1, int K1, const void* W2, int ldw2, int K2, void* out1, int ldo1,
                        void* out2, int ldo2, const void* gate, int ldg, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_linear_bwd_data",
               linear_bwd_data_t<T>((const T*)dY, ldd, M, M_dev, N, (const T*)W1, ldw1, K1,
                                    (const T*)W2, ldw2, K2, (T*)out1, ldo1, (T*)out2, ldo2,
                                    (const T*)gate, ldg, (cudaStream_t)stream))
}

size_t gfm_linear_bwd_weight_workspace_bytes(int M, int N, int K1, int K2, int with_bias, int dtype) {
  return dtype == GFM_F64 ? linear_bwd_weight_ws<double>(M, N, K1, K2, with_bias)
                          : linear_bwd_weight_ws<float>(M, N, K1, K2, with_bias);
}

int gfm_linear_bwd_weight(const void* dY, int ldd, int M, const int* M_dev, int N, const void* X1,
                          int ld1, int K1, const void* X2, int ld2, int K2, int with_bias,
                          void* g1, void* g2, void* gb, void* workspace, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_linear_bwd_weight",
               linear_bwd_weight_t<T>((const T*)dY, ldd, M, M_dev, N, (const T*)X1, ld1, K1,
                                      (const T*)X2, ld2, K2, with_bias, (T*)g1, (T*)g2, (T*)gb,
                                      (T*)workspace, (cudaStream_t)stream))
}

size_t gfm_force_fwd_workspace_bytes(int H, int e_cap, int dtype) {
  const size_t esz = dtype == GFM_F64 ? 8 : 4;
  return esz * (size_t)(e_cap > 0 ? e_cap : 1) * ceil_div(H, kBN) + 256;
}

int gfm_force_fwd(const void* h, int H, int n_nodes, const int* rowptr, const int* col_src,
                  const int* edge_dst, const void* edge_dx, int e_cap, const void* V,
                  const void* c, const void* u, void* f_pred, void* m_out, void* workspace,
                  int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_force_fwd",
               force_fwd_t<T>((const T*)h, H, n_nodes, rowptr, col_src, edge_dst,
                              (const T*)edge_dx, e_cap, (const T*)V, (const T*)c, (const T*)u,
                              (T*)workspace, (T*)f_pred, (T*)m_out, (cudaStream_t)stream))
}

size_t gfm_force_bwd_workspace_bytes(int H, int e_cap, int dtype) {
  return dtype == GFM_F64 ? force_bwd_ws<double>(H, e_cap) : force_bwd_ws<float>(H, e_cap);
}

int gfm_force_bwd(const void* h, int H, int n_nodes, const int* rowptr, const int* col_src,
                  const int* edge_dst, const void* edge_dx, int e_cap, const int* csc_ptr,
                  const int* csc_eid, const void* V, const void* c, const void* u,
                  const void* df, const void* dh_energy, void* grad_v, void* grad_c, void* grad_u,
                  void* dh_out, void* dz_out, void* workspace, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_force_bwd",
               force_bwd_t<T>((const T*)h, H, n_nodes, rowptr, col_src, edge_dst,
                              (const T*)edge_dx, e_cap, csc_ptr, csc_eid, (const T*)V,
                              (const T*)c, (const T*)u, (const T*)df, (const T*)dh_energy,
                              (T*)grad_v, (T*)grad_c, (T*)grad_u, (T*)dh_out, (T*)dz_out,
                              workspace, (cudaStream_t)stream))
}

int gfm_energy_readout(const void* y, int n_nodes, int G, const void* a, const void* c,
                       const int* node_offsets, int n_graphs, void* node_e, void* e_pred,
                       int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  GFM_DISPATCH(dtype, "gfm_energy_readout",
               (k_node_energy<T><<<grid_1d((long long)n_nodes * 32), 256, 0, s>>>(
                    (const T*)y, n_nodes, G, (const T*)a, (const T*)c, (T*)node_e),
                k_graph_pool<T><<<grid_1d(n_graphs), 256, 0, s>>>((const T*)node_e, node_offsets,
                                                                 n_graphs, (T*)e_pred),
                cudaGetLastError()))
}

int gfm_loss_seeds(const void* e_pred, const void* e_true, const int* n_per, int n_graphs,
                   const void* f_pred, const void* f_true, int n_nodes, double alpha_e,
                   double alpha_f, void* loss, void* de, void* df, float* contrib, int dtype,
                   void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  GFM_DISPATCH(dtype, "gfm_loss_seeds",
               (k_loss_seeds<T><<<1, 1024, 0, s>>>((const T*)e_pred, (const T*)e_true, n_per,
                                                   n_graphs, (const T*)f_pred, (const T*)f_true,
                                                   n_nodes, (T)alpha_e, (T)alpha_f, (T*)loss,
                                                   (T*)de, (T*)df, contrib),
                cudaGetLastError()))
}

int gfm_energy_seed(const void* de, const int* gnode, int n_nodes, int G, const void* a,
                    const void* y, void* ds, void* dz, int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  GFM_DISPATCH(dtype, "gfm_energy_seed",
               (k_energy_seed<T><<<grid_1d((long long)n_nodes * G), 256, 0, s>>>(
                    (const T*)de, gnode, n_nodes, G, (const T*)a, (const T*)y, (T*)ds, (T*)dz),
                cudaGetLastError()))
}

size_t gfm_embedding_grad_workspace_bytes(int n_nodes, int H, int chunk, int dtype) {
  const size_t esz = dtype == GFM_F64 ? 8 : 4;
  const int nch = ceil_div(n_nodes > 0 ? n_nodes : 1, chunk);
  return esz * (size_t)nch * 118 * H + (size_t)nch * 118 + 512;
}

int gfm_embedding_grad(const int* z, int n_nodes, const void* dh, int H, int chunk, void* grad,
                       void* workspace, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_embedding_grad",
               embedding_grad_t<T>(z, n_nodes, (const T*)dh, H, chunk, (T*)grad, workspace,
                                   (cudaStream_t)stream))
}

}  // extern "C"
