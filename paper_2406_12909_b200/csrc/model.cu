// Dense model pieces: node update / head linear layers (forward, data-grad,
// deterministic split-K weight-grad) on the tcgen05 engine (float32) or the
// SIMT engine (float64), the node-factored force head drivers (force.cu has
// the edge kernels), energy readout + graph pooling, the L1 MTL loss with its
// seeds, and the embedding gradient.
//
// Reference: forward_batch (model.py:344-400), mtl_loss (model.py:437-462),
// loss_and_grad (model.py:483-565).
#include <algorithm>
#include <type_traits>

#include "gemm_simt.cuh"
#include "tc_gemm.cuh"

namespace gfm {

static inline int grid_1d(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

// ------------------------------------------------------------ reductions
// out segment mapping for split-K weight grads: result matrix R[N][Kt] with
// Kt = K1 + K2 (+1 bias column) is written to three destinations.
// Split-K reduction: partials ws[split][R][C] (R x C = N x Kt, or Kt x N when
// trans) summed in split order in fp64.  A block owns a 32 x 32 tile; each
// thread keeps 4 independent sums (rows ty, ty + 8, ...) so 4 x unroll loads
// are in flight, then the tile goes out through smem so the [N][K] gradient
// rows are written coalesced in both layouts.
template <typename T>
__global__ void __launch_bounds__(256)
    k_splitk_reduce(const T* __restrict__ ws, int splits, int N, int K1, int K2, int with_bias,
                    T* __restrict__ g1, T* __restrict__ g2, T* __restrict__ gb, int trans) {
  pdl_entry();
  __shared__ T tile[32][33];
  const int Kt = K1 + K2 + with_bias;
  const int R = trans ? Kt : N, C = trans ? N : Kt;
  const long long total = (long long)R * C;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int c = c0 + tx;
#pragma unroll 4
  for (int sp = 0; sp < splits; ++sp) {
    const T* w = ws + (long long)sp * total;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ty + 8 * j;
      if (r < R && c < C) acc[j] += (double)w[(long long)r * C + c];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) tile[ty + 8 * j][tx] = (T)acc[j];
  __syncthreads();
  // write: element (n, k) of the [N][Kt] gradient; threads walk k fastest
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int n, k;
    T v;
    if (trans) {  // tile rows = k (r0..), cols = n (c0..)
      n = c0 + ty + 8 * j;
      k = r0 + tx;
      v = tile[tx][ty + 8 * j];
    } else {      // tile rows = n, cols = k
      n = r0 + ty + 8 * j;
      k = c0 + tx;
      v = tile[ty + 8 * j][tx];
    }
    if (n >= N || k >= Kt) continue;
    if (k < K1)
      g1[(long long)n * K1 + k] = v;
    else if (k < K1 + K2)
      g2[(long long)n * K2 + (k - K1)] = v;
    else
      gb[n] = v;
  }
}

// Small outputs: block = 32 x 8 threads, x over 32 consecutive partial
// elements, y over split groups (split = y, y + 8, ...); the 8 group sums are
// combined in order in smem -- fixed order, 8x the parallelism of a serial
// walk when there are too few 32 x 32 tiles to fill the GPU.
template <typename T>
__global__ void __launch_bounds__(256)
    k_splitk_reduce_narrow(const T* __restrict__ ws, int splits, int N, int K1, int K2,
                           int with_bias, T* __restrict__ g1, T* __restrict__ g2,
                           T* __restrict__ gb, int trans) {
  pdl_entry();
  __shared__ double red[8][33];
  const int Kt = K1 + K2 + with_bias;
  const long long total = (long long)N * Kt;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (long long base = (long long)blockIdx.x * 32; base < total; base += (long long)gridDim.x * 32) {
    const long long idx = base + tx;
    double acc = 0.0;
    if (idx < total) {
#pragma unroll 8  // loads in flight; adds in split order
      for (int k = ty; k < splits; k += 8) acc += (double)ws[(long long)k * total + idx];
    }
    red[ty][tx] = acc;
    __syncthreads();
    double a = 0.0;
    if (ty == 0)
      for (int q = 0; q < 8; ++q) a += red[q][tx];
    __syncthreads();
    if (ty != 0 || idx >= total) continue;
    const T v = (T)a;
    // partials are [N][Kt] (trans = 0) or [Kt][N] (trans = 1); idx walks them
    const int n = trans ? (int)(idx % N) : (int)(idx / Kt);
    const int k = trans ? (int)(idx / N) : (int)(idx % Kt);
    if (k < K1)
      g1[(long long)n * K1 + k] = v;
    else if (k < K1 + K2)
      g2[(long long)n * K2 + (k - K1)] = v;
    else
      gb[n] = v;
  }
}

template <typename T>
void splitk_reduce(const T* ws, int splits, int N, int K1, int K2, int with_bias, T* g1, T* g2,
                   T* gb, int trans, cudaStream_t s) {
  const int Kt = K1 + K2 + with_bias;
  const int R = trans ? Kt : N, C = trans ? N : Kt;
  const long long tiles = (long long)ceil_div(C, 32) * ceil_div(R, 32);
  if (tiles >= 2 * 148)
    launch_k(k_splitk_reduce<T>, dim3(ceil_div(C, 32), ceil_div(R, 32)), 256, 0, s,
        ws, splits, N, K1, K2, with_bias, g1, g2, gb, trans);
  else
    launch_k(k_splitk_reduce_narrow<T>, grid_1d((long long)N * Kt, 32), 256, 0, s,
        ws, splits, N, K1, K2, with_bias, g1, g2, gb, trans);
}

// node_e[i] = y[i] . a + c   (model.py:372)
template <typename T>
__global__ void k_node_energy(const T* __restrict__ y, int n, int G, const T* __restrict__ a,
                              const T* __restrict__ c, T* __restrict__ node_e) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += gridDim.x * (blockDim.x >> 5)) {
    T s = T(0);
    for (int g = lane; g < G; g += 32) s += y[(long long)i * G + g] * a[g];
    s = warp_sum(s);
    if (lane == 0) node_e[i] = s + c[0];
  }
}

// float32, G % 4 == 0, G/4 a power of two <= 32: LPN = G/4 lanes per node,
// one float4 of y and a per lane, group shuffle reduction (32/LPN nodes per
// warp, every load a full 16 B)
__global__ void k_node_energy4(const float* __restrict__ y, int n, int G, int lpn,
                               const float* __restrict__ a, const float* __restrict__ c,
                               float* __restrict__ node_e) {
  pdl_entry();
  const int lane = threadIdx.x & 31, sub = lane & (lpn - 1);
  const int per_warp = 32 / lpn;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const float4 av = reinterpret_cast<const float4*>(a)[sub];
  const float c0 = c[0];
  // base is warp-uniform, so every lane runs the group shuffles together
  for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * per_warp; base < n;
       base += warps * per_warp) {
    const int i = base + lane / lpn;
    float s = 0.f;
    if (i < n) {
      const float4 yv = reinterpret_cast<const float4*>(y + (long long)i * G)[sub];
      s = yv.x * av.x + yv.y * av.y + yv.z * av.z + yv.w * av.w;
    }
    for (int o = lpn >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (i < n && sub == 0) node_e[i] = s + c0;
  }
}

// e_pred[b] = add.reduceat(node_e, offsets) (model.py:373): x0 + pairwise(x1..)
template <typename T>
__global__ void k_graph_pool(const T* __restrict__ node_e, const int* __restrict__ off,
                             int n_graphs, T* __restrict__ e_pred) {
  pdl_entry();
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n_graphs; b += gridDim.x * blockDim.x) {
    const int lo = off[b], hi = off[b + 1];
    auto get = [&](long long i) -> T { return node_e[i]; };
    e_pred[b] = hi > lo ? add_rn(node_e[lo], np_pairwise<T>(get, lo + 1, hi - lo - 1)) : T(0);
  }
}

// L1 MTL loss + backward seeds (model.py:437-462, 510-516).  Grid-stride
// seeds; per-block float64 partial sums; the last block to finish (ticket
// counter) adds the partials in block order, so the result is deterministic.
constexpr int kLossBlocks = 64;
template <typename T>
__global__ void __launch_bounds__(256)
    k_loss_seeds(const T* __restrict__ e_pred, const T* __restrict__ e_true,
                 const int* __restrict__ n_per, int B_cap, const T* __restrict__ f_pred,
                 const T* __restrict__ f_true, int N_cap, const int* __restrict__ counts, T aE,
                 T aF, T* __restrict__ loss, T* __restrict__ de, T* __restrict__ df,
                 float* __restrict__ contrib, double* __restrict__ partial,
                 unsigned* __restrict__ ticket) {
  pdl_entry();
  __shared__ double red[2][8];
  __shared__ bool last;
  // ragged batches in a fixed-capacity step: the true graph / node counts
  // come from the device ([B, N]); the capacity tail gets zero seeds
  const int B = counts ? counts[0] : B_cap, N = counts ? counts[1] : N_cap;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  double se = 0.0, sf = 0.0;
  for (int b = tid; b < B_cap; b += nth) {
    if (b >= B) {
      de[b] = T(0);
      continue;
    }
    const T r = div_rn(sub_rn(e_pred[b], e_true[b]), (T)n_per[b]);
    se += (double)fabs(r);
    de[b] = div_rn(mul_rn(aE, sign_t(r)), (T)n_per[b] * (T)B);
  }
  // aF * sign(d) / (3N) takes only the values {q, -q, 0}: q = aF / (3N)
  const T q = div_rn(aF, T(3) * (T)N);
#pragma unroll 4
  for (int k = tid; k < 3 * N; k += nth) {
    const T d = sub_rn(f_pred[k], f_true[k]);
    sf += (double)fabs(d);
    df[k] = d > T(0) ? q : (d < T(0) ? -q : T(0));
  }
  for (int k = 3 * N + tid; k < 3 * N_cap; k += nth) df[k] = T(0);
  se = warp_sum(se);
  sf = warp_sum(sf);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = se;
    red[1][wid] = sf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double tot_e = 0.0, tot_f = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) {
      tot_e += ((volatile double*)partial)[2 * k];
      tot_f += ((volatile double*)partial)[2 * k + 1];
    }
    *ticket = 0u;  // ready for the next launch
    const T et = B > 0 ? (T)(tot_e / (double)B) : T(0);
    const T ft = N > 0 ? (T)(tot_f / (3.0 * (double)N)) : T(0);
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
                              T* __restrict__ ds, int ld_ds, T* __restrict__ dz) {
  pdl_entry();
  // 2D: y over nodes, x over the G columns (no 64-bit divides)
  for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < n; i += gridDim.y * blockDim.y) {
    const int gi = gnode[i];  // -1: capacity-tail node of a ragged batch
    const T s = gi >= 0 ? de[gi] : T(0);
    if (threadIdx.x < ld_ds) ds[(long long)i * ld_ds + threadIdx.x] = threadIdx.x == 0 ? s : T(0);
    const long long row = (long long)i * G;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      const T yy = y[row + g];
      dz[row + g] = mul_rn(mul_rn(s, a[g]), sub_rn(T(1), mul_rn(yy, yy)));
    }
  }
}

// float32, G % 4 == 0: one float4 of (y, dz) per thread, same per-element
// rounding as k_energy_seed (bit-identical output)
__global__ void k_energy_seed4(const float* __restrict__ de, const int* __restrict__ gnode, int n,
                               int G4, const float* __restrict__ a, const float* __restrict__ y,
                               float* __restrict__ ds, int ld_ds, float* __restrict__ dz) {
  pdl_entry();
  const long long total = (long long)n * G4;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / G4), q = (int)(t - (long long)i * G4);
    const int gi = gnode[i];
    const float s = gi >= 0 ? de[gi] : 0.f;
    if (q == 0)
      for (int k = 0; k < ld_ds; ++k) ds[(long long)i * ld_ds + k] = k == 0 ? s : 0.f;
    const float4 yv = reinterpret_cast<const float4*>(y)[t];
    const float4 av = reinterpret_cast<const float4*>(a)[q];
    float4 o;
    o.x = mul_rn(mul_rn(s, av.x), sub_rn(1.f, mul_rn(yv.x, yv.x)));
    o.y = mul_rn(mul_rn(s, av.y), sub_rn(1.f, mul_rn(yv.y, yv.y)));
    o.z = mul_rn(mul_rn(s, av.z), sub_rn(1.f, mul_rn(yv.z, yv.z)));
    o.w = mul_rn(mul_rn(s, av.w), sub_rn(1.f, mul_rn(yv.w, yv.w)));
    reinterpret_cast<float4*>(dz)[t] = o;
  }
}

// embedding gradient (model.py:564): grad_emb = onehot(z - 1)^T dh, i.e. a
// weight-gradient GEMM whose A operand is generated on the fly; absent
// elements are sums of exact zeros (stay 0.0).
template <typename T>
struct OneHotLd {  // A(row = element, k = node) = [z[node] - 1 == row]
  static constexpr bool kContigRow = false;
  const int* z;
  __device__ T operator()(int r, int k) const { return z[k] - 1 == r ? T(1) : T(0); }
  bool vec_ok(int K) const { return sizeof(T) == 4 && al16(z) && K % 4 == 0; }
  __device__ int src4(int r, int k, int, const float**, float4* imm) const {
    const int4 q = __ldg(reinterpret_cast<const int4*>(z + k));
    *imm = make_float4(q.x - 1 == r ? 1.f : 0.f, q.y - 1 == r ? 1.f : 0.f,
                       q.z - 1 == r ? 1.f : 0.f, q.w - 1 == r ? 1.f : 0.f);
    return -1;
  }
};

// ------------------------------------------------------------ typed drivers
// float32 GEMMs run on the tcgen05 tensor cores (3xTF32 by default,
// gemm_mode() == GFM_GEMM_TC3); float64 and GFM_GEMM_SIMT use the SIMT engine.
template <typename T>
inline bool use_tc() {
  return std::is_same<T, float>::value && gemm_mode() != GFM_GEMM_SIMT;
}
inline int tc_split3() { return gemm_mode() == GFM_GEMM_TC1 ? 0 : 1; }
// weight-gradient GEMMs (dW = X^T dY, embedding one-hot^T dh): 1xTF32 in MIXED
inline int tc_split3_wgrad() {
  return gemm_mode() == GFM_GEMM_TC1 || gemm_mode() == GFM_GEMM_MIXED ? 0 : 1;
}

template <typename T>
cudaError_t linear_fwd_t(const T* X1, int ld1, int K1, const T* X2, int ld2, int K2, const T* W1,
                         int ldw1, const T* W2, int ldw2, const T* bias, int M, const int* M_dev,
                         int N, int act, T* Y, int ldy, cudaStream_t s) {
  Rows2Ld<T> a{X1, ld1, K1, X2, ld2, K2};
  Rows2Ld<T> b{W1, ldw1, K1, W2, ldw2, K2};
  if constexpr (std::is_same<T, float>::value) {
    if (use_tc<T>()) {
      tc::TcEpiBiasAct epi{Y, ldy, bias, act};
      return tc::launch(M, M_dev, N, K1 + K2, nullptr, 1, tc_split3(), a, b, epi, s);
    }
  }
  EpiBiasAct<T> epi{Y, ldy, bias, act};
  return launch_simt_gemm<T>(M, M_dev, N, K1 + K2, nullptr, 1, a, b, epi, s);
}

template <typename T>
cudaError_t linear_bwd_data_t(const T* dY, int ldd, int M, const int* M_dev, int N, const T* W1,
                              int ldw1, int K1, const T* W2, int ldw2, int K2, T* o1, int ldo1,
                              T* o2, int ldo2, const T* gate, int ldg, cudaStream_t s,
                              const T* add = nullptr) {
  RowsLd<T> a{dY, ldd};
  Cols2Ld<T> b{W1, ldw1, K1, W2, ldw2, K2};
  if constexpr (std::is_same<T, float>::value) {
    if (use_tc<T>()) {
      tc::TcEpiSplitCols epi{o1, ldo1, K1, o2, ldo2, gate, ldg, add};
      return tc::launch(M, M_dev, K1 + K2, N, nullptr, 1, tc_split3(), a, b, epi, s);
    }
  }
  EpiSplitCols<T> epi{o1, ldo1, K1, o2, ldo2, gate, ldg, add};
  return launch_simt_gemm<T>(M, M_dev, K1 + K2, N, nullptr, 1, a, b, epi, s);
}

// U [rows][4H] (part-major columns p*H + c) -> Up [rows][4H] channel-major
// (4c + p): the B operand of the fused backward-data + aggregation prep
__global__ void k_permute_parts(const float* __restrict__ U, int rows, int H, int ldu,
                                float* __restrict__ Up) {
  pdl_entry();
  const long long total = (long long)rows * 4 * H;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / (4 * H)), j = (int)(idx % (4 * H));
    const int c = j >> 2, p = j & 3;
    Up[idx] = U[(long long)r * ldu + p * H + c];
  }
}

template <typename T>
int wgrad_splits(int M, int N, int Kt) {
  return use_tc<T>() ? tc::splits_for(N, Kt, M) : choose_splits(N, Kt, M);
}

template <typename T>
size_t linear_bwd_weight_ws(int M, int N, int K1, int K2, int with_bias) {
  const int Kt = K1 + K2 + with_bias;
  const int splits = std::max(choose_splits(N, Kt, M), tc::splits_for(Kt, N, M));
  // split-K partials + the [M][4] ones operand of the bias row
  return sizeof(T) * ((size_t)splits * N * Kt + 64 + 4 * (size_t)(M > 0 ? M : 1) + 64);
}

template <typename T>
__global__ void k_fill_ones(T* __restrict__ ones, int m) {  // ones[i][0] = 1, [1..3] = 0
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 4 * m; i += gridDim.x * blockDim.x)
    ones[i] = (i & 3) == 0 ? T(1) : T(0);
}

template <typename T>
cudaError_t colsum(const T* X, int n, int H, T* out, T* part, cudaStream_t s);  // force.cu
template <typename T>
cudaError_t colsum2(const T* X1, const T* X2, int n, int H, T* out1, T* out2, T* part,
                    cudaStream_t s);  // force.cu

// actual number of K splits after rounding the chunk to the engine's K step
inline int real_splits(int K, int splits, int kstep) {
  int k_chunk = ceil_div(ceil_div(K > 0 ? K : 1, splits), kstep) * kstep;
  return ceil_div(K > 0 ? K : 1, k_chunk);
}

template <typename T>
cudaError_t linear_bwd_weight_t(const T* dY, int ldd, int M, const int* M_dev, int N, const T* X1,
                                int ld1, int K1, const T* X2, int ld2, int K2, int with_bias,
                                T* g1, T* g2, T* gb, T* ws, cudaStream_t s,
                                gfm_reduce_job* defer = nullptr) {
  // with_bias == 2: the workspace already holds the ones operand (same M)
  const bool ones_ready = with_bias == 2;
  with_bias = with_bias ? 1 : 0;
  const int Kt = K1 + K2 + with_bias;
  cudaError_t e;
  int real, trans = 0;
  if constexpr (std::is_same<T, float>::value) {
    if (use_tc<T>()) {
      // tensor cores: C^T[Kt][N] = [X | 1]^T dY -- the wide operand X is read
      // once (one column tile), no half-empty 128-row tiles for N = H
      // the bias gradient rides in the GEMM as one more A row: a ones vector
      // [M][4] (column 0 = 1) that TMA loads as a third segment
      const int splits = tc::splits_for(Kt, N, M);
      Cols2Ld<T> a{X1, ld1, K1, X2, ld2, K2};
      if (with_bias) {
        T* ones = ws + (((size_t)splits * N * Kt + 63) & ~(size_t)63);
        if (!ones_ready) launch_k(k_fill_ones<T>, grid_1d(4LL * M), 256, 0, s, ones, M);
        a.ones = ones;
      }
      ColsLd<T> b{dY, ldd};
      tc::TcEpiPartial epi{ws, (long long)N * Kt, Kt, N};
      e = tc::launch(Kt, nullptr, N, M, M_dev, splits, tc_split3_wgrad(), a, b, epi, s);
      real = real_splits(M, splits, tc::kBK);
      trans = 1;
      goto reduce;
    }
  }
  {
    // rows = output features N, cols = Kt, reduction over the M batch rows
    const int splits = choose_splits(N, Kt, M);
    ColsLd<T> a{dY, ldd};
    Cols2Ld<T> b{X1, ld1, K1, X2, ld2, K2};
    EpiPartial<T> epi{ws, (long long)N * Kt};
    e = launch_simt_gemm<T>(N, nullptr, Kt, M, M_dev, splits, a, b, epi, s);
    real = real_splits(M, splits, kBK);
  }
reduce:
  if (e != cudaSuccess) return e;
  if (defer) {  // the caller reduces later, batched with other weight gradients
    *defer = gfm_reduce_job{ws, real, N, K1, K2, with_bias, trans, g1, g2, gb};
    return cudaGetLastError();
  }
  splitk_reduce<T>(ws, real, N, K1, K2, with_bias, g1, g2, gb, trans, s);
  return cudaGetLastError();
}

// All deferred split-K reductions of a backward pass in ONE launch: the 32x32
// tiles of every job form one flat grid (job found by prefix over the tile
// counts); each tile is k_splitk_reduce's (fp64 ordered sums, coalesced
// writes) -- deterministic and identical to the per-call reduce.
constexpr int kMaxReduceJobs = 24;
struct ReduceJobs {
  gfm_reduce_job job[kMaxReduceJobs];
  int tile0[kMaxReduceJobs + 1];  // first flat tile of each job
  int ncx[kMaxReduceJobs];        // tiles along C
  int rows[kMaxReduceJobs];       // tile height: 32 (4 sums / thread) or 8 (many splits)
};

template <typename T>
__global__ void __launch_bounds__(256) k_splitk_reduce_batch(const __grid_constant__ ReduceJobs J,
                                                             int n_jobs) {
  pdl_entry();
  __shared__ T tile[32][33];
  int q = 0;
  while (q + 1 < n_jobs && (int)blockIdx.x >= J.tile0[q + 1]) ++q;
  const gfm_reduce_job& jb = J.job[q];
  const int t = blockIdx.x - J.tile0[q];
  const T* ws = (const T*)jb.ws;
  const int N = jb.N, K1 = jb.K1, K2 = jb.K2, trans = jb.trans;
  const int Kt = K1 + K2 + jb.with_bias;
  const int R = trans ? Kt : N, C = trans ? N : Kt;
  const long long total = (long long)R * C;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int th = J.rows[q], nj = th / 8;
  const int r0 = (t / J.ncx[q]) * th, c0 = (t % J.ncx[q]) * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int c = c0 + tx;
  if (nj == 1) {  // one sum per thread, splits unrolled 8 deep (many-split jobs)
    const int r = r0 + ty;
    if (r < R && c < C) {
      const T* w = ws + (long long)r * C + c;
#pragma unroll 8
      for (int sp = 0; sp < jb.splits; ++sp) acc[0] += (double)w[(long long)sp * total];
    }
  } else {
#pragma unroll 4
    for (int sp = 0; sp < jb.splits; ++sp) {
      const T* w = ws + (long long)sp * total;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + ty + 8 * j;
        if (r < R && c < C) acc[j] += (double)w[(long long)r * C + c];
      }
    }
  }
  for (int j = 0; j < nj; ++j) tile[ty + 8 * j][tx] = (T)acc[j];
  __syncthreads();
  T* g1 = (T*)jb.g1;
  T* g2 = (T*)jb.g2;
  T* gb = (T*)jb.gb;
  // write: element (n, k) of the [N][Kt] gradient; th x 32 tile
  for (int e = threadIdx.x; e < th * 32; e += blockDim.x) {
    int n, k;
    T v;
    if (trans) {  // tile rows = k (r0 ..), cols = n (c0 ..): walk k fastest
      const int kk = e % th, nn = e / th;
      n = c0 + nn;
      k = r0 + kk;
      v = tile[kk][nn];
    } else {
      const int nn = e / 32, kk = e % 32;
      n = r0 + nn;
      k = c0 + kk;
      v = tile[nn][kk];
    }
    if (n >= N || k >= Kt) continue;
    if (k < K1)
      g1[(long long)n * K1 + k] = v;
    else if (k < K1 + K2)
      g2[(long long)n * K2 + (k - K1)] = v;
    else
      gb[n] = v;
  }
}

template <typename T>
cudaError_t splitk_reduce_batch(const gfm_reduce_job* jobs, int n_jobs, cudaStream_t s) {
  for (int base = 0; base < n_jobs; base += kMaxReduceJobs) {
    ReduceJobs J{};
    const int n = std::min(kMaxReduceJobs, n_jobs - base);
    int tiles = 0;
    for (int q = 0; q < n; ++q) {
      const gfm_reduce_job& jb = jobs[base + q];
      J.job[q] = jb;
      const int Kt = jb.K1 + jb.K2 + jb.with_bias;
      const int R = jb.trans ? Kt : jb.N, C = jb.trans ? jb.N : Kt;
      J.tile0[q] = tiles;
      J.ncx[q] = ceil_div(C, 32);
      J.rows[q] = jb.splits > 16 ? 8 : 32;
      tiles += J.ncx[q] * ceil_div(R, J.rows[q]);
    }
    J.tile0[n] = tiles;
    if (tiles > 0) launch_k(k_splitk_reduce_batch<T>, tiles, 256, 0, s, J, n);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t force_fwd_edges(const T* P, int n, int H, const int* rowptr, const int* col_src,
                            const T* dx, const T* c, const T* u, T* f, int flags, cudaStream_t s);
template <typename T>
cudaError_t force_bwd_edges(const T* P, int n, int H, const int* rowptr, const int* col_src,
                            const int* csc_ptr, const int* csc_eid, const int* csc_dst,
                            const T* dx, const T* df, const T* c, const T* u, T* Ddst, T* TU,
                            T* S, int flags, cudaStream_t s);
template <typename T>
cudaError_t colsum(const T* X, int n, int H, T* out, T* part, cudaStream_t s);

template <typename T>
cudaError_t force_fwd_t(const T* h, int H, int n, const int* rowptr, const int* col_src,
                        const T* dx, const T* V, const T* c, const T* u, T* P, T* f, int flags,
                        cudaStream_t s) {
  // P = h V^T  (the pair pre-activation is P[dst] + P[src] + c)
  cudaError_t e = linear_fwd_t<T>(h, H, H, nullptr, 0, 0, V, H, nullptr, 0, nullptr, n, nullptr, H,
                                  0, P, H, s);
  if (e != cudaSuccess) return e;
  return force_fwd_edges<T>(P, n, H, rowptr, col_src, dx, c, u, f, flags, s);
}

template <typename T>
size_t force_bwd_ws(int H, int n) {
  const size_t nh = (size_t)(n > 0 ? n : 1) * H;
  const size_t parts = 2 * (size_t)ceil_div(n > 0 ? n : 1, 128) * H;  // two colsums' partials
  return sizeof(T) * (3 * nh + parts + 64) + linear_bwd_weight_ws<T>(n, H, H, 0, 0) + 4096;
}

template <typename T>
cudaError_t force_bwd_t(const T* h, const T* P, int H, int n, const int* rowptr,
                        const int* col_src, const T* dx, const int* csc_ptr, const int* csc_eid,
                        const int* csc_dst, const T* V, const T* c, const T* u, const T* df,
                        const T* dh_e, T* gV, T* gc, T* gu, T* dz_out, void* ws, int flags,
                        cudaStream_t s, int stage = 7) {
  // stage bit 1: edge passes (S, D_dst, TU left in ws); bit 4: grad_V /
  // grad_c / grad_u from ws; bit 2: dz_out from S in ws -- separable so the
  // caller can overlap dh_energy and run the parameter gradients off the
  // critical path
  const size_t nh = (size_t)(n > 0 ? n : 1) * H;
  T* Ddst = (T*)ws;
  T* TU = Ddst + nh;
  T* S = TU + nh;
  T* part = S + nh;
  T* wws = part + 2 * (size_t)ceil_div(n > 0 ? n : 1, 128) * H + 64;
  wws = (T*)(((uintptr_t)wws + 255) & ~(uintptr_t)255);
  cudaError_t e;
  if (stage & 1) {
    e = force_bwd_edges<T>(P, n, H, rowptr, col_src, csc_ptr, csc_eid, csc_dst, dx, df, c, u,
                           Ddst, TU, S, flags, s);
    if (e != cudaSuccess) return e;
  }
  if (!(stage & 4)) goto finish;
  // grad_V = S^T h   (= sum_e dpre_e pair_e^T, model.py:543)
  e = linear_bwd_weight_t<T>(S, H, n, nullptr, H, h, H, H, nullptr, 0, 0, 0, gV, nullptr, nullptr,
                             wws, s);
  if (e != cudaSuccess) return e;
  // grad_c = colsum(D_dst) (model.py:544), grad_u = colsum(TU) (model.py:540): one launch pair
  if ((e = colsum2<T>(Ddst, TU, n, H, gc, gu, part, s)) != cudaSuccess) return e;
finish:
  if (!(stage & 2)) return cudaGetLastError();
  // dz_last = (dh_energy + S V) * (1 - h^2)   (model.py:545-547, 553)
  return linear_bwd_data_t<T>(S, H, n, nullptr, H, V, H, H, nullptr, 0, 0, dz_out, H, nullptr, 0,
                              h, H, s, dh_e);
}

template <typename T>
cudaError_t embedding_grad_t(const int* z, int n_nodes, const T* dh, int H, T* grad, T* ws,
                             cudaStream_t s) {
  constexpr int E = 118;
  const int splits = wgrad_splits<T>(n_nodes, E, H);
  OneHotLd<T> a{z};
  ColsLd<T> b{dh, H};
  cudaError_t e;
  int real;
  if constexpr (std::is_same<T, float>::value) {
    if (use_tc<T>()) {
      tc::TcEpiPartial epi{ws, (long long)E * H, E, H};
      e = tc::launch(E, nullptr, H, n_nodes, nullptr, splits, tc_split3_wgrad(), a, b, epi, s);
      real = real_splits(n_nodes, splits, tc::kBK);
      goto reduce;
    }
  }
  {
    EpiPartial<T> epi{ws, (long long)E * H};
    e = launch_simt_gemm<T>(E, nullptr, H, n_nodes, nullptr, splits, a, b, epi, s);
    real = real_splits(n_nodes, splits, kBK);
  }
reduce:
  if (e != cudaSuccess) return e;
  splitk_reduce<T>(ws, real, E, H, 0, 0, grad, nullptr, nullptr, 0, s);
  return cudaGetLastError();
}

}  // namespace gfm

using namespace gfm;

#define GFM_TRY_CUDA(expr)                                                 \
  do {                                                                     \
    cudaError_t _e2 = (expr);                                              \
    if (_e2 != cudaSuccess) {                                              \
      set_error("%s: %s", #expr, cudaGetErrorString(_e2));                 \
      return (int)_e2;                                                     \
    }                                                                      \
  } while (0)

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

int gfm_linear_bwd_weight_partials(const void* dY, int ldd, int M, const int* M_dev, int N,
                                   const void* X1, int ld1, int K1, const void* X2, int ld2,
                                   int K2, int with_bias, void* g1, void* g2, void* gb,
                                   void* workspace, gfm_reduce_job* job, int dtype,
                                   void* stream) {
  if (!job) {
    set_error("gfm_linear_bwd_weight_partials: job descriptor is NULL");
    return GFM_EINVAL;
  }
  GFM_DISPATCH(dtype, "gfm_linear_bwd_weight_partials",
               linear_bwd_weight_t<T>((const T*)dY, ldd, M, M_dev, N, (const T*)X1, ld1, K1,
                                      (const T*)X2, ld2, K2, with_bias, (T*)g1, (T*)g2, (T*)gb,
                                      (T*)workspace, (cudaStream_t)stream, job))
}

int gfm_splitk_reduce_batch(const gfm_reduce_job* jobs, int n_jobs, int dtype, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) {
    set_error("gfm_splitk_reduce_batch: bad job list");
    return GFM_EINVAL;
  }
  GFM_DISPATCH(dtype, "gfm_splitk_reduce_batch",
               splitk_reduce_batch<T>(jobs, n_jobs, (cudaStream_t)stream))
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

int gfm_force_fwd(const void* h, int H, int n_nodes, const int* rowptr, const int* col_src,
                  const void* edge_dx, const void* V, const void* c, const void* u, void* P,
                  void* f_pred, int dtype, int flags, void* stream) {
  GFM_DISPATCH(dtype, "gfm_force_fwd",
               force_fwd_t<T>((const T*)h, H, n_nodes, rowptr, col_src, (const T*)edge_dx,
                              (const T*)V, (const T*)c, (const T*)u, (T*)P, (T*)f_pred, flags,
                              (cudaStream_t)stream))
}

size_t gfm_force_bwd_workspace_bytes(int H, int n_nodes, int dtype) {
  return dtype == GFM_F64 ? force_bwd_ws<double>(H, n_nodes) : force_bwd_ws<float>(H, n_nodes);
}

int gfm_force_bwd(const void* h, const void* P, int H, int n_nodes, const int* rowptr,
                  const int* col_src, const void* edge_dx, const int* csc_ptr, const int* csc_eid,
                  const int* csc_dst, const void* V, const void* c, const void* u, const void* df,
                  const void* dh_energy, void* grad_v, void* grad_c, void* grad_u, void* dz_out,
                  void* workspace, int dtype, int flags, void* stream) {
  GFM_DISPATCH(dtype, "gfm_force_bwd",
               force_bwd_t<T>((const T*)h, (const T*)P, H, n_nodes, rowptr, col_src,
                              (const T*)edge_dx, csc_ptr, csc_eid, csc_dst, (const T*)V,
                              (const T*)c, (const T*)u, (const T*)df, (const T*)dh_energy,
                              (T*)grad_v, (T*)grad_c, (T*)grad_u, (T*)dz_out, workspace, flags,
                              (cudaStream_t)stream))
}

size_t gfm_layer_bwd_data_agg_workspace_bytes(int H) {
  return sizeof(float) * (size_t)H * 4 * H + 256;
}

int gfm_layer_bwd_data_agg(const void* dz, int M, int H, const void* W, const void* U,
                           const void* agg, const void* stat_mean, const int* rowptr, void* dh_in,
                           void* G, void* coef, void* dmax, void* workspace, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!use_tc<float>() || H <= 0 || (H % 4) || !G || !coef || !dmax) {
    set_error("gfm_layer_bwd_data_agg: needs the tensor-core engine, float32, H %% 4 == 0");
    return GFM_EINVAL;
  }
  float* Up = (float*)workspace;
  launch_k(k_permute_parts, grid_1d((long long)H * 4 * H), 256, 0, s, (const float*)U, H, H,
           4 * H, Up);
  RowsLd<float> a{(const float*)dz, H};
  Cols2Ld<float> b{(const float*)W, H, H, Up, 4 * H, 4 * H};
  tc::TcEpiAggPrep epi{(float*)dh_in, H, (float*)G, (float*)coef, (float*)dmax,
                       (const float*)agg, (const float*)stat_mean, rowptr};
  cudaError_t e = tc::launch(M, nullptr, 5 * H, H, nullptr, 1, tc_split3(), a, b, epi, s);
  if (e != cudaSuccess) {
    set_error("gfm_layer_bwd_data_agg: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

int gfm_force_bwd_edges(const void* h, const void* P, int H, int n_nodes, const int* rowptr,
                        const int* col_src, const void* edge_dx, const int* csc_ptr,
                        const int* csc_eid, const int* csc_dst, const void* V, const void* c,
                        const void* u, const void* df, void* grad_v, void* grad_c, void* grad_u,
                        void* workspace, int dtype, int flags, void* stream) {
  // grad pointers NULL: edge passes only (then gfm_force_bwd_grads)
  const int stage = grad_v ? 1 | 4 : 1;
  GFM_DISPATCH(dtype, "gfm_force_bwd_edges",
               force_bwd_t<T>((const T*)h, (const T*)P, H, n_nodes, rowptr, col_src,
                              (const T*)edge_dx, csc_ptr, csc_eid, csc_dst, (const T*)V,
                              (const T*)c, (const T*)u, (const T*)df, nullptr, (T*)grad_v,
                              (T*)grad_c, (T*)grad_u, nullptr, workspace, flags,
                              (cudaStream_t)stream, stage))
}

int gfm_force_bwd_grads(const void* h, int H, int n_nodes, void* grad_v, void* grad_c,
                        void* grad_u, void* workspace, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_force_bwd_grads",
               force_bwd_t<T>((const T*)h, nullptr, H, n_nodes, nullptr, nullptr, nullptr,
                              nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                              nullptr, (T*)grad_v, (T*)grad_c, (T*)grad_u, nullptr, workspace, 0,
                              (cudaStream_t)stream, 4))
}

int gfm_force_bwd_finish(const void* h, int H, int n_nodes, const void* V, const void* dh_energy,
                         void* dz_out, void* workspace, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_force_bwd_finish",
               force_bwd_t<T>((const T*)h, nullptr, H, n_nodes, nullptr, nullptr, nullptr,
                              nullptr, nullptr, nullptr, (const T*)V, nullptr, nullptr, nullptr,
                              (const T*)dh_energy, nullptr, nullptr, nullptr, (T*)dz_out,
                              workspace, 0, (cudaStream_t)stream, 2))
}

int gfm_energy_readout(const void* y, int n_nodes, int G, const void* a, const void* c,
                       const int* node_offsets, int n_graphs, void* node_e, void* e_pred,
                       int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int lpn = G / 4;
  if (dtype == GFM_F32 && G % 4 == 0 && lpn <= 32 && (lpn & (lpn - 1)) == 0 && al16(y) &&
      al16(a) && n_nodes > 0) {
    GFM_TRY_CUDA(launch_k(k_node_energy4, grid_1d((long long)n_nodes * lpn), 256, 0, s,
                          (const float*)y, n_nodes, G, lpn, (const float*)a, (const float*)c,
                          (float*)node_e));
    GFM_TRY_CUDA(launch_k(k_graph_pool<float>, grid_1d(n_graphs, 32), 32, 0, s,
                          (const float*)node_e, node_offsets, n_graphs, (float*)e_pred));
    GFM_TRY_CUDA(cudaGetLastError());
    return 0;
  }
  GFM_DISPATCH(dtype, "gfm_energy_readout",
               (launch_k(k_node_energy<T>, grid_1d((long long)n_nodes * 32), 256, 0, s,
                    (const T*)y, n_nodes, G, (const T*)a, (const T*)c, (T*)node_e),
                launch_k(k_graph_pool<T>, grid_1d(n_graphs, 32), 32, 0, s, (const T*)node_e, node_offsets,
                                                                 n_graphs, (T*)e_pred),
                cudaGetLastError()))
}

size_t gfm_loss_workspace_bytes(void) { return sizeof(double) * 2 * kLossBlocks + 256; }

int gfm_loss_seeds(const void* e_pred, const void* e_true, const int* n_per, int n_graphs,
                   const void* f_pred, const void* f_true, int n_nodes, const int* counts,
                   double alpha_e, double alpha_f, void* loss, void* de, void* df,
                   float* contrib, void* workspace, int dtype, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* partial = (double*)workspace;
  unsigned* ticket = (unsigned*)(partial + 2 * kLossBlocks);
  GFM_DISPATCH(dtype, "gfm_loss_seeds",
               (launch_k(k_loss_seeds<T>, kLossBlocks, 256, 0, s,
                    (const T*)e_pred, (const T*)e_true, n_per, n_graphs, (const T*)f_pred,
                    (const T*)f_true, n_nodes, counts, (T)alpha_e, (T)alpha_f, (T*)loss, (T*)de,
                    (T*)df,
                    contrib, partial, ticket),
                cudaGetLastError()))
}

int gfm_energy_seed(const void* de, const int* gnode, int n_nodes, int G, const void* a,
                    const void* y, void* ds, int ld_ds, void* dz, int dtype, void* stream) {
  if (ld_ds < 1) return GFM_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GFM_F32 && G % 4 == 0 && al16(y) && al16(a) && al16(dz) && n_nodes > 0) {
    GFM_TRY_CUDA(launch_k(k_energy_seed4, grid_1d((long long)n_nodes * (G / 4)), 256, 0, s,
                          (const float*)de, gnode, n_nodes, G / 4, (const float*)a,
                          (const float*)y, (float*)ds, ld_ds, (float*)dz));
    GFM_TRY_CUDA(cudaGetLastError());
    return 0;
  }
  GFM_DISPATCH(dtype, "gfm_energy_seed",
               (launch_k(k_energy_seed<T>, dim3(1, std::min(ceil_div(std::max(n_nodes, 1), 8), 65535)), dim3(32, 8), 0, s,
                    (const T*)de, gnode, n_nodes, G, (const T*)a, (const T*)y, (T*)ds, ld_ds,
                    (T*)dz),
                cudaGetLastError()))
}

size_t gfm_embedding_grad_workspace_bytes(int n_nodes, int H, int dtype) {
  return dtype == GFM_F64 ? linear_bwd_weight_ws<double>(n_nodes, 118, H, 0, 0)
                          : linear_bwd_weight_ws<float>(n_nodes, 118, H, 0, 0);
}

int gfm_embedding_grad(const int* z, int n_nodes, const void* dh, int H, void* grad,
                       void* workspace, int dtype, void* stream) {
  GFM_DISPATCH(dtype, "gfm_embedding_grad",
               embedding_grad_t<T>(z, n_nodes, (const T*)dh, H, (T*)grad, (T*)workspace,
                                   (cudaStream_t)stream))
}

}  // extern "C"
