// Tiled SIMT GEMM engine with pluggable operand loaders and epilogues.
//
// C[m][n] = sum_k A(m, k) * Bt(n, k), 64x64 CTA tile, BK = 16, 256 threads,
// 4x4 register micro-tile per thread.  This is the exact (fp32 / fp64) path:
// the float64 instantiation backs the parity tests, and the fp32
// instantiation is the generic fallback for shapes the tcgen05 kernels do
// not cover.  Loaders fuse the gathers the model needs (h[dst] + h[src]
// pairs, [h | agg] concatenation, a virtual ones column for bias grads);
// epilogues fuse bias + tanh, the force head's u-dot, and deterministic
// split-K partials.
#pragma once

#include "common.cuh"

namespace gfm {

constexpr int kBM = 64, kBN = 64, kBK = 16, kTM = 4, kTN = 4, kGemmThreads = 256;

// ---------------------------------------------------------------- loaders
// Each loader exposes  T operator()(int row, int k)  (row = m for A, n for
// Bt) and kContigRow: true when consecutive rows are adjacent in memory.
// For the tcgen05 engine's 16-byte cp.async staging they also expose
// vec_ok(K) (host: alignment / divisibility check) and
// src4(row, k, rows_left, &src, &imm): the global address of the 16-byte
// chunk (k..k+3 of a row for k-contiguous loaders, rows row..row+3 at k for
// row-contiguous ones) and its valid byte count, or -1 with an immediate.

__host__ __device__ inline bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }


template <typename T>
struct RowsLd {  // X[row * ld + k]
  static constexpr bool kContigRow = false;
  const T* p;
  int ld;
  __device__ T operator()(int r, int k) const { return p[(long long)r * ld + k]; }
  bool vec_ok(int K) const { return sizeof(T) == 4 && al16(p) && ld % 4 == 0 && K % 4 == 0; }
  __device__ int src4(int r, int k, int, const float** src, float4*) const {
    *src = reinterpret_cast<const float*>(p + (long long)r * ld + k);
    return 16;
  }
};

template <typename T>
struct Rows2Ld {  // [X1 | X2 | 1] along k
  static constexpr bool kContigRow = false;
  const T* p1;
  int ld1, k1;
  const T* p2;
  int ld2, k2;
  __device__ T operator()(int r, int k) const {
    if (k < k1) return p1[(long long)r * ld1 + k];
    k -= k1;
    if (k < k2) return p2[(long long)r * ld2 + k];
    return T(1);
  }
  bool vec_ok(int K) const {
    return sizeof(T) == 4 && al16(p1) && ld1 % 4 == 0 && k1 % 4 == 0 && K % 4 == 0 &&
           K <= k1 + k2 && (k2 == 0 || (al16(p2) && ld2 % 4 == 0 && k2 % 4 == 0));
  }
  __device__ int src4(int r, int k, int, const float** src, float4*) const {
    *src = reinterpret_cast<const float*>(k < k1 ? p1 + (long long)r * ld1 + k
                                                 : p2 + (long long)r * ld2 + (k - k1));
    return 16;
  }
};

template <typename T>
struct ColsLd {  // X[k * ld + row]  (transposed view)
  static constexpr bool kContigRow = true;
  const T* p;
  int ld;
  __device__ T operator()(int r, int k) const { return p[(long long)k * ld + r]; }
  bool vec_ok(int) const { return sizeof(T) == 4 && al16(p) && ld % 4 == 0; }
  __device__ int src4(int r, int k, int rows_left, const float** src, float4*) const {
    *src = reinterpret_cast<const float*>(p + (long long)k * ld + r);
    return (rows_left < 4 ? rows_left : 4) * 4;
  }
};

template <typename T>
struct Cols2Ld {  // rows split over [X1 | X2 | 1]: X1[k*ld1 + r], X2[k*ld2 + r - n1], ones
  static constexpr bool kContigRow = true;
  const T* p1;
  int ld1, n1;
  const T* p2;
  int ld2, n2;
  const T* ones = nullptr;  // optional [K][4] buffer (column 0 = 1): the ones row as a tensor
  __device__ T operator()(int r, int k) const {
    if (r < n1) return p1[(long long)k * ld1 + r];
    r -= n1;
    if (r < n2) return p2[(long long)k * ld2 + r];
    return T(1);
  }
  bool vec_ok(int) const {
    return sizeof(T) == 4 && al16(p1) && ld1 % 4 == 0 && n1 % 4 == 0 &&
           (n2 == 0 || (al16(p2) && ld2 % 4 == 0 && n2 % 4 == 0));
  }
  __device__ int src4(int r, int k, int rows_left, const float** src, float4* imm) const {
    const int nb = (rows_left < 4 ? rows_left : 4) * 4;
    if (r < n1) {
      *src = reinterpret_cast<const float*>(p1 + (long long)k * ld1 + r);
      return nb;
    }
    if (r < n1 + n2) {
      *src = reinterpret_cast<const float*>(p2 + (long long)k * ld2 + (r - n1));
      return nb;
    }
    *imm = make_float4(1.f, 0.f, 0.f, 0.f);  // the virtual ones row (bias gradient)
    return -1;
  }
};

template <typename T>
struct PairLd {  // pair[e][k] = h[dst[e]][k] + h[src[e]][k]   (model.py:379)
  static constexpr bool kContigRow = false;
  const T* h;
  int H;
  const int* dst;
  const int* src;
  __device__ T operator()(int e, int k) const {
    return h[(long long)dst[e] * H + k] + h[(long long)src[e] * H + k];
  }
  bool vec_ok(int) const { return false; }
  __device__ int src4(int, int, int, const float**, float4*) const { return 0; }
};

template <typename T>
struct PairColsLd {  // Bt(n, e) = pair[e][n]; row n == H is a ones column
  static constexpr bool kContigRow = true;
  const T* h;
  int H;
  const int* dst;
  const int* src;
  __device__ T operator()(int n, int e) const {
    if (n >= H) return T(1);
    return h[(long long)dst[e] * H + n] + h[(long long)src[e] * H + n];
  }
  bool vec_ok(int) const { return false; }
  __device__ int src4(int, int, int, const float**, float4*) const { return 0; }
};

// ---------------------------------------------------------------- epilogues
// Epilogue signature:
//   void operator()(T (&acc)[kTM][kTN], int m0, int n0, int M, int N,
//                   int split, int bm, int bn, int tx, int ty)
// rows m0 + i, cols n0 + j belong to this thread.

template <typename T>
struct EpiBiasAct {  // out = act(acc + bias)  (model.py:357-358, 370)
  T* out;
  int ldo;
  const T* bias;  // may be null
  int act;        // 0 identity, 1 tanh
  __device__ void operator()(T (&acc)[kTM][kTN], int m0, int n0, int M, int N, int, int, int, int,
                             int) const {
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
      int m = m0 + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < kTN; ++j) {
        int n = n0 + j;
        if (n >= N) continue;
        T v = acc[i][j];
        if (bias) v = v + bias[n];
        if (act == 1) v = tanh_t(v);
        out[(long long)m * ldo + n] = v;
      }
    }
  }
};

template <typename T>
struct EpiSplitCols {  // columns [0, n1) -> o1, [n1, N) -> o2; optional *(1 - g^2)
  T* o1;
  int ld1, n1;
  T* o2;
  int ld2;
  const T* gate;  // if set: out *= (1 - gate[m][n]^2), gate row stride ldg
  int ldg;
  const T* add;   // if set: o1 columns get + add[m][n] (row stride ld1) before the gate
  __device__ void operator()(T (&acc)[kTM][kTN], int m0, int n0, int M, int N, int, int, int, int,
                             int) const {
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
      int m = m0 + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < kTN; ++j) {
        int n = n0 + j;
        if (n >= N) continue;
        T v = acc[i][j];
        if (add && n < n1) v = add[(long long)m * ld1 + n] + v;
        if (gate) {
          T g = gate[(long long)m * ldg + n];
          v = v * (T(1) - g * g);
        }
        if (n < n1)
          o1[(long long)m * ld1 + n] = v;
        else
          o2[(long long)m * ld2 + (n - n1)] = v;
      }
    }
  }
};

template <typename T>
struct EpiPartial {  // split-K partial: ws[split][m][n]
  T* ws;
  long long split_stride;
  __device__ void operator()(T (&acc)[kTM][kTN], int m0, int n0, int M, int N, int split, int, int,
                             int, int) const {
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
      int m = m0 + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < kTN; ++j) {
        int n = n0 + j;
        if (n < N) ws[split * split_stride + (long long)m * N + n] = acc[i][j];
      }
    }
  }
};

// ---------------------------------------------------------------- engine
template <typename T, class AL, class BL, class Epi>
__global__ void __launch_bounds__(kGemmThreads)
    simt_gemm_kernel(int M, const int* M_dev, int N, int K, const int* K_dev, int k_chunk, AL a, BL b,
                     Epi epi) {
  pdl_entry();
  __shared__ __align__(16) T As[kBK][kBM + 4];
  __shared__ __align__(16) T Bs[kBK][kBN + 4];
  const int m_total = M_dev ? *M_dev : M;
  const int m_blk = blockIdx.x * kBM;
  if (m_blk >= m_total) return;
  const int n_blk = blockIdx.y * kBN;
  const int split = blockIdx.z;
  const int k_begin = split * k_chunk;
  const int k_end = min(K_dev ? *K_dev : K, k_begin + k_chunk);
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;

  T acc[kTM][kTN];
#pragma unroll
  for (int i = 0; i < kTM; ++i)
#pragma unroll
    for (int j = 0; j < kTN; ++j) acc[i][j] = T(0);

  for (int kt = k_begin; kt < k_end; kt += kBK) {
#pragma unroll
    for (int r = 0; r < (kBM * kBK) / kGemmThreads; ++r) {
      const int idx = tid + r * kGemmThreads;
      int mm, kk;
      if (AL::kContigRow) {
        mm = idx % kBM; kk = idx / kBM;
      } else {
        kk = idx % kBK; mm = idx / kBK;
      }
      const int gm = m_blk + mm, gk = kt + kk;
      As[kk][mm] = (gm < m_total && gk < k_end) ? a(gm, gk) : T(0);
    }
#pragma unroll
    for (int r = 0; r < (kBN * kBK) / kGemmThreads; ++r) {
      const int idx = tid + r * kGemmThreads;
      int nn, kk;
      if (BL::kContigRow) {
        nn = idx % kBN; kk = idx / kBN;
      } else {
        kk = idx % kBK; nn = idx / kBK;
      }
      const int gn = n_blk + nn, gk = kt + kk;
      Bs[kk][nn] = (gn < N && gk < k_end) ? b(gn, gk) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      T av[kTM], bv[kTN];
#pragma unroll
      for (int i = 0; i < kTM; ++i) av[i] = As[kk][ty * kTM + i];
#pragma unroll
      for (int j = 0; j < kTN; ++j) bv[j] = Bs[kk][tx * kTN + j];
#pragma unroll
      for (int i = 0; i < kTM; ++i)
#pragma unroll
        for (int j = 0; j < kTN; ++j) acc[i][j] += av[i] * bv[j];
    }
    __syncthreads();
  }
  epi(acc, m_blk + ty * kTM, n_blk + tx * kTN, m_total, N, split, blockIdx.x, blockIdx.y, tx, ty);
}

template <typename T, class AL, class BL, class Epi>
inline cudaError_t launch_simt_gemm(int M, const int* M_dev, int N, int K, const int* K_dev,
                                    int splits, AL a, BL b, Epi epi, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (splits < 1) splits = 1;
  int k_chunk = ceil_div(K > 0 ? K : 1, splits);
  k_chunk = ceil_div(k_chunk, kBK) * kBK;
  splits = ceil_div(K > 0 ? K : 1, k_chunk);
  dim3 grid(ceil_div(M, kBM), ceil_div(N, kBN), splits);
  launch_k(simt_gemm_kernel<T, AL, BL, Epi>, grid, kGemmThreads, 0, s, M, M_dev, N, K, K_dev, k_chunk, a, b,
                                                                 epi);
  return cudaGetLastError();
}

// Number of K splits for a reduction of length K producing an MxN result,
// chosen from the problem shape only (never from timing) so results are
// deterministic run to run.
inline int choose_splits(long long M, long long N, long long K) {
  long long tiles = (long long)ceil_div(M, kBM) * ceil_div(N, kBN);
  long long want = (2LL * 148 + tiles - 1) / tiles;  // fixed: results independent of device
  long long max_by_k = (K + 255) / 256;
  long long s = want < max_by_k ? want : max_by_k;
  if (s < 1) s = 1;
  if (s > 256) s = 256;
  return (int)s;
}

}  // namespace gfm
