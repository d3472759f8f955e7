// tcgen05 GEMM core for the model's skinny GEMMs (sm_100a).
//
// C[m][n] = sum_k A(m, k) * Bt(n, k) with a 128 x BN CTA tile and the
// accumulator in TMEM.  Operands are staged into shared memory by the CTA's
// threads -- not TMA -- because the A operands are gathers (h[dst] + h[src]
// pairs), concatenations ([h | agg]) or transposes that a tensor map cannot
// express; the same loaders as the SIMT engine feed it.  Staging writes the
// canonical K-major SWIZZLE_128B layout (8-row x 128-byte atoms, 16-byte
// chunk index XOR row%8) that the UMMA shared-memory descriptors describe.
//
// Precision: "3xTF32".  Each fp32 operand is split hi = rna_tf32(x),
// lo = x - hi, and the tile is accumulated as lo*hi + hi*lo + hi*hi with
// kind::tf32 MMAs -> ~22 mantissa bits per product, fp32 accumulation, i.e.
// float32-level results at tensor-core rate (1 x TF32 is selectable).
//
// Pipeline: 2 smem stages.  All 4 warps stage k-block kb+1 while the single
// elected thread's MMAs for kb run; tcgen05.commit arrives on the stage's
// mbarrier, which gates reuse of that stage.  Epilogue: each warp reads its
// 32 TMEM lanes (one output row per thread) with tcgen05.ld.32x32b.x16.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace gfm {
namespace tc {

constexpr int kBM = 128;           // MMA M (cta_group::1)
constexpr int kBK = 32;            // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 128;      // 4 warps: stage + epilogue; thread 0 issues MMAs
constexpr int kStages = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// byte offset of (row, k) inside a [rows][128B] K-major SWIZZLE_128B block
__device__ __forceinline__ uint32_t swz(int row, int k) {
  return (uint32_t)(row * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + ((k & 3) << 2));
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B (8-row
// group stride), LBO = 16 B (unused for swizzled K-major), version 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = bn
__host__ __device__ constexpr uint32_t make_idesc_tf32(int bn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n"
      :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(dst_smem)), "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

template <int NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "n"(NCOLS));
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
struct Smem {
  // per stage: A hi, A lo (128 x 128 B), B hi, B lo (BN x 128 B); 1024-aligned
  static constexpr int kA = kBM * 128;
  static constexpr int kB = BN * 128;
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kBytes = kStages * kStage + 1024 /*align*/ + 64 /*barriers, tmem ptr*/;
};

constexpr int tmem_cols(int bn) { return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256; }

// Stage rows [r0, r0 + ROWS) x one 32-wide k-block of a loader into hi/lo
// swizzled tiles.  All global loads of a thread are issued before any smem
// store (register batch) so each thread keeps up to 32 loads in flight.
// Mapping: k across lanes when k is contiguous in memory, rows otherwise.
template <int ROWS, class L>
__device__ __forceinline__ void stage(const L& ld, int r0, int rows_valid, int k0, int k_valid,
                                      uint8_t* hi, uint8_t* lo, bool split) {
  constexpr int kItems = ROWS * kBK / kThreads;  // elements per thread
  constexpr int kBatch = kItems < 32 ? kItems : 32;
  const int tid = threadIdx.x;
#pragma unroll
  for (int b0 = 0; b0 < kItems; b0 += kBatch) {
    float v[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int it = b0 + j;
      int r, k;
      if (!L::kContigRow) {
        r = (tid >> 5) + it * (kThreads / 32);
        k = tid & 31;
      } else {
        const int idx = tid + it * kThreads;
        r = idx % ROWS;
        k = idx / ROWS;
      }
      v[j] = (r < rows_valid && k < k_valid) ? ld(r0 + r, k0 + k) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int it = b0 + j;
      int r, k;
      if (!L::kContigRow) {
        r = (tid >> 5) + it * (kThreads / 32);
        k = tid & 31;
      } else {
        const int idx = tid + it * kThreads;
        r = idx % ROWS;
        k = idx / ROWS;
      }
      const uint32_t off = swz(r, k);
      const uint32_t h = split ? to_tf32(v[j]) : __float_as_uint(v[j]);
      *reinterpret_cast<uint32_t*>(hi + off) = h;
      if (split) *reinterpret_cast<float*>(lo + off) = v[j] - __uint_as_float(h);
    }
  }
}

// Persistent kernel: each CTA walks tiles t = blockIdx.x, += gridDim.x over
// (m tiles x n tiles x k splits).  TMEM and barriers are set up once.
// Epilogue concept (row owner; every thread calls every hook):
//   set_tile(bm, bn, split); begin(m, valid);
//   chunk(m, valid, n, v[16], ncols_valid) per 16-column chunk in order;
//   end(m, valid, n0, bm, bn, split).
template <int BN, class AL, class BL, class Epi>
__global__ void __launch_bounds__(kThreads)
    tc_gemm_kernel(int M, const int* __restrict__ M_dev, int N, int K, const int* __restrict__ K_dev,
                   int k_chunk, int splits, int split3, AL a, BL b, Epi epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = Smem<BN>;
  constexpr int NC = tmem_cols(BN);
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kStages * S::kStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kStages + 1);

  const int m_total = M_dev ? *M_dev : M;
  const int k_total = K_dev ? *K_dev : K;
  const int m_tiles = (m_total + kBM - 1) / kBM;
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_tiles * n_tiles * splits;
  if ((int)blockIdx.x >= n_work) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    mbar_init(&bars[kStages], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc<NC>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = make_idesc_tf32(BN);
  const bool split_on = split3 != 0;
  uint32_t phase[kStages] = {0, 0};
  uint32_t done_phase = 0;
  int g = 0;  // k-blocks issued by this CTA so far (stage ring position)

  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int split = w % splits;
    const int bn = (w / splits) % n_tiles;
    const int bm = w / (splits * n_tiles);
    const int m0 = bm * kBM, n0 = bn * BN;
    const int k_begin = split * k_chunk;
    const int k_end = min(k_total, k_begin + k_chunk);
    const int rows_a = min(kBM, m_total - m0);
    const int rows_b = min(BN, N - n0);
    const int nkb = k_end > k_begin ? (k_end - k_begin + kBK - 1) / kBK : 0;

    for (int kb = 0; kb < nkb; ++kb, ++g) {
      const int s = g % kStages;
      if (g >= kStages) {  // the MMAs that read this stage must have completed
        mbar_wait(&bars[s], phase[s]);
        phase[s] ^= 1;
      }
      uint8_t* st = base + s * S::kStage;
      uint8_t* a_hi = st;
      uint8_t* a_lo = st + S::kA;
      uint8_t* b_hi = st + 2 * S::kA;
      uint8_t* b_lo = st + 2 * S::kA + S::kB;
      const int k0 = k_begin + kb * kBK;
      const int kv = min(kBK, k_end - k0);
      stage<kBM>(a, m0, rows_a, k0, kv, a_hi, a_lo, split_on);
      stage<BN>(b, n0, rows_b, k0, kv, b_hi, b_lo, split_on);
      fence_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
        const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
        for (int ks = 0; ks < kBK / 8; ++ks) {  // K = 8 tf32 per MMA = 32 bytes
          const uint32_t o = ks * 32;
          const uint32_t acc0 = (kb > 0 || ks > 0) ? 1u : 0u;
          if (split_on) {
            mma_tf32(tmem, make_desc(al + o), make_desc(bh + o), idesc, acc0);
            mma_tf32(tmem, make_desc(ah + o), make_desc(bl + o), idesc, 1u);
            mma_tf32(tmem, make_desc(ah + o), make_desc(bh + o), idesc, 1u);
          } else {
            mma_tf32(tmem, make_desc(ah + o), make_desc(bh + o), idesc, acc0);
          }
        }
        mma_commit(&bars[s]);
      }
    }
    // all MMAs of this tile done -> accumulator readable
    if (threadIdx.x == 0) {
      if (nkb > 0)
        mma_commit(&bars[kStages]);
      else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&bars[kStages])) : "memory");
    }
    mbar_wait(&bars[kStages], done_phase);
    done_phase ^= 1;
    tc_fence_after();

    const int row = warp * 32 + lane;
    const int m = m0 + row;
    const bool valid = row < rows_a;
    epi.set_tile(bm, bn, split);
    epi.begin(m, valid);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      if (nkb > 0) {
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      epi.chunk(m, valid, n0 + c, v, min(16, N - (n0 + c)));
    }
    epi.end(m, valid, n0, bm, bn, split);
    tc_fence_before();
    __syncthreads();  // TMEM reads (and epilogue smem) finished before the next tile
    tc_fence_after();
  }
  if (warp == 0) tmem_free<NC>(tmem);
}

template <int BN, class AL, class BL, class Epi>
inline cudaError_t launch_bn(int M, const int* M_dev, int N, int K, const int* K_dev, int splits,
                             int split3, AL a, BL b, Epi epi, cudaStream_t s) {
  int k_chunk = ceil_div(ceil_div(K > 0 ? K : 1, splits), kBK) * kBK;
  splits = ceil_div(K > 0 ? K : 1, k_chunk);
  const int smem = Smem<BN>::kBytes;
  auto kern = tc_gemm_kernel<BN, AL, BL, Epi>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long long work = (long long)ceil_div(M, kBM) * ceil_div(N, BN) * splits;
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;
  const int grid = (int)std::min<long long>(work, 148LL * per_sm);
  kern<<<grid, kThreads, smem, s>>>(M, M_dev, N, K, K_dev, k_chunk, splits, split3, a, b, epi);
  return cudaGetLastError();
}

// BN chosen from N: one N tile when N <= 256 (rounded up to 32/64/128/256)
template <class AL, class BL, class Epi>
inline cudaError_t launch(int M, const int* M_dev, int N, int K, const int* K_dev, int splits,
                          int split3, AL a, BL b, Epi epi, cudaStream_t s, int bn_hint = 0) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (splits < 1) splits = 1;
  const int bn = bn_hint ? bn_hint : (N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
  switch (bn) {
    case 32: return launch_bn<32>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
    case 64: return launch_bn<64>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
    case 128: return launch_bn<128>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
    default: return launch_bn<256>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
  }
}

// Number of K splits for weight-gradient GEMMs (shape-only -> deterministic)
inline int splits_for(long long M, long long N, long long K, int bn) {
  long long tiles = (long long)ceil_div(M, kBM) * ceil_div(N, bn);
  long long want = (2LL * 148 + tiles - 1) / tiles;
  long long max_by_k = (K + 255) / 256;
  long long s = want < max_by_k ? want : max_by_k;
  if (s < 1) s = 1;
  if (s > 512) s = 512;
  return (int)s;
}

// ---------------------------------------------------------------- epilogues
struct TcEpiBiasAct {  // out[m][n] = act(acc + bias[n])
  float* out;
  int ldo;
  const float* bias;
  int act;
  __device__ void set_tile(int, int, int) {}
  __device__ void begin(int, bool) {}
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv) {
    if (!valid) return;
    float* o = out + (long long)m * ldo + n;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < nv) {
        float x = v[i] + (bias ? bias[n + i] : 0.f);
        o[i] = act ? tanhf(x) : x;
      }
    }
  }
  __device__ void end(int, bool, int, int, int, int) {}
};

struct TcEpiSplitCols {  // cols [0, n1) -> o1, [n1, N) -> o2, optional *(1 - gate^2) on o1
  float* o1;
  int ld1, n1;
  float* o2;
  int ld2;
  const float* gate;
  int ldg;
  const float* add;  // optional addend on the o1 columns (row stride ld1), before the gate
  __device__ void set_tile(int, int, int) {}
  __device__ void begin(int, bool) {}
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv) {
    if (!valid) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i >= nv) continue;
      const int c = n + i;
      float x = v[i];
      if (c < n1) {
        if (add) x = add[(long long)m * ld1 + c] + x;
        if (gate) {
          const float g = gate[(long long)m * ldg + c];
          x *= 1.f - g * g;
        }
        o1[(long long)m * ld1 + c] = x;
      } else {
        o2[(long long)m * ld2 + (c - n1)] = x;
      }
    }
  }
  __device__ void end(int, bool, int, int, int, int) {}
};

struct TcEpiPartial {  // split-K partial tile ws[split][m][n] (row-major, width N)
  float* ws;
  long long split_stride;
  int M, N;
  int split;
  __device__ void set_tile(int, int, int sp) { split = sp; }
  __device__ void begin(int, bool) {}
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv) {
    if (!valid) return;
    float* o = ws + split * split_stride + (long long)m * N + n;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nv) o[i] = v[i];
  }
  __device__ void end(int, bool, int, int, int, int) {}
};

}  // namespace tc
}  // namespace gfm
