// tcgen05 GEMM core for the model's node-level GEMMs (sm_100a).
//
// C[m][n] = sum_k A(m, k) * Bt(n, k) with a 128 x BN CTA tile (BN <= 128)
// and the accumulator in TMEM.  Operands are staged into shared memory by the
// CTA's threads -- not TMA -- because the A operands are concatenations
// ([h | agg]), transposes (weight gradients: dY^T) or generated one-hot rows
// that a tensor map cannot express; the same loaders as the SIMT engine feed
// it.  k-contiguous operands are staged K-major SWIZZLE_128B (8-row x
// 128-byte atoms, 16-byte chunk index XOR row % 8); row-contiguous operands
// (transposes) are staged MN-major SWIZZLE_128B_BASE32B so 16-byte global
// loads map to conflict-free 16-byte smem stores.
//
// Precision: "3xTF32".  Each fp32 operand is split hi = trunc_tf32(x),
// lo = x - hi (exact), and each tile is accumulated as lo*hi + hi*lo + hi*hi
// with kind::tf32 MMAs -> ~21 mantissa bits per product with fp32
// accumulation (measured max error ~3e-6 relative at K = 320, ~3x the SIMT
// fp32 engine); 1xTF32 (GFM_GEMM_TC1) skips the corrections.
//
// Schedule: one persistent CTA of 8 warps per SM walks (m tile, n tile,
// k split) work items as ONE flattened stream of 32-wide k-blocks.  Raw fp32
// tiles land in an S-deep smem ring via cp.async (16-byte, zero-fill for
// out-of-range chunks), L = S - 2 k-blocks ahead of the consumer, continuing
// across tile boundaries.  The raw tile is itself the "hi" TF32 operand (the
// tensor core ignores the low 13 mantissa bits); a light pass writes
// lo = x - trunc_tf32(x) into one of two lo buffers.  One thread issues the
// MMAs and tcgen05.commit arrives on the stage's mbarrier, which gates ring
// reuse.  Epilogue: warp w reads TMEM lanes 32*(w%4).. (one output row per
// thread) for column half w/4, 16 columns per tcgen05.ld.32x32b.x16.
#pragma once

#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "gemm_simt.cuh"

namespace gfm {
namespace tc {

// epilogues may define prefetch(m, n) -> state and store4(m, n, v, nv, split,
// state): the kernel then issues the four rows' prefetches of a chunk before
// any of their stores (their global loads overlap instead of serialising)
template <class E, class = void>
struct HasPrefetch : std::false_type {};
template <class E>
struct HasPrefetch<E, std::void_t<decltype(&E::prefetch)>> : std::true_type {};

// GFM_NO_TMA=1 forces the thread-staged (cp.async) engine (debug / A-B runs)
inline bool tma_disabled() {
  static int v = -1;
  if (v < 0) v = getenv("GFM_NO_TMA") ? atoi(getenv("GFM_NO_TMA")) : 0;
  return v != 0;
}

// GFM_NO_TMEM_A=1 keeps A in shared memory in the 3xTF32 TMA kernel (A/B runs)
inline bool at_disabled() {
  static int v = -1;
  if (v < 0) v = getenv("GFM_NO_TMEM_A") ? atoi(getenv("GFM_NO_TMEM_A")) : 0;
  return v != 0;
}

// CTA-pair (cta_group::2) 3xTF32 kernel for 64/128-wide tiles with a K-major
// A (default; GFM_TC_PAIR=0 / gfm_set_tc_pairs(0) for the single-CTA kernel)
inline bool pairs_enabled() { return tc_pairs(); }

// Accumulation flush depth in 32-wide k-blocks (TMA engine).  The tensor
// core's fp32 accumulator rounds toward zero, so its error grows linearly
// with the accumulation depth (tools/tf32_probe.py k: 1.0e-7 rms relative at
// K = 32, 6.0e-6 at 2,560, 1.9e-5 at 8,192, almost all of it a bias toward
// zero; IEEE FFMA chains: 9e-7 at 2,560).  Every 16 k-blocks (512 products)
// the epilogue warps fold the TMEM partial into fp32 registers (IEEE adds)
// while the MMAs fill the other accumulator, which bounds the biased run:
// 1.2e-6 rms at any K.  The last chunk is folded too and its accumulator
// released before the stores, so the next tile's MMAs do not wait on them.
// Measured at the C3 shapes (tools/gemm_time.py): every 16 k-blocks costs
// +5% forward, +0% backward-data, +4% weight gradient; every 8 costs up to
// +70% (register spills).  GFM_TC_FLUSH_KB overrides (0 = never flush).
inline int flush_kb() {
  static int v = -1;
  if (v < 0) v = getenv("GFM_TC_FLUSH_KB") ? atoi(getenv("GFM_TC_FLUSH_KB")) : 16;
  return v > 0 ? v : (1 << 30);
}

constexpr int kBM = 128;       // MMA M (cta_group::1)
constexpr int kBK = 32;        // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 256;  // 8 warps: staging + epilogue; thread 0 issues MMAs

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
// group stride), LBO = 16 B (ignored for swizzled K-major), version 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// MN-major SWIZZLE_128B_BASE32B descriptor (layout type 1): 128-byte rows
// hold 32 consecutive M (or N) tf32 of one k; 4 k-rows form a 512 B atom;
// LBO = byte stride between 32-element M/N atoms, SBO = stride between 4-k
// groups (an 8-deep tf32 MMA spans two).
__device__ __forceinline__ uint64_t make_desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

// instruction descriptor: D f32, A/B tf32, M = 128, N = bn; a_mn / b_mn
// select MN-major operands (bits 15 / 16)
__host__ __device__ constexpr uint32_t make_idesc_tf32(int bn, bool a_mn = false,
                                                       bool b_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
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

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gptr, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(saddr), "l"(gptr),
               "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory");
}

constexpr int tmem_cols(int cols) {
#ifdef GFM_TMEM_CAP256
  return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : 256;
#else
  return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
#endif
}

// ring depth by BN (192 KB of ring + lo buffers, one CTA per SM)
template <int BN>
struct Smem {
  static constexpr int kA = kBM * 128;  // one k-block of A: 128 rows x 128 B
  static constexpr int kB = BN * 128;
  static constexpr int kStage = kA + kB;
  static constexpr int kS = BN >= 128 ? 4 : BN >= 64 ? 6 : 7;  // ring stages
  static constexpr int kL = kS - 2;                              // lookahead
  static constexpr int kBytes = kS * kStage + 2 * kStage + 1024 /*align*/ + 512;
};

// MN-major tf32 tile of ROWS x 32 k in the SWIZZLE_128B_BASE32B layout (the
// only MN-major smem layout tcgen05 accepts for tf32): atoms of 4 k-rows x
// 128 B (32 rows) = 512 B; atom (k / 4, row / 32) at ((k/4) * ROWS/32 +
// row/32) * 512; inside, k-row kr = k % 4 at kr * 128 and the 32-byte chunk
// (row % 32) / 8 is XORed with kr.  A 16-byte row-quad is half a chunk.
template <int ROWS>
__device__ __forceinline__ uint32_t mn_off(int rq, int k) {
  const int r = rq << 2;
  const int kg = k >> 2, kr = k & 3, atom = r >> 5, c32 = (r & 31) >> 3, half = (r & 7) >> 2;
  return (uint32_t)((kg * (ROWS / 32) + atom) * 512 + kr * 128 + ((c32 ^ kr) << 5) + (half << 4));
}

// Issue one k-block of one operand into a raw tile.
//  VEC: 16-byte chunks -- loaders expose src4(r, k, rows_left, &src, &imm):
//       >= 0 -> cp.async from src with that many valid bytes (zero fill);
//       < 0  -> immediate value imm (stored directly).  k-contiguous loaders
//       give k..k+3 of row r (K-major chunk); row-contiguous ones give rows
//       r..r+3 at k (MN-major chunk).
//  scalar: synchronous register loads into the K-major layout.
template <int ROWS, bool VEC, int kThreads, class L>
__device__ __forceinline__ void issue_tile(const L& ld, int r0, int rows_valid, int k0, int k_valid,
                                           uint8_t* dst, int tid) {
  if constexpr (VEC) {
    constexpr int kChunks = ROWS * kBK / 4;
    const uint32_t sbase = smem_u32(dst);
#pragma unroll
    for (int j = 0; j < (kChunks + kThreads - 1) / kThreads; ++j) {
      const int idx = tid + j * kThreads;
      if (idx >= kChunks) break;
      int r, k;
      uint32_t off;
      if (!L::kContigRow) {
        r = idx >> 3;
        k = (idx & 7) << 2;
        off = (uint32_t)(r * 128 + (((idx & 7) ^ (r & 7)) << 4));
      } else {
        const int rq = idx % (ROWS / 4);
        r = rq << 2;
        k = idx / (ROWS / 4);
        off = mn_off<ROWS>(rq, k);
      }
      if (r < rows_valid && k < k_valid) {
        const float* src = nullptr;
        float4 imm;
        const int nb = ld.src4(r0 + r, k0 + k, rows_valid - r, &src, &imm);
        if (nb >= 0)
          cp_async16(sbase + off, src, nb);
        else
          *reinterpret_cast<float4*>(dst + off) = imm;
      } else {
        *reinterpret_cast<uint4*>(dst + off) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  } else {
    constexpr int kItems = ROWS * kBK / kThreads;
    constexpr int kBatch = kItems < 16 ? kItems : 16;
#pragma unroll
    for (int b0 = 0; b0 < kItems; b0 += kBatch) {
      float v[kBatch];
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        int r, k;
        if (!L::kContigRow) {
          r = (tid >> 5) + (b0 + j) * (kThreads / 32);
          k = tid & 31;
        } else {
          const int idx = tid + (b0 + j) * kThreads;
          r = idx % ROWS;
          k = idx / ROWS;
        }
        v[j] = (r < rows_valid && k < k_valid) ? ld(r0 + r, k0 + k) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        int r, k;
        if (!L::kContigRow) {
          r = (tid >> 5) + (b0 + j) * (kThreads / 32);
          k = tid & 31;
        } else {
          const int idx = tid + (b0 + j) * kThreads;
          r = idx % ROWS;
          k = idx / ROWS;
        }
        *reinterpret_cast<float*>(dst + swz(r, k)) = v[j];
      }
    }
  }
}

// lo = x - trunc_tf32(x) for every 16-byte chunk of a raw stage.  Explicit
// shared-space ld/st (the stage pointers are computed, so generic LD/ST would
// otherwise go through the slower generic path); all of a thread's loads are
// issued before its stores.
template <int BYTES, int kThreads>
__device__ __forceinline__ void make_lo(const uint8_t* raw, uint8_t* lo, int tid) {
  constexpr int kChunks = BYTES / 16;
  constexpr int kFull = kChunks / kThreads;
  const uint32_t r0 = smem_u32(raw), l0 = smem_u32(lo);
  const uint32_t m = 0xFFFFE000u;
  auto split = [&](uint4 x) {
    float4 l;
    l.x = __uint_as_float(x.x) - __uint_as_float(x.x & m);
    l.y = __uint_as_float(x.y) - __uint_as_float(x.y & m);
    l.z = __uint_as_float(x.z) - __uint_as_float(x.z & m);
    l.w = __uint_as_float(x.w) - __uint_as_float(x.w & m);
    return l;
  };
  uint4 x[kFull > 0 ? kFull : 1];
#pragma unroll
  for (int i = 0; i < kFull; ++i) {
    const uint32_t a = r0 + 16u * (uint32_t)(tid + i * kThreads);
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(x[i].x), "=r"(x[i].y), "=r"(x[i].z), "=r"(x[i].w) : "r"(a));
  }
#pragma unroll
  for (int i = 0; i < kFull; ++i) {
    const float4 l = split(x[i]);
    const uint32_t a = l0 + 16u * (uint32_t)(tid + i * kThreads);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "r"(a), "f"(l.x), "f"(l.y), "f"(l.z), "f"(l.w) : "memory");
  }
  for (int c = kFull * kThreads + tid; c < kChunks; c += kThreads) {
    uint4 y;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(y.x), "=r"(y.y), "=r"(y.z), "=r"(y.w) : "r"(r0 + 16u * (uint32_t)c));
    const float4 l = split(y);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "r"(l0 + 16u * (uint32_t)c), "f"(l.x), "f"(l.y), "f"(l.z), "f"(l.w) : "memory");
  }
}

// Work items are ordered split-major (w = split * tiles + tile): the CTAs in
// flight together share one K range, so a split-K GEMM streams each operand
// slice from HBM once and reuses it from L2 across all output tiles.
// Work item -> number of 32-wide k-blocks
__device__ __forceinline__ int item_nkb(int w, int tiles, int k_chunk, int k_total) {
  const int split = w / tiles;
  const int kb0 = split * k_chunk, kb1 = min(k_total, kb0 + k_chunk);
  return kb1 > kb0 ? (kb1 - kb0 + kBK - 1) / kBK : 0;
}

// Warp-specialised persistent kernel (one CTA per SM, 288 threads):
//   warps 0-3  producers: cp.async k-block p into ring stage p % S (after the
//              MMAs of p - S released it: empty[s]), and for k-block
//              q = p - L: wait its copies, write lo = x - trunc(x), arrive
//              full[q % S];
//   warp 8     MMA issuer (one elected lane): waits full[s], issues the 4 (or
//              12 with 3xTF32) tcgen05.mma of the k-block into TMEM
//              accumulator t % 2, commits empty[s]; at a tile's last k-block
//              commits tmem_full[t % 2] (waiting tmem_empty first for t >= 2);
//   warps 4-7  epilogue: wait tmem_full, tcgen05.ld rows (warp w owns TMEM
//              lanes 32*(w%4)), apply the epilogue, arrive tmem_empty.
// Phases: the n-th completion of a barrier has parity n & 1.
constexpr int kProducers = 128, kEpilogue = 128, kWSThreads = kProducers + kEpilogue + 32;

template <int BN, bool VA, bool VB, class AL, class BL, class Epi>
__global__ void __launch_bounds__(kWSThreads, 1)
    tc_gemm_kernel(int M, const int* __restrict__ M_dev, int N, int K, const int* __restrict__ K_dev,
                   int k_chunk, int splits, int split3, AL a, BL b, Epi epi) {
  pdl_entry();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = Smem<BN>;
  constexpr int NC = tmem_cols(2 * BN);  // two accumulators
  constexpr int kS = S::kS, kL = S::kL;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ring = base;                    // kS x [A raw | B raw]
  uint8_t* lobuf = base + kS * S::kStage;  // 2 x [A lo | B lo]
  uint64_t* full = reinterpret_cast<uint64_t*>(lobuf + 2 * S::kStage);
  uint64_t* empty = full + kS;
  uint64_t* tfull = empty + kS;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int m_total = M_dev ? *M_dev : M;
  const int k_total = K_dev ? *K_dev : K;
  const int m_tiles = (m_total + kBM - 1) / kBM;
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_tiles * n_tiles * splits;
  if ((int)blockIdx.x >= n_work) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int q = 0; q < kS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], kEpilogue / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc<NC>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool split_on = split3 != 0;

  auto tile_of = [&](int w, int& bm, int& bn, int& split) {
    split = w / (m_tiles * n_tiles);
    bn = (w % (m_tiles * n_tiles)) % n_tiles;
    bm = (w % (m_tiles * n_tiles)) / n_tiles;
  };

  if (warp < kProducers / 32) {
    // ================================================================ producers
    const int tid = threadIdx.x;
    int pw = blockIdx.x, pkb = 0, p = 0;  // issue cursor
    int cw = blockIdx.x, ckb = 0, q = 0;  // convert cursor
    auto skip_empty = [&](int& w, int& kb) {
      while (w < n_work && item_nkb(w, m_tiles * n_tiles, k_chunk, k_total) == 0) w += gridDim.x;
      kb = 0;
    };
    skip_empty(pw, pkb);
    skip_empty(cw, ckb);
    auto issue_one = [&]() {  // always commits one group (possibly empty)
      if (pw < n_work) {
        const int s = p % kS;
        if (p >= kS) mbar_wait(&empty[s], ((p / kS) - 1) & 1);
        int bm, bn, split;
        tile_of(pw, bm, bn, split);
        const int k_begin = split * k_chunk;
        const int k_end = min(k_total, k_begin + k_chunk);
        const int k0 = k_begin + pkb * kBK;
        const int kv = min(kBK, k_end - k0);
        uint8_t* st = ring + s * S::kStage;
        issue_tile<kBM, VA, kProducers>(a, bm * kBM, min(kBM, m_total - bm * kBM), k0, kv, st, tid);
        issue_tile<BN, VB, kProducers>(b, bn * BN, min(BN, N - bn * BN), k0, kv, st + S::kA, tid);
        ++p;
        if (++pkb == item_nkb(pw, m_tiles * n_tiles, k_chunk, k_total)) {
          pw += gridDim.x;
          skip_empty(pw, pkb);
        }
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int i = 0; i < kL; ++i) issue_one();
    while (cw < n_work) {
      issue_one();                 // k-block q + kL
      cp_async_wait<kL>();         // k-block q landed (own copies)
      asm volatile("bar.sync 1, %0;" :: "n"(kProducers) : "memory");  // everyone's copies
      const int s = q % kS;
      // lo[q & 1] was last read by the MMAs of k-block q - 2 (at the stream's
      // tail no later issue waited for them, so wait explicitly)
      if (split_on && q >= 2) mbar_wait(&empty[(q - 2) % kS], ((q - 2) / kS) & 1);
      if (split_on) make_lo<S::kStage, kProducers>(ring + s * S::kStage, lobuf + (q & 1) * S::kStage, tid);
      fence_async_smem();
      asm volatile("bar.sync 1, %0;" :: "n"(kProducers) : "memory");
      if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&full[s])) : "memory");
      ++q;
      if (++ckb == item_nkb(cw, m_tiles * n_tiles, k_chunk, k_total)) {
        cw += gridDim.x;
        skip_empty(cw, ckb);
      }
    }
    cp_async_wait<0>();
  } else if (warp == (kProducers + kEpilogue) / 32) {
    // ================================================================ MMA issuer
    constexpr bool kAmn = VA && AL::kContigRow;
    constexpr bool kBmn = VB && BL::kContigRow;
    const uint32_t idesc = make_idesc_tf32(BN, kAmn, kBmn);
    auto desc_a = [&](uint32_t addr, int ks) -> uint64_t {
      if constexpr (kAmn)
        return make_desc_mn(addr + ks * (kBM / 32) * 1024, 512, (kBM / 32) * 512);
      else
        return make_desc(addr + ks * 32);
    };
    auto desc_b = [&](uint32_t addr, int ks) -> uint64_t {
      if constexpr (kBmn)
        return make_desc_mn(addr + ks * (BN / 32) * 1024, 512, (BN / 32) * 512);
      else
        return make_desc(addr + ks * 32);
    };
    int q = 0, t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      const int nkb = item_nkb(w, m_tiles * n_tiles, k_chunk, k_total);
      const int acc = t & 1;
      if (t >= 2) mbar_wait(&tempty[acc], ((t >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * BN);
      for (int kb = 0; kb < nkb; ++kb, ++q) {
        const int s = q % kS;
        mbar_wait(&full[s], (q / kS) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ah = smem_u32(ring + s * S::kStage), bh = ah + S::kA;
          const uint32_t al = smem_u32(lobuf + (q & 1) * S::kStage), bl = al + S::kA;
#pragma unroll
          for (int ks = 0; ks < kBK / 8; ++ks) {
            const uint32_t acc0 = (kb > 0 || ks > 0) ? 1u : 0u;
            if (split_on) {
              mma_tf32(d, desc_a(al, ks), desc_b(bh, ks), idesc, acc0);
              mma_tf32(d, desc_a(ah, ks), desc_b(bl, ks), idesc, 1u);
              mma_tf32(d, desc_a(ah, ks), desc_b(bh, ks), idesc, 1u);
            } else {
              mma_tf32(d, desc_a(ah, ks), desc_b(bh, ks), idesc, acc0);
            }
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (nkb > 0)
          mma_commit(&tfull[acc]);
        else
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tfull[acc])) : "memory");
      }
      __syncwarp();
    }
  } else {
    // ================================================================ epilogue
    const int quarter = warp & 3;
    int t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      int bm, bn, split;
      tile_of(w, bm, bn, split);
      const int nkb = item_nkb(w, m_tiles * n_tiles, k_chunk, k_total);
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const int m0 = bm * kBM, n0 = bn * BN;
      const int row = quarter * 32 + lane;
      const int m = m0 + row;
      const bool valid = row < min(kBM, m_total - m0);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        if (nkb > 0) {
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c), v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        epi.chunk(m, valid, n0 + c, v, min(16, N - (n0 + c)), split);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tempty[acc])) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<NC>(tmem);
}

// ============================================================== TMA engine
// Host-built operand: up to two 2D fp32 segments.  K-major (mn = 0): rows x K
// with K contiguous, segments concatenated along K (split at k = split_at),
// box {32 k, ROWS rows}, SWIZZLE_128B == the K-major smem layout above.
// MN-major (mn = 1): memory X[k][row], segments concatenated along rows
// (split at row = split_at), box {32 rows, 32 k} per 32-row atom, swizzle
// 128B_ATOM_32B == SWIZZLE_128B_BASE32B with LBO = 4096 (atom), SBO = 512.
struct TmaOp {
  CUtensorMap map[3];
  // MN-major only: 3D view {32, K, extent / 32} of a segment whose extent is a
  // multiple of 32, so one TMA instruction fetches a whole 128-row tile (four
  // 32-row atoms, smem [atom][k][32]) instead of four 4 KB boxes -- the per-box
  // cost of narrow boxes, not bandwidth, bounds MN-major streaming
  CUtensorMap map3[3];
  int has3[3];
  int split_at;  // start of segment 1
  int split2;    // start of segment 2 (MN-major: the ones row of a bias gradient)
  int mn;
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

// 2D fp32 map: inner (contiguous) extent x outer extent, row stride ld elems
inline bool make_map(CUtensorMap* m, const float* base, long long inner, long long outer, long long ld,
                     int box_inner, int box_outer, CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || !base || inner <= 0 || outer <= 0) return false;
  if (((uintptr_t)base & 15) || ((ld * 4) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3D MN-major view: dims {32, K, extent / 32}, strides {ld, 32} elements,
// box {32, kBK, 4}
inline bool make_map3(CUtensorMap* m, const float* base, long long extent, long long K, long long ld,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, int atoms = 4) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || !base || extent <= 0 || extent % 32 || K <= 0) return false;
  if (((uintptr_t)base & 15) || ((ld * 4) & 15)) return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)(extent / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), 128};
  cuuint32_t box[3] = {32, (cuuint32_t)kBK, (cuuint32_t)atoms};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Loader -> TMA operand (false when the loader cannot be expressed)
template <class L>
inline bool build_tma(const L&, TmaOp*, int, long long, int,
                      CUtensorMapSwizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) {
  return false;
}

template <typename T>
inline bool build_tma(const RowsLd<T>& l, TmaOp* op, int rows_box, long long rows_total, int K,
                      CUtensorMapSwizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) {
  if (sizeof(T) != 4) return false;
  op->mn = 0;
  op->split_at = 1 << 30;
  op->split2 = 1 << 30;
  op->has3[0] = op->has3[1] = op->has3[2] = 0;
  return make_map(&op->map[0], (const float*)l.p, K, rows_total, l.ld, kBK, rows_box,
                  CU_TENSOR_MAP_SWIZZLE_128B);
}

template <typename T>
inline bool build_tma(const Rows2Ld<T>& l, TmaOp* op, int rows_box, long long rows_total, int K,
                      CUtensorMapSwizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) {
  if (sizeof(T) != 4 || K > l.k1 + l.k2) return false;
  op->mn = 0;
  op->split_at = l.k2 > 0 ? l.k1 : (1 << 30);
  op->split2 = 1 << 30;
  op->has3[0] = op->has3[1] = op->has3[2] = 0;
  if (l.k2 > 0 && l.k1 % kBK) return false;
  if (!make_map(&op->map[0], (const float*)l.p1, l.k1, rows_total, l.ld1, kBK, rows_box,
                CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  return l.k2 == 0 || make_map(&op->map[1], (const float*)l.p2, l.k2, rows_total, l.ld2, kBK,
                               rows_box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// MN-major operands: the 3D view fetches min(rows_box, 128) / 32 atoms per
// instruction (64-row B halves of CTA pairs: two)
template <typename T>
inline bool build_tma(const ColsLd<T>& l, TmaOp* op, int rows_box, long long rows_total, int K,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) {
  const int atoms = rows_box >= 128 ? 4 : (rows_box >= 32 ? rows_box / 32 : 1);
  if (sizeof(T) != 4) return false;
  op->mn = 1;
  op->split_at = 1 << 30;
  op->split2 = 1 << 30;
  op->has3[0] = op->has3[1] = op->has3[2] = 0;
  if (!make_map(&op->map[0], (const float*)l.p, rows_total, K, l.ld, 32, kBK, sw))
    return false;
  op->has3[0] = make_map3(&op->map3[0], (const float*)l.p, rows_total, K, l.ld, sw, atoms);
  return true;
}

template <typename T>
inline bool build_tma(const Cols2Ld<T>& l, TmaOp* op, int rows_box, long long rows_total, int K,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) {
  const int atoms = rows_box >= 128 ? 4 : (rows_box >= 32 ? rows_box / 32 : 1);
  // the virtual ones row (bias) needs the caller's ones buffer (a [K][4]
  // tensor whose column 0 is 1: inner extent 1, the rest of each 32-row box
  // is TMA zero fill)
  const bool bias = rows_total == l.n1 + l.n2 + 1;
  if (sizeof(T) != 4 || (rows_total > l.n1 + l.n2 && !(bias && l.ones))) return false;
  if ((l.n2 > 0 && l.n1 % 32) || (bias && (l.n1 + l.n2) % 32)) return false;
  op->mn = 1;
  op->has3[0] = op->has3[1] = op->has3[2] = 0;
  op->split_at = l.n2 > 0 ? l.n1 : (bias ? l.n1 : (1 << 30));
  op->split2 = bias ? l.n1 + l.n2 : (1 << 30);
  if (!make_map(&op->map[0], (const float*)l.p1, l.n1, K, l.ld1, 32, kBK, sw))
    return false;
  if (l.n2 > 0 && !make_map(&op->map[1], (const float*)l.p2, l.n2, K, l.ld2, 32, kBK, sw))
    return false;
  if (bias && !make_map(&op->map[2], (const float*)l.ones, 1, K, 4, 32, kBK, sw))
    return false;
  if (bias && l.n2 == 0) op->map[1] = op->map[2];  // segment 1 empty: route to the ones map
  op->has3[0] = make_map3(&op->map3[0], (const float*)l.p1, l.n1, K, l.ld1, sw, atoms);
  op->has3[1] = l.n2 > 0 && make_map3(&op->map3[1], (const float*)l.p2, l.n2, K, l.ld2, sw, atoms);
  op->has3[2] = 0;
  return true;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}

// load one k-block of an operand (ROWS rows starting at r0, k from k0)
template <int ROWS>
__device__ __forceinline__ void tma_tile(const TmaOp& op, uint32_t dst, int r0, int k0, uint64_t* bar) {
  if (op.mn == 0) {
    const int seg = k0 >= op.split_at;
    tma_load_2d(dst, &op.map[seg], seg ? k0 - op.split_at : k0, r0, bar);
  } else {
    // one 3D load when the whole tile lies in a segment with a 3D view (rows
    // past the last segment's end are TMA zero fill either way)
    // (whole 128-row tiles only: narrower 3D boxes measured slower than
    // 32-row 2D boxes -- C2 step +2%, pair weight gradients +12%)
    if constexpr (ROWS % 128 == 0) {
      constexpr int kBox = 128;
      const int seg = r0 >= op.split2 ? 2 : (r0 >= op.split_at ? 1 : 0);
      const int s0 = seg == 2 ? op.split2 : (seg == 1 ? op.split_at : 0);
      const int s1 = seg == 0 ? op.split_at : (seg == 1 ? op.split2 : (1 << 30));
      if (op.has3[seg] && (r0 + ROWS <= s1 || s1 >= (1 << 30))) {
#pragma unroll
        for (int at = 0; at < ROWS / kBox; ++at)
          tma_load_3d(dst + at * kBox * 128, &op.map3[seg], 0, k0, (r0 - s0) / 32 + at * (kBox / 32), bar);
        return;
      }
    }
#pragma unroll
    for (int at = 0; at < ROWS / 32; ++at) {
      const int ra = r0 + at * 32;
      const int seg = ra >= op.split2 ? 2 : (ra >= op.split_at ? 1 : 0);
      const int c0 = seg == 2 ? ra - op.split2 : (seg == 1 ? ra - op.split_at : ra);
      tma_load_2d(dst + at * 4096, &op.map[seg], c0, k0, bar);
    }
  }
}

// Smem: a deep ring of raw (= hi) k-block stages fed by TMA, and a separate
// 2-slot ring for the converted lo copies.  Decoupling the two lets TMA run
// kR k-blocks ahead (enough to cover L2/HBM latency at full MMA rate) while
// the lo buffers, which only live from conversion to MMA completion, stay few.
//
// AT (A in TMEM, 3xTF32 with a K-major A): the converter warps read each raw
// A row from smem once, split it into hi / lo in registers and tcgen05.st both
// into TMEM; the MMAs take A from TMEM, so per k-block the smem traffic drops
// from TMA 32K + lo pass 64K + 3 MMA reads of (A + B) 96K to TMA 32K + A read
// 16K + B lo pass 32K + 3 MMA reads of B 48K (BN = 128) -- the MMA loop is
// shared-memory-bandwidth bound, so this is its speed of light lever.
template <int BN, bool AT = false>
struct SmemT {
  static constexpr int kA = kBM * 128;
  static constexpr int kB = BN * 128;
  static constexpr int kRaw = kA + kB;
  static constexpr int kLo = AT ? kB : kRaw;  // lo slot: B only when A lives in TMEM
  // lo slots: conversion of k-block q + kL waits for the MMAs of q, so kL
  // bounds how far the converters run ahead of the tensor pipe (with A in
  // TMEM each slot also takes 64 TMEM columns; kL = 2 for 64-wide tiles, to
  // stay within 256 columns, measured 2% slower at C2)
  static constexpr int kL = AT ? 4 : 3;
  // epilogue transpose staging: 8 warps x 32 rows x (16 + 4 pad) floats
  static constexpr int kEpi = 8 * 32 * 20 * 4;
  static constexpr int kR = (224 * 1024 - kL * kLo - kEpi) / kRaw;  // raw stages
  static constexpr int kBars = (2 * kR + 2 * kL + 4) * 8 + 16;
  static constexpr int kBytes = kR * kRaw + kL * kLo + kEpi + 1024 + kBars;
  static_assert(kBytes <= 232448, "smem");
};

// 16 consecutive 32-bit TMEM columns of this warp's 32 lanes <- registers
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
         "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
         "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}

// D += A(TMEM) * B(smem descriptor)
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

constexpr int kConvWarps = 8;
// epilogue: two warps per TMEM lane quarter, each draining half the columns
constexpr int kEpiWarps = 8;
constexpr int kTmaThreads = (1 + kConvWarps + 1 + kEpiWarps) * 32;  // TMA, converters, MMA, epilogue

// One 32-deep k-block of MMAs + the commits that release its buffers, issued
// by the whole (converged) MMA warp with one elected lane inside the asm, so
// descriptors stay in uniform registers (no per-MMA waterfall) and advance by
// one 64-bit add per k-step (K-major: +32 B, MN-major: +1024 B).
//   kb_at3: 3xTF32, A hi/lo in TMEM (ta = hi column; lo = ta + 32)
//   kb_ss3: 3xTF32, all operands in smem descriptors
//   kb_ss1: 1xTF32
#define GFM_KB_PRE(ACC)                                             \
  "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a0, a1, b0, b1;\n\t"        \
  ".reg .b32 h, l;\n\t"                                              \
  "elect.sync _|e, 0xffffffff;\n\t"                                  \
  "setp.ne.b32 p, " ACC ", 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
#define GFM_MMA_T(A, B, EN, ID) \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [" A "], " B ", " ID ", " EN ";\n\t"
#define GFM_MMA_S(A, B, EN, ID) \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], " A ", " B ", " ID ", " EN ";\n\t"
#define GFM_COMMIT(BAR) \
  "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [" BAR "];\n\t"
#define GFM_STEP_T(BI) \
  "add.u32 h, h, 8;\n\tadd.u32 l, l, 8;\n\tadd.s64 b0, b0, " BI ";\n\tadd.s64 b1, b1, " BI ";\n\t"
#define GFM_STEP_S(AI, BI) \
  "add.s64 a0, a0, " AI ";\n\tadd.s64 a1, a1, " AI ";\n\tadd.s64 b0, b0, " BI ";\n\tadd.s64 b1, b1, " BI ";\n\t"

__device__ __forceinline__ void kb_at3(uint32_t d, uint32_t ta, uint64_t bh, uint64_t bl,
                                       uint64_t binc, uint32_t idesc, uint32_t acc0,
                                       uint32_t bar0, uint32_t bar1) {
#define T3 GFM_MMA_T("l", "b0", "t", "%5") GFM_MMA_T("h", "b1", "t", "%5") GFM_MMA_T("h", "b0", "t", "%5")
  asm volatile(
      GFM_KB_PRE("%6")
      "mov.b64 b0, %2;\n\tmov.b64 b1, %3;\n\tmov.b32 h, %1;\n\tadd.u32 l, h, 32;\n\t"
      GFM_MMA_T("l", "b0", "p", "%5") GFM_MMA_T("h", "b1", "t", "%5") GFM_MMA_T("h", "b0", "t", "%5")
      GFM_STEP_T("%4") T3 GFM_STEP_T("%4") T3 GFM_STEP_T("%4") T3
      GFM_COMMIT("%7") GFM_COMMIT("%8") "}\n"
      :: "r"(d), "r"(ta), "l"(bh), "l"(bl), "l"(binc), "r"(idesc), "r"(acc0), "r"(bar0),
         "r"(bar1) : "memory");
#undef T3
}

__device__ __forceinline__ void kb_ss3(uint32_t d, uint64_t ah, uint64_t al, uint64_t ainc,
                                       uint64_t bh, uint64_t bl, uint64_t binc, uint32_t idesc,
                                       uint32_t acc0, uint32_t bar0, uint32_t bar1) {
#define S3 GFM_MMA_S("a1", "b0", "t", "%7") GFM_MMA_S("a0", "b1", "t", "%7") GFM_MMA_S("a0", "b0", "t", "%7")
  asm volatile(
      GFM_KB_PRE("%8")
      "mov.b64 a0, %1;\n\tmov.b64 a1, %2;\n\tmov.b64 b0, %4;\n\tmov.b64 b1, %5;\n\t"
      GFM_MMA_S("a1", "b0", "p", "%7") GFM_MMA_S("a0", "b1", "t", "%7") GFM_MMA_S("a0", "b0", "t", "%7")
      GFM_STEP_S("%3", "%6") S3 GFM_STEP_S("%3", "%6") S3 GFM_STEP_S("%3", "%6") S3
      GFM_COMMIT("%9") GFM_COMMIT("%10") "}\n"
      :: "r"(d), "l"(ah), "l"(al), "l"(ainc), "l"(bh), "l"(bl), "l"(binc), "r"(idesc),
         "r"(acc0), "r"(bar0), "r"(bar1) : "memory");
#undef S3
}

__device__ __forceinline__ void kb_ss1(uint32_t d, uint64_t ah, uint64_t ainc, uint64_t bh,
                                       uint64_t binc, uint32_t idesc, uint32_t acc0,
                                       uint32_t bar0) {
  asm volatile(
      GFM_KB_PRE("%6")
      "mov.b64 a0, %1;\n\tmov.b64 b0, %3;\n\tmov.b64 a1, 0;\n\tmov.b64 b1, 0;\n\t"
      GFM_MMA_S("a0", "b0", "p", "%5") GFM_STEP_S("%2", "%4")
      GFM_MMA_S("a0", "b0", "t", "%5") GFM_STEP_S("%2", "%4")
      GFM_MMA_S("a0", "b0", "t", "%5") GFM_STEP_S("%2", "%4")
      GFM_MMA_S("a0", "b0", "t", "%5")
      GFM_COMMIT("%7") "}\n"
      :: "r"(d), "l"(ah), "l"(ainc), "l"(bh), "l"(binc), "r"(idesc), "r"(acc0), "r"(bar0)
      : "memory");
}
#undef GFM_KB_PRE
#undef GFM_MMA_T
#undef GFM_MMA_S
#undef GFM_COMMIT
#undef GFM_STEP_T
#undef GFM_STEP_S

// AT: 0 = A in smem; 1 = A in TMEM, staged K-major SWIZZLE_128B; 2 = A in
// TMEM, staged MN-major without swizzle ([32-row atom][k][32], so converter
// lane r reads its row down the k column conflict-free)
// FLUSH: work items deeper than the flush depth (see flush_kb) accumulate in
// chunks folded into registers; shallow GEMMs take the plain instantiation
template <int BN, class Epi, int AT, bool FLUSH>
__global__ void __launch_bounds__(kTmaThreads, 1)
    tc_gemm_tma_kernel(int M, const int* __restrict__ M_dev, int N, int K, int k_chunk, int splits,
                       int split3, int fkb, const __grid_constant__ TmaOp ta,
                       const __grid_constant__ TmaOp tb, Epi epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = SmemT<BN, AT != 0>;
  // TMEM: two BN-column accumulators, then (AT) kL A slots of 32 hi + 32 lo columns
  constexpr int kACol = 2 * BN;
  constexpr int NC = tmem_cols(2 * BN + (AT ? S::kL * 64 : 0));
  constexpr int kR = S::kR, kL = S::kL;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* lo_base = base + kR * S::kRaw;
  float* epi_stage = reinterpret_cast<float*>(lo_base + kL * S::kLo);  // [8][32][20]
  uint64_t* tfl = reinterpret_cast<uint64_t*>(lo_base + kL * S::kLo + S::kEpi);  // TMA landed [kR]
  uint64_t* empty = tfl + kR;    // MMAs done with the raw stage [kR]
  uint64_t* cvt = empty + kR;    // lo written [kL]
  uint64_t* lofree = cvt + kL;   // MMAs done with the lo slot [kL]
  uint64_t* tfull = lofree + kL; // accumulator ready [2]
  uint64_t* tempty = tfull + 2;  // accumulator drained [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool split_on = split3 != 0;
  constexpr int kMmaWarp = 1 + kConvWarps;

  // prologue (barriers, descriptor prefetch, TMEM) touches no predecessor
  // output, so it runs before the programmatic-dependency wait
  if (threadIdx.x == 0) {
    for (int q = 0; q < kR; ++q) {
      mbar_init(&tfl[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < kL; ++q) {
      mbar_init(&cvt[q], kConvWarps);
      mbar_init(&lofree[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&ta.map[0]) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tb.map[0]) : "memory");
  }
  if (warp == 0) tmem_alloc<NC>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();

  const int m_total = M_dev ? *M_dev : M;
  const int m_tiles = (m_total + kBM - 1) / kBM;
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_tiles * n_tiles * splits;
  if ((int)blockIdx.x >= n_work) {
    if (warp == 0) tmem_free<NC>(tmem);
    return;
  }

  auto tile_of = [&](int w, int& bm, int& bn, int& split) {
    split = w / (m_tiles * n_tiles);
    bn = (w % (m_tiles * n_tiles)) % n_tiles;
    bm = (w % (m_tiles * n_tiles)) / n_tiles;
  };
  auto nkb_of = [&](int w) { return item_nkb(w, m_tiles * n_tiles, k_chunk, K); };
  // accumulation chunks of a work item (>= 1: an empty item still completes once)
  auto nch_of = [&](int nkb) {
    if constexpr (!FLUSH) return 1;
    return nkb > 0 ? (nkb + fkb - 1) / fkb : 1;
  };

  if (warp == 0) {
    // ============================================================ TMA producer
    if (lane == 0) {
      int p = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        int bm, bn, split;
        tile_of(w, bm, bn, split);
        const int nkb = nkb_of(w);
        for (int kb = 0; kb < nkb; ++kb, ++p) {
          const int s = p % kR;
          if (p >= kR) mbar_wait(&empty[s], ((p / kR) - 1) & 1);
          const int k0 = split * k_chunk + kb * kBK;
          const uint32_t st = smem_u32(base + s * S::kRaw);
          mbar_expect_tx(&tfl[s], S::kRaw);
          tma_tile<kBM>(ta, st, bm * kBM, k0, &tfl[s]);
          tma_tile<BN>(tb, st + S::kA, bn * BN, k0, &tfl[s]);
        }
      }
    }
  } else if (warp <= kConvWarps) {
    // ============================================================ lo converters
    if (split_on) {
      const int ctid = threadIdx.x - 32;
      int q = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int nkb = nkb_of(w);
        for (int kb = 0; kb < nkb; ++kb, ++q) {
          const int s = q % kR, l = q % kL;
          mbar_wait(&tfl[s], (q / kR) & 1);
          if (q >= kL) mbar_wait(&lofree[l], ((q / kL) - 1) & 1);
          if constexpr (AT != 0) {
            // A row r = 32 * (warp % 4) + lane (this warp's TMEM lane quarter),
            // k half h = (warp - 1) / 4 -> 16 hi / lo values
            const int q4 = warp & 3, h = (warp - 1) >> 2;
            const int r = q4 * 32 + lane;
            uint32_t hi[16], lo[16];
            if constexpr (AT == 1) {  // 4 swizzled 16-byte chunks of the row
              const uint32_t ra = smem_u32(base + s * S::kRaw) + (uint32_t)(r * 128);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t a = ra + (uint32_t)((((4 * h + j) ^ (r & 7)) & 7) << 4);
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(hi[4 * j]), "=r"(hi[4 * j + 1]), "=r"(hi[4 * j + 2]),
                               "=r"(hi[4 * j + 3]) : "r"(a));
              }
            } else {  // atom q4, column lane, k rows 16h.. (128-byte row stride)
              const uint32_t ra = smem_u32(base + s * S::kRaw) +
                                  (uint32_t)(q4 * 4096 + (16 * h) * 128 + lane * 4);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(hi[j]) : "r"(ra + 128u * j));
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const uint32_t x = hi[e];
              hi[e] = x & 0xFFFFE000u;
              lo[e] = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi[e]));
            }
            const uint32_t ta_ = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(kACol + l * 64 + 16 * h);
            tmem_st16(ta_, hi);
            tmem_st16(ta_ + 32, lo);
            make_lo<S::kB, kConvWarps * 32>(base + s * S::kRaw + S::kA, lo_base + l * S::kLo, ctid);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
          } else {
            make_lo<S::kRaw, kConvWarps * 32>(base + s * S::kRaw, lo_base + l * S::kRaw, ctid);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&cvt[l])) : "memory");
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ============================================================ MMA issuer
    // (A from TMEM is always row = lane, k = column: K-major in the idesc)
    const bool a_mn = AT == 0 && ta.mn != 0, b_mn = tb.mn != 0;
    const uint32_t idesc = make_idesc_tf32(BN, a_mn, b_mn);
    // k-step 0 descriptor; later k-steps add ainc / binc (address field is >> 4)
    auto desc0 = [&](bool mn, uint32_t addr) -> uint64_t {
      return mn ? make_desc_mn(addr, 4096, 512) : make_desc(addr);
    };
    const uint64_t ainc = a_mn ? 1024 >> 4 : 32 >> 4, binc = b_mn ? 1024 >> 4 : 32 >> 4;
    int q = 0, t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
     const int nkb = nkb_of(w), nch = nch_of(nkb);
     for (int ch = 0; ch < nch; ++ch, ++t) {  // one accumulator per chunk
      const int acc = t & 1;
      if (t >= 2) mbar_wait(&tempty[acc], ((t >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * BN);
      const int kb_end = min(nkb, (ch + 1) * fkb);
      for (int kb = ch * fkb; kb < kb_end; ++kb, ++q) {
        const int s = q % kR, l = q % kL;
        mbar_wait(&tfl[s], (q / kR) & 1);
        if (split_on) mbar_wait(&cvt[l], (q / kL) & 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(base + s * S::kRaw), bh = ah + S::kA;
        const uint32_t al = smem_u32(lo_base + l * S::kLo), bl = AT != 0 ? al : al + S::kA;
        const uint32_t acc0 = kb > ch * fkb ? 1u : 0u;
        const uint32_t e_bar = smem_u32(&empty[s]), l_bar = smem_u32(&lofree[l]);
        if constexpr (AT != 0) {
          kb_at3(d, tmem + (uint32_t)(kACol + l * 64), desc0(b_mn, bh), desc0(b_mn, bl), binc,
                 idesc, acc0, e_bar, l_bar);
        } else if (split_on) {
          kb_ss3(d, desc0(a_mn, ah), desc0(a_mn, al), ainc, desc0(b_mn, bh), desc0(b_mn, bl),
                 binc, idesc, acc0, e_bar, l_bar);
        } else {
          kb_ss1(d, desc0(a_mn, ah), ainc, desc0(b_mn, bh), binc, idesc, acc0, e_bar);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (nkb > 0)
          mma_commit(&tfull[acc]);
        else
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tfull[acc])) : "memory");
      }
      __syncwarp();
     }
    }
  } else {
    // ============================================================ epilogue
    const int quarter = warp & 3;                       // TMEM lanes 32 * quarter ..
    const int half = (warp - (kMmaWarp + 1)) / 4;       // column half of the tile
    constexpr int kHalf = BN / 2 >= 16 ? BN / 2 : 16;
    int t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      int bm, bn, split;
      tile_of(w, bm, bn, split);
      const int nkb = nkb_of(w), nch = nch_of(nkb);
      // chunks before the last: fold each TMEM partial into fp32 registers
      // (IEEE adds, in chunk order) and hand the accumulator back at once
      constexpr int kRegs = (BN / 2 >= 16 ? BN / 2 : 16);
      float racc[kRegs];
      const int c_lo = half * kHalf, c_hi = min(BN, (half + 1) * kHalf);
      for (int ch = 0; ch + 1 < nch; ++ch, ++t) {
        const int acc = t & 1;
        mbar_wait(&tfull[acc], (t >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < kRegs / 16; ++j) {
          if (c_lo + 16 * j >= c_hi) continue;
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c_lo + 16 * j), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) racc[16 * j + i] = ch == 0 ? v[i] : racc[16 * j + i] + v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tempty[acc])) : "memory");
      }
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const int m0 = bm * kBM, n0 = bn * BN;
      // per 16-column chunk: registers (row = lane) -> this warp's smem stage
      // -> read back transposed so each store instruction writes 8 rows x 64
      // contiguous bytes (full sectors) instead of 32 rows x 16 bytes
      float* stg = epi_stage + (warp - (kMmaWarp + 1)) * (32 * 20);
      const int m_lim = min(kBM, m_total - m0);
      auto store16 = [&](int c, const float (&v)[16]) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(stg + lane * 20 + 4 * q) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
        if constexpr (HasPrefetch<Epi>::value) {
          decltype(epi.prefetch(0, 0)) pre[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3;
            const int col = n0 + c + 4 * q;
            const int rr = quarter * 32 + r;
            if (rr < m_lim && col < N) pre[j] = epi.prefetch(m0 + rr, col);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3;
            const int col = n0 + c + 4 * q;
            const int rr = quarter * 32 + r;
            if (rr < m_lim && col < N)
              epi.store4(m0 + rr, col, *reinterpret_cast<const float4*>(stg + r * 20 + 4 * q),
                         min(4, N - col), split, pre[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3;
            const int col = n0 + c + 4 * q;
            const int rr = quarter * 32 + r;
            if (rr < m_lim && col < N)
              epi.store4(m0 + rr, col, *reinterpret_cast<const float4*>(stg + r * 20 + 4 * q),
                         min(4, N - col), split);
          }
        }
        __syncwarp();
      };
      if (nch > 1) {
        // last chunk: fold it too and hand the accumulator back BEFORE the
        // stores, so the next tile's MMAs are not held up by this epilogue
#pragma unroll
        for (int j = 0; j < kRegs / 16; ++j) {
          if (c_lo + 16 * j >= c_hi) continue;
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c_lo + 16 * j), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) racc[16 * j + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tempty[acc])) : "memory");
#pragma unroll
        for (int j = 0; j < kRegs / 16; ++j) {
          const int c = c_lo + 16 * j;
          if (c >= c_hi || n0 + c >= N) continue;
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = racc[16 * j + i];
          store16(c, v);
        }
        continue;
      }
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        if (nkb > 0) {
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c), v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (n0 + c >= N) continue;
        store16(c, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tempty[acc])) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<NC>(tmem);
}

// ---------------------------------------------------------------- CTA pairs
// cta_group::2 variant of the A-in-TMEM 3xTF32 kernel: a cluster of two CTAs
// (one TPC) computes a 256 x BN tile with M = 256 MMAs issued by the leader.
// Each CTA stages its own 128 A rows (converted into its own TMEM, as in the
// single-CTA kernel) and HALF of the BN B rows (raw + lo): the tensor cores
// read each B half from its owner's smem, so per SM the TMA bytes, the B lo
// pass and the MMAs' B reads halve (per 32-deep k-block and SM ~80 KB of
// shared-memory traffic instead of ~128 KB) while the MMA time per SM stays.
// Barriers: TMA landed / ring free / lo free / accumulator full are per CTA
// (the leader's commits multicast to both); lo written and accumulator
// drained live in the leader and count both CTAs' warps.
template <int BN>
struct SmemP {
  static constexpr int kA = kBM * 128;
  static constexpr int kB = (BN / 2) * 128;  // this CTA's half of the B rows
  static constexpr int kRaw = kA + kB;
  static constexpr int kLo = kB;
  static constexpr int kL = 4;
  static constexpr int kEpi = 8 * 32 * 20 * 4;
  static constexpr int kR = (224 * 1024 - kL * kLo - kEpi) / kRaw;
  static constexpr int kBars = (2 * kR + 2 * kL + 4) * 8 + 16;
  static constexpr int kBytes = kR * kRaw + kL * kLo + kEpi + 1024 + kBars;
  static_assert(kBytes <= 232448, "smem");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of p's twin in CTA `rank` of the pair
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) { return peer_addr(p, 0); }
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  // default (.release.cta) semantics, as CUTLASS's ClusterBarrier: a
  // .release.cluster arrive costs a cluster-scope MEMBAR per k-block
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(caddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n"
      :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// commit the leader's MMAs to the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      :: "r"(smem_u32(bar)), "h"((unsigned short)3) : "memory");
}

// kb_at3 with M = 256 pair MMAs (A from both CTAs' TMEM, B halves from both
// CTAs' smem) and multicast commits
__device__ __forceinline__ void kb_at3_pair(uint32_t d, uint32_t ta, uint64_t bh, uint64_t bl,
                                            uint64_t binc, uint32_t idesc, uint32_t acc0,
                                            uint32_t bar0, uint32_t bar1) {
#define GFM_P_MMA(A, B, EN) \
  "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [" A "], " B ", %5, " EN ";\n\t"
#define GFM_P_T3 GFM_P_MMA("l", "b0", "t") GFM_P_MMA("h", "b1", "t") GFM_P_MMA("h", "b0", "t")
#define GFM_P_STEP \
  "add.u32 h, h, 8;\n\tadd.u32 l, l, 8;\n\tadd.s64 b0, b0, %4;\n\tadd.s64 b1, b1, %4;\n\t"
#define GFM_P_COMMIT(BAR) \
  "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [" BAR "], m;\n\t"
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 b0, b1;\n\t.reg .b32 h, l;\n\t.reg .b16 m;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b16 m, 3;\n\t"
      "mov.b64 b0, %2;\n\tmov.b64 b1, %3;\n\tmov.b32 h, %1;\n\tadd.u32 l, h, 32;\n\t"
      GFM_P_MMA("l", "b0", "p") GFM_P_MMA("h", "b1", "t") GFM_P_MMA("h", "b0", "t")
      GFM_P_STEP GFM_P_T3 GFM_P_STEP GFM_P_T3 GFM_P_STEP GFM_P_T3
      GFM_P_COMMIT("%7") GFM_P_COMMIT("%8") "}\n"
      :: "r"(d), "r"(ta), "l"(bh), "l"(bl), "l"(binc), "r"(idesc), "r"(acc0), "r"(bar0),
         "r"(bar1) : "memory");
#undef GFM_P_MMA
#undef GFM_P_T3
#undef GFM_P_STEP
#undef GFM_P_COMMIT
}

template <int BN, class Epi, int AT, bool FLUSH>
__global__ void __launch_bounds__(kTmaThreads, 1)
    tc_gemm_tma_pair_kernel(int M, const int* __restrict__ M_dev, int N, int K, int k_chunk, int splits,
                       int split3, int fkb, const __grid_constant__ TmaOp ta,
                       const __grid_constant__ TmaOp tb, Epi epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  static_assert(AT != 0 && BN >= 64, "pairs: A in TMEM, B halves of >= 32 rows");
  using S = SmemP<BN>;
  // TMEM: two BN-column accumulators, then (AT) kL A slots of 32 hi + 32 lo columns
  constexpr int kACol = 2 * BN;
  constexpr int NC = tmem_cols(2 * BN + (AT ? S::kL * 64 : 0));
  constexpr int kR = S::kR, kL = S::kL;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* lo_base = base + kR * S::kRaw;
  float* epi_stage = reinterpret_cast<float*>(lo_base + kL * S::kLo);  // [8][32][20]
  uint64_t* tfl = reinterpret_cast<uint64_t*>(lo_base + kL * S::kLo + S::kEpi);  // TMA landed [kR]
  uint64_t* empty = tfl + kR;    // MMAs done with the raw stage [kR]
  uint64_t* cvt = empty + kR;    // lo written [kL]
  uint64_t* lofree = cvt + kL;   // MMAs done with the lo slot [kL]
  uint64_t* tfull = lofree + kL; // accumulator ready [2]
  uint64_t* tempty = tfull + 2;  // accumulator drained [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool split_on = split3 != 0;
  constexpr int kMmaWarp = 1 + kConvWarps;

  // prologue (barriers, descriptor prefetch, TMEM) touches no predecessor
  // output, so it runs before the programmatic-dependency wait
  if (threadIdx.x == 0) {
    for (int q = 0; q < kR; ++q) {
      mbar_init(&tfl[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < kL; ++q) {
      mbar_init(&cvt[q], 2 * kConvWarps);  // both CTAs' converters (leader's copy)
      mbar_init(&lofree[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], 2 * kEpiWarps);  // both CTAs' epilogues (leader's copy)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&ta.map[0]) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tb.map[0]) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_slot)), "n"(NC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits and the TMEM address visible pair-wide
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();

  const int rank = (int)cluster_rank();
  const int cid = (int)blockIdx.x >> 1, ncl = (int)gridDim.x >> 1;
  const int m_total = M_dev ? *M_dev : M;
  const int m_tiles = (m_total + kBM - 1) / kBM;
  const int m_pairs = (m_tiles + 1) / 2;  // a pair owns m tiles 2p (leader) and 2p + 1
  const int n_tiles = (N + BN - 1) / BN;
  const int n_work = m_pairs * n_tiles * splits;

  auto tile_of = [&](int w, int& bm, int& bn, int& split) {
    split = w / (m_pairs * n_tiles);
    bn = (w % (m_pairs * n_tiles)) % n_tiles;
    bm = 2 * ((w % (m_pairs * n_tiles)) / n_tiles) + rank;
  };
  auto nkb_of = [&](int w) { return item_nkb(w, m_pairs * n_tiles, k_chunk, K); };
  // accumulation chunks of a work item (>= 1: an empty item still completes once)
  auto nch_of = [&](int nkb) {
    if constexpr (!FLUSH) return 1;
    return nkb > 0 ? (nkb + fkb - 1) / fkb : 1;
  };

  if (cid >= n_work) {
    // no work for this pair: straight to the teardown
  } else if (warp == 0) {
    // ============================================================ TMA producer
    if (lane == 0) {
      int p = 0;
      for (int w = cid; w < n_work; w += ncl) {
        int bm, bn, split;
        tile_of(w, bm, bn, split);
        const int nkb = nkb_of(w);
        for (int kb = 0; kb < nkb; ++kb, ++p) {
          const int s = p % kR;
          if (p >= kR) mbar_wait_cl(&empty[s], ((p / kR) - 1) & 1);
          const int k0 = split * k_chunk + kb * kBK;
          const uint32_t st = smem_u32(base + s * S::kRaw);
          mbar_expect_tx(&tfl[s], S::kRaw);
          tma_tile<kBM>(ta, st, bm * kBM, k0, &tfl[s]);
          tma_tile<BN / 2>(tb, st + S::kA, bn * BN + rank * (BN / 2), k0, &tfl[s]);
        }
      }
    }
  } else if (warp <= kConvWarps) {
    // ============================================================ lo converters
    if (split_on) {
      const int ctid = threadIdx.x - 32;
      int q = 0;
      for (int w = cid; w < n_work; w += ncl) {
        const int nkb = nkb_of(w);
        for (int kb = 0; kb < nkb; ++kb, ++q) {
          const int s = q % kR, l = q % kL;
          mbar_wait(&tfl[s], (q / kR) & 1);
          if (q >= kL) mbar_wait_cl(&lofree[l], ((q / kL) - 1) & 1);
          if constexpr (AT != 0) {
            // A row r = 32 * (warp % 4) + lane (this warp's TMEM lane quarter),
            // k half h = (warp - 1) / 4 -> 16 hi / lo values
            const int q4 = warp & 3, h = (warp - 1) >> 2;
            const int r = q4 * 32 + lane;
            uint32_t hi[16], lo[16];
            if constexpr (AT == 1) {  // 4 swizzled 16-byte chunks of the row
              const uint32_t ra = smem_u32(base + s * S::kRaw) + (uint32_t)(r * 128);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t a = ra + (uint32_t)((((4 * h + j) ^ (r & 7)) & 7) << 4);
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(hi[4 * j]), "=r"(hi[4 * j + 1]), "=r"(hi[4 * j + 2]),
                               "=r"(hi[4 * j + 3]) : "r"(a));
              }
            } else {  // atom q4, column lane, k rows 16h.. (128-byte row stride)
              const uint32_t ra = smem_u32(base + s * S::kRaw) +
                                  (uint32_t)(q4 * 4096 + (16 * h) * 128 + lane * 4);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(hi[j]) : "r"(ra + 128u * j));
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const uint32_t x = hi[e];
              hi[e] = x & 0xFFFFE000u;
              lo[e] = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi[e]));
            }
            const uint32_t ta_ = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(kACol + l * 64 + 16 * h);
            tmem_st16(ta_, hi);
            tmem_st16(ta_ + 32, lo);
            make_lo<S::kB, kConvWarps * 32>(base + s * S::kRaw + S::kA, lo_base + l * S::kLo, ctid);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
          } else {
            make_lo<S::kRaw, kConvWarps * 32>(base + s * S::kRaw, lo_base + l * S::kRaw, ctid);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&cvt[l]));
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (rank != 0) {
      // the leader's MMA warp issues for the pair
    } else {
    // ============================================================ MMA issuer
    // (A from TMEM is always row = lane, k = column: K-major in the idesc)
    const bool a_mn = AT == 0 && ta.mn != 0, b_mn = tb.mn != 0;
    const uint32_t idesc = make_idesc_tf32(BN, a_mn, b_mn) + ((uint32_t)(kBM >> 4) << 24);  // M = 256
    // k-step 0 descriptor; later k-steps add ainc / binc (address field is >> 4)
    auto desc0 = [&](bool mn, uint32_t addr) -> uint64_t {
      return mn ? make_desc_mn(addr, 4096, 512) : make_desc(addr);
    };
    const uint64_t ainc = a_mn ? 1024 >> 4 : 32 >> 4, binc = b_mn ? 1024 >> 4 : 32 >> 4;
    int q = 0, t = 0;
    for (int w = cid; w < n_work; w += ncl) {
     const int nkb = nkb_of(w), nch = nch_of(nkb);
     for (int ch = 0; ch < nch; ++ch, ++t) {  // one accumulator per chunk
      const int acc = t & 1;
      if (t >= 2) mbar_wait_cl(&tempty[acc], ((t >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * BN);
      const int kb_end = min(nkb, (ch + 1) * fkb);
      for (int kb = ch * fkb; kb < kb_end; ++kb, ++q) {
        const int s = q % kR, l = q % kL;
        mbar_wait_cl(&cvt[l], (q / kL) & 1);  // both CTAs' rows landed and converted
        tc_fence_after();
        const uint32_t ah = smem_u32(base + s * S::kRaw), bh = ah + S::kA;
        const uint32_t al = smem_u32(lo_base + l * S::kLo), bl = AT != 0 ? al : al + S::kA;
        const uint32_t acc0 = kb > ch * fkb ? 1u : 0u;
        const uint32_t e_bar = smem_u32(&empty[s]), l_bar = smem_u32(&lofree[l]);
        (void)ah;
        kb_at3_pair(d, tmem + (uint32_t)(kACol + l * 64), desc0(b_mn, bh), desc0(b_mn, bl), binc,
                    idesc, acc0, e_bar, l_bar);
        __syncwarp();
      }
      if (lane == 0) {
        if (nkb > 0) {
          mma_commit_pair(&tfull[acc]);
        } else {  // empty item: complete both CTAs' accumulators by hand
          mbar_arrive_cluster(peer_addr(&tfull[acc], 0));
          mbar_arrive_cluster(peer_addr(&tfull[acc], 1));
        }
      }
      __syncwarp();
     }
    }
    }
  } else {
    // ============================================================ epilogue
    const int quarter = warp & 3;                       // TMEM lanes 32 * quarter ..
    const int half = (warp - (kMmaWarp + 1)) / 4;       // column half of the tile
    constexpr int kHalf = BN / 2 >= 16 ? BN / 2 : 16;
    int t = 0;
    for (int w = cid; w < n_work; w += ncl, ++t) {
      int bm, bn, split;
      tile_of(w, bm, bn, split);
      const int nkb = nkb_of(w), nch = nch_of(nkb);
      // chunks before the last: fold each TMEM partial into fp32 registers
      // (IEEE adds, in chunk order) and hand the accumulator back at once
      constexpr int kRegs = (BN / 2 >= 16 ? BN / 2 : 16);
      float racc[kRegs];
      const int c_lo = half * kHalf, c_hi = min(BN, (half + 1) * kHalf);
      for (int ch = 0; ch + 1 < nch; ++ch, ++t) {
        const int acc = t & 1;
        mbar_wait_cl(&tfull[acc], (t >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < kRegs / 16; ++j) {
          if (c_lo + 16 * j >= c_hi) continue;
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c_lo + 16 * j), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) racc[16 * j + i] = ch == 0 ? v[i] : racc[16 * j + i] + v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[acc]));
      }
      const int acc = t & 1;
      mbar_wait_cl(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const int m0 = bm * kBM, n0 = bn * BN;
      // per 16-column chunk: registers (row = lane) -> this warp's smem stage
      // -> read back transposed so each store instruction writes 8 rows x 64
      // contiguous bytes (full sectors) instead of 32 rows x 16 bytes
      float* stg = epi_stage + (warp - (kMmaWarp + 1)) * (32 * 20);
      const int m_lim = min(kBM, m_total - m0);
      auto store16 = [&](int c, const float (&v)[16]) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(stg + lane * 20 + 4 * q) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
        if constexpr (HasPrefetch<Epi>::value) {
          decltype(epi.prefetch(0, 0)) pre[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3;
            const int col = n0 + c + 4 * q;
            const int rr = quarter * 32 + r;
            if (rr < m_lim && col < N) pre[j] = epi.prefetch(m0 + rr, col);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3;
            const int col = n0 + c + 4 * q;
            const int rr = quarter * 32 + r;
            if (rr < m_lim && col < N)
              epi.store4(m0 + rr, col, *reinterpret_cast<const float4*>(stg + r * 20 + 4 * q),
                         min(4, N - col), split, pre[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), q = lane & 3;
            const int col = n0 + c + 4 * q;
            const int rr = quarter * 32 + r;
            if (rr < m_lim && col < N)
              epi.store4(m0 + rr, col, *reinterpret_cast<const float4*>(stg + r * 20 + 4 * q),
                         min(4, N - col), split);
          }
        }
        __syncwarp();
      };
      if (nch > 1) {
        // last chunk: fold it too and hand the accumulator back BEFORE the
        // stores, so the next tile's MMAs are not held up by this epilogue
#pragma unroll
        for (int j = 0; j < kRegs / 16; ++j) {
          if (c_lo + 16 * j >= c_hi) continue;
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c_lo + 16 * j), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) racc[16 * j + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[acc]));
#pragma unroll
        for (int j = 0; j < kRegs / 16; ++j) {
          const int c = c_lo + 16 * j;
          if (c >= c_hi || n0 + c >= N) continue;
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = racc[16 * j + i];
          store16(c, v);
        }
        continue;
      }
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        if (nkb > 0) {
          tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + c), v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (n0 + c >= N) continue;
        store16(c, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[acc]));
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the peer no longer touches this CTA's smem / barriers
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(NC));
}

template <int BN, class AL, class BL, class Epi>
inline cudaError_t launch_bn(int M, const int* M_dev, int N, int K, const int* K_dev, int splits,
                             int split3, AL a, BL b, Epi epi, cudaStream_t s) {
  int k_chunk = ceil_div(ceil_div(K > 0 ? K : 1, splits), kBK) * kBK;
  splits = ceil_div(K > 0 ? K : 1, k_chunk);
  const long long work = (long long)ceil_div(M, kBM) * ceil_div(N, BN) * splits;
  const int grid = (int)std::min<long long>(work, 148LL);
  if (!K_dev && !tma_disabled()) {
    TmaOp ta, tb;
    if (build_tma(a, &ta, kBM, M, K) && build_tma(b, &tb, BN, N, K)) {
      // 3xTF32: A goes through TMEM (K-major as staged; MN-major re-mapped
      // without swizzle for the converters)
      int at = 0;
      if (split3 != 0 && !at_disabled()) {
        if (ta.mn == 0)
          at = 1;
        else if (build_tma(a, &ta, kBM, M, K, CU_TENSOR_MAP_SWIZZLE_NONE))
          at = 2;
        else
          build_tma(a, &ta, kBM, M, K);
      }
      const bool flush = ceil_div(k_chunk, kBK) > flush_kb();
      if constexpr (BN >= 64) {
        // CTA pairs (cta_group::2): B halves per CTA
        TmaOp tbh;
        // (K-major A only: with the MN-major A of the weight gradients the
        // pair kernel measured 28% slower, forward / backward-data 4-8% faster)
        // (deep GEMMs only: below K = 512 -- every C2 GEMM -- the pair's
        // cluster launch and cross-CTA handshakes cost more than it saves)
        if (at == 1 && pairs_enabled() && ceil_div(M, kBM) >= 2 && K >= 512 &&
            build_tma(b, &tbh, BN / 2, N, K)) {
          auto kp = flush ? (at == 1 ? tc_gemm_tma_pair_kernel<BN, Epi, 1, true>
                                     : tc_gemm_tma_pair_kernel<BN, Epi, 2, true>)
                          : (at == 1 ? tc_gemm_tma_pair_kernel<BN, Epi, 1, false>
                                     : tc_gemm_tma_pair_kernel<BN, Epi, 2, false>);
          const int smem = SmemP<BN>::kBytes;
          cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          if (e != cudaSuccess) return e;
          // persistent: as many pairs as can be co-resident (not every TPC
          // may take a pair of these 1-CTA-per-SM CTAs at once; a second
          // wave of pairs would double the time of a persistent kernel)
          static int max_pairs = 0;
          if (max_pairs == 0) {
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(148);
            qc.blockDim = dim3(kTmaThreads);
            qc.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 2;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            qc.attrs = qa;
            qc.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kp, &qc) != cudaSuccess || n <= 0) n = 64;
            max_pairs = n < 74 ? n : 74;
            if (getenv("GFM_TC_DEBUG")) fprintf(stderr, "tc pairs: %d co-resident (BN %d)\n", n, BN);
          }
          const long long pw = (long long)ceil_div(ceil_div(M, kBM), 2) * ceil_div(N, BN) * splits;
          const int pgrid = 2 * (int)std::min<long long>(pw, (long long)max_pairs);
          launch_kc(kp, pgrid, kTmaThreads, smem, s, 2, M, M_dev, N, K, k_chunk, splits, split3,
                    flush_kb(), ta, tbh, epi);
          ++g_pair_launches;
          return cudaGetLastError();
        }
      }
      auto kern = flush ? (at == 1   ? tc_gemm_tma_kernel<BN, Epi, 1, true>
                           : at == 2 ? tc_gemm_tma_kernel<BN, Epi, 2, true>
                                     : tc_gemm_tma_kernel<BN, Epi, 0, true>)
                        : (at == 1   ? tc_gemm_tma_kernel<BN, Epi, 1, false>
                           : at == 2 ? tc_gemm_tma_kernel<BN, Epi, 2, false>
                                     : tc_gemm_tma_kernel<BN, Epi, 0, false>);
      const int smem = at ? SmemT<BN, true>::kBytes : SmemT<BN, false>::kBytes;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      launch_k(kern, grid, kTmaThreads, smem, s, M, M_dev, N, K, k_chunk, splits, split3,
               flush_kb(), ta, tb, epi);
      return cudaGetLastError();
    }
  }
  const int smem = Smem<BN>::kBytes;
  const bool va = a.vec_ok(K), vb = b.vec_ok(K);
  auto kern = va ? (vb ? tc_gemm_kernel<BN, true, true, AL, BL, Epi>
                       : tc_gemm_kernel<BN, true, false, AL, BL, Epi>)
                 : (vb ? tc_gemm_kernel<BN, false, true, AL, BL, Epi>
                       : tc_gemm_kernel<BN, false, false, AL, BL, Epi>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  launch_k(kern, grid, kWSThreads, smem, s, M, M_dev, N, K, K_dev, k_chunk, splits, split3, a, b, epi);
  return cudaGetLastError();
}

inline int bn_cap() {  // GFM_TC_BN_MAX (32 / 64 / 128) caps the column tile (A/B runs)
  static int v = -1;
  if (v < 0) v = getenv("GFM_TC_BN_MAX") ? atoi(getenv("GFM_TC_BN_MAX")) : 128;
  return v;
}
inline int pick_bn(int n) {
  const int bn = n <= 32 ? 32 : n <= 64 ? 64 : 128;
  return bn < bn_cap() ? bn : (bn_cap() >= 128 ? 128 : bn_cap() >= 64 ? 64 : 32);
}

// BN from N (32 / 64 / 128; N > 128 is tiled in 128-wide column tiles)
template <class AL, class BL, class Epi>
inline cudaError_t launch(int M, const int* M_dev, int N, int K, const int* K_dev, int splits,
                          int split3, AL a, BL b, Epi epi, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (splits < 1) splits = 1;
  switch (pick_bn(N)) {
    case 32: return launch_bn<32>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
    case 64: return launch_bn<64>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
    default: return launch_bn<128>(M, M_dev, N, K, K_dev, splits, split3, a, b, epi, s);
  }
}

// Number of K splits for weight-gradient GEMMs (shape-only -> deterministic):
// enough (tile x split) work items to give every SM one, chunks >= 256.
inline int splits_for(long long M, long long N, long long K) {
  long long tiles = (long long)ceil_div(M, kBM) * ceil_div(N, pick_bn((int)std::min<long long>(N, 128)));
  long long want = (148LL + tiles - 1) / tiles;
  long long max_by_k = (K + 255) / 256;
  // <= 8192-deep fp32 TMEM accumulations (error ~ sqrt(depth) * 2^-24 stays
  // ~1e-5 relative, far inside the 3xTF32 bound); the split partials are summed
  // in fp64
  long long min_by_k = (K + 8191) / 8192;
  long long s = want < max_by_k ? want : max_by_k;
  if (s < min_by_k) s = min_by_k;
  if (s < 1) s = 1;
  if (s > 512) s = 512;
  return (int)s;
}

// ---------------------------------------------------------------- epilogues
// Epilogue stores: 16 consecutive floats per thread-row; when the whole chunk
// is valid and 16-byte aligned they go out as 4 x st.global.v4 (2 full
// sectors per thread), else element by element.
__device__ __forceinline__ bool chunk_vec(const void* p, int nv) {
  return nv == 16 && (((uintptr_t)p) & 15) == 0;
}
// 4 consecutive outputs (nv valid) -> one st.global.v4 when aligned
__device__ __forceinline__ void put4(float* o, const float (&x)[4], int nv) {
  if (nv == 4 && (((uintptr_t)o) & 15) == 0) {
    *reinterpret_cast<float4*>(o) = make_float4(x[0], x[1], x[2], x[3]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < nv) o[i] = x[i];
  }
}

struct TcEpiBiasAct {  // out[m][n] = act(acc + bias[n])
  float* out;
  int ldo;
  const float* bias;
  int act;
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv, int) const {
    if (!valid) return;
    float* o = out + (long long)m * ldo + n;
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float t = v[i] + (bias && i < nv ? bias[n + i] : 0.f);
      x[i] = act ? tanh_fast(t) : t;
    }
    if (chunk_vec(o, nv)) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<float4*>(o)[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nv) o[i] = x[i];
    }
  }
  __device__ void store4(int m, int n, float4 v, int nv, int) const;
};

// (TcEpiBiasAct::store4) the transposed-epilogue entry: row m, columns n..n+3
__device__ __forceinline__ void bias_act4(float (&x)[4], const float* bias, int n, int nv, int act) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float t = x[i] + (bias && i < nv ? bias[n + i] : 0.f);
    x[i] = act ? tanh_fast(t) : t;
  }
}

__device__ __forceinline__ void TcEpiBiasAct::store4(int m, int n, float4 v, int nv, int) const {
  float x[4] = {v.x, v.y, v.z, v.w};
  bias_act4(x, bias, n, nv, act);
  put4(out + (long long)m * ldo + n, x, nv);
}

struct TcEpiSplitCols {  // cols [0, n1) -> o1 (+ add, * (1 - gate^2)), [n1, N) -> o2
  float* o1;
  int ld1, n1;
  float* o2;
  int ld2;
  const float* gate;
  int ldg;
  const float* add;  // optional addend on the o1 columns (row stride ld1), before the gate
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv, int) const {
    if (!valid) return;
    if (n + 16 <= n1 || n >= n1) {  // chunk entirely in one output
      const bool first = n < n1;
      float* o = first ? o1 + (long long)m * ld1 + n : o2 + (long long)m * ld2 + (n - n1);
      float x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = v[i];
      if (first && (add || gate)) {
        const float* ap = add ? add + (long long)m * ld1 + n : nullptr;
        const float* gp = gate ? gate + (long long)m * ldg + n : nullptr;
        if (nv == 16 && (!ap || chunk_vec(ap, 16)) && (!gp || chunk_vec(gp, 16))) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (ap) {
              const float4 a4 = reinterpret_cast<const float4*>(ap)[q];
              x[4 * q] = a4.x + x[4 * q]; x[4 * q + 1] = a4.y + x[4 * q + 1];
              x[4 * q + 2] = a4.z + x[4 * q + 2]; x[4 * q + 3] = a4.w + x[4 * q + 3];
            }
            if (gp) {
              const float4 g4 = reinterpret_cast<const float4*>(gp)[q];
              x[4 * q] *= 1.f - g4.x * g4.x; x[4 * q + 1] *= 1.f - g4.y * g4.y;
              x[4 * q + 2] *= 1.f - g4.z * g4.z; x[4 * q + 3] *= 1.f - g4.w * g4.w;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i >= nv) continue;
            if (ap) x[i] = ap[i] + x[i];
            if (gp) x[i] *= 1.f - gp[i] * gp[i];
          }
        }
      }
      if (chunk_vec(o, nv)) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          reinterpret_cast<float4*>(o)[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < nv) o[i] = x[i];
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i >= nv) continue;
      const int c = n + i;
      float x = v[i];
      if (c < n1) {
        if (add) x = add[(long long)m * ld1 + c] + x;
        if (gate) {
          const float gg = gate[(long long)m * ldg + c];
          x *= 1.f - gg * gg;
        }
        o1[(long long)m * ld1 + c] = x;
      } else {
        o2[(long long)m * ld2 + (c - n1)] = x;
      }
    }
  }
  __device__ void store4(int m, int n, float4 v, int nv, int) const;
};

__device__ __forceinline__ void split_cols4(const TcEpiSplitCols& e, int m, int n, float4 v,
                                            int nv) {
  float x[4] = {v.x, v.y, v.z, v.w};
  if (n + 4 <= e.n1 || n >= e.n1) {
    const bool first = n < e.n1;
    if (first && (e.add || e.gate)) {
      const float* ap = e.add ? e.add + (long long)m * e.ld1 + n : nullptr;
      const float* gp = e.gate ? e.gate + (long long)m * e.ldg + n : nullptr;
      if (nv == 4 && (!ap || (((uintptr_t)ap) & 15) == 0) && (!gp || (((uintptr_t)gp) & 15) == 0)) {
        if (ap) {
          const float4 a4 = *reinterpret_cast<const float4*>(ap);
          x[0] = a4.x + x[0]; x[1] = a4.y + x[1]; x[2] = a4.z + x[2]; x[3] = a4.w + x[3];
        }
        if (gp) {
          const float4 g4 = *reinterpret_cast<const float4*>(gp);
          x[0] *= 1.f - g4.x * g4.x; x[1] *= 1.f - g4.y * g4.y;
          x[2] *= 1.f - g4.z * g4.z; x[3] *= 1.f - g4.w * g4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= nv) continue;
          if (ap) x[i] = ap[i] + x[i];
          if (gp) x[i] *= 1.f - gp[i] * gp[i];
        }
      }
    }
    put4(first ? e.o1 + (long long)m * e.ld1 + n : e.o2 + (long long)m * e.ld2 + (n - e.n1), x, nv);
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nv) continue;
    const int c = n + i;
    float y = x[i];
    if (c < e.n1) {
      if (e.add) y = e.add[(long long)m * e.ld1 + c] + y;
      if (e.gate) {
        const float gg = e.gate[(long long)m * e.ldg + c];
        y *= 1.f - gg * gg;
      }
      e.o1[(long long)m * e.ld1 + c] = y;
    } else {
      e.o2[(long long)m * e.ld2 + (c - e.n1)] = y;
    }
  }
}

__device__ __forceinline__ void TcEpiSplitCols::store4(int m, int n, float4 v, int nv, int) const {
  split_cols4(*this, m, n, v, nv);
}

// Layer backward-data fused with the PNA aggregation-backward prep
// (model.py:549-558 + 325-341): columns [0, H) are dh_in = dz W; columns
// [H, 5H) are dz U with U's columns PERMUTED channel-major (4c + p, parts
// sum | mean | max | std), so every 4-column store holds one channel's four
// part gradients and the epilogue writes the gather's inputs directly:
//   G = dsum + dmean / deg - coef * mean,  coef = dstd / (deg * std) (std > 0)
//   dmax  (read by the argmax-routed gather)
// -- the [N][4H] dagg never reaches memory and the prep pass disappears.
struct TcEpiAggPrep {
  float* dh;  // [M][H] (ld H)
  int H;
  float* G;
  float* coef;
  float* dmax;
  const float* agg;    // [M][4H] forward output (std part at column 3H)
  const float* smean;  // [M][H]
  const int* rowptr;
  struct Pre {
    int deg;
    float sd, mu;
  };
  __device__ Pre prefetch(int m, int n) const {
    Pre p{0, 0.f, 0.f};
    if (n >= H) {
      const int c = (n - H) >> 2;
      p.deg = __ldg(rowptr + m + 1) - __ldg(rowptr + m);
      p.sd = __ldg(agg + (long long)m * 4 * H + 3 * H + c);
      p.mu = __ldg(smean + (long long)m * H + c);
    }
    return p;
  }
  __device__ void store4(int m, int n, float4 v, int nv, int, const Pre& p) const {
    if (n < H) {
      const float x[4] = {v.x, v.y, v.z, v.w};
      put4(dh + (long long)m * H + n, x, nv);
      return;
    }
    const int c = (n - H) >> 2;
    float g = v.x;
    if (p.deg > 0) g += __fdiv_rn(v.y, (float)p.deg);
    float cf = 0.f;
    if (p.deg > 0 && p.sd > 0.f) {
      const float k = v.w / ((float)p.deg * p.sd);
      g -= k * p.mu;
      cf = k;
    }
    const long long o = (long long)m * H + c;
    G[o] = g;
    coef[o] = cf;
    dmax[o] = v.z;
  }
  __device__ void store4(int m, int n, float4 v, int nv, int split) const {
    store4(m, n, v, nv, split, prefetch(m, n));
  }
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv, int split) const {
    if (!valid) return;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (4 * q < nv)
        store4(m, n + 4 * q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]),
               min(4, nv - 4 * q), split);
  }
};

struct TcEpiPartial {  // split-K partial tile ws[split][m][n] (row-major, width N)
  float* ws;
  long long split_stride;
  int M, N;
  __device__ void chunk(int m, bool valid, int n, const float (&v)[16], int nv, int split) const {
    if (!valid) return;
    float* o = ws + split * split_stride + (long long)m * N + n;
    if (chunk_vec(o, nv)) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nv) o[i] = v[i];
    }
  }
  __device__ void store4(int m, int n, float4 v, int nv, int split) const {
    const float x[4] = {v.x, v.y, v.z, v.w};
    put4(ws + split * split_stride + (long long)m * N + n, x, nv);
  }
};

}  // namespace tc
}  // namespace gfm
