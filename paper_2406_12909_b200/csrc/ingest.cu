// Record payloads -> device arrays (container ingest straight into HBM,
// SURVEY 8(f) row 4; the host codec is records.py:126-183):
//   u32 n_atoms | u32 edge_count | u32 tag_len | u8 z[n] | f64 pos[n,3] |
//   u32 edges[m,2] | f64 energy | f64 forces[n,3] | tag utf-8 | u32 crc32
// little-endian, records packed back to back at arbitrary byte offsets.
//   gfm_record_scan    one thread per record: header, length check, zlib CRC32
//   gfm_record_decode  one warp per record: fields scattered into the store's
//                      concatenated arrays (+ per-node in-degree counts)
// Byte and integer work: HBM-bound, no arithmetic to speak of.
#include <cstdint>

#include "common.cuh"

namespace gfm {

__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) {  // unaligned little-endian
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
__device__ __forceinline__ double ld_f64(const uint8_t* p) {
  const unsigned long long lo = ld_u32(p), hi = ld_u32(p + 4);
  return __longlong_as_double((long long)(lo | (hi << 32)));
}

// status: 0 ok, 1 truncated (shorter than header + crc), 2 length mismatch,
// 3 checksum mismatch
__global__ void k_record_scan(const uint8_t* __restrict__ blob, const long long* __restrict__ off,
                              const long long* __restrict__ len, int n_rec, int* __restrict__ n_atoms,
                              int* __restrict__ n_edges, int* __restrict__ status) {
  pdl_entry();
  __shared__ uint32_t tab[256];  // zlib's reflected CRC-32 table, built per block
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = c & 1u ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    tab[i] = c;
  }
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rec; r += gridDim.x * blockDim.x) {
    const uint8_t* p = blob + off[r];
    const long long L = len[r];
    n_atoms[r] = 0;
    n_edges[r] = 0;
    if (L < 16) {
      status[r] = 1;
      continue;
    }
    const uint32_t n = ld_u32(p), m = ld_u32(p + 4), tl = ld_u32(p + 8);
    const long long want = 12LL + n + 48LL * n + 8LL * m + 8 + tl + 4;
    if (L != want) {
      status[r] = 2;
      continue;
    }
    // byte-wise up to a 16-byte boundary, then 16-byte loads (one load per
    // 16 table steps instead of one per byte), then the tail
    uint32_t c = 0xFFFFFFFFu;
    const long long body = L - 4;
    long long i = 0;
    const long long head = (16 - (long long)((uintptr_t)p & 15)) & 15;
    for (; i < head && i < body; ++i) c = tab[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    for (; i + 16 <= body; i += 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t x = w[q];
#pragma unroll
        for (int b = 0; b < 4; ++b, x >>= 8) c = tab[(c ^ x) & 0xFFu] ^ (c >> 8);
      }
    }
    for (; i < body; ++i) c = tab[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    if ((c ^ 0xFFFFFFFFu) != ld_u32(p + L - 4)) {
      status[r] = 3;
      continue;
    }
    status[r] = 0;
    n_atoms[r] = (int)n;
    n_edges[r] = (int)m;
  }
}

// warp per record; atom_off / edge_off: exclusive prefix sums (the record's
// first row in the concatenated arrays); deg (optional): in-degree counts of
// the global node ids (integer atomics: order independent)
__global__ void k_record_decode(const uint8_t* __restrict__ blob, const long long* __restrict__ off,
                                int n_rec, const long long* __restrict__ atom_off,
                                const long long* __restrict__ edge_off, int* __restrict__ z,
                                double* __restrict__ pos, double* __restrict__ forces,
                                double* __restrict__ energy, int* __restrict__ edges,
                                int* __restrict__ deg, int* __restrict__ bad) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rec; r += warps) {
    const uint8_t* p = blob + off[r];
    const int n = (int)ld_u32(p), m = (int)ld_u32(p + 4);
    const long long a0 = atom_off[r], e0 = edge_off[r];
    const uint8_t* pz = p + 12;
    const uint8_t* pp = pz + n;
    const uint8_t* pe = pp + 24LL * n;
    const uint8_t* pen = pe + 8LL * m;
    const uint8_t* pf = pen + 8;
    for (int i = lane; i < n; i += 32) z[a0 + i] = pz[i];
    for (int i = lane; i < 3 * n; i += 32) {
      pos[3 * a0 + i] = ld_f64(pp + 8LL * i);
      forces[3 * a0 + i] = ld_f64(pf + 8LL * i);
    }
    for (int i = lane; i < 2 * m; i += 32) {
      const uint32_t v = ld_u32(pe + 4LL * i);
      edges[2 * e0 + i] = (int)v;
      if (v >= (uint32_t)n && bad) atomicOr(bad, 1);  // endpoint out of range
    }
    if (deg)
      for (int i = lane; i < m; i += 32) {
        const uint32_t d = ld_u32(pe + 8LL * i + 4);
        if (d < (uint32_t)n) atomicAdd(&deg[a0 + d], 1);
      }
    if (lane == 0) energy[r] = ld_f64(pen);
  }
}

}  // namespace gfm

using namespace gfm;

extern "C" {

int gfm_record_scan(const void* blob, const long long* offsets, const long long* lengths, int n_rec,
                    int* n_atoms, int* n_edges, int* status, void* stream) {
  if (n_rec <= 0) return 0;
  const int grid = (n_rec + 127) / 128 < 148 * 8 ? (n_rec + 127) / 128 : 148 * 8;
  launch_k(k_record_scan, grid, 128, 0, (cudaStream_t)stream, (const uint8_t*)blob, offsets,
           lengths, n_rec, n_atoms, n_edges, status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_record_scan: %s", cudaGetErrorString(e));
  return (int)e;
}

int gfm_record_decode(const void* blob, const long long* offsets, int n_rec,
                      const long long* atom_offsets, const long long* edge_offsets, int* z,
                      double* pos, double* forces, double* energy, int* edges, int* deg,
                      int* bad, void* stream) {
  if (n_rec <= 0) return 0;
  const long long warps = n_rec;
  const int grid = (int)((warps * 32 + 255) / 256 < 148 * 16 ? (warps * 32 + 255) / 256 : 148 * 16);
  launch_k(k_record_decode, grid, 256, 0, (cudaStream_t)stream, (const uint8_t*)blob, offsets,
           n_rec, atom_offsets, edge_offsets, z, pos, forces, energy, edges, deg, bad);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error("gfm_record_decode: %s", cudaGetErrorString(e));
  return (int)e;
}

}  // extern "C"
