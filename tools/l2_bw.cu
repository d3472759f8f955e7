// L2 (LTS) read-throughput probe: every SM streams float4 loads over a
// buffer that fits in L2 (and, for comparison, one that does not), CUDA-event
// timed after warm-up.  The gather-bound aggregation kernels are judged
// against the L2-resident figure (bench.py roofline "l2_*" keys).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw tools/l2_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_read(const float4* __restrict__ p, long long n4, int reps,
                                             float* __restrict__ sink) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldcg(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.f) sink[0] = acc;  // keeps the loads alive
}

static double run(long long bytes, int reps, int sms) {
  float4* p;
  float* sink;
  cudaMalloc(&p, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(p, 0, bytes);
  const long long n4 = bytes / 16;
  const int grid = sms * 4, block = 512;
  k_read<<<grid, block>>>(p, n4, 1, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_read<<<grid, block>>>(p, n4, reps, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(p);
  cudaFree(sink);
  return (double)bytes * reps / (ms * 1e-3) / 1e9;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double l2 = 0, hbm = 0;
  for (long long mb : {16LL, 32LL, 48LL, 64LL}) {
    const double g = run(mb << 20, 200, sms);
    printf("resident %3lld MB: %8.0f GB/s\n", mb, g);
    if (g > l2) l2 = g;
  }
  hbm = run(8LL << 30, 3, sms);
  printf("streaming 8 GB: %8.0f GB/s\n", hbm);
  printf("{\"l2_read_gbs\": %.0f, \"hbm_read_gbs\": %.0f, \"sms\": %d}\n", l2, hbm, sms);
  return 0;
}
