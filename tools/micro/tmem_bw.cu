// TMEM read / write bandwidth per SM (microbenchmark, not product code): the
// epilogues of the GEMM and attention kernels drain fp32 accumulators with
// tcgen05.ld, so bytes/clock/SM of tcgen05.ld bounds them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2010_13382_b200/csrc -o tmem_bw tmem_bw.cu
// One CTA per SM, W warps (warp w reads lane quadrant w % 4), each warp loops
// over all 512 columns with 32x32b.x{16,32,64} loads (one wait per load or one
// wait per 4 loads); reports bytes per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "ptx.cuh"

using namespace ff;

template <int X>
__device__ __forceinline__ void ld_x(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld_x<16>(uint32_t taddr, uint32_t* r) {
  tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(r));
}
template <>
__device__ __forceinline__ void ld_x<32>(uint32_t taddr, uint32_t* r) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
}

template <int X, int BATCH>
__global__ void __launch_bounds__(512, 1) k_tmem_ld(unsigned long long* cycles, uint32_t* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  uint32_t r[BATCH][X];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 512; c += X * BATCH) {
#pragma unroll
      for (int b = 0; b < BATCH; ++b) ld_x<X>(base + c + b * X, r[b]);
      tmem_wait_ld();
#pragma unroll
      for (int b = 0; b < BATCH; ++b) acc ^= r[b][0] ^ r[b][X - 1];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

template <int X, int BATCH>
void run(int warps) {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  const int iters = 200;
  k_tmem_ld<X, BATCH><<<148, 32 * warps>>>(cyc, sink, iters);
  k_tmem_ld<X, BATCH><<<148, 32 * warps>>>(cyc, sink, iters);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
  // bytes read per CTA: warps x (32 lanes x 512 cols x 4 B) x iters
  const double bytes = (double)warps * 32 * 512 * 4 * iters;
  printf("tcgen05.ld 32x32b.x%-2d batch %d, %2d warps: %.1f B/clk/SM (%s)\n", X, BATCH, warps, bytes / mean,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<16, 1>(w);
    run<16, 2>(w);
    run<32, 1>(w);
    run<32, 2>(w);
  }
  return 0;
}
