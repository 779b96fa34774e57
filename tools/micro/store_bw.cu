// Output-store throughput of the GEMM epilogue pattern (microbenchmark, not
// product code).  The C3 QKV GEMM writes a 32768 x 1536 fp16 result (100 MB,
// head-major: [1536/64 * M rows x 64 cols], 128-byte rows) and measured as fast
// with its operands left in smem as with them loaded (tools/mma_rate.py), so
// the epilogue's stores bound it.  One CTA per SM, 16 warps; per 128 x 256
// tile each warp writes a 32-row x 64-column block (4 KB contiguous in the
// head-major layout) as
//   0: two TMA stores of 32 x 32 (64-byte rows, 64B swizzle; the kernel today)
//   1: one TMA store of 32 x 64 (128-byte rows, 128B swizzle)
//   2: st.global.v4, lane = 16-byte piece, 8 rows x 128 B per instruction pass
// with NBUF staging buffers per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2010_13382_b200/csrc -o store_bw store_bw.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace ff;

constexpr int M = 32768, N = 1536, BM = 128, BN = 256;
constexpr int WARPS = 16;

template <int MODE, int NBUF>
__global__ void __launch_bounds__(WARPS * 32, 1)
    store_kernel(const __grid_constant__ CUtensorMap map32, const __grid_constant__ CUtensorMap map64, __half* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = smem + warp * NBUF * 4096;
  const int q = warp & 3, cg = warp >> 2;  // rows [32q, +32), columns [64 cg, +64) of the tile
  const int m_tiles = M / BM, n_tiles = N / BN;
  int nb = 0;
  for (int tile = blockIdx.x; tile < m_tiles * n_tiles; tile += gridDim.x) {
    const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
    const int row0 = mt * BM + q * 32;
    const int col0 = nt * BN + cg * 64;  // one 64-column head block
    const int hrow = (col0 >> 6) * M + row0;
    uint8_t* b = buf + (nb % NBUF) * 4096;
    if (MODE == 2) {
      // 4 KB contiguous: 32 rows x 128 B; lane writes 16 B pieces
      uint4* dst = reinterpret_cast<uint4*>(out + (size_t)hrow * 64);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i * 32 + lane] = make_uint4(tile, i, lane, 0x3C003C00);
    } else {
      if (lane == 0) {
        if (NBUF == 1) bulk_wait_read<0>();
        else bulk_wait_read<NBUF - 1>();
      }
      __syncwarp();
      // fill the staging buffer (contents irrelevant; layout = 32 rows x 128 B)
#pragma unroll
      for (int i = 0; i < 8; ++i) reinterpret_cast<uint4*>(b)[i * 32 + lane] = make_uint4(tile, i, lane, 0x3C003C00);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (MODE == 0) {
          tma_store_2d(&map32, b, 0, hrow);
          tma_store_2d(&map32, b + 2048, 32, hrow);
        } else {
          tma_store_2d(&map64, b, 0, hrow);
        }
        bulk_commit();
      }
      ++nb;
    }
  }
  if (lane == 0) bulk_wait<0>();
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  __half* out;
  cudaMalloc(&out, (size_t)M * N * 2);
  uint8_t* junk;
  cudaMalloc(&junk, 256 << 20);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  PFN enc = reinterpret_cast<PFN>(fn);
  CUtensorMap m32, m64;
  cuuint64_t dims[2] = {64, (cuuint64_t)(N / 64) * M};
  cuuint64_t str[1] = {128};
  cuuint32_t box32[2] = {32, 32}, box64[2] = {64, 32}, es[2] = {1, 1};
  enc(&m32, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, out, dims, str, box32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m64, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, out, dims, str, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name, int nbuf) {
    const int smem = WARPS * nbuf * 4096 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e9f;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(junk, it, 256 << 20);  // flush L2
      cudaEventRecord(e0);
      kern<<<148, WARPS * 32, smem>>>(m32, m64, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-40s %7.1f us  %6.0f GB/s (%s)\n", name, best * 1e3, (double)M * N * 2 / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(store_kernel<0, 1>, "TMA 2 x (32x32), 1 buf", 1);
  run(store_kernel<0, 2>, "TMA 2 x (32x32), 2 bufs", 2);
  run(store_kernel<1, 1>, "TMA 1 x (32x64), 1 buf", 1);
  run(store_kernel<1, 2>, "TMA 1 x (32x64), 2 bufs", 2);
  run(store_kernel<1, 3>, "TMA 1 x (32x64), 3 bufs", 3);
  run(store_kernel<2, 1>, "st.global.v4 contiguous", 1);
  return 0;
}
