// Check + time TMA tile::gather4: gather 128 rows (128-byte slices of a
// [rows x 128] bf16 tensor) by row index into a 128B-swizzled smem tile;
// index -1 must zero-fill.  Verifies against a host reference.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

__global__ void gather_kernel(const __grid_constant__ CUtensorMap tm, const int* idx, int col0, uint8_t* out,
                              int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const uint32_t dst = smem_u32(smem);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, 128 * 128);
    __syncwarp();
    // lane l gathers rows 4l..4l+3 of the tile
    const int* r = idx + blockIdx.x * 128 + 4 * threadIdx.x;
    gather4(dst + threadIdx.x * 512, &tm, &bar, col0, r[0], r[1], r[2], r[3]);
    mbar_wait(&bar, it & 1);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  for (int i = threadIdx.x; i < 128 * 128 / 16; i += 32)
    reinterpret_cast<uint4*>(out + blockIdx.x * 16384)[i] = reinterpret_cast<const uint4*>(smem)[i];
}

int main() {
  const int rows = 4096, C = 128;  // bf16 elements
  std::vector<uint16_t> h(rows * C);
  for (int i = 0; i < rows * C; ++i) h[i] = (uint16_t)(i * 2654435761u >> 16);
  uint16_t* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  const int tiles = 4;
  std::vector<int> idx(tiles * 128);
  for (int i = 0; i < tiles * 128; ++i) idx[i] = (i % 17 == 3) ? -1 : (i * 37) % rows;
  int* didx;
  cudaMalloc(&didx, idx.size() * 4);
  cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
  uint8_t* dout;
  cudaMalloc(&dout, tiles * 16384);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 8);

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)C * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;
  for (int col0 : {0, 64}) {
    gather_kernel<<<tiles, 32, 16384 + 1024>>>(tm, didx, col0, dout, 1, dcyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("col0=%d kernel: %s\n", col0, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<uint8_t> out(tiles * 16384);
    cudaMemcpy(out.data(), dout, out.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < tiles; ++t)
      for (int row = 0; row < 128; ++row)
        for (int j = 0; j < 8; ++j) {  // 16-byte chunk j of the row stored at chunk j ^ (row % 8)
          const uint8_t* got = out.data() + t * 16384 + row * 128 + ((j ^ (row & 7)) << 4);
          const int src = idx[t * 128 + row];
          for (int b = 0; b < 16; ++b) {
            uint8_t want = 0;
            if (src >= 0) want = reinterpret_cast<const uint8_t*>(h.data())[(size_t)src * C * 2 + col0 * 2 + j * 16 + b];
            if (got[b] != want) ++bad;
          }
        }
    printf("col0=%d mismatched bytes: %d (swizzled layout check)\n", col0, bad);
  }
  gather_kernel<<<148, 32, 16384 + 1024>>>(tm, didx, 0, dout, 1000, dcyc);
  cudaDeviceSynchronize();
  unsigned long long cyc;
  cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  printf("gather 16 KB per iteration (1 CTA/SM, serialized): %.0f cycles/iter -> %.1f B/cycle/SM\n", cyc / 1000.0,
         16384.0 / (cyc / 1000.0));
  return 0;
}
