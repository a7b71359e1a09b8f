// TMA 2D tile-load throughput per SM for filter-like traffic: every CTA (one
// per SM) streams [box_rows x 128 B] boxes of a [rows x cols] bf16 matrix
// with `stages` loads in flight.  Shared: all CTAs read the same matrix (the
// conv filter case); private: each CTA reads its own copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu -lcuda
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__global__ void tma_kernel(const __grid_constant__ CUtensorMap tm_shared, const __grid_constant__ CUtensorMap tm_priv,
                           int priv, int nkb, int box_bytes, int stages, int iters, int rot,
                           unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const CUtensorMap* tm = priv ? &tm_priv : &tm_shared;
  const int row0 = priv ? blockIdx.x * 128 : 0;   // private copies stacked along rows
  const int start = rot ? (blockIdx.x * 7) % nkb : 0;
  long long t0 = clock64();
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) mbar_wait(&bar[s], ((it - stages) / stages) & 1);
    if (it < iters) {
      mbar_arrive_expect_tx(&bar[s], box_bytes);
      const int kb = (start + it) % nkb;
      tma_load_2d(smem_u32(base + s * box_bytes), tm, &bar[s], kb * 64, row0);
    }
  }
  long long t1 = clock64();
  cyc[blockIdx.x] = t1 - t0;
}


// 3D boxes {64 elems, rows, depth}: depth consecutive 128-byte K blocks per load.
// issuers: number of warps issuing (each warp lane 0 owns stages w, w+issuers, ...)
__global__ void tma3_kernel(const __grid_constant__ CUtensorMap tm, int nkb, int depth, int box_bytes, int stages,
                            int iters, int issuers, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w >= issuers) return;
  long long t0 = clock64();
  for (int it = w; it < iters + stages; it += issuers) {
    const int s = it % stages;
    if (it >= stages) mbar_wait(&bar[s], ((it - stages) / stages) & 1);
    if (it < iters) {
      mbar_arrive_expect_tx(&bar[s], box_bytes);
      const int kb = (it * depth) % nkb;
      tma_load_3d(smem_u32(base + s * box_bytes), &tm, &bar[s], 0, 0, kb);
    }
  }
  long long t1 = clock64();
  if (w == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int cols = 2304, box_rows_list[2] = {128, 256};
  const int nsm = 148;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  uint16_t* d;
  const size_t rows_priv = (size_t)nsm * 256;
  cudaMalloc(&d, rows_priv * cols * 2);
  cudaMemset(d, 1, rows_priv * cols * 2);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, nsm * 8);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int box_rows : box_rows_list) {
    CUtensorMap tms, tmp;
    cuuint64_t dims_s[2] = {(cuuint64_t)cols, (cuuint64_t)box_rows};
    cuuint64_t dims_p[2] = {(cuuint64_t)cols, (cuuint64_t)rows_priv};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    encode(&tms, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims_s, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    encode(&tmp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims_p, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int box_bytes = box_rows * 128;
    for (int priv = 0; priv < 2; ++priv)
      for (int rot = 0; rot < 2; ++rot)
        for (int stages : {2, 4, 8}) {
          if (stages * box_bytes > 190 * 1024) continue;
          const int iters = 2000;
          tma_kernel<<<nsm, 32, stages * box_bytes + 1024>>>(tms, tmp, priv, cols / 64, box_bytes, stages, iters, rot,
                                                             dcyc);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<unsigned long long> c(nsm);
          cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
          double mx = 0;
          for (auto v : c) mx = v > mx ? v : mx;
          printf("box %3d rows (%5d B) %s rot=%d stages=%d: %.0f cycles/load, %.1f B/cycle/SM\n", box_rows, box_bytes,
                 priv ? "private" : "shared ", rot, stages, mx / iters, box_bytes * (double)iters / mx);
        }
  }
  cudaFuncSetAttribute(tma3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rows : {128, 256})
    for (int depth : {1, 2, 4}) {
      CUtensorMap tm;
      cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
      cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)rows, (cuuint32_t)depth};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode3d rows=%d depth=%d failed %d\n", rows, depth, (int)r); continue; }
      const int box_bytes = rows * 128 * depth;
      for (int issuers : {1, 4})
        for (int stages : {2, 4, 8}) {
          if (stages * box_bytes > 190 * 1024 || stages < issuers) continue;
          const int iters = 1000;
          tma3_kernel<<<nsm, 128, stages * box_bytes + 1024>>>(tm, cols / 64, depth, box_bytes, stages, iters,
                                                               issuers, dcyc);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<unsigned long long> c(nsm);
          cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
          double mx = 0;
          for (auto v : c) mx = v > mx ? v : mx;
          printf("3d box %3d rows x %d blocks (%6d B) issuers=%d stages=%d: %.0f cycles/load, %.1f B/cycle/SM\n", rows,
                 depth, box_bytes, issuers, stages, mx / iters, box_bytes * (double)iters / mx);
        }
    }
  return 0;
}
