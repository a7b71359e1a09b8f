// How TMA loads overlap per issuing thread on a B200: every CTA (one per SM)
// streams 16 KB boxes (128 rows x 128 B) of its own slice of a 2 GiB buffer
// (HBM-resident: every box is a first touch) or of a 4 MiB buffer (L2
// resident), with `issuers` issuing threads placed either one per warp
// (lane 0 of warps 0..k-1) or as lanes 0..k-1 of warp 0, each thread keeping
// `depth` boxes in flight on its own barriers.  Reports cycles per box per SM
// and B/cycle/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_issue tma_issue.cu -lcuda
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

constexpr int kBox = 16384;

__global__ void issue_kernel(const __grid_constant__ CUtensorMap tm, int rows_per_cta, int issuers, int per_warp,
                             int depth, int boxes, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[64];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 64; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int id = -1;
  if (per_warp) { if (lane == 0 && warp < issuers) id = warp; }
  else if (warp == 0 && lane < issuers) id = lane;
  if (id < 0) return;
  const int row0 = blockIdx.x * rows_per_cta;
  long long t0 = clock64();
  // thread `id` owns boxes id, id + issuers, ... and barriers id*depth .. id*depth + depth-1
  int k = 0;
  for (int b = id; b < boxes + depth * issuers; b += issuers, ++k) {
    const int slot = id * depth + (k % depth);
    if (k >= depth) mbar_wait(&bar[slot], ((k - depth) / depth) & 1);
    if (b < boxes) {
      mbar_arrive_expect_tx(&bar[slot], kBox);
      const int r = (b * 128) % rows_per_cta;
      tma_load_2d(smem_u32(base + slot * kBox), &tm, &bar[slot], 0, row0 + r);
    }
  }
  long long t1 = clock64();
  if (id == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int nsm = 148;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const size_t big = size_t(2) << 30, small = size_t(4) << 20;
  uint8_t* d;
  cudaMalloc(&d, big);
  cudaMemset(d, 1, big);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, nsm * 8);
  cudaFuncSetAttribute(issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int hbm = 1; hbm >= 0; --hbm) {
    const size_t bytes = hbm ? big : small;
    const int rows_total = (int)(bytes / 128);
    const int rows_per_cta = hbm ? rows_total / nsm / 128 * 128 : rows_total / 128 * 128 / nsm / 128 * 128;
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int boxes = hbm ? rows_per_cta / 128 : 400;
    for (int per_warp = 1; per_warp >= 0; --per_warp)
      for (int issuers : {1, 2, 4, 8})
        for (int depth : {1, 2, 4}) {
          if (issuers * depth > 12) continue;
          if (per_warp && issuers > 8) continue;
          issue_kernel<<<nsm, 256, issuers * depth * kBox + 1024>>>(tm, rows_per_cta, issuers, per_warp, depth, boxes,
                                                                    dcyc);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<unsigned long long> c(nsm);
          cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
          double mx = 0;
          for (auto v : c) mx = v > mx ? v : mx;
          printf("%s issuers=%d (%s) depth=%d: %6.0f cycles/box  %6.1f B/cycle/SM  in flight %3d KB\n",
                 hbm ? "HBM" : "L2 ", issuers, per_warp ? "one per warp" : "lanes of warp 0", depth, mx / boxes,
                 kBox * (double)boxes / mx, issuers * depth * 16);
        }
  }
  return 0;
}
