// The dense-A kernel's load skeleton in isolation: one CTA per SM, a ring of
// `stages` stages, each = one 16 KB A box (128 rows x 128 B, streamed from a
// private slice of a 2 GiB buffer: first-touch HBM, or re-read from a 4 MiB
// L2-resident one) + one B box of `brows` x 128 B from a small buffer every
// CTA reads (L2-resident); `issuers` threads (lane 0 of warps 0..) issue the
// stages round-robin; one consumer warp waits on each stage's full barrier
// and releases it either with tcgen05.commit (what the kernel does after its
// MMAs) or a plain mbarrier arrive.  Reports cycles per stage per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ring tma_ring.cu -lcuda
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__global__ void ring_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                            int a_rows_per_cta, int stages, int issuers, int use_commit, int nstage, int bbytes,
                            unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cw = 4;   // consumer warp
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  if (warp == cw) tmem_alloc<32>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t sA = smem_u32(smem), sB = sA + stages * 16384;
  long long t0 = clock64();
  if (warp < issuers && lane == 0) {
    for (int q = warp; q < nstage; q += issuers) {
      const int st = q % stages;
      mbar_wait(&empty[st], (uint32_t)((q / stages) & 1) ^ 1u);
      mbar_arrive_expect_tx(&full[st], 16384 + bbytes);
      tma_load_2d(sB + st * bbytes, &tb, &full[st], 0, (q % 16) * (bbytes / 128));
      tma_load_2d(sA + st * 16384, &ta, &full[st], 0, blockIdx.x * a_rows_per_cta + (q * 128) % a_rows_per_cta);
    }
  } else if (warp == cw) {
    for (int q = 0; q < nstage; ++q) {
      const int st = q % stages;
      mbar_wait(&full[st], (uint32_t)((q / stages) & 1));
      tc_fence_after();
      if (lane == 0) {
        if (use_commit) tc_commit(&empty[st]);
        else mbar_arrive(&empty[st]);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == cw) tmem_dealloc<32>(tslot);
}

int main() {
  const int nsm = 148;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const size_t big = size_t(2) << 30, small = size_t(4) << 20;
  uint8_t *d, *db;
  cudaMalloc(&d, big);
  cudaMemset(d, 1, big);
  cudaMalloc(&db, small);
  cudaMemset(db, 1, small);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, nsm * 8);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int hbm = 1; hbm >= 0; --hbm) {
    const size_t abytes = hbm ? big : small;
    const int a_rows_total = (int)(abytes / 128);
    const int a_rows_per_cta = a_rows_total / nsm / 128 * 128;
    CUtensorMap ta, tb;
    cuuint64_t dims[2] = {64, (cuuint64_t)a_rows_total};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    encode(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int brows : {0, 128, 256}) {
      if (brows) {
        cuuint64_t bd[2] = {64, (cuuint64_t)(small / 128)};
        cuuint32_t bbox[2] = {64, (cuuint32_t)brows};
        encode(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, db, bd, strides, bbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        tb = ta;
      }
      const int bbytes = brows * 128;
      for (int stages : {4, 8})
        for (int issuers : {1, 4})
          for (int commit = 0; commit < 2; ++commit) {
            if (stages * (16384 + bbytes) > 215 * 1024 || issuers > stages) continue;
            if (brows == 0) continue;   // (B always present)
            const int nstage = hbm ? a_rows_per_cta / 128 : 600;
            ring_kernel<<<nsm, 160, stages * (16384 + bbytes) + 1024>>>(ta, tb, a_rows_per_cta, stages, issuers, commit,
                                                                        nstage, bbytes, dcyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<unsigned long long> c(nsm);
            cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (auto v : c) mx = v > mx ? v : mx;
            printf("A %s  B %3d rows  stages %d issuers %d release %-7s: %6.0f cycles/stage  %6.1f B/cycle/SM\n",
                   hbm ? "HBM" : "L2 ", brows, stages, issuers, commit ? "commit" : "arrive", mx / nstage,
                   (16384.0 + bbytes) * nstage / mx);
          }
    }
  }
  return 0;
}
