// Check a "sliding window" A operand for tcgen05.mma: A row m starts 16 bytes
// after row m-1 in one contiguous smem buffer (rows overlap), described with
// the no-swizzle K-major layout (core matrix = 8 rows x 16 B).  Tries both
// assignments of the K-direction / M-direction core-matrix strides to the
// descriptor's LBO / SBO fields and reports which one reproduces the CPU
// result.  M=128, N=64, K=16, bf16 -> f32.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version
  return d;                 // layout bits 61-63 = 0: no swizzle
}

__global__ void kern(const uint16_t* row, const uint16_t* bmat, float* out, int variant, int nrow_elems) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint16_t* sRow = reinterpret_cast<uint16_t*>(smem);            // sliding source (A)
  uint8_t* sB = smem + 8192;                                      // B, 64 x 16, core-matrix layout
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < nrow_elems; i += blockDim.x) sRow[i] = row[i];
  // B[n][k] at core matrix (n/8, k/8): K-dir stride 128 B, N-dir stride 256 B
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    const int off = (n / 8) * 256 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<uint16_t*>(sB + off) = bmat[i];
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<64>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    if (elect_one()) {
      const uint32_t a_addr = smem_u32(sRow), b_addr = smem_u32(sB);
      uint64_t ad, bd;
      if (variant == 0) { ad = desc_noswz(a_addr, 16, 128); bd = desc_noswz(b_addr, 128, 256); }
      else { ad = desc_noswz(a_addr, 128, 16); bd = desc_noswz(b_addr, 256, 128); }
      tc_mma<false>(tmem, ad, bd, make_idesc<false>(128, 64), 0u);
      tc_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32;
  uint32_t v[32];
  for (int half = 0; half < 2; ++half) {
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(w * 32) << 16) + half * 32, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(w * 32 + (threadIdx.x & 31)) * 64 + half * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<64>(tmem); }
}

// Rate: `iters` back-to-back MMAs (M=128, N=64, K=16) from one thread.
// mode 0: sliding no-swizzle A (LBO 16, SBO 128); 1: ordinary no-swizzle A
// (distinct rows, LBO 128, SBO 256); 2: SW128 K-major A.  B no-swizzle.
__global__ void rate(int mode, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bars2[8];
  __shared__ uint32_t tslot;
  if (threadIdx.x < 8) mbar_init(&bars2[threadIdx.x], 1);
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t a_addr = smem_u32(smem), b_addr = smem_u32(smem + 32768 + 16384);
    uint64_t ad;
    if (mode == 0) ad = desc_noswz(a_addr, 16, 128);
    else if (mode == 1) ad = desc_noswz(a_addr, 128, 256);
    else ad = sw128_kmajor_desc(a_addr);
    const uint64_t bd = desc_noswz(b_addr, 128, 256);
    long long t0 = clock64();
    if (elect_one()) {
      if (mode < 3) {
        for (int i = 0; i < iters; ++i) tc_mma<false>(tmem, ad, bd, make_idesc<false>(128, 64), i > 0 ? 1u : 0u);
      } else if (mode == 4) {   // row-kernel tiles: 14 MMAs + 2 commits per tile, 4 accumulators
        const uint64_t a0 = desc_noswz(0, 16, 128), b0 = desc_noswz(b_addr, 128, 512);
        for (int t = 0; t < iters / 14; ++t) {
          for (int i = 0; i < 14; ++i) {
            const int ky = i >> 1, j = i & 1;
            const uint64_t adj = a0 + ((a_addr + ky * 2112 + 32 * j) >> 4);
            const uint64_t bdj = b0 + ((ky * 64 * 64 + j * 256) >> 4);
            tc_mma<false>(tmem + (t & 3) * 64, adj, bdj, make_idesc<false>(128, 64), i > 0 ? 1u : 0u);
          }
          tc_commit(&bars2[t & 3]);
          tc_commit(&bars2[4 + (t & 3)]);
        }
      } else {   // mode 3: the row kernel's pattern: 7 A rows 2112 B apart, 7 B blocks, 2 K steps each
        const uint64_t a0 = desc_noswz(0, 16, 128), b0 = desc_noswz(b_addr, 128, 512);
        for (int i = 0; i < iters; ++i) {
          const int ky = (i >> 1) % 7, j = i & 1;
          const uint64_t adj = a0 + ((a_addr + ky * 2112 + 32 * j) >> 4);
          const uint64_t bdj = b0 + ((ky * 64 * 64 + j * 256) >> 4);
          tc_mma<false>(tmem, adj, bdj, make_idesc<false>(128, 64), i > 0 ? 1u : 0u);
        }
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

static uint16_t to_bf16(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }

int main() {
  const int nrow = 128 * 8 + 64;   // elements
  std::vector<uint16_t> row(nrow), b(64 * 16);
  std::vector<float> rowf(nrow), bf(64 * 16);
  for (int i = 0; i < nrow; ++i) { rowf[i] = (float)((i * 7) % 9 - 4); row[i] = to_bf16(rowf[i]); }
  for (int i = 0; i < 64 * 16; ++i) { bf[i] = (float)((i * 5) % 7 - 3); b[i] = to_bf16(bf[i]); }
  uint16_t *drow, *db; float* dout;
  cudaMalloc(&drow, nrow * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(drow, row.data(), nrow * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dout, 0, 128 * 64 * 4);
    kern<<<1, 128, 16384 + 1024>>>(drow, db, dout, variant, nrow);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("variant %d: %s\n", variant, cudaGetErrorString(e)); return 1; }
    std::vector<float> out(128 * 64);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        float ref = 0.f;
        for (int k = 0; k < 16; ++k) ref += rowf[8 * m + k] * bf[n * 16 + k];   // row m starts 16 B = 8 elements later
        if (out[m * 64 + n] != ref) ++bad;
      }
    printf("variant %d (%s): %d / %d mismatches\n", variant, variant ? "LBO=M-dir 16B? swapped" : "LBO=K-dir 16B, SBO=M-dir 128B",
           bad, 128 * 64);
  }
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 5; ++mode) {
    rate<<<1, 128, 96 * 1024>>>(mode, 2002, dcyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("rate mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    unsigned long long c;
    cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cycles per M128 N64 K16 MMA\n", mode,
           mode == 0 ? "sliding no-swizzle A" : mode == 1 ? "no-swizzle A" : mode == 2 ? "SW128 A" : mode == 3 ? "row-kernel pattern" : "row tiles + commits",
           c / 2002.0);
  }
  return 0;
}
