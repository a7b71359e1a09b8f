// Check the CTA-pair (cta_group::2) MMA mechanics on B200: a cluster of two
// CTAs, TMEM allocated with cta_group::2 by a warp in each CTA, one
// M=256 N=128 K=16 bf16 MMA issued by the leader with A rows 0..127 / 128..255
// and B rows 0..63 / 64..127 in CTA 0 / CTA 1 shared memory (same offsets),
// completion multicast to both CTAs' mbarriers, each CTA reading its 128 TMEM
// lanes.  Compared against the CPU.
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void __cluster_dims__(2, 1, 1) pair_kernel(const uint16_t* a, const uint16_t* b, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_ctarank();
  uint8_t* sA = smem;              // 128 x 16 bf16, core matrices: (m/8, k/8) at ((m/8)*2 + k/8)*128
  uint8_t* sB = smem + 4096;       // 64 x 16
  for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    *reinterpret_cast<uint16_t*>(sA + ((m / 8) * 2 + k / 8) * 128 + (m % 8) * 16 + (k % 8) * 2) = a[(rank * 128 + m) * 16 + k];
  }
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    *reinterpret_cast<uint16_t*>(sB + ((n / 8) * 2 + k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = b[(rank * 64 + n) * 16 + k];
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (rank == 0 && threadIdx.x < 32) {
    if (elect_one()) {
      const uint64_t ad = desc_noswz(smem_u32(sA), 128, 256), bd = desc_noswz(smem_u32(sB), 128, 256);
      const uint32_t idesc = make_idesc<false>(256, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
          ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32;
  uint32_t v[32];
  for (int q = 0; q < 4; ++q) {
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(w * 32) << 16) + q * 32, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j)
      out[(rank * 128 + w * 32 + (threadIdx.x & 31)) * 128 + q * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
  }
}

static uint16_t to_bf16(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }

int main() {
  std::vector<float> af(256 * 16), bf(128 * 16);
  std::vector<uint16_t> a(256 * 16), b(128 * 16);
  for (int i = 0; i < 256 * 16; ++i) { af[i] = (float)((i * 7) % 9 - 4); a[i] = to_bf16(af[i]); }
  for (int i = 0; i < 128 * 16; ++i) { bf[i] = (float)((i * 5) % 7 - 3); b[i] = to_bf16(bf[i]); }
  uint16_t *da, *db; float* dout;
  cudaMalloc(&da, a.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dout, 256 * 128 * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dout, 0, 256 * 128 * 4);
  pair_kernel<<<2, 128, 16384>>>(da, db, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> out(256 * 128);
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 128; ++n) {
      float ref = 0.f;
      for (int k = 0; k < 16; ++k) ref += af[m * 16 + k] * bf[n * 16 + k];
      if (out[m * 128 + n] != ref) ++bad;
    }
  printf("pair MMA M=256 N=128 K=16: %d / %d mismatches\n", bad, 256 * 128);
  return 0;
}
