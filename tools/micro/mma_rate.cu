// Microbenchmark: raw tcgen05.mma issue/execute rate for one CTA per SM,
// single issuing thread, operands resident in smem (128B-swizzle K-major),
// no barriers in the loop.  Prints cycles per MMA for N = 64/128/256 and
// kind::f16 / kind::i8.
#include <cstdio>
#include <cuda.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;


template <bool kI8, int N, int kVar>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                  // 128 x 128 B
  uint8_t* sB = smem + 16384;          // N x 128 B
  __shared__ uint64_t bar;
  __shared__ uint64_t bars[8];
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (kVar == 7 && threadIdx.x < 32) {
    // whole warp runs the loop; one elected lane issues (uniform operands)
    constexpr uint32_t idesc = make_idesc<kI8>(128, N);
    const uint64_t ad = sw128_kmajor_desc(smem_u32(sA));
    const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
    if (elect_one()) mbar_arrive(&done);
    __syncwarp();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&done, 0);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k) tc_mma<kI8>(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
        tc_commit(&bars[it & 7]);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  } else if (kVar == 9 && threadIdx.x == 0) {
    // the uint8 gather kernel's pattern: one N-wide MMA + one N=16 MMA (row sums) per K step
    constexpr uint32_t idesc = make_idesc<kI8>(128, N);
    constexpr uint32_t idesc16 = make_idesc<kI8>(128, 16);
    const uint64_t ad = sw128_kmajor_desc(smem_u32(sA));
    const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tc_mma<kI8>(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
        tc_mma<kI8>(tmem + N, ad + 2 * k, bd + 2 * k, idesc16, (it | k) != 0);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  } else if ((kVar < 7 || kVar == 8) && threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc<kI8>(128, N);
    const uint64_t ad = sw128_kmajor_desc(smem_u32(sA));
    const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
    long long t0 = clock64();
    if (kVar >= 3) mbar_arrive(&done);  // phase 0 of `done` completes: waits on parity 0 return at once
    for (int it = 0; it < iters; ++it) {
      if (kVar == 3) mbar_wait(&done, 0);
      if (kVar == 4) {  // relaxed try_wait
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&done)), "r"(0) : "memory");
        }
      }
      if (kVar == 5) {  // test_wait spin
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&done)), "r"(0) : "memory");
        }
      }
      if (kVar == 6 && (it & 1) == 0) mbar_wait(&done, 0);
      if (kVar >= 2 && kVar != 8) tc_fence_after();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // var 0: one accumulator; var 8: two accumulators alternated
        // (breaks the accumulate-dependency chain between consecutive MMAs)
        const uint32_t dd = (kVar == 8 && (k & 1)) ? tmem + N : tmem;
        tc_mma<kI8>(dd, ad + 2 * k, bd + 2 * k, idesc, (it | (k >> 1)) != 0);
      }
      if (kVar >= 1 && kVar != 8) tc_commit(&bars[it & 7]);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

template <bool kI8, int N, int kVar = 0>
void run(unsigned long long* d) {
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(mma_rate<kI8, N, kVar>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  mma_rate<kI8, N, kVar><<<148, 128, smem>>>(iters, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  mma_rate<kI8, N, kVar><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double macs = 148.0 * iters * 4 * 128.0 * N * (kI8 ? 32 : 16);
  printf("var%d %s N=%3d: %.1f cycles/MMA (ideal %d), %.0f T%s/s, err=%s\n", kVar, kI8 ? "i8 " : "f16", N,
         (double)cyc / (iters * 4), 128 * N / 256, 2 * macs / (ms * 1e-3) / 1e12, kI8 ? "OP" : "FLOP",
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<false, 128, 2>(d); run<false, 128, 3>(d); run<false, 128, 7>(d); run<false, 64, 7>(d);
  run<false, 64, 0>(d); run<false, 64, 8>(d); run<false, 128, 0>(d); run<false, 128, 8>(d); run<false, 32, 0>(d);
  run<false, 32, 8>(d); run<true, 64, 0>(d); run<true, 128, 0>(d); run<true, 256, 0>(d);
  // uint8 row-sum options: a separate N=16 MMA per K step vs ones rows fused into the filter tile (N + 16)
  run<true, 16, 0>(d); run<true, 32, 0>(d); run<true, 144, 0>(d); run<true, 160, 0>(d); run<true, 192, 0>(d);
  run<true, 128, 9>(d); run<true, 240, 0>(d); run<false, 144, 0>(d); run<false, 256, 0>(d);
  return 0;
}
