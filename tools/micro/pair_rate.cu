// Issue rate of CTA-pair (cta_group::2) MMAs, M=256 x N x K16 bf16, from the
// leader's elected thread, with SW128 K-major descriptors.  Patterns (A, B):
//   0: fixed; 1: K steps (+32 B); 2: 3x3 taps sliding A rows (row width 29,
//   unaligned starts) + K steps, B advancing one N/2 x 128 B block per tap
// (the window kernel's stream).  Ideal: N/2 cycles per MMA (each SM computes
// 128 x N x 16).
#include <cstdio>
#include <cuda.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

// kTraffic: warps 4.. of BOTH CTAs stream 16-byte st.shared (1) or ld.shared
// (2) over a 64 KB scratch region while the MMAs run -- how much does other
// shared-memory traffic (TMA fills, epilogue staging) slow the tensor core's
// operand reads?  out[1] = bytes moved by CTA 0's traffic warps.
template <int kMode, int kN, int kTraffic = 0>
__global__ void __cluster_dims__(2, 1, 1) rate(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ uint64_t done_bar;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done_bar, 1); fence_mbar_init(); mbar_arrive(&done_bar); }
  if (threadIdx.x < 32) tmem_alloc2<256>(&tslot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (kTraffic == 3 && threadIdx.x >= 128) {
    // epilogue-like TMEM reads of the columns next to the accumulator while the MMAs run
    const int w = threadIdx.x >> 5;
    const uint32_t taddr = tmem + ((uint32_t)((w & 3) * 32) << 16) + kN;
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!mbar_try_wait(&bar, 0)) {
      for (int rep = 0; rep < 8; ++rep) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr, v);
        tmem_ld_wait_regs(v);
        acc += v[0] + v[31];
      }
      n += 8;
    }
    if (acc == 0x12345678u) cyc[3] = acc;
    if (rank == 0 && (threadIdx.x & 31) == 0) atomicAdd(cyc + 1, n);
  } else
  if (kTraffic && threadIdx.x >= 128) {
    const uint32_t base = smem_u32(smem) + 131072 + (threadIdx.x - 128) * 16;
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!mbar_try_wait(&bar, 0)) {
      for (int rep = 0; rep < 16; ++rep) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t addr = base + i * 4096;   // (<= 384 traffic threads: 6 KB per row of the sweep)
          if (kTraffic == 1) {
            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(acc) : "memory");
          } else {
            uint32_t x, y, z, w;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr) : "memory");
            acc += x + y + z + w;
          }
        }
      }
      n += 16 * 16 * 16;
    }
    if (acc == 0x12345678u) cyc[3] = acc;
    if (rank == 0) atomicAdd(cyc + 1, n);
  } else
  if (rank == 0 && threadIdx.x < 32) {
    const uint32_t a_addr = smem_u32(smem), b_addr = smem_u32(smem + 65536);
    const uint64_t ad0 = sw128_kmajor_desc(a_addr), bd0 = sw128_kmajor_desc(b_addr);
    long long t0 = clock64();
    if (kMode < 3) {
      if (elect_one()) {
        for (int g = 0; g < iters / 36; ++g) {
#pragma unroll
          for (int j = 0; j < 36; ++j) {
            const int tap = j / 4, k = j % 4;
            uint32_t ao = 0, bo = 0;
            if (kMode == 1) { ao = 32 * k; bo = 32 * k; }
            if (kMode == 2) { ao = ((tap / 3) * 29 + tap % 3) * 128 + 32 * k; bo = 32 * k + tap * (kN / 2) * 128; }
            tc_mma2<false>(tmem, ad0 + (ao >> 4), bd0 + (bo >> 4), make_idesc<false>(256, kN), (g | j) ? 1u : 0u);
          }
        }
        tc_commit2_mc(&bar, 3);
      }
    } else {
      // the window kernel's MMA loop shape: per tap a (completed) barrier wait,
      // fence, elected issue of 4 MMAs, warp sync (mode 4: + a commit per tap)
      __shared__ int32_t taps[9];
      if (threadIdx.x < 9) taps[threadIdx.x] = ((threadIdx.x / 3) * 29 + threadIdx.x % 3);
      __syncwarp();
      for (int g = 0; g < iters / 36; ++g) {
        for (int tap = 0; tap < 9; ++tap) {
          mbar_wait(&done_bar, 0);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t toff = (uint64_t)(taps[tap] * 8);
            const uint64_t bd = bd0 + ((tap * (kN / 2) * 128) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma2<false>(tmem, ad0 + toff + 2 * k, bd + 2 * k, make_idesc<false>(256, kN), (g | tap | k) ? 1u : 0u);
            if (kMode == 4) tc_commit2_mc(&done_bar + 0, 0);
          }
          __syncwarp();
        }
      }
      if (elect_one()) tc_commit2_mc(&bar, 3);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
  } else {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc2<256>(tmem); }
}

template <int kMode, int kN, int kTraffic>
void run_traffic(unsigned long long* d, int warps) {
  cudaFuncSetAttribute(rate<kMode, kN, kTraffic>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaMemset(d, 0, 32);
  rate<kMode, kN, kTraffic><<<2, 128 + 32 * warps, 205 * 1024>>>(36000, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("traffic: %s\n", cudaGetErrorString(e)); return; }
  unsigned long long c[2];
  cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
  if (kTraffic == 3)
    printf("pair M256 N%d K steps + %d warps of tcgen05.ld.x32 per CTA: %6.1f cycles per MMA (ideal %d), %6.1f cycles per load per warp\n",
           kN, warps, c[0] / 36000.0, kN / 2, (double)c[0] * warps / (double)c[1]);
  else
  printf("pair M256 N%d K steps + %d warps of %s.shared.v4 per CTA: %6.1f cycles per MMA (ideal %d), traffic %5.1f B/cycle/SM\n",
         kN, warps, kTraffic == 1 ? "st" : "ld", c[0] / 36000.0, kN / 2, (double)c[1] / (double)c[0]);
}

template <int kMode, int kN>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(rate<kMode, kN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  rate<kMode, kN><<<2, 128, 205 * 1024>>>(3600, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("mode %d: %s\n", kMode, cudaGetErrorString(e)); return; }
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"fixed", "K steps", "3x3 sliding taps", "kernel loop shape", "loop + commit/tap"};
  printf("pair M256 N%d %-18s: %6.1f cycles per MMA (ideal %d)\n", kN, names[kMode], c / 3600.0, kN / 2);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<0, 128>(d); run<1, 128>(d); run<2, 128>(d); run<3, 128>(d);
  run<0, 256>(d); run<1, 256>(d);
  run<0, 64>(d); run<1, 64>(d); run<2, 64>(d);
  for (int w : {1, 2, 4, 8, 12}) run_traffic<1, 128, 1>(d, w);
  for (int w : {1, 2, 4, 8, 12}) run_traffic<1, 128, 2>(d, w);
  for (int w : {4, 12}) run_traffic<1, 256, 1>(d, w);
  for (int w : {4, 12}) run_traffic<1, 64, 1>(d, w);
  for (int w : {4, 8}) run_traffic<1, 128, 3>(d, w);
  for (int w : {4, 8}) run_traffic<1, 64, 3>(d, w);
  return 0;
}
