// Check a "sliding window" A operand in the canonical 128B-swizzle K-major
// layout: a buffer of pixel rows (128 B = 64 bf16 channels each, written with
// the TMA 128B swizzle: 16-byte chunk j of row r at j ^ (r % 8), 1024-byte
// aligned base) and an MMA whose A row m is pixel row s + m, i.e. the
// descriptor start address is base + 128*s (+32*k for the K step).  Tries the
// descriptor's base-offset field = 0 and = (start >> 7) & 7, for several
// slides s, and reports which reproduces the CPU result.  M=128, N=64, K=64,
// bf16 -> f32.  Then times back-to-back sliding MMAs (M128 N128 K16).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

constexpr int kRows = 128 + 64;   // pixel rows in the window

__device__ __forceinline__ uint64_t sw128_desc_bo(uint32_t addr, uint32_t base_off) {
  uint64_t d = sw128_kmajor_desc(addr);
  d |= (uint64_t)(base_off & 7) << 49;
  return d;
}

__global__ void kern(const uint16_t* win, const uint16_t* bmat, float* out, int slide, int use_bo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;                    // kRows x 128 B, swizzled
  uint8_t* sB = smem + kRows * 128 + 1024 - (kRows * 128) % 1024;   // 64 x 128 B, swizzled
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < kRows * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    *reinterpret_cast<uint16_t*>(sW + r * 128 + (((c / 8) ^ (r % 8)) * 16) + (c % 8) * 2) = win[i];
  }
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    *reinterpret_cast<uint16_t*>(sB + r * 128 + (((c / 8) ^ (r % 8)) * 16) + (c % 8) * 2) = bmat[i];
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
      const uint32_t a0 = smem_u32(sW) + 128 * slide, b0 = smem_u32(sB);
      for (int k = 0; k < 4; ++k) {
        const uint32_t aa = a0 + 32 * k;
        const uint64_t ad = sw128_desc_bo(aa, use_bo ? (aa >> 7) & 7 : 0);
        const uint64_t bd = sw128_kmajor_desc(b0 + 32 * k);
        tc_mma<false>(tmem, ad, bd, make_idesc<false>(128, 64), k > 0 ? 1u : 0u);
      }
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

// Rate: iters (multiple of 36) MMAs M128 x N x K16 from one thread, 36 per
// fully unrolled group (descriptor offsets are immediates).  Pattern (A, B):
//   0: A fixed,            B fixed
//   1: A +32k (K step),    B +32k
//   2: A 3x3 taps at row width 29 (unaligned slides) + 32k, B +32k + tap*BN*128
//   3: A 3x3 taps at 8-row aligned slides + 32k,             B as 2
//   4: A 3x3 taps unaligned, no K step, B fixed
template <int kMode, int kN>
__global__ void rate(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t a_addr = smem_u32(smem), b_addr = smem_u32(smem + 32768);
    const uint64_t ad0 = sw128_kmajor_desc(a_addr), bd0 = sw128_kmajor_desc(b_addr);
    long long t0 = clock64();
    if (elect_one()) {
      for (int g = 0; g < iters / 36; ++g) {
#pragma unroll
        for (int j = 0; j < 36; ++j) {
          const int tap = j / 4, k = j % 4;
          uint32_t ao = 0, bo = 0;
          if (kMode == 1) { ao = 32 * k; bo = 32 * k; }
          if (kMode == 2) { ao = ((tap / 3) * 29 + tap % 3) * 128 + 32 * k; bo = 32 * k + tap * kN * 128; }
          if (kMode == 3) { ao = tap * 1024 + 32 * k; bo = 32 * k + tap * kN * 128; }
          if (kMode == 4) { ao = ((tap / 3) * 29 + tap % 3) * 128; }
          tc_mma<false>(tmem, ad0 + (ao >> 4), bd0 + (bo >> 4), make_idesc<false>(128, kN), (g | j) ? 1u : 0u);
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

template <int kMode, int kN>
void run_rate(unsigned long long* dcyc) {
  cudaFuncSetAttribute(rate<kMode, kN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  rate<kMode, kN><<<1, 128, 205 * 1024>>>(1800, dcyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("rate mode %d: %s\n", kMode, cudaGetErrorString(e)); exit(1); }
  unsigned long long c;
  cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"A,B fixed", "A,B K-steps", "3x3 unaligned slides", "3x3 8-row slides", "3x3 slides, no K step"};
  printf("rate N=%d %-24s: %6.1f cycles per MMA (ideal %d)\n", kN, names[kMode], c / 1800.0, kN / 2);
}

static uint16_t to_bf16(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }

int main() {
  std::vector<uint16_t> win(kRows * 64), b(64 * 64);
  std::vector<float> winf(kRows * 64), bf(64 * 64);
  for (int i = 0; i < kRows * 64; ++i) { winf[i] = (float)((i * 7 + i / 64) % 9 - 4); win[i] = to_bf16(winf[i]); }
  for (int i = 0; i < 64 * 64; ++i) { bf[i] = (float)((i * 5) % 7 - 3); b[i] = to_bf16(bf[i]); }
  uint16_t *dw, *db; float* dout;
  cudaMalloc(&dw, win.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(dw, win.data(), win.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int slides[] = {0, 1, 3, 5, 7, 8, 13, 29, 58};
  for (int use_bo = 0; use_bo < 2; ++use_bo) {
    int total_bad = 0;
    for (int s : slides) {
      cudaMemset(dout, 0, 128 * 64 * 4);
      kern<<<1, 128, 48 * 1024>>>(dw, db, dout, s, use_bo);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("slide %d: %s\n", s, cudaGetErrorString(e)); return 1; }
      std::vector<float> out(128 * 64);
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          float ref = 0.f;
          for (int k = 0; k < 64; ++k) ref += winf[(s + m) * 64 + k] * bf[n * 64 + k];
          if (out[m * 64 + n] != ref) ++bad;
        }
      printf("base_offset=%s slide %2d: %d / %d mismatches\n", use_bo ? "(addr>>7)&7" : "0", s, bad, 128 * 64);
      total_bad += bad;
    }
    printf("SUMMARY base_offset=%s: %s\n", use_bo ? "(addr>>7)&7" : "0", total_bad ? "WRONG" : "EXACT");
  }
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 8);
  run_rate<0, 128>(dcyc); run_rate<1, 128>(dcyc); run_rate<2, 128>(dcyc); run_rate<3, 128>(dcyc); run_rate<4, 128>(dcyc);
  run_rate<0, 256>(dcyc); run_rate<1, 256>(dcyc); run_rate<2, 256>(dcyc); run_rate<3, 256>(dcyc); run_rate<4, 256>(dcyc);
  return 0;
}
