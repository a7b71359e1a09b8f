// tcgen05.ld (TMEM -> registers) latency and throughput on a B200: one CTA
// per SM allocates 512 TMEM columns; `warps` warps (warp w reads lane
// quarter w % 4) each loop `iters` times over: issue `batch` loads of
// 32x32b.x32 (32 columns) or one .x64 / .x128, then tcgen05.wait::ld, and
// fold the registers so nothing is dead.  Reports cycles per load batch per
// warp and TMEM bytes per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu
#include <cstdio>
#include <vector>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__device__ __forceinline__ void ld_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

template <int kMode>   // 0: one x32 per wait, 1: two x32 per wait, 2: one x64 per wait
__global__ void tmem_kernel(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = (uint32_t)((i * 64 + warp * 128) & 511);
    if constexpr (kMode == 0) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(base + (col & 480), r);
      tmem_ld_wait_regs(r);
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k];
    } else if constexpr (kMode == 1) {
      uint32_t r[32], q[32];
      tmem_ld_32x32b_x32(base + (col & 448), r);
      tmem_ld_32x32b_x32(base + (col & 448) + 32, q);
      tmem_ld_wait_regs(r);
      tmem_ld_wait_regs(q);
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k] ^ q[k];
    } else {
      uint32_t r[64];
      ld_x64(base + (col & 448), r);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 64; ++k) acc += r[k];
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0 && warp == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int kMode>
void run(int warps, unsigned long long* dcyc, uint32_t* sink) {
  const int iters = 4000;
  tmem_kernel<kMode><<<148, 32 * warps>>>(iters, dcyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  std::vector<unsigned long long> c(148);
  cudaMemcpy(c.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (auto v : c) mx = v > mx ? v : mx;
  const int cols = kMode == 0 ? 32 : 64;
  printf("mode %s warps %2d: %6.0f cycles per wait (per warp), %6.1f B/cycle/SM\n",
         kMode == 0 ? "x32      " : kMode == 1 ? "2 x x32  " : "x64      ", warps, mx / iters,
         (double)warps * iters * cols * 32 * 4 / mx);
}

int main() {
  unsigned long long* dcyc;
  uint32_t* sink;
  cudaMalloc(&dcyc, 148 * 8);
  cudaMalloc(&sink, 64);
  for (int warps : {4, 8, 16}) {
    run<0>(warps, dcyc, sink);
    run<1>(warps, dcyc, sink);
    run<2>(warps, dcyc, sink);
  }
  return 0;
}
