// TMA rate of the window kernel's box shape: a 4-D NHWC bf16 tensor
// (C=128, W=28, H=28, N=64: cfg2), boxes {64 ch, bw px, bh rows, 1 image}
// (128-byte swizzle) loaded by one thread per SM with `stages` loads in
// flight, every SM walking different windows.  Variants: start column -1
// (one out-of-bounds zero column per row, as the kernel does) vs 0; box rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_window tma_window.cu -lcuda
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_cl(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

__device__ __forceinline__ void arrive_remote_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ int g_wait_mode;
__device__ int g_relaxed;
__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t parity) {
  if (g_wait_mode == 1) { while (!mbar_test(bar, parity)) {} }
  else if (g_wait_mode == 2) { while (!mbar_try_cl(bar, parity)) {} }
  else mbar_wait(bar, parity);
}

__global__ void win_kernel(const __grid_constant__ CUtensorMap tm, int box_bytes, int stages, int iters, int x0,
                           int bh, int cbs, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) mbar_wait(&bar[s], ((it - stages) / stages) & 1);
    if (it < iters) {
      mbar_arrive_expect_tx(&bar[s], box_bytes);
      const int w = blockIdx.x * 37 + it;
      const int n = (w / 4) % 64, y = (w % 4) * 7 - 1, cb = (w / 256) % cbs;
      tma_load_4d(smem_u32(base + s * ((box_bytes + 1023) / 1024 * 1024)), &tm, &bar[s], cb * 64, x0, y < 0 ? 0 : y, n);
    }
  }
  long long t1 = clock64();
  cyc[blockIdx.x] = t1 - t0;
}

// the same, launched as 2-CTA clusters (no inter-CTA interaction)
__global__ void __cluster_dims__(2, 1, 1) win_cl_kernel(const __grid_constant__ CUtensorMap tm, int box_bytes, int stages, int iters, int x0,
                           int bh, int cbs, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) mbar_wait(&bar[s], ((it - stages) / stages) & 1);
    if (it < iters) {
      mbar_arrive_expect_tx(&bar[s], box_bytes);
      const int w = blockIdx.x * 37 + it;
      const int n = (w / 4) % 64, y = (w % 4) * 7 - 1, cb = (w / 256) % cbs;
      tma_load_4d(smem_u32(base + s * ((box_bytes + 1023) / 1024 * 1024)), &tm, &bar[s], cb * 64, x0, y < 0 ? 0 : y, n);
    }
  }
  long long t1 = clock64();
  cyc[blockIdx.x] = t1 - t0;
}

// CTA-pair version: both CTAs of a cluster load their own window into their
// own smem, completion counted at the leader's barrier (the window kernel's
// .cta_group::2 path); the leader waits and releases the peer via a remote
// arrive on the peer's "empty" barrier.
__global__ void __cluster_dims__(2, 1, 1) win_pair_kernel(const __grid_constant__ CUtensorMap tm, int box_bytes,
                                                          int stages, int iters, int x0, int cbs,
                                                          unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  cluster_sync_all();
  const int slot = (box_bytes + 1023) / 1024 * 1024;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (it >= stages) wait_mode(&empty[s], ((it - stages) / stages) & 1);
      if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * box_bytes);
      const int w = blockIdx.x * 37 + it;
      const int n = (w / 4) % 64, y = (w % 4) * 7 - 1, cb = (w / 256) % cbs;
      tma_load_4d_cg2(smem_u32(base + s * slot), &tm, mapa_rank(smem_u32(&full[s]), 0), cb * 64, x0, y < 0 ? 0 : y, n);
    }
  } else if (threadIdx.x == 32 && rank == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      wait_mode(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
      (g_relaxed ? arrive_remote_relaxed : mbar_arrive_remote)(mapa_rank(smem_u32(&empty[s]), 1));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  cluster_sync_all();
}

// Forwarded variant: each CTA's TMA completes on its OWN barrier; the peer
// waits on it and forwards one remote arrive to the leader's full barrier
// (count 2: the leader's expect_tx arrive + the peer's forward).
__global__ void __cluster_dims__(2, 1, 1) win_fwd_kernel(const __grid_constant__ CUtensorMap tm, int box_bytes,
                                                         int stages, int iters, int x0, int cbs,
                                                         unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16], local[16];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 2); mbar_init(&empty[s], 1); mbar_init(&local[s], 1); }
    fence_mbar_init();
  }
  cluster_sync_all();
  const int slot = (box_bytes + 1023) / 1024 * 1024;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (it >= stages) wait_mode(&empty[s], ((it - stages) / stages) & 1);
      const int w = blockIdx.x * 37 + it;
      const int n = (w / 4) % 64, y = (w % 4) * 7 - 1, cb = (w / 256) % cbs;
      uint64_t* bar = rank == 0 ? &full[s] : &local[s];
      mbar_arrive_expect_tx(bar, box_bytes);
      tma_load_4d(smem_u32(base + s * slot), &tm, bar, cb * 64, x0, y < 0 ? 0 : y, n);
    }
  } else if (threadIdx.x == 32 && rank == 1) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      wait_mode(&local[s], (it / stages) & 1);
      (g_relaxed ? arrive_remote_relaxed : mbar_arrive_remote)(mapa_rank(smem_u32(&full[s]), 0));
    }
  } else if (threadIdx.x == 64 && rank == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      wait_mode(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
      (g_relaxed ? arrive_remote_relaxed : mbar_arrive_remote)(mapa_rank(smem_u32(&empty[s]), 1));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  cluster_sync_all();
}

int main() {
  const int nsm = 148, C = 128, W = 28, H = 28, N = 64;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  uint16_t* d;
  cudaMalloc(&d, (size_t)N * H * W * C * 2);
  cudaMemset(d, 1, (size_t)N * H * W * C * 2);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, nsm * 8);
  cudaFuncSetAttribute(win_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(win_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(win_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(win_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct V { int bw, bh, x0; const char* what; } vs[] = {
      {29, 8, -1, "29 px x 8 rows from x=-1 (kernel)"}, {28, 8, 0, "28 px x 8 rows from x=0"},
      {29, 4, -1, "29 px x 4 rows from x=-1"}, {28, 4, 0, "28 px x 4 rows from x=0"},
      {32, 8, -2, "32 px x 8 rows from x=-2"}};
  for (auto v : vs) {
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)v.bw, (cuuint32_t)v.bh, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    const int box_bytes = v.bw * v.bh * 128;
    for (int stages : {1, 2, 4}) {
      const int iters = 400;
      win_kernel<<<nsm, 32, stages * ((box_bytes + 1023) / 1024 * 1024) + 1024>>>(tm, box_bytes, stages, iters, v.x0,
                                                                                  v.bh, C / 64, dcyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<unsigned long long> c(nsm);
      cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (auto x : c) mx = x > mx ? x : mx;
      printf("%-36s (%5d B) stages=%d: %5.0f cycles/load, %5.1f B/cycle/SM\n", v.what, box_bytes, stages, mx / iters,
             box_bytes * (double)iters / mx);
      win_cl_kernel<<<nsm, 32, stages * ((box_bytes + 1023) / 1024 * 1024) + 1024>>>(tm, box_bytes, stages, iters, v.x0,
                                                                                    v.bh, C / 64, dcyc);
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("cl error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
      mx = 0;
      for (auto x : c) mx = x > mx ? x : mx;
      printf("%-36s (%5d B) stages=%d CLUSTER-LOCAL: %5.0f cycles/load\n", v.what, box_bytes, stages, mx / iters);
      for (int mode = 0; mode < 4; ++mode) {
      const int wm = mode == 3 ? 0 : mode, rel = mode == 3;
      cudaMemcpyToSymbol(g_wait_mode, &wm, 4);
      cudaMemcpyToSymbol(g_relaxed, &rel, 4);
      win_pair_kernel<<<nsm, 64, stages * ((box_bytes + 1023) / 1024 * 1024) + 1024>>>(tm, box_bytes, stages, iters,
                                                                                       v.x0, C / 64, dcyc);
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("pair error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
      mx = 0;
      for (auto x : c) mx = x > mx ? x : mx;
      printf("%-36s (%5d B) stages=%d PAIR wait=%s: %5.0f cycles/load, %5.1f B/cycle/SM\n", v.what, box_bytes, stages,
             mode == 0 ? "try_sleep" : mode == 1 ? "test_spin" : mode == 2 ? "try_cluster" : "try_sleep+relaxed_remote", mx / iters, box_bytes * (double)iters / mx);
      }
      { const int one = 1; cudaMemcpyToSymbol(g_relaxed, &one, 4); }
      win_fwd_kernel<<<nsm, 96, stages * ((box_bytes + 1023) / 1024 * 1024) + 1024>>>(tm, box_bytes, stages, iters,
                                                                                      v.x0, C / 64, dcyc);
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("fwd error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
      mx = 0;
      for (auto x : c) mx = x > mx ? x : mx;
      printf("%-36s (%5d B) stages=%d FWD(relaxed):  %5.0f cycles/load, %5.1f B/cycle/SM\n", v.what, box_bytes, stages,
             mx / iters, box_bytes * (double)iters / mx);
    }
  }
  return 0;
}
