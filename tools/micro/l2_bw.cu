// L2 -> SM bandwidth on an L2-resident buffer: plain LDG.128 and cp.async
// (LDGSTS 16B) into shared memory.  One pass = every block streams its
// slice of a 32 MiB buffer; reported as aggregate GB/s.
#include <cstdio>
#include <cstdint>

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n, int reps, uint4* out) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678) out[0] = acc;
}

__global__ void cpasync_kernel(const uint4* __restrict__ p, size_t n, int reps, uint4* out) {
  extern __shared__ uint4 sm[];
  const int slots = 8192;  // 128 KB ring
  int k = threadIdx.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + (k & (slots - 1)));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(p + i) : "memory");
      k += blockDim.x;
      if ((k & 2047) < blockDim.x) asm volatile("cp.async.wait_group 4;\n cp.async.commit_group;" ::: "memory");
    }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (sm[threadIdx.x].x == 0x12345678) out[0] = sm[threadIdx.x];
}

int main() {
  const size_t bytes = 32ull << 20;
  const size_t n = bytes / 16;
  uint4 *p, *out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(p, 1, bytes);
  cudaFuncSetAttribute(cpasync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 20;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      ldg_kernel<<<148 * bps, threads>>>(p, n, 1, out);
      cudaEventRecord(a);
      ldg_kernel<<<148 * bps, threads>>>(p, n, reps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("LDG.128   threads=%4d blocks/SM=%d: %8.0f GB/s\n", threads, bps, reps * bytes / (ms * 1e-3) / 1e9);
    }
  }
  for (int threads : {256, 512, 1024}) {
    cpasync_kernel<<<148, threads, 131072>>>(p, n, 1, out);
    cudaEventRecord(a);
    cpasync_kernel<<<148, threads, 131072>>>(p, n, reps, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDGSTS.16 threads=%4d: %8.0f GB/s (%s)\n", threads, reps * bytes / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
