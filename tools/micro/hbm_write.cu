// HBM write bandwidth on a B200 by store path (what an output-heavy layer can
// reach): cudaMemsetAsync, 16-byte st.global from every thread, and 1-D bulk
// stores (cp.async.bulk.global.shared, TMA) of 16 KB smem blocks; plus the
// read-only and 1:1 copy rates for scale.  1 GiB buffers, best of 10.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_write hbm_write.cu
#include <cstdio>
#include <cstdint>

__global__ void st16(uint4* p, size_t n) {
  const uint4 v = make_uint4(1, 2, 3, 4);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void ld16(const uint4* __restrict__ p, size_t n, uint4* out) {
  uint4 a = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    a.x ^= v.x; a.y ^= v.y; a.z ^= v.z; a.w ^= v.w;
  }
  if (a.x == 0x1234567) out[0] = a;
}
__global__ void cp16(const uint4* __restrict__ s, uint4* d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = __ldcs(s + i);
}
// bulk stores: each CTA owns a contiguous slice; `issuers` warps (lane 0) each
// store 16 KB blocks from smem, `inflight` bulk groups outstanding per issuer
__global__ void bulk_st(uint8_t* p, size_t bytes_per_cta, int issuers, int inflight) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) || w >= issuers) return;
  uint8_t* base = p + blockIdx.x * bytes_per_cta;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
  int k = 0;
  for (size_t off = (size_t)w * 16384; off < bytes_per_cta; off += (size_t)issuers * 16384, ++k) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(base + off), "r"(src) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (inflight == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float m = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    m = ms < m ? ms : m;
  }
  return m;
}

int main() {
  const size_t bytes = size_t(1) << 30;
  uint8_t *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  const size_t n = bytes / 16;
  const int blocks = 148 * 8;
  float t = best([&] { cudaMemsetAsync(b, 3, bytes); });
  printf("cudaMemsetAsync        %8.1f GB/s\n", bytes / t / 1e6);
  t = best([&] { st16<<<blocks, 256>>>((uint4*)b, n); });
  printf("st.global 16B          %8.1f GB/s\n", bytes / t / 1e6);
  t = best([&] { ld16<<<blocks, 256>>>((const uint4*)a, n, (uint4*)b); });
  printf("ld.global 16B (read)   %8.1f GB/s\n", bytes / t / 1e6);
  t = best([&] { cp16<<<blocks, 256>>>((const uint4*)a, (uint4*)b, n); });
  printf("copy 16B (r+w)         %8.1f GB/s\n", 2 * bytes / t / 1e6);
  cudaFuncSetAttribute(bulk_st, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (int issuers : {1, 2, 4})
    for (int inflight : {2, 8}) {
      const size_t per = bytes / 148 / 16384 * 16384;
      t = best([&] { bulk_st<<<148, 128, 16384>>>(b, per, issuers, inflight); });
      printf("bulk store issuers=%d inflight=%d %8.1f GB/s\n", issuers, inflight, per * 148 / t / 1e6);
    }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
