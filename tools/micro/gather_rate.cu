// How fast can one CTA per SM gather 128-byte rows through row indices into
// a ring of 128B-swizzled 16 KB smem tiles (the IB-gather kernel's A fill)?
// Every CTA walks "tiles" of 128 output pixels x taps x channel blocks of a
// synthetic NHWC u8 input with the cfg4 / cfg2 geometries (or a linear
// pattern), a consumer thread releases each stage as soon as it is full.
//   mode 0: LDGSTS (cp.async 16 B, 8 lanes per row, 4 rows per instruction)
//   mode 1: TMA tile::gather4, one instruction per 4 rows, issued by the
//           lanes of the producer warps
//   mode 2: LDGSTS, 16 lanes per row covering both channel blocks of a pixel
//           (256 contiguous bytes per row request; two stages filled at once)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/gather_rate gather_rate.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1907_02129_b200/csrc/sm100_ptx.cuh"
using namespace icv;

struct Geo {
  int H, W, C;       // input (bytes per pixel = C)
  int OH, OW, S, P;  // output grid, stride, pad (3x3 taps)
  int linear;        // 1: row r of stage q = consecutive 128-byte rows (no conv pattern)
  int tiles;         // M tiles in total
  int cblocks;
};

// idx[cta][local stage q][row]: byte offset / 128 of the row's 128-byte block (host-built: the "indirection buffer")
// (copied to shared memory before the timed loop, like the kernel's staged index slices)
__device__ __forceinline__ const int* stage_idx(const int* idx, long long stages_per_cta, long long q) {
  return idx + q * 128;
}

template <int kMode>
__global__ void __launch_bounds__(1024, 1) gather_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* x, const int* idx, long long spc, Geo g,
                                                         int prod_warps, int stages, unsigned long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], kMode == 1 ? 1 : kMode == 9 ? 65 : 32 * prod_warps);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  {
    int* sidx = reinterpret_cast<int*>(smem + stages * 16384);
    const int* src = idx + (long long)blockIdx.x * spc * 128;
    for (int i = threadIdx.x; i < spc * 128; i += blockDim.x) sidx[i] = src[i];
    idx = sidx;
  }
  __syncthreads();
  const int nkb = 9 * g.cblocks;
  long long my_tiles = 0;
  for (long long t = blockIdx.x; t < g.tiles; t += 148) ++my_tiles;   // (the table is built for 148 CTAs)
  const long long total = my_tiles * nkb;
  long long t0 = clock64();
  if (warp < prod_warps) {
    const int rows_w = prod_warps == 31 ? 4 : 128 / prod_warps;   // (31: rows 124..127 idle -- rate probe only)   // rows per producer warp
    if (kMode == 0 || kMode == 4 || kMode == 5) {
      const int chunk = lane & 7, sub = lane >> 3;
      int stage = 0;
      uint32_t phase = 0;
      int nxt[8];
      for (int i = 0; i < rows_w / 4; ++i) nxt[i] = stage_idx(idx, spc, 0)[warp * rows_w + 4 * i + sub];
      for (long long q = 0; q < total; ++q) {
        int cur[8];
        for (int i = 0; i < rows_w / 4; ++i) cur[i] = nxt[i];
        if (q + 1 < total)
          for (int i = 0; i < rows_w / 4; ++i) nxt[i] = stage_idx(idx, spc, q + 1)[warp * rows_w + 4 * i + sub];
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t base = smem_u32(smem) + stage * 16384;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < rows_w / 4) {
            const int row = warp * rows_w + 4 * i + sub;
            const int dc = kMode == 4 ? chunk : kMode == 5 ? (chunk ^ ((row & 3) << 1)) : (chunk ^ (row & 7));
            cp_async_16_full(base + row * 128 + (dc << 4), x + (long long)cur[i] * 128 + chunk * 16);
          }
        }
        cp_async_mbar_arrive_noinc(&full[stage]);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    } else if (kMode == 9) {
      // split fill: rows [0, 64) by LDGSTS from producer warps 0-1 (mode 0's pattern), rows [64, 128) by
      // TMA gather4 from 16 lanes of producer warp 2 -- do the two paths add up?
      // full barrier: 64 LDGSTS-thread arrivals + 1 expect_tx arrival (8 KB)
      const int chunk = lane & 7, sub = lane >> 3;
      const int bpp = g.C / 128;
      int stage = 0;
      uint32_t phase = 0;
      for (long long q = 0; q < total; ++q) {
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t base = smem_u32(smem) + stage * 16384;
        if (warp < 2) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = warp * 32 + 4 * i + sub;
            cp_async_16_full(base + row * 128 + ((chunk ^ (row & 7)) << 4),
                             x + (long long)stage_idx(idx, spc, q)[row] * 128 + chunk * 16);
          }
          cp_async_mbar_arrive_noinc(&full[stage]);
        } else if (warp == 2) {
          if (lane == 0) mbar_arrive_expect_tx(&full[stage], 8192);
          __syncwarp();
          if (lane < 16) {
            const int j = 16 + lane;   // rows 4j .. 4j+3
            const int* r = stage_idx(idx, spc, q) + 4 * j;
            tma_gather4(base + j * 512, &tm, &full[stage], (r[0] % bpp) * 128, r[0] / bpp, r[1] / bpp, r[2] / bpp,
                        r[3] / bpp);
          }
        }
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    } else if (kMode == 8) {
      // LDG.128 into registers (all of a stage's rows of this warp in flight), then STS.128 into the
      // swizzled tile, proxy fence, plain mbarrier arrive -- the data passes through registers (row sums possible)
      const int chunk = lane & 7, sub = lane >> 3;
      int stage = 0;
      uint32_t phase = 0;
      for (long long q = 0; q < total; ++q) {
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < rows_w / 4) {
            const int row = warp * rows_w + 4 * i + sub;
            v[i] = __ldcg(reinterpret_cast<const uint4*>(x + (long long)stage_idx(idx, spc, q)[row] * 128 + chunk * 16));
          }
        }
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* base = smem + stage * 16384;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < rows_w / 4) {
            const int row = warp * rows_w + 4 * i + sub;
            *reinterpret_cast<uint4*>(base + row * 128 + ((chunk ^ (row & 7)) << 4)) = v[i];
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&full[stage]);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    } else if (kMode == 6 || kMode == 7) {
      // no mbarriers at all: mode 0's loads into the ring, throttled only by wait_group (l2_bw.cu's scheme);
      // mode 7 also skips the index lookup (linear addresses computed from q)
      const int chunk = lane & 7, sub = lane >> 3;
      int stage = 0;
      for (long long q = 0; q < total; ++q) {
        const uint32_t base = smem_u32(smem) + stage * 16384;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < rows_w / 4) {
            const int row = warp * rows_w + 4 * i + sub;
            const long long blk = kMode == 7 ? ((long long)blockIdx.x * spc + q) * 128 + row
                                             : (long long)stage_idx(idx, spc, q)[row];
            cp_async_16_full(base + row * 128 + ((chunk ^ (row & 7)) << 4), x + blk * 128 + chunk * 16);
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 6;" ::: "memory");
        if (++stage == stages) stage = 0;
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else if (kMode == 3) {
      // mode 0's loads, completion by commit_group / wait_group: stage q - kLag is
      // arrived on (plain mbarrier arrive) once its group has landed
      constexpr int kLag = 3;
      const int chunk = lane & 7, sub = lane >> 3;
      int stage = 0;
      uint32_t phase = 0;
      for (long long q = 0; q < total + kLag; ++q) {
        if (q < total) {
          int cur[8];
          for (int i = 0; i < rows_w / 4; ++i) cur[i] = stage_idx(idx, spc, q)[warp * rows_w + 4 * i + sub];
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t base = smem_u32(smem) + stage * 16384;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i < rows_w / 4) {
              const int row = warp * rows_w + 4 * i + sub;
              cp_async_16_full(base + row * 128 + ((chunk ^ (row & 7)) << 4), x + (long long)cur[i] * 128 + chunk * 16);
            }
          }
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (q >= kLag) {
          asm volatile("cp.async.wait_group %0;" ::"n"(kLag) : "memory");
          fence_proxy_async_smem();
          mbar_arrive(&full[(q - kLag) % stages]);
        }
      }
    } else if (kMode == 2) {
      // 16 lanes per pixel row (cblocks == 2): one instruction covers 2 rows x 256 bytes, filling stages q, q+1
      const int chunk = lane & 7, cbl = (lane >> 3) & 1, sub = lane >> 4;
      int stage = 0;
      uint32_t phase = 0;
      for (long long q = 0; q < total; q += 2) {
        int cur[16];
        for (int i = 0; i < rows_w / 2; ++i) cur[i] = stage_idx(idx, spc, q + cbl)[warp * rows_w + 2 * i + sub];
        const int st2 = stage + 1 == stages ? 0 : stage + 1;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_wait(&empty[st2], st2 == 0 ? phase : phase ^ 1);
        const uint32_t base = smem_u32(smem) + (cbl ? st2 : stage) * 16384;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i < rows_w / 2) {
            const int row = warp * rows_w + 2 * i + sub;
            cp_async_16_full(base + row * 128 + ((chunk ^ (row & 7)) << 4), x + (long long)cur[i] * 128 + chunk * 16);
          }
        }
        cp_async_mbar_arrive_noinc(&full[stage]);
        cp_async_mbar_arrive_noinc(&full[st2]);
        stage += 2;
        if (stage >= stages) { stage -= stages; phase ^= 1; }
      }
    } else {
      // gather4: 32 instructions per stage, lane l of warp w issues instruction j = w + prod_warps * l' ...
      const int per_warp = 32 / prod_warps;   // instructions per warp per stage (prod_warps <= 32)
      int stage = 0;
      uint32_t phase = 0;
      const int bpp = g.C / 128;   // 128-byte blocks per pixel
      for (long long q = 0; q < total; ++q) {
        int r[4] = {0, 0, 0, 0};
        if (lane < per_warp) {
          const int j = warp * per_warp + lane;   // rows 4j .. 4j+3
          for (int k = 0; k < 4; ++k) r[k] = stage_idx(idx, spc, q)[4 * j + k];
        }
        mbar_wait(&empty[stage], phase ^ 1);
        if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&full[stage], 16384);
        __syncwarp();
        if (lane < per_warp) {
          const int j = warp * per_warp + lane;
          tma_gather4(smem_u32(smem) + stage * 16384 + j * 512, &tm, &full[stage], (r[0] % bpp) * 128, r[0] / bpp,
                      r[1] / bpp, r[2] / bpp, r[3] / bpp);
        }
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == prod_warps && lane == 0 && kMode != 6 && kMode != 7) {
    int stage = 0;
    uint32_t phase = 0;
    for (long long q = 0; q < total; ++q) {
      mbar_wait(&full[stage], phase);
      mbar_arrive(&empty[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 148 * 8);
  uint8_t* flush;
  cudaMalloc(&flush, 512u << 20);
  struct Case { const char* name; Geo g; int N; };
  Case cases[] = {
      {"cfg4 (s2, 256 B pixels)", {28, 28, 256, 14, 14, 2, 1, 0, 196, 2}, 128},
      {"cfg2 (s1, 256 B pixels)", {28, 28, 256, 28, 28, 1, 1, 0, 392, 2}, 64},
      {"cfg3b-like (s1, 512 B pixels)", {64, 64, 512, 64, 64, 1, 1, 0, 296, 4}, 16},
      {"linear", {28, 28, 256, 14, 14, 2, 1, 1, 196, 2}, 128},
  };
  for (auto& c : cases) {
    Geo g = c.g;
    size_t bytes = g.linear ? (size_t)g.tiles * 9 * g.cblocks * 16384 : (size_t)c.N * g.H * g.W * g.C;
    uint8_t* x;
    cudaMalloc(&x, bytes);
    cudaMemset(x, 1, bytes);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)g.C, (cuuint64_t)(bytes / g.C)};
    cuuint64_t strides[1] = {(cuuint64_t)g.C};
    cuuint32_t box[2] = {128, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    // per-CTA stage lists (tile t of CTA b = b + t * 148; stage = (tap, channel block))
    const int nkb = 9 * g.cblocks;
    const long long spc = (long long)((g.tiles + 147) / 148) * nkb;
    std::vector<int> hidx((size_t)148 * spc * 128, 0);
    for (int b = 0; b < 148; ++b) {
      long long q = 0;
      for (long long t = b; t < g.tiles; t += 148)
        for (int kb = 0; kb < nkb; ++kb, ++q)
          for (int row = 0; row < 128; ++row) {
            long long off;
            if (g.linear) {
              off = ((t * nkb + kb) * 128 + row) * 128;
            } else {
              const int tap = kb / g.cblocks, cb = kb % g.cblocks;
              const long long p = t * 128 + row;
              const int ohw = g.OH * g.OW;
              const long long n = p / ohw;
              const int r = (int)(p - n * ohw);
              const int oy = r / g.OW, ox = r - oy * g.OW;
              int iy = oy * g.S - g.P + tap / 3, ix = ox * g.S - g.P + tap % 3;
              iy = iy < 0 ? 0 : (iy >= g.H ? g.H - 1 : iy);   // (clamped instead of the zero row)
              ix = ix < 0 ? 0 : (ix >= g.W ? g.W - 1 : ix);
              off = (((n * g.H + iy) * g.W + ix) * (long long)g.C) + cb * 128;
            }
            hidx[((size_t)b * spc + q) * 128 + row] = (int)(off / 128);
          }
    }
    int* idx;
    cudaMalloc(&idx, hidx.size() * 4);
    cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice);
    const double gathered = (double)g.tiles * 9 * g.cblocks * 16384;
    printf("== %s: input %.1f MB, gathered %.1f MB\n", c.name, bytes / 1e6, gathered / 1e6);
    for (int grid : {148})
    for (int mode : {0, 1, 2, 9}) {
      if (mode == 2 && g.cblocks != 2) continue;
      if ((mode == 1 || mode == 9) && g.linear) continue;
      if (mode == 2 && g.cblocks != 2) continue;
      if (mode == 1 && g.linear) continue;
      for (int pw : {4, 8}) {
        if (mode == 9 && pw != 4) continue;
        for (int stages : {10}) {
          for (int cold = 0; cold < 1; ++cold) {
            const int smem = stages * 16384 + 1024 + (int)spc * 512;
            const int threads = 32 * (pw + 1);
            if (smem > 232448) continue;
            float best = 1e9f;
            for (int rep = 0; rep < 3; ++rep) {
              if (cold) cudaMemset(flush, rep, 512u << 20);
              cudaEvent_t a, b;
              cudaEventCreate(&a); cudaEventCreate(&b);
              cudaEventRecord(a);
              if (mode == 0) {
                cudaFuncSetAttribute(gather_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<0><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 1) {
                cudaFuncSetAttribute(gather_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<1><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 9) {
                cudaFuncSetAttribute(gather_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<9><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 8) {
                cudaFuncSetAttribute(gather_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<8><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 6) {
                cudaFuncSetAttribute(gather_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<6><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 7) {
                cudaFuncSetAttribute(gather_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<7><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 4) {
                cudaFuncSetAttribute(gather_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<4><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 5) {
                cudaFuncSetAttribute(gather_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<5><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else if (mode == 3) {
                cudaFuncSetAttribute(gather_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<3><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              } else {
                cudaFuncSetAttribute(gather_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                gather_kernel<2><<<grid, threads, smem>>>(tm, x, idx, spc, g, pw, stages, dcyc);
              }
              cudaEventRecord(b);
              cudaEventSynchronize(b);
              float ms;
              cudaEventElapsedTime(&ms, a, b);
              if (ms < best) best = ms;
              cudaEventDestroy(a); cudaEventDestroy(b);
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long hc[148];
            cudaMemcpy(hc, dcyc, sizeof(hc), cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = hc[i] > mx ? hc[i] : mx;
            printf("grid %3d mode %d  prod warps %2d  stages %2d  %s: %7.2f us  %6.2f TB/s | in-kernel loop %6llu cycles (max)  %5.1f B/cycle/SM\n",
                   grid, mode, pw, stages, cold ? "cold" : "warm", best * 1e3, gathered / (best * 1e-3) / 1e12, mx,
                   (double)((g.tiles + 147) / 148) * 9 * g.cblocks * 16384 / (double)mx);
          }
        }
      }
    }
    cudaFree(x);
    cudaFree(idx);
  }
  return 0;
}
