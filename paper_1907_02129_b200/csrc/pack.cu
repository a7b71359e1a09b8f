// K7: filter packing (replaces pack_filter, reference gemm.py:135-167).
//
// Tensor-core families: KRSC weights -> rows of `row_bytes` per output
// channel, each row = R*S taps x `cblocks` 128-byte channel blocks (zero
// padded past C), rows zero padded to a multiple of the kernel's BLOCK_N.
// This is exactly the K-major B operand the tcgen05 kernel TMA-loads with a
// 128-byte swizzle: one (tap, channel-block) k-step is one 128-byte column
// of this matrix.  Bias (and, for uint8, the zero-point corrections) are
// folded into one int32/f32 epilogue constant per output channel.
//
// CUDA-core / exact families: KRSC copied (converted to the compute dtype)
// plus the bias.  One-time setup work, off the timed path (gemm.py:135,
// bench.py:220).
#include <cuda_bf16.h>

#include "icv_internal.h"

namespace icv {
namespace {

template <typename Tin>
__device__ __forceinline__ float to_f32(Tin v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// bf16 tensor-core layout: element (n, e, c') of a [n_pad][RS][cblocks*64] bf16 array.
template <typename Tin>
__global__ void pack_tc_bf16(const Tin* __restrict__ w, __nv_bfloat16* __restrict__ out, int K, int RS, int C,
                             int cpad, int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % cpad);
    const int64_t ne = i / cpad;
    const int e = (int)(ne % RS);
    const int n = (int)(ne / RS);
    float v = 0.f;
    if (n < K && c < C) v = to_f32<Tin>(w[((int64_t)n * RS + e) * C + c]);
    out[i] = __float2bfloat16_rn(v);
  }
}

__global__ void pack_tc_u8(const uint8_t* __restrict__ w, uint8_t* __restrict__ out, int K, int RS, int C, int cpad,
                           int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % cpad);
    const int64_t ne = i / cpad;
    const int e = (int)(ne % RS);
    const int n = (int)(ne / RS);
    out[i] = (n < K && c < C) ? w[((int64_t)n * RS + e) * C + c] : (uint8_t)0;
  }
}

// channel-poor layout: out[n][k] = w[n][k] for k < R*S*C (KRSC order = e*C + c), else 0
template <typename Tin>
__global__ void pack_kpacked_bf16(const Tin* __restrict__ w, __nv_bfloat16* __restrict__ out, int K, int kk,
                                  int kpad, int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % kpad);
    const int n = (int)(i / kpad);
    out[i] = __float2bfloat16_rn((n < K && k < kk) ? to_f32<Tin>(w[(int64_t)n * kk + k]) : 0.f);
  }
}

// row-sliding layout (igemm_rows.cu): per kernel row ky a [n_pad][32] K-major
// no-swizzle block, k = kx*4 + c (kx < 8, c < 4), core matrices of 8 rows x
// 8 elements: byte ((n/8)*4 + k/8)*128 + (n%8)*16 + (k%8)*2.
template <typename Tin>
__global__ void pack_rows_bf16(const Tin* __restrict__ w, uint8_t* __restrict__ out, int K, int R, int S, int C,
                               int n_pad, int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % 32);
    const int64_t nk = i / 32;
    const int n = (int)(nk % n_pad);
    const int ky = (int)(nk / n_pad);
    const int kx = k / 4, c = k % 4;
    float v = 0.f;
    if (n < K && kx < S && c < C) v = to_f32<Tin>(w[(((int64_t)n * R + ky) * S + kx) * C + c]);
    const int64_t off = (int64_t)ky * n_pad * 64 + ((n / 8) * 4 + k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(out + off) = __float2bfloat16_rn(v);
  }
}

template <typename Tin, typename Tout>
__global__ void pack_copy(const Tin* __restrict__ w, Tout* __restrict__ out, int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(Tout) == 2) out[i] = __float2bfloat16_rn(to_f32<Tin>(w[i]));
    else out[i] = (Tout)w[i];
  }
}

__global__ void pack_bias_f32(const float* __restrict__ bias, float* __restrict__ out, int K, int n_pad) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_pad; n += gridDim.x * blockDim.x)
    out[n] = (bias != nullptr && n < K) ? bias[n] : 0.f;
}

// uint8: one block per output channel; int64 block reduction of sum(w).
//   tensor-core family: const[n] = bias[n] - zx*sum_w[n] + RS*C*zx*zw
//     (the kernel adds S1 = sum x*w - zw * sum x on top)
//   CUDA-core family:   const[n] = bias[n] (the kernel accumulates (x-zx)(w-zw))
__global__ void pack_bias_u8(const uint8_t* __restrict__ w, const int32_t* __restrict__ bias,
                             int32_t* __restrict__ out, int K, int n_pad, int64_t kk, int zx, int zw, int fold) {
  __shared__ long long part[32];
  const int n = blockIdx.x;
  long long s = 0;
  if (n < K && fold)
    for (int64_t i = threadIdx.x; i < kk; i += blockDim.x) s += w[(int64_t)n * kk + i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += part[i];
    long long v = 0;
    if (n < K) {
      v = bias ? bias[n] : 0;
      if (fold) v += -(long long)zx * tot + kk * (long long)zx * zw;
    }
    out[n] = (int32_t)v;
  }
}

// uint8 tensor-core family: out[e][n] = zx * sum_c (w[n][e][c] - zw), the
// contribution a padded tap (x = zx) has that a zero-filled one (x = 0) lacks
// relative to the folded constants; one block per (e, n).
__global__ void pack_tapcorr_u8(const uint8_t* __restrict__ w, int32_t* __restrict__ out, int K, int n_pad, int RS,
                                int C, int zx, int zw) {
  const int e = blockIdx.x / n_pad, n = blockIdx.x - e * n_pad;
  int s = 0;
  if (n < K)
    for (int c = threadIdx.x; c < C; c += blockDim.x) s += (int)w[((int64_t)n * RS + e) * C + c] - zw;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[(int64_t)e * n_pad + n] = zx * s;
}

int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

int launch_pack(const Geom& g, const PackedLayout& L, int32_t w_dtype, const void* w, const void* bias,
                const icv_quant* q, void* packed, cudaStream_t st) {
  uint8_t* base = static_cast<uint8_t*>(packed);
  const int RS = g.R * g.S;
  const int64_t kk = (int64_t)RS * g.C;
  int launches = 0;
  switch (L.family) {
    case kFamTcBf16: {
      const int cpad = L.cblocks * 64;
      const int64_t total = (int64_t)L.n_pad * RS * cpad;
      auto* out = reinterpret_cast<__nv_bfloat16*>(base + L.w_off);
      if (w_dtype == ICV_F32)
        pack_tc_bf16<float><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(w), out, g.K, RS, g.C, cpad, total);
      else
        pack_tc_bf16<__nv_bfloat16><<<grid_for(total), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w), out, g.K,
                                                                       RS, g.C, cpad, total);
      pack_bias_f32<<<grid_for(L.n_pad), 256, 0, st>>>(static_cast<const float*>(bias),
                                                         reinterpret_cast<float*>(base + L.bias_off), g.K, L.n_pad);
      launches = 2;
      break;
    }
    case kFamStemBf16: {
      const int kpad = L.cblocks * 64;
      const int64_t total = (int64_t)L.n_pad * kpad;
      auto* out = reinterpret_cast<__nv_bfloat16*>(base + L.w_off);
      if (w_dtype == ICV_F32)
        pack_kpacked_bf16<float><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(w), out, g.K, (int)kk,
                                                                   kpad, total);
      else
        pack_kpacked_bf16<__nv_bfloat16><<<grid_for(total), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w), out,
                                                                           g.K, (int)kk, kpad, total);
      pack_bias_f32<<<grid_for(L.n_pad), 256, 0, st>>>(static_cast<const float*>(bias),
                                                         reinterpret_cast<float*>(base + L.bias_off), g.K, L.n_pad);
      launches = 2;
      if (L.rows_off) {
        const int64_t rtotal = (int64_t)g.R * L.n_pad * 32;
        if (w_dtype == ICV_F32)
          pack_rows_bf16<float><<<grid_for(rtotal), 256, 0, st>>>(static_cast<const float*>(w), base + L.rows_off, g.K,
                                                                  g.R, g.S, g.C, L.n_pad, rtotal);
        else
          pack_rows_bf16<__nv_bfloat16><<<grid_for(rtotal), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w),
                                                                          base + L.rows_off, g.K, g.R, g.S, g.C,
                                                                          L.n_pad, rtotal);
        ++launches;
      }
      break;
    }
    case kFamTcU8: {
      const int cpad = L.cblocks * 128;
      const int64_t total = (int64_t)L.n_pad * RS * cpad;
      pack_tc_u8<<<grid_for(total), 256, 0, st>>>(static_cast<const uint8_t*>(w), base + L.w_off, g.K, RS, g.C, cpad,
                                                  total);
      pack_bias_u8<<<L.n_pad, 256, 0, st>>>(static_cast<const uint8_t*>(w), static_cast<const int32_t*>(bias),
                                            reinterpret_cast<int32_t*>(base + L.bias_off), g.K, L.n_pad, kk,
                                            q->input_zero_point, q->kernel_zero_point, 1);
      pack_tapcorr_u8<<<(unsigned)(RS * L.n_pad), 32, 0, st>>>(static_cast<const uint8_t*>(w),
                                                               reinterpret_cast<int32_t*>(base + L.tapcorr_off), g.K,
                                                               L.n_pad, (int)RS, g.C, q->input_zero_point,
                                                               q->kernel_zero_point);
      launches = 3;
      break;
    }
    case kFamF32Exact: {
      const int64_t total = (int64_t)g.K * kk;
      pack_copy<float, float><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(w),
                                                                reinterpret_cast<float*>(base + L.w_off), total);
      pack_bias_f32<<<grid_for(g.K), 256, 0, st>>>(static_cast<const float*>(bias),
                                                     reinterpret_cast<float*>(base + L.bias_off), g.K, g.K);
      launches = 2;
      break;
    }
    case kFamCoreBf16: {
      const int64_t total = (int64_t)g.K * kk;
      auto* out = reinterpret_cast<__nv_bfloat16*>(base + L.w_off);
      if (w_dtype == ICV_F32)
        pack_copy<float, __nv_bfloat16><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(w), out, total);
      else
        pack_copy<__nv_bfloat16, __nv_bfloat16><<<grid_for(total), 256, 0, st>>>(
            static_cast<const __nv_bfloat16*>(w), out, total);
      pack_bias_f32<<<grid_for(g.K), 256, 0, st>>>(static_cast<const float*>(bias),
                                                     reinterpret_cast<float*>(base + L.bias_off), g.K, g.K);
      launches = 2;
      break;
    }
    case kFamCoreU8: {
      const int64_t total = (int64_t)g.K * kk;
      pack_copy<uint8_t, uint8_t><<<grid_for(total), 256, 0, st>>>(static_cast<const uint8_t*>(w), base + L.w_off,
                                                                    total);
      pack_bias_u8<<<g.K, 256, 0, st>>>(static_cast<const uint8_t*>(w), static_cast<const int32_t*>(bias),
                                        reinterpret_cast<int32_t*>(base + L.bias_off), g.K, g.K, kk,
                                        q->input_zero_point, q->kernel_zero_point, 0);
      launches = 2;
      break;
    }
    default:
      return fail(ICV_ERR_UNSUPPORTED, "unknown packing family");
  }
  note_launch(launches);
  return cuda_check(cudaGetLastError(), "pack launch");
}

}  // namespace icv
