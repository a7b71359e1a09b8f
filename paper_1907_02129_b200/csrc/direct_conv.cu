// Direct convolution on the device: the correctness oracle of the GPU
// benchmark harness (harness.py), restating the reference's
// convbench.reference.direct_conv (reference.py:30-84): each output starts
// from its bias (+0.0 without one) and accumulates, for ky, kx, c ascending,
// fl(acc + fl(x * w)) -- one rounded multiply and one rounded add per tap
// (__fmul_rn / __fadd_rn, never contracted into an FMA) -- with out-of-bounds
// (padding) taps SKIPPED rather than read from a zero row.  Independent of
// the indirection buffer.  Inputs may be float32 or bfloat16 (a bf16 value
// is exact in float32, so a bf16 layer's oracle is this float32 convolution
// of the bf16 operands); the output is float32.
//
// One thread per output element (n, oy, ox, k), k fastest: the threads of a
// warp share one input pixel's taps (broadcast loads) and read 32 filter
// rows.  It is a gate, not a hot path.
#include <cuda_bf16.h>

#include "icv_internal.h"

namespace icv {
namespace {

template <typename T>
__device__ __forceinline__ float ld_f32(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld_f32<float>(const float* p, int64_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float ld_f32<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

template <typename TX, typename TW>
__global__ void direct_conv_kernel(Geom g, int64_t total, const TX* __restrict__ x, const TW* __restrict__ w,
                                   const float* __restrict__ bias, float* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int k = (int)(i % g.K);
    int64_t pix = i / g.K;
    const int ox = (int)(pix % g.OW);
    pix /= g.OW;
    const int oy = (int)(pix % g.OH);
    const int64_t n = pix / g.OH;
    float acc = bias ? bias[k] : 0.0f;
    const TW* wk = w + (int64_t)k * g.R * g.S * g.C;
    for (int ky = 0; ky < g.R; ++ky) {
      const int iy = oy * g.SY + ky * g.DY - g.PT;
      if (iy < 0 || iy >= g.H) continue;   // padding taps are skipped (reference.py:60-83)
      for (int kx = 0; kx < g.S; ++kx) {
        const int ix = ox * g.SX + kx * g.DX - g.PL;
        if (ix < 0 || ix >= g.W) continue;
        const int64_t xo = ((n * g.H + iy) * g.W + ix) * g.C;
        const int64_t wo = ((int64_t)ky * g.S + kx) * g.C;
        for (int c = 0; c < g.C; ++c) acc = __fadd_rn(acc, __fmul_rn(ld_f32(x, xo + c), ld_f32(wk, wo + c)));
      }
    }
    y[i] = acc;
  }
}

template <typename TX, typename TW>
int launch_t(const Geom& g, int64_t batch, const void* x, const void* w, const float* bias, float* y,
             cudaStream_t st) {
  const int64_t total = batch * g.OH * g.OW * g.K;
  if (total == 0) return ICV_OK;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 32) blocks = 148 * 32;
  direct_conv_kernel<TX, TW><<<blocks, 256, 0, st>>>(g, total, static_cast<const TX*>(x),
                                                      static_cast<const TW*>(w), bias, y);
  note_launch();
  return cuda_check(cudaGetLastError(), "direct_conv launch");
}

}  // namespace
}  // namespace icv

using namespace icv;

extern "C" ICV_API int icv_direct_conv(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch,
                                       int32_t x_dtype, const void* x, int32_t w_dtype, const void* w,
                                       const float* bias, float* y, void* stream) {
  Geom g;
  if (int s = make_geom(desc, in, &g)) return s;
  if (batch < 1 || batch > in->n) return fail(ICV_ERR_ARG, "batch must be within the physical input batch");
  if (!x || !w || !y) return fail(ICV_ERR_ARG, "icv_direct_conv: null tensor");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool xf = x_dtype == ICV_F32, xb = x_dtype == ICV_BF16, wf = w_dtype == ICV_F32, wb = w_dtype == ICV_BF16;
  if (xf && wf) return launch_t<float, float>(g, batch, x, w, bias, y, st);
  if (xb && wb) return launch_t<__nv_bfloat16, __nv_bfloat16>(g, batch, x, w, bias, y, st);
  if (xb && wf) return launch_t<__nv_bfloat16, float>(g, batch, x, w, bias, y, st);
  if (xf && wb) return launch_t<float, __nv_bfloat16>(g, batch, x, w, bias, y, st);
  return fail(ICV_ERR_ARG, "icv_direct_conv: input and filter must be float32 or bfloat16");
}
