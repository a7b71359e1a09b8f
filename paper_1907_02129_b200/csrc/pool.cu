// NHWC max pooling (the 3x3/2 p1 pool after the ResNet-50 stem, cfg5).
// Not part of the reference operator: the conv stack of SURVEY.md §8(d)
// needs it between the stem and stage 1.  HBM-bound: one thread per output
// pixel and 8-channel group (16-byte loads of each in-window pixel, bf16
// max with __hmax2); padding taps are skipped (= -inf padding).  Other
// channel counts / dtypes use the element-wise variant.
#include <cuda_bf16.h>

#include "icv_internal.h"

namespace icv {
namespace {

struct PoolGeom {
  int n, h, w, c, oh, ow, kh, kw, sh, sw, ph, pw;
};

__global__ void maxpool_bf16x8(const uint4* __restrict__ x, uint4* __restrict__ y, PoolGeom g, int64_t total) {
  const int cg = g.c / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i % cg);
    int64_t pix = i / cg;
    const int ox = (int)(pix % g.ow);
    pix /= g.ow;
    const int oy = (int)(pix % g.oh);
    const int n = (int)(pix / g.oh);
    __nv_bfloat162 m[4];
    bool any = false;
    for (int ky = 0; ky < g.kh; ++ky) {
      const int iy = oy * g.sh - g.ph + ky;
      if (iy < 0 || iy >= g.h) continue;
      for (int kx = 0; kx < g.kw; ++kx) {
        const int ix = ox * g.sw - g.pw + kx;
        if (ix < 0 || ix >= g.w) continue;
        const uint4 v = __ldg(x + (((int64_t)n * g.h + iy) * g.w + ix) * cg + q);
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = any ? __hmax2(m[j], b[j]) : b[j];
        any = true;
      }
    }
    uint4 out = make_uint4(0, 0, 0, 0);
    if (any) out = *reinterpret_cast<const uint4*>(m);
    y[i] = out;
  }
}

template <typename T>
__global__ void maxpool_scalar(const T* __restrict__ x, T* __restrict__ y, PoolGeom g, int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % g.c);
    int64_t pix = i / g.c;
    const int ox = (int)(pix % g.ow);
    pix /= g.ow;
    const int oy = (int)(pix % g.oh);
    const int n = (int)(pix / g.oh);
    float m = 0.f;
    bool any = false;
    for (int ky = 0; ky < g.kh; ++ky) {
      const int iy = oy * g.sh - g.ph + ky;
      if (iy < 0 || iy >= g.h) continue;
      for (int kx = 0; kx < g.kw; ++kx) {
        const int ix = ox * g.sw - g.pw + kx;
        if (ix < 0 || ix >= g.w) continue;
        const float v = (float)x[(((int64_t)n * g.h + iy) * g.w + ix) * g.c + ch];
        m = any ? fmaxf(m, v) : v;
        any = true;
      }
    }
    y[i] = (T)m;
  }
}

}  // namespace

int launch_maxpool(const icv_shape4& in, int kh, int kw, int sh, int sw, int ph, int pw, int dtype, const void* x,
                   void* y, cudaStream_t st) {
  PoolGeom g{(int)in.n, (int)in.h, (int)in.w, (int)in.c, 0, 0, kh, kw, sh, sw, ph, pw};
  g.oh = (g.h + 2 * ph - kh) / sh + 1;
  g.ow = (g.w + 2 * pw - kw) / sw + 1;
  const int64_t pixels = (int64_t)g.n * g.oh * g.ow;
  const bool vec = dtype == ICV_BF16 && g.c % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  const int64_t total = vec ? pixels * (g.c / 8) : pixels * g.c;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  if (vec) {
    maxpool_bf16x8<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint4*>(x), static_cast<uint4*>(y), g, total);
  } else if (dtype == ICV_BF16) {
    maxpool_scalar<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                                      static_cast<__nv_bfloat16*>(y), g, total);
  } else if (dtype == ICV_F32) {
    maxpool_scalar<float><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const float*>(x), static_cast<float*>(y), g,
                                                              total);
  } else {
    return fail(ICV_ERR_UNSUPPORTED, "max pool: bf16 or f32 only");
  }
  note_launch();
  return cuda_check(cudaGetLastError(), "maxpool launch");
}

}  // namespace icv
