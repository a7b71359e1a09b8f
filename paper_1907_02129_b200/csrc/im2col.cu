// im2row patch matrix on the device: the GEMM-based baseline the paper
// compares the indirect algorithm against (reference im2col.py:48-114).
//
// Row p (output pixel, n / oy / ox row-major) holds at column e*C + c
// (e = ky*S + kx) the input element at iy = oy*SY + ky*DY - PT,
// ix = ox*SX + kx*DX - PL, or the padding value when the tap is out of
// bounds: zeros (the reference's 0.0) or, when given, the zero row (uint8:
// the input zero point).  HBM-bound by construction -- the matrix is R*S
// times the input -- which is the cost the indirection buffer avoids.
// 16-byte pieces (or elements for rows that are not 16-byte multiples).
#include "icv_internal.h"

namespace icv {
namespace {

struct I2CGeom {
  int32_t H, W, C, S, SY, SX, DY, DX, PT, PL, OH, OW, RS;
};

// One warp per output pixel (index math once per pixel); its R*S*C row is
// contiguous in the patch matrix, so lane j of each step writes piece j of
// a 32-piece run: every store instruction covers 512 contiguous bytes.
template <typename V>
__global__ void __launch_bounds__(256) im2col_kernel(const V* __restrict__ x, const V* __restrict__ zero,
                                                     V* __restrict__ out, I2CGeom g, int32_t vpr, int64_t pixels) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int32_t row_vecs = g.RS * vpr;
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < pixels; p += nwarps) {
    const int64_t img_row = p / g.OW;
    const int32_t ox = (int32_t)(p - img_row * g.OW);
    const int64_t n = img_row / g.OH;
    const int32_t oy = (int32_t)(img_row - n * g.OH);
    const V* xn = x + (int64_t)n * g.H * g.W * vpr;
    V* dst = out + p * row_vecs;
    int32_t e = lane / vpr, q = lane - (lane / vpr) * vpr;   // piece `lane` of the row
#pragma unroll 4
    for (int32_t j = lane; j < row_vecs; j += 32) {
      const int32_t ky = e / g.S, kx = e - ky * g.S;
      const int32_t iy = oy * g.SY + ky * g.DY - g.PT, ix = ox * g.SX + kx * g.DX - g.PL;
      V v;
      if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) v = __ldg(xn + ((int64_t)iy * g.W + ix) * vpr + q);
      else if (zero != nullptr) v = __ldg(zero + q);
      else v = V{};
      dst[j] = v;
      q += 32;
      while (q >= vpr) { q -= vpr; ++e; }
    }
  }
}

template <typename V>
int launch_i2c(const Geom& gm, int64_t batch, int elem, const void* x, const void* zero, void* out, cudaStream_t st) {
  I2CGeom g{(int32_t)gm.H, (int32_t)gm.W, gm.C, gm.S, gm.SY, gm.SX, gm.DY, gm.DX, gm.PT, gm.PL,
            (int32_t)gm.OH, (int32_t)gm.OW, gm.RS()};
  const int32_t vpr = (int32_t)((int64_t)gm.C * elem / (int64_t)sizeof(V));
  const int64_t pixels = batch * gm.OH * gm.OW;
  if (pixels == 0) return ICV_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (pixels + 7) / 8;   // 8 warps (pixels) per block
  const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
  im2col_kernel<V><<<grid, 256, 0, st>>>(static_cast<const V*>(x), static_cast<const V*>(zero), static_cast<V*>(out),
                                         g, vpr, pixels);
  note_launch();
  return cuda_check(cudaGetLastError(), "im2col launch");
}

}  // namespace

int launch_im2col(const Geom& g, int64_t batch, int elem, const void* x, const void* zero, void* out,
                  cudaStream_t st) {
  const int64_t row_bytes = (int64_t)g.C * elem;
  const bool a16 = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (reinterpret_cast<uintptr_t>(zero) & 15) == 0;
  if (a16) return launch_i2c<uint4>(g, batch, elem, x, zero, out, st);
  if (elem == 4) return launch_i2c<uint32_t>(g, batch, elem, x, zero, out, st);
  if (elem == 2) return launch_i2c<uint16_t>(g, batch, elem, x, zero, out, st);
  return launch_i2c<uint8_t>(g, batch, elem, x, zero, out, st);
}

}  // namespace icv
