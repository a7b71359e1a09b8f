// CUDA-core indirect-GEMM kernels (K5 and the channel-poor variant).
//
//   kExactF32  bit-exact restatement of the reference's float32 indirect
//              convolution (indirect.py:272-300 under the arithmetic
//              contract of gemm.py:6-15): each output starts from its bias,
//              then for e = 0..RS-1 and c = 0..C-1 (ascending) does
//              acc = fl(acc + fl(x * w)) with __fmul_rn/__fadd_rn, which the
//              compiler never contracts into an FMA.  Padding taps read the
//              bound zero row, exactly as the reference does (:291).
//   kBf16      bf16 inputs, fp32 accumulation, bf16 output: the
//              "warp-level CUDA-core variant" for layers whose pixel rows are
//              not 16-byte aligned (C % 8 != 0, e.g. the 3-channel stem).
//   kU8        uint8 inputs, exact int32 accumulation of (x - zx)(w - zw),
//              fixed-point requantization epilogue (C % 16 != 0 fallback).
//
// Tiling: a CTA owns 64 output pixels x 64 output channels; per tap it reads
// the 64 row references of its pixels from the indirection buffer (the
// paper's Listing 3: per kernel element, load fresh row pointers, then
// C-long dot products into the same accumulators), stages 16-channel slices
// of those rows and of the filter in shared memory and each of the 256
// threads accumulates a 4 x 4 block of outputs.
#include <cuda_bf16.h>

#include "icv_internal.h"
#include "requant.cuh"

namespace icv {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

enum Mode { kExactF32 = 0, kBf16 = 1, kU8 = 2 };

template <int M>
struct Traits;
template <>
struct Traits<kExactF32> {
  using In = float;
  using Acc = float;
  using Out = float;
};
template <>
struct Traits<kBf16> {
  using In = __nv_bfloat16;
  using Acc = float;
  using Out = __nv_bfloat16;
};
template <>
struct Traits<kU8> {
  using In = uint8_t;
  using Acc = int32_t;
  using Out = uint8_t;
};

struct CoreArgs {
  const void* x;
  const void* zero_row;
  const void* ib;
  int ib_is_i32;
  int ib_per_image;
  int64_t mr, P, ohw, img_elems;
  int RS, C, K;
  const void* w;       // KRSC, compute dtype
  const void* bias;    // f32 (float modes) / int32 (u8)
  void* y;
  int32_t zx, zw, zo, qmin, qmax, m0, shift;
};

template <int M>
__device__ __forceinline__ typename Traits<M>::Acc load_in(const typename Traits<M>::In* p, int32_t z) {
  if constexpr (M == kExactF32) return *p;
  else if constexpr (M == kBf16) return __bfloat162float(*p);
  else return (int32_t)(*p) - z;
}

template <int M>
__device__ __forceinline__ typename Traits<M>::Acc madd(typename Traits<M>::Acc acc, typename Traits<M>::Acc a,
                                                        typename Traits<M>::Acc b) {
  if constexpr (M == kExactF32) return __fadd_rn(acc, __fmul_rn(a, b));   // gemm.py:6-15, no FMA
  else if constexpr (M == kBf16) return fmaf(a, b, acc);
  else return acc + a * b;
}

template <int M>
__global__ void __launch_bounds__(NT) conv_core_kernel(CoreArgs a) {
  using In = typename Traits<M>::In;
  using Acc = typename Traits<M>::Acc;
  using Out = typename Traits<M>::Out;
  __shared__ Acc As[BK][BM];
  __shared__ Acc Ws[BK][BN];
  __shared__ const In* rows[BM];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const In* x = static_cast<const In*>(a.x);
  const In* zero = static_cast<const In*>(a.zero_row);
  const In* w = static_cast<const In*>(a.w);

  Acc acc[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + tx * 4 + j;
    Acc b0;
    if constexpr (M == kU8) b0 = n < a.K ? static_cast<const int32_t*>(a.bias)[n] : 0;
    else b0 = n < a.K ? static_cast<const float*>(a.bias)[n] : 0.f;   // bias is the accumulator init
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][j] = b0;
  }

  for (int e = 0; e < a.RS; ++e) {
    __syncthreads();
    if (tid < BM) {
      int64_t p = m0 + tid;
      p = p < a.P ? p : a.P - 1;                        // clamped lane (indirect.py:111)
      int64_t base = 0;
      if (a.ib_per_image) {                             // image-relative buffer of image 0
        const int64_t n = p / a.ohw;
        p -= n * a.ohw;
        base = n * a.img_elems;
      }
      const int64_t ent = ((p / a.mr) * a.RS + e) * a.mr + p % a.mr;
      int64_t off = a.ib_is_i32 ? (int64_t) static_cast<const int32_t*>(a.ib)[ent]
                                : static_cast<const int64_t*>(a.ib)[ent];
      if (off >= 0) off += base;
      rows[tid] = off < 0 ? zero : x + off;             // ZERO_REF -> zero row (indirect.py:291)
    }
    for (int c0 = 0; c0 < a.C; c0 += BK) {
      const int cn = a.C - c0 < BK ? a.C - c0 : BK;
      __syncthreads();
      for (int i = tid; i < BK * BM; i += NT) {
        const int r = i % BM, c = i / BM;
        As[c][r] = c < cn ? load_in<M>(rows[r] + c0 + c, a.zx) : (Acc)0;
      }
      for (int i = tid; i < BK * BN; i += NT) {
        const int c = i % BK, n = i / BK;
        const int ng = n0 + n;
        Ws[c][n] = (c < cn && ng < a.K) ? load_in<M>(w + ((int64_t)ng * a.RS + e) * a.C + c0 + c, a.zw) : (Acc)0;
      }
      __syncthreads();
      for (int c = 0; c < cn; ++c) {                    // exactly C products per tap, ascending
        Acc av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[c][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Ws[c][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = madd<M>(acc[i][j], av[i], bv[j]);
      }
    }
  }

  Out* y = static_cast<Out*>(a.y);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t p = m0 + ty * 4 + i;
    if (p >= a.P) continue;                              // tail lanes dropped (indirect.py:299)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= a.K) continue;
      if constexpr (M == kExactF32) y[p * a.K + n] = acc[i][j];
      else if constexpr (M == kBf16) y[p * a.K + n] = __float2bfloat16_rn(acc[i][j]);
      else y[p * a.K + n] = requant_u8(acc[i][j], a.m0, a.shift, a.zo, a.qmin, a.qmax);
    }
  }
}

template <int M>
int launch_mode(const ConvArgs& c, cudaStream_t st) {
  CoreArgs a;
  a.x = c.x;
  a.zero_row = c.zero_row;
  a.ib = c.ib;
  a.ib_is_i32 = c.ib_is_i32;
  a.ib_per_image = c.ib_per_image;
  a.ohw = c.g.OH * c.g.OW;
  a.img_elems = c.g.H * c.g.W * (int64_t)c.g.C;
  a.mr = c.mr;
  a.P = c.P;
  a.RS = c.g.RS();
  a.C = c.g.C;
  a.K = c.g.K;
  a.w = c.packed + c.L.w_off;
  a.bias = c.packed + c.L.bias_off;
  a.y = c.y;
  a.zx = c.zx; a.zw = c.zw; a.zo = c.zo; a.qmin = c.qmin; a.qmax = c.qmax; a.m0 = c.m0; a.shift = c.shift;
  const int64_t mt = (c.P + BM - 1) / BM;
  if (mt > 0x7fffffff) return fail(ICV_ERR_UNSUPPORTED, "too many pixel tiles");
  dim3 grid((unsigned)mt, (unsigned)((c.g.K + BN - 1) / BN));
  if (grid.y > 65535) return fail(ICV_ERR_UNSUPPORTED, "too many output channels");
  conv_core_kernel<M><<<grid, NT, 0, st>>>(a);
  note_launch();
  return cuda_check(cudaGetLastError(), "conv_core launch");
}

}  // namespace

int launch_conv_f32_exact(const ConvArgs& a, cudaStream_t st) { return launch_mode<kExactF32>(a, st); }

int launch_conv_core(const ConvArgs& a, cudaStream_t st) {
  if (a.L.family == kFamCoreBf16) return launch_mode<kBf16>(a, st);
  if (a.L.family == kFamCoreU8) return launch_mode<kU8>(a, st);
  return fail(ICV_ERR_UNSUPPORTED, "not a CUDA-core family");
}

}  // namespace icv
