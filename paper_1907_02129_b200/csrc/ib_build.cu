// K1: indirection-buffer construction on the device.
//
// Restates _compute_offsets (reference indirect.py:98-126) as one thread per
// buffer entry: entry [t, e, m] (tile-major, then kernel element, then lane;
// indirect.py:14-16) serves output pixel p = min(t*mr + m, P - 1) (trailing
// lanes clamp to the last real pixel, :111) and tap e = ky*S + kx; it holds
// the element offset ((n*H + iy)*W + ix)*C of the input pixel row that tap
// reads, or ZERO_REF = -1 when the tap falls in the padding (:120-125).
//
// HBM-bound integer work: consecutive threads write consecutive entries
// (fully coalesced 8- or 4-byte stores); the grid is a multiple of the SM
// count and grid-strides over the entries.
#include "icv_internal.h"

namespace icv {
namespace {

struct IbArgs {
  int32_t R, S, SY, SX, DY, DX, PT, PL;
  int64_t H, W, C, OH, OW, P;
  int64_t mr, rs_mr, first_entry, end_entry;
};

template <typename Idx, typename Out>
__global__ void __launch_bounds__(256) ib_build_kernel(IbArgs a, Out* __restrict__ ib) {
  const Idx stride = (Idx)gridDim.x * blockDim.x;
  const Idx mr = (Idx)a.mr, rs_mr = (Idx)a.rs_mr, S = (Idx)a.S;
  const Idx ohw = (Idx)(a.OH * a.OW), ow = (Idx)a.OW, plast = (Idx)(a.P - 1);
  for (Idx i = (Idx)a.first_entry + (Idx)blockIdx.x * blockDim.x + threadIdx.x; i < (Idx)a.end_entry; i += stride) {
    const Idx t = i / rs_mr;
    const Idx rem = i - t * rs_mr;
    const Idx e = rem / mr;
    const Idx m = rem - e * mr;
    Idx p = t * mr + m;
    p = p < plast ? p : plast;                       // indirect.py:111
    const Idx n = p / ohw;
    const Idx r2 = p - n * ohw;
    const Idx oy = r2 / ow;
    const Idx ox = r2 - oy * ow;
    const Idx ky = e / S;
    const Idx kx = e - ky * S;
    const int64_t iy = (int64_t)oy * a.SY + (int64_t)ky * a.DY - a.PT;   // :120
    const int64_t ix = (int64_t)ox * a.SX + (int64_t)kx * a.DX - a.PL;   // :121
    const bool valid = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;        // :122
    const int64_t off = (((int64_t)n * a.H + iy) * a.W + ix) * a.C;     // :123
    ib[i] = valid ? (Out)off : (Out)-1;                                   // :124-125
  }
}

// Count entries that differ from the canonical buffer (same formula as above).
template <typename Idx, typename In>
__global__ void __launch_bounds__(256) ib_check_kernel(IbArgs a, const In* __restrict__ ib, int32_t* mismatches) {
  const Idx stride = (Idx)gridDim.x * blockDim.x;
  const Idx mr = (Idx)a.mr, rs_mr = (Idx)a.rs_mr, S = (Idx)a.S;
  const Idx ohw = (Idx)(a.OH * a.OW), ow = (Idx)a.OW, plast = (Idx)(a.P - 1);
  int32_t bad = 0;
  for (Idx i = (Idx)a.first_entry + (Idx)blockIdx.x * blockDim.x + threadIdx.x; i < (Idx)a.end_entry; i += stride) {
    const Idx t = i / rs_mr;
    const Idx rem = i - t * rs_mr;
    const Idx e = rem / mr;
    const Idx m = rem - e * mr;
    Idx p = t * mr + m;
    p = p < plast ? p : plast;
    const Idx n = p / ohw;
    const Idx r2 = p - n * ohw;
    const Idx oy = r2 / ow;
    const Idx ox = r2 - oy * ow;
    const Idx ky = e / S;
    const Idx kx = e - ky * S;
    const int64_t iy = (int64_t)oy * a.SY + (int64_t)ky * a.DY - a.PT;
    const int64_t ix = (int64_t)ox * a.SX + (int64_t)kx * a.DX - a.PL;
    const bool valid = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
    const int64_t off = (((int64_t)n * a.H + iy) * a.W + ix) * a.C;
    bad += (int64_t)ib[i] != (valid ? off : (int64_t)-1);
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatches, bad);
}

static IbArgs ib_args(const Geom& g, int64_t batch, int32_t mr) {
  IbArgs a;
  a.R = g.R; a.S = g.S; a.SY = g.SY; a.SX = g.SX; a.DY = g.DY; a.DX = g.DX; a.PT = g.PT; a.PL = g.PL;
  a.H = g.H; a.W = g.W; a.C = g.C; a.OH = g.OH; a.OW = g.OW;
  a.P = batch * g.OH * g.OW;
  a.mr = mr;
  a.rs_mr = (int64_t)g.RS() * mr;
  a.first_entry = 0;
  a.end_entry = ((a.P + mr - 1) / mr) * a.rs_mr;
  return a;
}

}  // namespace

int launch_ib_check(const Geom& g, int64_t batch, int32_t mr, int32_t ib_dtype, const void* ib, int32_t* mismatches,
                    cudaStream_t st) {
  const IbArgs a = ib_args(g, batch, mr);
  if (cudaError_t e = cudaMemsetAsync(mismatches, 0, sizeof(int32_t), st)) return cuda_check(e, "ib_check memset");
  const int64_t n = a.end_entry;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  const int blocks = (int)(want < (int64_t)sms * 8 ? (want > 0 ? want : 1) : (int64_t)sms * 8);
  const bool small = a.end_entry < (int64_t(1) << 31);
  if (ib_dtype == ICV_I64) {
    if (small) ib_check_kernel<uint32_t, int64_t><<<blocks, 256, 0, st>>>(a, static_cast<const int64_t*>(ib), mismatches);
    else ib_check_kernel<uint64_t, int64_t><<<blocks, 256, 0, st>>>(a, static_cast<const int64_t*>(ib), mismatches);
  } else {
    if (small) ib_check_kernel<uint32_t, int32_t><<<blocks, 256, 0, st>>>(a, static_cast<const int32_t*>(ib), mismatches);
    else ib_check_kernel<uint64_t, int32_t><<<blocks, 256, 0, st>>>(a, static_cast<const int32_t*>(ib), mismatches);
  }
  note_launch();
  return cuda_check(cudaGetLastError(), "ib_check launch");
}

int launch_ib_build(const Geom& g, int64_t batch, int32_t mr, int64_t first_tile, int32_t ib_dtype, void* ib,
                    cudaStream_t st) {
  IbArgs a;
  a.R = g.R; a.S = g.S; a.SY = g.SY; a.SX = g.SX; a.DY = g.DY; a.DX = g.DX; a.PT = g.PT; a.PL = g.PL;
  a.H = g.H; a.W = g.W; a.C = g.C; a.OH = g.OH; a.OW = g.OW;
  a.P = batch * g.OH * g.OW;
  a.mr = mr;
  a.rs_mr = (int64_t)g.RS() * mr;
  const int64_t tiles = (a.P + mr - 1) / mr;
  a.first_entry = first_tile * a.rs_mr;
  a.end_entry = tiles * a.rs_mr;
  const int64_t n = a.end_entry - a.first_entry;
  if (n <= 0) return ICV_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  const int blocks = (int)(want < cap ? want : cap);
  const bool small = a.end_entry < (int64_t(1) << 31) && a.P < (int64_t(1) << 31);
  if (ib_dtype == ICV_I64) {
    if (small) ib_build_kernel<uint32_t, int64_t><<<blocks, 256, 0, st>>>(a, static_cast<int64_t*>(ib));
    else ib_build_kernel<uint64_t, int64_t><<<blocks, 256, 0, st>>>(a, static_cast<int64_t*>(ib));
  } else {
    if (small) ib_build_kernel<uint32_t, int32_t><<<blocks, 256, 0, st>>>(a, static_cast<int32_t*>(ib));
    else ib_build_kernel<uint64_t, int32_t><<<blocks, 256, 0, st>>>(a, static_cast<int32_t*>(ib));
  }
  note_launch();
  return cuda_check(cudaGetLastError(), "ib_build launch");
}

}  // namespace icv
