// Internal declarations shared by the libicv translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/icv.h"

namespace icv {

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
void note_launch(int n = 1);
struct Geom;
int launch_im2col(const Geom& g, int64_t batch, int elem, const void* x, const void* zero, void* out,
                  cudaStream_t st);
int launch_maxpool(const icv_shape4& in, int kh, int kw, int sh, int sw, int ph, int pw, int dtype, const void* x,
                   void* y, cudaStream_t st);

// ---- geometry --------------------------------------------------------------
struct Geom {
  int R, S, SY, SX, DY, DX, PT, PL, PB, PR, C, K;
  int64_t N, H, W;   // bound input extent
  int64_t OH, OW;    // output extent
  int RS() const { return R * S; }
};
// Validates desc/in and fills g (ICV_ERR_ARG / ICV_ERR_GEOMETRY on failure).
int make_geom(const icv_conv_desc* d, const icv_shape4* in, Geom* g);

// ---- kernel families ---------------------------------------------------------
enum Family { kFamF32Exact = 0, kFamTcBf16 = 1, kFamTcU8 = 2, kFamCoreBf16 = 3, kFamCoreU8 = 4, kFamStemBf16 = 5 };
bool stem_kernel_eligible(int C, int RS, int K);
constexpr int kMaxRsTc = 24;   // taps per pixel handled by the tensor-core kernels
int family_for(int32_t dtype, int C, int RS, int K);
// Output-channel tile width of the tensor-core kernels for this problem.
int tc_block_n(int family, int K);
// Packed-filter layout (byte offsets inside the icv_pack_filter buffer).
struct PackedLayout {
  int family;
  int block_n;        // tensor-core families
  int n_pad;          // packed rows (output channels, zero padded)
  int cblocks;        // 128-byte channel blocks per tap (tensor-core families)
  int64_t row_bytes;  // bytes per packed output channel row
  int64_t w_off, w_bytes, bias_off, bias_bytes, total;
  int64_t rows_off;   // channel-poor family: row-sliding filter copy (0 = absent)
  int64_t tapcorr_off; // uint8 tensor-core family: [RS][n_pad] int32 zx * sum_c (w - zw) per tap (0 = absent)
};
int packed_layout(const icv_conv_desc* d, int32_t dtype, PackedLayout* L);

// ---- kernels (launchers) ---------------------------------------------------
int launch_ib_build(const Geom& g, int64_t batch, int32_t mr, int64_t first_tile, int32_t ib_dtype, void* ib,
                    cudaStream_t st);
int launch_ib_check(const Geom& g, int64_t batch, int32_t mr, int32_t ib_dtype, const void* ib, int32_t* mismatches,
                    cudaStream_t st);
int launch_pack(const Geom& g, const PackedLayout& L, int32_t w_dtype, const void* w, const void* bias,
                const icv_quant* q, void* packed, cudaStream_t st);

struct ConvArgs {
  Geom g;
  int64_t P;  // output pixels = batch * OH * OW
  int32_t mr;
  const void* x;
  const void* zero_row;
  const void* ib;
  int32_t ib_is_i32;
  int32_t ib_per_image;  // entries are image-relative (ICV_IB_PER_IMAGE)
  int32_t ib_canonical;  // caller guarantees the icv_ib_build layout (ICV_IB_CANONICAL)
  int32_t zero_known;    // caller guarantees the zero row is all zero bytes (ICV_ZERO_ROW_ZEROS)
  int32_t zero_is_zp;    // uint8: caller guarantees every zero-row byte is the input zero point (ICV_ZERO_ROW_ZP)
  const uint8_t* packed;
  PackedLayout L;
  void* y;
  // uint8 requantization
  int32_t zx, zw, zo, qmin, qmax, m0, shift;
};
int launch_conv_f32_exact(const ConvArgs& a, cudaStream_t st);
int launch_conv_core(const ConvArgs& a, cudaStream_t st);       // bf16 / u8, any C (CUDA cores)
int launch_conv_tc(const ConvArgs& a, cudaStream_t st);         // bf16 / u8 tcgen05
bool win_kernel_eligible(const ConvArgs& a);                   // stride-1 window kernel applies
int launch_conv_win(const ConvArgs& a, cudaStream_t st);        // bf16 / u8 tcgen05, sliding window A
const char* tc_kernel_name(const ConvArgs& a);
int launch_conv_stem(const ConvArgs& a, cudaStream_t st);   // channel-poor bf16 (tcgen05)
bool rows_kernel_eligible(const Geom& g);
bool rows_filter_eligible(int R, int S, int SY, int SX, int DY, int DX, int C, int K);
int launch_conv_rows(const ConvArgs& a, cudaStream_t st);   // channel-poor, stride 2, row-sliding A

}  // namespace icv
