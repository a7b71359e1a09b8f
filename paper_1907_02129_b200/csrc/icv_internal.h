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

// ---- tuning knobs (icv_set_tuning) -------------------------------------------
// Plan choices exposed for A/B measurement and tests.  The defaults are the
// measured-best plans; nothing reads the environment.  Values
// are process-wide atomics, read once per icv_conv call.
enum TuneKey {
  kTuneWin = 0,          // window kernel: -1 auto, 0 never (IB-gather kernel), 1 whenever it fits
  kTuneWinMinUsefulPm,   // auto mode: minimum fraction (per mille) of computed rows that are real pixels
  kTuneWinS2,            // 1: stride-2 phase-plane window kernel (measured slower; opt-in)
  kTuneWinU8,            // 1: uint8 window kernel (measured slower; opt-in)
  kTuneWinWs,            // window stages (0 = plan default)
  kTuneWinTma,           // 1: TMA windows when the zero row allows, 0: cp.async windows
  kTuneWinU8Cls,         // 1: uint8 padding corrections per border class, 0: per tap
  kTuneWinSplit,         // TMA issuers per window
  kTuneWinDebug,         // 1: print the window plan to stderr
  kTuneWinCs,            // 2: CTA pairs allowed, 1: single CTAs only
  kTuneWinMt,            // 2: two-tile units allowed, 1: one tile per unit
  kTuneWinRes,           // 1: resident-filter plans allowed
  kTuneWinU8Bn,          // uint8 window tile width when K = 256 (256 or 128)
  kTuneCluster,          // gather kernel: 2 = CTA pairs (measured slower; opt-in), 1 = single CTAs
  kTuneU8Bn,             // gather kernel uint8 tile width: 256 (opt-in) or 0 = default 128
  kTuneTmaStore,         // 1: TMA tile stores in the epilogue, 0: thread stores
  kTuneRowsRp,           // row kernel: output rows per tile (1, or 2 = opt-in)
  kTuneDenseA,           // 1: 1x1 stride-1 layers load A as dense TMA boxes, 0: IB gathers
  kTuneDenseCs,          // dense A on CTA pairs (M = 256): 0 = auto (long K loops), 1 = never, 2 = always
  kTunePdl,              // 1: persistent conv kernels use programmatic dependent launch
  kTuneDensePf,          // dense A: L2 bulk prefetch of the A rows this many tiles ahead (0 = off)
  kTuneRowsPf,           // row kernel: L2 bulk prefetch of the input rows this many tiles ahead (0 = off)
  kTuneDenseResB,        // dense A: keep the filter blocks resident when they fit in this many KB (0 = off)
  kTuneEpiWide,          // bf16 epilogue: 64-column chunks with 4 KB TMA stores (1) or 32-column chunks (0)
  kTuneSmallTileBn,      // bf16 gather/dense: BLOCK_N 128 instead of 256 when tiles < this % of the SM count (0 = never)
  kTuneWinFiltLanes,     // window kernel: filter-block issuing lanes per filter producer warp
  kTuneRowsLoaders,      // row kernel: lanes issuing the raw-row bulk copies
  kTuneIm2colA,          // im2col TMA A tiles: 0 off, 1 auto (long K loops; over the window kernel on small images), 2 wherever eligible
  kTuneCount
};
int tune(TuneKey k);

// One-time per (kernel, device) setup before a launch: opt in to
// `smem_bytes` of dynamic shared memory and, for cluster launches
// (cluster > 1), query how many clusters of `threads`-thread CTAs can be
// co-resident (written to *max_clusters; 0 otherwise).  Function attributes
// are per device, so a process driving several GPUs sets them on each.
int kernel_setup(const void* fn, int smem_bytes, int cluster, int threads, int* max_clusters);

// Launch a persistent conv kernel: thread-block clusters of `cluster` CTAs
// (1 = none) and, unless knob pdl = 0, programmatic dependent launch -- the
// kernel may start while the previous kernel in the stream drains (its
// setup overlaps that kernel's tail; it calls griddep_wait() before touching
// any tensor a previous kernel may write).
template <typename... KArgs, typename... Args>
int launch_conv_kernel(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       int cluster, const char* what, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  int n = 0;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (tune(kTunePdl)) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = n;
  if (cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...); e != cudaSuccess) return cuda_check(e, what);
  note_launch();
  return cuda_check(cudaGetLastError(), what);
}

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
  int32_t prefer_gather; // caller asks for the IB-gather kernels (ICV_PREFER_GATHER)
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
bool dense_a_eligible(const ConvArgs& a);                      // 1x1 stride-1: A is the dense input matrix
bool im2col_a_eligible(const ConvArgs& a);                     // canonical buffer, zero zero row: A tiles by im2col TMA
int tma_a_mode(const ConvArgs& a);                             // 0 IB gather, 1 dense TMA boxes, 2 im2col TMA
int launch_conv_win(const ConvArgs& a, cudaStream_t st);        // bf16 / u8 tcgen05, sliding window A
const char* tc_kernel_name(const ConvArgs& a);
int launch_conv_stem(const ConvArgs& a, cudaStream_t st);   // channel-poor bf16 (tcgen05)
bool rows_kernel_eligible(const Geom& g);
bool rows_filter_eligible(int R, int S, int SY, int SX, int DY, int DX, int C, int K);
int launch_conv_rows(const ConvArgs& a, cudaStream_t st);   // channel-poor, stride 2, row-sliding A

}  // namespace icv
