// libicv C ABI (include/icv.h): argument validation, geometry, kernel-family
// selection and dispatch.  No compute happens on the host; every entry that
// touches tensor data launches a device kernel on the caller's stream.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "icv_internal.h"

namespace icv {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ICV_OK;
  return fail(ICV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int kernel_setup(const void* fn, int smem_bytes, int cluster, int threads, int* max_clusters) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, int> done;   // (kernel, device, smem) -> max clusters
  int dev = 0;
  if (int s = cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) return s;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(fn, dev, smem_bytes);
  auto it = done.find(key);
  if (it == done.end()) {
    if (int s = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes),
                           "cudaFuncSetAttribute(max dynamic smem)"))
      return s;
    int mc = 0;
    if (cluster > 1) {
      cudaLaunchConfig_t q = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.gridDim = dim3(cluster * 74);
      q.blockDim = dim3(threads);
      q.dynamicSmemBytes = smem_bytes;
      q.attrs = at;
      q.numAttrs = 1;
      if (int s = cuda_check(cudaOccupancyMaxActiveClusters(&mc, fn, &q), "cudaOccupancyMaxActiveClusters")) return s;
    }
    it = done.emplace(key, mc).first;
  }
  if (max_clusters) *max_clusters = it->second;
  return ICV_OK;
}

// ---- tuning knobs --------------------------------------------------------------
static const char* const kTuneNames[kTuneCount] = {
    "win", "win_min_useful_pm", "win_s2", "win_u8", "win_ws", "win_tma", "win_u8_cls", "win_split",
    "win_debug", "win_cs", "win_mt", "win_res", "win_u8_bn", "cluster", "u8_bn", "tma_store", "rows_rp",
    "dense_a", "dense_cs", "pdl", "dense_pf", "rows_pf", "dense_resb", "epi_wide", "small_tile_bn", "win_filt_lanes", "rows_loaders", "im2col_a"};
static const int kTuneDefaults[kTuneCount] = {-1, 700, 0, 0, 0, 1, 1, 1, 0, 2, 2, 1, 256, 1, 0, 1, 1, 1, 0, 1, 0, 0, 128, 1, 0, 1, 1, 1};
static std::atomic<int> g_tune[kTuneCount];
static std::once_flag g_tune_once;
static void tune_init() {
  std::call_once(g_tune_once, [] {
    for (int i = 0; i < kTuneCount; ++i) g_tune[i].store(kTuneDefaults[i], std::memory_order_relaxed);
  });
}
int tune(TuneKey k) {
  tune_init();
  return g_tune[k].load(std::memory_order_relaxed);
}
static int tune_index(const char* key) {
  if (!key) return -1;
  for (int i = 0; i < kTuneCount; ++i)
    if (std::strcmp(key, kTuneNames[i]) == 0) return i;
  return -1;
}

int make_geom(const icv_conv_desc* d, const icv_shape4* in, Geom* g) {
  if (!d || !in || !g) return fail(ICV_ERR_ARG, "null argument");
  const int32_t pos[] = {d->kernel_h, d->kernel_w, d->stride_h, d->stride_w,
                         d->dilation_h, d->dilation_w, d->in_channels, d->out_channels};
  for (int32_t v : pos)
    if (v < 1) return fail(ICV_ERR_ARG, "kernel/stride/dilation/channels must be >= 1");
  if (d->pad_top < 0 || d->pad_left < 0 || d->pad_bottom < 0 || d->pad_right < 0)
    return fail(ICV_ERR_ARG, "pads must be >= 0");
  if (in->n < 1 || in->h < 1 || in->w < 1 || in->c < 1) return fail(ICV_ERR_ARG, "input extent must be >= 1");
  // tensors.py:191-194
  if (in->c != d->in_channels)
    return fail(ICV_ERR_ARG, "input has " + std::to_string(in->c) + " channels, params expect " +
                                 std::to_string(d->in_channels));
  // tensors.py:195-211
  const int64_t span_h = in->h + d->pad_top + d->pad_bottom - (int64_t)d->dilation_h * (d->kernel_h - 1) - 1;
  const int64_t span_w = in->w + d->pad_left + d->pad_right - (int64_t)d->dilation_w * (d->kernel_w - 1) - 1;
  if (span_h < 0 || span_w < 0) return fail(ICV_ERR_GEOMETRY, "dilated kernel does not fit in padded input");
  g->R = d->kernel_h; g->S = d->kernel_w; g->SY = d->stride_h; g->SX = d->stride_w;
  g->DY = d->dilation_h; g->DX = d->dilation_w; g->PT = d->pad_top; g->PL = d->pad_left;
  g->PB = d->pad_bottom; g->PR = d->pad_right; g->C = d->in_channels; g->K = d->out_channels;
  g->N = in->n; g->H = in->h; g->W = in->w;
  g->OH = span_h / d->stride_h + 1;
  g->OW = span_w / d->stride_w + 1;
  return ICV_OK;
}

int family_for(int32_t dtype, int C, int RS, int K) {
  // tensor-core kernels need 16-byte pixel rows, an indirection slice that
  // fits in shared memory (R*S <= 24) and at most 2048 output channels
  const bool tc_ok = RS <= kMaxRsTc && K <= 2048;
  switch (dtype) {
    case ICV_F32: return kFamF32Exact;
    case ICV_BF16:
      if (C % 8 == 0 && tc_ok) return kFamTcBf16;
      return stem_kernel_eligible(C, RS, K) ? kFamStemBf16 : kFamCoreBf16;
    case ICV_U8: return (C % 16 == 0 && tc_ok) ? kFamTcU8 : kFamCoreU8;
    default: return -1;
  }
}

int tc_block_n(int family, int K) {
  if (family == kFamTcBf16) return K <= 64 ? 64 : (K <= 128 ? 128 : 256);
  if (family == kFamTcU8) return K <= 64 ? 64 : 128;   // + 16 TMEM columns for the row sums
  if (family == kFamStemBf16) return K <= 64 ? 64 : 128;
  return 0;
}

static int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

int packed_layout(const icv_conv_desc* d, int32_t dtype, PackedLayout* L) {
  if (!d || !L) return fail(ICV_ERR_ARG, "null argument");
  if (d->in_channels < 1 || d->out_channels < 1 || d->kernel_h < 1 || d->kernel_w < 1)
    return fail(ICV_ERR_ARG, "bad filter geometry");
  const int fam = family_for(dtype, d->in_channels, d->kernel_h * d->kernel_w, d->out_channels);
  if (fam < 0) return fail(ICV_ERR_ARG, "unsupported compute dtype");
  const int64_t K = d->out_channels, C = d->in_channels, RS = (int64_t)d->kernel_h * d->kernel_w;
  std::memset(L, 0, sizeof(*L));
  L->family = fam;
  if (fam == kFamTcBf16 || fam == kFamTcU8) {
    const int eb = fam == kFamTcBf16 ? 2 : 1;
    L->block_n = tc_block_n(fam, (int)K);
    L->n_pad = (int)align_up(K, L->block_n);
    L->cblocks = (int)((C * eb + 127) / 128);
    L->row_bytes = RS * L->cblocks * 128;
    L->w_off = 0;
    L->w_bytes = (int64_t)L->n_pad * L->row_bytes;
    L->bias_off = align_up(L->w_bytes, 256);
    L->bias_bytes = 4 * (int64_t)L->n_pad;
  } else if (fam == kFamStemBf16) {
    // one row per output channel: k = e*C + c over the whole receptive field,
    // zero padded to whole 128-byte blocks of 16-element MMA steps
    L->block_n = tc_block_n(fam, (int)K);
    L->n_pad = L->block_n;
    const int64_t ksteps = (RS * C + 15) / 16;
    L->cblocks = (int)((ksteps * 16 + 63) / 64);
    L->row_bytes = (int64_t)L->cblocks * 128;
    L->w_off = 0;
    L->w_bytes = (int64_t)L->n_pad * L->row_bytes;
    L->bias_off = align_up(L->w_bytes, 256);
    L->bias_bytes = 4 * (int64_t)L->n_pad;
    // plus, for stride-2 layers, the row-sliding kernel's copy: per kernel row
    // a [n_pad][32] (kx < 8, c < 4) no-swizzle K-major block
    if (rows_filter_eligible(d->kernel_h, d->kernel_w, d->stride_h, d->stride_w, d->dilation_h, d->dilation_w,
                             (int)C, (int)K))
      L->rows_off = align_up(L->bias_off + L->bias_bytes, 1024);
  } else {
    const int eb = fam == kFamF32Exact ? 4 : (fam == kFamCoreBf16 ? 2 : 1);
    L->n_pad = (int)K;
    L->row_bytes = RS * C * eb;
    L->w_off = 0;
    L->w_bytes = K * L->row_bytes;
    L->bias_off = align_up(L->w_bytes, 256);
    L->bias_bytes = 4 * K;
  }
  L->total = align_up(L->bias_off + L->bias_bytes, 256);
  if (fam == kFamTcU8) {   // per-tap padding corrections for zero-filled (TMA) windows
    L->tapcorr_off = L->total;
    L->total = align_up(L->tapcorr_off + RS * L->n_pad * 4, 256);
  }
  if (L->rows_off) L->total = align_up(L->rows_off + (int64_t)d->kernel_h * L->n_pad * 64, 256);
  return ICV_OK;
}

}  // namespace icv

using namespace icv;

extern "C" {

ICV_API int32_t icv_abi_version(void) { return ICV_ABI_VERSION; }

ICV_API const char* icv_last_error(void) { return g_last_error.c_str(); }

ICV_API int64_t icv_launch_count(void) { return g_launches.load(); }

ICV_API int icv_set_tuning(const char* key, int32_t value) {
  const int i = tune_index(key);
  if (i < 0) return fail(ICV_ERR_ARG, std::string("icv_set_tuning: unknown key ") + (key ? key : "(null)"));
  tune_init();
  g_tune[i].store(value < 0 && i != kTuneWin ? kTuneDefaults[i] : value, std::memory_order_relaxed);
  return ICV_OK;
}

ICV_API int icv_get_tuning(const char* key, int32_t* value) {
  const int i = tune_index(key);
  if (i < 0) return fail(ICV_ERR_ARG, std::string("icv_get_tuning: unknown key ") + (key ? key : "(null)"));
  if (value) *value = tune((TuneKey)i);
  return ICV_OK;
}

ICV_API int icv_maxpool2d(const icv_shape4* in, int32_t kh, int32_t kw, int32_t sh, int32_t sw, int32_t ph,
                          int32_t pw, int32_t dtype, const void* x, void* y, void* stream) {
  if (!in || !x || !y) return fail(ICV_ERR_ARG, "icv_maxpool2d: null argument");
  if (in->n < 1 || in->h < 1 || in->w < 1 || in->c < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0 ||
      ph >= kh || pw >= kw)
    return fail(ICV_ERR_ARG, "icv_maxpool2d: invalid geometry");
  if (in->h + 2 * ph < kh || in->w + 2 * pw < kw) return fail(ICV_ERR_GEOMETRY, "icv_maxpool2d: window does not fit");
  return launch_maxpool(*in, kh, kw, sh, sw, ph, pw, dtype, x, y, static_cast<cudaStream_t>(stream));
}

ICV_API int icv_device_info(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int v;
  if (int s = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device), "sm count")) return s;
  if (sm_count) *sm_count = v;
  if (int s = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device), "cc major")) return s;
  if (cc_major) *cc_major = v;
  if (int s = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device), "cc minor")) return s;
  if (cc_minor) *cc_minor = v;
  return ICV_OK;
}

ICV_API int icv_im2col(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t dtype, const void* x,
                       const void* zero_row, void* patches, void* stream) {
  Geom g;
  if (int s = make_geom(desc, in, &g)) return s;
  if (!x || !patches) return fail(ICV_ERR_ARG, "icv_im2col: null tensor");
  if (batch < 1 || batch > in->n) return fail(ICV_ERR_ARG, "batch must be within the physical input batch");
  const int elem = dtype == ICV_F32 ? 4 : dtype == ICV_BF16 ? 2 : dtype == ICV_U8 ? 1 : 0;
  if (elem == 0) return fail(ICV_ERR_ARG, "icv_im2col: unsupported dtype");
  return launch_im2col(g, batch, elem, x, zero_row, patches, static_cast<cudaStream_t>(stream));
}

ICV_API int icv_out_shape(const icv_conv_desc* desc, const icv_shape4* in, icv_shape4* out) {
  Geom g;
  if (int s = make_geom(desc, in, &g)) return s;
  if (!out) return fail(ICV_ERR_ARG, "null out");
  out->n = in->n; out->h = g.OH; out->w = g.OW; out->c = desc->out_channels;
  return ICV_OK;
}

ICV_API int icv_ib_entries(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t mr, int64_t* tiles,
                   int64_t* entries) {
  Geom g;
  if (int s = make_geom(desc, in, &g)) return s;
  if (mr < 1) return fail(ICV_ERR_ARG, "mr must be >= 1");
  if (batch < 1 || batch > in->n) return fail(ICV_ERR_ARG, "batch must be within the physical input batch");
  const int64_t pixels = batch * g.OH * g.OW;
  const int64_t t = (pixels + mr - 1) / mr;
  if (tiles) *tiles = t;
  if (entries) *entries = t * g.RS() * mr;
  return ICV_OK;
}

ICV_API int icv_ib_build(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t mr, int64_t first_tile,
                 int32_t ib_dtype, void* ib, void* stream) {
  Geom g;
  if (int s = make_geom(desc, in, &g)) return s;
  if (mr < 1) return fail(ICV_ERR_ARG, "mr must be >= 1");
  if (batch < 1 || batch > in->n) return fail(ICV_ERR_ARG, "batch must be within the physical input batch");
  const bool per_image = (ib_dtype & ICV_IB_PER_IMAGE) != 0;
  ib_dtype &= ~ICV_IB_PER_IMAGE;
  if (ib_dtype != ICV_I64 && ib_dtype != ICV_I32) return fail(ICV_ERR_ARG, "ib dtype must be int64 or int32");
  if (!ib) return fail(ICV_ERR_ARG, "null ib");
  if (per_image) batch = 1;   // image 0's buffer serves every image
  const int64_t pixels = batch * g.OH * g.OW;
  const int64_t tiles = (pixels + mr - 1) / mr;
  if (first_tile < 0 || first_tile > tiles) return fail(ICV_ERR_ARG, "first_tile out of range");
  if (ib_dtype == ICV_I32 && g.N * g.H * g.W * g.C >= (int64_t(1) << 31))
    return fail(ICV_ERR_ARG, "input too large for int32 offsets");
  return launch_ib_build(g, batch, mr, first_tile, ib_dtype, ib, (cudaStream_t)stream);
}

ICV_API int icv_ib_check(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t mr, int32_t ib_dtype,
                         const void* ib, int32_t* mismatches, void* stream) {
  Geom g;
  if (int s = make_geom(desc, in, &g)) return s;
  if (mr < 1) return fail(ICV_ERR_ARG, "mr must be >= 1");
  if (batch < 1 || batch > in->n) return fail(ICV_ERR_ARG, "batch must be within the physical input batch");
  const bool per_image = (ib_dtype & ICV_IB_PER_IMAGE) != 0;
  ib_dtype &= ~(ICV_IB_PER_IMAGE | ICV_IB_CANONICAL);
  if (ib_dtype != ICV_I64 && ib_dtype != ICV_I32) return fail(ICV_ERR_ARG, "ib dtype must be int64 or int32");
  if (!ib || !mismatches) return fail(ICV_ERR_ARG, "icv_ib_check: null pointer");
  return launch_ib_check(g, per_image ? 1 : batch, mr, ib_dtype, ib, mismatches, (cudaStream_t)stream);
}

ICV_API int icv_packed_filter_bytes(const icv_conv_desc* desc, int32_t compute_dtype, int64_t* bytes) {
  PackedLayout L;
  if (int s = packed_layout(desc, compute_dtype, &L)) return s;
  if (bytes) *bytes = L.total;
  return ICV_OK;
}

ICV_API int icv_requant_params(float input_scale, float kernel_scale, float output_scale, int32_t* multiplier,
                       int32_t* shift) {
  const double real = ((double)input_scale * (double)kernel_scale) / (double)output_scale;
  if (!(real > 0.0 && real < 1.0)) return fail(ICV_ERR_ARG, "requantization scale must be in (0, 1)");
  int e = 0;
  const double q = std::frexp(real, &e);  // real = q * 2^e, q in [0.5, 1)
  int64_t m0 = (int64_t)std::floor(q * 2147483648.0 + 0.5);
  if (m0 == (int64_t(1) << 31)) {
    m0 = int64_t(1) << 30;
    e += 1;
  }
  const int sh = -e;
  if (sh < 0 || sh > 31) return fail(ICV_ERR_ARG, "requantization shift out of [0, 31]");
  if (multiplier) *multiplier = (int32_t)m0;
  if (shift) *shift = sh;
  return ICV_OK;
}

ICV_API int icv_pack_filter(const icv_conv_desc* desc, int32_t compute_dtype, int32_t w_dtype, const void* w_krsc,
                    const void* bias, const icv_quant* quant, void* packed, void* stream) {
  PackedLayout L;
  if (int s = packed_layout(desc, compute_dtype, &L)) return s;
  if (!w_krsc || !packed) return fail(ICV_ERR_ARG, "null weights or output");
  if (compute_dtype == ICV_U8) {
    if (w_dtype != ICV_U8) return fail(ICV_ERR_ARG, "uint8 convolution needs uint8 weights");
    if (!quant) return fail(ICV_ERR_ARG, "uint8 convolution needs quantization parameters");
    const int64_t kk = (int64_t)desc->kernel_h * desc->kernel_w * desc->in_channels;
    if (kk * 255 * 255 * 4 >= (int64_t(1) << 31))
      return fail(ICV_ERR_UNSUPPORTED, "R*S*C too large for exact int32 accumulation");
  } else if (w_dtype != ICV_F32 && w_dtype != ICV_BF16) {
    return fail(ICV_ERR_ARG, "float convolution needs float32 or bfloat16 weights");
  }
  if (compute_dtype == ICV_F32 && w_dtype != ICV_F32)
    return fail(ICV_ERR_ARG, "float32 convolution needs float32 weights");
  Geom g{};
  g.R = desc->kernel_h; g.S = desc->kernel_w; g.C = desc->in_channels; g.K = desc->out_channels;
  return launch_pack(g, L, w_dtype, w_krsc, bias, quant, packed, (cudaStream_t)stream);
}

static const char* kernel_name_for(const ConvArgs& a) {
  switch (a.L.family) {
    case kFamF32Exact: return "icv_conv_f32_exact";
    case kFamCoreBf16: return "icv_conv_core<bf16>";
    case kFamCoreU8: return "icv_conv_core<u8>";
    case kFamTcBf16:
    case kFamTcU8: return tc_kernel_name(a);
    case kFamStemBf16:
      return (!a.prefer_gather && a.ib_canonical && a.L.rows_off && rows_kernel_eligible(a.g))
                 ? "icv_igemm_rows<bf16>" : "icv_igemm_stem<bf16>";
  }
  return "?";
}

ICV_API int icv_conv_kernel_name(const icv_conv_desc* desc, const icv_shape4* in, int32_t dtype, int32_t flags,
                                 const char** name) {
  ConvArgs a{};
  if (int s = make_geom(desc, in, &a.g)) return s;
  if (int s = packed_layout(desc, dtype, &a.L)) return s;
  a.P = in->n * a.g.OH * a.g.OW;
  a.ib_per_image = (flags & ICV_IB_PER_IMAGE) != 0;
  a.ib_canonical = (flags & ICV_IB_CANONICAL) != 0;
  a.zero_known = (flags & ICV_ZERO_ROW_ZEROS) != 0;
  a.zero_is_zp = (flags & ICV_ZERO_ROW_ZP) != 0;
  a.prefer_gather = (flags & ICV_PREFER_GATHER) != 0;
  a.x = reinterpret_cast<const void*>(uintptr_t(256));   // (16-byte aligned tensors assumed)
  a.y = reinterpret_cast<void*>(uintptr_t(256));
  a.zero_row = a.x;
  if (name) *name = kernel_name_for(a);
  return ICV_OK;
}

ICV_API int icv_conv(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t dtype, const void* x,
             const void* zero_row, const void* ib, int32_t ib_dtype, int32_t mr, const void* packed,
             const icv_quant* quant, void* y, void* stream) {
  ConvArgs a{};
  if (int s = make_geom(desc, in, &a.g)) return s;
  if (batch < 1 || batch > in->n) return fail(ICV_ERR_ARG, "batch must be within the physical input batch");
  if (mr < 1) return fail(ICV_ERR_ARG, "mr must be >= 1");
  a.ib_per_image = (ib_dtype & ICV_IB_PER_IMAGE) != 0;
  a.ib_canonical = (ib_dtype & ICV_IB_CANONICAL) != 0;
  a.zero_known = (ib_dtype & ICV_ZERO_ROW_ZEROS) != 0;
  a.zero_is_zp = (ib_dtype & ICV_ZERO_ROW_ZP) != 0;
  a.prefer_gather = (ib_dtype & ICV_PREFER_GATHER) != 0;
  ib_dtype &= ~(ICV_IB_PER_IMAGE | ICV_IB_CANONICAL | ICV_ZERO_ROW_ZEROS | ICV_ZERO_ROW_ZP | ICV_PREFER_GATHER);
  if (ib_dtype != ICV_I64 && ib_dtype != ICV_I32) return fail(ICV_ERR_ARG, "ib dtype must be int64 or int32");
  if (!x || !zero_row || !ib || !packed || !y) return fail(ICV_ERR_ARG, "null tensor pointer");
  if (int s = packed_layout(desc, dtype, &a.L)) return s;
  a.P = batch * a.g.OH * a.g.OW;
  a.mr = mr;
  a.x = x;
  a.zero_row = zero_row;
  a.ib = ib;
  a.ib_is_i32 = ib_dtype == ICV_I32;
  a.packed = static_cast<const uint8_t*>(packed);
  a.y = y;
  if (a.L.family == kFamTcBf16 || a.L.family == kFamTcU8 || a.L.family == kFamStemBf16) {
    // the tensor-core kernels move 16-byte vectors of x, the zero row and y
    const uintptr_t mis = (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(zero_row) |
                           reinterpret_cast<uintptr_t>(y)) & 15;
    if (mis) return fail(ICV_ERR_UNSUPPORTED, "tensor-core convolution needs 16-byte aligned input, zero row and output");
  }
  if (dtype == ICV_U8) {
    if (!quant) return fail(ICV_ERR_ARG, "uint8 convolution needs quantization parameters");
    if (quant->output_min < 0 || quant->output_max > 255 || quant->output_min > quant->output_max)
      return fail(ICV_ERR_ARG, "output clamp range must lie in [0, 255]");
    if (quant->input_zero_point < 0 || quant->input_zero_point > 255 || quant->kernel_zero_point < 0 ||
        quant->kernel_zero_point > 255)
      return fail(ICV_ERR_ARG, "zero points must lie in [0, 255]");
    if (int s = icv_requant_params(quant->input_scale, quant->kernel_scale, quant->output_scale, &a.m0, &a.shift))
      return s;
    a.zx = quant->input_zero_point;
    a.zw = quant->kernel_zero_point;
    a.zo = quant->output_zero_point;
    a.qmin = quant->output_min;
    a.qmax = quant->output_max;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (a.L.family) {
    case kFamF32Exact: return launch_conv_f32_exact(a, st);
    case kFamCoreBf16:
    case kFamCoreU8: return launch_conv_core(a, st);
    case kFamTcBf16:
    case kFamTcU8: return launch_conv_tc(a, st);
    case kFamStemBf16: return launch_conv_stem(a, st);
  }
  return fail(ICV_ERR_UNSUPPORTED, "no kernel family");
}

}  // extern "C"
