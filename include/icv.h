/*
 * icv.h — C ABI of libicv.so, the B200 (sm_100a) indirect-convolution engine.
 *
 * The reference (arXiv 1907.02129 "convbench", /root/reference/pkg) has no
 * FFI: its hot path is the in-process Python API re-exported by
 * convbench/__init__.py:31-49.  This header is the native boundary that a
 * binding of that API calls instead; every entry point names the reference
 * function it replaces.  Plain pointers and sizes only: no torch types.
 *
 * Conventions
 *   - Tensor pointers are DEVICE pointers (caller-allocated).  The library
 *     allocates no persistent device memory.
 *   - Every launch is stream-ordered on `stream` (a cudaStream_t; NULL = the
 *     legacy default stream).  No call synchronizes the device.
 *   - Return value: ICV_OK (0) or a negative icv_status.  icv_last_error()
 *     returns a thread-local message describing the last failure.
 *   - Reentrant; the per-process kernel-attribute cache is set up once under
 *     a mutex.
 */
#ifndef ICV_H_
#define ICV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICV_ABI_VERSION 2

#if defined(__GNUC__)
#define ICV_API __attribute__((visibility("default")))
#else
#define ICV_API
#endif

typedef enum icv_status {
  ICV_OK = 0,
  ICV_ERR_ARG = -1,          /* maps to ValueError / TypeError            */
  ICV_ERR_GEOMETRY = -2,     /* maps to InvalidGeometryError (ValueError) */
  ICV_ERR_STALE = -3,        /* maps to StaleBufferError (RuntimeError)   */
  ICV_ERR_UNSUPPORTED = -4,  /* no kernel for this dtype/geometry         */
  ICV_ERR_CUDA = -5          /* a CUDA runtime call failed                */
} icv_status;

typedef enum icv_dtype {
  ICV_F32 = 0,
  ICV_BF16 = 1,
  ICV_U8 = 2,
  ICV_I32 = 3,
  ICV_I64 = 4
} icv_dtype;

/* Indirection-buffer layout flag, OR-ed into the `ib_dtype` arguments.
 * Canonical (flag clear): the reference's (T, R*S, mr) buffer over all
 * `batch` images, T = ceil(batch*Ho*Wo / mr).  Per-image (flag set): the
 * buffer of image 0 only, T = ceil(Ho*Wo / mr); entry (n, q, e) of the
 * canonical buffer equals entry (0, q, e) + n*H*W*C (ZERO_REF kept), so one
 * small, L2-resident buffer serves any batch (SPEC.md:325 leaves the row
 * reference representation to the implementation). */
#define ICV_IB_PER_IMAGE 0x100

/* Flag OR-ed into icv_conv's `ib_dtype`: the buffer is exactly what
 * icv_ib_build produced for this geometry (icv_ib_check can verify it).  It
 * lets channel-poor stride-2 layers consume the buffer at input-row
 * granularity (row-sliding kernel); without it they gather tap by tap. */
#define ICV_IB_CANONICAL 0x200

/* Flag OR-ed into icv_conv's `ib_dtype`: the bound zero row is all zero
 * bytes (and, per the reference's contract, read-only: indirect.py:42).
 * Stride-1 layers may then realize padding as out-of-bounds zero fill of
 * their TMA windows instead of reading the zero row. */
#define ICV_ZERO_ROW_ZEROS 0x400

/* Flag OR-ed into icv_conv's `ib_dtype` (uint8): every byte of the bound
 * zero row equals quant->input_zero_point (as the reference semantics
 * prescribe for quantized padding).  Windowed layers may then zero-fill
 * padding and add the packed per-tap correction zx * sum_c (w - zw). */
#define ICV_ZERO_ROW_ZP 0x800

/* Flag OR-ed into icv_conv's `ib_dtype`: run the IB-gather kernels (every
 * A row fetched through its indirection-buffer entry, the paper's mainloop),
 * not the window / row-sliding / dense-A specialisations that a canonical
 * buffer otherwise permits.  For measuring the indirect algorithm itself. */
#define ICV_PREFER_GATHER 0x1000

/* Convolution geometry; field-for-field convbench.tensors.ConvParams
 * (tensors.py:41-72). */
typedef struct icv_conv_desc {
  int32_t kernel_h, kernel_w;
  int32_t stride_h, stride_w;
  int32_t dilation_h, dilation_w;
  int32_t pad_top, pad_left, pad_bottom, pad_right;
  int32_t in_channels, out_channels;
} icv_conv_desc;

/* (n, h, w, c) extent; convbench.tensors.Shape4 (tensors.py:18-38). */
typedef struct icv_shape4 {
  int64_t n, h, w, c;
} icv_shape4;

/* QNNPACK-style asymmetric quantization of one uint8 convolution.  No
 * reference counterpart (the reference is float32-only, tensors.py:107-108);
 * semantics in DESIGN.md §uint8. */
typedef struct icv_quant {
  int32_t input_zero_point;
  float input_scale;
  int32_t kernel_zero_point;
  float kernel_scale;
  int32_t output_zero_point;
  float output_scale;
  int32_t output_min, output_max;
} icv_quant;

/* ---- library ---------------------------------------------------------- */
ICV_API int32_t icv_abi_version(void);
ICV_API const char* icv_last_error(void);
/* Number of SMs / compute capability of `device` (for host-side planning). */
ICV_API int icv_device_info(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---- geometry --------------------------------------------------------- */
/* Output extent.  Replaces conv_output_shape, tensors.py:184-211
 * (ICV_ERR_ARG on channel mismatch :191-194, ICV_ERR_GEOMETRY when the
 * dilated kernel does not fit :203-208). */
ICV_API int icv_out_shape(const icv_conv_desc* desc, const icv_shape4* in, icv_shape4* out);

/* Tile and entry count of an indirection buffer built for `batch` images at
 * tile height `mr`: tiles = ceil(batch*Ho*Wo / mr), entries = tiles*R*S*mr
 * (indirect.py:94-95, :117). */
ICV_API int icv_ib_entries(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t mr,
                   int64_t* tiles, int64_t* entries);

/* ---- indirection buffer (hot path, K1) -------------------------------- */
/* Write entries for tiles [first_tile, T) of the (T, R*S, mr) buffer at
 * `ib` (element type ICV_I64 — the canonical form, ZERO_REF = -1 — or
 * ICV_I32).  Entry [t, e, m] = element offset of the input pixel row read by
 * tap e of output pixel min(t*mr + m, P - 1), or -1 for a padding tap.
 * Replaces _compute_offsets (indirect.py:98-126) as called by
 * init_indirection_buffer (:129-164; first_tile = 0) and
 * update_for_batch_growth (:185-192; first_tile = old full-tile count).
 * `ib` points at the START of the buffer (tile 0).  With ICV_IB_PER_IMAGE
 * in `ib_dtype` the per-image buffer is written and `batch` is ignored. */
ICV_API int icv_ib_build(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t mr,
                 int64_t first_tile, int32_t ib_dtype, void* ib, void* stream);

/* ---- filter packing (K7) ---------------------------------------------- */
/* Bytes of device storage icv_pack_filter writes for `compute_dtype`
 * (weights + per-channel epilogue constants). */
/* Count the entries of `ib` (layout flags as for icv_ib_build) that differ
 * from the canonical buffer of this geometry; the count is written to the
 * DEVICE int32 `mismatches` (stream-ordered, no synchronization). */
ICV_API int icv_ib_check(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t mr, int32_t ib_dtype,
                         const void* ib, int32_t* mismatches, void* stream);

ICV_API int icv_packed_filter_bytes(const icv_conv_desc* desc, int32_t compute_dtype, int64_t* bytes);

/* Repack KRSC weights (`w_dtype` ICV_F32 / ICV_BF16 / ICV_U8) into the
 * device layout the `compute_dtype` kernel reads, and fold the bias (f32 for
 * float paths, int32 for ICV_U8; NULL = zeros) plus, for uint8, the
 * zero-point corrections into the per-channel epilogue constants.  Replaces
 * pack_filter (gemm.py:135-167).  `quant` is required iff compute_dtype ==
 * ICV_U8. */
ICV_API int icv_pack_filter(const icv_conv_desc* desc, int32_t compute_dtype, int32_t w_dtype, const void* w_krsc,
                    const void* bias, const icv_quant* quant, void* packed, void* stream);

/* Requantization multiplier/shift for real_scale = sx*sw/so computed in
 * float64 from the float32 scales. */
ICV_API int icv_requant_params(float input_scale, float kernel_scale, float output_scale, int32_t* multiplier,
                       int32_t* shift);

/* ---- indirect convolution (hot path, K2/K3/K5) ------------------------ */
/* y[p, k] = bias[k] + sum_{e, c} X[ib(p, e) + c] * W[k, e, c] for the first
 * `batch` images (batch <= the buffer's batch; logical truncation,
 * indirect.py:265-275).  `x` is the bound NHWC input (`dtype`), `zero_row`
 * the C-element row substituted for ZERO_REF entries, `ib` the (T, R*S, mr)
 * buffer built for this geometry, `packed` the output of icv_pack_filter
 * for `dtype`.  Output `y` is NHWC (batch, Ho, Wo, K): float32 for ICV_F32,
 * bf16 for ICV_BF16, uint8 for ICV_U8.
 *   ICV_F32:  bit-exact with the reference (bias init, e then c ascending,
 *             separate multiply and add roundings; gemm.py:6-15).
 *   ICV_BF16: tcgen05 kind::f16 MMA, fp32 accumulate, bf16 out.
 *   ICV_U8:   tcgen05 kind::i8 MMA, int32 accumulate, fixed-point requant.
 * Replaces indirect_conv (indirect.py:239-300). */
ICV_API int icv_conv(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t dtype, const void* x,
             const void* zero_row, const void* ib, int32_t ib_dtype, int32_t mr, const void* packed,
             const icv_quant* quant, void* y, void* stream);

/* Which kernel icv_conv would launch for this problem (for tests/benches)
 * given the layout flags of its `ib_dtype` argument (ICV_IB_CANONICAL,
 * ICV_ZERO_ROW_ZEROS, ICV_PREFER_GATHER, ...) and 16-byte aligned tensors:
 * writes a static NUL-terminated name into *name. */
ICV_API int icv_conv_kernel_name(const icv_conv_desc* desc, const icv_shape4* in, int32_t dtype, int32_t flags,
                                 const char** name);

/* Plan knobs for A/B measurement (DESIGN.md §4 lists them; the defaults are
 * the measured-best plans): set / read a process-wide value by name.
 * Unknown names return ICV_ERR_ARG; a negative value restores the default
 * (except "win", where -1 is the default "auto").  Not synchronized with
 * concurrent icv_conv calls: set knobs before launching. */
ICV_API int icv_set_tuning(const char* key, int32_t value);
ICV_API int icv_get_tuning(const char* key, int32_t* value);

/* Launch counter: number of kernels this library has launched in this
 * process (all entry points).  For the bench's gpu_launches claim. */
ICV_API int64_t icv_launch_count(void);

/* NHWC max pooling (bf16 / f32), padding taps skipped (-inf padding).  Not
 * part of the reference operator: the ResNet-50 conv stack (cfg5, SURVEY.md
 * §8(d)) pools the stem output 3x3 / stride 2 / pad 1 before stage 1.
 * Output shape (n, (h + 2*ph - kh)/sh + 1, (w + 2*pw - kw)/sw + 1, c). */
ICV_API int icv_maxpool2d(const icv_shape4* in, int32_t kh, int32_t kw, int32_t sh, int32_t sw, int32_t ph,
                          int32_t pw, int32_t dtype, const void* x, void* y, void* stream);

/* ---- GEMM-based baseline: im2row patch matrix (reference im2col.py:48-114) --
 * Writes the (batch*OH*OW) x (R*S*C) patch matrix of `x` (dtype ICV_F32 /
 * ICV_BF16 / ICV_U8, NHWC): row p = output pixel, column e*C + c = tap e's
 * channel c, padding taps = `zero_row` (C elements) or zeros when NULL.
 * Replaces build_patch_matrix's copy loop (im2col.py:86-113); the paper's
 * GEMM baseline multiplies it with the filter (gemm_conv, im2col.py:117-131). */
ICV_API int icv_im2col(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t dtype, const void* x,
                       const void* zero_row, void* patches, void* stream);

/* ---- direct convolution: the harness's correctness oracle ----------------
 * Float32 output of the direct convolution of `x` (ICV_F32 / ICV_BF16 NHWC,
 * first `batch` images) with the KRSC filter `w` (ICV_F32 / ICV_BF16) plus
 * `bias` (float32, NULL = none): bias init, then ky, kx, c ascending with a
 * rounded multiply and a rounded add per tap, padding taps skipped -- the
 * reference's convbench.reference.direct_conv (reference.py:30-84),
 * bit-exact with it for float32.  No indirection buffer involved. */
ICV_API int icv_direct_conv(const icv_conv_desc* desc, const icv_shape4* in, int64_t batch, int32_t x_dtype,
                            const void* x, int32_t w_dtype, const void* w, const float* bias, float* y,
                            void* stream);

/* ---- filter replication for the batch-sharded operator --
 * The convolution shards by image (reference indirect.py:112-125: an
 * image's buffer entries, sums and outputs depend only on that image and
 * the replicated filter), so a data-parallel deployment has exactly one
 * collective: broadcasting the packed filter (icv_pack_filter's bytes) from
 * the source rank once per model load.  NCCL is loaded at run time
 * (libnccl.so.2); without it these return ICV_ERR_UNSUPPORTED.  `comm` is an
 * opaque ncclComm_t.  The reference has no multi-device path (SURVEY.md
 * §2.3); these replace nothing in it. */
#define ICV_NCCL_UNIQUE_ID_BYTES 128
ICV_API int icv_nccl_version(int32_t* version);
/* Rank 0 creates the id (ICV_NCCL_UNIQUE_ID_BYTES bytes) and ships it to the
 * other ranks out of band (torch.distributed's store in dist.py). */
ICV_API int icv_nccl_unique_id(void* id_out);
/* One process per GPU: each rank, its device current, joins the communicator. */
ICV_API int icv_nccl_init_rank(void** comm, int32_t nranks, const void* unique_id, int32_t rank);
/* One process driving `ndev` local GPUs (devices NULL = 0..ndev-1): one
 * communicator per device into comms[0..ndev). */
ICV_API int icv_nccl_init_all(void** comms, int32_t ndev, const int32_t* devices);
ICV_API int icv_nccl_comm_size(void* comm, int32_t* nranks);
/* Broadcast `bytes` from `root`'s sendbuf (NULL = in place in recvbuf) into
 * every rank's recvbuf, stream-ordered on `stream`. */
ICV_API int icv_nccl_broadcast(const void* sendbuf, void* recvbuf, int64_t bytes, int32_t root, void* comm,
                               void* stream);
ICV_API int icv_nccl_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* ICV_H_ */
