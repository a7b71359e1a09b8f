// K4: channel-poor indirect convolution on tcgen05 ("stem" kernel).
//
// For layers whose pixel rows are a few bytes (the 7x7/2 ResNet stem: C = 3
// bf16 = 6-byte rows) a per-tap 128-byte channel block would be 97 % padding,
// and cp.async cannot address 6-byte rows.  Here the GEMM K dimension is
// the whole receptive field, k = e*C + c (e = ky*S + kx, the reference's
// reduction order, indirect.py:287-294), padded to a multiple of 16:
// 147 -> 160 for the stem.  Each producer thread owns one output pixel (one
// A row): per tap it reads the row reference from the indirection buffer
// (ZERO_REF -> bound zero row), loads the tap's C elements with two aligned
// 32-bit loads and a funnel shift, packs them into registers at their K
// position and writes every completed 16-byte chunk straight into the
// 128B-swizzled A tile (st.shared.v4).  The packed filter (K_out <= 128 rows
// x K) stays resident in smem for the whole kernel (one TMA load), the MMA
// warp issues ceil(R*S*C/16) tcgen05.mma per 128-pixel tile, and the shared
// epilogue streams the bf16 output (the dominant HBM traffic of the layer).
#include <climits>

#include "igemm_common.cuh"

namespace icv {
namespace {

constexpr int kProdWarpsStem = 8;        // two producer threads per A row (tap halves)
constexpr int kProdThreads = 32 * kProdWarpsStem;
constexpr int kEpiWarpsStem = 4;
constexpr int kMmaWarpStem = kProdWarpsStem + kEpiWarpsStem;
constexpr int kThreadsStem = 32 * (kMmaWarpStem + 1);
#ifndef ICV_STEM_ACC
#define ICV_STEM_ACC 2
#endif
constexpr int kAccStagesStem = ICV_STEM_ACC;       // TMEM accumulators in flight (MMA runs ahead of the epilogue)
constexpr int kStagesStem = 2;          // A tiles in flight
constexpr int kPrefetch = 4;            // L2 prefetch distance of input windows (tiles, image-major)

// Byte offset of element offset `d` (a multiple of C) in the pixel-slot
// window (8 bytes per pixel): d / C * 8 = d * kSlotMul (mod 2^32).
__host__ __device__ constexpr uint32_t inv_odd(uint32_t c) {
  uint32_t x = c;   // Newton iterations for the inverse of an odd c mod 2^32
  for (int i = 0; i < 5; ++i) x *= 2u - c * x;
  return x;
}
template <int C>
constexpr uint32_t kSlotMul = (C & 1) ? 8u * inv_odd(C) : 8u / C;

// Tile schedule of the stem kernel: CTA b owns the contiguous virtual tiles
// [V*b/G, V*(b+1)/G).  With a per-image indirection buffer and whole tiles
// per image (Ho*Wo % 128 == 0), virtual tile v is pattern j = v / N of image
// n = v % N: consecutive tiles of a CTA share one reference pattern (the
// buffer is batch invariant), so its window layout and slot offsets are
// computed once per pattern and only the window's image offset changes.
struct StemTiles {
  int32_t total;     // tiles
  int32_t n_img;     // images sharing a pattern (1 unless image-major)
  int32_t tpi;       // tiles per image (image-major)
};
struct StemPos {
  int32_t key, img;  // pattern (image-0 tile, or the tile itself) and image of a local tile
};
struct StemSched {
  int32_t begin, n, n_img, tpi;
  __device__ __forceinline__ explicit StemSched(const StemTiles& t)
      : begin((int32_t)((int64_t)t.total * blockIdx.x / gridDim.x)),
        n((int32_t)((int64_t)t.total * (blockIdx.x + 1) / gridDim.x) - begin),
        n_img(t.n_img),
        tpi(t.tpi) {}
  __device__ __forceinline__ int64_t count() const { return n; }
  __device__ __forceinline__ StemPos pos(int64_t k) const {
    const int32_t v = begin + (int32_t)k;
    return n_img > 1 ? StemPos{v / n_img, v % n_img} : StemPos{v, 0};
  }
  __device__ __forceinline__ void advance(StemPos& p) const {
    if (++p.img == n_img) { p.img = 0; ++p.key; }
  }
  __device__ __forceinline__ int64_t tile(StemPos p) const {
    return n_img > 1 ? (int64_t)p.img * tpi + p.key : (int64_t)p.key;
  }
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return tile(pos(k)); }
};

#if defined(ICV_TRACE) || defined(ICV_STEM_PHASES)
// debug build: per-CTA cycle accumulators of the producer / MMA phases
// (slots 26..39 of g_icv_trace, tools/trace_stem.py), kept in registers
#define STEM_T0(cond) long long _t = clock64(), _acc[5] = {0, 0, 0, 0, 0}; const bool _tr = (cond)
#define STEM_ACC(i)                    \
  do {                                 \
    const long long _n = clock64();    \
    _acc[i] += _n - _t;                \
    _t = _n;                           \
  } while (0)
#define STEM_FLUSH(slot0, n) \
  if (_tr)                   \
    for (int _i = 0; _i < (n); ++_i) g_icv_trace[blockIdx.x][(slot0) + _i] = (unsigned long long)_acc[_i]
#else
#define STEM_T0(cond)
#define STEM_ACC(i)
#define STEM_FLUSH(slot0, n)
#endif

template <int C, int RS, int BN>
struct CfgStem {
  static constexpr int kK = RS * C;                         // real reduction length
  static constexpr int kKSteps = (kK + 15) / 16;            // MMA K steps (16 bf16 each)
  static constexpr int kBlocks = (kKSteps * 16 + 63) / 64;  // 128-byte K blocks per row
  static constexpr int kABytes = kBM * kBlocks * 128;       // one A tile
  static constexpr int kBBytes = BN * kBlocks * 128;        // resident filter
  static constexpr int kEpiBytes = kEpiWarpsStem * kEpiWarpBytes<false>;
  // Taps are assembled in groups of 8: 8 taps x C elements = C whole 16-byte
  // chunks of the A row.  kGroups groups cover the kKSteps*16 elements the
  // MMA reads (taps past R*S read a zero slot); the two producer halves take
  // groups [0, kG0) and [kG0, kGroups).
  static constexpr int kGroups = (kKSteps * 2 + C - 1) / C;
  static constexpr int kG0 = (kGroups + 1) / 2;
  static constexpr int kTapsHalf = kG0 * 8;                 // taps per producer thread (max)
  static constexpr int kTaps = kGroups * 8;
  // input-window capacity in pixels (cfg3a needs <= 1834; a 128-wide
  // resident 7x7x3 filter leaves room for half of that)
  static constexpr int kWinPix = (BN > 64 && RS * C > 64) ? 1024 : 2048;
  // staged input window: raw NHWC bytes of up to kWinPix pixels (cp.async)
  static constexpr int kStageBytes = kWinPix * C * 2;
  // pixel-slot window: 8 bytes per pixel (C elements, zero padded), then two
  // slots: the bound zero row (ZERO_REF taps) and true zeros (taps past R*S)
  static constexpr int kSlotBytes = (kWinPix + 2) * 8;
  static constexpr int kRelBytes = kTaps * kBM * 2;         // [kTaps/2][128][2] uint16 slot byte offsets
  static constexpr int kHalfPix = kWinPix / 2;              // even pixels, then odd pixels
  static constexpr int kMiscBytes = 1024;                   // bias, reductions, window bases
  static constexpr int kSmemBytes = 1024 + kStagesStem * kABytes + kBBytes + kEpiBytes + 2 * kStageBytes +
                                    2 * kSlotBytes + 2 * kRelBytes + kMiscBytes + 256;
  static_assert(kSmemBytes <= 232448, "shared memory overflow");
  static_assert(C >= 1 && C <= 4, "channel-poor kernel handles 1..4 channels");
  static_assert(kGroups * C * 8 <= kBlocks * 64, "tap groups overflow the A row");
  static_assert(kSlotBytes < 65536, "slot offsets are 16-bit");
};

// 16-byte chunk q (elements 8q .. 8q+7) of row `row` in the swizzled A tile.
__device__ __forceinline__ uint32_t a_chunk_addr(uint32_t tile, int row, int q) {
  const int blk = q >> 3, j = q & 7;
  return tile + blk * (kBM * 128) + row * 128 + ((j ^ (row & 7)) << 4);
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

// element j (0 .. 2*N-1) of a little-endian array of N packed bf16 pairs
template <int N>
__device__ __forceinline__ uint32_t elem16(const uint32_t (&v)[N], int j) {
  return (v[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
}

// Place tap i (0..7) of a group -- its C elements are the low 16*C bits of
// (hi:lo) -- at element i*C of the group's 4*C words.
template <int C>
__device__ __forceinline__ void place_tap(uint32_t (&w)[4 * C], int i, uint32_t lo, uint32_t hi) {
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const uint32_t v = c < 2 ? (lo >> (16 * c)) & 0xFFFFu : (hi >> (16 * (c - 2))) & 0xFFFFu;
    const int k = i * C + c;
    if (k & 1) w[k >> 1] |= v << 16;
    else w[k >> 1] = v;
  }
}

template <int C>
__device__ __forceinline__ void store_group(const uint32_t (&w)[4 * C], uint32_t tileA, int row, int g) {
#pragma unroll
  for (int j = 0; j < C; ++j) sts128(a_chunk_addr(tileA, row, g * C + j), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}

template <int C, int RS, int BN, typename IbT>
__global__ void __launch_bounds__(kThreadsStem, 1) igemm_stem_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                                     const __grid_constant__ CUtensorMap tmap_y,
                                                                     const TcArgs a, int32_t x_elems,
                                                                     const StemTiles tiles) {
  using Cf = CfgStem<C, RS, BN>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base (SW128 atoms); pointer arithmetic keeps the
  // shared address space visible to the compiler (no generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStagesStem * Cf::kABytes;
  uint8_t* sEpi = sB + Cf::kBBytes;
  uint8_t* sStage = sEpi + Cf::kEpiBytes;                            // [2] raw input windows
  uint8_t* sSlot = sStage + 2 * Cf::kStageBytes;                     // [2] pixel-slot windows (+ 2 zero slots)
  uint8_t* sRel = sSlot + 2 * Cf::kSlotBytes;                        // [2][kTaps/2][128][2] slot offsets
  uint8_t* sMisc = sRel + 2 * Cf::kRelBytes;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(sMisc);                         // 128 x 4 B
  int32_t* sRed = reinterpret_cast<int32_t*>(sMisc + 512);                      // [2][2][8] min/max per warp
  int32_t* sWin = reinterpret_cast<int32_t*>(sMisc + 512 + 128);                // [2] pixel groups (or -1)
  int32_t* sKeyW0 = reinterpret_cast<int32_t*>(sMisc + 512 + 144);              // [2] pattern window start
  int32_t* sKeyGroups = reinterpret_cast<int32_t*>(sMisc + 512 + 160);          // [2] pattern window groups
  uint64_t* full = reinterpret_cast<uint64_t*>(sMisc + Cf::kMiscBytes);
  uint64_t* empty = full + kStagesStem;
  uint64_t* tfull = empty + kStagesStem;
  uint64_t* tempty = tfull + kAccStagesStem;
  uint64_t* bfull = tempty + kAccStagesStem;
  uint64_t* winbar = bfull + 1;                                      // [2] raw window landed (bulk copy)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(winbar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const StemSched sched(tiles);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesStem; ++s) {
      mbar_init(&full[s], kProdThreads);   // every producer thread (st.shared + proxy fence + arrive)
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kAccStagesStem; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarpsStem);   // one arrival per epilogue warp
    }
    mbar_init(bfull, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&winbar[s], 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmap_b);
  }
  for (int i = threadIdx.x; i < a.n_pad; i += blockDim.x) sBias[i] = __ldg(static_cast<const uint32_t*>(a.bias) + i);
  if (threadIdx.x < 16) {   // the two fixed slots of each slot buffer: bound zero row, then true zeros
    const int j = threadIdx.x & 7;
    const uint16_t* z = reinterpret_cast<const uint16_t*>(a.zero_row);
    uint16_t* slot = reinterpret_cast<uint16_t*>(sSlot + (threadIdx.x >> 3) * Cf::kSlotBytes + Cf::kWinPix * 8);
    slot[j] = (j < 4 && j < C) ? __ldg(z + j) : (uint16_t)0;
  }
  constexpr uint32_t kTmemCols = kAccStagesStem * BN <= 256 ? 256 : 512;
  if (warp == kMmaWarpStem) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();   // (setup read only constants; tensors may belong to the previous kernel)
  griddep_launch_dependents();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t sA_u32 = smem_u32(sA);
  const uint32_t sB_u32 = smem_u32(sB);

  if (threadIdx.x == 0) {   // resident filter: one TMA box per 128-byte K block
    mbar_arrive_expect_tx(bfull, Cf::kBBytes);
    tma_load_3d(sB_u32, &tmap_b, bfull, 0, 0, 0);   // all kBlocks K blocks in one box
  }

  if (warp < kProdWarpsStem) {
    // ------------------------------------------------------------ producers
    // Thread (half, row) assembles half of A row `row` (one output pixel).
    // Per tile, the row references of its 128 pixels (indirection buffer)
    // bound the span of input pixels the tile reads (the "window").  Two
    // tiles ahead, the window's raw NHWC bytes are copied into smem with
    // coalesced 16-byte cp.async and every reference becomes a 16-bit slot
    // offset; when the tile comes up, the window is re-laid out as one
    // 8-byte slot per pixel, so each tap is a single aligned 8-byte shared
    // load.  A window wider than Cf::kWinPix pixels (never for the ResNet stem)
    // falls back to reading the taps straight from global memory.
    const int half = warp >> 2;
    const int row = threadIdx.x & (kBM - 1);
    const int g_begin = half ? Cf::kG0 : 0;
    const int g_end = half ? Cf::kGroups : Cf::kG0;
    const int e_begin = g_begin * 8;
    const int n_real = min((g_end - g_begin) * 8, RS - e_begin);   // taps below R*S
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(a.x);
    const uint32_t sStage_u32 = smem_u32(sStage);
    const uint32_t sSlot_u32 = smem_u32(sSlot);
    const uint32_t sRel_u32 = smem_u32(sRel);
    const int64_t my_tiles = sched.count();
    constexpr int kWordsPerRef = sizeof(IbT) / 4;   // low word of an int64 reference (offsets < 2^31)
    int32_t ref[Cf::kTapsHalf];        // raw references of this thread's taps (image-relative if per-image)
    int32_t base = 0;                  // element offset of this row's image (per-image buffers)
    // a new reference pattern starts at local tile k (position p)
    auto new_key = [&](int64_t k, StemPos p) { return k == 0 || p.img == 0; };

    auto load_refs = [&](int64_t k, StemPos p) {  // row references of local tile k's pattern -> registers
      if (k >= my_tiles || !new_key(k, p)) return;
      const RowRef rr = row_ref(a, p.key, row);     // image 0's tile (image-major) or the tile itself
      const int32_t* ib = reinterpret_cast<const int32_t*>(static_cast<const IbT*>(a.ib) + rr.ent0 +
                                                           (int64_t)e_begin * a.mr);
      const int64_t stride = a.mr * kWordsPerRef;
      base = (int32_t)rr.base;
#pragma unroll
      for (int i = 0; i < Cf::kTapsHalf; ++i) ref[i] = i < n_real ? __ldg(ib + i * stride) : -2;
    };
    // Window of local tile k.  For a new pattern: the CTA-wide pixel span of
    // its valid references -> (sKeyW0, sKeyGroups)[key & 1] and the slot
    // offsets -> sRel[key & 1].  Then the raw window bytes of tile k (the
    // pattern's window moved to tile k's image) -> sStage[k & 1].
    auto prepare = [&](int64_t k, StemPos p) {
      if (k < my_tiles) {
        const int buf = (int)(k & 1);
        const int ks = p.key & 1;
        if (new_key(k, p)) {
          uint32_t lo = 0xFFFFFFFFu;   // ZERO_REF (-1) and padding (-2) are the largest as unsigned
          int32_t hi = -1;
#pragma unroll
          for (int i = 0; i < Cf::kTapsHalf; ++i) {
            lo = min(lo, (uint32_t)ref[i]);
            hi = max(hi, ref[i]);
          }
          const bool row_valid = hi >= 0;
          if (row_valid) { lo += base; hi += base; }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          }
          if (lane == 0) { sRed[ks * 16 + warp] = (int32_t)lo; sRed[ks * 16 + 8 + warp] = hi; }
          named_bar_sync(1, kProdThreads);   // also: every producer finished assembling tile k-2
          lo = 0xFFFFFFFFu;
          hi = -1;
#pragma unroll
          for (int i = 0; i < kProdWarpsStem; ++i) {
            lo = min(lo, (uint32_t)sRed[ks * 16 + i]);
            hi = max(hi, sRed[ks * 16 + 8 + i]);
          }
          const int32_t w0 = hi < 0 ? 0 : (int32_t)(lo / (8 * C) * (8 * C));   // 8-pixel (16C-byte) aligned
          const int32_t groups = hi < 0 ? 0 : ((hi - w0) / C + 8) / 8;           // 8-pixel groups spanned
          if (threadIdx.x == 0) { sKeyW0[ks] = w0; sKeyGroups[ks] = groups; }
          // pixel s of the window lives in slot (s & 1) * kHalfPix + (s >> 1); ZERO_REF -> slot Cf::kWinPix
          // (pixel 2 * Cf::kWinPix), taps past R*S -> slot Cf::kWinPix + 1
          const int32_t d = row_valid ? w0 - base : -2 * Cf::kWinPix * C;
          const uint32_t zc = (uint32_t)(2 * Cf::kWinPix * C + d);
          const uint32_t rel_base = sRel_u32 + ks * Cf::kRelBytes + ((g_begin * 4) * kBM + row) * 4;
#pragma unroll
          for (int i = 0; i < Cf::kTapsHalf; i += 2) {
            if (i < (g_end - g_begin) * 8) {
              uint32_t r2 = 0;
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const uint32_t px = (min((uint32_t)ref[i + j], zc) - (uint32_t)d) * kSlotMul<C> / 8;
                const uint32_t off = i + j < n_real ? ((px & 1) * Cf::kHalfPix + (px >> 1)) * 8
                                                    : (uint32_t)(Cf::kWinPix + 1) * 8;
                r2 |= (off & 0xFFFFu) << (16 * j);
              }
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(rel_base + (i / 2) * kBM * 4), "r"(r2) : "memory");
            }
          }
        }
        // One bulk copy of the window's bytes (contiguous NHWC pixels) into
        // sStage[k & 1], tracked by winbar[k & 1] (the stage buffer is free:
        // every producer converted tile k-2 before the last barrier).  With
        // the image-major schedule the same pattern's window kPrefetch images
        // later is pulled into L2 at the same time.
        if (threadIdx.x == 0) {
          const int32_t groups = sKeyGroups[ks];
          const int32_t w0 = sKeyW0[ks] + p.img * (int32_t)a.img_elems;
          const bool fits = groups * 8 <= Cf::kWinPix;
          sWin[buf] = fits ? groups : -1;
          if (fits && groups > 0) {
            const int64_t end = (int64_t)w0 + groups * 8 * C;            // window end (elements)
            const int64_t lim = end < x_elems ? end : x_elems;
            const uint32_t bytes = (uint32_t)(((lim - w0) * 2) & ~15LL);   // whole 16-byte chunks in bounds
            const uint32_t dst = sStage_u32 + buf * Cf::kStageBytes;
            // a ragged tail (< 16 bytes, only the tensor's last chunk) is copied by this thread
            for (int64_t b = bytes; b < (lim - w0) * 2; b += 2)
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst + (uint32_t)b),
                           "h"(__ldg(reinterpret_cast<const uint16_t*>(a.x) + w0 + b / 2)) : "memory");
            mbar_arrive_expect_tx(&winbar[buf], bytes);
            if (bytes) bulk_load(dst, a.x + (int64_t)w0 * 2, bytes, &winbar[buf]);
            if (sched.n_img > 1 && p.img + kPrefetch < sched.n_img && k + kPrefetch < my_tiles) {
              const int64_t pw0 = (int64_t)w0 + (int64_t)kPrefetch * a.img_elems;
              const int64_t pend = pw0 + groups * 8 * C < x_elems ? pw0 + groups * 8 * C : x_elems;
              const uint32_t pbytes = (uint32_t)(((pend - pw0) * 2) & ~15LL);
              if (pbytes) bulk_prefetch_l2(a.x + pw0 * 2, pbytes);
            }
          } else {
            mbar_arrive(&winbar[buf]);
          }
        }
      }
    };

    // prologue: windows of tiles 0 and 1
    StemPos pb = sched.pos(0);       // tile being assembled (k)
    StemPos pp = pb;                 // tile being prepared (k + 2)
    load_refs(0, pp);
    prepare(0, pp);
    sched.advance(pp);
    load_refs(1, pp);
    prepare(1, pp);
    sched.advance(pp);
    int stage = 0;
    uint32_t phase = 0;
    STEM_T0(threadIdx.x == 0 || threadIdx.x == 128);
    for (int64_t k = 0; k < my_tiles; ++k) {
      load_refs(k + 2, pp);                   // lands while tile k is assembled
      const int buf = (int)(k & 1);
      mbar_wait(&winbar[buf], (uint32_t)(k >> 1) & 1u);   // window k landed (and sWin[buf] published)
      STEM_ACC(0);
      const int32_t groups = sWin[buf];
      const uint32_t slots = sSlot_u32 + buf * Cf::kSlotBytes;
      if (groups > 0) {                       // raw window -> pixel slots (even pixels, then odd pixels)
        const uint32_t src = sStage_u32 + buf * Cf::kStageBytes;
        for (int g = threadIdx.x; g < groups; g += kProdThreads) {
          uint32_t v[4 * C];                  // 8 pixels x C elements
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const uint4 t = lds128(src + (g * C + q) * 16);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
          }
          uint32_t s[16];                     // 8 slots x 2 words
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            s[2 * p] = elem16(v, p * C) | (C > 1 ? elem16(v, p * C + 1) << 16 : 0u);
            s[2 * p + 1] = (C > 2 ? elem16(v, p * C + 2) : 0u) | (C > 3 ? elem16(v, p * C + 3) << 16 : 0u);
          }
#pragma unroll
          for (int par = 0; par < 2; ++par) {
            const uint32_t dst = slots + (par * Cf::kHalfPix + g * 4) * 8;
            sts128(dst, s[2 * par], s[2 * par + 1], s[2 * par + 4], s[2 * par + 5]);
            sts128(dst + 16, s[2 * par + 8], s[2 * par + 9], s[2 * par + 12], s[2 * par + 13]);
          }
        }
      }
      // slots of tile k ready; every producer finished tile k-1 (so slot buffer
      // buf^1 and its stage are free for tile k+1) and has read sWin[buf]
      named_bar_sync(1, kProdThreads);
      STEM_ACC(1);
      mbar_wait(&empty[stage], phase ^ 1);
      STEM_ACC(2);
      const uint32_t tileA = sA_u32 + stage * Cf::kABytes;
#ifdef ICV_EXP_STEM_NOBUILD
      if (false) {
#else
      if (groups >= 0) {
#endif
        const uint32_t rel_base = sRel_u32 + (pb.key & 1) * Cf::kRelBytes + row * 4;
#pragma unroll 2
        for (int g = g_begin; g < g_end; ++g) {
          uint32_t w[4 * C];
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const uint32_t r2 = lds32(rel_base + (g * 4 + i / 2) * kBM * 4);
            const uint2 v0 = lds64(slots + (r2 & 0xFFFFu));
            const uint2 v1 = lds64(slots + (r2 >> 16));
            place_tap<C>(w, i, v0.x, v0.y);
            place_tap<C>(w, i + 1, v1.x, v1.y);
          }
          store_group<C>(w, tileA, row, g);
        }
      } else if (groups < 0) {
        // window too wide: read the taps from global memory
        const RowRef rr = row_ref(a, sched.tile(pb), row);
        const IbT* ib = static_cast<const IbT*>(a.ib) + rr.ent0;
        const uint2 zr = lds64(slots + Cf::kWinPix * 8);
#pragma unroll 1
        for (int g = g_begin; g < g_end; ++g) {
          uint32_t w[4 * C];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int e = g * 8 + i;
            uint32_t lo = 0, hi = 0;
            if (e < RS) {
              const int64_t raw = (int64_t)__ldg(ib + (int64_t)e * a.mr);
              if (raw >= 0) {
                const int64_t off = raw + rr.base;
                const int64_t wi = off >> 1;
                const uint32_t sh = (uint32_t)(off & 1) * 16;
                const uint32_t l = __ldg(x32 + wi);
                uint32_t h = 0u;
                if (2 * (wi + 1) + 1 < x_elems) h = __ldg(x32 + wi + 1);
                else if (2 * (wi + 1) < x_elems) h = __ldg(reinterpret_cast<const uint16_t*>(a.x) + 2 * (wi + 1));
                lo = __funnelshift_r(l, h, sh);
                hi = h >> sh;
              } else {
                lo = zr.x;
                hi = zr.y;
              }
            }
            place_tap<C>(w, i, lo, hi);
          }
          store_group<C>(w, tileA, row, g);
        }
      }
      fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
      mbar_arrive(&full[stage]);
      STEM_ACC(3);
      if (++stage == kStagesStem) { stage = 0; phase ^= 1; }
      prepare(k + 2, pp);
      sched.advance(pp);
      sched.advance(pb);
      STEM_ACC(4);
    }
    STEM_FLUSH(30 + 5 * half, 5);
  } else if (warp == kMmaWarpStem) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc<false>(kBM, BN);
    mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int as = 0;
    uint32_t aphase = 0;
    const int64_t n_local = sched.count();
    STEM_T0(lane == 0);
    for (int64_t k = 0; k < n_local; ++k) {
      mbar_wait(&tempty[as], aphase ^ 1);
      STEM_ACC(0);
      mbar_wait(&full[stage], phase);
      STEM_ACC(1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = tmem_base + as * BN;
        const uint32_t tileA = sA_u32 + stage * Cf::kABytes;
#pragma unroll
        for (int ks = 0; ks < Cf::kKSteps; ++ks) {
          const int blk = ks >> 2, kk = ks & 3;
          const uint64_t ad = sw128_kmajor_desc(tileA + blk * kBM * 128) + 2 * kk;
          const uint64_t bd = sw128_kmajor_desc(sB_u32 + blk * BN * 128) + 2 * kk;
          tc_mma<false>(d, ad, bd, idesc, ks != 0);
        }
        tc_commit(&empty[stage]);
        tc_commit(&tfull[as]);
      }
      __syncwarp();
      if (++stage == kStagesStem) { stage = 0; phase ^= 1; }
      if (++as == kAccStagesStem) { as = 0; aphase ^= 1; }
    }
    STEM_FLUSH(26, 2);
  } else {
    epilogue_loop<false, BN, kEpiWarpsStem, BN, StemSched, kAccStagesStem>(a, warp - kProdWarpsStem, lane, tmem_base,
                                                                         sEpi, sBias, tfull, tempty,
                                                 sched, a.use_tma_y ? &tmap_y : nullptr);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarpStem) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

template <int C, int RS, int BN, typename IbT>
int launch_stem_t(const ConvArgs& c, cudaStream_t st) {
  using Cf = CfgStem<C, RS, BN>;
  const int64_t x_elems = c.g.N * c.g.H * c.g.W * (int64_t)c.g.C;
  if (x_elems >= (int64_t(1) << 31)) return fail(ICV_ERR_UNSUPPORTED, "stem kernel: input too large");
  auto kernel = igemm_stem_kernel<C, RS, BN, IbT>;
  if (int s = kernel_setup(reinterpret_cast<const void*>(kernel), Cf::kSmemBytes, 1, 0, nullptr)) return s;
  CUtensorMap tmap;
  if (int s = make_filter_tmap(c, BN, Cf::kBlocks, &tmap)) return s;
  TcArgs a;
  fill_tc_args(c, BN, &a);
  const int sms = sm_count();
  const int grid = (int)(a.total_tiles < sms ? a.total_tiles : sms);
  if (a.total_tiles >= (int64_t(1) << 31)) return fail(ICV_ERR_UNSUPPORTED, "stem kernel: too many tiles");
  StemTiles tiles{(int32_t)a.total_tiles, 1, (int32_t)a.total_tiles};
  if (a.ib_per_image && a.ohw % kBM == 0 && a.P / a.ohw > 1 && a.total_tiles == a.P / kBM) {
    tiles.n_img = (int32_t)(a.P / a.ohw);   // image-major: consecutive tiles share one reference pattern
    tiles.tpi = (int32_t)(a.ohw / kBM);
  }
  CUtensorMap tmap_y;
  a.use_tma_y = make_output_tmap(c, &tmap_y) == ICV_OK;
  if (!a.use_tma_y) tmap_y = tmap;   // unused placeholder
  return launch_conv_kernel(kernel, (unsigned)grid, kThreadsStem, Cf::kSmemBytes, st, 1, "igemm_stem launch", tmap,
                            tmap_y, a, (int32_t)x_elems, tiles);
}

template <typename IbT>
int dispatch_stem(const ConvArgs& c, cudaStream_t st) {
  const int rs = c.g.RS(), bn = c.L.block_n;
  if (c.g.C == 3 && rs == 49) return bn == 64 ? launch_stem_t<3, 49, 64, IbT>(c, st) : launch_stem_t<3, 49, 128, IbT>(c, st);
  if (c.g.C == 3 && rs == 9) return bn == 64 ? launch_stem_t<3, 9, 64, IbT>(c, st) : launch_stem_t<3, 9, 128, IbT>(c, st);
  if (c.g.C == 1 && rs == 9) return bn == 64 ? launch_stem_t<1, 9, 64, IbT>(c, st) : launch_stem_t<1, 9, 128, IbT>(c, st);
  return fail(ICV_ERR_UNSUPPORTED, "no channel-poor tensor-core kernel for this shape");
}

}  // namespace

bool stem_kernel_eligible(int C, int RS, int K) {
  return K <= 128 && ((C == 3 && (RS == 49 || RS == 9)) || (C == 1 && RS == 9));
}

int launch_conv_stem(const ConvArgs& c, cudaStream_t st) {
  // stride-2 layers with a canonical buffer: the row-sliding kernel (igemm_rows.cu)
  if (!c.prefer_gather && c.ib_canonical && c.L.rows_off && rows_kernel_eligible(c.g)) return launch_conv_rows(c, st);
  if (c.ib_is_i32) return dispatch_stem<int32_t>(c, st);
  return dispatch_stem<int64_t>(c, st);
}

}  // namespace icv
