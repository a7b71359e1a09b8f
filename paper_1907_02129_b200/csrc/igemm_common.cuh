// Pieces shared by the two tcgen05 indirect-GEMM kernels (igemm_tc.cu:
// A operand gathered into shared memory; igemm_tmem.cu: A operand gathered
// into tensor memory): kernel arguments, indirection-buffer addressing, the
// TMEM -> registers -> HBM epilogue, and the TMA descriptor of the packed
// filter.
#pragma once
#include <type_traits>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "icv_internal.h"
#include "requant.cuh"
#include "sm100_ptx.cuh"

namespace icv {

constexpr int kBM = 128;                // output pixels per tile (TMEM lanes / MMA M)
constexpr int kABytes = kBM * 128;      // one 128-byte K block of the A tile
constexpr int kMaxBias = 2048;          // output channels whose epilogue constants live in smem

#if (defined(ICV_STEM_PHASES) || defined(ICV_ROWS_PHASES) || defined(ICV_ROWS_TIMELINE)) && !defined(ICV_TRACE)
extern __device__ unsigned long long g_icv_trace[1024][128];
#define TRACE(slot)
#elif defined(ICV_TRACE)
// Debug-build timeline (tools/trace_conv.py): per CTA, globaltimer (ns) at
// kernel entry [0], after setup [1], MMA warp's last commit of tile i [2+i],
// epilogue's tmem-full wakeup of tile i [10+i] and release [18+i], producer
// start of tile i [26+i] (i < 8).  Never compiled into the shipped library.
extern __device__ unsigned long long g_icv_trace[1024][128];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot) g_icv_trace[blockIdx.x][slot] = gtime()
#else
#define TRACE(slot)
#endif

struct TcArgs {
  const uint8_t* x;
  const uint8_t* zero_row;
  const void* ib;
  int64_t mr, P;
  int32_t RS, c_bytes, cblocks, elem_bytes, K, n_tiles;
  int64_t total_tiles;
  const void* bias;  // f32 (bf16) or int32 (u8) epilogue constant per padded output channel
  void* y;
  int32_t zw, zo, qmin, qmax, m0, shift;
  int32_t n_pad;
  int32_t cblock_elems;      // elements per 128-byte channel block
  int32_t c_tz;              // C = odd << c_tz
  uint32_t c_inv;            // odd^-1 mod 2^32
  int32_t use_tma_x;         // input tensor map valid (TMA gathers allowed)
  int32_t ib_per_image;      // buffer holds image 0's (image-relative) references
  int32_t use_tma_y;         // output tensor map valid: epilogue stores tiles with TMA
  int32_t tiles_per_row;     // row-tiled kernels: tile = (output row, 128-pixel block); 3-D output map
  int32_t ow;                // row-tiled kernels: output row width (pixels >= ow are not stored)
  int64_t ohw, img_elems;    // Ho*Wo, H*W*C
  int32_t oh;                // row-pair tiles (kSubRows 2): output rows per image
  int32_t dense_pf;          // dense A: L2-prefetch the A rows this many local tiles ahead (0 = off)
  int32_t epi_wide;          // bf16 epilogue: 64-column chunks, 128-byte-swizzled staging, 64 x 32 TMA boxes
  int64_t x_rows;            // dense A: pixel rows of the bound input
  // im2col A (use_tma_x == 2): output width, kernel width, strides, dilations, leading pads
  int32_t im_ow, im_s, im_sx, im_sy, im_dx, im_dy, im_pl, im_pt;
  // uint8 im2col A: padded taps are zero-filled by TMA instead of holding the
  // zero point; the epilogue adds the per-channel correction of the pixel's
  // border class (row class x column class: which taps leave the image)
  const int32_t* tapcorr;    // [RS][n_pad] zx * sum_c (w - zw) per (tap, channel); nullptr = no corrections
  int32_t im_r, im_h, im_w, im_oh;
  int32_t ncls, cls_tb, cls_ohb, cls_nr, cls_lb, cls_owb, cls_ncc;
};

// Border classes of an output row / column index v of n classes: the top
// (left) prefix v < tb one class each, the bottom (right) suffix v >= ohb one
// class each, everything between the single interior class n - 1; border_rep
// gives a representative index of class k.
__device__ __forceinline__ int border_class(int v, int tb, int ohb, int n) {
  return v < tb ? v : (v >= ohb ? tb + v - ohb : n - 1);
}
__device__ __forceinline__ int border_rep(int k, int tb, int ohb, int n) {
  return k < tb ? k : (k < n - 1 ? ohb + k - tb : tb);
}

// Where the references of output pixel p = tile_m*128 + row live: entry of
// tap 0 (tap e adds e*mr; layout tile-major, kernel element, lane,
// indirect.py:14-16) and the element offset to add to non-ZERO_REF entries.
// p is clamped to the last real pixel (indirect.py:111).  Canonical buffer:
// entry ((p / mr) * RS) * mr + p % mr, base 0.  Per-image buffer: the same for
// q = p mod (Ho*Wo) in image 0's buffer, base n*H*W*C.
struct RowRef {
  int64_t ent0;
  int64_t base;
};
__device__ __forceinline__ RowRef row_ref(const TcArgs& a, int64_t tile_m, int row) {
  int64_t p = tile_m * kBM + row;
  p = p < a.P ? p : a.P - 1;
  int64_t base = 0;
  if (a.ib_per_image) {
    const int64_t n = p / a.ohw;
    p -= n * a.ohw;
    base = n * a.img_elems;
  }
  const int64_t t = p / a.mr;
  return {t * a.RS * a.mr + (p - t * a.mr), base};
}
__device__ __forceinline__ int64_t resolve_ref(int64_t raw, int64_t base) { return raw < 0 ? raw : raw + base; }

// Pixel-row index of an element offset (offsets are multiples of C).
__device__ __forceinline__ int32_t pixel_row(const TcArgs& a, int64_t off) {
  return (int32_t)(((uint32_t)off >> a.c_tz) * a.c_inv);
}

template <typename IbT>
__device__ __forceinline__ int64_t load_ref(const TcArgs& a, int64_t ent) {
  return (int64_t)__ldg(static_cast<const IbT*>(a.ib) + ent);
}

// ----------------------------------------------------------------------------
// Epilogue (K6).  Epilogue warp `ew` (warp_id % 4 == ew % 4, which fixes the
// TMEM lane quarter it may read) owns 32 rows of the tile and, when there are
// 8 epilogue warps, half of its columns.  Per 32-column chunk: tcgen05.ld the
// fp32/s32 accumulators (the next chunk's load is in flight while this one is
// converted), add the folded bias / zero-point constants from smem, cast to
// bf16 or requantize to uint8, stage the 32 x 32 block in smem and write it out
// with row-contiguous 16-byte stores.  Tail rows (>= P) and columns (>= K) are
// never stored (indirect.py:299).
// Epilogue store of the first min(n, 16) bytes of `val` (misaligned or
// ragged output rows); a rolled loop, so the fast path is not if-converted
// into predicated byte stores.
__device__ __forceinline__ void store_partial(uint8_t* dst, uint4 val, int n) {
#pragma unroll 1
  for (int j = 0; j < 16 && j < n; ++j) {
    const uint32_t word = j < 4 ? val.x : j < 8 ? val.y : j < 12 ? val.z : val.w;
    dst[j] = (uint8_t)(word >> (8 * (j & 3)));
  }
}

#ifdef ICV_ROWS_PHASES   // debug: epilogue phase cycle accumulators (warp 0, lane 0) -> g_icv_trace[cta][42..47]
#define EP_ACC(i) do { const long long _n = clock64(); _ep[i] += _n - _et; _et = _n; } while (0)
#else
#define EP_ACC(i)
#endif

// Tile schedule: local tile k of this CTA is tile_of(k), k < n_local
// (default: tiles blockIdx.x, blockIdx.x + gridDim.x, ...).
struct StridedTiles {
  int64_t total;
  __device__ __forceinline__ int64_t count() const {
    return blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  }
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return blockIdx.x + k * gridDim.x; }
};

// Epilogue staging per warp: two 32-row tiles of one 32-column chunk (the
// TMA-store path double-buffers them; the fallback path uses 80/48-byte
// padded rows in the same space).  1024-byte aligned in the TMA kernels.
template <bool kI8>
constexpr int kEpiWarpBytes = kI8 ? 2048 : 4096;

// kTileGroups > 1: the epilogue warps split into groups of 4 that take
// alternate tiles (each warp all BN columns of its 32 rows), so several
// tiles are in the epilogue at once; otherwise extra warps split columns.
template <bool kI8, int BN, int kEpiWarps, int kAccStride, typename Sched = StridedTiles, int kAccStages = 2,
          bool kRowTiles = false, int kTileGroups = 1, int kSubRows = 1>
__device__ __forceinline__ void epilogue_loop(const TcArgs& a, int ew, int lane, uint32_t tmem_base, uint8_t* sEpi,
                                              const uint32_t* sBias, uint64_t* tfull, uint64_t* tempty,
                                              Sched sched = Sched{0}, const CUtensorMap* tmap_y = nullptr,
                                              uint32_t tempty_remote = 0, const int32_t* smem_sums = nullptr,
                                              const int32_t* cls_corr = nullptr) {
  constexpr int kOutRowBytes = kI8 ? 32 : 64;
  constexpr int kStageRowBytes = kI8 ? 48 : 80;  // padded: row-per-lane staging writes are conflict free
  const int slot = ew & 3;
  constexpr int kColGroups = kEpiWarps / 4 / kTileGroups;
  constexpr int kColsPerWarp = BN / kColGroups;
  const int group = kTileGroups > 1 ? ew / 4 : 0;
  const int col0 = kTileGroups > 1 ? 0 : (ew / 4) * kColsPerWarp;
  uint8_t* stg = sEpi + ew * kEpiWarpBytes<kI8>;
  const bool vec_ok = kI8 ? (a.K & 15) == 0 : (a.K & 7) == 0;
  const bool use_tma = tmap_y != nullptr;
  int chunk_seq = 0;
  int as = 0;
  uint32_t aphase = 0;
  if constexpr (std::is_same<Sched, StridedTiles>::value) sched.total = a.total_tiles;
  const int64_t n_local = sched.count();
#ifdef ICV_TRACE
  long long t_prev = clock64(), t_wait = 0, t_work = 0;
#endif
#ifdef ICV_ROWS_PHASES
  long long _et = clock64(), _ep[6] = {0, 0, 0, 0, 0, 0};
#endif
  // kSubRows 2 (row-tiled, two groups): a tile covers two output rows, one
  // accumulator each; group g stores row g of every tile
  static_assert(kSubRows == 1 || (kRowTiles && kTileGroups == 2), "sub-rows: one group per row");
  constexpr int kTileStep = kSubRows > 1 ? 1 : kTileGroups;
  if constexpr (kTileGroups > 1 && kSubRows == 1) {   // this group's first tile
    as = group % kAccStages;
    aphase = (uint32_t)(group / kAccStages) & 1u;
  }
  for (int64_t ti = kSubRows > 1 ? 0 : group; ti < n_local; ti += kTileStep) {
    const int64_t tile = sched(ti);
    const int64_t mt = a.n_tiles == 1 ? tile : tile / a.n_tiles;
    const int nt = a.n_tiles == 1 ? 0 : (int)(tile - mt * a.n_tiles);
    EP_ACC(5);
    mbar_wait(&tfull[as], aphase);
    tc_fence_after();
    EP_ACC(0);
#ifdef ICV_TRACE
    {   // slot 28: cycles waiting for accumulators, 29: cycles working (warp 0, lane 0)
      const long long t = clock64();
      t_wait += t - t_prev;
      t_prev = t;
    }
#endif
    const int ti_ = (int)ti;
    if (ew == 0 && lane == 0 && ti_ < 8) TRACE(10 + ti_);
    // first pixel of this warp's rows; row-tiled: (output row, first pixel of the block)
    int64_t row0 = mt * kBM + slot * 32;
    int32_t rt_row = 0, rt_ox0 = 0;
    bool row_valid = true;
    if constexpr (kRowTiles) {
      rt_row = (int32_t)((uint32_t)mt / (uint32_t)a.tiles_per_row);
      rt_ox0 = ((int32_t)mt - rt_row * a.tiles_per_row) * kBM + slot * 32;
      if constexpr (kSubRows > 1) {   // rt_row is a row-pair index: (image, output row 2 * pair + group)
        const int32_t ohp = (a.oh + 1) >> 1;
        const int32_t img = (int32_t)((uint32_t)rt_row / (uint32_t)ohp);
        const int32_t oy = 2 * (rt_row - img * ohp) + group;
        row_valid = oy < a.oh;
        rt_row = img * a.oh + oy;
      }
      row0 = (int64_t)rt_row * a.ow + rt_ox0;
    }
    const uint32_t taddr = tmem_base + ((uint32_t)(slot * 32) << 16) + as * kAccStride + (kSubRows > 1 ? group * BN : 0);
    int32_t rowsum = 0;
    if constexpr (kI8) {
      if (smem_sums) {   // (row sums computed by the kernel's row-sum warps: [accumulator stage][row])
        rowsum = smem_sums[as * kBM + slot * 32 + lane];
      } else {
        uint32_t rs;
        tmem_ld_32x32b_x1(taddr + BN, rs);
        tmem_ld_wait();
        rowsum = (int32_t)rs;
      }
    }
    // uint8 over zero-filled (im2col TMA) A tiles: this lane's pixel's border
    // class selects the staged correction vector ([class][n_pad], smem)
    const int32_t* my_corr = nullptr;
    if constexpr (kI8) {
      if (cls_corr != nullptr) {
        int64_t p = row0 + lane;
        p = p < a.P ? p : a.P - 1;
        const int64_t n = p / a.ohw;
        const int32_t r = (int32_t)(p - n * a.ohw);
        const int32_t oy = r / a.im_ow, ox = r - oy * a.im_ow;
        my_corr = cls_corr + (border_class(oy, a.cls_tb, a.cls_ohb, a.cls_nr) * a.cls_ncc +
                              border_class(ox, a.cls_lb, a.cls_owb, a.cls_ncc)) * a.n_pad;
      }
    }
    const int cols_left = a.K - nt * BN - col0;
#ifdef ICV_EXP_NOEPI   // experiment: release the accumulators without storing
    const int nchunks = 0;
    (void)cols_left;
#else
    const int nchunks = cols_left > 0 && row_valid ? (min(kColsPerWarp, cols_left) + 31) / 32 : 0;
#endif
    bool done_wide = false;
    if constexpr (!kI8 && kColsPerWarp % 64 == 0) {
      if (use_tma && a.epi_wide) {
        // 64-column chunks: two TMEM loads under one wait, the 32 x 64 block
        // staged 128-byte swizzled (conflict-free row-per-lane writes) and
        // stored as one 4 KB TMA box -- half the fences, stores and waits of
        // the 32-column path.  One staging buffer per warp: the previous
        // box must have been read before it is rewritten (that wait overlaps
        // this chunk's TMEM loads and conversion).
        const int nw = nchunks > 0 ? (min(kColsPerWarp, cols_left) + 63) / 64 : 0;
        const uint32_t sb = smem_u32(stg);
#pragma unroll 1
        for (int ci = 0; ci < nw; ++ci) {
          const int c = col0 + ci * 64;
          const int n = nt * BN + c;
          uint32_t v0[32], v1[32];
          tmem_ld_32x32b_x32(taddr + c, v0);
          tmem_ld_32x32b_x32(taddr + c + 32, v1);
          tmem_ld_wait_regs(v0);
          tmem_ld_wait_regs(v1);
          EP_ACC(1);
          uint32_t w[32];
          const float4* bias4 = reinterpret_cast<const float4*>(sBias + n);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float4 b = bias4[q];
            const uint32_t* vv = q < 8 ? v0 : v1;
            const int o = 4 * (q & 7);
            __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(vv[o + 0]) + b.x, __uint_as_float(vv[o + 1]) + b.y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(vv[o + 2]) + b.z, __uint_as_float(vv[o + 3]) + b.w);
            w[2 * q] = *reinterpret_cast<uint32_t*>(&lo);
            w[2 * q + 1] = *reinterpret_cast<uint32_t*>(&hi);
          }
          EP_ACC(2);
          if (chunk_seq > 0) {
            if (lane == 0) bulk_wait_group_read<0>();
            __syncwarp();
          }
          EP_ACC(5);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            sts128(sb + lane * 128 + ((q ^ (lane & 7)) << 4), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          EP_ACC(3);
          if (lane == 0) {
            if constexpr (kRowTiles)   // (channel, pixel in the output row, output row); pixels >= Wo clipped
              tma_store_3d(tmap_y, sb, n, rt_ox0, rt_row);
            else
              tma_store_2d(tmap_y, sb, n, (int32_t)row0);
            bulk_commit_group();
          }
          EP_ACC(4);
          ++chunk_seq;
        }
        done_wide = true;
      }
    }
    if (!done_wide) {
    uint32_t v[32];
    if (nchunks > 0) {
      tmem_ld_32x32b_x32(taddr + col0, v);
      tmem_ld_wait_regs(v);
    }
    EP_ACC(1);
#pragma unroll 1
    for (int ci = 0; ci < nchunks; ++ci) {
      const int c = col0 + ci * 32;
      const int n = nt * BN + c;
      uint32_t vn[32];
      if (ci + 1 < nchunks) tmem_ld_32x32b_x32(taddr + c + 32, vn);
      uint32_t w[kI8 ? 8 : 16];
      if constexpr (!kI8) {
        const float4* bias4 = reinterpret_cast<const float4*>(sBias + n);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b = bias4[q];
          __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(v[4 * q + 0]) + b.x,
                                                    __uint_as_float(v[4 * q + 1]) + b.y);
          __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(v[4 * q + 2]) + b.z,
                                                    __uint_as_float(v[4 * q + 3]) + b.w);
          w[2 * q] = *reinterpret_cast<uint32_t*>(&lo);
          w[2 * q + 1] = *reinterpret_cast<uint32_t*>(&hi);
        }
      } else {
        const int4* cst4 = reinterpret_cast<const int4*>(sBias + n);
        // exact mod 2^32: the true accumulator fits int32
        const uint32_t corr = 0u - (uint32_t)a.zw * (uint32_t)rowsum;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          int4 b = cst4[q];
          if (my_corr != nullptr) {
            const int4 t = reinterpret_cast<const int4*>(my_corr + n)[q];
            b.x += t.x; b.y += t.y; b.z += t.z; b.w += t.w;
          }
          const int bb[4] = {b.x, b.y, b.z, b.w};
          uint32_t word = 0;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int32_t acc = (int32_t)(v[4 * q + h] + (uint32_t)bb[h] + corr);
            word |= (uint32_t)requant_u8(acc, a.m0, a.shift, a.zo, a.qmin, a.qmax) << (8 * h);
          }
          w[q] = word;
        }
      }
      EP_ACC(2);
      if (use_tma) {
        // stage the 32 x 32 block as the TMA box (bf16: 64-byte rows with the
        // 64-byte swizzle, conflict-free row-per-lane writes; u8: dense
        // 32-byte rows) and let one lane store it; TMA clips rows >= P and
        // columns >= K.  Two buffers: wait until the store issued two chunks
        // ago has read its source.
        const uint32_t sb = smem_u32(stg) + (chunk_seq & 1) * (32 * kOutRowBytes);
        if (chunk_seq >= 2) {
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
        }
#ifndef ICV_EXP_EPI_NOSTS   // experiment: no staging writes (and no stores)
#pragma unroll
        for (int q = 0; q < kOutRowBytes / 16; ++q) {
          const int phys = kI8 ? q : (q ^ ((lane >> 1) & 3));
          sts128(sb + lane * kOutRowBytes + phys * 16, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
#ifndef ICV_EXP_EPI_NOSTORE   // experiment: staged, never stored
        fence_proxy_async_smem();
        __syncwarp();
        EP_ACC(3);
        if (lane == 0) {
          if constexpr (kRowTiles)   // (channel, pixel in the output row, output row); pixels >= Wo clipped
            tma_store_3d(tmap_y, sb, n, rt_ox0, rt_row);
          else
            tma_store_2d(tmap_y, sb, n, (int32_t)row0);
          bulk_commit_group();
        }
#endif
#else
        if (w[0] == 0x12345678u && w[15] == 0x9abcdef0u) sts128(sb, w[1], w[2], w[3], w[4]);   // keep the math
#endif
        ++chunk_seq;
        EP_ACC(4);
        if (ci + 1 < nchunks) {
          tmem_ld_wait_regs(vn);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = vn[i];
        }
        continue;
      }
      uint4* my = reinterpret_cast<uint4*>(stg + lane * kStageRowBytes);
#pragma unroll
      for (int q = 0; q < kOutRowBytes / 16; ++q) my[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      __syncwarp();
      constexpr int kChunks = kOutRowBytes / 16;  // 16-byte chunks per staged row
      constexpr int kRowsPerPass = 32 / kChunks;
      constexpr int eb = kI8 ? 1 : 2;
#pragma unroll
      for (int pass = 0; pass < 32 / kRowsPerPass; ++pass) {
        const int rr = pass * kRowsPerPass + lane / kChunks;
        const int q = lane % kChunks;
        const int64_t p = row0 + rr;
        if (kRowTiles ? rt_ox0 + rr < a.ow : p < a.P) {
          const uint4 val = *reinterpret_cast<const uint4*>(stg + rr * kStageRowBytes + q * 16);
          const int col = n + q * (16 / eb);
          uint8_t* dst = static_cast<uint8_t*>(a.y) + (p * a.K + col) * eb;
          if (vec_ok && col + 16 / eb <= a.K) *reinterpret_cast<uint4*>(dst) = val;
          else store_partial(dst, val, (a.K - col) * eb);   // ragged / misaligned rows only
        }
      }
      __syncwarp();
      if (ci + 1 < nchunks) {
        tmem_ld_wait_regs(vn);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = vn[i];
      }
    }
    }   // !done_wide
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {   // one arrival per epilogue warp (at the pair leader for a pair peer)
      if (tempty_remote) mbar_arrive_remote_relaxed(tempty_remote + as * 8);
      else mbar_arrive(&tempty[as]);
    }
#ifdef ICV_ROWS_TIMELINE
    if (ew == 0 && lane == 0 && ti < 24) g_icv_trace[blockIdx.x][80 + ti] = ({ unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); t_; });
#endif
#ifdef ICV_TRACE
    {
      const long long t = clock64();
      t_work += t - t_prev;
      t_prev = t;
    }
#endif
    if (ew == 0 && lane == 0 && ti_ < 8) TRACE(18 + ti_);
    if constexpr (kSubRows > 1) {
      if (++as == kAccStages) { as = 0; aphase ^= 1; }
    } else if constexpr (kTileGroups > 1) {
      static_assert(kAccStages % kTileGroups == 0, "groups must map to fixed accumulator stages");
      as += kTileGroups;
      if (as >= kAccStages) { as -= kAccStages; aphase ^= 1; }
    } else if (++as == kAccStages) {
      as = 0;
      aphase ^= 1;
    }
  }
  if (use_tma && lane == 0) bulk_wait_group<0>();   // output written before the CTA exits
#ifdef ICV_ROWS_PHASES
  if (ew == 0 && lane == 0)
    for (int i = 0; i < 6; ++i) g_icv_trace[blockIdx.x][42 + i] = (unsigned long long)_ep[i];
#endif
#ifdef ICV_TRACE
  if (ew == 0 && lane == 0) {
    g_icv_trace[blockIdx.x][28] = (unsigned long long)t_wait;
    g_icv_trace[blockIdx.x][29] = (unsigned long long)t_work;
  }
#endif
}

// ----------------------------------------------------------------------------
// Host side: TMA map of the packed filter rows (K-major, 128-byte column
// blocks, 128-byte swizzle) and the common argument block.
PFN_cuTensorMapEncodeTiled_v12000 get_tensor_map_encoder();
int make_filter_tmap(const ConvArgs& c, int block_n, int depth, CUtensorMap* tmap);
int make_input_tmap(const ConvArgs& c, CUtensorMap* tmap);
int make_input_tmap_im2col(const ConvArgs& c, CUtensorMap* tmap);
int make_output_tmap(const ConvArgs& c, CUtensorMap* tmap, bool wide = false);
void fill_tc_args(const ConvArgs& c, int block_n, TcArgs* a);
int sm_count();

}  // namespace icv
