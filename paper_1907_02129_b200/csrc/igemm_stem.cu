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
constexpr int kStagesStem = 2;          // A tiles in flight
constexpr int kWinBufs = 3;             // input windows in flight (tile k assembling, k+1 landing, k+2 issued)

template <int C, int RS, int BN>
struct CfgStem {
  static constexpr int kK = RS * C;                         // real reduction length
  static constexpr int kKSteps = (kK + 15) / 16;            // MMA K steps (16 bf16 each)
  static constexpr int kBlocks = (kKSteps * 16 + 63) / 64;  // 128-byte K blocks per row
  static constexpr int kABytes = kBM * kBlocks * 128;       // one A tile
  static constexpr int kBBytes = BN * kBlocks * 128;        // resident filter
  static constexpr int kEpiBytes = kEpiWarpsStem * 32 * 80;
  // Taps are assembled in groups of 8: 8 taps x C elements = C whole 16-byte
  // chunks of the A row.  kGroups groups cover the kKSteps*16 elements the
  // MMA reads (taps past R*S read a zero slot); the two producer halves take
  // groups [0, kG0) and [kG0, kGroups).
  static constexpr int kGroups = (kKSteps * 2 + C - 1) / C;
  static constexpr int kG0 = (kGroups + 1) / 2;
  static constexpr int kTapsHalf = kG0 * 8;                 // taps per producer thread (max)
  static constexpr int kTaps = kGroups * 8;
  // elements per staged input window: 16 KB of bf16 (8 KB when a 128-wide
  // resident filter leaves less room); two 8-element slots follow it: the
  // bound zero row (ZERO_REF taps) and true zeros (taps past R*S)
  static constexpr int kWinElems = (BN <= 64 || RS * C <= 64) ? 8192 : 4096;
  static constexpr int kWinBytes = kWinElems * 2 + 32;
  static constexpr int kRelBytes = kTaps * kBM * 2;         // [kTaps/2][128][2] uint16 window indices
  static constexpr int kMiscBytes = 1024;                   // bias, reductions, window bases
  static constexpr int kSmemBytes = 1024 + kStagesStem * kABytes + kBBytes + kEpiBytes + kWinBufs * kWinBytes +
                                    kWinBufs * kRelBytes + kMiscBytes + 256;
  static_assert(kSmemBytes <= 232448, "shared memory overflow");
  static_assert(C >= 1 && C <= 4, "channel-poor kernel handles 1..4 channels");
  static_assert(kGroups * C * 8 <= kBlocks * 64, "tap groups overflow the A row");
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
  for (int j = 0; j < C; ++j)
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a_chunk_addr(tileA, row, g * C + j)),
                 "r"(w[4 * j]), "r"(w[4 * j + 1]), "r"(w[4 * j + 2]), "r"(w[4 * j + 3]) : "memory");
}

template <int C, int RS, int BN, typename IbT>
__global__ void __launch_bounds__(kThreadsStem, 1) igemm_stem_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                                     const TcArgs a, int32_t x_elems) {
  using Cf = CfgStem<C, RS, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStagesStem * Cf::kABytes;
  uint8_t* sEpi = sB + Cf::kBBytes;
  uint8_t* sWin = sEpi + Cf::kEpiBytes;                              // [3] windows (+ zero slots)
  uint8_t* sRel = sWin + kWinBufs * Cf::kWinBytes;                   // [3][kTaps/2][128][2] uint16
  uint8_t* sMisc = sRel + kWinBufs * Cf::kRelBytes;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(sMisc);                         // 128 x 4 B
  int32_t* sRed = reinterpret_cast<int32_t*>(sMisc + 512);                      // [3][2][8] min/max per warp
  int32_t* sWinLo = reinterpret_cast<int32_t*>(sMisc + 512 + 192);              // [3] window start (or -1)
  uint64_t* full = reinterpret_cast<uint64_t*>(sMisc + Cf::kMiscBytes);
  uint64_t* empty = full + kStagesStem;
  uint64_t* tfull = empty + kStagesStem;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesStem; ++s) {
      mbar_init(&full[s], kProdThreads);   // every producer thread (st.shared + proxy fence + arrive)
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 32 * kEpiWarpsStem);
    }
    mbar_init(bfull, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmap_b);
  }
  for (int i = threadIdx.x; i < a.n_pad; i += blockDim.x) sBias[i] = __ldg(static_cast<const uint32_t*>(a.bias) + i);
  if (threadIdx.x < kWinBufs * 8) {   // zero slots behind every window: bound zero row, then true zeros
    const int b = threadIdx.x >> 3, j = threadIdx.x & 7;
    const uint16_t* z = reinterpret_cast<const uint16_t*>(a.zero_row);
    uint16_t* slot = reinterpret_cast<uint16_t*>(sWin + b * Cf::kWinBytes) + Cf::kWinElems;
    slot[j] = j < C ? __ldg(z + j) : (uint16_t)0;
    slot[8 + j] = 0;
  }
  if (warp == kMmaWarpStem) tmem_alloc<(2 * BN <= 128 ? 128 : 256)>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t sA_u32 = smem_u32(sA);
  const uint32_t sB_u32 = smem_u32(sB);

  if (threadIdx.x == 0) {   // resident filter: one TMA box per 128-byte K block
    mbar_arrive_expect_tx(bfull, Cf::kBBytes);
    for (int b = 0; b < Cf::kBlocks; ++b) tma_load_2d(sB_u32 + b * BN * 128, &tmap_b, bfull, b * 128, 0);
  }

  if (warp < kProdWarpsStem) {
    // ------------------------------------------------------------ producers
    // Thread (half, row) assembles half of A row `row` (one output pixel).
    // Per tile, the row references of its 128 pixels (indirection buffer)
    // bound the span of input elements the tile reads; that span (the
    // "window") is copied into smem with coalesced 16-byte cp.async two
    // tiles ahead, the references become 16-bit window indices, and rows are
    // assembled from the window with shared-memory loads.  A window larger
    // than the buffer (never for the ResNet stem) falls back to reading the
    // taps straight from global memory.
    const int half = warp >> 2;
    const int row = threadIdx.x & (kBM - 1);
    const int g_begin = half ? Cf::kG0 : 0;
    const int g_end = half ? Cf::kGroups : Cf::kG0;
    const int e_begin = g_begin * 8;
    const int n_taps = (g_end - g_begin) * 8;
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(a.x);
    const uint32_t sWin_u32 = smem_u32(sWin);
    const uint32_t sRel_u32 = smem_u32(sRel);
    const int64_t my_tiles = blockIdx.x < a.total_tiles ? (a.total_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    constexpr int32_t kPad = -2;        // tap past R*S
    int32_t ref[Cf::kTapsHalf];         // resolved element offsets (ZERO_REF = -1, padding = -2)

    auto load_refs = [&](int64_t k) {   // row references of local tile k -> registers
      if (k >= my_tiles) return;
      const RowRef rr = row_ref(a, blockIdx.x + k * gridDim.x, row);
      const IbT* ib = static_cast<const IbT*>(a.ib) + rr.ent0 + (int64_t)e_begin * a.mr;
      const int32_t base = (int32_t)rr.base;
#pragma unroll
      for (int i = 0; i < Cf::kTapsHalf; ++i) {
        if (i < n_taps && e_begin + i < RS) {
          const int32_t raw = (int32_t)__ldg(ib + (int64_t)i * a.mr);
          ref[i] = raw + (base & ~(raw >> 31));          // ZERO_REF (-1) stays -1
        } else {
          ref[i] = kPad;
        }
      }
    };
    // window of local tile k: CTA-wide min/max of the valid offsets, window
    // indices -> sRel, 16-byte cp.async copies -> sWin
    auto prepare = [&](int64_t k) {
      const int buf = (int)(k % kWinBufs);
      if (k < my_tiles) {
        uint32_t lo = 0xFFFFFFFFu;
        int32_t hi = -1;
#pragma unroll
        for (int i = 0; i < Cf::kTapsHalf; ++i) {
          lo = min(lo, ref[i] >= 0 ? (uint32_t)ref[i] : 0xFFFFFFFFu);
          hi = max(hi, ref[i]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) { sRed[buf * 16 + warp] = (int32_t)lo; sRed[buf * 16 + 8 + warp] = hi; }
      }
      named_bar_sync(1, kProdThreads);
      if (k < my_tiles) {
        uint32_t lo = 0xFFFFFFFFu;
        int32_t hi = -1;
#pragma unroll
        for (int i = 0; i < kProdWarpsStem; ++i) {
          lo = min(lo, (uint32_t)sRed[buf * 16 + i]);
          hi = max(hi, sRed[buf * 16 + 8 + i]);
        }
        const int32_t w0 = hi < 0 ? 0 : (int32_t)(lo & ~7u);        // 16-byte aligned start
        const int32_t w1 = hi < 0 ? 0 : ((hi + C + 7) & ~7);          // covers the last reference's C elements
        const bool fits = w1 - w0 <= Cf::kWinElems;
        if (threadIdx.x == 0) sWinLo[buf] = fits ? w0 : -1;
        const uint32_t rel_base = sRel_u32 + buf * Cf::kRelBytes + ((g_begin * 4) * kBM + row) * 4;
#pragma unroll
        for (int i = 0; i < Cf::kTapsHalf; i += 2) {
          if (i < n_taps) {
            uint32_t r2 = 0;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int32_t r = ref[i + j];
              const uint32_t rel = r >= 0 ? (uint32_t)(r - w0) : (r == -1 ? Cf::kWinElems : Cf::kWinElems + 8);
              r2 |= rel << (16 * j);
            }
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(rel_base + (i / 2) * kBM * 4), "r"(r2) : "memory");
          }
        }
        if (fits) {
          const uint32_t dst = sWin_u32 + buf * Cf::kWinBytes;
          for (int32_t ch = threadIdx.x; ch * 8 < w1 - w0; ch += kProdThreads) {
            const int32_t e0 = w0 + ch * 8;
            int32_t valid = (x_elems - e0) * 2;
            valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
            cp_async_16(dst + (uint32_t)ch * 16, a.x + (valid ? (int64_t)e0 * 2 : 0), (uint32_t)valid);
          }
        }
      }
      cp_async_commit();
    };

    // prologue: windows of tiles 0 and 1
    load_refs(0);
    prepare(0);
    load_refs(1);
    prepare(1);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t k = 0; k < my_tiles; ++k) {
      load_refs(k + 2);                       // lands while tile k is assembled
      asm volatile("cp.async.wait_group 1;" ::: "memory");   // window k (window k+1 may still fly)
      named_bar_sync(1, kProdThreads);
      const int buf = (int)(k % kWinBufs);
      const bool in_window = sWinLo[buf] >= 0;
      mbar_wait(&empty[stage], phase ^ 1);
      const uint32_t tileA = sA_u32 + stage * Cf::kABytes;
      if (in_window) {
        const uint32_t win = sWin_u32 + buf * Cf::kWinBytes;
        const uint32_t rel_base = sRel_u32 + buf * Cf::kRelBytes + row * 4;
#pragma unroll 1
        for (int g = g_begin; g < g_end; ++g) {
          uint32_t w[4 * C];
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const uint32_t r2 = lds32(rel_base + (g * 4 + i / 2) * kBM * 4);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint32_t rel = j ? r2 >> 16 : r2 & 0xFFFFu;
              const uint32_t addr = win + ((rel * 2) & ~3u);
              const uint32_t sh = (rel & 1) * 16;
              const uint32_t lo = lds32(addr), hi = lds32(addr + 4);
              place_tap<C>(w, i + j, __funnelshift_r(lo, hi, sh), hi >> sh);
            }
          }
          store_group<C>(w, tileA, row, g);
        }
      } else {
        // window too large: read the taps from global memory
        const RowRef rr = row_ref(a, blockIdx.x + k * gridDim.x, row);
        const IbT* ib = static_cast<const IbT*>(a.ib) + rr.ent0;
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
                const uint32_t* z = reinterpret_cast<const uint32_t*>(sWin + buf * Cf::kWinBytes) + Cf::kWinElems / 2;
                lo = z[0];
                hi = z[1];
              }
            }
            place_tap<C>(w, i, lo, hi);
          }
          store_group<C>(w, tileA, row, g);
        }
      }
      fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
      mbar_arrive(&full[stage]);
      if (++stage == kStagesStem) { stage = 0; phase ^= 1; }
      prepare(k + 2);              // every producer finished reading window k+2's buffer (tile k-1)
    }
  } else if (warp == kMmaWarpStem) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc<false>(kBM, BN);
    mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int as = 0;
    uint32_t aphase = 0;
    for (int64_t tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[as], aphase ^ 1);
      mbar_wait(&full[stage], phase);
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
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
  } else {
    epilogue_loop<false, BN, kEpiWarpsStem, BN>(a, warp - kProdWarpsStem, lane, tmem_base, sEpi, sBias, tfull, tempty);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarpStem) {
    tc_fence_after();
    tmem_dealloc<(2 * BN <= 128 ? 128 : 256)>(tmem_base);
  }
}

template <int C, int RS, int BN, typename IbT>
int launch_stem_t(const ConvArgs& c, cudaStream_t st) {
  using Cf = CfgStem<C, RS, BN>;
  const int64_t x_elems = c.g.N * c.g.H * c.g.W * (int64_t)c.g.C;
  if (x_elems >= (int64_t(1) << 31)) return fail(ICV_ERR_UNSUPPORTED, "stem kernel: input too large");
  auto kernel = igemm_stem_kernel<C, RS, BN, IbT>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [&] {
    err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmemBytes);
  });
  if (err != cudaSuccess) return cuda_check(err, "cudaFuncSetAttribute(stem smem)");
  CUtensorMap tmap;
  if (int s = make_filter_tmap(c, BN, &tmap)) return s;
  TcArgs a;
  fill_tc_args(c, BN, &a);
  const int sms = sm_count();
  const int grid = (int)(a.total_tiles < sms ? a.total_tiles : sms);
  kernel<<<grid, kThreadsStem, Cf::kSmemBytes, st>>>(tmap, a, (int32_t)x_elems);
  note_launch();
  return cuda_check(cudaGetLastError(), "igemm_stem launch");
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
  if (c.ib_is_i32) return dispatch_stem<int32_t>(c, st);
  return dispatch_stem<int64_t>(c, st);
}

}  // namespace icv
