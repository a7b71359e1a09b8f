// K2/K3/K6: the indirect-GEMM mainloop on sm_100a tensor cores.
//
// Replaces indirect_conv's hot loop (reference indirect.py:287-294) for
// bf16 (tcgen05 kind::f16, fp32 accumulate) and uint8 (kind::i8, s32
// accumulate) when pixel rows are 16-byte aligned.  GEMM view:
// M = output pixels, N = output channels, K = R*S taps x C channels.
//
// Persistent, warp-specialised CTA (one per SM, 288 threads):
//   warps 0-3  A producers.  Thread r owns row r of the 128-pixel M tile.
//              Per tap e it reads that pixel's row reference from the
//              indirection buffer (the paper's "load fresh row pointers per
//              kernel element", Listing 3), resolves ZERO_REF to the bound
//              zero row, and gathers the row's 128-byte channel block with
//              eight 16-byte cp.async into the stage's A tile in the
//              canonical 128B-swizzle K-major layout.  Completion is
//              signalled on the stage's mbarrier (cp.async.mbarrier.arrive
//              .noinc).  Thread 0 also issues the TMA load of the matching
//              128-byte column block of the packed filter (B operand).
//   warp 8     MMA issuer (one elected lane): 4 x tcgen05.mma (K = 32 bytes
//              each) per stage into a TMEM accumulator; tcgen05.commit frees
//              the smem stage and, after the last k-step, publishes the
//              accumulator.  For uint8 a second N=16 MMA against an all-ones
//              B tile accumulates the per-pixel input row sum needed by the
//              zero-point correction.
//   warps 4-7  epilogue: tcgen05.ld the accumulator (warp w reads TMEM lanes
//              32*(w%4)..), add the folded bias / zero-point constants, cast
//              to bf16 or requantize to uint8, store NHWC rows.  Two TMEM
//              accumulator stages let the epilogue of tile i overlap the
//              mainloop of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "icv_internal.h"
#include "requant.cuh"
#include "sm100_ptx.cuh"

namespace icv {
namespace {

#ifndef ICV_EPI_WARPS
#define ICV_EPI_WARPS 8
#endif
constexpr int kEpiWarps = ICV_EPI_WARPS;          // 4 or 8 (two column halves)
constexpr int kMmaWarp = 4 + kEpiWarps;
constexpr int kThreads = 32 * (kMmaWarp + 1);     // 4 producer warps + epilogue warps + 1 MMA warp
constexpr int kMaxBias = 2048;                    // output channels whose epilogue constants live in smem
constexpr int kBM = 128;
constexpr int kABytes = kBM * 128;  // one 128-byte K block per row

template <bool kI8, int BN>
struct Cfg {
  static constexpr int kBBytes = BN * 128;
  // One smem "slot" holds one 128-byte K block of A (128 rows) and of B
  // (BN rows).  A pipeline stage groups kKB slots behind one full/empty
  // mbarrier pair, so the MMA warp pays one barrier wait per kKB*4 MMAs:
  // a wait + issue round costs ~330 cycles, more than four N=128 MMAs take
  // (256 cycles), so narrow tiles batch two K blocks per stage.
  static constexpr int kKB = BN >= 256 ? 1 : 2;
  static constexpr int kSlotBytes = kABytes + kBBytes;
#ifndef ICV_SLOT_KB
#define ICV_SLOT_KB 192
#endif
  static constexpr int kSlotsRaw = (ICV_SLOT_KB * 1024) / kSlotBytes;
  static constexpr int kSlots = (kSlotsRaw > 8 ? 8 : kSlotsRaw) / kKB * kKB;
  static constexpr int kStages = kSlots / kKB;
  static constexpr int kOnesBytes = kI8 ? 16 * 128 : 0;
  static constexpr int kAccStride = kI8 ? 2 * BN : BN;  // TMEM columns per accumulator stage
  static constexpr int kTmemNeed = 2 * kAccStride;
  static constexpr uint32_t kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128
                                        : kTmemNeed <= 256 ? 256 : 512;
  // epilogue staging: per epilogue warp, 32 rows x 32 output columns, rows
  // padded to a 16-byte multiple that keeps the row-per-lane writes
  // bank-conflict free
  static constexpr int kOutRowBytes = kI8 ? 32 : 64;
  static constexpr int kStageRowBytes = kI8 ? 48 : 80;
  static constexpr int kEpiBytes = kEpiWarps * 32 * kStageRowBytes;
  static constexpr int kBiasBytes = 4 * kMaxBias;
  static constexpr int kBarBytes = 256;
  static constexpr int kSmemBytes =
      1024 /*align slack*/ + kSlots * kSlotBytes + kOnesBytes + kEpiBytes + kBiasBytes + kBarBytes;
  static_assert(kTmemNeed <= 512, "TMEM overflow");
  static_assert(kSmemBytes <= 232448, "shared memory overflow");
};

#ifdef ICV_STATS
// Debug-build timeline counters (per CTA): 0 producer empty-wait, 1 producer
// loop, 2 MMA full-wait, 3 MMA tmem-empty-wait, 4 MMA loop, 5 epilogue
// tmem-full-wait, 6 epilogue loop, 7 k-blocks.  Not compiled in release.
__device__ unsigned long long g_icv_stats[1024][8];
#define STAT_BEGIN(v) long long v = clock64()
#define STAT_ADD(slot, v) atomicAdd(&g_icv_stats[blockIdx.x][slot], (unsigned long long)(clock64() - (v)))
#define STAT_INC(slot) atomicAdd(&g_icv_stats[blockIdx.x][slot], 1ull)
#else
#define STAT_BEGIN(v)
#define STAT_ADD(slot, v)
#define STAT_INC(slot)
#endif

#ifdef ICV_TRACE
// Debug-build timeline: per CTA, globaltimer (ns) at kernel entry [0], after
// setup [1], MMA thread's last commit of tile i [2+i], epilogue thread 128's
// tmem-full wakeup of tile i [10+i] and release [18+i], producer 0 start of
// tile i [26+i] (i < 8).
__device__ unsigned long long g_icv_trace[1024][34];
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
  const void* bias;  // f32 (bf16) or int32 (u8) per padded output channel
  void* y;
  int32_t zw, zo, qmin, qmax, m0, shift;
  int32_t n_pad;
};

// First buffer entry of output pixel p (clamped to the last real pixel,
// indirect.py:111): ((p / mr) * RS) * mr + p % mr; tap e adds e * mr.
__device__ __forceinline__ int64_t first_entry(const TcArgs& a, int64_t tile_m, int row) {
  int64_t p = tile_m * kBM + row;
  p = p < a.P ? p : a.P - 1;
  const int64_t t = p / a.mr;
  return t * a.RS * a.mr + (p - t * a.mr);
}

template <typename IbT>
__device__ __forceinline__ int64_t load_ref(const TcArgs& a, int64_t ent) {
  return (int64_t)__ldg(static_cast<const IbT*>(a.ib) + ent);
}

template <bool kI8, int BN, typename IbT>
__global__ void __launch_bounds__(kThreads, 1) igemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                               const TcArgs a) {
  using C = Cfg<kI8, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::kSlots * kABytes;
  uint8_t* sOnes = sB + C::kSlots * C::kBBytes;
  uint8_t* sEpi = sOnes + C::kOnesBytes;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(sEpi + C::kEpiBytes);   // f32 or int32 per output channel
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + C::kEpiBytes + C::kBiasBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 128 + 1);  // 128 producer cp.async arrivals + 1 expect_tx arrival
      mbar_init(&empty[s], 1);       // tcgen05.commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);       // tcgen05.commit after the last k-step
      mbar_init(&tempty[s], 32 * kEpiWarps);   // every epilogue thread
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmap_b);
  }
  if constexpr (kI8) {
    // all-ones B tile (16 rows x 128 bytes) for the per-pixel row-sum MMA
    if (threadIdx.x >= 128 && threadIdx.x < 256) {
      reinterpret_cast<uint4*>(sOnes)[threadIdx.x - 128] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u,
                                                                      0x01010101u);
      fence_proxy_async_smem();
    }
  }
  // epilogue constants (bias / folded zero-point terms) for every padded
  // output channel, staged once per CTA
  for (int i = threadIdx.x; i < a.n_pad && i < kMaxBias; i += blockDim.x)
    sBias[i] = __ldg(static_cast<const uint32_t*>(a.bias) + i);
  if (warp == kMmaWarp) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);
  const int num_kb = a.RS * a.cblocks;
  const uint32_t sA_u32 = smem_u32(sA);
  const uint32_t sB_u32 = smem_u32(sB);

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    // Warp w gathers rows [32w, 32w+32) of the A tile.  Each lane loads the
    // row reference of ONE row per tap (lane l -> row 32w+l, one coalesced
    // read of the buffer); the references are then shuffled so that 8
    // consecutive lanes copy the 8 16-byte chunks of one row: every cp.async
    // instruction moves 4 whole 128-byte rows (full L2 lines), and every
    // row lands as 128 contiguous (swizzled) shared-memory bytes.
    const int chunk = lane & 7;
    const int sub = lane >> 3;
    int stage = 0;
    uint32_t phase = 0;
    STAT_BEGIN(tloop);
    int64_t tile = blockIdx.x;
    int64_t ent0 = tile < a.total_tiles ? first_entry(a, tile / a.n_tiles, warp * 32 + lane) : 0;
    int64_t off_next = tile < a.total_tiles ? load_ref<IbT>(a, ent0) : 0;
    for (int ti = 0; tile < a.total_tiles; tile += gridDim.x, ++ti) {
      if (threadIdx.x == 0 && ti < 8) TRACE(26 + ti);
      const int nt = (int)(tile % a.n_tiles);
      const int64_t next_tile = tile + gridDim.x;
      int kb = 0;
      for (int e = 0; e < a.RS; ++e) {
        const int64_t off_own = off_next;
        // prefetch the next tap's reference (or the next tile's first tap)
        if (e + 1 < a.RS) {
          off_next = load_ref<IbT>(a, ent0 + (int64_t)(e + 1) * a.mr);
        } else if (next_tile < a.total_tiles) {
          ent0 = first_entry(a, next_tile / a.n_tiles, warp * 32 + lane);
          off_next = load_ref<IbT>(a, ent0);
        }
        const uint8_t* src[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t off = __shfl_sync(0xffffffffu, off_own, 4 * i + sub);
          src[i] = off < 0 ? a.zero_row : a.x + off * a.elem_bytes;      // ZERO_REF -> bound zero row
        }
        for (int cb = 0; cb < a.cblocks; ++cb, ++kb) {
          const int j = kb % C::kKB;                       // slot within the stage
          if (j == 0) {
            STAT_BEGIN(tw);
            mbar_wait(&empty[stage], phase ^ 1);
            if (threadIdx.x == 0) {
              STAT_ADD(0, tw);
              const int nsub = min(C::kKB, num_kb - kb);
              mbar_arrive_expect_tx(&full[stage], nsub * C::kBBytes);
            }
          }
          const int slot = stage * C::kKB + j;
          if (threadIdx.x == 0)
            tma_load_2d(sB_u32 + slot * C::kBBytes, &tmap_b, &full[stage], kb * 128, nt * BN);
          const int b = cb * 128 + chunk * 16;
          int valid = a.c_bytes - b;
          valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
          const uint32_t dst0 = sA_u32 + slot * kABytes;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = warp * 32 + 4 * i + sub;
            cp_async_16(dst0 + row * 128 + ((chunk ^ (row & 7)) << 4), src[i] + (valid ? b : 0), (uint32_t)valid);
          }
          if (j == C::kKB - 1 || kb == num_kb - 1) {
            cp_async_mbar_arrive_noinc(&full[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
    if (threadIdx.x == 0) STAT_ADD(1, tloop);
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (so stage/descriptor values are
    // warp-uniform and live in uniform registers); one elected lane issues
    // the tcgen05.mma / tcgen05.commit instructions.
    constexpr uint32_t idesc = make_idesc<kI8>(kBM, BN);
    constexpr uint32_t idesc_ones = make_idesc<kI8>(kBM, 16);
    const uint64_t ones_desc = sw128_kmajor_desc(smem_u32(sOnes));
    const int stages_per_tile = (num_kb + C::kKB - 1) / C::kKB;
    int stage = 0;
    uint32_t phase = 0;
    int as = 0;
    uint32_t aphase = 0;
    STAT_BEGIN(mloop);
    for (int64_t tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
      STAT_BEGIN(mw);
      mbar_wait(&tempty[as], aphase ^ 1);
      if (lane == 0) STAT_ADD(3, mw);
      tc_fence_after();
      const uint32_t d = tmem_base + as * C::kAccStride;
      for (int si = 0; si < stages_per_tile; ++si) {
        const int nsub = min(C::kKB, num_kb - si * C::kKB);
        STAT_BEGIN(fw);
        mbar_wait(&full[stage], phase);
        if (lane == 0) { STAT_ADD(2, fw); STAT_INC(7); }
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < nsub; ++j) {
            const int slot = stage * C::kKB + j;
            const uint64_t adesc = sw128_kmajor_desc(sA_u32 + slot * kABytes);
            const uint64_t bdesc = sw128_kmajor_desc(sB_u32 + slot * C::kBBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x 32-byte K steps per 128-byte block
              const uint32_t acc = (si | j | k) != 0;
              tc_mma<kI8>(d, adesc + 2 * k, bdesc + 2 * k, idesc, acc);
              if constexpr (kI8) tc_mma<true>(d + BN, adesc + 2 * k, ones_desc + 2 * k, idesc_ones, acc);
            }
          }
          tc_commit(&empty[stage]);
          if (si == stages_per_tile - 1) tc_commit(&tfull[as]);
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) {
        const int ti = (int)((tile - blockIdx.x) / gridDim.x);
        if (ti < 8) TRACE(2 + ti);
      }
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
    if (lane == 0) STAT_ADD(4, mloop);
  } else {
    // ------------------------------------------------------------ epilogue
    // Epilogue warp e reads TMEM lanes 32*(e%4).. (its 32 rows; the lane
    // quarter a warp may access is fixed by warp_id % 4) and, with 8
    // epilogue warps, one half of the tile's columns.  32 columns per
    // tcgen05.ld; the next chunk's load is in flight while the current one
    // is converted.  Finished values go through a per-warp staging buffer
    // so global stores are row-contiguous (16-byte chunks, whole rows).
    const int ew = warp - 4;
    const int slot = ew & 3;
    constexpr int kColGroups = kEpiWarps / 4;
    constexpr int kColsPerWarp = BN / kColGroups;
    const int col0 = (ew / 4) * kColsPerWarp;
    uint8_t* stg = sEpi + ew * 32 * C::kStageRowBytes;
    const bool vec_ok = kI8 ? (a.K & 15) == 0 : (a.K & 7) == 0;
    int as = 0;
    uint32_t aphase = 0;
    STAT_BEGIN(eloop);
    for (int64_t tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
      const int64_t mt = tile / a.n_tiles;
      const int nt = (int)(tile - mt * a.n_tiles);
      STAT_BEGIN(ewt);
      mbar_wait(&tfull[as], aphase);
      if (threadIdx.x == 128) STAT_ADD(5, ewt);
      const int ti_ = (int)((tile - blockIdx.x) / gridDim.x);
      if (threadIdx.x == 128 && ti_ < 8) TRACE(10 + ti_);
      tc_fence_after();
      const int64_t row0 = mt * kBM + slot * 32;  // first pixel of this warp's rows
      const uint32_t taddr = tmem_base + ((uint32_t)(slot * 32) << 16) + as * C::kAccStride;
      int32_t rowsum = 0;
      if constexpr (kI8) {
        uint32_t rs;
        tmem_ld_32x32b_x1(taddr + BN, rs);
        tmem_ld_wait();
        rowsum = (int32_t)rs;
      }
      const int nchunks = min(kColsPerWarp, a.K - nt * BN - col0) > 0
                              ? (min(kColsPerWarp, a.K - nt * BN - col0) + 31) / 32 : 0;
      uint32_t v[32];
      if (nchunks > 0) {
        tmem_ld_32x32b_x32(taddr + col0, v);
        tmem_ld_wait_regs(v);
      }
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
          const long long corr = -(long long)a.zw * rowsum;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int4 b = cst4[q];
            const int bb[4] = {b.x, b.y, b.z, b.w};
            uint32_t word = 0;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int32_t acc = (int32_t)((long long)(int32_t)v[4 * q + h] + bb[h] + corr);
              word |= (uint32_t)requant_u8(acc, a.m0, a.shift, a.zo, a.qmin, a.qmax) << (8 * h);
            }
            w[q] = word;
          }
        }
        // stage: lane = row
        uint4* my = reinterpret_cast<uint4*>(stg + lane * C::kStageRowBytes);
#pragma unroll
        for (int q = 0; q < C::kOutRowBytes / 16; ++q) my[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        __syncwarp();
        // write out: lanes cover (row, 16-byte chunk) pairs
        constexpr int kChunks = C::kOutRowBytes / 16;      // 4 (bf16) or 2 (u8) chunks per row
        constexpr int kRowsPerPass = 32 / kChunks;
        constexpr int eb = kI8 ? 1 : 2;
#pragma unroll
        for (int pass = 0; pass < 32 / kRowsPerPass; ++pass) {
          const int rr = pass * kRowsPerPass + lane / kChunks;
          const int q = lane % kChunks;
          const int64_t p = row0 + rr;
          if (p < a.P) {
            const uint4 val = *reinterpret_cast<const uint4*>(stg + rr * C::kStageRowBytes + q * 16);
            const int col = n + q * (16 / eb);
            uint8_t* dst = static_cast<uint8_t*>(a.y) + (p * a.K + col) * eb;
            if (vec_ok && col + 16 / eb <= a.K) {
              *reinterpret_cast<uint4*>(dst) = val;
            } else {
              const uint8_t* bytes = reinterpret_cast<const uint8_t*>(&val);
              for (int j = 0; j < 16 / eb; ++j)
                if (col + j < a.K)
                  for (int t = 0; t < eb; ++t) dst[j * eb + t] = bytes[j * eb + t];
            }
          }
        }
        __syncwarp();
        if (ci + 1 < nchunks) {
          tmem_ld_wait_regs(vn);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = vn[i];
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[as]);
      if (threadIdx.x == 128 && ti_ < 8) TRACE(18 + ti_);
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
    if (threadIdx.x == 128) STAT_ADD(6, eloop);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

template <bool kI8, int BN, typename IbT>
int launch_tc(const ConvArgs& c, cudaStream_t st) {
  using Cf = Cfg<kI8, BN>;
  auto kernel = igemm_tc_kernel<kI8, BN, IbT>;
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [&] {
    attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return cuda_check(attr_err, "cudaFuncSetAttribute(smem)");

  auto encode = get_encode();
  if (!encode) return fail(ICV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)c.L.row_bytes, (cuuint64_t)c.L.n_pad};
  const cuuint64_t strides[1] = {(cuuint64_t)c.L.row_bytes};
  const cuuint32_t box[2] = {128, (cuuint32_t)BN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(c.packed + c.L.w_off), dims,
                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(ICV_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));

  TcArgs a;
  a.x = static_cast<const uint8_t*>(c.x);
  a.zero_row = static_cast<const uint8_t*>(c.zero_row);
  a.ib = c.ib;
  a.mr = c.mr;
  a.P = c.P;
  a.RS = c.g.RS();
  a.elem_bytes = kI8 ? 1 : 2;
  a.c_bytes = c.g.C * a.elem_bytes;
  a.cblocks = c.L.cblocks;
  a.K = c.g.K;
  a.n_tiles = c.L.n_pad / BN;
  const int64_t m_tiles = (c.P + kBM - 1) / kBM;
  a.total_tiles = m_tiles * a.n_tiles;
  a.bias = c.packed + c.L.bias_off;
  a.y = c.y;
  a.zw = c.zw; a.zo = c.zo; a.qmin = c.qmin; a.qmax = c.qmax; a.m0 = c.m0; a.shift = c.shift;
  a.n_pad = c.L.n_pad;
  if (c.L.n_pad > kMaxBias) return fail(ICV_ERR_UNSUPPORTED, "more than 2048 output channels");

  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(a.total_tiles < sms ? a.total_tiles : sms);
  kernel<<<grid, kThreads, Cf::kSmemBytes, st>>>(tmap, a);
  note_launch();
  return cuda_check(cudaGetLastError(), "igemm_tc launch");
}

template <typename IbT>
int dispatch_bn(const ConvArgs& c, int bn, cudaStream_t st) {
  if (c.L.family == kFamTcBf16) {
    if (bn == 64) return launch_tc<false, 64, IbT>(c, st);
    if (bn == 128) return launch_tc<false, 128, IbT>(c, st);
    if (bn == 256) return launch_tc<false, 256, IbT>(c, st);
  } else if (c.L.family == kFamTcU8) {
    if (bn == 64) return launch_tc<true, 64, IbT>(c, st);
    if (bn == 128) return launch_tc<true, 128, IbT>(c, st);
  }
  return fail(ICV_ERR_UNSUPPORTED, "no tensor-core kernel for this tile width");
}

}  // namespace

#ifdef ICV_TRACE
extern "C" ICV_API int icv_debug_trace(unsigned long long* host, int reset) {
  if (host && cudaMemcpyFromSymbol(host, g_icv_trace, sizeof(g_icv_trace)) != cudaSuccess) return ICV_ERR_CUDA;
  if (reset) {
    static unsigned long long zeros[1024][34];
    if (cudaMemcpyToSymbol(g_icv_trace, zeros, sizeof(zeros)) != cudaSuccess) return ICV_ERR_CUDA;
  }
  return ICV_OK;
}
#endif

#ifdef ICV_STATS
extern "C" ICV_API int icv_debug_stats(unsigned long long* host, int reset) {
  if (host && cudaMemcpyFromSymbol(host, g_icv_stats, sizeof(g_icv_stats)) != cudaSuccess) return ICV_ERR_CUDA;
  if (reset) {
    static unsigned long long zeros[1024][8];
    if (cudaMemcpyToSymbol(g_icv_stats, zeros, sizeof(zeros)) != cudaSuccess) return ICV_ERR_CUDA;
  }
  return ICV_OK;
}
#endif

int launch_conv_tc(const ConvArgs& c, cudaStream_t st) {
  const int bn = c.L.block_n;
  if (c.ib_is_i32) return dispatch_bn<int32_t>(c, bn, st);
  return dispatch_bn<int64_t>(c, bn, st);
}

}  // namespace icv
