// K2/K3: indirect-GEMM mainloop on sm_100a tensor cores, A operand staged in
// SHARED memory ("kernel S", the IB-gather kernel).
//
// Replaces indirect_conv's hot loop (reference indirect.py:287-294).  GEMM
// view: M = output pixels, N = output channels, K = R*S taps x C channels.
// Persistent, warp-specialised CTA (one per SM):
//   warps 0-3  A producers.  The CTA's slice of the indirection buffer for
//              its next tile (128 pixels x R*S taps, tile-major / tap / lane,
//              indirect.py:14-16) is copied into smem by cp.async one tile
//              ahead, so reading the row references never stalls the gather.
//              Per tap the warp reads the references of its 32 rows (the
//              paper's "load fresh row pointers per kernel element",
//              Listing 3), resolves ZERO_REF to the bound zero row, and
//              gathers 4 whole 128-byte rows per cp.async instruction (8
//              lanes per row) into the slot's A tile in the canonical
//              128B-swizzle K-major layout.  Thread 0 also TMA-loads the
//              matching packed-filter block (B).
//   warps 4-7  epilogue (igemm_common.cuh).
//   warp 8     MMA: one elected lane issues 4 x tcgen05.mma per 128-byte K
//              block into a TMEM accumulator (uint8: 16 all-ones rows behind
//              the filter rows of every B block make the same MMA, N = BN + 16,
//              produce the per-pixel input row sums of the zero-point
//              correction); tcgen05.commit releases smem stages and publishes
//              finished accumulators.
//
// The same kernel runs two TMA-fed plans over a canonical buffer (IbT =
// DenseA: no index slices, the producer warps' lane 0 issue tile loads):
//   dense   1x1 stride-1 unpadded layers: the A tile is 128 consecutive pixel
//           rows, one 2-D box per channel block;
//   im2col  any geometry with an all-zero (uint8: zero-point) zero row: one
//           im2col tile load per (tap, channel block), the TMA unit walks the
//           128 output pixels and zero-fills padded taps (uint8: corrected per
//           border class in the epilogue);
// both also on CTA pairs (cta_group::2, M = 256: each member loads its own A
// rows and half of every filter block, every load completes on the leader's
// barrier).  Opt-in: uint8 BLOCK_N 256 with row-sum warps (knob u8_bn).
#include <cstdio>
#include <cstdlib>

#include "igemm_common.cuh"

namespace icv {

#if defined(ICV_TRACE) || defined(ICV_STEM_PHASES) || defined(ICV_ROWS_PHASES) || defined(ICV_ROWS_TIMELINE)
__device__ unsigned long long g_icv_trace[1024][128];
#endif

namespace {

// Epilogue warps: 8 for uint8 (the q31 requantization is the heavier
// epilogue; measured 47 -> 41 us on cfg4), 4 for bf16 (8 measured slower).
// Output-heavy bf16 layers (K >= 4 C: the ResNet-50 1x1 expansions) run 8
// (s1b1_1x1b 131 -> 102 us, s2 1x1b 78 -> 63 us; the 1x1 reductions and
// strided 3x3s measured 4-8 us slower with 8).
template <bool kI8>
constexpr int kEpiWarpsS = kI8 ? 8 : 4;
// Gather (producer) warps: each covers 128 / kProdWarpsS A rows.
#ifndef ICV_PROD_WARPS_BF16
#define ICV_PROD_WARPS_BF16 4   // 8 measured equal on cfg2 / cfg3b (the fill is L2->SM bound, not issue bound)
#endif
#ifndef ICV_PROD_WARPS_U8
#define ICV_PROD_WARPS_U8 4
#endif
template <bool kI8>
constexpr int kProdWarpsS = kI8 ? ICV_PROD_WARPS_U8 : ICV_PROD_WARPS_BF16;
template <bool kI8, int kEpiW = kEpiWarpsS<kI8>>
constexpr int kMmaWarpS = kProdWarpsS<kI8> + kEpiW;
template <bool kI8, int kEpiW = kEpiWarpsS<kI8>>
constexpr int kThreadsS = 32 * (kMmaWarpS<kI8, kEpiW> + 1);

// Index type tag of the dense-A instantiation (no indirection buffer read:
// the A tile is TMA-loaded as 128 consecutive pixel rows; dense_a_eligible).
struct DenseA {};
template <typename IbT>
constexpr bool kIsDense = std::is_same<IbT, DenseA>::value;

template <bool kI8, int BN, int kPair = 1, int kEpiW = kEpiWarpsS<kI8>, bool kDense = false>
struct CfgS {
  // uint8 row sums (the zero-point correction needs sum_k x[p][k] per output
  // pixel): 16 all-ones rows sit behind the BN filter rows of every B block
  // in smem and the MMA runs N = BN + 16 -- tcgen05 time is linear in N (72
  // vs 64 cycles at N 144 / 128, tools/micro/mma_rate.cu), while a separate
  // N = 16 MMA per K step costs its 45-cycle floor (107 cycles per pair).
  // CTA pairs and BN 256 (N <= 256) keep the separate ones tile.
  static constexpr bool kFuseOnes = kI8 && kPair == 1 && BN + 16 <= 256;
  // bytes one K block of the filter tile occupies in smem / brings in by TMA
  // (a CTA pair splits the BN rows)
  static constexpr int kBLoadBytes = BN * 128 / kPair;
  static constexpr int kBBytes = kBLoadBytes + (kFuseOnes ? 16 * 128 : 0);
  // One smem slot = one 128-byte K block of A (128 rows) and of B (BN rows).
  // A stage groups kKB slots behind one full/empty barrier pair so the MMA
  // warp pays one barrier round trip per kKB*4 MMAs.
#ifndef ICV_KKB
#define ICV_KKB 2
#endif
  // (dense A: one K block per stage -- 1x1 layers have few K blocks per
  // tile, and the stages then run straight across tile boundaries)
  // (fused ones rows: one TMA box per K block, and the larger slots would
  // leave only two 2-block stages)
  static constexpr int kKB = (kDense || BN >= 256 || kFuseOnes) ? 1 : ICV_KKB;
  static constexpr int kSlotBytes = kABytes + kBBytes;
#ifndef ICV_MAX_SLOTS
#define ICV_MAX_SLOTS 8
#endif
  static constexpr int kMaxSlots = kDense ? 12 : ICV_MAX_SLOTS;
  // BN 256 (single CTA): two 256-column accumulators fill TMEM, so the row
  // sums are computed by four extra warps that read each full A stage from
  // shared memory (one row per thread, dp4a) and hand the per-tile sums to
  // the epilogue through smem ([2][128] int32 in the ones-tile region).
  static constexpr int kSumWarps = (kI8 && !kFuseOnes && kPair == 1) ? 4 : 0;
  static constexpr int kOnesBytes = kSumWarps ? 2 * kBM * 4 : (kI8 && !kFuseOnes) ? 16 * 128 : 0;
  // TMEM columns per accumulator stage (uint8: row sums at +BN; BN = 256
  // keeps 32 columns for them and runs one accumulator stage)
  static constexpr int kAccStride = kI8 ? (kSumWarps ? BN : BN == 256 ? BN + 32 : 2 * BN) : BN;
  static constexpr int kAccStages = 2 * kAccStride <= 512 ? 2 : 1;
  static constexpr int kTmemNeed = kAccStages * kAccStride;
  static constexpr uint32_t kTmemCols = kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
  static constexpr int kEpiBytes = kEpiW * kEpiWarpBytes<kI8>;
  static constexpr int kBarBytes = 256;
  static_assert(kTmemNeed <= 512, "TMEM overflow");
};

// Runtime shared-memory plan of kernel S: the ring gets whatever the index
// slices, epilogue staging and constants leave of the 227 KB.
struct PlanS {
  int slots, stages;
  int off_b, off_ones, off_epi, off_bias, off_ib, off_corr, off_bar, bytes;
  int res_b;   // dense A: filter blocks of this CTA's N tile kept resident (0 = streamed per stage)
};

// Border classes of a layer's output pixels (igemm_common.cuh border_class):
// rows / columns whose receptive field leaves the image at the top (left) or
// bottom (right) are one class each, the interior one class.
struct BorderClasses {
  int ncls, tb, ohb, nr, lb, owb, ncc;
};
bool im2col_u8_classes(const ConvArgs& c, BorderClasses* b);

template <bool kI8, int BN, typename IbT, int kPair = 1, int kEpiW = kEpiWarpsS<kI8>>
bool plan_smem(int rs, int n_pad, PlanS* p, int res_kb = 0, int corr_bytes = 0) {
  using C = CfgS<kI8, BN, kPair, kEpiW, kIsDense<IbT>>;
  const int bias = (n_pad * 4 + 15) / 16 * 16;
  const int ib = kIsDense<IbT> ? 0 : 2 * rs * kBM * 4 + 2 * kBM * 4;   // int32 index slices + per-row bases
  // resident filter (dense A only): res_kb blocks of B, the ring holds A only
  const int res = res_kb * C::kBBytes;
  const int slot_bytes = res_kb ? kABytes : C::kSlotBytes;
  // (corr_bytes: uint8 im2col A -- border-class correction vectors, [classes][n_pad] int32)
  const int fixed = 1024 + C::kOnesBytes + C::kEpiBytes + bias + ib + corr_bytes + C::kBarBytes + res;
  int slots = (232448 - fixed) / slot_bytes;
  slots = (slots > C::kMaxSlots ? C::kMaxSlots : slots) / C::kKB * C::kKB;
  if (slots < 2 * C::kKB) return false;
  p->res_b = res_kb;
  p->slots = slots;
  p->stages = slots / C::kKB;
  p->off_b = slots * kABytes;
  p->off_ones = p->off_b + (res_kb ? res : slots * C::kBBytes);
  p->off_epi = p->off_ones + C::kOnesBytes;
  p->off_bias = p->off_epi + C::kEpiBytes;
  p->off_ib = p->off_bias + bias;
  p->off_corr = p->off_ib + ib;
  p->off_bar = p->off_corr + corr_bytes;
  p->bytes = 1024 + p->off_bar + C::kBarBytes;
  return true;
}

// Tile schedule.  kCS = 1: CTA b takes tiles b, b + G, ...  kCS > 1: a
// cluster of kCS CTAs takes groups of kCS consecutive M tiles with the same
// N tile (CTA rank r takes M tile group*kCS + r), so the cluster shares
// every filter block: each CTA TMA-loads 1/kCS of a stage's filter blocks
// and multicasts it to all kCS CTAs.  M tiles past the end are dummies
// (clamped references, nothing stored) so the CTAs of a cluster stay in
// step.
template <int kCS>
struct ClusterTiles {
  int64_t m_tiles;
  int32_t n_tiles;
  __device__ __forceinline__ int64_t groups() const { return (m_tiles + kCS - 1) / kCS * n_tiles; }
  __device__ __forceinline__ int64_t count() const {
    const int64_t nc = gridDim.x / kCS, c = blockIdx.x / kCS, g = groups();
    return c < g ? (g - c + nc - 1) / nc : 0;
  }
  __device__ __forceinline__ int64_t operator()(int64_t k) const {
    const int64_t g = blockIdx.x / kCS + k * (gridDim.x / kCS);
    const int64_t mg = g / n_tiles;
    const int64_t nt = g - mg * n_tiles;
    return (mg * kCS + blockIdx.x % kCS) * n_tiles + nt;
  }
};

// (+ the row-sum warps of the uint8 BN 256 plan)
template <bool kI8, int BN, int kCS, int kEpiW>
constexpr int kThreadsK = kThreadsS<kI8, kEpiW> + 32 * CfgS<kI8, BN, kCS, kEpiW, false>::kSumWarps;

template <bool kI8, int BN, typename IbT, int kCS, int kEpiW>
__global__ void __launch_bounds__(kThreadsK<kI8, BN, kCS, kEpiW>, 1) igemm_smem_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                                  const __grid_constant__ CUtensorMap tmap_x,
                                                                  const __grid_constant__ CUtensorMap tmap_y,
                                                                  const TcArgs a, const PlanS pl) {
  // kCS == 2: CTA pair -- the leader (rank 0) issues cta_group::2 MMAs with
  // M = 256 (its 128 rows + the peer's 128 rows); each CTA gathers its own A
  // rows and TMA-loads its half of the filter rows, so each SM receives half
  // the filter bytes of the single-CTA kernel.
  using C = CfgS<kI8, BN, kCS, kEpiW, kIsDense<IbT>>;
  static_assert(kCS == 1 || kCS == 2, "single CTA or CTA pair");
  constexpr uint16_t kMask = (uint16_t)((1u << kCS) - 1);
  const ClusterTiles<kCS> sched{a.total_tiles / a.n_tiles, a.n_tiles};
  const uint32_t crank = kCS > 1 ? cluster_ctarank() : 0;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base (SW128 atoms); pointer arithmetic keeps the
  // shared address space visible to the compiler (no generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + pl.off_b;
  uint8_t* sOnes = smem + pl.off_ones;
  uint8_t* sEpi = smem + pl.off_epi;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(smem + pl.off_bias);
  int32_t* sRowBase = reinterpret_cast<int32_t*>(smem + pl.off_ib);   // [2][128] per-image base offsets
  // [2][RS][128] index slices and [2][128] per-row image bases, 32-bit (the
  // launcher requires N*H*W*C < 2^31; an int64 entry's low word is its value)
  int32_t* sIB = reinterpret_cast<int32_t*>(smem + pl.off_ib + 2 * kBM * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  const int kStages = pl.stages;
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;                                        // resident filter landed (dense A)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(0);
  // Dense A (a.use_tma_x): a 1x1 stride-1 layer with a canonical buffer
  // references pixel p at tap 0 for output pixel p, so the A tile of M tile
  // mt is the 128 consecutive pixel rows [128 mt, 128 mt + 128) of the input
  // -- one 2-D TMA box per 128-byte channel block (rows past the batch and
  // channels past C are zero-filled; those rows are never stored).  The
  // launcher sets it only for such layers (and for the GEMM baseline's patch
  // matrix, a 1 x P image of R*S*C channels).
  constexpr bool dense_a = kIsDense<IbT>;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      // TMA path: 1 expect_tx arrival; cp.async path: 128 producer arrivals + 1
      // cp.async path: 128 producer arrivals + 1 expect_tx (+ 1 forwarded from the peer, pair leader)
      // dense A: the issuing thread's expect_tx arrival; gather: 32 per producer
      // warp + 1 expect_tx; a pair leader also counts the peer's forwarded arrival
      // (dense pairs: both CTAs' TMA loads complete on the leader's barrier, armed by the leader's issuer)
      mbar_init(&full[s], (dense_a ? 1 : 32 * kProdWarpsS<kI8> + 1) + (kCS == 2 && crank == 0 && !dense_a ? 1 : 0));
      mbar_init(&empty[s], 1 + C::kSumWarps);   // tcgen05.commit (multicast to both CTAs of a pair) + row-sum warps
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1 + C::kSumWarps);    // tcgen05.commit after the last K block (+ the tile's row sums)
      // one arrival per epilogue warp (of both CTAs at the pair leader)
      mbar_init(&tempty[s], (kCS == 2 && crank == 0) ? 2 * kEpiW : kEpiW);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmap_b);
    if (dense_a) tma_prefetch_desc(&tmap_x);
  }
  if constexpr (C::kFuseOnes) {
    // 16 all-ones rows behind the filter rows of every B block (TMA writes
    // only the first BN rows, so they stay); all-ones is swizzle-invariant
    const int nblk = pl.res_b ? pl.res_b : pl.slots;
    for (int i = threadIdx.x; i < nblk * 128; i += blockDim.x)
      reinterpret_cast<uint4*>(sB + (i >> 7) * C::kBBytes + C::kBLoadBytes)[i & 127] =
          make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fence_proxy_async_smem();
  } else if constexpr (kI8 && C::kSumWarps == 0) {
    if (threadIdx.x >= 128 && threadIdx.x < 256) {  // all-ones B tile (16 rows x 128 bytes)
      reinterpret_cast<uint4*>(sOnes)[threadIdx.x - 128] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u,
                                                                      0x01010101u);
      fence_proxy_async_smem();
    }
  }
  for (int i = threadIdx.x; i < a.n_pad; i += blockDim.x) sBias[i] = __ldg(static_cast<const uint32_t*>(a.bias) + i);
  int32_t* sCorr = reinterpret_cast<int32_t*>(smem + pl.off_corr);
  if (warp == kMmaWarpS<kI8, kEpiW>) {
    if constexpr (kCS == 2) tmem_alloc2<C::kTmemCols>(tmem_slot);
    else tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (kCS > 1) cluster_sync_all();   // peers' barriers initialised before any remote arrival
  else __syncthreads();
  tc_fence_after();
  // setup above read only constants (bias, zero row); the input activation
  // and the output may belong to the previous kernel in the stream.  The
  // filter does not: with dense A the first ring pass's filter blocks (or the
  // resident filter) are requested before the wait, so under programmatic
  // dependent launch they arrive while the previous kernel drains.
  if constexpr (dense_a && kCS == 1) {
    constexpr int kPWd = kProdWarpsS<kI8>;
    if (warp < kPWd && lane == 0) {
      const int64_t my_tiles0 = sched.count();
      const int nkb = a.RS * a.cblocks;
      if (pl.res_b) {
        if (warp == 0 && my_tiles0 > 0) {
          const int nt0 = (int)(sched(0) % a.n_tiles);
          mbar_arrive_expect_tx(bres, pl.res_b * C::kBLoadBytes);
          for (int kb = 0; kb < pl.res_b; ++kb)
            tma_load_3d(smem_u32(sB) + kb * C::kBBytes, &tmap_b, bres, 0, nt0 * BN, kb);
        }
      } else {
        const int niss = pl.stages < kPWd ? pl.stages : kPWd;
        for (int64_t q = warp; warp < niss && q < pl.stages && q < my_tiles0 * nkb; q += niss) {
          const int nt0 = (int)(sched(q / nkb) % a.n_tiles);
          mbar_arrive_expect_tx(&full[q], kABytes + C::kBLoadBytes);
          tma_load_3d(smem_u32(sB) + (int)q * C::kBBytes, &tmap_b, &full[q], 0, nt0 * BN, (int)(q % nkb));
        }
      }
    }
  }
  griddep_wait();
  griddep_launch_dependents();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);
  const int num_kb = a.RS * a.cblocks;
  const uint32_t sA_u32 = smem_u32(sA);
  const uint32_t sB_u32 = smem_u32(sB);

  if (warp < kProdWarpsS<kI8>) {
    // ------------------------------------------------------------ producers
    constexpr int kPW = kProdWarpsS<kI8>;
    constexpr int kRowsW = kBM / kPW;          // A rows per producer warp (32 or 16)
    const int chunk = lane & 7;
    const int sub = lane >> 3;
    const int slice_elems = a.RS * kBM;
    const int64_t my_tiles = sched.count();
    // cp.async the (R*S taps x 128 pixels) index slice of local tile k into buffer k&1
    auto stage_index_slice = [&](int64_t k) {
      if constexpr (!dense_a) {
        if (k < my_tiles && threadIdx.x < kBM) {
          const int64_t mt = sched(k) / a.n_tiles;
          const uint32_t base = smem_u32(sIB + (k & 1) * slice_elems) + threadIdx.x * 4;
          const RowRef rr = row_ref(a, mt, threadIdx.x);                        // row = threadIdx.x
          const IbT* src = static_cast<const IbT*>(a.ib) + rr.ent0;
          sRowBase[(k & 1) * kBM + threadIdx.x] = (int32_t)rr.base;
          for (int e = 0; e < a.RS; ++e)
            cp_async_ca<4>(base + e * kBM * 4, src + (int64_t)e * a.mr);
        }
      }
      cp_async_commit();
    };
    stage_index_slice(0);
    cp_async_wait_committed();
    named_bar_sync(1, 32 * kProdWarpsS<kI8>);
    int stage = 0;
    uint32_t phase = 0;
#ifdef ICV_TRACE
    long long p_begin = clock64(), p_wait = 0;
#endif
    for (int64_t k = 0; k < my_tiles; ++k) {
      const int64_t tile = sched(k);
      if (threadIdx.x == 0 && k < 8) TRACE(26 + k);
      stage_index_slice(k + 1);
      const int32_t* slice = sIB + (k & 1) * slice_elems;
      const int32_t* rbase = sRowBase + (k & 1) * kBM;
      const int nt = (int)(tile % a.n_tiles);
      if constexpr (dense_a) {
        // Stage q of the CTA's K-block sequence (kKB = 1: one A box + one
        // filter box under one expect_tx, no thread-side arrivals) is issued
        // by lane 0 of producer warp q % kPW: a thread's TMA loads issue one
        // after another at ~450 cycles each whatever their size
        // (tools/micro/tma_rate.cu), so one issuer would cap the ring at
        // ~50 B/cycle; kPW issuers keep several stages in flight.
        // At most kStages issuers: an issuer's previous stage, q - niss,
        // waited for the consumption of q - niss - kStages, so with
        // niss <= kStages the empty barrier of stage q is at most one phase
        // behind and its parity wait is unambiguous.
        static_assert(C::kKB == 1, "dense A: one K block per stage");
        const int niss = kStages < kPW ? kStages : kPW;
        const int64_t mt = tile / a.n_tiles;
        // L2 prefetch of the A rows of local tile k + dense_pf (one
        // contiguous range of 128 pixel rows), by a thread that issues no
        // TMA loads: the stage ring then reads A from L2, not from HBM
        if (a.dense_pf > 0 && threadIdx.x == 1 && k + a.dense_pf < my_tiles) {
          const int64_t mtp = sched(k + a.dense_pf) / a.n_tiles;
          const int64_t rows = min((int64_t)kBM, a.x_rows - mtp * kBM);
          if (rows > 0) {
            const uint8_t* src = a.x + mtp * kBM * (int64_t)a.c_bytes;
            int64_t bytes = rows * (int64_t)a.c_bytes;
            while (bytes > 0) {
              const uint32_t b = (uint32_t)(bytes < 65536 ? bytes : 65536);
              bulk_prefetch_l2(src, b);
              src += b;
              bytes -= b;
            }
          }
        }
        // im2col A (a.use_tma_x == 2): base input position (tap 0) of the tile's
        // first output pixel; the TMA unit walks the 128 output pixels itself
        int32_t im_w0 = 0, im_h0 = 0, im_n0 = 0;
        if (a.use_tma_x == 2 && lane == 0) {
          const int64_t p0 = mt * kBM;
          const int64_t n0 = p0 / a.ohw;
          const int32_t r0 = (int32_t)(p0 - n0 * a.ohw);
          const int32_t oy0 = r0 / a.im_ow;
          im_n0 = (int32_t)n0;
          im_h0 = oy0 * a.im_sy - a.im_pt;
          im_w0 = (r0 - oy0 * a.im_ow) * a.im_sx - a.im_pl;
        }
        const int64_t q0 = k * num_kb;
        for (int kb = 0; kb < num_kb; ++kb) {
          const int64_t q = q0 + kb;
          if (lane == 0 && (int)(q % niss) == warp) {
            const int st = (int)(q % kStages);
            mbar_wait(&empty[st], (uint32_t)((q / kStages) & 1) ^ 1u);
#ifdef ICV_TRACE
            if (k == (my_tiles > 1 ? 1 : 0) && kb < 16) TRACE(64 + kb);   // stage free
#endif
            if (pl.res_b) {   // resident filter: the stage holds A only
              mbar_arrive_expect_tx(&full[st], kABytes);
            } else if (kCS == 1 && q < kStages) {
              // (first ring pass: expect_tx and the filter block were issued before griddep_wait)
            } else if constexpr (kCS == 2) {
              // CTA pair: each member loads its own 128 A rows and its half of
              // the BN filter rows into its own smem; every load completes on
              // the LEADER's full barrier (TMA .cta_group::2), which the
              // leader's issuer arms with the bytes of both members -- no
              // forwarding hop.  (A member's complete_tx may precede the arming:
              // the phase cannot complete before the leader's arrival.)
              if (crank == 0) mbar_arrive_expect_tx(&full[st], 2 * (kABytes + C::kBLoadBytes));
              tma_load_3d_cg2(sB_u32 + st * C::kBBytes, &tmap_b, mapa_rank(smem_u32(&full[st]), 0), 0,
                              nt * BN + (int)crank * (BN / kCS), kb);
            } else {
              mbar_arrive_expect_tx(&full[st], kABytes + C::kBLoadBytes);
              tma_load_3d(sB_u32 + st * C::kBBytes, &tmap_b, &full[st], 0, nt * BN, kb);
            }
            if (a.use_tma_x == 2) {
              // K block kb = (tap e, channel block cb), cb fastest (the packed filter's order)
              const int e = kb / a.cblocks, cb = kb - e * a.cblocks;
              const int ky = e / a.im_s, kx = e - ky * a.im_s;
              const uint16_t ow_ = (uint16_t)(kx * a.im_dx), oh_ = (uint16_t)(ky * a.im_dy);
              if constexpr (kCS == 2)
                tma_load_im2col_4d_cg2(sA_u32 + st * kABytes, &tmap_x, mapa_rank(smem_u32(&full[st]), 0),
                                       cb * a.cblock_elems, im_w0, im_h0, im_n0, ow_, oh_);
              else
                tma_load_im2col_4d(sA_u32 + st * kABytes, &tmap_x, &full[st], cb * a.cblock_elems, im_w0, im_h0, im_n0,
                                   ow_, oh_);
            } else if constexpr (kCS == 2) {
              tma_load_2d_cg2(sA_u32 + st * kABytes, &tmap_x, mapa_rank(smem_u32(&full[st]), 0), kb * a.cblock_elems,
                              (int32_t)(mt * kBM));
            } else {
              tma_load_2d(sA_u32 + st * kABytes, &tmap_x, &full[st], kb * a.cblock_elems, (int32_t)(mt * kBM));
            }
#ifdef ICV_TRACE
            if (k == (my_tiles > 1 ? 1 : 0) && kb < 16) TRACE(96 + kb);   // stage issued
#endif
          }
        }
      } else {
        // IB gather (cp.async, any zero row): 8 lanes per 128-byte row (lane & 7 =
        // 16-byte chunk), 4 rows per instruction -- whole 128-byte lines per
        // request, which the LSU/L2 path moves fastest.  Per tap each lane
        // resolves ONE row reference (its own row of the warp's 32) and the 8
        // row pointers an instruction needs are exchanged by shuffles; rows
        // 4i+sub with the same i&1 share one swizzle pattern, so the shared
        // destinations are two registers plus immediates, and with the
        // channel-block count known at compile time the source offsets are
        // immediates too.
        const int myrow = warp * kRowsW + (lane & (kRowsW - 1));
        const int64_t mybase = rbase[myrow];
        const bool c_full = (a.c_bytes & 127) == 0;
        uint32_t dofs[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) dofs[b] = (warp * kRowsW + 4 * b + sub) * 128 + ((chunk ^ (4 * b + sub)) << 4);
        auto gather_tile = [&](auto cbc) {
          constexpr int kCBc = decltype(cbc)::value;   // 0: runtime channel-block count
          const int cblocks = kCBc ? kCBc : a.cblocks;
          int kb = 0;
          int stage_seq = (int)(k * ((num_kb + C::kKB - 1) / C::kKB));
          for (int e = 0; e < a.RS; ++e) {
            const int64_t off = resolve_ref((int64_t)slice[e * kBM + myrow], mybase);
            const uint8_t* mine = off < 0 ? a.zero_row : a.x + off * a.elem_bytes;   // ZERO_REF -> zero row
            const uint8_t* src[kRowsW / 4];
#pragma unroll
            for (int i = 0; i < kRowsW / 4; ++i)
              src[i] = reinterpret_cast<const uint8_t*>(
                           __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(mine), 4 * i + sub)) +
                       chunk * 16;
#pragma unroll(kCBc ? kCBc : 1)
            for (int cb = 0; cb < cblocks; ++cb, ++kb) {
              const int j = kb % C::kKB;
              if (j == 0) {
#ifdef ICV_TRACE
                long long pw0 = clock64();
#endif
                mbar_wait(&empty[stage], phase ^ 1);
#ifdef ICV_TRACE
                p_wait += clock64() - pw0;
                if (threadIdx.x == 0 && k == 1 && kb / C::kKB < 16) TRACE(64 + kb / C::kKB);   // stage free
#endif
                // the stage's filter blocks: one 3-D box (kKB K blocks; a tail
                // block past the filter is zero-filled and never multiplied),
                // issued by the producer warps in turn
                if (lane == 0 && warp == (stage_seq % kPW)) {
#ifdef ICV_EXP_NOB   // experiment: no filter loads
                  mbar_arrive(&full[stage]);
#else
                  mbar_arrive_expect_tx(&full[stage], C::kKB * C::kBLoadBytes);
                  // (a pair member loads its half of the BN filter rows)
                  tma_load_3d(sB_u32 + stage * C::kKB * C::kBBytes, &tmap_b, &full[stage], 0,
                              nt * BN + (int)crank * (BN / kCS), kb);
#endif
                }
                ++stage_seq;
              }
              const uint32_t slot_base = sA_u32 + (stage * C::kKB + j) * kABytes;
              const uint32_t d0 = slot_base + dofs[0], d1 = slot_base + dofs[1];
#ifndef ICV_EXP_NOA   // experiment: no A gathers
              if (c_full || cb + 1 < cblocks) {
#pragma unroll
                for (int i = 0; i < kRowsW / 4; ++i)
                  cp_async_16_full((i & 1 ? d1 : d0) + (i >> 1) * 1024, src[i] + cb * 128);
              } else {   // partial last channel block: zero-fill past C
                int valid = a.c_bytes - (cb * 128 + chunk * 16);
                valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
#pragma unroll
                for (int i = 0; i < kRowsW / 4; ++i)
                  cp_async_16((i & 1 ? d1 : d0) + (i >> 1) * 1024, valid ? src[i] + cb * 128 : a.x, (uint32_t)valid);
              }
#endif
              if (j == C::kKB - 1 || kb == num_kb - 1) {
#ifdef ICV_TRACE
                if (threadIdx.x == 0 && k == 1 && kb / C::kKB < 16) TRACE(96 + kb / C::kKB);   // stage issued
#endif
                cp_async_mbar_arrive_noinc(&full[stage]);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
              }
            }
          }
        };
        if (c_full && a.cblocks == 1) gather_tile(std::integral_constant<int, 1>{});
        else if (c_full && a.cblocks == 2) gather_tile(std::integral_constant<int, 2>{});
        else if (c_full && a.cblocks == 4) gather_tile(std::integral_constant<int, 4>{});
        else gather_tile(std::integral_constant<int, 0>{});
      }
      if (threadIdx.x == 0 && k < 8) TRACE(40 + k);   // producer: all of tile k's loads issued
      if constexpr (!dense_a) {
        // slice k+1 landed (its group was committed before this tile's gathers)
        // and every producer is done reading slice k
        cp_async_wait_committed();
        if (threadIdx.x == 0 && k < 8) TRACE(48 + k);   // producer: next slice landed
        named_bar_sync(1, 32 * kProdWarpsS<kI8>);
      }
    }
#ifdef ICV_TRACE
    if (threadIdx.x == 0) {
      g_icv_trace[blockIdx.x][37] = (unsigned long long)(clock64() - p_begin);
      g_icv_trace[blockIdx.x][38] = (unsigned long long)p_wait;
    }
#endif
  } else if (warp == kMmaWarpS<kI8, kEpiW> && kCS == 2 && crank != 0) {
    // ------------------------------------------------------------ pair peer: forwarder
    // The leader's MMAs read this CTA's stages too: once a stage is full here
    // (own gathers + own filter half), tell the leader's full barrier.
    const int stages_per_tile = (num_kb + C::kKB - 1) / C::kKB;
    const int64_t n_local = dense_a ? 0 : sched.count();   // (dense A: the member's loads signal the leader directly)
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = 0; t < n_local; ++t)
      for (int si = 0; si < stages_per_tile; ++si) {
        mbar_wait(&full[stage], phase);
        if (lane == 0) mbar_arrive_remote(mapa_rank(smem_u32(&full[stage]), 0));
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
  } else if (warp == kMmaWarpS<kI8, kEpiW>) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc<kI8>(kBM * kCS, BN + (C::kFuseOnes ? 16 : 0));
    constexpr uint32_t idesc_ones = make_idesc<kI8>(kBM * kCS, 16);
    const uint64_t ones_desc = sw128_kmajor_desc(smem_u32(sOnes));
    const int stages_per_tile = (num_kb + C::kKB - 1) / C::kKB;
    int stage = 0;
    uint32_t phase = 0;
    int as = 0;
    uint32_t aphase = 0;
#ifdef ICV_TRACE
    long long c_wait_full = 0, c_wait_tempty = 0, c_begin = clock64();
#endif
    const int64_t n_local = sched.count();
    if (pl.res_b && n_local > 0) {   // resident filter landed
      mbar_wait(bres, 0);
      tc_fence_after();
    }
    for (int64_t ti_local = 0; ti_local < n_local; ++ti_local) {
#ifdef ICV_TRACE
      long long c0 = clock64();
#endif
      mbar_wait(&tempty[as], aphase ^ 1);
#ifdef ICV_TRACE
      c_wait_tempty += clock64() - c0;
#endif
      tc_fence_after();
      const uint32_t d = tmem_base + as * C::kAccStride;
      for (int si = 0; si < stages_per_tile; ++si) {
        const int nsub = min(C::kKB, num_kb - si * C::kKB);
#ifdef ICV_TRACE
        long long c1 = clock64();
#endif
        mbar_wait(&full[stage], phase);
#ifdef ICV_TRACE
        c_wait_full += clock64() - c1;
        if (lane == 0 && ti_local == (n_local > 1 ? 1 : 0) && si < 16) TRACE(80 + si);   // stage full (MMA warp wakes)
#endif
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < nsub; ++j) {
            const int slot = stage * C::kKB + j;
            const uint64_t adesc = sw128_kmajor_desc(sA_u32 + slot * kABytes);
            const uint64_t bdesc = sw128_kmajor_desc(sB_u32 + (pl.res_b ? si * C::kKB + j : slot) * C::kBBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x 32-byte K steps per 128-byte block
              const uint32_t acc = (si | j | k) != 0;
              if constexpr (kCS == 1) {
#ifndef ICV_EXP_NOMMA   // experiment: fills only
                tc_mma<kI8>(d, adesc + 2 * k, bdesc + 2 * k, idesc, acc);
#endif
                if constexpr (kI8 && !C::kFuseOnes && !C::kSumWarps)
                  tc_mma<true>(d + BN, adesc + 2 * k, ones_desc + 2 * k, idesc_ones, acc);
              } else {
                tc_mma2<kI8>(d, adesc + 2 * k, bdesc + 2 * k, idesc, acc);
                if constexpr (kI8) tc_mma2<true>(d + BN, adesc + 2 * k, ones_desc + 2 * k, idesc_ones, acc);
              }
            }
          }
          if constexpr (kCS == 1) {
            tc_commit(&empty[stage]);
            if (si == stages_per_tile - 1) tc_commit(&tfull[as]);
          } else {   // the stage is free, and the accumulator ready, in both CTAs
            tc_commit2_mc(&empty[stage], kMask);
            if (si == stages_per_tile - 1) tc_commit2_mc(&tfull[as], kMask);
          }
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) {
        const int ti = (int)ti_local;
        if (ti < 8) TRACE(2 + ti);
      }
      if (++as == C::kAccStages) { as = 0; aphase ^= 1; }
    }
#ifdef ICV_TRACE
    if (lane == 0) {
      g_icv_trace[blockIdx.x][34] = (unsigned long long)(clock64() - c_begin);
      g_icv_trace[blockIdx.x][35] = (unsigned long long)c_wait_full;
      g_icv_trace[blockIdx.x][36] = (unsigned long long)c_wait_tempty;
    }
#endif
  } else if (C::kSumWarps > 0 && warp > kMmaWarpS<kI8, kEpiW>) {
    // ------------------------------------------------------------ row sums (uint8, BN 256)
    // Thread r of the four warps sums row r of every A stage of the tile:
    // the 128 bytes of the row in its swizzled order (chunk j ^ (r & 7):
    // conflict-free across a quarter warp).  Padding taps hold the bound
    // zero row, zero-filled channel tails add nothing -- the same bytes the
    // MMA multiplies.  The stage is released by the MMA commit AND these
    // warps; the sums reach the epilogue through smem under the tfull barrier.
    static_assert(C::kSumWarps == 0 || C::kKB == 1, "row-sum warps: one K block per stage");
    const int row = (warp - kMmaWarpS<kI8, kEpiW> - 1) * 32 + lane;
    int32_t* sSum = reinterpret_cast<int32_t*>(sOnes);
    const int64_t n_local = sched.count();
    int stage = 0, as = 0;
    uint32_t phase = 0, aphase = 0;
    for (int64_t t = 0; t < n_local; ++t) {
      uint32_t acc = 0;
      for (int si = 0; si < num_kb; ++si) {
        mbar_wait(&full[stage], phase);
        const uint8_t* rowp = sA + stage * kABytes + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 v = *reinterpret_cast<const uint4*>(rowp + ((j ^ (row & 7)) << 4));
          acc = __dp4a(v.x, 0x01010101u, acc);
          acc = __dp4a(v.y, 0x01010101u, acc);
          acc = __dp4a(v.z, 0x01010101u, acc);
          acc = __dp4a(v.w, 0x01010101u, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      mbar_wait(&tempty[as], aphase ^ 1);   // the epilogue has read the sums of the tile two back
      sSum[as * kBM + row] = (int32_t)acc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfull[as]);
      if (++as == C::kAccStages) { as = 0; aphase ^= 1; }
    }
  } else {
    // uint8 over zero-filled im2col tiles: per border class (row class x
    // column class) the sum of the per-tap corrections zx * sum_c (w - zw) of
    // the taps that leave the image there -- what those taps would have
    // contributed had they read the zero point (the zero row) instead of TMA's
    // zero fill.  Staged by the epilogue warps while the first tile's
    // mainloop runs (off the producers' and the MMA's critical path).
    if constexpr (kI8) {
      if (a.ncls > 0) {
        for (int i = threadIdx.x - 32 * kProdWarpsS<kI8>; i < a.ncls * a.n_pad; i += 32 * kEpiW) {
          const int cl = i / a.n_pad, n = i - cl * a.n_pad;
          const int oy = border_rep(cl / a.cls_ncc, a.cls_tb, a.cls_ohb, a.cls_nr);
          const int ox = border_rep(cl % a.cls_ncc, a.cls_lb, a.cls_owb, a.cls_ncc);
          int32_t sum = 0;
          for (int ky = 0; ky < a.im_r; ++ky) {
            const int iy = oy * a.im_sy - a.im_pt + ky * a.im_dy;
            const bool row_out = iy < 0 || iy >= a.im_h;
            for (int kx = 0; kx < a.im_s; ++kx) {
              const int ix = ox * a.im_sx - a.im_pl + kx * a.im_dx;
              if (row_out || ix < 0 || ix >= a.im_w) sum += __ldg(a.tapcorr + (int64_t)(ky * a.im_s + kx) * a.n_pad + n);
            }
          }
          sCorr[i] = sum;
        }
        named_bar_sync(3, 32 * kEpiW);
      }
    }
    // a pair peer releases accumulators at the leader (which issues the next MMAs)
    const uint32_t tempty_remote = (kCS == 2 && crank != 0) ? mapa_rank(smem_u32(tempty), 0) : 0u;
    epilogue_loop<kI8, BN, kEpiW, C::kAccStride, std::remove_const_t<decltype(sched)>, C::kAccStages>(
        a, warp - kProdWarpsS<kI8>, lane, tmem_base, sEpi, sBias, tfull, tempty, sched, a.use_tma_y ? &tmap_y : nullptr,
        tempty_remote, C::kSumWarps ? reinterpret_cast<const int32_t*>(sOnes) : nullptr,
        (kI8 && a.ncls > 0) ? sCorr : nullptr);
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (kCS > 1) cluster_sync_all();   // both CTAs done: no peer still signals, writes or reads TMEM
  if (warp == kMmaWarpS<kI8, kEpiW>) {
    tc_fence_after();
    if constexpr (kCS == 2) tmem_dealloc2<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <bool kI8, int BN, typename IbT, int kCS, int kEpiW>
int launch_smem_cs(const ConvArgs& c, cudaStream_t st) {
  auto kernel = igemm_smem_kernel<kI8, BN, IbT, kCS, kEpiW>;
  PlanS pl;
  // uint8 im2col A: border-class correction vectors staged in smem
  BorderClasses bc;
  int corr_bytes = 0;
  if constexpr (kI8 && kIsDense<IbT>)
    if (tma_a_mode(c) == 2 && im2col_u8_classes(c, &bc)) corr_bytes = bc.ncls * c.L.n_pad * 4;
  if (!plan_smem<kI8, BN, IbT, kCS, kEpiW>(c.g.RS(), c.L.n_pad, &pl, 0, corr_bytes))
    return fail(ICV_ERR_UNSUPPORTED, "indirection slice of this kernel size does not fit in shared memory");
  // dense A with few K blocks: keep the CTA's filter blocks resident (the
  // grid is then a multiple of the N-tile count, so every CTA keeps one N
  // tile) when they fit in dense_resb KB and the A ring keeps >= 4 stages
  int grid_mult = 1;
  if constexpr (kIsDense<IbT> && kCS == 1) {
    using Cd = CfgS<kI8, BN, 1, kEpiW, true>;
    const int kbs = c.g.RS() * c.L.cblocks;   // K blocks per tile
    const int n_tiles = c.L.n_pad / BN;
    PlanS pr;
    if (tune(kTuneDenseResB) > 0 && kbs * Cd::kBBytes <= tune(kTuneDenseResB) * 1024 && n_tiles <= 8 &&
        plan_smem<kI8, BN, IbT, kCS, kEpiW>(1, c.L.n_pad, &pr, kbs, corr_bytes) && pr.stages >= 4) {
      pl = pr;
      grid_mult = n_tiles;
    }
  }
  if (c.g.N * c.g.H * c.g.W * (int64_t)c.g.C >= (int64_t(1) << 31))
    return fail(ICV_ERR_UNSUPPORTED, "tensor-core kernel: input tensors of 2^31 or more elements are not supported");
  int max_clusters = 0;
  constexpr int kThreads = kThreadsK<kI8, BN, kCS, kEpiW>;
  if (int s = kernel_setup(reinterpret_cast<const void*>(kernel), 232448, kCS, kThreads, &max_clusters))
    return s;
  CUtensorMap tmap, tmap_x;
  if (int s = make_filter_tmap(c, BN / kCS, CfgS<kI8, BN, kCS, kEpiW, kIsDense<IbT>>::kKB, &tmap)) return s;
  TcArgs a;
  fill_tc_args(c, BN, &a);
  // dense A: 1x1 stride-1 layers with a canonical buffer (and the GEMM
  // baseline's patch matrix) load the A tile as TMA boxes of consecutive rows
  a.use_tma_x = 0;
  if constexpr (kIsDense<IbT>) {   // (single CTAs and pairs alike: each CTA loads its own 128 rows)
    const int mode = tma_a_mode(c);
    if (mode == 2) {
      if (int s = make_input_tmap_im2col(c, &tmap_x)) return fail(s, "im2col input tensor map");
      a.im_ow = (int32_t)c.g.OW; a.im_s = c.g.S; a.im_sx = c.g.SX; a.im_sy = c.g.SY;
      a.im_dx = c.g.DX; a.im_dy = c.g.DY; a.im_pl = c.g.PL; a.im_pt = c.g.PT;
      a.im_r = c.g.R; a.im_h = (int32_t)c.g.H; a.im_w = (int32_t)c.g.W; a.im_oh = (int32_t)c.g.OH;
      if (corr_bytes) {   // (uint8, zero row = zero point: TMA's zero fill needs the padded taps' corrections)
        a.tapcorr = reinterpret_cast<const int32_t*>(c.packed + c.L.tapcorr_off);
        a.ncls = bc.ncls;
        a.cls_tb = bc.tb; a.cls_ohb = bc.ohb; a.cls_nr = bc.nr;
        a.cls_lb = bc.lb; a.cls_owb = bc.owb; a.cls_ncc = bc.ncc;
      }
    } else if (int s = make_input_tmap(c, &tmap_x)) {
      return fail(s, "dense-A input tensor map");
    }
    a.use_tma_x = mode == 2 ? 2 : 1;
    a.dense_pf = tune(kTuneDensePf);
    a.x_rows = c.g.N * c.g.H * c.g.W;
  } else {
    tmap_x = tmap;   // unused placeholder
  }
  CUtensorMap tmap_y;
  // wide epilogue chunks when each epilogue warp owns a multiple of 64 columns
  constexpr bool kWideOk = !kI8 && (BN / (kEpiW / 4)) % 64 == 0;
  a.epi_wide = kWideOk && tune(kTuneEpiWide) != 0;
  a.use_tma_y = make_output_tmap(c, &tmap_y, a.epi_wide) == ICV_OK;
  if (!a.use_tma_y) a.epi_wide = 0;
  if (!a.use_tma_y) tmap_y = tmap;   // unused placeholder
  const int sms = sm_count();
  int64_t grid;
  if constexpr (kCS == 1) {
    grid = a.total_tiles < sms ? a.total_tiles : sms;
    if (grid_mult > 1) grid = grid / grid_mult * grid_mult;   // (resident filter: one N tile per CTA)
  } else {
    const int64_t groups = (a.total_tiles / a.n_tiles + kCS - 1) / kCS * a.n_tiles;
    int64_t clusters = sms / kCS;
    if (max_clusters > 0 && clusters > max_clusters) clusters = max_clusters;
    if (clusters > groups) clusters = groups;
    grid = clusters * kCS;
  }
  if (tune(kTuneWinDebug))   // (knob "win_debug" prints every tensor-core plan)
    fprintf(stderr, "igemm_smem: i8 %d BN %d CS %d epi %d dense %d | grid %lld max_clusters %d stages %d slots %d "
                    "smem %d tiles %lld n_tiles %d resident filter blocks %d\n", (int)kI8, BN, kCS, kEpiW,
            (int)kIsDense<IbT>, (long long)grid, max_clusters, pl.stages, pl.slots, pl.bytes, (long long)a.total_tiles,
            a.n_tiles, pl.res_b);
  return launch_conv_kernel(kernel, (unsigned)grid, kThreads, pl.bytes, st, kCS, "igemm_smem launch", tmap,
                            tmap_x, tmap_y, a, pl);
}

// CTA pairs (cta_group::2, M = 256): tuning knob "cluster" = 2 (see the kernel).
bool use_clusters() { return tune(kTuneCluster) == 2; }

// Dense-A layers on CTA pairs (knob "dense_cs": 0 auto, 1 never, 2 always).
// A pair member streams its own A rows and HALF of every filter block, so the
// L2 -> SM bytes per tile drop by a third at BN 256.  That pays once the K loop
// is long enough for the filter re-stream to dominate the fill (ResNet-50,
// N = 256, single CTA -> pair: 512->256 at 28x28 59.5 -> 53.1 us, 1024->512 at
// 14x14 53.2 -> 45.9, 2048->512 at 7x7 37.0 -> 32.9, 256->1024 39.2 -> 36.9 us)
// and loses on short K loops (64->64 37.7 -> 45.1, 128->512 53.3 -> 56.4 us):
// auto takes pairs from four 128-byte channel blocks up.
bool dense_pair_wanted(const ConvArgs& c) {
  const int mode = tune(kTuneDenseCs);
  if (mode == 2) return true;
  if (mode == 1) return false;
  return c.L.family == kFamTcBf16 && c.g.RS() * c.L.cblocks >= 4;
}


template <bool kI8, int BN, typename IbT>
int launch_smem(const ConvArgs& c, cudaStream_t st) {
  if (use_clusters()) return launch_smem_cs<kI8, BN, IbT, 2, kEpiWarpsS<kI8>>(c, st);
  if (tma_a_mode(c)) {
    PlanS pl;
    const bool wide_out = !kI8 && (int64_t)c.g.K >= 4 * (int64_t)c.g.C;
    if (dense_pair_wanted(c)) {
      // CTA pairs (M = 256): each SM streams its own A rows and half of the
      // filter block, so the L2 -> SM bytes per MMA drop by a third at BN 256
      if (wide_out && plan_smem<kI8, BN, DenseA, 2, 8>(1, c.L.n_pad, &pl))
        return launch_smem_cs<kI8, BN, DenseA, 2, 8>(c, st);
      if (plan_smem<kI8, BN, DenseA, 2, kEpiWarpsS<kI8>>(1, c.L.n_pad, &pl))
        return launch_smem_cs<kI8, BN, DenseA, 2, kEpiWarpsS<kI8>>(c, st);
    }
    if (wide_out && plan_smem<kI8, BN, DenseA, 1, 8>(1, c.L.n_pad, &pl))
      return launch_smem_cs<kI8, BN, DenseA, 1, 8>(c, st);
    if (plan_smem<kI8, BN, DenseA, 1, kEpiWarpsS<kI8>>(1, c.L.n_pad, &pl))
      return launch_smem_cs<kI8, BN, DenseA, 1, kEpiWarpsS<kI8>>(c, st);
  }
  if constexpr (!kI8) {
    // output-heavy layers (K >= 4 C) get 8 epilogue warps
    PlanS pl;
    if ((int64_t)c.g.K >= 4 * (int64_t)c.g.C && plan_smem<kI8, BN, IbT, 1, 8>(c.g.RS(), c.L.n_pad, &pl))
      return launch_smem_cs<kI8, BN, IbT, 1, 8>(c, st);
  }
  return launch_smem_cs<kI8, BN, IbT, 1, kEpiWarpsS<kI8>>(c, st);
}

// knob u8_bn = 256: uint8 layers with a multiple of 256 output channels run
// BLOCK_N 256 (half the A gathers per output, one accumulator stage); correct
// but measured slower on cfg4 (51 vs 40 us: 1.3 waves of tiles, no epilogue
// overlap), so BLOCK_N 128 stays the default
template <bool kI8, int BN>
bool smem_plan_ok(const ConvArgs& c);
int smem_block_n(const ConvArgs& c) {
  if (c.L.family == kFamTcU8 && c.L.n_pad % 256 == 0 && tune(kTuneU8Bn) == 256 && smem_plan_ok<true, 256>(c)) return 256;
  // few tiles: BLOCK_N 256 would leave a partial last wave of tiles (e.g.
  // ResNet-50 stage 4: 196 tiles on 148 SMs = 1.32 waves); half-width tiles
  // double the count (2.65 waves) -- the packed layout serves any BLOCK_N
  // dividing n_pad
  if (c.L.family == kFamTcBf16 && c.L.block_n == 256 && tune(kTuneSmallTileBn) > 0) {
    const int64_t m_tiles = (c.P + kBM - 1) / kBM;
    const int64_t tiles = m_tiles * (c.L.n_pad / 256);
    if (tiles * 100 < (int64_t)sm_count() * tune(kTuneSmallTileBn)) return 128;
  }
  return c.L.block_n;
}

template <typename IbT>
int dispatch_smem(const ConvArgs& c, cudaStream_t st) {
  const int bn = smem_block_n(c);
  if (c.L.family == kFamTcBf16) {
    if (bn == 64) return launch_smem<false, 64, IbT>(c, st);
    if (bn == 128) return launch_smem<false, 128, IbT>(c, st);
    if (bn == 256) return launch_smem<false, 256, IbT>(c, st);
  } else if (c.L.family == kFamTcU8) {
    if (bn == 64) return launch_smem<true, 64, IbT>(c, st);
    if (bn == 128) return launch_smem<true, 128, IbT>(c, st);
    if (bn == 256) return launch_smem<true, 256, IbT>(c, st);
  }
  return fail(ICV_ERR_UNSUPPORTED, "no tensor-core kernel for this tile width");
}

template <bool kI8, int BN>
bool smem_plan_ok(const ConvArgs& c) {
  PlanS pl;
  return c.ib_is_i32 ? plan_smem<kI8, BN, int32_t>(c.g.RS(), c.L.n_pad, &pl)
                     : plan_smem<kI8, BN, int64_t>(c.g.RS(), c.L.n_pad, &pl);
}

}  // namespace

// ---------------------------------------------------------------- host helpers
PFN_cuTensorMapEncodeTiled_v12000 get_tensor_map_encoder() {
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

int make_filter_tmap(const ConvArgs& c, int block_n, int depth, CUtensorMap* tmap) {
  auto encode = get_tensor_map_encoder();
  if (!encode) return fail(ICV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  // packed rows viewed as [K blocks][n_pad rows][128 B]; box = depth K blocks of block_n rows
  const cuuint64_t dims[3] = {128, (cuuint64_t)c.L.n_pad, (cuuint64_t)(c.L.row_bytes / 128)};
  const cuuint64_t strides[2] = {(cuuint64_t)c.L.row_bytes, 128};
  const cuuint32_t box[3] = {128, (cuuint32_t)block_n, (cuuint32_t)depth};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = encode(tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(c.packed + c.L.w_off), dims,
                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(ICV_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
  return ICV_OK;
}

// 2-D view of the output (rows = output pixels of the batch, columns = K)
// for the epilogue's TMA tile stores: box = 32 columns x 32 rows; bf16 rows
// of the box are 64 bytes with the 64-byte swizzle, uint8 rows 32 bytes
// unswizzled.  Needs 16-byte aligned rows (K*elem % 16 == 0).
int make_output_tmap(const ConvArgs& c, CUtensorMap* tmap, bool wide) {
  if (tune(kTuneTmaStore) == 0) return ICV_ERR_UNSUPPORTED;
  const bool i8 = c.L.family == kFamTcU8;
  if (!i8 && c.L.family != kFamTcBf16 && c.L.family != kFamStemBf16) return ICV_ERR_UNSUPPORTED;
  const int eb = i8 ? 1 : 2;
  if ((c.g.K * eb) % 16 != 0 || (reinterpret_cast<uintptr_t>(c.y) & 15) != 0) return ICV_ERR_UNSUPPORTED;
  if (c.P >= (int64_t(1) << 31)) return ICV_ERR_UNSUPPORTED;
  auto encode = get_tensor_map_encoder();
  if (!encode) return ICV_ERR_CUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)c.g.K, (cuuint64_t)c.P};
  const cuuint64_t strides[1] = {(cuuint64_t)c.g.K * eb};
  // box: 32 columns x 32 rows (bf16: 64-byte swizzle), or for the wide bf16
  // epilogue 64 columns x 32 rows with the 128-byte swizzle
  const bool w64 = wide && !i8;
  const cuuint32_t box[2] = {w64 ? 64u : 32u, 32};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(tmap, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c.y, dims, strides,
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       i8 ? CU_TENSOR_MAP_SWIZZLE_NONE : (w64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return cr == CUDA_SUCCESS ? ICV_OK : ICV_ERR_CUDA;
}

// A 1x1, stride-1, unpadded layer over a canonical buffer reads pixel row p
// for output pixel p (indirect.py:112-125 with R = S = 1), so its A operand
// is the dense [pixels][C] input matrix.
namespace {
bool im2col_u8_classes(const ConvArgs& c, BorderClasses* b) {
  if (c.L.family != kFamTcU8 || c.L.tapcorr_off == 0) return false;
  const Geom& g = c.g;
  // top rows: tap row 0 above the image; bottom rows: the last tap row below it
  const auto border = [](int64_t O, int64_t I, int P, int span, int st, int* tb, int* ohb, int* n) {
    const int64_t t = std::min<int64_t>(O, (P + st - 1) / st);
    const int64_t first_bot = std::max<int64_t>(0, (I + P - span + st) / st);   // ceil((I + P - span + 1) / st)
    const int64_t b0 = std::max<int64_t>(t, std::min<int64_t>(O, first_bot));
    *tb = (int)t; *ohb = (int)b0; *n = (int)(t + (O - b0) + 1);
  };
  border(g.OH, g.H, g.PT, (g.R - 1) * g.DY + 1, g.SY, &b->tb, &b->ohb, &b->nr);
  border(g.OW, g.W, g.PL, (g.S - 1) * g.DX + 1, g.SX, &b->lb, &b->owb, &b->ncc);
  b->ncls = b->nr * b->ncc;
  return b->ncls >= 1 && (int64_t)b->ncls * c.L.n_pad * 4 <= 24576;
}
}  // namespace

// im2col TMA A tiles (tma_a_mode 2).  The buffer must be canonical and the
// zero row all zeros (padding = out-of-bounds zero fill); bf16 with whole
// 128-byte channel blocks; corners / offsets inside the TMA encoding's 8-bit
// fields (two spatial dimensions).
bool im2col_a_eligible(const ConvArgs& c) {
  const Geom& g = c.g;
  if (c.prefer_gather || !c.ib_canonical) return false;
  if (c.L.family == kFamTcU8) {
    // zero row = input zero point: TMA's zero fill is corrected per border
    // class in the epilogue (needs the packed per-tap corrections)
    if (!c.zero_known) {
      BorderClasses b;
      if (!c.zero_is_zp || !im2col_u8_classes(c, &b)) return false;
    }
  } else if (c.L.family != kFamTcBf16 || !c.zero_known) {
    return false;
  }
  const int eb = c.L.family == kFamTcU8 ? 1 : 2;
  if ((reinterpret_cast<uintptr_t>(c.x) & 15) != 0 || (g.C * eb) % 128 != 0) return false;
  const int uw = g.PR - (g.S - 1) * g.DX, uh = g.PB - (g.R - 1) * g.DY;
  if (g.PL > 128 || g.PT > 128 || uw < -128 || uw > 127 || uh < -128 || uh > 127) return false;
  if ((g.S - 1) * g.DX >= 255 || (g.R - 1) * g.DY >= 255) return false;
  if (g.SX > 8 || g.SY > 8) return false;   // (traversal strides: 3-bit fields)
  return g.N * g.H * g.W < (int64_t(1) << 31) && c.P < (int64_t(1) << 31);
}

bool dense_a_eligible(const ConvArgs& c) {
  const Geom& g = c.g;
  if (c.prefer_gather || !c.ib_canonical) return false;
  if (g.R != 1 || g.S != 1 || g.SY != 1 || g.SX != 1 || g.PT || g.PL || g.PB || g.PR) return false;
  const int eb = c.L.family == kFamTcU8 ? 1 : 2;
  if ((reinterpret_cast<uintptr_t>(c.x) & 15) != 0 || (g.C * eb) % 16 != 0) return false;
  return g.N * g.H * g.W < (int64_t(1) << 31);
}

// How the A tile can be brought in by TMA instead of the IB gather: 1 = dense
// (1x1 stride-1 unpadded: 128 consecutive pixel rows), 2 = im2col TMA (any
// kernel size / stride / dilation / padding over a canonical buffer with an
// all-zero zero row: the tile's references are a function of the geometry and
// the TMA unit generates them itself), 0 = neither.
int tma_a_mode(const ConvArgs& c) {
  if (tune(kTuneDenseA) && dense_a_eligible(c)) return 1;
  // im2col re-reads every input pixel once per tap that uses it, like the
  // gather, but at TMA rates and on CTA pairs; measured against the IB-gather
  // kernel (ResNet-50, N = 256, us): 512 ch 3x3/2 75.7 -> 57.3, 256 ch 3x3/2
  // 55.3 -> 51.1, the 1x1/2 projections 71.7 -> 65.5, 55.3 -> 52.1, 51.3 ->
  // 49.2, but 128 ch 3x3/2 77.9 -> 80.0: auto takes it from four channel
  // blocks up (knob im2col_a: 0 off, 1 auto, 2 wherever eligible).
  const int mode = tune(kTuneIm2colA);
  if (mode && im2col_a_eligible(c) && (mode == 2 || c.L.cblocks >= 4 || c.L.family == kFamTcU8)) return 2;
  return 0;
}

// 2-D view of the bound input for dense-A TMA loads: rows = N*H*W pixels,
// columns = C elements; box = one 128-byte channel block of 128 rows,
// 128-byte swizzle (the A tile's canonical K-major layout).  Rows past the
// tensor and columns past C are zero-filled.
int make_input_tmap(const ConvArgs& c, CUtensorMap* tmap) {
  if (c.L.family != kFamTcBf16 && c.L.family != kFamTcU8) return ICV_ERR_UNSUPPORTED;
  const int64_t rows = c.g.N * c.g.H * c.g.W;
  auto encode = get_tensor_map_encoder();
  if (!encode) return ICV_ERR_CUDA;
  const bool i8 = c.L.family == kFamTcU8;
  const int eb = i8 ? 1 : 2;
  const cuuint64_t dims[2] = {(cuuint64_t)c.g.C, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)c.g.C * eb};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / eb), (cuuint32_t)kBM};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(tmap, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                       const_cast<void*>(c.x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return cr == CUDA_SUCCESS ? ICV_OK : ICV_ERR_CUDA;
}

// 4-D NHWC im2col map of the bound input (cuTensorMapEncodeIm2col): bounding
// box corners from the padding and the kernel extent, traversal strides = the
// convolution strides, 128 output pixels x one 128-byte channel block per
// load, 128-byte swizzle (the A tile's canonical K-major layout).
int make_input_tmap_im2col(const ConvArgs& c, CUtensorMap* tmap) {
  typedef CUresult (*EncodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
  static EncodeIm2col fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2col>(p);
  });
  if (!fn) return ICV_ERR_CUDA;
  const Geom& g = c.g;
  const bool i8 = c.L.family == kFamTcU8;
  const cuuint64_t eb = i8 ? 1 : 2;
  const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
  const cuuint64_t strides[3] = {(cuuint64_t)g.C * eb, (cuuint64_t)g.W * g.C * eb, (cuuint64_t)g.H * g.W * g.C * eb};
  const int lower[2] = {-g.PL, -g.PT};
  const int upper[2] = {g.PR - (g.S - 1) * g.DX, g.PB - (g.R - 1) * g.DY};
  const cuuint32_t estr[4] = {1, (cuuint32_t)g.SX, (cuuint32_t)g.SY, 1};
  CUresult cr = fn(tmap, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                   const_cast<void*>(c.x), dims, strides, lower, upper,
                   (cuuint32_t)(128 / eb), (cuuint32_t)kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return ICV_ERR_CUDA;
  // drivers up to 13.1 encode im2col maps of tensors under 128 KB with a bit
  // the hardware rejects (the workaround CUTLASS applies, copy_traits_sm90_im2col.hpp)
  int drv = 0;
  if (cudaDriverGetVersion(&drv) == cudaSuccess && drv <= 13010 &&
      (uint64_t)g.N * g.H * g.W * g.C * eb < 131072)
    reinterpret_cast<uint64_t*>(tmap)[1] &= ~(1ull << 21);
  return ICV_OK;
}

void fill_tc_args(const ConvArgs& c, int block_n, TcArgs* a) {
  const bool i8 = c.L.family == kFamTcU8;
  a->use_tma_y = 0;
  a->dense_pf = 0;
  a->tapcorr = nullptr;
  a->ncls = 0;
  a->im_ow = 1;
  a->epi_wide = 0;
  a->x_rows = c.g.N * c.g.H * c.g.W;
  a->tiles_per_row = 1;
  a->ow = 0;
  a->x = static_cast<const uint8_t*>(c.x);
  a->zero_row = static_cast<const uint8_t*>(c.zero_row);
  a->ib = c.ib;
  a->mr = c.mr;
  a->P = c.P;
  a->RS = c.g.RS();
  a->elem_bytes = i8 ? 1 : 2;
  a->c_bytes = c.g.C * a->elem_bytes;
  a->cblocks = c.L.cblocks;
  a->K = c.g.K;
  a->n_tiles = c.L.n_pad / block_n;
  a->total_tiles = ((c.P + kBM - 1) / kBM) * a->n_tiles;
  a->bias = c.packed + c.L.bias_off;
  a->y = c.y;
  a->zw = c.zw; a->zo = c.zo; a->qmin = c.qmin; a->qmax = c.qmax; a->m0 = c.m0; a->shift = c.shift;
  a->n_pad = c.L.n_pad;
  a->cblock_elems = 128 / a->elem_bytes;
  // exact division of element offsets (multiples of C) by C: C = odd << tz,
  // off / C = (off >> tz) * odd^-1 (mod 2^32)
  uint32_t odd = (uint32_t)c.g.C, tz = 0;
  while ((odd & 1u) == 0) { odd >>= 1; ++tz; }
  uint32_t inv = odd;                         // Newton iteration for the inverse mod 2^32
  for (int i = 0; i < 5; ++i) inv *= 2u - odd * inv;
  a->c_tz = (int32_t)tz;
  a->c_inv = inv;
  a->use_tma_x = 0;
  a->ib_per_image = c.ib_per_image;
  a->ohw = c.g.OH * c.g.OW;
  a->img_elems = c.g.H * c.g.W * (int64_t)c.g.C;
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

bool tc_kernel_available(const ConvArgs& c) {
  if (c.L.n_pad > kMaxBias) return false;
  const int bn = c.L.block_n;
  if (c.L.family == kFamTcU8) return bn == 64 ? smem_plan_ok<true, 64>(c) : smem_plan_ok<true, 128>(c);
  return bn == 64 ? smem_plan_ok<false, 64>(c) : bn == 128 ? smem_plan_ok<false, 128>(c) : smem_plan_ok<false, 256>(c);
}

// The im2col TMA kernel instead of the window kernel: on small images with
// many channels the window kernel's virtual grid computes many junk pixels and
// re-streams a large filter per unit (ResNet-50 256 ch 14x14 3x3: window 58.4,
// im2col pairs 49.2 us; 512 ch 7x7: 58.4 vs 57.4), while with few channels or
// large images reading each input pixel once wins (128 ch 28x28: 54.3 vs
// 75.8 us; cfg3b 62.4 vs 63.5).  Auto: four channel blocks up and output rows
// of at most 16 pixels; knob im2col_a = 2: wherever eligible (A/B).
static bool im2col_over_window(const ConvArgs& c) {
  if (tma_a_mode(c) != 2) return false;
  if (tune(kTuneIm2colA) == 2) return true;
  return tune(kTuneWin) != 1 && c.g.OW <= 16;   // (win = 1 forces the window kernel)
}

int launch_conv_tc(const ConvArgs& c, cudaStream_t st) {
  if (c.L.n_pad > kMaxBias) return fail(ICV_ERR_UNSUPPORTED, "more than 2048 output channels");
  if (win_kernel_eligible(c) && !im2col_over_window(c)) return launch_conv_win(c, st);
  if (c.ib_is_i32) return dispatch_smem<int32_t>(c, st);
  return dispatch_smem<int64_t>(c, st);
}

const char* tc_kernel_name(const ConvArgs& c) {
  const bool i8 = c.L.family == kFamTcU8;
  if (win_kernel_eligible(c) && !im2col_over_window(c)) return i8 ? "icv_igemm_win<u8>" : "icv_igemm_win<bf16>";
  if (const int mode = use_clusters() ? 0 : tma_a_mode(c)) {
    if (mode == 2 && i8) return dense_pair_wanted(c) ? "icv_igemm_smem<u8,im2col,pair>" : "icv_igemm_smem<u8,im2col>";
    if (mode == 2) return dense_pair_wanted(c) ? "icv_igemm_smem<bf16,im2col,pair>" : "icv_igemm_smem<bf16,im2col>";
    if (dense_pair_wanted(c)) return i8 ? "icv_igemm_smem<u8,dense,pair>" : "icv_igemm_smem<bf16,dense,pair>";
    return i8 ? "icv_igemm_smem<u8,dense>" : "icv_igemm_smem<bf16,dense>";
  }
  return i8 ? "icv_igemm_smem<u8>" : "icv_igemm_smem<bf16>";
}

}  // namespace icv

#if defined(ICV_TRACE) || defined(ICV_STEM_PHASES) || defined(ICV_ROWS_PHASES) || defined(ICV_ROWS_TIMELINE)
extern "C" ICV_API int icv_debug_trace(unsigned long long* host, int reset) {
  if (host && cudaMemcpyFromSymbol(host, icv::g_icv_trace, sizeof(icv::g_icv_trace)) != cudaSuccess)
    return ICV_ERR_CUDA;
  if (reset) {
    static unsigned long long zeros[1024][128];
    if (cudaMemcpyToSymbol(icv::g_icv_trace, zeros, sizeof(zeros)) != cudaSuccess) return ICV_ERR_CUDA;
  }
  return ICV_OK;
}
#endif
