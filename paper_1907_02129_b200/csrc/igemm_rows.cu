// K4b: row-sliding channel-poor kernel (the 7x7/2 ResNet stem and other
// stride-2 layers with C <= 4).
//
// The indirection buffer of such a layer (built by icv_ib_build, verified
// canonical by icv_ib_check once per buffer) has a fixed structure: for an
// output row oy and kernel row ky, the references of the row's pixels and of
// the taps kx = 0..S-1 are one arithmetic progression through input row
// iy = 2*oy - PT + ky (ZERO_REF exactly where it leaves the image).  This
// kernel consumes the buffer at that granularity: one input row per (output
// row, ky), converted once into shared memory as 8-byte pixels (C padded to
// 4, zero padding columns on both sides), and the tcgen05 A operand of tap
// row ky is a "sliding window" over it -- A row m (output pixel ox) starts
// 16 bytes (two pixels) after row m-1, described with the no-swizzle K-major
// layout (LBO = 16 B along K, SBO = 128 B along M; tools/micro/slide_mma.cu
// checks the encoding on a B200).  Per 128-pixel tile of one output row that
// is R x ceil(S*4/16) MMAs with A straight from the converted rows: there is
// no per-tap gather at all.  The filter stays resident in smem; each tile
// brings in only the input rows it adds (2 for stride 2), one bulk copy.
//
// Roles: warps 0-3 convert new input rows into a 16-row ring, warps 4-7 run
// the shared TMA-store epilogue (3-D output map: pixels past Wo are clipped),
// warp 8 issues the MMAs, warp 9 issues the bulk copies.
#include "igemm_common.cuh"

namespace icv {
namespace {

#ifdef ICV_ROWS_PHASES   // debug: per-role cycle accumulators -> g_icv_trace[cta][30..39]
#define RP_T0() long long _rt = clock64(), _ra[4] = {0, 0, 0, 0}
#define RP_ACC(i) do { const long long _n = clock64(); _ra[i] += _n - _rt; _rt = _n; } while (0)
#define RP_FLUSH(slot0, cond) if (cond) for (int _i = 0; _i < 4; ++_i) g_icv_trace[blockIdx.x][(slot0) + _i] = _ra[_i]
#else
#define RP_T0()
#define RP_ACC(i)
#define RP_FLUSH(slot0, cond)
#endif
#ifdef ICV_ROWS_TIMELINE   // debug: globaltimer per tile (CTA b < 8, tile k < 24) -> g_icv_trace[b][...]
__device__ __forceinline__ unsigned long long rt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define RT(slot) g_icv_trace[blockIdx.x][slot] = rt_now()
#define RTK(base, k) do { if ((k) < 24) g_icv_trace[blockIdx.x][(base) + (k)] = rt_now(); } while (0)
#else
#define RT(slot)
#define RTK(base, k)
#endif

#ifndef ICV_ROWS_RING
#define ICV_ROWS_RING 32
#endif
#ifndef ICV_ROWS_STAGES
#define ICV_ROWS_STAGES 6
#endif
#ifndef ICV_ROWS_READY
#define ICV_ROWS_READY 12
#endif
constexpr int kRingBig = ICV_ROWS_RING;   // converted input rows resident (power of 2) when the smem plan fits, else 16
constexpr int kConvWarps = 4;
constexpr int kConvThreads = 32 * kConvWarps;
#ifndef ICV_ROWS_EPI
#define ICV_ROWS_EPI 8
#endif
constexpr int kEpiWarpsR = ICV_ROWS_EPI;
constexpr int kMmaWarpR = kConvWarps + kEpiWarpsR;
constexpr int kLoadWarpR = kMmaWarpR + 1;
constexpr int kThreadsR = 32 * (kLoadWarpR + 1);
constexpr int kMDone = 4;                 // MMA-done barriers (tile k -> k % 4)
constexpr int kStagesR = ICV_ROWS_STAGES;             // raw-row stages in flight (the loader runs this many tiles ahead)
constexpr int kRowsReady = ICV_ROWS_READY;            // converted-tile barriers (converters run up to kLag + 1 tiles ahead of the MMA)
// TMEM accumulators (the MMA may run kAccR tiles ahead of the epilogue)
template <int BN>
constexpr int kAccRFor = BN <= 64 ? 8 : 4;

struct RowsArgs {
  TcArgs t;                     // epilogue fields (y, K, bias, n_tiles = 1, tiles_per_row, P)
  const uint8_t* wrows;         // packed row-sliding filter: [R][BN/8][4][8][8] bf16
  int32_t H, W, C, R, S, PT, PL, OH, tpr;
  int32_t rp, OHT;              // output rows per tile (1 or 2), row tiles per image = ceil(OH / rp)
  int32_t ring_row_bytes;       // 8 * padded pixels
  int32_t row_bytes;            // W * C * 2 (one raw input row)
  int32_t ksteps;               // MMA K steps per kernel row (1 or 2)
  int64_t total_tiles;          // N * OH * tpr
  int32_t pf;                   // loader: L2-prefetch the rows this many tiles ahead (0 = off)
  int32_t loaders;              // loader lanes issuing the raw-row copies round-robin
};

struct RowsPlan {
  int off_b, off_ring, off_stage, off_epi, off_bias, off_bar, bytes, stage_bytes;
};

// no-swizzle K-major smem descriptor
__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

struct RowTiles {   // contiguous tile ranges per CTA (epilogue schedule); begin computed once
  int64_t first, n;
  __device__ __forceinline__ static RowTiles make(int64_t total) {
    const int64_t b = total * blockIdx.x / gridDim.x;
    return RowTiles{b, total * (blockIdx.x + 1) / gridDim.x - b};
  }
  __device__ __forceinline__ int64_t begin() const { return first; }
  __device__ __forceinline__ int64_t count() const { return n; }
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return first + k; }
};

// Input rows a tile reads (clipped to the image) and the ones it adds to the
// ring after the previous tile of the same CTA.  Walks the CTA's tiles in
// order with 32-bit counters (no divisions per tile).
struct TileRows {
  int32_t n, oy, oxb, lo, hi, new_lo, new_hi;
  bool fresh;   // first tile of the CTA or of a new image
};
struct TileWalk {
  int32_t n, oy, oxb, prev_n, prev_hi;
  __device__ __forceinline__ void start(const RowsArgs& a, int64_t t0) {
    const int32_t row = (int32_t)(t0 / a.tpr);
    oxb = (int32_t)(t0 - (int64_t)row * a.tpr);
    n = row / a.OHT;
    oy = (row - n * a.OHT) * a.rp;
    prev_n = -1;
    prev_hi = -1;
  }
  // rows of the current tile; then advance to the next tile
  __device__ __forceinline__ TileRows next(const RowsArgs& a) {
    TileRows r;
    r.n = n;
    r.oy = oy;
    r.oxb = oxb;
    const int32_t first = 2 * oy - a.PT;
    const int32_t nrows = min(a.rp, a.OH - oy);
    r.lo = max(first, 0);
    r.hi = min(first + 2 * (nrows - 1) + a.R - 1, a.H - 1);
    r.fresh = prev_n != n;
    r.new_lo = r.fresh ? r.lo : max(r.lo, prev_hi + 1);
    r.new_hi = r.hi;
    prev_n = n;
    prev_hi = r.hi;
    if (++oxb == a.tpr) {
      oxb = 0;
      oy += a.rp;
      if (oy >= a.OH) { oy = 0; ++n; }
    }
    return r;
  }
};

template <int BN, int kR, int kKS, int kC, int kRing, int kRP>
__global__ void __launch_bounds__(kThreadsR, 1) igemm_rows_kernel(const __grid_constant__ CUtensorMap tmap_y,
                                                                  const RowsArgs a, const RowsPlan pl) {
  constexpr int kAccR = kAccRFor<BN> / kRP;   // tiles in TMEM (kRP accumulators each)
  // Ring-slot reuse: the 2 rows tile k adds evict rows last read by tile
  // k - (kRing + 1 - kR) / 2 or earlier, so within an image the converters
  // only wait for the MMAs of tile k - kLag (bounded by the accumulator ring
  // so the tfull phase they wait on is unambiguous); a new image may evict
  // anything, so its first tile waits for all earlier MMAs.
  constexpr int kLagRing = (kRing + 1 - (kR + 2 * (kRP - 1))) / (2 * kRP);
  constexpr int kLagCap = kAccR - 1 < kRowsReady - 2 ? kAccR - 1 : kRowsReady - 2;
  constexpr int kLag = kLagRing < kLagCap ? kLagRing : kLagCap;
  static_assert(kLag + 2 <= kRowsReady, "rows_ready phases must stay unambiguous");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem + pl.off_b;
  uint8_t* sRing = smem + pl.off_ring;           // kRing rows + 1 zero row
  uint8_t* sStage = smem + pl.off_stage;         // [kStagesR] raw new rows
  uint8_t* sEpi = smem + pl.off_epi;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(smem + pl.off_bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  uint64_t* stage_full = bars;                    // [kStagesR] raw rows landed (bulk copy)
  uint64_t* stage_free = stage_full + kStagesR;   // [kStagesR] converters done with the raw rows
  uint64_t* rows_ready = stage_free + kStagesR;   // [kRowsReady] tile's rows converted
  uint64_t* mdone = rows_ready + kRowsReady;      // [4] (unused)
  uint64_t* tfull = mdone + kMDone;               // [kAccR]
  uint64_t* tempty = tfull + kAccR;               // [kAccR]
  uint64_t* bfull = tempty + kAccR;
  int32_t* sInfo = reinterpret_cast<int32_t*>(bfull + 1);   // [kStagesR][2] new_lo, new_hi of the staged rows
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sInfo + 2 * kStagesR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const RowTiles sched = RowTiles::make(a.total_tiles);
  const int64_t t0 = sched.begin();
  const int64_t my_tiles = sched.count();
  const uint32_t ring_u32 = smem_u32(sRing);
  const uint32_t zero_row = ring_u32 + kRing * a.ring_row_bytes;

  if (threadIdx.x == 0) RT(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesR; ++s) {
      mbar_init(&stage_full[s], 1);
      mbar_init(&stage_free[s], kConvWarps);   // one arrival per converter warp
    }
    for (int s = 0; s < kRowsReady; ++s) mbar_init(&rows_ready[s], kConvWarps);
    for (int s = 0; s < kAccR; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4 * kRP);   // one arrival per warp of the epilogue group(s) storing the tile
    }
    for (int s = 0; s < kMDone; ++s) mbar_init(&mdone[s], 1);
    mbar_init(bfull, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < a.t.n_pad; i += blockDim.x) sBias[i] = __ldg(static_cast<const uint32_t*>(a.t.bias) + i);
  // ring (and zero row) start all-zero: padding columns / channels are never written again
  for (int i = threadIdx.x; i < (kRing + 1) * a.ring_row_bytes / 16; i += blockDim.x)
    sts128(ring_u32 + i * 16, 0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  if (warp == kMmaWarpR) tmem_alloc<(kAccR * kRP * BN <= 256 ? 256 : 512)>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();   // (setup read only constants; tensors may belong to the previous kernel)
  griddep_launch_dependents();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) RT(1);

  if (warp == kLoadWarpR) {
    // ------------------------------------------------------------ loader
    // Lanes 0 .. nload-1 issue the raw-row copies of tiles k = lane, lane +
    // nload, ...: each copy is small (the ~2 rows a tile adds) and one
    // thread's bulk copies are served one after another, so a single loader
    // caps the kernel at one tile per copy latency.  nload <= kStagesR keeps
    // every stage barrier's parity wait within one phase.
    const int nload = a.loaders < 1 ? 1 : (a.loaders > kStagesR ? kStagesR : a.loaders);
    if (lane < nload) {
      if (lane == 0) {
        const uint32_t b_bytes = (uint32_t)(a.R * BN * 64);
        mbar_arrive_expect_tx(bfull, b_bytes);
        bulk_load(smem_u32(sB), a.wrows, b_bytes, bfull);
      }
      RP_T0();
      TileWalk walk;
      walk.start(a, t0);
      // L2 prefetch of the rows `a.pf` tiles ahead (lane 0; knob rows_pf)
      TileWalk pwalk;
      pwalk.start(a, t0);
      auto prefetch_next = [&]() {
        const TileRows pr = pwalk.next(a);
        const int32_t pc = pr.new_hi - pr.new_lo + 1;
        if (pc > 0) bulk_prefetch_l2(a.t.x + ((int64_t)pr.n * a.H + pr.new_lo) * a.row_bytes, (uint32_t)(pc * a.row_bytes));
      };
      if (lane == 0)
        for (int64_t k = 0; k < a.pf && k < my_tiles; ++k) prefetch_next();
      for (int64_t k = 0; k < my_tiles; ++k) {
        const int s = (int)(k % kStagesR);
        if (lane == 0 && a.pf > 0 && k + a.pf < my_tiles) prefetch_next();
        const TileRows tr = walk.next(a);
        if ((int)(k % nload) != lane) continue;
        RP_ACC(1);
        if (k >= kStagesR) mbar_wait(&stage_free[s], (uint32_t)((k / kStagesR - 1) & 1));
        RP_ACC(0);
        sInfo[2 * s] = tr.new_lo;
        sInfo[2 * s + 1] = tr.new_hi;
        const int32_t cnt = tr.new_hi - tr.new_lo + 1;
        if (cnt > 0) {
          const uint32_t bytes = (uint32_t)(cnt * a.row_bytes);
          mbar_arrive_expect_tx(&stage_full[s], bytes);
          bulk_load(smem_u32(sStage) + s * pl.stage_bytes,
                    a.t.x + ((int64_t)tr.n * a.H + tr.new_lo) * a.row_bytes, bytes, &stage_full[s]);
        } else {
          mbar_arrive(&stage_full[s]);
        }
        RTK(8, k);
        RP_ACC(2);
      }
      RP_FLUSH(30, true);
    }
  } else if (warp < kConvWarps) {
    // ------------------------------------------------------------ converters
    // raw NHWC row (C bf16 per pixel) -> ring row (8-byte pixels at padded
    // position PL + ix, channels C..3 zero)
    const int tid = threadIdx.x;
    RP_T0();
    TileWalk walk;
    walk.start(a, t0);
    const uint32_t stage_u32 = smem_u32(sStage);
    for (int64_t k = 0; k < my_tiles; ++k) {
      const int s = (int)(k % kStagesR);
      const int rs = (int)(k % kRowsReady);
      const TileRows tr = walk.next(a);
      // the ring rows this tile overwrites are free once the MMAs of tile
      // k - kLag (same image) or of tile k-1 (a new image) have completed
      const int64_t need = tr.fresh ? k - 1 : k - kLag;
      RP_ACC(3);
      if (need >= 0) mbar_wait(&tfull[need % kAccR], (uint32_t)(need / kAccR) & 1u);   // MMAs of tile `need` done
      RP_ACC(0);
      mbar_wait(&stage_full[s], (uint32_t)((k / kStagesR) & 1));
      RP_ACC(1);
      const int32_t new_lo = sInfo[2 * s], new_hi = sInfo[2 * s + 1];
      const int32_t cnt = new_hi - new_lo + 1;
      // one thread per 8-pixel group of a new row: C 16-byte loads of the raw
      // row, eight 8-byte pixel slots out (W % 8 == 0)
      const int32_t groups_per_row = a.W / 8;
#ifndef ICV_EXP_ROWS_NOCONV
      const int32_t ngroups = cnt * groups_per_row;
#else
      const int32_t ngroups = 0;
#endif
      for (int32_t gi = tid; gi < ngroups; gi += kConvThreads) {
        const int32_t r = gi / groups_per_row, g = gi - r * groups_per_row;
        const uint32_t src = stage_u32 + s * pl.stage_bytes + r * a.row_bytes + g * (16 * kC);
        const uint32_t dst = ring_u32 + ((new_lo + r) & (kRing - 1)) * a.ring_row_bytes + (a.PL + 8 * g) * 8;
        uint32_t v[4 * kC];
#pragma unroll
        for (int q = 0; q < kC; ++q) {
          const uint4 t4 = lds128(src + q * 16);
          v[4 * q] = t4.x; v[4 * q + 1] = t4.y; v[4 * q + 2] = t4.z; v[4 * q + 3] = t4.w;
        }
#pragma unroll
        for (int px = 0; px < 8; ++px) {
          uint32_t e[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int idx = px * kC + c;   // element index in the group
            e[c] = c < kC ? (v[idx >> 1] >> (16 * (idx & 1))) & 0xFFFFu : 0u;
          }
          asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(dst + px * 8), "r"(e[0] | (e[1] << 16)),
                       "r"(e[2] | (e[3] << 16)) : "memory");
        }
      }
#ifndef ICV_EXP_NOFENCE
      fence_proxy_async_smem();   // ring writes -> visible to the tensor core
#endif
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&stage_free[s]);
        mbar_arrive(&rows_ready[rs]);
      }
      if (tid == 0) RTK(32, k);
      RP_ACC(2);
    }
    RP_FLUSH(34, tid == 0);
  } else if (warp == kMmaWarpR) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc<false>(kBM, BN);
    const uint32_t sB_u32 = smem_u32(sB);
    mbar_wait(bfull, 0);
    int as = 0;
    uint32_t aphase = 0;
    RP_T0();
    TileWalk walk;
    walk.start(a, t0);
    // descriptor constant parts (address field = bits 0..13, smem < 256 KB)
    const uint64_t adesc0 = desc_noswz(0, 16, 128), bdesc0 = desc_noswz(sB_u32, 128, 512);
    for (int64_t k = 0; k < my_tiles; ++k) {
      const TileRows tr = walk.next(a);
      RP_ACC(3);
      mbar_wait(&tempty[as], aphase ^ 1);
      RP_ACC(0);
      mbar_wait(&rows_ready[k % kRowsReady], (uint32_t)(k / kRowsReady) & 1u);
      RP_ACC(1);
      tc_fence_after();
      RP_ACC(3);
      if (elect_one()) {
        const uint32_t col0 = (uint32_t)tr.oxb * kBM * 2 * 8;   // padded pixel 2*ox of the tile's first pixel
#pragma unroll
        for (int sr = 0; sr < kRP; ++sr) {   // output row oy + sr -> accumulator sr of the tile
          const uint32_t d = tmem_base + (as * kRP + sr) * BN;
          // all row addresses first (independent), then kR*kKS back-to-back MMAs
          uint32_t rowa[kR];
#pragma unroll
          for (int ky = 0; ky < kR; ++ky) {
            const int32_t iy = 2 * (tr.oy + sr) - a.PT + ky;
            rowa[ky] = (iy >= 0 && iy < a.H) ? ring_u32 + (uint32_t)(iy & (kRing - 1)) * a.ring_row_bytes + col0
                                             : zero_row;
          }
#pragma unroll
          for (int ky = 0; ky < kR; ++ky) {
#pragma unroll
            for (int j = 0; j < kKS; ++j) {
              const uint64_t ad = adesc0 + ((rowa[ky] + 32 * j) >> 4);
              const uint64_t bd = bdesc0 + ((ky * BN * 64 + j * 256) >> 4);
#ifndef ICV_EXP_NOMMA
              tc_mma<false>(d, ad, bd, idesc, (ky | j) != 0 ? 1u : 0u);
#endif
            }
          }
        }
#ifdef ICV_ROWS_PHASES
        { const long long _n = clock64(); _ra[2] += _n - _rt; _rt = _n; }
#endif
        tc_commit(&tfull[as]);   // accumulator ready (epilogue) and the tile's ring rows free (converters)
        RTK(56, k);
      }
      __syncwarp();
      RP_ACC(3);
      if (++as == kAccR) { as = 0; aphase ^= 1; }
    }
    RP_FLUSH(38, lane == 0);
  } else {
    static_assert(kRP == 1 || kEpiWarpsR == 8, "row pairs: one epilogue group per row");
    epilogue_loop<false, BN, kEpiWarpsR, BN * kRP, RowTiles, kAccR, true, kEpiWarpsR / 4, kRP>(a.t, warp - kConvWarps, lane, tmem_base, sEpi, sBias,
                                                                 tfull, tempty, sched,
                                                                 a.t.use_tma_y ? &tmap_y : nullptr);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarpR) {
    tc_fence_after();
    tmem_dealloc<(kAccR * kRP * BN <= 256 ? 256 : 512)>(tmem_base);
  }
}

bool plan_rows(const ConvArgs& c, int BN, int tpr, int kRing, int rp, RowsPlan* p, int* ring_row_bytes) {
  const int ring_px_needed = 2 * (tpr * kBM - 1) + 8;
  int ring_px = ring_px_needed > c.g.PL + (int)c.g.W ? ring_px_needed : c.g.PL + (int)c.g.W;
  ring_px = (ring_px + 1) / 2 * 2;   // 16-byte rows
  *ring_row_bytes = ring_px * 8;
  const int b = c.g.R * BN * 64;
  const int ring = (kRing + 1) * *ring_row_bytes;
  const int stage = ((c.g.R + 2 * (rp - 1)) * (int)c.g.W * c.g.C * 2 + 15) / 16 * 16;   // a fresh tile's rows
  const int epi = kEpiWarpsR * kEpiWarpBytes<false>;
  (void)BN;
  int off = 0;
  p->off_epi = off;  off += epi;                       // 1024-aligned (TMA-store staging)
  p->off_b = off;    off += (b + 1023) / 1024 * 1024;
  p->off_ring = off; off += (ring + 127) / 128 * 128;
  p->off_stage = off; off += kStagesR * stage;
  p->stage_bytes = stage;
  p->off_bias = off; off += (c.L.n_pad * 4 + 15) / 16 * 16;
  p->off_bar = off;  off += 512;
  p->bytes = off + 1024;
  return p->bytes <= 232448;
}

template <int BN, int kR, int kKS, int kC, int kRing, int kRP>
int launch_rows_ring(const ConvArgs& c, cudaStream_t st, const RowsPlan& pl, int ring_row_bytes, int tpr) {
  auto kernel = igemm_rows_kernel<BN, kR, kKS, kC, kRing, kRP>;
  if (int s = kernel_setup(reinterpret_cast<const void*>(kernel), 232448, 1, kThreadsR, nullptr)) return s;
  RowsArgs a;
  fill_tc_args(c, BN, &a.t);
  a.t.tiles_per_row = tpr;
  a.t.ow = (int32_t)c.g.OW;
  a.wrows = c.packed + c.L.rows_off;
  a.H = (int32_t)c.g.H;
  a.W = (int32_t)c.g.W;
  a.C = c.g.C;
  a.R = c.g.R;
  a.S = c.g.S;
  a.PT = c.g.PT;
  a.PL = c.g.PL;
  a.OH = (int32_t)c.g.OH;
  a.tpr = tpr;
  a.ring_row_bytes = ring_row_bytes;
  a.row_bytes = (int32_t)(c.g.W * c.g.C * 2);
  a.ksteps = c.g.S * 4 <= 16 ? 1 : 2;
  a.rp = kRP;
  a.OHT = (int32_t)((c.g.OH + kRP - 1) / kRP);
  a.t.oh = (int32_t)c.g.OH;
  a.total_tiles = c.P / (c.g.OH * c.g.OW) * a.OHT * tpr;
  // 3-D output view (channel, pixel in the row, output row)
  CUtensorMap tmap_y;
  {
    auto encode = get_tensor_map_encoder();
    if (!encode) return fail(ICV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {(cuuint64_t)c.g.K, (cuuint64_t)c.g.OW, (cuuint64_t)(c.P / c.g.OW)};
    const cuuint64_t strides[2] = {(cuuint64_t)c.g.K * 2, (cuuint64_t)(c.g.OW * c.g.K * 2)};
    // box: 32 channels x 32 pixels (64-byte swizzle), or for the wide
    // epilogue 64 channels x 32 pixels (128-byte swizzle)
    a.t.epi_wide = tune(kTuneEpiWide) != 0 && BN % 64 == 0;
    const cuuint32_t box[3] = {a.t.epi_wide ? 64u : 32u, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode(&tmap_y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, c.y, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         a.t.epi_wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(ICV_ERR_CUDA, "row kernel: output tensor map");
  }
  a.t.use_tma_y = tune(kTuneTmaStore) != 0;
  a.pf = tune(kTuneRowsPf);
  a.loaders = tune(kTuneRowsLoaders);
  const int sms = sm_count();
  const int grid = (int)(a.total_tiles < sms ? a.total_tiles : sms);
  return launch_conv_kernel(kernel, (unsigned)grid, kThreadsR, pl.bytes, st, 1, "igemm_rows launch", tmap_y, a, pl);
}

// The deeper ring (converters up to kAccR - 1 tiles ahead of the MMA: cfg3a
// 30.8 -> 28.7 us) when the smem plan fits, else 16 rows (wide input rows).
template <int BN, int kR, int kKS, int kC>
int launch_rows_t(const ConvArgs& c, cudaStream_t st) {
  const int tpr = (int)((c.g.OW + kBM - 1) / kBM);
  RowsPlan pl;
  int ring_row_bytes = 0;
  // opt-in knob rows_rp = 2: tiles of two output rows (half the per-tile
  // hand-offs; BN 64: 8 accumulators = 4 tile pairs).  Correct, measured
  // slower (cfg3a 30.8 vs 28.7 us): the kernel is bound by shared-memory
  // bandwidth per output row, not by hand-offs per tile
  const bool rp2 = BN == 64 && tune(kTuneRowsRp) == 2;
  if (rp2 && plan_rows(c, BN, tpr, kRingBig, 2, &pl, &ring_row_bytes))
    return launch_rows_ring<BN, kR, kKS, kC, kRingBig, 2>(c, st, pl, ring_row_bytes, tpr);
  if (plan_rows(c, BN, tpr, kRingBig, 1, &pl, &ring_row_bytes))
    return launch_rows_ring<BN, kR, kKS, kC, kRingBig, 1>(c, st, pl, ring_row_bytes, tpr);
  if (plan_rows(c, BN, tpr, 16, 1, &pl, &ring_row_bytes))
    return launch_rows_ring<BN, kR, kKS, kC, 16, 1>(c, st, pl, ring_row_bytes, tpr);
  return fail(ICV_ERR_UNSUPPORTED, "row kernel: smem plan");
}

}  // namespace

// Filter geometry the row-sliding kernel handles (decides the packed copy).
bool rows_filter_eligible(int R, int S, int SY, int SX, int DY, int DX, int C, int K) {
  // instantiated shapes: 7 kernel rows x 5..8 columns (2 K steps), 3 x 1..4 (1 K step)
  const bool shape = (R == 7 && S > 4 && S <= 8) || (R == 3 && S <= 4);
  return shape && SX == 2 && SY == 2 && DX == 1 && DY == 1 && (C == 1 || C == 3) && K % 8 == 0 && K <= 128;
}
// ... and the input geometry (the IB must also be canonical).
bool rows_kernel_eligible(const Geom& g) {
  return rows_filter_eligible(g.R, g.S, g.SY, g.SX, g.DY, g.DX, g.C, g.K) && g.W % 8 == 0 && g.OW >= 32;
}

int launch_conv_rows(const ConvArgs& c, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(c.x) & 15) || (reinterpret_cast<uintptr_t>(c.y) & 15))
    return fail(ICV_ERR_UNSUPPORTED, "row kernel: 16-byte aligned tensors required");
  const bool n64 = c.L.block_n == 64;
  if (c.g.R == 7) {
    if (c.g.C == 3) return n64 ? launch_rows_t<64, 7, 2, 3>(c, st) : launch_rows_t<128, 7, 2, 3>(c, st);
    return n64 ? launch_rows_t<64, 7, 2, 1>(c, st) : launch_rows_t<128, 7, 2, 1>(c, st);
  }
  if (c.g.C == 3) return n64 ? launch_rows_t<64, 3, 1, 3>(c, st) : launch_rows_t<128, 3, 1, 3>(c, st);
  return n64 ? launch_rows_t<64, 3, 1, 1>(c, st) : launch_rows_t<128, 3, 1, 1>(c, st);
}

}  // namespace icv
