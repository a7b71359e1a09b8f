// K2w: window kernel -- the tcgen05 indirect GEMM for stride-1 layers with
// 16-byte pixel rows (bf16 C % 8 == 0, u8 C % 16 == 0), any kernel size,
// padding and dilation.
//
// The indirection buffer of a stride-1 layer (built by icv_ib_build; the call
// carries ICV_IB_CANONICAL) has a fixed structure: the reference of output
// pixel (n, oy, ox) at tap (ky, kx) is input pixel (oy - PT + ky*DY,
// ox - PL + kx*DX) of image n, or ZERO_REF where that leaves the image
// (indirect.py:112-125).  The kernel lays the batch out as one "stacked
// padded plane": rows of Wp = W + Zc positions (Zc = max(PL, PR) zero
// columns, shared by the right pad of one input row and the left pad of the
// next), each image preceded by Zr = max(PT, PB) zero rows (shared by the
// bottom pad of one image and the top pad of the next).  On the matching
// "virtual" output grid -- Hz = H + Zr rows of Wp pixels per image; rows
// oy >= Ho and columns ox >= Wo are computed and never stored -- the
// reference of virtual pixel q at tap e is plane position
//     q + (Zr - PT)*Wp + (Zc - PL) + off(e),   off(e) = ky*DY*Wp + kx*DX,
// the same affine map for every tap, shifted by a constant.  So a tile of 128
// consecutive virtual pixels reads, per tap, 128 CONSECUTIVE positions of one
// window of WR plane rows; tiles run straight across image boundaries.  The
// window is staged once per 128-byte channel block by TMA (128-byte swizzle;
// one box per image the window touches, from a set of tensor maps with box
// heights 1..WR, so boxes never overlap; zero rows and columns are
// out-of-bounds zero fill) -- or, when the bound zero row is not all zeros,
// gathered with cp.async from the zero row.  The tcgen05 A operand of tap e
// is the window itself with the descriptor start moved by off(e) rows: the
// swizzle is a function of the absolute smem address, so a 128-byte-row
// slide needs no re-layout (tools/micro/slide_sw128.cu checks it bit-exact on
// a B200 and shows the sliding operand runs at the full M128 N128 K16 rate).
// Each input pixel is read from L2 once per (tile, channel block) instead of
// R*S times.
//
// Work units: one or two M tiles per CTA (two accumulators sharing every
// filter block); CTA pairs (cta_group::2, M = 256) split each filter block's
// rows between the two SMs.  The schedule gives every cluster two-tile units
// while at least two rounds of work remain and one-tile units in the last
// round, which evens out the tail (cfg2: 3 tile-times per SM instead of 4).
//
// Roles: warps 0-3 producers (thread 0 issues the window and filter TMA
// loads; all 128 threads gather in cp.async mode), 8 epilogue warps, one MMA
// warp (one elected lane; the pair leader's only).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>

#include "igemm_common.cuh"

namespace icv {
namespace {

constexpr int kEpiWarpsW = 8;                    // two groups of 4 (TMEM lane quarters)
constexpr int kProdWarpsW = 4;
constexpr int kMmaWarpW = kProdWarpsW + kEpiWarpsW;
constexpr int kThreadsW = 32 * (kMmaWarpW + 1);
constexpr int kEpiRowBytes = 80;                 // staged output row (64 B + 16 B pad: conflict-free)
constexpr int kEpiWarpBytesW = 32 * kEpiRowBytes;
constexpr int kMaxWinStages = 4;
constexpr int kMaxBSlots = 40;                   // (resident filters: one slot per K block)
constexpr int kEpiBarId = 2;                     // named barrier of the epilogue warps
#ifndef ICV_MAX_WR
#define ICV_MAX_WR 32
#endif
constexpr int kMaxWR = ICV_MAX_WR;               // window rows (one tensor map per box height)

struct WinMaps {
  CUtensorMap m[kMaxWR];   // m[h-1]: box of h plane rows (x Wp positions x one 128-byte channel block)
};

struct WinArgs {
  TcArgs t;              // epilogue / filter fields (y, K, bias, n_tiles, quantization, cblocks, RS)
  int32_t H, W, OH, OW, S, DY, DX, PT, PL, Zc, Zr, Hz, Wp;
  int32_t WR, WR2;       // window rows of one tile / of two consecutive tiles (a two-tile unit shares one window)
  int32_t dpair;         // CTA pairs, one-tile units: the peer takes tile t + dpair (same window column), 0: t + 1
  int32_t batch;         // images convolved
  int32_t tiles;         // 128-pixel M tiles of the virtual grid
  int32_t two_units;     // leading units with two M tiles per CTA (then one-tile units)
  int32_t units;         // (two_units + one-tile units) * n_tiles
  int32_t cbe;           // elements per 128-byte channel block
  int32_t win_lead;      // bytes from a slot's start to the window's first row (1024-aligned)
  int32_t zero_known;    // host certifies the zero row is all zeros (no in-kernel check)
  int32_t win_split;     // TMA windows: rows split over this many issuing threads (lane 0 of warps 0..)
  int32_t filt_lanes;    // filter-block issuers per remaining producer warp (lanes 0..filt_lanes-1)
  // stride 2: the input is read as nph phase planes (row parity py, column
  // parity px); php[p] = 2 * py + px of the p-th plane holding taps
  int32_t sy;            // 1 or 2 (both directions)
  int32_t nph;
  int32_t php[4];
  int32_t g_shift, rel_shift;   // window row / in-window position of a tile's first pixel (see win_tile)
  const int32_t* tapcorr;       // u8 with TMA windows: per (tap, channel) zx * sum_c (w - zw), added for padded taps
  // u8 border classes (ncls > 0): a pixel's padded-tap set depends only on
  // its row class (top rows oy < cls_tb, bottom rows oy >= cls_ohb, one
  // interior class) and its column class; the epilogue adds one staged
  // correction vector per class instead of one per padded tap
  int32_t ncls, cls_tb, cls_ohb, cls_nr, cls_lb, cls_owb, cls_ncc;
};

// (border_class / border_rep: igemm_common.cuh)

struct PlanW {
  int wstages, bslots;
  int resident;          // the CTA's filter rows stay in smem: every K block loaded once, never released
  int win_stage;         // bytes per window stage (one window of up to WR2 rows + pair slack)
  int off_b, off_ones, off_epi, off_bias, off_tap, off_corr, off_bar, bytes;
};

template <bool kI8, int BN, int kMT, int kCS>
struct CfgW {
  // TMEM columns per M tile (u8: row sums at +BN; BN = 256 keeps 32 columns for them)
  static constexpr int kAccTile = kI8 ? (BN == 256 ? BN + 32 : 2 * BN) : BN;
  static constexpr int kAccStage = kMT * kAccTile;
  static constexpr int kAS = 2 * kAccStage <= 512 ? 2 : 1;   // accumulator stages (2: epilogue overlaps the next unit)
  static constexpr int kTmemNeed = kAS * kAccStage;
  static constexpr uint32_t kTmemCols = kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
  static constexpr int kBBytes = BN * 128 / kCS;        // this CTA's filter rows of one K block
  static constexpr int kOnesBytes = kI8 ? 16 * 128 : 0;
  static_assert(kTmemNeed <= 512, "TMEM overflow");
};

template <bool kI8, int BN, int kMT, int kCS, bool kS2>
bool plan_win(int win_stage, int rs, int kblocks, int n_pad, bool resident, PlanW* p) {
  using C = CfgW<kI8, BN, kMT, kCS>;
  const int bias = (n_pad * 4 + 15) / 16 * 16;
  const int tap = (rs * 8 + 9 * 4 + 15) / 16 * 16;   // sTap[rs], sTapE[rs], sPh[5], sPhP[4]
  const int bars = 1024;
  const int corr = kI8 ? rs * BN * 4 : 0;   // u8: staged per-tap padding corrections of the N tile
  const int fixed = 1024 + C::kOnesBytes + kEpiWarpsW * kEpiWarpBytesW + bias + tap + corr + bars;
  p->resident = 0;
  if (resident) {   // every K block of this CTA's filter rows + as many window stages (2..4) as fit
    if (kblocks > kMaxBSlots || fixed + 2 * win_stage + kblocks * C::kBBytes > 232448) return false;
    int ws = tune(kTuneWinWs) > 0 ? tune(kTuneWinWs) : kMaxWinStages;
    ws = ws > kMaxWinStages ? kMaxWinStages : (ws < 2 ? 2 : ws);
    while (ws > 2 && fixed + ws * win_stage + kblocks * C::kBBytes > 232448) --ws;
    p->resident = 1;
    p->wstages = ws;
    p->bslots = kblocks;
    p->win_stage = win_stage;
    p->off_b = ws * win_stage;
    p->off_ones = p->off_b + kblocks * C::kBBytes;
    p->off_epi = p->off_ones + C::kOnesBytes;
    p->off_bias = p->off_epi + kEpiWarpsW * kEpiWarpBytesW;
    p->off_tap = p->off_bias + bias;
    p->off_corr = p->off_tap + tap;
    p->off_bar = p->off_corr + corr;
    p->bytes = 1024 + p->off_bar + bars;
    return true;
  }
  const int ws_max = tune(kTuneWinWs) > 0 ? tune(kTuneWinWs) : (kS2 ? kMaxWinStages : 3);   // knob: force the stage count
  for (int ws = ws_max; ws >= 2; --ws) {
    const int left = 232448 - fixed - ws * win_stage;
    int bs = left / C::kBBytes;
    if (bs > 16) bs = 16;
    if (bs >= (ws == 2 ? 3 : 6)) {
      p->wstages = ws;
      p->bslots = bs;
      p->win_stage = win_stage;
      p->off_b = ws * win_stage;
      p->off_ones = p->off_b + bs * C::kBBytes;
      p->off_epi = p->off_ones + C::kOnesBytes;
      p->off_bias = p->off_epi + kEpiWarpsW * kEpiWarpBytesW;
      p->off_tap = p->off_bias + bias;
      p->off_corr = p->off_tap + tap;
      p->off_bar = p->off_corr + corr;
      p->bytes = 1024 + p->off_bar + bars;
      return true;
    }
  }
  return false;
}

// Tile t of the virtual grid: first virtual pixel, first window row of the
// stacked plane, position of pixel q0's tap-0 reference inside the window.
struct WinTile {
  int32_t q0, g0, rel0;
};
__device__ __forceinline__ WinTile win_tile(const WinArgs& a, int32_t t) {
  WinTile w;
  w.q0 = t * kBM;
  const int32_t v0 = w.q0 / a.Wp;
  w.g0 = v0 + a.g_shift;
  w.rel0 = w.q0 - v0 * a.Wp + a.rel_shift;
  return w;
}

// Unit u: `cnt` (1 or 2) consecutive M tiles per CTA starting at tile
// `first` for CTA rank crank, and the leader's first tile.  Single CTA: the
// unit's tiles in order.  Pair, consecutive mode: the leader takes the
// unit's first cnt tiles, the peer the next cnt (its window shifted to the
// leader's column).  Pair, dpair mode (one-tile units): the peer takes tile
// t + dpair, whose window column equals the leader's (dpair*128 = 0 mod Wp).
// A CTA whose tiles start past the end repeats the leader's tile (nothing of
// it is stored); tiles past the end are never stored.
struct UnitTiles {
  int32_t first, lead;
  int cnt;
  bool stand_in;
};
template <int kCS>
__device__ __forceinline__ UnitTiles unit_tiles(const WinArgs& a, int32_t u, uint32_t crank) {
  const int32_t b = u / a.t.n_tiles;
  int32_t pt;   // first pair tile (kCS tiles each)
  UnitTiles r;
  if (b < a.two_units) {
    pt = 2 * b;
    r.cnt = 2;
  } else {
    pt = 2 * a.two_units + (b - a.two_units);
    r.cnt = 1;
  }
  if (kCS == 1) {
    r.first = r.lead = pt;
  } else if (a.dpair > 0) {
    const int32_t blk = pt / a.dpair, j = pt - blk * a.dpair;
    r.lead = blk * 2 * a.dpair + j;
    r.first = r.lead + (int32_t)crank * a.dpair;
  } else {
    r.lead = pt * kCS;
    r.first = r.lead + (int32_t)crank * r.cnt;
  }
  r.stand_in = r.first >= a.tiles;
  if (r.stand_in) r.first = r.lead;   // (whole CTA past the end: never stored)
  return r;
}

#ifdef ICV_WEXP_PREFETCH   // experiment: L2 prefetch of the next window (measured slower: cfg2 25.5 -> 27.5 us)
constexpr bool kNoPrefetch = false;
#else
constexpr bool kNoPrefetch = true;
#endif


#ifdef ICV_WEXP_DIRECT   // experiment: epilogue stores straight from registers
constexpr bool kDirect = true;
#else
constexpr bool kDirect = false;
#endif

// Prefetch into L2 the input rows a unit's window covers (every channel: the
// rows of one image are contiguous), one bulk prefetch per image touched.
__device__ __forceinline__ void prefetch_window(const WinArgs& a, const UnitTiles& ut) {
  if (ut.stand_in) return;
  const WinTile tw = win_tile(a, ut.first);
  int32_t g = tw.g0;
  const int32_t gend = g + (ut.cnt == 2 ? a.WR2 : a.WR);
  const int64_t row_b = (int64_t)a.W * a.t.c_bytes;
  while (g < gend) {
    const int32_t n = g / a.Hz;
    if (n >= a.batch) break;
    const int32_t r = g - n * a.Hz;
    const int32_t h = min(gend - g, a.Hz - r);
    const int32_t iy0 = max(r - a.Zr, 0), iy1 = min(r + h - a.Zr, a.H);
    if (iy1 > iy0) {
      int64_t bytes = (int64_t)(iy1 - iy0) * row_b;
      const uint8_t* src = a.t.x + ((int64_t)n * a.H + iy0) * row_b;
      while (bytes > 0) {   // (bulk prefetch sizes are 32-bit; 16-byte multiples)
        const uint32_t b = (uint32_t)(bytes < (1 << 20) ? bytes : (1 << 20));
        bulk_prefetch_l2(src, b & ~15u);
        src += b;
        bytes -= b;
      }
    }
    g += h;
  }
}

template <bool kI8, int BN, int kMT, int kCS, bool kS2>
__global__ void __launch_bounds__(kThreadsW, 1) igemm_win_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                            const __grid_constant__ WinMaps maps,
                                                            const WinArgs a, const PlanW pl) {
  // kCS == 2: CTA pair.  The leader (rank 0) issues cta_group::2 MMAs with
  // M = 256 (its 128 window rows + the peer's); each CTA loads its own
  // windows and HALF of every filter block (BN/2 rows), both signalling the
  // leader's full barriers (TMA .cta_group::2), so each SM receives half the
  // filter bytes and the per-MMA shared-memory reads drop from A + B to
  // A + B/2.  A pair MMA reads A at the same smem address in both CTAs: the
  // peer shifts its window inside the slot by (rel0_leader - rel0_peer) rows
  // so its tile starts where the leader's does.  Commits multicast to both
  // CTAs; the peer's epilogue releases accumulators at the leader.
  using C = CfgW<kI8, BN, kMT, kCS>;
  static_assert(kCS == 1 || kCS == 2, "single CTA or CTA pair");
  constexpr uint16_t kMask = (uint16_t)((1u << kCS) - 1);
  const uint32_t crank = kCS > 1 ? cluster_ctarank() : 0;
  const int32_t cid = kCS > 1 ? (int32_t)(blockIdx.x / kCS) : (int32_t)blockIdx.x;   // cluster id
  const int32_t ncl = kCS > 1 ? (int32_t)(gridDim.x / kCS) : (int32_t)gridDim.x;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sWin = smem;
  uint8_t* sB = smem + pl.off_b;
  uint8_t* sOnes = smem + pl.off_ones;
  uint8_t* sEpi = smem + pl.off_epi;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(smem + pl.off_bias);
  int32_t* sTap = reinterpret_cast<int32_t*>(smem + pl.off_tap);   // window offset of the i-th tap (plane order)
  int32_t* sTapE = sTap + a.t.RS;                                      // its tap index e = ky * S + kx
  int32_t* sPh = sTapE + a.t.RS;                                       // taps of plane p: [sPh[p], sPh[p + 1])
  int32_t* sPhP = sPh + 5;                                             // plane p's parities 2 * py + px
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  uint64_t* wempty = wfull + kMaxWinStages;
  uint64_t* bfull = wempty + kMaxWinStages;
  uint64_t* bempty = bfull + kMaxBSlots;
  uint64_t* tfull = bempty + kMaxBSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(0);
#ifdef ICV_TRACE
  if (threadIdx.x == 0) g_icv_trace[blockIdx.x][62] = (unsigned long long)clock64();
#endif
  // TMA windows realize padding as out-of-bounds (zero-filled) pixels: only
  // valid when the bound zero row is all zeros.  The host certifies that
  // (zero_known) or the CTA checks it; otherwise the producers gather the
  // window with cp.async, reading the zero row for padding pixels (single
  // CTA only: the pair kernel is launched only with a certified zero row).
  int nonzero = 0;
  if (a.t.use_tma_x && !a.zero_known)
    for (int i = threadIdx.x; i < a.t.c_bytes / 16; i += blockDim.x) {
      const uint4 z = __ldg(reinterpret_cast<const uint4*>(a.t.zero_row) + i);
      nonzero |= (z.x | z.y | z.z | z.w) != 0;
    }
  const bool tma_win = a.t.use_tma_x && (a.zero_known ? true : !__syncthreads_or(nonzero));
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.wstages; ++s) {
      mbar_init(&wfull[s], tma_win ? 1 : 32 * kProdWarpsW);
      mbar_init(&wempty[s], 1);
    }
    for (int s = 0; s < pl.bslots; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int s = 0; s < C::kAS; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kCS * kEpiWarpsW);   // both CTAs' epilogue warps arrive at the leader
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmap_b);
  }
#ifndef ICV_WEXP_NODESCPF
  if (warp == 1 && lane < kMaxWR && lane < (a.WR2 > a.WR ? a.WR2 : a.WR)) tma_prefetch_desc(&maps.m[lane]);
#endif
  if constexpr (kI8) {
    if (threadIdx.x < 128) {   // all-ones B tile (16 rows x 128 bytes): per-pixel input sums
      reinterpret_cast<uint4*>(sOnes)[threadIdx.x] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
      fence_proxy_async_smem();
    }
  }
  const int nph = kS2 ? a.nph : 1;
  if constexpr (!kS2) {
    for (int e = threadIdx.x; e < a.t.RS; e += blockDim.x) {
      const int ky = e / a.S, kx = e - ky * a.S;
      sTap[e] = ky * a.DY * a.Wp + kx * a.DX;
    }
  } else if (threadIdx.x == 0) {
    // taps grouped by input plane.  Stride 1: one plane, off(e) = ky*DY*Wp +
    // kx*DX.  Stride 2: tap (ky, kx) reads plane (py, px) at row qy + Zr and
    // column qx + Zc past the output pixel, ky*DY - PT = 2*qy + py (floor),
    // kx*DX - PL = 2*qx + px.
    int i = 0;
    for (int p = 0; p < a.nph; ++p) {
      sPh[p] = i;
      for (int e = 0; e < a.t.RS; ++e) {
        const int ky = e / a.S, kx = e - ky * a.S;
        int off, ph = 0;
        if (a.sy == 1) {
          off = ky * a.DY * a.Wp + kx * a.DX;
        } else {
          const int ay = ky * a.DY - a.PT, ax = kx * a.DX - a.PL;
          const int qy = ay >= 0 ? ay / 2 : -((1 - ay) / 2), qx = ax >= 0 ? ax / 2 : -((1 - ax) / 2);
          ph = 2 * (ay - 2 * qy) + (ax - 2 * qx);
          off = (qy + a.Zr) * a.Wp + qx + a.Zc;
        }
        if (ph == a.php[p]) {
          sTap[i] = off;
          sTapE[i] = e;
          ++i;
        }
      }
    }
    sPh[a.nph] = i;
#pragma unroll
    for (int p = 0; p < 4; ++p) sPhP[p] = a.php[p];
  }
  if (warp == kMmaWarpW) {
    if constexpr (kCS == 2) tmem_alloc2<C::kTmemCols>(tmem_slot);
    else tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (kCS > 1) cluster_sync_all();   // the peer's barriers exist before any remote signal
  else __syncthreads();
  tc_fence_after();
  const int cblocks = a.t.cblocks;
  const int RS = a.t.RS;
  const uint32_t sWin_u32 = smem_u32(sWin);
  const uint32_t sB_u32 = smem_u32(sB);
  const int32_t row_bytes = a.Wp * 128;   // one plane row of one channel block

  // resident filter: K-block slot `slot` = (channel block cb, tap e) of this CTA's rows
  auto load_filter_slot = [&](int slot) {
    const int cb = slot / RS, e = slot - cb * RS;
    if (crank == 0) mbar_arrive_expect_tx(&bfull[slot], kCS * C::kBBytes);
    if constexpr (kCS == 2)
      tma_load_3d_cg2(sB_u32 + slot * C::kBBytes, &tmap_b, mapa_rank(smem_u32(&bfull[slot]), 0), 0,
                      (int)crank * (BN / kCS), e * cblocks + cb);
    else
      tma_load_3d(sB_u32 + slot * C::kBBytes, &tmap_b, &bfull[slot], 0, 0, e * cblocks + cb);
  };
  // Filter-block issue order (the producer loop below and the pre-issue):
  // TMA windows -- the producer warps past the window issuers load filter
  // blocks round-robin over the ring sequence fq (at most bslots threads, so
  // a slot's parity wait is never more than one phase ahead; lanes
  // 0 .. filt_lanes-1 of each such warp issue independently).
  const int nfilt = tma_win ? min((kProdWarpsW - a.win_split) * a.filt_lanes, pl.bslots) : 1;
  const int fidx = tma_win ? (warp - a.win_split) * a.filt_lanes + lane : 0;
  const bool filt_thread = warp < kProdWarpsW &&
                           (tma_win ? (lane < a.filt_lanes && warp >= a.win_split && fidx < nfilt) : threadIdx.x == 0);
  // The filter is not written by the previous kernel, so the first unit's
  // filter blocks (the whole filter when it is resident; otherwise the first
  // ring pass) are requested before griddep_wait: under programmatic
  // dependent launch they land while the previous kernel drains.
  int64_t pre_fq = 0;   // ring blocks issued before the wait (non-resident)
  if (filt_thread && cid < a.units) {
    const int32_t nt0 = cid % a.t.n_tiles;
    int64_t fq = 0;
    for (int st = 0; st < cblocks * nph && fq < (pl.resident ? (int64_t)1 << 40 : (int64_t)pl.bslots); ++st) {
      const int cb = kS2 ? st / nph : st, pi = kS2 ? st - cb * nph : 0;
      for (int i = kS2 ? sPh[pi] : 0; i < (kS2 ? sPh[pi + 1] : RS); ++i, ++fq) {
        if (!pl.resident && fq >= pl.bslots) break;
        if ((int)(fq % nfilt) != fidx) continue;
        const int e = kS2 ? sTapE[i] : i;
        if (pl.resident) {
          load_filter_slot(cb * RS + e);
        } else {
          const int bs = (int)fq;   // first ring pass: slot fq, phase 0 (free)
          if (crank == 0) mbar_arrive_expect_tx(&bfull[bs], kCS * C::kBBytes);
          if constexpr (kCS == 2)
            tma_load_3d_cg2(sB_u32 + bs * C::kBBytes, &tmap_b, mapa_rank(smem_u32(&bfull[bs]), 0), 0,
                            nt0 * BN + (int)crank * (BN / kCS), e * cblocks + cb);
          else
            tma_load_3d(sB_u32 + bs * C::kBBytes, &tmap_b, &bfull[bs], 0, nt0 * BN, e * cblocks + cb);
        }
      }
    }
    pre_fq = pl.resident ? 0 : (fq < pl.bslots ? fq : pl.bslots);
  }
  griddep_wait();   // (setup read only constants; tensors may belong to the previous kernel)
  griddep_launch_dependents();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);
  if (warp < kProdWarpsW) {
    // ------------------------------------------------------------ producers
    // TMA windows: lane 0 of warps 0 .. win_split-1 each load a share of
    // the window's rows, and lane 0 of the last producer warp loads the
    // filter blocks -- separate threads, because one thread's TMA loads are
    // served one after another (~450 cycles each, tools/micro/tma_rate.cu)
    // and a window must not queue behind filter loads waiting for free slots
    // (nor the reverse).  cp.async windows: all producer threads gather,
    // thread 0 loads the filter.  (An idle thread must not trail the barrier
    // phases it waits on, hence the exits.)
    // TMA windows: the producer warps past the window issuers all load filter
    // blocks, taking the stage's taps round-robin (each filter block is one
    // TMA load of BN / kCS rows, so at ~450 cycles per load one thread would
    // cap a stage at RS loads * 450 cycles).
    const bool win_thread = !tma_win || (lane == 0 && warp < a.win_split);
    if (!win_thread && !filt_thread) goto done;
    {
      int ws = 0;
      uint32_t wph = 0;
      int64_t fq = 0;   // filter blocks issued so far by all filter threads (ring sequence)
      int uk = 0;
      for (int32_t u = cid; u < a.units; u += ncl, ++uk) {
        if (threadIdx.x == 0 && uk < 8) TRACE(26 + uk);
        const int32_t nt = u % a.t.n_tiles;
        const UnitTiles ut = unit_tiles<kCS>(a, u, crank);
        const WinTile tw = win_tile(a, ut.first);
        const int32_t rows = ut.cnt == 2 ? a.WR2 : a.WR;   // window of this CTA's tiles
        // pair: shift the window so this CTA's first tile starts at the leader's column
        const int32_t shift = kCS > 1 ? (win_tile(a, ut.lead).rel0 - tw.rel0) * 128 : 0;
        // L2 prefetch of the NEXT unit's window (all channel blocks): its TMA
        // loads then hit L2 instead of waiting on HBM behind this unit's MMAs
        if (threadIdx.x == 0 && u + ncl < a.units && !kNoPrefetch) prefetch_window(a, unit_tiles<kCS>(a, u + ncl, crank));
        for (int st = 0; st < cblocks * nph; ++st) {   // stages: (channel block, input plane)
          const int cb = kS2 ? st / nph : st, pi = kS2 ? st - cb * nph : 0;
          const int py = kS2 ? sPhP[pi] >> 1 : 0, px = kS2 ? sPhP[pi] & 1 : 0;
          if (!win_thread) {
            // (filter thread only)
          } else {
          mbar_wait(&wempty[ws], wph ^ 1);
          if (threadIdx.x == 0 && uk < 4 && st < 2) TRACE(64 + uk * 2 + st);
          const uint32_t wbase = sWin_u32 + ws * pl.win_stage + a.win_lead;
          if (tma_win) {
            // completion of both CTAs' windows is counted at the leader
            if (crank == 0 && threadIdx.x == 0) mbar_arrive_expect_tx(&wfull[ws], kCS * rows * row_bytes);
            const uint32_t bar = kCS > 1 ? mapa_rank(smem_u32(&wfull[ws]), 0) : smem_u32(&wfull[ws]);
            // this thread's share of the rows; one box per image block it touches
            const int32_t r0 = rows * warp / a.win_split, r1 = rows * (warp + 1) / a.win_split;
            int32_t g = tw.g0 + r0;
            const int32_t gend = tw.g0 + r1;
            uint32_t dst = wbase + shift + r0 * row_bytes;
            while (g < gend) {
              const int32_t n = g / a.Hz;
              const int32_t r = g - n * a.Hz;          // row inside the image block
              const int32_t h = min(gend - g, a.Hz - r);
              const CUtensorMap* m = &maps.m[h - 1];
              // stride 2: plane row r is input row 2 (r - Zr) + py, plane column
              // c input column 2 (c - Zc) + px (the maps step 2 in W and H)
              const int32_t cx = !kS2 ? -a.Zc : px - 2 * a.Zc;
              const int32_t cy = !kS2 ? r - a.Zr : 2 * (r - a.Zr) + py;
              if constexpr (kCS == 2)
                tma_load_4d_cg2(dst, m, bar, cb * a.cbe, cx, cy, n);
              else
                tma_load_4d(dst, m, &wfull[ws], cb * a.cbe, cx, cy, n);
              dst += h * row_bytes;
              g += h;
            }
          } else {
            // cp.async window gather: 8 lanes per 128-byte pixel block, written
            // in the TMA 128-byte swizzle; padding pixels read the zero row
            const int positions = rows * a.Wp;
            const int chunk = threadIdx.x & 7;
            const int cofs = cb * 128 + chunk * 16;
            int valid_bytes = a.t.c_bytes - cofs;
            valid_bytes = valid_bytes < 0 ? 0 : (valid_bytes > 16 ? 16 : valid_bytes);
            for (int r = threadIdx.x >> 3; r < positions; r += 32 * kProdWarpsW / 8) {
              const int row = r / a.Wp;
              const int g = tw.g0 + row;
              const int n = g / a.Hz;
              const int iy = g - n * a.Hz - a.Zr;
              const int ix = r - row * a.Wp - a.Zc;
              const bool inside = n < a.batch && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
              const uint8_t* src = inside ? a.t.x + ((((int64_t)n * a.H + iy) * a.W + ix) * a.t.c_bytes + cofs)
                                          : a.t.zero_row + cofs;
              cp_async_16(wbase + r * 128 + ((chunk ^ (r & 7)) << 4), valid_bytes ? src : a.t.x, (uint32_t)valid_bytes);
            }
            cp_async_mbar_arrive_noinc(&wfull[ws]);
          }
          if (++ws == pl.wstages) { ws = 0; wph ^= 1; }
          }
          // this CTA's rows of the filter blocks of this stage, one per tap
          // (resident filter: loaded during the first unit only)
          if (filt_thread && pl.resident) {
            // (resident: every slot was requested before griddep_wait)
          } else if (filt_thread) {
            for (int i = kS2 ? sPh[pi] : 0; i < (kS2 ? sPh[pi + 1] : RS); ++i, ++fq) {
              if ((int)(fq % nfilt) != fidx || fq < pre_fq) continue;
              const int e = kS2 ? sTapE[i] : i;
              const int bs = (int)(fq % pl.bslots);
              mbar_wait(&bempty[bs], (uint32_t)((fq / pl.bslots) & 1) ^ 1u);
              if (crank == 0) mbar_arrive_expect_tx(&bfull[bs], kCS * C::kBBytes);
              if constexpr (kCS == 2)
                tma_load_3d_cg2(sB_u32 + bs * C::kBBytes, &tmap_b, mapa_rank(smem_u32(&bfull[bs]), 0), 0,
                                nt * BN + (int)crank * (BN / kCS), e * cblocks + cb);
              else
                tma_load_3d(sB_u32 + bs * C::kBBytes, &tmap_b, &bfull[bs], 0, nt * BN, e * cblocks + cb);
            }
          }
        }
        if (threadIdx.x == 0 && uk < 8) { TRACE(40 + uk); TRACE(48 + uk); }
      }
    }
  } else if (warp == kMmaWarpW && crank == 0) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    constexpr uint32_t idesc = make_idesc<kI8>(kBM * kCS, BN);
    constexpr uint32_t idesc_ones = make_idesc<kI8>(kBM * kCS, 16);
    const uint64_t ones_desc = sw128_kmajor_desc(smem_u32(sOnes));
    int ws = 0, bs = 0, as = 0;
    uint32_t wph = 0, bph = 0, aph = 0;
    int uk = 0;
#ifdef ICV_TRACE
    long long c_wait_full = 0, c_wait_tempty = 0, c_begin = clock64();
#endif
    for (int32_t u = cid; u < a.units; u += ncl, ++uk) {
      const UnitTiles ut = unit_tiles<kCS>(a, u, 0);
      const int cnt = ut.cnt;
      const int32_t rel0 = win_tile(a, ut.lead).rel0;
#ifdef ICV_TRACE
      long long c0 = clock64();
#endif
      mbar_wait(&tempty[as], aph ^ 1);
#ifdef ICV_TRACE
      c_wait_tempty += clock64() - c0;
#endif
      tc_fence_after();
      const uint32_t d = tmem_base + as * C::kAccStage;
      for (int st = 0; st < cblocks * nph; ++st) {   // stages: (channel block, input plane)
        const int cb = kS2 ? st / nph : st, pi = kS2 ? st - cb * nph : 0;
        const bool last_stage = st == cblocks * nph - 1;
        mbar_wait(&wfull[ws], wph);
        if (lane == 0 && uk < 4 && st < 2) TRACE(72 + uk * 2 + st);
        tc_fence_after();
        // tile i of the unit: 128 window rows after tile i - 1
        uint64_t adesc[kMT];
#pragma unroll
        for (int i = 0; i < kMT; ++i)
          adesc[i] = sw128_kmajor_desc(sWin_u32 + ws * pl.win_stage + a.win_lead + (rel0 + i * kBM) * 128);
        const int i_beg = kS2 ? sPh[pi] : 0;
        const int i_end = kS2 ? sPh[pi + 1] : RS;
        // One elected lane issues the whole stage: per tap only the filter
        // slot's barrier (skipped for a resident filter after the first
        // unit: its slots are never reloaded), the descriptors and the MMAs
        // -- no per-tap warp reconvergence (the issue loop has to keep up
        // with 4 MMAs of N/2 cycles each per tap).
        if (elect_one()) {
          int bsl = bs;
          uint32_t bphl = bph;
          for (int ti = i_beg; ti < i_end; ++ti) {
            const int e = kS2 ? sTapE[ti] : ti;   // (stride 1: taps in order)
            const int bslot = pl.resident ? cb * RS + e : bsl;
            if (!pl.resident || uk == 0) {
#ifdef ICV_TRACE
              long long c1 = clock64();
#endif
              mbar_wait(&bfull[bslot], pl.resident ? 0u : bphl);
#ifdef ICV_TRACE
              c_wait_full += clock64() - c1;
              if (uk == 1 && st == 0 && ti - i_beg < 12) TRACE(96 + ti - i_beg);    // tap's filter block seen
#endif
              tc_fence_after();
            }
            const uint64_t toff = (uint64_t)(sTap[ti] * 8);   // (off(e) * 128 bytes) >> 4
            const uint64_t bdesc = sw128_kmajor_desc(sB_u32 + bslot * C::kBBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // 4 x 32-byte K steps per 128-byte block
              const uint32_t acc = (st | ti | k) != 0;
#pragma unroll
              for (int i = 0; i < kMT; ++i) {
                if (i >= cnt) break;
#ifndef ICV_WEXP_NOMMA   // experiment: no MMAs
                if constexpr (kCS == 1) {
                  tc_mma<kI8>(d + i * C::kAccTile, adesc[i] + toff + 2 * k, bdesc + 2 * k, idesc, acc);
                  if constexpr (kI8)
                    tc_mma<true>(d + i * C::kAccTile + BN, adesc[i] + toff + 2 * k, ones_desc + 2 * k, idesc_ones, acc);
                } else {
                  tc_mma2<kI8>(d + i * C::kAccTile, adesc[i] + toff + 2 * k, bdesc + 2 * k, idesc, acc);
                  if constexpr (kI8)
                    tc_mma2<true>(d + i * C::kAccTile + BN, adesc[i] + toff + 2 * k, ones_desc + 2 * k, idesc_ones, acc);
                }
#endif
              }
            }
            if constexpr (kCS == 1) {
              if (!pl.resident) tc_commit(&bempty[bsl]);
              if (ti == i_end - 1) {
                tc_commit(&wempty[ws]);
                if (last_stage) tc_commit(&tfull[as]);
              }
            } else {   // stage free / accumulators ready in both CTAs
              if (!pl.resident) tc_commit2_mc(&bempty[bsl], kMask);
              if (ti == i_end - 1) {
                tc_commit2_mc(&wempty[ws], kMask);
                if (last_stage) tc_commit2_mc(&tfull[as], kMask);
              }
            }
            if (++bsl == pl.bslots) { bsl = 0; bphl ^= 1; }
#ifdef ICV_TRACE
            if (uk == 1 && st == 0 && ti - i_beg < 12) TRACE(108 + ti - i_beg);   // tap's MMAs and commits issued
#endif
          }
        }
        __syncwarp();
        for (int ti = i_beg; ti < i_end; ++ti)   // (every lane keeps the slot counters)
          if (++bs == pl.bslots) { bs = 0; bph ^= 1; }
        if (lane == 0 && uk < 4 && st < 2) TRACE(80 + uk * 2 + st);
        if (++ws == pl.wstages) { ws = 0; wph ^= 1; }
      }
      if (lane == 0 && uk < 8) TRACE(2 + uk);
      if (++as == C::kAS) { as = 0; aph ^= 1; }
    }
#ifdef ICV_TRACE
    if (lane == 0) {
      g_icv_trace[blockIdx.x][34] = (unsigned long long)(clock64() - c_begin);
      g_icv_trace[blockIdx.x][35] = (unsigned long long)c_wait_full;
      g_icv_trace[blockIdx.x][36] = (unsigned long long)c_wait_tempty;
    }
#endif
  } else if (warp >= kProdWarpsW && warp < kMmaWarpW) {
    // ------------------------------------------------------------ epilogue
    // Two groups of 4 warps; warp w reads TMEM lane quarter (w % 4) = 32
    // rows.  A two-tile unit: group g takes M tile g (all columns); a
    // one-tile unit: group g takes column half g.  Per 32-column chunk:
    // tcgen05.ld, + bias / zero-point constants, bf16 cast or q31 requant,
    // stage the 32 rows in smem and store whole 16-byte pieces of the valid
    // rows (virtual pixel -> output pixel; junk rows / columns are never
    // stored).
    constexpr int kGroups = kEpiWarpsW / 4;
    constexpr int kOutRowBytes = kI8 ? 32 : 64;
    constexpr int kChunks16 = kOutRowBytes / 16;
    constexpr int kRowsPerPass = 32 / kChunks16;
    constexpr int eb = kI8 ? 1 : 2;
    static_assert(kMT <= kGroups, "epilogue groups");
    const int ew = warp - kProdWarpsW;
    const int grp = ew / 4;
    const int slot = warp & 3;
    uint8_t* stg = sEpi + ew * kEpiWarpBytesW;
    const bool vec_ok = kI8 ? (a.t.K & 15) == 0 : (a.t.K & 7) == 0;
    // epilogue constants (loaded here, off the producers' / MMA's critical path)
    for (int i = threadIdx.x - 32 * kProdWarpsW; i < a.t.n_pad; i += 32 * kEpiWarpsW)
      sBias[i] = __ldg(static_cast<const uint32_t*>(a.t.bias) + i);
    // u8 padding corrections: staged once when the layer has one N tile
    int32_t* sCorr = reinterpret_cast<int32_t*>(smem + pl.off_corr);
    const bool corr_staged = kI8 && a.tapcorr != nullptr && a.t.n_tiles == 1;
    if (corr_staged)
      for (int i = threadIdx.x - 32 * kProdWarpsW; i < a.t.RS * BN; i += 32 * kEpiWarpsW) {
        const int e = i / BN, n = i - e * BN;
        sCorr[i] = __ldg(a.tapcorr + (int64_t)e * a.t.n_pad + n);
      }
    named_bar_sync(kEpiBarId, 32 * kEpiWarpsW);
    const bool cls_mode = corr_staged && a.ncls > 0;
    if (cls_mode) {
      // per-class sums of the staged per-tap corrections, written in place
      // over the per-tap table (ncls <= RS, at most kClsPer entries a thread)
      constexpr int kClsPer = 16;
      const int R = a.t.RS / a.S;
      int32_t tmp[kClsPer];
#pragma unroll
      for (int j = 0; j < kClsPer; ++j) {
        const int idx = threadIdx.x - 32 * kProdWarpsW + j * 32 * kEpiWarpsW;
        tmp[j] = 0;
        if (idx < a.ncls * BN) {
          const int cl = idx / BN, n = idx - cl * BN;
          const int oy = border_rep(cl / a.cls_ncc, a.cls_tb, a.cls_ohb, a.cls_nr);
          const int ox = border_rep(cl % a.cls_ncc, a.cls_lb, a.cls_owb, a.cls_ncc);
          int32_t sum = 0;
          for (int ky = 0; ky < R; ++ky) {
            const int iy = oy * a.sy - a.PT + ky * a.DY;
            const bool row_out = iy < 0 || iy >= a.H;
            for (int kx = 0; kx < a.S; ++kx) {
              const int ix = ox * a.sy - a.PL + kx * a.DX;
              if (row_out || ix < 0 || ix >= a.W) sum += sCorr[(ky * a.S + kx) * BN + n];
            }
          }
          tmp[j] = sum;
        }
      }
      named_bar_sync(kEpiBarId, 32 * kEpiWarpsW);
#pragma unroll
      for (int j = 0; j < kClsPer; ++j) {
        const int idx = threadIdx.x - 32 * kProdWarpsW + j * 32 * kEpiWarpsW;
        if (idx < a.ncls * BN) sCorr[idx] = tmp[j];
      }
      named_bar_sync(kEpiBarId, 32 * kEpiWarpsW);
    }
    const uint32_t tempty_remote = kCS == 2 && crank != 0 ? mapa_rank(smem_u32(tempty), 0) : 0u;
    const int32_t img_px = a.Hz * a.Wp;   // virtual pixels per image
    int as = 0;
    uint32_t aph = 0;
    int uk = 0;
    for (int32_t u = cid; u < a.units; u += ncl, ++uk) {
      const int32_t nt = u % a.t.n_tiles;
      const UnitTiles ut = unit_tiles<kCS>(a, u, crank);
      const int cnt = ut.cnt;
      // this group's tile and columns
      const bool split_cols = cnt == 1;
      const int i = split_cols ? 0 : grp;
      const int cols_w = split_cols ? BN / kGroups : BN;
      const int col0 = split_cols ? grp * cols_w : 0;
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      if (ew == 0 && lane == 0 && uk < 8) TRACE(10 + uk);
      const int32_t my_tile = ut.first + i;
      if (!ut.stand_in && my_tile < a.tiles) {
        const WinTile tl = win_tile(a, my_tile);
        // this lane's row: virtual pixel q -> output pixel p (or -1)
        const int32_t q = tl.q0 + slot * 32 + lane;
        const int32_t n = q / img_px;
        const int32_t r = q - n * img_px;
        const int32_t oy = r / a.Wp;
        const int32_t ox = r - oy * a.Wp;
        const int32_t myp = (n < a.batch && oy < a.OH && ox < a.OW) ? (n * a.OH + oy) * a.OW + ox : -1;
        // u8 with zero-filled TMA windows: padded taps contributed x = 0
        // instead of the zero point; their per-channel correction is added below
        uint64_t oob = 0;
        const int32_t* clsCorr = sCorr;
        if (cls_mode)
          clsCorr = sCorr + (border_class(oy < a.OH ? oy : a.OH - 1, a.cls_tb, a.cls_ohb, a.cls_nr) * a.cls_ncc +
                             border_class(ox < a.OW ? ox : a.OW - 1, a.cls_lb, a.cls_owb, a.cls_ncc)) * BN;
        else if (kI8 && a.tapcorr != nullptr && myp >= 0)
          for (int e = 0; e < a.t.RS; ++e) {
            const int ky = e / a.S, kx = e - ky * a.S;
            const int iy = oy * a.sy - a.PT + ky * a.DY, ix = ox * a.sy - a.PL + kx * a.DX;
            if (iy < 0 || iy >= a.H || ix < 0 || ix >= a.W) oob |= 1ull << e;
          }
        // the rows this lane stores in each pass (fixed for the tile)
        uint8_t* rowptr[32 / kRowsPerPass];
#pragma unroll
        for (int pass = 0; pass < 32 / kRowsPerPass; ++pass) {
          const int32_t p = __shfl_sync(0xffffffffu, myp, pass * kRowsPerPass + lane / kChunks16);
          rowptr[pass] = p >= 0 ? static_cast<uint8_t*>(a.t.y) + (int64_t)p * a.t.K * eb + (lane % kChunks16) * 16
                                : nullptr;
        }
        const uint32_t taddr = tmem_base + ((uint32_t)(slot * 32) << 16) + as * C::kAccStage + i * C::kAccTile;
        int32_t rowsum = 0;
        if constexpr (kI8) {
          uint32_t rs;
          tmem_ld_32x32b_x1(taddr + BN, rs);
          tmem_ld_wait();
          rowsum = (int32_t)rs;
        }
        const int cols_left = a.t.K - nt * BN - col0;
#ifdef ICV_WEXP_NOEPI   // experiment: release accumulators without storing
        const int nchunks = 0;
        (void)cols_left;
#else
        const int nchunks = cols_left > 0 ? (min(cols_w, cols_left) + 31) / 32 : 0;
#endif
        uint32_t v[32];
        if (nchunks > 0) {
          tmem_ld_32x32b_x32(taddr + col0, v);
          tmem_ld_wait_regs(v);
        }
#pragma unroll 1
        for (int ci = 0; ci < nchunks; ++ci) {
          const int c = col0 + ci * 32;
          const int n0 = nt * BN + c;
          uint32_t vn[32];
          if (ci + 1 < nchunks) tmem_ld_32x32b_x32(taddr + c + 32, vn);
          uint32_t w[kI8 ? 8 : 16];
          if constexpr (!kI8) {
            const float4* bias4 = reinterpret_cast<const float4*>(sBias + n0);
#pragma unroll
            for (int qd = 0; qd < 8; ++qd) {
              const float4 b = bias4[qd];
              __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(v[4 * qd + 0]) + b.x,
                                                        __uint_as_float(v[4 * qd + 1]) + b.y);
              __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(v[4 * qd + 2]) + b.z,
                                                        __uint_as_float(v[4 * qd + 3]) + b.w);
              w[2 * qd] = *reinterpret_cast<uint32_t*>(&lo);
              w[2 * qd + 1] = *reinterpret_cast<uint32_t*>(&hi);
            }
          } else {
            const int4* cst4 = reinterpret_cast<const int4*>(sBias + n0);
            // exact mod 2^32: the true accumulator fits int32
            const uint32_t corr = 0u - (uint32_t)a.t.zw * (uint32_t)rowsum;
#pragma unroll
            for (int qd = 0; qd < 8; ++qd) {
              int4 b = cst4[qd];
              if (cls_mode) {
                const int4 t = reinterpret_cast<const int4*>(clsCorr + (n0 - nt * BN))[qd];
                b.x += t.x; b.y += t.y; b.z += t.z; b.w += t.w;
              }
              for (uint64_t m = oob; m != 0; m &= m - 1) {
                const int e = __ffsll((long long)m) - 1;
                const int4 t = corr_staged ? reinterpret_cast<const int4*>(sCorr + e * BN + (n0 - nt * BN))[qd]
                                           : __ldg(reinterpret_cast<const int4*>(a.tapcorr + (int64_t)e * a.t.n_pad + n0) + qd);
                b.x += t.x; b.y += t.y; b.z += t.z; b.w += t.w;
              }
              const int bb[4] = {b.x, b.y, b.z, b.w};
              uint32_t word = 0;
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const int32_t acc = (int32_t)(v[4 * qd + h] + (uint32_t)bb[h] + corr);
#ifndef ICV_WEXP_NOREQ
                word |= (uint32_t)requant_u8(acc, a.t.m0, a.t.shift, a.t.zo, a.t.qmin, a.t.qmax) << (8 * h);
#else   // experiment: no requantization (timing only)
                word |= ((uint32_t)acc & 0xFFu) << (8 * h);
#endif
              }
              w[qd] = word;
            }
          }
          const bool full = vec_ok && n0 + 32 <= a.t.K;
          if (kDirect && full) {
            // straight from registers: this lane's pixel row, 16-byte pieces
            // (no smem staging: the mainloop's MMAs need the smem bandwidth)
            if (myp >= 0) {
              uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(a.t.y) + (int64_t)myp * a.t.K * eb + n0 * eb);
#pragma unroll
              for (int qd = 0; qd < kChunks16; ++qd)
                dst[qd] = make_uint4(w[4 * qd], w[4 * qd + 1], w[4 * qd + 2], w[4 * qd + 3]);
            }
            if (ci + 1 < nchunks) {
              tmem_ld_wait_regs(vn);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = vn[j];
            }
            continue;
          }
          uint4* my = reinterpret_cast<uint4*>(stg + lane * kEpiRowBytes);
#pragma unroll
          for (int qd = 0; qd < kChunks16; ++qd)
            my[qd] = make_uint4(w[4 * qd], w[4 * qd + 1], w[4 * qd + 2], w[4 * qd + 3]);
          __syncwarp();
#pragma unroll
          for (int pass = 0; pass < 32 / kRowsPerPass; ++pass) {
            const int rr = pass * kRowsPerPass + lane / kChunks16;
            const int qd = lane % kChunks16;
            if (rowptr[pass] != nullptr) {
              const uint4 val = *reinterpret_cast<const uint4*>(stg + rr * kEpiRowBytes + qd * 16);
              uint8_t* dst = rowptr[pass] + n0 * eb;
              if (full) {
                *reinterpret_cast<uint4*>(dst) = val;
              } else {
                const int col = n0 + qd * (16 / eb);
                if (vec_ok && col + 16 / eb <= a.t.K) *reinterpret_cast<uint4*>(dst) = val;
                else if (col < a.t.K) store_partial(dst, val, (a.t.K - col) * eb);
              }
            }
          }
          __syncwarp();
          if (ci + 1 < nchunks) {
            tmem_ld_wait_regs(vn);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = vn[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {   // one arrival per epilogue warp, at the pair leader
        if (tempty_remote) mbar_arrive_remote_relaxed(tempty_remote + as * 8);
        else mbar_arrive(&tempty[as]);
      }
      if (ew == 0 && lane == 0 && uk < 8) TRACE(18 + uk);
      if (++as == C::kAS) { as = 0; aph ^= 1; }
    }
  }

done:
  tc_fence_before();
  __syncthreads();
#ifdef ICV_TRACE
  if (threadIdx.x == 0) { g_icv_trace[blockIdx.x][60] = (unsigned long long)clock64(); TRACE(61); }
#endif
  if constexpr (kCS > 1) cluster_sync_all();   // no peer still signals, writes or reads TMEM
  if (warp == kMmaWarpW) {
    tc_fence_after();
    if constexpr (kCS == 2) tmem_dealloc2<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}


// TMA (zero-filled) windows are exact for this call's zero row
bool tma_zero_ok(const ConvArgs& c) {
  return c.zero_known || (c.L.family == kFamTcU8 && c.zero_is_zp && c.L.tapcorr_off != 0 && c.g.RS() <= 64);
}

// Geometry of the window schedule (host).
struct WinGeom {
  int Zc, Zr, Hz, Wp, WR, WR2, tiles;
  double useful;   // stored output pixels / computed rows
  int sy, nph, php[4], g_shift, rel_shift;
};

// floor division by 2
static inline int fdiv2(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }

// Stride 2 (both directions): the batch is read as up to four phase planes
// (input rows of parity py, columns of parity px), each stacked like the
// stride-1 plane but on the OUTPUT grid: per image Hz = OH + (qy range) rows
// of Wp = OW + (qx range) positions; plane position (r, c) of image n holds
// input pixel (2 (r - Zr) + py, 2 (c - Zc) + px), zero outside the image.
// Virtual pixel q = (n Hz + oy) Wp + ox reads, at tap e, position q + off(e)
// of plane ph(e) (off(e) = (qy + Zr) Wp + qx + Zc): again one affine shift
// per tap, so the same sliding-descriptor mainloop applies plane by plane.
bool win_geom_s2(const ConvArgs& c, WinGeom* w) {
  const Geom& g = c.g;
  int qy0 = 1 << 30, qy1 = -(1 << 30), qx0 = 1 << 30, qx1 = -(1 << 30);
  bool used[4] = {false, false, false, false};
  for (int ky = 0; ky < g.R; ++ky)
    for (int kx = 0; kx < g.S; ++kx) {
      const int ay = ky * g.DY - g.PT, ax = kx * g.DX - g.PL;
      const int qy = fdiv2(ay), qx = fdiv2(ax);
      used[2 * (ay - 2 * qy) + (ax - 2 * qx)] = true;
      qy0 = qy < qy0 ? qy : qy0; qy1 = qy > qy1 ? qy : qy1;
      qx0 = qx < qx0 ? qx : qx0; qx1 = qx > qx1 ? qx : qx1;
    }
  w->sy = 2;
  w->nph = 0;
  for (int p = 0; p < 4; ++p)
    if (used[p]) w->php[w->nph++] = p;
  w->Zr = -qy0;
  w->Zc = -qx0;
  w->Hz = (int)g.OH + (qy1 - qy0);
  w->Wp = (int)g.OW + (qx1 - qx0);
  w->g_shift = 0;
  w->rel_shift = 0;
  if (w->Wp > 128) return false;   // (box width 2 Wp input columns <= 256)
  const int64_t span = (int64_t)(w->Wp - 1) + (kBM - 1) + (int64_t)(qy1 - qy0) * w->Wp + (qx1 - qx0) + 1;
  const int64_t wr = (span + w->Wp - 1) / w->Wp;
  const int64_t wr2 = (span + kBM + w->Wp - 1) / w->Wp;
  if (wr > kMaxWR || wr > 128) return false;
  w->WR = (int)wr;
  w->WR2 = (int)(wr2 <= kMaxWR && wr2 <= 128 ? wr2 : 0);
  const int64_t batch = c.P / (g.OH * g.OW);
  const int64_t vpx = ((batch - 1) * w->Hz + g.OH) * (int64_t)w->Wp;
  if (vpx >= (int64_t(1) << 30)) return false;
  w->tiles = (int)((vpx + kBM - 1) / kBM);
  w->useful = (double)c.P / ((double)w->tiles * kBM);
  return true;
}

bool win_geom(const ConvArgs& c, WinGeom* w) {
  const Geom& g = c.g;
  if (g.SY == 2 && g.SX == 2) return win_geom_s2(c, w);
  if (g.SY != 1 || g.SX != 1) return false;
  w->sy = 1;
  w->nph = 1;
  w->php[0] = 0;
  w->g_shift = (g.PT > g.PB ? g.PT : g.PB) - g.PT;
  w->rel_shift = (g.PL > g.PR ? g.PL : g.PR) - g.PL;
  w->Zc = g.PL > g.PR ? g.PL : g.PR;
  w->Zr = g.PT > g.PB ? g.PT : g.PB;
  w->Wp = (int)g.W + w->Zc;
  w->Hz = (int)g.H + w->Zr;
  if (w->Wp > 256) return false;
  // window rows: from the tile's first row to the last row its last pixel's
  // last tap reads (tile start column <= Wp - 1)
  const int64_t span = (int64_t)(w->Wp - 1) - g.PL + w->Zc + (kBM - 1) + (int64_t)(g.R - 1) * g.DY * w->Wp +
                       (int64_t)(g.S - 1) * g.DX + 1;
  const int64_t wr = (span + w->Wp - 1) / w->Wp;
  const int64_t wr2 = (span + kBM + w->Wp - 1) / w->Wp;   // two consecutive tiles
  if (wr > kMaxWR) return false;
  w->WR = (int)wr;
  w->WR2 = (int)(wr2 <= kMaxWR ? wr2 : 0);                  // 0: no two-tile units
  const int64_t batch = c.P / (g.OH * g.OW);
  const int64_t vpx = ((batch - 1) * w->Hz + g.OH) * (int64_t)w->Wp;   // virtual pixels up to the last stored one
  if (vpx >= (int64_t(1) << 30)) return false;
  w->tiles = (int)((vpx + kBM - 1) / kBM);
  w->useful = (double)c.P / ((double)w->tiles * kBM);
  return true;
}

// Window tensor maps (box heights 1..WR) of a bound input: cached, the
// encode costs host time and the input buffer of a layer rarely changes.
int window_maps(const ConvArgs& c, const WinGeom& w, WinMaps* out) {
  auto encode = get_tensor_map_encoder();
  if (!encode) return ICV_ERR_CUDA;
  const bool i8 = c.L.family == kFamTcU8;
  const int eb = i8 ? 1 : 2;
  const int64_t batch = c.P / (c.g.OH * c.g.OW);
  using Key = std::tuple<const void*, int64_t, int64_t, int64_t, int64_t, int, int, int, int>;
  static std::mutex mu;
  static std::map<Key, WinMaps> cache;
  const Key key{c.x, (int64_t)c.g.C, c.g.W, c.g.H, batch, w.Wp, w.WR2 > w.WR ? w.WR2 : w.WR, eb, w.sy};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return ICV_OK;
  }
  const cuuint64_t dims[4] = {(cuuint64_t)c.g.C, (cuuint64_t)c.g.W, (cuuint64_t)c.g.H, (cuuint64_t)batch};
  const cuuint64_t strides[3] = {(cuuint64_t)c.g.C * eb, (cuuint64_t)(c.g.W * c.g.C * eb),
                                 (cuuint64_t)(c.g.H * c.g.W * c.g.C * eb)};
  // stride 2: every other input column and row (one phase plane per load)
  const cuuint32_t estr[4] = {1, (cuuint32_t)w.sy, (cuuint32_t)w.sy, 1};
  WinMaps m;
  std::memset(&m, 0, sizeof(m));
  const int hmax = w.WR2 > w.WR ? w.WR2 : w.WR;
  for (int h = 1; h <= hmax; ++h) {
    const cuuint32_t box[4] = {(cuuint32_t)(128 / eb), (cuuint32_t)(w.sy * w.Wp), (cuuint32_t)(w.sy * h), 1};
    CUresult cr = encode(&m.m[h - 1], i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                         const_cast<void*>(c.x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return ICV_ERR_CUDA;
  }
  if (cache.size() > 256) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return ICV_OK;
}

// Pairing of a CTA pair's tiles: one-tile units pair tile t with t + D
// (D*128 = 0 mod Wp: the same window column, no shift); two-tile units pair
// consecutive tiles and shift the peer's window inside its slot.
int pair_stride(const WinGeom& w, int kmt, int kcs) {
  if (kcs == 1 || kmt == 2) return 0;
  int a = kBM, b = w.Wp;
  while (b) { const int t = a % b; a = b; b = t; }
  return w.Wp / a;
}
// window slot: [lead slack][rows][tail slack]; the slack (one plane row on
// each side, rounded) absorbs a shifted peer window
bool slot_slack(int kmt, int kcs) { return kcs > 1 && kmt == 2; }
int slot_lead(const WinGeom& w, int kmt, int kcs) { return slot_slack(kmt, kcs) ? (w.Wp * 128 + 1023) / 1024 * 1024 : 0; }
int slot_bytes(const WinGeom& w, int kmt, int kcs) {
  const int rows = kmt == 2 ? w.WR2 : w.WR;
  return (slot_lead(w, kmt, kcs) + rows * w.Wp * 128 + (slot_slack(kmt, kcs) ? w.Wp * 128 : 0) + 1023) / 1024 * 1024;
}

// resident filter: one-tile units, a single N tile, and every K block of
// this CTA's filter rows fits beside two window stages
template <bool kI8, int BN, int kMT, int kCS, bool kS2>
bool win_plan_for(const ConvArgs& c, const WinGeom& w, PlanW* pl, bool resident = false) {
  if (kMT == 2 && w.WR2 == 0) return false;
  if (resident && c.L.n_pad != BN) return false;
  return plan_win<kI8, BN, kMT, kCS, kS2>(slot_bytes(w, kMT, kCS), c.g.RS(), c.g.RS() * c.L.cblocks, c.L.n_pad, resident,
                                     pl);
}

template <bool kI8, int BN, int kMT, int kCS, bool kS2>
int launch_win(const ConvArgs& c, const WinGeom& w, cudaStream_t st, bool resident) {
  auto kernel = igemm_win_kernel<kI8, BN, kMT, kCS, kS2>;
  PlanW pl;
  if (!win_plan_for<kI8, BN, kMT, kCS, kS2>(c, w, &pl, resident))
    return fail(ICV_ERR_UNSUPPORTED, "window does not fit in shared memory");
  int max_clusters = 0;
  if (int s = kernel_setup(reinterpret_cast<const void*>(kernel), 232448, kCS, kThreadsW, &max_clusters)) return s;
  WinArgs a;
  fill_tc_args(c, BN, &a.t);
  CUtensorMap tmap_b;
  if (int s = make_filter_tmap(c, BN / kCS, 1, &tmap_b)) return s;
  WinMaps maps;
  a.t.use_tma_x = tune(kTuneWinTma) == 1 && window_maps(c, w, &maps) == ICV_OK;
  if (!a.t.use_tma_x) {
    if (kCS > 1) return fail(ICV_ERR_UNSUPPORTED, "window pair kernel needs TMA window maps");
    if (w.sy != 1) return fail(ICV_ERR_UNSUPPORTED, "stride-2 window kernel needs TMA window maps");
    std::memset(&maps, 0, sizeof(maps));   // unused (cp.async windows)
  }
  // zero-filled TMA windows are exact when the zero row is zeros, and for
  // uint8 also when it holds the input zero point (plus the per-tap correction)
  a.zero_known = tma_zero_ok(c);
  a.tapcorr = (kI8 && !c.zero_known && c.zero_is_zp && c.L.tapcorr_off)
                  ? reinterpret_cast<const int32_t*>(c.packed + c.L.tapcorr_off) : nullptr;
  a.ncls = 0;
  if (a.tapcorr != nullptr && tune(kTuneWinU8Cls) == 1) {
    // border classes (WinArgs): top rows iy0 < 0, bottom rows with the last tap row >= H
    const auto border = [&](int64_t O, int64_t I, int P, int span, int st, int* tb, int* ohb, int* n) {
      const int64_t t = std::min<int64_t>(O, (P + st - 1) / st);
      const int64_t first_bot = std::max<int64_t>(0, (I + P - span + st) / st);   // ceil((I + P - span + 1) / st)
      const int64_t b0 = std::max<int64_t>(t, std::min<int64_t>(O, first_bot));
      *tb = (int)t; *ohb = (int)b0; *n = (int)(t + (O - b0) + 1);
    };
    int nr, ncc;
    border(c.g.OH, c.g.H, c.g.PT, (c.g.R - 1) * c.g.DY + 1, w.sy, &a.cls_tb, &a.cls_ohb, &nr);
    border(c.g.OW, c.g.W, c.g.PL, (c.g.S - 1) * c.g.DX + 1, w.sy, &a.cls_lb, &a.cls_owb, &ncc);
    a.cls_nr = nr;
    a.cls_ncc = ncc;
    const int ncls = nr * ncc;
    if (ncls <= c.g.RS() && ncls * BN <= 16 * 32 * kEpiWarpsW && c.L.n_pad <= BN) a.ncls = ncls;
  }
  a.sy = w.sy;
  a.nph = w.nph;
  for (int p = 0; p < 4; ++p) a.php[p] = p < w.nph ? w.php[p] : 0;
  a.g_shift = w.g_shift;
  a.rel_shift = w.rel_shift;
  a.win_split = tune(kTuneWinSplit);
  a.filt_lanes = tune(kTuneWinFiltLanes) < 1 ? 1 : (tune(kTuneWinFiltLanes) > 8 ? 8 : tune(kTuneWinFiltLanes));
  if (a.win_split < 1) a.win_split = 1;
  if (a.win_split > kProdWarpsW) a.win_split = kProdWarpsW;
  if (a.win_split > w.WR) a.win_split = w.WR;
  a.H = (int32_t)c.g.H; a.W = (int32_t)c.g.W; a.OH = (int32_t)c.g.OH; a.OW = (int32_t)c.g.OW;
  a.S = c.g.S; a.DY = c.g.DY; a.DX = c.g.DX; a.PT = c.g.PT; a.PL = c.g.PL;
  a.Zc = w.Zc; a.Zr = w.Zr; a.Hz = w.Hz; a.Wp = w.Wp; a.WR = w.WR; a.WR2 = w.WR2;
  a.batch = (int32_t)(c.P / (c.g.OH * c.g.OW));
  a.tiles = w.tiles;
  a.dpair = pair_stride(w, kMT, kCS);
  int64_t pair_tiles;
  if (a.dpair > 0) {
    const int64_t blk = 2 * (int64_t)a.dpair, full = w.tiles / blk, rest = w.tiles - full * blk;
    pair_tiles = full * a.dpair + (rest < a.dpair ? rest : a.dpair);
  } else {
    pair_tiles = (w.tiles + kCS - 1) / kCS;
  }
  const int sms = sm_count();
  int64_t clusters = sms / kCS;
  if (kCS > 1 && max_clusters > 0 && clusters > max_clusters) clusters = max_clusters;
  // two-tile units while at least two rounds of work remain, one-tile units
  // in the last round (each cluster then ends within one tile-time of the rest)
  int64_t two = 0, one = 0, rem = pair_tiles;
  const int64_t per_round = clusters / a.t.n_tiles > 0 ? clusters / a.t.n_tiles : 1;
  if (kMT == 2) {
    while (rem > 0) {
      if (rem >= 2 * per_round) { two += per_round; rem -= 2 * per_round; }
      else if (rem > per_round) { two += rem - per_round; one += 2 * per_round - rem; rem = 0; }
      else { one += rem; rem = 0; }
    }
  } else {
    one = rem;
  }
  a.two_units = (int32_t)two;
  a.units = (int32_t)((two + one) * a.t.n_tiles);
  a.cbe = 128 / a.t.elem_bytes;
  a.win_lead = slot_lead(w, kMT, kCS);
  if (clusters > a.units) clusters = a.units;
  if (tune(kTuneWinDebug))
    fprintf(stderr, "igemm_win: BN %d MT %d CS %d S2 %d resident %d wstages %d bslots %d win_stage %d smem %d | "
                    "Wp %d Hz %d WR %d WR2 %d tiles %d units %d (two %d) clusters %lld split %d\n",
            BN, kMT, kCS, (int)kS2, pl.resident, pl.wstages, pl.bslots, pl.win_stage, pl.bytes, w.Wp, w.Hz, w.WR, w.WR2,
            w.tiles, a.units, a.two_units, (long long)clusters, a.win_split);
  return launch_conv_kernel(kernel, (unsigned)(clusters * kCS), kThreadsW, pl.bytes, st, kCS, "igemm_win launch", tmap_b,
                            maps, a, pl);
}


template <bool kI8, int BN, int kMT>
constexpr bool mt_fits() {
  return 2 * kMT * (kI8 ? 2 * BN : BN) <= 512;
}

// dispatch on (dtype, BN, kMT, kCS); `launch` false: only check the plan
template <bool kI8, int BN, bool kS2>
int dispatch_bn(const ConvArgs& c, const WinGeom& w, cudaStream_t st, bool launch) {
  PlanW pl;
  // CTA pairs need TMA windows, hence a zero row the host certifies
  const bool pair = tma_zero_ok(c) && tune(kTuneWinCs) == 2;
  const bool mt2 = tune(kTuneWinMt) == 2;
  const bool res = tune(kTuneWinRes) == 1;
  // preference: pair with two-tile units (measured fastest on every stride-1
  // layer: cfg2 25.5 vs 27.5 us resident, ResNet-50 s1 3x3 85 vs 121 us --
  // two tiles share each filter block and one window of WR2 rows), pair
  // with a resident filter, pair, then the single-CTA kernels
  if constexpr (mt_fits<kI8, BN, 2>()) {
    // two-tile units with the filter resident (one N tile whose blocks fit
    // beside the windows: the C = K = 64 / 128 layers) load no filter block
    // after the first unit
    if (pair && mt2 && res && win_plan_for<kI8, BN, 2, 2, kS2>(c, w, &pl, true))
      return launch ? launch_win<kI8, BN, 2, 2, kS2>(c, w, st, true) : ICV_OK;
    if (pair && mt2 && win_plan_for<kI8, BN, 2, 2, kS2>(c, w, &pl))
      return launch ? launch_win<kI8, BN, 2, 2, kS2>(c, w, st, false) : ICV_OK;
  }
  if (pair && res && win_plan_for<kI8, BN, 1, 2, kS2>(c, w, &pl, true))
    return launch ? launch_win<kI8, BN, 1, 2, kS2>(c, w, st, true) : ICV_OK;
  if (pair && win_plan_for<kI8, BN, 1, 2, kS2>(c, w, &pl)) return launch ? launch_win<kI8, BN, 1, 2, kS2>(c, w, st, false) : ICV_OK;
  if constexpr (mt_fits<kI8, BN, 2>()) {
    if (mt2 && win_plan_for<kI8, BN, 2, 1, kS2>(c, w, &pl)) return launch ? launch_win<kI8, BN, 2, 1, kS2>(c, w, st, false) : ICV_OK;
  }
  if (res && win_plan_for<kI8, BN, 1, 1, kS2>(c, w, &pl, true))
    return launch ? launch_win<kI8, BN, 1, 1, kS2>(c, w, st, true) : ICV_OK;
  if (win_plan_for<kI8, BN, 1, 1, kS2>(c, w, &pl)) return launch ? launch_win<kI8, BN, 1, 1, kS2>(c, w, st, false) : ICV_OK;
  return ICV_ERR_UNSUPPORTED;
}

template <bool kS2>
int dispatch_win_s(const ConvArgs& c, const WinGeom& w, cudaStream_t st, bool launch) {
  int bn = c.L.block_n;
  // uint8 with 256 output channels: one N tile of 256 (the TMEM layout keeps
  // 32 columns for the row sums, one accumulator stage)
  if (c.L.family == kFamTcU8 && c.L.n_pad == 256 && tune(kTuneWinU8Bn) == 256) bn = 256;
  if (c.L.family == kFamTcBf16) {
    if (bn == 64) return dispatch_bn<false, 64, kS2>(c, w, st, launch);
    if (bn == 128) return dispatch_bn<false, 128, kS2>(c, w, st, launch);
    if (bn == 256) return dispatch_bn<false, 256, kS2>(c, w, st, launch);
  } else if (c.L.family == kFamTcU8) {
    if (bn == 64) return dispatch_bn<true, 64, kS2>(c, w, st, launch);
    if (bn == 128) return dispatch_bn<true, 128, kS2>(c, w, st, launch);
    if (bn == 256) return dispatch_bn<true, 256, kS2>(c, w, st, launch);
  }
  return ICV_ERR_UNSUPPORTED;
}

int dispatch_win(const ConvArgs& c, const WinGeom& w, cudaStream_t st, bool launch) {
  return w.sy == 2 ? dispatch_win_s<true>(c, w, st, launch) : dispatch_win_s<false>(c, w, st, launch);
}

}  // namespace

// The window kernel takes a stride-1 tensor-core layer when the call
// certifies a canonical buffer, the window geometry fits, and at least
// win_min_useful_pm / 1000 (default 0.7) of the computed rows are real
// output pixels.  Knob win = 0 or the call flag ICV_PREFER_GATHER disable it
// (tap-by-tap IB-gather kernel); win = 1 forces it whenever it fits.
bool win_kernel_eligible(const ConvArgs& c) {
  const int mode = tune(kTuneWin);
  if (mode == 0 || c.prefer_gather) return false;
  if (!c.ib_canonical) return false;
  if (c.L.family != kFamTcBf16 && c.L.family != kFamTcU8) return false;
  if (c.L.n_pad > kMaxBias) return false;
  if (c.P >= (int64_t(1) << 31)) return false;
  if ((reinterpret_cast<uintptr_t>(c.x) & 15) != 0) return false;
  // 1x1 layers have no tap re-reads for the window to save; measured slower
  // than the gather kernel on every ResNet-50 1x1 (profiles/r01d_cfg5_layers.json)
  if (c.g.R * c.g.S == 1 && mode != 1) return false;
  WinGeom w;
  if (!win_geom(c, &w)) return false;
  if (w.sy == 2 && !tma_zero_ok(c)) return false;   // (no cp.async phase-plane gather)
  // Opt-in only (win = 1, or win_s2 = 1 / win_u8 = 1), measured slower
  // than the gather kernel today: stride-2 phase planes (ResNet-50 s2b1 3x3
  // 115 vs 84 us, s3b1 88 vs 60 us) and the uint8 epilogue (cfg4 85 vs 41 us).
  const bool forced = mode == 1;
  if (w.sy == 2 && !forced && tune(kTuneWinS2) != 1) return false;
  if (c.L.family == kFamTcU8 && !forced && tune(kTuneWinU8) != 1) return false;
  const double min_useful = forced ? 0.0 : tune(kTuneWinMinUsefulPm) / 1000.0;
  if (w.useful < min_useful) return false;
  return dispatch_win(c, w, nullptr, false) == ICV_OK;
}

int launch_conv_win(const ConvArgs& c, cudaStream_t st) {
  WinGeom w;
  if (!win_geom(c, &w)) return fail(ICV_ERR_UNSUPPORTED, "window kernel: geometry not supported");
  const int s = dispatch_win(c, w, st, true);
  if (s == ICV_ERR_UNSUPPORTED) return fail(ICV_ERR_UNSUPPORTED, "window kernel: no plan for this layer");
  return s;
}

}  // namespace icv
