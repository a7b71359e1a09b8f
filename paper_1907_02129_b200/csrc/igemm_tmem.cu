// K2/K3: indirect-GEMM mainloop on sm_100a tensor cores with the gathered A
// operand staged in TENSOR memory ("kernel T").
//
// Why: with the A tile in shared memory (igemm_tc.cu) every 128-byte K block
// costs 16 KB of smem writes (the gather) plus 16 KB of smem reads (the MMA)
// on top of the filter tile, and the cp.async -> mbarrier -> MMA round trip
// puts the full L2 latency on the critical path of every ring slot.  Here the
// producers gather pixel rows through the indirection buffer into REGISTERS
// (prefetched two K blocks ahead, decoupled from slot availability) and write
// them into TMEM with tcgen05.st; tcgen05.mma then reads A from TMEM
// (`[a_tmem]` operand) and only the packed filter (B) streams through smem via
// TMA.  TMEM budget (512 columns): two accumulator stages (2 x BLOCK_N, plus
// 16 row-sum columns each for uint8) and up to eight 32-column A slots.
//
// Warp roles (416 threads, one persistent CTA per SM):
//   warps 0-7  producers.  Warp w gathers the 32 rows of TMEM lane quarter
//              w%4; warps 0-3 fill the first K block of each 2-block stage,
//              warps 4-7 the second; each prefetches two of its K blocks
//              ahead in registers (6 K blocks in flight per SM).  Per tile the
//              CTA's slice of the
//              indirection buffer (128 pixels x R*S taps, indirect.py:14-16)
//              is copied into smem one tile ahead; a thread resolves the row
//              references of its 4 rows (ZERO_REF -> bound zero row,
//              indirect.py:291) and loads 4 x 32 bytes of each row per K
//              block (8-byte pieces; 4 lanes cover one 32-byte sector).
//   warps 8-11 epilogue (igemm_common.cuh).
//   warp 12    TMEM allocation and MMA issue (one elected lane).
#include "igemm_common.cuh"

namespace icv {
namespace {

constexpr int kProdWarpsT = 8;
constexpr int kEpiWarp0T = 8;
constexpr int kEpiWarpsT = 4;
constexpr int kMmaWarpT = 12;
constexpr int kThreadsT = 32 * (kMmaWarpT + 1);
constexpr int kMaxRST = 16;      // taps whose per-tile buffer slice fits in smem
constexpr int kMinKBT = 8;       // tile-ahead index staging needs >= 4 stage uses per tile

template <bool kI8, int BN, typename IbT>
struct CfgT {
  static constexpr int kAccStride = kI8 ? BN + 16 : BN;   // + per-pixel row-sum columns (uint8)
  static constexpr int kAccCols = 2 * kAccStride;
  static constexpr int kASlotsRaw = (512 - kAccCols) / 32;
  static constexpr int kKB = 2;                            // K blocks per stage (one barrier round trip)
  static constexpr int kSlots = (kASlotsRaw > 8 ? 8 : kASlotsRaw) / kKB * kKB;
  static constexpr int kStages = kSlots / kKB;
  static constexpr int kABase = kAccCols;                  // first TMEM column of A slot 0
  static constexpr int kBBytes = BN * 128;
  static constexpr int kOnesBytes = kI8 ? 16 * 128 : 0;
  static constexpr int kIbBytes = kMaxRST * kBM * (int)sizeof(IbT);   // one tile's index slice
  static constexpr int kEpiBytes = kEpiWarpsT * kEpiWarpBytes<kI8>;
  static constexpr int kBiasBytes = 4 * kMaxBias;
  static constexpr int kBarBytes = 256;
  static constexpr int kSmemBytes =
      1024 + kSlots * kBBytes + kOnesBytes + 2 * kIbBytes + kEpiBytes + kBiasBytes + kBarBytes;
  static_assert(kStages >= 2, "too few A slots");
  static_assert(kABase + kSlots * 32 <= 512, "TMEM overflow");
  static_assert(kSmemBytes <= 232448, "shared memory overflow");
};

// One K block of the 4 rows a producer thread owns: 4 rows x 4 pieces of 8 bytes.
struct ARegs {
  uint2 v[4][4];
};

template <bool kI8, int BN, typename IbT>
__global__ void __launch_bounds__(kThreadsT, 1) igemm_tmem_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                                  const TcArgs a) {
  using C = CfgT<kI8, BN, IbT>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base (SW128 atoms); pointer arithmetic keeps the
  // shared address space visible to the compiler (no generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;
  uint8_t* sOnes = sB + C::kSlots * C::kBBytes;
  IbT* sIB = reinterpret_cast<IbT*>(sOnes + C::kOnesBytes);              // [2][kMaxRST][128]
  uint8_t* sEpi = reinterpret_cast<uint8_t*>(sIB) + 2 * C::kIbBytes;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(sEpi + C::kEpiBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sBias) + C::kBiasBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 32 * kProdWarpsT + 1);   // every producer thread + 1 expect_tx arrival
      mbar_init(&empty[s], 1);                     // tcgen05.commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarpsT);   // one arrival per epilogue warp
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmap_b);
  }
  if constexpr (kI8) {
    if (threadIdx.x >= 256 && threadIdx.x < 384) {  // all-ones B tile (16 rows x 128 bytes)
      reinterpret_cast<uint4*>(sOnes)[threadIdx.x - 256] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u,
                                                                      0x01010101u);
      fence_proxy_async_smem();
    }
  }
  for (int i = threadIdx.x; i < a.n_pad && i < kMaxBias; i += blockDim.x)
    sBias[i] = __ldg(static_cast<const uint32_t*>(a.bias) + i);
  if (warp == kMmaWarpT) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);
  const int num_kb = a.RS * a.cblocks;
  const int spt = (num_kb + C::kKB - 1) / C::kKB;   // stage uses per tile
  const uint32_t sB_u32 = smem_u32(sB);

  if (warp < kProdWarpsT) {
    // ------------------------------------------------------------ producers
    const int q = warp & 3;          // TMEM lane quarter (rows 32q .. 32q+31)
    const int h = warp >> 2;         // which K block of each 2-block stage
    const int t0 = lane & 3, t1 = lane >> 2;
    const int ptid = threadIdx.x;    // 0 .. 255
    const int64_t my_tiles = blockIdx.x < a.total_tiles ? (a.total_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int64_t total_items = my_tiles * spt;      // one item = one stage use (K block 2*si + h)
    const uint32_t sIB_u32 = smem_u32(sIB);

    // copy the (128 pixels x R*S taps) index slice of local tile k into buffer k&1
    auto stage_index_slice = [&](int64_t k) {
      if (k >= my_tiles) return;
      const int64_t tile = blockIdx.x + k * gridDim.x;
      const int64_t mt = tile / a.n_tiles;
      const uint32_t base = sIB_u32 + (uint32_t)((k & 1) * C::kIbBytes);
      for (int idx = ptid; idx < kBM * a.RS; idx += 32 * kProdWarpsT) {
        const int e = idx / kBM, row = idx - e * kBM;
        const int64_t ent = row_ref(a, mt, row).ent0 + (int64_t)e * a.mr;
        cp_async_ca<sizeof(IbT)>(base + (uint32_t)((e * kBM + row) * sizeof(IbT)), static_cast<const IbT*>(a.ib) + ent);
      }
    };
    auto issue = [&](int64_t n, ARegs& r) {
      if (n >= total_items) return;
      const int64_t k = n / spt;
      const int kb = 2 * (int)(n - k * spt) + h;
      if (kb >= num_kb) return;
      const int e = kb / a.cblocks, cb = kb - e * a.cblocks;
      const IbT* slice = sIB + (k & 1) * (C::kIbBytes / (int)sizeof(IbT)) + e * kBM;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 32 * q + 16 * (i >> 1) + 8 * (i & 1) + t1;
        const int64_t off = (int64_t)slice[row];
        const uint8_t* src = off < 0 ? a.zero_row : a.x + off * a.elem_bytes;   // ZERO_REF -> bound zero row
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int b = cb * 128 + 32 * p + 8 * t0;
          r.v[i][p] = b + 8 <= a.c_bytes ? __ldg(reinterpret_cast<const uint2*>(src + b)) : make_uint2(0u, 0u);
        }
      }
    };
    auto commit = [&](int64_t n, const ARegs& r) {
      if (n >= total_items) return;
      const int64_t k = n / spt;
      const int si = (int)(n - k * spt);
      const int kb = 2 * si + h;
      const int stage = (int)(n % C::kStages);
      const uint32_t phase = (uint32_t)((n / C::kStages) & 1);
      mbar_wait(&empty[stage], phase ^ 1);
      if (warp == 0 && lane == 0) {
        const int64_t tile = blockIdx.x + k * gridDim.x;
        const int nt = (int)(tile % a.n_tiles);
        const int nsub = min(C::kKB, num_kb - 2 * si);
        (void)nsub;
        mbar_arrive_expect_tx(&full[stage], C::kKB * C::kBBytes);   // tail blocks past the filter are zero-filled
        tma_load_3d(sB_u32 + stage * C::kKB * C::kBBytes, &tmap_b, &full[stage], 0, nt * BN, C::kKB * si);
      }
      if (kb < num_kb) {
        const uint32_t col = C::kABase + (uint32_t)(stage * C::kKB + h) * 32;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          uint32_t regs[16];
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            regs[4 * p + 0] = r.v[2 * g][p].x;
            regs[4 * p + 1] = r.v[2 * g][p].y;
            regs[4 * p + 2] = r.v[2 * g + 1][p].x;
            regs[4 * p + 3] = r.v[2 * g + 1][p].y;
          }
          tmem_st_16x256b_x4(tmem_base + ((uint32_t)(32 * q + 16 * g) << 16) + col, regs);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      mbar_arrive(&full[stage]);
    };
    auto before_item = [&](int64_t n) {
      if (n >= total_items) return;
      const int64_t k = n / spt;
      const int si = (int)(n - k * spt);
      if (si == 0) stage_index_slice(k + 1);
      if (si == spt - 2) {
        cp_async_wait_all();
        named_bar_sync(1, 32 * kProdWarpsT);
      }
    };

    stage_index_slice(0);
    cp_async_wait_all();
    named_bar_sync(1, 32 * kProdWarpsT);
    ARegs r0, r1, r2;
    issue(0, r0);
    issue(1, r1);
    for (int64_t n = 0; n < total_items; n += 3) {
      before_item(n);
      issue(n + 2, r2);
      commit(n, r0);
      before_item(n + 1);
      issue(n + 3, r0);
      commit(n + 1, r1);
      before_item(n + 2);
      issue(n + 4, r1);
      commit(n + 2, r2);
    }
  } else if (warp == kMmaWarpT) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc<kI8>(kBM, BN);
    constexpr uint32_t idesc_ones = make_idesc<kI8>(kBM, 16);
    const uint64_t ones_desc = sw128_kmajor_desc(smem_u32(sOnes));
    int stage = 0;
    uint32_t phase = 0;
    int as = 0;
    uint32_t aphase = 0;
    for (int64_t tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[as], aphase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + as * C::kAccStride;
      for (int si = 0; si < spt; ++si) {
        const int nsub = min(C::kKB, num_kb - si * C::kKB);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < nsub; ++j) {
            const int slot = stage * C::kKB + j;
            const uint32_t at = tmem_base + C::kABase + slot * 32;
            const uint64_t bdesc = sw128_kmajor_desc(sB_u32 + slot * C::kBBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x 32-byte K steps (8 TMEM columns each)
              const uint32_t acc = (si | j | k) != 0;
              tc_mma_ts<kI8>(d, at + 8 * k, bdesc + 2 * k, idesc, acc);
              if constexpr (kI8) tc_mma_ts<true>(d + BN, at + 8 * k, ones_desc + 2 * k, idesc_ones, acc);
            }
          }
          tc_commit(&empty[stage]);
          if (si == spt - 1) tc_commit(&tfull[as]);
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
  } else {
    epilogue_loop<kI8, BN, kEpiWarpsT, C::kAccStride>(a, warp - kEpiWarp0T, lane, tmem_base, sEpi, sBias, tfull,
                                                      tempty);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarpT) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

template <bool kI8, int BN, typename IbT>
int launch_tmem(const ConvArgs& c, cudaStream_t st) {
  using Cf = CfgT<kI8, BN, IbT>;
  auto kernel = igemm_tmem_kernel<kI8, BN, IbT>;
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [&] {
    attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return cuda_check(attr_err, "cudaFuncSetAttribute(smem)");
  CUtensorMap tmap;
  if (int s = make_filter_tmap(c, BN, Cf::kKB, &tmap)) return s;
  TcArgs a;
  fill_tc_args(c, BN, &a);
  const int sms = sm_count();
  const int grid = (int)(a.total_tiles < sms ? a.total_tiles : sms);
  kernel<<<grid, kThreadsT, Cf::kSmemBytes, st>>>(tmap, a);
  note_launch();
  return cuda_check(cudaGetLastError(), "igemm_tmem launch");
}

template <typename IbT>
int dispatch_tmem(const ConvArgs& c, cudaStream_t st) {
  const int bn = c.L.block_n;
  if (c.L.family == kFamTcBf16) {
    if (bn == 64) return launch_tmem<false, 64, IbT>(c, st);
    if (bn == 128) return launch_tmem<false, 128, IbT>(c, st);
  } else if (c.L.family == kFamTcU8) {
    if (bn == 64) return launch_tmem<true, 64, IbT>(c, st);
    if (bn == 128) return launch_tmem<true, 128, IbT>(c, st);
  }
  return fail(ICV_ERR_UNSUPPORTED, "no TMEM-A kernel for this tile width");
}

}  // namespace

bool tmem_kernel_eligible(const ConvArgs& c) {
  if (c.ib_per_image) return false;                    // canonical buffers only
  if (c.L.block_n > 128) return false;                 // two 256-column accumulators leave no TMEM for A
  if (c.g.RS() > kMaxRST) return false;                // per-tile index slice must fit in smem
  return c.g.RS() * c.L.cblocks >= kMinKBT;
}

int launch_conv_tmem(const ConvArgs& c, cudaStream_t st) {
  if (c.ib_is_i32) return dispatch_tmem<int32_t>(c, st);
  return dispatch_tmem<int64_t>(c, st);
}

}  // namespace icv
