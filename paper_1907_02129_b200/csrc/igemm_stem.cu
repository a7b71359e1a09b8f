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
#include "igemm_common.cuh"

namespace icv {
namespace {

constexpr int kEpiWarpsStem = 4;
constexpr int kMmaWarpStem = 8;
constexpr int kThreadsStem = 32 * (kMmaWarpStem + 1);
constexpr int kStagesStem = 3;

template <int C, int RS, int BN>
struct CfgStem {
  static constexpr int kK = RS * C;                         // real reduction length
  static constexpr int kKSteps = (kK + 15) / 16;            // MMA K steps (16 bf16 each)
  static constexpr int kBlocks = (kKSteps * 16 + 63) / 64;  // 128-byte K blocks per row
  static constexpr int kWords = kBlocks * 32;               // 32-bit words per A row
  static constexpr int kABytes = kBM * kBlocks * 128;       // one A tile
  static constexpr int kBBytes = BN * kBlocks * 128;        // resident filter
  static constexpr int kEpiBytes = kEpiWarpsStem * 32 * 80;
  static constexpr int kSmemBytes = 1024 + kStagesStem * kABytes + kBBytes + kEpiBytes + 4 * 256 + 256;
  static_assert(kSmemBytes <= 232448, "shared memory overflow");
  static_assert(C >= 1 && C <= 4, "channel-poor kernel handles 1..4 channels");
};

// 16-byte chunk q (elements 8q .. 8q+7) of row `row` in the swizzled A tile.
__device__ __forceinline__ uint32_t a_chunk_addr(uint32_t tile, int row, int q) {
  const int blk = q >> 3, j = q & 7;
  return tile + blk * (kBM * 128) + row * 128 + ((j ^ (row & 7)) << 4);
}

template <int C, int RS, int BN, typename IbT>
__global__ void __launch_bounds__(kThreadsStem, 1) igemm_stem_kernel(const __grid_constant__ CUtensorMap tmap_b,
                                                                     const TcArgs a, int64_t x_elems) {
  using Cf = CfgStem<C, RS, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStagesStem * Cf::kABytes;
  uint8_t* sEpi = sB + Cf::kBBytes;
  uint32_t* sBias = reinterpret_cast<uint32_t*>(sEpi + Cf::kEpiBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sBias) + 4 * 256);
  uint64_t* empty = full + kStagesStem;
  uint64_t* tfull = empty + kStagesStem;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesStem; ++s) {
      mbar_init(&full[s], 128);   // every producer thread (st.shared + proxy fence + arrive)
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

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    const int row = threadIdx.x;
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(a.x);
    const uint16_t* x16 = reinterpret_cast<const uint16_t*>(a.x);
    const uint16_t* z16 = reinterpret_cast<const uint16_t*>(a.zero_row);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
      const IbT* ref = static_cast<const IbT*>(a.ib) + first_entry(a, tile, row);
      int64_t offs[RS];
#pragma unroll
      for (int e = 0; e < RS; ++e) offs[e] = (int64_t)__ldg(ref + (int64_t)e * a.mr);
      mbar_wait(&empty[stage], phase ^ 1);
      const uint32_t tileA = sA_u32 + stage * Cf::kABytes;
      uint32_t w[Cf::kWords];
#pragma unroll
      for (int i = 0; i < Cf::kWords; ++i) w[i] = 0u;
#pragma unroll
      for (int e = 0; e < RS; ++e) {
        const int64_t off = offs[e];
        uint32_t h[C];
        if (off >= 0) {
          // C elements at element offset `off`: two aligned words + funnel shift
          const int64_t wi = off >> 1;
          const uint32_t w0 = __ldg(x32 + wi);
          uint32_t w1 = 0u;
          if (2 * (wi + 1) + 1 < x_elems) w1 = __ldg(x32 + wi + 1);
          else if (2 * (wi + 1) < x_elems) w1 = (uint32_t)__ldg(x16 + 2 * (wi + 1));
          const uint64_t v = ((uint64_t)w1 << 32 | w0) >> ((off & 1) * 16);
#pragma unroll
          for (int c = 0; c < C; ++c) h[c] = (uint32_t)(v >> (16 * c)) & 0xFFFFu;
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) h[c] = __ldg(z16 + c);    // ZERO_REF -> bound zero row
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int k = e * C + c;
          w[k >> 1] |= h[c] << (16 * (k & 1));
        }
        // flush the 16-byte chunks completed by this tap
        const int q_lo = e == 0 ? 0 : ((e * C) >> 3);
        const int q_hi = ((e + 1) * C) >> 3;   // chunks [q_lo, q_hi) are complete
#pragma unroll
        for (int q = q_lo; q < q_hi; ++q)
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a_chunk_addr(tileA, row, q)),
                       "r"(w[4 * q]), "r"(w[4 * q + 1]), "r"(w[4 * q + 2]), "r"(w[4 * q + 3]) : "memory");
      }
#pragma unroll
      for (int q = (RS * C) >> 3; q < Cf::kBlocks * 8; ++q)   // the partial last chunk and zero padding
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a_chunk_addr(tileA, row, q)),
                     "r"(w[4 * q]), "r"(w[4 * q + 1]), "r"(w[4 * q + 2]), "r"(w[4 * q + 3]) : "memory");
      fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
      mbar_arrive(&full[stage]);
      if (++stage == kStagesStem) { stage = 0; phase ^= 1; }
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
    epilogue_loop<false, BN, kEpiWarpsStem, BN>(a, warp - 4, lane, tmem_base, sEpi, sBias, tfull, tempty);
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
  auto kernel = igemm_stem_kernel<C, RS, BN, IbT>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [&] { err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmemBytes); });
  if (err != cudaSuccess) return cuda_check(err, "cudaFuncSetAttribute(stem smem)");
  CUtensorMap tmap;
  if (int s = make_filter_tmap(c, BN, &tmap)) return s;
  TcArgs a;
  fill_tc_args(c, BN, &a);
  const int sms = sm_count();
  const int grid = (int)(a.total_tiles < sms ? a.total_tiles : sms);
  kernel<<<grid, kThreadsStem, Cf::kSmemBytes, st>>>(tmap, a, c.g.N * c.g.H * c.g.W * (int64_t)c.g.C);
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
