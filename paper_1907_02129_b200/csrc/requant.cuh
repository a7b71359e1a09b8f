// Fixed-point requantization shared by the uint8 epilogues (K6).
// gemmlowp / QNNPACK "q31" convention, identical to oracle/quant.py:
//   y = SaturatingRoundingDoublingHighMul(acc, M0)
//   y = RoundingDivideByPOT(y, shift)          (ties away from zero)
//   y = clamp(y + zo, qmin, qmax)
// Written in the cheapest exact form (one 32x32->64 multiply, the rest 32-bit
// ops): tests/test_requant_form.py compiles this header on the host and checks
// it against the oracle's restatement on edge and random values.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define ICV_QFN __host__ __device__ __forceinline__
#else
#define ICV_QFN inline
#endif

namespace icv {

// SRDHM: trunc((a*b + nudge) / 2^31), nudge = 2^30 for a*b >= 0, 1 - 2^30
// otherwise.  Both cases equal floor((a*b + 2^30) / 2^31): for a*b < 0,
// trunc(s / 2^31) = floor((s + 2^31 - 1) / 2^31) with s = a*b + 1 - 2^30.
ICV_QFN int32_t srdhm(int32_t a, int32_t b) {
  if (a == INT32_MIN && b == INT32_MIN) return INT32_MAX;
  return (int32_t)(((long long)a * (long long)b + (1LL << 30)) >> 31);
}

// RoundingDivideByPOT, e in [0, 31], all in 32 bits.
ICV_QFN int32_t rounding_divide_by_pot(int32_t x, int e) {
  const int32_t mask = (int32_t)((1u << e) - 1u);
  const int32_t rem = x & mask;
  const int32_t thr = (mask >> 1) + (x < 0 ? 1 : 0);
  return (x >> e) + (rem > thr ? 1 : 0);
}

ICV_QFN uint8_t requant_u8(int32_t acc, int32_t m0, int32_t shift, int32_t zo, int32_t qmin, int32_t qmax) {
  // clamp before adding the zero point: y + zo never wraps (oracle adds in int64)
  const int32_t lo = qmin - zo, hi = qmax - zo;
  int32_t y = rounding_divide_by_pot(srdhm(acc, m0), shift);
  y = y < lo ? lo : (y > hi ? hi : y);
  return (uint8_t)(y + zo);
}

}  // namespace icv
