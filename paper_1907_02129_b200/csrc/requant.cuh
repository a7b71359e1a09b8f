// Fixed-point requantization shared by the uint8 epilogues (K6).
// gemmlowp / QNNPACK "q31" convention, identical to oracle/quant.py:
//   y = SaturatingRoundingDoublingHighMul(acc, M0)
//   y = RoundingDivideByPOT(y, shift)          (ties away from zero)
//   y = clamp(y + zo, qmin, qmax)
#pragma once
#include <cstdint>

namespace icv {

__device__ __forceinline__ int32_t srdhm(int32_t a, int32_t b) {
  if (a == INT32_MIN && b == INT32_MIN) return INT32_MAX;
  const long long ab = (long long)a * (long long)b;
  const long long nudge = ab >= 0 ? (1LL << 30) : (1LL - (1LL << 30));
  return (int32_t)((ab + nudge) / 2147483648LL);   // C division truncates toward zero
}

__device__ __forceinline__ int32_t rounding_divide_by_pot(int32_t x, int e) {
  const long long mask = (1LL << e) - 1;
  const long long rem = (long long)x & mask;
  const long long thr = (mask >> 1) + (x < 0 ? 1 : 0);
  return (int32_t)(((long long)x >> e) + (rem > thr ? 1 : 0));
}

__device__ __forceinline__ uint8_t requant_u8(int32_t acc, int32_t m0, int32_t shift, int32_t zo, int32_t qmin,
                                              int32_t qmax) {
  int32_t y = rounding_divide_by_pot(srdhm(acc, m0), shift) + zo;
  y = y < qmin ? qmin : (y > qmax ? qmax : y);
  return (uint8_t)y;
}

}  // namespace icv
