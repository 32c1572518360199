// bdk_frag.cuh -- register-level code extraction shared by the decode kernels.
//
// The packed words (bdk_common.cuh) are loaded with ldmatrix so that each
// 32-bit register holds two 16-bit words of adjacent MMA fragment rows; field
// POS (counted from the LSB) of both halves is turned into an exact fp16 pair
// by the magic-number trick: lop3 ORs the field into the mantissa of 1024.0
// (0x6400) and one HSUB2 / HFMA2 removes the bias (and the power-of-two field
// shift) exactly.  Two instructions per half2, no integer->float converts.
#pragma once
#include "bdk_common.cuh"

namespace bdk {

template <int SHIFT>
struct MagicConst {
  // fp16 bits of 2^-SHIFT and of -1024 * 2^-SHIFT, duplicated in both halves
  static constexpr uint32_t scale_h = static_cast<uint32_t>(15 - SHIFT) << 10;
  static constexpr uint32_t bias_h = 0x8000u | (static_cast<uint32_t>(25 - SHIFT) << 10);
  static constexpr uint32_t scale2 = scale_h | (scale_h << 16);
  static constexpr uint32_t bias2 = bias_h | (bias_h << 16);
};

// Code at bit position POS of both 16-bit halves of r as an exact fp16 pair.
// lop3 ORs the field into the mantissa of 1024.0 (0x6400); the power-of-two
// rescale is exact, so the result equals the integer code.
template <int BITS, int POS>
__device__ __forceinline__ __half2 ext(uint32_t r, uint32_t r8) {
  if constexpr (BITS == 16) {
    return u2h(r);
  } else {
    constexpr int PB = 8 / BITS;  // fields per byte
    constexpr int SUB = POS % PB;
    const uint32_t src = (POS / PB) ? r8 : r;
    constexpr uint32_t MASK = (((1u << BITS) - 1u) * 0x00010001u) << (SUB * BITS);
    const uint32_t x = lop3_and_or(src, MASK, 0x64006400u);
    if constexpr (SUB == 0) {
      return __hsub2(u2h(x), u2h(0x64006400u));
    } else {
      using M = MagicConst<SUB * BITS>;
      return __hfma2(u2h(x), u2h(M::scale2), u2h(M::bias2));
    }
  }
}



}  // namespace bdk

namespace bdk {

// ------------------------------------------------------------- subnormal mode
// The fast kernel never materializes integer codes: a field masked into an
// otherwise-zero half (exponent bits 0) IS the fp16 subnormal c * 2^(sh-24),
// exactly, where sh is the field's bit offset.  One AND per half2 (plus one
// shift per register for the high byte); the 2^(sh-24) factors are folded
// into per-row logit scales (K) and into the P operand (V).  Tensor cores
// multiply fp16 subnormals exactly (probe: tools/micro/subnormal_mma.cu);
// the fp32 accumulation keeps ~2^-17 relative, far below fp16 P rounding.
template <int BITS, int POS>
struct SubShift {  // bit offset of field POS once the high byte is shifted down
  static constexpr int value = (POS * BITS) % 8;
};

template <int BITS, int POS>
__device__ __forceinline__ uint32_t ext_sub(uint32_t r, uint32_t r8) {
  constexpr int FPB = 8 / BITS;  // fields per byte
  constexpr uint32_t M = (((1u << BITS) - 1u) * 0x00010001u) << SubShift<BITS, POS>::value;
  return (POS / FPB ? r8 : r) & M;
}

}  // namespace bdk
