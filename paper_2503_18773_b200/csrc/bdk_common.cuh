// bdk_common.cuh -- shared device helpers for the sm_100a BitDecoding path.
//
// Device data layout:
//   one BLOCK RECORD per (cell, block slot), cell = b * heads_kv + h:
//     [ K words | V words | K params | V params ]  padded to 128 B
//   K/V words: the reference PackedBlock word array (kvcache.cpp:79-95):
//     row c (channel) holds N_r/P = 8*W_n u16 words, word g packs tokens
//     g*P .. g*P+P-1 of channel c, field k (MSB first) = token order[k]
//     (layout.cpp:45-61).  A row is 16*W_n bytes = W_n 16-byte chunks; chunk
//     j of row c is stored at chunk position j ^ swz(c) (the reference's XOR
//     swizzle, layout.hpp:49, in 16-byte units) so that the ldmatrix reads of
//     8 consecutive rows hit 8 distinct bank groups.  Readback undoes it, so
//     the logical words are byte-identical to the reference.
//   params: the reference QuantParams data (quant.hpp:38-47): u16 pairs
//     (scale, zero) = one u32 per group, KChannel [N_r/g][d], KToken [N_r][d/g].
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace bdk {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kMinScale = 6.103515625e-05f;  // quant.hpp:52, 2^-14

// ---------------------------------------------------------------- geometry
struct Geom {
  int batch, heads_kv, d, warp_n, bits, k_axis, g, interleave;
  int n_r;          // 8 * warp_n * (16 / bits)           (layout.cpp:74-77)
  int pack;         // P = 16 / bits
  int max_blocks;   // block slots per cell
  int wbytes;       // K (or V) word bytes per block = d * 16 * warp_n
  int kp_bytes;     // K param bytes per block
  int vp_bytes;     // V param bytes per block
  int rec_bytes;    // record stride (128-B aligned)
};

__host__ __device__ inline int swz(int row, int warp_n) {
  // chunk XOR pattern: 8 / warp_n rows share a 128-B line; rotate per line.
  return ((row * warp_n) >> 3) & (warp_n - 1);
}

// token held by bit-field position p (counted from the LSB of a 16-bit word)
// given the permutation order[] (field k from the MSB holds token order[k]).
__host__ __device__ inline int pos_token(int p, int pack, int interleave) {
  if (pack == 1) return 0;
  const int k = pack - 1 - p;  // field index from the MSB
  if (!interleave) return k;   // identity_order (layout.cpp:36-43)
  // interleave_order (layout.cpp:21-34): odd indices descending, then even
  // indices descending ("75316420" for P = 8, "3120" for P = 4).
  const int half = pack / 2;
  return k < half ? pack - 1 - 2 * k : pack - 2 - 2 * (k - half);
}

// inverse of pos_token: bit-field position (from the LSB) holding token
// offset j of a word
__host__ __device__ inline int field_of_token(int j, int pack, int interleave) {
  if (pack == 1) return 0;
  int k;  // field index from the MSB
  if (!interleave)
    k = j;
  else
    k = (j & 1) ? (pack - 1 - j) / 2 : pack / 2 + (pack - 2 - j) / 2;
  return pack - 1 - k;
}

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D = A(16x16, row) * B(16x8, col) + D, f16 inputs, f32 accumulate
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic) {
  uint32_t r;
  // (a & mask) | magic   -> immLut = (0xF0 & 0xCC) | 0xAA = 0xEA
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(a), "r"(mask), "r"(magic));
  return r;
}

// ---------------------------------------------------------- mbarrier / TMA
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// wait with a suspend-time hint: producer-side waits that are expected to
// block (ring full) park the warp instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completes on bar.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// programmatic dependent launch (PDL): let the next kernel in the stream start
// launching / wait until the previous kernel's memory is visible
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// named barrier over the first n threads of the CTA (n a multiple of 32)
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// -------------------------------------------------------- warp reductions
__device__ __forceinline__ float warp_max_xor(float v, int from) {
  for (int o = from; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------ element readback
// Element (token t, channel ch) of one block record, dequantized exactly as
// packed_tile stages it (kvcache.cpp:289-309): round_f16(code*scale + zero)
// in fp32 (the fp32 product is exact); passthrough blocks hold raw fp16 bits.
// which = 0 keys, 1 values.
__device__ __forceinline__ __half packed_elem(const Geom& G, const uint8_t* rec, int t, int ch,
                                              int which) {
  const int rb = 16 * G.warp_n, P = G.pack;
  const uint32_t mask = G.bits == 16 ? 0xFFFFu : ((1u << G.bits) - 1u);
  const int wi = t / P, j = wi / 8;
  const int p = field_of_token(t % P, P, G.interleave);
  const uint8_t* words = rec + which * G.wbytes;
  const uint16_t w = *reinterpret_cast<const uint16_t*>(
      words + (size_t)ch * rb + ((j ^ swz(ch, G.warp_n)) << 4) + (wi % 8) * 2);
  const uint32_t code = (w >> (p * G.bits)) & mask;
  if (G.bits == 16) return __ushort_as_half(static_cast<uint16_t>(code));
  const uint32_t* par =
      reinterpret_cast<const uint32_t*>(rec + 2 * G.wbytes + (which ? G.kp_bytes : 0));
  const int gi = (which == 0 && G.k_axis == 0) ? (t / G.g) * G.d + ch
                                               : t * (G.d / G.g) + ch / G.g;
  const uint32_t pr = par[gi];
  const float s = __half2float(__ushort_as_half(static_cast<uint16_t>(pr & 0xFFFF)));
  const float z = __half2float(__ushort_as_half(static_cast<uint16_t>(pr >> 16)));
  return __float2half_rn(__fadd_rn(__fmul_rn(static_cast<float>(code), s), z));
}

}  // namespace bdk
