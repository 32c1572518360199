// bdk_qpack_fast.cuh -- tile-staged fused quantize-and-pack (sm_100a).
//
// Same bit-exact result as qpack_block (bdk_qpack.cuh; kvcache.cpp:184-206,
// quant.cpp:18-93, layout.cpp:45-61) for the BASELINE geometry (d = 128,
// group 128, KChannel K, token-wise V), restructured for HBM throughput:
//
//   * one CTA per (block, 128-token group, cell, tensor): K and V of a block
//     are independent, and with group 128 so are the 128-token halves of an
//     N_r = 256 block, so a CTA stages ONE [128][128] fp16 tile (32 KB) with
//     a single TMA bulk copy and four CTAs per SM overlap their loads with
//     each other's arithmetic;
//   * group (min, max) over the staged tile with half2 min/max (exact on
//     binary16 values; the sign of a zero extremum is taken from the first
//     zero in scan order, the reference's strict-compare tie rule);
//   * code = rint((x - z) / s) via x * rcp(s): the product is within 2^-22
//     relative of the quotient, so it rounds to the same integer unless it
//     lies within 4 * 2^-22 * 2^BITS of a half-integer -- those elements
//     (exact .5 quotients are common on fp16 grids) take the exact IEEE
//     division (__fdiv_rn), so every code equals the reference's;
//   * the params are assembled in shared memory and written with one TMA
//     bulk store; the words go out as 16-byte stores in the record's
//     (swizzled) row layout.
#pragma once
#include "bdk_common.cuh"
#include "bdk_qpack.cuh"

namespace bdk {

constexpr int QF_D = 128;        // head_dim served
constexpr int QF_THREADS = 256;  // threads per CTA

__host__ __device__ inline bool qpack_fast_ok(const Geom& G) {
  return G.d == QF_D && G.g == QF_D && G.k_axis == 0 &&
         (G.bits == 2 || G.bits == 4 || G.bits == 8) && G.n_r % QF_D == 0 && G.warp_n <= 8;
}

struct QfSmem {
  uint32_t tile, out, pout, fs, part, bar, total;
};

__host__ __device__ inline QfSmem qf_layout(const Geom& G) {
  (void)G;
  QfSmem L;
  L.tile = 0;
  L.out = (uint32_t)(QF_D * QF_D * 2);  // staged fp16 tile [128 tokens][128]
  L.pout = L.out;                        // (words go straight to global)
  L.fs = L.pout + QF_D * 4;              // u32 params of the tile (record layout)
  L.part = L.fs + QF_D * 16;             // float4 (s, z, 1/s, -) per group
  L.bar = L.part + 2u * 4u * 64u * 4u;   // K partial half2 (lo, hi) per part
  L.total = L.bar + 16u;
  return L;
}

__device__ __forceinline__ void tma_bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

// One word with the exact IEEE quotient (quant.cpp:30-38): the rare case of a
// product within 1e-4 of a half-integer.  Out of line to keep the fast path
// small.
template <int BITS>
__device__ __noinline__ uint32_t exact_word(const __half* tile, const uint32_t* prm, int tsr, int tw,
                                            int ch, int interleave) {
  constexpr int P = 16 / BITS;
  const float qmax = static_cast<float>((1u << BITS) - 1u);
  uint32_t word = 0;
  for (int p = 0; p < P; ++p) {
    const int t = tw + pos_token(p, P, interleave);
    const uint32_t u = prm[tsr != 0 ? t : ch];
    const float s = __half2float(__ushort_as_half(static_cast<uint16_t>(u & 0xFFFFu)));
    const float z = __half2float(__ushort_as_half(static_cast<uint16_t>(u >> 16)));
    word |= quant_code(__half2float(tile[(size_t)t * QF_D + ch]), s, z, qmax) << (p * BITS);
  }
  return word;
}

// Fast-path constants of one group: fs = (tie threshold, z, 1/s, -z/s).
// q = fma(x, 1/s, -z/s) differs from the reference's rn(rn(x - z) / s) by at
// most (qmax + 1) 2^-22 + |z/s| 2^-24 (the rounding of 1/s, of -z/s, of the
// FMA, and the reference's own roundings of x - z and of the quotient), so a
// q farther than 4x that from a half-integer rounds like the reference; the
// others take the exact path (exact_word).  Constant groups (s = kMinScale,
// huge |z/s|) get a negative threshold: always exact.
__device__ __forceinline__ float4 qf_group_consts(float s, float z, float qmax) {
  const float r = __frcp_rn(s);
  const float c = -__fmul_rn(z, r);
  const float margin = 4.f * ((qmax + 1.f) * (1.f / 4194304.f) + fabsf(c) * (1.f / 16777216.f));
  return make_float4(0.5f - margin, z, r, c);
}

// codes + pack of one 128-token tile (tokens [hf*128, hf*128+128) of the
// block): item (chunk j of the tile, channel pair cp) -> the 8 words (8*P
// tokens) of channels 2cp and 2cp+1, stored as 16 bytes each at their
// swizzled row position in the record; one half2 load feeds both channels.
// TOKEN_PARAMS: V (a (scale, zero) per token) else K (per channel; the tile
// is one 128-token group).  Codes need no clamp here: z = lo exactly and
// s >= (hi - lo) / qmax * (1 - 2^-11), so every in-group quotient lies in
// [0, qmax + 0.5).
// (NT: threads [0, NT) of the CTA take part; `tile` may be shared or global)
// max(|a|, |b|, c) with NaN propagation (one FMNMX3.NAN): a NaN or infinite
// quotient's deviation reaches the tie test below
__device__ __forceinline__ float absmax3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(fabsf(a)), "f"(fabsf(b)), "f"(c));
  return d;
}

// wthr (TOKEN_PARAMS): per word of P tokens, the smallest tie threshold of its
// tokens (V: one (scale, zero) per token), so a word needs one compare
template <int BITS, bool TOKEN_PARAMS, bool IL, int NT = QF_THREADS>
__device__ __forceinline__ void qf_pack(const __half* tile, const float4* fs, const uint32_t* prm,
                                        uint8_t* words, const Geom& G, int hf,
                                        const float* wthr = nullptr) {
  constexpr int P = 16 / BITS;
  constexpr int CPT = QF_D / (8 * P);  // 16-byte chunks per row in one tile
  // SPLIT threads share a chunk (4 / SPLIT word pairs each) so that all
  // NT threads have an item at 2-bit too
  constexpr int SPLIT = NT / (CPT * (QF_D / 2)) < 1 ? 1 : NT / (CPT * (QF_D / 2));
  constexpr int NP = 4 / SPLIT;  // u32 word pairs per item
  const __half2* tile2 = reinterpret_cast<const __half2*>(tile);
  const int wn = G.warp_n, rb = 16 * wn;
  // IL: the token order is a compile-time constant, so every tile offset
  // below folds into the load's immediate
  int tok[P];
#pragma unroll
  for (int p = 0; p < P; ++p) tok[p] = pos_token(p, P, IL ? 1 : 0);
  // q + 1.5 * 2^23 lands in [2^23, 2^24), where the ulp is 1: the FADD rounds q
  // to an integer (ties to even, as rintf) and leaves it in the low mantissa
  // bits, so rint + float->int costs one FADD instead of two XU-pipe ops.  The
  // exponent bits ride along through the shifted sums and are subtracted once.
  constexpr float MAGIC = 12582912.f;
  constexpr uint32_t MAGIC_BITS = 0x4B400000u;
  uint32_t bias = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) bias += MAGIC_BITS << (p * BITS);
  static_assert((SPLIT * CPT * (QF_D / 2)) % NT == 0, "every lane of a warp has an item");
  for (int item = threadIdx.x; item < SPLIT * CPT * (QF_D / 2); item += NT) {
    const int sp = item / (CPT * (QF_D / 2));
    const int jl = (item / (QF_D / 2)) % CPT, cp = item % (QF_D / 2);
    const int t0 = jl * 8 * P + sp * NP * 2 * P;  // first token (tile-relative)
    const int j = hf * CPT + jl;                   // chunk index in the row
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = pa;
    float thr = 0.f;
    if (!TOKEN_PARAMS) {
      pa = fs[2 * cp];
      pb = fs[2 * cp + 1];
      // the pair's words go to the exact path together: one threshold
      thr = fminf(pa.x, pb.x);
    }
    uint32_t w0[NP], w1[NP];
#pragma unroll
    for (int i2 = 0; i2 < NP; ++i2) {
      uint32_t p0 = 0, p1 = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int tw = t0 + (i2 * 2 + h) * P;  // first token of the word
        uint32_t a0 = 0, a1 = 0;
        // largest |q - rint(q)| over the word's codes of both channels (NaN
        // propagating); the word pair takes the exact path when it reaches
        // the threshold
        float dev = 0.f;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int t = tw + tok[p];
          if (TOKEN_PARAMS) pa = pb = fs[t];
          const float2 x = __half22float2(tile2[(size_t)t * 64 + cp]);
          // q = (x - z) / s as one FMA (qf_group_consts)
          const float q0 = __fmaf_rn(x.x, pa.z, pa.w);
          const float q1 = __fmaf_rn(x.y, pb.z, pb.w);
          const float t0m = __fadd_rn(q0, MAGIC), t1m = __fadd_rn(q1, MAGIC);
          const float r0 = __fsub_rn(t0m, MAGIC), r1 = __fsub_rn(t1m, MAGIC);
          dev = absmax3_nan(q0 - r0, q1 - r1, dev);
          a0 += __float_as_uint(t0m) << (p * BITS);
          a1 += __float_as_uint(t1m) << (p * BITS);
        }
        a0 -= bias;
        a1 -= bias;
        // unordered: a NaN or infinite quotient (NaN deviation) takes the
        // exact path, which gives the reference's code (clamp + cast on x86)
        const bool tie = !(dev <= (TOKEN_PARAMS ? wthr[tw / P] : thr));
        if (__any_sync(0xffffffffu, tie) && tie) {
          a0 = exact_word<BITS>(tile, prm, TOKEN_PARAMS, tw, 2 * cp, G.interleave);
          a1 = exact_word<BITS>(tile, prm, TOKEN_PARAMS, tw, 2 * cp + 1, G.interleave);
        }
        p0 |= a0 << (16 * h);
        p1 |= a1 << (16 * h);
      }
      w0[i2] = p0;
      w1[i2] = p1;
    }
    const int ca = 2 * cp, cb = 2 * cp + 1;
    uint8_t* da = words + (size_t)ca * rb + ((j ^ swz(ca, wn)) << 4) + sp * NP * 4;
    uint8_t* db = words + (size_t)cb * rb + ((j ^ swz(cb, wn)) << 4) + sp * NP * 4;
    if constexpr (NP == 4) {
      *reinterpret_cast<uint4*>(da) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
      *reinterpret_cast<uint4*>(db) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
    } else if constexpr (NP == 2) {
      *reinterpret_cast<uint2*>(da) = make_uint2(w0[0], w0[1]);
      *reinterpret_cast<uint2*>(db) = make_uint2(w1[0], w1[1]);
    } else {
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        reinterpret_cast<uint32_t*>(da)[i] = w0[i];
        reinterpret_cast<uint32_t*>(db)[i] = w1[i];
      }
    }
  }
}

// grid (nb * H + 1, cells, 2) with H = N_r / 128 tiles per block: x < nb*H
// packs tile x % H of block x / H of cell (cell_begin + y), tensor z (0 = K,
// 1 = V); x == nb*H, z == 0 copies the residual tail and sets the cell's
// lengths (prefill_kernel's tail branch).
template <int BITS>
__global__ void __launch_bounds__(QF_THREADS) qpack_fast_kernel(DevCache c, const __half* k,
                                                                const __half* v, int len,
                                                                int cell_begin) {
  const float qmax = static_cast<float>((1u << BITS) - 1u);
  extern __shared__ __align__(128) uint8_t smem[];
  const Geom& G = c.G;
  const int cell = cell_begin + blockIdx.y;
  const int nb = len / G.n_r;
  const int H = G.n_r / QF_D;
  const int tsr = blockIdx.z;
  if ((int)blockIdx.x >= nb * H) {  // residual tail + lengths
    if (tsr != 0) return;
    const int tail = len - nb * G.n_r;
    const size_t src = (size_t)blockIdx.y * len * QF_D + (size_t)nb * G.n_r * QF_D;
    const size_t dst = (size_t)cell * G.n_r * QF_D;
    for (int i = threadIdx.x; i < tail * QF_D; i += blockDim.x) {
      c.res_k[dst + i] = k[src + i];
      c.res_v[dst + i] = v[src + i];
    }
    if (threadIdx.x == 0) {
      c.packed_blocks[cell] = nb;
      c.res_len[cell] = tail;
    }
    return;
  }
  const int blk = blockIdx.x / H, hf = blockIdx.x % H;
  const QfSmem L = qf_layout(G);
  const __half* tile = reinterpret_cast<const __half*>(smem + L.tile);
  const __half2* tile2 = reinterpret_cast<const __half2*>(tile);
  uint32_t* pout = reinterpret_cast<uint32_t*>(smem + L.pout);
  float4* fs = reinterpret_cast<float4*>(smem + L.fs);
  float* wthr_sm = reinterpret_cast<float*>(smem + L.part);  // V: per-word tie threshold
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  constexpr uint32_t TILE_BYTES = QF_D * QF_D * 2;
  const __half* src = (tsr ? v : k) + (size_t)blockIdx.y * len * QF_D +
                      ((size_t)blk * G.n_r + (size_t)hf * QF_D) * QF_D;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_expect_tx(bar, TILE_BYTES);
    tma_bulk_g2s(smem + L.tile, src, TILE_BYTES, bar, policy_evict_first());
  }
  __syncthreads();
  mbar_wait(bar, 0);

  const int tid = threadIdx.x;
  if (tsr == 0) {
    // ---- K: KChannel group = this tile's 128 tokens of one channel, param
    // [gr = hf][c].  Thread (channel pair, quarter) scans 32 tokens with half2
    // min/max; the first-zero lookup (tie rule) runs only for a zero extremum.
    __half2* plo = reinterpret_cast<__half2*>(smem + L.part);  // [part][cp]
    __half2* phi = plo + 4 * 64;
    {
      const int cp = tid % 64, part = tid / 64;
      const int t0 = part * 32;
      __half2 lo = tile2[(size_t)t0 * 64 + cp], hi = lo;
#pragma unroll 8
      for (int t = t0 + 1; t < t0 + 32; ++t) {
        const __half2 x = tile2[(size_t)t * 64 + cp];
        lo = __hmin2(lo, x);
        hi = __hmax2(hi, x);
      }
      plo[part * 64 + cp] = lo;
      phi[part * 64 + cp] = hi;
    }
    __syncthreads();
    if (tid < QF_D) {
      const int ch = tid;
      float lo = INFINITY, hi = -INFINITY;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const __half2 l2 = plo[p * 64 + ch / 2], h2 = phi[p * 64 + ch / 2];
        lo = fminf(lo, __half2float((ch & 1) ? __high2half(l2) : __low2half(l2)));
        hi = fmaxf(hi, __half2float((ch & 1) ? __high2half(h2) : __low2half(h2)));
      }
      if (lo == 0.f || hi == 0.f) {  // sign of the first zero in token order
        for (int t = 0; t < QF_D; ++t) {
          const float x = __half2float(tile[(size_t)t * QF_D + ch]);
          if (x == 0.f) {
            if (lo == 0.f) lo = x;
            if (hi == 0.f) hi = x;
            break;
          }
        }
      }
      float s, z;
      group_params(lo, hi, qmax, s, z);
      fs[ch] = qf_group_consts(s, z, qmax);
      pout[ch] = param_u32(s, z);
    }
  } else {
    // ---- V: token groups (the 128 channels of one token), param [t].
    // Thread per token; the scan is staggered by token so the 32 rows of a
    // warp hit 32 distinct banks.
    if (tid < QF_D) {
      const int t = tid;
      const __half2* row = tile2 + (size_t)t * 64;
      __half2 lo = row[t & 63], hi = lo;
#pragma unroll 8
      for (int i = 1; i < 64; ++i) {
        const __half2 x = row[(i + t) & 63];
        lo = __hmin2(lo, x);
        hi = __hmax2(hi, x);
      }
      float flo = fminf(__low2float(lo), __high2float(lo));
      float fhi = fmaxf(__low2float(hi), __high2float(hi));
      if (flo == 0.f || fhi == 0.f) {  // sign of the first zero in channel order
        for (int ch = 0; ch < QF_D; ++ch) {
          const float x = __half2float(tile[(size_t)t * QF_D + ch]);
          if (x == 0.f) {
            if (flo == 0.f) flo = x;
            if (fhi == 0.f) fhi = x;
            break;
          }
        }
      }
      float s, z;
      group_params(flo, fhi, qmax, s, z);
      const float4 k4 = qf_group_consts(s, z, qmax);
      fs[t] = k4;
      pout[t] = param_u32(s, z);
      // the word of tokens [t & ~(P-1), +P): smallest tie threshold
      constexpr int P = 16 / BITS;
      float wt = k4.x;
#pragma unroll
      for (int o = 1; o < P; o <<= 1) wt = fminf(wt, __shfl_xor_sync(0xffffffffu, wt, o));
      if (t % P == 0) wthr_sm[t / P] = wt;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + blk) * G.rec_bytes;
  if (threadIdx.x == 0) {  // this tile's params: 128 u32, contiguous in the record
    tma_bulk_s2g(rec + 2 * G.wbytes + (tsr ? G.kp_bytes : 0) + hf * QF_D * 4, pout, QF_D * 4);
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  }
  if (tsr == 0) {
    if (G.interleave)
      qf_pack<BITS, false, true>(tile, fs, pout, rec, G, hf);
    else
      qf_pack<BITS, false, false>(tile, fs, pout, rec, G, hf);
  } else {
    if (G.interleave)
      qf_pack<BITS, true, true>(tile, fs, pout, rec + G.wbytes, G, hf, wthr_sm);
    else
      qf_pack<BITS, true, false>(tile, fs, pout, rec + G.wbytes, G, hf, wthr_sm);
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// Fused flush of one full residual window (build_block + commit_block,
// kvcache.cpp:208-237) by the combine grid: threads [0, NT) of a CTA pack the
// window's tiles item0, item0 + istep, ... (item i < N_r/128: K tile i, else
// V tile i - N_r/128), so the CTAs of one cell split the window.  Same
// arithmetic as qpack_fast_kernel -- bit-exact with the reference -- but the
// 128-token tiles are read straight from the (L2-resident) window instead of
// being staged.  `sm` >= 3 KB of shared scratch: fs (128 float4) + K partial
// (lo, hi) half2 per (part, channel pair).  Synchronized by named barrier
// `bar` over NT threads.
template <int BITS, int NT>
__device__ __forceinline__ void qf_flush_window(const Geom& G, const __half* rk, const __half* rv,
                                                uint8_t* rec, uint8_t* sm, int bar, int item0,
                                                int istep) {
  static_assert(NT >= 64 && NT % 64 == 0, "channel pairs x token parts");
  constexpr int PARTS = NT / 64, TPP = QF_D / PARTS;  // K scan: token parts, tokens per part
  constexpr int TB = 8;                               // V rows per load batch of a warp
  const float qmax = static_cast<float>((1u << BITS) - 1u);
  float4* fs = reinterpret_cast<float4*>(sm);
  __half2* plo = reinterpret_cast<__half2*>(sm + QF_D * 16);
  __half2* phi = plo + PARTS * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* kp = reinterpret_cast<uint32_t*>(rec + 2 * G.wbytes);
  uint32_t* vp = reinterpret_cast<uint32_t*>(rec + 2 * G.wbytes + G.kp_bytes);
  const int H = G.n_r / QF_D;
  for (int item = item0; item < 2 * H; item += istep) {
    if (item < H) {
      // ---- K tile hf: KChannel group = the tile's 128 tokens of one channel
      const int hf = item;
      const __half* kt = rk + (size_t)hf * QF_D * QF_D;
      const __half2* kt2 = reinterpret_cast<const __half2*>(kt);
      {
        const int cp = tid % 64, part = tid / 64;
        const int t0 = part * TPP;
        __half2 lo = kt2[(size_t)t0 * 64 + cp], hi = lo;
#pragma unroll 16
        for (int t = t0 + 1; t < t0 + TPP; ++t) {
          const __half2 x = kt2[(size_t)t * 64 + cp];
          lo = __hmin2(lo, x);
          hi = __hmax2(hi, x);
        }
        plo[part * 64 + cp] = lo;
        phi[part * 64 + cp] = hi;
      }
      named_bar(bar, NT);
      for (int ch = tid; ch < QF_D; ch += NT) {
        float lo = INFINITY, hi = -INFINITY;
#pragma unroll
        for (int p = 0; p < PARTS; ++p) {
          const __half2 l2 = plo[p * 64 + ch / 2], h2 = phi[p * 64 + ch / 2];
          lo = fminf(lo, __half2float((ch & 1) ? __high2half(l2) : __low2half(l2)));
          hi = fmaxf(hi, __half2float((ch & 1) ? __high2half(h2) : __low2half(h2)));
        }
        if (lo == 0.f || hi == 0.f) {  // sign of the first zero in token order
          for (int t = 0; t < QF_D; ++t) {
            const float x = __half2float(kt[(size_t)t * QF_D + ch]);
            if (x == 0.f) {
              if (lo == 0.f) lo = x;
              if (hi == 0.f) hi = x;
              break;
            }
          }
        }
        float s, z;
        group_params(lo, hi, qmax, s, z);
        fs[ch] = qf_group_consts(s, z, qmax);
        kp[hf * QF_D + ch] = param_u32(s, z);
      }
      named_bar(bar, NT);
      if (G.interleave)
        qf_pack<BITS, false, true, NT>(kt, fs, kp + hf * QF_D, rec, G, hf);
      else
        qf_pack<BITS, false, false, NT>(kt, fs, kp + hf * QF_D, rec, G, hf);
    } else {
      // ---- V tile hf: token groups (the 128 channels of one token); warp per
      // token, TB rows of a warp in flight per batch
      const int hf = item - H;
      const __half* vt = rv + (size_t)hf * QF_D * QF_D;
      const __half2* vt2 = reinterpret_cast<const __half2*>(vt);
      for (int tb = warp * TB; tb < QF_D; tb += (NT / 32) * TB) {
        __half2 a[TB], b[TB];
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          a[i] = vt2[(size_t)(tb + i) * 64 + lane];
          b[i] = vt2[(size_t)(tb + i) * 64 + 32 + lane];
        }
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          const int t = tb + i;
          const __half2 lo2 = __hmin2(a[i], b[i]), hi2 = __hmax2(a[i], b[i]);
          float lo = fminf(__low2float(lo2), __high2float(lo2));
          float hi = fmaxf(__low2float(hi2), __high2float(hi2));
          // first zero in channel order (channels 2*lane, 2*lane+1, 64+2*lane, ...)
          int zf = 0x7fffffff;
          if (__low2float(a[i]) == 0.f) zf = 2 * lane;
          else if (__high2float(a[i]) == 0.f) zf = 2 * lane + 1;
          else if (__low2float(b[i]) == 0.f) zf = 64 + 2 * lane;
          else if (__high2float(b[i]) == 0.f) zf = 65 + 2 * lane;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            zf = min(zf, __shfl_xor_sync(0xffffffffu, zf, o));
          }
          if (lo == 0.f || hi == 0.f) {
            const float x = __half2float(vt[(size_t)t * QF_D + zf]);
            if (lo == 0.f) lo = x;
            if (hi == 0.f) hi = x;
          }
          if (lane == 0) {
            float s, z;
            group_params(lo, hi, qmax, s, z);
            fs[t] = qf_group_consts(s, z, qmax);
            vp[hf * QF_D + t] = param_u32(s, z);
          }
        }
      }
      named_bar(bar, NT);
      // per word of P tokens: the smallest tie threshold (qf_pack)
      constexpr int P = 16 / BITS;
      float* wthr = reinterpret_cast<float*>(plo);
      for (int w = tid; w < QF_D / P; w += NT) {
        float wt = fs[w * P].x;
#pragma unroll
        for (int i = 1; i < P; ++i) wt = fminf(wt, fs[w * P + i].x);
        wthr[w] = wt;
      }
      named_bar(bar, NT);
      if (G.interleave)
        qf_pack<BITS, true, true, NT>(vt, fs, vp + hf * QF_D, rec + G.wbytes, G, hf, wthr);
      else
        qf_pack<BITS, true, false, NT>(vt, fs, vp + hf * QF_D, rec + G.wbytes, G, hf, wthr);
    }
    named_bar(bar, NT);  // fs is reused
  }
}

}  // namespace bdk
