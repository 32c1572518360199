// bdk_qpack.cuh -- fused quantize-and-pack of one N_r-token block (sm_100a).
//
// Bit-exact restatement of KVCache::make_block_from (kvcache.cpp:184-206):
//   quantize_tile (quant.cpp:47-93) with compute_group_params /
//   quantize_group (quant.cpp:18-38), then pack_block_codes
//   (kvcache.cpp:79-95) / pack_word (layout.cpp:45-61).
// Numerics follow SURVEY.md F2: IEEE __fsub_rn / __fdiv_rn (never x*rcp),
// rintf (round-half-even, = nearbyintf), __float2half_rn (RNE).  Group min /
// max keep the reference's tie rule (the FIRST element equal to the extremum
// wins, which only matters for the sign of a zero) -- see first_zero below.
//
// Two passes over a [N_r, d] tile (all CTA threads participate):
//   pass 1: per group -> (scale, zero) u32 param + u8 codes in shared scratch
//   pass 2: thread per channel row packs P codes per u16 word, 8 words per
//           16-byte chunk, chunk j stored at j ^ swz(row) (bdk_common.cuh)
#pragma once
#include "bdk_common.cuh"

namespace bdk {

// quant.cpp:18-28 (lo, hi already reduced; lo is binary16-representable)
__device__ __forceinline__ void group_params(float lo, float hi, float qmax, float& s, float& z) {
  float sc = __half2float(__float2half_rn(__fdiv_rn(__fsub_rn(hi, lo), qmax)));
  if (!(sc >= kMinScale)) sc = kMinScale;
  s = sc;
  z = __half2float(__float2half_rn(lo));
}

// quant.cpp:30-38
__device__ __forceinline__ uint32_t quant_code(float x, float s, float z, float qmax) {
  float c = rintf(__fdiv_rn(__fsub_rn(x, z), s));
  c = c < 0.0f ? 0.0f : (qmax < c ? qmax : c);
  return static_cast<uint32_t>(c);
}

__device__ __forceinline__ uint32_t param_u32(float s, float z) {
  const uint32_t sb = __half_as_ushort(__float2half_rn(s));
  const uint32_t zb = __half_as_ushort(__float2half_rn(z));
  return sb | (zb << 16);
}

// Pass 1 for a channel-wise-grouped tensor (K with QuantAxis::KChannel):
// item (c, gr) scans tokens gr*g .. gr*g+g-1 of channel c in order, exactly
// like the reference loop, so the tie rule holds by construction.
__device__ inline void qpass_channel(const __half* src, int ld, int n_r, int d, int g, float qmax,
                                     uint32_t* params, uint8_t* codes) {
  const int ngr = n_r / g;
  for (int it = threadIdx.x; it < d * ngr; it += blockDim.x) {
    const int c = it % d, gr = it / d;
    const __half* col = src + (size_t)gr * g * ld + c;
    float lo = __half2float(col[0]), hi = lo;
    for (int i = 0; i < g; ++i) {
      const float x = __half2float(col[(size_t)i * ld]);
      lo = x < lo ? x : lo;  // std::min(lo, x)
      hi = hi < x ? x : hi;  // std::max(hi, x)
    }
    float s, z;
    group_params(lo, hi, qmax, s, z);
    params[gr * d + c] = param_u32(s, z);
    for (int i = 0; i < g; ++i) {
      const float x = __half2float(col[(size_t)i * ld]);
      codes[(gr * g + i) * d + c] = static_cast<uint8_t>(quant_code(x, s, z, qmax));
    }
  }
}

// Pass 1 for a token-wise-grouped tensor (V always; K with KToken): one warp
// per token row; lane owns channels lane + 32*i.  Groups of g >= 32 channels
// reduce over i then across the warp; groups of g < 32 (g | 32) reduce within
// lane segments.  min/max values are order-independent except for the sign
// of a zero extremum, which is taken from the first (lowest-channel) element
// equal to it -- the reference's strict-compare scan keeps the first one.
__device__ inline void qpass_token(const __half* src, int ld, int n_r, int d, int g, float qmax,
                                   uint32_t* params, uint8_t* codes) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int groups = d / g;
  for (int t = warp; t < n_r; t += nwarps) {
    const __half* row = src + (size_t)t * ld;
    if (g >= 32) {
      const int ipg = g / 32;
      for (int gc = 0; gc < groups; ++gc) {
        float lo = INFINITY, hi = -INFINITY;
        int zfirst = 0x7fffffff;
        for (int i = 0; i < ipg; ++i) {
          const int c = gc * g + i * 32 + lane;
          const float x = __half2float(row[c]);
          lo = fminf(lo, x);
          hi = fmaxf(hi, x);
          if (x == 0.0f) zfirst = min(zfirst, c);
        }
        for (int o = 16; o >= 1; o >>= 1) {
          lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          zfirst = min(zfirst, __shfl_xor_sync(0xffffffffu, zfirst, o));
        }
        if (lo == 0.0f) lo = __half2float(row[zfirst]);
        if (hi == 0.0f) hi = __half2float(row[zfirst]);
        float s, z;
        group_params(lo, hi, qmax, s, z);
        if (lane == 0) params[t * groups + gc] = param_u32(s, z);
        for (int i = 0; i < ipg; ++i) {
          const int c = gc * g + i * 32 + lane;
          codes[t * d + c] = static_cast<uint8_t>(quant_code(__half2float(row[c]), s, z, qmax));
        }
      }
    } else {
      // g < 32 (a power of two dividing d): lanes form aligned g-lane
      // segments; lanes past d (d < 32 or d % 32 != 0) carry neutral values
      for (int i = 0; i < (d + 31) / 32; ++i) {
        const int c = i * 32 + lane;
        const bool valid = c < d;
        const float x = valid ? __half2float(row[c]) : 0.0f;
        float lo = valid ? x : INFINITY, hi = valid ? x : -INFINITY;
        int zfirst = valid && x == 0.0f ? c : 0x7fffffff;
        for (int o = g / 2; o >= 1; o >>= 1) {
          lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          zfirst = min(zfirst, __shfl_xor_sync(0xffffffffu, zfirst, o));
        }
        if (!valid) continue;  // after the shuffles: every lane took part
        if (lo == 0.0f) lo = __half2float(row[zfirst]);
        if (hi == 0.0f) hi = __half2float(row[zfirst]);
        float s, z;
        group_params(lo, hi, qmax, s, z);
        if ((lane % g) == 0) params[t * groups + c / g] = param_u32(s, z);
        codes[t * d + c] = static_cast<uint8_t>(quant_code(x, s, z, qmax));
      }
    }
  }
}

// Pass 2: pack codes (u8 [n_r][d] in shared memory) into the word rows.
template <int BITS>
__device__ inline void qpass_pack(const uint8_t* codes, int n_r, int d, int warp_n, int interleave,
                                  uint8_t* words) {
  constexpr int P = 16 / BITS;
  const int rb = 16 * warp_n;
  int tok[P];
#pragma unroll
  for (int p = 0; p < P; ++p) tok[p] = pos_token(p, P, interleave);
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    for (int j = 0; j < warp_n; ++j) {
      uint32_t w[4];
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {
        uint32_t pair = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int wi = j * 8 + i2 * 2 + h;  // word index in the row
          uint32_t word = 0;
#pragma unroll
          for (int p = 0; p < P; ++p)
            word |= static_cast<uint32_t>(codes[(wi * P + tok[p]) * d + c]) << (p * BITS);
          pair |= word << (16 * h);
        }
        w[i2] = pair;
      }
      *reinterpret_cast<uint4*>(words + (size_t)c * rb + ((j ^ swz(c, warp_n)) << 4)) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  (void)n_r;
}

// Passthrough (num_bits == 16, kvcache.cpp:186-196): raw binary16 bits, P = 1,
// so word (c, t) = bits of x[t][c] -- a transpose into the row layout.
__device__ inline void qpass_raw(const __half* src, int ld, int d, int warp_n, uint8_t* words) {
  const int rb = 16 * warp_n;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    for (int j = 0; j < warp_n; ++j) {
      uint32_t w[4];
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {
        const int t = j * 8 + i2 * 2;
        w[i2] = static_cast<uint32_t>(__half_as_ushort(src[(size_t)t * ld + c])) |
                (static_cast<uint32_t>(__half_as_ushort(src[(size_t)(t + 1) * ld + c])) << 16);
      }
      *reinterpret_cast<uint4*>(words + (size_t)c * rb + ((j ^ swz(c, warp_n)) << 4)) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// make_block_from for one block: k/v rows [n_r][ld] (fp16, global), record
// out, `scratch` >= n_r*d bytes of shared memory.  Ends with __syncthreads.
template <int BITS>
__device__ inline void qpack_block(const Geom& G, const __half* k, const __half* v, int ld,
                                   uint8_t* rec, uint8_t* scratch) {
  uint8_t* kw = rec;
  uint8_t* vw = rec + G.wbytes;
  uint32_t* kp = reinterpret_cast<uint32_t*>(rec + 2 * G.wbytes);
  uint32_t* vp = reinterpret_cast<uint32_t*>(rec + 2 * G.wbytes + G.kp_bytes);
  if constexpr (BITS == 16) {
    qpass_raw(k, ld, G.d, G.warp_n, kw);
    qpass_raw(v, ld, G.d, G.warp_n, vw);
    __syncthreads();
  } else {
    const float qmax = static_cast<float>((1u << BITS) - 1u);
    if (G.k_axis == 0)
      qpass_channel(k, ld, G.n_r, G.d, G.g, qmax, kp, scratch);
    else
      qpass_token(k, ld, G.n_r, G.d, G.g, qmax, kp, scratch);
    __syncthreads();
    qpass_pack<BITS>(scratch, G.n_r, G.d, G.warp_n, G.interleave, kw);
    __syncthreads();
    qpass_token(v, ld, G.n_r, G.d, G.g, qmax, vp, scratch);
    __syncthreads();
    qpass_pack<BITS>(scratch, G.n_r, G.d, G.warp_n, G.interleave, vw);
    __syncthreads();
  }
}

// Fused flush of one full residual window (build_block + commit_block,
// kvcache.cpp:208-237) by a CTA that has other warps busy or gone: threads
// [0, nthr) only, synchronized by named barrier `bar` (nthr threads), no
// shared memory.  Geometry of the fast decode kernel: KChannel K with
// g | N_r, per-token V groups of g = d (one (scale, zero) per token).
// Same arithmetic as qpass_channel / qpass_token / qpass_pack (bit-exact
// with the reference): K item (c, gr) scans its g tokens in order; V token t
// reduces its row per warp with the first-zero sign rule; codes are packed
// straight into the swizzled word rows (thread per channel row), the V
// params read back from the record the first pass wrote.
// (G by value: the callers' geometry is a kernel parameter, whose address
// would make them keep it in local memory)
template <int BITS>
__device__ __noinline__ void flush_window(const Geom G, const __half* rk, const __half* rv,
                                    uint8_t* rec, int nthr, int bar) {
  constexpr int P = 16 / BITS;
  const float qmax = static_cast<float>((1u << BITS) - 1u);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const int d = G.d, n_r = G.n_r, g = G.g, rb = 16 * G.warp_n;
  uint8_t* kw = rec;
  uint8_t* vw = rec + G.wbytes;
  uint32_t* kp = reinterpret_cast<uint32_t*>(rec + 2 * G.wbytes);
  uint32_t* vp = reinterpret_cast<uint32_t*>(rec + 2 * G.wbytes + G.kp_bytes);
  int tok[P];
#pragma unroll
  for (int p = 0; p < P; ++p) tok[p] = pos_token(p, P, G.interleave);
  // ---- K: thread per (channel, group): params, then its words
  const int ngr = n_r / g, wpg = g / P;  // words per group in a row
  for (int it = tid; it < d * ngr; it += nthr) {
    const int c = it % d, gr = it / d;
    const __half* col = rk + (size_t)gr * g * d + c;
    float lo = __half2float(col[0]), hi = lo;
    for (int i = 0; i < g; ++i) {
      const float x = __half2float(col[(size_t)i * d]);
      lo = x < lo ? x : lo;  // std::min(lo, x)
      hi = hi < x ? x : hi;  // std::max(hi, x)
    }
    float sc, z;
    group_params(lo, hi, qmax, sc, z);
    kp[gr * d + c] = param_u32(sc, z);
    for (int w8 = 0; w8 < wpg; w8 += 8) {  // one 16-byte chunk: 8 words
      uint32_t q4[4];
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {
        uint32_t pair = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int wi = gr * wpg + w8 + 2 * i2 + h;  // word index in the row
          uint32_t word = 0;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            const float x = __half2float(rk[(size_t)(wi * P + tok[p]) * d + c]);
            word |= quant_code(x, sc, z, qmax) << (p * BITS);
          }
          pair |= word << (16 * h);
        }
        q4[i2] = pair;
      }
      const int j = (gr * wpg + w8) / 8;
      *reinterpret_cast<uint4*>(kw + (size_t)c * rb + ((j ^ swz(c, G.warp_n)) << 4)) =
          make_uint4(q4[0], q4[1], q4[2], q4[3]);
    }
  }
  // ---- V params: warp per token, lanes over channels (qpass_token, g >= 32)
  const int groups = d / g, ipg = g / 32;
  for (int t = warp; t < n_r; t += nwarps) {
    const __half* row = rv + (size_t)t * d;
    for (int gc = 0; gc < groups; ++gc) {
      float lo = INFINITY, hi = -INFINITY;
      int zfirst = 0x7fffffff;
      for (int i = 0; i < ipg; ++i) {
        const int c = gc * g + i * 32 + lane;
        const float x = __half2float(row[c]);
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
        if (x == 0.0f) zfirst = min(zfirst, c);
      }
      for (int o = 16; o >= 1; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        zfirst = min(zfirst, __shfl_xor_sync(0xffffffffu, zfirst, o));
      }
      if (lo == 0.0f) lo = __half2float(row[zfirst]);
      if (hi == 0.0f) hi = __half2float(row[zfirst]);
      float sc, z;
      group_params(lo, hi, qmax, sc, z);
      if (lane == 0) vp[t * groups + gc] = param_u32(sc, z);
    }
  }
  named_bar(bar, nthr);  // V params visible to every thread of the flush
  // ---- V words: thread per channel row, codes with the token's params
  for (int c = tid; c < d; c += nthr) {
    const int gc = c / g;
    for (int j = 0; j < G.warp_n; ++j) {
      uint32_t q4[4];
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {
        uint32_t pair = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int wi = j * 8 + 2 * i2 + h;
          uint32_t word = 0;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            const int t = wi * P + tok[p];
            const uint32_t pr = vp[t * groups + gc];
            const float sc = __half2float(__ushort_as_half(static_cast<uint16_t>(pr & 0xFFFFu)));
            const float z = __half2float(__ushort_as_half(static_cast<uint16_t>(pr >> 16)));
            word |= quant_code(__half2float(rv[(size_t)t * d + c]), sc, z, qmax) << (p * BITS);
          }
          pair |= word << (16 * h);
        }
        q4[i2] = pair;
      }
      *reinterpret_cast<uint4*>(vw + (size_t)c * rb + ((j ^ swz(c, G.warp_n)) << 4)) =
          make_uint4(q4[0], q4[1], q4[2], q4[3]);
    }
  }
  named_bar(bar, nthr);
}

}  // namespace bdk
