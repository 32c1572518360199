// bdk_kernels.cu -- sm_100a kernels of the BitDecoding decode hot path.
//
//   prefill_kernel  KVCache::prefill (kvcache.cpp:155-168): fused quantize +
//                   pack of every full N_r block (bdk_qpack.cuh) + residual tail
//   append_kernel   KVCache::append_token (kvcache.cpp:170-182)
//   flush_kernel    KVCache::flush_residual (kvcache.cpp:245-251)
//   decode_kernel   decode_step's residual_attend + packed_attend
//                   (attention.cpp:92-140, 164-242), one CTA per (split, cell):
//                     part 0      append + fp16 residual attention + qpack of a
//                                 full residual into the next block slot
//                     part 1..S   split-KV attention over packed blocks:
//                                 TMA bulk copies (UBLKCP) of whole block
//                                 records into a 4-stage mbarrier ring fed by
//                                 a producer warp; 4 consumer warps each own
//                                 one 16-byte chunk (8*P tokens) of every
//                                 block row, dequantize in registers
//                                 (lop3 magic-number int->fp16 + HFMA2) and
//                                 run mma.sync m16n8k16 in swap-AB form:
//                                 S^T = K Q^T (tokens in M, GQA heads in N)
//                                 and O^T += V^T P^T.
//   combine_kernel  combine (attention.cpp:142-162) over the parts + the
//                   cache-update phase (attention.cpp:235-240)
//
// Fragment <-> packed-layout mapping: with ldmatrix.trans on
// [channel rows x word columns], lane (gid,t4) receives (w[c][g], w[c+1][g])
// for c = 2*t4 (+8), g = 8j+gid; bit position p of each half is the code of
// token g*P + order[P-1-p].  Rows gid / gid+8 of an S^T tile take positions
// (2pi, 2pi+1) of the same register, so one ldmatrix register feeds P/2
// M-tiles.  Plain ldmatrix of the SAME V rows yields (w[c][8j+2t4],
// w[c][8j+2t4+1]) = the V^T A fragment with the identical token labelling,
// so softmax/PV see a consistent (permuted) token order and the packed
// words never need unpacking in memory.
#include <cfloat>

#include "bdk_launch.h"
#include "bdk_frag.cuh"
#include <cstdlib>

#include "bdk_qpack.cuh"
#include "bdk_qpack_fast.cuh"

namespace bdk {

// ------------------------------------------------------------ small kernels

template <int BITS>
__global__ void __launch_bounds__(256) prefill_kernel(DevCache c, const __half* k, const __half* v,
                                                      int len, int cell_begin) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Geom& G = c.G;
  const int cell = cell_begin + blockIdx.y;
  const int nb = len / G.n_r;
  const __half* kc = k + (size_t)blockIdx.y * len * G.d;
  const __half* vc = v + (size_t)blockIdx.y * len * G.d;
  if ((int)blockIdx.x < nb) {
    uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + blockIdx.x) * G.rec_bytes;
    const size_t off = (size_t)blockIdx.x * G.n_r * G.d;
    qpack_block<BITS>(G, kc + off, vc + off, G.d, rec, smem);
  } else {
    const int tail = len - nb * G.n_r;
    const size_t src = (size_t)nb * G.n_r * G.d, dst = (size_t)cell * G.n_r * G.d;
    for (int i = threadIdx.x; i < tail * G.d; i += blockDim.x) {
      c.res_k[dst + i] = kc[src + i];
      c.res_v[dst + i] = vc[src + i];
    }
    if (threadIdx.x == 0) {
      c.packed_blocks[cell] = nb;
      c.res_len[cell] = tail;
    }
  }
}

__global__ void append_kernel(DevCache c, int cell, const __half* k_row, const __half* v_row) {
  const Geom& G = c.G;
  const int r = c.res_len[cell];
  for (int i = threadIdx.x; i < G.d; i += blockDim.x) {
    c.res_k[((size_t)cell * G.n_r + r) * G.d + i] = k_row[i];
    c.res_v[((size_t)cell * G.n_r + r) * G.d + i] = v_row[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) c.res_len[cell] = r + 1;
}

template <int BITS>
__global__ void __launch_bounds__(256) flush_kernel(DevCache c, int cell, int commit) {
  // flush_residual (commit = 1) / build_block (commit = 0, kvcache.cpp:
  // 208-219): pack the full residual into the next block slot; only a flush
  // updates the lengths
  extern __shared__ __align__(128) uint8_t smem[];
  const Geom& G = c.G;
  const int slot = c.packed_blocks[cell];
  uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + slot) * G.rec_bytes;
  const size_t base = (size_t)cell * G.n_r * G.d;
  qpack_block<BITS>(G, c.res_k + base, c.res_v + base, G.d, rec, smem);
  if (commit && threadIdx.x == 0) {
    c.packed_blocks[cell] = slot + 1;
    c.res_len[cell] = 0;
  }
}

// flush of every residual that the step filled (decode_step's build_block +
// commit_block, attention.cpp:103, :235-240): one CTA per cell, no-op unless
// res_len == N_r
template <int BITS>
__global__ void __launch_bounds__(256) flush_full_kernel(DevCache c) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Geom& G = c.G;
  const int cell = blockIdx.x;
  if (c.res_len[cell] != G.n_r) return;
  const int slot = c.packed_blocks[cell];
  uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + slot) * G.rec_bytes;
  const size_t base = (size_t)cell * G.n_r * G.d;
  qpack_block<BITS>(G, c.res_k + base, c.res_v + base, G.d, rec, smem);
  if (threadIdx.x == 0) {
    c.packed_blocks[cell] = slot + 1;
    c.res_len[cell] = 0;
  }
}

// Host-API step inputs: pinned (mapped) host staging -> device, as a kernel
// rather than a copy-engine transfer so that the decode kernel, launched as its
// programmatic dependent, starts streaming packed blocks while the inputs are
// still crossing PCIe (it reads them only after griddepcontrol.wait).
__global__ void __launch_bounds__(256) stage_in_kernel(const uint4* __restrict__ src,
                                                       uint4* __restrict__ dst, size_t n16) {
  pdl_launch_dependents();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// packed_tile dequant: blocks [blk0, blk0 + gridDim.x) of a cell -> fp16 rows
__global__ void dequant_kernel(DevCache c, int cell, int blk0, __half* k_out, __half* v_out) {
  const Geom& G = c.G;
  const int blk = blk0 + blockIdx.x;
  const uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + blk) * G.rec_bytes;
  for (int i = threadIdx.x; i < G.n_r * G.d; i += blockDim.x) {
    const int t = i / G.d, ch = i % G.d;
    const size_t o = (size_t)blockIdx.x * G.n_r * G.d + i;
    k_out[o] = packed_elem(G, rec, t, ch, 0);
    v_out[o] = packed_elem(G, rec, t, ch, 1);
  }
}

// ---------------------------------------------------------------- decode

template <int BITS, int D, int WN>
struct Cfg {
  static constexpr int P = 16 / BITS;
  static constexpr int RB = 16 * WN;               // bytes per channel row
  static constexpr int NW = 4;                     // consumer warps
  static constexpr int NT = (NW + 1) * 32;         // + 1 TMA producer warp
  static constexpr int SB = NW >= WN ? NW / WN : 1;  // blocks per stage
  static constexpr int CPW = WN > NW ? WN / NW : 1;  // chunks per warp per block
  static constexpr int NS = 4;                     // pipeline stages
  static constexpr int NPAIR = P >= 2 ? P / 2 : 1;  // S^T M-tiles per chunk
  static constexpr int KT = D / 16;                // 16-channel tiles
};

struct SoftState {
  float m0, m1;  // running max (log2 domain) of heads 2*t4, 2*t4+1
  float l0, l1;  // thread-partial exp sums
};

// Online-softmax step over NPAIR S^T tiles of 16 tokens (attend_tile,
// attention.cpp:66-89, in the exp2 domain).  Produces the P^T B fragments
// (movmatrix transposes the 8x8 accumulator blocks) and rescales O on a
// warp-uniform max change only.
template <int NPAIR, int KT>
__device__ __forceinline__ void softmax_step(float (&s)[NPAIR][4], SoftState& st,
                                             float (&o)[KT][4], float scale,
                                             uint32_t (&pb)[NPAIR][2], uint32_t (&pl)[NPAIR][2],
                                             bool precise) {
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    mx0 = fmaxf(mx0, fmaxf(s[i][0], s[i][2]));
    mx1 = fmaxf(mx1, fmaxf(s[i][1], s[i][3]));
  }
#pragma unroll
  for (int off = 4; off <= 16; off <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
  }
  const float mn0 = fmaxf(st.m0, mx0 * scale);
  const float mn1 = fmaxf(st.m1, mx1 * scale);
  if (__any_sync(0xffffffffu, mn0 != st.m0 || mn1 != st.m1)) {
    const float r0 = st.m0 == -INFINITY ? 0.f : ex2(st.m0 - mn0);
    const float r1 = st.m1 == -INFINITY ? 0.f : ex2(st.m1 - mn1);
#pragma unroll
    for (int mt = 0; mt < KT; ++mt) {
      o[mt][0] *= r0;
      o[mt][1] *= r1;
      o[mt][2] *= r0;
      o[mt][3] *= r1;
    }
    st.l0 *= r0;
    st.l1 *= r1;
    st.m0 = mn0;
    st.m1 = mn1;
  }
  const float b0 = st.m0 == -INFINITY ? 0.f : st.m0;
  const float b1 = st.m1 == -INFINITY ? 0.f : st.m1;
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    const float p0 = ex2(fmaf(s[i][0], scale, -b0));
    const float p1 = ex2(fmaf(s[i][1], scale, -b1));
    const float p2 = ex2(fmaf(s[i][2], scale, -b0));
    const float p3 = ex2(fmaf(s[i][3], scale, -b1));
    st.l0 += p0 + p2;
    st.l1 += p1 + p3;
    const __half2 h01 = __floats2half2_rn(p0, p1);
    const __half2 h23 = __floats2half2_rn(p2, p3);
    pb[i][0] = movmatrix_t(h2u(h01));
    pb[i][1] = movmatrix_t(h2u(h23));
    if (precise) {
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      pl[i][0] = movmatrix_t(pack_h2(p0 - f01.x, p1 - f01.y));
      pl[i][1] = movmatrix_t(pack_h2(p2 - f23.x, p3 - f23.y));
    }
  }
}


// Per-warp state -> shared -> merged CTA partial (unnormalized O, m, l).
template <int D, int NW>
__device__ __forceinline__ void finalize_part(SoftState st, float (&o)[D / 16][4], float* sm,
                                              float* part_o, float* part_ml, int ng) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int off = 4; off <= 16; off <<= 1) {
    st.l0 += __shfl_xor_sync(0xffffffffu, st.l0, off);
    st.l1 += __shfl_xor_sync(0xffffffffu, st.l1, off);
  }
  constexpr int WS = 8 * D + 16;  // per-warp floats
  named_bar(1, NW * 32);          // every consumer is done with the stage ring
  float* so = sm + warp * WS;
  const int h0 = 2 * t4, h1 = 2 * t4 + 1;
#pragma unroll
  for (int mt = 0; mt < D / 16; ++mt) {
    so[h0 * D + mt * 16 + gid] = o[mt][0];
    so[h1 * D + mt * 16 + gid] = o[mt][1];
    so[h0 * D + mt * 16 + 8 + gid] = o[mt][2];
    so[h1 * D + mt * 16 + 8 + gid] = o[mt][3];
  }
  if (gid == 0) {
    so[8 * D + h0] = st.m0;
    so[8 * D + h1] = st.m1;
    so[8 * D + 8 + h0] = st.l0;
    so[8 * D + 8 + h1] = st.l1;
  }
  named_bar(1, NW * 32);
  for (int i = threadIdx.x; i < ng * D; i += NW * 32) {
    const int h = i / D, ch = i % D;
    float ms = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) ms = fmaxf(ms, sm[w * WS + 8 * D + h]);
    float acc = 0.f, l = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = sm[w * WS + 8 * D + h];
      if (mw == -INFINITY) continue;
      const float f = ex2(mw - ms);
      acc += sm[w * WS + h * D + ch] * f;
      l += sm[w * WS + 8 * D + 8 + h] * f;
    }
    part_o[h * D + ch] = acc;
    if (ch == 0) {
      part_ml[2 * h] = ms;
      part_ml[2 * h + 1] = l;
    }
  }
}

template <int BITS, int D, int WN>
__global__ void __launch_bounds__(Cfg<BITS, D, WN>::NT, 3)
    decode_kernel(DevCache c, DecodeArgs a) {
  using C = Cfg<BITS, D, WN>;
  constexpr int P = C::P, KT = C::KT, NPAIR = C::NPAIR;
  extern __shared__ __align__(128) uint8_t smem[];
  const Geom& G = c.G;
  const int cell = blockIdx.y, part = blockIdx.x, n_parts = gridDim.x;
  const int bidx = cell / G.heads_kv, hk = cell % G.heads_kv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
  const int ng = a.n_group;
  float* part_o = a.part_o + ((size_t)cell * n_parts + part) * ng * D;
  float* part_ml = a.part_ml + ((size_t)cell * n_parts + part) * ng * 2;

  // Q^T B fragments (b0: channels kt*16+2t4.., b1: +8; column n = head gid)
  uint32_t qb[KT][2];
  {
    const __half* qh = a.q + ((size_t)bidx * a.heads_q + (size_t)hk * ng + gid) * D;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      qb[kt][0] = gid < ng ? *reinterpret_cast<const uint32_t*>(qh + kt * 16 + 2 * t4) : 0u;
      qb[kt][1] = gid < ng ? *reinterpret_cast<const uint32_t*>(qh + kt * 16 + 8 + 2 * t4) : 0u;
    }
  }
  const float scale = a.sm_scale_log2;
  const bool precise = a.precise != 0;

  // ===================================================== part 0: residual
  if (part == 0) {
    const int rl0 = a.skip_residual ? 0 : c.res_len[cell];
    const int slot = c.packed_blocks[cell];
    __half* rk = c.res_k + (size_t)cell * G.n_r * D;
    __half* rv = c.res_v + (size_t)cell * G.n_r * D;
    int rlen = rl0;
    if (a.k_new != nullptr) {  // append_token (kvcache.cpp:170-182)
      const __half* kn = a.k_new + (size_t)cell * D;
      const __half* vn = a.v_new + (size_t)cell * D;
      for (int i = threadIdx.x; i < D; i += blockDim.x) {
        rk[(size_t)rl0 * D + i] = kn[i];
        rv[(size_t)rl0 * D + i] = vn[i];
      }
      rlen = rl0 + 1;
    }
    __syncthreads();
    if (warp < C::NW) {
      SoftState st{-INFINITY, -INFINITY, 0.f, 0.f};
      float o[KT][4];
#pragma unroll
      for (int mt = 0; mt < KT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
      for (int tile = warp; tile * 16 < rlen; tile += C::NW) {
        const int t0 = tile * 16;
        const bool v0 = t0 + gid < rlen, v1 = t0 + gid + 8 < rlen;
        float s[1][4] = {{0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          uint32_t af[4];
          const __half* r0 = rk + (size_t)(t0 + gid) * D + kt * 16 + 2 * t4;
          const __half* r1 = r0 + 8 * D;
          af[0] = v0 ? *reinterpret_cast<const uint32_t*>(r0) : 0u;
          af[1] = v1 ? *reinterpret_cast<const uint32_t*>(r1) : 0u;
          af[2] = v0 ? *reinterpret_cast<const uint32_t*>(r0 + 8) : 0u;
          af[3] = v1 ? *reinterpret_cast<const uint32_t*>(r1 + 8) : 0u;
          mma16816(s[0], af, qb[kt][0], qb[kt][1]);
        }
        if (!v0) s[0][0] = s[0][1] = -INFINITY;
        if (!v1) s[0][2] = s[0][3] = -INFINITY;
        uint32_t pb[1][2], pl[1][2];
        softmax_step<1, KT>(s, st, o, scale, pb, pl, precise);
        const int ta = t0 + 2 * t4;  // k rows 2t4, 2t4+1 (and +8)
#pragma unroll
        for (int mt = 0; mt < KT; ++mt) {
          auto ldv = [&](int t, int ch) -> uint32_t {
            return t < rlen ? static_cast<uint32_t>(__half_as_ushort(rv[(size_t)t * D + ch])) : 0u;
          };
          const int ch0 = mt * 16 + gid, ch1 = ch0 + 8;
          uint32_t af[4];
          af[0] = ldv(ta, ch0) | (ldv(ta + 1, ch0) << 16);
          af[1] = ldv(ta, ch1) | (ldv(ta + 1, ch1) << 16);
          af[2] = ldv(ta + 8, ch0) | (ldv(ta + 9, ch0) << 16);
          af[3] = ldv(ta + 8, ch1) | (ldv(ta + 9, ch1) << 16);
          mma16816(o[mt], af, pb[0][0], pb[0][1]);
          if (precise) mma16816(o[mt], af, pl[0][0], pl[0][1]);
        }
      }
      finalize_part<D, C::NW>(st, o, reinterpret_cast<float*>(smem), part_o, part_ml, ng);
    }
    if (a.k_new != nullptr && rlen == G.n_r) {
      // the residual is full: quantize + pack it into block slot `slot`
      // (residual_attend -> build_block, attention.cpp:103; committed by the
      // combine kernel after every part has read the lengths)
      __syncthreads();
      uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + slot) * G.rec_bytes;
      qpack_block<BITS>(G, rk, rv, D, rec, smem);
    }
    return;
  }

  // ============================================= parts 1..S: packed blocks
  const int nblk_cell = c.packed_blocks[cell];
  const int lo_blk = max(a.blk_begin, 0), hi_blk = min(a.blk_end, nblk_cell);
  const int b0 = lo_blk + (part - 1) * a.blocks_per_split;
  const int nblocks = max(0, min(b0 + a.blocks_per_split, hi_blk) - b0);
  const int nst = (nblocks + C::SB - 1) / C::SB;
  const int REC = G.rec_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)C::NS * C::SB * REC);
  uint64_t* empty = full + C::NS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::NW) {  // ---------------- TMA producer warp
    if (lane == 0 && nst > 0) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* src0 = c.records + ((size_t)cell * G.max_blocks + b0) * REC;
      for (int it = 0; it < nst; ++it) {
        const int s = it % C::NS;
        if (it >= C::NS) mbar_wait(&empty[s], ((it / C::NS) - 1) & 1);
        const int nb = min(C::SB, nblocks - it * C::SB);
        const uint32_t bytes = static_cast<uint32_t>(nb * REC);
        mbar_expect_tx(&full[s], bytes);
        tma_bulk_g2s(smem + (size_t)s * C::SB * REC, src0 + (size_t)it * C::SB * REC, bytes,
                     &full[s], pol);
      }
    }
    return;
  }

  // ------------------------------------------------------ consumer warps
  SoftState st{-INFINITY, -INFINITY, 0.f, 0.f};
  float o[KT][4];
#pragma unroll
  for (int mt = 0; mt < KT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  const int vgroups = G.bits == 16 ? 1 : D / G.g;

  for (int it = 0; it < nst; ++it) {
    const int s = it % C::NS;
    mbar_wait(&full[s], (it / C::NS) & 1);
    const uint8_t* stage = smem + (size_t)s * C::SB * REC;
#pragma unroll 1
    for (int u = 0; u < C::CPW; ++u) {
      int kb, j;
      if constexpr (C::SB > 1) {
        kb = warp / WN;
        j = warp % WN;
        if (it * C::SB + kb >= nblocks) break;
      } else {
        kb = 0;
        j = warp * C::CPW + u;
      }
      const uint8_t* rec = stage + (size_t)kb * REC;
      const uint32_t kw = smem_u32(rec), vw = smem_u32(rec + G.wbytes);
      const uint32_t* kp = reinterpret_cast<const uint32_t*>(rec + 2 * G.wbytes);
      const uint32_t* vp = reinterpret_cast<const uint32_t*>(rec + 2 * G.wbytes + G.kp_bytes);

      // ---- S^T = K Q^T over the chunk's 8*P tokens
      float sacc[NPAIR][4];
#pragma unroll
      for (int i = 0; i < NPAIR; ++i) sacc[i][0] = sacc[i][1] = sacc[i][2] = sacc[i][3] = 0.f;
      {
        uint32_t kr[D / 32][4];
#pragma unroll
        for (int kc = 0; kc < D / 32; ++kc) {
          const int row = kc * 32 + lane;
          ldsm_x4_t(kw + row * C::RB + ((j ^ swz(row, WN)) << 4), kr[kc][0], kr[kc][1], kr[kc][2],
                    kr[kc][3]);
        }
        const int kgr = G.k_axis == 0 ? (j * 8 * P) / (G.bits == 16 ? 1 : G.g) : 0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const uint32_t rl = kr[kt / 2][2 * (kt % 2)], rh = kr[kt / 2][2 * (kt % 2) + 1];
          const uint32_t rl8 = rl >> 8, rh8 = rh >> 8;
          __half2 sl, zl, sh, zh;
          if constexpr (BITS != 16) {
            if (G.k_axis == 0) {
              const uint2 pl = *reinterpret_cast<const uint2*>(kp + kgr * D + kt * 16 + 2 * t4);
              const uint2 ph = *reinterpret_cast<const uint2*>(kp + kgr * D + kt * 16 + 8 + 2 * t4);
              sl = u2h(prmt(pl.x, pl.y, 0x5410));
              zl = u2h(prmt(pl.x, pl.y, 0x7632));
              sh = u2h(prmt(ph.x, ph.y, 0x5410));
              zh = u2h(prmt(ph.x, ph.y, 0x7632));
            }
          }
#pragma unroll
          for (int pi = 0; pi < NPAIR; ++pi) {
            uint32_t af[4];
            if constexpr (BITS == 16) {
              af[0] = rl;
              af[1] = 0u;
              af[2] = rh;
              af[3] = 0u;
            } else {
              __half2 c0, c1, c2, c3;
              switch (pi) {  // positions (2pi, 2pi+1)
#define BDK_EXT(PI)                                            \
  case PI:                                                     \
    c0 = ext<BITS, (2 * PI) % P>(rl, rl8);                     \
    c1 = ext<BITS, (2 * PI + 1) % P>(rl, rl8);                 \
    c2 = ext<BITS, (2 * PI) % P>(rh, rh8);                     \
    c3 = ext<BITS, (2 * PI + 1) % P>(rh, rh8);                 \
    break;
                BDK_EXT(0)
                BDK_EXT(1)
                BDK_EXT(2)
                BDK_EXT(3)
#undef BDK_EXT
              }
              if (G.k_axis == 0) {
                af[0] = h2u(__hfma2(c0, sl, zl));
                af[1] = h2u(__hfma2(c1, sl, zl));
                af[2] = h2u(__hfma2(c2, sh, zh));
                af[3] = h2u(__hfma2(c3, sh, zh));
              } else {  // KToken keys: (scale, zero) per (token, channel group)
                const int kg = D / G.g, cg = (kt * 16) / G.g;
                const int te = (8 * j + gid) * P + pos_token(2 * pi, P, G.interleave);
                const int tf = (8 * j + gid) * P + pos_token(2 * pi + 1, P, G.interleave);
                const uint32_t pe = kp[te * kg + cg], pf = kp[tf * kg + cg];
                const __half2 se = u2h(prmt(pe, pe, 0x1010)), ze = u2h(prmt(pe, pe, 0x3232));
                const __half2 sf = u2h(prmt(pf, pf, 0x1010)), zf = u2h(prmt(pf, pf, 0x3232));
                af[0] = h2u(__hfma2(c0, se, ze));
                af[1] = h2u(__hfma2(c1, sf, zf));
                af[2] = h2u(__hfma2(c2, se, ze));
                af[3] = h2u(__hfma2(c3, sf, zf));
              }
            }
            mma16816(sacc[pi], af, qb[kt][0], qb[kt][1]);
          }
        }
      }
      if constexpr (BITS == 16) sacc[0][2] = sacc[0][3] = -INFINITY;  // no second label

      uint32_t pb[NPAIR][2], pl[NPAIR][2];
      softmax_step<NPAIR, KT>(sacc, st, o, scale, pb, pl, precise);

      // ---- O^T += V^T P^T
      uint32_t vr[D / 32][4];
#pragma unroll
      for (int vc = 0; vc < D / 32; ++vc) {
        const int row = vc * 32 + lane;
        ldsm_x4(vw + row * C::RB + ((j ^ swz(row, WN)) << 4), vr[vc][0], vr[vc][1], vr[vc][2],
                vr[vc][3]);
      }
      // V params for the k rows (tokens) of each pair: low half token
      // (8j+2t4)*P + tok(pos), high half (8j+2t4+1)*P + tok(pos)
      __half2 vs[NPAIR][2], vz[NPAIR][2];
      auto load_vparams = [&](int cg) {
#pragma unroll
        for (int pi = 0; pi < NPAIR; ++pi) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ta = (8 * j + 2 * t4) * P + pos_token((2 * pi + e) % P, P, G.interleave);
            const uint32_t pa = vp[ta * vgroups + cg], pbv = vp[(ta + P) * vgroups + cg];
            vs[pi][e] = u2h(prmt(pa, pbv, 0x5410));
            vz[pi][e] = u2h(prmt(pa, pbv, 0x7632));
          }
        }
      };
      if constexpr (BITS != 16) {
        if (vgroups == 1) load_vparams(0);
      }
#pragma unroll
      for (int mt = 0; mt < KT; ++mt) {
        const uint32_t ra = vr[mt / 2][2 * (mt % 2)], rb = vr[mt / 2][2 * (mt % 2) + 1];
        const uint32_t ra8 = ra >> 8, rb8 = rb >> 8;
        if constexpr (BITS != 16) {
          if (vgroups != 1) load_vparams((mt * 16) / G.g);
        }
#pragma unroll
        for (int pi = 0; pi < NPAIR; ++pi) {
          uint32_t af[4];
          if constexpr (BITS == 16) {
            af[0] = ra;
            af[1] = rb;
            af[2] = 0u;
            af[3] = 0u;
          } else {
            __half2 c0, c1, c2, c3;
            switch (pi) {
#define BDK_EXTV(PI)                                           \
  case PI:                                                     \
    c0 = ext<BITS, (2 * PI) % P>(ra, ra8);                     \
    c1 = ext<BITS, (2 * PI) % P>(rb, rb8);                     \
    c2 = ext<BITS, (2 * PI + 1) % P>(ra, ra8);                 \
    c3 = ext<BITS, (2 * PI + 1) % P>(rb, rb8);                 \
    break;
              BDK_EXTV(0)
              BDK_EXTV(1)
              BDK_EXTV(2)
              BDK_EXTV(3)
#undef BDK_EXTV
            }
            af[0] = h2u(__hfma2(c0, vs[pi][0], vz[pi][0]));
            af[1] = h2u(__hfma2(c1, vs[pi][0], vz[pi][0]));
            af[2] = h2u(__hfma2(c2, vs[pi][1], vz[pi][1]));
            af[3] = h2u(__hfma2(c3, vs[pi][1], vz[pi][1]));
          }
          mma16816(o[mt], af, pb[pi][0], pb[pi][1]);
          if (precise) mma16816(o[mt], af, pl[pi][0], pl[pi][1]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  finalize_part<D, C::NW>(st, o, reinterpret_cast<float*>(smem), part_o, part_ml, ng);
}

// combine (attention.cpp:142-162) + cache-update phase (attention.cpp:235-240)
__global__ void combine_kernel(DevCache c, DecodeArgs a, int n_parts, int d) {
  const Geom& G = c.G;
  const int cell = blockIdx.x, ng = a.n_group;
  const int bidx = cell / G.heads_kv, hk = cell % G.heads_kv;
  const float* ml = a.part_ml + (size_t)cell * n_parts * ng * 2;
  const float* po = a.part_o + (size_t)cell * n_parts * ng * d;
  for (int i = threadIdx.x; i < ng * d; i += blockDim.x) {
    const int h = i / d, ch = i % d;
    float ms = -INFINITY;
    for (int p = 0; p < n_parts; ++p) ms = fmaxf(ms, ml[(p * ng + h) * 2]);
    float acc = 0.f, l = 0.f;
    for (int p = 0; p < n_parts; ++p) {
      const float m = ml[(p * ng + h) * 2];
      if (m == -INFINITY) continue;
      const float w = ex2(m - ms);
      acc += po[(p * ng + h) * d + ch] * w;
      l += ml[(p * ng + h) * 2 + 1] * w;
    }
    const size_t row = (size_t)bidx * a.heads_q + (size_t)hk * ng + h;
    a.out[row * d + ch] = l > 0.f ? acc / l : 0.f;
    if (a.out_lse != nullptr && ch == 0) a.out_lse[row] = l > 0.f ? ms + __log2f(l) : -INFINITY;
  }
  if (threadIdx.x == 0 && a.k_new != nullptr) {
    const int r = c.res_len[cell] + 1;
    if (r == G.n_r) {
      c.packed_blocks[cell] += 1;
      c.res_len[cell] = 0;
    } else {
      c.res_len[cell] = r;
    }
  }
}

__global__ void merge_partials_kernel(const float* o, const float* lse, int n_parts, int rows,
                                      int d, size_t o_stride, size_t lse_stride, float* out) {
  const int row = blockIdx.x;
  for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
    float ms = -INFINITY;
    for (int p = 0; p < n_parts; ++p) ms = fmaxf(ms, lse[p * lse_stride + row]);
    float acc = 0.f, l = 0.f;
    for (int p = 0; p < n_parts; ++p) {
      const float m = lse[p * lse_stride + row];
      if (m == -INFINITY) continue;
      const float w = ex2(m - ms);
      acc += o[p * o_stride + (size_t)row * d + ch] * w;
      l += w;
    }
    out[(size_t)row * d + ch] = l > 0.f ? acc / l : 0.f;
  }
}

// Sequence-split exchange over peer memory.
// Rank r's normalized partial [rows*d o | rows lse] (bdk_decode_partial)
// sits in slot step%2 of its own buffer; one launch per rank (1) publishes
// "rank r has step s" with a system-scope release of its monotonic step flag
// (the partial was written by the previous kernel in this stream), (2) waits
// for every peer's flag with system-scope acquires, (3) reads the peers'
// partials straight from their HBM (NVLink P2P loads through the peer
// mapping; plain loads for the local rank) and LSE-merges them (combine,
// attention.cpp:142-162).  Two slots suffice: a rank can only reach step s+2
// after its step s+1 merge saw every peer publish s+1, which each peer does
// after finishing its own step-s merge.  A stuck peer trips the timeout and
// sets *err instead of hanging the GPU.
__global__ void __launch_bounds__(128) peer_merge_kernel(PeerMergeArgs a) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(a.flags[a.rank]),
                   "r"((unsigned)a.step)
                   : "memory");
    }
    int good = 1;
    const unsigned long long t0 = globaltimer();
    for (int p = 0; p < a.world && good; ++p) {
      if (p == a.rank) continue;
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.flags[p]) : "memory");
        if ((int)(v - (unsigned)a.step) >= 0) break;  // monotonic step counter, wrap-safe
        if (globaltimer() - t0 > a.timeout_ns) {
          good = 0;
          atomicExch(a.err, 1);
          break;
        }
        __nanosleep(100);
      }
    }
    ok = good;
  }
  __syncthreads();
  if (!ok) return;
  const int rows = a.rows, d = a.d;
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    float ms = -INFINITY;
    for (int p = 0; p < a.world; ++p) ms = fmaxf(ms, __ldcv(a.parts[p] + (size_t)rows * d + row));
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
      float acc = 0.f, l = 0.f;
      for (int p = 0; p < a.world; ++p) {
        const float m = __ldcv(a.parts[p] + (size_t)rows * d + row);
        if (m == -INFINITY) continue;
        const float w = ex2(m - ms);
        acc = fmaf(__ldcv(a.parts[p] + (size_t)row * d + ch), w, acc);
        l += w;
      }
      a.out[(size_t)row * d + ch] = l > 0.f ? acc / l : 0.f;
      if (a.out_lse != nullptr && ch == 0) a.out_lse[row] = l > 0.f ? ms + __log2f(l) : -INFINITY;
    }
  }
}

// ------------------------------------------------- quant.hpp utilities
// quantize_tile / dequantize_tile / compute_group_params (quant.cpp:18-110)
// for callers of the reference's quant API: one thread per group scanning it
// in the reference's order (strict compares keep the first extremum, so the
// sign of a zero extremum needs no special case), the same IEEE arithmetic
// as the packing kernels.  axis 0 = KChannel (groups along rows, params
// [rows/g][d]), 1 = KToken (groups along d, params [rows][d/g]).
__global__ void quantize_tile_kernel(const float* x, int rows, int d, int bits, int axis, int g,
                                     uint16_t* codes, uint32_t* params) {
  const int n_groups = axis == 0 ? (rows / g) * d : rows * (d / g);
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= n_groups) return;
  // element i of group gi: KChannel group (gr, c) runs over rows gr*g..; KToken (t, gc) over cols
  int base, stride;
  if (axis == 0) {
    const int gr = gi / d, c = gi % d;
    base = gr * g * d + c;
    stride = d;
  } else {
    const int t = gi / (d / g), gc = gi % (d / g);
    base = t * d + gc * g;
    stride = 1;
  }
  float lo = x[base], hi = lo;
  for (int i = 1; i < g; ++i) {
    const float v = x[base + i * stride];
    lo = v < lo ? v : lo;
    hi = hi < v ? v : hi;
  }
  const float qmax = static_cast<float>((1u << bits) - 1u);
  float s, z;
  group_params(lo, hi, qmax, s, z);
  params[gi] = param_u32(s, z);
  for (int i = 0; i < g; ++i)
    codes[base + i * stride] = static_cast<uint16_t>(quant_code(x[base + i * stride], s, z, qmax));
}

// out = round_f16(code * scale + zero), the product and sum each rounded in
// fp32 like the reference's non-contracted `code * scale + zero`
__global__ void dequantize_tile_kernel(const uint16_t* codes, const uint32_t* params, int rows,
                                       int d, int axis, int g, int round16, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * d) return;
  const int t = i / d, c = i % d;
  const int gi = axis == 0 ? (t / g) * d + c : t * (d / g) + c / g;
  const uint32_t p = params[gi];
  const float s = __half2float(__ushort_as_half(static_cast<unsigned short>(p & 0xFFFF)));
  const float z = __half2float(__ushort_as_half(static_cast<unsigned short>(p >> 16)));
  const float v = __fadd_rn(__fmul_rn(static_cast<float>(codes[i]), s), z);
  out[i] = round16 ? __half2float(__float2half_rn(v)) : v;
}

// quantize_group / dequantize_group (quant.cpp:30-44) with explicit fp32
// (scale, zero): codes as quantize_tile, values in fp32 without rounding
__global__ void quantize_group_kernel(const float* x, int n, float s, float z, int bits,
                                      uint16_t* codes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n)
    codes[i] = static_cast<uint16_t>(quant_code(x[i], s, z, static_cast<float>((1u << bits) - 1u)));
}

__global__ void dequantize_group_kernel(const uint16_t* codes, int n, float s, float z,
                                        float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __fadd_rn(__fmul_rn(static_cast<float>(codes[i]), s), z);
}

// ------------------------------------------------------------- launchers

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size high-water mark) instead of on every launch (host-side latency of the
// steady-state decode loop).
static cudaError_t ensure_smem(const void* kern, size_t bytes) {
  struct Entry {
    const void* k;
    int dev;
    size_t bytes;
  };
  static Entry table[256];
  static int n = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < n; ++i)
    if (table[i].k == kern && table[i].dev == dev && table[i].bytes >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(std::max<size_t>(bytes, 16)));
  if (e != cudaSuccess) return e;
  for (int i = 0; i < n; ++i)
    if (table[i].k == kern && table[i].dev == dev) {
      table[i].bytes = bytes;
      return cudaSuccess;
    }
  if (n < 256) table[n++] = Entry{kern, dev, bytes};
  return cudaSuccess;
}

bool fast_path_ok(const Geom& G) {
  if (G.d != 128) return false;
  if (!(G.warp_n == 1 || G.warp_n == 2 || G.warp_n == 4 || G.warp_n == 8)) return false;
  if (G.bits == 16) return true;
  if (G.g % 16 != 0 || G.d % G.g != 0) return false;
  if (G.k_axis == 0 && (G.g % (8 * G.pack) != 0)) return false;
  return true;
}

template <int BITS, int D, int WN>
static cudaError_t decode_launch(const DevCache& c, const DecodeArgs& a, cudaStream_t s) {
  using C = Cfg<BITS, D, WN>;
  const size_t ring = (size_t)C::NS * C::SB * c.G.rec_bytes + 2 * C::NS * sizeof(uint64_t);
  const size_t merge = (size_t)C::NW * (8 * D + 16) * sizeof(float);
  const size_t qp = (size_t)c.G.n_r * D;
  const size_t smem = std::max(ring, std::max(merge, qp));
  auto kern = decode_kernel<BITS, D, WN>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  dim3 grid(1 + a.n_splits, c.G.batch * c.G.heads_kv);
  if (a.ev_begin) cudaEventRecord(a.ev_begin, s);
  kern<<<grid, C::NT, smem, s>>>(c, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (a.ev_end) cudaEventRecord(a.ev_end, s);
  const int nthr = std::min(1024, std::max(32, a.n_group * D));
  combine_kernel<<<c.G.batch * c.G.heads_kv, nthr, 0, s>>>(c, a, 1 + a.n_splits, D);
  return cudaGetLastError();
}

template <int BITS>
static cudaError_t decode_bits(const DevCache& c, const DecodeArgs& a, cudaStream_t s) {
  switch (c.G.warp_n) {
    case 1: return decode_launch<BITS, 128, 1>(c, a, s);
    case 2: return decode_launch<BITS, 128, 2>(c, a, s);
    case 4: return decode_launch<BITS, 128, 4>(c, a, s);
    case 8: return decode_launch<BITS, 128, 8>(c, a, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_decode(const DevCache& c, const DecodeArgs& a, cudaStream_t s) {
  switch (c.G.bits) {
    case 2: return decode_bits<2>(c, a, s);
    case 4: return decode_bits<4>(c, a, s);
    case 8: return decode_bits<8>(c, a, s);
    case 16: return decode_bits<16>(c, a, s);
  }
  return cudaErrorInvalidValue;
}

int max_ctas_per_sm(const Geom&) { return 3; }

template <int BITS>
static cudaError_t prefill_bits(const DevCache& c, const __half* k, const __half* v, int len,
                                int cell_begin, int n_cells, cudaStream_t s) {
  if constexpr (BITS != 16) {
    static const bool fast_off = getenv("BDK_QPACK_FAST") && atoi(getenv("BDK_QPACK_FAST")) == 0;
    if (qpack_fast_ok(c.G) && !fast_off) {
      const QfSmem L = qf_layout(c.G);
      auto kern = qpack_fast_kernel<BITS>;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(L.total));
      if (e != cudaSuccess) return e;
      dim3 grid((len / c.G.n_r) * (c.G.n_r / QF_D) + 1, n_cells, 2);
      kern<<<grid, QF_THREADS, L.total, s>>>(c, k, v, len, cell_begin);
      return cudaGetLastError();
    }
  }
  const size_t smem = (size_t)c.G.n_r * c.G.d;
  auto kern = prefill_kernel<BITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(std::max<size_t>(smem, 16)));
  if (e != cudaSuccess) return e;
  dim3 grid(len / c.G.n_r + 1, n_cells);
  kern<<<grid, 256, smem, s>>>(c, k, v, len, cell_begin);
  return cudaGetLastError();
}

cudaError_t launch_prefill(const DevCache& c, const __half* k, const __half* v, int len,
                           int cell_begin, int n_cells, cudaStream_t s) {
  switch (c.G.bits) {
    case 2: return prefill_bits<2>(c, k, v, len, cell_begin, n_cells, s);
    case 4: return prefill_bits<4>(c, k, v, len, cell_begin, n_cells, s);
    case 8: return prefill_bits<8>(c, k, v, len, cell_begin, n_cells, s);
    case 16: return prefill_bits<16>(c, k, v, len, cell_begin, n_cells, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_append(const DevCache& c, int cell, const __half* k_row, const __half* v_row,
                          cudaStream_t s) {
  append_kernel<<<1, 128, 0, s>>>(c, cell, k_row, v_row);
  return cudaGetLastError();
}

template <int BITS>
static cudaError_t flush_bits(const DevCache& c, int cell, int commit, cudaStream_t s) {
  const size_t smem = (size_t)c.G.n_r * c.G.d;
  auto kern = flush_kernel<BITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(std::max<size_t>(smem, 16)));
  if (e != cudaSuccess) return e;
  kern<<<1, 256, smem, s>>>(c, cell, commit);
  return cudaGetLastError();
}

static cudaError_t flush_any(const DevCache& c, int cell, int commit, cudaStream_t s) {
  switch (c.G.bits) {
    case 2: return flush_bits<2>(c, cell, commit, s);
    case 4: return flush_bits<4>(c, cell, commit, s);
    case 8: return flush_bits<8>(c, cell, commit, s);
    case 16: return flush_bits<16>(c, cell, commit, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_flush(const DevCache& c, int cell, cudaStream_t s) {
  return flush_any(c, cell, 1, s);
}

cudaError_t launch_build(const DevCache& c, int cell, cudaStream_t s) {
  return flush_any(c, cell, 0, s);
}

template <int BITS>
static cudaError_t flush_full_bits(const DevCache& c, cudaStream_t s) {
  const size_t smem = (size_t)c.G.n_r * c.G.d;
  auto kern = flush_full_kernel<BITS>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  kern<<<c.G.batch * c.G.heads_kv, 256, smem, s>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_flush_full(const DevCache& c, cudaStream_t s) {
  switch (c.G.bits) {
    case 2: return flush_full_bits<2>(c, s);
    case 4: return flush_full_bits<4>(c, s);
    case 8: return flush_full_bits<8>(c, s);
    case 16: return flush_full_bits<16>(c, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_stage_in(const void* src_host, void* dst, size_t bytes, cudaStream_t s) {
  const size_t n16 = (bytes + 15) / 16;
  if (n16 == 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<size_t>((n16 + 255) / 256, 148));
  stage_in_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(src_host),
                                        static_cast<uint4*>(dst), n16);
  return cudaGetLastError();
}

cudaError_t launch_dequant(const DevCache& c, int cell, int blk0, int nblk, __half* k_out,
                           __half* v_out, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  dequant_kernel<<<nblk, 256, 0, s>>>(c, cell, blk0, k_out, v_out);
  return cudaGetLastError();
}

cudaError_t launch_merge_partials(const float* o, const float* lse, int n_parts, int rows, int d,
                                  size_t o_stride, size_t lse_stride, float* out, cudaStream_t s) {
  merge_partials_kernel<<<rows, 128, 0, s>>>(o, lse, n_parts, rows, d, o_stride, lse_stride, out);
  return cudaGetLastError();
}

cudaError_t launch_peer_merge(const PeerMergeArgs& a, cudaStream_t s) {
  const int grid = std::max(1, std::min(a.rows, 16));  // few CTAs: never crowd out a peer
  peer_merge_kernel<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_quantize_tile(const float* x, int rows, int d, int bits, int axis, int g,
                                 uint16_t* codes, uint32_t* params, cudaStream_t s) {
  const int n_groups = axis == 0 ? (rows / g) * d : rows * (d / g);
  quantize_tile_kernel<<<(n_groups + 127) / 128, 128, 0, s>>>(x, rows, d, bits, axis, g, codes,
                                                              params);
  return cudaGetLastError();
}

cudaError_t launch_dequantize_tile(const uint16_t* codes, const uint32_t* params, int rows, int d,
                                   int axis, int g, int round16, float* out, cudaStream_t s) {
  dequantize_tile_kernel<<<(rows * d + 255) / 256, 256, 0, s>>>(codes, params, rows, d, axis, g,
                                                                round16, out);
  return cudaGetLastError();
}

cudaError_t launch_quantize_group(const float* x, int n, float s, float z, int bits,
                                  uint16_t* codes, cudaStream_t st) {
  quantize_group_kernel<<<(n + 255) / 256, 256, 0, st>>>(x, n, s, z, bits, codes);
  return cudaGetLastError();
}

cudaError_t launch_dequantize_group(const uint16_t* codes, int n, float s, float z, float* out,
                                    cudaStream_t st) {
  dequantize_group_kernel<<<(n + 255) / 256, 256, 0, st>>>(codes, n, s, z, out);
  return cudaGetLastError();
}

}  // namespace bdk
