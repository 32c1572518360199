// bdk_decode_fast.cu -- the sm_100a decode hot kernel (fast mode).
//
// A step of decode_step for every cell (attention.cpp:164-242) is two grids:
//   decode_fast_kernel   residual_attend + packed_attend as stream-K
//                        partials, with the append of the new token fused in;
//   combine_fast_kernel  combine (the LSE merge of each cell's partials), the
//                        commit of the cell's lengths and the flush of a
//                        residual window the step filled (kvcache.cpp:
//                        208-237); a programmatic dependent of the first.
//
// Schedule -- stream-K over units.  Cell c (= b * heads_kv + h) owns
// nb_c + 1 units: its packed blocks (in the attended range) and, last, its
// residual window.  The grid is exactly the resident CTA capacity of the GPU;
// CTA i takes units [i*T/N, (i+1)*T/N) of the flattened sequence, so every
// SM streams the same number of blocks whatever the batch / context shape
// (b=1 128K and b=32 8K alike).  A CTA range may span several cells; each
// (CTA, cell) segment leaves one partial (unnormalized O, running max, sum)
// in slot i + c (injective); the combine grid merges the slots of cell c,
// those of CTAs cta_of_unit(first unit of c) .. cta_of_unit(last unit of c).
//
// CTA = WN consumer warps + 1 TMA warp + 1 prep warp:
//   TMA warp   one lane streams whole block records (K words | V words |
//              K params | V params, ~17 KB) HBM -> SMEM with cp.async.bulk
//              into an NS-stage mbarrier ring (full / empty barriers).
//   prep warp  per block: folds the channel-wise K scales into the query,
//              Q'[h][c] = fp16(q[h][c] * s_c), and the zero-points into one
//              scalar per head, Z[h] = sum_c q[h][c] z_c (fp32); converts the
//              per-token V (scale, zero) to fp32.  Signals a prep barrier.
//   consumers  warp w owns 16-byte chunk w (8*P tokens) of every channel row:
//              ldmatrix.trans (K) / ldmatrix (V) of the packed words, exact
//              code extraction (lop3 + hsub2/hfma2, bdk_frag.cuh), mma.sync
//              m16n8k16 in swap-AB form  S^T = codes_K . Q'^T  (tokens in M,
//              GQA heads in N), online softmax in the exp2 domain with the
//              logits S = S' + Z, then O^T += codes_V^T . (P s_t)^T  plus the
//              per-head zero term sum_t P z_t accumulated in fp32.
//
// Numerics (fast mode): the folds replace the
// reference's round_f16(code*scale + zero) staging by fp16(q*s) and fp16(P*s)
// roundings of the same magnitude; the fp32 accumulation is unchanged.  The
// bit-faithful dequant path is the exact kernel in bdk_kernels.cu.
#include <cfloat>
#include <cstdlib>

#include "bdk_frag.cuh"
#include "bdk_launch.h"
#include "bdk_qpack.cuh"
#include "bdk_qpack_fast.cuh"

namespace bdk {

namespace {

constexpr int D = 128;
constexpr int KT = D / 16;
constexpr int QP_ROW = 272;                    // bytes per Q' head row (256 + 16 pad)
constexpr int QP_BYTES = 8 * QP_ROW + 8 * 4;  // Q' [8 heads] + Z [8] per K group
constexpr int OT = KT;                        // O^T accumulator tiles
constexpr int MERGE_KC = 64;                   // contributors per merge round
constexpr int MERGE_LB = 20;                   // slot loads in flight per thread

template <int BITS, int WN, int MINB_, int GRP_>
struct FC {
  static constexpr int P = 16 / BITS;
  static constexpr int NPAIR = P / 2;          // S^T m16 tiles per chunk (P >= 2)
  static constexpr int RB = 16 * WN;           // bytes per channel row
  static constexpr int NC = WN * GRP_;         // consumer warps (+ TMA warp + GRP_ prep warps)
};

// Record geometry of the fast path, fixed by (bits, W_n): d = 128, g = 128,
// KChannel K (fast_decode_ok), N_r = 8 W_n (16 / bits).  Word bytes per
// tensor 16 W_n d, K params (N_r / 128) d (scale, zero) u16 pairs, V params
// N_r pairs, the record padded to 128 B (bdk_api.cu's Geom, checked at launch)
template <int BITS, int WN>
struct FG {
  static constexpr int NR = 8 * WN * (16 / BITS);
  static constexpr int GPB = NR / 128 > 0 ? NR / 128 : 1;
  static constexpr int WB = 16 * WN * 128;
  static constexpr int KPB = GPB * 128 * 4;
  static constexpr int VPB = NR * 4;
  static constexpr int REC = (2 * WB + KPB + VPB + 127) / 128 * 128;
  static constexpr int PREP_STRIDE = (GPB * (8 * 272 + 8 * 4) + 127) / 128 * 128;
};

struct Smem {
  uint32_t ring, prep, merge;  // byte offsets
  uint32_t prep_stride;
  uint32_t merge_floats;
  uint32_t total;
};

// column packing: with n_group <= 4 an S^T tile only fills accumulator
// columns 0..3 (heads); the partner tile (same field shifts) is accumulated
// into columns 4..7 of the same registers, halving the softmax work.  Used
// at 2-bit (4 tiles per chunk: measured +1% on C2); at 4-bit the two tiles
// per chunk leave too little to share (measured -3% on C5).
__host__ __device__ inline int col_pack(const Geom& G, int ng) {
  return (ng <= 4 && G.bits == 2) ? 2 : 1;
}

__host__ __device__ inline Smem smem_layout(const Geom& G, int ng, int NS, int grp) {
  Smem L;
  const int gpb = G.k_axis == 0 ? G.n_r / G.g : 1;
  L.ring = 0;
  L.prep_stride = (uint32_t)((gpb * QP_BYTES + 127) / 128 * 128);
  L.prep = L.ring + NS * G.rec_bytes;
  L.merge = L.prep + NS * L.prep_stride;
  const uint32_t merge_bytes = (uint32_t)(
      max(G.warp_n * grp * (((ng <= 4 && (G.bits == 2 || G.bits == 4)) ? 2 : 1) * ng * D + 16), 24 + 2 * MERGE_KC * 8 + 4 * 32 * G.warp_n * grp) *
          4 +
      64);
  L.merge_floats = merge_bytes / 4;
  L.total = L.merge + merge_bytes + 3 * NS * 8 + 48 + 128;  // + flag, claims, schedule scratch
  return L;
}

__device__ __forceinline__ int cta_of_unit(long long u, long long T, int N) {
  return (int)(((u + 1) * (long long)N - 1) / T);
}

// The step's schedule.  Cell c owns nb_c packed blocks of the attended range
// then max(1, ceil(rlen_c / rt)) residual units of rt tokens.  Lengths live in
// the half of the double buffer that no CTA writes during this step
// (DevCache::len2, FastArgs::par).  Host schedule (dev == 0): the unit counts
// come from the launch arguments (uniform cells) or the uploaded prefix
// arrays; device schedule (dev == 1, graph steps): from the lengths (L2 loads).
struct Sched {
  // a view of the launch parameters (__grid_constant__: read from the
  // constant bank on use, so nothing here occupies registers in the hot loop)
  const DevCache* c;
  const FastArgs* a;
  int cells, rt;
  __device__ __forceinline__ const int* pb() const { return c->len2 + (size_t)a->par * 2 * cells; }
  __device__ __forceinline__ const int* rl() const { return pb() + cells; }
  __device__ __forceinline__ int* pb_n() const { return c->len2 + (size_t)(a->par ^ 1) * 2 * cells; }
  __device__ __forceinline__ int* rl_n() const { return pb_n() + cells; }
  __device__ __forceinline__ int radd() const {
    return a->skip_residual ? -1 : (a->k_new != nullptr ? 1 : 0);
  }
  __device__ __forceinline__ int nb(int cell) const {
    if (!a->dev_sched) return a->uni_units ? a->uni_nb : __ldg(a->unit_nb + cell);
    return max(0, min(a->blk_end, __ldcg(pb() + cell)) - a->blk_begin);
  }
  __device__ __forceinline__ int rlen(int cell) const {
    return radd() < 0 ? 0 : __ldcg(rl() + cell) + radd();
  }
  __device__ __forceinline__ int units(int cell, int nbc) const {
    if (!a->dev_sched)
      return a->uni_units ? a->uni_units : __ldg(a->unit_off + cell + 1) - __ldg(a->unit_off + cell);
    return nbc + max(1, (rlen(cell) + rt - 1) / rt) + a->res_extra;
  }
};

__device__ __forceinline__ Sched make_sched(const DevCache& c, const FastArgs& a, int cells, int rt) {
  return Sched{&c, &a, cells, rt};
}

__device__ __forceinline__ int ld_acquire_gpu_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct SchedOut {
  long long T, off0;  // total units; first unit of cell0
  int cell0;
};

// host schedule: the cell holding unit u (largest c with unit_off[c] <= u)
__device__ __forceinline__ int find_cell(const int* off, int cells, long long u) {
  int lo = 0, hi = cells - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)__ldg(off + mid) <= u)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ SchedOut sched_host(const Sched& S, const FastArgs& a, int cells) {
  const long long T = a.total_units;
  const long long neff = min((long long)gridDim.x, T);
  const long long ub = (long long)blockIdx.x < neff ? (long long)blockIdx.x * T / neff : T;
  if (ub >= T) return SchedOut{T, T, cells};
  if (a.uni_units) {
    const int c0 = (int)(ub / a.uni_units);
    return SchedOut{T, (long long)c0 * a.uni_units, c0};
  }
  const int c0 = find_cell(a.unit_off, cells, ub);
  return SchedOut{T, (long long)__ldg(a.unit_off + c0), c0};
}

// Block-wide scan of the cells' unit counts: total T and, for this CTA's
// first unit u_begin = blockIdx.x * T / N, the cell holding it and that
// cell's first unit.  All threads of the CTA; ends with __syncthreads.
__device__ __forceinline__ SchedOut sched_scan(const Sched& S, int cells, long long* sm) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nt >> 5;
  const int per = (cells + nt - 1) / nt;
  const int c0 = min(cells, tid * per), c1 = min(cells, c0 + per);
  long long s = 0;
  for (int cc = c0; cc < c1; ++cc) s += S.units(cc, S.nb(cc));
  long long x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < nw ? sm[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) sm[lane] = w;
  }
  __syncthreads();
  const long long T = sm[nw - 1];
  const long long excl = x - s + (warp ? sm[warp - 1] : 0);
  // CTAs [0, min(N, T)) share the units (no empty range between two CTAs
  // of one cell); the rest are idle
  const long long neff = min((long long)gridDim.x, T);
  const long long ub = (long long)blockIdx.x < neff ? (long long)blockIdx.x * T / neff : T;
  __syncthreads();  // sm is reused for the result
  if (s > 0 && excl <= ub && ub < excl + s) {
    long long off = excl;
    for (int cc = c0; cc < c1; ++cc) {
      const long long u = S.units(cc, S.nb(cc));
      if (ub < off + u) {
        sm[0] = cc;
        sm[1] = off;
        break;
      }
      off += u;
    }
  }
  if (ub >= T && tid == 0) {  // idle CTA (T < N)
    sm[0] = cells;
    sm[1] = T;
  }
  __syncthreads();
  SchedOut r{T, sm[1], (int)sm[0]};
  __syncthreads();
  return r;
}

// next block index from a chunk position's claim counter (lane 0 claims,
// the warp shares it)
__device__ __forceinline__ int claim_next(int* ctr, int lane) {
  int k = 0;
  if (lane == 0) k = atomicAdd(ctr, 1);
  return __shfl_sync(0xffffffffu, k, 0);
}

// online-softmax state of one consumer warp (columns = heads 2*t4, 2*t4+1)
struct Soft {
  float m0, m1, l0, l1, z0, z1;  // z: sum_t P_t * zero_t (V zero-point term)
};

template <int KTILES>
__device__ __forceinline__ void rescale(Soft& st, float (&o)[KTILES][4], float r0, float r1) {
#pragma unroll
  for (int mt = 0; mt < KTILES; ++mt) {
    o[mt][0] *= r0;
    o[mt][1] *= r1;
    o[mt][2] *= r0;
    o[mt][3] *= r1;
  }
  st.l0 *= r0;
  st.l1 *= r1;
  st.z0 *= r0;
  st.z1 *= r1;
}

// Online softmax over NPAIR S^T tiles of logits x (log2 domain), in place:
// x <- exp2(x - m).  Lazy rescaling: the running max m (warp-uniform per
// head) is only raised -- with the cross-lane reduction and the O rescale --
// when some logit exceeds it by more than TAU, so P <= 2^TAU and the common
// path costs one vote instead of three shuffle rounds.  Exact in real
// arithmetic; m only sets the scale of the fp32 state.
constexpr float TAU = 6.f;

template <int NPAIR>
__device__ __forceinline__ void softmax_update(float (&x)[NPAIR][4], Soft& st, float (&o)[OT][4]) {
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    mx0 = fmaxf(mx0, fmaxf(x[i][0], x[i][2]));
    mx1 = fmaxf(mx1, fmaxf(x[i][1], x[i][3]));
  }
  if (__any_sync(0xffffffffu, mx0 > st.m0 + TAU || mx1 > st.m1 + TAU)) {
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(st.m0, mx0), mn1 = fmaxf(st.m1, mx1);
    const float r0 = st.m0 == -INFINITY ? 0.f : ex2(st.m0 - mn0);
    const float r1 = st.m1 == -INFINITY ? 0.f : ex2(st.m1 - mn1);
    rescale<OT>(st, o, r0, r1);
    st.m0 = mn0;
    st.m1 = mn1;
  }
  const float b0 = st.m0 == -INFINITY ? 0.f : st.m0;
  const float b1 = st.m1 == -INFINITY ? 0.f : st.m1;
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    x[i][0] = ex2(x[i][0] - b0);
    x[i][1] = ex2(x[i][1] - b1);
    x[i][2] = ex2(x[i][2] - b0);
    x[i][3] = ex2(x[i][3] - b1);
    st.l0 += x[i][0] + x[i][2];
    st.l1 += x[i][1] + x[i][3];
  }
}

// consumer-warp partial of a segment -> CTA partial in `slot`.  With column
// packing (CP = 2) accumulator columns 4..7 hold a second online-softmax
// stream of heads 0..3 (the partner tiles), merged here like another warp.
template <int NC, int CP>
__device__ __forceinline__ void finalize_segment(Soft st, float (&o)[OT][4], float* sm, int ng,
                                                 float* slot, float oscale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int off = 4; off <= 16; off <<= 1) {
    st.l0 += __shfl_xor_sync(0xffffffffu, st.l0, off);
    st.l1 += __shfl_xor_sync(0xffffffffu, st.l1, off);
    st.z0 += __shfl_xor_sync(0xffffffffu, st.z0, off);
    st.z1 += __shfl_xor_sync(0xffffffffu, st.z1, off);
  }
  const int nvc = CP * ng;  // virtual columns: (stream, head)
  const int WS = nvc * D + 16;
  float* so = sm + warp * WS;
  // accumulator columns 2*t4, 2*t4+1 -> (stream, head) -> virtual column
  const int c0 = 2 * t4, c1 = 2 * t4 + 1;
  const int hh0 = CP == 2 ? (c0 & 3) : c0, hh1 = CP == 2 ? (c1 & 3) : c1;
  const int v0 = CP == 2 ? (c0 >> 2) * ng + hh0 : c0, v1 = CP == 2 ? (c1 >> 2) * ng + hh1 : c1;
#pragma unroll
  for (int mt = 0; mt < KT; ++mt) {
    const int ch = mt * 16 + gid;
    // undo the subnormal-mode scale of the V codes (2^(24 - SH_REF)) and add
    // the zero-point term
    if (hh0 < ng) {
      so[v0 * D + ch] = fmaf(o[mt][0], oscale, st.z0);
      so[v0 * D + ch + 8] = fmaf(o[mt][2], oscale, st.z0);
    }
    if (hh1 < ng) {
      so[v1 * D + ch] = fmaf(o[mt][1], oscale, st.z1);
      so[v1 * D + ch + 8] = fmaf(o[mt][3], oscale, st.z1);
    }
  }
  if (gid == 0) {
    if (hh0 < ng) {
      so[nvc * D + v0] = st.m0;
      so[nvc * D + 8 + v0] = st.l0;
    }
    if (hh1 < ng) {
      so[nvc * D + v1] = st.m1;
      so[nvc * D + 8 + v1] = st.l1;
    }
  }
  named_bar(1, NC * 32);
  for (int i = threadIdx.x; i < ng * D; i += NC * 32) {
    const int h = i / D, ch = i % D;
    float ms = -INFINITY;
#pragma unroll
    for (int w = 0; w < NC; ++w)
#pragma unroll
      for (int sidx = 0; sidx < CP; ++sidx) ms = fmaxf(ms, sm[w * WS + nvc * D + sidx * ng + h]);
    float acc = 0.f, l = 0.f;
#pragma unroll
    for (int w = 0; w < NC; ++w) {
#pragma unroll
      for (int sidx = 0; sidx < CP; ++sidx) {
        const int vc = sidx * ng + h;
        const float mw = sm[w * WS + nvc * D + vc];
        const float f = mw == -INFINITY ? 0.f : ex2(mw - ms);
        acc += sm[w * WS + vc * D + ch] * f;
        l += sm[w * WS + nvc * D + 8 + vc] * f;
      }
    }
    slot[i] = acc;
    if (ch == 0) {
      slot[ng * D + 2 * h] = ms;
      slot[ng * D + 2 * h + 1] = l;
    }
  }
  named_bar(1, NC * 32);
}

// f32 += f16 * f16 as one FHFMA (sm_100): the product of two binary16 values
// is exact in fp32, so this equals fmaf(float(a), float(b), c) bit for bit
__device__ __forceinline__ float fhfma(uint16_t a, uint16_t b, float c) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"(a), "h"(b));
  return c;
}

// Fold of one staged block for the prep warp: Q'[h][c] = fp16(q[h][c] s_c)
// and Z[h] = sum_c q[h][c] z_c for every K group of the block (q2: this
// lane's query channels as half2).  The params are (scale | zero << 16) u32
// per channel; the zero terms take the high halves directly (FHFMA half
// selects: no conversions, no repacking).
// GPB: K groups per block, N_r / 128 -- a compile-time constant of the
// kernel (N_r = 8 W_n (16 / bits), and the fast path has g = 128)
template <int NH, int GPB>
__device__ __forceinline__ void prep_fold(const uint8_t* rec, uint8_t* pp, const Geom& G, int ng,
                                          const uint32_t (&q2)[D / (32 / NH) / 2]) {
  constexpr int LPH = 32 / NH;  // lanes per head
  constexpr int CPL = D / LPH;  // channels per lane
  constexpr int H2 = CPL / 2;   // half2 per lane
  const int lane = threadIdx.x & 31;
  const int h = lane % NH, cbk = lane / NH;
  constexpr int gpb = GPB;
  const uint32_t* kp = reinterpret_cast<const uint32_t*>(rec + 2 * G.wbytes);
#pragma unroll
  for (int gr = 0; gr < gpb; ++gr) {
    uint8_t* qp = pp + gr * QP_BYTES;
    float za = 0.f, zb = 0.f;
    uint32_t qo[H2];
    uint32_t pw[CPL];
    if constexpr (CPL % 4 == 0) {
#pragma unroll
      for (int v = 0; v < CPL / 4; ++v) {
        const uint4 x = *reinterpret_cast<const uint4*>(kp + gr * D + cbk * CPL + 4 * v);
        pw[4 * v] = x.x;
        pw[4 * v + 1] = x.y;
        pw[4 * v + 2] = x.z;
        pw[4 * v + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int v = 0; v < CPL / 2; ++v) {
        const uint2 x = *reinterpret_cast<const uint2*>(kp + gr * D + cbk * CPL + 2 * v);
        pw[2 * v] = x.x;
        pw[2 * v + 1] = x.y;
      }
    }
#pragma unroll
    for (int i = 0; i < H2; ++i) {
      const uint32_t p0 = pw[2 * i], p1 = pw[2 * i + 1];
      const __half2 s2 = u2h(prmt(p0, p1, 0x5410));
      qo[i] = h2u(__hmul2(u2h(q2[i]), s2));
      za = fhfma((uint16_t)(q2[i] & 0xFFFFu), (uint16_t)(p0 >> 16), za);
      zb = fhfma((uint16_t)(q2[i] >> 16), (uint16_t)(p1 >> 16), zb);
    }
    if (h < ng) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(qp + h * QP_ROW + cbk * CPL * 2);
      if constexpr (H2 % 4 == 0) {
#pragma unroll
        for (int v = 0; v < H2 / 4; ++v)
          reinterpret_cast<uint4*>(dst)[v] =
              make_uint4(qo[4 * v], qo[4 * v + 1], qo[4 * v + 2], qo[4 * v + 3]);
      } else {
#pragma unroll
        for (int v = 0; v < H2; ++v) dst[v] = qo[v];
      }
    }
    float zacc = za + zb;
#pragma unroll
    for (int off = NH; off < 32; off <<= 1) zacc += __shfl_xor_sync(0xffffffffu, zacc, off);
    if (cbk == 0 && h < ng) reinterpret_cast<float*>(qp + 8 * QP_ROW)[h] = zacc;
  }
}

struct PrepCtx {
  const uint8_t* ring;
  uint8_t* prep;
  uint64_t* full;
  uint64_t* ready;
  unsigned long long* tr;
  int rec, prep_stride, pgrp;
  long long u_begin, u_end, off0;
  int cell0;
  int rt;  // residual tokens per unit
};

// Prep warp: per packed block of its consumer group, fold the channel-wise K
// scales into the query, Q'[h][c] = fp16(q[h][c] s_c), and the zero points
// into Z[h] = sum_c q[h][c] z_c (fp32), for every K group of the block.
// NH = n_group rounded up to a power of two: lane -> (head lane % NH, a block
// of 4*NH channels), so only real heads cost work; Q' rows of heads >= n_group
// stay zero (prep areas are zeroed at kernel start).
template <int NH, int NS, int GRP, int GPB>
__device__ __forceinline__ void prep_loop(const DevCache& c, const FastArgs& a, const PrepCtx& px) {
  constexpr int LPH = 32 / NH;  // lanes per head
  constexpr int CPL = D / LPH;  // channels per lane
  constexpr int H2 = CPL / 2;   // half2 per lane
  const Geom& G = c.G;
  const int lane = threadIdx.x & 31;
  const int h = lane % NH, cbk = lane / NH;
  const int ng = a.n_group;
  const Sched S = make_sched(c, a, G.batch * G.heads_kv, px.rt);
  int it = 0;
  long long u = px.u_begin, off = px.off0;
  for (int cell = px.cell0; u < px.u_end; ++cell) {
    const int nbc = S.nb(cell);
    const long long ce = off + S.units(cell, nbc);
    const long long seg_end = min(px.u_end, ce);
    const long long pk_end = min(seg_end, off + nbc);
    if (u < pk_end) {
      const int bidx = cell / G.heads_kv, hk = cell % G.heads_kv;
      uint32_t q2[H2];
#pragma unroll
      for (int i = 0; i < H2; ++i) q2[i] = 0u;
      if (h < ng) {
        const uint32_t* qs = reinterpret_cast<const uint32_t*>(
            a.q + ((size_t)bidx * a.heads_q + (size_t)hk * ng + h) * D + cbk * CPL);
#pragma unroll
        for (int i = 0; i < H2; ++i) q2[i] = __ldg(qs + i);
      }
      for (long long x = u; x < pk_end; ++x, ++it) {
        if (GRP > 1 && (it % GRP) != px.pgrp) continue;
        const int s = it % NS;
        const unsigned long long tw = (px.tr && lane == 0) ? globaltimer() : 0ull;
        mbar_wait_sleep(&px.full[s], (it / NS) & 1);
        const unsigned long long tb = (px.tr && lane == 0) ? globaltimer() : 0ull;
        if (px.tr && lane == 0) px.tr[12] += tb - tw;
        if (!(a.dev_flags & 2)) {
          prep_fold<NH, GPB>(px.ring + (size_t)s * px.rec, px.prep + (size_t)s * px.prep_stride, G,
                             ng, q2);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&px.ready[s]);
        if (px.tr && lane == 0) px.tr[13] += globaltimer() - tb;
      }
    }
    u = seg_end;
    off = ce;
  }
}

// One packed block (one 16-byte chunk j of every channel row) of a consumer
// warp, in four stages (so the consumer loop can software-pipeline them):
//   qk_stage   S^T = codes_K . Q'^T -> logits (log2 domain, zero term folded)
//   soft_stage online softmax, zero term, P' = P * s_t -> P'^T fragments
//   ldv_stage  ldmatrix of the V words into registers, release of the stage
//   pv_stage   O^T += codes_V^T . P'^T
// `rec` is the staged block record, `qp` its folded query (prep warp).
template <int BITS, int WN, int CP>
struct Stg {
  using C = FC<BITS, WN, 1, 1>;
  static constexpr int P = C::P, NPAIR = C::NPAIR, RB = C::RB;
  static constexpr int NPK = NPAIR / CP;
  static constexpr int NPH = CP == 2 ? NPK : 1;
  static constexpr int SH_REF = BITS == 8 ? 0 : 2;
};

template <int BITS, int WN, int CP>
__device__ __forceinline__ void qk_stage(const uint8_t* rec, const uint8_t* qp, int j, float scale,
                                         float (&sacc)[Stg<BITS, WN, CP>::NPK][4]) {
  using T = Stg<BITS, WN, CP>;
  constexpr int P = T::P, NPAIR = T::NPAIR, RB = T::RB, NPK = T::NPK;
  const int lane = threadIdx.x & 31, t4 = lane & 3;
  // Q'^T B fragments (ldmatrix of the [head][channel] rows; rows >= n_group
  // are zero).  CP = 2: qh = the same heads in columns 4..7 (each lane's
  // row address is r ^ 4, so columns 0..3 read the zero rows 4..7)
  uint32_t qb[KT][2], qh[CP == 2 ? KT : 1][2];
  {
    const int mi = lane >> 3, r = lane & 7;
#pragma unroll
    for (int kk = 0; kk < KT / 2; ++kk) {
      const int kt = 2 * kk + (mi >> 1);
      const int cof = (kt * 16 + (mi & 1) * 8) * 2;
      ldsm_x4(smem_u32(qp + r * QP_ROW + cof), qb[2 * kk][0], qb[2 * kk][1], qb[2 * kk + 1][0],
              qb[2 * kk + 1][1]);
      if constexpr (CP == 2)
        ldsm_x4(smem_u32(qp + (r ^ 4) * QP_ROW + cof), qh[2 * kk][0], qh[2 * kk][1],
                qh[2 * kk + 1][0], qh[2 * kk + 1][1]);
    }
  }
  const float2 zz =
      *reinterpret_cast<const float2*>(qp + 8 * QP_ROW + 8 * (CP == 2 ? (t4 & 1) : t4));
  const float zs0 = zz.x * scale, zs1 = zz.y * scale;

  // ---- S^T = codes_K . Q'^T over the chunk's 8*P tokens.  Tile pi goes
  // to packed accumulator pi % NPK (columns 0..3 for pi < HALF, 4..7 for
  // the partner pi >= HALF when CP = 2).  Independent HMMA chains: one per
  // (accumulator, column half), and per channel-tile parity when few.
  constexpr int HALF = NPAIR / 2;
  constexpr bool KSPLIT = NPAIR <= 2;
  constexpr int NCH = NPK * CP * (KSPLIT ? 2 : 1);
  float chn[NCH][4];
#pragma unroll
  for (int i = 0; i < NCH; ++i) chn[i][0] = chn[i][1] = chn[i][2] = chn[i][3] = 0.f;
  {
    const uint32_t kw = smem_u32(rec);
    uint32_t kr[4][4];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      const int row = kc * 32 + lane;
      ldsm_x4_t(kw + row * RB + ((j ^ swz(row, WN)) << 4), kr[kc][0], kr[kc][1], kr[kc][2],
                kr[kc][3]);
    }
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const uint32_t rl = kr[kt / 2][2 * (kt % 2)], rh = kr[kt / 2][2 * (kt % 2) + 1];
      const uint32_t rl8 = rl >> 8, rh8 = rh >> 8;
#pragma unroll
      for (int pi = 0; pi < NPAIR; ++pi) {
        uint32_t af[4];
#define BDK_KEXT(PI)                                 \
  if (pi == PI) {                                    \
    af[0] = ext_sub<BITS, (2 * PI) % P>(rl, rl8);     \
    af[1] = ext_sub<BITS, (2 * PI + 1) % P>(rl, rl8); \
    af[2] = ext_sub<BITS, (2 * PI) % P>(rh, rh8);     \
    af[3] = ext_sub<BITS, (2 * PI + 1) % P>(rh, rh8); \
  }
        BDK_KEXT(0)
        BDK_KEXT(1)
        BDK_KEXT(2)
        BDK_KEXT(3)
#undef BDK_KEXT
        const int f = (CP == 2 && pi >= HALF) ? 1 : 0;
        const int ci = pi % NPK + NPK * (f + CP * (KSPLIT ? (kt & 1) : 0));
        if (f)
          mma16816(chn[ci], af, qh[CP == 2 ? kt : 0][0], qh[CP == 2 ? kt : 0][1]);
        else
          mma16816(chn[ci], af, qb[kt][0], qb[kt][1]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NPK; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float x = chn[i][r];
#pragma unroll
      for (int k = 1; k < NCH / NPK; ++k) x += chn[i + k * NPK][r];
      sacc[i][r] = x;
    }
  // ---- logits (log2 domain): S = S' 2^(24 - sh) + Z (rows gid / gid+8
  // hold fields 2i / 2i+1; the partner tile i + HALF has the same field
  // shifts)
#pragma unroll
  for (int i = 0; i < NPK; ++i) {
    const float al = scale * (float)(1 << (24 - ((2 * i) % P) * BITS % 8));
    const float ah = scale * (float)(1 << (24 - ((2 * i + 1) % P) * BITS % 8));
    sacc[i][0] = fmaf(sacc[i][0], al, zs0);
    sacc[i][1] = fmaf(sacc[i][1], al, zs1);
    sacc[i][2] = fmaf(sacc[i][2], ah, zs0);
    sacc[i][3] = fmaf(sacc[i][3], ah, zs1);
  }
}

template <int BITS, int WN, int CP>
__device__ __forceinline__ void soft_stage(const uint8_t* rec, const Geom& G, int j,
                                           const int (&vtok)[Stg<BITS, WN, CP>::NPK][2],
                                           float (&sacc)[Stg<BITS, WN, CP>::NPK][4], Soft& st,
                                           float (&o)[OT][4],
                                           uint32_t (&pb)[Stg<BITS, WN, CP>::NPK][2],
                                           uint32_t (&pbh)[Stg<BITS, WN, CP>::NPH][2]) {
  using T = Stg<BITS, WN, CP>;
  constexpr int P = T::P, NPK = T::NPK, SH_REF = T::SH_REF;
  const int lane = threadIdx.x & 31, gid = lane >> 2;
  using F = FG<BITS, WN>;
  const uint32_t* vpr = reinterpret_cast<const uint32_t*>(rec + 2 * F::WB + F::KPB);
  softmax_update<NPK>(sacc, st, o);
  // ---- P' = P * s_t (V token scale folded), zero term, P'^T fragments
#pragma unroll
  for (int i = 0; i < NPK; ++i) {
    // V (scale, zero) of the tokens of rows gid / gid+8 (fields 2i / 2i+1
    // of this lane's tile); the scale carries 2^(SH_REF - sh) of the
    // field's subnormal shift
    const int g0 = (8 * j + gid) * P;
    const float2 pa = __half22float2(u2h(vpr[g0 + vtok[i][0]]));
    const float2 pz = __half22float2(u2h(vpr[g0 + vtok[i][1]]));
    const float2 sz0 = make_float2(
        pa.x * (float)(1 << (SH_REF + 8)) / (float)(1 << (8 + ((2 * i) % P) * BITS % 8)), pa.y);
    const float2 sz1 = make_float2(
        pz.x * (float)(1 << (SH_REF + 8)) / (float)(1 << (8 + ((2 * i + 1) % P) * BITS % 8)),
        pz.y);
    st.z0 = fmaf(sacc[i][0], sz0.y, fmaf(sacc[i][2], sz1.y, st.z0));
    st.z1 = fmaf(sacc[i][1], sz0.y, fmaf(sacc[i][3], sz1.y, st.z1));
    pb[i][0] = movmatrix_t(pack_h2(sacc[i][0] * sz0.x, sacc[i][1] * sz0.x));
    pb[i][1] = movmatrix_t(pack_h2(sacc[i][2] * sz1.x, sacc[i][3] * sz1.x));
  }
  // CP = 2: P'^T of tile i keeps only its column half (head columns n =
  // gid after the transpose)
  if constexpr (CP == 2) {
#pragma unroll
    for (int i = 0; i < NPK; ++i) {
      pbh[i][0] = gid >= 4 ? pb[i][0] : 0u;
      pbh[i][1] = gid >= 4 ? pb[i][1] : 0u;
      pb[i][0] = gid < 4 ? pb[i][0] : 0u;
      pb[i][1] = gid < 4 ? pb[i][1] : 0u;
    }
  }
}

// V words of the chunk into registers; then the ring slot and its prep slot
// are free (every read of the stage is done)
template <int BITS, int WN, int CP>
__device__ __forceinline__ void ldv_stage(const uint8_t* rec, const Geom& G, int j,
                                          uint32_t (&vr)[4][4], uint64_t* empty_s) {
  constexpr int RB = Stg<BITS, WN, CP>::RB;
  const int lane = threadIdx.x & 31;
  const uint32_t vw = smem_u32(rec + FG<BITS, WN>::WB);
#pragma unroll
  for (int vc = 0; vc < 4; ++vc) {
    const int row = vc * 32 + lane;
    ldsm_x4(vw + row * RB + ((j ^ swz(row, WN)) << 4), vr[vc][0], vr[vc][1], vr[vc][2], vr[vc][3]);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_s);  // ring slot + prep slot are free
}

template <int BITS, int WN, int CP>
__device__ __forceinline__ void pv_stage(const uint32_t (&vr)[4][4],
                                         const uint32_t (&pb)[Stg<BITS, WN, CP>::NPK][2],
                                         const uint32_t (&pbh)[Stg<BITS, WN, CP>::NPH][2],
                                         float (&o)[OT][4]) {
  using T = Stg<BITS, WN, CP>;
  constexpr int P = T::P, NPAIR = T::NPAIR, NPK = T::NPK;
  constexpr int HALF = NPAIR / 2;
#pragma unroll
  for (int mt = 0; mt < KT; ++mt) {
    const uint32_t ra = vr[mt / 2][2 * (mt % 2)], rb = vr[mt / 2][2 * (mt % 2) + 1];
    const uint32_t ra8 = ra >> 8, rb8 = rb >> 8;
#pragma unroll
    for (int pi = 0; pi < NPAIR; ++pi) {
      uint32_t af[4];
#define BDK_VEXT(PI)                                 \
  if (pi == PI) {                                    \
    af[0] = ext_sub<BITS, (2 * PI) % P>(ra, ra8);     \
    af[1] = ext_sub<BITS, (2 * PI) % P>(rb, rb8);     \
    af[2] = ext_sub<BITS, (2 * PI + 1) % P>(ra, ra8); \
    af[3] = ext_sub<BITS, (2 * PI + 1) % P>(rb, rb8); \
  }
      BDK_VEXT(0)
      BDK_VEXT(1)
      BDK_VEXT(2)
      BDK_VEXT(3)
#undef BDK_VEXT
      if (CP == 2 && pi >= HALF)
        mma16816(o[mt], af, pbh[CP == 2 ? pi - HALF : 0][0], pbh[CP == 2 ? pi - HALF : 0][1]);
      else
        mma16816(o[mt], af, pb[pi % NPK][0], pb[pi % NPK][1]);
    }
  }
}

// The four stages back to back (the unpipelined consumer).
template <int BITS, int WN, int CP>
__device__ __forceinline__ void consume_block(const uint8_t* rec, const uint8_t* qp, const Geom& G,
                                              int j, float scale,
                                              const int (&vtok)[Stg<BITS, WN, CP>::NPK][2],
                                              Soft& st, float (&o)[OT][4], uint64_t* empty_s) {
  using T = Stg<BITS, WN, CP>;
  float sacc[T::NPK][4];
  uint32_t pb[T::NPK][2], pbh[T::NPH][2], vr[4][4];
  qk_stage<BITS, WN, CP>(rec, qp, j, scale, sacc);
  soft_stage<BITS, WN, CP>(rec, G, j, vtok, sacc, st, o, pb, pbh);
  ldv_stage<BITS, WN, CP>(rec, G, j, vr, empty_s);
  pv_stage<BITS, WN, CP>(vr, pb, pbh, o);
}

// Residual tokens [t_lo, t_hi) of `cell` (fp16 window, residual_attend,
// attention.cpp:92-105), split over the NC consumer warps in 16-token tiles;
// writes the appended token first if row rl0 falls in the range.
template <int NC, int CP>
__device__ __forceinline__ void consume_residual(const DevCache& c, const FastArgs& a, int cell,
                                                 int t_lo, int t_hi, int rl0, bool app,
                                                 float scale, Soft& st, float (&o)[OT][4]) {
  const Geom& G = c.G;
  const int ng = a.n_group;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
  constexpr int RT = 16 * NC;
  const int bidx = cell / G.heads_kv, hk = cell % G.heads_kv;
  __half* rk = c.res_k + (size_t)cell * G.n_r * D;
  __half* rv = c.res_v + (size_t)cell * G.n_r * D;
      if (app && rl0 >= t_lo && rl0 < t_hi) {  // append_token (kvcache.cpp:170-182)
    const __half* kn = a.k_new + (size_t)cell * D;
    const __half* vn = a.v_new + (size_t)cell * D;
    for (int i = threadIdx.x; i < D; i += NC * 32) {
      rk[(size_t)rl0 * D + i] = kn[i];
      rv[(size_t)rl0 * D + i] = vn[i];
    }
    named_bar(1, NC * 32);
  }
  uint32_t qb[KT][2];
  {
    const __half* qh = a.q + ((size_t)bidx * a.heads_q + (size_t)hk * ng + gid) * D;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      qb[kt][0] = gid < ng ? *reinterpret_cast<const uint32_t*>(qh + kt * 16 + 2 * t4) : 0u;
      qb[kt][1] = gid < ng ? *reinterpret_cast<const uint32_t*>(qh + kt * 16 + 8 + 2 * t4) : 0u;
    }
  }
  for (int t0 = t_lo + 16 * warp; t0 < t_hi; t0 += RT) {
    const bool v0 = t0 + gid < t_hi, v1 = t0 + gid + 8 < t_hi;
    const __half* k0 = rk + (size_t)(t0 + gid) * D + 2 * t4;
    const __half* k1 = k0 + 8 * D;
    float sacc[1][4] = {{0.f, 0.f, 0.f, 0.f}};
    uint32_t ka[KT][4];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      ka[kt][0] = v0 ? *reinterpret_cast<const uint32_t*>(k0 + kt * 16) : 0u;
      ka[kt][1] = v1 ? *reinterpret_cast<const uint32_t*>(k1 + kt * 16) : 0u;
      ka[kt][2] = v0 ? *reinterpret_cast<const uint32_t*>(k0 + kt * 16 + 8) : 0u;
      ka[kt][3] = v1 ? *reinterpret_cast<const uint32_t*>(k1 + kt * 16 + 8) : 0u;
    }
    // V rows in the natural [token][channel] fragment; movmatrix.trans
    // turns each 8x8 block into the V^T A-fragment (channel rows)
    const __half* w0 = rv + (size_t)(t0 + gid) * D + 2 * t4;
    const __half* w1 = w0 + 8 * D;
    uint32_t va[KT][4];
#pragma unroll
    for (int mt = 0; mt < KT; ++mt) {
      va[mt][0] = v0 ? *reinterpret_cast<const uint32_t*>(w0 + mt * 16) : 0u;
      va[mt][1] = v0 ? *reinterpret_cast<const uint32_t*>(w0 + mt * 16 + 8) : 0u;
      va[mt][2] = v1 ? *reinterpret_cast<const uint32_t*>(w1 + mt * 16) : 0u;
      va[mt][3] = v1 ? *reinterpret_cast<const uint32_t*>(w1 + mt * 16 + 8) : 0u;
    }
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) mma16816(sacc[0], ka[kt], qb[kt][0], qb[kt][1]);
    // CP = 2: columns 4..7 are the partner stream, which the residual
    // tokens do not feed
    const bool live = CP == 1 || t4 < 2;
    sacc[0][0] = v0 && live ? sacc[0][0] * scale : -INFINITY;
    sacc[0][1] = v0 && live ? sacc[0][1] * scale : -INFINITY;
    sacc[0][2] = v1 && live ? sacc[0][2] * scale : -INFINITY;
    sacc[0][3] = v1 && live ? sacc[0][3] * scale : -INFINITY;
    softmax_update<1>(sacc, st, o);
    const uint32_t pb0 = movmatrix_t(pack_h2(sacc[0][0], sacc[0][1]));
    const uint32_t pb1 = movmatrix_t(pack_h2(sacc[0][2], sacc[0][3]));
#pragma unroll
    for (int mt = 0; mt < KT; ++mt) {
      uint32_t af[4];
      af[0] = movmatrix_t(va[mt][0]);
      af[1] = movmatrix_t(va[mt][1]);
      af[2] = movmatrix_t(va[mt][2]);
      af[3] = movmatrix_t(va[mt][3]);
      mma16816(o[mt], af, pb0, pb1);
    }
  }
}

// NHT: the prep warp's head layout (n_group rounded up to a power of two)
// fixed at compile time (only that prep loop in the kernel body: measured
// +1.4% C5, +0.8% C2 from the smaller body), or 0 = chosen at run time
template <int BITS, int WN, int NS, int MINB, int GRP, int CP, int SWP, int NHT = 0>
__global__ void __maxnreg__(GRP >= 3 ? 128 : (MINB >= 3 ? 112 : 168))
    decode_fast_kernel(const __grid_constant__ DevCache c, const __grid_constant__ FastArgs a) {
  using C = FC<BITS, WN, MINB, GRP>;
  constexpr int P = C::P, NPAIR = C::NPAIR, NC = C::NC;
  static_assert(CP == 1 || (CP == 2 && NPAIR % 2 == 0), "column packing pairs tiles");
  constexpr int NPK = NPAIR / CP;  // packed S^T accumulators per chunk
  static_assert(NS % GRP == 0, "stage s must always belong to consumer group s % GRP");
  // subnormal mode: the V operand P s is pre-scaled by 2^(SH_REF - sh) so the
  // accumulator holds O * 2^(SH_REF - 24) for every field shift sh
  constexpr int SH_REF = BITS == 8 ? 0 : 2;
  const float oscale = exp2f((float)(24 - SH_REF));
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& G = c.G;
  const int cells = G.batch * G.heads_kv;
  const int ng = a.n_group;
  const Smem L = smem_layout(G, ng, NS, GRP);
  uint8_t* ring = smem + L.ring;
  uint8_t* prep = smem + L.prep;
  float* merge_sm = reinterpret_cast<float*>(smem + L.merge);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.total - 3 * NS * 8 - 48);
  uint64_t* empty = full + NS;
  uint64_t* ready = empty + NS;
  int* flag = reinterpret_cast<int*>(ready + NS);
  int* claim = flag + 2;  // [WN] next block per chunk position (GRP > 1)
  long long* sched_sm =
      reinterpret_cast<long long*>(smem + L.total - 3 * NS * 8 - 48 - 128);  // [16]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t4 = lane & 3;
  constexpr int REC = FG<BITS, WN>::REC;  // == G.rec_bytes (checked at launch)

  // zero the prep areas once: Q' rows of heads >= n_group stay zero
  for (uint32_t i = threadIdx.x * 16; i < NS * L.prep_stride; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(prep + i) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WN);  // the WN warps of the group that owns stage s
      mbar_init(&ready[s], 1);
    }
    for (int i = 0; i < WN; ++i) claim[i] = 0;
    fence_mbar_init();
  }
  __syncthreads();

  // PDL: the next kernel may launch its CTAs as soon as every CTA of this one
  // is resident (the grid is one wave, so this cannot starve it)
  pdl_launch_dependents();
  // ---- the step's schedule
  const Sched S = make_sched(c, a, cells, 16 * NC);
  SchedOut so;
  if (a.dev_sched) {
    // the lengths may still be being committed by the previous step
    if (a.pdl) pdl_wait();
    so = sched_scan(S, cells, sched_sm);
  } else {
    so = sched_host(S, a, cells);
  }
  const long long T = so.T;
  const int N = (int)min((long long)gridDim.x, T);  // CTAs sharing the units
  const long long u_begin = (int)blockIdx.x < N ? (long long)blockIdx.x * T / N : T;
  const long long u_end = (int)blockIdx.x < N ? (long long)(blockIdx.x + 1) * T / N : T;
  const int cell0 = so.cell0;
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 16 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();

  // ------------------------------------------------------------ TMA warp
  if (warp == NC) {
    if (lane == 0 && u_begin < u_end) {
      const uint64_t pol = policy_evict_first();
      // the first NS records may stream in before the previous kernel ends
      // when no packed record changed since (host schedule only: the records
      // are immutable and the schedule is in the arguments)
      bool waited = !a.pdl || a.dev_sched;
      if (!a.prefetch_ok && !waited) {
        pdl_wait();
        waited = true;
      }
      int it = 0;
      long long u = u_begin, off = so.off0;
      for (int cell = cell0; u < u_end; ++cell) {
        const int nbc = S.nb(cell);
        const long long ce = off + S.units(cell, nbc);
        const long long seg_end = min(u_end, ce);
        const long long pk_end = min(seg_end, off + nbc);
        const uint8_t* base = c.records + (size_t)cell * G.max_blocks * REC;
        for (long long x = u; x < pk_end; ++x, ++it) {
          const int s = it % NS;
          if (!waited && it == NS) {
            pdl_wait();
            waited = true;
          }
          if (it >= NS) {
            const unsigned long long tw = tr ? globaltimer() : 0ull;
            mbar_wait_sleep(&empty[s], ((it / NS) - 1) & 1);
            if (tr) tr[11] += globaltimer() - tw;
          }
          mbar_expect_tx(&full[s], (uint32_t)REC);
          const int blk = a.blk_begin + (int)(x - off);
          tma_bulk_g2s(ring + (size_t)s * REC, base + (size_t)blk * REC, (uint32_t)REC, &full[s],
                       pol);
        }
        u = seg_end;
        off = ce;
      }
    }
    return;
  }
  // q, lengths, counters and slots: after the previous kernel
  if (a.pdl && !a.dev_sched) pdl_wait();
  // the previous step's completion counters (its combine grid has finished)
  // start the next step at zero
  if (a.done != nullptr && warp < NC)
    for (int i = blockIdx.x * (NC * 32) + threadIdx.x; i < cells; i += gridDim.x * (NC * 32))
      a.done[(size_t)(a.par ^ 1) * cells + i] = 0;

  // ---------------------------------------------------------- prep warps
  if (warp > NC) {
    if (u_begin >= u_end) return;
    const int pgrp = warp - NC - 1;  // prepares the blocks of consumer group pgrp
    const int nh = ng <= 1 ? 1 : ng <= 2 ? 2 : ng <= 4 ? 4 : 8;
    PrepCtx px{ring, prep, full, ready, tr, REC, (int)L.prep_stride, pgrp, u_begin, u_end,
               so.off0, cell0, 16 * NC};
    // K groups per block: N_r / 128 (fast_decode_ok: g = 128, N_r % g = 0)
    constexpr int GPB = (WN * (16 / BITS)) / 16 > 0 ? (WN * (16 / BITS)) / 16 : 1;
    if constexpr (NHT > 0) {
      (void)nh;
      prep_loop<NHT, NS, GRP, GPB>(c, a, px);
    } else {
      if (nh == 1) prep_loop<1, NS, GRP, GPB>(c, a, px);
      else if (nh == 2) prep_loop<2, NS, GRP, GPB>(c, a, px);
      else if (nh == 4) prep_loop<4, NS, GRP, GPB>(c, a, px);
      else prep_loop<8, NS, GRP, GPB>(c, a, px);
    }
    return;
  }

  // ------------------------------------------------------ consumer warps
  const int j = warp % WN;    // 16-byte chunk of every channel row
  const int tok_base = 8 * j * P;
  const int kgr = G.k_axis == 0 ? tok_base / G.g : 0;
  const float scale = a.sm_scale_log2;
  int tok_lab[2 * NPAIR];  // token offset of field position e (labels (g, e))
#pragma unroll
  for (int e = 0; e < 2 * NPAIR; ++e) tok_lab[e] = pos_token(e, P, G.interleave);
  // per lane: token offsets of the rows of its tile in packed accumulator i
  // (lanes t4 >= 2 hold the partner tile i + NPAIR/2 when CP = 2)
  int vtok[NPK][2];
#pragma unroll
  for (int i = 0; i < NPK; ++i) {
    const bool partner = CP == 2 && t4 >= 2;
    vtok[i][0] = partner ? tok_lab[2 * (i + NPAIR / 2)] : tok_lab[2 * i];
    vtok[i][1] = partner ? tok_lab[2 * (i + NPAIR / 2) + 1] : tok_lab[2 * i + 1];
  }
  const int stride_slot = slot_stride(ng);

  int it = 0;
  long long u = u_begin, off = so.off0;
  for (int cell = cell0; u < u_end; ++cell) {
    const int nbc = S.nb(cell);
    const long long cb = off, ce = off + S.units(cell, nbc);
    const long long seg_end = min(u_end, ce);
    const long long res_begin = cb + nbc;  // 1st residual unit
    const long long pk_end = min(seg_end, res_begin);
    Soft st{-INFINITY, -INFINITY, 0.f, 0.f, 0.f, 0.f};
    float o[OT][4];  // O^T (subnormal-mode scaled, see oscale)
#pragma unroll
    for (int mt = 0; mt < OT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;

    // ---------------- packed blocks: CTA blocks [it, it_end) of this cell.
    // GRP > 1: the warps at chunk position j (one per group) claim blocks
    // dynamically from a shared-memory counter, so the groups stay busy to
    // the end of the cell whatever the warp scheduler favours
    const int it_end = it + (int)max(0LL, pk_end - u);
    if constexpr (SWP) {
      // software-pipelined consumer (GRP == 1): block k's QK^T is issued in
      // the same basic block as block k-1's PV (independent HMMA chains and
      // extraction for the scheduler to interleave); block k-1's V words are
      // already in registers and its stage released.  The O updates keep the
      // unpipelined order (PV(k-1) before softmax(k)'s rescale): bit-identical.
      static_assert(GRP == 1, "the pipelined consumer walks its blocks in order");
      using TS = Stg<BITS, WN, CP>;
      if (a.dev_flags & 1) {  // dev probe: stream only (no compute)
        for (int k = it; k < it_end; ++k) {
          const int s = k % NS;
          mbar_wait(&ready[s], (k / NS) & 1);
          mbar_wait(&full[s], (k / NS) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
      } else if (it < it_end) {
        float sacc[TS::NPK][4];
        uint32_t pb[TS::NPK][2], pbh[TS::NPH][2], vr[4][4];
        {
          const int s = it % NS;
          mbar_wait(&ready[s], (it / NS) & 1);
          mbar_wait(&full[s], (it / NS) & 1);
          if (tr && threadIdx.x == 0 && it == 0) tr[1] = globaltimer();
          const uint8_t* rec = ring + (size_t)s * REC;
          qk_stage<BITS, WN, CP>(rec, prep + (size_t)s * FG<BITS, WN>::PREP_STRIDE + kgr * QP_BYTES, j, scale,
                                 sacc);
          soft_stage<BITS, WN, CP>(rec, G, j, vtok, sacc, st, o, pb, pbh);
          ldv_stage<BITS, WN, CP>(rec, G, j, vr, &empty[s]);
        }
        for (int k = it + 1; k < it_end; ++k) {
          const int s = k % NS;
          unsigned long long tw = 0;
          if (tr && threadIdx.x == 0) tw = globaltimer();
          mbar_wait(&ready[s], (k / NS) & 1);
          mbar_wait(&full[s], (k / NS) & 1);
          if (tr && threadIdx.x == 0) tr[9] += globaltimer() - tw;
          const uint8_t* rec = ring + (size_t)s * REC;
          qk_stage<BITS, WN, CP>(rec, prep + (size_t)s * FG<BITS, WN>::PREP_STRIDE + kgr * QP_BYTES, j, scale,
                                 sacc);
          pv_stage<BITS, WN, CP>(vr, pb, pbh, o);
          soft_stage<BITS, WN, CP>(rec, G, j, vtok, sacc, st, o, pb, pbh);
          ldv_stage<BITS, WN, CP>(rec, G, j, vr, &empty[s]);
        }
        pv_stage<BITS, WN, CP>(vr, pb, pbh, o);
      }
    }
    int kn = SWP ? it_end : (GRP > 1 ? claim_next(claim + j, lane) : it);
    for (int k = kn; k < it_end; k = kn) {
      kn = GRP > 1 ? claim_next(claim + j, lane) : k + 1;  // next claim, in flight
      const int s = k % NS;
      unsigned long long tw = 0;
      if (tr && threadIdx.x == 0) tw = globaltimer();
      mbar_wait(&ready[s], (k / NS) & 1);
      mbar_wait(&full[s], (k / NS) & 1);
      if (tr && threadIdx.x == 0) {
        const unsigned long long now = globaltimer();
        if (k == 0) tr[1] = now; else tr[9] += now - tw;
      }
      if (a.dev_flags & 1) {  // dev probe: stream only (no compute)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }
      consume_block<BITS, WN, CP>(ring + (size_t)s * REC,
                                  prep + (size_t)s * FG<BITS, WN>::PREP_STRIDE + kgr * QP_BYTES, G, j, scale,
                                  vtok, st, o, &empty[s]);
    }

    it = it_end;
    if (tr && threadIdx.x == 0) tr[2] = globaltimer();
    // ---------------- residual window (fp16), append fused.  Residual unit r
    // of a cell covers tokens [r*RT, (r+1)*RT) (RT = 16 per consumer warp);
    // the CTA whose range holds row res_len writes the new token there.
    // the cell's lengths: from the arguments when the host schedule found
    // them uniform, else from the current half
    const int rl0 = a.uni_len ? a.uni_rl : __ldcg(S.rl() + cell);
    const bool app = a.k_new != nullptr && !a.skip_residual;
    float oscale_seg = oscale;
    if (seg_end > res_begin && !a.skip_residual) {
      // the packed-block O is held at scale 2^(SH_REF - 24) (subnormal-mode
      // V codes); the residual V is plain fp16: bring O to unit scale first
#pragma unroll
      for (int mt = 0; mt < KT; ++mt) {
        o[mt][0] *= oscale;
        o[mt][1] *= oscale;
        o[mt][2] *= oscale;
        o[mt][3] *= oscale;
      }
      oscale_seg = 1.f;
      constexpr int RT = 16 * NC;
      const int rlen = rl0 + (app ? 1 : 0);
      const int t_lo = (int)(max(u, res_begin) - res_begin) * RT;
      const int t_hi = min(rlen, (int)(seg_end - res_begin) * RT);
      consume_residual<NC, CP>(c, a, cell, t_lo, t_hi, rl0, app, scale, st, o);
    }

    // ---------------- segment partial -> slot (CTA + cell), completion count
    if (tr && threadIdx.x == 0) tr[3] = globaltimer();
    float* slot = a.slots + (size_t)(blockIdx.x + cell) * stride_slot;
    finalize_segment<NC, CP>(st, o, merge_sm, ng, slot, oscale_seg);  // ends with a barrier
    // the segment's partial is complete: count it for the combine grid (the
    // barrier orders every consumer thread's slot writes before this release)
    if (a.done != nullptr && threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.done + (size_t)a.par * cells + cell)
                   : "memory");
    if (tr && threadIdx.x == 0) tr[4] = globaltimer();
    if (tr && threadIdx.x == 0) {
      tr[5] = globaltimer();
      tr[6] = 0;
      tr[7] = (unsigned long long)(u_end - u_begin);
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[8] = smid;
    }
    // every consumer warp has left its claim loop: restart the claims at the
    // next cell's first block
    if (GRP > 1 && threadIdx.x < WN) claim[threadIdx.x] = it;
    named_bar(1, NC * 32);  // merge smem reuse by the next segment
    u = seg_end;
    off = ce;
  }
}

// ---------------------------------------------------------------------------
// combine (attention.cpp:142-162) + the step's commit (kvcache.cpp:170-251).
// A separate small grid chained to the attention grid by programmatic
// dependent launch: CTA (cell, h) LSE-merges the cell's partial slots for
// query head h of the group (thread = channel; every (max, sum) pair and O
// value of a batch of contributors in flight at once), so the merge runs on
// cells x n_group CTAs in parallel instead of on the tail of the CTA that
// finished a cell last.  CTA (cell, 0) then commits the cell's next lengths
// into the other half of len2 and, when the step filled the residual window,
// quantizes + packs it into the cell's next block slot (the fused flush).
constexpr int CMB_LB = 40;  // contributors per load batch (one round for C1-C5: <= 38)

template <int BITS, int WN>
__global__ void __launch_bounds__(D) combine_fast_kernel(const __grid_constant__ DevCache c,
                                                         const __grid_constant__ FastArgs a) {
  __shared__ __align__(16) uint8_t sm[4096];
  pdl_launch_dependents();  // the next step's prologue and prefetch may start
  const Geom& G = c.G;
  const int cells = G.batch * G.heads_kv;
  const int cell = blockIdx.x, h = blockIdx.y, ch = threadIdx.x;
  const int ng = a.n_group;
  const Sched S = make_sched(c, a, cells, a.rt);
  // host schedule: everything but the partials comes from the arguments (or
  // the schedule upload that precedes the attention grid), so it is worked
  // out before griddepcontrol.wait; the device schedule reads the lengths
  // after it
  if (a.pdl && a.dev_sched) pdl_wait();
  // the cell's unit range [cb, ce) and total T: host schedule from the
  // arguments, device schedule by a block reduction over the lengths
  long long cb, ce, T;
  if (!a.dev_sched) {
    T = a.total_units;
    if (a.uni_units) {
      cb = (long long)cell * a.uni_units;
      ce = cb + a.uni_units;
    } else {
      cb = __ldg(a.unit_off + cell);
      ce = __ldg(a.unit_off + cell + 1);
    }
  } else {
    long long* red = reinterpret_cast<long long*>(sm);
    long long before = 0, all = 0, mine = 0;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) {
      const long long u = S.units(i, S.nb(i));
      all += u;
      if (i < cell) before += u;
      if (i == cell) mine = u;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
      mine += __shfl_xor_sync(0xffffffffu, mine, o);
    }
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      red[warp] = before;
      red[8 + warp] = all;
      red[16 + warp] = mine;
    }
    __syncthreads();
    before = all = mine = 0;
    for (int w = 0; w < nw; ++w) {
      before += red[w];
      all += red[8 + w];
      mine += red[16 + w];
    }
    __syncthreads();
    cb = before;
    ce = before + mine;
    T = all;
  }
  const int N = (int)min((long long)a.n_ctas, T);
  const int lo = cta_of_unit(cb, T, N), hi = cta_of_unit(ce - 1, T, N);
  const int nk = hi - lo + 1;
  const int stride = slot_stride(ng);
  const float* base = a.slots + (size_t)(lo + cell) * stride;
  // the step's commit of this cell (lengths from the arguments when uniform)
  const bool app = a.k_new != nullptr && !a.skip_residual;
  int rl0 = a.uni_rl, pb0 = a.uni_pb;
  if (a.spin && a.done != nullptr && !a.dev_sched) {
    // host schedule: start as soon as this cell's nk partials are written
    // (the attention grid's CTAs count them), not when its last CTA exits
    if (threadIdx.x == 0) {
      const int* cnt = a.done + (size_t)a.par * cells + cell;
      while (ld_acquire_gpu_i(cnt) < nk) __nanosleep(64);
    }
    __syncthreads();
  } else if (a.pdl && !a.dev_sched) {
    pdl_wait();  // the attention grid's partials
  }
  if (a.dev_flags & 8) return;  // dev probe: the combine grid's cost in the step
  if (!a.uni_len) {
    rl0 = __ldcg(S.rl() + cell);
    pb0 = __ldcg(S.pb() + cell);
  }
  const bool fill = app && rl0 + 1 == G.n_r;
  // online LSE merge over the contributors, CMB_LB loads of each kind in flight
  float M = -INFINITY, L = 0.f, acc = 0.f;
  for (int k0 = 0; k0 < nk; k0 += CMB_LB) {
    float mk[CMB_LB], lk[CMB_LB], ok[CMB_LB];
#pragma unroll
    for (int i = 0; i < CMB_LB; ++i) {
      const int k = k0 + i;
      if (k < nk) {
        const float* sl = base + (size_t)k * stride;
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(sl + ng * D + 2 * h));
        mk[i] = ml.x;
        lk[i] = ml.y;
        ok[i] = __ldcg(sl + h * D + ch);
      } else {
        mk[i] = -INFINITY;
        lk[i] = 0.f;
        ok[i] = 0.f;
      }
    }
    float mx = M;
#pragma unroll
    for (int i = 0; i < CMB_LB; ++i) mx = fmaxf(mx, mk[i]);
    const float r = M == -INFINITY ? 0.f : ex2(M - mx);
    acc *= r;
    L *= r;
#pragma unroll
    for (int i = 0; i < CMB_LB; ++i) {
      const float w = mk[i] == -INFINITY ? 0.f : ex2(mk[i] - mx);
      acc = fmaf(ok[i], w, acc);
      L = fmaf(lk[i], w, L);
    }
    M = mx;
  }
  const int bidx = cell / G.heads_kv, hk = cell % G.heads_kv;
  const size_t row = (size_t)bidx * a.heads_q + (size_t)hk * ng + h;
  a.out[row * D + ch] = L > 0.f ? acc / L : 0.f;
  if (a.out_lse != nullptr && ch == 0) a.out_lse[row] = L > 0.f ? M + __log2f(L) : -INFINITY;
  if (h != 0 && !fill) return;
  // ---- the commit (every contributor has read the window)
  if (fill) {
    // build_block + commit_block (kvcache.cpp:208-237) after the step's
    // attention (attention.cpp:235-240); the cell's n_group CTAs split the
    // window's K and V tiles
    constexpr int P = 16 / BITS;
    const size_t wo = (size_t)cell * G.n_r * D;
    uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + pb0) * G.rec_bytes;
    if constexpr (BITS != 8 && (WN * P) % 16 == 0) {
      qf_flush_window<BITS, D>(G, c.res_k + wo, c.res_v + wo, rec, sm, 1, h, ng);
    } else if (h == 0) {
      flush_window<BITS>(G, c.res_k + wo, c.res_v + wo, rec, D, 1);
    }
  }
  if (h != 0) return;
  if (threadIdx.x == 0) {
    S.pb_n()[cell] = fill ? pb0 + 1 : pb0;
    S.rl_n()[cell] = fill ? 0 : rl0 + (app ? 1 : 0);
  }
}

}  // namespace

bool fast_decode_ok(const Geom& G, int n_group) {
  if (G.d != D || n_group < 1 || n_group > 8) return false;
  if (!(G.bits == 2 || G.bits == 4 || G.bits == 8)) return false;
  if (!(G.warp_n == 1 || G.warp_n == 2 || G.warp_n == 4 || G.warp_n == 8)) return false;
  if (G.k_axis != 0) return false;
  if (G.g != D) return false;  // V: one (scale, zero) per token
  if (G.n_r % G.g != 0) return false;       // KChannel groups tile the block
  if (G.g % (8 * G.pack) != 0) return false;  // a warp's chunk lies in one K group
  return true;
}

// Variant table: (bits, warp_n) -> kernel with its ring depth and the CTAs
// per SM it is built for.  BDK_FAST_VARIANT (env, dev knob) picks an
// alternative ring/occupancy point for the W_n = 4 kernels.
struct Variant {
  const void* fn;
  int ns, grp;
  const void* combine;  // combine_fast_kernel of the same geometry
};

// software-pipelined consumer loop (GRP == 1 kernels); dev knob BDK_SWP=0|1|2
static int swp_knob() {
  static int v = [] {
    const char* e = getenv("BDK_SWP");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// the pipelined W_n = 4 kernels (the BASELINE geometry) with the prep
// layout fixed for n_group's power of two
template <int BITS, int NS, int MINB, int CP>
static const void* swp_nh_kernel(int ng) {
  const int nh = ng <= 1 ? 1 : ng <= 2 ? 2 : ng <= 4 ? 4 : 8;
  if (nh == 1) return reinterpret_cast<const void*>(decode_fast_kernel<BITS, 4, NS, MINB, 1, CP, 1, 1>);
  if (nh == 2) return reinterpret_cast<const void*>(decode_fast_kernel<BITS, 4, NS, MINB, 1, CP, 1, 2>);
  if constexpr (CP == 2) {  // column packing needs n_group <= 4
    return reinterpret_cast<const void*>(decode_fast_kernel<BITS, 4, NS, MINB, 1, CP, 1, 4>);
  } else {
    if (nh == 4)
      return reinterpret_cast<const void*>(decode_fast_kernel<BITS, 4, NS, MINB, 1, CP, 1, 4>);
    return reinterpret_cast<const void*>(decode_fast_kernel<BITS, 4, NS, MINB, 1, CP, 1, 8>);
  }
}

template <int BITS, int WN, int NS, int MINB, int GRP>
static Variant variant(int cp, bool swp, int ng) {
  const void* comb = reinterpret_cast<const void*>(combine_fast_kernel<BITS, WN>);
  if constexpr (WN == 4 && GRP == 1) {
    if (swp) {
      if constexpr (BITS != 8)
        if (cp == 2) return Variant{swp_nh_kernel<BITS, NS, MINB, 2>(ng), NS, GRP, comb};
      return Variant{swp_nh_kernel<BITS, NS, MINB, 1>(ng), NS, GRP, comb};
    }
  }
  if constexpr (BITS != 8) {
    if (cp == 2) {
      if constexpr (GRP == 1 && WN != 4)
        if (swp)
          return Variant{
              reinterpret_cast<const void*>(decode_fast_kernel<BITS, WN, NS, MINB, GRP, 2, 1>), NS,
              GRP, comb};
      return Variant{reinterpret_cast<const void*>(decode_fast_kernel<BITS, WN, NS, MINB, GRP, 2, 0>),
                     NS, GRP, comb};
    }
  }
  if constexpr (GRP == 1 && WN != 4)
    if (swp)
      return Variant{reinterpret_cast<const void*>(decode_fast_kernel<BITS, WN, NS, MINB, GRP, 1, 1>),
                     NS, GRP, comb};
  return Variant{reinterpret_cast<const void*>(decode_fast_kernel<BITS, WN, NS, MINB, GRP, 1, 0>), NS,
                 GRP, comb};
}

static int variant_knob() {
  static int v = [] {
    const char* e = getenv("BDK_FAST_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// default: two co-resident CTAs per SM, one consumer group each, 4-stage ring
// (measured best on B200).  Dev knob BDK_FAST_VARIANT: 2 = one CTA per SM with
// two consumer groups claiming chunks from a shared 8-stage ring, 3 = three
// groups at 128 registers (both measured 6-15% slower).
// swp: the software-pipelined consumer loop (measured: C5 +3.8%, C2 +-0.3%;
// C1, under one block per CTA, -3%: chosen when CTAs average >= 2 blocks)
static Variant fast_kernel(const Geom& G, int ng, bool swp = true) {
  const int v = variant_knob();
  swp = swp && swp_knob() != 0;
  // dev knob BDK_COLPACK: 0 = never, 2 = wherever the layout allows (4-bit too)
  static const int cp_knob = getenv("BDK_COLPACK") ? atoi(getenv("BDK_COLPACK")) : -1;
  const int cp = cp_knob == 0 ? 1
                 : cp_knob == 2 ? ((ng <= 4 && (G.bits == 2 || G.bits == 4)) ? 2 : 1)
                                : col_pack(G, ng);
#define BDK_SEL(B, W, NS, MB, GR) \
  if (G.bits == B && G.warp_n == W) return variant<B, W, NS, MB, GR>(cp, swp, ng);
  if (v == 2) {
    BDK_SEL(2, 4, 8, 1, 2) BDK_SEL(4, 4, 8, 1, 2)
  } else if (v == 3) {
    BDK_SEL(2, 4, 6, 1, 3) BDK_SEL(4, 4, 9, 1, 3)
  }
  BDK_SEL(2, 1, 4, 2, 1) BDK_SEL(2, 2, 4, 2, 1) BDK_SEL(2, 4, 4, 2, 1) BDK_SEL(2, 8, 4, 1, 1)
  BDK_SEL(4, 1, 4, 2, 1) BDK_SEL(4, 2, 4, 2, 1) BDK_SEL(4, 4, 4, 2, 1) BDK_SEL(4, 8, 4, 1, 1)
  BDK_SEL(8, 1, 4, 2, 1) BDK_SEL(8, 2, 4, 2, 1) BDK_SEL(8, 4, 4, 2, 1) BDK_SEL(8, 8, 4, 1, 1)
#undef BDK_SEL
  return Variant{nullptr, 0, 1, nullptr};
}

static int fast_threads(const Geom& G, const Variant& k) {
  return (G.warp_n * k.grp + 1 + k.grp) * 32;
}

static uint32_t fast_smem(const Geom& G, int ng, const Variant& k) {
  return smem_layout(G, ng, k.ns, k.grp).total;
}

int fast_residual_tokens(const Geom& G) { return 16 * G.warp_n * fast_kernel(G, 1).grp; }

int fast_decode_ctas_per_sm(const Geom& G, int n_group) {
  const Variant k = fast_kernel(G, n_group);
  if (!k.fn) return 0;
  const uint32_t smem = fast_smem(G, n_group, k);
  // both consumer-loop variants (launch_decode_fast picks one per step)
  for (const bool swp : {true, false})
    if (cudaFuncSetAttribute(fast_kernel(G, n_group, swp).fn,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k.fn, fast_threads(G, k), smem) !=
      cudaSuccess)
    return 0;
  return n;
}

cudaError_t launch_decode_fast(const DevCache& c, const FastArgs& a, cudaStream_t s) {
  // graph steps (device schedule) hold for any lengths: pipelined.  Dev knob
  // BDK_SWP: 0 never, 1 by this rule (default), 2 always
  const bool swp = a.dev_sched || a.total_units >= 2LL * a.n_ctas || swp_knob() == 2;
  const Variant k = fast_kernel(c.G, a.n_group, swp);
  if (!k.fn) return cudaErrorInvalidValue;
  // the kernels bake the record geometry in (FG); it must be the cache's
  {
    const Geom& G = c.G;
    const int P = 16 / G.bits, nr = 8 * G.warp_n * P, gpb = nr / 128 > 0 ? nr / 128 : 1;
    const int rec = (2 * 16 * G.warp_n * 128 + gpb * 512 + nr * 4 + 127) / 128 * 128;
    if (G.rec_bytes != rec || G.wbytes != 16 * G.warp_n * 128 || G.kp_bytes != gpb * 512 ||
        G.n_r != nr || G.g != 128 || G.k_axis != 0 ||
        (int)smem_layout(G, a.n_group, k.ns, k.grp).prep_stride !=
            (gpb * QP_BYTES + 127) / 128 * 128)
      return cudaErrorInvalidValue;
  }
  const uint32_t smem = fast_smem(c.G, a.n_group, k);
  DevCache cc = c;
  FastArgs aa = a;
  aa.rt = 16 * c.G.warp_n * k.grp;
  void* args[] = {&cc, &aa};
  if (a.ev_begin) cudaEventRecord(a.ev_begin, s);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.n_ctas);
  cfg.blockDim = dim3(fast_threads(c.G, k));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelExC(&cfg, k.fn, args);
  if (e != cudaSuccess) return e;
  // combine: one CTA per (cell, query head of the group), a programmatic
  // dependent of the attention grid (it waits for the partials itself)
  cudaLaunchConfig_t cfg2 = {};
  cfg2.gridDim = dim3(c.G.batch * c.G.heads_kv, a.n_group);
  cfg2.blockDim = dim3(D);
  cfg2.dynamicSmemBytes = 0;
  cfg2.stream = s;
  cfg2.attrs = attr;
  cfg2.numAttrs = 1;
  e = cudaLaunchKernelExC(&cfg2, k.combine, args);
  if (e != cudaSuccess) return e;
  if (a.ev_end) cudaEventRecord(a.ev_end, s);
  return cudaSuccess;
}

}  // namespace bdk
