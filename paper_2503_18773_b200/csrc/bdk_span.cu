// bdk_span.cu -- general span attention on sm_100a.
//
// The fast kernels (bdk_decode_fast.cu, bdk_kernels.cu) serve head_dim 128
// with n_group <= 8.  Everything else the reference accepts -- any head_dim,
// any n_group, the attention internals a caller can reach directly
// (attend_tile, partitioned_rowmax, residual_attend, packed_attend, combine;
// attention.cpp:32-162) -- runs here, still on the device.
//
// One CTA walks one contiguous token span in tiles with exactly the
// reference's online-softmax step per tile (attend_tile,
// attention.cpp:52-90).  Every dot product, row sum and P.V sum runs in the
// reference's order with unfused fp32 operations (__fmul_rn/__fadd_rn, no
// FMA contraction), so the one difference from the host is expf (CUDA,
// <= 2 ulp) against libm.  q, the score tile, the per-row rescale factors,
// the running P.V sums and a 32-token chunk of K or V rows (dequantized once
// from the packed block records) sit in shared memory; the partial state
// (o, m, l) stays in the parts buffer, each element owned by one thread
// across tiles.  This path is latency-bound by construction; the hot path's
// throughput lives in the fast kernels.
#include <cfloat>

#include "bdk_launch.h"

namespace bdk {

namespace {

constexpr int kSpanThreads = 256;

struct SpanCtx {
  const SpanArgs* a;
  int cell;
  int mode;    // 0 fp32 arrays, 1 packed segment, 2 residual window
  int stored;  // residual tokens already in the buffer (mode 2)
};

__device__ __forceinline__ float span_kv(const SpanCtx& x, int t, int ch, int which) {
  const SpanArgs& a = *x.a;
  const Geom& G = a.c.G;
  if (x.mode == 0) return (which ? a.v32 : a.k32)[(size_t)t * a.d + ch];
  if (x.mode == 2) {
    if (t < x.stored)
      return __half2float(
          (which ? a.c.res_v : a.c.res_k)[((size_t)x.cell * G.n_r + t) * G.d + ch]);
    return __half2float((which ? a.v_new : a.k_new)[(size_t)x.cell * G.d + ch]);
  }
  const uint8_t* rec = a.c.records + ((size_t)x.cell * G.max_blocks + t / G.n_r) * G.rec_bytes;
  return __half2float(packed_elem(G, rec, t % G.n_r, ch, which));
}

// K/V rows staged per chunk of the tile: dequantized once into shared memory
// (row stride d + 1, so the S loop's strided rows hit distinct banks)
constexpr int kSpanChunk = 32;

__device__ __forceinline__ void stage_rows(const SpanCtx& x, int t0, int m, int d, int which,
                                           float* kv) {
  for (int i = threadIdx.x; i < m * d; i += blockDim.x) {
    const int j = i / d, c = i % d;
    kv[j * (d + 1) + c] = span_kv(x, t0 + j, c, which);
  }
}

// K/V element j of the current chunk: the staged row, or (when the staged
// layout does not fit in shared memory) straight from the source
__device__ __forceinline__ float chunk_kv(const SpanCtx& x, const float* kv, int d, int t0, int j,
                                          int c, int which) {
  return kv ? kv[j * (d + 1) + c] : span_kv(x, t0 + j, c, which);
}

// online softmax over tokens [t_begin, t_end) in tiles of tile_n.  kv (the
// chunk stage) may be null and pacc may live in global memory: the large
// geometries the reference accepts (e.g. n_group 64, d 256, N_r 512) keep
// only q, the score tile and the rescale factors in shared memory.
__device__ void span_walk(const SpanCtx& x, const float* q, int rows, int d, float scale,
                          int tile_n, int t_begin, int t_end, float* o, float* m, float* l,
                          float* s, float* resc, float* pacc, float* kv) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int t0 = t_begin; t0 < t_end; t0 += tile_n) {
    const int n = min(tile_n, t_end - t0);
    // S = scale * q k^T, sequential over channels
    for (int c0 = 0; c0 < n; c0 += kSpanChunk) {
      const int mc = min(kSpanChunk, n - c0);
      if (kv) stage_rows(x, t0 + c0, mc, d, 0, kv);
      __syncthreads();
      for (int i = tid; i < rows * mc; i += nt) {
        const int r = i / mc, j = i % mc;
        float acc = 0.f;
        for (int c = 0; c < d; ++c)
          acc = __fadd_rn(acc, __fmul_rn(q[r * d + c], chunk_kv(x, kv, d, t0 + c0, j, c, 0)));
        s[r * n + c0 + j] = __fmul_rn(acc, scale);
      }
      __syncthreads();
    }
    // row max (a partitioned max is the same number), rescale, P, row sum
    for (int r = tid; r < rows; r += nt) {
      float tm = -INFINITY;
      for (int j = 0; j < n; ++j) tm = fmaxf(tm, s[r * n + j]);
      const float m_old = m[r];
      const float m_new = fmaxf(m_old, tm);
      const float rs = m_old == -INFINITY ? 0.f : expf(__fadd_rn(m_old, -m_new));
      float sum = 0.f;
      for (int j = 0; j < n; ++j) {
        const float p = expf(__fadd_rn(s[r * n + j], -m_new));
        s[r * n + j] = p;
        sum = __fadd_rn(sum, p);
      }
      l[r] = __fadd_rn(__fmul_rn(l[r], rs), sum);
      m[r] = m_new;
      resc[r] = rs;
    }
    for (int i = tid; i < rows * d; i += nt) pacc[i] = 0.f;
    // O' = P V + rescale * O, sequential over the tile's tokens (the running
    // sum carries across chunks, so the order is the reference's; element i
    // of pacc is owned by one thread throughout)
    for (int c0 = 0; c0 < n; c0 += kSpanChunk) {
      const int mc = min(kSpanChunk, n - c0);
      __syncthreads();
      if (kv) stage_rows(x, t0 + c0, mc, d, 1, kv);
      __syncthreads();
      for (int i = tid; i < rows * d; i += nt) {
        const int r = i / d, c = i % d;
        float acc = pacc[i];
        for (int j = 0; j < mc; ++j)
          acc = __fadd_rn(acc, __fmul_rn(s[r * n + c0 + j], chunk_kv(x, kv, d, t0 + c0, j, c, 1)));
        pacc[i] = acc;
      }
    }
    __syncthreads();
    for (int i = tid; i < rows * d; i += nt) o[i] = __fadd_rn(pacc[i], __fmul_rn(resc[i / d], o[i]));
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSpanThreads) span_parts_kernel(SpanArgs a) {
  extern __shared__ float sm[];
  const int rows = a.rows, d = a.d;
  const int cell = a.cell0 + blockIdx.y, part = blockIdx.x;
  const Geom& G = a.c.G;
  const int tile_max = a.source == kSpanFp32 ? a.len32 : max(a.tile_n, G.n_r);
  // shared layout: q | resc | s [rows * tile_max] | kv chunk (opt.) | pacc (opt.)
  float* q = sm;
  float* resc = q + rows * d;
  float* s = resc + rows;
  float* kv = a.kv_smem ? s + (size_t)rows * tile_max : nullptr;
  float* pacc = a.pacc_smem
                    ? s + (size_t)rows * tile_max + (a.kv_smem ? kSpanChunk * (d + 1) : 0)
                    : a.scratch + ((size_t)blockIdx.y * a.n_parts + part) * rows * d;
  float* st = a.parts + ((size_t)blockIdx.y * a.n_parts + part) * rows * (d + 2);
  float* o = st;
  float* m = st + rows * d;
  float* l = m + rows;

  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    if (a.q32 != nullptr) {
      q[i] = a.q32[i];
    } else {
      const int r = i / d, c = i % d;
      const int b = cell / G.heads_kv, hk = cell % G.heads_kv;
      const size_t row = (size_t)b * a.heads_q + (size_t)hk * rows + r;
      q[i] = __fmul_rn(__half2float(a.q16[row * d + c]), a.q_scale);
    }
    if (!a.keep_state) o[i] = 0.f;
  }
  if (!a.keep_state)
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      m[r] = -INFINITY;
      l[r] = 0.f;
    }

  SpanCtx x{&a, cell, 0, 0};
  int t_begin = 0, t_end = 0, tile = a.tile_n;
  if (a.source == kSpanFp32) {
    t_end = a.len32;
  } else if (part < a.residual) {
    // residual window (residual_attend, attention.cpp:92-105): one tile of
    // every stored token plus the token this step appends
    x.mode = 2;
    x.stored = a.c.res_len[cell];
    t_end = x.stored + (a.k_new != nullptr ? 1 : 0);
    tile = max(t_end, 1);
    if (a.k_new != nullptr)
      for (int c = threadIdx.x; c < G.d; c += blockDim.x) {
        const size_t dst = ((size_t)cell * G.n_r + x.stored) * G.d + c;
        a.c.res_k[dst] = a.k_new[(size_t)cell * G.d + c];
        a.c.res_v[dst] = a.v_new[(size_t)cell * G.d + c];
      }
  } else {
    // packed split (packed_attend, attention.cpp:107-140): tiles of tile_n
    // over the block range, base + (s < rem) tiles per split
    x.mode = 1;
    const int lo = a.blk_begin * G.n_r;
    const int hi = min(a.blk_end, a.c.packed_blocks[cell]) * G.n_r;
    const int len = max(0, hi - lo);
    const int n_tiles = (len + a.tile_n - 1) / a.tile_n;
    const int sp = part - a.residual, splits = max(1, a.splits);
    const int base = n_tiles / splits, rem = n_tiles % splits;
    const int first = sp * base + min(sp, rem), count = base + (sp < rem ? 1 : 0);
    t_begin = lo + first * a.tile_n;
    t_end = count ? min(lo + (first + count) * a.tile_n, hi) : t_begin;
  }
  __syncthreads();
  span_walk(x, q, rows, d, a.scale, tile, t_begin, t_end, o, m, l, s, resc, pacc, kv);
}

__global__ void __launch_bounds__(256)
    span_combine_kernel(const float* parts, int n_parts, int rows, int d, int heads_kv,
                        int heads_q, float* out, float* out_lse, int* res_len) {
  const int cell = blockIdx.x;
  const size_t stride = (size_t)rows * (d + 2);
  const float* P = parts + (size_t)cell * n_parts * stride;
  const int b = cell / heads_kv, hk = cell % heads_kv;
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    const int r = i / d;
    float ms = -INFINITY;
    for (int p = 0; p < n_parts; ++p) ms = fmaxf(ms, P[p * stride + rows * d + r]);
    float acc = 0.f, l = 0.f;
    for (int p = 0; p < n_parts; ++p) {
      const float mp = P[p * stride + rows * d + r];
      const float w = mp == -INFINITY ? 0.f : expf(__fadd_rn(mp, -ms));
      l = __fadd_rn(l, __fmul_rn(P[p * stride + rows * d + rows + r], w));
      acc = __fadd_rn(acc, __fmul_rn(P[p * stride + i], w));
    }
    const size_t row = (size_t)b * heads_q + (size_t)hk * rows + r;
    out[row * d + i % d] = __fdiv_rn(acc, l);
    if (out_lse != nullptr && i % d == 0)
      out_lse[row] = l > 0.f ? __fadd_rn(__fmul_rn(ms, kLog2e), log2f(l)) : -INFINITY;
  }
  if (res_len != nullptr && threadIdx.x == 0) res_len[cell] += 1;
}

__global__ void partitioned_rowmax_kernel(const float* s, int rows, int cols, int w, float* out) {
  const int slice = cols / w;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    float mr = -INFINITY;
    for (int p = 0; p < w; ++p) {
      float mp = -INFINITY;
      for (int j = 0; j < slice; ++j) mp = fmaxf(mp, s[(size_t)r * cols + p * slice + j]);
      mr = fmaxf(mr, mp);
    }
    out[r] = mr;
  }
}

}  // namespace

// the minimal layout (q, rescale factors, score tile): what a geometry needs
// to run at all
size_t span_smem_bytes(int rows, int d, int tile) {
  return (size_t)rows * (d + 1 + tile) * sizeof(float);
}

cudaError_t launch_span_parts(const SpanArgs& a_in, int n_cells, cudaStream_t s) {
  if (n_cells <= 0 || a_in.n_parts <= 0) return cudaSuccess;
  SpanArgs a = a_in;
  const int tile = a.source == kSpanFp32 ? a.len32 : max(a.tile_n, a.c.G.n_r);
  // stage the K/V chunk and the running P.V sums in shared memory when they
  // fit (227 KB per CTA); otherwise read K/V from the source and keep the
  // sums in a stream-ordered global scratch
  constexpr size_t kMax = 227u << 10;
  const size_t kv_b = (size_t)kSpanChunk * (a.d + 1) * sizeof(float);
  const size_t pacc_b = (size_t)a.rows * a.d * sizeof(float);
  size_t smem = span_smem_bytes(a.rows, a.d, tile);
  a.kv_smem = smem + kv_b <= kMax;
  if (a.kv_smem) smem += kv_b;
  a.pacc_smem = smem + pacc_b <= kMax;
  if (a.pacc_smem) smem += pacc_b;
  float* scratch = nullptr;
  cudaError_t e;
  if (!a.pacc_smem) {
    e = cudaMallocAsync(&scratch, (size_t)n_cells * a.n_parts * pacc_b, s);
    if (e != cudaSuccess) return e;
    a.scratch = scratch;
  }
  e = cudaFuncSetAttribute(span_parts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
  if (e == cudaSuccess) {
    span_parts_kernel<<<dim3(a.n_parts, n_cells), kSpanThreads, smem, s>>>(a);
    e = cudaGetLastError();
  }
  if (scratch) {
    const cudaError_t f = cudaFreeAsync(scratch, s);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

cudaError_t launch_span_combine(const float* parts, int n_cells, int n_parts, int rows, int d,
                                int heads_kv, int heads_q, float* out, float* out_lse,
                                int* res_len, cudaStream_t s) {
  if (n_cells <= 0) return cudaSuccess;
  const int nt = min(256, max(32, (rows * d + 31) / 32 * 32));
  span_combine_kernel<<<n_cells, nt, 0, s>>>(parts, n_parts, rows, d, heads_kv, heads_q, out,
                                             out_lse, res_len);
  return cudaGetLastError();
}

cudaError_t launch_partitioned_rowmax(const float* s, int rows, int cols, int warp_n, float* out,
                                      cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  partitioned_rowmax_kernel<<<(rows + 127) / 128, 128, 0, st>>>(s, rows, cols, warp_n, out);
  return cudaGetLastError();
}

}  // namespace bdk
