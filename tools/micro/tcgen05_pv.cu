// tcgen05_pv.cu -- micro-benchmark: the PV stage of the 2-bit decode consumer
// (O^T += codes_V^T . P'^T over one 256-token block of 128 channel rows) on
//   (A) mma.sync m16n8k16, the production path: each of 4 warps owns a 64-token
//       chunk of every row (ldmatrix, one LOP3 per half2, 32 HMMA into an
//       O^T[128 ch][8 heads] register accumulator);
//   (B) tcgen05.mma with A in TMEM: thread = channel row (a warp's TMEM lane
//       quarter = its 32 channels), the same LOP3 extraction into half2
//       registers, tcgen05.st of them into TMEM, one elected thread issues
//       kind::f16 MMAs (M = 128 channels, N = 16 heads, K = 16 tokens) with
//       B = P'^T from shared memory, accumulator O^T in TMEM; the A region is
//       double-buffered per 128-token half and released by tcgen05.commit.
// Same codes, same P, 2 CTAs of 4 warps per SM, 296 CTAs, the block data
// resident in shared memory (no HBM traffic): cycles per (CTA, block), and
// both results checked against a double-precision host reference.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_18773_b200/csrc \
//      tools/micro/tcgen05_pv.cu -o tools/micro/bin/tcgen05_pv
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include "bdk_common.cuh"

using namespace bdk;

constexpr int ROWS = 128;      // channels
constexpr int TOK = 256;       // tokens per 2-bit block (N_r at W_n 4)
constexpr int RB = 64;         // bytes per row (32 u16 words)
constexpr int NH = 16;         // MMA N (heads padded)
constexpr int NB = 512;        // blocks per CTA (timing loop)
constexpr int NCTA = 296;

// value of field f (0..7) of a 2-bit word as the production extraction makes
// it: fields 0..3 masked in place, 4..7 after >> 8: code << 2(f%4), as an fp16
// subnormal (x 2^-24)
static double field_val(uint16_t w, int f) {
  const int code = (w >> (2 * f)) & 3;
  return (double)(code << (2 * (f % 4))) * std::ldexp(1.0, -24);
}

template <int F>
__device__ __forceinline__ uint32_t ext2(uint32_t r, uint32_t r8) {
  constexpr uint32_t M = (3u * 0x00010001u) << (2 * (F % 4));
  return (F < 4 ? r : r8) & M;
}

// ---------------------------------------------------------------- (A) HMMA
// smem words: row c at c*RB, 16-byte chunk j at (j ^ (c & 3)) * 16 (a swizzle
// that makes 8 consecutive rows' ldmatrix reads conflict-free at RB = 64)
__global__ void __launch_bounds__(128) hmma_pv(const uint16_t* words, const uint32_t* pfrag,
                                               float* out, long long* cyc) {
  __shared__ __align__(128) uint8_t sw[ROWS * RB];
  for (int i = threadIdx.x; i < ROWS * RB / 16; i += 128) {
    const int c = i / (RB / 16), j = i % (RB / 16);
    reinterpret_cast<uint4*>(sw)[c * (RB / 16) + (j ^ (c & 3))] =
        reinterpret_cast<const uint4*>(words)[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
  // P'^T B-fragments of this warp's 64 tokens: 4 tiles of 16 tokens
  uint32_t pb[4][2];
  for (int i = 0; i < 4; ++i) {
    pb[i][0] = pfrag[((j * 4 + i) * 2 + 0) * 32 + lane];
    pb[i][1] = pfrag[((j * 4 + i) * 2 + 1) * 32 + lane];
  }
  float o[8][4] = {};
  const uint32_t base = smem_u32(sw);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < NB; ++it) {
    uint32_t vr[4][4];
#pragma unroll
    for (int vc = 0; vc < 4; ++vc) {
      const int row = vc * 32 + lane;
      ldsm_x4(base + row * RB + ((j ^ (row & 3)) << 4), vr[vc][0], vr[vc][1], vr[vc][2], vr[vc][3]);
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const uint32_t ra = vr[mt / 2][2 * (mt % 2)], rb = vr[mt / 2][2 * (mt % 2) + 1];
      const uint32_t ra8 = ra >> 8, rb8 = rb >> 8;
      uint32_t af[4];
#define PV_TILE(PI)                          \
  af[0] = ext2<2 * PI>(ra, ra8);             \
  af[1] = ext2<2 * PI>(rb, rb8);             \
  af[2] = ext2<2 * PI + 1>(ra, ra8);         \
  af[3] = ext2<2 * PI + 1>(rb, rb8);         \
  mma16816(o[mt], af, pb[PI][0], pb[PI][1]);
      PV_TILE(0)
      PV_TILE(1)
      PV_TILE(2)
      PV_TILE(3)
#undef PV_TILE
    }
  }
  const long long t1 = clock64();
  // O^T partial of this warp's tokens: [channel][head 0..7]
  const int gid = lane >> 2, t4 = lane & 3;
  float* ob = out + ((size_t)blockIdx.x * 4 + j) * ROWS * 8;
  for (int mt = 0; mt < 8; ++mt) {
    ob[(mt * 16 + gid) * 8 + 2 * t4] = o[mt][0];
    ob[(mt * 16 + gid) * 8 + 2 * t4 + 1] = o[mt][1];
    ob[(mt * 16 + gid + 8) * 8 + 2 * t4] = o[mt][2];
    ob[(mt * 16 + gid + 8) * 8 + 2 * t4 + 1] = o[mt][3];
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// -------------------------------------------------------------- (B) tcgen05
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE (bits 61-63)
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, N, M
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                       uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
      smem_u32(bar)));
}

#define ST32(OFF)                                                                               \
  asm volatile(                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"  \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"( \
          ta + (OFF)),                                                                          \
      "r"(h[OFF + 0]), "r"(h[OFF + 1]), "r"(h[OFF + 2]), "r"(h[OFF + 3]), "r"(h[OFF + 4]),      \
      "r"(h[OFF + 5]), "r"(h[OFF + 6]), "r"(h[OFF + 7]), "r"(h[OFF + 8]), "r"(h[OFF + 9]),      \
      "r"(h[OFF + 10]), "r"(h[OFF + 11]), "r"(h[OFF + 12]), "r"(h[OFF + 13]), "r"(h[OFF + 14]), \
      "r"(h[OFF + 15]), "r"(h[OFF + 16]), "r"(h[OFF + 17]), "r"(h[OFF + 18]), "r"(h[OFF + 19]), \
      "r"(h[OFF + 20]), "r"(h[OFF + 21]), "r"(h[OFF + 22]), "r"(h[OFF + 23]), "r"(h[OFF + 24]), \
      "r"(h[OFF + 25]), "r"(h[OFF + 26]), "r"(h[OFF + 27]), "r"(h[OFF + 28]), "r"(h[OFF + 29]), \
      "r"(h[OFF + 30]), "r"(h[OFF + 31]))

// TMEM columns: D [0, 16) (O^T, f32), A buffers [32, 96) and [96, 160)
// (128 tokens each as fp16 pairs).  smem: words (row-major, RB per row, the
// 4 chunks of a row rotated by row & 3), P'^T core matrices (8 n x 8 k fp16,
// 128 B each; core (n/8, k/8) at n/8 * SBO + k/8 * LBO).
constexpr uint32_t LBO = 128, SBO = (TOK / 8) * 128;

// mode (attribution runs): 0 = full; 1 = no MMAs (extraction + tcgen05.st +
// the hand-off); 2 = no tcgen05.st (extraction + the hand-off + MMAs)
__global__ void __launch_bounds__(128) tc_pv(const uint16_t* words, const uint16_t* pT,
                                             float* out, long long* cyc, int mode) {
  __shared__ __align__(128) uint8_t sw[ROWS * RB];
  __shared__ __align__(128) uint8_t sp[NH * TOK * 2];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tmem_sh;
  for (int i = threadIdx.x; i < ROWS * RB / 16; i += 128) {
    const int c = i / (RB / 16), j = i % (RB / 16);
    reinterpret_cast<uint4*>(sw)[c * (RB / 16) + (j ^ (c & 3))] =
        reinterpret_cast<const uint4*>(words)[i];
  }
  for (int i = threadIdx.x; i < NH * TOK; i += 128) {  // pT is [n][k]
    const int n = i / TOK, k = i % TOK;
    const uint32_t off = (n / 8) * SBO + (k / 8) * LBO + (n % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<uint16_t*>(sp + off) = pT[i];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
        smem_u32(&tmem_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // sp for the MMA (async proxy)
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_sh;
  const uint32_t idesc = idesc_f16(128, NH);
  const int row = warp * 32 + lane;  // this thread's channel = its TMEM lane
  const uint32_t rbase = smem_u32(sw) + row * RB;
  const uint32_t pbase = smem_u32(sp);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < NB; ++it) {
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int use = 2 * it + hb;  // A-buffer use count
      const int b = use & 1;
      // the MMAs that last read buffer b (use - 2) must be done
      if (use >= 2) mbar_wait(&bar[b], ((use - 2) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      // the row's words of tokens [128 hb, 128 hb + 128): chunks 2hb, 2hb+1
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int jj = 2 * hb + q;
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(w[4 * q]), "=r"(w[4 * q + 1]), "=r"(w[4 * q + 2]), "=r"(w[4 * q + 3])
                     : "r"(rbase + ((jj ^ (row & 3)) << 4)));
      }
      // column i*8 + f: (low, high) = field f of words (2i, 2i+1)
      uint32_t h[64];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t r8 = w[i] >> 8;
        h[i * 8 + 0] = ext2<0>(w[i], r8);
        h[i * 8 + 1] = ext2<1>(w[i], r8);
        h[i * 8 + 2] = ext2<2>(w[i], r8);
        h[i * 8 + 3] = ext2<3>(w[i], r8);
        h[i * 8 + 4] = ext2<4>(w[i], r8);
        h[i * 8 + 5] = ext2<5>(w[i], r8);
        h[i * 8 + 6] = ext2<6>(w[i], r8);
        h[i * 8 + 7] = ext2<7>(w[i], r8);
      }
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 32 + 64 * b;
      if (mode != 2) {
        ST32(0);
        ST32(32);
      } else {
        uint32_t x = 0;  // keep the extraction live
#pragma unroll
        for (int i = 0; i < 64; ++i) x ^= h[i];
        if (x == 0x12345678u) out[0] = 0.f;
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t k0 = 128 * hb + 16 * kk;  // first K index of this MMA
          if (mode != 1)
            tc_mma(tmem, tmem + 32 + 64 * b + 8 * kk, smem_desc(pbase + (k0 / 8) * LBO, LBO, SBO),
                   idesc, (uint32_t)(use | kk));
        }
        tc_commit(&bar[b]);
      }
    }
  }
  // drain: the last use of each buffer
  const int last = 2 * NB - 1;
  mbar_wait(&bar[last & 1], (last >> 1) & 1);
  mbar_wait(&bar[(last - 1) & 1], ((last - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const long long t1 = clock64();
  uint32_t d[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
        "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
        "=r"(d[14]), "=r"(d[15])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int n = 0; n < NH; ++n) out[((size_t)blockIdx.x * ROWS + row) * NH + n] = __uint_as_float(d[n]);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

static uint16_t f2h(float f) {
  __half h = __float2half(f);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static float h2f(uint16_t u) {
  __half h;
  memcpy(&h, &u, 2);
  return __half2float(h);
}

int main() {
  srand(7);
  // codes: row c = 32 u16 words; word g holds 8 tokens (field f = bits 2f..2f+1)
  std::vector<uint16_t> words(ROWS * TOK / 8);
  for (auto& w : words) w = (uint16_t)(rand() & 0xFFFF);
  // P'^T values for (token slot, head) in the ORDER each path consumes them.
  // Path A: warp j, tile pi (16 tokens), HMMA A rows m: gid -> word (8 j + gid
  // within ra/rb?) -- both paths share one definition of token t: word t / 8,
  // field t % 8, and P[t][n].
  std::vector<float> P(TOK * NH);
  for (auto& p : P) p = h2f(f2h((float)(rand() % 1000) / 1000.f));
  // host reference O^T[c][n] = sum_t val(c, t) P[t][n]
  std::vector<double> ref(ROWS * NH, 0.0);
  for (int c = 0; c < ROWS; ++c)
    for (int t = 0; t < TOK; ++t) {
      const double v = field_val(words[c * (TOK / 8) + t / 8], t % 8);
      for (int n = 0; n < NH; ++n) ref[c * NH + n] += v * P[t * NH + n];
    }
  // (A) fragments: ldmatrix (non-trans) of rows (channels) vc*32+lane, chunk j
  // -> per lane: ra = words (c, 8j'..) ... the production mapping: for tile
  // mt (channels mt*16..+15) lane (gid, t4) holds words at row mt*16+gid
  // (+8) and word index 8j + 2*t4 (+1): register = (word 8j+2t4, word 8j+2t4+1)
  // of that row; field f of both halves -> tokens (8(8j+2t4)+f, 8(8j+2t4+1)+f).
  // af[0] (rows gid, k-pair 2t4,2t4+1) = field 2PI of ra; af[1] (rows gid+8)
  // = field 2PI of rb; af[2] (k + 8) = field 2PI+1 of ra; af[3] = of rb.
  // So for tile PI the HMMA K index k (0..15): k = 2t4 + s (s = half) for
  // field 2PI (k < 8) and 8 + 2t4 + s for field 2PI+1, token =
  // 8(8j + 2t4 + s) + field.  B fragment (k, n): b0 = (k = 2t4, 2t4+1; n = gid),
  // b1 = (k = 8 + 2t4, +1; n = gid).
  std::vector<uint32_t> pfrag(4 * 4 * 2 * 32);
  for (int j = 0; j < 4; ++j)
    for (int pi = 0; pi < 4; ++pi)
      for (int lane = 0; lane < 32; ++lane) {
        const int gid = lane >> 2, t4 = lane & 3;
        for (int reg = 0; reg < 2; ++reg) {
          uint32_t v = 0;
          for (int s = 0; s < 2; ++s) {
            const int field = 2 * pi + reg;
            const int t = 8 * (8 * j + 2 * t4 + s) + field;
            v |= (uint32_t)f2h(P[t * NH + gid]) << (16 * s);
          }
          pfrag[((j * 4 + pi) * 2 + reg) * 32 + lane] = v;
        }
      }
  // (B) P'^T [n][k]: K index k of half hb, MMA kk: column col = (k - 128 hb) / 2
  // of the A buffer = i*8 + f, half s = k % 2 -> word 16 hb + 2i + s, field f
  std::vector<uint16_t> pT(NH * TOK);
  for (int k = 0; k < TOK; ++k) {
    const int hb = k / 128, col = (k % 128) / 2, s = k % 2;
    const int i = col / 8, f = col % 8;
    const int t = 8 * (16 * hb + 2 * i + s) + f;
    for (int n = 0; n < NH; ++n) pT[n * TOK + k] = f2h(P[t * NH + n]);
  }
  uint16_t *dw, *dp;
  uint32_t* dpf;
  float *oa, *ob;
  long long* cyc;
  cudaMalloc(&dw, words.size() * 2);
  cudaMalloc(&dp, pT.size() * 2);
  cudaMalloc(&dpf, pfrag.size() * 4);
  cudaMalloc(&oa, (size_t)NCTA * 4 * ROWS * 8 * 4);
  cudaMalloc(&ob, (size_t)NCTA * ROWS * NH * 4);
  cudaMalloc(&cyc, NCTA * 8);
  cudaMemcpy(dw, words.data(), words.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, pT.data(), pT.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dpf, pfrag.data(), pfrag.size() * 4, cudaMemcpyHostToDevice);
  std::vector<long long> hc(NCTA);
  auto report = [&](const char* name, float ms) {
    cudaMemcpy(hc.data(), cyc, NCTA * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (auto x : hc) s += (double)x;
    printf("%-8s %8.1f cycles per (CTA, block)   kernel %.3f ms for %d blocks x %d CTAs\n", name,
           s / NCTA / NB, ms, NB, NCTA);
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // 96 KB of (unused) dynamic shared memory per CTA: two CTAs per SM, as in
  // the decode kernel
  const int pad = 96 * 1024;
  cudaFuncSetAttribute(hmma_pv, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaFuncSetAttribute(tc_pv, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0);
    hmma_pv<<<NCTA, 128, pad>>>(dw, dpf, oa, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) report("mma.sync", ms);
    const char* names[3] = {"tcgen05", "  st only", "  mma only"};
    for (int mode = 2; mode >= 0; --mode) {  // mode 0 last: its D is checked below
      cudaEventRecord(e0);
      tc_pv<<<NCTA, 128, pad>>>(dw, dp, ob, cyc, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) report(names[mode], ms);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  // checks (CTA 0): A sums its 4 warps' partials over heads 0..7; B heads 0..15
  std::vector<float> ha((size_t)4 * ROWS * 8), hb((size_t)ROWS * NH);
  cudaMemcpy(ha.data(), oa, ha.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb.data(), ob, hb.size() * 4, cudaMemcpyDeviceToHost);
  double ea = 0, eb = 0, mx = 0;
  for (int c = 0; c < ROWS; ++c)
    for (int n = 0; n < NH; ++n) {
      const double r = ref[c * NH + n] * NB;
      mx = fmax(mx, fabs(r));
      if (n < 8) {
        double a = 0;
        for (int j = 0; j < 4; ++j) a += ha[((size_t)j * ROWS + c) * 8 + n];
        ea = fmax(ea, fabs(a - r));
      }
      eb = fmax(eb, fabs(hb[(size_t)c * NH + n] - r));
    }
  printf("max |ref| %.4e   max-abs error: mma.sync %.3e  tcgen05 %.3e  (relative %.2e / %.2e)\n", mx,
         ea, eb, ea / mx, eb / mx);
  // both are correct computations of the same sums (a layout error would be
  // O(1)); the tcgen05 path's larger error is its handling of the subnormal
  // fp16 codes (mma.sync: exact, tools/micro/subnormal_mma.cu)
  return (ea / mx < 1e-3 && eb / mx < 1e-3) ? 0 : 2;
}
