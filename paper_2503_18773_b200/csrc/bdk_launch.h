// bdk_launch.h -- host-side launchers for the sm_100a kernels (internal; the
// public boundary is include/bitdecode_b200.h).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bdk_common.cuh"

namespace bdk {

// Device state of one cache (owned by bdk_cache in bdk_api.cpp).
struct DevCache {
  Geom G;
  uint8_t* records = nullptr;  // [cells][max_blocks][rec_bytes]
  __half* res_k = nullptr;     // [cells][n_r][d]
  __half* res_v = nullptr;
  // current lengths (the host points these at the live half of len2 before
  // every launch; kernels other than the fast decode update them in place)
  int* packed_blocks = nullptr;  // [cells]
  int* res_len = nullptr;        // [cells]
  // double-buffered lengths of the fast decode: [2][packed_blocks | res_len][cells].
  // Fast step s reads half (s & 1) -- FastArgs::par, from the host's step
  // count -- and its merging CTAs write every cell's next lengths into the
  // other half, so nothing a step reads changes while it runs.
  int* len2 = nullptr;
};

struct DecodeArgs {
  const __half* q = nullptr;      // [batch][heads_q][d]
  const __half* k_new = nullptr;  // [batch][heads_kv][d] (nullptr: no append)
  const __half* v_new = nullptr;
  float* out = nullptr;           // [batch][heads_q][d] normalized output
  float* out_lse = nullptr;       // optional [batch][heads_q] log2-sum-exp (partial mode)
  float* part_o = nullptr;        // workspace [cells][n_parts][n_group][d]
  float* part_ml = nullptr;       // workspace [cells][n_parts][n_group][2]
  int heads_q = 0, n_group = 0;
  int n_splits = 1, blocks_per_split = 1;
  int blk_begin = 0, blk_end = 1 << 30;  // packed block range attended
  int precise = 0;                        // hi/lo split P
  int skip_residual = 0;                  // partial decode without the residual
  float sm_scale_log2 = 0.f;
  // optional CUDA events recorded on the launching stream immediately before
  // and after the attention kernel (bdk_profile_begin/end)
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
};

// Fast decode (bdk_decode_fast.cu): stream-K over (cell, unit) with unit =
// one packed block or the residual window of a cell; the LSE combine, the
// length commit and the fused flush run in the combine grid launched after it.
struct FastArgs {
  const __half* q = nullptr;      // [batch][heads_q][d]
  const __half* k_new = nullptr;  // [batch][heads_kv][d] (nullptr: no append)
  const __half* v_new = nullptr;
  float* out = nullptr;      // [batch][heads_q][d]
  float* out_lse = nullptr;  // optional [batch][heads_q] (log2 domain)
  float* slots = nullptr;    // [n_ctas + cells][n_group][d + 2] partials
  int* done = nullptr;       // [2][cells] partials written per cell, by step parity
  int spin = 0;              // host schedule: the combine grid starts on `done` counts
  int n_ctas = 0, heads_q = 0, n_group = 0;
  int blk_begin = 0, blk_end = 1 << 30;  // packed block range attended
  int skip_residual = 0;  // residual units attend nothing (sequence-split ranks)
  int par = 0;            // half of DevCache::len2 this step reads (step & 1)
  int rt = 0;             // residual tokens per unit (set by launch_decode_fast)
  // schedule.  dev_sched = 0: from the host mirror of the lengths -- every
  // cell uni_units units of which uni_nb packed, or (uni_units == 0) the
  // uploaded prefix unit_off [cells + 1] and unit_nb [cells]; total_units.
  // dev_sched = 1: scanned on the device from len2 (a launch whose arguments
  // hold for any lengths: the steps of a captured CUDA graph)
  int dev_sched = 0;
  long long total_units = 0;
  int uni_units = 0, uni_nb = 0;
  int uni_len = 0, uni_pb = 0, uni_rl = 0;  // host schedule: every cell has these lengths
  // extra (empty) residual units per cell: the schedule charges a cell's
  // residual tail + segment switch this many more blocks' worth of time, so
  // the CTAs that hold one take fewer packed blocks
  int res_extra = 0;
  const int* unit_off = nullptr;
  const int* unit_nb = nullptr;
  float sm_scale_log2 = 0.f;
  unsigned long long* trace = nullptr;  // dev: [n_ctas][16] globaltimer stamps
  int dev_flags = 0;                    // dev probes (BDK_DEV_FLAGS): 1 no compute, 2 no prep
  int pdl = 0;  // launched as a programmatic dependent of the previous kernel
  int prefetch_ok = 0;  // no packed record changed since the previous kernel: the
                        // TMA warp may stream the first ring stages before
                        // griddepcontrol.wait
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
};

// floats per partial slot of the fast kernel: n_group x [d] unnormalized O,
// then n_group (max, sum) pairs; padded to a float4 multiple
__host__ __device__ inline int slot_stride(int n_group) {
  return (n_group * 130 + 3) / 4 * 4;
}

bool fast_path_ok(const Geom& G);
// geometry served by the folded-dequant stream-K kernel
bool fast_decode_ok(const Geom& G, int n_group);
// resident CTAs per SM of the fast kernel for this geometry (occupancy API)
int fast_decode_ctas_per_sm(const Geom& G, int n_group);
// tokens per residual unit of the fast kernel's schedule
int fast_residual_tokens(const Geom& G);
cudaError_t launch_decode_fast(const DevCache& c, const FastArgs& a, cudaStream_t s);
// quantize+pack every full residual window into its next block slot and
// commit (packed_blocks++, res_len = 0): Algorithm 2's flush after the step
cudaError_t launch_flush_full(const DevCache& c, cudaStream_t s);
int max_ctas_per_sm(const Geom& G);

cudaError_t launch_prefill(const DevCache& c, const __half* k, const __half* v, int len,
                           int cell_begin, int n_cells, cudaStream_t s);
cudaError_t launch_append(const DevCache& c, int cell, const __half* k_row, const __half* v_row,
                          cudaStream_t s);
cudaError_t launch_flush(const DevCache& c, int cell, cudaStream_t s);
cudaError_t launch_build(const DevCache& c, int cell, cudaStream_t s);  // pack, no commit
cudaError_t launch_decode(const DevCache& c, const DecodeArgs& a, cudaStream_t s);
// copy bytes (rounded up to 16) from mapped pinned host memory to the device;
// a PDL primary for the decode launch that follows
cudaError_t launch_stage_in(const void* src_host, void* dst, size_t bytes, cudaStream_t s);
// dequantize blocks [blk0, blk0+nblk) of a cell into fp16 [nblk*n_r][d] rows
cudaError_t launch_dequant(const DevCache& c, int cell, int blk0, int nblk, __half* k_out,
                           __half* v_out, cudaStream_t s);
// merge normalized (o, lse) partials of n_parts ranks: o [n_parts][rows][d],
// lse [n_parts][rows] (log2 domain) -> out [rows][d]
// sequence-split exchange over peer memory (bdk_peer_merge)
constexpr int kMaxPeers = 8;
struct PeerMergeArgs {
  const float* parts[kMaxPeers];  // slot of each rank: [rows*d o | rows lse] (peer-mapped)
  unsigned* flags[kMaxPeers];     // each rank's monotonic step flag (peer-mapped)
  int world = 1, rank = 0;
  long long step = 0;
  int rows = 0, d = 0;
  float* out = nullptr;
  float* out_lse = nullptr;
  int* err = nullptr;
  unsigned long long timeout_ns = 0;
};
cudaError_t launch_peer_merge(const PeerMergeArgs& a, cudaStream_t s);

// General span attention (bdk_span.cu): decode_step for geometry outside the
// fast kernels' envelope and the reference's attention internals
// (attend_tile / residual_attend / packed_attend / combine).  One CTA per
// (part, cell); a part is a cell's residual window or one split of its packed
// segment, split by the reference's rule (attention.cpp:116-130).  A part's
// state is [rows*d o | rows m | rows l] fp32, unnormalized (PartialOutput).
enum SpanSource { kSpanCache = 0, kSpanFp32 = 1 };
struct SpanArgs {
  DevCache c;
  int source = kSpanCache;
  const float* k32 = nullptr;  // kSpanFp32: tokens [len32][d]
  const float* v32 = nullptr;
  int len32 = 0;
  const __half* q16 = nullptr;  // [batch][heads_q][d], times q_scale in fp32 (decode)
  const float* q32 = nullptr;   // [rows][d] as given (one cell)
  float q_scale = 1.f, scale = 1.f;
  const __half* k_new = nullptr;  // decode append rows [cells][d]; written by the residual part
  const __half* v_new = nullptr;
  int heads_q = 0, rows = 0, d = 0;
  int cell0 = 0;
  int residual = 1;  // part 0 of every cell is its residual window
  int tile_n = 64, splits = 1;
  int blk_begin = 0, blk_end = 1 << 30;
  int warp_n = 1;
  int keep_state = 0;  // parts already hold the initial state
  float* parts = nullptr;  // [cells][n_parts][rows * (d + 2)]
  int n_parts = 1;
  // set by launch_span_parts: which stages fit in shared memory (else the K/V
  // chunk is read from the source and the P.V sums live in `scratch`)
  int kv_smem = 1, pacc_smem = 1;
  float* scratch = nullptr;
};
// minimal dynamic shared memory of one span CTA (tile = the longest tile it
// walks); the K/V chunk stage and P.V sums are added when they fit
size_t span_smem_bytes(int rows, int d, int tile);
cudaError_t launch_span_parts(const SpanArgs& a, int n_cells, cudaStream_t s);
// combine (attention.cpp:142-162) of each cell's n_parts states -> out rows
// b*heads_q + hk*rows + r; optional log2-sum-exp; res_len (nullable) += 1
cudaError_t launch_span_combine(const float* parts, int n_cells, int n_parts, int rows, int d,
                                int heads_kv, int heads_q, float* out, float* out_lse,
                                int* res_len, cudaStream_t s);
cudaError_t launch_partitioned_rowmax(const float* s, int rows, int cols, int warp_n, float* out,
                                      cudaStream_t st);

// quant.hpp utilities (bdk_quantize_tile / bdk_dequantize_tile)
cudaError_t launch_quantize_tile(const float* x, int rows, int d, int bits, int axis, int g,
                                 uint16_t* codes, uint32_t* params, cudaStream_t s);
cudaError_t launch_dequantize_tile(const uint16_t* codes, const uint32_t* params, int rows, int d,
                                   int axis, int g, int round16, float* out, cudaStream_t s);

cudaError_t launch_quantize_group(const float* x, int n, float s, float z, int bits,
                                  uint16_t* codes, cudaStream_t st);
cudaError_t launch_dequantize_group(const uint16_t* codes, int n, float s, float z, float* out,
                                    cudaStream_t st);

cudaError_t launch_merge_partials(const float* o, const float* lse, int n_parts, int rows, int d,
                                  size_t o_stride, size_t lse_stride, float* out, cudaStream_t s);

}  // namespace bdk
