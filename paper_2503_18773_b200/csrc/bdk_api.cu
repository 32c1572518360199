// bdk_api.cu -- host implementation of the C-ABI (include/bitdecode_b200.h).
//
// Owns the device arena of one cache and an authoritative host mirror of the
// per-cell lengths (packed blocks, residual fill).  The mirror drives the
// reference's precondition checks (StateError / CapacityError / ShapeError,
// kvcache.cpp:155-251, attention.cpp:164-179) before any launch, and the
// split planning of the decode grid.  No exception crosses the boundary and
// there is no host compute path: every numeric step runs in the sm_100a
// kernels of bdk_kernels.cu.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/bitdecode_b200.h"
#include "bdk_launch.h"

using bdk::DevCache;
using bdk::Geom;

struct bdk_cache {
  DevCache dev;
  bdk_cache_desc desc{};
  int device = 0;
  int num_sms = 148;
  int precise = 1;  // the reference's 1e-5 contract unless the caller opts into fast
  uint32_t kp_u16 = 0, vp_u16 = 0, wpb = 0;
  std::vector<int> packed_blocks, res_len;  // host mirror
  // decode workspace
  float* part_o = nullptr;
  float* part_ml = nullptr;
  size_t part_floats = 0, part_ml_floats = 0;
  // span-path partial states (bdk_span.cu)
  float* span_parts = nullptr;
  size_t span_floats = 0;
  // host-API staging (pinned host + device)
  void* h_stage = nullptr;
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  // fast-path (stream-K) resources
  uint64_t fast_steps = 0;            // fast decode steps (their parity picks the len2 half)
  bool capturing_pdl_off = false;     // graph capture without programmatic launch edges
  int* unit_off = nullptr;            // device host-schedule [unit_off (cells + 1) | unit_nb (cells)]
  std::vector<int> unit_off_host;     // last uploaded host schedule
  bool blocks_written = true;         // a packed record may have changed since the last fast step
  int graphs = 0;                     // live bdk_graph objects (workspaces are pinned)
  float* slots = nullptr;             // device partial slots
  int* done = nullptr;                // device [2][cells] partials written per cell
  bool done_live = false;             // the last fast step kept `done` counted
  size_t slot_floats = 0;
  int fast_ctas_per_sm = -1, fast_ng = -1;
  // attention-kernel timing (bdk_profile_begin/end): one event pair per launch
  bool profiling = false;
  mutable uint64_t launches = 0;  // kernels this cache has launched (all entry points)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  size_t events_used = 0;
};

namespace {

thread_local std::string g_err;

bdk_status fail(bdk_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

bdk_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return BDK_CUDA_ERROR;
}

// Makes `dev` current for the scope of one C-ABI call and restores the
// caller's device on exit: every allocation and launch of a cache lands on the
// cache's own GPU, and a call never changes the calling thread's device.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DevGuard(const DevGuard&) = delete;
  DevGuard& operator=(const DevGuard&) = delete;
};

#define BDK_CUDA(call, where)                  \
  do {                                         \
    cudaError_t e_ = (call);                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int cell_of(const bdk_cache* c, uint32_t b, uint32_t h) {
  return static_cast<int>(b * c->desc.heads_kv + h);
}

bdk_status check_cell(const bdk_cache* c, uint32_t b, uint32_t h) {
  if (!c) return fail(BDK_INVALID_ARGUMENT, "null cache");
  if (b >= c->desc.batch || h >= c->desc.heads_kv)
    return fail(BDK_SHAPE_ERROR, "cell index out of range");
  return BDK_OK;
}

uint32_t param_u16(uint32_t n_r, uint32_t d, uint32_t bits, uint32_t axis, uint32_t g) {
  if (bits == 16) return 0;
  const uint32_t groups = axis == 0 ? (n_r / g) * d : n_r * (d / g);
  return 2 * groups;  // (scale, zero) halves, quant.hpp:38-47
}

size_t word_offset(const Geom& G, uint32_t word) {
  // logical word index -> byte offset inside the swizzled word array
  const uint32_t per_row = 8 * G.warp_n;
  const uint32_t c = word / per_row, wi = word % per_row, j = wi / 8;
  return (size_t)c * 16 * G.warp_n + ((j ^ bdk::swz(c, G.warp_n)) << 4) + (wi % 8) * 2;
}

bdk_status ensure_workspace(bdk_cache* c, int n_parts, int ng) {
  const size_t cells = (size_t)c->desc.batch * c->desc.heads_kv;
  const size_t need = cells * n_parts * ng * c->desc.head_dim;
  const size_t need_ml = cells * n_parts * ng * 2;
  if (need > c->part_floats) {
    if (c->part_o) cudaFree(c->part_o);
    c->part_o = nullptr;
    BDK_CUDA(cudaMalloc(&c->part_o, need * sizeof(float)), "cudaMalloc(partials)");
    c->part_floats = need;
  }
  if (need_ml > c->part_ml_floats) {
    if (c->part_ml) cudaFree(c->part_ml);
    c->part_ml = nullptr;
    BDK_CUDA(cudaMalloc(&c->part_ml, need_ml * sizeof(float)), "cudaMalloc(partials)");
    c->part_ml_floats = need_ml;
  }
  return BDK_OK;
}

bdk_status ensure_stage(bdk_cache* c, size_t bytes) {
  if (bytes <= c->stage_bytes) return BDK_OK;
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->d_stage) cudaFree(c->d_stage);
  c->h_stage = c->d_stage = nullptr;
  BDK_CUDA(cudaMallocHost(&c->h_stage, bytes), "cudaMallocHost(stage)");
  BDK_CUDA(cudaMalloc(&c->d_stage, bytes), "cudaMalloc(stage)");
  c->stage_bytes = bytes;
  return BDK_OK;
}

bdk_status validate(const bdk_attn_config* cfg) {
  auto req = [](bool ok, const char* what) { return ok ? BDK_OK : fail(BDK_CONFIG_ERROR, what); };
  bdk_status s;
  if ((s = req(cfg->batch > 0, "batch must be > 0"))) return s;
  if ((s = req(cfg->heads_q > 0, "heads_q must be > 0"))) return s;
  if ((s = req(cfg->heads_kv > 0, "heads_kv must be > 0"))) return s;
  if ((s = req(cfg->head_dim > 0, "head_dim must be > 0"))) return s;
  if ((s = req(cfg->tile_m > 0, "tile_m must be > 0"))) return s;
  if ((s = req(cfg->tile_n > 0, "tile_n must be > 0"))) return s;
  if ((s = req(cfg->num_splits >= 1, "num_splits must be >= 1"))) return s;
  if ((s = req(cfg->warp_n > 0, "warp_n must be > 0"))) return s;
  if ((s = req(cfg->warp_m > 0, "warp_m must be > 0"))) return s;
  if ((s = req(cfg->heads_q % cfg->heads_kv == 0, "heads_q must be divisible by heads_kv")))
    return s;
  if ((s = req(cfg->tile_n % (cfg->warp_n * 8) == 0, "tile_n must be divisible by warp_n*8")))
    return s;
  return BDK_OK;
}

// geometry the tensor-core decode kernels serve; anything else the reference
// accepts runs on the span path (bdk_span.cu)
bool exact_ok(const bdk_cache* c, const bdk_attn_config* cfg) {
  return bdk::fast_path_ok(c->dev.G) && cfg->heads_q / cfg->heads_kv <= 8;
}

constexpr size_t kSpanSmemMax = 227u << 10;

// decode_step shape checks (attention.cpp:164-179) + capacity of the append
bdk_status check_decode(bdk_cache* c, const bdk_attn_config* cfg, bool appends) {
  if (!c || !cfg) return fail(BDK_INVALID_ARGUMENT, "null argument");
  bdk_status s = validate(cfg);
  if (s) return s;
  if (cfg->batch != c->desc.batch || cfg->heads_kv != c->desc.heads_kv ||
      cfg->head_dim != c->desc.head_dim)
    return fail(BDK_SHAPE_ERROR, "decode_step: cache geometry does not match config");
  if (!exact_ok(c, cfg)) {
    const int tile = static_cast<int>(std::max<uint32_t>(cfg->tile_n, c->dev.G.n_r));
    if (bdk::span_smem_bytes(cfg->heads_q / cfg->heads_kv, cfg->head_dim, tile) > kSpanSmemMax)
      return fail(BDK_UNSUPPORTED, "n_group * (head_dim + max(tile_n, N_r)) exceeds shared memory");
  }
  if (appends) {
    const int n_r = c->dev.G.n_r;
    for (size_t i = 0; i < c->res_len.size(); ++i) {
      if (c->res_len[i] == n_r)
        return fail(BDK_CAPACITY_ERROR, "residual is full; flush before appending");
      if (c->res_len[i] + 1 == n_r && c->packed_blocks[i] >= c->dev.G.max_blocks)
        return fail(BDK_CAPACITY_ERROR, "cache arena full (raise max_tokens)");
    }
  }
  return BDK_OK;
}

bdk_status next_events(bdk_cache* c, cudaEvent_t* e0, cudaEvent_t* e1) {
  *e0 = *e1 = nullptr;
  if (!c->profiling) return BDK_OK;
  if (c->events_used == c->events.size()) {
    cudaEvent_t a, b;
    BDK_CUDA(cudaEventCreate(&a), "cudaEventCreate");
    BDK_CUDA(cudaEventCreate(&b), "cudaEventCreate");
    c->events.emplace_back(a, b);
  }
  *e0 = c->events[c->events_used].first;
  *e1 = c->events[c->events_used].second;
  c->events_used++;
  return BDK_OK;
}

// The live half of the double-buffered device lengths (DevCache::len2) for
// kernels that update lengths in place (prefill, append, flush, precise and
// span decode, readback): half (fast steps & 1).
void point_lengths(bdk_cache* c) {
  const size_t cells = (size_t)c->desc.batch * c->desc.heads_kv;
  const size_t par = c->fast_steps & 1;
  c->dev.packed_blocks = c->dev.len2 + par * 2 * cells;
  c->dev.res_len = c->dev.packed_blocks + cells;
}

// mirror of one fast step's commit: every cell +1 token when it appends, a
// full window becomes a block (written by the step's merging CTA); the
// lengths now live in the other half of len2
void advance_fast_step(bdk_cache* c, bool appends) {
  c->blocks_written = false;
  if (appends) {
    for (size_t i = 0; i < c->res_len.size(); ++i) {
      if (++c->res_len[i] == c->dev.G.n_r) {
        c->res_len[i] = 0;
        c->packed_blocks[i] += 1;
        c->blocks_written = true;
      }
    }
  }
  c->fast_steps += 1;
  point_lengths(c);
}

// Stream-K fast path (bdk_decode_fast.cu): ONE launch per step -- append,
// attention, combine and the flush of any residual the step fills.  Eager
// steps take their schedule from the host mirror of the lengths (arguments,
// plus an upload when it is not uniform and changed); graph-captured steps
// (dev_sched) scan the device lengths instead, so their arguments hold for any
// lengths and a captured graph of steps replays correctly.  Both give the
// same unit partition, hence bit-identical results.
bdk_status run_decode_fast(bdk_cache* c, const bdk_attn_config* cfg, const void* q,
                           const void* k_new, const void* v_new, float* out, float* lse,
                           int blk_begin, int blk_end, cudaStream_t stream, bool no_res,
                           bool dev_sched = false) {
  const int cells = static_cast<int>(c->desc.batch * c->desc.heads_kv);
  const int ng = static_cast<int>(cfg->heads_q / cfg->heads_kv);
  const Geom& G = c->dev.G;
  DevGuard dev_guard_(c->device);
  if (c->fast_ng != ng) {
    c->fast_ctas_per_sm = bdk::fast_decode_ctas_per_sm(G, ng);
    c->fast_ng = ng;
    if (c->fast_ctas_per_sm <= 0)
      return fail(BDK_CUDA_ERROR, "fast decode kernel does not fit on this device");
  }
  const int n_ctas = c->fast_ctas_per_sm * c->num_sms;  // one wave, every step
  const size_t need = (size_t)(n_ctas + cells) * bdk::slot_stride(ng);
  if (need > c->slot_floats) {
    if (c->graphs > 0)
      return fail(BDK_STATE_ERROR, "decode workspace would move under a live bdk_graph");
    if (c->slots) {
      BDK_CUDA(cudaStreamSynchronize(stream), "slots resize");
      cudaFree(c->slots);
    }
    c->slots = nullptr;
    BDK_CUDA(cudaMalloc(&c->slots, need * sizeof(float)), "cudaMalloc(slots)");
    c->slot_floats = need;
  }
  if (!c->done) BDK_CUDA(cudaMalloc(&c->done, 2 * cells * sizeof(int)), "cudaMalloc(done)");
  bdk::FastArgs a;
  // the combine grid starts on per-cell completion counts when it is small
  // enough to sit resident beside the attention grid's tail (C1, C2, C5);
  // a large one (C3: 1024 CTAs) waits for the grid instead (measured)
  a.spin = (size_t)cells * ng <= (size_t)n_ctas ? 1 : 0;
  // counted only when the combine spins on them (the release adds cost a
  // fence per segment: C3's 1024 cells); a step that starts counting again
  // after steps that did not finds both parities zeroed
  if (a.spin && !c->done_live)
    BDK_CUDA(cudaMemsetAsync(c->done, 0, 2 * cells * sizeof(int), stream), "memset(done)");
  c->done_live = a.spin != 0;
  a.done = a.spin ? c->done : nullptr;
  a.q = static_cast<const __half*>(q);
  a.k_new = static_cast<const __half*>(k_new);
  a.v_new = static_cast<const __half*>(v_new);
  a.out = out;
  a.out_lse = lse;
  a.slots = c->slots;
  a.n_ctas = n_ctas;
  a.heads_q = static_cast<int>(cfg->heads_q);
  a.n_group = ng;
  a.blk_begin = blk_begin;
  a.blk_end = blk_end;
  a.skip_residual = no_res ? 1 : 0;
  a.sm_scale_log2 = (1.0f / std::sqrt(static_cast<float>(cfg->head_dim))) * bdk::kLog2e;
  a.par = static_cast<int>(c->fast_steps & 1);
  // schedule weight of a cell's residual tail + segment switch: 3 extra
  // (empty) units when CTAs average >= 2 packed blocks (measured: C5 +2.2%,
  // C2 +4.3%, C3 +0.5%; C1, under one block per CTA, loses with it).  Any
  // value gives the same partials' union, so graph steps keep the one they
  // were captured with.  Dev knob BDK_RESW overrides.
  {
    static const int resw_knob = getenv("BDK_RESW") ? atoi(getenv("BDK_RESW")) : -1;
    long long nb_all = 0;
    for (int i = 0; i < cells; ++i)
      nb_all += std::max(0, std::min(blk_end, c->packed_blocks[i]) - blk_begin);
    a.res_extra = resw_knob >= 0 ? resw_knob : (nb_all >= 2LL * n_ctas ? 3 : 0);
  }
  static const bool dev_sched_knob = getenv("BDK_DEVSCHED") && atoi(getenv("BDK_DEVSCHED")) == 1;
  if (dev_sched_knob) dev_sched = true;
  a.dev_sched = dev_sched ? 1 : 0;
  if (!dev_sched) {
    // schedule: [unit_off (cells + 1) | unit_nb (cells)]; a cell's units are
    // its packed blocks in range then ceil(res_len' / rt) residual units
    const int rt = bdk::fast_residual_tokens(G);
    std::vector<int> off(2 * cells + 1, 0);
    for (int i = 0; i < cells; ++i) {
      const int nb = std::max(0, std::min(blk_end, c->packed_blocks[i]) - blk_begin);
      const int rlen = no_res ? 0 : c->res_len[i] + (k_new != nullptr ? 1 : 0);
      off[i + 1] = off[i] + nb + std::max(1, (rlen + rt - 1) / rt) + a.res_extra;
      off[cells + 1 + i] = nb;
    }
    bool uni = true;
    for (int i = 1; i < cells && uni; ++i)
      uni = off[i + 1] - off[i] == off[1] - off[0] && off[cells + 1 + i] == off[cells + 1];
    a.total_units = off[cells];
    a.uni_units = uni ? off[1] - off[0] : 0;
    a.uni_nb = uni ? off[cells + 1] : 0;
    bool uni_len = true;
    for (int i = 1; i < cells && uni_len; ++i)
      uni_len = c->packed_blocks[i] == c->packed_blocks[0] && c->res_len[i] == c->res_len[0];
    a.uni_len = uni_len ? 1 : 0;
    a.uni_pb = c->packed_blocks[0];
    a.uni_rl = c->res_len[0];
    if (!uni) {
      if (!c->unit_off)
        BDK_CUDA(cudaMalloc(&c->unit_off, (2 * cells + 1) * sizeof(int)), "cudaMalloc(schedule)");
      if (off != c->unit_off_host) {
        BDK_CUDA(cudaMemcpyAsync(c->unit_off, off.data(), (2 * cells + 1) * sizeof(int),
                                 cudaMemcpyHostToDevice, stream),
                 "H2D schedule");
        c->unit_off_host = off;
      }
      a.unit_off = c->unit_off;
      a.unit_nb = c->unit_off + cells + 1;
    }
  }
  // the first ring stages may stream before the previous kernel ends when no
  // packed record changed since the last fast step (dev knob BDK_PREFETCH=0)
  static const bool prefetch_off = getenv("BDK_PREFETCH") && atoi(getenv("BDK_PREFETCH")) == 0;
  a.prefetch_ok = (c->blocks_written || prefetch_off) ? 0 : 1;
  bdk_status st = next_events(c, &a.ev_begin, &a.ev_end);
  if (st) return st;
  // dev knob: BDK_TRACE=<file> appends per-CTA globaltimer stamps of every
  // fast launch (synchronizes; never set in measurements)
  static const char* trace_path = getenv("BDK_TRACE");
  static const int dev_flags = getenv("BDK_DEV_FLAGS") ? atoi(getenv("BDK_DEV_FLAGS")) : 0;
  static const bool pdl_off = getenv("BDK_PDL") && atoi(getenv("BDK_PDL")) == 0;
  a.dev_flags = dev_flags;
  // PDL: overlap this launch's prologue with the tail of the previous kernel
  a.pdl = pdl_off || a.ev_begin || c->capturing_pdl_off ? 0 : 1;
  unsigned long long* trace = nullptr;
  if (trace_path) {
    BDK_CUDA(cudaMalloc(&trace, (size_t)n_ctas * 16 * 8), "cudaMalloc(trace)");
    BDK_CUDA(cudaMemsetAsync(trace, 0, (size_t)n_ctas * 16 * 8, stream), "memset(trace)");
    a.trace = trace;
  }
  BDK_CUDA(bdk::launch_decode_fast(c->dev, a, stream), "fast decode launch");
  c->launches += 2;  // attention grid + combine grid
  if (trace) {
    std::vector<unsigned long long> h((size_t)n_ctas * 16);
    BDK_CUDA(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, stream),
             "D2H trace");
    BDK_CUDA(cudaStreamSynchronize(stream), "trace sync");
    cudaFree(trace);
    if (FILE* f = fopen(trace_path, "a")) {
      fprintf(f, "launch n_ctas=%d\n", n_ctas);
      for (int i = 0; i < n_ctas; ++i) {
        for (int k = 0; k < 16; ++k) fprintf(f, "%llu ", h[(size_t)i * 16 + k]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  // the step's length commit, mirrored: the device lengths now live in the
  // other half of the double buffer
  advance_fast_step(c, k_new != nullptr && !no_res);
  return BDK_OK;
}

bdk_status ensure_span(bdk_cache* c, size_t floats) {
  if (floats <= c->span_floats) return BDK_OK;
  if (c->span_parts) cudaFree(c->span_parts);
  c->span_parts = nullptr;
  BDK_CUDA(cudaMalloc(&c->span_parts, floats * sizeof(float)), "cudaMalloc(span parts)");
  c->span_floats = floats;
  return BDK_OK;
}

// decode_step on the span path (bdk_span.cu): the reference's own
// decomposition -- residual window (with the appended token) as part 0, then
// packed splits of cfg->tile_n tiles by the reference's split rule -- combined
// in that order, then the flush of any residual the step filled.  The split
// count is cfg->num_splits raised so that no CTA walks more than 4 tiles
// (capped at 1024 splits and by a 256 MiB partial-state budget).
bdk_status run_decode_span(bdk_cache* c, const bdk_attn_config* cfg, const void* q,
                           const void* k_new, const void* v_new, float* out, float* lse,
                           int blk_begin, int blk_end, cudaStream_t stream, bool no_res) {
  const int cells = static_cast<int>(c->desc.batch * c->desc.heads_kv);
  const int ng = static_cast<int>(cfg->heads_q / cfg->heads_kv), d = c->desc.head_dim;
  bdk::SpanArgs a;
  a.c = c->dev;
  a.q16 = static_cast<const __half*>(q);
  a.q_scale = 1.0f / std::sqrt(static_cast<float>(d));  // attention.cpp:198
  a.k_new = static_cast<const __half*>(k_new);
  a.v_new = static_cast<const __half*>(v_new);
  a.heads_q = static_cast<int>(cfg->heads_q);
  a.rows = ng;
  a.d = d;
  a.residual = no_res ? 0 : 1;
  a.tile_n = static_cast<int>(cfg->tile_n);
  // the reference's num_splits, raised so that no CTA walks more than 4
  // tiles (a CTA's walk is sequential; results are split-invariant within
  // the reference's 1e-5, test_attention.cpp:312-340)
  {
    int nblk = 0;
    for (int i = 0; i < cells; ++i) nblk = std::max(nblk, c->packed_blocks[i]);
    const long long lo = std::max(0, blk_begin), hi = std::min<long long>(blk_end, nblk);
    const long long toks = std::max(0LL, hi - lo) * c->dev.G.n_r;
    const long long tiles = (toks + cfg->tile_n - 1) / cfg->tile_n;
    const long long per_split = (long long)cells * ng * (d + 2);  // floats of one split
    const long long budget = std::max(1LL, (64LL << 20) / std::max(1LL, per_split) - 1);
    const long long raised = std::min({1024LL, (tiles + 3) / 4, budget});
    a.splits = static_cast<int>(std::max<long long>(cfg->num_splits, raised));
  }
  a.blk_begin = std::max(0, blk_begin);
  a.blk_end = blk_end;
  a.warp_n = static_cast<int>(cfg->warp_n);
  a.n_parts = a.residual + a.splits;
  bdk_status s = ensure_span(c, (size_t)cells * a.n_parts * ng * (d + 2));
  if (s) return s;
  a.parts = c->span_parts;
  DevGuard dev_guard_(c->device);
  BDK_CUDA(bdk::launch_span_parts(a, cells, stream), "span launch");
  BDK_CUDA(bdk::launch_span_combine(c->span_parts, cells, a.n_parts, ng, d,
                                    static_cast<int>(c->desc.heads_kv),
                                    static_cast<int>(cfg->heads_q), out, lse,
                                    k_new != nullptr ? c->dev.res_len : nullptr, stream),
           "span combine launch");
  c->launches += 2;
  c->blocks_written = true;  // packed records may change (no PDL prefetch next)
  if (k_new != nullptr) {
    bool full = false;
    for (int i = 0; i < cells; ++i) full |= c->res_len[i] + 1 == c->dev.G.n_r;
    if (full) {
      BDK_CUDA(bdk::launch_flush_full(c->dev, stream), "flush launch");
      c->launches += 1;
    }
    for (int i = 0; i < cells; ++i) {
      if (++c->res_len[i] == c->dev.G.n_r) {
        c->res_len[i] = 0;
        c->packed_blocks[i] += 1;
      }
    }
  }
  return BDK_OK;
}

bdk_status run_decode(bdk_cache* c, const bdk_attn_config* cfg, const void* q, const void* k_new,
                      const void* v_new, float* out, float* lse, int blk_begin, int blk_end,
                      cudaStream_t stream, bool no_res = false) {
  DevGuard dev_guard_(c->device);  // workspaces and launches on the cache's GPU
  const int cells = static_cast<int>(c->desc.batch * c->desc.heads_kv);
  if (!exact_ok(c, cfg))
    return run_decode_span(c, cfg, q, k_new, v_new, out, lse, blk_begin, blk_end, stream, no_res);
  if (!c->precise && bdk::fast_decode_ok(c->dev.G, static_cast<int>(cfg->heads_q / cfg->heads_kv)))
    return run_decode_fast(c, cfg, q, k_new, v_new, out, lse, std::max(0, blk_begin), blk_end,
                           stream, no_res);
  int nblk_max = 0;
  for (int i = 0; i < cells; ++i) nblk_max = std::max(nblk_max, c->packed_blocks[i]);
  const int lo = std::max(0, blk_begin), hi = std::min(blk_end, nblk_max);
  const int span = std::max(0, hi - lo);
  // split planning: ~3 resident CTAs per SM worth of packed blocks, <= 256
  // splits per cell (attention.cpp:116-130 splits on the CPU; the GPU picks
  // its own -- results are split-invariant, test_attention.cpp:312-340)
  const long target = (long)c->num_sms * bdk::max_ctas_per_sm(c->dev.G);
  int bps = 1;
  if (span > 0) {
    bps = static_cast<int>(std::max<long>(1, ((long)cells * span + target - 1) / target));
    bps = std::max(bps, (span + 255) / 256);
  }
  const int n_splits = span > 0 ? (span + bps - 1) / bps : 1;
  const int ng = static_cast<int>(cfg->heads_q / cfg->heads_kv);
  bdk_status s = ensure_workspace(c, n_splits + 1, ng);
  if (s) return s;

  bdk::DecodeArgs a;
  a.q = static_cast<const __half*>(q);
  a.k_new = static_cast<const __half*>(k_new);
  a.v_new = static_cast<const __half*>(v_new);
  a.out = out;
  a.out_lse = lse;
  a.part_o = c->part_o;
  a.part_ml = c->part_ml;
  a.heads_q = static_cast<int>(cfg->heads_q);
  a.n_group = ng;
  a.n_splits = n_splits;
  a.blocks_per_split = bps;
  a.blk_begin = lo;
  a.blk_end = hi;
  a.skip_residual = no_res ? 1 : 0;
  a.precise = c->precise;
  a.sm_scale_log2 = (1.0f / std::sqrt(static_cast<float>(cfg->head_dim))) * bdk::kLog2e;
  {
    bdk_status st = next_events(c, &a.ev_begin, &a.ev_end);
    if (st) return st;
  }
  BDK_CUDA(bdk::launch_decode(c->dev, a, stream), "decode launch");
  c->blocks_written = true;  // packed records may change (no PDL prefetch next)
  c->launches += 2;  // split-KV kernel + combine kernel
  if (k_new != nullptr) {  // mirror of the cache-update phase
    for (int i = 0; i < cells; ++i) {
      if (++c->res_len[i] == c->dev.G.n_r) {
        c->res_len[i] = 0;
        c->packed_blocks[i] += 1;
      }
    }
  }
  return BDK_OK;
}

}  // namespace

extern "C" {

const char* bdk_last_error(void) { return g_err.c_str(); }

const char* bdk_status_name(bdk_status s) {
  switch (s) {
    case BDK_OK: return "OK";
    case BDK_CONFIG_ERROR: return "ConfigError";
    case BDK_SHAPE_ERROR: return "ShapeError";
    case BDK_UNSUPPORTED_BITS: return "UnsupportedBits";
    case BDK_CODE_OVERFLOW: return "CodeOverflow";
    case BDK_CAPACITY_ERROR: return "CapacityError";
    case BDK_STATE_ERROR: return "StateError";
    case BDK_FORMAT_ERROR: return "FormatError";
    case BDK_EMPTY_INPUT: return "EmptyInput";
    case BDK_CUDA_ERROR: return "CudaError";
    case BDK_UNSUPPORTED: return "Unsupported";
    case BDK_INVALID_ARGUMENT: return "InvalidArgument";
  }
  return "Unknown";
}

bdk_status bdk_validate_config(const bdk_attn_config* cfg) {
  if (!cfg) return fail(BDK_INVALID_ARGUMENT, "null config");
  return validate(cfg);
}

bdk_status bdk_cache_create(const bdk_cache_desc* d, bdk_cache** out) {
  if (!d || !out) return fail(BDK_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (d->batch == 0 || d->heads_kv == 0 || d->head_dim == 0 || d->warp_n == 0)
    return fail(BDK_CONFIG_ERROR, "cache geometry fields must be > 0");
  if (d->num_bits != 2 && d->num_bits != 4 && d->num_bits != 8 && d->num_bits != 16)
    return fail(BDK_UNSUPPORTED_BITS, "num_bits must be one of 2, 4, 8, 16");
  if (d->k_axis > 1) return fail(BDK_CONFIG_ERROR, "k_axis must be 0 (KChannel) or 1 (KToken)");
  const uint32_t pack = 16 / d->num_bits;
  const uint32_t n_r = 8 * d->warp_n * pack;
  if (d->num_bits != 16) {
    if (d->group_size == 0 || d->head_dim % d->group_size != 0)
      return fail(BDK_CONFIG_ERROR, "group_size must divide head_dim (token-wise V groups)");
    if (d->k_axis == 0 && n_r % d->group_size != 0)
      return fail(BDK_CONFIG_ERROR, "channel-wise group_size must divide N_r");
  }
  Geom G{};
  G.batch = d->batch;
  G.heads_kv = d->heads_kv;
  G.d = d->head_dim;
  G.warp_n = d->warp_n;
  G.bits = d->num_bits;
  G.k_axis = d->k_axis;
  G.g = d->num_bits == 16 ? 1 : d->group_size;
  G.interleave = d->interleave ? 1 : 0;
  G.n_r = n_r;
  G.pack = pack;
  G.max_blocks = d->max_tokens / n_r + 1;
  G.wbytes = d->head_dim * 16 * d->warp_n;
  const uint32_t kp = param_u16(n_r, d->head_dim, d->num_bits, d->k_axis, G.g);
  const uint32_t vp = param_u16(n_r, d->head_dim, d->num_bits, 1, G.g);
  G.kp_bytes = 2 * kp;
  G.vp_bytes = 2 * vp;
  G.rec_bytes = ((2 * G.wbytes + G.kp_bytes + G.vp_bytes) + 127) / 128 * 128;
  // any geometry the reference accepts can be stored, prefilled, flushed,
  // read back and serialized; only decode needs the attention kernels'
  // envelope (checked in check_decode).  The chunk swizzle needs a
  // power-of-two warp_n.
  if (d->warp_n & (d->warp_n - 1))
    return fail(BDK_UNSUPPORTED, "warp_n must be a power of two (chunk swizzle)");

  bdk_cache* c = new bdk_cache();
  c->desc = *d;
  c->device = d->device;
  c->kp_u16 = kp;
  c->vp_u16 = vp;
  c->wpb = d->head_dim * 8 * d->warp_n;
  c->dev.G = G;
  const size_t cells = (size_t)d->batch * d->heads_kv;
  c->packed_blocks.assign(cells, 0);
  c->res_len.assign(cells, 0);
  DevGuard dev_guard_(d->device);
  int n_dev = 0;
  cudaError_t e = cudaGetDeviceCount(&n_dev);
  if (e == cudaSuccess && (d->device < 0 || d->device >= n_dev)) e = cudaErrorInvalidDevice;
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, d->device);
  if (e == cudaSuccess)
    e = cudaMalloc(&c->dev.records, cells * G.max_blocks * (size_t)G.rec_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->dev.res_k, cells * n_r * d->head_dim * 2);
  if (e == cudaSuccess) e = cudaMalloc(&c->dev.res_v, cells * n_r * d->head_dim * 2);
  if (e == cudaSuccess) e = cudaMalloc(&c->dev.len2, 4 * cells * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->dev.len2, 0, 4 * cells * sizeof(int));
  point_lengths(c);
  if (e != cudaSuccess) {
    bdk_cache_destroy(c);
    return cuda_fail(e, "bdk_cache_create");
  }
  *out = c;
  return BDK_OK;
}

bdk_status bdk_cache_destroy(bdk_cache* c) {
  if (!c) return BDK_OK;
  DevGuard dev_guard_(c->device);
  cudaFree(c->dev.records);
  cudaFree(c->dev.res_k);
  cudaFree(c->dev.res_v);
  cudaFree(c->dev.len2);
  cudaFree(c->unit_off);
  cudaFree(c->part_o);
  cudaFree(c->part_ml);
  cudaFree(c->span_parts);
  cudaFree(c->slots);
  cudaFree(c->done);
  for (auto& ev : c->events) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  if (c->h_stage) cudaFreeHost(c->h_stage);
  cudaFree(c->d_stage);
  delete c;
  return BDK_OK;
}

bdk_status bdk_cache_get_info(const bdk_cache* c, bdk_cache_info* info) {
  if (!c || !info) return fail(BDK_INVALID_ARGUMENT, "null argument");
  info->n_r = c->dev.G.n_r;
  info->pack_num = c->dev.G.pack;
  info->words_per_block = c->wpb;
  info->k_param_u16 = c->kp_u16;
  info->v_param_u16 = c->vp_u16;
  info->record_bytes = c->dev.G.rec_bytes;
  info->max_blocks = c->dev.G.max_blocks;
  info->fast_path = bdk::fast_path_ok(c->dev.G) ? 1 : 0;
  return BDK_OK;
}

bdk_status bdk_cache_lengths(const bdk_cache* c, uint32_t b, uint32_t h, uint32_t* packed_len,
                             uint32_t* res_len) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (packed_len) *packed_len = c->packed_blocks[i] * c->dev.G.n_r;
  if (res_len) *res_len = c->res_len[i];
  return BDK_OK;
}

bdk_status bdk_prefill(bdk_cache* c, uint32_t b, uint32_t h, const void* k, const void* v,
                       uint32_t len, void* stream) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (c->packed_blocks[i] != 0 || c->res_len[i] != 0)
    return fail(BDK_STATE_ERROR, "prefill into a non-empty cell");
  const int nb = static_cast<int>(len / c->dev.G.n_r);
  if (nb > c->dev.G.max_blocks) return fail(BDK_CAPACITY_ERROR, "prefill exceeds max_tokens");
  if (len > 0 && (!k || !v)) return fail(BDK_INVALID_ARGUMENT, "null k/v");
  c->blocks_written = true;  // packed records may change (no PDL prefetch next)
  DevGuard dev_guard_(c->device);
  c->launches += 1;
  BDK_CUDA(bdk::launch_prefill(c->dev, static_cast<const __half*>(k),
                               static_cast<const __half*>(v), static_cast<int>(len), i, 1,
                               as_stream(stream)),
           "prefill launch");
  c->packed_blocks[i] = nb;
  c->res_len[i] = static_cast<int>(len % c->dev.G.n_r);
  return BDK_OK;
}

bdk_status bdk_cache_reset(bdk_cache* c, void* stream) {
  if (!c) return fail(BDK_INVALID_ARGUMENT, "null cache");
  const size_t cells = c->res_len.size();
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaMemsetAsync(c->dev.packed_blocks, 0, cells * sizeof(int), as_stream(stream)),
           "reset packed_blocks");
  BDK_CUDA(cudaMemsetAsync(c->dev.res_len, 0, cells * sizeof(int), as_stream(stream)),
           "reset res_len");
  std::fill(c->packed_blocks.begin(), c->packed_blocks.end(), 0);
  std::fill(c->res_len.begin(), c->res_len.end(), 0);
  c->blocks_written = true;
  return BDK_OK;
}

bdk_status bdk_prefill_all(bdk_cache* c, const void* k, const void* v, uint32_t len,
                           void* stream) {
  if (!c) return fail(BDK_INVALID_ARGUMENT, "null cache");
  for (size_t i = 0; i < c->res_len.size(); ++i)
    if (c->packed_blocks[i] != 0 || c->res_len[i] != 0)
      return fail(BDK_STATE_ERROR, "prefill into a non-empty cell");
  const int nb = static_cast<int>(len / c->dev.G.n_r);
  if (nb > c->dev.G.max_blocks) return fail(BDK_CAPACITY_ERROR, "prefill exceeds max_tokens");
  c->blocks_written = true;  // packed records may change (no PDL prefetch next)
  const int cells = static_cast<int>(c->res_len.size());
  DevGuard dev_guard_(c->device);
  c->launches += 1;
  BDK_CUDA(bdk::launch_prefill(c->dev, static_cast<const __half*>(k),
                               static_cast<const __half*>(v), static_cast<int>(len), 0, cells,
                               as_stream(stream)),
           "prefill launch");
  for (int i = 0; i < cells; ++i) {
    c->packed_blocks[i] = nb;
    c->res_len[i] = static_cast<int>(len % c->dev.G.n_r);
  }
  return BDK_OK;
}

bdk_status bdk_append_token(bdk_cache* c, uint32_t b, uint32_t h, const void* k, const void* v,
                            void* stream) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  c->blocks_written = true;  // packed records may change (no PDL prefetch next)
  if (c->res_len[i] == c->dev.G.n_r)
    return fail(BDK_CAPACITY_ERROR, "residual is full; flush before appending");
  DevGuard dev_guard_(c->device);
  c->launches += 1;
  BDK_CUDA(bdk::launch_append(c->dev, i, static_cast<const __half*>(k),
                              static_cast<const __half*>(v), as_stream(stream)),
           "append launch");
  c->res_len[i] += 1;
  return BDK_OK;
}

bdk_status bdk_flush_residual(bdk_cache* c, uint32_t b, uint32_t h, void* stream) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (c->res_len[i] != c->dev.G.n_r)
    return fail(BDK_STATE_ERROR, "flush_residual requires res_len == N_r, have " +
                                     std::to_string(c->res_len[i]));
  if (c->packed_blocks[i] >= c->dev.G.max_blocks)
    return fail(BDK_CAPACITY_ERROR, "cache arena full (raise max_tokens)");
  DevGuard dev_guard_(c->device);
  c->launches += 1;
  BDK_CUDA(bdk::launch_flush(c->dev, i, as_stream(stream)), "flush launch");
  c->blocks_written = true;
  c->packed_blocks[i] += 1;
  c->res_len[i] = 0;
  return BDK_OK;
}

bdk_status bdk_decode_step(bdk_cache* c, const bdk_attn_config* cfg, const void* q,
                           const void* k_new, const void* v_new, float* out, void* stream) {
  bdk_status s = check_decode(c, cfg, true);
  if (s) return s;
  if (!q || !k_new || !v_new || !out) return fail(BDK_INVALID_ARGUMENT, "null tensor");
  return run_decode(c, cfg, q, k_new, v_new, out, nullptr, 0, 1 << 30, as_stream(stream));
}

bdk_status bdk_decode_partial(bdk_cache* c, const bdk_attn_config* cfg, const void* q,
                              const void* k_new, const void* v_new, uint32_t blk_begin,
                              uint32_t blk_end, uint32_t flags, float* out, float* lse,
                              void* stream) {
  const bool appends = k_new != nullptr;
  bdk_status s = check_decode(c, cfg, appends);
  if (s) return s;
  if (!q || !out || !lse || (appends && !v_new))
    return fail(BDK_INVALID_ARGUMENT, "null tensor");
  const bool no_res = (flags & BDK_PARTIAL_NO_RESIDUAL) != 0;
  if (no_res && appends)
    return fail(BDK_STATE_ERROR, "decode_partial: an append needs the residual window");
  return run_decode(c, cfg, q, k_new, v_new, out, lse, static_cast<int>(blk_begin),
                    static_cast<int>(std::min<uint32_t>(blk_end, 1u << 30)), as_stream(stream),
                    no_res);
}

struct bdk_graph {
  bdk_cache* cache = nullptr;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // by the parity of the first step
  uint32_t n_steps = 0;
};

bdk_status bdk_graph_create(bdk_cache* c, const bdk_attn_config* cfg, const void* q,
                            const void* k_new, const void* v_new, float* out, uint32_t n_steps,
                            bdk_graph** graph) {
  if (!graph) return fail(BDK_INVALID_ARGUMENT, "null graph");
  *graph = nullptr;
  bdk_status s = check_decode(c, cfg, true);
  if (s) return s;
  if (!q || !k_new || !v_new || !out) return fail(BDK_INVALID_ARGUMENT, "null tensor");
  if (n_steps == 0) return fail(BDK_INVALID_ARGUMENT, "n_steps must be > 0");
  if (c->profiling) return fail(BDK_STATE_ERROR, "graph capture while profiling");
  const int ng = static_cast<int>(cfg->heads_q / cfg->heads_kv);
  if (c->precise || !exact_ok(c, cfg) || !bdk::fast_decode_ok(c->dev.G, ng))
    return fail(BDK_UNSUPPORTED, "graph capture needs the fast decode path (set_precise(0))");
  DevGuard dev_guard_(c->device);
  cudaStream_t st = nullptr;
  BDK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
  // the workspaces a step uses exist before capture (allocations do not
  // belong in a graph): one attend-only launch sizes them
  s = run_decode_fast(c, cfg, q, nullptr, nullptr, out, nullptr, 0, 1 << 30, st, false);
  if (s == BDK_OK && cudaStreamSynchronize(st) != cudaSuccess)
    s = cuda_fail(cudaGetLastError(), "graph warm-up");
  // two captures, one per parity of the first step (node i reads the len2
  // half (p + i) & 1).  The host mirror advances as the steps are recorded
  // (capacity checks run per step) and is restored afterwards -- the steps
  // happen when the graph is launched
  const auto pb0 = c->packed_blocks, rl0 = c->res_len;
  const uint64_t steps0 = c->fast_steps, launches0 = c->launches;
  const size_t nq = (size_t)cfg->batch * cfg->heads_q * cfg->head_dim;
  const size_t nk = (size_t)cfg->batch * cfg->heads_kv * cfg->head_dim;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  for (int pass = 0; pass < 2 && s == BDK_OK; ++pass) {
    c->packed_blocks = pb0;
    c->res_len = rl0;
    c->fast_steps = steps0 + pass;
    point_lengths(c);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaStreamBeginCapture");
    for (uint32_t i = 0; s == BDK_OK && i < n_steps; ++i) {
      s = check_decode(c, cfg, true);
      if (s == BDK_OK)
        s = run_decode_fast(c, cfg, static_cast<const __half*>(q) + i * nq,
                            static_cast<const __half*>(k_new) + i * nk,
                            static_cast<const __half*>(v_new) + i * nk, out + i * nq, nullptr, 0,
                            1 << 30, st, false, /*dev_sched=*/true);
    }
    if (e == cudaSuccess) {
      const cudaError_t e2 = cudaStreamEndCapture(st, &g);
      if (s == BDK_OK && e2 != cudaSuccess) s = cuda_fail(e2, "cudaStreamEndCapture");
    }
    if (s == BDK_OK) {
      e = cudaGraphInstantiate(&exec[(steps0 + pass) & 1], g, 0);
      if (e != cudaSuccess) s = cuda_fail(e, "cudaGraphInstantiate");
    }
    if (g) cudaGraphDestroy(g);
  }
  c->packed_blocks = pb0;
  c->res_len = rl0;
  c->fast_steps = steps0;
  c->launches = launches0;
  c->blocks_written = true;
  point_lengths(c);
  cudaStreamDestroy(st);
  if (s) {
    for (auto& x : exec)
      if (x) cudaGraphExecDestroy(x);
    return s;
  }
  auto* gr = new bdk_graph;
  gr->cache = c;
  gr->exec[0] = exec[0];
  gr->exec[1] = exec[1];
  gr->n_steps = n_steps;
  c->graphs += 1;
  *graph = gr;
  return BDK_OK;
}

bdk_status bdk_graph_launch(bdk_graph* gr, void* stream) {
  if (!gr || !gr->exec[0] || !gr->exec[1]) return fail(BDK_INVALID_ARGUMENT, "null graph");
  bdk_cache* c = gr->cache;
  // capacity of the n_steps appends, on a copy of the mirror
  {
    auto pb = c->packed_blocks;
    auto rl = c->res_len;
    const int n_r = c->dev.G.n_r;
    for (uint32_t i = 0; i < gr->n_steps; ++i)
      for (size_t k = 0; k < rl.size(); ++k) {
        if (rl[k] + 1 == n_r && pb[k] >= c->dev.G.max_blocks)
          return fail(BDK_CAPACITY_ERROR, "cache arena full (raise max_tokens)");
        if (++rl[k] == n_r) {
          rl[k] = 0;
          pb[k] += 1;
        }
      }
  }
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaGraphLaunch(gr->exec[c->fast_steps & 1], as_stream(stream)), "cudaGraphLaunch");
  for (uint32_t i = 0; i < gr->n_steps; ++i) advance_fast_step(c, true);
  c->launches += 2 * (uint64_t)gr->n_steps;
  return BDK_OK;
}

bdk_status bdk_graph_destroy(bdk_graph* gr) {
  if (!gr) return BDK_OK;
  DevGuard dev_guard_(gr->cache->device);
  for (auto& x : gr->exec)
    if (x) cudaGraphExecDestroy(x);
  gr->cache->graphs -= 1;
  delete gr;
  return BDK_OK;
}

bdk_status bdk_merge_partials(const float* o, const float* lse, uint32_t n_parts, uint32_t rows,
                              uint32_t d, uint64_t o_stride, uint64_t lse_stride, float* out,
                              void* stream) {
  if (n_parts == 0) return fail(BDK_EMPTY_INPUT, "combine: no partial outputs");
  if (!o || !lse || !out) return fail(BDK_INVALID_ARGUMENT, "null tensor");
  if (o_stride < (uint64_t)rows * d || lse_stride < rows)
    return fail(BDK_SHAPE_ERROR, "merge_partials: part stride smaller than a part");
  BDK_CUDA(bdk::launch_merge_partials(o, lse, static_cast<int>(n_parts), static_cast<int>(rows),
                                      static_cast<int>(d), o_stride, lse_stride, out,
                                      as_stream(stream)),
           "merge launch");
  return BDK_OK;
}

// ------------------------------------------------- attention internals
// attend_tile / partitioned_rowmax / residual_attend / packed_attend /
// combine (attention.hpp:17-70) on the device (bdk_span.cu): host buffers in
// and out, synchronous.  Same validation and error classes as the reference.
namespace {
struct DevF {  // scoped device float buffer
  float* p = nullptr;
  ~DevF() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(float)); }
};

bdk_status span_fits(uint32_t rows, uint32_t d, uint32_t tile) {
  if (bdk::span_smem_bytes(rows, d, tile) > kSpanSmemMax)
    return fail(BDK_UNSUPPORTED, "rows * (d + tile) exceeds shared memory");
  return BDK_OK;
}

// state [rows*d o | rows m | rows l] <-> the three host arrays
bdk_status put_state(float* dst, const float* o, const float* m, const float* l, size_t rows,
                     size_t d) {
  BDK_CUDA(cudaMemcpy(dst, o, rows * d * 4, cudaMemcpyHostToDevice), "H2D state");
  BDK_CUDA(cudaMemcpy(dst + rows * d, m, rows * 4, cudaMemcpyHostToDevice), "H2D state");
  BDK_CUDA(cudaMemcpy(dst + rows * d + rows, l, rows * 4, cudaMemcpyHostToDevice), "H2D state");
  return BDK_OK;
}
bdk_status get_state(const float* src, float* o, float* m, float* l, size_t rows, size_t d) {
  BDK_CUDA(cudaMemcpy(o, src, rows * d * 4, cudaMemcpyDeviceToHost), "D2H state");
  BDK_CUDA(cudaMemcpy(m, src + rows * d, rows * 4, cudaMemcpyDeviceToHost), "D2H state");
  BDK_CUDA(cudaMemcpy(l, src + rows * d + rows, rows * 4, cudaMemcpyDeviceToHost), "D2H state");
  return BDK_OK;
}
}  // namespace

bdk_status bdk_attend_tile_host(float* o, float* m, float* l, uint32_t rows, uint32_t d,
                                const float* q, const float* k, const float* v, uint32_t tile_n,
                                float scale, uint32_t warp_n, int32_t device) {
  if (!o || !m || !l || !q || (tile_n && (!k || !v)))
    return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (rows == 0 || d == 0 || tile_n == 0) return BDK_OK;
  bdk_status s = span_fits(rows, d, tile_n);
  if (s) return s;
  DevGuard dev_guard_(device);
  DevF bq, bk, bv, bs;
  BDK_CUDA(bq.alloc((size_t)rows * d), "cudaMalloc");
  BDK_CUDA(bk.alloc((size_t)tile_n * d), "cudaMalloc");
  BDK_CUDA(bv.alloc((size_t)tile_n * d), "cudaMalloc");
  BDK_CUDA(bs.alloc((size_t)rows * (d + 2)), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bq.p, q, (size_t)rows * d * 4, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(cudaMemcpy(bk.p, k, (size_t)tile_n * d * 4, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(cudaMemcpy(bv.p, v, (size_t)tile_n * d * 4, cudaMemcpyHostToDevice), "H2D");
  if ((s = put_state(bs.p, o, m, l, rows, d))) return s;
  bdk::SpanArgs a;
  a.source = bdk::kSpanFp32;
  a.k32 = bk.p;
  a.v32 = bv.p;
  a.len32 = static_cast<int>(tile_n);
  a.q32 = bq.p;
  a.scale = scale;
  a.rows = static_cast<int>(rows);
  a.d = static_cast<int>(d);
  a.residual = 0;
  a.tile_n = static_cast<int>(tile_n);
  a.warp_n = static_cast<int>(warp_n);
  a.keep_state = 1;
  a.parts = bs.p;
  a.n_parts = 1;
  BDK_CUDA(bdk::launch_span_parts(a, 1, nullptr), "attend_tile launch");
  return get_state(bs.p, o, m, l, rows, d);
}

bdk_status bdk_partitioned_rowmax_host(const float* sc, uint32_t rows, uint32_t cols,
                                       uint32_t warp_n, float* out, int32_t device) {
  if (warp_n == 0 || cols % warp_n != 0)
    return fail(BDK_SHAPE_ERROR,
                "partitioned_rowmax: cols must divide evenly across warp_n partitions");
  if (!sc || !out) return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (rows == 0) return BDK_OK;
  DevGuard dev_guard_(device);
  DevF bs, bo;
  BDK_CUDA(bs.alloc((size_t)rows * cols), "cudaMalloc");
  BDK_CUDA(bo.alloc(rows), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bs.p, sc, (size_t)rows * cols * 4, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(bdk::launch_partitioned_rowmax(bs.p, (int)rows, (int)cols, (int)warp_n, bo.p, nullptr),
           "rowmax launch");
  BDK_CUDA(cudaMemcpy(out, bo.p, rows * 4, cudaMemcpyDeviceToHost), "D2H");
  return BDK_OK;
}

bdk_status bdk_residual_attend_host(const bdk_cache* c, uint32_t b, uint32_t h, const float* q,
                                    uint32_t q_rows, float scale, float* o, float* m, float* l) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  if (!q || !o || !m || !l) return fail(BDK_INVALID_ARGUMENT, "null argument");
  const int i = cell_of(c, b, h);
  if (c->res_len[i] == 0) return fail(BDK_STATE_ERROR, "residual_attend: residual cache is empty");
  if (q_rows == 0) return BDK_OK;
  const uint32_t d = c->desc.head_dim;
  if ((s = span_fits(q_rows, d, c->dev.G.n_r))) return s;
  DevGuard dev_guard_(c->device);
  DevF bq, bs;
  BDK_CUDA(bq.alloc((size_t)q_rows * d), "cudaMalloc");
  BDK_CUDA(bs.alloc((size_t)q_rows * (d + 2)), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bq.p, q, (size_t)q_rows * d * 4, cudaMemcpyHostToDevice), "H2D");
  if ((s = put_state(bs.p, o, m, l, q_rows, d))) return s;
  bdk::SpanArgs a;
  a.c = c->dev;
  a.q32 = bq.p;
  a.scale = scale;
  a.rows = static_cast<int>(q_rows);
  a.d = static_cast<int>(d);
  a.cell0 = i;
  a.residual = 1;
  a.splits = 0;
  a.tile_n = c->dev.G.n_r;
  a.keep_state = 1;
  a.parts = bs.p;
  a.n_parts = 1;
  c->launches += 1;
  BDK_CUDA(bdk::launch_span_parts(a, 1, nullptr), "residual_attend launch");
  return get_state(bs.p, o, m, l, q_rows, d);
}

bdk_status bdk_packed_attend_host(const bdk_cache* c, uint32_t b, uint32_t h, const float* q,
                                  uint32_t q_rows, uint32_t tile_n, uint32_t num_splits,
                                  float scale, float* o, float* m, float* l, uint32_t* n_parts) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  if (!q || !o || !m || !l || !n_parts) return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (tile_n == 0) return fail(BDK_SHAPE_ERROR, "packed_attend: tile_n must be > 0");
  *n_parts = 0;
  const int i = cell_of(c, b, h);
  const uint64_t plen = (uint64_t)c->packed_blocks[i] * c->dev.G.n_r;
  if (plen == 0 || q_rows == 0) return BDK_OK;
  const uint32_t d = c->desc.head_dim;
  if ((s = span_fits(q_rows, d, std::max<uint32_t>(tile_n, c->dev.G.n_r)))) return s;
  // splits past the tile count are empty (attention.cpp:124-130) and omitted
  const uint64_t n_tiles = (plen + tile_n - 1) / tile_n;
  const uint32_t splits = (uint32_t)std::min<uint64_t>(std::max<uint32_t>(1, num_splits), n_tiles);
  DevGuard dev_guard_(c->device);
  DevF bq, bs;
  const size_t stride = (size_t)q_rows * (d + 2);
  BDK_CUDA(bq.alloc((size_t)q_rows * d), "cudaMalloc");
  BDK_CUDA(bs.alloc(stride * splits), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bq.p, q, (size_t)q_rows * d * 4, cudaMemcpyHostToDevice), "H2D");
  bdk::SpanArgs a;
  a.c = c->dev;
  a.q32 = bq.p;
  a.scale = scale;
  a.rows = static_cast<int>(q_rows);
  a.d = static_cast<int>(d);
  a.cell0 = i;
  a.residual = 0;
  a.tile_n = static_cast<int>(tile_n);
  a.splits = static_cast<int>(splits);
  a.parts = bs.p;
  a.n_parts = static_cast<int>(splits);
  c->launches += 1;
  BDK_CUDA(bdk::launch_span_parts(a, 1, nullptr), "packed_attend launch");
  for (uint32_t p = 0; p < splits; ++p)
    if ((s = get_state(bs.p + p * stride, o + (size_t)p * q_rows * d, m + (size_t)p * q_rows,
                       l + (size_t)p * q_rows, q_rows, d)))
      return s;
  *n_parts = splits;
  return BDK_OK;
}

bdk_status bdk_combine_host(const float* o, const float* m, const float* l, uint32_t n_parts,
                            uint32_t rows, uint32_t d, float* out, int32_t device) {
  if (n_parts == 0) return fail(BDK_EMPTY_INPUT, "combine: no partial outputs");
  if (!o || !m || !l || !out) return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (rows == 0 || d == 0) return BDK_OK;
  DevGuard dev_guard_(device);
  const size_t stride = (size_t)rows * (d + 2);
  DevF bs, bo;
  BDK_CUDA(bs.alloc(stride * n_parts), "cudaMalloc");
  BDK_CUDA(bo.alloc((size_t)rows * d), "cudaMalloc");
  for (uint32_t p = 0; p < n_parts; ++p) {
    bdk_status s = put_state(bs.p + p * stride, o + (size_t)p * rows * d, m + (size_t)p * rows,
                             l + (size_t)p * rows, rows, d);
    if (s) return s;
  }
  BDK_CUDA(bdk::launch_span_combine(bs.p, 1, (int)n_parts, (int)rows, (int)d, 1, (int)rows, bo.p,
                                    nullptr, nullptr, nullptr),
           "combine launch");
  BDK_CUDA(cudaMemcpy(out, bo.p, (size_t)rows * d * 4, cudaMemcpyDeviceToHost), "D2H");
  return BDK_OK;
}

bdk_status bdk_peer_merge(const float* const* parts, uint32_t* const* flags, uint32_t world,
                          uint32_t rank, uint64_t step, uint32_t rows, uint32_t d, float* out,
                          float* out_lse, int* err, uint64_t timeout_ns, void* stream) {
  if (world == 0 || world > (uint32_t)bdk::kMaxPeers)
    return fail(BDK_CONFIG_ERROR, "peer_merge: world must be 1..8");
  if (rank >= world) return fail(BDK_CONFIG_ERROR, "peer_merge: rank out of range");
  if (!parts || !flags || !out || !err) return fail(BDK_INVALID_ARGUMENT, "null argument");
  bdk::PeerMergeArgs a;
  for (uint32_t p = 0; p < world; ++p) {
    if (!parts[p] || !flags[p]) return fail(BDK_INVALID_ARGUMENT, "null peer pointer");
    a.parts[p] = parts[p];
    a.flags[p] = flags[p];
  }
  a.world = (int)world;
  a.rank = (int)rank;
  a.step = (long long)step;
  a.rows = (int)rows;
  a.d = (int)d;
  a.out = out;
  a.out_lse = out_lse;
  a.err = err;
  a.timeout_ns = timeout_ns ? timeout_ns : 2000000000ull;
  BDK_CUDA(bdk::launch_peer_merge(a, as_stream(stream)), "peer merge launch");
  return BDK_OK;
}

bdk_status bdk_set_precise(bdk_cache* c, int precise) {
  if (!c) return fail(BDK_INVALID_ARGUMENT, "null cache");
  c->precise = precise ? 1 : 0;
  return BDK_OK;
}

// host fp32 tensors -> fp16 into the pinned staging buffer (values are
// binary16-representable, so RNE narrowing is exact; fp16.hpp:13-70).  F16C
// converts 8 lanes per instruction; the scalar loop covers CPUs without it
// and the tail.
namespace {
__attribute__((target("avx,f16c"))) void f32_to_f16_f16c(const float* in, uint16_t* out,
                                                          size_t n) {
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const __m256 x = _mm256_loadu_ps(in + i);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(out + i),
                     _mm256_cvtps_ph(x, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC));
  }
  for (; i < n; ++i) out[i] = static_cast<uint16_t>(_cvtss_sh(in[i], _MM_FROUND_TO_NEAREST_INT));
}

void f32_to_f16_serial(const float* in, uint16_t* out, size_t n) {
  static const bool f16c = __builtin_cpu_supports("f16c") && __builtin_cpu_supports("avx");
  if (f16c) {
    f32_to_f16_f16c(in, out, n);
    return;
  }
  for (size_t i = 0; i < n; ++i) {
    const __half h = __float2half_rn(in[i]);
    std::memcpy(out + i, &h, 2);
  }
}

// large host tensors (e.g. b32 MHA: 1.5 MB of fp32 inputs per step) are
// converted / copied by several host threads: a single core's memory
// bandwidth would otherwise dominate the host-API step
constexpr size_t kParallelHost = size_t(1) << 14;  // elements (back-to-back calls keep the pool warm)
constexpr int kHostThreads = 8;

void f32_to_f16_host(const float* in, uint16_t* out, size_t n) {
  if (n < kParallelHost) {
    f32_to_f16_serial(in, out, n);
    return;
  }
  const size_t chunk = (n / kHostThreads + 7) & ~size_t(7);
#pragma omp parallel for num_threads(kHostThreads) schedule(static)
  for (int t = 0; t < kHostThreads; ++t) {
    const size_t lo = std::min(n, (size_t)t * chunk), hi = std::min(n, lo + chunk);
    if (hi > lo) f32_to_f16_serial(in + lo, out + lo, hi - lo);
  }
}

// q, k_new, v_new -> one contiguous fp16 staging run [q | k | v], one
// parallel region for the three
void f32_to_f16_host3(const float* q, size_t nq, const float* k, const float* v, size_t nk,
                      uint16_t* out) {
  const size_t n = nq + 2 * nk;
  auto src = [&](size_t i, size_t& len) -> const float* {  // run containing element i
    if (i < nq) return len = nq - i, q + i;
    if (i < nq + nk) return len = nq + nk - i, k + (i - nq);
    return len = n - i, v + (i - nq - nk);
  };
  auto convert = [&](size_t lo, size_t hi) {
    while (lo < hi) {
      size_t len;
      const float* p = src(lo, len);
      len = std::min(len, hi - lo);
      f32_to_f16_serial(p, out + lo, len);
      lo += len;
    }
  };
  if (n < kParallelHost) {
    convert(0, n);
    return;
  }
  const size_t chunk = (n / kHostThreads + 7) & ~size_t(7);
#pragma omp parallel for num_threads(kHostThreads) schedule(static)
  for (int t = 0; t < kHostThreads; ++t) {
    const size_t lo = std::min(n, (size_t)t * chunk), hi = std::min(n, lo + chunk);
    convert(lo, hi);
  }
}

void copy_host(float* dst, const float* src, size_t n) {
  if (n < kParallelHost) {
    std::memcpy(dst, src, n * 4);
    return;
  }
  const size_t chunk = (n / kHostThreads + 15) & ~size_t(15);
#pragma omp parallel for num_threads(kHostThreads) schedule(static)
  for (int t = 0; t < kHostThreads; ++t) {
    const size_t lo = std::min(n, (size_t)t * chunk), hi = std::min(n, lo + chunk);
    if (hi > lo) std::memcpy(dst + lo, src + lo, (hi - lo) * 4);
  }
}
}  // namespace

// Host-tensor decode_step: the step's inputs go host fp32 -> pinned fp16
// (F16C) -> one H2D copy; for small outputs the decode kernel writes its fp32
// output straight into the pinned staging buffer (mapped, UVA), so the only
// device round trip after the kernel is the stream synchronization.
bdk_status bdk_decode_step_host(bdk_cache* c, const bdk_attn_config* cfg, const float* q,
                                const float* k_new, const float* v_new, float* out) {
  bdk_status s = check_decode(c, cfg, true);
  if (s) return s;
  if (!q || !k_new || !v_new || !out) return fail(BDK_INVALID_ARGUMENT, "null tensor");
  const size_t d = cfg->head_dim;
  const size_t nq = (size_t)cfg->batch * cfg->heads_q * d;
  const size_t nk = (size_t)cfg->batch * cfg->heads_kv * d;
  const size_t n_in = nq + 2 * nk;
  // staging layout (host and device alike): fp16 [q | k | v], fp32 out (128-B aligned)
  const size_t out_off = (n_in * 2 + 127) & ~size_t(127);
  const size_t bytes = out_off + nq * 4;
  DevGuard dev_guard_(c->device);
  s = ensure_stage(c, bytes);
  if (s) return s;
  uint16_t* hin = static_cast<uint16_t*>(c->h_stage);
  f32_to_f16_host3(q, nq, k_new, v_new, nk, hin);
  __half* dh = static_cast<__half*>(c->d_stage);
  float* hout = reinterpret_cast<float*>(static_cast<uint8_t*>(c->h_stage) + out_off);
  // small outputs (<= 256 KiB) are stored by the kernel over PCIe into the
  // pinned buffer (saves the D2H copy's latency); larger ones (e.g. b32 MHA,
  // 512 KiB) go through HBM and one D2H copy, which streams faster
  static const int zc_env = getenv("BDK_E2E_ZC") ? atoi(getenv("BDK_E2E_ZC")) : -1;
  const bool zc = zc_env >= 0 ? zc_env != 0 : nq * 4 <= (256u << 10);
  float* dout = zc ? hout : reinterpret_cast<float*>(static_cast<uint8_t*>(c->d_stage) + out_off);
  cudaStream_t st = 0;
  // small inputs cross PCIe in a kernel the decode kernel overlaps its start
  // with (C5: +8% e2e); large ones stream faster on the copy engine (C3).
  // Staging buffers are padded past n_in, so the 16-byte round-up stays inside.
  if (n_in * 2 <= (256u << 10)) {
    BDK_CUDA(bdk::launch_stage_in(hin, dh, n_in * 2, st), "H2D stage-in");
    c->launches += 1;
  } else {
    BDK_CUDA(cudaMemcpyAsync(dh, hin, n_in * 2, cudaMemcpyHostToDevice, st), "H2D");
  }
  s = run_decode(c, cfg, dh, dh + nq, dh + nq + nk, dout, nullptr, 0, 1 << 30, st);
  if (s) return s;
  if (!zc) BDK_CUDA(cudaMemcpyAsync(hout, dout, nq * 4, cudaMemcpyDeviceToHost, st), "D2H");
  BDK_CUDA(cudaStreamSynchronize(st), "decode_step_host");
  copy_host(out, hout, nq);
  return BDK_OK;
}

bdk_status bdk_prefill_host(bdk_cache* c, uint32_t b, uint32_t h, const uint16_t* k,
                            const uint16_t* v, uint32_t len) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  if (len > 0 && (!k || !v)) return fail(BDK_INVALID_ARGUMENT, "null k/v");
  const size_t n = (size_t)len * c->desc.head_dim;
  DevGuard dev_guard_(c->device);
  void* d = nullptr;
  if (n) {
    BDK_CUDA(cudaMalloc(&d, 2 * n * 2), "cudaMalloc(prefill staging)");
    cudaError_t e = cudaMemcpy(d, k, n * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(static_cast<uint16_t*>(d) + n, v, n * 2, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(d);
      return cuda_fail(e, "H2D prefill");
    }
  }
  s = bdk_prefill(c, b, h, d, n ? static_cast<uint16_t*>(d) + n : nullptr, len, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(d);
  if (s) return s;
  if (e != cudaSuccess) return cuda_fail(e, "prefill");
  return BDK_OK;
}

bdk_status bdk_append_token_host(bdk_cache* c, uint32_t b, uint32_t h, const uint16_t* k,
                                 const uint16_t* v) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  if (!k || !v) return fail(BDK_INVALID_ARGUMENT, "null k/v row");
  const size_t d = c->desc.head_dim;
  DevGuard dev_guard_(c->device);
  s = ensure_stage(c, 4 * d + 256);
  if (s) return s;
  uint16_t* dk = static_cast<uint16_t*>(c->d_stage);
  BDK_CUDA(cudaMemcpy(dk, k, d * 2, cudaMemcpyHostToDevice), "H2D row");
  BDK_CUDA(cudaMemcpy(dk + d, v, d * 2, cudaMemcpyHostToDevice), "H2D row");
  s = bdk_append_token(c, b, h, dk, dk + d, nullptr);
  if (s) return s;
  BDK_CUDA(cudaDeviceSynchronize(), "append");
  return BDK_OK;
}

bdk_status bdk_packed_tile_host(const bdk_cache* c, uint32_t b, uint32_t h, uint32_t t0,
                                uint32_t len, uint16_t* k_out, uint16_t* v_out) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  const uint32_t n_r = c->dev.G.n_r;
  if ((uint64_t)t0 + len > (uint64_t)c->packed_blocks[i] * n_r)
    return fail(BDK_SHAPE_ERROR, "packed_tile: range past packed segment");
  if (len == 0) return BDK_OK;
  if (!k_out || !v_out) return fail(BDK_INVALID_ARGUMENT, "null output");
  const uint32_t blk0 = t0 / n_r, blk1 = (t0 + len + n_r - 1) / n_r, nb = blk1 - blk0;
  const size_t d = c->desc.head_dim, rows = (size_t)nb * n_r;
  DevGuard dev_guard_(c->device);
  uint16_t* dbuf = nullptr;
  BDK_CUDA(cudaMalloc(&dbuf, 2 * rows * d * 2), "cudaMalloc(dequant)");
  s = bdk_dequant_blocks(c, b, h, blk0, nb, dbuf, dbuf + rows * d, nullptr);
  cudaError_t e = s ? cudaSuccess : cudaDeviceSynchronize();
  const size_t off = (size_t)(t0 - blk0 * n_r) * d;
  if (!s && e == cudaSuccess)
    e = cudaMemcpy(k_out, dbuf + off, (size_t)len * d * 2, cudaMemcpyDeviceToHost);
  if (!s && e == cudaSuccess)
    e = cudaMemcpy(v_out, dbuf + rows * d + off, (size_t)len * d * 2, cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (s) return s;
  if (e != cudaSuccess) return cuda_fail(e, "packed_tile");
  return BDK_OK;
}

// D2H of one block record (cell i, slot blk), un-swizzled into the
// reference's word arrays
static bdk_status read_record(const bdk_cache* c, int i, uint32_t blk, uint16_t* kw,
                              uint16_t* vw, uint16_t* kp, uint16_t* vp) {
  const Geom& G = c->dev.G;
  std::vector<uint8_t> rec(G.rec_bytes);
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaDeviceSynchronize(), "sync");
  BDK_CUDA(cudaMemcpy(rec.data(),
                      c->dev.records + ((size_t)i * G.max_blocks + blk) * G.rec_bytes,
                      G.rec_bytes, cudaMemcpyDeviceToHost),
           "D2H block");
  for (uint32_t w = 0; w < c->wpb; ++w) {  // undo the 16-byte chunk swizzle
    const size_t off = word_offset(G, w);
    if (kw) std::memcpy(kw + w, rec.data() + off, 2);
    if (vw) std::memcpy(vw + w, rec.data() + G.wbytes + off, 2);
  }
  if (kp) std::memcpy(kp, rec.data() + 2 * G.wbytes, G.kp_bytes);
  if (vp) std::memcpy(vp, rec.data() + 2 * G.wbytes + G.kp_bytes, G.vp_bytes);
  return BDK_OK;
}

bdk_status bdk_read_block(const bdk_cache* c, uint32_t b, uint32_t h, uint32_t blk,
                          uint16_t* kw, uint16_t* vw, uint16_t* kp, uint16_t* vp) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (static_cast<int>(blk) >= c->packed_blocks[i])
    return fail(BDK_SHAPE_ERROR, "block index past the packed segment");
  return read_record(c, i, blk, kw, vw, kp, vp);
}

bdk_status bdk_build_block(bdk_cache* c, uint32_t b, uint32_t h, uint16_t* kw, uint16_t* vw,
                           uint16_t* kp, uint16_t* vp) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  c->blocks_written = true;  // packed records may change (no PDL prefetch next)
  if (c->res_len[i] != c->dev.G.n_r)
    return fail(BDK_STATE_ERROR, "build_block requires a full residual (res_len == N_r)");
  if (c->packed_blocks[i] >= c->dev.G.max_blocks)
    return fail(BDK_CAPACITY_ERROR, "cache arena full (raise max_tokens)");
  DevGuard dev_guard_(c->device);
  c->launches += 1;
  BDK_CUDA(bdk::launch_build(c->dev, i, nullptr), "build launch");
  return read_record(c, i, (uint32_t)c->packed_blocks[i], kw, vw, kp, vp);
}

bdk_status bdk_commit_block(bdk_cache* c, uint32_t b, uint32_t h, const uint16_t* kw,
                            const uint16_t* vw, const uint16_t* kp, const uint16_t* vp) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (c->res_len[i] != c->dev.G.n_r)
    return fail(BDK_STATE_ERROR, "commit_block requires a full residual (res_len == N_r)");
  s = bdk_adopt_block(c, b, h, kw, vw, kp, vp);
  if (s) return s;
  const int zero = 0;
  BDK_CUDA(cudaMemcpy(c->dev.res_len + i, &zero, sizeof(int), cudaMemcpyHostToDevice),
           "H2D res_len");
  c->res_len[i] = 0;
  return BDK_OK;
}

bdk_status bdk_adopt_block(bdk_cache* c, uint32_t b, uint32_t h, const uint16_t* kw,
                           const uint16_t* vw, const uint16_t* kp, const uint16_t* vp) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  if (!kw || !vw || ((c->kp_u16 && !kp) || (c->vp_u16 && !vp)))
    return fail(BDK_INVALID_ARGUMENT, "null block field");
  const int i = cell_of(c, b, h);
  const Geom& G = c->dev.G;
  if (c->packed_blocks[i] >= G.max_blocks)
    return fail(BDK_CAPACITY_ERROR, "cache arena full (raise max_tokens)");
  std::vector<uint8_t> rec(G.rec_bytes, 0);
  for (uint32_t w = 0; w < c->wpb; ++w) {
    const size_t off = word_offset(G, w);
    std::memcpy(rec.data() + off, kw + w, 2);
    std::memcpy(rec.data() + G.wbytes + off, vw + w, 2);
  }
  if (G.kp_bytes) std::memcpy(rec.data() + 2 * G.wbytes, kp, G.kp_bytes);
  if (G.vp_bytes) std::memcpy(rec.data() + 2 * G.wbytes + G.kp_bytes, vp, G.vp_bytes);
  const int slot = c->packed_blocks[i];
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaDeviceSynchronize(), "sync");
  BDK_CUDA(cudaMemcpy(c->dev.records + ((size_t)i * G.max_blocks + slot) * G.rec_bytes,
                      rec.data(), G.rec_bytes, cudaMemcpyHostToDevice),
           "H2D block");
  const int nb = slot + 1;
  BDK_CUDA(cudaMemcpy(c->dev.packed_blocks + i, &nb, sizeof(int), cudaMemcpyHostToDevice),
           "H2D length");
  c->packed_blocks[i] = nb;
  c->blocks_written = true;
  return BDK_OK;
}

bdk_status bdk_read_residual(const bdk_cache* c, uint32_t b, uint32_t h, uint16_t* k,
                             uint16_t* v) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  const size_t n = (size_t)c->res_len[i] * c->desc.head_dim;
  const size_t base = (size_t)i * c->dev.G.n_r * c->desc.head_dim;
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaDeviceSynchronize(), "sync");
  if (k && n) BDK_CUDA(cudaMemcpy(k, c->dev.res_k + base, n * 2, cudaMemcpyDeviceToHost), "D2H");
  if (v && n) BDK_CUDA(cudaMemcpy(v, c->dev.res_v + base, n * 2, cudaMemcpyDeviceToHost), "D2H");
  return BDK_OK;
}

bdk_status bdk_dequant_blocks(const bdk_cache* c, uint32_t b, uint32_t h, uint32_t blk0,
                              uint32_t nblk, void* k_out, void* v_out, void* stream) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (static_cast<int>(blk0 + nblk) > c->packed_blocks[i])
    return fail(BDK_SHAPE_ERROR, "packed_tile: range past packed segment");
  DevGuard dev_guard_(c->device);
  c->launches += 1;
  BDK_CUDA(bdk::launch_dequant(c->dev, i, static_cast<int>(blk0), static_cast<int>(nblk),
                               static_cast<__half*>(k_out), static_cast<__half*>(v_out),
                               as_stream(stream)),
           "dequant launch");
  return BDK_OK;
}

bdk_status bdk_memory(const bdk_cache* c, uint64_t out[4]) {
  if (!c || !out) return fail(BDK_INVALID_ARGUMENT, "null argument");
  out[0] = out[1] = out[2] = out[3] = 0;
  for (size_t i = 0; i < c->res_len.size(); ++i) {
    out[0] += (uint64_t)c->packed_blocks[i] * c->wpb * 2;
    out[1] += (uint64_t)c->packed_blocks[i] * c->wpb * 2;
    out[2] += (uint64_t)c->packed_blocks[i] * (c->kp_u16 + c->vp_u16) * 2;
    out[3] += (uint64_t)c->res_len[i] * c->desc.head_dim * 2 * 2;
  }
  return BDK_OK;
}

bdk_status bdk_corrupt_word(bdk_cache* c, uint32_t b, uint32_t h, uint32_t blk, uint32_t word,
                            uint16_t value) {
  bdk_status s = check_cell(c, b, h);
  if (s) return s;
  const int i = cell_of(c, b, h);
  if (static_cast<int>(blk) >= c->packed_blocks[i] || word >= c->wpb)
    return fail(BDK_SHAPE_ERROR, "corrupt_word: index out of range");
  const Geom& G = c->dev.G;
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaDeviceSynchronize(), "sync");
  BDK_CUDA(cudaMemcpy(c->dev.records + ((size_t)i * G.max_blocks + blk) * G.rec_bytes +
                          word_offset(G, word),
                      &value, 2, cudaMemcpyHostToDevice),
           "H2D word");
  c->blocks_written = true;
  return BDK_OK;
}

bdk_status bdk_profile_begin(bdk_cache* c) {
  if (!c) return fail(BDK_INVALID_ARGUMENT, "null cache");
  c->profiling = true;
  c->events_used = 0;
  return BDK_OK;
}

bdk_status bdk_profile_end(bdk_cache* c, float* total_ms, uint32_t* launches) {
  if (!c || !total_ms || !launches) return fail(BDK_INVALID_ARGUMENT, "null argument");
  c->profiling = false;
  DevGuard dev_guard_(c->device);
  float sum = 0.f;
  for (size_t i = 0; i < c->events_used; ++i) {
    BDK_CUDA(cudaEventSynchronize(c->events[i].second), "cudaEventSynchronize");
    float ms = 0.f;
    BDK_CUDA(cudaEventElapsedTime(&ms, c->events[i].first, c->events[i].second),
             "cudaEventElapsedTime");
    sum += ms;
  }
  *total_ms = sum;
  *launches = static_cast<uint32_t>(c->events_used);
  c->events_used = 0;
  return BDK_OK;
}

bdk_status bdk_launch_count(const bdk_cache* c, uint64_t* n) {
  if (!c || !n) return fail(BDK_INVALID_ARGUMENT, "null argument");
  *n = c->launches;
  return BDK_OK;
}

bdk_status bdk_synchronize(void) {
  BDK_CUDA(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  return BDK_OK;
}


// ------------------------------------------------------------- BDKV v1
// The reference's on-disk cache format (serialize.hpp:11-20,
// serialize.cpp:87-194), all integers little-endian:
//   "BDKV" | version u8 (1) | flags u8 (bit0 = interleaved layout)
//   u32 num_bits, k_axis, group_size, N_r, head_dim, batch, heads_kv
//   per cell (batch-major): u32 packed_len, u32 res_len, then the K words of
//   every block, the K params of every block, the V words, the V params
//   (u16 arrays in block order), then res_len*d residual K binary16 bits and
//   the same for V.
// The device records hold the same words (only chunk-swizzled) and the same
// (scale, zero) u16 pairs, so a dump is a per-cell D2H copy plus the
// un-swizzle, and a load the reverse.  FormatError messages carry the byte
// offset like the reference's FormatError::offset.
namespace {

void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

bdk_status format_fail(const std::string& what, uint64_t offset) {
  return fail(BDK_FORMAT_ERROR, what + " (at byte offset " + std::to_string(offset) + ")");
}

struct BdkvReader {
  const uint8_t* p;
  uint64_t n, off = 0;
  bool u8(uint8_t& v) {
    if (off + 1 > n) return false;
    v = p[off++];
    return true;
  }
  bool u32(uint32_t& v) {
    if (off + 4 > n) return false;
    v = (uint32_t)p[off] | (uint32_t)p[off + 1] << 8 | (uint32_t)p[off + 2] << 16 |
        (uint32_t)p[off + 3] << 24;
    off += 4;
    return true;
  }
  bool skip(uint64_t bytes) {
    if (bytes > n - off) return false;
    off += bytes;
    return true;
  }
};

bdk_status serialize(const bdk_cache* c, std::vector<uint8_t>& o) {
  const Geom& G = c->dev.G;
  const uint32_t d = c->desc.head_dim;
  o.clear();
  const char magic[4] = {'B', 'D', 'K', 'V'};
  o.insert(o.end(), magic, magic + 4);
  o.push_back(1);
  o.push_back(c->desc.interleave ? 1 : 0);
  put_u32(o, c->desc.num_bits);
  put_u32(o, c->desc.k_axis);
  put_u32(o, c->desc.group_size);
  put_u32(o, (uint32_t)G.n_r);
  put_u32(o, d);
  put_u32(o, c->desc.batch);
  put_u32(o, c->desc.heads_kv);
  DevGuard dev_guard_(c->device);
  BDK_CUDA(cudaDeviceSynchronize(), "sync");
  std::vector<uint8_t> recs;
  std::vector<uint16_t> res;
  const size_t cells = c->res_len.size();
  for (size_t i = 0; i < cells; ++i) {
    const uint32_t nb = (uint32_t)c->packed_blocks[i], rl = (uint32_t)c->res_len[i];
    put_u32(o, nb * (uint32_t)G.n_r);
    put_u32(o, rl);
    recs.resize((size_t)nb * G.rec_bytes);
    if (nb)
      BDK_CUDA(cudaMemcpy(recs.data(), c->dev.records + (size_t)i * G.max_blocks * G.rec_bytes,
                          recs.size(), cudaMemcpyDeviceToHost),
               "D2H records");
    // K words | K params | V words | V params, each for every block in order
    for (int part = 0; part < 4; ++part) {
      for (uint32_t blk = 0; blk < nb; ++blk) {
        const uint8_t* rec = recs.data() + (size_t)blk * G.rec_bytes;
        if (part == 0 || part == 2) {
          const uint8_t* words = rec + (part == 2 ? G.wbytes : 0);
          for (uint32_t w = 0; w < c->wpb; ++w) {
            const uint8_t* src = words + word_offset(G, w);
            o.push_back(src[0]);
            o.push_back(src[1]);
          }
        } else {
          const uint8_t* prm = rec + 2 * G.wbytes + (part == 3 ? G.kp_bytes : 0);
          const uint32_t nbytes = 2 * (part == 1 ? c->kp_u16 : c->vp_u16);
          o.insert(o.end(), prm, prm + nbytes);
        }
      }
    }
    res.resize((size_t)rl * d);
    for (int t = 0; t < 2; ++t) {
      if (rl)
        BDK_CUDA(cudaMemcpy(res.data(), (t ? c->dev.res_v : c->dev.res_k) + i * (size_t)G.n_r * d,
                            res.size() * 2, cudaMemcpyDeviceToHost),
                 "D2H residual");
      for (uint16_t x : res) {
        o.push_back(static_cast<uint8_t>(x & 0xFF));
        o.push_back(static_cast<uint8_t>(x >> 8));
      }
    }
  }
  return BDK_OK;
}

}  // namespace

bdk_status bdk_dump_cache(const bdk_cache* c, uint8_t* buf, uint64_t capacity, uint64_t* size) {
  if (!c || !size) return fail(BDK_INVALID_ARGUMENT, "null argument");
  std::vector<uint8_t> o;
  bdk_status s = serialize(c, o);
  if (s) return s;
  *size = o.size();
  if (!buf) return BDK_OK;
  if (capacity < o.size())
    return fail(BDK_CAPACITY_ERROR, "dump buffer too small: need " + std::to_string(o.size()));
  std::memcpy(buf, o.data(), o.size());
  return BDK_OK;
}

bdk_status bdk_dump_cache_file(const bdk_cache* c, const char* path) {
  if (!c || !path) return fail(BDK_INVALID_ARGUMENT, "null argument");
  std::vector<uint8_t> o;
  bdk_status s = serialize(c, o);
  if (s) return s;
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(BDK_INVALID_ARGUMENT, std::string("cannot open ") + path + " for writing");
  const bool ok = std::fwrite(o.data(), 1, o.size(), f) == o.size();
  if (std::fclose(f) != 0 || !ok)
    return fail(BDK_INVALID_ARGUMENT, std::string("write to ") + path + " failed");
  return BDK_OK;
}

bdk_status bdk_load_cache(const uint8_t* buf, uint64_t size, uint32_t max_tokens, int32_t device,
                          bdk_cache** out) {
  if (!out || (!buf && size)) return fail(BDK_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  BdkvReader r{buf, size};
  const auto eof = [&]() { return format_fail("unexpected end of file", r.n); };
  if (size < 4) return format_fail("unexpected end of file", size);
  if (std::memcmp(buf, "BDKV", 4) != 0) return format_fail("bad magic", 0);
  r.off = 4;
  uint8_t version = 0, flags = 0;
  if (!r.u8(version)) return eof();
  if (version != 1) return format_fail("unsupported version " + std::to_string(version), 4);
  if (!r.u8(flags)) return eof();
  uint32_t bits, axis, g, n_r, d, batch, heads;
  if (!r.u32(bits)) return eof();
  if (!r.u32(axis)) return eof();
  if (axis > 1) return format_fail("bad quant axis", r.off - 4);
  if (!r.u32(g) || !r.u32(n_r) || !r.u32(d) || !r.u32(batch) || !r.u32(heads)) return eof();
  if (bits == 0 || bits > 16 || n_r == 0 || n_r % (8 * (16 / bits)) != 0)
    return format_fail("N_r inconsistent with num_bits", 10);
  const uint32_t warp_n = n_r / (8 * (16 / bits));
  // pass 1: validate every cell and size the arena
  const uint64_t wpb = (uint64_t)n_r * d * bits / 16;
  const bool pass = bits == 16;
  const uint64_t kp = pass ? 0
                      : 2ull * (axis == 0 ? (uint64_t)(g ? n_r / g : 0) * d
                                          : (uint64_t)n_r * (g ? d / g : 0));
  const uint64_t vp = pass ? 0 : 2ull * n_r * (g ? d / g : 0);
  const uint64_t body = r.off;
  uint64_t need = 0;
  const uint64_t cells = (uint64_t)batch * heads;
  for (uint64_t i = 0; i < cells; ++i) {
    uint32_t plen, rlen;
    if (!r.u32(plen) || !r.u32(rlen)) return eof();
    if (plen % n_r != 0) return format_fail("packed_len not block-aligned", r.off - 8);
    if (rlen >= n_r) return format_fail("res_len must be < N_r", r.off - 4);
    const uint64_t blocks = plen / n_r;
    if (!r.skip(2 * blocks * (2 * wpb + kp + vp) + 4ull * rlen * d))
      return format_fail("unexpected end of file", r.n);
    need = std::max<uint64_t>(need, (uint64_t)plen + rlen);
  }
  bdk_cache_desc desc{};
  desc.batch = batch;
  desc.heads_kv = heads;
  desc.head_dim = d;
  desc.warp_n = warp_n;
  desc.num_bits = bits;
  desc.k_axis = axis;
  desc.group_size = g;
  desc.interleave = flags & 1;
  desc.max_tokens = (uint32_t)std::max<uint64_t>(max_tokens, need + n_r);
  desc.device = device;
  bdk_cache* c = nullptr;
  bdk_status s = bdk_cache_create(&desc, &c);
  if (s) return s;
  const Geom& G = c->dev.G;
  if (c->wpb != wpb || c->kp_u16 != kp || c->vp_u16 != vp) {  // cannot happen for valid geometry
    bdk_cache_destroy(c);
    return format_fail("array sizes inconsistent with the header", 6);
  }
  // pass 2: fill the device arena
  r.off = body;
  std::vector<uint8_t> recs;
  std::vector<int> nbs(cells), rls(cells);
  for (uint64_t i = 0; i < cells; ++i) {
    uint32_t plen, rlen;
    r.u32(plen);
    r.u32(rlen);
    const uint32_t nb = plen / n_r;
    recs.assign((size_t)nb * G.rec_bytes, 0);
    for (int part = 0; part < 4; ++part) {
      for (uint32_t blk = 0; blk < nb; ++blk) {
        uint8_t* rec = recs.data() + (size_t)blk * G.rec_bytes;
        if (part == 0 || part == 2) {
          uint8_t* words = rec + (part == 2 ? G.wbytes : 0);
          for (uint32_t w = 0; w < wpb; ++w) {
            std::memcpy(words + word_offset(G, w), buf + r.off, 2);
            r.off += 2;
          }
        } else {
          const uint64_t nbytes = 2 * (part == 1 ? kp : vp);
          std::memcpy(rec + 2 * G.wbytes + (part == 3 ? G.kp_bytes : 0), buf + r.off, nbytes);
          r.off += nbytes;
        }
      }
    }
    cudaError_t e = cudaSuccess;
    if (nb)
      e = cudaMemcpy(c->dev.records + (size_t)i * G.max_blocks * G.rec_bytes, recs.data(),
                     recs.size(), cudaMemcpyHostToDevice);
    for (int t = 0; t < 2 && e == cudaSuccess; ++t) {
      if (rlen)
        e = cudaMemcpy((t ? c->dev.res_v : c->dev.res_k) + i * (size_t)G.n_r * d, buf + r.off,
                       (size_t)rlen * d * 2, cudaMemcpyHostToDevice);
      r.off += (uint64_t)rlen * d * 2;
    }
    if (e != cudaSuccess) {
      bdk_cache_destroy(c);
      return cuda_fail(e, "H2D load");
    }
    nbs[i] = (int)nb;
    rls[i] = (int)rlen;
  }
  cudaError_t e = cudaMemcpy(c->dev.packed_blocks, nbs.data(), cells * sizeof(int),
                             cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(c->dev.res_len, rls.data(), cells * sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    bdk_cache_destroy(c);
    return cuda_fail(e, "H2D lengths");
  }
  c->packed_blocks = nbs;
  c->res_len = rls;
  *out = c;
  return BDK_OK;
}

bdk_status bdk_load_cache_file(const char* path, uint32_t max_tokens, int32_t device,
                               bdk_cache** out) {
  if (!path || !out) return fail(BDK_INVALID_ARGUMENT, "null argument");
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(BDK_INVALID_ARGUMENT, std::string("cannot open ") + path);
  std::vector<uint8_t> data;
  uint8_t chunk[1 << 16];
  size_t n;
  while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) data.insert(data.end(), chunk, chunk + n);
  std::fclose(f);
  return bdk_load_cache(data.data(), data.size(), max_tokens, device, out);
}


// ------------------------------------------------- quant.hpp utilities
// quantize_tile / dequantize_tile / compute_group_params / quantize_group /
// dequantize_group (quant.hpp:56-80) on the device: host buffers in and out,
// synchronous.  Same validation and error classes as the reference.
namespace {
struct DevBuf {  // scoped device allocation
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

bdk_status quant_common(uint32_t bits, int32_t device) {
  if (bits == 0 || bits > 16) return fail(BDK_UNSUPPORTED_BITS, "num_bits must be 1..16");
  DevGuard dev_guard_(device);
  return BDK_OK;
}
}  // namespace

bdk_status bdk_quantize_tile(const float* x, uint32_t rows, uint32_t d, uint32_t bits,
                             uint32_t axis, uint32_t group_size, uint16_t* codes,
                             uint16_t* params, int32_t device) {
  if (!x || !codes || !params) return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (axis > 1) return fail(BDK_CONFIG_ERROR, "axis must be 0 (KChannel) or 1 (KToken)");
  const uint32_t extent = axis == 0 ? rows : d;
  if (group_size == 0 || extent % group_size != 0)
    return fail(BDK_SHAPE_ERROR, "group_size (" + std::to_string(group_size) +
                                     ") must divide the grouped extent (" +
                                     std::to_string(extent) + ")");
  bdk_status s = quant_common(bits, device);
  if (s) return s;
  const size_t n = (size_t)rows * d;
  const size_t groups = n / group_size;
  if (n == 0) return BDK_OK;
  DevBuf bx, bc, bp;
  BDK_CUDA(cudaMalloc(&bx.p, n * 4), "cudaMalloc");
  BDK_CUDA(cudaMalloc(&bc.p, n * 2), "cudaMalloc");
  BDK_CUDA(cudaMalloc(&bp.p, groups * 4), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bx.p, x, n * 4, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(bdk::launch_quantize_tile(static_cast<float*>(bx.p), (int)rows, (int)d, (int)bits,
                                     (int)axis, (int)group_size, static_cast<uint16_t*>(bc.p),
                                     static_cast<uint32_t*>(bp.p), nullptr),
           "quantize_tile launch");
  BDK_CUDA(cudaMemcpy(codes, bc.p, n * 2, cudaMemcpyDeviceToHost), "D2H codes");
  BDK_CUDA(cudaMemcpy(params, bp.p, groups * 4, cudaMemcpyDeviceToHost), "D2H params");
  return BDK_OK;
}

bdk_status bdk_dequantize_tile(const uint16_t* codes, const uint16_t* params, uint32_t rows,
                               uint32_t d, uint32_t axis, uint32_t group_size, float* out,
                               int32_t device) {
  if (!codes || !params || !out) return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (axis > 1) return fail(BDK_CONFIG_ERROR, "axis must be 0 (KChannel) or 1 (KToken)");
  const uint32_t extent = axis == 0 ? rows : d;
  if (group_size == 0 || extent % group_size != 0)
    return fail(BDK_SHAPE_ERROR, "dequantize_tile: group_size must divide the grouped extent");
  DevGuard dev_guard_(device);
  const size_t n = (size_t)rows * d;
  const size_t groups = n / group_size;
  if (n == 0) return BDK_OK;
  DevBuf bc, bp, bo;
  BDK_CUDA(cudaMalloc(&bc.p, n * 2), "cudaMalloc");
  BDK_CUDA(cudaMalloc(&bp.p, groups * 4), "cudaMalloc");
  BDK_CUDA(cudaMalloc(&bo.p, n * 4), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bc.p, codes, n * 2, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(cudaMemcpy(bp.p, params, groups * 4, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(bdk::launch_dequantize_tile(static_cast<uint16_t*>(bc.p),
                                       static_cast<uint32_t*>(bp.p), (int)rows, (int)d, (int)axis,
                                       (int)group_size, 1, static_cast<float*>(bo.p), nullptr),
           "dequantize_tile launch");
  BDK_CUDA(cudaMemcpy(out, bo.p, n * 4, cudaMemcpyDeviceToHost), "D2H");
  return BDK_OK;
}

bdk_status bdk_compute_group_params(const float* x, uint32_t n, uint32_t bits, float* scale,
                                    float* zero, int32_t device) {
  if (!x || !scale || !zero) return fail(BDK_INVALID_ARGUMENT, "null argument");
  if (n == 0) return fail(BDK_EMPTY_INPUT, "compute_group_params: empty group");
  std::vector<uint16_t> codes(n), prm(2);
  bdk_status s = bdk_quantize_tile(x, n, 1, bits, 0, n, codes.data(), prm.data(), device);
  if (s) return s;
  __half hs, hz;
  std::memcpy(&hs, &prm[0], 2);
  std::memcpy(&hz, &prm[1], 2);
  *scale = __half2float(hs);
  *zero = __half2float(hz);
  return BDK_OK;
}

bdk_status bdk_quantize_group(const float* x, uint32_t n, float scale, float zero, uint32_t bits,
                              uint16_t* codes, int32_t device) {
  if (!x || !codes) return fail(BDK_INVALID_ARGUMENT, "null argument");
  bdk_status s = quant_common(bits, device);
  if (s) return s;
  if (n == 0) return BDK_OK;
  DevBuf bx, bc;
  BDK_CUDA(cudaMalloc(&bx.p, (size_t)n * 4), "cudaMalloc");
  BDK_CUDA(cudaMalloc(&bc.p, (size_t)n * 2), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bx.p, x, (size_t)n * 4, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(bdk::launch_quantize_group(static_cast<float*>(bx.p), (int)n, scale, zero, (int)bits,
                                      static_cast<uint16_t*>(bc.p), nullptr),
           "quantize_group launch");
  BDK_CUDA(cudaMemcpy(codes, bc.p, (size_t)n * 2, cudaMemcpyDeviceToHost), "D2H");
  return BDK_OK;
}

bdk_status bdk_dequantize_group(const uint16_t* codes, uint32_t n, float scale, float zero,
                                float* values, int32_t device) {
  if (!codes || !values) return fail(BDK_INVALID_ARGUMENT, "null argument");
  DevGuard dev_guard_(device);
  if (n == 0) return BDK_OK;
  DevBuf bc, bo;
  BDK_CUDA(cudaMalloc(&bc.p, (size_t)n * 2), "cudaMalloc");
  BDK_CUDA(cudaMalloc(&bo.p, (size_t)n * 4), "cudaMalloc");
  BDK_CUDA(cudaMemcpy(bc.p, codes, (size_t)n * 2, cudaMemcpyHostToDevice), "H2D");
  BDK_CUDA(bdk::launch_dequantize_group(static_cast<uint16_t*>(bc.p), (int)n, scale, zero,
                                        static_cast<float*>(bo.p), nullptr),
           "dequantize_group launch");
  BDK_CUDA(cudaMemcpy(values, bo.p, (size_t)n * 4, cudaMemcpyDeviceToHost), "D2H");
  return BDK_OK;
}

}  // extern "C"
