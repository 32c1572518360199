// ref_shim.cpp -- extern "C" handle API over the UNMODIFIED reference engine
// (/root/reference/proj/src/*.cpp, compiled where the sources lie by
// oracle/Makefile into oracle/_ref/libbitkv_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (to pin the C restatement in
// oracle/bitkv_oracle.c and to generate tests/golden/) and by bench.py's
// reference/cpu_baseline arm.  Nothing here is on the product path.
//
// Exceptions never cross this boundary: every entry point returns the status
// code of the reference exception class (errors.hpp:14-54).
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <algorithm>
#include <vector>

#include "bitkv/attention.hpp"
#include "bitkv/bench.hpp"
#include "bitkv/errors.hpp"
#include "bitkv/kvcache.hpp"
#include "bitkv/layout.hpp"
#include "bitkv/serialize.hpp"

using namespace bitkv;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const ShapeError*>(&e)) return 2;
  if (dynamic_cast<const UnsupportedBits*>(&e)) return 3;
  if (dynamic_cast<const CodeOverflow*>(&e)) return 4;
  if (dynamic_cast<const CapacityError*>(&e)) return 5;
  if (dynamic_cast<const StateError*>(&e)) return 6;
  if (dynamic_cast<const FormatError*>(&e)) return 7;
  if (dynamic_cast<const EmptyInput*>(&e)) return 8;
  return 99;
}

#define GUARD(...)                           \
  try {                                      \
    __VA_ARGS__;                             \
    return 0;                                \
  } catch (const std::exception& e) {        \
    return status_of(e);                     \
  }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_pack_word(const uint16_t* codes, uint32_t bits, int interleave, uint16_t* word) {
  GUARD({
    const InterleavePerm p = interleave ? interleave_order(bits) : identity_order(bits);
    *word = pack_word(std::span<const uint16_t>(codes, p.pack_num), p);
  })
}

int ref_unpack_word(uint16_t word, uint32_t bits, int interleave, uint16_t* codes) {
  GUARD({
    const InterleavePerm p = interleave ? interleave_order(bits) : identity_order(bits);
    unpack_word(word, p, std::span<uint16_t>(codes, p.pack_num));
  })
}

int ref_group_params(const float* x, size_t n, uint32_t bits, float* scale, float* zero) {
  GUARD({
    const GroupParams p = compute_group_params(std::span<const float>(x, n), bits);
    *scale = p.scale;
    *zero = p.zero;
  })
}

struct RefCache {
  KVCache cache;
};

int ref_cache_create(size_t batch, size_t heads_kv, size_t d, size_t warp_n, uint32_t bits,
                     uint32_t k_axis, size_t g, int interleave, void** out) {
  GUARD({
    QuantSpec spec{bits, k_axis ? QuantAxis::KToken : QuantAxis::KChannel, g};
    *out = new RefCache{KVCache(batch, heads_kv, d, warp_n, spec, CacheBackend::Contiguous, 16,
                                0, interleave != 0)};
  })
}

void ref_cache_destroy(void* c) { delete static_cast<RefCache*>(c); }

size_t ref_cache_n_r(void* c) { return static_cast<RefCache*>(c)->cache.n_r(); }
size_t ref_cache_packed_len(void* c, size_t b, size_t h) {
  return static_cast<RefCache*>(c)->cache.packed_len(b, h);
}
size_t ref_cache_res_len(void* c, size_t b, size_t h) {
  return static_cast<RefCache*>(c)->cache.res_len(b, h);
}

int ref_cache_prefill(void* c, size_t b, size_t h, const float* k, const float* v, size_t len) {
  GUARD(static_cast<RefCache*>(c)->cache.prefill(b, h, k, v, len))
}

int ref_cache_append(void* c, size_t b, size_t h, const float* k, const float* v) {
  GUARD(static_cast<RefCache*>(c)->cache.append_token(b, h, k, v))
}

int ref_cache_flush(void* c, size_t b, size_t h) {
  GUARD(static_cast<RefCache*>(c)->cache.flush_residual(b, h))
}

// which: 0 k_words, 1 v_words, 2 k_params, 3 v_params.  Copies up to cap u16
// and returns the element count through *n.
int ref_cache_block(void* c, size_t b, size_t h, size_t blk, int which, uint16_t* dst,
                    size_t cap, size_t* n) {
  GUARD({
    const PackedBlock& pb = static_cast<RefCache*>(c)->cache.packed(b, h).blocks.at(blk);
    const std::vector<uint16_t>& src = which == 0   ? pb.k_words
                                       : which == 1 ? pb.v_words
                                       : which == 2 ? pb.k_params.data
                                                    : pb.v_params.data;
    *n = src.size();
    std::memcpy(dst, src.data(), std::min(cap, src.size()) * 2);
  })
}

int ref_cache_reconstruct(void* c, size_t b, size_t h, float* k_out, float* v_out) {
  GUARD({
    std::vector<float> k, v;
    static_cast<RefCache*>(c)->cache.reconstruct(b, h, k, v);
    std::memcpy(k_out, k.data(), k.size() * 4);
    std::memcpy(v_out, v.data(), v.size() * 4);
  })
}

int ref_cache_memory(void* c, size_t* out4) {
  GUARD({
    const auto m = static_cast<RefCache*>(c)->cache.memory();
    out4[0] = m.k_packed_payload_bytes;
    out4[1] = m.v_packed_payload_bytes;
    out4[2] = m.params_bytes;
    out4[3] = m.residual_bytes;
  })
}

// BDKV dump (serialize.cpp:87-120).  Returns the byte count through *n; copies
// up to cap bytes.
int ref_cache_dump(void* c, uint8_t* dst, size_t cap, size_t* n) {
  GUARD({
    std::ostringstream os(std::ios::binary);
    dump_cache(static_cast<RefCache*>(c)->cache, os);
    const std::string s = os.str();
    *n = s.size();
    std::memcpy(dst, s.data(), std::min(cap, s.size()));
  })
}

int ref_cache_load(const uint8_t* src, size_t n, void** out) {
  GUARD({
    std::istringstream is(std::string(reinterpret_cast<const char*>(src), n), std::ios::binary);
    *out = new RefCache{load_cache(is)};
  })
}

// decode_step (attention.cpp:164-242) with caller-provided fp32 tensors.
int ref_decode_step(void* c, size_t heads_q, size_t tile_n, size_t num_splits, size_t warp_n,
                    const float* q, const float* k_new, const float* v_new, float* out) {
  GUARD({
    KVCache& cache = static_cast<RefCache*>(c)->cache;
    AttentionConfig cfg;
    cfg.batch = cache.batch();
    cfg.heads_q = heads_q;
    cfg.heads_kv = cache.heads_kv();
    cfg.head_dim = cache.head_dim();
    cfg.tile_m = std::max<size_t>(1, heads_q / cache.heads_kv());
    cfg.tile_n = tile_n;
    cfg.num_splits = num_splits;
    cfg.warp_n = warp_n;
    const size_t d = cfg.head_dim;
    Tensor tq({cfg.batch, heads_q, d});
    Tensor tk({cfg.batch, cfg.heads_kv, d});
    Tensor tv({cfg.batch, cfg.heads_kv, d});
    for (size_t i = 0; i < tq.numel(); ++i) tq.set(i, q[i]);
    for (size_t i = 0; i < tk.numel(); ++i) tk.set(i, k_new[i]);
    for (size_t i = 0; i < tv.numel(); ++i) tv.set(i, v_new[i]);
    const AttnOutput o = decode_step(cache, cfg, tq, tk, tv);
    std::memcpy(out, o.data.data(), o.data.size() * 4);
  })
}

// naive oracle (oracle.cpp:12-37)
void ref_naive_attention(const float* q, size_t rows, const float* k, const float* v,
                         size_t len, size_t d, float* out) {
  const auto o = naive_attention(q, rows, k, v, len, d);
  std::memcpy(out, o.data(), o.size() * 4);
}

// run_bench (bench.cpp:80-210): the reference's own timing harness.
// out: [0] prefill_seconds [1] mean_ms [2] p50_ms [3] p99_ms [4] tokens/s
//      [5] checksum (bit-cast u64) [6..9] memory fields [10] n_r
int ref_run_bench(int mode, size_t seq_len, size_t batch, size_t heads_q, size_t heads_kv,
                  size_t head_dim, uint32_t bits, size_t group_size, uint32_t k_axis,
                  size_t num_splits, size_t steps, uint64_t seed, size_t tile_n, size_t warp_n,
                  int interleave, int verify, double* out, double* oracle3, double* step_ms,
                  size_t step_cap) {
  GUARD({
    WorkloadSpec s;
    s.mode = mode == 0 ? WorkloadMode::Single
                       : (mode == 1 ? WorkloadMode::Batches : WorkloadMode::Page);
    s.seq_len = seq_len;
    s.batch = batch;
    s.heads_q = heads_q;
    s.heads_kv = heads_kv;
    s.head_dim = head_dim;
    s.bits = bits;
    s.group_size = group_size;
    s.quant_axis = k_axis ? QuantAxis::KToken : QuantAxis::KChannel;
    s.num_splits = num_splits;
    s.steps = steps;
    s.seed = seed;
    s.tile_n = tile_n;
    s.warp_n = warp_n;
    s.interleave = interleave != 0;
    s.verify = verify != 0;
    const BenchReport r = run_bench(s);
    out[0] = r.prefill_seconds;
    out[1] = r.mean_ms;
    out[2] = r.p50_ms;
    out[3] = r.p99_ms;
    out[4] = r.tokens_per_second;
    std::memcpy(&out[5], &r.output_checksum, 8);
    out[6] = double(r.memory.k_packed_payload_bytes);
    out[7] = double(r.memory.v_packed_payload_bytes);
    out[8] = double(r.memory.params_bytes);
    out[9] = double(r.memory.residual_bytes);
    out[10] = double(r.n_r);
    for (size_t i = 0; step_ms && i < std::min(step_cap, r.step_seconds.size()); ++i)
      step_ms[i] = r.step_seconds[i] * 1e3;
    if (oracle3) {
      oracle3[0] = r.oracle.max_abs_err;
      oracle3[1] = r.oracle.rel_l2_err;
      oracle3[2] = r.oracle.cosine_similarity;
    }
  })
}

// run_verify battery (bench.cpp:602-613); returns the number of failures.
int ref_run_verify(uint64_t seed_begin, uint64_t seed_end, uint32_t bits) {
  try {
    int fails = 0;
    for (const auto& r : run_verify(seed_begin, seed_end, bits)) fails += r.pass ? 0 : 1;
    return fails;
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

}  // extern "C"
