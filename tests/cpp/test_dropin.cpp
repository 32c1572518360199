// test_dropin.cpp -- the C++ drop-in (include/bitkv_b200.hpp) used exactly like
// the reference engine's API, checked against the CPU oracle (oracle/, test
// infrastructure only).  Mirrors the reference doctest cases it cites.
//
//   build: tests/test_cpp_dropin.py (g++ -std=c++20 ... -lbitdecode_b200 -loracle)
//   run:   needs a B200 (cuda:0); exit code = number of failed checks
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "bitkv_b200.hpp"
extern "C" {
#include "bitkv_oracle.h"
}

static int g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)

template <class E, class F>
static bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

using namespace bitkv;

static std::vector<float> gauss(orc_gauss& g, size_t n) {
  std::vector<float> v(n);
  orc_gauss_fill_rounded(&g, v.data(), n);
  return v;
}

// test_kvcache.cpp:27-57 (prefill split) + :110-130 (flushed block ==
// offline reference bit-exact), at d = 128 on the device cache
static void prefill_is_bit_exact(uint32_t bits, size_t warp_n, size_t g, QuantAxis axis) {
  const size_t d = 128, len = 3 * residual_block_size(bits, warp_n) + 37;
  KVCache cache(1, 2, d, warp_n, QuantSpec{bits, axis, g});
  int st = 0;
  orc_cache* oc = orc_cache_create(1, 2, d, warp_n, bits, (uint32_t)axis, g, 1, len + 512, &st);
  CHECK(st == 0);
  orc_gauss rng;
  orc_gauss_init(&rng, bits * 31 + warp_n);
  for (size_t h = 0; h < 2; ++h) {
    const auto k = gauss(rng, len * d), v = gauss(rng, len * d);
    cache.prefill(0, h, k.data(), v.data(), len);
    CHECK(orc_cache_prefill(oc, 0, h, k.data(), v.data(), len) == 0);
    CHECK(cache.packed_len(0, h) == orc_cache_packed_len(oc, 0, h));
    CHECK(cache.res_len(0, h) == orc_cache_res_len(oc, 0, h));
    const PackedKV pk = cache.packed(0, h);
    for (size_t i = 0; i < pk.blocks.size(); ++i) {
      const PackedBlock& b = pk.blocks[i];
      const uint16_t* kw = orc_cache_block(oc, 0, h, i, 0);
      const uint16_t* vw = orc_cache_block(oc, 0, h, i, 1);
      const uint16_t* kp = orc_cache_block(oc, 0, h, i, 2);
      const uint16_t* vp = orc_cache_block(oc, 0, h, i, 3);
      CHECK(std::memcmp(b.k_words.data(), kw, b.k_words.size() * 2) == 0);
      CHECK(std::memcmp(b.v_words.data(), vw, b.v_words.size() * 2) == 0);
      CHECK(std::memcmp(b.k_params.data.data(), kp, b.k_params.data.size() * 2) == 0);
      CHECK(std::memcmp(b.v_params.data.data(), vp, b.v_params.data.size() * 2) == 0);
    }
    // reconstruct == oracle reconstruct (dequantized packed tokens + residual)
    std::vector<float> rk, rv;
    cache.reconstruct(0, h, rk, rv);
    std::vector<float> ok(rk.size()), ov(rv.size());
    CHECK(orc_cache_reconstruct(oc, 0, h, ok.data(), ov.data()) == 0);
    CHECK(rk == ok && rv == ov);
  }
  orc_cache_destroy(oc);
}

// test_attention.cpp:350-441: engine decode vs the reference algorithm, in
// the precise mode at the reference's 1e-5 and in the fast mode at its stated
// tolerance; the N_r-th step flushes exactly once (:401-421)
static void decode_matches_oracle(bool precise, uint32_t bits, size_t hq, size_t hkv) {
  const size_t d = 128, warp_n = 4, batch = 2;
  const size_t n_r = residual_block_size(bits, warp_n), len = 4 * n_r - 2;
  KVCache cache(batch, hkv, d, warp_n, QuantSpec{bits, QuantAxis::KChannel, 128});
  cache.set_precise(precise);
  int st = 0;
  orc_cache* oc = orc_cache_create(batch, hkv, d, warp_n, bits, 0, 128, 1, len + 512, &st);
  orc_gauss rng;
  orc_gauss_init(&rng, 99 + bits + hq);
  for (size_t b = 0; b < batch; ++b)
    for (size_t h = 0; h < hkv; ++h) {
      const auto k = gauss(rng, len * d), v = gauss(rng, len * d);
      cache.prefill(b, h, k.data(), v.data(), len);
      orc_cache_prefill(oc, b, h, k.data(), v.data(), len);
    }
  AttentionConfig cfg;
  cfg.batch = batch;
  cfg.heads_q = hq;
  cfg.heads_kv = hkv;
  cfg.head_dim = d;
  cfg.warp_n = warp_n;
  double worst = 0.0, ref2 = 0.0, err2 = 0.0;
  for (int step = 0; step < 4; ++step) {  // crosses the flush at step 2
    Tensor q({batch, hq, d}), kn({batch, hkv, d}), vn({batch, hkv, d});
    for (size_t i = 0; i < q.numel(); ++i) q.set(i, orc_gauss_next(&rng));
    for (size_t i = 0; i < kn.numel(); ++i) kn.set(i, orc_gauss_next(&rng));
    for (size_t i = 0; i < vn.numel(); ++i) vn.set(i, orc_gauss_next(&rng));
    const AttnOutput out = decode_step(cache, cfg, q, kn, vn);
    std::vector<float> ref(q.numel());
    CHECK(orc_decode_step(oc, hq, 64, 4, warp_n, q.data(), kn.data(), vn.data(), ref.data(), 1) ==
          0);
    for (size_t i = 0; i < ref.size(); ++i) {
      worst = std::max(worst, (double)std::fabs(out.data[i] - ref[i]));
      ref2 += (double)ref[i] * ref[i];
      err2 += (double)(out.data[i] - ref[i]) * (out.data[i] - ref[i]);
    }
    for (size_t b = 0; b < batch; ++b)
      for (size_t h = 0; h < hkv; ++h) {
        CHECK(cache.packed_len(b, h) == orc_cache_packed_len(oc, b, h));
        CHECK(cache.res_len(b, h) == orc_cache_res_len(oc, b, h));
      }
  }
  const double rel = std::sqrt(err2 / ref2);
  std::printf("decode bits=%u hq=%zu hkv=%zu precise=%d: max-abs %.3e rel-L2 %.3e\n", bits, hq,
              hkv, (int)precise, worst, rel);
  if (precise)
    CHECK(worst < 1e-5);
  else
    CHECK(worst < 2e-3 && rel < 1e-3);
  orc_cache_destroy(oc);
}

// the reference's error behaviour at the API boundary (errors.hpp)
static void errors_map_to_reference_exceptions() {
  KVCache cache(1, 1, 128, 1, QuantSpec{8, QuantAxis::KChannel, 16});  // N_r = 16
  std::vector<float> row(128, 0.5f);
  for (int t = 0; t < 16; ++t) cache.append_token(0, 0, row.data(), row.data());
  CHECK(cache.res_len(0, 0) == 16);
  CHECK(throws_as<CapacityError>([&] { cache.append_token(0, 0, row.data(), row.data()); }));
  cache.flush_residual(0, 0);  // test_kvcache.cpp:76-91
  CHECK(cache.res_len(0, 0) == 0 && cache.packed_len(0, 0) == 16);
  CHECK(throws_as<StateError>([&] { cache.flush_residual(0, 0); }));
  CHECK(throws_as<StateError>([&] { cache.prefill(0, 0, row.data(), row.data(), 1); }));
  AttentionConfig bad;
  bad.heads_q = 32;
  bad.heads_kv = 5;
  CHECK(throws_as<ConfigError>([&] { validate_config(bad); }));
  CHECK(throws_as<UnsupportedBits>(
      [&] { KVCache(1, 1, 128, 4, QuantSpec{3, QuantAxis::KChannel, 64}); }));
  // constant block -> zero words, exact params (test_kvcache.cpp:93-108)
  const KVCache::Memory m = cache.memory();
  CHECK(m.k_packed_payload_bytes == 16 * 128 * 8 / 8);
  const PackedBlock b = cache.packed(0, 0).blocks.at(0);
  bool zeros = true;
  for (uint16_t w : b.k_words) zeros &= (w == 0);
  CHECK(zeros);
  CHECK(b.k_params.zero(0) == 0.5f && b.k_params.scale(0) == kMinScale);
}

// test_serialize.cpp:44-82 on the device cache: dump -> load reproduces
// every cell, re-dump is byte-identical; truncation / bad magic ->
// FormatError with an offset (:84-104)
static void serialize_round_trip(uint32_t bits) {
  const size_t d = 128, n_r = residual_block_size(bits, 4);
  KVCache cache(2, 2, d, 4, QuantSpec{bits, QuantAxis::KChannel, 128}, CacheBackend::Contiguous,
                16, 0, true, 4 * n_r);
  orc_gauss rng;
  orc_gauss_init(&rng, 500 + bits);
  for (size_t b = 0; b < 2; ++b)
    for (size_t h = 0; h < 2; ++h) {
      const size_t len = n_r + 13 * (b * 2 + h + 1);
      const auto k = gauss(rng, len * d), v = gauss(rng, len * d);
      cache.prefill(b, h, k.data(), v.data(), len);
    }
  std::ostringstream os(std::ios::binary);
  dump_cache(cache, os);
  const std::string bytes = os.str();
  std::istringstream is(bytes, std::ios::binary);
  KVCache loaded = load_cache(is);
  CHECK(loaded.n_r() == cache.n_r() && loaded.batch() == 2 && loaded.heads_kv() == 2);
  for (size_t b = 0; b < 2; ++b)
    for (size_t h = 0; h < 2; ++h) {
      CHECK(loaded.packed_len(b, h) == cache.packed_len(b, h));
      CHECK(loaded.res_len(b, h) == cache.res_len(b, h));
      CHECK(loaded.packed(b, h).blocks == cache.packed(b, h).blocks);
    }
  std::ostringstream os2(std::ios::binary);
  dump_cache(loaded, os2);
  CHECK(os2.str() == bytes);
  for (size_t cut : {size_t{0}, size_t{3}, size_t{9}, bytes.size() / 2, bytes.size() - 1}) {
    std::istringstream t(bytes.substr(0, cut), std::ios::binary);
    CHECK(throws_as<FormatError>([&] { load_cache(t); }));
  }
  std::string bad = bytes;
  bad[0] = 'X';
  std::istringstream tb(bad, std::ios::binary);
  try {
    load_cache(tb);
    CHECK(false);
  } catch (const FormatError& e) {
    CHECK(e.offset == 0);
  }
}

// layout.hpp / quant.hpp API of the drop-in (test_layout.cpp:13-39,
// test_quant.cpp:27-69)
static void quant_and_layout_api() {
  const InterleavePerm p2 = interleave_order(2);
  const uint8_t want2[8] = {7, 5, 3, 1, 6, 4, 2, 0};
  CHECK(std::memcmp(p2.order.data(), want2, 8) == 0);
  const uint16_t c4[4] = {1, 2, 3, 4};
  CHECK(pack_word(c4, interleave_order(4)) == 0x4231);
  uint16_t back[4] = {};
  unpack_word(0x4231, interleave_order(4), back);
  CHECK(std::memcmp(back, c4, 8) == 0);
  const uint16_t big[4] = {16, 0, 0, 0};
  CHECK(throws_as<CodeOverflow>([&] { pack_word(big, interleave_order(4)); }));
  const float g[4] = {-1.f, 0.f, 2.f, 5.f};
  uint16_t codes[4] = {};
  quantize_group(g, 0.4f, -1.0f, 4, codes);  // round half to even: {0, 2, 8, 15}
  CHECK(codes[0] == 0 && codes[1] == 2 && codes[2] == 8 && codes[3] == 15);
  const GroupParams gp = compute_group_params(g, 4);
  CHECK(gp.zero == -1.0f && gp.scale == round_f16(6.0f / 15.0f));
  // quantize_tile -> pack_block_codes == the cache's own packed block
  const size_t d = 128, n_r = 128;
  orc_gauss rng;
  orc_gauss_init(&rng, 77);
  const auto k = gauss(rng, n_r * d), v = gauss(rng, n_r * d);
  KVCache cache(1, 1, d, 4, QuantSpec{4, QuantAxis::KChannel, 128});
  cache.prefill(0, 0, k.data(), v.data(), n_r);
  const PackedBlock blk = cache.packed(0, 0).blocks.at(0);
  const QuantizedTile qk = quantize_tile(k.data(), n_r, d, 4, QuantAxis::KChannel, 128);
  CHECK(pack_block_codes(qk.codes, n_r, d, interleave_order(4)) == blk.k_words);
  CHECK(qk.params.data == blk.k_params.data);
  CHECK(unpack_block_codes(blk.k_words, n_r, d, interleave_order(4)) == qk.codes);
}

int main() {
  prefill_is_bit_exact(4, 4, 128, QuantAxis::KChannel);
  prefill_is_bit_exact(2, 4, 128, QuantAxis::KChannel);
  prefill_is_bit_exact(8, 2, 32, QuantAxis::KChannel);
  prefill_is_bit_exact(4, 2, 32, QuantAxis::KToken);
  decode_matches_oracle(false, 4, 32, 8);
  decode_matches_oracle(false, 2, 32, 8);
  decode_matches_oracle(true, 4, 32, 8);
  decode_matches_oracle(true, 2, 8, 8);
  errors_map_to_reference_exceptions();
  serialize_round_trip(4);
  serialize_round_trip(2);
  quant_and_layout_api();
  std::printf("%s: %d failed checks\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail;
}
