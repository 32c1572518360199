/*
 * bitkv_oracle.c -- CPU restatement of the reference decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see bitkv_oracle.h).  Compiled with
 * -ffp-contract=off and no -march so that, like the reference Release build
 * (proj/CMakeLists.txt:6-13, no -march), no FMA contraction changes the
 * summation results; the decode outputs then agree bit-for-bit with the
 * reference compiled the same way (pinned by tests/test_oracle.py).
 *
 * Citations are relative to /root/reference/proj.
 */
#include "bitkv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ fp16 */

/* include/bitkv/fp16.hpp:13-38 (RNE narrowing, saturate to inf, NaN->7E00) */
uint16_t orc_f32_to_f16_bits(float value) {
  uint32_t f;
  memcpy(&f, &value, 4);
  const uint32_t sign = f & 0x80000000u;
  f ^= sign;
  uint16_t out;
  if (f >= 0x47800000u) {
    out = f > 0x7F800000u ? 0x7E00u : 0x7C00u;
  } else if (f < 0x38800000u) {
    float aligned;
    memcpy(&aligned, &f, 4);
    aligned += 0.5f;
    uint32_t bits;
    memcpy(&bits, &aligned, 4);
    out = (uint16_t)(bits - 0x3F000000u);
  } else {
    const uint32_t mant_odd = (f >> 13) & 1u;
    f += 0xC8000FFFu;
    f += mant_odd;
    out = (uint16_t)(f >> 13);
  }
  return (uint16_t)(out | (sign >> 16));
}

/* include/bitkv/fp16.hpp:40-65 (exact widening) */
float orc_f16_bits_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu;
  uint32_t mant = h & 0x3FFu;
  uint32_t bits;
  if (e == 0) {
    if (mant == 0) {
      bits = sign;
    } else {
      e = 1;
      while (!(mant & 0x400u)) {
        mant <<= 1;
        --e;
      }
      mant &= 0x3FFu;
      bits = sign | ((e + 112u) << 23) | (mant << 13);
    }
  } else if (e == 31) {
    bits = sign | 0x7F800000u | (mant << 13);
  } else {
    bits = sign | ((e + 112u) << 23) | (mant << 13);
  }
  float out;
  memcpy(&out, &bits, 4);
  return out;
}

/* fp16.hpp:68-70 */
float orc_round_f16(float v) { return orc_f16_bits_to_f32(orc_f32_to_f16_bits(v)); }

/* ---------------------------------------------------------------- layout */

static int bits_ok(uint32_t bits) { return bits == 2 || bits == 4 || bits == 8 || bits == 16; }

/* layout.cpp:21-43: interleaved = odd indices descending then even
 * descending ("75316420" for 8 fields); identity = 0..P-1 */
int orc_perm(uint32_t bits, int interleave, uint8_t order[8], uint32_t* pack_num) {
  if (!bits_ok(bits)) return ORC_UNSUPPORTED_BITS;
  const uint32_t p = 16 / bits;
  memset(order, 0, 8);
  if (interleave) {
    uint32_t k = 0;
    for (uint32_t i = p; i-- > 0;)
      if (i % 2 == 1) order[k++] = (uint8_t)i;
    for (uint32_t i = p; i-- > 0;)
      if (i % 2 == 0) order[k++] = (uint8_t)i;
  } else {
    for (uint32_t i = 0; i < p; ++i) order[i] = (uint8_t)i;
  }
  *pack_num = p;
  return ORC_OK;
}

/* layout.cpp:45-61: field k (from the MSB) holds codes[order[k]] */
int orc_pack_word(const uint16_t* codes, uint32_t bits, int interleave, uint16_t* word) {
  uint8_t order[8];
  uint32_t p;
  int st = orc_perm(bits, interleave, order, &p);
  if (st) return st;
  const uint32_t limit = bits >= 16 ? 0x10000u : (1u << bits);
  uint32_t w = 0;
  for (uint32_t k = 0; k < p; ++k) {
    const uint32_t code = codes[order[k]];
    if (code >= limit) return ORC_CODE_OVERFLOW;
    w |= code << (16 - (k + 1) * bits);
  }
  *word = (uint16_t)w;
  return ORC_OK;
}

/* layout.cpp:63-72 */
int orc_unpack_word(uint16_t word, uint32_t bits, int interleave, uint16_t* codes) {
  uint8_t order[8];
  uint32_t p;
  int st = orc_perm(bits, interleave, order, &p);
  if (st) return st;
  const uint32_t mask = bits >= 16 ? 0xFFFFu : (1u << bits) - 1u;
  for (uint32_t k = 0; k < p; ++k)
    codes[order[k]] = (uint16_t)((word >> (16 - (k + 1) * bits)) & mask);
  return ORC_OK;
}

/* layout.cpp:74-77: N_r = 8 * W_n * (16 / B) */
size_t orc_residual_block_size(uint32_t bits, size_t warp_n) {
  if (!bits_ok(bits)) return 0;
  return 8 * warp_n * (16 / bits);
}

/* ----------------------------------------------------------------- quant */

static const float kMinScale = 6.103515625e-05f; /* quant.hpp:52, 2^-14 */

/* quant.cpp:18-28: zero = min, scale = round_f16((max-min)/qmax) clamped */
void orc_group_params(const float* x, size_t stride, size_t n, uint32_t bits, float* scale,
                      float* zero) {
  float lo = x[0], hi = x[0];
  for (size_t i = 0; i < n; ++i) {
    const float v = x[i * stride];
    lo = v < lo ? v : lo; /* std::min(lo, x) */
    hi = hi < v ? v : hi; /* std::max(hi, x) */
  }
  float s = orc_round_f16((hi - lo) / (float)((1u << bits) - 1u));
  if (!(s >= kMinScale)) s = kMinScale;
  *scale = s;
  *zero = orc_round_f16(lo);
}

/* quant.cpp:30-38: code = clamp(nearbyint((x - zero) / scale), 0, qmax) */
void orc_quantize_group(const float* x, size_t stride, size_t n, float scale, float zero,
                        uint32_t bits, uint16_t* codes, size_t code_stride) {
  const float qmax = (float)((1u << bits) - 1u);
  for (size_t i = 0; i < n; ++i) {
    float c = nearbyintf((x[i * stride] - zero) / scale);
    c = c < 0.0f ? 0.0f : (qmax < c ? qmax : c); /* std::clamp */
    codes[i * code_stride] = (uint16_t)c;
  }
}

size_t orc_param_count(size_t n_r, size_t d, uint32_t bits, uint32_t axis, size_t g) {
  if (bits == 16) return 0;
  const size_t groups = axis == 0 ? (n_r / g) * d : n_r * (d / g);
  return 2 * groups;
}

/* quant.cpp:47-93 quantize_tile: codes row-major [rows, d]; param push order
 * [gr][c] for KChannel, [t][gc] for KToken (quant.cpp:71, :88) */
static void quantize_tile(const float* tile, size_t rows, size_t d, uint32_t bits, uint32_t axis,
                          size_t g, uint16_t* codes, uint16_t* params) {
  size_t np = 0;
  if (axis == 0) {
    for (size_t gr = 0; gr < rows / g; ++gr) {
      for (size_t c = 0; c < d; ++c) {
        float s, z;
        const float* base = tile + gr * g * d + c;
        orc_group_params(base, d, g, bits, &s, &z);
        orc_quantize_group(base, d, g, s, z, bits, codes + gr * g * d + c, d);
        params[np++] = orc_f32_to_f16_bits(s);
        params[np++] = orc_f32_to_f16_bits(z);
      }
    }
  } else {
    for (size_t t = 0; t < rows; ++t) {
      for (size_t gc = 0; gc < d / g; ++gc) {
        float s, z;
        const float* base = tile + t * d + gc * g;
        orc_group_params(base, 1, g, bits, &s, &z);
        orc_quantize_group(base, 1, g, s, z, bits, codes + t * d + gc * g, 1);
        params[np++] = orc_f32_to_f16_bits(s);
        params[np++] = orc_f32_to_f16_bits(z);
      }
    }
  }
}

/* kvcache.cpp:79-95 pack_block_codes: words[c * (n_r/P) + g] packs tokens
 * g*P .. g*P+P-1 of channel c */
static void pack_block_codes(const uint16_t* codes, size_t n_r, size_t d, uint32_t bits,
                             int interleave, uint16_t* words) {
  const size_t p = 16 / bits, groups = n_r / p;
  uint16_t tmp[8];
  for (size_t c = 0; c < d; ++c) {
    for (size_t g = 0; g < groups; ++g) {
      for (size_t k = 0; k < p; ++k) tmp[k] = codes[(g * p + k) * d + c];
      orc_pack_word(tmp, bits, interleave, &words[c * groups + g]);
    }
  }
}

/* kvcache.cpp:97-112 */
static void unpack_block_codes(const uint16_t* words, size_t n_r, size_t d, uint32_t bits,
                               int interleave, uint16_t* codes) {
  const size_t p = 16 / bits, groups = n_r / p;
  uint16_t tmp[8];
  for (size_t c = 0; c < d; ++c) {
    for (size_t g = 0; g < groups; ++g) {
      orc_unpack_word(words[c * groups + g], bits, interleave, tmp);
      for (size_t k = 0; k < p; ++k) codes[(g * p + k) * d + c] = tmp[k];
    }
  }
}

/* kvcache.cpp:184-206 make_block_from */
int orc_make_block(const float* k, const float* v, size_t n_r, size_t d, uint32_t bits,
                   uint32_t k_axis, size_t g, int interleave, uint16_t* k_words,
                   uint16_t* v_words, uint16_t* k_params, uint16_t* v_params) {
  if (!bits_ok(bits)) return ORC_UNSUPPORTED_BITS;
  uint16_t* kc = (uint16_t*)malloc(n_r * d * 2);
  uint16_t* vc = (uint16_t*)malloc(n_r * d * 2);
  if (bits == 16) { /* passthrough: raw binary16 bits, P = 1, no params */
    for (size_t i = 0; i < n_r * d; ++i) {
      kc[i] = orc_f32_to_f16_bits(k[i]);
      vc[i] = orc_f32_to_f16_bits(v[i]);
    }
  } else {
    quantize_tile(k, n_r, d, bits, k_axis, g, kc, k_params);
    quantize_tile(v, n_r, d, bits, 1, g, vc, v_params);
  }
  pack_block_codes(kc, n_r, d, bits, interleave, k_words);
  pack_block_codes(vc, n_r, d, bits, interleave, v_words);
  free(kc);
  free(vc);
  return ORC_OK;
}

/* kvcache.cpp:263-312 packed_tile: round_f16(code * scale + zero) */
void orc_dequant_block(const uint16_t* k_words, const uint16_t* v_words,
                       const uint16_t* k_params, const uint16_t* v_params, size_t n_r, size_t d,
                       uint32_t bits, uint32_t k_axis, size_t g, int interleave, float* k_out,
                       float* v_out) {
  uint16_t* kc = (uint16_t*)malloc(n_r * d * 2);
  uint16_t* vc = (uint16_t*)malloc(n_r * d * 2);
  unpack_block_codes(k_words, n_r, d, bits, interleave, kc);
  unpack_block_codes(v_words, n_r, d, bits, interleave, vc);
  if (bits == 16) {
    for (size_t i = 0; i < n_r * d; ++i) {
      k_out[i] = orc_f16_bits_to_f32(kc[i]);
      v_out[i] = orc_f16_bits_to_f32(vc[i]);
    }
  } else {
    const size_t vcols = d / g;
    for (size_t row = 0; row < n_r; ++row) {
      for (size_t c = 0; c < d; ++c) {
        const size_t kg = k_axis == 0 ? (row / g) * d + c : row * (d / g) + c / g;
        const size_t vg = row * vcols + c / g;
        const float ks = orc_f16_bits_to_f32(k_params[2 * kg]);
        const float kz = orc_f16_bits_to_f32(k_params[2 * kg + 1]);
        const float vs = orc_f16_bits_to_f32(v_params[2 * vg]);
        const float vz = orc_f16_bits_to_f32(v_params[2 * vg + 1]);
        k_out[row * d + c] = orc_round_f16((float)kc[row * d + c] * ks + kz);
        v_out[row * d + c] = orc_round_f16((float)vc[row * d + c] * vs + vz);
      }
    }
  }
  free(kc);
  free(vc);
}

/* ----------------------------------------------------------------- cache */

struct orc_cache {
  size_t batch, heads_kv, d, warp_n, n_r, g, max_blocks;
  uint32_t bits, k_axis;
  int interleave;
  size_t wpb, kpc, vpc; /* words per block, param u16 counts */
  size_t* packed_len;
  size_t* res_len;
  uint16_t *kw, *vw, *kp, *vp;
  float *rk, *rv; /* [cells][n_r][d] */
};

size_t orc_cache_n_r(const orc_cache* c) { return c->n_r; }

/* kvcache.cpp:114-148 constructor checks */
orc_cache* orc_cache_create(size_t batch, size_t heads_kv, size_t d, size_t warp_n,
                            uint32_t bits, uint32_t k_axis, size_t g, int interleave,
                            size_t max_tokens, int* status) {
  *status = ORC_OK;
  if (batch == 0 || heads_kv == 0 || d == 0 || warp_n == 0) {
    *status = ORC_CONFIG_ERROR;
    return NULL;
  }
  if (!bits_ok(bits)) {
    *status = ORC_UNSUPPORTED_BITS;
    return NULL;
  }
  const size_t n_r = orc_residual_block_size(bits, warp_n);
  if (bits != 16) {
    if (g == 0 || d % g != 0 || (k_axis == 0 && n_r % g != 0)) {
      *status = ORC_CONFIG_ERROR;
      return NULL;
    }
  }
  orc_cache* c = (orc_cache*)calloc(1, sizeof(orc_cache));
  c->batch = batch;
  c->heads_kv = heads_kv;
  c->d = d;
  c->warp_n = warp_n;
  c->n_r = n_r;
  c->g = g;
  c->bits = bits;
  c->k_axis = k_axis;
  c->interleave = interleave;
  c->max_blocks = max_tokens / n_r + 1;
  c->wpb = d * n_r / (16 / bits);
  c->kpc = orc_param_count(n_r, d, bits, k_axis, g);
  c->vpc = orc_param_count(n_r, d, bits, 1, g);
  const size_t cells = batch * heads_kv;
  c->packed_len = (size_t*)calloc(cells, sizeof(size_t));
  c->res_len = (size_t*)calloc(cells, sizeof(size_t));
  c->kw = (uint16_t*)malloc(cells * c->max_blocks * c->wpb * 2);
  c->vw = (uint16_t*)malloc(cells * c->max_blocks * c->wpb * 2);
  c->kp = (uint16_t*)malloc(cells * c->max_blocks * (c->kpc + 1) * 2);
  c->vp = (uint16_t*)malloc(cells * c->max_blocks * (c->vpc + 1) * 2);
  c->rk = (float*)malloc(cells * n_r * d * 4);
  c->rv = (float*)malloc(cells * n_r * d * 4);
  if (!c->kw || !c->vw || !c->kp || !c->vp || !c->rk || !c->rv) {
    orc_cache_destroy(c);
    *status = ORC_CAPACITY_ERROR;
    return NULL;
  }
  return c;
}

void orc_cache_destroy(orc_cache* c) {
  if (!c) return;
  free(c->packed_len);
  free(c->res_len);
  free(c->kw);
  free(c->vw);
  free(c->kp);
  free(c->vp);
  free(c->rk);
  free(c->rv);
  free(c);
}

static size_t cell_of(const orc_cache* c, size_t b, size_t h) { return b * c->heads_kv + h; }
size_t orc_cache_packed_len(const orc_cache* c, size_t b, size_t h) {
  return c->packed_len[cell_of(c, b, h)];
}
size_t orc_cache_res_len(const orc_cache* c, size_t b, size_t h) {
  return c->res_len[cell_of(c, b, h)];
}
size_t orc_cache_words_per_block(const orc_cache* c) { return c->wpb; }
size_t orc_cache_k_param_count(const orc_cache* c) { return c->kpc; }
size_t orc_cache_v_param_count(const orc_cache* c) { return c->vpc; }

static uint16_t* blk_kw(const orc_cache* c, size_t cell, size_t i) {
  return c->kw + (cell * c->max_blocks + i) * c->wpb;
}
static uint16_t* blk_vw(const orc_cache* c, size_t cell, size_t i) {
  return c->vw + (cell * c->max_blocks + i) * c->wpb;
}
static uint16_t* blk_kp(const orc_cache* c, size_t cell, size_t i) {
  return c->kp + (cell * c->max_blocks + i) * (c->kpc + 1);
}
static uint16_t* blk_vp(const orc_cache* c, size_t cell, size_t i) {
  return c->vp + (cell * c->max_blocks + i) * (c->vpc + 1);
}

const uint16_t* orc_cache_block(const orc_cache* c, size_t b, size_t h, size_t blk, int which) {
  const size_t cell = cell_of(c, b, h);
  if (blk >= c->packed_len[cell] / c->n_r) return NULL;
  switch (which) {
    case 0: return blk_kw(c, cell, blk);
    case 1: return blk_vw(c, cell, blk);
    case 2: return blk_kp(c, cell, blk);
    default: return blk_vp(c, cell, blk);
  }
}

const float* orc_cache_residual(const orc_cache* c, size_t b, size_t h, int which) {
  const size_t cell = cell_of(c, b, h);
  return (which == 0 ? c->rk : c->rv) + cell * c->n_r * c->d;
}

/* kvcache.cpp:184-206 into a block slot */
static int build_into(orc_cache* c, size_t cell, size_t slot, const float* k, const float* v) {
  if (slot >= c->max_blocks) return ORC_CAPACITY_ERROR;
  return orc_make_block(k, v, c->n_r, c->d, c->bits, c->k_axis, c->g, c->interleave,
                        blk_kw(c, cell, slot), blk_vw(c, cell, slot), blk_kp(c, cell, slot),
                        blk_vp(c, cell, slot));
}

/* kvcache.cpp:170-182 append_token */
int orc_cache_append(orc_cache* c, size_t b, size_t h, const float* k_row, const float* v_row) {
  const size_t cell = cell_of(c, b, h);
  if (c->res_len[cell] == c->n_r) return ORC_CAPACITY_ERROR;
  const size_t r = c->res_len[cell];
  memcpy(c->rk + (cell * c->n_r + r) * c->d, k_row, c->d * 4);
  memcpy(c->rv + (cell * c->n_r + r) * c->d, v_row, c->d * 4);
  c->res_len[cell] = r + 1;
  return ORC_OK;
}

/* kvcache.cpp:155-168 prefill */
int orc_cache_prefill(orc_cache* c, size_t b, size_t h, const float* k, const float* v,
                      size_t len) {
  const size_t cell = cell_of(c, b, h);
  if (c->packed_len[cell] != 0 || c->res_len[cell] != 0) return ORC_STATE_ERROR;
  const size_t n_p = len - len % c->n_r;
  if (n_p / c->n_r > c->max_blocks) return ORC_CAPACITY_ERROR;
  for (size_t t0 = 0; t0 < n_p; t0 += c->n_r) {
    int st = build_into(c, cell, t0 / c->n_r, k + t0 * c->d, v + t0 * c->d);
    if (st) return st;
  }
  c->packed_len[cell] = n_p;
  for (size_t t = n_p; t < len; ++t) orc_cache_append(c, b, h, k + t * c->d, v + t * c->d);
  return ORC_OK;
}

/* kvcache.cpp:245-251 flush_residual = commit_block(build_block) */
int orc_cache_flush(orc_cache* c, size_t b, size_t h) {
  const size_t cell = cell_of(c, b, h);
  if (c->res_len[cell] != c->n_r) return ORC_STATE_ERROR;
  int st = build_into(c, cell, c->packed_len[cell] / c->n_r, c->rk + cell * c->n_r * c->d,
                      c->rv + cell * c->n_r * c->d);
  if (st) return st;
  c->packed_len[cell] += c->n_r;
  c->res_len[cell] = 0;
  return ORC_OK;
}

/* kvcache.cpp:263-312 for tokens [t0, t0+len) of the packed segment */
static void packed_tile(const orc_cache* c, size_t cell, size_t t0, size_t len, float* k_out,
                        float* v_out, float* scratch_k, float* scratch_v) {
  size_t written = 0;
  const size_t d = c->d;
  while (written < len) {
    const size_t t = t0 + written;
    const size_t bi = t / c->n_r, local = t % c->n_r;
    size_t take = c->n_r - local;
    if (len - written < take) take = len - written;
    orc_dequant_block(blk_kw(c, cell, bi), blk_vw(c, cell, bi), blk_kp(c, cell, bi),
                      blk_vp(c, cell, bi), c->n_r, d, c->bits, c->k_axis, c->g, c->interleave,
                      scratch_k, scratch_v);
    memcpy(k_out + written * d, scratch_k + local * d, take * d * 4);
    memcpy(v_out + written * d, scratch_v + local * d, take * d * 4);
    written += take;
  }
}

/* kvcache.cpp:314-324 */
int orc_cache_reconstruct(const orc_cache* c, size_t b, size_t h, float* k_out, float* v_out) {
  const size_t cell = cell_of(c, b, h);
  const size_t plen = c->packed_len[cell], d = c->d;
  float* sk = (float*)malloc(c->n_r * d * 4);
  float* sv = (float*)malloc(c->n_r * d * 4);
  if (plen) packed_tile(c, cell, 0, plen, k_out, v_out, sk, sv);
  free(sk);
  free(sv);
  memcpy(k_out + plen * d, c->rk + cell * c->n_r * d, c->res_len[cell] * d * 4);
  memcpy(v_out + plen * d, c->rv + cell * c->n_r * d, c->res_len[cell] * d * 4);
  return ORC_OK;
}

/* ------------------------------------------------------------- attention */

typedef struct {
  size_t rows, d;
  float *o, *m, *l;
} partial;

static void partial_init(partial* p, size_t rows, size_t d) {
  p->rows = rows;
  p->d = d;
  p->o = (float*)calloc(rows * d, 4);
  p->m = (float*)malloc(rows * 4);
  p->l = (float*)calloc(rows, 4);
  for (size_t i = 0; i < rows; ++i) p->m[i] = -INFINITY;
}
static void partial_free(partial* p) {
  free(p->o);
  free(p->m);
  free(p->l);
}

/* attention.cpp:52-90 attend_tile (the W_n-partitioned row max of :32-50 is
 * an exact max, so it is taken directly) */
static void attend_tile(partial* st, const float* q, const float* k, const float* v,
                        size_t tile_n, size_t d, float scale_factor, float* s) {
  const size_t rows = st->rows;
  for (size_t i = 0; i < rows; ++i) {
    for (size_t j = 0; j < tile_n; ++j) {
      float acc = 0.0f;
      for (size_t c = 0; c < d; ++c) acc += q[i * d + c] * k[j * d + c];
      s[i * tile_n + j] = acc * scale_factor;
    }
  }
  for (size_t i = 0; i < rows; ++i) {
    float tmax = -INFINITY;
    for (size_t j = 0; j < tile_n; ++j) tmax = tmax < s[i * tile_n + j] ? s[i * tile_n + j] : tmax;
    const float m_new = st->m[i] < tmax ? tmax : st->m[i];
    const float rescale = st->m[i] == -INFINITY ? 0.0f : expf(st->m[i] - m_new);
    float rowsum = 0.0f;
    for (size_t j = 0; j < tile_n; ++j) {
      const float p = expf(s[i * tile_n + j] - m_new);
      s[i * tile_n + j] = p;
      rowsum += p;
    }
    float* o = st->o + i * d;
    for (size_t c = 0; c < d; ++c) {
      float acc = 0.0f;
      for (size_t j = 0; j < tile_n; ++j) acc += s[i * tile_n + j] * v[j * d + c];
      o[c] = acc + rescale * o[c];
    }
    st->l[i] = st->l[i] * rescale + rowsum;
    st->m[i] = m_new;
  }
}

/* attention.cpp:142-162 combine (partials in list order) */
static void combine(const partial* ps, size_t n, float* out) {
  const size_t rows = ps[0].rows, d = ps[0].d;
  memset(out, 0, rows * d * 4);
  for (size_t i = 0; i < rows; ++i) {
    float m_star = -INFINITY;
    for (size_t p = 0; p < n; ++p) m_star = m_star < ps[p].m[i] ? ps[p].m[i] : m_star;
    float l = 0.0f;
    for (size_t p = 0; p < n; ++p) {
      const float w = ps[p].m[i] == -INFINITY ? 0.0f : expf(ps[p].m[i] - m_star);
      l += ps[p].l[i] * w;
      for (size_t c = 0; c < d; ++c) out[i * d + c] += ps[p].o[i * d + c] * w;
    }
    for (size_t c = 0; c < d; ++c) out[i * d + c] /= l;
  }
}

typedef struct {
  orc_cache* c;
  size_t heads_q, tile_n, num_splits, n_group;
  const float* q;
  float* out;
  int* pending; /* per cell: 1 if the residual was full */
  size_t next;
  pthread_mutex_t mu;
} step_ctx;

/* per-cell body of decode_step (attention.cpp:203-232) */
static void decode_cell(step_ctx* x, size_t item) {
  orc_cache* c = x->c;
  const size_t d = c->d, ng = x->n_group, b = item / c->heads_kv, h = item % c->heads_kv;
  const float inv_sqrt_d = 1.0f / sqrtf((float)d);
  float* q_tile = (float*)malloc(ng * d * 4);
  for (size_t g = 0; g < ng; ++g)
    for (size_t cc = 0; cc < d; ++cc)
      q_tile[g * d + cc] = x->q[(b * x->heads_q + h * ng + g) * d + cc] * inv_sqrt_d;

  const size_t plen = c->packed_len[item];
  const size_t n_tiles = (plen + x->tile_n - 1) / x->tile_n;
  const size_t splits = x->num_splits < 1 ? 1 : x->num_splits;
  partial* ps = (partial*)calloc(splits + 1, sizeof(partial));
  size_t nps = 0;
  const size_t smax = (x->tile_n > c->n_r ? x->tile_n : c->n_r);
  float* s = (float*)malloc(ng * smax * 4);

  /* residual_attend (attention.cpp:92-105) */
  const size_t rlen = c->res_len[item];
  partial_init(&ps[nps], ng, d);
  attend_tile(&ps[nps], q_tile, c->rk + item * c->n_r * d, c->rv + item * c->n_r * d, rlen, d,
              1.0f, s);
  ++nps;
  x->pending[item] = rlen == c->n_r;

  /* packed_attend (attention.cpp:107-140) */
  if (plen > 0) {
    const size_t base = n_tiles / splits, rem = n_tiles % splits;
    float* kt = (float*)malloc(x->tile_n * d * 4);
    float* vt = (float*)malloc(x->tile_n * d * 4);
    float* sk = (float*)malloc(c->n_r * d * 4);
    float* sv = (float*)malloc(c->n_r * d * 4);
    size_t tile_begin = 0;
    for (size_t sp = 0; sp < splits; ++sp) {
      const size_t count = base + (sp < rem ? 1 : 0);
      if (count == 0) continue;
      const size_t t_begin = tile_begin * x->tile_n;
      size_t t_end = (tile_begin + count) * x->tile_n;
      if (t_end > plen) t_end = plen;
      tile_begin += count;
      partial_init(&ps[nps], ng, d);
      for (size_t t0 = t_begin; t0 < t_end; t0 += x->tile_n) {
        const size_t len = x->tile_n < t_end - t0 ? x->tile_n : t_end - t0;
        packed_tile(c, item, t0, len, kt, vt, sk, sv);
        attend_tile(&ps[nps], q_tile, kt, vt, len, d, 1.0f, s);
      }
      ++nps;
    }
    free(kt);
    free(vt);
    free(sk);
    free(sv);
  }
  float* merged = (float*)malloc(ng * d * 4);
  combine(ps, nps, merged);
  for (size_t g = 0; g < ng; ++g)
    memcpy(x->out + (b * x->heads_q + h * ng + g) * d, merged + g * d, d * 4);
  for (size_t i = 0; i < nps; ++i) partial_free(&ps[i]);
  free(ps);
  free(merged);
  free(s);
  free(q_tile);
}

static void* worker(void* arg) {
  step_ctx* x = (step_ctx*)arg;
  const size_t items = x->c->batch * x->c->heads_kv;
  for (;;) {
    pthread_mutex_lock(&x->mu);
    const size_t i = x->next++;
    pthread_mutex_unlock(&x->mu);
    if (i >= items) break;
    decode_cell(x, i);
  }
  return NULL;
}

/* attention.cpp:164-242 decode_step */
int orc_decode_step(orc_cache* c, size_t heads_q, size_t tile_n, size_t num_splits,
                    size_t warp_n, const float* q, const float* k_new, const float* v_new,
                    float* out, int threads) {
  (void)warp_n; /* only shapes the (exact) partitioned row max */
  if (heads_q == 0 || heads_q % c->heads_kv != 0 || tile_n == 0 || num_splits < 1)
    return ORC_CONFIG_ERROR;
  const size_t d = c->d, items = c->batch * c->heads_kv;
  /* append phase (attention.cpp:181-190); reference appends cell by cell and
   * would throw CapacityError on the first full residual */
  for (size_t i = 0; i < items; ++i)
    if (c->res_len[i] == c->n_r) return ORC_CAPACITY_ERROR;
  for (size_t i = 0; i < items; ++i)
    orc_cache_append(c, i / c->heads_kv, i % c->heads_kv, k_new + i * d, v_new + i * d);

  step_ctx x;
  x.c = c;
  x.heads_q = heads_q;
  x.tile_n = tile_n;
  x.num_splits = num_splits;
  x.n_group = heads_q / c->heads_kv;
  x.q = q;
  x.out = out;
  x.pending = (int*)calloc(items, sizeof(int));
  x.next = 0;
  pthread_mutex_init(&x.mu, NULL);
  size_t nt = threads > 0 ? (size_t)threads : (size_t)sysconf(_SC_NPROCESSORS_ONLN);
  if (nt > items) nt = items;
  if (nt <= 1) {
    for (size_t i = 0; i < items; ++i) decode_cell(&x, i);
  } else {
    pthread_t* th = (pthread_t*)malloc(nt * sizeof(pthread_t));
    for (size_t t = 0; t < nt; ++t) pthread_create(&th[t], NULL, worker, &x);
    for (size_t t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&x.mu);
  /* cache-update phase (attention.cpp:235-240) */
  int st = ORC_OK;
  for (size_t i = 0; i < items; ++i)
    if (x.pending[i] && !st) st = orc_cache_flush(c, i / c->heads_kv, i % c->heads_kv);
  free(x.pending);
  return st;
}

/* --------------------------------------------------------------- oracle.cpp */

/* oracle.cpp:12-37 */
void orc_naive_attention(const float* q, size_t q_rows, const float* k, const float* v,
                         size_t len, size_t d, float* out) {
  const float inv_sqrt_d = 1.0f / sqrtf((float)d);
  float* scores = (float*)malloc((len ? len : 1) * 4);
  for (size_t i = 0; i < q_rows; ++i) {
    for (size_t j = 0; j < len; ++j) {
      float s = 0.0f;
      for (size_t c = 0; c < d; ++c) s += q[i * d + c] * k[j * d + c];
      scores[j] = s * inv_sqrt_d;
    }
    float m = -INFINITY;
    for (size_t j = 0; j < len; ++j) m = m < scores[j] ? scores[j] : m;
    float l = 0.0f;
    for (size_t j = 0; j < len; ++j) {
      scores[j] = expf(scores[j] - m);
      l += scores[j];
    }
    for (size_t c = 0; c < d; ++c) {
      float acc = 0.0f;
      for (size_t j = 0; j < len; ++j) acc += scores[j] * v[j * d + c];
      out[i * d + c] = acc / l;
    }
  }
  free(scores);
}

/* oracle.cpp:42-61 reference_roundtrip_group */
static void roundtrip_group(const float* x, size_t stride, size_t n, uint32_t bits, float* out) {
  float lo = x[0], hi = x[0];
  for (size_t i = 1; i < n; ++i) {
    lo = x[i * stride] < lo ? x[i * stride] : lo;
    hi = hi < x[i * stride] ? x[i * stride] : hi;
  }
  const float qmax = (float)((1u << bits) - 1u);
  float scale = orc_round_f16((hi - lo) / qmax);
  if (!(scale >= kMinScale)) scale = kMinScale;
  const float zero = orc_round_f16(lo);
  for (size_t i = 0; i < n; ++i) {
    float c = nearbyintf((x[i * stride] - zero) / scale);
    c = c < 0.0f ? 0.0f : (qmax < c ? qmax : c);
    out[i * stride] = orc_round_f16(c * scale + zero);
  }
}

/* oracle.cpp:84-96 offline_quant_reference */
void orc_offline_quant_reference(const float* k, const float* v, size_t len, size_t d,
                                 uint32_t bits, uint32_t k_axis, size_t g, size_t n_r,
                                 float* k_out, float* v_out) {
  memcpy(k_out, k, len * d * 4);
  memcpy(v_out, v, len * d * 4);
  if (bits == 16) return;
  const size_t full = len - len % n_r;
  for (size_t t0 = 0; t0 < full; t0 += n_r) {
    for (int which = 0; which < 2; ++which) {
      const float* src = (which ? v : k) + t0 * d;
      float* dst = (which ? v_out : k_out) + t0 * d;
      const uint32_t axis = which ? 1u : k_axis;
      if (axis == 0) {
        for (size_t gr = 0; gr < n_r / g; ++gr)
          for (size_t c = 0; c < d; ++c)
            roundtrip_group(src + gr * g * d + c, d, g, bits, dst + gr * g * d + c);
      } else {
        for (size_t t = 0; t < n_r; ++t)
          for (size_t gc = 0; gc < d / g; ++gc)
            roundtrip_group(src + t * d + gc * g, 1, g, bits, dst + t * d + gc * g);
      }
    }
  }
}

/* ------------------------------------------------------------- bench.cpp */

/* std::mt19937_64 (the C++ standard fixes its output sequence) */
void orc_gauss_init(orc_gauss* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
  g->has_spare = 0;
  g->spare = 0.0;
}

static uint64_t mt_next(orc_gauss* g) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  if (g->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1ULL];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[x & 1ULL];
    }
    x = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ MAG[x & 1ULL];
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* bench.cpp:32-35: (0, 1] */
static double uniform01(orc_gauss* g) { return ((double)(mt_next(g) >> 11) + 1.0) * 0x1.0p-53; }

/* bench.cpp:18-30 Box-Muller with a cached spare */
float orc_gauss_next(orc_gauss* g) {
  if (g->has_spare) {
    g->has_spare = 0;
    return (float)g->spare;
  }
  const double u1 = uniform01(g), u2 = uniform01(g);
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  g->spare = r * sin(theta);
  g->has_spare = 1;
  return (float)(r * cos(theta));
}

void orc_gauss_fill_rounded(orc_gauss* g, float* dst, size_t n) {
  for (size_t i = 0; i < n; ++i) dst[i] = orc_round_f16(orc_gauss_next(g));
}

/* The same stream as orc_gauss_fill_rounded, with the Box-Muller transforms
 * (log/sqrt/sin/cos, the cost) spread over threads: the Mersenne Twister
 * words are drawn sequentially, then pair k = (u1, u2) gives outputs 2k
 * (r cos) and 2k+1 (r sin) independently.  Bit-identical to the sequential
 * fill (tests/test_oracle.py). */
typedef struct {
  const uint64_t* raw;
  float* dst;
  size_t p0, p1;
} gauss_job;

static void* gauss_pairs(void* arg) {
  const gauss_job* j = (const gauss_job*)arg;
  for (size_t k = j->p0; k < j->p1; ++k) {
    const double u1 = ((double)(j->raw[2 * k] >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = ((double)(j->raw[2 * k + 1] >> 11) + 1.0) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    j->dst[2 * k] = orc_round_f16((float)(r * cos(theta)));
    j->dst[2 * k + 1] = orc_round_f16((float)(r * sin(theta)));
  }
  return NULL;
}

void orc_gauss_fill_rounded_par(orc_gauss* g, float* dst, size_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  size_t i = 0;
  if (n && g->has_spare) dst[i++] = orc_round_f16(orc_gauss_next(g));
  const size_t chunk_pairs = (size_t)1 << 22;
  uint64_t* raw = (uint64_t*)malloc(2 * chunk_pairs * sizeof(uint64_t));
  while (raw && n - i >= 2) {
    const size_t pairs = (n - i) / 2 < chunk_pairs ? (n - i) / 2 : chunk_pairs;
    for (size_t k = 0; k < 2 * pairs; ++k) raw[k] = mt_next(g);
    pthread_t tid[64];
    gauss_job job[64];
    const int nt = pairs < 4096 ? 1 : threads;
    for (int t = 0; t < nt; ++t) {
      job[t].raw = raw;
      job[t].dst = dst + i;
      job[t].p0 = pairs * t / nt;
      job[t].p1 = pairs * (t + 1) / nt;
      if (t > 0) pthread_create(&tid[t], NULL, gauss_pairs, &job[t]);
    }
    gauss_pairs(&job[0]);
    for (int t = 1; t < nt; ++t) pthread_join(tid[t], NULL);
    i += 2 * pairs;
  }
  free(raw);
  for (; i < n; ++i) dst[i] = orc_round_f16(orc_gauss_next(g));
}

void orc_gauss_fill_f16(orc_gauss* g, uint16_t* dst, size_t n) {
  for (size_t i = 0; i < n; ++i) dst[i] = orc_f32_to_f16_bits(orc_gauss_next(g));
}

/* bench.cpp:37-45 */
uint64_t orc_fnv1a64(const void* data, size_t len, uint64_t h) {
  const uint8_t* p = (const uint8_t*)data;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
