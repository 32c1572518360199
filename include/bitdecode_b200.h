/*
 * bitdecode_b200.h -- C-ABI drop-in boundary for the BitDecoding decode hot
 * path on B200 (sm_100a).  Plain C: pointers, sizes, status codes; no C++
 * types, no torch types, no exceptions cross this boundary.
 *
 * Every entry point replaces one piece of the reference engine's C++ API
 * (/root/reference/proj/include/bitkv, "bitkv::"), cited per function.  The
 * C++ drop-in (include/bitkv_b200.hpp) and the Python binding
 * (paper_2503_18773_b200/bitkv.py) re-expose the reference API on top of it;
 * INTEGRATION.md shows how a reference-side caller binds it.
 *
 * Memory model: the cache lives in device memory (HBM) and is owned by the
 * library.  Tensor arguments named *_dev are device pointers to binary16
 * values (row-major, the reference shapes); *_host arguments are host fp32
 * arrays holding binary16-representable values (the reference Tensor
 * contract, tensor.hpp:16-46).  `stream` is a cudaStream_t (NULL = legacy
 * default stream); device-pointer calls are stream-ordered and asynchronous.
 */
#ifndef BITDECODE_B200_H
#define BITDECODE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BDK_API __attribute__((visibility("default")))
#else
#define BDK_API
#endif

/* 1:1 with the reference exception classes (errors.hpp:14-54). */
typedef enum bdk_status {
  BDK_OK = 0,
  BDK_CONFIG_ERROR = 1,     /* bitkv::ConfigError */
  BDK_SHAPE_ERROR = 2,      /* bitkv::ShapeError */
  BDK_UNSUPPORTED_BITS = 3, /* bitkv::UnsupportedBits */
  BDK_CODE_OVERFLOW = 4,    /* bitkv::CodeOverflow */
  BDK_CAPACITY_ERROR = 5,   /* bitkv::CapacityError */
  BDK_STATE_ERROR = 6,      /* bitkv::StateError */
  BDK_FORMAT_ERROR = 7,     /* bitkv::FormatError */
  BDK_EMPTY_INPUT = 8,      /* bitkv::EmptyInput */
  BDK_CUDA_ERROR = 20,      /* device / driver failure (message in bdk_last_error) */
  BDK_UNSUPPORTED = 21,     /* geometry outside the sm_100a kernels' envelope */
  BDK_INVALID_ARGUMENT = 22 /* NULL handle / pointer */
} bdk_status;

typedef struct bdk_cache bdk_cache;

/* KVCache(batch, heads_kv, head_dim, warp_n, QuantSpec{num_bits, k_axis,
 * group_size}, Contiguous, page_size, max_pages, interleave)
 * (kvcache.hpp:107-109, quant.hpp:19-25).  max_tokens is the per-cell token
 * capacity the device arena is sized for (the reference grows vectors). */
typedef struct bdk_cache_desc {
  uint32_t batch;
  uint32_t heads_kv;
  uint32_t head_dim;
  uint32_t warp_n;
  uint32_t num_bits;   /* 2, 4, 8, or 16 (fp16 passthrough) */
  uint32_t k_axis;     /* 0 = QuantAxis::KChannel, 1 = QuantAxis::KToken */
  uint32_t group_size;
  uint32_t interleave; /* 1 = interleave_order, 0 = identity_order */
  uint32_t max_tokens;
  int32_t device;
} bdk_cache_desc;

/* AttentionConfig (config.hpp:13-25). */
typedef struct bdk_attn_config {
  uint32_t batch;
  uint32_t heads_q;
  uint32_t heads_kv;
  uint32_t head_dim;
  uint32_t tile_m;
  uint32_t tile_n;
  uint32_t num_splits;
  uint32_t warp_n;
  uint32_t warp_m;
} bdk_attn_config;

typedef struct bdk_cache_info {
  uint32_t n_r;             /* KVCache::n_r(), residual_block_size (layout.cpp:74-77) */
  uint32_t pack_num;        /* 16 / num_bits */
  uint32_t words_per_block; /* u16 words per block per tensor */
  uint32_t k_param_u16;     /* QuantParams::data.size() per block, K */
  uint32_t v_param_u16;     /* ... V */
  uint32_t record_bytes;    /* device block-record stride */
  uint32_t max_blocks;      /* block slots per cell */
  uint32_t fast_path;       /* 1 if the tensor-core decode kernel serves this geometry */
} bdk_cache_info;

/* ---------------------------------------------------------------- errors */
BDK_API const char* bdk_last_error(void);         /* thread-local message */
BDK_API const char* bdk_status_name(bdk_status s); /* "ConfigError", ... */

/* validate_config (config.hpp:29, config.cpp:10-30) */
BDK_API bdk_status bdk_validate_config(const bdk_attn_config* cfg);

/* ------------------------------------------------------- cache lifetime */
/* KVCache::KVCache (kvcache.cpp:114-148) */
BDK_API bdk_status bdk_cache_create(const bdk_cache_desc* desc, bdk_cache** out);
BDK_API bdk_status bdk_cache_destroy(bdk_cache* cache);
BDK_API bdk_status bdk_cache_get_info(const bdk_cache* cache, bdk_cache_info* info);
/* KVCache::packed_len / res_len (kvcache.hpp:145-147) */
BDK_API bdk_status bdk_cache_lengths(const bdk_cache* cache, uint32_t b, uint32_t h,
                                     uint32_t* packed_len, uint32_t* res_len);

/* Empty every cell (packed_len = res_len = 0), stream-ordered; the arena is
 * kept.  Equivalent to constructing a fresh KVCache of the same geometry
 * (kvcache.cpp:114-148) without reallocating device memory. */
BDK_API bdk_status bdk_cache_reset(bdk_cache* cache, void* stream);

/* ------------------------------------------------- cache state machine */
/* KVCache::prefill (kvcache.cpp:155-168): fused quantize+pack of the first
 * len - len % N_r tokens (bit-exact), tail into the residual.
 * k_dev/v_dev: binary16 [len][head_dim]. */
BDK_API bdk_status bdk_prefill(bdk_cache* cache, uint32_t b, uint32_t h, const void* k_dev,
                               const void* v_dev, uint32_t len, void* stream);
/* prefill of every cell with the same length; k_dev/v_dev:
 * [batch][heads_kv][len][head_dim] (run_bench's prefill loop,
 * bench.cpp:132-139, in one launch). */
BDK_API bdk_status bdk_prefill_all(bdk_cache* cache, const void* k_dev, const void* v_dev,
                                   uint32_t len, void* stream);
/* Host-buffer variants (binary16 bits in host memory; synchronous): the entry
 * points the C++ drop-in (bitkv_b200.hpp) binds for the reference's
 * host-pointer API (KVCache::prefill / append_token / packed_tile). */
BDK_API bdk_status bdk_prefill_host(bdk_cache* cache, uint32_t b, uint32_t h,
                                    const uint16_t* k_host, const uint16_t* v_host, uint32_t len);
BDK_API bdk_status bdk_append_token_host(bdk_cache* cache, uint32_t b, uint32_t h,
                                         const uint16_t* k_row_host, const uint16_t* v_row_host);
/* KVCache::packed_tile (kvcache.cpp:263-312): dequantized tokens
 * [t0, t0 + len) of the packed segment, binary16 bits [len][head_dim]. */
BDK_API bdk_status bdk_packed_tile_host(const bdk_cache* cache, uint32_t b, uint32_t h, uint32_t t0,
                                        uint32_t len, uint16_t* k_host, uint16_t* v_host);
/* KVCache::append_token (kvcache.cpp:170-182); rows binary16 [head_dim]. */
BDK_API bdk_status bdk_append_token(bdk_cache* cache, uint32_t b, uint32_t h,
                                    const void* k_row_dev, const void* v_row_dev, void* stream);
/* KVCache::flush_residual (kvcache.cpp:245-251). */
BDK_API bdk_status bdk_flush_residual(bdk_cache* cache, uint32_t b, uint32_t h, void* stream);

/* ----------------------------------------------------------- decode step */
/* decode_step (attention.hpp:87-88, attention.cpp:164-242): append the new
 * token of every cell, residual + packed split-KV attention, LSE combine,
 * commit of any full residual block.
 * q_dev [batch][heads_q][d], k_new_dev/v_new_dev [batch][heads_kv][d]
 * (binary16), out_dev fp32 [batch][heads_q][d]. */
BDK_API bdk_status bdk_decode_step(bdk_cache* cache, const bdk_attn_config* cfg,
                                   const void* q_dev, const void* k_new_dev,
                                   const void* v_new_dev, float* out_dev, void* stream);
/* A CUDA graph of n_steps consecutive decode steps (decode_step,
 * attention.cpp:164-242, Algorithm 2's steady-state loop): step i reads
 * q_dev + i*batch*heads_q*d, k_new_dev/v_new_dev + i*batch*heads_kv*d
 * (binary16) and writes out_dev + i*batch*heads_q*d (fp32).  Every step is
 * a fixed pair of launches -- the attention grid (append, residual and
 * packed attention) and its combine grid (LSE merge, length commit and the
 * flush of a residual window that fills, build_block + commit_block,
 * kvcache.cpp:208-237) -- scheduled on the device from the cache's device
 * lengths, so one captured
 * graph replays correctly at any cache state, flush steps included, and
 * bit-identically to the same steps run eagerly.  Fast mode only
 * (bdk_set_precise(cache, 0); else BDK_UNSUPPORTED).  Each launch checks the
 * host mirror's capacity for n_steps more tokens first (CapacityError) and
 * advances it.  The graph keeps pointers to the cache's workspaces: destroy
 * it before the cache. */
typedef struct bdk_graph bdk_graph;
BDK_API bdk_status bdk_graph_create(bdk_cache* cache, const bdk_attn_config* cfg,
                                    const void* q_dev, const void* k_new_dev,
                                    const void* v_new_dev, float* out_dev, uint32_t n_steps,
                                    bdk_graph** graph);
BDK_API bdk_status bdk_graph_launch(bdk_graph* graph, void* stream);
BDK_API bdk_status bdk_graph_destroy(bdk_graph* graph);
/* Same contract with host fp32 tensors (the reference's by-value Tensor /
 * AttnOutput interface); synchronous; host<->device copies included. */
BDK_API bdk_status bdk_decode_step_host(bdk_cache* cache, const bdk_attn_config* cfg,
                                        const float* q_host, const float* k_new_host,
                                        const float* v_new_host, float* out_host);
/* Partial decode for sequence-split multi-GPU: attends packed blocks
 * [blk_begin, blk_end) of every cell plus (unless flags has
 * BDK_PARTIAL_NO_RESIDUAL) the residual window; appends only when
 * k_new_dev != NULL.  Writes the NORMALIZED partial output out_dev
 * [batch][heads_q][d] and its log2-sum-exp lse_dev [batch][heads_q]; the
 * partials of all ranks merge with bdk_merge_partials (combine,
 * attention.cpp:142-162). */
#define BDK_PARTIAL_NO_RESIDUAL 1u
BDK_API bdk_status bdk_decode_partial(bdk_cache* cache, const bdk_attn_config* cfg,
                                      const void* q_dev, const void* k_new_dev,
                                      const void* v_new_dev, uint32_t blk_begin,
                                      uint32_t blk_end, uint32_t flags, float* out_dev,
                                      float* lse_dev, void* stream);
/* LSE merge of n_parts normalized partials: part p is o_dev + p*o_stride
 * ([rows][d] fp32) and lse_dev + p*lse_stride ([rows], log2 domain), strides
 * in floats (so one all-gathered [n_parts][rows*d + rows] buffer merges in
 * place) -> out_dev [rows][d]. */
BDK_API bdk_status bdk_merge_partials(const float* o_dev, const float* lse_dev, uint32_t n_parts,
                                      uint32_t rows, uint32_t d, uint64_t o_stride,
                                      uint64_t lse_stride, float* out_dev, void* stream);
/* Sequence-split exchange over peer memory, one launch per rank (the
 * all-gather + combine of attention.cpp:142-162 without NCCL): parts[p]
 * points at rank p's partial for this step ([rows*d] o then [rows] lse, as
 * bdk_decode_partial wrote it; a peer-mapped pointer for p != rank) and
 * flags[p] at rank p's u32 step counter.  The kernel publishes `step` in
 * flags[rank], waits until every peer's flag reaches it, reads the peers'
 * partials directly and LSE-merges into out [rows][d] (and out_lse).  Each
 * rank keeps two slots and uses slot step % 2.  A peer that does not publish
 * within timeout_ns (0 = 2 s) sets *err = 1 instead of hanging. */
BDK_API bdk_status bdk_peer_merge(const float* const* parts, uint32_t* const* flags,
                                  uint32_t world, uint32_t rank, uint64_t step, uint32_t rows,
                                  uint32_t d, float* out_dev, float* out_lse_dev, int* err_dev,
                                  uint64_t timeout_ns, void* stream);
/* ------------------------------------------------ attention internals
 * The reference's decode decomposition (attention.hpp:17-70), on the device,
 * host buffers in and out, synchronous.  A PartialOutput state is three
 * arrays: o [rows][d] (unnormalized), m [rows] (running max, -inf initially),
 * l [rows] (running exp-sum, 0 initially).
 * attend_tile (attention.cpp:52-90): one online-softmax step over tile_n
 * tokens k/v [tile_n][d]; state in/out.  warp_n only picks the row-max
 * partition, which does not change the result. */
BDK_API bdk_status bdk_attend_tile_host(float* o, float* m, float* l, uint32_t rows, uint32_t d,
                                        const float* q, const float* k, const float* v,
                                        uint32_t tile_n, float scale, uint32_t warp_n,
                                        int32_t device);
/* partitioned_rowmax (attention.cpp:32-50): ShapeError unless warp_n | cols. */
BDK_API bdk_status bdk_partitioned_rowmax_host(const float* s, uint32_t rows, uint32_t cols,
                                               uint32_t warp_n, float* out, int32_t device);
/* residual_attend (attention.cpp:92-105): one tile over the res_len residual
 * tokens of cell (b, h); state in/out; StateError if the residual is empty.
 * (The block build of a full residual is bdk_build_block.) */
BDK_API bdk_status bdk_residual_attend_host(const bdk_cache* cache, uint32_t b, uint32_t h,
                                            const float* q, uint32_t q_rows, float scale,
                                            float* o, float* m, float* l);
/* packed_attend (attention.cpp:107-140): the packed segment of cell (b, h)
 * in tiles of tile_n, num_splits contiguous tile ranges; writes the
 * *n_parts non-empty splits' states (capacity max(1, num_splits) each). */
BDK_API bdk_status bdk_packed_attend_host(const bdk_cache* cache, uint32_t b, uint32_t h,
                                          const float* q, uint32_t q_rows, uint32_t tile_n,
                                          uint32_t num_splits, float scale, float* o, float* m,
                                          float* l, uint32_t* n_parts);
/* combine (attention.cpp:142-162) of n_parts states (o [n_parts][rows][d],
 * m/l [n_parts][rows]) -> out [rows][d]; EmptyInput when n_parts == 0. */
BDK_API bdk_status bdk_combine_host(const float* o, const float* m, const float* l,
                                    uint32_t n_parts, uint32_t rows, uint32_t d, float* out,
                                    int32_t device);

/* Decode numerics of a cache.  1 = precise (the default for every new or
 * loaded cache): bit-faithful round_f16(code*scale + zero) dequant and the
 * P = P_hi + P_lo split PV, within the reference's own 1e-5 decode tolerance
 * (proj/tests/test_attention.cpp:350-441).  0 = fast: scales folded into Q and
 * P, fp16 P (the throughput kernel; rel-L2 ~1e-3), an
 * explicit opt-in. */
BDK_API bdk_status bdk_set_precise(bdk_cache* cache, int precise);

/* --------------------------------------------------------- readback/IO */
/* PackedBlock of cell (b, h) (kvcache.hpp:17-26) in the reference layout
 * (kvcache.cpp:79-95, quant.cpp:71/:88), host outputs; any pointer may be
 * NULL.  Sizes from bdk_cache_get_info. */
BDK_API bdk_status bdk_read_block(const bdk_cache* cache, uint32_t b, uint32_t h, uint32_t blk,
                                  uint16_t* k_words, uint16_t* v_words, uint16_t* k_params,
                                  uint16_t* v_params);
/* KVCache::build_block (kvcache.cpp:208-219): quantize + pack the full
 * residual into host word/param arrays without committing; StateError unless
 * res_len == N_r. */
BDK_API bdk_status bdk_build_block(bdk_cache* cache, uint32_t b, uint32_t h, uint16_t* k_words,
                                   uint16_t* v_words, uint16_t* k_params, uint16_t* v_params);
/* KVCache::commit_block (kvcache.cpp:231-237): adopt the block and clear the
 * residual; StateError unless res_len == N_r. */
BDK_API bdk_status bdk_commit_block(bdk_cache* cache, uint32_t b, uint32_t h,
                                    const uint16_t* k_words, const uint16_t* v_words,
                                    const uint16_t* k_params, const uint16_t* v_params);
/* KVCache::adopt_block (kvcache.cpp:239-243): append an already-packed block
 * (reference layout, host inputs). */
BDK_API bdk_status bdk_adopt_block(bdk_cache* cache, uint32_t b, uint32_t h,
                                   const uint16_t* k_words, const uint16_t* v_words,
                                   const uint16_t* k_params, const uint16_t* v_params);
/* KVCache::residual_tile (kvcache.cpp:253-261) as binary16 bits, host
 * [res_len][d] each. */
BDK_API bdk_status bdk_read_residual(const bdk_cache* cache, uint32_t b, uint32_t h,
                                     uint16_t* k_host, uint16_t* v_host);
/* KVCache::packed_tile dequant (kvcache.cpp:263-312) of blocks [blk0,
 * blk0+nblk) into binary16 device rows [nblk*N_r][d]. */
BDK_API bdk_status bdk_dequant_blocks(const bdk_cache* cache, uint32_t b, uint32_t h,
                                      uint32_t blk0, uint32_t nblk, void* k_out_dev,
                                      void* v_out_dev, void* stream);
/* KVCache::memory (kvcache.cpp:330-345): {k payload, v payload, params,
 * residual} bytes. */
BDK_API bdk_status bdk_memory(const bdk_cache* cache, uint64_t out[4]);

/* ------------------------------------------------- quant.hpp utilities */
/* quant.hpp:56-80 on the device, host buffers in/out (synchronous).
 * quantize_tile: x [rows][d] fp32 -> codes [rows][d] and params as (scale,
 * zero) binary16 pairs in push order: KChannel (axis 0) [rows/g][d], KToken
 * (axis 1) [rows][d/g] (quant.cpp:47-93); ShapeError unless g divides the
 * grouped extent.  dequantize_tile rounds every value to binary16 storage
 * (quant.cpp:95-110); dequantize_group does not (quant.cpp:40-44). */
BDK_API bdk_status bdk_quantize_tile(const float* x, uint32_t rows, uint32_t d, uint32_t num_bits,
                                     uint32_t axis, uint32_t group_size, uint16_t* codes,
                                     uint16_t* params, int32_t device);
BDK_API bdk_status bdk_dequantize_tile(const uint16_t* codes, const uint16_t* params,
                                       uint32_t rows, uint32_t d, uint32_t axis,
                                       uint32_t group_size, float* out, int32_t device);
BDK_API bdk_status bdk_compute_group_params(const float* x, uint32_t n, uint32_t num_bits,
                                            float* scale, float* zero, int32_t device);
BDK_API bdk_status bdk_quantize_group(const float* x, uint32_t n, float scale, float zero,
                                      uint32_t num_bits, uint16_t* codes, int32_t device);
BDK_API bdk_status bdk_dequantize_group(const uint16_t* codes, uint32_t n, float scale,
                                        float zero, float* values, int32_t device);

/* ------------------------------------------------ BDKV v1 cache files */
/* dump_cache / load_cache (serialize.hpp:11-23, serialize.cpp:87-194): the
 * reference's byte format.  bdk_dump_cache writes into buf (capacity bytes)
 * and sets *size; buf == NULL queries the size.  bdk_load_cache builds a new
 * cache (contiguous backend) with max(max_tokens, longest cell + N_r) token
 * capacity; bad magic / version / fields or truncation -> BDK_FORMAT_ERROR
 * with the byte offset in bdk_last_error(). */
BDK_API bdk_status bdk_dump_cache(const bdk_cache* cache, uint8_t* buf, uint64_t capacity,
                                  uint64_t* size);
BDK_API bdk_status bdk_load_cache(const uint8_t* buf, uint64_t size, uint32_t max_tokens,
                                  int32_t device, bdk_cache** out);
/* dump_cache_file / load_cache_file (serialize.hpp:22-23) */
BDK_API bdk_status bdk_dump_cache_file(const bdk_cache* cache, const char* path);
BDK_API bdk_status bdk_load_cache_file(const char* path, uint32_t max_tokens, int32_t device,
                                       bdk_cache** out);
/* KVCache::corrupt_word (kvcache.cpp:326-328): fault injection on K words. */
BDK_API bdk_status bdk_corrupt_word(bdk_cache* cache, uint32_t b, uint32_t h, uint32_t blk,
                                    uint32_t word, uint16_t value);
/* Attention-kernel timing: between begin and end every decode launch of the
 * cache records a CUDA event pair on its launching stream immediately around
 * the split-KV attention kernel.  end synchronizes on the events and returns
 * the summed kernel time and the number of launches (measurement hook for
 * bench.py's roofline; no reference counterpart). */
BDK_API bdk_status bdk_profile_begin(bdk_cache* cache);
BDK_API bdk_status bdk_profile_end(bdk_cache* cache, float* total_ms, uint32_t* launches);
/* Total sm_100a kernels launched on behalf of this cache so far (every entry
 * point; bench.py reports the delta over its timed region). */
BDK_API bdk_status bdk_launch_count(const bdk_cache* cache, uint64_t* n);
/* Blocks until all work on the cache's device is done; reports async errors. */
BDK_API bdk_status bdk_synchronize(void);

#ifdef __cplusplus
}
#endif
#endif /* BITDECODE_B200_H */
