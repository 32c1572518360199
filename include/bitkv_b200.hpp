// bitkv_b200.hpp -- C++20 drop-in for the reference engine's public API
// (/root/reference/proj/include/bitkv, namespace bitkv) over the sm_100a
// C-ABI in bitdecode_b200.h.
//
// Include this header INSTEAD of the reference headers and link
// libbitdecode_b200.so: the names, argument meaning, value semantics and
// exception classes follow the reference (cited per symbol), while the cache
// lives in HBM and every numeric step -- fused quantize+pack, dequant,
// decode attention, LSE combine -- runs in the CUDA kernels.  The only code in
// this header is host bookkeeping: shape checks, status -> exception mapping,
// and the binary16 <-> fp32 value conversions of the reference Tensor contract
// (tensor.hpp:16-46, all API values are binary16-representable).
//
// Extensions (documented, no reference counterpart): the KVCache constructor
// takes an optional per-cell token capacity (the device arena is sized once;
// the reference grows host vectors) and a CUDA device ordinal.
#pragma once

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <utility>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <istream>
#include <iterator>
#include <ostream>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "bitdecode_b200.h"

namespace bitkv {

// ------------------------------------------------------------ errors.hpp
struct Error : std::runtime_error {  // errors.hpp:9-12
  using std::runtime_error::runtime_error;
};
struct ConfigError : Error {  // errors.hpp:14-54
  using Error::Error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct UnsupportedBits : Error {
  using Error::Error;
};
struct CodeOverflow : Error {
  using Error::Error;
};
struct CapacityError : Error {
  using Error::Error;
};
struct StateError : Error {
  using Error::Error;
};
struct FormatError : Error {  // errors.hpp: carries the byte offset
  explicit FormatError(const std::string& m) : Error(m), offset(parse_offset(m)) {}
  size_t offset;

 private:
  static size_t parse_offset(const std::string& m) {
    const auto p = m.rfind("byte offset ");
    return p == std::string::npos ? 0 : static_cast<size_t>(std::stoull(m.substr(p + 12)));
  }
};
struct EmptyInput : Error {
  using Error::Error;
};
struct CudaError : Error {  // device / driver failure (no reference counterpart)
  using Error::Error;
};
struct Unsupported : Error {  // geometry outside the sm_100a kernels' envelope
  using Error::Error;
};

namespace detail {
inline void check(bdk_status s) {
  if (s == BDK_OK) return;
  const std::string msg = bdk_last_error();
  switch (s) {
    case BDK_CONFIG_ERROR: throw ConfigError(msg);
    case BDK_SHAPE_ERROR: throw ShapeError(msg);
    case BDK_UNSUPPORTED_BITS: throw UnsupportedBits(msg);
    case BDK_CODE_OVERFLOW: throw CodeOverflow(msg);
    case BDK_CAPACITY_ERROR: throw CapacityError(msg);
    case BDK_STATE_ERROR: throw StateError(msg);
    case BDK_FORMAT_ERROR: throw FormatError(msg);
    case BDK_EMPTY_INPUT: throw EmptyInput(msg);
    case BDK_CUDA_ERROR: throw CudaError(msg);
    case BDK_UNSUPPORTED: throw Unsupported(msg);
    default: throw Error(msg);
  }
}
}  // namespace detail

// -------------------------------------------------------------- fp16.hpp
// IEEE binary16 <-> binary32 with round-to-nearest-even (fp16.hpp:13-70).
inline uint16_t f32_to_f16_bits(float value) {
  return std::bit_cast<uint16_t>(static_cast<_Float16>(value));
}
inline float f16_bits_to_f32(uint16_t bits) {
  return static_cast<float>(std::bit_cast<_Float16>(bits));
}
inline float round_f16(float value) { return f16_bits_to_f32(f32_to_f16_bits(value)); }

// ------------------------------------------------------------ tensor.hpp
class Tensor {  // tensor.hpp:16-81: row-major fp32 storage of binary16 values
 public:
  Tensor() = default;
  explicit Tensor(std::vector<size_t> shape) : shape_(std::move(shape)) {
    data_.assign(count(shape_), 0.0f);
  }
  static Tensor from_values(std::vector<size_t> shape, const std::vector<float>& values) {
    Tensor t(std::move(shape));
    if (values.size() != t.data_.size())
      throw ShapeError("from_values: element count does not match shape");
    for (size_t i = 0; i < values.size(); ++i) t.data_[i] = round_f16(values[i]);
    return t;
  }
  const std::vector<size_t>& shape() const { return shape_; }
  size_t ndim() const { return shape_.size(); }
  size_t dim(size_t i) const { return shape_.at(i); }
  size_t numel() const { return data_.size(); }
  float at(size_t flat) const { return data_[flat]; }
  float operator()(size_t i, size_t j) const { return data_[flat2(i, j)]; }
  float operator()(size_t i, size_t j, size_t k) const { return data_[flat3(i, j, k)]; }
  void set(size_t flat, float v) { data_[flat] = round_f16(v); }
  void set(size_t i, size_t j, float v) { data_[flat2(i, j)] = round_f16(v); }
  void set(size_t i, size_t j, size_t k, float v) { data_[flat3(i, j, k)] = round_f16(v); }
  const float* data() const { return data_.data(); }
  const std::vector<float>& values() const { return data_; }
  bool same_elements(const Tensor& other) const { return data_ == other.data_; }  // tensor.hpp:62

 private:
  static size_t count(const std::vector<size_t>& s) {
    size_t n = 1;
    for (size_t d : s) n *= d;
    return n;
  }
  size_t flat2(size_t i, size_t j) const {
    if (shape_.size() != 2) throw ShapeError("2-d index into non-2-d tensor");
    return i * shape_[1] + j;
  }
  size_t flat3(size_t i, size_t j, size_t k) const {
    if (shape_.size() != 3) throw ShapeError("3-d index into non-3-d tensor");
    return (i * shape_[1] + j) * shape_[2] + k;
  }
  std::vector<size_t> shape_;
  std::vector<float> data_;
};

// ------------------------------------------------------------- quant.hpp
enum class QuantAxis : uint32_t { KChannel = 0, KToken = 1 };  // quant.hpp:12-15

struct QuantSpec {  // quant.hpp:19-25
  uint32_t num_bits = 4;
  QuantAxis k_axis = QuantAxis::KChannel;
  size_t group_size = 64;
  bool passthrough() const { return num_bits == 16; }
};

struct QuantParams {  // quant.hpp:38-47: (scale, zero) binary16 pairs
  size_t rows = 0;
  size_t cols = 0;
  std::vector<uint16_t> data;
  size_t group_count() const { return rows * cols; }
  float scale(size_t g) const { return f16_bits_to_f32(data[2 * g]); }
  float zero(size_t g) const { return f16_bits_to_f32(data[2 * g + 1]); }
  void push(float scale, float zero) {
    data.push_back(f32_to_f16_bits(scale));
    data.push_back(f32_to_f16_bits(zero));
  }
  bool operator==(const QuantParams&) const = default;
};

inline constexpr float kMinScale = 6.103515625e-05f;  // quant.hpp:52

// ----------------------------------------------------------- quant.hpp
// quant.hpp:45-80 on the device (bdk_quantize_tile & co.), same values.
struct GroupParams {
  float scale;
  float zero;
};
struct QuantizedTile {  // quant.hpp:62-65
  std::vector<uint16_t> codes;
  QuantParams params;
};

inline GroupParams compute_group_params(std::span<const float> group, uint32_t num_bits,
                                        int device = 0) {
  GroupParams g{};
  detail::check(bdk_compute_group_params(group.data(), static_cast<uint32_t>(group.size()),
                                         num_bits, &g.scale, &g.zero, device));
  return g;
}

inline void quantize_group(std::span<const float> group, float scale, float zero,
                           uint32_t num_bits, std::span<uint16_t> codes_out, int device = 0) {
  detail::check(bdk_quantize_group(group.data(), static_cast<uint32_t>(group.size()), scale, zero,
                                   num_bits, codes_out.data(), device));
}

inline void dequantize_group(std::span<const uint16_t> codes, float scale, float zero,
                             std::span<float> values_out, int device = 0) {
  detail::check(bdk_dequantize_group(codes.data(), static_cast<uint32_t>(codes.size()), scale,
                                     zero, values_out.data(), device));
}

inline QuantizedTile quantize_tile(const float* tile, size_t rows, size_t d, uint32_t num_bits,
                                   QuantAxis axis, size_t group_size, int device = 0) {
  QuantizedTile out;
  out.codes.assign(rows * d, 0);
  const size_t groups = group_size ? rows * d / group_size : 0;
  out.params.data.assign(2 * groups, 0);
  detail::check(bdk_quantize_tile(tile, static_cast<uint32_t>(rows), static_cast<uint32_t>(d),
                                  num_bits, static_cast<uint32_t>(axis),
                                  static_cast<uint32_t>(group_size), out.codes.data(),
                                  out.params.data.data(), device));
  out.params.rows = axis == QuantAxis::KChannel ? rows / group_size : rows;
  out.params.cols = axis == QuantAxis::KChannel ? d : d / group_size;
  return out;
}

inline void dequantize_tile(const std::vector<uint16_t>& codes, const QuantParams& params,
                            size_t rows, size_t d, QuantAxis axis, size_t group_size, float* out,
                            int device = 0) {
  if (codes.size() != rows * d) throw ShapeError("dequantize_tile: codes do not cover the tile");
  detail::check(bdk_dequantize_tile(codes.data(), params.data.data(), static_cast<uint32_t>(rows),
                                    static_cast<uint32_t>(d), static_cast<uint32_t>(axis),
                                    static_cast<uint32_t>(group_size), out, device));
}

// ------------------------------------------------------------ layout.hpp
// ---------------------------------------------------------- layout.hpp
// Word-layout metadata (which field holds which element): integer helpers
// mirroring layout.cpp:21-86 and kvcache.cpp:79-112, the layout contract the
// device cache keeps byte-identical.
struct InterleavePerm {  // layout.hpp:13-24
  uint32_t num_bits = 0;
  uint32_t pack_num = 0;
  std::array<uint8_t, 8> order{};
  std::array<uint8_t, 8> inverse() const {
    std::array<uint8_t, 8> inv{};
    for (uint32_t k = 0; k < pack_num; ++k) inv[order[k]] = static_cast<uint8_t>(k);
    return inv;
  }
};

namespace detail {
inline uint32_t pack_num_of(uint32_t num_bits) {
  if (num_bits != 2 && num_bits != 4 && num_bits != 8 && num_bits != 16)
    throw UnsupportedBits("num_bits must be one of 2, 4, 8, 16");
  return 16 / num_bits;
}
}  // namespace detail

inline InterleavePerm interleave_order(uint32_t num_bits) {  // layout.cpp:21-34
  InterleavePerm p{num_bits, detail::pack_num_of(num_bits), {}};
  uint32_t k = 0;
  for (int i = (int)p.pack_num - 1; i >= 0; --i)
    if (i % 2 == 1) p.order[k++] = static_cast<uint8_t>(i);
  for (int i = (int)p.pack_num - 1; i >= 0; --i)
    if (i % 2 == 0) p.order[k++] = static_cast<uint8_t>(i);
  return p;
}

inline InterleavePerm identity_order(uint32_t num_bits) {  // layout.cpp:36-43
  InterleavePerm p{num_bits, detail::pack_num_of(num_bits), {}};
  for (uint32_t k = 0; k < p.pack_num; ++k) p.order[k] = static_cast<uint8_t>(k);
  return p;
}

inline uint16_t pack_word(std::span<const uint16_t> codes, const InterleavePerm& perm) {
  uint32_t w = 0;  // layout.cpp:45-61: field k (from the MSB) holds codes[order[k]]
  for (uint32_t k = 0; k < perm.pack_num; ++k) {
    const uint32_t c = codes[perm.order[k]];
    if (perm.num_bits < 16 && (c >> perm.num_bits) != 0)
      throw CodeOverflow("pack_word: code does not fit in num_bits");
    w |= c << (16 - (k + 1) * perm.num_bits);
  }
  return static_cast<uint16_t>(w);
}

inline void unpack_word(uint16_t word, const InterleavePerm& perm,
                        std::span<uint16_t> codes_out) {  // layout.cpp:63-72
  const uint32_t mask = perm.num_bits == 16 ? 0xFFFFu : ((1u << perm.num_bits) - 1u);
  for (uint32_t k = 0; k < perm.pack_num; ++k)
    codes_out[perm.order[k]] = static_cast<uint16_t>((word >> (16 - (k + 1) * perm.num_bits)) & mask);
}

inline size_t iteration_count(size_t tile_n, size_t warp_n) {  // layout.cpp:79-86
  const size_t stride = warp_n * 8;
  if (stride == 0 || tile_n % stride != 0) throw ShapeError("tile_n must be a multiple of warp_n*8");
  return tile_n / stride;
}

inline size_t swizzle_col(size_t row, size_t col) { return row ^ col; }  // layout.hpp:49

inline size_t residual_block_size(uint32_t num_bits, size_t warp_n) {  // layout.cpp:74-77
  if (num_bits != 2 && num_bits != 4 && num_bits != 8 && num_bits != 16)
    throw UnsupportedBits("num_bits must be one of 2, 4, 8, 16");
  return 8 * warp_n * (16 / num_bits);
}

// ------------------------------------------------------------ config.hpp
struct AttentionConfig {  // config.hpp:13-25
  size_t batch = 1;
  size_t heads_q = 32;
  size_t heads_kv = 8;
  size_t head_dim = 128;
  size_t tile_m = 1;
  size_t tile_n = 64;
  size_t num_splits = 1;
  size_t warp_n = 4;
  size_t warp_m = 1;
  size_t n_group() const { return heads_q / heads_kv; }
};

namespace detail {
inline bdk_attn_config to_c(const AttentionConfig& c) {
  bdk_attn_config o{};
  o.batch = static_cast<uint32_t>(c.batch);
  o.heads_q = static_cast<uint32_t>(c.heads_q);
  o.heads_kv = static_cast<uint32_t>(c.heads_kv);
  o.head_dim = static_cast<uint32_t>(c.head_dim);
  o.tile_m = static_cast<uint32_t>(c.tile_m);
  o.tile_n = static_cast<uint32_t>(c.tile_n);
  o.num_splits = static_cast<uint32_t>(c.num_splits);
  o.warp_n = static_cast<uint32_t>(c.warp_n);
  o.warp_m = static_cast<uint32_t>(c.warp_m);
  return o;
}
}  // namespace detail

// gqa_transform / gqa_untransform (config.hpp:31-38, config.cpp:32-68):
// regroup the query heads sharing a KV head, [1, heads_q, d] <->
// [n_group, heads_kv, d]; a pure element permutation
inline Tensor gqa_transform(const Tensor& q, size_t n_group) {
  if (q.ndim() != 3 || q.dim(0) != 1) throw ShapeError("gqa_transform expects shape [1, heads_q, d]");
  const size_t heads_q = q.dim(1), d = q.dim(2);
  if (n_group == 0 || heads_q % n_group != 0) throw ShapeError("heads_q must be divisible by n_group");
  const size_t heads_kv = heads_q / n_group;
  Tensor out({n_group, heads_kv, d});
  for (size_t h = 0; h < heads_kv; ++h)
    for (size_t g = 0; g < n_group; ++g)
      for (size_t k = 0; k < d; ++k) out.set(g, h, k, q(0, h * n_group + g, k));
  return out;
}

inline Tensor gqa_untransform(const Tensor& q, size_t n_group) {
  if (q.ndim() != 3 || q.dim(0) != n_group)
    throw ShapeError("gqa_untransform expects shape [n_group, heads_kv, d]");
  const size_t heads_kv = q.dim(1), d = q.dim(2);
  Tensor out({1, heads_kv * n_group, d});
  for (size_t h = 0; h < heads_kv; ++h)
    for (size_t g = 0; g < n_group; ++g)
      for (size_t k = 0; k < d; ++k) out.set(size_t{0}, h * n_group + g, k, q(g, h, k));
  return out;
}

inline AttentionConfig validate_config(const AttentionConfig& cfg) {  // config.cpp:10-30
  const bdk_attn_config c = detail::to_c(cfg);
  detail::check(bdk_validate_config(&c));
  return cfg;
}

// ----------------------------------------------------------- kvcache.hpp
struct PackedBlock {  // kvcache.hpp:17-26
  std::vector<uint16_t> k_words;
  std::vector<uint16_t> v_words;
  QuantParams k_params;
  QuantParams v_params;
  bool operator==(const PackedBlock&) const = default;
};

struct PackedKV {  // kvcache.hpp:28-43
  std::vector<PackedBlock> blocks;
  size_t packed_len = 0;
  size_t k_word_count() const {
    size_t n = 0;
    for (const auto& b : blocks) n += b.k_words.size();
    return n;
  }
  size_t v_word_count() const {
    size_t n = 0;
    for (const auto& b : blocks) n += b.v_words.size();
    return n;
  }
};

struct ResidualCache {  // kvcache.hpp:45-50 (host view of a residual window)
  std::vector<float> k;
  std::vector<float> v;
  size_t res_len = 0;
};

// ---- paged residual bookkeeping (kvcache.hpp:52-97): host-side token pages
// for callers that manage their own residual tails.  The device cache keeps
// its residual window contiguous in HBM (CacheBackend::Paged is accepted and
// observationally identical, test_kvcache.cpp:243-283).
class PagePool {
 public:
  PagePool() = default;
  PagePool(size_t page_size, size_t head_dim, size_t max_pages = 0)
      : page_size_(page_size), head_dim_(head_dim), max_pages_(max_pages) {}

  // Pages live in one growing slab ([k rows | v rows] per page).  Released
  // handles form an intrusive LIFO list threaded through next_free_, so the
  // most recently released page is handed out first (the reference's
  // recycling order, kvcache.hpp:50-52).
  uint32_t alloc() {
    if (head_ != kNone) {
      const uint32_t id = head_;
      head_ = next_free_[id];
      next_free_[id] = kLive;
      --n_free_;
      return id;
    }
    const size_t n = next_free_.size();
    if (max_pages_ != 0 && n == max_pages_) throw CapacityError("PagePool: all pages in use");
    slab_.resize(slab_.size() + 2 * page_floats(), 0.0f);
    next_free_.push_back(kLive);
    return static_cast<uint32_t>(n);
  }
  void release(uint32_t id) {
    next_free_[id] = head_;
    head_ = id;
    ++n_free_;
  }

  float* k_row(uint32_t page, size_t slot) { return slab_.data() + row_off(page, slot, 0); }
  float* v_row(uint32_t page, size_t slot) { return slab_.data() + row_off(page, slot, 1); }
  const float* k_row(uint32_t page, size_t slot) const { return slab_.data() + row_off(page, slot, 0); }
  const float* v_row(uint32_t page, size_t slot) const { return slab_.data() + row_off(page, slot, 1); }

  size_t page_size() const { return page_size_; }
  size_t live_pages() const { return next_free_.size() - n_free_; }

 private:
  static constexpr uint32_t kNone = 0xFFFFFFFFu, kLive = 0xFFFFFFFEu;
  size_t page_floats() const { return page_size_ * head_dim_; }
  size_t row_off(uint32_t page, size_t slot, int half) const {
    return (2 * (size_t)page + (size_t)half) * page_floats() + slot * head_dim_;
  }
  std::vector<float> slab_;
  std::vector<uint32_t> next_free_;  // per page: next released page, or kLive
  uint32_t head_ = kNone;
  size_t n_free_ = 0;
  size_t page_size_ = 0, head_dim_ = 0, max_pages_ = 0;
};

struct PageTable {  // logical tokens -> pool pages; pages == ceil(length / page_size)
  size_t page_size = 16;
  std::vector<uint32_t> pages;
  size_t length = 0;
};

inline void paged_append(PageTable& pt, PagePool& pool, const float* k_row, const float* v_row,
                         size_t d) {
  if (pt.pages.size() * pt.page_size == pt.length) pt.pages.push_back(pool.alloc());  // last page full
  const uint32_t page = pt.pages.back();
  const size_t slot = pt.length - (pt.pages.size() - 1) * pt.page_size;
  std::copy(k_row, k_row + d, pool.k_row(page, slot));
  std::copy(v_row, v_row + d, pool.v_row(page, slot));
  pt.length += 1;
}

// tokens [t0, t0 + len) page run by page run (rows of a page are contiguous)
inline void paged_gather(const PageTable& pt, const PagePool& pool, size_t t0, size_t len,
                         size_t d, float* k_out, float* v_out) {
  if (len > pt.length || t0 > pt.length - len)
    throw ShapeError("paged_gather: tokens [t0, t0 + len) exceed the table");
  size_t done = 0;
  while (done < len) {
    const size_t t = t0 + done;
    const size_t slot = t % pt.page_size;
    const size_t run = std::min(len - done, pt.page_size - slot);
    const uint32_t page = pt.pages[t / pt.page_size];
    std::copy(pool.k_row(page, slot), pool.k_row(page, slot) + run * d, k_out + done * d);
    std::copy(pool.v_row(page, slot), pool.v_row(page, slot) + run * d, v_out + done * d);
    done += run;
  }
}

inline void paged_pop_front(PageTable& pt, PagePool& pool, size_t n_tokens) {
  if (n_tokens > pt.length) throw StateError("paged_pop_front: fewer tokens resident");
  const size_t whole = n_tokens / pt.page_size;
  if (whole * pt.page_size != n_tokens) throw StateError("paged_pop_front: partial page");
  std::for_each(pt.pages.begin(), pt.pages.begin() + static_cast<std::ptrdiff_t>(whole),
                [&pool](uint32_t id) { pool.release(id); });
  std::rotate(pt.pages.begin(), pt.pages.begin() + static_cast<std::ptrdiff_t>(whole), pt.pages.end());
  pt.pages.resize(pt.pages.size() - whole);
  pt.length -= n_tokens;
}

enum class CacheBackend { Contiguous, Paged };  // kvcache.hpp:100

class KVCache {  // kvcache.hpp:103-189, cache resident in HBM
 public:
  KVCache(size_t batch, size_t heads_kv, size_t head_dim, size_t warp_n, QuantSpec spec,
          CacheBackend backend = CacheBackend::Contiguous, size_t page_size = 16,
          size_t max_pages = 0, bool interleave = true, size_t max_tokens = 65536,
          int device = 0)
      : batch_(batch), heads_kv_(heads_kv), head_dim_(head_dim), warp_n_(warp_n), spec_(spec),
        backend_(backend), page_size_(page_size), interleave_(interleave) {
    (void)max_pages;
    if (backend == CacheBackend::Paged) {
      const size_t n_r = residual_block_size(spec.num_bits, warp_n);
      if (page_size == 0 || n_r % page_size != 0)
        throw ConfigError("page_size must divide N_r");
    }
    bdk_cache_desc d{};
    d.batch = static_cast<uint32_t>(batch);
    d.heads_kv = static_cast<uint32_t>(heads_kv);
    d.head_dim = static_cast<uint32_t>(head_dim);
    d.warp_n = static_cast<uint32_t>(warp_n);
    d.num_bits = spec.num_bits;
    d.k_axis = static_cast<uint32_t>(spec.k_axis);
    d.group_size = static_cast<uint32_t>(spec.group_size);
    d.interleave = interleave ? 1u : 0u;
    d.max_tokens = static_cast<uint32_t>(max_tokens);
    d.device = device;
    detail::check(bdk_cache_create(&d, &h_));
    detail::check(bdk_cache_get_info(h_, &info_));
  }
  KVCache(const KVCache&) = delete;
  KVCache& operator=(const KVCache&) = delete;
  KVCache(KVCache&& o) noexcept { *this = std::move(o); }
  KVCache& operator=(KVCache&& o) noexcept {
    std::swap(h_, o.h_);
    batch_ = o.batch_;
    heads_kv_ = o.heads_kv_;
    head_dim_ = o.head_dim_;
    warp_n_ = o.warp_n_;
    spec_ = o.spec_;
    backend_ = o.backend_;
    page_size_ = o.page_size_;
    interleave_ = o.interleave_;
    info_ = o.info_;
    snap_ = std::move(o.snap_);
    return *this;
  }
  ~KVCache() {
    if (h_) bdk_cache_destroy(h_);
  }

  size_t batch() const { return batch_; }
  size_t heads_kv() const { return heads_kv_; }
  size_t head_dim() const { return head_dim_; }
  size_t warp_n() const { return warp_n_; }
  size_t n_r() const { return info_.n_r; }
  const QuantSpec& spec() const { return spec_; }
  CacheBackend backend() const { return backend_; }
  size_t page_size() const { return page_size_; }
  bool interleaved() const { return interleave_; }
  // KVCache::perm (kvcache.hpp:120): the word permutation of this cache
  InterleavePerm perm() const {
    return interleave_ ? interleave_order(spec_.num_bits) : identity_order(spec_.num_bits);
  }
  bdk_cache* handle() const { return h_; }

  // KVCache::prefill (kvcache.cpp:155-168): fused quantize+pack on device
  void prefill(size_t b, size_t h, const float* k, const float* v, size_t len) {
    std::vector<uint16_t> kb(len * head_dim_), vb(len * head_dim_);
    for (size_t i = 0; i < kb.size(); ++i) {
      kb[i] = f32_to_f16_bits(k[i]);
      vb[i] = f32_to_f16_bits(v[i]);
    }
    detail::check(bdk_prefill_host(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                   kb.data(), vb.data(), static_cast<uint32_t>(len)));
  }
  // KVCache::append_token (kvcache.cpp:170-182)
  void append_token(size_t b, size_t h, const float* k_row, const float* v_row) {
    std::vector<uint16_t> kb(head_dim_), vb(head_dim_);
    for (size_t i = 0; i < head_dim_; ++i) {
      kb[i] = f32_to_f16_bits(k_row[i]);
      vb[i] = f32_to_f16_bits(v_row[i]);
    }
    detail::check(bdk_append_token_host(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                        kb.data(), vb.data()));
  }
  // KVCache::flush_residual (kvcache.cpp:245-251)
  void flush_residual(size_t b, size_t h) {
    detail::check(
        bdk_flush_residual(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h), nullptr));
    detail::check(bdk_synchronize());
  }
  // KVCache::adopt_block (kvcache.cpp:239-243)
  void adopt_block(size_t b, size_t h, const PackedBlock& blk) {
    detail::check(bdk_adopt_block(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                  blk.k_words.data(), blk.v_words.data(),
                                  blk.k_params.data.data(), blk.v_params.data.data()));
  }

  size_t packed_len(size_t b, size_t h) const { return lengths(b, h).first; }
  size_t res_len(size_t b, size_t h) const { return lengths(b, h).second; }
  size_t total_len(size_t b, size_t h) const {
    const auto l = lengths(b, h);
    return l.first + l.second;
  }

  // KVCache::packed(b, h) (kvcache.hpp:148). The segment lives in HBM; this
  // refreshes a per-cell host snapshot and returns a reference to it, so the
  // reference's `const PackedBlock& blk = cache.packed(b, h).blocks[0];`
  // stays valid until the next packed(b, h) call on the same cell.
  const PackedKV& packed(size_t b, size_t h) const {
    if (b >= batch_ || h >= heads_kv_) throw ConfigError("packed: cell out of range");
    if (snap_.size() != batch_ * heads_kv_) snap_.assign(batch_ * heads_kv_, PackedKV{});
    PackedKV& out = snap_[b * heads_kv_ + h];
    out.packed_len = packed_len(b, h);
    const size_t nb = out.packed_len / n_r();
    out.blocks.resize(nb);
    for (size_t i = 0; i < nb; ++i) out.blocks[i] = block(b, h, i);
    return out;
  }
  // KVCache::build_block (kvcache.cpp:208-219): pack the full residual on the
  // device without committing
  PackedBlock build_block(size_t b, size_t h) const {
    PackedBlock blk = empty_block();
    detail::check(bdk_build_block(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                  blk.k_words.data(), blk.v_words.data(),
                                  blk.k_params.data.data(), blk.v_params.data.data()));
    return blk;
  }
  // KVCache::commit_block (kvcache.cpp:231-237)
  void commit_block(size_t b, size_t h, const PackedBlock& blk) {
    detail::check(bdk_commit_block(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                   blk.k_words.data(), blk.v_words.data(),
                                   blk.k_params.data.data(), blk.v_params.data.data()));
  }

  PackedBlock block(size_t b, size_t h, size_t i) const {
    PackedBlock blk = empty_block();
    detail::check(bdk_read_block(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                 static_cast<uint32_t>(i), blk.k_words.data(), blk.v_words.data(),
                                 blk.k_params.data.data(), blk.v_params.data.data()));
    return blk;
  }
  // a block sized for this geometry, params grids as quant.cpp:59-91
  PackedBlock empty_block() const {
    PackedBlock blk;
    blk.k_words.resize(info_.words_per_block);
    blk.v_words.resize(info_.words_per_block);
    blk.k_params.data.resize(info_.k_param_u16);
    blk.v_params.data.resize(info_.v_param_u16);
    const size_t g = spec_.passthrough() ? 1 : spec_.group_size;
    if (!spec_.passthrough()) {  // quant.cpp:59-91 grids
      if (spec_.k_axis == QuantAxis::KChannel) {
        blk.k_params.rows = n_r() / g;
        blk.k_params.cols = head_dim_;
      } else {
        blk.k_params.rows = n_r();
        blk.k_params.cols = head_dim_ / g;
      }
      blk.v_params.rows = n_r();
      blk.v_params.cols = head_dim_ / g;
    }
    return blk;
  }
  // KVCache::residual_tile (kvcache.cpp:253-261): [res_len, d] fp32 each
  void residual_tile(size_t b, size_t h, float* k_out, float* v_out) const {
    const size_t n = res_len(b, h) * head_dim_;
    std::vector<uint16_t> kb(n), vb(n);
    detail::check(bdk_read_residual(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                    kb.data(), vb.data()));
    for (size_t i = 0; i < n; ++i) {
      k_out[i] = f16_bits_to_f32(kb[i]);
      v_out[i] = f16_bits_to_f32(vb[i]);
    }
  }
  // KVCache::packed_tile (kvcache.cpp:263-312): device dequant, [len, d] fp32
  void packed_tile(size_t b, size_t h, size_t t0, size_t len, float* k_out, float* v_out) const {
    std::vector<uint16_t> kb(len * head_dim_), vb(len * head_dim_);
    detail::check(bdk_packed_tile_host(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                       static_cast<uint32_t>(t0), static_cast<uint32_t>(len),
                                       kb.data(), vb.data()));
    for (size_t i = 0; i < kb.size(); ++i) {
      k_out[i] = f16_bits_to_f32(kb[i]);
      v_out[i] = f16_bits_to_f32(vb[i]);
    }
  }
  // KVCache::reconstruct (kvcache.cpp:314-324)
  void reconstruct(size_t b, size_t h, std::vector<float>& k_out, std::vector<float>& v_out) const {
    const size_t p = packed_len(b, h), r = res_len(b, h);
    k_out.assign((p + r) * head_dim_, 0.f);
    v_out.assign((p + r) * head_dim_, 0.f);
    if (p) packed_tile(b, h, 0, p, k_out.data(), v_out.data());
    if (r) residual_tile(b, h, k_out.data() + p * head_dim_, v_out.data() + p * head_dim_);
  }
  // KVCache::corrupt_word (kvcache.cpp:326-328)
  void corrupt_word(size_t b, size_t h, size_t blk, size_t word, uint16_t value) {
    detail::check(bdk_corrupt_word(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h),
                                   static_cast<uint32_t>(blk), static_cast<uint32_t>(word),
                                   value));
  }
  struct Memory {  // kvcache.hpp:165-171
    size_t k_packed_payload_bytes = 0;
    size_t v_packed_payload_bytes = 0;
    size_t params_bytes = 0;
    size_t residual_bytes = 0;
  };
  Memory memory() const {  // kvcache.cpp:330-345
    uint64_t m[4];
    detail::check(bdk_memory(h_, m));
    return Memory{m[0], m[1], m[2], m[3]};
  }
  // precise (true, the default: bit-faithful dequant + hi/lo split PV, the
  // reference's own 1e-5 tolerances) or fast (false: folded
  // scales, fp16 P -- the throughput kernel, an explicit opt-in)
  void set_precise(bool precise) { detail::check(bdk_set_precise(h_, precise ? 1 : 0)); }
  // empty every cell, keeping the device arena (a fresh KVCache of the same
  // geometry without reallocating)
  void reset() { detail::check(bdk_cache_reset(h_, nullptr)); }

  // adopt a handle the C-ABI created (load_cache); geometry from the BDKV
  // header fields (serialize.hpp:11-20)
  static KVCache adopt(bdk_cache* h, uint32_t bits, uint32_t axis, uint32_t g, uint32_t n_r,
                       uint32_t d, uint32_t batch, uint32_t heads, bool interleave) {
    KVCache c;
    c.h_ = h;
    c.batch_ = batch;
    c.heads_kv_ = heads;
    c.head_dim_ = d;
    c.warp_n_ = n_r / (8 * (16 / bits));
    c.spec_ = QuantSpec{bits, static_cast<QuantAxis>(axis), g};
    c.interleave_ = interleave;
    detail::check(bdk_cache_get_info(h, &c.info_));
    return c;
  }

 private:
  KVCache() = default;
  std::pair<size_t, size_t> lengths(size_t b, size_t h) const {
    uint32_t p = 0, r = 0;
    detail::check(bdk_cache_lengths(h_, static_cast<uint32_t>(b), static_cast<uint32_t>(h), &p,
                                    &r));
    return {p, r};
  }
  bdk_cache* h_ = nullptr;
  size_t batch_ = 1, heads_kv_ = 1, head_dim_ = 0, warp_n_ = 1;
  QuantSpec spec_;
  CacheBackend backend_ = CacheBackend::Contiguous;
  size_t page_size_ = 16;
  bool interleave_ = true;
  bdk_cache_info info_{};
  mutable std::vector<PackedKV> snap_;  // host snapshots handed out by packed()
};

// --------------------------------------------------------- attention.hpp
struct AttnOutput {  // attention.hpp:73-84
  size_t batch = 0;
  size_t heads = 0;
  size_t d = 0;
  std::vector<float> data;
  float* row(size_t b, size_t h) { return data.data() + (b * heads + h) * d; }
  const float* row(size_t b, size_t h) const { return data.data() + (b * heads + h) * d; }
};

// The reference's decode decomposition (attention.hpp:17-70).  Every call
// runs on the device (bdk_span.cu) through the C-ABI; the structs are the
// reference's host-side value types.
struct PartialOutput {  // attention.hpp:17-26
  size_t rows = 0;
  size_t d = 0;
  std::vector<float> o;  // rows * d, unnormalized
  std::vector<float> m;  // rows, starts at -inf
  std::vector<float> l;  // rows, starts at 0
  static PartialOutput init(size_t rows, size_t d) {
    PartialOutput p;
    p.rows = rows;
    p.d = d;
    p.o.assign(rows * d, 0.0f);
    p.m.assign(rows, -INFINITY);
    p.l.assign(rows, 0.0f);
    return p;
  }
};

// attention.hpp:28-36.  The device kernels keep their own staging in shared
// memory; the struct stays for signature compatibility.
struct StagingBuffer {
  std::vector<float> partition_max;
  std::vector<float> p_tile;
  void reserve(size_t warp_n, size_t tile_m, size_t tile_n) {
    partition_max.resize(warp_n);
    p_tile.resize(tile_m * tile_n);
  }
};

namespace detail {
// device of the cache-less calls (attend_tile, partitioned_rowmax, combine)
inline int& compute_device() {
  static int dev = 0;
  return dev;
}
}  // namespace detail

// partitioned_rowmax (attention.cpp:32-50)
inline void partitioned_rowmax(const float* s, size_t rows, size_t cols, size_t warp_n,
                               StagingBuffer& buf, float* rowmax_out) {
  if (warp_n != 0) buf.partition_max.resize(warp_n);
  detail::check(bdk_partitioned_rowmax_host(s, static_cast<uint32_t>(rows),
                                            static_cast<uint32_t>(cols),
                                            static_cast<uint32_t>(warp_n), rowmax_out,
                                            detail::compute_device()));
}

// attend_tile (attention.cpp:52-90): one online-softmax step
inline void attend_tile(PartialOutput& state, const float* q, const float* k, const float* v,
                        size_t tile_n, size_t d, float scale_factor, size_t warp_n,
                        StagingBuffer& buf) {
  (void)buf;
  if (state.d != d || state.o.size() != state.rows * d)
    throw ShapeError("attend_tile: state shape does not match d");
  detail::check(bdk_attend_tile_host(state.o.data(), state.m.data(), state.l.data(),
                                     static_cast<uint32_t>(state.rows), static_cast<uint32_t>(d),
                                     q, k, v, static_cast<uint32_t>(tile_n), scale_factor,
                                     static_cast<uint32_t>(warp_n), detail::compute_device()));
}

// residual_attend (attention.cpp:92-105): attention over the residual of
// cell (b, h); the packed block of a full residual, for the caller to commit
inline std::optional<PackedBlock> residual_attend(const KVCache& cache, size_t b, size_t h,
                                                  const float* q, size_t q_rows,
                                                  float scale_factor, size_t warp_n,
                                                  PartialOutput& state, StagingBuffer& buf) {
  (void)warp_n;
  (void)buf;
  if (cache.res_len(b, h) == 0) throw StateError("residual_attend: residual cache is empty");
  if (state.rows != q_rows) throw ShapeError("residual_attend: state rows != q rows");
  if (state.d != cache.head_dim()) throw ShapeError("residual_attend: state d != head_dim");
  detail::check(bdk_residual_attend_host(cache.handle(), static_cast<uint32_t>(b),
                                         static_cast<uint32_t>(h), q,
                                         static_cast<uint32_t>(q_rows), scale_factor,
                                         state.o.data(), state.m.data(), state.l.data()));
  if (cache.res_len(b, h) == cache.n_r()) return cache.build_block(b, h);
  return std::nullopt;
}

// packed_attend (attention.cpp:107-140): one state per non-empty split
inline std::vector<PartialOutput> packed_attend(const KVCache& cache, size_t b, size_t h,
                                                const float* q, size_t q_rows, size_t tile_n,
                                                size_t num_splits, float scale_factor,
                                                size_t warp_n) {
  (void)warp_n;
  const size_t d = cache.head_dim();
  const size_t cap = std::max<size_t>(1, num_splits);
  std::vector<float> o(cap * q_rows * d), m(cap * q_rows), l(cap * q_rows);
  uint32_t n = 0;
  detail::check(bdk_packed_attend_host(cache.handle(), static_cast<uint32_t>(b),
                                       static_cast<uint32_t>(h), q,
                                       static_cast<uint32_t>(q_rows),
                                       static_cast<uint32_t>(tile_n),
                                       static_cast<uint32_t>(num_splits), scale_factor, o.data(),
                                       m.data(), l.data(), &n));
  std::vector<PartialOutput> parts(n);
  for (uint32_t p = 0; p < n; ++p) {
    parts[p].rows = q_rows;
    parts[p].d = d;
    parts[p].o.assign(o.begin() + p * q_rows * d, o.begin() + (p + 1) * q_rows * d);
    parts[p].m.assign(m.begin() + p * q_rows, m.begin() + (p + 1) * q_rows);
    parts[p].l.assign(l.begin() + p * q_rows, l.begin() + (p + 1) * q_rows);
  }
  return parts;
}

// combine (attention.cpp:142-162): LSE reduction of the partial states
inline std::vector<float> combine(std::span<const PartialOutput> partials) {
  if (partials.empty()) throw EmptyInput("combine: no partial outputs");
  const size_t rows = partials[0].rows, d = partials[0].d;
  for (const auto& p : partials)
    if (p.rows != rows || p.d != d) throw ShapeError("combine: partial shapes differ");
  std::vector<float> o, m, l, out(rows * d);
  o.reserve(partials.size() * rows * d);
  for (const auto& p : partials) {
    o.insert(o.end(), p.o.begin(), p.o.end());
    m.insert(m.end(), p.m.begin(), p.m.end());
    l.insert(l.end(), p.l.begin(), p.l.end());
  }
  detail::check(bdk_combine_host(o.data(), m.data(), l.data(),
                                 static_cast<uint32_t>(partials.size()),
                                 static_cast<uint32_t>(rows), static_cast<uint32_t>(d), out.data(),
                                 detail::compute_device()));
  return out;
}

// decode_step (attention.hpp:87-88, attention.cpp:164-242)
inline AttnOutput decode_step(KVCache& cache, const AttentionConfig& cfg, const Tensor& q,
                              const Tensor& k_new, const Tensor& v_new) {
  validate_config(cfg);
  if (q.ndim() != 3 || q.dim(0) != cfg.batch || q.dim(1) != cfg.heads_q ||
      q.dim(2) != cfg.head_dim)
    throw ShapeError("decode_step: q must be [batch, heads_q, d]");
  if (k_new.ndim() != 3 || k_new.dim(0) != cfg.batch || k_new.dim(1) != cfg.heads_kv ||
      k_new.dim(2) != cfg.head_dim || v_new.ndim() != 3 || v_new.dim(0) != cfg.batch ||
      v_new.dim(1) != cfg.heads_kv || v_new.dim(2) != cfg.head_dim)
    throw ShapeError("decode_step: k_new / v_new must be [batch, heads_kv, d]");
  AttnOutput out;
  out.batch = cfg.batch;
  out.heads = cfg.heads_q;
  out.d = cfg.head_dim;
  out.data.assign(cfg.batch * cfg.heads_q * cfg.head_dim, 0.f);
  const bdk_attn_config c = detail::to_c(cfg);
  detail::check(bdk_decode_step_host(cache.handle(), &c, q.data(), k_new.data(), v_new.data(),
                                     out.data.data()));
  return out;
}

// kvcache.hpp:199-205: row-major [n_r, d] codes <-> channel-major words,
// pack_num consecutive tokens per word
inline std::vector<uint16_t> pack_block_codes(const std::vector<uint16_t>& codes, size_t n_r,
                                              size_t d, const InterleavePerm& perm) {
  if (codes.size() != n_r * d) throw ShapeError("pack_block_codes: codes do not cover block");
  if (n_r % perm.pack_num != 0) throw ShapeError("pack_block_codes: N_r not pack-aligned");
  const size_t groups = n_r / perm.pack_num;
  std::vector<uint16_t> words(groups * d), tmp(perm.pack_num);
  for (size_t c = 0; c < d; ++c)
    for (size_t g = 0; g < groups; ++g) {
      for (size_t k = 0; k < perm.pack_num; ++k) tmp[k] = codes[(g * perm.pack_num + k) * d + c];
      words[c * groups + g] = pack_word(tmp, perm);
    }
  return words;
}

inline std::vector<uint16_t> unpack_block_codes(const std::vector<uint16_t>& words, size_t n_r,
                                                size_t d, const InterleavePerm& perm) {
  const size_t groups = n_r / perm.pack_num;
  if (words.size() != groups * d) throw ShapeError("unpack_block_codes: word count mismatch");
  std::vector<uint16_t> codes(n_r * d), tmp(perm.pack_num);
  for (size_t c = 0; c < d; ++c)
    for (size_t g = 0; g < groups; ++g) {
      unpack_word(words[c * groups + g], perm, tmp);
      for (size_t k = 0; k < perm.pack_num; ++k) codes[(g * perm.pack_num + k) * d + c] = tmp[k];
    }
  return codes;
}

// ------------------------------------------------------------ serialize.hpp
// BDKV v1 (serialize.hpp:11-23): the reference's byte format, produced from
// and loaded into the device cache by the C-ABI (bdk_dump_cache /
// bdk_load_cache).  max_tokens / device size the loaded cache's arena.
inline void dump_cache(const KVCache& cache, std::ostream& os) {
  uint64_t n = 0;
  detail::check(bdk_dump_cache(cache.handle(), nullptr, 0, &n));
  std::vector<uint8_t> buf(n);
  detail::check(bdk_dump_cache(cache.handle(), buf.data(), n, &n));
  os.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(n));
  os.flush();
}

namespace detail {
inline KVCache adopt_loaded(bdk_cache* h, const std::vector<uint8_t>& hdr) {
  uint32_t f[7];
  std::memcpy(f, hdr.data() + 6, sizeof f);  // little-endian host
  return KVCache::adopt(h, f[0], f[1], f[2], f[3], f[4], f[5], f[6], (hdr[5] & 1) != 0);
}
}  // namespace detail

inline KVCache load_cache(std::istream& is, size_t max_tokens = 0, int device = 0) {
  std::vector<uint8_t> buf((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
  bdk_cache* h = nullptr;
  detail::check(bdk_load_cache(buf.data(), buf.size(), static_cast<uint32_t>(max_tokens), device,
                               &h));
  return detail::adopt_loaded(h, buf);
}

inline void dump_cache_file(const KVCache& cache, const std::string& path) {
  detail::check(bdk_dump_cache_file(cache.handle(), path.c_str()));
}

inline KVCache load_cache_file(const std::string& path, size_t max_tokens = 0, int device = 0) {
  bdk_cache* h = nullptr;
  detail::check(bdk_load_cache_file(path.c_str(), static_cast<uint32_t>(max_tokens), device, &h));
  std::vector<uint8_t> hdr(34, 0);
  if (FILE* f = std::fopen(path.c_str(), "rb")) {
    const size_t got = std::fread(hdr.data(), 1, hdr.size(), f);
    std::fclose(f);
    (void)got;
  }
  return detail::adopt_loaded(h, hdr);
}

}  // namespace bitkv
