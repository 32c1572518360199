// bitkv/oracle.hpp for the reference test suite built against the drop-in:
// the reference's brute-force test references (oracle.hpp:17-40) served by
// this repo's C restatement (oracle/bitkv_oracle.c).  TEST INFRASTRUCTURE
// ONLY -- linked into the ref-suite test binaries, never into the library.
#pragma once
#include <cmath>
#include <span>
#include <vector>

#include "bitkv_b200.hpp"
extern "C" {
#include "bitkv_oracle.h"
}

namespace bitkv {

inline std::vector<float> naive_attention(const float* q, size_t q_rows, const float* k,
                                          const float* v, size_t len, size_t d) {
  std::vector<float> out(q_rows * d);
  orc_naive_attention(q, q_rows, k, v, len, d, out.data());
  return out;
}

inline void offline_quant_reference(const float* k, const float* v, size_t len, size_t d,
                                    const QuantSpec& spec, size_t n_r, float* k_out,
                                    float* v_out) {
  orc_offline_quant_reference(k, v, len, d, spec.num_bits, static_cast<uint32_t>(spec.k_axis),
                              spec.group_size, n_r, k_out, v_out);
}

struct OracleReport {
  double max_abs_err = 0.0;
  double rel_l2_err = 0.0;
  double cosine_similarity = 1.0;
};

inline OracleReport compare(std::span<const float> a, std::span<const float> b) {
  if (a.size() != b.size()) throw ShapeError("compare: length mismatch");
  OracleReport r;
  double diff2 = 0, ref2 = 0, dot = 0, a2 = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double x = a[i], y = b[i];
    r.max_abs_err = std::max(r.max_abs_err, std::fabs(x - y));
    diff2 += (x - y) * (x - y);
    ref2 += y * y;
    dot += x * y;
    a2 += x * x;
  }
  r.rel_l2_err = ref2 > 0 ? std::sqrt(diff2) / std::sqrt(ref2) : std::sqrt(diff2);
  if (a2 == 0 && ref2 == 0)
    r.cosine_similarity = 1.0;
  else if (a2 == 0 || ref2 == 0)
    r.cosine_similarity = 0.0;
  else
    r.cosine_similarity = dot / (std::sqrt(a2) * std::sqrt(ref2));
  return r;
}

}  // namespace bitkv
