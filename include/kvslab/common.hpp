// kvslab/common.hpp -- value types, error classes and KV geometry.
//
// The error classes are the reference's own hierarchy (proj/core/include/
// slabsim/common.hpp:31-95, restated in this repo's slabsim/common.hpp), so
// code written against slabsim keeps its catch clauses; the C ABI maps them
// 1:1 onto ks_status codes.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "slabsim/common.hpp"

namespace kvslab {

// The value types and the exception hierarchy ARE slabsim's (one set of
// classes, declared in slabsim/common.hpp): code written against the
// reference catches exactly what this library throws.
using slabsim::Bytes;
using slabsim::Error;
using slabsim::InvalidConfigError;
using slabsim::InvalidFreeError;
using slabsim::InvalidKeyError;
using slabsim::InvalidProfileError;
using slabsim::PoolExhaustedError;
using slabsim::Seconds;
using slabsim::Tokens;

// The geometry subset of slabsim::ModelProfile that token_size and
// kv_block_size read (precision.hpp:168-176).
struct KvGeometry {
  std::uint32_t num_kv_heads = 0;
  std::uint32_t head_dim = 0;
  std::uint32_t num_layers = 1;
  std::uint32_t tp_degree = 1;
  Tokens tokens_per_block = 16;
  Bytes quant_param_bytes_per_block = 0;
  int kv_bits = 16;
};

// precision.cpp:76-89: (kv_heads/tp) * head_dim * 2 * kv_bits / 8, in bits.
inline Bytes token_size(const KvGeometry& g) {
  if (g.tp_degree == 0 || g.num_kv_heads % g.tp_degree != 0) {
    throw InvalidProfileError("num_kv_heads not divisible by tp_degree");
  }
  const std::uint64_t bits = static_cast<std::uint64_t>(g.num_kv_heads / g.tp_degree) *
                             g.head_dim * 2 * static_cast<std::uint64_t>(g.kv_bits);
  if (bits % 8 != 0) throw InvalidProfileError("fractional-byte token size rejected");
  return bits / 8;
}

// precision.cpp:91-99: num_layers * (tpb * token_size + quant params).
inline Bytes kv_block_size(const KvGeometry& g) {
  if (g.tokens_per_block < 1) throw InvalidProfileError("tokens_per_block must be >= 1");
  return static_cast<Bytes>(g.num_layers) *
         (g.tokens_per_block * token_size(g) + g.quant_param_bytes_per_block);
}

}  // namespace kvslab
