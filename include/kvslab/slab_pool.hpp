// kvslab/slab_pool.hpp -- host half of the KV-slab data path (C++ API).
//
// A from-scratch allocator with the same public API and the same observable
// semantics as slabsim::SlabPool (reference: proj/core/include/slabsim/
// slab_pool.hpp:101-202, proj/core/src/slab_pool.cpp:51-386): identical
// slab choice (lowest-id PARTIAL slab of the key, else lowest FREE slab),
// identical handles and global ids, identical byte-exact fragmentation
// ledger, identical errors.  Parity is pinned against the compiled reference
// (tests/golden/*, tests/test_slab_pool_parity.py).
//
// Internals are different and sized for a 180 GB B200 pool: structure-of-
// arrays slab metadata, one occupancy arena, and two-level find-first-set
// bitsets for the FREE list and every per-key PARTIAL list, so alloc/free are
// O(1) word scans instead of std::set operations.  The pool also records
// which slabs changed so the device slab table can be delta-synced.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <ostream>
#include <string>
#include <utility>
#include <vector>

#include "kvslab/common.hpp"

namespace kvslab {

enum class SlabState { kFree, kPartial, kFull };

// slab_pool.hpp:41-46
struct SlabPoolConfig {
  Bytes capacity_bytes = 0;
  Bytes slab_size_bytes = 0;
  std::vector<Bytes> block_size_keys;
  bool require_lcm_alignment = true;
};

// slab_pool.hpp:53-60
struct BlockHandle {
  std::uint32_t slab_id = 0;
  std::uint32_t local_block_id = 0;
  std::uint64_t global_block_id = 0;
  Bytes key = 0;
  bool operator==(const BlockHandle&) const = default;
};

// slab_pool.hpp:67-78
struct FragmentationStats {
  Bytes allocated_bytes = 0;
  Bytes free_block_bytes = 0;
  Bytes slab_residue_bytes = 0;
  Bytes free_slab_bytes = 0;
  Bytes usable_capacity() const {
    return allocated_bytes + free_block_bytes + slab_residue_bytes + free_slab_bytes;
  }
  bool operator==(const FragmentationStats&) const = default;
};

// slab_pool.hpp:80-89
struct OpLogRecord {
  std::uint64_t seq = 0;
  double time = 0.0;
  const char* op = "";
  Bytes key = 0;
  std::uint32_t slab_id = 0;
  std::uint32_t local_block_id = 0;
  std::uint64_t global_block_id = 0;
};

void write_op_log_line(std::ostream& out, const OpLogRecord& rec);

// One planned compaction move (K3); new, no reference counterpart.
struct BlockMove {
  BlockHandle src;
  BlockHandle dst;
};

// Find-first-set bitset with a one-word-per-64-words summary level.
class FfsBitset {
 public:
  void resize(std::uint32_t n);
  void set(std::uint32_t i);
  void clear(std::uint32_t i);
  bool test(std::uint32_t i) const { return (leaf_[i >> 6] >> (i & 63)) & 1u; }
  // lowest set index, or UINT32_MAX
  std::uint32_t first() const;
  std::uint32_t count() const { return count_; }
  bool operator==(const FfsBitset& o) const { return leaf_ == o.leaf_; }
  template <class F>
  void for_each(F&& f) const {
    for (std::size_t w = 0; w < leaf_.size(); ++w) {
      std::uint64_t bits = leaf_[w];
      while (bits) {
        f(static_cast<std::uint32_t>(w * 64 + __builtin_ctzll(bits)));
        bits &= bits - 1;
      }
    }
  }

 private:
  std::vector<std::uint64_t> leaf_;
  std::vector<std::uint64_t> summary_;
  std::uint32_t count_ = 0;
};

class SlabPool {
 public:
  explicit SlabPool(const SlabPoolConfig& config);

  BlockHandle alloc_block(Bytes key);
  std::optional<BlockHandle> try_alloc_block(Bytes key);
  void free_block(const BlockHandle& handle);

  std::uint64_t blocks_per_slab(Bytes key) const;
  FragmentationStats snapshot_stats() const { return stats_; }

  const SlabPoolConfig& config() const { return config_; }
  std::uint32_t slab_count() const { return nslabs_; }
  Bytes slab_size() const { return config_.slab_size_bytes; }
  Bytes tail_remainder_bytes() const { return tail_remainder_; }
  Bytes usable_capacity_bytes() const { return usable_capacity_; }

  SlabState slab_state(std::uint32_t slab_id) const;
  Bytes slab_key(std::uint32_t slab_id) const;
  std::uint32_t slab_blocks_total(std::uint32_t slab_id) const;
  std::uint32_t slab_blocks_used(std::uint32_t slab_id) const;

  std::uint64_t free_blocks_for_key(Bytes key) const;
  std::uint64_t allocated_block_count() const { return allocated_blocks_; }
  std::uint64_t allocated_block_count(Bytes key) const;

  static std::uint64_t global_block_id(std::uint32_t slab_id, std::uint32_t local_block_id,
                                       std::uint64_t blocks_per_slab) {
    return static_cast<std::uint64_t>(slab_id) * blocks_per_slab + local_block_id;
  }
  static std::pair<std::uint32_t, std::uint32_t> split_global_block_id(
      std::uint64_t global_id, std::uint64_t blocks_per_slab) {
    return {static_cast<std::uint32_t>(global_id / blocks_per_slab),
            static_cast<std::uint32_t>(global_id % blocks_per_slab)};
  }
  // slab * slab_size + local * key (== gid * key only under LCM alignment)
  Bytes block_byte_offset(Bytes key, std::uint64_t global_id) const;

  bool operator==(const SlabPool& other) const;
  bool check_integrity(std::string* why = nullptr) const;

  void set_op_log(std::function<void(const OpLogRecord&)> sink) { op_log_ = std::move(sink); }
  void set_clock(std::function<double()> clock) { clock_ = std::move(clock); }
  void debug_flip_occupancy_bit(std::uint32_t slab_id, std::uint32_t local_block_id);

  // ---- extensions (not in the reference) ----
  // Deterministic compaction plan for one key.  Applies
  // the moves to the table and returns them; the caller moves the bytes (K3)
  // and rewrites its block tables.
  std::vector<BlockMove> plan_compaction(Bytes key, std::uint64_t max_moves,
                                         std::uint32_t* slabs_freed = nullptr);
  // Slabs whose (key, blocks_total, state) changed since the last call.
  void drain_dirty_slabs(std::vector<std::uint32_t>* out);
  // Slabs formatted to a key other than the one whose bytes they last held
  // (device memory starts zero-filled, which is clean for every key): their
  // stale bytes must be cleared before a kernel reads a block slot past a
  // sequence's context (a foreign format's bytes can be NaN patterns).
  void drain_scrub_slabs(std::vector<std::uint32_t>* out);
  bool has_scrub_slabs() const noexcept { return !scrub_.empty(); }

 private:
  int key_index(Bytes key) const;  // -1 if unregistered
  void format_slab(std::uint32_t slab_id, int kidx);
  void unformat_slab(std::uint32_t slab_id);
  std::uint32_t take_first_free(std::uint32_t slab_id);
  void take_specific(std::uint32_t slab_id, std::uint32_t local);
  void release(std::uint32_t slab_id, std::uint32_t local, int kidx);
  void log_op(const char* op, const BlockHandle& h);
  void mark_dirty(std::uint32_t slab_id);
  std::uint64_t* occ(std::uint32_t slab_id) { return &occ_[std::size_t(slab_id) * words_per_slab_]; }
  const std::uint64_t* occ(std::uint32_t slab_id) const {
    return &occ_[std::size_t(slab_id) * words_per_slab_];
  }

  SlabPoolConfig config_;
  Bytes tail_remainder_ = 0;
  Bytes usable_capacity_ = 0;
  std::uint32_t nslabs_ = 0;
  std::uint32_t words_per_slab_ = 0;
  std::vector<Bytes> keys_;              // sorted, deduplicated
  std::vector<std::uint32_t> bps_;       // blocks per slab, per key index
  std::vector<std::uint64_t> alloc_by_key_;
  // per-slab SoA; kidx_ = key index + 1, 0 = unformatted
  std::vector<std::uint16_t> kidx_;
  std::vector<std::uint32_t> total_, used_, hint_;
  std::vector<std::uint64_t> occ_;
  FfsBitset free_slabs_;
  std::vector<FfsBitset> partial_;  // per key index
  FragmentationStats stats_;
  std::uint64_t allocated_blocks_ = 0;
  std::uint64_t op_seq_ = 0;
  std::vector<std::uint8_t> dirty_flag_;
  std::vector<std::uint32_t> dirty_;
  std::vector<Bytes> bytes_key_;  // per slab: key whose format its device bytes hold, 0 = zeros
  std::vector<std::uint32_t> scrub_;
  std::function<void(const OpLogRecord&)> op_log_;
  std::function<double()> clock_;
};

}  // namespace kvslab
