// kvslab/seq_table.hpp -- engine-side per-sequence block table (C++ API).
//
// The reference keeps each running request's blocks in LiveRequest::blocks
// (proj/core/src/simulator.cpp:33-40) and drives the allocator from three
// call sites: the prefill claim of ceil(prompt/tpb) blocks with rollback
// (:500-526), the decode growth rule need = ceil((cached+1)/tpb) with a
// per-request stall (:561-578), and the release of every handle on
// completion / eviction / stop (:583-596, :621, :745-747).  SeqTable is that
// bookkeeping as a native object over a kvslab::SlabPool: one row per
// sequence slot, the handles in logical-block order, the cached-token count,
// and a list of (row, col, gid) entries changed since the last upload, which
// the C ABI scatters into the engine's int32 device table.  It also carries
// the reference's internal-fragmentation metric (simulator.cpp:80-89).
#pragma once

#include <cstdint>
#include <unordered_map>
#include <vector>

#include "kvslab/slab_pool.hpp"

namespace kvslab {

struct SeqTableStats {
  std::uint32_t live_seqs = 0;      // rows holding at least one block
  std::uint64_t held_blocks = 0;    // held_blocks_total (simulator.cpp:75-79)
  std::uint64_t cached_tokens = 0;  // cached_total (simulator.cpp:70-74)
  Bytes internal_frag_bytes = 0;    // simulator.cpp:80-89
};

class SeqTable {
 public:
  // useful_token_bytes = num_layers * token_size, block_metadata_bytes =
  // num_layers * quant params per block (simulator.cpp:53-54, 210-212).
  SeqTable(SlabPool* pool, Bytes key, std::uint32_t max_seqs, std::uint32_t max_blocks_per_seq,
           Tokens tokens_per_block, Bytes useful_token_bytes, Bytes block_metadata_bytes);

  // simulator.cpp:561-578: claim blocks until ceil(tokens/tpb) are held.
  // false = stalled (the blocks claimed so far are kept, as in do_decode).
  bool ensure_capacity(std::uint32_t seq, Tokens tokens);
  // simulator.cpp:500-526: claim the prompt's blocks or none (rollback);
  // on success the row's cached count is the prompt length.
  bool admit(std::uint32_t seq, Tokens prompt_tokens);
  // One decode step of a batch (simulator.cpp:561-578 then :609-612): each
  // listed sequence grows for its next token; the ones that got their block
  // advance by one token, the others are marked in `stalled` (nullable).
  // Returns the number that advanced.
  std::uint32_t step(const std::uint32_t* seqs, std::uint32_t n, std::uint8_t* stalled);
  // simulator.cpp:621 / :583-596: free every handle of the row.
  void release(std::uint32_t seq);
  // Moves a sequence to an empty row (no allocator traffic): an engine keeps
  // its running batch in rows 0..B-1 by moving the last row into a released
  // one.  The destination row's device entries join the pending upload.
  void move_row(std::uint32_t src, std::uint32_t dst);

  Tokens cached(std::uint32_t seq) const { return cached_.at(seq); }
  void set_cached(std::uint32_t seq, Tokens tokens);
  const std::vector<BlockHandle>& blocks(std::uint32_t seq) const { return rows_.at(seq); }
  std::uint32_t max_seqs() const { return static_cast<std::uint32_t>(rows_.size()); }
  std::uint32_t max_blocks_per_seq() const { return max_blocks_; }
  Bytes key() const { return key_; }
  Tokens tokens_per_block() const { return tpb_; }
  SeqTableStats stats() const;

  // Compaction (K3): rewrite every held handle whose gid was moved; the
  // rewritten entries join the pending device upload.  Returns how many.
  std::uint64_t remap(const std::unordered_map<std::uint64_t, BlockHandle>& moved);

  // Entries (row, col, gid) changed since the last drain, in change order.
  struct Delta {
    std::int32_t row, col, gid;
  };
  const std::vector<Delta>& pending() const { return pending_; }
  // Keeps only the last change of each (row, col): one scatter launch
  // applies its entries in no particular order.
  void dedupe_pending();
  void clear_pending() { pending_.clear(); }

 private:
  void push(std::uint32_t seq, std::uint32_t col, std::uint64_t gid);

  SlabPool* pool_;
  Bytes key_;
  std::uint32_t max_blocks_;
  Tokens tpb_;
  Bytes useful_token_bytes_, block_metadata_bytes_;
  std::vector<std::vector<BlockHandle>> rows_;
  std::vector<Tokens> cached_;
  std::vector<Delta> pending_;
};

}  // namespace kvslab
