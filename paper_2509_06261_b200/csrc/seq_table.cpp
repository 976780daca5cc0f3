// seq_table.cpp -- kvslab::SeqTable (see include/kvslab/seq_table.hpp).
#include "kvslab/seq_table.hpp"

#include <algorithm>
#include <limits>
#include <stdexcept>
#include <string>

namespace kvslab {

SeqTable::SeqTable(SlabPool* pool, Bytes key, std::uint32_t max_seqs,
                   std::uint32_t max_blocks_per_seq, Tokens tokens_per_block,
                   Bytes useful_token_bytes, Bytes block_metadata_bytes)
    : pool_(pool),
      key_(key),
      max_blocks_(max_blocks_per_seq),
      tpb_(tokens_per_block),
      useful_token_bytes_(useful_token_bytes),
      block_metadata_bytes_(block_metadata_bytes),
      rows_(max_seqs),
      cached_(max_seqs, 0) {
  if (!pool_) throw InvalidConfigError("sequence table needs a pool");
  if (tpb_ == 0) throw InvalidConfigError("tokens_per_block must be >= 1");
  if (max_seqs == 0 || max_blocks_per_seq == 0) {
    throw InvalidConfigError("sequence table needs at least one row and one column");
  }
  pool_->blocks_per_slab(key_);  // InvalidKeyError when the key is not registered
  // device entries are int32 global ids
  const std::uint64_t max_gid = std::uint64_t{pool_->slab_count()} * pool_->blocks_per_slab(key_);
  if (max_gid > static_cast<std::uint64_t>(std::numeric_limits<std::int32_t>::max())) {
    throw InvalidConfigError("global block ids of key " + std::to_string(key_) +
                             " exceed the int32 device table");
  }
  for (auto& r : rows_) r.reserve(max_blocks_per_seq);
}

void SeqTable::push(std::uint32_t seq, std::uint32_t col, std::uint64_t gid) {
  pending_.push_back({static_cast<std::int32_t>(seq), static_cast<std::int32_t>(col),
                      static_cast<std::int32_t>(gid)});
}

bool SeqTable::ensure_capacity(std::uint32_t seq, Tokens tokens) {
  auto& hs = rows_.at(seq);
  const Tokens need = (tokens + tpb_ - 1) / tpb_;
  if (need > max_blocks_) {
    throw std::out_of_range("sequence " + std::to_string(seq) + " needs " + std::to_string(need) +
                            " blocks, table row holds " + std::to_string(max_blocks_));
  }
  while (hs.size() < need) {
    auto h = pool_->try_alloc_block(key_);
    if (!h) return false;
    push(seq, static_cast<std::uint32_t>(hs.size()), h->global_block_id);
    hs.push_back(*h);
  }
  return true;
}

bool SeqTable::admit(std::uint32_t seq, Tokens prompt_tokens) {
  auto& hs = rows_.at(seq);
  if (!hs.empty()) throw std::invalid_argument("admit into a row that still holds blocks");
  const std::size_t mark = pending_.size();
  if (!ensure_capacity(seq, prompt_tokens)) {
    for (const BlockHandle& h : hs) pool_->free_block(h);
    hs.clear();
    pending_.resize(mark);
    return false;
  }
  cached_[seq] = prompt_tokens;
  return true;
}

std::uint32_t SeqTable::step(const std::uint32_t* seqs, std::uint32_t n, std::uint8_t* stalled) {
  std::uint32_t active = 0;
  for (std::uint32_t i = 0; i < n; ++i) {
    const std::uint32_t s = seqs[i];
    const bool ok = ensure_capacity(s, cached_.at(s) + 1);
    if (stalled) stalled[i] = ok ? 0 : 1;
    if (ok) {
      ++cached_[s];
      ++active;
    }
  }
  return active;
}

void SeqTable::release(std::uint32_t seq) {
  auto& hs = rows_.at(seq);
  for (const BlockHandle& h : hs) pool_->free_block(h);
  hs.clear();
  cached_[seq] = 0;
}

void SeqTable::move_row(std::uint32_t src, std::uint32_t dst) {
  if (src == dst) return;
  auto& from = rows_.at(src);
  auto& to = rows_.at(dst);
  if (!to.empty()) throw std::invalid_argument("move into a row that still holds blocks");
  to.swap(from);
  cached_[dst] = cached_[src];
  cached_[src] = 0;
  for (std::size_t c = 0; c < to.size(); ++c) {
    push(dst, static_cast<std::uint32_t>(c), to[c].global_block_id);
  }
}

void SeqTable::set_cached(std::uint32_t seq, Tokens tokens) {
  const Tokens need = (tokens + tpb_ - 1) / tpb_;
  if (need > rows_.at(seq).size()) {
    throw std::out_of_range("cached tokens exceed the row's blocks");
  }
  cached_[seq] = tokens;
}

SeqTableStats SeqTable::stats() const {
  SeqTableStats st;
  for (std::size_t s = 0; s < rows_.size(); ++s) {
    const Bytes held = rows_[s].size();
    if (held == 0) continue;
    ++st.live_seqs;
    st.held_blocks += held;
    st.cached_tokens += cached_[s];
    // simulator.cpp:80-89: held*key - (cached*useful_token_bytes + held*metadata)
    st.internal_frag_bytes +=
        held * key_ - (cached_[s] * useful_token_bytes_ + held * block_metadata_bytes_);
  }
  return st;
}

std::uint64_t SeqTable::remap(const std::unordered_map<std::uint64_t, BlockHandle>& moved) {
  std::uint64_t n = 0;
  for (std::size_t s = 0; s < rows_.size(); ++s) {
    auto& hs = rows_[s];
    for (std::size_t c = 0; c < hs.size(); ++c) {
      const auto it = moved.find(hs[c].global_block_id);
      if (it == moved.end()) continue;
      hs[c] = it->second;
      push(static_cast<std::uint32_t>(s), static_cast<std::uint32_t>(c), it->second.global_block_id);
      ++n;
    }
  }
  return n;
}

void SeqTable::dedupe_pending() {
  if (pending_.size() < 2) return;
  std::vector<std::uint32_t> idx(pending_.size());
  for (std::uint32_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](std::uint32_t a, std::uint32_t b) {
    const Delta& x = pending_[a];
    const Delta& y = pending_[b];
    if (x.row != y.row) return x.row < y.row;
    if (x.col != y.col) return x.col < y.col;
    return a < b;
  });
  std::vector<Delta> out;
  out.reserve(pending_.size());
  for (std::size_t i = 0; i < idx.size(); ++i) {
    const bool last = i + 1 == idx.size() || pending_[idx[i + 1]].row != pending_[idx[i]].row ||
                      pending_[idx[i + 1]].col != pending_[idx[i]].col;
    if (last) out.push_back(pending_[idx[i]]);
  }
  pending_.swap(out);
}

}  // namespace kvslab
