// slab_pool.cpp -- kvslab::SlabPool (see include/kvslab/slab_pool.hpp).
//
// Semantics follow slabsim::SlabPool (proj/core/src/slab_pool.cpp); every
// public method cites the reference lines it mirrors.  The data structures
// are this library's own: SoA slab metadata, a single occupancy arena and
// find-first-set bitsets instead of std::map/std::set.
#include "kvslab/slab_pool.hpp"

#include <algorithm>
#include <bit>
#include <numeric>
#include <set>

namespace kvslab {

// ---------------------------------------------------------------- FfsBitset
void FfsBitset::resize(std::uint32_t n) {
  leaf_.assign((n + 63) / 64, 0);
  summary_.assign((leaf_.size() + 63) / 64, 0);
  count_ = 0;
}
void FfsBitset::set(std::uint32_t i) {
  std::uint64_t& w = leaf_[i >> 6];
  const std::uint64_t b = std::uint64_t{1} << (i & 63);
  if (w & b) return;
  w |= b;
  summary_[i >> 12] |= std::uint64_t{1} << ((i >> 6) & 63);
  ++count_;
}
void FfsBitset::clear(std::uint32_t i) {
  std::uint64_t& w = leaf_[i >> 6];
  const std::uint64_t b = std::uint64_t{1} << (i & 63);
  if (!(w & b)) return;
  w &= ~b;
  if (w == 0) summary_[i >> 12] &= ~(std::uint64_t{1} << ((i >> 6) & 63));
  --count_;
}
std::uint32_t FfsBitset::first() const {
  for (std::size_t s = 0; s < summary_.size(); ++s) {
    if (summary_[s]) {
      const std::size_t w = s * 64 + static_cast<std::size_t>(std::countr_zero(summary_[s]));
      return static_cast<std::uint32_t>(w * 64 + std::countr_zero(leaf_[w]));
    }
  }
  return UINT32_MAX;
}

// ---------------------------------------------------------------- helpers
void write_op_log_line(std::ostream& out, const OpLogRecord& rec) {
  // slab_pool.cpp:45-49: "seq time op key slab local gid"
  out << rec.seq << ' ' << rec.time << ' ' << rec.op << ' ' << rec.key << ' ' << rec.slab_id
      << ' ' << rec.local_block_id << ' ' << rec.global_block_id << '\n';
}

namespace {
[[noreturn]] void unregistered(Bytes key) {
  throw InvalidKeyError("block-size key " + std::to_string(key) + " is not registered");
}
}  // namespace

// ---------------------------------------------------------------- ctor
// slab_pool.cpp:51-98
SlabPool::SlabPool(const SlabPoolConfig& config) : config_(config) {
  if (config_.slab_size_bytes == 0) throw InvalidConfigError("slab size must be positive");
  if (config_.block_size_keys.empty()) {
    throw InvalidConfigError("at least one block-size key must be registered");
  }
  keys_ = config_.block_size_keys;
  std::sort(keys_.begin(), keys_.end());
  keys_.erase(std::unique(keys_.begin(), keys_.end()), keys_.end());
  config_.block_size_keys = keys_;
  if (keys_.size() > 65534) throw InvalidConfigError("too many block-size keys");
  for (Bytes k : keys_) {
    if (k == 0) throw InvalidConfigError("block-size key must be >= 1");
    if (k > config_.slab_size_bytes) {
      throw InvalidConfigError("block-size key " + std::to_string(k) + " exceeds slab size " +
                               std::to_string(config_.slab_size_bytes));
    }
  }
  if (config_.require_lcm_alignment) {
    std::uint64_t l = 1;
    bool too_big = false;
    for (Bytes k : keys_) {
      l = std::lcm(l, k);
      if (l > config_.slab_size_bytes) {
        too_big = true;
        break;
      }
    }
    if (too_big || config_.slab_size_bytes % l != 0) {
      throw InvalidConfigError("slab size " + std::to_string(config_.slab_size_bytes) +
                               " is not a multiple of lcm(block-size keys)");
    }
  }
  const std::uint64_t n = config_.capacity_bytes / config_.slab_size_bytes;
  if (n == 0) throw InvalidConfigError("capacity smaller than one slab");
  if (n > UINT32_MAX / 2) throw InvalidConfigError("too many slabs");
  nslabs_ = static_cast<std::uint32_t>(n);
  tail_remainder_ = config_.capacity_bytes % config_.slab_size_bytes;
  usable_capacity_ = n * config_.slab_size_bytes;

  std::uint64_t max_bps = 0;
  for (Bytes k : keys_) {
    const std::uint64_t b = config_.slab_size_bytes / k;
    if (b > UINT32_MAX) throw InvalidConfigError("too many blocks per slab");
    bps_.push_back(static_cast<std::uint32_t>(b));
    max_bps = std::max(max_bps, b);
  }
  words_per_slab_ = static_cast<std::uint32_t>((max_bps + 63) / 64);
  alloc_by_key_.assign(keys_.size(), 0);
  kidx_.assign(nslabs_, 0);
  total_.assign(nslabs_, 0);
  used_.assign(nslabs_, 0);
  hint_.assign(nslabs_, 0);
  occ_.assign(std::size_t(nslabs_) * words_per_slab_, 0);
  free_slabs_.resize(nslabs_);
  for (std::uint32_t i = 0; i < nslabs_; ++i) free_slabs_.set(i);
  partial_.resize(keys_.size());
  for (auto& p : partial_) p.resize(nslabs_);
  dirty_flag_.assign(nslabs_, 0);
  bytes_key_.assign(nslabs_, 0);
  stats_.free_slab_bytes = usable_capacity_;
}

int SlabPool::key_index(Bytes key) const {
  auto it = std::lower_bound(keys_.begin(), keys_.end(), key);
  if (it == keys_.end() || *it != key) return -1;
  return static_cast<int>(it - keys_.begin());
}

// slab_pool.cpp:104-113
SlabState SlabPool::slab_state(std::uint32_t slab_id) const {
  if (slab_id >= nslabs_) throw std::out_of_range("slab id out of range");
  if (kidx_[slab_id] == 0) return SlabState::kFree;
  return used_[slab_id] == total_[slab_id] ? SlabState::kFull : SlabState::kPartial;
}
Bytes SlabPool::slab_key(std::uint32_t slab_id) const {
  if (slab_id >= nslabs_) throw std::out_of_range("slab id out of range");
  return kidx_[slab_id] ? keys_[kidx_[slab_id] - 1] : 0;
}
std::uint32_t SlabPool::slab_blocks_total(std::uint32_t slab_id) const { return total_.at(slab_id); }
std::uint32_t SlabPool::slab_blocks_used(std::uint32_t slab_id) const { return used_.at(slab_id); }

// slab_pool.cpp:115-122
std::uint64_t SlabPool::blocks_per_slab(Bytes key) const {
  const int k = key_index(key);
  if (k < 0) unregistered(key);
  return bps_[k];
}

// slab_pool.cpp:124-133
std::uint64_t SlabPool::free_blocks_for_key(Bytes key) const {
  const int k = key_index(key);
  if (k < 0) unregistered(key);
  std::uint64_t n = std::uint64_t{free_slabs_.count()} * bps_[k];
  partial_[k].for_each([&](std::uint32_t s) { n += total_[s] - used_[s]; });
  return n;
}

// slab_pool.cpp:135-141
std::uint64_t SlabPool::allocated_block_count(Bytes key) const {
  const int k = key_index(key);
  if (k < 0) unregistered(key);
  return alloc_by_key_[k];
}

Bytes SlabPool::block_byte_offset(Bytes key, std::uint64_t gid) const {
  const std::uint64_t b = blocks_per_slab(key);
  return (gid / b) * config_.slab_size_bytes + (gid % b) * key;
}

void SlabPool::mark_dirty(std::uint32_t s) {
  if (!dirty_flag_[s]) {
    dirty_flag_[s] = 1;
    dirty_.push_back(s);
  }
}
void SlabPool::drain_scrub_slabs(std::vector<std::uint32_t>* out) {
  out->clear();
  out->swap(scrub_);
}
void SlabPool::drain_dirty_slabs(std::vector<std::uint32_t>* out) {
  out->clear();
  out->swap(dirty_);
  for (std::uint32_t s : *out) dirty_flag_[s] = 0;
}

// slab_pool.cpp:143-158
void SlabPool::format_slab(std::uint32_t s, int k) {
  if (bytes_key_[s] != 0 && bytes_key_[s] != keys_[k]) scrub_.push_back(s);
  bytes_key_[s] = keys_[k];
  kidx_[s] = static_cast<std::uint16_t>(k + 1);
  total_[s] = bps_[k];
  used_[s] = 0;
  hint_[s] = 0;
  std::fill_n(occ(s), words_per_slab_, 0);
  free_slabs_.clear(s);
  partial_[k].set(s);
  const Bytes block_bytes = Bytes{bps_[k]} * keys_[k];
  stats_.free_slab_bytes -= config_.slab_size_bytes;
  stats_.free_block_bytes += block_bytes;
  stats_.slab_residue_bytes += config_.slab_size_bytes - block_bytes;
  mark_dirty(s);
}

// slab_pool.cpp:160-169
void SlabPool::unformat_slab(std::uint32_t s) {
  const int k = kidx_[s] - 1;
  const Bytes block_bytes = Bytes{total_[s]} * keys_[k];
  stats_.free_block_bytes -= block_bytes;
  stats_.slab_residue_bytes -= config_.slab_size_bytes - block_bytes;
  stats_.free_slab_bytes += config_.slab_size_bytes;
  partial_[k].clear(s);
  kidx_[s] = 0;
  total_[s] = used_[s] = hint_[s] = 0;
  std::fill_n(occ(s), words_per_slab_, 0);
  free_slabs_.set(s);
  mark_dirty(s);
}

// slab_pool.cpp:171-191: lowest clear bit at or after the hint's word.
std::uint32_t SlabPool::take_first_free(std::uint32_t s) {
  std::uint64_t* w = occ(s);
  const std::uint32_t total = total_[s];
  const std::uint32_t nwords = (total + 63) / 64;
  for (std::uint32_t i = hint_[s] / 64; i < nwords; ++i) {
    std::uint64_t bits = w[i];
    const std::uint32_t valid = std::min<std::uint32_t>(64, total - i * 64);
    if (valid < 64) bits |= ~std::uint64_t{0} << valid;
    if (bits != ~std::uint64_t{0}) {
      const std::uint32_t b = static_cast<std::uint32_t>(std::countr_one(bits));
      const std::uint32_t local = i * 64 + b;
      w[i] |= std::uint64_t{1} << b;
      ++used_[s];
      hint_[s] = local + 1;
      return local;
    }
  }
  throw Error("internal: slab advertised a free block but none found");
}

void SlabPool::take_specific(std::uint32_t s, std::uint32_t local) {
  occ(s)[local / 64] |= std::uint64_t{1} << (local % 64);
  ++used_[s];
  // keep the reference's hint invariant: every bit below the hint is set
  if (hint_[s] == local) {
    std::uint32_t h = local + 1;
    while (h < total_[s] && ((occ(s)[h / 64] >> (h % 64)) & 1u)) ++h;
    hint_[s] = h;
  }
}

// slab_pool.cpp:193-226
std::optional<BlockHandle> SlabPool::try_alloc_block(Bytes key) {
  const int k = key_index(key);
  if (k < 0) unregistered(key);
  std::uint32_t s = partial_[k].first();
  if (s == UINT32_MAX) {
    s = free_slabs_.first();
    if (s == UINT32_MAX) return std::nullopt;
    format_slab(s, k);
  }
  const std::uint32_t local = take_first_free(s);
  if (used_[s] == total_[s]) {
    partial_[k].clear(s);
    mark_dirty(s);
  }
  stats_.allocated_bytes += key;
  stats_.free_block_bytes -= key;
  ++allocated_blocks_;
  ++alloc_by_key_[k];
  BlockHandle h;
  h.slab_id = s;
  h.local_block_id = local;
  h.global_block_id = global_block_id(s, local, total_[s]);
  h.key = key;
  log_op("alloc", h);
  return h;
}

// slab_pool.cpp:228-235
BlockHandle SlabPool::alloc_block(Bytes key) {
  auto h = try_alloc_block(key);
  if (!h) {
    throw PoolExhaustedError("pool exhausted: no PARTIAL slab of key " + std::to_string(key) +
                             " and no FREE slab");
  }
  return *h;
}

void SlabPool::release(std::uint32_t s, std::uint32_t local, int k) {
  const bool was_full = used_[s] == total_[s];
  occ(s)[local / 64] &= ~(std::uint64_t{1} << (local % 64));
  --used_[s];
  hint_[s] = std::min(hint_[s], local);
  stats_.allocated_bytes -= keys_[k];
  stats_.free_block_bytes += keys_[k];
  --allocated_blocks_;
  --alloc_by_key_[k];
  if (was_full) {
    partial_[k].set(s);
    mark_dirty(s);
  }
}

// slab_pool.cpp:237-272
void SlabPool::free_block(const BlockHandle& h) {
  if (h.slab_id >= nslabs_) {
    throw InvalidFreeError("free of unknown slab id " + std::to_string(h.slab_id));
  }
  const std::uint32_t s = h.slab_id;
  const int k = static_cast<int>(kidx_[s]) - 1;
  if (k < 0 || keys_[k] != h.key || h.local_block_id >= total_[s] ||
      h.global_block_id != global_block_id(s, h.local_block_id, total_[s])) {
    throw InvalidFreeError("free of handle that was never issued");
  }
  if (!((occ(s)[h.local_block_id / 64] >> (h.local_block_id % 64)) & 1u)) {
    throw InvalidFreeError("double free of block " + std::to_string(h.global_block_id) +
                           " (key " + std::to_string(h.key) + ")");
  }
  release(s, h.local_block_id, k);
  log_op("free", h);
  if (used_[s] == 0) unformat_slab(s);
}

// slab_pool.cpp:274-286
void SlabPool::log_op(const char* op, const BlockHandle& h) {
  ++op_seq_;
  if (!op_log_) return;
  OpLogRecord r;
  r.seq = op_seq_;
  r.time = clock_ ? clock_() : static_cast<double>(op_seq_);
  r.op = op;
  r.key = h.key;
  r.slab_id = h.slab_id;
  r.local_block_id = h.local_block_id;
  r.global_block_id = h.global_block_id;
  op_log_(r);
}

// slab_pool.cpp:288-296 (op sequence excluded, as in the reference)
bool SlabPool::operator==(const SlabPool& o) const {
  if (config_.capacity_bytes != o.config_.capacity_bytes ||
      config_.slab_size_bytes != o.config_.slab_size_bytes || keys_ != o.keys_ ||
      nslabs_ != o.nslabs_ || !(stats_ == o.stats_) || allocated_blocks_ != o.allocated_blocks_ ||
      alloc_by_key_ != o.alloc_by_key_ || !(free_slabs_ == o.free_slabs_)) {
    return false;
  }
  for (std::size_t k = 0; k < partial_.size(); ++k) {
    if (!(partial_[k] == o.partial_[k])) return false;
  }
  for (std::uint32_t s = 0; s < nslabs_; ++s) {
    if (kidx_[s] != o.kidx_[s] || total_[s] != o.total_[s] || used_[s] != o.used_[s] ||
        hint_[s] != o.hint_[s]) {
      return false;
    }
    const std::uint32_t nw = (total_[s] + 63) / 64;
    if (!std::equal(occ(s), occ(s) + nw, o.occ(s))) return false;
  }
  return true;
}

// slab_pool.cpp:298-379
bool SlabPool::check_integrity(std::string* why) const {
  auto fail = [&](const std::string& r) {
    if (why) *why = r;
    return false;
  };
  FragmentationStats re;
  std::uint64_t used_total = 0;
  std::vector<std::uint64_t> by_key(keys_.size(), 0);
  for (std::uint32_t s = 0; s < nslabs_; ++s) {
    const std::uint64_t* w = occ(s);
    if (kidx_[s] == 0) {
      for (std::uint32_t i = 0; i < words_per_slab_; ++i) {
        if (w[i]) return fail("unformatted slab " + std::to_string(s) + " has residual metadata");
      }
      if (used_[s] || total_[s]) {
        return fail("unformatted slab " + std::to_string(s) + " has residual metadata");
      }
      if (!free_slabs_.test(s)) {
        return fail("FREE slab " + std::to_string(s) + " missing from free-slab list");
      }
      re.free_slab_bytes += config_.slab_size_bytes;
      continue;
    }
    const int k = kidx_[s] - 1;
    if (total_[s] != bps_[k]) return fail("slab " + std::to_string(s) + " has wrong block count");
    std::uint64_t pop = 0;
    for (std::uint32_t i = 0; i < words_per_slab_; ++i) {
      std::uint64_t bits = w[i];
      const std::uint64_t lo = std::uint64_t{i} * 64;
      if (lo + 64 > total_[s]) {
        const std::uint64_t valid = total_[s] > lo ? total_[s] - lo : 0;
        const std::uint64_t mask = valid >= 64 ? ~std::uint64_t{0} : ((std::uint64_t{1} << valid) - 1);
        if (bits & ~mask) return fail("slab " + std::to_string(s) + " has out-of-range bit set");
      }
      pop += static_cast<std::uint64_t>(std::popcount(bits));
    }
    if (pop != used_[s]) return fail("slab " + std::to_string(s) + " blocks_used disagrees with bitmap");
    if (pop == 0) return fail("formatted slab " + std::to_string(s) + " is empty");
    if ((pop < total_[s]) != partial_[k].test(s)) {
      return fail("slab " + std::to_string(s) + " partial-list membership disagrees with state");
    }
    if (free_slabs_.test(s)) {
      return fail("formatted slab " + std::to_string(s) + " present in free-slab list");
    }
    const Bytes block_bytes = Bytes{total_[s]} * keys_[k];
    re.allocated_bytes += pop * keys_[k];
    re.free_block_bytes += (total_[s] - pop) * keys_[k];
    re.slab_residue_bytes += config_.slab_size_bytes - block_bytes;
    used_total += pop;
    by_key[k] += pop;
  }
  if (!(re == stats_)) return fail("fragmentation counters disagree with recomputation");
  if (re.usable_capacity() != usable_capacity_) {
    return fail("conservation violated: components do not sum to capacity");
  }
  if (used_total != allocated_blocks_) return fail("allocated block count disagrees with bitmaps");
  if (by_key != alloc_by_key_) return fail("per-key allocated counts disagree with bitmaps");
  return true;
}

// slab_pool.cpp:381-386
void SlabPool::debug_flip_occupancy_bit(std::uint32_t s, std::uint32_t local) {
  if (s >= nslabs_ || local >= std::uint64_t{words_per_slab_} * 64) {
    throw std::out_of_range("flip out of range");
  }
  occ(s)[local / 64] ^= std::uint64_t{1} << (local % 64);
}

// ------------------------------------------------------------ compaction
// New (no reference; SPEC.md:223 forbids migration in the reference).
// Sources: PARTIAL slabs of the key in (used asc, slab desc) order; a source
// is evacuated only when every block fits into the other non-evacuated slabs
// of the key; each move goes to the fullest such slab (ties: lowest id),
// lowest free local id first.  Mirrors oracle/kvslab_oracle.c
// orc_compact_plan move for move.
std::vector<BlockMove> SlabPool::plan_compaction(Bytes key, std::uint64_t max_moves,
                                                 std::uint32_t* slabs_freed) {
  const int k = key_index(key);
  if (k < 0) unregistered(key);
  std::vector<BlockMove> moves;
  std::uint32_t freed = 0;
  std::vector<std::uint32_t> cand;
  partial_[k].for_each([&](std::uint32_t s) { cand.push_back(s); });
  std::sort(cand.begin(), cand.end(), [&](std::uint32_t a, std::uint32_t b) {
    return used_[a] != used_[b] ? used_[a] < used_[b] : a > b;
  });
  // Targets: every slab of the key (PARTIAL or FULL) that is not evacuated.
  // A move keeps the key's free-block count (dst -1, src +1), so the room
  // available to a source is the running total minus the source's own free
  // blocks; evacuating a (then empty) source removes its blocks.  Open
  // targets sit in an ordered set by (used desc, id asc): the fill order of
  // a fresh fullest-first sort, kept current move by move in O(log n).
  std::uint64_t room = 0;
  std::set<std::pair<std::int64_t, std::uint32_t>> open;
  for (std::uint32_t s = 0; s < nslabs_; ++s) {
    if (kidx_[s] != k + 1) continue;
    room += total_[s] - used_[s];
    if (used_[s] < total_[s]) open.insert({-std::int64_t{used_[s]}, s});
  }
  std::vector<std::uint8_t> recv(nslabs_, 0);
  for (std::uint32_t S : cand) {
    if (recv[S] || kidx_[S] != k + 1) continue;
    const std::uint32_t need = used_[S];
    const std::uint64_t own = total_[S] - used_[S];
    if (room - own < need || moves.size() + need > max_moves) break;
    open.erase({-std::int64_t{used_[S]}, S});
    const std::uint32_t bps = total_[S];
    for (std::uint32_t l = 0; l < bps && used_[S] > 0; ++l) {
      if (!((occ(S)[l / 64] >> (l % 64)) & 1u)) continue;
      const auto top = open.begin();
      const std::uint32_t D = top->second;
      open.erase(top);
      const std::uint32_t dl = take_first_free(D);
      if (used_[D] < total_[D]) open.insert({-std::int64_t{used_[D]}, D});
      stats_.allocated_bytes += key;
      stats_.free_block_bytes -= key;
      ++allocated_blocks_;
      ++alloc_by_key_[k];
      if (used_[D] == total_[D]) {
        partial_[k].clear(D);
        mark_dirty(D);
      }
      recv[D] = 1;
      BlockMove m;
      m.src = {S, l, global_block_id(S, l, bps), key};
      m.dst = {D, dl, global_block_id(D, dl, total_[D]), key};
      log_op("alloc", m.dst);
      release(S, l, k);
      log_op("free", m.src);
      moves.push_back(m);
    }
    room -= total_[S];
    unformat_slab(S);
    ++freed;
  }
  if (slabs_freed) *slabs_freed = freed;
  return moves;
}

}  // namespace kvslab
