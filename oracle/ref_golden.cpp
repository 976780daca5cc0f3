// ref_golden.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Drives the UNMODIFIED reference allocator (slabsim::SlabPool, compiled by
// oracle/Makefile straight from /root/reference/proj/core/src) and the
// reference precision arithmetic, and prints their answers as line-oriented
// golden vectors.  oracle/make_golden.py feeds it op scripts and turns the
// output into tests/golden/*.json|*.npz, which are committed because
// /root/reference does not exist on the GPU box.
//
// Reference interfaces exercised (file:line under /root/reference/proj):
//   SlabPool ctor / alloc / try_alloc / free / stats   core/src/slab_pool.cpp:51-272
//   global_block_id / split_global_block_id             core/include/slabsim/slab_pool.hpp:140-151
//   check_integrity / operator== / flip hook            core/src/slab_pool.cpp:288-386
//   WholeSlabRefModel (the reference's own oracle)      core/src/oracles.cpp:21-85
//   token_size / kv_block_size                          core/src/precision.cpp:76-99
//   Rng::uniform01 (mt19937_64)                         core/include/slabsim/workload.hpp:32-48
//
// Input: one command per line on stdin (see make_golden.py for the grammar).
#include <cinttypes>
#include <cstdio>
#include <iostream>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <typeinfo>
#include <vector>

#include "slabsim/oracles.hpp"
#include "slabsim/precision.hpp"
#include "slabsim/slab_pool.hpp"
#include "slabsim/workload.hpp"

using namespace slabsim;

namespace {

const char* err_name(const std::exception& e) {
  if (dynamic_cast<const InvalidConfigError*>(&e)) return "InvalidConfigError";
  if (dynamic_cast<const InvalidKeyError*>(&e)) return "InvalidKeyError";
  if (dynamic_cast<const InvalidFreeError*>(&e)) return "InvalidFreeError";
  if (dynamic_cast<const PoolExhaustedError*>(&e)) return "PoolExhaustedError";
  if (dynamic_cast<const InvalidProfileError*>(&e)) return "InvalidProfileError";
  if (dynamic_cast<const Error*>(&e)) return "Error";
  return "std::exception";
}

void print_stats(const SlabPool& p) {
  const FragmentationStats s = p.snapshot_stats();
  std::printf(" S %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64, s.allocated_bytes,
              s.free_block_bytes, s.slab_residue_bytes, s.free_slab_bytes);
}

struct Fnv {
  std::uint64_t total = 0;
  std::uint64_t n = 0;
  void add(std::initializer_list<std::uint64_t> fields) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t f : fields) {
      h ^= f;
      h *= 0x100000001b3ull;
    }
    total += h * (2 * n + 1);
    ++n;
  }
};

SlabPoolConfig read_config(std::istringstream& in) {
  SlabPoolConfig cfg;
  int lcm = 1;
  std::size_t nkeys = 0;
  in >> cfg.capacity_bytes >> cfg.slab_size_bytes >> lcm >> nkeys;
  cfg.require_lcm_alignment = lcm != 0;
  cfg.block_size_keys.resize(nkeys);
  for (auto& k : cfg.block_size_keys) in >> k;
  return cfg;
}

// Randomised churn in the shape of test_slab_pool.cpp:240-290 (remove_mode 0,
// order-preserving erase) and acceptance_test.cpp:87-162 (remove_mode 1,
// swap-with-back).  Every op is cross-checked against WholeSlabRefModel; the
// first n_record records are printed, all of them are folded into a hash.
void churn(std::istringstream& in) {
  SlabPoolConfig cfg = read_config(in);
  std::uint64_t seed = 0, nops = 0, n_record = 0;
  int pfree_milli = 0, remove_mode = 0;
  in >> seed >> nops >> pfree_milli >> remove_mode >> n_record;
  const double pfree = pfree_milli / 1000.0;
  SlabPool pool(cfg);
  WholeSlabRefModel ref(cfg);
  Rng rng(seed);
  std::vector<BlockHandle> live;
  Fnv fnv;
  std::uint64_t draws = 0;
  for (std::uint64_t i = 0; i < nops; ++i) {
    std::uint64_t kind, key, slab = 0, local = 0, gid = 0;
    bool do_free = false;
    if (!live.empty()) {
      ++draws;
      do_free = rng.uniform01() < pfree;
    }
    if (do_free) {
      ++draws;
      const std::size_t pick = static_cast<std::size_t>(rng.uniform01() * live.size());
      const BlockHandle h = live[pick];
      pool.free_block(h);
      ref.on_free(h.key, h.slab_id);
      if (remove_mode == 0) {
        live.erase(live.begin() + static_cast<std::ptrdiff_t>(pick));
      } else {
        live[pick] = live.back();
        live.pop_back();
      }
      kind = 2;
      key = h.key;
      slab = h.slab_id;
      local = h.local_block_id;
      gid = h.global_block_id;
    } else {
      ++draws;
      key = cfg.block_size_keys[static_cast<std::size_t>(
          rng.uniform01() * cfg.block_size_keys.size())];
      const bool expect = ref.would_succeed(key);
      auto h = pool.try_alloc_block(key);
      if (h.has_value() != expect) {
        std::fprintf(stderr, "reference disagrees with its own oracle at op %" PRIu64 "\n", i);
        std::exit(3);
      }
      if (h) {
        if (h->slab_id != ref.on_alloc(key)) {
          std::fprintf(stderr, "slab choice mismatch at op %" PRIu64 "\n", i);
          std::exit(3);
        }
        live.push_back(*h);
        kind = 0;
        slab = h->slab_id;
        local = h->local_block_id;
        gid = h->global_block_id;
      } else {
        kind = 1;
      }
    }
    const FragmentationStats s = pool.snapshot_stats();
    if (!(s == ref.ledger())) {
      std::fprintf(stderr, "ledger mismatch at op %" PRIu64 "\n", i);
      std::exit(3);
    }
    fnv.add({kind, key, slab, local, gid, s.allocated_bytes, s.free_block_bytes,
             s.slab_residue_bytes, s.free_slab_bytes});
    if (i < n_record) {
      std::printf("C %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64
                  " %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64 "\n",
                  kind, key, slab, local, gid, s.allocated_bytes, s.free_block_bytes,
                  s.slab_residue_bytes, s.free_slab_bytes);
    }
  }
  std::string why;
  const bool ok = pool.check_integrity(&why);
  std::printf("CH %" PRIu64 " %" PRIu64 " %" PRIu64 " %d %zu", fnv.total, fnv.n, draws,
              ok ? 1 : 0, live.size());
  print_stats(pool);
  std::printf("\n");
}

void run_script(std::istream& in) {
  std::unique_ptr<SlabPool> pool;
  std::unique_ptr<SlabPool> saved;
  std::vector<std::optional<BlockHandle>> results;
  std::string line;
  std::size_t op = 0;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string cmd;
    ls >> cmd;
    if (cmd == "end") {
      std::printf("END\n");
      std::fflush(stdout);
      pool.reset();
      saved.reset();
      results.clear();
      op = 0;
      continue;
    }
    if (cmd == "churn") {
      churn(ls);
      std::fflush(stdout);
      continue;
    }
    if (cmd == "oplog") {  // churn with the reference's own op-log writer
      SlabPoolConfig cfg = read_config(ls);
      std::uint64_t seed = 0, nops = 0;
      ls >> seed >> nops;
      SlabPool pool(cfg);
      pool.set_op_log([](const OpLogRecord& r) {
        std::ostringstream os;
        write_op_log_line(os, r);
        std::printf("L %s", os.str().c_str());
      });
      Rng rng(seed);
      std::vector<BlockHandle> live;
      for (std::uint64_t i = 0; i < nops; ++i) {
        if (!live.empty() && rng.uniform01() < 0.45) {
          const std::size_t pick = static_cast<std::size_t>(rng.uniform01() * live.size());
          pool.free_block(live[pick]);
          live[pick] = live.back();
          live.pop_back();
        } else {
          const Bytes key = cfg.block_size_keys[static_cast<std::size_t>(
              rng.uniform01() * cfg.block_size_keys.size())];
          auto h = pool.try_alloc_block(key);
          if (h) live.push_back(*h);
        }
      }
      std::printf("END\n");
      continue;
    }
    if (cmd == "rng") {
      std::uint64_t seed = 0, n = 0;
      ls >> seed >> n;
      Rng rng(seed);
      std::printf("RNG");
      for (std::uint64_t i = 0; i < n; ++i) std::printf(" %a", rng.uniform01());
      std::printf("\n");
      continue;
    }
    if (cmd == "prec") {
      ModelProfile p;
      p.model_id = "g";
      std::uint64_t qp = 0, tpb = 0;
      ls >> p.num_kv_heads >> p.head_dim >> p.num_layers >> p.tp_degree >> tpb >> qp >>
          p.precision.kv_bits;
      p.tokens_per_block = tpb;
      p.quant_param_bytes_per_block = qp;
      try {
        const Bytes ts = token_size(p);
        const Bytes bs = kv_block_size(p);
        std::printf("P %" PRIu64 " %" PRIu64 "\n", ts, bs);
      } catch (const std::exception& e) {
        std::printf("E %s\n", err_name(e));
      }
      continue;
    }
    std::printf("R %zu", op);
    results.emplace_back();
    try {
      if (cmd == "config") {
        SlabPoolConfig cfg = read_config(ls);
        pool = std::make_unique<SlabPool>(cfg);
        std::printf(" CFG %u %" PRIu64 " %" PRIu64, pool->slab_count(),
                    pool->tail_remainder_bytes(), pool->usable_capacity_bytes());
        print_stats(*pool);
      } else if (cmd == "alloc" || cmd == "try_alloc") {
        Bytes key = 0;
        ls >> key;
        std::optional<BlockHandle> h;
        if (cmd == "alloc") {
          h = pool->alloc_block(key);
        } else {
          h = pool->try_alloc_block(key);
        }
        if (h) {
          std::printf(" H %u %u %" PRIu64 " %" PRIu64, h->slab_id, h->local_block_id,
                      h->global_block_id, h->key);
          results.back() = h;
        } else {
          std::printf(" NONE");
        }
        print_stats(*pool);
      } else if (cmd == "free") {
        std::size_t ref = 0;
        ls >> ref;
        pool->free_block(*results.at(ref));
        std::printf(" OK");
        print_stats(*pool);
      } else if (cmd == "free_raw") {
        BlockHandle h;
        ls >> h.slab_id >> h.local_block_id >> h.global_block_id >> h.key;
        pool->free_block(h);
        std::printf(" OK");
        print_stats(*pool);
      } else if (cmd == "bps") {
        Bytes key = 0;
        ls >> key;
        std::printf(" V %" PRIu64, pool->blocks_per_slab(key));
      } else if (cmd == "free_blocks") {
        Bytes key = 0;
        ls >> key;
        std::printf(" V %" PRIu64, pool->free_blocks_for_key(key));
      } else if (cmd == "alloc_count") {
        Bytes key = 0;
        ls >> key;
        std::printf(" V %" PRIu64,
                    key == 0 ? pool->allocated_block_count() : pool->allocated_block_count(key));
      } else if (cmd == "states") {
        std::printf(" ST %u", pool->slab_count());
        for (std::uint32_t i = 0; i < pool->slab_count(); ++i) {
          std::printf(" %d %" PRIu64, static_cast<int>(pool->slab_state(i)), pool->slab_key(i));
        }
      } else if (cmd == "integrity") {
        std::string why;
        std::printf(" I %d", pool->check_integrity(&why) ? 1 : 0);
      } else if (cmd == "flip") {
        std::uint32_t s = 0, l = 0;
        ls >> s >> l;
        pool->debug_flip_occupancy_bit(s, l);
        std::printf(" OK");
      } else if (cmd == "save") {
        saved = std::make_unique<SlabPool>(*pool);
        std::printf(" OK");
      } else if (cmd == "equal_saved") {
        std::printf(" EQ %d", (*pool == *saved) ? 1 : 0);
      } else if (cmd == "gid") {
        std::uint64_t s = 0, l = 0, bps = 0;
        ls >> s >> l >> bps;
        const auto g = SlabPool::global_block_id(static_cast<std::uint32_t>(s),
                                                 static_cast<std::uint32_t>(l), bps);
        const auto [s2, l2] = SlabPool::split_global_block_id(g, bps);
        std::printf(" G %" PRIu64 " %u %u", g, s2, l2);
      } else {
        std::printf(" E UnknownCommand");
      }
    } catch (const std::exception& e) {
      std::printf(" E %s", err_name(e));
    }
    std::printf("\n");
    ++op;
  }
}

}  // namespace

int main() {
  run_script(std::cin);
  return 0;
}
