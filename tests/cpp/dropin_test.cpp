// Compiles reference-style code (slabsim:: names, reference headers' paths)
// against libkvslab.so and re-runs checks of proj/tests/test_slab_pool.cpp.
#include <cstdio>
#include <optional>
#include <string>
#include <vector>

#include "slabsim/slab_pool.hpp"

using namespace slabsim;

static int failures = 0;
#define CHECK(x) do { if (!(x)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); ++failures; } } while (0)
template <class E, class F>
static bool throws(F f) { try { f(); } catch (const E&) { return true; } catch (...) { return false; } return false; }

int main() {
  constexpr Bytes kKiB = 1024;
  SlabPoolConfig two;  // test_slab_pool.cpp:28-34
  two.capacity_bytes = 4 * 64 * kKiB;
  two.slab_size_bytes = 64 * kKiB;
  two.block_size_keys = {64 * kKiB, 32 * kKiB};
  {  // :78-100 global ids
    SlabPoolConfig cfg = two;
    cfg.block_size_keys = {32 * kKiB};
    SlabPool pool(cfg);
    CHECK(pool.blocks_per_slab(32 * kKiB) == 2);
    BlockHandle a = pool.alloc_block(32 * kKiB), b = pool.alloc_block(32 * kKiB),
                c = pool.alloc_block(32 * kKiB);
    CHECK(a.global_block_id == 0 && b.global_block_id == 1);
    CHECK(c.slab_id == 1 && c.local_block_id == 0 && c.global_block_id == 2);
    auto [s, l] = SlabPool::split_global_block_id(c.global_block_id, 2);
    CHECK(s == 1 && l == 0);
  }
  {  // :117-130 exhaustion and key mismatch
    SlabPool pool(two);
    for (int i = 0; i < 3; ++i) pool.alloc_block(64 * kKiB);
    pool.alloc_block(32 * kKiB);
    CHECK(pool.free_blocks_for_key(32 * kKiB) == 1);
    CHECK(pool.try_alloc_block(64 * kKiB) == std::nullopt);
    CHECK(throws<PoolExhaustedError>([&] { pool.alloc_block(64 * kKiB); }));
    CHECK(throws<InvalidKeyError>([&] { pool.alloc_block(1234); }));
  }
  {  // :132-160 free transitions
    SlabPoolConfig cfg = two;
    cfg.capacity_bytes = 2 * 64 * kKiB;
    cfg.block_size_keys = {32 * kKiB, 64 * kKiB};
    SlabPool pool(cfg);
    BlockHandle a = pool.alloc_block(32 * kKiB), b = pool.alloc_block(32 * kKiB);
    CHECK(pool.slab_state(a.slab_id) == SlabState::kFull);
    pool.free_block(a);
    CHECK(pool.slab_state(a.slab_id) == SlabState::kPartial);
    pool.free_block(b);
    CHECK(pool.slab_state(a.slab_id) == SlabState::kFree);
    BlockHandle c = pool.alloc_block(64 * kKiB);
    CHECK(c.slab_id == 0);
    CHECK(throws<InvalidFreeError>([&] { pool.free_block(b); }));
    pool.free_block(c);
    CHECK(throws<InvalidFreeError>([&] { pool.free_block(c); }));
  }
  {  // :162-186 residue with relaxed alignment
    SlabPoolConfig u;
    u.capacity_bytes = 45;
    u.slab_size_bytes = 15;
    u.block_size_keys = {4};
    CHECK(throws<InvalidConfigError>([&] { SlabPool p(u); }));
    u.require_lcm_alignment = false;
    SlabPool relaxed(u);
    relaxed.alloc_block(4);
    FragmentationStats st = relaxed.snapshot_stats();
    CHECK(st.slab_residue_bytes == 3 && st.allocated_bytes == 4 && st.free_block_bytes == 8 &&
          st.free_slab_bytes == 30 && st.usable_capacity() == 45);
  }
  {  // :204-212 round trip + :292-300 integrity + :302-313 op log
    SlabPool pool(two);
    pool.alloc_block(32 * kKiB);
    const SlabPool before = pool;
    const BlockHandle h = pool.alloc_block(64 * kKiB);
    CHECK(!(pool == before));
    pool.free_block(h);
    CHECK(pool == before);
    std::vector<OpLogRecord> log;
    pool.set_op_log([&](const OpLogRecord& r) { log.push_back(r); });
    const BlockHandle g = pool.alloc_block(32 * kKiB);
    pool.free_block(g);
    CHECK(log.size() == 2 && std::string(log[0].op) == "alloc" && std::string(log[1].op) == "free");
    std::string why;
    CHECK(pool.check_integrity(&why));
    pool.debug_flip_occupancy_bit(0, 1);
    CHECK(!pool.check_integrity(&why) && !why.empty());
  }
  kvslab::KvGeometry g;  // precision.cpp:76-99, test_precision.cpp:23-51 (kvslab's geometry helpers)
  g.num_kv_heads = 8;
  g.head_dim = 128;
  g.kv_bits = 8;
  g.quant_param_bytes_per_block = 64;
  CHECK(kvslab::token_size(g) == 2048 && kvslab::kv_block_size(g) == 32832);
  // kvslab's errors ARE slabsim's: a reference-style catch clause sees them
  CHECK(throws<slabsim::InvalidKeyError>([&] { SlabPool p(two); p.alloc_block(3); }));
  CHECK(throws<slabsim::Error>([&] { SlabPool p(two); p.free_block(BlockHandle{}); }));
  std::printf(failures ? "dropin: %d failures\n" : "dropin: all checks passed\n", failures);
  return failures ? 1 : 0;
}
