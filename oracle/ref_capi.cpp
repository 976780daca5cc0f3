// ref_capi.cpp -- TEST / BASELINE INFRASTRUCTURE ONLY (never linked into the product).
//
// A C shim over the UNMODIFIED reference allocator (slabsim::SlabPool,
// /root/reference/proj/core/src/slab_pool.cpp) so Python tests and the
// bench.py CPU-baseline leg can drive the reference itself:
//   - parity: replay an op stream on the reference and on our product pool;
//   - baseline: time the reference's own host path (alloc/free per decode
//     step, and the churn of benchmarks/bench_slab_pool.cpp:34-58).
// Built into oracle/_ref/libslabsim_ref.so by oracle/Makefile (`make ref`).
#include <chrono>
#include <cstdint>
#include <vector>

#include "slabsim/slab_pool.hpp"
#include "slabsim/workload.hpp"

using namespace slabsim;

extern "C" {

void* ref_pool_create(std::uint64_t capacity, std::uint64_t slab, const std::uint64_t* keys,
                      std::uint32_t nkeys, int require_lcm) {
  SlabPoolConfig cfg;
  cfg.capacity_bytes = capacity;
  cfg.slab_size_bytes = slab;
  cfg.block_size_keys.assign(keys, keys + nkeys);
  cfg.require_lcm_alignment = require_lcm != 0;
  try {
    return new SlabPool(cfg);
  } catch (...) {
    return nullptr;
  }
}

void ref_pool_destroy(void* p) { delete static_cast<SlabPool*>(p); }

// out = {slab, local, gid, key}; returns 0 ok, 3 exhausted, 2 invalid key
int ref_try_alloc(void* p, std::uint64_t key, std::uint64_t* out) {
  try {
    auto h = static_cast<SlabPool*>(p)->try_alloc_block(key);
    if (!h) return 3;
    out[0] = h->slab_id;
    out[1] = h->local_block_id;
    out[2] = h->global_block_id;
    out[3] = h->key;
    return 0;
  } catch (...) {
    return 2;
  }
}

int ref_free(void* p, const std::uint64_t* hv) {
  BlockHandle h;
  h.slab_id = static_cast<std::uint32_t>(hv[0]);
  h.local_block_id = static_cast<std::uint32_t>(hv[1]);
  h.global_block_id = hv[2];
  h.key = hv[3];
  try {
    static_cast<SlabPool*>(p)->free_block(h);
    return 0;
  } catch (...) {
    return 4;
  }
}

void ref_stats(void* p, std::uint64_t* out) {
  const FragmentationStats s = static_cast<SlabPool*>(p)->snapshot_stats();
  out[0] = s.allocated_bytes;
  out[1] = s.free_block_bytes;
  out[2] = s.slab_residue_bytes;
  out[3] = s.free_slab_bytes;
}

// Mirror of bm_alloc_free_churn (benchmarks/bench_slab_pool.cpp:25-58):
// 1024 slabs of 48 KiB, keys {4,8,12,24} KiB (first num_keys), seed 42.
// Returns nanoseconds per op over `ops` operations.
double ref_bench_churn(int num_keys, std::uint64_t ops) {
  SlabPoolConfig cfg;
  cfg.slab_size_bytes = 12 * 4096;
  cfg.capacity_bytes = 1024 * cfg.slab_size_bytes;
  const std::vector<Bytes> keys = {4096, 2 * 4096, 3 * 4096, 6 * 4096};
  cfg.block_size_keys.assign(keys.begin(), keys.begin() + num_keys);
  SlabPool pool(cfg);
  Rng rng(42);
  std::vector<BlockHandle> live;
  live.reserve(1 << 16);
  const auto t0 = std::chrono::steady_clock::now();
  for (std::uint64_t i = 0; i < ops; ++i) {
    if (!live.empty() && rng.uniform01() < 0.5) {
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
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return s * 1e9 / static_cast<double>(ops);
}

}  // extern "C"
