// capi.cpp -- the extern "C" boundary (include/kvslab.h).
//
// Exceptions never cross this layer: each entry point catches the kvslab
// error classes (named after slabsim's, common.hpp:31-59) and maps them to
// ks_status, keeping the message in a thread-local for ks_last_error().
#include "kvslab.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "kvslab/seq_table.hpp"
#include "kvslab/slab_pool.hpp"
#include "launch.hpp"

using kvslab::BlockHandle;
using kvslab::SeqTable;
using kvslab::SlabPool;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

ks_status fail(ks_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

template <class F>
ks_status guarded(F&& f) {
  try {
    return f();
  } catch (const kvslab::InvalidConfigError& e) {
    return fail(KS_INVALID_CONFIG, e.what());
  } catch (const kvslab::InvalidKeyError& e) {
    return fail(KS_INVALID_KEY, e.what());
  } catch (const kvslab::PoolExhaustedError& e) {
    return fail(KS_EXHAUSTED, e.what());
  } catch (const kvslab::InvalidFreeError& e) {
    return fail(KS_INVALID_FREE, e.what());
  } catch (const kvslab::InvalidProfileError& e) {
    return fail(KS_INVALID_PROFILE, e.what());
  } catch (const std::out_of_range& e) {
    return fail(KS_INVALID_ARGUMENT, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(KS_INVALID_ARGUMENT, e.what());
  } catch (const std::bad_alloc&) {
    return fail(KS_INTERNAL, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(KS_INTERNAL, e.what());
  }
}

ks_status cuda_fail(cudaError_t e, const char* where) {
  return fail(KS_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

ks_block_handle to_c(const BlockHandle& h) {
  ks_block_handle o;
  o.slab_id = h.slab_id;
  o.local_block_id = h.local_block_id;
  o.global_block_id = h.global_block_id;
  o.key = h.key;
  return o;
}
BlockHandle from_c(const ks_block_handle& h) {
  BlockHandle o;
  o.slab_id = h.slab_id;
  o.local_block_id = h.local_block_id;
  o.global_block_id = h.global_block_id;
  o.key = h.key;
  return o;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

constexpr size_t kStageWords = 1u << 20;  // 4 MiB of uint32 staging

}  // namespace

namespace kvslab {
Tuning Tuning::from_env() {
  Tuning t;
  auto num = [](const char* name, long dflt) {
    const char* v = std::getenv(name);
    return v ? std::strtol(v, nullptr, 0) : dflt;
  };
  t.decode_max_ctas = static_cast<int>(num("KVSLAB_DECODE_MAX_CTAS", 0));
  t.decode_hg = static_cast<uint32_t>(num("KVSLAB_DECODE_HG", 0));
  t.decode_smem = static_cast<uint32_t>(num("KVSLAB_DECODE_SMEM", 0));
  t.merge_threads = static_cast<uint32_t>(num("KVSLAB_MERGE_THREADS", 0));
  t.merge_dc = static_cast<uint32_t>(num("KVSLAB_MERGE_DC", 0));
  t.decode_pack = static_cast<uint32_t>(num("KVSLAB_DECODE_PACK", 0));
  t.pdl = num("KVSLAB_NO_PDL", 0) ? 0 : 1;
  t.append_per_sm = static_cast<uint32_t>(num("KVSLAB_APPEND_PER_SM", 0));
  t.decode_min_blocks = static_cast<uint32_t>(num("KVSLAB_DECODE_MIN_BLOCKS", 0));
  t.prefill_nt = static_cast<uint32_t>(num("KVSLAB_PREFILL_NT", 0));
  t.prefill_tc = static_cast<int>(num("KVSLAB_PREFILL_TC", 2));
  t.prefill_expand = static_cast<int>(num("KVSLAB_PREFILL_EXPAND", -1));
  t.prefill_split = static_cast<int>(num("KVSLAB_PREFILL_SPLIT", 1));
  if (kProbes) {
    t.decode_debug = static_cast<int>(num("KVSLAB_DECODE_DEBUG", 0));
    t.prefill_debug = static_cast<int>(num("KVSLAB_PREFILL_DEBUG", 0));
  }
  return t;
}
}  // namespace kvslab

struct ks_pool {
  // Pinned host -> device staging ring for small control uploads (table
  // deltas, move lists).  A slot is reused only after the kernel that read it
  // completed (its event), so calls on different streams never race.
  static constexpr int kSlots = 8;
  static constexpr size_t kSlotWords = kStageWords / kSlots;
  struct Slot {
    uint32_t* h = nullptr;
    uint32_t* d = nullptr;
  };

  std::unique_ptr<SlabPool> pool;
  int device = -1;
  int num_sms = 0;
  uint8_t* d_base = nullptr;
  uint64_t d_bytes = 0;
  void* d_slab_table = nullptr;
  uint32_t* h_stage = nullptr;  // pinned, kStageWords
  uint32_t* d_stage = nullptr;  // device, kStageWords
  cudaEvent_t slot_ev[kSlots] = {};
  bool slot_pending[kSlots] = {};
  int next_slot = 0;
  ks_op_log_fn log_fn = nullptr;
  void* log_user = nullptr;
  ks_clock_fn clock_fn = nullptr;
  void* clock_user = nullptr;
  std::vector<uint32_t> dirty;
  std::map<uint64_t, uint32_t> cta_budget;  // per key: K2 CTAs (SM share), 0 = all
  // Engine tables registered on this pool (ks_seq_table_create); compaction
  // remaps every table of the compacted key, whoever owns it.
  std::vector<ks_seq_table*> tables;
  // Compaction fence: source slabs return FREE on the host before their
  // bytes leave on the compaction stream, so until that work completes every
  // launch on another stream waits for it (wait_fence).
  cudaEvent_t fence = nullptr;
  cudaStream_t fence_stream = nullptr;
  bool fence_pending = false;
  // Tuning overrides, read from the environment once at pool creation.
  kvslab::Tuning tuning;
  std::vector<uint32_t> scrub;  // scratch for scrub_slabs
  uint64_t scrubbed_bytes = 0;

  ~ks_pool();
  void destroy_device() {
    if (device >= 0) {
      DeviceGuard g(device);
      // A pool may be destroyed (e.g. by a garbage collector) while another
      // stream of this thread is being captured into a graph; in the default
      // global capture mode cudaFree / cudaEventSynchronize would invalidate
      // that capture.  Relaxed mode for this thread while we tear down.
      cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
      const bool swapped = cudaThreadExchangeStreamCaptureMode(&mode) == cudaSuccess;
      if (fence) cudaEventSynchronize(fence), cudaEventDestroy(fence);
      for (int i = 0; i < kSlots; ++i)
        if (slot_ev[i]) cudaEventSynchronize(slot_ev[i]), cudaEventDestroy(slot_ev[i]);
      cudaFree(d_base);
      cudaFree(d_slab_table);
      cudaFree(d_stage);
      cudaFreeHost(h_stage);
      if (swapped) cudaThreadExchangeStreamCaptureMode(&mode);
    }
  }
  // Next staging slot, waiting for its previous consumer if still running.
  cudaError_t acquire(int* idx, Slot* s) {
    const int i = next_slot;
    next_slot = (next_slot + 1) % kSlots;
    if (slot_pending[i]) {
      slot_pending[i] = false;
      cudaError_t e = cudaEventSynchronize(slot_ev[i]);
      if (e != cudaSuccess) return e;
    }
    *idx = i;
    s->h = h_stage + i * kSlotWords;
    s->d = d_stage + i * kSlotWords;
    return cudaSuccess;
  }
  cudaError_t upload(const Slot& s, size_t words, cudaStream_t st) {
    return cudaMemcpyAsync(s.d, s.h, words * 4, cudaMemcpyHostToDevice, st);
  }
  // Marks the slot busy until the work just enqueued on `st` finishes.
  cudaError_t release(int i, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(slot_ev[i], st);
    slot_pending[i] = e == cudaSuccess;
    return e;
  }
};

struct ks_seq_table {
  ks_pool* owner = nullptr;  // null once the pool is destroyed
  std::unique_ptr<kvslab::SeqTable> t;
  int32_t* d_table = nullptr;
  uint32_t row_stride = 0;
};

ks_pool::~ks_pool() {
  for (ks_seq_table* t : tables) t->owner = nullptr;
  destroy_device();
}

namespace {

// Orders `s` after a pending compaction (see ks_pool::fence).  Eager launches
// only: a stream being captured into a graph is left alone (graphs are
// replayed later, after the compaction stream's work was enqueued).
cudaError_t wait_fence(ks_pool* p, cudaStream_t s) {
  if (!p->fence_pending) return cudaSuccess;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &cs);
  if (e != cudaSuccess || cs != cudaStreamCaptureStatusNone) return e;
  e = cudaEventQuery(p->fence);
  if (e == cudaSuccess) {
    p->fence_pending = false;
    return cudaSuccess;
  }
  if (e != cudaErrorNotReady) return e;
  if (s == p->fence_stream) return cudaSuccess;
  return cudaStreamWaitEvent(s, p->fence, 0);
}

// Clears the slabs the allocator re-formatted to a different key since the
// last call (SlabPool::drain_scrub_slabs), on `s`, ahead of the launch that
// follows.  Not while `s` is being captured: a graph must not replay it.
cudaError_t scrub_slabs(ks_pool* p, cudaStream_t s) {
  if (!p->pool->has_scrub_slabs()) return cudaSuccess;  // the common case: no runtime call
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &cs);
  if (e != cudaSuccess || cs != cudaStreamCaptureStatusNone) return e;
  p->pool->drain_scrub_slabs(&p->scrub);
  const uint64_t slab = p->pool->slab_size();
  for (uint32_t id : p->scrub) {
    e = cudaMemsetAsync(p->d_base + static_cast<uint64_t>(id) * slab, 0, slab, s);
    if (e != cudaSuccess) return e;
  }
  p->scrubbed_bytes += p->scrub.size() * slab;
  return cudaSuccess;
}

// The launch prologue of every device entry point that reads or writes KV:
// order after a pending compaction, then clear re-formatted slabs.
cudaError_t prepare(ks_pool* p, cudaStream_t s) {
  cudaError_t e = wait_fence(p, s);
  return e != cudaSuccess ? e : scrub_slabs(p, s);
}

uint32_t fmt_bits(uint32_t dt) { return dt == KS_KV_FP16 ? 16 : (dt == KS_KV_INT4 ? 4 : 8); }

struct FmtInfo {
  uint64_t token_size, chunk, layer_bytes, key, natural_qp;
};
ks_status fmt_info(const ks_kv_format* f, FmtInfo* o) {
  if (!f) return fail(KS_INVALID_ARGUMENT, "null format");
  if (f->kv_dtype > KS_KV_INT4) return fail(KS_INVALID_ARGUMENT, "unknown kv_dtype");
  if (f->num_kv_heads == 0 || f->head_dim == 0 || f->num_layers == 0 || f->tokens_per_block == 0)
    return fail(KS_INVALID_ARGUMENT, "format counts must be positive");
  if (f->num_q_heads == 0 || f->num_q_heads % f->num_kv_heads != 0)
    return fail(KS_INVALID_ARGUMENT, "num_q_heads must be a positive multiple of num_kv_heads");
  const uint64_t bits = fmt_bits(f->kv_dtype);
  const uint64_t H = f->num_kv_heads, T = f->tokens_per_block;
  o->token_size = H * f->head_dim * 2 * bits / 8;
  o->chunk = T * f->head_dim * bits / 8;
  o->layer_bytes = T * o->token_size + f->quant_param_bytes_per_block;
  o->key = f->num_layers * o->layer_bytes;
  switch (f->kv_dtype) {
    case KS_KV_FP8_E4M3: o->natural_qp = 2 * H * 4; break;
    case KS_KV_INT8: o->natural_qp = 2 * H * T * 2; break;
    case KS_KV_INT4: o->natural_qp = 2 * H * T * 4; break;
    default: o->natural_qp = 0;
  }
  const uint64_t qp = f->quant_param_bytes_per_block;
  const bool qp_ok = qp == o->natural_qp || (f->kv_dtype == KS_KV_FP8_E4M3 && qp == 0);
  if (!qp_ok)
    return fail(KS_INVALID_ARGUMENT, "quant_param_bytes_per_block must be the format's natural size");
  return KS_OK;
}

ks_status check_kernel_format(const ks_pool* pool, const ks_kv_format* f, FmtInfo* fi) {
  ks_status s = fmt_info(f, fi);
  if (s != KS_OK) return s;
  if (f->head_dim != 128) return fail(KS_NOT_SUPPORTED, "kernels require head_dim == 128");
  if (f->tokens_per_block != 16) return fail(KS_NOT_SUPPORTED, "kernels require tokens_per_block == 16");
  if (f->num_q_heads / f->num_kv_heads > 16) return fail(KS_NOT_SUPPORTED, "GQA group > 16");
  if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
  if (pool->device < 0 || !pool->d_base) return fail(KS_INVALID_ARGUMENT, "pool has no device tensor");
  if (pool->pool->slab_size() % 16 != 0 || fi->key % 16 != 0 || fi->layer_bytes % 16 != 0)
    return fail(KS_NOT_SUPPORTED, "slab size, key and layer stride must be multiples of 16 bytes");
  pool->pool->blocks_per_slab(fi->key);  // throws InvalidKeyError when unregistered
  return KS_OK;
}

}  // namespace

extern "C" {

uint32_t ks_abi_version(void) { return KS_ABI_VERSION; }
const char* ks_last_error(void) { return g_err.c_str(); }
uint64_t ks_launch_count(void) { return g_launches.load(); }

const char* ks_status_name(ks_status s) {
  switch (s) {
    case KS_OK: return "KS_OK";
    case KS_INVALID_CONFIG: return "KS_INVALID_CONFIG";
    case KS_INVALID_KEY: return "KS_INVALID_KEY";
    case KS_EXHAUSTED: return "KS_EXHAUSTED";
    case KS_INVALID_FREE: return "KS_INVALID_FREE";
    case KS_INVALID_PROFILE: return "KS_INVALID_PROFILE";
    case KS_INVALID_ARGUMENT: return "KS_INVALID_ARGUMENT";
    case KS_CUDA_ERROR: return "KS_CUDA_ERROR";
    case KS_NOT_SUPPORTED: return "KS_NOT_SUPPORTED";
    default: return "KS_INTERNAL";
  }
}

// ------------------------------------------------------------- geometry
static kvslab::KvGeometry to_geo(const ks_model_geometry* g) {
  kvslab::KvGeometry o;
  o.num_kv_heads = g->num_kv_heads;
  o.head_dim = g->head_dim;
  o.num_layers = g->num_layers;
  o.tp_degree = g->tp_degree;
  o.tokens_per_block = g->tokens_per_block;
  o.quant_param_bytes_per_block = g->quant_param_bytes_per_block;
  o.kv_bits = g->kv_bits;
  return o;
}
ks_status ks_token_size(const ks_model_geometry* g, uint64_t* out) {
  return guarded([&] {
    if (!g || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = kvslab::token_size(to_geo(g));
    return KS_OK;
  });
}
ks_status ks_kv_block_size(const ks_model_geometry* g, uint64_t* out) {
  return guarded([&] {
    if (!g || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = kvslab::kv_block_size(to_geo(g));
    return KS_OK;
  });
}

// ------------------------------------------------------------- pool
ks_status ks_pool_create(const ks_pool_config* cfg, int device, ks_pool** out) {
  return guarded([&] {
    if (!cfg || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    kvslab::SlabPoolConfig c;
    c.capacity_bytes = cfg->capacity_bytes;
    c.slab_size_bytes = cfg->slab_size_bytes;
    if (cfg->num_keys && !cfg->block_size_keys) return fail(KS_INVALID_ARGUMENT, "null keys");
    c.block_size_keys.assign(cfg->block_size_keys, cfg->block_size_keys + cfg->num_keys);
    c.require_lcm_alignment = cfg->require_lcm_alignment != 0;
    auto p = std::make_unique<ks_pool>();
    p->pool = std::make_unique<SlabPool>(c);
    if (device >= 0) {
      DeviceGuard g(device);
      if (!g.ok) return fail(KS_CUDA_ERROR, "cudaSetDevice failed");
      p->device = device;
      cudaError_t e = cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
      if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
      p->d_bytes = p->pool->usable_capacity_bytes();
      e = cudaMalloc(&p->d_base, p->d_bytes);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(KV tensor)");
      // Zero-filled once: the slots of a block past a sequence's context are
      // read by the kernels and masked through P = 0, which would turn a NaN
      // or Inf bit pattern left in fresh device memory into a NaN output.
      // (Reused blocks hold earlier appended, finite values.)
      e = cudaMemset(p->d_base, 0, p->d_bytes);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(KV tensor)");
      const size_t tbytes = static_cast<size_t>(p->pool->slab_count()) * 16;
      e = cudaMalloc(&p->d_slab_table, tbytes);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(slab table)");
      e = cudaMemset(p->d_slab_table, 0, tbytes);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(slab table)");
      e = cudaMallocHost(&p->h_stage, kStageWords * 4);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost(staging)");
      e = cudaMalloc(&p->d_stage, kStageWords * 4);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
      for (int i = 0; i < ks_pool::kSlots; ++i) {
        e = cudaEventCreateWithFlags(&p->slot_ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
      }
      e = cudaEventCreateWithFlags(&p->fence, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
      p->tuning = kvslab::Tuning::from_env();
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
    }
    *out = p.release();
    return KS_OK;
  });
}

ks_status ks_pool_destroy(ks_pool* pool) {
  delete pool;
  return KS_OK;
}

ks_status ks_pool_get_info(const ks_pool* pool, ks_pool_info* out) {
  if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
  const SlabPool& p = *pool->pool;
  out->slab_count = p.slab_count();
  out->num_keys = static_cast<uint32_t>(p.config().block_size_keys.size());
  out->slab_size_bytes = p.slab_size();
  out->tail_remainder_bytes = p.tail_remainder_bytes();
  out->usable_capacity_bytes = p.usable_capacity_bytes();
  out->allocated_blocks = p.allocated_block_count();
  out->device = pool->device;
  out->require_lcm_alignment = p.config().require_lcm_alignment ? 1 : 0;
  return KS_OK;
}

ks_status ks_pool_scrubbed_bytes(const ks_pool* pool, uint64_t* bytes) {
  if (!pool || !bytes) return fail(KS_INVALID_ARGUMENT, "null argument");
  *bytes = pool->scrubbed_bytes;
  return KS_OK;
}

ks_status ks_pool_keys(const ks_pool* pool, uint64_t* keys_out, uint32_t capacity) {
  if (!pool || (!keys_out && capacity)) return fail(KS_INVALID_ARGUMENT, "null argument");
  const auto& k = pool->pool->config().block_size_keys;
  if (capacity < k.size()) return fail(KS_INVALID_ARGUMENT, "capacity too small");
  std::copy(k.begin(), k.end(), keys_out);
  return KS_OK;
}

ks_status ks_alloc_block(ks_pool* pool, uint64_t key, ks_block_handle* out) {
  return guarded([&] {
    if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = to_c(pool->pool->alloc_block(key));
    return KS_OK;
  });
}

ks_status ks_try_alloc_block(ks_pool* pool, uint64_t key, ks_block_handle* out, int32_t* ok) {
  return guarded([&] {
    if (!pool || !out || !ok) return fail(KS_INVALID_ARGUMENT, "null argument");
    auto h = pool->pool->try_alloc_block(key);
    *ok = h ? 1 : 0;
    if (h) *out = to_c(*h);
    return KS_OK;
  });
}

ks_status ks_alloc_blocks(ks_pool* pool, uint64_t key, uint32_t n, ks_block_handle* out,
                          uint32_t* n_done) {
  return guarded([&] {
    if (!pool || (!out && n) || !n_done) return fail(KS_INVALID_ARGUMENT, "null argument");
    *n_done = 0;
    for (uint32_t i = 0; i < n; ++i) {
      auto h = pool->pool->try_alloc_block(key);
      if (!h) break;
      out[i] = to_c(*h);
      ++*n_done;
    }
    return KS_OK;
  });
}

ks_status ks_free_block(ks_pool* pool, const ks_block_handle* h) {
  return guarded([&] {
    if (!pool || !h) return fail(KS_INVALID_ARGUMENT, "null argument");
    pool->pool->free_block(from_c(*h));
    return KS_OK;
  });
}

ks_status ks_free_blocks(ks_pool* pool, const ks_block_handle* hs, uint32_t n) {
  return guarded([&] {
    if (!pool || (!hs && n)) return fail(KS_INVALID_ARGUMENT, "null argument");
    for (uint32_t i = 0; i < n; ++i) pool->pool->free_block(from_c(hs[i]));
    return KS_OK;
  });
}

ks_status ks_blocks_per_slab(const ks_pool* pool, uint64_t key, uint64_t* out) {
  return guarded([&] {
    if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = pool->pool->blocks_per_slab(key);
    return KS_OK;
  });
}

ks_status ks_snapshot_stats(const ks_pool* pool, ks_frag_stats* out) {
  if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
  const auto s = pool->pool->snapshot_stats();
  out->allocated_bytes = s.allocated_bytes;
  out->free_block_bytes = s.free_block_bytes;
  out->slab_residue_bytes = s.slab_residue_bytes;
  out->free_slab_bytes = s.free_slab_bytes;
  return KS_OK;
}

ks_status ks_free_blocks_for_key(const ks_pool* pool, uint64_t key, uint64_t* out) {
  return guarded([&] {
    if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = pool->pool->free_blocks_for_key(key);
    return KS_OK;
  });
}

ks_status ks_allocated_block_count(const ks_pool* pool, uint64_t key, uint64_t* out) {
  return guarded([&] {
    if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = key == 0 ? pool->pool->allocated_block_count() : pool->pool->allocated_block_count(key);
    return KS_OK;
  });
}

ks_status ks_slab_state(const ks_pool* pool, uint32_t slab_id, int32_t* state, uint64_t* key) {
  return guarded([&] {
    if (!pool || !state || !key) return fail(KS_INVALID_ARGUMENT, "null argument");
    *state = static_cast<int32_t>(pool->pool->slab_state(slab_id));
    *key = pool->pool->slab_key(slab_id);
    return KS_OK;
  });
}

ks_status ks_check_integrity(const ks_pool* pool, int32_t* ok) {
  if (!pool || !ok) return fail(KS_INVALID_ARGUMENT, "null argument");
  std::string why;
  *ok = pool->pool->check_integrity(&why) ? 1 : 0;
  if (!*ok) g_err = why;
  return KS_OK;
}

ks_status ks_pool_equal(const ks_pool* a, const ks_pool* b, int32_t* equal) {
  if (!a || !b || !equal) return fail(KS_INVALID_ARGUMENT, "null argument");
  *equal = (*a->pool == *b->pool) ? 1 : 0;
  return KS_OK;
}

ks_status ks_pool_clone_host(const ks_pool* pool, ks_pool** out) {
  return guarded([&] {
    if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    auto p = std::make_unique<ks_pool>();
    p->pool = std::make_unique<SlabPool>(*pool->pool);
    p->pool->set_op_log(nullptr);
    p->pool->set_clock(nullptr);
    *out = p.release();
    return KS_OK;
  });
}

ks_status ks_set_op_log(ks_pool* pool, ks_op_log_fn fn, void* user) {
  if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
  pool->log_fn = fn;
  pool->log_user = user;
  if (!fn) {
    pool->pool->set_op_log(nullptr);
    return KS_OK;
  }
  pool->pool->set_op_log([pool](const kvslab::OpLogRecord& r) {
    ks_op_record c;
    c.seq = r.seq;
    c.time = r.time;
    c.op = r.op;
    c.key = r.key;
    c.slab_id = r.slab_id;
    c.local_block_id = r.local_block_id;
    c.global_block_id = r.global_block_id;
    pool->log_fn(&c, pool->log_user);
  });
  return KS_OK;
}

ks_status ks_set_clock(ks_pool* pool, ks_clock_fn fn, void* user) {
  if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
  pool->clock_fn = fn;
  pool->clock_user = user;
  if (!fn) {
    pool->pool->set_clock(nullptr);
  } else {
    pool->pool->set_clock([pool]() { return pool->clock_fn(pool->clock_user); });
  }
  return KS_OK;
}

ks_status ks_debug_flip_occupancy_bit(ks_pool* pool, uint32_t slab_id, uint32_t local) {
  return guarded([&] {
    if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
    pool->pool->debug_flip_occupancy_bit(slab_id, local);
    return KS_OK;
  });
}

uint64_t ks_global_block_id(uint32_t slab_id, uint32_t local_block_id, uint64_t bps) {
  return SlabPool::global_block_id(slab_id, local_block_id, bps);
}
void ks_split_global_block_id(uint64_t gid, uint64_t bps, uint32_t* slab_id, uint32_t* local) {
  const auto [s, l] = SlabPool::split_global_block_id(gid, bps);
  if (slab_id) *slab_id = s;
  if (local) *local = l;
}
ks_status ks_block_byte_offset(const ks_pool* pool, uint64_t key, uint64_t gid, uint64_t* out) {
  return guarded([&] {
    if (!pool || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = pool->pool->block_byte_offset(key, gid);
    return KS_OK;
  });
}

// ------------------------------------------------------------- formats
ks_status ks_natural_qparams(const ks_kv_format* fmt, uint64_t* out) {
  if (!fmt || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
  ks_kv_format f = *fmt;
  FmtInfo fi;
  // natural size does not depend on the declared qparams; probe with it
  const uint64_t H = f.num_kv_heads, T = f.tokens_per_block;
  switch (f.kv_dtype) {
    case KS_KV_FP16: *out = 0; break;
    case KS_KV_FP8_E4M3: *out = 2 * H * 4; break;
    case KS_KV_INT8: *out = 2 * H * T * 2; break;
    case KS_KV_INT4: *out = 2 * H * T * 4; break;
    default: return fail(KS_INVALID_ARGUMENT, "unknown kv_dtype");
  }
  (void)fi;
  return KS_OK;
}

ks_status ks_format_key(const ks_kv_format* fmt, uint64_t* out) {
  if (!out) return fail(KS_INVALID_ARGUMENT, "null argument");
  FmtInfo fi;
  ks_status s = fmt_info(fmt, &fi);
  if (s != KS_OK) return s;
  *out = fi.key;
  return KS_OK;
}

ks_status ks_validate_format(const ks_pool* pool, const ks_kv_format* fmt) {
  return guarded([&] {
    FmtInfo fi;
    return check_kernel_format(pool, fmt, &fi);
  });
}

// ------------------------------------------------------------- device
ks_status ks_device_base(const ks_pool* pool, void** d_base, uint64_t* bytes) {
  if (!pool || !d_base) return fail(KS_INVALID_ARGUMENT, "null argument");
  *d_base = pool->d_base;
  if (bytes) *bytes = pool->d_bytes;
  return KS_OK;
}

ks_status ks_slab_table_device(const ks_pool* pool, const void** d_table) {
  if (!pool || !d_table) return fail(KS_INVALID_ARGUMENT, "null argument");
  *d_table = pool->d_slab_table;
  return KS_OK;
}

ks_status ks_slab_table_sync(ks_pool* pool, void* stream) {
  return guarded([&] {
    if (!pool || pool->device < 0) return fail(KS_INVALID_ARGUMENT, "pool has no device tensor");
    DeviceGuard g(pool->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    pool->pool->drain_dirty_slabs(&pool->dirty);
    size_t i = 0;
    while (i < pool->dirty.size()) {
      const size_t n = std::min(pool->dirty.size() - i, ks_pool::kSlotWords / 5);
      int si = 0;
      ks_pool::Slot sl;
      cudaError_t e = pool->acquire(&si, &sl);
      if (e != cudaSuccess) return cuda_fail(e, "staging wait");
      for (size_t j = 0; j < n; ++j) {
        const uint32_t slab = pool->dirty[i + j];
        const uint64_t key = pool->pool->slab_key(slab);
        uint32_t* w = sl.h + 5 * j;
        w[0] = slab;
        w[1] = static_cast<uint32_t>(key);
        w[2] = static_cast<uint32_t>(key >> 32);
        w[3] = pool->pool->slab_blocks_total(slab);
        w[4] = static_cast<uint32_t>(pool->pool->slab_state(slab));
      }
      e = pool->upload(sl, 5 * n, s);
      if (e != cudaSuccess) return cuda_fail(e, "staging upload");
      e = kvslab::launch_slab_table_scatter(pool->d_slab_table, sl.d, static_cast<uint32_t>(n), s);
      if (e != cudaSuccess) return cuda_fail(e, "slab table scatter");
      e = pool->release(si, s);
      if (e != cudaSuccess) return cuda_fail(e, "staging release");
      ++g_launches;
      i += n;
    }
    return KS_OK;
  });
}

ks_status ks_block_table_update(ks_pool* pool, int32_t* d_table, uint32_t row_stride,
                                const int32_t* rows, const int32_t* cols, const int32_t* vals,
                                uint32_t n, void* stream) {
  return guarded([&] {
    if (!pool || pool->device < 0) return fail(KS_INVALID_ARGUMENT, "pool has no device tensor");
    if (n == 0) return KS_OK;
    if (!d_table || !rows || !cols || !vals) return fail(KS_INVALID_ARGUMENT, "null argument");
    DeviceGuard g(pool->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t fe = prepare(pool, s);
    if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
    uint32_t i = 0;
    while (i < n) {
      const uint32_t m = static_cast<uint32_t>(std::min<size_t>(n - i, ks_pool::kSlotWords / 3));
      int si = 0;
      ks_pool::Slot sl;
      cudaError_t e = pool->acquire(&si, &sl);
      if (e != cudaSuccess) return cuda_fail(e, "staging wait");
      for (uint32_t j = 0; j < m; ++j) {
        sl.h[3 * j] = static_cast<uint32_t>(rows[i + j]);
        sl.h[3 * j + 1] = static_cast<uint32_t>(cols[i + j]);
        sl.h[3 * j + 2] = static_cast<uint32_t>(vals[i + j]);
      }
      e = pool->upload(sl, 3 * static_cast<size_t>(m), s);
      if (e != cudaSuccess) return cuda_fail(e, "staging upload");
      e = kvslab::launch_table_scatter(d_table, row_stride, reinterpret_cast<const int32_t*>(sl.d),
                                       m, s);
      if (e != cudaSuccess) return cuda_fail(e, "table scatter");
      e = pool->release(si, s);
      if (e != cudaSuccess) return cuda_fail(e, "staging release");
      ++g_launches;
      i += m;
    }
    return KS_OK;
  });
}

ks_status ks_block_table_validate(ks_pool* pool, uint64_t key, const int32_t* d_table,
                                  uint32_t row_stride, const int32_t* d_ctx_lens, uint32_t rows,
                                  uint32_t tpb, void* stream, uint64_t* n_bad) {
  return guarded([&] {
    if (!pool || pool->device < 0 || !n_bad || tpb == 0)
      return fail(KS_INVALID_ARGUMENT, "bad argument");
    const uint64_t bps = pool->pool->blocks_per_slab(key);
    DeviceGuard g(pool->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int si = 0;
    ks_pool::Slot sl;
    cudaError_t e = pool->acquire(&si, &sl);
    if (e != cudaSuccess) return cuda_fail(e, "staging wait");
    e = cudaMemsetAsync(sl.d, 0, 8, s);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
    e = kvslab::launch_table_validate(d_table, row_stride, d_ctx_lens, rows, tpb,
                                      pool->d_slab_table, pool->pool->slab_count(), key,
                                      kvslab::dev::make_fastdiv(static_cast<uint32_t>(bps)),
                                      reinterpret_cast<unsigned long long*>(sl.d), s);
    if (e != cudaSuccess) return cuda_fail(e, "validate");
    ++g_launches;
    unsigned long long bad = 0;
    e = cudaMemcpyAsync(&bad, sl.d, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "validate readback");
    *n_bad = bad;
    return KS_OK;
  });
}

ks_status ks_kv_append(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_k,
                       const void* d_v, uint32_t n_tokens, const int32_t* d_tok_seq,
                       const int32_t* d_tok_pos, const int32_t* d_block_table, uint32_t bt_stride,
                       const float* d_kv_scales, void* stream) {
  return guarded([&] {
    FmtInfo fi;
    ks_status st = check_kernel_format(pool, fmt, &fi);
    if (st != KS_OK) return st;
    if (layer >= fmt->num_layers) return fail(KS_INVALID_ARGUMENT, "layer out of range");
    if (n_tokens == 0) return KS_OK;
    if (!d_k || !d_v || !d_tok_seq || !d_tok_pos || !d_block_table)
      return fail(KS_INVALID_ARGUMENT, "null device pointer");
    DeviceGuard g(pool->device);
    kvslab::AppendParams p{};
    p.pool = pool->d_base;
    p.geom.slab_size = pool->pool->slab_size();
    p.geom.key = fi.key;
    p.geom.bps = kvslab::dev::make_fastdiv(static_cast<uint32_t>(pool->pool->blocks_per_slab(fi.key)));
    p.layer_off = static_cast<uint64_t>(layer) * fi.layer_bytes;
    p.H = fmt->num_kv_heads;
    p.D = fmt->head_dim;
    p.tpb = fmt->tokens_per_block;
    p.chunk_bytes = static_cast<uint32_t>(fi.chunk);
    p.params_off = static_cast<uint32_t>(2 * p.H * fi.chunk);
    p.fp8_inblock = fmt->kv_dtype == KS_KV_FP8_E4M3 && fmt->quant_param_bytes_per_block > 0;
    p.k = static_cast<const __half*>(d_k);
    p.v = static_cast<const __half*>(d_v);
    p.n_tokens = n_tokens;
    p.tok_seq = d_tok_seq;
    p.tok_pos = d_tok_pos;
    p.block_table = d_block_table;
    p.bt_stride = bt_stride;
    p.kv_scales = d_kv_scales;
    p.ctas_per_sm = pool->tuning.append_per_sm;
    cudaError_t fe = prepare(pool, static_cast<cudaStream_t>(stream));
    if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
    cudaError_t e = kvslab::launch_kv_append(p, static_cast<int>(fmt->kv_dtype),
                                             static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "kv_append launch");
    ++g_launches;
    return KS_OK;
  });
}

ks_status ks_paged_decode_workspace_size(const ks_pool* pool, const ks_kv_format* fmt,
                                         uint32_t batch, size_t* bytes) {
  if (!pool || !fmt || !bytes) return fail(KS_INVALID_ARGUMENT, "null argument");
  const int sms = pool->num_sms > 0 ? pool->num_sms : 148;
  const size_t part = kvslab::decode_partials_bytes(sms, static_cast<int>(fmt->num_q_heads / std::max(1u, fmt->num_kv_heads)));
  (void)batch;  // the partials are sized per SM, not per sequence
  *bytes = part;
  return KS_OK;
}

static ks_status decode_impl(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                             const void* d_k_new, const void* d_v_new, void* d_out, float* d_lse, const int32_t* d_block_table,
                          uint32_t bt_stride, const int32_t* d_ctx_lens, uint32_t batch,
                          float sm_scale, const float* d_kv_scales, void* d_workspace,
                          size_t workspace_bytes, void* stream) {
  return guarded([&] {
    FmtInfo fi;
    ks_status st = check_kernel_format(pool, fmt, &fi);
    if (st != KS_OK) return st;
    if (layer >= fmt->num_layers) return fail(KS_INVALID_ARGUMENT, "layer out of range");
    if (batch == 0) return KS_OK;
    if (!d_q || !d_out || !d_block_table || !d_ctx_lens || !d_workspace)
      return fail(KS_INVALID_ARGUMENT, "null device pointer");
    size_t need = 0;
    ks_paged_decode_workspace_size(pool, fmt, batch, &need);
    if (workspace_bytes < need) return fail(KS_INVALID_ARGUMENT, "workspace too small");
    if (batch > 8192) return fail(KS_NOT_SUPPORTED, "batch > 8192 per launch");
    DeviceGuard g(pool->device);
    kvslab::DecodeParams p{};
    p.pool = pool->d_base;
    p.geom.slab_size = pool->pool->slab_size();
    p.geom.key = fi.key;
    p.geom.bps = kvslab::dev::make_fastdiv(static_cast<uint32_t>(pool->pool->blocks_per_slab(fi.key)));
    p.layer_off = static_cast<uint64_t>(layer) * fi.layer_bytes;
    p.H = fmt->num_kv_heads;
    p.G = fmt->num_q_heads / fmt->num_kv_heads;
    p.q = static_cast<const __half*>(d_q);
    p.out = static_cast<__half*>(d_out);
    p.lse = d_lse;
    p.block_table = d_block_table;
    p.bt_stride = bt_stride;
    p.ctx_lens = d_ctx_lens;
    p.batch = batch;
    const float scale = sm_scale > 0.f ? sm_scale : 1.0f / std::sqrt(static_cast<float>(fmt->head_dim));
    p.sm_scale_log2 = scale * 1.4426950408889634f;
    p.kv_scales = fmt->kv_dtype == KS_KV_FP8_E4M3 ? d_kv_scales : nullptr;
    p.k_new = static_cast<const __half*>(d_k_new);
    p.v_new = static_cast<const __half*>(d_v_new);
    p.params_off = static_cast<uint32_t>(2 * p.H * fi.chunk);
    p.fp8_inblock = fmt->kv_dtype == KS_KV_FP8_E4M3 && fmt->quant_param_bytes_per_block > 0;
    if ((d_k_new == nullptr) != (d_v_new == nullptr))
      return fail(KS_INVALID_ARGUMENT, "k_new and v_new must both be set or both be null");
    p.partials = static_cast<float*>(d_workspace);
    const kvslab::Tuning& tu = pool->tuning;
    p.max_ctas = 0;
    {
      auto it = pool->cta_budget.find(fi.key);
      if (it != pool->cta_budget.end()) p.max_ctas = static_cast<int>(it->second);
    }
    if (tu.decode_max_ctas) p.max_ctas = tu.decode_max_ctas;
    p.hg_max = tu.decode_hg;
    p.smem_budget = tu.decode_smem;
    p.merge_threads = tu.merge_threads;
    p.merge_dc = tu.merge_dc;
    p.pack_mode = tu.decode_pack;
    p.debug = tu.decode_debug;
    p.pdl = tu.pdl;
    p.min_blocks = tu.decode_min_blocks;
    p.trace = tu.decode_trace;  // probe builds only (Tuning::from_env)
    cudaError_t fe = prepare(pool, static_cast<cudaStream_t>(stream));
    if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
    cudaError_t e = kvslab::launch_paged_decode(p, static_cast<int>(fmt->kv_dtype), pool->num_sms,
                                                static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "paged_decode launch");
    g_launches += 2;  // decode + merge
    return KS_OK;
  });
}

ks_status ks_paged_decode(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                          void* d_out, float* d_lse, const int32_t* d_block_table,
                          uint32_t bt_stride, const int32_t* d_ctx_lens, uint32_t batch,
                          float sm_scale, const float* d_kv_scales, void* d_workspace,
                          size_t workspace_bytes, void* stream) {
  return decode_impl(pool, fmt, layer, d_q, nullptr, nullptr, d_out, d_lse, d_block_table,
                     bt_stride, d_ctx_lens, batch, sm_scale, d_kv_scales, d_workspace,
                     workspace_bytes, stream);
}

ks_status ks_paged_decode_append(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer,
                                 const void* d_q, const void* d_k_new, const void* d_v_new,
                                 void* d_out, float* d_lse, const int32_t* d_block_table,
                                 uint32_t bt_stride, const int32_t* d_ctx_lens, uint32_t batch,
                                 float sm_scale, const float* d_kv_scales, void* d_workspace,
                                 size_t workspace_bytes, void* stream) {
  if (!d_k_new || !d_v_new) return fail(KS_INVALID_ARGUMENT, "null k_new/v_new");
  return decode_impl(pool, fmt, layer, d_q, d_k_new, d_v_new, d_out, d_lse, d_block_table,
                     bt_stride, d_ctx_lens, batch, sm_scale, d_kv_scales, d_workspace,
                     workspace_bytes, stream);
}

static int prefill_sms(const ks_pool* pool) {
  if (pool && pool->num_sms > 0) return pool->num_sms;
  int dev = 0, n = 0;  // the size query has no pool: the current device's SMs
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
    return n;
  cudaGetLastError();
  return 148;
}

// Workspace layout: [split-KV partials][expand scratch]
ks_status ks_paged_prefill_workspace_size(const ks_kv_format* fmt, uint32_t batch, uint32_t bt_stride,
                                          uint32_t max_q_len, size_t* bytes) {
  if (!fmt || !bytes) return fail(KS_INVALID_ARGUMENT, "null argument");
  const uint32_t H = fmt->num_kv_heads, G = H ? fmt->num_q_heads / H : 0;
  const uint32_t splits = G ? kvslab::prefill_kv_splits(batch, H, G, max_q_len, prefill_sms(nullptr)) : 1;
  *bytes = (G ? kvslab::prefill_partial_bytes(batch, H, G, max_q_len, splits) : 0) +
           (fmt->kv_dtype == KS_KV_FP16 ? 0 : kvslab::prefill_expand_bytes(H, batch, bt_stride));
  return KS_OK;
}

// Expand-once pays off when each KV tile would otherwise be dequantised by
// several query-tile CTAs of a head (two 128-row tiles per CTA).
static bool prefill_expands(const kvslab::Tuning& tu, uint32_t max_q_len, uint32_t G) {
  if (tu.prefill_expand >= 0) return tu.prefill_expand != 0;
  return static_cast<uint64_t>(max_q_len) * G >= 1024;
}

static ks_status prefill_impl(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                              void* d_out, float* d_lse, const int32_t* d_block_table,
                              uint32_t bt_stride, const int32_t* d_cu_q, const int32_t* d_ctx_lens,
                              uint32_t batch, uint32_t max_q_len, float sm_scale,
                              const float* d_kv_scales, void* d_workspace, size_t workspace_bytes,
                              void* stream) {
  return guarded([&] {
    FmtInfo fi;
    ks_status st = check_kernel_format(pool, fmt, &fi);
    if (st != KS_OK) return st;
    if (layer >= fmt->num_layers) return fail(KS_INVALID_ARGUMENT, "layer out of range");
    const uint32_t G = fmt->num_q_heads / fmt->num_kv_heads;
    if (G == 0 || 16 % G != 0) return fail(KS_NOT_SUPPORTED, "prefill needs a GQA group dividing 16");
    if (batch == 0 || max_q_len == 0) return KS_OK;
    if (!d_q || !d_out || !d_block_table || !d_cu_q || !d_ctx_lens)
      return fail(KS_INVALID_ARGUMENT, "null device pointer");
    if (static_cast<uint64_t>(batch) * fmt->num_kv_heads > 0x7fffffffULL)
      return fail(KS_NOT_SUPPORTED, "batch x kv heads too large");
    DeviceGuard g(pool->device);
    kvslab::PrefillParams p{};
    p.pool = pool->d_base;
    p.geom.slab_size = pool->pool->slab_size();
    p.geom.key = fi.key;
    p.geom.bps = kvslab::dev::make_fastdiv(static_cast<uint32_t>(pool->pool->blocks_per_slab(fi.key)));
    p.layer_off = static_cast<uint64_t>(layer) * fi.layer_bytes;
    p.H = fmt->num_kv_heads;
    p.G = G;
    p.q = static_cast<const __half*>(d_q);
    p.out = static_cast<__half*>(d_out);
    p.lse = d_lse;
    p.block_table = d_block_table;
    p.bt_stride = bt_stride;
    p.cu_q = d_cu_q;
    p.ctx_lens = d_ctx_lens;
    p.batch = batch;
    p.max_q_len = max_q_len;
    const float scale = sm_scale > 0.f ? sm_scale : 1.0f / std::sqrt(static_cast<float>(fmt->head_dim));
    p.sm_scale_log2 = scale * 1.4426950408889634f;
    p.kv_scales = fmt->kv_dtype == KS_KV_FP8_E4M3 ? d_kv_scales : nullptr;
    const kvslab::Tuning& tu = pool->tuning;
    p.nt = tu.prefill_nt;
    p.use_tc = tu.prefill_tc;
    p.debug = tu.prefill_debug;
    cudaError_t fe = prepare(pool, static_cast<cudaStream_t>(stream));
    if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
    // Workspace use (kvslab.h): split-KV partials when the query tiles alone
    // would leave SMs idle (tcgen05 path) and, for quantised formats with long
    // chunks, the expand-once scratch.  A workspace too small for both drops
    // the split first, then takes the expand in sequence groups.
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    const bool expand = ws != nullptr && fmt->kv_dtype != KS_KV_FP16 && p.use_tc &&
                        prefill_expands(tu, max_q_len, G);
    const size_t full_expand = expand ? kvslab::prefill_expand_bytes(p.H, batch, bt_stride) : 0;
    if (ws && p.use_tc && tu.prefill_split != 0) {
      const uint32_t splits = kvslab::prefill_kv_splits(batch, p.H, G, max_q_len, prefill_sms(pool));
      const size_t pb = kvslab::prefill_partial_bytes(batch, p.H, G, max_q_len, splits);
      if (splits > 1 && workspace_bytes >= pb + full_expand) {
        p.kv_splits = splits;
        p.part = reinterpret_cast<float*>(ws);
        ws += pb;
        workspace_bytes -= pb;
      }
    }
    const size_t per_seq = kvslab::prefill_expand_bytes(p.H, 1, bt_stride);
    if (expand && per_seq > 0 && workspace_bytes >= per_seq) {
      // a workspace smaller than the whole batch's takes the sequences in groups
      const uint32_t group = static_cast<uint32_t>(std::min<size_t>(batch, workspace_bytes / per_seq));
      for (uint32_t g0 = 0; g0 < batch; g0 += group) {
        kvslab::PrefillParams q = p;
        q.batch = std::min(group, batch - g0);
        q.block_table = p.block_table + static_cast<size_t>(g0) * bt_stride;
        q.cu_q = p.cu_q + g0;  // row offsets stay absolute
        q.ctx_lens = p.ctx_lens + g0;
        cudaError_t e = kvslab::launch_paged_prefill_expand(q, static_cast<int>(fmt->kv_dtype), ws,
                                                            static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_fail(e, "paged_prefill (expand) launch");
        g_launches += 2;
      }
      return KS_OK;
    }
    cudaError_t e = kvslab::launch_paged_prefill(p, static_cast<int>(fmt->kv_dtype),
                                                 static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "paged_prefill launch");
    ++g_launches;
    return KS_OK;
  });
}

ks_status ks_paged_prefill(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                           void* d_out, float* d_lse, const int32_t* d_block_table,
                           uint32_t bt_stride, const int32_t* d_cu_q, const int32_t* d_ctx_lens,
                           uint32_t batch, uint32_t max_q_len, float sm_scale,
                           const float* d_kv_scales, void* stream) {
  return prefill_impl(pool, fmt, layer, d_q, d_out, d_lse, d_block_table, bt_stride, d_cu_q, d_ctx_lens,
                      batch, max_q_len, sm_scale, d_kv_scales, nullptr, 0, stream);
}

ks_status ks_paged_prefill_ws(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                              void* d_out, float* d_lse, const int32_t* d_block_table,
                              uint32_t bt_stride, const int32_t* d_cu_q, const int32_t* d_ctx_lens,
                              uint32_t batch, uint32_t max_q_len, float sm_scale,
                              const float* d_kv_scales, void* d_workspace, size_t workspace_bytes,
                              void* stream) {
  return prefill_impl(pool, fmt, layer, d_q, d_out, d_lse, d_block_table, bt_stride, d_cu_q, d_ctx_lens,
                      batch, max_q_len, sm_scale, d_kv_scales, d_workspace, workspace_bytes, stream);
}

ks_status ks_probe_set_decode_trace(ks_pool* pool, void* d_trace) {
  if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
  if (!kvslab::kProbes) return fail(KS_NOT_SUPPORTED, "timestamp probes need a -DKVSLAB_PROBES build");
  pool->tuning.decode_trace = static_cast<unsigned long long*>(d_trace);
  return KS_OK;
}

ks_status ks_set_decode_sm_share(ks_pool* pool, uint64_t key, uint32_t max_ctas) {
  return guarded([&] {
    if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
    pool->pool->blocks_per_slab(key);  // InvalidKeyError when unregistered
    if (max_ctas == 0) pool->cta_budget.erase(key);
    else pool->cta_budget[key] = max_ctas;
    return KS_OK;
  });
}

ks_status ks_compact_plan(ks_pool* pool, uint64_t key, uint32_t max_moves, ks_block_move* moves,
                          uint32_t* n_moves, uint32_t* slabs_freed) {
  return guarded([&] {
    if (!pool || !n_moves || (!moves && max_moves)) return fail(KS_INVALID_ARGUMENT, "null argument");
    uint32_t freed = 0;
    auto mv = pool->pool->plan_compaction(key, max_moves, &freed);
    for (size_t i = 0; i < mv.size(); ++i) {
      moves[i].src_global_block_id = mv[i].src.global_block_id;
      moves[i].dst_global_block_id = mv[i].dst.global_block_id;
    }
    *n_moves = static_cast<uint32_t>(mv.size());
    if (slabs_freed) *slabs_freed = freed;
    return KS_OK;
  });
}

ks_status ks_compact_apply(ks_pool* pool, uint64_t key, const ks_block_move* moves, uint32_t n,
                           void* stream) {
  return guarded([&] {
    if (!pool || pool->device < 0) return fail(KS_INVALID_ARGUMENT, "pool has no device tensor");
    if (n == 0) return KS_OK;
    if (!moves) return fail(KS_INVALID_ARGUMENT, "null moves");
    if (key % 16 != 0 || pool->pool->slab_size() % 16 != 0)
      return fail(KS_NOT_SUPPORTED, "key and slab size must be multiples of 16 bytes");
    const uint64_t bps = pool->pool->blocks_per_slab(key);
    DeviceGuard g(pool->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t fe = prepare(pool, s);
    if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
    uint32_t i = 0;
    while (i < n) {
      const uint32_t m = static_cast<uint32_t>(std::min<size_t>(n - i, ks_pool::kSlotWords / 2));
      int si = 0;
      ks_pool::Slot sl;
      cudaError_t e = pool->acquire(&si, &sl);
      if (e != cudaSuccess) return cuda_fail(e, "staging wait");
      for (uint32_t j = 0; j < m; ++j) {
        sl.h[j] = static_cast<uint32_t>(moves[i + j].src_global_block_id);
        sl.h[m + j] = static_cast<uint32_t>(moves[i + j].dst_global_block_id);
      }
      e = pool->upload(sl, 2 * static_cast<size_t>(m), s);
      if (e != cudaSuccess) return cuda_fail(e, "staging upload");
      kvslab::CompactParams p{};
      p.pool = pool->d_base;
      p.geom.slab_size = pool->pool->slab_size();
      p.geom.key = key;
      p.geom.bps = kvslab::dev::make_fastdiv(static_cast<uint32_t>(bps));
      p.src_gid = sl.d;
      p.dst_gid = sl.d + m;
      p.n_moves = m;
      e = kvslab::launch_compact(p, pool->num_sms, s);
      if (e != cudaSuccess) return cuda_fail(e, "compact launch");
      e = pool->release(si, s);
      if (e != cudaSuccess) return cuda_fail(e, "staging release");
      ++g_launches;
      i += m;
    }
    return KS_OK;
  });
}

// Rewrites table entries through the sorted move list, in chunks of one
// staging slot.  Sources and destinations of one plan are disjoint (a slab
// that received blocks is never evacuated, an evacuated slab never receives),
// so chunked passes remap every entry at most once.
static ks_status remap_table(ks_pool* pool, int32_t* d_table, uint64_t n_entries,
                             const std::vector<std::pair<uint32_t, uint32_t>>& v, cudaStream_t s) {
  const size_t per = ks_pool::kSlotWords / 2;
  for (size_t i0 = 0; i0 < v.size(); i0 += per) {
    const uint32_t n = static_cast<uint32_t>(std::min(per, v.size() - i0));
    int si = 0;
    ks_pool::Slot sl;
    cudaError_t e = pool->acquire(&si, &sl);
    if (e != cudaSuccess) return cuda_fail(e, "staging wait");
    for (uint32_t i = 0; i < n; ++i) {
      sl.h[i] = v[i0 + i].first;
      sl.h[n + i] = v[i0 + i].second;
    }
    e = pool->upload(sl, 2 * static_cast<size_t>(n), s);
    if (e != cudaSuccess) return cuda_fail(e, "staging upload");
    e = kvslab::launch_table_remap(d_table, n_entries, sl.d, sl.d + n, n, s);
    if (e != cudaSuccess) return cuda_fail(e, "remap launch");
    e = pool->release(si, s);
    if (e != cudaSuccess) return cuda_fail(e, "staging release");
    ++g_launches;
  }
  return KS_OK;
}

ks_status ks_block_table_remap(ks_pool* pool, int32_t* d_table, uint64_t n_entries,
                               const ks_block_move* moves, uint32_t n, void* stream) {
  return guarded([&] {
    if (!pool || pool->device < 0) return fail(KS_INVALID_ARGUMENT, "pool has no device tensor");
    if (n == 0 || n_entries == 0) return KS_OK;
    if (!d_table || !moves) return fail(KS_INVALID_ARGUMENT, "null argument");
    std::vector<std::pair<uint32_t, uint32_t>> v(n);
    for (uint32_t i = 0; i < n; ++i)
      v[i] = {static_cast<uint32_t>(moves[i].src_global_block_id),
              static_cast<uint32_t>(moves[i].dst_global_block_id)};
    std::sort(v.begin(), v.end());
    DeviceGuard g(pool->device);
    return remap_table(pool, d_table, n_entries, v, static_cast<cudaStream_t>(stream));
  });
}

// ------------------------------------------------------------- engine tables
static ks_status seq_table_sync_impl(ks_seq_table* t, cudaStream_t s) {
  ks_pool* pool = t->owner;
  t->t->dedupe_pending();
  const auto& pend = t->t->pending();
  if (pend.empty()) return KS_OK;
  if (!t->d_table || pool->device < 0) {  // host-only table: nothing to mirror
    t->t->clear_pending();
    return KS_OK;
  }
  DeviceGuard g(pool->device);
  cudaError_t fe = prepare(pool, s);
  if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
  size_t i = 0;
  while (i < pend.size()) {
    const size_t m = std::min(pend.size() - i, ks_pool::kSlotWords / 3);
    int si = 0;
    ks_pool::Slot sl;
    cudaError_t e = pool->acquire(&si, &sl);
    if (e != cudaSuccess) return cuda_fail(e, "staging wait");
    std::memcpy(sl.h, pend.data() + i, m * sizeof(SeqTable::Delta));
    e = pool->upload(sl, 3 * m, s);
    if (e != cudaSuccess) return cuda_fail(e, "staging upload");
    e = kvslab::launch_table_scatter(t->d_table, t->row_stride, reinterpret_cast<const int32_t*>(sl.d),
                                     static_cast<uint32_t>(m), s);
    if (e != cudaSuccess) return cuda_fail(e, "table scatter");
    e = pool->release(si, s);
    if (e != cudaSuccess) return cuda_fail(e, "staging release");
    ++g_launches;
    i += m;
  }
  t->t->clear_pending();
  return KS_OK;
}

#define KS_TABLE_GUARD(t)                                                     \
  if (!(t)) return fail(KS_INVALID_ARGUMENT, "null table");                   \
  if (!(t)->owner) return fail(KS_INVALID_ARGUMENT, "table's pool was destroyed")

ks_status ks_seq_table_create(ks_pool* pool, const ks_seq_table_config* cfg, ks_seq_table** out) {
  return guarded([&] {
    if (!pool || !cfg || !out) return fail(KS_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (cfg->d_table && cfg->row_stride < cfg->max_blocks_per_seq)
      return fail(KS_INVALID_ARGUMENT, "row_stride < max_blocks_per_seq");
    auto t = std::make_unique<ks_seq_table>();
    t->t = std::make_unique<SeqTable>(pool->pool.get(), cfg->key, cfg->max_seqs,
                                      cfg->max_blocks_per_seq, cfg->tokens_per_block,
                                      cfg->useful_token_bytes, cfg->block_metadata_bytes);
    t->owner = pool;
    t->d_table = cfg->d_table;
    t->row_stride = cfg->d_table ? cfg->row_stride : cfg->max_blocks_per_seq;
    pool->tables.push_back(t.get());
    *out = t.release();
    return KS_OK;
  });
}

ks_status ks_seq_table_destroy(ks_seq_table* t) {
  if (!t) return KS_OK;
  if (t->owner) {
    auto& v = t->owner->tables;
    v.erase(std::remove(v.begin(), v.end(), t), v.end());
  }
  delete t;
  return KS_OK;
}

ks_status ks_seq_table_admit(ks_seq_table* t, uint32_t seq, uint64_t prompt_tokens, int32_t* ok) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!ok) return fail(KS_INVALID_ARGUMENT, "null argument");
    *ok = t->t->admit(seq, prompt_tokens) ? 1 : 0;
    return KS_OK;
  });
}

ks_status ks_seq_table_ensure(ks_seq_table* t, uint32_t seq, uint64_t tokens, int32_t* ok) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!ok) return fail(KS_INVALID_ARGUMENT, "null argument");
    *ok = t->t->ensure_capacity(seq, tokens) ? 1 : 0;
    return KS_OK;
  });
}

ks_status ks_seq_table_step(ks_seq_table* t, const uint32_t* seqs, uint32_t n, uint8_t* stalled,
                            uint32_t* n_active) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if ((!seqs && n) || !n_active) return fail(KS_INVALID_ARGUMENT, "null argument");
    *n_active = t->t->step(seqs, n, stalled);
    return KS_OK;
  });
}

ks_status ks_seq_table_release(ks_seq_table* t, uint32_t seq) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    t->t->release(seq);
    return KS_OK;
  });
}

ks_status ks_seq_table_move_row(ks_seq_table* t, uint32_t src, uint32_t dst) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    t->t->move_row(src, dst);
    return KS_OK;
  });
}

ks_status ks_seq_table_cached(const ks_seq_table* t, uint32_t seq, uint64_t* tokens) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!tokens) return fail(KS_INVALID_ARGUMENT, "null argument");
    *tokens = t->t->cached(seq);
    return KS_OK;
  });
}

ks_status ks_seq_table_set_cached(ks_seq_table* t, uint32_t seq, uint64_t tokens) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    t->t->set_cached(seq, tokens);
    return KS_OK;
  });
}

ks_status ks_seq_table_ctx_lens(const ks_seq_table* t, int32_t* out, uint32_t n, int32_t plus) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!out && n) return fail(KS_INVALID_ARGUMENT, "null argument");
    if (n > t->t->max_seqs()) return fail(KS_INVALID_ARGUMENT, "more rows than the table has");
    for (uint32_t s = 0; s < n; ++s)
      out[s] = t->t->blocks(s).empty() ? 0 : static_cast<int32_t>(t->t->cached(s)) + plus;
    return KS_OK;
  });
}

ks_status ks_seq_table_blocks(const ks_seq_table* t, uint32_t seq, ks_block_handle* out,
                              uint32_t capacity, uint32_t* n) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!n || (!out && capacity)) return fail(KS_INVALID_ARGUMENT, "null argument");
    const auto& hs = t->t->blocks(seq);
    *n = static_cast<uint32_t>(hs.size());
    const size_t m = std::min<size_t>(hs.size(), capacity);
    for (size_t i = 0; i < m; ++i) out[i] = to_c(hs[i]);
    return KS_OK;
  });
}

ks_status ks_seq_table_get_stats(const ks_seq_table* t, ks_seq_table_stats* out) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!out) return fail(KS_INVALID_ARGUMENT, "null argument");
    const auto st = t->t->stats();
    out->live_seqs = st.live_seqs;
    out->held_blocks = st.held_blocks;
    out->cached_tokens = st.cached_tokens;
    out->internal_frag_bytes = st.internal_frag_bytes;
    return KS_OK;
  });
}

ks_status ks_seq_table_pending(const ks_seq_table* t, uint32_t* n) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    if (!n) return fail(KS_INVALID_ARGUMENT, "null argument");
    *n = static_cast<uint32_t>(t->t->pending().size());
    return KS_OK;
  });
}

ks_status ks_seq_table_sync(ks_seq_table* t, void* stream) {
  return guarded([&] {
    KS_TABLE_GUARD(t);
    return seq_table_sync_impl(t, static_cast<cudaStream_t>(stream));
  });
}

// K3 over every registered table of the key, all-or-nothing on the host.
ks_status ks_compact(ks_pool* pool, uint64_t key, uint32_t max_moves, void* stream,
                     uint32_t* n_moves, uint32_t* slabs_freed) {
  return guarded([&] {
    if (!pool) return fail(KS_INVALID_ARGUMENT, "null pool");
    if (pool->device < 0) return fail(KS_INVALID_ARGUMENT, "pool has no device tensor");
    if (key % 16 != 0 || pool->pool->slab_size() % 16 != 0)
      return fail(KS_NOT_SUPPORTED, "key and slab size must be multiples of 16 bytes");
    const uint64_t bps = pool->pool->blocks_per_slab(key);  // InvalidKeyError first
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    {  // before the snapshot: the rollback must not resurrect drained scrubs
      DeviceGuard g(pool->device);
      cudaError_t fe = prepare(pool, s);
      if (fe != cudaSuccess) return cuda_fail(fe, "launch prologue (fence / slab scrub)");
    }
    std::vector<ks_seq_table*> mine;
    for (ks_seq_table* t : pool->tables)
      if (t->t->key() == key) mine.push_back(t);
    // snapshot for rollback: the host table and the affected engine tables
    SlabPool before(*pool->pool);
    std::vector<SeqTable> rows_before;
    rows_before.reserve(mine.size());
    for (ks_seq_table* t : mine) rows_before.push_back(*t->t);
    uint32_t freed = 0;
    const auto mv = pool->pool->plan_compaction(key, max_moves, &freed);
    auto rollback = [&](ks_status st) {
      *pool->pool = before;
      for (size_t i = 0; i < mine.size(); ++i) *mine[i]->t = rows_before[i];
      return st;
    };
    if (!mv.empty()) {
      DeviceGuard g(pool->device);
      // bytes
      const size_t per = ks_pool::kSlotWords / 2;
      for (size_t i0 = 0; i0 < mv.size(); i0 += per) {
        const uint32_t m = static_cast<uint32_t>(std::min(per, mv.size() - i0));
        int si = 0;
        ks_pool::Slot sl;
        cudaError_t e = pool->acquire(&si, &sl);
        if (e != cudaSuccess) return rollback(cuda_fail(e, "staging wait"));
        for (uint32_t j = 0; j < m; ++j) {
          sl.h[j] = static_cast<uint32_t>(mv[i0 + j].src.global_block_id);
          sl.h[m + j] = static_cast<uint32_t>(mv[i0 + j].dst.global_block_id);
        }
        e = pool->upload(sl, 2 * static_cast<size_t>(m), s);
        if (e != cudaSuccess) return rollback(cuda_fail(e, "staging upload"));
        kvslab::CompactParams p{};
        p.pool = pool->d_base;
        p.geom.slab_size = pool->pool->slab_size();
        p.geom.key = key;
        p.geom.bps = kvslab::dev::make_fastdiv(static_cast<uint32_t>(bps));
        p.src_gid = sl.d;
        p.dst_gid = sl.d + m;
        p.n_moves = m;
        e = kvslab::launch_compact(p, pool->num_sms, s);
        if (e != cudaSuccess) return rollback(cuda_fail(e, "compact launch"));
        e = pool->release(si, s);
        if (e != cudaSuccess) return rollback(cuda_fail(e, "staging release"));
        ++g_launches;
      }
      // handles + device entries of every table of the key
      std::unordered_map<uint64_t, BlockHandle> moved;
      moved.reserve(mv.size() * 2);
      for (const auto& m : mv) moved.emplace(m.src.global_block_id, m.dst);
      for (ks_seq_table* t : mine) {
        t->t->remap(moved);
        ks_status st = seq_table_sync_impl(t, s);
        if (st != KS_OK) return rollback(st);
      }
      cudaError_t e = cudaEventRecord(pool->fence, s);
      if (e != cudaSuccess) return rollback(cuda_fail(e, "fence record"));
      pool->fence_stream = s;
      pool->fence_pending = true;
    }
    if (n_moves) *n_moves = static_cast<uint32_t>(mv.size());
    if (slabs_freed) *slabs_freed = freed;
    return KS_OK;
  });
}

}  // extern "C"
