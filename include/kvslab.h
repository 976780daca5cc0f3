/* kvslab.h -- C ABI of the B200-native KV-slab data path (libkvslab.so).
 *
 * Drop-in boundary for the reference's slab allocator.  The reference
 * (FineServe "slabsim", /root/reference/proj) exposes this path only as the
 * C++ class slabsim::SlabPool plus two geometry functions; it has no C ABI,
 * FFI or plugin registry.  Every entry point below
 * cites the reference interface it replaces; the C++ wrapper in
 * include/kvslab/slab_pool.hpp re-exposes them with the reference's class
 * and exception names.  INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *   - every function returns ks_status; exceptions never cross the ABI.
 *     The reference's exception classes map 1:1 (common.hpp:36-59):
 *       InvalidConfigError -> KS_INVALID_CONFIG, InvalidKeyError -> KS_INVALID_KEY,
 *       PoolExhaustedError -> KS_EXHAUSTED,      InvalidFreeError -> KS_INVALID_FREE,
 *       InvalidProfileError -> KS_INVALID_PROFILE.
 *     ks_last_error() returns the thread-local message of the last failure.
 *   - plain pointers and sizes only; `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).  Device pointers are marked d_.
 *   - threading: one writer per pool; device work is
 *     asynchronous and ordered on the caller's stream.
 */
#ifndef KVSLAB_H_
#define KVSLAB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_ABI_VERSION 1

typedef enum ks_status {
  KS_OK = 0,
  KS_INVALID_CONFIG = 1,  /* slabsim::InvalidConfigError */
  KS_INVALID_KEY = 2,     /* slabsim::InvalidKeyError */
  KS_EXHAUSTED = 3,       /* slabsim::PoolExhaustedError */
  KS_INVALID_FREE = 4,    /* slabsim::InvalidFreeError */
  KS_INVALID_PROFILE = 5, /* slabsim::InvalidProfileError */
  KS_INVALID_ARGUMENT = 6,
  KS_CUDA_ERROR = 7,
  KS_NOT_SUPPORTED = 8,
  KS_INTERNAL = 9
} ks_status;

typedef enum ks_slab_state_code { KS_SLAB_FREE = 0, KS_SLAB_PARTIAL = 1, KS_SLAB_FULL = 2 } ks_slab_state_code;

typedef enum ks_kv_dtype {
  KS_KV_FP16 = 0,     /* 16-bit, copied verbatim */
  KS_KV_FP8_E4M3 = 1, /* OCP e4m3, static per-(K|V, head) fp32 scale */
  KS_KV_INT8 = 2,     /* symmetric, fp16 scale per (K|V, head, token) */
  KS_KV_INT4 = 3      /* asymmetric QoQ-style, fp16 (scale, zero) per (K|V, head, token) */
} ks_kv_dtype;

typedef struct ks_pool ks_pool;

/* slabsim::SlabPoolConfig (slab_pool.hpp:41-46) */
typedef struct ks_pool_config {
  uint64_t capacity_bytes;
  uint64_t slab_size_bytes;
  const uint64_t* block_size_keys;
  uint32_t num_keys;
  int32_t require_lcm_alignment; /* nonzero = reference default (true) */
} ks_pool_config;

/* slabsim::BlockHandle (slab_pool.hpp:53-60) */
typedef struct ks_block_handle {
  uint32_t slab_id;
  uint32_t local_block_id;
  uint64_t global_block_id;
  uint64_t key;
} ks_block_handle;

/* slabsim::FragmentationStats (slab_pool.hpp:67-78) */
typedef struct ks_frag_stats {
  uint64_t allocated_bytes;
  uint64_t free_block_bytes;
  uint64_t slab_residue_bytes;
  uint64_t free_slab_bytes;
} ks_frag_stats;

/* slabsim::OpLogRecord (slab_pool.hpp:80-89); op is "alloc" or "free" */
typedef struct ks_op_record {
  uint64_t seq;
  double time;
  const char* op;
  uint64_t key;
  uint32_t slab_id;
  uint32_t local_block_id;
  uint64_t global_block_id;
} ks_op_record;
typedef void (*ks_op_log_fn)(const ks_op_record* rec, void* user);
typedef double (*ks_clock_fn)(void* user);

typedef struct ks_pool_info {
  uint32_t slab_count;           /* SlabPool::slab_count            hpp:125 */
  uint32_t num_keys;             /* registered (sorted, deduped) keys        */
  uint64_t slab_size_bytes;      /* SlabPool::slab_size             hpp:126 */
  uint64_t tail_remainder_bytes; /* SlabPool::tail_remainder_bytes  hpp:127 */
  uint64_t usable_capacity_bytes;/* SlabPool::usable_capacity_bytes hpp:128 */
  uint64_t allocated_blocks;     /* SlabPool::allocated_block_count hpp:137 */
  int32_t device;                /* -1: host-only pool (no KV tensor) */
  int32_t require_lcm_alignment;
} ks_pool_info;

/* ------------------------------------------------------------------ */
/* Library                                                            */
/* ------------------------------------------------------------------ */
uint32_t ks_abi_version(void);
const char* ks_last_error(void);
const char* ks_status_name(ks_status s);

/* ------------------------------------------------------------------ */
/* Geometry -- precision.hpp:104-108 / precision.cpp:76-99             */
/* ------------------------------------------------------------------ */
typedef struct ks_model_geometry {
  uint32_t num_kv_heads;
  uint32_t head_dim;
  uint32_t num_layers;
  uint32_t tp_degree;
  uint64_t tokens_per_block;
  uint64_t quant_param_bytes_per_block;
  int32_t kv_bits;
} ks_model_geometry;
/* token_size(profile): (kv_heads/tp)*head_dim*2*kv_bits/8, computed in bits */
ks_status ks_token_size(const ks_model_geometry* g, uint64_t* out);
/* kv_block_size(profile) = num_layers*(tpb*token_size + quant params) = slab key */
ks_status ks_kv_block_size(const ks_model_geometry* g, uint64_t* out);

/* ------------------------------------------------------------------ */
/* Slab pool -- slabsim::SlabPool (slab_pool.hpp:101-202)              */
/* ------------------------------------------------------------------ */
/* SlabPool(const SlabPoolConfig&) (slab_pool.cpp:51-98).  device >= 0 also
 * reserves the single KV tensor (usable capacity bytes, zero-filled once) and
 * the device slab table on that GPU -- the only device allocation the pool
 * ever makes.  device < 0 builds a host-only pool. */
ks_status ks_pool_create(const ks_pool_config* cfg, int device, ks_pool** out);
ks_status ks_pool_destroy(ks_pool* pool);
ks_status ks_pool_get_info(const ks_pool* pool, ks_pool_info* out);
/* Device bytes cleared so far because a slab was re-formatted to another key.
 * A block's slots past a sequence's context are read and masked (P = 0), so
 * they must not hold NaN patterns; fresh memory is zero-filled at creation,
 * and a slab whose previous key's bytes (e.g. INT4 nibbles read as FP8) may
 * form such patterns is cleared (one memset) by the next stream-taking call
 * on the pool -- table upload, append, decode, prefill, compaction -- on that
 * call's stream, before its own work.  Graph captures never include it:
 * upload the new blocks' table entries eagerly before replaying a graph. */
ks_status ks_pool_scrubbed_bytes(const ks_pool* pool, uint64_t* bytes);
/* sorted, deduplicated keys (config().block_size_keys, slab_pool.cpp:58-61) */
ks_status ks_pool_keys(const ks_pool* pool, uint64_t* keys_out, uint32_t capacity);

/* alloc_block (slab_pool.cpp:232-235): KS_EXHAUSTED when no room */
ks_status ks_alloc_block(ks_pool* pool, uint64_t key, ks_block_handle* out);
/* try_alloc_block (slab_pool.cpp:193-226): *ok = 0 and KS_OK when no room */
ks_status ks_try_alloc_block(ks_pool* pool, uint64_t key, ks_block_handle* out, int32_t* ok);
/* batched try-alloc of n blocks of one key; *n_done receives how many
 * succeeded (the first *n_done handles are valid) */
ks_status ks_alloc_blocks(ks_pool* pool, uint64_t key, uint32_t n, ks_block_handle* out,
                          uint32_t* n_done);
/* free_block (slab_pool.cpp:237-272) */
ks_status ks_free_block(ks_pool* pool, const ks_block_handle* handle);
ks_status ks_free_blocks(ks_pool* pool, const ks_block_handle* handles, uint32_t n);

ks_status ks_blocks_per_slab(const ks_pool* pool, uint64_t key, uint64_t* out);       /* cpp:115-122 */
ks_status ks_snapshot_stats(const ks_pool* pool, ks_frag_stats* out);                 /* hpp:122 */
ks_status ks_free_blocks_for_key(const ks_pool* pool, uint64_t key, uint64_t* out);   /* cpp:124-133 */
/* key == 0: all keys (hpp:137), else per key (cpp:135-141) */
ks_status ks_allocated_block_count(const ks_pool* pool, uint64_t key, uint64_t* out);
ks_status ks_slab_state(const ks_pool* pool, uint32_t slab_id, int32_t* state, uint64_t* key); /* hpp:130-132 */
/* check_integrity (cpp:298-379); message via ks_last_error when *ok == 0 */
ks_status ks_check_integrity(const ks_pool* pool, int32_t* ok);
/* operator== (cpp:288-296) */
ks_status ks_pool_equal(const ks_pool* a, const ks_pool* b, int32_t* equal);
/* deep copy of the host table (no device tensor); for state snapshots */
ks_status ks_pool_clone_host(const ks_pool* pool, ks_pool** out);
ks_status ks_set_op_log(ks_pool* pool, ks_op_log_fn fn, void* user); /* hpp:162-164 */
ks_status ks_set_clock(ks_pool* pool, ks_clock_fn fn, void* user);   /* hpp:165 */
ks_status ks_debug_flip_occupancy_bit(ks_pool* pool, uint32_t slab_id, uint32_t local_block_id); /* hpp:167-170 */

/* static id arithmetic (slab_pool.hpp:140-151) */
uint64_t ks_global_block_id(uint32_t slab_id, uint32_t local_block_id, uint64_t blocks_per_slab);
void ks_split_global_block_id(uint64_t global_id, uint64_t blocks_per_slab, uint32_t* slab_id,
                              uint32_t* local_block_id);
/* byte offset of a block inside the KV tensor: slab*slab_size + local*key.
 * Equals gid*key only under LCM alignment (hard part 1). */
ks_status ks_block_byte_offset(const ks_pool* pool, uint64_t key, uint64_t global_block_id,
                               uint64_t* out);

/* ------------------------------------------------------------------ */
/* Device data path (new: no reference counterpart)    */
/* ------------------------------------------------------------------ */
/* Per-model KV format.  head_dim must be 128 and tokens_per_block 16 for the
 * CUDA kernels.  quant_param_bytes_per_block (per layer) must be the format's
 * natural size (ks_natural_qparams) -- or 0 for FP8, meaning the per-head
 * scales are passed at call time only. */
typedef struct ks_kv_format {
  uint32_t kv_dtype; /* ks_kv_dtype */
  uint32_t num_kv_heads; /* per shard */
  uint32_t num_q_heads;  /* per shard, multiple of num_kv_heads */
  uint32_t head_dim;
  uint32_t num_layers;
  uint32_t tokens_per_block;
  uint64_t quant_param_bytes_per_block;
} ks_kv_format;
ks_status ks_natural_qparams(const ks_kv_format* fmt, uint64_t* out);
/* slab key of the format == kv_block_size of the equivalent profile */
ks_status ks_format_key(const ks_kv_format* fmt, uint64_t* out);
ks_status ks_validate_format(const ks_pool* pool, const ks_kv_format* fmt);

/* The single pre-allocated KV tensor. */
ks_status ks_device_base(const ks_pool* pool, void** d_base, uint64_t* bytes);
/* Device slab table: slab_count entries of {uint64 key; uint32 blocks_total;
 * uint32 state} mirroring the host table.  sync uploads the slabs changed
 * since the last sync (delta) on `stream`. */
ks_status ks_slab_table_device(const ks_pool* pool, const void** d_table);
ks_status ks_slab_table_sync(ks_pool* pool, void* stream);

/* Block tables are engine-owned int32 device arrays [rows][row_stride] of
 * global block ids (the engine's logical table, simulator.cpp:36).
 * Delta upload: d_table[rows[i]*row_stride + cols[i]] = vals[i] (host arrays),
 * staged through the pool's pinned buffer. */
ks_status ks_block_table_update(ks_pool* pool, int32_t* d_table, uint32_t row_stride,
                                const int32_t* rows, const int32_t* cols, const int32_t* vals,
                                uint32_t n, void* stream);
/* Debug/validation: checks every referenced entry of a block table against the
 * device slab table (slab formatted to `key`, local < blocks_total).
 * *n_bad receives the number of bad entries (synchronises the stream). */
ks_status ks_block_table_validate(ks_pool* pool, uint64_t key, const int32_t* d_table,
                                  uint32_t row_stride, const int32_t* d_ctx_lens, uint32_t rows,
                                  uint32_t tokens_per_block, void* stream, uint64_t* n_bad);

/* K1 -- KV append with on-the-fly quantisation (replaces the cost stand-in
 * of simulator.cpp:602-604 together with K2).  d_k, d_v: fp16 [n_tokens][Hkv][d].
 * Token i belongs to sequence d_tok_seq[i] at position d_tok_pos[i]; its
 * block is d_block_table[seq*bt_stride + pos/tpb] (allocated by the caller
 * via ks_alloc_block on the growth rule of simulator.cpp:561-578).
 * d_kv_scales: fp32 [2][Hkv] FP8 scales (NULL = 1.0); ignored otherwise. */
ks_status ks_kv_append(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_k,
                       const void* d_v, uint32_t n_tokens, const int32_t* d_tok_seq,
                       const int32_t* d_tok_pos, const int32_t* d_block_table,
                       uint32_t bt_stride, const float* d_kv_scales, void* stream);

/* K2 -- slab-indexed paged decode attention.
 * d_q, d_out: fp16 [batch][Hq][d]; d_lse: fp32 [batch][Hq] natural-log
 * log-sum-exp (nullable); d_ctx_lens: int32 [batch]; sm_scale <= 0 means
 * 1/sqrt(d).  The workspace (>= ks_paged_decode_workspace_size bytes) holds
 * the fp32 partials of sequence-heads split across CTAs; it needs no
 * initialisation, but launches that may run concurrently (different streams)
 * need distinct workspaces.
 * Programmatic dependent launch: each K2 grid lets the next kernel on its
 * stream start early, and issues the bulk copies of its first KV blocks
 * before waiting for its predecessor.  Back-to-back launches on the same
 * stream must therefore not read a block the previous launch writes -- i.e.
 * two ks_paged_decode_append calls in a row must target different layers (a
 * decode step appends layer by layer, so this holds for one step per layer;
 * with a 1-layer format put any other kernel between two steps). */
ks_status ks_paged_decode_workspace_size(const ks_pool* pool, const ks_kv_format* fmt,
                                         uint32_t batch, size_t* bytes);
ks_status ks_paged_decode(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                          void* d_out, float* d_lse, const int32_t* d_block_table,
                          uint32_t bt_stride, const int32_t* d_ctx_lens, uint32_t batch,
                          float sm_scale, const float* d_kv_scales, void* d_workspace,
                          size_t workspace_bytes, void* stream);

/* K1+K2 fused, the decode-step form: first appends the new token of every
 * sequence (d_k_new, d_v_new: fp16 [batch][Hkv][d], the token at position
 * d_ctx_lens[s]-1, whose block must already be in the table), then attends
 * over all d_ctx_lens[s] tokens.  The warp that owns a sequence-head's last
 * block writes the token before its bulk copy reads the block, so there is no
 * separate K1 launch and no inter-kernel dependency.  Bytes written are
 * identical to ks_kv_append. */
ks_status ks_paged_decode_append(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer,
                                 const void* d_q, const void* d_k_new, const void* d_v_new,
                                 void* d_out, float* d_lse, const int32_t* d_block_table,
                                 uint32_t bt_stride, const int32_t* d_ctx_lens, uint32_t batch,
                                 float sm_scale, const float* d_kv_scales, void* d_workspace,
                                 size_t workspace_bytes, void* stream);

/* K4 -- chunked-prefill attention over slab blocks (the
 * prefill block claim is simulator.cpp:500-526).  The chunk's K/V must
 * already be in the blocks (ks_kv_append).  d_q, d_out: fp16
 * [T_total][Hq][d], the rows of sequence s being d_cu_q[s]..d_cu_q[s+1]-1
 * (int32 [batch+1], device), at positions d_ctx_lens[s]-n_s..d_ctx_lens[s]-1
 * (so d_ctx_lens[s] >= n_s); each query attends causally to keys 0..its
 * position.  max_q_len >= every n_s (sizes the grid).  d_lse: fp32
 * [T_total][Hq] natural-log LSE (nullable).  GQA group must divide 16.
 * Runs on the tcgen05 tensor cores (TMEM accumulators) for every KV format;
 * no workspace; no host synchronisation. */
ks_status ks_paged_prefill(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                           void* d_out, float* d_lse, const int32_t* d_block_table,
                           uint32_t bt_stride, const int32_t* d_cu_q, const int32_t* d_ctx_lens,
                           uint32_t batch, uint32_t max_q_len, float sm_scale,
                           const float* d_kv_scales, void* stream);

/* K4 with a workspace (quantised formats).  When the chunk is long enough
 * that every KV tile would be dequantised by several query-tile CTAs
 * (max_q_len x GQA group >= 1024), the context blocks are first expanded
 * once into fp16 scratch blocks (block b of sequence s at s*bt_stride + b,
 * laid out like FP16 slab blocks) and attended by the FP16 tcgen05 kernel.
 * The workspace also enables split-KV: when batch x kv heads x query tiles
 * would leave SMs idle (short chunks over long contexts), each query tile's
 * KV range is cut over up to 8 CTAs whose fp32 partials are merged by a
 * second kernel.  ks_paged_prefill_workspace_size gives the bytes for both
 * (partials first, then the expand scratch; FP16 needs only the partials); a
 * smaller workspace drops the split first, then takes the expand in
 * sequence groups (at least one sequence's blocks, batch = 1).  A null
 * workspace runs exactly ks_paged_prefill. */
ks_status ks_paged_prefill_workspace_size(const ks_kv_format* fmt, uint32_t batch, uint32_t bt_stride,
                                          uint32_t max_q_len, size_t* bytes);
ks_status ks_paged_prefill_ws(ks_pool* pool, const ks_kv_format* fmt, uint32_t layer, const void* d_q,
                              void* d_out, float* d_lse, const int32_t* d_block_table,
                              uint32_t bt_stride, const int32_t* d_cu_q, const int32_t* d_ctx_lens,
                              uint32_t batch, uint32_t max_q_len, float sm_scale,
                              const float* d_kv_scales, void* d_workspace, size_t workspace_bytes,
                              void* stream);

/* Spatial sharing between co-located models (MPS-style SM partitioning,
 * PAPER.md section 2.4): cap the persistent K2 grid of the model with slab
 * key `key` at max_ctas SMs (the kernel places one CTA per SM, two for INT8),
 * so co-located models' decode kernels issued on different streams run side
 * by side.  0 = whole GPU. */
ks_status ks_set_decode_sm_share(ks_pool* pool, uint64_t key, uint32_t max_ctas);

/* K3 -- slab compaction for one key (new; the reference never migrates,
 * SPEC.md:223).  plan: host-side, deterministic; it
 * moves blocks out of the least-occupied PARTIAL slabs of `key` so they
 * return FREE and can be reformatted for any key.  The host table is
 * updated immediately; the bytes move when ks_compact_apply runs on the
 * stream, which must precede the next K1/K2 on that stream. */
typedef struct ks_block_move {
  uint64_t src_global_block_id;
  uint64_t dst_global_block_id;
} ks_block_move;
ks_status ks_compact_plan(ks_pool* pool, uint64_t key, uint32_t max_moves, ks_block_move* moves,
                          uint32_t* n_moves, uint32_t* slabs_freed);
/* copies `key` bytes per move inside the KV tensor (K3 kernel) */
ks_status ks_compact_apply(ks_pool* pool, uint64_t key, const ks_block_move* moves, uint32_t n,
                           void* stream);
/* rewrites block-table entries equal to a moved src id to its dst id (any
 * number of moves; taken in chunks) */
ks_status ks_block_table_remap(ks_pool* pool, int32_t* d_table, uint64_t n_entries,
                               const ks_block_move* moves, uint32_t n, void* stream);

/* ------------------------------------------------------------------ */
/* Engine block tables (simulator.cpp:33-40 LiveRequest::blocks)      */
/* ------------------------------------------------------------------ */
/* A sequence table is the engine-side logical block table of one model: a
 * row per sequence slot holding its handles in logical-block order and its
 * cached-token count, driven by the reference's three allocator call sites
 * -- prefill claim with rollback (simulator.cpp:500-526), decode growth
 * need = ceil((cached+1)/tpb) with per-request stall (:561-578), release on
 * completion / eviction (:583-596, :621) -- and mirrored into the engine's
 * int32 device table [max_seqs][row_stride] of global block ids by delta
 * upload (ks_seq_table_sync).  Tables register with their pool, so
 * ks_compact rewrites every table of the compacted key, whichever model owns
 * it.  Destroying a table does not free its blocks (release rows first);
 * destroying the pool detaches its tables (later calls fail). */
typedef struct ks_seq_table ks_seq_table;
typedef struct ks_seq_table_config {
  uint64_t key;                  /* the model's slab key (kv_block_size) */
  uint32_t max_seqs;
  uint32_t max_blocks_per_seq;
  uint32_t tokens_per_block;
  uint32_t reserved;
  uint64_t useful_token_bytes;   /* num_layers * token_size (simulator.cpp:210) */
  uint64_t block_metadata_bytes; /* num_layers * quant params per block (:211-212) */
  int32_t* d_table;              /* engine-owned device table; NULL = host only */
  uint32_t row_stride;           /* entries per device row, >= max_blocks_per_seq */
} ks_seq_table_config;
typedef struct ks_seq_table_stats {
  uint32_t live_seqs;            /* rows holding blocks */
  uint64_t held_blocks;          /* held_blocks_total (simulator.cpp:75-79) */
  uint64_t cached_tokens;        /* cached_total (simulator.cpp:70-74) */
  uint64_t internal_frag_bytes;  /* internal_frag_bytes (simulator.cpp:80-89) */
} ks_seq_table_stats;
ks_status ks_seq_table_create(ks_pool* pool, const ks_seq_table_config* cfg, ks_seq_table** out);
ks_status ks_seq_table_destroy(ks_seq_table* t);
/* prefill claim: ceil(prompt/tpb) blocks or none; *ok = 0 when the pool cannot back it */
ks_status ks_seq_table_admit(ks_seq_table* t, uint32_t seq, uint64_t prompt_tokens, int32_t* ok);
/* growth to ceil(tokens/tpb) blocks; *ok = 0 = stalled (blocks claimed so far are kept) */
ks_status ks_seq_table_ensure(ks_seq_table* t, uint32_t seq, uint64_t tokens, int32_t* ok);
/* one decode step of a batch: each listed row grows for its next token and,
 * if it got the block, advances by one; stalled[i] (nullable) = 1 otherwise */
ks_status ks_seq_table_step(ks_seq_table* t, const uint32_t* seqs, uint32_t n, uint8_t* stalled,
                            uint32_t* n_active);
ks_status ks_seq_table_release(ks_seq_table* t, uint32_t seq);
/* moves a sequence to an empty row (no allocator traffic), e.g. to keep the
 * running batch in rows 0..B-1; the destination row is re-uploaded */
ks_status ks_seq_table_move_row(ks_seq_table* t, uint32_t src, uint32_t dst);
ks_status ks_seq_table_cached(const ks_seq_table* t, uint32_t seq, uint64_t* tokens);
ks_status ks_seq_table_set_cached(ks_seq_table* t, uint32_t seq, uint64_t tokens);
/* out[s] = cached(s) + plus for rows 0..n-1 that hold blocks, 0 for empty rows */
ks_status ks_seq_table_ctx_lens(const ks_seq_table* t, int32_t* out, uint32_t n, int32_t plus);
/* *n = blocks held by the row; the first min(*n, capacity) handles are written */
ks_status ks_seq_table_blocks(const ks_seq_table* t, uint32_t seq, ks_block_handle* out,
                              uint32_t capacity, uint32_t* n);
ks_status ks_seq_table_get_stats(const ks_seq_table* t, ks_seq_table_stats* out);
/* number of entries changed since the last sync */
ks_status ks_seq_table_pending(const ks_seq_table* t, uint32_t* n);
ks_status ks_seq_table_sync(ks_seq_table* t, void* stream);

/* K3 as one transaction: plan (<= max_moves), move the bytes, and rewrite
 * the handles and device entries of every registered table of `key`, all on
 * `stream`.  On any failure the host slab table and the tables are restored
 * and nothing is reported as moved.  `stream` must be ordered after every
 * earlier launch that touches blocks of `key`; later launches through this
 * library on other streams wait for the compaction automatically (eager
 * launches; capture graphs after the compaction has been issued on the
 * replay stream).  Tables that are not registered can be rewritten with
 * ks_compact_plan / ks_compact_apply / ks_block_table_remap. */
ks_status ks_compact(ks_pool* pool, uint64_t key, uint32_t max_moves, void* stream,
                     uint32_t* n_moves, uint32_t* slabs_freed);

/* Design probes only: in a -DKVSLAB_PROBES build, the following K2 launches
 * write per-CTA globaltimer stamps to d_trace (NULL = off; scripts/
 * probe_timeline.py).  KS_NOT_SUPPORTED in release builds. */
ks_status ks_probe_set_decode_trace(ks_pool* pool, void* d_trace);

/* Number of kernel launches this process issued through the library
 * (per kernel family); used by bench.py for its gpu_launches claim. */
uint64_t ks_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KVSLAB_H_ */
