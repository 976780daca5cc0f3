/* kvslab_oracle.h -- CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * as the timed CPU baseline.  The product path (paper_2509_06261_b200) never
 * links, loads or calls it.
 *
 * What it restates, and how it is pinned:
 *   - token/block geometry       precision.cpp:76-99          pinned: tests/golden/precision.json
 *   - slab allocator             slab_pool.cpp:51-272         pinned: tests/golden/slab_*.json|npz
 *   - mt19937_64 uniform01       workload.hpp:32-48           pinned: tests/golden/rng.json
 *   - KV byte format, quantised append, fp64 paged decode, compaction plan:
 *     NO reference implementation exists (SURVEY.md
 *     section 8c).  These follow the byte-size formulas of PAPER.md:231-239 /
 *     precision.cpp:91-99 and the layout written down in DESIGN.md section 3.
 *     They are "parity unpinned" with respect to the reference: the CUDA path
 *     is bit-exact / within tolerance against THIS restatement only.
 */
#ifndef KVSLAB_ORACLE_H_
#define KVSLAB_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- RNG (workload.hpp:32-48) ---------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
void orc_rng_fill_uniform(orc_rng* r, double* out, size_t n);

/* ---------------- geometry (precision.cpp:76-99) ---------------- */
/* returns 0 on success, -1 on the reference's InvalidProfileError cases */
int orc_token_size(uint32_t num_kv_heads, uint32_t head_dim, uint32_t tp_degree,
                   int kv_bits, uint64_t* out);
int orc_kv_block_size(uint32_t num_kv_heads, uint32_t head_dim, uint32_t tp_degree,
                      int kv_bits, uint64_t tokens_per_block, uint64_t qparams_per_block,
                      uint32_t num_layers, uint64_t* out);

/* ---------------- slab allocator restatement (slab_pool.cpp) ---------------- */
typedef struct orc_pool orc_pool;
enum { ORC_OK = 0, ORC_INVALID_CONFIG = 1, ORC_INVALID_KEY = 2, ORC_EXHAUSTED = 3,
       ORC_INVALID_FREE = 4 };
typedef struct {
  uint32_t slab_id, local_block_id;
  uint64_t global_block_id, key;
} orc_handle;
int orc_pool_create(uint64_t capacity, uint64_t slab_size, const uint64_t* keys, uint32_t nkeys,
                    int require_lcm, orc_pool** out);
void orc_pool_destroy(orc_pool* p);
/* try-alloc semantics: returns ORC_EXHAUSTED with *out untouched when no room */
int orc_pool_alloc(orc_pool* p, uint64_t key, orc_handle* out);
int orc_pool_free(orc_pool* p, const orc_handle* h);
void orc_pool_stats(const orc_pool* p, uint64_t out[4]);
uint32_t orc_pool_slab_count(const orc_pool* p);
/* state: 0 FREE, 1 PARTIAL, 2 FULL */
void orc_pool_slab(const orc_pool* p, uint32_t slab, int* state, uint64_t* key, uint32_t* used,
                   uint32_t* total);
/* occupancy bit of (slab, local); -1 when out of range */
int orc_pool_bit(const orc_pool* p, uint32_t slab, uint32_t local);

/* ---------------- KV byte format ---------------- */
enum { ORC_FP16 = 0, ORC_FP8 = 1, ORC_INT8 = 2, ORC_INT4 = 3 };
typedef struct {
  uint32_t kv_dtype;
  uint32_t num_kv_heads; /* per shard */
  uint32_t num_q_heads;  /* per shard */
  uint32_t head_dim;
  uint32_t num_layers;
  uint32_t tokens_per_block;
  uint64_t qparams; /* quant-param bytes per block per layer */
} orc_fmt;
uint64_t orc_fmt_token_size(const orc_fmt* f);  /* bytes per token per layer */
uint64_t orc_fmt_chunk_bytes(const orc_fmt* f); /* tpb*d*bits/8 */
uint64_t orc_fmt_layer_bytes(const orc_fmt* f); /* tpb*token_size + qparams */
uint64_t orc_fmt_key(const orc_fmt* f);         /* num_layers * layer_bytes */
/* natural quant-param bytes of the format (FP8: in-block per-head scales) */
uint64_t orc_fmt_natural_qparams(const orc_fmt* f);
/* 128-byte swizzle of 16-byte granules inside a K/V chunk */
uint64_t orc_swz(uint64_t chunk_offset);

/* block byte offset inside the pool for (slab, local) */
uint64_t orc_block_offset(uint64_t slab_size, uint64_t key, uint64_t bps, uint64_t gid);

uint8_t orc_f32_to_e4m3(float x);
float orc_e4m3_to_f32(uint8_t c);
uint16_t orc_f32_to_f16(float x);
float orc_f16_to_f32(uint16_t h);

/* Quantised append (K1 restated).  k, v: fp16 [n_tok][H][d].  For token i,
 * sequence tok_seq[i] at position tok_pos[i]: block = block_table[seq*bt_stride
 * + pos/tpb] (a global block id of key orc_fmt_key), slot = pos%tpb.
 * kv_scales: fp32 [2][H] (FP8 only; NULL = 1.0). */
void orc_append(uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                uint32_t layer, const uint16_t* k, const uint16_t* v, uint32_t n_tok,
                const int32_t* tok_seq, const int32_t* tok_pos, const int32_t* block_table,
                uint32_t bt_stride, const float* kv_scales);

/* dequantised K/V of one (layer, head, token slot) of a block, fp64 [d] */
void orc_dequant(const uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                 uint32_t layer, uint64_t gid, uint32_t kv, uint32_t head, uint32_t slot,
                 const float* kv_scales, double* out);

/* fp64 paged decode (K2 restated).  q: fp16 [B][Hq][d]; out fp64 [B][Hq][d];
 * lse (natural log, nullable) fp64 [B][Hq].  OpenMP over (seq, head) when
 * nthreads > 1. */
void orc_paged_decode(const uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                      uint32_t layer, const uint16_t* q, const int32_t* block_table,
                      uint32_t bt_stride, const int32_t* ctx_lens, uint32_t batch,
                      double sm_scale, const float* kv_scales, double* out, double* lse,
                      int nthreads);

/* algorithmic bytes of one decode launch */
/* chunked prefill: queries of sequence s are rows cu_q[s]..cu_q[s+1]-1 of q,
 * at positions ctx_lens[s]-n_s..ctx_lens[s]-1, causal over keys 0..pos */
void orc_paged_prefill(const uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                       uint32_t layer, const uint16_t* q, const int32_t* block_table,
                       uint32_t bt_stride, const int32_t* cu_q, const int32_t* ctx_lens,
                       uint32_t batch, double sm_scale, const float* kv_scales, double* out,
                       double* lse, int nthreads);
uint64_t orc_decode_bytes(const orc_fmt* f, const int32_t* ctx_lens, uint32_t batch);

/* ---------------- compaction plan (K3 restated; new, no reference) --------- */
/* Plans moves for one key: sources are PARTIAL slabs of the key taken in
 * (blocks_used asc, slab_id desc) order; a source is evacuated only if all
 * its blocks fit into free blocks of the remaining destination slabs, taken
 * in (blocks_used desc, slab_id asc) order, lowest free local id first.
 * Applies the moves to the pool (alloc-at + free) and writes (src_gid,dst_gid)
 * pairs.  Returns the number of moves (<= max_moves). */
uint32_t orc_compact_plan(orc_pool* p, uint64_t key, uint32_t max_moves, uint64_t* src_gid,
                          uint64_t* dst_gid, uint32_t* slabs_freed);

#ifdef __cplusplus
}
#endif
#endif
