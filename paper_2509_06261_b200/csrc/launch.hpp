// launch.hpp -- kernel parameter blocks and host-side launchers (internal).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "kvslab_geom.hpp"

namespace kvslab {

constexpr int kDecodeWarps = 4;

// Probe builds (-DKVSLAB_PROBES) compile the per-warp timestamp hooks into
// the decode kernels; release builds compile them out.
#ifdef KVSLAB_PROBES
constexpr bool kProbes = true;
#else
constexpr bool kProbes = false;
#endif

// Tuning overrides for experiments (scripts/ab_decode.py and friends).  Read
// from KVSLAB_* environment variables once, when a pool is created -- never
// on the launch path.  Zero / -1 = the library's default.
struct Tuning {
  int decode_max_ctas = 0;         // KVSLAB_DECODE_MAX_CTAS
  uint32_t decode_hg = 0;          // KVSLAB_DECODE_HG
  uint32_t decode_smem = 0;        // KVSLAB_DECODE_SMEM
  uint32_t merge_threads = 0;      // KVSLAB_MERGE_THREADS
  uint32_t merge_dc = 0;           // KVSLAB_MERGE_DC
  uint32_t decode_pack = 0;        // KVSLAB_DECODE_PACK
  int decode_debug = 0;            // KVSLAB_DECODE_DEBUG (probe builds only)
  unsigned long long* decode_trace = nullptr;  // KVSLAB_DECODE_TRACE (probe builds only)
  int pdl = 1;                     // KVSLAB_NO_PDL=1 -> 0
  uint32_t append_per_sm = 0;      // KVSLAB_APPEND_PER_SM (K1 CTAs per SM, 0 = occupancy)
  uint32_t decode_min_blocks = 0;  // KVSLAB_DECODE_MIN_BLOCKS (K2 blocks per CTA floor, 0 = default)
  uint32_t prefill_nt = 0;         // KVSLAB_PREFILL_NT
  int prefill_tc = 2;              // KVSLAB_PREFILL_TC
  int prefill_debug = 0;           // KVSLAB_PREFILL_DEBUG (probe builds only)
  int prefill_expand = -1;         // KVSLAB_PREFILL_EXPAND (-1 auto)
  int prefill_split = 1;           // KVSLAB_PREFILL_SPLIT
  static Tuning from_env();
};

struct DecodeParams {
  const uint8_t* pool;
  dev::SlabGeom geom;
  uint64_t layer_off;  // layer * layer_bytes
  uint32_t H, G;       // kv heads, query heads per kv head
  const __half* q;
  __half* out;
  float* lse;
  const int32_t* block_table;
  uint32_t bt_stride;
  const int32_t* ctx_lens;
  uint32_t batch;
  float sm_scale_log2;
  const float* kv_scales;  // FP8 [2][H]
  const __half* k_new;     // fused append: new token K/V [batch][H][d] (nullable)
  const __half* v_new;
  uint32_t params_off;     // 2*H*chunk: quant params inside a layer sub-block
  bool fp8_inblock;
  float* partials;
  // filled by the launcher
  uint32_t stage_bytes, bar_offset, qbuf_offset, prefix_offset, hg, stages;
  int max_ctas;  // SMs the grid may cover (x CTAs per SM); 0 = persistent full machine
  uint32_t hg_max;        // 0 = default head-group size
  uint32_t smem_budget;   // ring bytes per CTA; 0 = default
  uint32_t merge_threads; // merge CTA size cap; 0 = default (256)
  uint32_t merge_dc;      // probe override of the merge's dims split (0 = auto)
  uint32_t pack_mode;     // packed G<=4 step: 0 = auto, 1 = off, 2-4 A/B forms (decode.cu)
  int debug;     // bit0: skip math, bit1: skip partial merge (probes only)
  int pdl;       // launch with programmatic stream serialization
  uint32_t min_blocks;    // >= this many blocks per CTA (0 = kMinBlocksPerCta)
  unsigned long long* trace;  // probes: per-warp globaltimer stamps (nullable)
};

struct PrefillParams {
  const uint8_t* pool;
  dev::SlabGeom geom;
  uint64_t layer_off;
  uint32_t H, G;
  const __half* q;         // [T_total][H*G][d]
  __half* out;
  float* lse;
  const int32_t* block_table;
  uint32_t bt_stride;
  const int32_t* cu_q;     // [batch+1] query-row offsets
  const int32_t* ctx_lens; // [batch] cached tokens including the chunk
  uint32_t batch, max_q_len;
  float sm_scale_log2;
  const float* kv_scales;  // FP8 [2][H]
  const float* exp_sz;     // expand scratch: K scale/zero per (seq, block, head) (EXP kernels)
  uint32_t kv_splits;      // split-KV CTAs per query tile (tcgen05 kernel; needs part)
  float* part;             // split-KV partials [row][split][kD + 4]
  uint32_t nt;  // query rows per warp / 8 (1 or 2; 0 = default: 1, or 2 when G > 8)
  int use_tc;   // tcgen05 kernel (prefill_tc.cu) unless 0 (then mma.sync, prefill.cu)
  int debug;    // probes: bit0 no KV loads after the first two tiles, bit1 no softmax math
  // filled by the launcher
  uint32_t tiles, stages, stage_bytes, qbuf_offset, bar_offset;
};

struct AppendParams {
  uint8_t* pool;
  dev::SlabGeom geom;
  uint64_t layer_off;
  uint32_t H, D, tpb;
  uint32_t chunk_bytes, params_off;
  bool fp8_inblock;
  const __half* k;
  const __half* v;
  uint32_t n_tokens;
  const int32_t* tok_seq;
  const int32_t* tok_pos;
  const int32_t* block_table;
  uint32_t bt_stride;
  const float* kv_scales;
  uint32_t ctas_per_sm;  // 0 = every resident slot (occupancy); else at most this many per SM
};

struct CompactParams {
  uint8_t* pool;
  dev::SlabGeom geom;
  const uint32_t* src_gid;
  const uint32_t* dst_gid;
  uint32_t n_moves;
};

cudaError_t launch_paged_decode(const DecodeParams& p, int kv_dtype, int num_sms,
                                cudaStream_t stream);
size_t decode_partials_bytes(int num_sms, int G);
cudaError_t launch_paged_prefill(const PrefillParams& p, int kv_dtype, cudaStream_t stream);
cudaError_t launch_paged_prefill_tc(const PrefillParams& p, int kv_dtype, cudaStream_t stream);  // tcgen05
// quantised formats: expand the context once into fp16 scratch, then the FP16 kernel
size_t prefill_expand_bytes(uint32_t H, uint32_t batch, uint32_t bt_stride);
// split-KV: CTAs per query tile that fill the SMs (1 = none), and the partials' bytes
uint32_t prefill_kv_splits(uint32_t batch, uint32_t H, uint32_t G, uint32_t max_q_len, int num_sms);
size_t prefill_partial_bytes(uint32_t batch, uint32_t H, uint32_t G, uint32_t max_q_len, uint32_t splits);
cudaError_t launch_paged_prefill_expand(const PrefillParams& p, int kv_dtype, uint8_t* scratch,
                                        cudaStream_t stream);
cudaError_t launch_kv_append(const AppendParams& p, int kv_dtype, cudaStream_t stream);
cudaError_t launch_compact(const CompactParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_table_scatter(int32_t* table, uint32_t row_stride, const int32_t* triples,
                                 uint32_t n, cudaStream_t stream);
cudaError_t launch_table_remap(int32_t* table, uint64_t n_entries, const uint32_t* src_sorted,
                               const uint32_t* dst_sorted, uint32_t n, cudaStream_t stream);
cudaError_t launch_table_validate(const int32_t* table, uint32_t row_stride,
                                  const int32_t* ctx_lens, uint32_t rows, uint32_t tpb,
                                  const void* slab_table, uint32_t slab_count, uint64_t key,
                                  dev::FastDiv bps, unsigned long long* n_bad,
                                  cudaStream_t stream);
cudaError_t launch_slab_table_scatter(void* table, const void* entries, uint32_t n,
                                      cudaStream_t stream);

}  // namespace kvslab
