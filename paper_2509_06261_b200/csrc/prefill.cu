// prefill.cu -- K4: chunked-prefill attention over slab blocks for sm_100a.
//
// the step before decode on the same blocks.  The
// reference claims ceil(prompt/tpb) blocks per admitted request
// (simulator.cpp:500-526) and charges the prefill as a cost (:536-538); here
// K1 writes the chunk's K/V into those blocks and this kernel attends the
// chunk's queries causally over every cached token of the sequence through
// the slab indirection.  Output matches oracle/kvslab_oracle.c
// orc_paged_prefill (fp64) within 1e-3 (FP16/FP8) or 1e-2 (INT8/INT4).
//
// Work: one CTA per (sequence, kv head, query tile).  A tile is 8 consumer
// warps x 8 query rows (8/G tokens x the G query heads of the kv head), so a
// CTA streams the head's blocks 0..(last position)/16 once for 64 query rows.
// A producer warp copies each block's K chunk, V chunk and params of the head
// (cp.async.bulk, TMA engine) into a STAGES-deep ring; each consumer warp runs
// the shared tensor-core step (attend.cuh) over the blocks its rows can see,
// masking only the diagonal blocks.  Tiles are launched heaviest first
// (latest positions), so the causal work imbalance drains in the tail.
#include <cuda_runtime.h>
#include <stdint.h>

#include "attend.cuh"
#include "kvslab_device.cuh"
#include "func_cache.hpp"
#include "launch.hpp"

namespace kvslab {
namespace dev {

// consumer warps per CTA: 8*NT query rows each; the CTA (W+1 warps) fits one
// SM's register file per sub-partition (NT=1: <= 152 regs, NT=2: <= 240)
template <int NT>
constexpr int kPrefillWarps = NT == 1 ? 11 : 6;

template <int FMT, int NT>
__global__ void __maxnreg__(NT == 1 ? 152 : 240) prefill_kernel(const PrefillParams p) {
  using Gm = Geo<FMT>;
  constexpr int W = kPrefillWarps<NT>;
  constexpr int R = 8 * NT;  // query rows per consumer warp
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t s = blockIdx.x / p.H, h = blockIdx.x % p.H;
  const uint32_t tile = p.tiles - 1 - blockIdx.y;  // heaviest (latest) tiles first
  const int q0 = p.cu_q[s], nq = p.cu_q[s + 1] - q0;
  const uint32_t G = p.G, TPW = R / G;             // tokens per consumer warp
  const int QT = static_cast<int>(W * TPW);       // tokens per tile
  const int tok0 = static_cast<int>(tile) * QT;
  if (tok0 >= nq) return;  // uniform across the CTA
  const int ctx = p.ctx_lens[s];
  const int pos0 = ctx - nq;  // position of the chunk's first query
  const int tok_end = min(nq, tok0 + QT);
  const uint32_t nb = static_cast<uint32_t>(pos0 + tok_end - 1) / kTPB + 1;  // blocks the CTA streams
  const uint32_t S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_offset);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], W);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t chunk = Gm::kChunk, prm = Gm::kParam;

  if (warp == W) {
    // ============================ producer warp ============================
    // K chunk, V chunk, K params, V params of head h: 2 (or 4) bulk copies.
    const uint32_t stage_tx = 2 * chunk + 2 * prm;
    const uint64_t pol = policy_evict_last();  // every later tile of (s, h) re-reads these blocks
    const int32_t* bt = p.block_table + static_cast<uint64_t>(s) * p.bt_stride;
    uint32_t st = 0, ph = 0;
    const uint32_t ring = smem_u32(smem);
    int32_t ent = lane < static_cast<int>(nb) ? __ldg(bt + lane) : 0;
    for (uint32_t b = 0; b < nb; ++b) {
      if ((b & 31) == 0 && b > 0)
        ent = b + lane < nb ? __ldg(bt + b + lane) : 0;
      const uint32_t gid = static_cast<uint32_t>(__shfl_sync(0xffffffffu, ent, b & 31));
      mbar_wait(&empty[st], ph ^ 1);
      if (lane == 0) {
        const uint8_t* base = p.pool + block_offset(p.geom, gid) + p.layer_off;
        const uint32_t sb = ring + st * p.stage_bytes;
        mbar_expect_tx(&full[st], stage_tx);
        bulk_g2s_u32(sb, base + static_cast<uint64_t>(h) * chunk, chunk, &full[st], pol);
        bulk_g2s_u32(sb + chunk, base + static_cast<uint64_t>(p.H + h) * chunk, chunk, &full[st], pol);
        if constexpr (Gm::kParam > 0) {
          const uint8_t* pp = base + 2ull * p.H * chunk + static_cast<uint64_t>(h) * prm;
          bulk_g2s_u32(sb + 2 * chunk, pp, prm, &full[st], pol);
          bulk_g2s_u32(sb + 2 * chunk + prm, pp + static_cast<uint64_t>(p.H) * prm, prm, &full[st], pol);
        }
      }
      if (++st == S) {
        st = 0;
        ph ^= 1;
      }
    }
    return;
  }

  // ============================ consumer warps ============================
  // Query rows of this warp: column c = token (c / G) x head (c % G).
  const int wtok0 = tok0 + warp * static_cast<int>(TPW);
  const int wtok_end = min(tok_end, wtok0 + static_cast<int>(TPW));  // may be <= wtok0
  const uint32_t Hq = p.H * G;
  uint8_t* sq = smem + p.qbuf_offset + warp * R * kD * 2;
  // stage the warp's R query rows in shared memory (row r = token r/G x head r%G)
  for (int i = lane; i < R * 16; i += 32) {
    const int r = i >> 4, part = i & 15;
    const int tok = wtok0 + r / static_cast<int>(G);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (tok < wtok_end)
      v = __ldg(reinterpret_cast<const uint4*>(p.q + (static_cast<uint64_t>(q0 + tok) * Hq + h * G + r % G) * kD) +
                part);
    reinterpret_cast<uint4*>(sq + r * kD * 2)[part] = v;
  }
  __syncwarp();
  const FragOff fo = make_offsets<FMT>(g, t);
  uint32_t qf[NT][8][2];
  load_q_frags<FMT, NT>(smem_u32(sq), g, t, R, qf);
  float qsb[NT][2], qst[NT][2];
  UnitState<NT> us;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    qsb[nt][0] = qsb[nt][1] = qst[nt][0] = qst[nt][1] = 0.f;
    if constexpr (Gm::kBiased) {
      float lo = 0.f, hi = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const float2 f0 = __half22float2(*reinterpret_cast<__half2*>(&qf[nt][kk][0]));
        const float2 f1 = __half22float2(*reinterpret_cast<__half2*>(&qf[nt][kk][1]));
        lo += f0.x + f0.y;
        hi += f1.x + f1.y;
      }
      float sbq = lo + hi, stq = FMT == kINT4 ? lo + 16.f * hi : sbq;
      sbq += __shfl_xor_sync(0xffffffffu, sbq, 1);
      sbq += __shfl_xor_sync(0xffffffffu, sbq, 2);
      stq += __shfl_xor_sync(0xffffffffu, stq, 1);
      stq += __shfl_xor_sync(0xffffffffu, stq, 2);
      qsb[nt][0] = __shfl_sync(0xffffffffu, sbq, (2 * t) * 4);
      qsb[nt][1] = __shfl_sync(0xffffffffu, sbq, (2 * t + 1) * 4);
      qst[nt][0] = __shfl_sync(0xffffffffu, stq, (2 * t) * 4);
      qst[nt][1] = __shfl_sync(0xffffffffu, stq, (2 * t + 1) * 4);
    }
    us.m[nt][0] = us.m[nt][1] = -INFINITY;
    us.l[nt][0] = us.l[nt][1] = 0.f;
    us.zb[nt][0] = us.zb[nt][1] = 0.f;
    us.zz[nt][0] = us.zz[nt][1] = 0.f;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
      us.acc[mt][nt][0] = us.acc[mt][nt][1] = us.acc[mt][nt][2] = us.acc[mt][nt][3] = 0.f;
  }
  float kscale = 1.f, vscale = 1.f;
  if constexpr (FMT == kFP8) {
    if (p.kv_scales) {
      kscale = p.kv_scales[h];
      vscale = p.kv_scales[p.H + h];
    }
  }
  // positions of this lane's two query columns (2t, 2t+1); padding columns
  // reuse the warp's last valid position (computed, never stored)
  const int wlast = wtok_end > wtok0 ? pos0 + wtok_end - 1 : pos0;
  int qpos[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int tok = wtok0 + (nt * 8 + 2 * t + c) / static_cast<int>(G);
      qpos[nt][c] = tok < wtok_end ? pos0 + tok : wlast;
    }
  const int wfirst = wtok_end > wtok0 ? pos0 + wtok0 : pos0;
  const uint32_t nb_w = wtok_end > wtok0 ? static_cast<uint32_t>(wlast) / kTPB + 1 : 0u;
  const float sml2 = p.sm_scale_log2;
  const uint32_t ring = smem_u32(smem);
  uint32_t st = 0, ph = 0, since_flush = 0;
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == S) {
      st = 0;
      ph ^= 1;
    }
  };
  for (uint32_t b = 0; b < nb;) {
    const int bstart = static_cast<int>(b) * kTPB;
    if constexpr (NT == 1) {
      // two whole blocks per step (independent score tiles: more ILP)
      if (b + 1 < nb_w && bstart + 2 * kTPB - 1 <= wfirst) {
        const uint32_t st1 = st + 1 == S ? 0 : st + 1, ph1 = st + 1 == S ? ph ^ 1 : ph;
        mbar_wait(&full[st], ph);
        mbar_wait(&full[st1], ph1);
        const uint32_t sbs[2] = {ring + st * p.stage_bytes, ring + st1 * p.stage_bytes};
        const int valid[2] = {kTPB, kTPB};
        attend<FMT, NT, 2, false, false>(us, sbs, valid, 0u, 2 * chunk, chunk, prm, fo, qf, qsb, qst, kscale,
                                         sml2, g, t);
        release();
        release();
        b += 2;
        if ((since_flush += 2) >= kBiasFlush) {
          flush_bias<FMT, NT>(us);
          since_flush = 0;
        }
        continue;
      }
    }
    mbar_wait(&full[st], ph);
    if (b < nb_w) {
      const uint32_t sbs[1] = {ring + st * p.stage_bytes};
      const int valid[1] = {kTPB};
      if (bstart + kTPB - 1 <= wfirst) {  // every row of the warp sees the whole block
        attend<FMT, NT, 1, false, false>(us, sbs, valid, 0u, 2 * chunk, chunk, prm, fo, qf, qsb, qst, kscale,
                                         sml2, g, t);
      } else {  // diagonal block: causal mask per query column
        int lim[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          lim[nt][0] = qpos[nt][0] - bstart + 1;
          lim[nt][1] = qpos[nt][1] - bstart + 1;
        }
        attend<FMT, NT, 1, true, true>(us, sbs, valid, 0u, 2 * chunk, chunk, prm, fo, qf, qsb, qst, kscale,
                                       sml2, g, t, lim);
      }
      if (++since_flush >= kBiasFlush) {
        flush_bias<FMT, NT>(us);
        since_flush = 0;
      }
    }
    release();
    ++b;
  }
  if (nb_w == 0) return;
  // ---- epilogue: normalise and store the warp's valid rows ----
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float l = us.l[nt][c], zb = us.zb[nt][c], zz = us.zz[nt][c];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
        if constexpr (Gm::kBiased) zb += __shfl_xor_sync(0xffffffffu, zb, o);
        if constexpr (FMT == kINT4) zz += __shfl_xor_sync(0xffffffffu, zz, o);
      }
      const int col = nt * 8 + 2 * t + c;
      const int tok = wtok0 + col / static_cast<int>(G);
      if (tok >= wtok_end) continue;
      const float inv = 1.f / l;
      const uint64_t row = static_cast<uint64_t>(q0 + tok) * Hq + h * G + col % G;
      __half* orow = p.out + row * kD;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int d0 = vdim<FMT>(mt, g, 0);
        const float lo = us.acc[mt][nt][c] * vscale + zb + zz;
        float hi;
        if constexpr (FMT == kINT4) hi = (us.acc[mt][nt][2 + c] + zb) * 0.0625f + zz;
        else hi = us.acc[mt][nt][2 + c] * vscale + zb + zz;
        *reinterpret_cast<__half2*>(orow + d0) = __floats2half2_rn(lo * inv, hi * inv);
      }
      if (p.lse && g == 0) p.lse[row] = (us.m[nt][c] + __log2f(l)) * 0.69314718055994531f;
    }
}

template <int FMT, int NT>
static cudaError_t launch_prefill_fmt(const PrefillParams& p0, cudaStream_t stream) {
  using Gm = Geo<FMT>;
  constexpr int W = kPrefillWarps<NT>;
  PrefillParams p = p0;
  p.stage_bytes = (2 * (Gm::kChunk + Gm::kParam) + 127) / 128 * 128;
  const uint32_t qbytes = W * 8 * NT * kD * 2;
  uint32_t stages = (200 * 1024 - qbytes) / p.stage_bytes;
  if (stages > 16) stages = 16;
  p.stages = stages;
  p.qbuf_offset = stages * p.stage_bytes;
  p.bar_offset = p.qbuf_offset + qbytes;
  const size_t smem = p.bar_offset + 2 * stages * 8;
  auto kern = prefill_kernel<FMT, NT>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const uint32_t qt = W * (8 * NT / p.G);  // tokens per tile
  p.tiles = (p.max_q_len + qt - 1) / qt;
  if (p.tiles == 0) return cudaSuccess;
  kern<<<dim3(p.batch * p.H, p.tiles), (W + 1) * 32, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace dev

cudaError_t launch_paged_prefill(const PrefillParams& p, int kv_dtype, cudaStream_t stream) {
  using namespace dev;
  // 8 query rows per warp (default: more warps, two-block steps) or 16 (GQA 16)
  // tcgen05 kernel (two 128-row query tiles per CTA), except for quantised KV
  // when every chunk has <= 64 query rows: the dequantising loaders then
  // stream the whole context for a quarter-full tile, and the mma.sync kernel
  // measured faster (INT4, 16 x chunk 16 at ctx 4k: 142 vs 186 us; at chunk
  // 32 the tcgen05 kernel wins, 187 vs 295)
  const bool small = kv_dtype != kFP16 && p.max_q_len * p.G <= 64;
  // ... unless the tcgen05 kernel splits the KV range (few CTAs: small batch,
  // long context), which wins there (B=1 INT4 chunk 16 at ctx 8k: 258 -> 61 us)
  if (p.use_tc == 1 || (p.use_tc && (!small || p.kv_splits > 1)))  // 1: forced
    return launch_paged_prefill_tc(p, kv_dtype, stream);
  const bool two = p.nt == 2 || p.G > 8;
  switch (kv_dtype) {
    case kFP16: return two ? launch_prefill_fmt<kFP16, 2>(p, stream) : launch_prefill_fmt<kFP16, 1>(p, stream);
    case kFP8: return two ? launch_prefill_fmt<kFP8, 2>(p, stream) : launch_prefill_fmt<kFP8, 1>(p, stream);
    case kINT8: return two ? launch_prefill_fmt<kINT8, 2>(p, stream) : launch_prefill_fmt<kINT8, 1>(p, stream);
    case kINT4: return two ? launch_prefill_fmt<kINT4, 2>(p, stream) : launch_prefill_fmt<kINT4, 1>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace kvslab
