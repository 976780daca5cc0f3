// decode.cu -- K2: slab-indexed paged decode attention for sm_100a.
//
// Replaces the reference's simulated attention cost (simulator.cpp:602-604,
// "dur = gamma + delta*active + epsilon*sum(cached)") with the real read of
// every cached K/V byte through the slab indirection.  Output matches
// oracle/kvslab_oracle.c orc_paged_decode (fp64) within 1e-3 (FP16/FP8) or
// 1e-2 (INT8/INT4) relative.
//
// Design:
//  * Work = every (sequence, kv-head group, block) of the batch, flattened
//    seq-major and cut into one equal contiguous range per CTA of a
//    persistent grid (stream-K), so ragged contexts balance exactly.  A unit
//    (sequence, head group) cut by a range boundary leaves fp32 partials that
//    merge_kernel, launched behind with programmatic dependent launch,
//    combines; whole units are written directly.
//  * CTA = HG consumer warps (one kv head each) + one producer warp.  The
//    producer streams each block's K, V and params of the group with
//    cp.async.bulk (TMA engine; one copy when the group spans all kv heads)
//    into a STAGES-deep ring of full/empty mbarriers, and the group's Q rows
//    (plus, for the fused append, the new token's K/V rows) at unit starts.
//  * QK^T and PV run on tensor cores as m16n8k16 tiles with the query group
//    as N (8 or 16): S^T = K.Q^T (M = 16 tokens), O^T += V^T.P^T (M = dims).
//    Quantised K/V enter the MMA as exact small integers (or e4m3 -> f16);
//    per-token scales/zeros are applied to the 16x8 score tile and folded
//    into P, so dequantisation costs no extra multiply per element.
//  * The swizzled chunk layout plus the per-format fragment <-> dim/token
//    permutations make every shared-memory fragment load conflict-free.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "attend.cuh"
#include "kvslab_device.cuh"
#include "func_cache.hpp"
#include "launch.hpp"

namespace kvslab {
namespace dev {

// ------------------------------------------------------------------ cursor
// Walks the flattened (seq, head, block) space using the per-CTA prefix.
struct Cursor {
  uint32_t s, h, b, nblk;
};
__device__ __forceinline__ uint32_t nblk_of(const uint32_t* pre, uint32_t s, uint32_t H) {
  return (pre[s + 1] - pre[s]) / H;
}
__device__ __forceinline__ void cursor_seek(Cursor& c, const uint32_t* pre, uint32_t batch,
                                            uint32_t H, uint32_t idx) {
  // largest s with pre[s] <= idx
  uint32_t lo = 0, hi = batch;  // pre[batch] = total > idx
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (pre[mid] <= idx) lo = mid; else hi = mid;
  }
  c.s = lo;
  c.nblk = nblk_of(pre, lo, H);
  const uint32_t off = idx - pre[lo];
  c.h = off / c.nblk;
  c.b = off - c.h * c.nblk;
}
__device__ __forceinline__ void cursor_next(Cursor& c, const uint32_t* pre, uint32_t batch,
                                            uint32_t H) {
  if (++c.b < c.nblk) return;
  c.b = 0;
  if (++c.h < H) return;
  c.h = 0;
  do {
    ++c.s;
  } while (c.s < batch && pre[c.s + 1] == pre[c.s]);
  if (c.s < batch) c.nblk = nblk_of(pre, c.s, H);
}

// First flat index (CTA range start) of CTA c: floor(c * total / C), with
// 32-bit arithmetic only (c, r0 < C <= 2^16): c*q0 + (c*r0)/C.
struct CtaSplit {
  uint32_t total, C, q0, r0;
};
__device__ __forceinline__ CtaSplit make_split(uint32_t total, uint32_t C) {
  return CtaSplit{total, C, total / C, total % C};
}
__device__ __forceinline__ uint32_t cta_start(uint32_t c, const CtaSplit& sp) {
  return c * sp.q0 + (c * sp.r0) / sp.C;
}
// CTA whose range contains flat index f: the largest c with
// floor(c*total/C) <= f, i.e. c*total < (f+1)*C.
__device__ __forceinline__ uint32_t cta_of(uint32_t f, const CtaSplit& sp) {
  return static_cast<uint32_t>(((static_cast<uint64_t>(f) + 1) * sp.C - 1) / sp.total);
}

constexpr uint32_t kMinBlocksPerCta = 4;
// CTAs a launch uses: >= kMinBlocksPerCta blocks each, but at least one per
// (sequence, head group) unit when the grid allows (units <= batch x NG):
// with very short contexts (a few blocks per unit) four units serialised on
// one CTA -- a Q load, the fused append and an epilogue each -- cost more
// than the blocks (FP8 B8 ctx 16: 9.3 us per launch against 3.7 us at B1).
__device__ __forceinline__ uint32_t effective_ctas(uint32_t total, uint32_t grid, uint32_t units,
                                                   uint32_t min_blocks) {
  const uint32_t mb = min_blocks ? min_blocks : kMinBlocksPerCta;
  const uint32_t want = max((total + mb - 1) / mb, min(units, total));
  return max(1u, min(grid, want));
}

// ------------------------------------------------------------ merge kernel
// Combines the fp32 partials of every (sequence, head) unit that the decode
// kernel's CTA ranges cut:  O = sum_j 2^(m_j-M) acc_j / sum_j 2^(m_j-M) l_j.
// One CTA per (sequence, head).  Before griddepcontrol.wait -- i.e. while the
// decode grid still runs -- it recomputes the unit's CTA span from ctx_lens
// (block prefix, the same equal-range split as the decode kernel), so after
// the wait only the partial loads remain.  Warp (q, w) merges segments
// c = ca + w (mod WS) of query q online (SB loads in flight, 4 dims per lane);
// with WS > 1 the per-warp states are combined through shared memory.  The
// CTAs are small (<= 56 registers, <= 4 KB shared) so they co-reside with the
// running decode CTAs and with the next layer's.
template <int DC>  // dims split over DC CTAs per (sequence, head) (small batches)
__global__ void __maxnreg__(56) merge_kernel(const DecodeParams p, uint32_t WS, uint32_t grid) {
  constexpr int VW = 4 / DC;  // floats per lane
  pdl_launch_dependents();
  const uint64_t tm0 = (kProbes && p.trace) ? gtimer() : 0;
  extern __shared__ float4 msm[];  // WS > 1: o[G*WS][32], then m[G*WS], l[G*WS]
  __shared__ uint32_t red[2][32];
  const uint32_t unit = blockIdx.x / DC, dc = blockIdx.x % DC;
  const uint32_t s = unit / p.H, h = unit % p.H;
  const uint32_t HG = p.hg, NG = p.H / p.hg, grp = h / HG, hw = h % HG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t G = p.G;
  const uint32_t q = warp / WS, w = warp % WS;
  const int ctx_s = p.ctx_lens[s];
  // CTA 0 always waits for the decode grid, so this grid never completes
  // before it (a PDL successor that waits on the merge then also sees the
  // decode kernel's direct outputs, even when every unit was whole)
  if (ctx_s <= 0) {  // empty sequence: written by decode CTA 0
    if (blockIdx.x == 0) pdl_wait();
    return;
  }
  // blocks before sequence s and in total (ctx_lens is not written by the
  // PDL predecessor: same contract as the decode kernel's prologue)
  uint32_t before = 0, all = 0;
  for (uint32_t i = threadIdx.x; i < p.batch; i += blockDim.x) {
    const int c = p.ctx_lens[i];
    const uint32_t nb = c > 0 ? (static_cast<uint32_t>(c) + kTPB - 1) / kTPB : 0;
    all += nb;
    before += i < s ? nb : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    before += __shfl_xor_sync(0xffffffffu, before, o);
    all += __shfl_xor_sync(0xffffffffu, all, o);
  }
  if (lane == 0) {
    red[0][warp] = before;
    red[1][warp] = all;
  }
  __syncthreads();
  before = all = 0;
  for (uint32_t i = 0; i < blockDim.x / 32; ++i) {
    before += red[0][i];
    all += red[1][i];
  }
  const uint32_t nblk = (static_cast<uint32_t>(ctx_s) + kTPB - 1) / kTPB;
  const uint32_t total = all * NG;
  const uint32_t U0 = before * NG + grp * nblk;
  const CtaSplit sp = make_split(total, effective_ctas(total, grid, p.batch * NG, p.min_blocks));
  const uint32_t ca = cta_of(U0, sp), cb = cta_of(U0 + nblk - 1, sp);
  if (ca == cb) {  // whole unit: the decode kernel wrote it
    if (blockIdx.x == 0) pdl_wait();
    return;
  }
  // the unit is the last segment of CTA ca (its first if it starts there)
  // and the first segment of every later CTA
  const uint32_t slot_a = cta_start(ca, sp) < U0 ? 1u : 0u;
  pdl_wait();  // partials come from the decode kernel
  if (kProbes && p.trace && threadIdx.x == 0) {  // probes: [2048] first merge CTA past the wait
    const uint64_t tw = gtimer();
    atomicMin(p.trace + 2048, static_cast<unsigned long long>(tw));
    p.trace[2050 + 3 * blockIdx.x] = tm0;
    p.trace[2051 + 3 * blockIdx.x] = tw;
  }
  const uint32_t hdr = (2 * G + 3) & ~3u;
  const uint32_t slot_f = hdr + G * kD;
  constexpr int SB = DC == 1 ? 4 : (DC == 2 ? 8 : 10);  // loads in flight (<= 56 registers)
  const uint32_t d0 = dc * (kD / DC) + lane * VW;  // first dim of this lane
  float M = -INFINITY, L = 0.f;
  float o[VW];
#pragma unroll
  for (int v = 0; v < VW; ++v) o[v] = 0.f;
  // slot of CTA c: (2c + [c == ca ? slot_a : 0]) * HG + hw; header (m, l) pairs
  const uint32_t cstride = 2 * HG * slot_f;  // floats between consecutive CTAs' slots
  const float* pbase = p.partials + static_cast<uint64_t>(hw) * slot_f;
  const uint32_t a_off = slot_a * HG * slot_f;
  for (uint32_t c0 = ca + w; c0 <= cb; c0 += SB * WS) {
    float mv[SB], lv[SB];
    float av[SB][VW];
#pragma unroll
    for (int j = 0; j < SB; ++j) {
      const uint32_t c = c0 + j * WS;
      const bool valid = c <= cb;
      const float* pp = pbase + (c * cstride + (c == ca ? a_off : 0u));
      const float2 ml = valid ? __ldcg(reinterpret_cast<const float2*>(pp) + q) : make_float2(-INFINITY, 0.f);
      mv[j] = ml.x;
      lv[j] = ml.y;
      const float* pa = pp + hdr + q * kD + d0;
      if constexpr (VW == 4) {
        const float4 x = valid ? __ldcg(reinterpret_cast<const float4*>(pa)) : make_float4(0.f, 0.f, 0.f, 0.f);
        av[j][0] = x.x; av[j][1] = x.y; av[j][2] = x.z; av[j][3] = x.w;
      } else if constexpr (VW == 2) {
        const float2 x = valid ? __ldcg(reinterpret_cast<const float2*>(pa)) : make_float2(0.f, 0.f);
        av[j][0] = x.x; av[j][1] = x.y;
      } else {
        av[j][0] = valid ? __ldcg(pa) : 0.f;
      }
    }
    float Mb = M;
#pragma unroll
    for (int j = 0; j < SB; ++j) Mb = fmaxf(Mb, mv[j]);
    const float a = M == -INFINITY ? 0.f : ex2(M - Mb);
    L *= a;
#pragma unroll
    for (int v = 0; v < VW; ++v) o[v] *= a;
#pragma unroll
    for (int j = 0; j < SB; ++j) {
      const float f = mv[j] == -INFINITY ? 0.f : ex2(mv[j] - Mb);
      L += f * lv[j];
#pragma unroll
      for (int v = 0; v < VW; ++v) o[v] += f * av[j][v];
    }
    M = Mb;
  }
  if (WS > 1) {
    float* s_m = reinterpret_cast<float*>(msm + G * WS * 32);
    float* s_l = s_m + G * WS;
    s_m[warp] = M;
    s_l[warp] = L;
    float* mo = reinterpret_cast<float*>(msm + warp * 32 + lane);
#pragma unroll
    for (int v = 0; v < VW; ++v) mo[v] = o[v];
    __syncthreads();
    if (w != 0) return;
    float Mq = -INFINITY;
    for (uint32_t i = 0; i < WS; ++i) Mq = fmaxf(Mq, s_m[warp + i]);
    float Lq = 0.f;
    float oq[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) oq[v] = 0.f;
    for (uint32_t i = 0; i < WS; ++i) {
      const float mi = s_m[warp + i];
      const float f = mi == -INFINITY ? 0.f : ex2(mi - Mq);
      Lq += f * s_l[warp + i];
      const float* vi = reinterpret_cast<const float*>(msm + (warp + i) * 32 + lane);
#pragma unroll
      for (int v = 0; v < VW; ++v) oq[v] += f * vi[v];
    }
    M = Mq;
    L = Lq;
#pragma unroll
    for (int v = 0; v < VW; ++v) o[v] = oq[v];
  }
  const uint32_t Hq = p.H * G;
  const float inv = 1.f / L;
  __half* orow = p.out + (static_cast<uint64_t>(s) * Hq + h * G + q) * kD + d0;
  if constexpr (VW == 1) {
    *orow = __float2half_rn(o[0] * inv);
  } else {
#pragma unroll
    for (int v = 0; v < VW; v += 2)
      *reinterpret_cast<__half2*>(orow + v) = __floats2half2_rn(o[v] * inv, o[v + 1] * inv);
  }
  if (p.lse && lane == 0 && dc == 0)
    p.lse[static_cast<uint64_t>(s) * Hq + h * G + q] = (M + __log2f(L)) * 0.69314718055994531f;
  if (kProbes && p.trace && lane == 0) {
    const uint64_t te = gtimer();
    atomicMax(p.trace + 2049, static_cast<unsigned long long>(te));
    p.trace[2052 + 3 * blockIdx.x] = te;
  }
}

// Probe stamps (p.trace only): per CTA, the time the producer issues stage k
// (k < 32) and the time consumer warp 0 sees it full.
constexpr uint32_t kTrStage = 12288, kTrReady = kTrStage + 148 * 4 * 32;
// Compiled in only with -DKVSLAB_STAGE_PROBES (scripts/probe_stages.py): the
// per-block checks cost the consumer loop ~1 % even when p.trace is null.
__device__ __forceinline__ void trace_ready(const DecodeParams& p, int warp, int lane, uint32_t k) {
#ifdef KVSLAB_STAGE_PROBES
  if (kProbes && p.trace && warp == 0 && lane == 0 && k < 32) p.trace[kTrReady + blockIdx.x * 32 + k] = gtimer();
#else
  (void)p, (void)warp, (void)lane, (void)k;
#endif
}

// Formats whose consumer step runs two full blocks at a time (measured per format
// with scripts/microbench_consumer.cu and in the kernel).
template <int FMT, int NT, int PK>
constexpr bool kPairs = NT == 1 && (PK != 0 || FMT != kFP16);  // FP16 unpacked: no gain, spills
// PK = 2: the packed step with the integer QK (attend_iq; INT8/INT4 only)
template <int FMT, int PK>
constexpr bool kIQ = PK == 2 && (FMT == kINT8 || FMT == kINT4);

// ------------------------------------------------------------------ kernel
// CTA = HG consumer warps (one KV head each, a head group) + 1 producer warp.
// Work = the flattened list of (sequence, head group, block) cut into one
// equal contiguous range per CTA of a persistent grid (stream-K: ragged
// contexts balance exactly).  The producer streams each block's K, V and
// params for the whole head group with ONE bulk copy each (they are
// contiguous in the layer sub-block) into a shared STAGES-deep ring
// (full/empty mbarriers), and the group's Q rows into a ping-pong Q buffer at
// each unit start.  Every consumer warp runs the tensor-core online softmax
// for its head; a (sequence, head) cut by a CTA-range boundary leaves an fp32
// partial that merge_kernel (the PDL-launched successor) combines.
// <= 152 registers for the 9-warp CTA: three warps on one SM sub-partition
// then leave room for a merge warp (<= 56 registers) of a co-resident merge CTA
// PK: packed step for G <= 4 (1: attend_pk, 2: attend_iq -- IMMA QK for the
// integer formats): tile columns 0-3 and 4-7 attend alternate blocks of the
// segment, folded at the segment end.
template <int FMT, int NT, int PK>
__global__ void __maxnreg__(NT == 1 ? 152 : 255) paged_decode_kernel(const DecodeParams p) {
  using Gm = Geo<FMT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t HG = p.hg, NG = p.H / p.hg, S = p.stages;
  // PDL contract: before griddepcontrol.wait this kernel reads only data no
  // PDL-enabled predecessor writes (ctx_lens, block tables, KV of other
  // layers); Q, new K/V, outputs and the workspace come after the wait.
  pdl_launch_dependents();
  const uint64_t t0 = (kProbes && p.trace) ? gtimer() : 0;

  // ---- per-CTA prefix of blocks over sequences (x NG head groups) ----
  uint32_t* pre = reinterpret_cast<uint32_t*>(smem + p.prefix_offset);
  __shared__ uint32_t wsum[9];
  {
    const uint32_t nthr = blockDim.x, per = (p.batch + nthr - 1) / nthr;
    const uint32_t b0 = min(p.batch, threadIdx.x * per), b1 = min(p.batch, b0 + per);
    uint32_t sum = 0;
    for (uint32_t s = b0; s < b1; ++s) {
      const int c = p.ctx_lens[s];
      sum += c > 0 ? (static_cast<uint32_t>(c) + kTPB - 1) / kTPB : 0;
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += wsum[w];
    uint32_t run = wbase + incl - sum;
    for (uint32_t s = b0; s < b1; ++s) {
      pre[s] = run * NG;
      const int c = p.ctx_lens[s];
      run += c > 0 ? (static_cast<uint32_t>(c) + kTPB - 1) / kTPB : 0;
    }
    if (threadIdx.x == nthr - 1) pre[p.batch] = run * NG;
  }
  // barriers: full[S], empty[S], qfull[2], qempty[2]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_offset);
  uint64_t* empty = full + S;
  uint64_t* qfull = empty + S;
  uint64_t* qempty = qfull + 2;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], HG);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], HG);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t total = pre[p.batch];

  // Sequences with no context (empty slots of a fixed-size batch) get zero
  // outputs and -inf LSE, after the predecessor finished: spread over the
  // grid, one sequence per CTA at a time, 16-byte stores by the whole CTA
  // (one thread per sequence writing 2-byte zeros made a 64-slot batch with
  // 8 live sequences 10x slower).
  {
    bool waited = false;
    const uint32_t hq = p.H * p.G;
    const bool v16 = (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
    for (uint32_t s = blockIdx.x; s < p.batch; s += gridDim.x) {
      if (pre[s + 1] != pre[s]) continue;  // uniform: pre is in shared memory
      if (!waited) {
        pdl_wait();
        waited = true;
      }
      __half* orow = p.out + static_cast<uint64_t>(s) * hq * kD;
      if (v16) {
        for (uint32_t i = threadIdx.x; i < hq * kD / 8; i += blockDim.x)
          reinterpret_cast<uint4*>(orow)[i] = make_uint4(0u, 0u, 0u, 0u);
      } else {
        for (uint32_t i = threadIdx.x; i < hq * kD; i += blockDim.x) orow[i] = __float2half(0.f);
      }
      if (p.lse)
        for (uint32_t i = threadIdx.x; i < hq; i += blockDim.x) p.lse[static_cast<uint64_t>(s) * hq + i] = -INFINITY;
    }
  }

  // small launches use fewer CTAs (>= kMinBlocksPerCta blocks each) so a unit
  // is not cut into more partials than the work justifies
  const uint32_t C = effective_ctas(total, gridDim.x, p.batch * NG, p.min_blocks);
  if (blockIdx.x >= C) return;  // uniform across the CTA
  const CtaSplit sp = make_split(total, C);
  const uint32_t cs = cta_start(blockIdx.x, sp), ce = cta_start(blockIdx.x + 1, sp);
  if (cs >= ce) return;  // uniform across the CTA
  const uint32_t n = ce - cs;
  const uint32_t Hq = p.H * p.G;
  const uint32_t kvq = HG * Gm::kChunk;          // bytes of the group's K (or V) chunks
  const uint32_t pq = HG * Gm::kParam;           // bytes of the group's K (or V) params
  const uint32_t qbytes = HG * p.G * kD * 2;
  // a Q slot also carries the group's new K/V rows when the step appends
  const uint32_t nbytes = HG * kD * 2;
  const uint32_t qslot = qbytes + (p.k_new != nullptr ? 2 * nbytes : 0u);
  uint64_t* meta = reinterpret_cast<uint64_t*>(smem + p.bar_offset) + 2 * S + 4;  // [S] stage block address
  uint8_t* ring = smem;
  uint8_t* qbuf = smem + p.qbuf_offset;

  const bool compute_only = kProbes && (p.debug & 4) != 0;  // probe: no copies; consumers reuse stage data
  if (warp == static_cast<int>(HG)) {
    if (compute_only) return;
    // ============================ producer warp ============================
    // Per-block work is precomputed 32 blocks at a time, one block per lane
    // (cursor, block-table entry, slab address, unit start), so each stage
    // costs a few shuffles and one bulk copy when the head group spans all
    // kv heads (K, V and params of a layer sub-block are contiguous), else
    // four.
    const uint64_t pol = policy_evict_first();
    const bool one_copy = HG == p.H;
    const uint32_t stage_tx = 2 * kvq + 2 * pq;
    struct Win {
      uint64_t src;  // K of head g0 in the block's layer sub-block (g0 = 0 if one_copy)
      uint32_t g0;   // first head of the group; bit 31: the segment it opens holds the unit's last block
      int32_t qrow;  // first Q row of the unit if the block opens a unit segment, else -1
    };
    auto load_window = [&](uint32_t base) -> Win {
      Win w{0, 0, -1};
      if (base + lane < n) {
        Cursor c;
        cursor_seek(c, pre, p.batch, NG, cs + base + lane);
        const int32_t ent = __ldg(p.block_table + static_cast<uint64_t>(c.s) * p.bt_stride + c.b);
        w.g0 = c.h * HG;
        w.src = reinterpret_cast<uint64_t>(p.pool) + block_offset(p.geom, static_cast<uint32_t>(ent)) +
                p.layer_off + static_cast<uint64_t>(w.g0) * Gm::kChunk;
        if (c.b == 0 || base + lane == 0) {
          w.qrow = static_cast<int32_t>(c.s * Hq + w.g0 * p.G);
          if (n - (base + lane) >= c.nblk - c.b) w.g0 |= 0x80000000u;
        }
      }
      return w;
    };
    Win win0 = load_window(0);
    Win win1 = n > 32 ? load_window(32) : Win{0, 0, -1};
    bool dep_ready = false;
    uint32_t ui = 0, st = 0, ph = 0;
    uint64_t t_first = 0;
    const uint32_t ring_u = smem_u32(ring);
    for (uint32_t k = 0; k < n; ++k) {
      if (kProbes && k == 1 && p.trace) t_first = gtimer();
      if ((k & 31) == 0 && k > 0 && k + 32 < n) {
        if ((k >> 5) & 1) win0 = load_window(k + 32);
        else win1 = load_window(k + 32);
      }
      const Win& w = ((k >> 5) & 1) ? win1 : win0;
      const uint32_t j = k & 31;
      const uint64_t src = (static_cast<uint64_t>(__shfl_sync(0xffffffffu, static_cast<uint32_t>(w.src >> 32), j)) << 32) |
                           __shfl_sync(0xffffffffu, static_cast<uint32_t>(w.src), j);
      const int32_t qrow = __shfl_sync(0xffffffffu, w.qrow, j);
      const uint32_t gw = __shfl_sync(0xffffffffu, w.g0, j);
      const uint32_t g0 = gw & 0x7fffffffu;
      mbar_wait(&empty[st], ph ^ 1);
#ifdef KVSLAB_STAGE_PROBES
      if (kProbes && p.trace && lane == 0 && k < 32) p.trace[kTrStage + blockIdx.x * 32 + k] = gtimer();
#endif
      if (lane == 0) {
        const uint32_t sb = ring_u + st * p.stage_bytes;
        meta[st] = src - static_cast<uint64_t>(g0) * Gm::kChunk;  // layer sub-block (fused append)
        mbar_expect_tx(&full[st], stage_tx);
        const uint8_t* blk = reinterpret_cast<const uint8_t*>(src);
        if (one_copy) {
          bulk_g2s_u32(sb, blk, stage_tx, &full[st], pol);
        } else {
          bulk_g2s_u32(sb, blk, kvq, &full[st], pol);
          bulk_g2s_u32(sb + kvq, blk + static_cast<uint64_t>(p.H) * Gm::kChunk, kvq, &full[st], pol);
          if constexpr (Gm::kParam > 0) {
            const uint8_t* prm = blk + (2ull * p.H - g0) * Gm::kChunk + static_cast<uint64_t>(g0) * Gm::kParam;
            bulk_g2s_u32(sb + 2 * kvq, prm, pq, &full[st], pol);
            bulk_g2s_u32(sb + 2 * kvq + pq, prm + static_cast<uint64_t>(p.H) * Gm::kParam, pq, &full[st],
                         pol);
          }
        }
      }
      if (qrow >= 0) {
        if (!dep_ready) {  // Q comes from the predecessor
          pdl_wait();
          dep_ready = true;
        }
        if (lane == 0) {
          const uint32_t qs = ui & 1;
          const bool app = p.k_new != nullptr && (gw >> 31);
          mbar_wait(&qempty[qs], ((ui >> 1) & 1) ^ 1);
          mbar_expect_tx(&qfull[qs], qbytes + (app ? 2 * nbytes : 0u));
          uint8_t* qd = qbuf + qs * qslot;
          bulk_g2s(qd, p.q + static_cast<uint64_t>(qrow) * kD, qbytes, &qfull[qs], pol);
          if (app) {  // the new token's K and V rows of the group (fused K1)
            const uint64_t nrow = static_cast<uint64_t>(qrow / static_cast<int32_t>(Hq)) * p.H + g0;
            bulk_g2s(qd + qbytes, p.k_new + nrow * kD, nbytes, &qfull[qs], pol);
            bulk_g2s(qd + qbytes + nbytes, p.v_new + nrow * kD, nbytes, &qfull[qs], pol);
          }
        }
        ++ui;
      }
      if (++st == S) {
        st = 0;
        ph ^= 1;
      }
    }
    if (kProbes && p.trace && lane == 0) {
      unsigned long long* tr = p.trace + static_cast<uint64_t>(blockIdx.x) * 8;
      tr[0] = t0;
      tr[1] = t_first;
      tr[2] = gtimer();
      tr[3] = n;
    }
    return;
  }

  // ============================ consumer warps ============================
  // The CTA range is walked one unit segment at a time: the inner loop over
  // a segment's full blocks is just wait -> attend -> release; the unit's last
  // (partial, possibly freshly appended) block is peeled off.
  const FragOff fo = make_offsets<FMT>(g, t);
  uint32_t qf[kIQ<FMT, PK> ? 1 : NT][kIQ<FMT, PK> ? 1 : 8][2];
  uint32_t qi[4][2];
  float qsc = 0.f, qzs = 0.f;  // integer QK: query t's score scale and zero term
  UnitState<NT> us;
  float qsb[NT][2], qst[NT][2];
  float kscale = 1.f, vscale = 1.f;
  uint32_t ui = 0, st = 0, ph = 0;
  const uint32_t ring_u32 = smem_u32(ring), ring_end = ring_u32 + S * p.stage_bytes;
  uint32_t sb = ring_u32;  // shared address of stage st
  Cursor cc;
  cursor_seek(cc, pre, p.batch, NG, cs);
  const uint32_t slot_hdr = (2 * p.G + 3) & ~3u;  // (m, l)[G], padded to 16 B
  const uint32_t slot_f = slot_hdr + p.G * kD;
  const float sml2 = p.sm_scale_log2;
  const uint32_t wK = warp * Gm::kChunk, wP = 2 * kvq + warp * Gm::kParam;
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
  auto release = [&]() {
    __syncwarp();
    if (lane == 0 && !compute_only) mbar_arrive_s(empty_s + 8 * st);
    sb += p.stage_bytes;
    if (++st == S) {
      st = 0;
      ph ^= 1;
      sb = ring_u32;
    }
  };
  if (kProbes && p.trace && warp == 0 && lane == 0) p.trace[blockIdx.x * 8 + 4] = gtimer();
  const long long c_loop0 = clock64();

  for (uint32_t k = 0; k < n;) {
    const uint32_t head = cc.h * HG + warp;
    const uint32_t seg_b0 = cc.b;
    const uint32_t seg_len = min(cc.nblk - cc.b, n - k);
    const bool has_last = seg_b0 + seg_len == cc.nblk;  // holds the unit's last block
    const int ctx_cur = p.ctx_lens[cc.s];
    uint2 new_k = make_uint2(0, 0), new_v = make_uint2(0, 0);  // fused K1: this lane's 4 values
    {  // ---- unit segment start: Q fragments, state ----
      const uint32_t qs = ui & 1;
      if (!compute_only) mbar_wait(&qfull[qs], (ui >> 1) & 1);
      if constexpr (kIQ<FMT, PK>)
        load_q_iq<FMT>(smem_u32(qbuf + qs * qslot) + warp * p.G * kD * 2, g, t, p.G, sml2, qi, qsc, qzs);
      else
        load_q_frags<FMT, NT, PK != 0>(smem_u32(qbuf + qs * qslot) + warp * p.G * kD * 2, g, t, p.G, qf);
      if (p.k_new != nullptr && has_last) {  // staged with Q by the producer
        const uint32_t nk = smem_u32(qbuf + qs * qslot + qbytes) + warp * kD * 2 + lane * 8;
        new_k = lds64(nk);
        new_v = lds64(nk + nbytes);
      }
      __syncwarp();
      if (lane == 0 && !compute_only) mbar_arrive(&qempty[qs]);
      ++ui;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        if constexpr (Gm::kBiased && !kIQ<FMT, PK>) {
          // lo: k-slots 2t, 2t+1; hi: 2t+8, 2t+9 (carry 1/16 for INT4)
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
        // packed: finite so a column stream that sees no block stays NaN-free
        us.m[nt][0] = us.m[nt][1] = PK != 0 ? -1e30f : -INFINITY;
        us.l[nt][0] = us.l[nt][1] = 0.f;
        us.zb[nt][0] = us.zb[nt][1] = 0.f;
        us.zz[nt][0] = us.zz[nt][1] = 0.f;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
          us.acc[mt][nt][0] = us.acc[mt][nt][1] = us.acc[mt][nt][2] = us.acc[mt][nt][3] = 0.f;
      }
      if constexpr (FMT == kFP8) {
        if (p.kv_scales) {
          kscale = p.kv_scales[head];
          vscale = p.kv_scales[p.H + head];
        }
      }
    }
    // fused K1: the new token lands in the unit's last block; fetch its K/V
    // row now so the load latency is hidden behind the full blocks
    const bool app = p.k_new != nullptr && has_last;

    // ---- full blocks: all 16 tokens valid ----
    const uint32_t nfull = seg_len - (has_last ? 1u : 0u);
    // packed: each column stream sees every other block, so twice the blocks
    // between flushes keep the same per-stream bias bound
    constexpr uint32_t kFlush = PK ? 2 * kBiasFlush : kBiasFlush;
    uint32_t i = 0;
    if constexpr (kPairs<FMT, NT, PK>) {
      // two full blocks per step: two independent score tiles, one softmax
      // update (INT4: the dequant-heavy step gains from the extra ILP)
      for (; i + 1 < nfull; i += 2) {
        const uint32_t sb1 = sb + p.stage_bytes == ring_end ? ring_u32 : sb + p.stage_bytes;
        const uint32_t st1 = st + 1 == S ? 0 : st + 1, ph1 = st + 1 == S ? ph ^ 1 : ph;
        if (!compute_only) {
          mbar_wait_s(full_s + 8 * st, ph);
          mbar_wait_s(full_s + 8 * st1, ph1);
        }
        trace_ready(p, warp, lane, k + i);
        trace_ready(p, warp, lane, k + i + 1);
        const uint32_t sbs[2] = {sb, sb1};
        const int valid[2] = {kTPB, kTPB};
        if constexpr (kIQ<FMT, PK>)
          attend_iq<FMT, 2, false>(us, sbs, valid, wK, wP, kvq, pq, fo, qi, qsc, qzs, g, t);
        else if constexpr (PK != 0)
          attend_pk<FMT, 2, false>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, kscale, sml2, g, t);
        else
          attend<FMT, NT, 2, false>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, kscale, sml2, g, t);
        release();
        release();
        if ((i % kFlush) == kFlush - 2) {  // every kFlush blocks
          if constexpr (kIQ<FMT, PK>) flush_bias_iq<FMT>(us, g, t);
          else flush_bias<FMT, NT>(us);
        }
      }
    }
    for (; i < nfull; ++i) {
      if (!compute_only) mbar_wait_s(full_s + 8 * st, ph);
      trace_ready(p, warp, lane, k + i);
      if constexpr (PK != 0) {
        const uint32_t sbs[2] = {sb, sb};
        const int valid[2] = {kTPB, 0};
        if constexpr (kIQ<FMT, PK>)
          attend_iq<FMT, 1, false>(us, sbs, valid, wK, wP, kvq, pq, fo, qi, qsc, qzs, g, t);
        else
          attend_pk<FMT, 1, false>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, kscale, sml2, g, t);
      } else {
        const uint32_t sbs[1] = {sb};
        const int valid[1] = {kTPB};
        if (!kProbes || !(p.debug & 8))  // probe: stream only
          attend<FMT, NT, 1, false>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, kscale, sml2, g, t);
      }
      release();
      if (i % kFlush == kFlush - 1) {
        if constexpr (kIQ<FMT, PK>) flush_bias_iq<FMT>(us, g, t);
        else flush_bias<FMT, NT>(us);
      }
    }
    // ---- the unit's last block (partial; holds the appended token) ----
    if (has_last) {
      if (!compute_only) mbar_wait_s(full_s + 8 * st, ph);
      trace_ready(p, warp, lane, k + nfull);
      if (app) {
        // Fused K1: the block holding the new token (position ctx-1) was
        // copied before the token existed.  Quantise it once (quant_row,
        // bit-identical to K1), write it to its slab block in HBM, and patch
        // the staged copy so this step's attention includes it.
        uint8_t* gblk = reinterpret_cast<uint8_t*>(meta[st]);  // the block's layer sub-block
        const uint32_t slot = static_cast<uint32_t>(ctx_cur - 1) % kTPB;
        const float sck = (FMT == kFP8 && p.kv_scales) ? kscale : 1.0f;
        const float scv = (FMT == kFP8 && p.kv_scales) ? vscale : 1.0f;
        const QRow rk = quant_row<FMT>(new_k, sck), rv = quant_row<FMT>(new_v, scv);
        put_row<FMT>(gblk + static_cast<uint64_t>(head) * Gm::kChunk, gblk + p.params_off, slot, 0, head,
                     p.H, kTPB, rk, sck, p.fp8_inblock, lane);
        put_row<FMT>(gblk + static_cast<uint64_t>(p.H + head) * Gm::kChunk, gblk + p.params_off, slot, 1,
                     head, p.H, kTPB, rv, scv, p.fp8_inblock, lane);
        uint8_t* sst = ring + (sb - ring_u32);
        uint8_t* sprm = sst + 2 * kvq;  // [K params x HG][V params x HG]
        put_row<FMT>(sst + warp * Gm::kChunk, sprm, slot, 0, warp, HG, kTPB, rk, sck, false, lane);
        put_row<FMT>(sst + kvq + warp * Gm::kChunk, sprm, slot, 1, warp, HG, kTPB, rv, scv, false, lane);
        __syncwarp();
      }
      const int vlast = ctx_cur - static_cast<int>(cc.nblk - 1) * kTPB;
      if constexpr (PK != 0) {
        const uint32_t sbs[2] = {sb, sb};
        const int valid[2] = {vlast, 0};
        if constexpr (kIQ<FMT, PK>)
          attend_iq<FMT, 1, true>(us, sbs, valid, wK, wP, kvq, pq, fo, qi, qsc, qzs, g, t);
        else
          attend_pk<FMT, 1, true>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, kscale, sml2, g, t);
      } else {
        const uint32_t sbs[1] = {sb};
        const int valid[1] = {vlast};
        attend<FMT, NT, 1, true>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, kscale, sml2, g, t);
      }
      release();
    }
    if constexpr (kIQ<FMT, PK>) iq_state_to_acc(us, g, t);
    if constexpr (PK != 0) fold_halves(us);
    const bool first_seg = k == 0;  // the segment opens this CTA's range
    k += seg_len;
    cc.b = seg_b0 + seg_len - 1;  // last block consumed

    // ---- end of the unit segment: output or fp32 partial ----
    {
      const bool whole = (seg_b0 == 0) && has_last;
      float lf[NT][2], zbf[NT][2], zzf[NT][2];
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
          lf[nt][c] = l;
          zbf[nt][c] = zb;
          zzf[nt][c] = zz;
        }
      // O rows g (lo) and g+8 (hi) of m-tile mt for query column c, unnormalised
      auto o_lo = [&](int mt, int nt, int c) {
        // kIQ INT4: row g carried the whole byte (load_v_frags_iq)
        if constexpr (kIQ<FMT, PK> && FMT == kINT4) return us.acc[mt][nt][c] - us.acc[mt][nt][2 + c] + zzf[nt][c];
        return us.acc[mt][nt][c] * vscale + zbf[nt][c] + zzf[nt][c];
      };
      auto o_hi = [&](int mt, int nt, int c) {
        if constexpr (FMT == kINT4) return (us.acc[mt][nt][2 + c] + zbf[nt][c]) * 0.0625f + zzf[nt][c];
        else return us.acc[mt][nt][2 + c] * vscale + zbf[nt][c] + zzf[nt][c];
      };
      // Vector stores: a lane's O values of one query column are the
      // contiguous dims vdim(mt, g, r8) -- m-tiles 4h..4h+3 form 8 dims (one
      // 16-byte fp16 store), m-tiles 2j, 2j+1 four (one 16-byte fp32 piece).
      // After fold_halves (PK) lanes t and t^2 hold the same two columns, so
      // each writes half of them and all 32 lanes store (the STG.64 form cost
      // ~1 us per segment end at B16: 16 scattered stores per active lane).
      auto half_run = [&](int nt, int c, int h, float inv) {
        auto w = [&](int k) { return pack_h2(o_lo(4 * h + k, nt, c) * inv, o_hi(4 * h + k, nt, c) * inv); };
        return make_uint4(w(0), w(1), w(2), w(3));
      };
      auto piece = [&](int nt, int c, int j) {
        return make_float4(o_lo(2 * j, nt, c), o_hi(2 * j, nt, c), o_lo(2 * j + 1, nt, c), o_hi(2 * j + 1, nt, c));
      };
      if (whole) {
        if constexpr (PK != 0) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int q = 2 * (t & 1) + c, h = t >> 1;
            if (q >= static_cast<int>(p.G)) continue;
            const float inv = 1.f / lf[0][c];
            __half* orow = p.out + (static_cast<uint64_t>(cc.s) * Hq + head * p.G + q) * kD;
            const uint4 r0 = half_run(0, c, 0, inv), r1 = half_run(0, c, 1, inv);  // static indices
            *reinterpret_cast<uint4*>(orow + vdim<FMT>(4 * h, g, 0)) =
                h ? r1 : r0;
            if (p.lse && g == 0 && t < 2)
              p.lse[static_cast<uint64_t>(cc.s) * Hq + head * p.G + q] =
                  (us.m[0][c] + __log2f(lf[0][c])) * 0.69314718055994531f;
          }
        } else {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int q = nt * 8 + 2 * t + c;
              if (q >= static_cast<int>(p.G)) continue;
              const float inv = 1.f / lf[nt][c];
              __half* orow = p.out + (static_cast<uint64_t>(cc.s) * Hq + head * p.G + q) * kD;
#pragma unroll
              for (int h = 0; h < 2; ++h)
                *reinterpret_cast<uint4*>(orow + vdim<FMT>(4 * h, g, 0)) = half_run(nt, c, h, inv);
              if (p.lse && g == 0)
                p.lse[static_cast<uint64_t>(cc.s) * Hq + head * p.G + q] =
                    (us.m[nt][c] + __log2f(lf[nt][c])) * 0.69314718055994531f;
            }
        }
      } else {
        // partial slot: (2*cta + [0 first | 1 last segment of the CTA]) * HG + warp
        float* ps = p.partials + ((2ull * blockIdx.x + (first_seg ? 0 : 1)) * HG + warp) * slot_f;
        if constexpr (PK != 0) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int q = 2 * (t & 1) + c;
            if (q >= static_cast<int>(p.G)) continue;
            if (g == 0 && t < 2) *reinterpret_cast<float2*>(ps + 2 * q) = make_float2(us.m[0][c], lf[0][c]);
            // pieces 2i + (t >> 1): lanes t, t^2 fill adjacent 16 bytes (one 32-byte sector)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int j = 2 * i + (t >> 1);
              const float4 a0 = piece(0, c, 2 * i), a1 = piece(0, c, 2 * i + 1);  // static indices
              *reinterpret_cast<float4*>(ps + slot_hdr + q * kD + vdim<FMT>(2 * j, g, 0)) = (t >> 1) ? a1 : a0;
            }
          }
        } else {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int q = nt * 8 + 2 * t + c;
              if (q >= static_cast<int>(p.G)) continue;
              if (g == 0) *reinterpret_cast<float2*>(ps + 2 * q) = make_float2(us.m[nt][c], lf[nt][c]);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<float4*>(ps + slot_hdr + q * kD + vdim<FMT>(2 * j, g, 0)) = piece(nt, c, j);
            }
        }
      }
    }
    cursor_next(cc, pre, p.batch, NG);
  }
  if (kProbes && p.trace && warp == 0 && lane == 0) {
    p.trace[blockIdx.x * 8 + 5] = gtimer();
    p.trace[blockIdx.x * 8 + 6] = static_cast<unsigned long long>(clock64() - c_loop0);
    p.trace[blockIdx.x * 8 + 7] = n;
  }
}

// Ring depth per format: ~150-200 KB in flight per SM with one CTA (HG
// consumer warps + a producer) per SM.
template <int FMT, int NT, int PK>
static cudaError_t launch_fmt(const DecodeParams& p0, int num_sms, cudaStream_t stream) {
  using Gm = Geo<FMT>;
  DecodeParams p = p0;
  // (INT8 with head groups of 4 and two CTAs per SM measured 1-6 % faster
  // alone but 6 % slower co-located in BASELINE configs[3]: not used)
  uint32_t hg_max = NT == 1 ? 8 : 4;
  if (p.hg_max > 0) hg_max = p.hg_max < (NT == 1 ? 8u : 4u) ? p.hg_max : (NT == 1 ? 8u : 4u);
  uint32_t hg = 1;
  while (hg * 2 <= hg_max && p.H % (hg * 2) == 0) hg *= 2;
  p.hg = hg;
  p.stage_bytes = (2 * hg * (Gm::kChunk + Gm::kParam) + 127) / 128 * 128;
  const uint32_t qbytes = hg * p.G * kD * 2 + (p.k_new != nullptr ? 2 * hg * kD * 2 : 0);  // Q slot
  const size_t budget = p.smem_budget > 0 ? p.smem_budget
                                          : 220 * 1024 - (p.batch + 1) * 4 - 2 * qbytes - 512;
  uint32_t stages = static_cast<uint32_t>(budget / p.stage_bytes);
  if (stages > 16) stages = 16;
  if (stages < 2) stages = 2;
  p.stages = stages;
  p.qbuf_offset = stages * p.stage_bytes;
  p.bar_offset = (p.qbuf_offset + 2 * qbytes + 15) / 16 * 16;
  p.prefix_offset = p.bar_offset + (2 * stages + 4) * 8 + stages * 8;  // + stage block addresses
  const size_t smem = p.prefix_offset + (p.batch + 1) * 4;
  auto kern = paged_decode_kernel<FMT, NT, PK>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int threads = static_cast<int>((hg + 1) * 32);
  int per_sm = 0;
  e = cached_occupancy(reinterpret_cast<const void*>(kern), threads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  if (per_sm > 4) per_sm = 4;  // workspace partials are sized for <= 4 CTAs per SM
  int grid = per_sm * num_sms;
  // FP16 is HBM-bound with consumers to spare: 3/4 of the SMs still saturate
  // HBM (~62 GB/s per SM of TMA issue), and the free quarter lets the next
  // launch's CTAs start, read their tables and prefetch their rings while this
  // one drains and merges (scripts/ab_decode.py, 8-layer graphs: 3-7 % faster
  // at every shape measured, B=1..64, ctx 2k..32k).  The quantised formats are
  // consumer-limited at large batch and keep every SM.
  if (FMT == kFP16 && p.max_ctas == 0) grid = std::max(1, grid * 3 / 4);
  // FP8 is consumer-limited at large batch and keeps every SM, but its short
  // launches gain from the same hand-over (B16 ctx 2k 19.0 -> 18.3 us, B4 ctx
  // 8k 19.2 -> 18.4; INT8/INT4, whose consumers are slower, lose 5-15 % at
  // B8-16 and keep the full grid).  The launch itself must be smaller -- an
  // in-kernel early exit of the extra CTAs measured no gain: every launched
  // CTA has to be resident before the next launch may start.  The host only
  // knows the table bound batch x bt_stride (an overestimate keeps the full grid).
  if (FMT == kFP8 && p.max_ctas == 0 &&
      static_cast<uint64_t>(p.batch) * p.bt_stride * (p.H / hg) < static_cast<uint64_t>(grid) * 24)
    grid = std::max(1, grid * 3 / 4);
  // a model's SM share (ks_set_decode_sm_share) caps the SMs its grid may
  // cover: per_sm CTAs on each
  if (p.max_ctas > 0 && grid > p.max_ctas * per_sm) grid = p.max_ctas * per_sm;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p);
  if (e != cudaSuccess) return e;
  // merge the partials of units cut by CTA ranges (early-exits otherwise).
  // Warps per query from the expected segments per unit (about grid / units,
  // +1), SB = 4 loads in flight per warp; <= 128 threads (one warp per SM
  // sub-partition) by default so a merge CTA fits beside a decode CTA.
  const uint32_t units = p.batch * (p.H / hg);
  const uint32_t segs = (static_cast<uint32_t>(grid) + units - 1) / units + 1;
  // Many merge CTAs (>= 64): <= 128 threads each, so they co-reside with the
  // decode CTAs.  Few (small batch, long context: many segments per unit):
  // up to 1024 threads, so each warp merges <= 2 batches of SB segments.
  const uint32_t mt = p.merge_threads ? p.merge_threads : (p.batch * p.H >= 64 ? 128u : 1024u);
  uint32_t ws = 1;
  while (ws < 32 && ws * 4 * 2 < segs && p.G * 32 * ws * 2 <= mt) ws *= 2;
  // and few (sequence, head) merges are spread over DC CTAs each (dims split)
  const uint32_t heads = p.batch * p.H;
  int DC = heads >= 64 ? 1 : (heads >= 32 ? 2 : 4);
  if (p.merge_dc == 1 || p.merge_dc == 2 || p.merge_dc == 4) DC = static_cast<int>(p.merge_dc);  // probe override
  cudaLaunchConfig_t mcfg = cfg;
  mcfg.gridDim = dim3(heads * DC);
  mcfg.blockDim = dim3(p.G * 32 * ws);
  mcfg.dynamicSmemBytes = ws > 1 ? p.G * ws * (32 * 16 + 8) : 0;
  const uint32_t g32 = static_cast<uint32_t>(grid);
  if (DC == 1) return cudaLaunchKernelEx(&mcfg, merge_kernel<1>, p, ws, g32);
  if (DC == 2) return cudaLaunchKernelEx(&mcfg, merge_kernel<2>, p, ws, g32);
  return cudaLaunchKernelEx(&mcfg, merge_kernel<4>, p, ws, g32);
}

}  // namespace dev

cudaError_t launch_paged_decode(const DecodeParams& p, int kv_dtype, int num_sms,
                                cudaStream_t stream) {
  using namespace dev;
  const bool two = p.G > 8;
  // packed G <= 4 step.  Default (pack_mode 0): the integer-QK packed step
  // (attend_iq) for INT4 -- B64 ctx 4k 62.8 -> 57.1 us, B64 ctx 1300 28.4 ->
  // 27.0 against the packed HMMA step -- and the plain step for the rest:
  // INT8 on attend_iq measured neutral at B64 (HBM-bound) and 0.4 us slower at
  // B16 (the per-segment Q split), packed HMMA neutral at large batch and
  // ~0.5 us slower at B16 for FP8/INT8, neutral for FP16.  A/B switches:
  // pack_mode 1 plain everywhere; 2 packed HMMA for every format; 3 packed
  // HMMA for INT4 only (the previous default); 4 attend_iq for INT8 and INT4.
  const bool small_g = p.G <= 4;
  const bool integer = kv_dtype == kINT8 || kv_dtype == kINT4;
  const int pk = !small_g || p.pack_mode == 1 ? 0
                 : p.pack_mode == 0           ? (kv_dtype == kINT4 ? 2 : 0)
                 : p.pack_mode == 2           ? 1
                 : p.pack_mode == 3           ? (kv_dtype == kINT4 ? 1 : 0)
                                              : (integer ? 2 : 0);
#define KVSLAB_DECODE_CASE(F)                                          \
  case F:                                                              \
    if (two) return launch_fmt<F, 2, 0>(p, num_sms, stream);           \
    if (pk == 1) return launch_fmt<F, 1, 1>(p, num_sms, stream);       \
    if constexpr (F == kINT8 || F == kINT4)                            \
      if (pk == 2) return launch_fmt<F, 1, 2>(p, num_sms, stream);     \
    return launch_fmt<F, 1, 0>(p, num_sms, stream);
  switch (kv_dtype) {
    KVSLAB_DECODE_CASE(kFP16)
    KVSLAB_DECODE_CASE(kFP8)
    KVSLAB_DECODE_CASE(kINT8)
    KVSLAB_DECODE_CASE(kINT4)
    default: return cudaErrorInvalidValue;
  }
#undef KVSLAB_DECODE_CASE
}

size_t decode_partials_bytes(int num_sms, int G) {
  // <= 4 CTAs per SM (smem) x 2 segments x (group heads x G) <= 64 query rows
  (void)G;
  const size_t ctas = static_cast<size_t>(num_sms) * 4;
  return ctas * 2 * 64 * (dev::kD + 4) * sizeof(float);
}

}  // namespace kvslab
