// prefill_tc.cu -- K4 on the 5th-generation tensor cores (tcgen05 / TMEM),
// FP16 KV.  Same contract and oracle as prefill.cu (orc_paged_prefill, 1e-3).
//
// One CTA (4 warps) per (sequence, kv head, tile of 128 query rows = 128/G
// tokens x the G query heads).  The rows are the M=128 operand of UMMA:
//   S[128 x 64]  = Q[128 x 128] . K_t^T           (8 x tcgen05.mma K=16, TMEM)
//   O[128 x 128] += P[128 x 64] . V_t[64 x 128]   (4 x tcgen05.mma K=16, TMEM)
// per KV tile t of 64 tokens (4 slab blocks).  Thread r owns query row r: it
// reads its S row from TMEM (tcgen05.ld 32x32b), runs the online softmax with
// no shuffles (lazy rescale: O is rescaled in TMEM only when the row max grows
// by more than 2^8), and writes its P row into shared memory.  Operands live
// in shared memory in the UMMA canonical 128-byte-swizzled layouts (Q, K, P
// K-major; V token-major = MN-major B), so the slab chunk's own swizzled rows
// are re-laid out by the cp.async copies themselves:
// each 16-byte granule goes from its slab position straight to its operand
// position, double-buffered one tile ahead.  Blocks past the sequence are
// zero-filled.  Thread 0 issues the MMAs; tcgen05.commit signals mbarriers.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "attend.cuh"
#include "kvslab_device.cuh"
#include "func_cache.hpp"
#include "launch.hpp"

namespace kvslab {
namespace dev {
namespace tc {

constexpr uint32_t kRows = 128;   // UMMA M: query rows per CTA
constexpr uint32_t kTile = 64;    // KV tokens per tile (UMMA N of S, K of PV)
constexpr uint32_t kThreads = 128;
// shared memory map (1024-aligned): Q | K[2] | V[2] | P
constexpr uint32_t kQ = 0, kQBytes = kRows * kD * 2;                // 32 KB
constexpr uint32_t kK = kQ + kQBytes, kKVBytes = kTile * kD * 2;     // 16 KB each
constexpr uint32_t kV = kK + 2 * kKVBytes;
constexpr uint32_t kP = kV + 2 * kKVBytes, kPBytes = kRows * kTile * 2;  // 16 KB
constexpr uint32_t kSmem = kP + kPBytes;
constexpr uint32_t kTmemCols = 256;  // S: [0, 64), O: [64, 192)
constexpr uint32_t kTmemO = kTile;

// byte offset of element (row, k) of a K-major 128B-swizzled operand whose
// 64-element column j is a [rows][128 B] region
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t gran /*16B of the 128B row*/) {
  return row * 128 + ((gran ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (2ull << 61);  // sm100, SWIZZLE_128B
}
__device__ __forceinline__ void umma_f16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// 32 consecutive TMEM columns of this thread's lane -> registers
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

// 16 columns at a time (the O rescale runs while the 64 scores are live)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

// ---------------------------------------------------------------------------
// v2: warp-specialised, two query tiles per CTA (FA4-style ping-pong).
//   warps 0-3 / 4-7: softmax of query tile A / B (thread = row)
//   warp 8 lane 0  : MMA issuer (S_A, S_B, PV_A, PV_B in a software pipeline)
//   warps 9-11     : cp.async loaders (Q tiles, then a 3-stage K/V ring)
// While one tile's softmax runs the tensor core works on the other tile, and
// the K/V ring keeps two tiles in flight.  TMEM: S_A | S_B | O_A | O_B.
constexpr uint32_t kLoadWarp0 = 9;
// FP16 needs only Q gathers and bulk copies from its 3 loader warps (12 warps);
// the dequantising formats get 7 (16 warps, <= 128 registers; with the O
// rescale in 16-column TMEM chunks the spills are small): measured +6-14 %
// EXP: INT8/INT4 over the expand scratch -- K as exact integers and V
// dequantised, both fp16 operands as stored, so the loaders only issue bulk
// copies like FP16 (plus the tile's K scale/zero arrays)
template <int FMT, bool EXP = false>
constexpr uint32_t kLoadersOf = (FMT == kFP16 || EXP) ? 96u : 224u;
template <int FMT, bool EXP = false>
constexpr uint32_t kThreadsOf = kLoadWarp0 * 32 + kLoadersOf<FMT, EXP>;
constexpr uint32_t k2TmemCols = 512;
constexpr uint32_t kPartStride = kD + 4;  // split-KV partial per row: acc[128], m, l (+pad)
// Shared memory per format: Q (2 x 32 KB) | fp16 K/V operand ring | P (2 x
// 16 KB) | raw ring.  FP16 chunks are operands as stored (3 operand stages,
// no raw ring); FP8/INT8/INT4 chunks and their per-token params land raw
// (bulk copies, 2 stages) and the loader warps dequantise them into the
// operand ring.
template <int FMT, bool EXP = false>
struct TcCfg {
  static constexpr bool kOperands = FMT == kFP16 || EXP;  // chunks are fp16 operands as stored
  static constexpr uint32_t kStages = kOperands ? 3 : 2;
  static constexpr uint32_t kRawStages = 3;  // raw blocks land two tiles ahead of the dequant
  static constexpr uint32_t kChunk = Geo<FMT>::kChunk, kParam = Geo<FMT>::kParam;
  static constexpr uint32_t kRawBlock = 2 * kChunk + 2 * kParam;  // K, V, K params, V params
  static constexpr uint32_t kRawBytes = kOperands ? 0 : (4 * kRawBlock + 127) / 128 * 128;
  static constexpr uint32_t kQo = 0, kKV = 2 * kQBytes, kP = kKV + kStages * 2 * kKVBytes;
  static constexpr uint32_t kRaw = kP + 2 * kPBytes;
  // INT8/INT4: K enters the MMA as exact integers; its per-token scale (and
  // zero) are applied to S in fp32 from these arrays ([stage][64] x 2 floats)
  static constexpr uint32_t kSZ = kRaw + kRawStages * kRawBytes;
  static constexpr uint32_t kSmem = kSZ + kStages * kTile * 8;
};
// bulk-copy source for blocks past the sequence (a chunk half of zeros)
__device__ __align__(128) uint8_t g_zero_half[kTPB * 128];

// a row's 64 scores with one load and one wait
__device__ __forceinline__ void tmem_ld64_to(uint32_t taddr, float* v) {
  uint32_t u[64];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31]), "=r"(u[32]), "=r"(u[33]), "=r"(u[34]), "=r"(u[35]), "=r"(u[36]), "=r"(u[37]), "=r"(u[38]), "=r"(u[39]), "=r"(u[40]), "=r"(u[41]), "=r"(u[42]), "=r"(u[43]), "=r"(u[44]), "=r"(u[45]), "=r"(u[46]), "=r"(u[47]), "=r"(u[48]), "=r"(u[49]), "=r"(u[50]), "=r"(u[51]), "=r"(u[52]), "=r"(u[53]), "=r"(u[54]), "=r"(u[55]), "=r"(u[56]), "=r"(u[57]), "=r"(u[58]), "=r"(u[59]), "=r"(u[60]), "=r"(u[61]), "=r"(u[62]), "=r"(u[63])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(u[i]);
}
__device__ __forceinline__ void tmem_ld32_to(uint32_t taddr, float* v) {
  float t[32];
  tmem_ld32(taddr, t);
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = t[i];
}

// 16 raw bytes of K or V (token `tok` of block `bi`, dims d0.. of the
// format's row) -> fp16 operand granules at their swizzled tile positions.
// FP8 is converted exactly (its static per-head scale is applied in fp32 to S
// and O); INT8 / INT4 apply the token's scale (and zero) in one fp16 rounding.
template <int FMT>
__device__ __forceinline__ void dequant_granule(uint8_t* tile, uint32_t row, uint32_t d0, uint4 w, uint32_t sz,
                                                bool exact) {
  auto put = [&](uint32_t d, uint32_t a, uint32_t b, uint32_t c, uint32_t e) {  // 8 dims at d
    const uint32_t half = d >> 6, gran = (d & 63) >> 3;
    *reinterpret_cast<uint4*>(tile + half * (kTile * 128) + sw128(row, gran)) = make_uint4(a, b, c, e);
  };
  const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
  if constexpr (FMT == kFP8) {
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = e4m3x2_to_f16x2(static_cast<uint16_t>(wd[i] & 0xffff));
      o[2 * i + 1] = e4m3x2_to_f16x2(static_cast<uint16_t>(wd[i] >> 16));
    }
    put(d0, o[0], o[1], o[2], o[3]);
    put(d0 + 8, o[4], o[5], o[6], o[7]);
  } else if constexpr (FMT == kINT8) {
    // K (exact): the integer itself; V: times the token's fp16 scale
    const uint32_t s2 = exact ? 0x3C003C00u : ((sz & 0xffffu) | (sz << 16));
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t x = wd[i] ^ 0x80808080u;  // exact 1152 + b, minus 1152, times s
      o[2 * i] = hmul2_u32(hsub2_u32(__byte_perm(x, 0x64646464u, 0x4140), 0x64806480u), s2);
      o[2 * i + 1] = hmul2_u32(hsub2_u32(__byte_perm(x, 0x64646464u, 0x4342), 0x64806480u), s2);
    }
    put(d0, o[0], o[1], o[2], o[3]);
    put(d0 + 8, o[4], o[5], o[6], o[7]);
  } else {  // INT4: 32 dims, byte k = (dim 2k low nibble, dim 2k+1 high nibble)
    // K (exact): n itself, i.e. scale 1 and zero 0; V: s*n + z (one rounding)
    const uint32_t sc = exact ? 0x3C00u : (sz & 0xffffu), z = exact ? 0u : (sz >> 16);
    const uint32_t s2 = sc | (hmul2_u32(sc, 0x2C00u) << 16);  // (s, s/16): the high nibble enters as 16 n
    const uint32_t z2 = z | (z << 16);
    uint32_t o[16];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t y = __byte_perm(wd[i], 0, k | (k << 8) | (k << 16) | (k << 24));
        const uint32_t n = hsub2_u32(lop3_and_or(y, 0x00F0000Fu, 0x64006400u), 0x64006400u);
        o[4 * i + k] = hfma2_u32(n, s2, z2);
      }
    put(d0, o[0], o[1], o[2], o[3]);
    put(d0 + 8, o[4], o[5], o[6], o[7]);
    put(d0 + 16, o[8], o[9], o[10], o[11]);
    put(d0 + 24, o[12], o[13], o[14], o[15]);
  }
}

// INT4 V granule of the token-pair layout: 16 dims
// (bytes j .. j+7) of two tokens interleaved in 2-byte units,
// w = [A.j A.j+1 B.j B.j+1][A.j+2 ...]; scaled as in dequant_granule.
__device__ __forceinline__ void dequant_int4_vpair(uint8_t* tile, uint32_t row_a, uint32_t row_b, uint32_t d0,
                                                   uint4 w, uint32_t sza, uint32_t szb) {
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const uint32_t sel = side ? 0x7632u : 0x5410u, sz = side ? szb : sza;
    const uint32_t wd[2] = {__byte_perm(w.x, w.y, sel), __byte_perm(w.z, w.w, sel)};
    const uint32_t sc = sz & 0xffffu, z = sz >> 16;
    const uint32_t s2 = sc | (hmul2_u32(sc, 0x2C00u) << 16);
    const uint32_t z2 = z | (z << 16);
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t y = __byte_perm(wd[i], 0, k | (k << 8) | (k << 16) | (k << 24));
        const uint32_t n = hsub2_u32(lop3_and_or(y, 0x00F0000Fu, 0x64006400u), 0x64006400u);
        o[4 * i + k] = hfma2_u32(n, s2, z2);
      }
    const uint32_t row = side ? row_b : row_a;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t d = d0 + 8 * h, half = d >> 6, gran = (d & 63) >> 3;
      *reinterpret_cast<uint4*>(tile + half * (kTile * 128) + sw128(row, gran)) =
          make_uint4(o[4 * h], o[4 * h + 1], o[4 * h + 2], o[4 * h + 3]);
    }
  }
}

template <int FMT, bool EXP = false, bool SPLIT = false>
__global__ void __launch_bounds__(kThreadsOf<FMT, EXP>, 1) prefill_tc2_kernel(const PrefillParams p) {
  using Cfg = TcCfg<FMT, EXP>;
  constexpr uint32_t kLoaders = kLoadersOf<FMT, EXP>;
  constexpr uint32_t kStages = Cfg::kStages, k2Q = Cfg::kQo, k2KV = Cfg::kKV, k2P = Cfg::kP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t q_full, kv_full[kStages], kv_empty[kStages], s_full[2], p_full[2], pv_done[2], o_final;
  __shared__ uint64_t raw_full[Cfg::kRawStages], raw_empty[Cfg::kRawStages];
  __shared__ uint32_t tmem_base;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t s = blockIdx.x / p.H, h = blockIdx.x % p.H;
  const uint32_t G = p.G, TPC = 2 * kRows / G;  // tokens per CTA
  const uint32_t tile = p.tiles - 1 - blockIdx.y;
  const int q0 = p.cu_q[s], nq = p.cu_q[s + 1] - q0;
  const int tok0 = static_cast<int>(tile * TPC);
  if (tok0 >= nq) return;
  const int ctx = p.ctx_lens[s];
  const int pos0 = ctx - nq;
  const int tok_end = min(nq, tok0 + static_cast<int>(TPC));
  const int pos_last = pos0 + tok_end - 1;
  const uint32_t ntiles = static_cast<uint32_t>(pos_last) / kTile + 1;
  // split-KV (gridDim.z > 1; short chunks over long contexts would leave SMs
  // idle): CTA z of the query tile attends KV tiles [t0, t0 + niter) and
  // leaves an fp32 partial (acc, m, l) per row for prefill_merge_kernel
  // (a separate instantiation: the unsplit kernel keeps its exact code)
  const uint32_t nsplit = SPLIT ? gridDim.z : 1u, z = SPLIT ? blockIdx.z : 0u;
  const uint32_t t0 = SPLIT ? z * ntiles / nsplit : 0u;
  const uint32_t niter = SPLIT ? (z + 1) * ntiles / nsplit - t0 : ntiles;
  const uint32_t nblk = (static_cast<uint32_t>(ctx) + kTPB - 1) / kTPB;
  const uint32_t Hq = p.H * G;
  const uint32_t sbase = smem_u32(smem);

  if (tid == 0) {
    mbar_init(&q_full, kLoaders);
    for (uint32_t i = 0; i < kStages; ++i) {
      mbar_init(&kv_full[i], Cfg::kOperands ? 1u : kLoaders);
      mbar_init(&kv_empty[i], 1);
    }
    for (uint32_t i = 0; i < Cfg::kRawStages; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], kLoaders);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], kRows);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(&o_final, 1);
    fence_mbar_init();
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(k2TmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp >= kLoadWarp0) {
    // ============================ loaders ============================
    const uint32_t lt = tid - kLoadWarp0 * 32;
    for (uint32_t i = lt; i < 2 * kRows * 16; i += kLoaders) {
      const uint32_t x = i >> 11, rem = i & 2047, r = rem >> 4, c = rem & 15;
      const uint32_t rr = x * kRows + r;
      const int tok = tok0 + static_cast<int>(rr / G);
      const bool ok = tok < tok_end;
      const __half* src = p.q + (static_cast<uint64_t>(ok ? q0 + tok : q0) * Hq + h * G + rr % G) * kD + c * 8;
      cp_async16(sbase + k2Q + x * kQBytes + (c >> 3) * (kRows * 128) + sw128(r, c & 7), src, ok ? 16u : 0u);
    }
    cp_async_commit();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async();
    mbar_arrive(&q_full);
    if constexpr (!Cfg::kOperands) {
      // ---- raw blocks (bulk copies, one thread) -> dequantised operand tiles (96 threads) ----
      constexpr uint32_t kC = Cfg::kChunk, kPm = Cfg::kParam, kRB = Cfg::kRawBlock;
      const int32_t* bt = p.block_table + static_cast<uint64_t>(s) * p.bt_stride;
      const uint32_t raw0 = sbase + Cfg::kRaw;
      constexpr uint32_t RS = Cfg::kRawStages;
      auto issue_raw = [&](uint32_t t) {
        const uint32_t rs = t % RS;
        if (t >= RS) mbar_wait(&raw_empty[rs], ((t / RS) - 1) & 1);
        mbar_expect_tx(&raw_full[rs], 4 * kRB);
        const uint64_t pol = policy_evict_last();
        for (uint32_t bi = 0; bi < 4; ++bi) {
          const uint32_t b = (t0 + t) * 4 + bi;
          const uint32_t dst = raw0 + rs * Cfg::kRawBytes + bi * kRB;
          if (b < nblk) {
            const uint8_t* blk = p.pool + block_offset(p.geom, static_cast<uint32_t>(__ldg(bt + b))) + p.layer_off;
            bulk_g2s_u32(dst, blk + static_cast<uint64_t>(h) * kC, kC, &raw_full[rs], pol);
            bulk_g2s_u32(dst + kC, blk + static_cast<uint64_t>(p.H + h) * kC, kC, &raw_full[rs], pol);
            if constexpr (kPm > 0) {
              const uint8_t* prm = blk + 2ull * p.H * kC + static_cast<uint64_t>(h) * kPm;
              bulk_g2s_u32(dst + 2 * kC, prm, kPm, &raw_full[rs], pol);
              bulk_g2s_u32(dst + 2 * kC + kPm, prm + static_cast<uint64_t>(p.H) * kPm, kPm, &raw_full[rs], pol);
            }
          } else {  // past the sequence: zeros (scale 0 -> exact 0)
            for (uint32_t o = 0; o < kRB; o += kTPB * 128) {
              const uint32_t n = min(kTPB * 128, kRB - o);
              bulk_g2s_u32(dst + o, g_zero_half, n, &raw_full[rs], pol);
            }
          }
        }
      };
      if (lt == 0)
        for (uint32_t t = 0; t + 1 < RS && t < niter; ++t) issue_raw(t);
      constexpr uint32_t kRowB = kD * Fmt<FMT>::kBits / 8;     // raw bytes per token row
      constexpr uint32_t kGran = 2 * 4 * kC / 16;               // raw 16-byte granules per tile
      for (uint32_t t = 0; t < niter; ++t) {
        if (lt == 0 && t + RS - 1 < niter) issue_raw(t + RS - 1);
        const uint32_t rs = t % RS, st = t % kStages;
        mbar_wait(&raw_full[rs], (t / RS) & 1);
        if (t >= kStages) mbar_wait(&kv_empty[st], ((t / kStages) - 1) & 1);
        const uint8_t* raw = smem + Cfg::kRaw + rs * Cfg::kRawBytes;
        uint8_t* kt = smem + k2KV + st * 2 * kKVBytes;
#pragma unroll 4
        for (uint32_t i = lt; i < ((kProbes && (p.debug & 4)) ? 0u : kGran); i += kLoaders) {
          const uint32_t kv = i / (4 * kC / 16), rem = i % (4 * kC / 16);
          const uint32_t bi = rem / (kC / 16), gi = rem % (kC / 16);  // physical granule of the chunk
          const uint32_t off = gi * 16, line = off >> 7;
          const uint32_t lo = (off & 127) ^ ((line & 7) << 4);          // unswizzle: logical byte in the line
          const uint32_t lb = (line << 7) | lo;                          // logical byte in the chunk
          const uint32_t tok = lb / kRowB, d0 = (lb % kRowB) * 8 / Fmt<FMT>::kBits;
          const uint8_t* rb = raw + bi * kRB;
          const uint4 w = *reinterpret_cast<const uint4*>(rb + kv * kC + off);
          if constexpr (FMT == kINT4) {
            if (kv == 1) {  // token-pair line: tokens (tok_a, tok_b) [+8], 16 dims each
              const uint32_t tp = line >> 1;
              const uint32_t ta = (tp & 1) + ((tp >> 1) << 2) + 8 * (line & 1), tb = ta + 2;
              const uint8_t* pv = rb + 2 * kC + kPm;
              dequant_int4_vpair(kt + kKVBytes, bi * kTPB + ta, bi * kTPB + tb, 2 * ((lo >> 4) * 8), w,
                                 *reinterpret_cast<const uint32_t*>(pv + ta * 4),
                                 *reinterpret_cast<const uint32_t*>(pv + tb * 4));
              continue;
            }
          }
          uint32_t sz = 0;
          if constexpr (FMT == kINT8) sz = *reinterpret_cast<const uint16_t*>(rb + 2 * kC + kv * kPm + tok * 2);
          if constexpr (FMT == kINT4) sz = *reinterpret_cast<const uint32_t*>(rb + 2 * kC + kv * kPm + tok * 4);
          dequant_granule<FMT>(kt + kv * kKVBytes, bi * kTPB + tok, d0, w, sz, kv == 0 && FMT != kFP8);
        }
        if constexpr (FMT == kINT8 || FMT == kINT4) {  // K scale / zero of the tile's 64 tokens, fp32
          if (lt < kTile) {
            const uint8_t* rp = raw + (lt / kTPB) * kRB + 2 * kC + (lt % kTPB) * (FMT == kINT8 ? 2 : 4);
            float* sz = reinterpret_cast<float*>(smem + Cfg::kSZ + st * kTile * 8);
            // pre-multiplied by the softmax scale (log2 domain): S = s'*dot + z'*sum(q)
            if constexpr (FMT == kINT8) {
              sz[lt] = __half2float(*reinterpret_cast<const __half*>(rp)) * p.sm_scale_log2;
              sz[kTile + lt] = 0.f;
            } else {
              const __half2 v = *reinterpret_cast<const __half2*>(rp);
              sz[lt] = __low2float(v) * p.sm_scale_log2;
              sz[kTile + lt] = __high2float(v) * p.sm_scale_log2;
            }
          }
        }
        fence_proxy_async();
        mbar_arrive(&kv_full[st]);
        mbar_arrive(&raw_empty[rs]);
      }
    } else if (tid == kLoadWarp0 * 32) {
      // K/V: each FP16 chunk half (16 tokens x 64 dims, 2 KB) is already a
      // 128B-swizzled operand slice, so one bulk copy (TMA engine) per half
      // places it at rows 16*bi.. of the tile; 16 copies per 64-token tile
      const int32_t* bt = p.block_table + static_cast<uint64_t>(s) * p.bt_stride;
      const uint64_t pol = policy_evict_last();  // every query tile of the head re-reads them
      pdl_wait();  // launched behind expand_kernel (PDL): its scratch blocks are complete
      for (uint32_t t = 0; t < niter; ++t) {
        const uint32_t st = t % kStages;
        if (t >= kStages) mbar_wait(&kv_empty[st], ((t / kStages) - 1) & 1);
        const uint32_t kb = sbase + k2KV + st * 2 * kKVBytes;
        mbar_expect_tx(&kv_full[st], 2 * kKVBytes + (EXP ? kTile * 8 : 0u));
#pragma unroll
        for (uint32_t bi = 0; bi < 4; ++bi) {
          const uint32_t b = (t0 + t) * 4 + bi;
          // null table: the expand scratch, block b of sequence s at s * bt_stride + b
          const uint32_t gid = p.block_table ? static_cast<uint32_t>(__ldg(bt + b)) : s * p.bt_stride + b;
          const uint8_t* blk = b < nblk ? p.pool + block_offset(p.geom, gid) + p.layer_off : nullptr;
#pragma unroll
          for (uint32_t kv = 0; kv < 2; ++kv)
#pragma unroll
            for (uint32_t half = 0; half < 2; ++half) {
              const uint8_t* src = blk ? blk + static_cast<uint64_t>(kv * p.H + h) * (kTPB * kD * 2) + half * (kTPB * 128)
                                       : g_zero_half;
              bulk_g2s_u32(kb + kv * kKVBytes + half * (kTile * 128) + bi * (kTPB * 128), src, kTPB * 128,
                           &kv_full[st], pol);
            }
          if constexpr (EXP) {  // the block's 16 K scales', then 16 zeros' (fp32, x sm_scale_log2)
            const uint8_t* zs = b < nblk ? reinterpret_cast<const uint8_t*>(
                                               p.exp_sz + ((static_cast<uint64_t>(s) * p.bt_stride + b) * p.H + h) * 32)
                                         : g_zero_half;
            const uint32_t szs = sbase + Cfg::kSZ + st * kTile * 8 + bi * kTPB * 4;
            bulk_g2s_u32(szs, zs, kTPB * 4, &kv_full[st], pol);
            bulk_g2s_u32(szs + kTile * 4, zs + kTPB * 4, kTPB * 4, &kv_full[st], pol);
          }
        }
      }
    }
  } else if (warp == 8) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      const uint32_t idesc_s = (1u << 4) | ((kTile >> 3) << 17) | ((kRows >> 4) << 24);
      const uint32_t idesc_pv = (1u << 4) | (1u << 16) | ((kD >> 3) << 17) | ((kRows >> 4) << 24);
      auto mma_s = [&](uint32_t x, uint32_t st, uint32_t sb) {  // sb: S buffer (tile parity)
#pragma unroll
        for (uint32_t k = 0; k < kD / 16; ++k) {
          const uint64_t ad = umma_desc(sbase + k2Q + x * kQBytes + (k >> 2) * (kRows * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd =
              umma_desc(sbase + k2KV + st * 2 * kKVBytes + (k >> 2) * (kTile * 128) + (k & 3) * 32, 16, 1024);
          umma_f16(tmem + x * 2 * kTile + sb * kTile, ad, bd, idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[x]);
      };
      auto mma_pv = [&](uint32_t x, uint32_t st, bool first) {
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k) {
          const uint64_t ad = umma_desc(sbase + k2P + x * kPBytes + k * 32, 16, 1024);
          const uint64_t bd = umma_desc(sbase + k2KV + st * 2 * kKVBytes + kKVBytes + k * 2048, kTile * 128, 1024);
          umma_f16(tmem + 4 * kTile + x * kD, ad, bd, idesc_pv, (!first || k > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[x]);
      };
      // S is double-buffered in TMEM, so S(t+1) of a tile runs while its
      // softmax of t is still reading S(t):  S_A(t+1), PV_A(t), S_B(t+1), PV_B(t)
      mbar_wait(&q_full, 0);
      tc_fence_after();
      if (niter > 0) {
        mbar_wait(&kv_full[0], 0);
        tc_fence_after();
        mma_s(0, 0, 0);
        mma_s(1, 0, 0);
      }
      for (uint32_t t = 0; t < niter; ++t) {
        const uint32_t st = t % kStages, nst = (t + 1) % kStages;
        const bool more = t + 1 < niter;
        if (more) {  // both tiles' next S first: neither waits on the other's softmax
          mbar_wait(&kv_full[nst], ((t + 1) / kStages) & 1);
          tc_fence_after();
          mma_s(0, nst, (t + 1) & 1);  // buffer (t+1)&1 was read by softmax(t-1): p_full(t-1) waited
          mma_s(1, nst, (t + 1) & 1);
        }
        mbar_wait(&p_full[0], t & 1);
        tc_fence_after();
        mma_pv(0, st, t == 0);
        mbar_wait(&p_full[1], t & 1);
        tc_fence_after();
        mma_pv(1, st, t == 0);
        umma_commit(&kv_empty[st]);
      }
      if (niter > 0) umma_commit(&o_final);
      else mbar_arrive(&o_final);  // empty split: nothing to wait for
    }
    __syncwarp();
  } else {
    // ============================ softmax (row per thread) ============================
    const uint32_t x = warp >> 2, r = tid & (kRows - 1);
    const uint32_t rr = x * kRows + r;
    const int rtok = tok0 + static_cast<int>(rr / G);
    const bool rvalid = rtok < tok_end;
    const int rpos = rvalid ? pos0 + rtok : pos_last;
    const uint32_t lanes = ((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lanes + x * 2 * kTile, tO = tmem + lanes + 4 * kTile + x * kD;
    float sml2 = p.sm_scale_log2, oscale = 1.f;
    if constexpr (FMT == kFP8 || FMT == kFP16) {  // static per-head scales (FP8, also when expanded to fp16): K into S, V into O
      if (p.kv_scales) {
        sml2 *= p.kv_scales[h];
        oscale = p.kv_scales[p.H + h];
      }
    }
    uint8_t* prow = smem + k2P + x * kPBytes;
    float m = -INFINITY, l = 0.f, qsum = 0.f;
    for (uint32_t t = 0; t < niter; ++t) {
      mbar_wait(&s_full[x], t & 1);
      tc_fence_after();
      float sc[kTile];
      tmem_ld64_to(tS + (t & 1) * kTile, sc);
      if (kProbes && (p.debug & 2)) {
#pragma unroll
        for (int j = 0; j < static_cast<int>(kTile); ++j) sc[j] = 0.f;
      }
      const int kbase = static_cast<int>((t0 + t) * kTile);
      if constexpr (FMT == kINT8 || FMT == kINT4) {
        if (t == 0 && FMT == kINT4) {  // sum of this row's (exact fp16) query, for the zero term
          const uint8_t* qr = smem + k2Q + x * kQBytes;
          float acc = 0.f;
#pragma unroll
          for (uint32_t c = 0; c < 16; ++c) {
            const uint4 v = *reinterpret_cast<const uint4*>(qr + (c >> 3) * (kRows * 128) + sw128(r, c & 7));
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&wv[i]));
              acc += f.x + f.y;
            }
          }
          qsum = acc;
        }
        const float* sz = reinterpret_cast<const float*>(smem + Cfg::kSZ + (t % kStages) * kTile * 8);
        const float2 qs2 = make_float2(qsum, qsum);
#pragma unroll
        for (int j = 0; j < static_cast<int>(kTile); j += 4) {  // packed fp32x2, 16-byte scale loads
          const float4 a = *reinterpret_cast<const float4*>(sz + j);
          float2 lo = make_float2(sc[j], sc[j + 1]), hi = make_float2(sc[j + 2], sc[j + 3]);
          if constexpr (FMT == kINT8) {
            lo = fmul2(lo, make_float2(a.x, a.y));
            hi = fmul2(hi, make_float2(a.z, a.w));
          } else {
            const float4 z = *reinterpret_cast<const float4*>(sz + kTile + j);
            lo = ffma2(lo, make_float2(a.x, a.y), fmul2(make_float2(z.x, z.y), qs2));
            hi = ffma2(hi, make_float2(a.z, a.w), fmul2(make_float2(z.z, z.w), qs2));
          }
          sc[j] = lo.x;
          sc[j + 1] = lo.y;
          sc[j + 2] = hi.x;
          sc[j + 3] = hi.y;
        }
      }
      if (kbase + static_cast<int>(kTile) - 1 > rpos) {  // diagonal tile only: causal mask
#pragma unroll
        for (int j = 0; j < static_cast<int>(kTile); ++j)
          if (kbase + j > rpos) sc[j] = -INFINITY;
      }
      // FP16/FP8 keep raw scores: the scale rides in the exp2's FFMA below
      constexpr bool kRaw = !(FMT == kINT8 || FMT == kINT4);
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < static_cast<int>(kTile); ++j) mx = fmaxf(mx, sc[j]);
      if constexpr (kRaw) mx *= sml2;
      const bool grow = mx > m + kRescaleSlack;
      const float alpha = grow ? ex2(m - mx) : 1.f;
      // O and the P buffer are free once PV of tile t-1 completed
      if (t > 0) {
        mbar_wait(&pv_done[x], (t - 1) & 1);
        tc_fence_after();
      }
      if (t > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
        for (uint32_t c = 0; c < kD; c += 16) {
          float o[16];
          tmem_ld16(tO + c, o);
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] *= alpha;
          tmem_st16(tO + c, o);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (grow) {
        l *= alpha;
        m = mx;
      }
      float2 l2 = make_float2(0.f, 0.f);
      const float2 sml22 = make_float2(sml2, sml2), nm2 = make_float2(-m, -m);
#pragma unroll
      for (uint32_t c = 0; c < kTile / 8; ++c) {
        float pv[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {  // two scores per FFMA2 / FADD2
          const float2 sj = make_float2(sc[c * 8 + j], sc[c * 8 + j + 1]);
          const float2 xj = kRaw ? ffma2(sj, sml22, nm2) : fadd2(sj, nm2);
          pv[j] = ex2(xj.x);
          pv[j + 1] = ex2(xj.y);
          l2 = fadd2(l2, make_float2(pv[j], pv[j + 1]));
        }
        uint4 w;
        w.x = pack_h2(pv[0], pv[1]);
        w.y = pack_h2(pv[2], pv[3]);
        w.z = pack_h2(pv[4], pv[5]);
        w.w = pack_h2(pv[6], pv[7]);
        *reinterpret_cast<uint4*>(prow + sw128(r, c)) = w;
      }
      l += l2.x + l2.y;
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&p_full[x]);
    }
    mbar_wait(&o_final, 0);
    tc_fence_after();
    if (SPLIT) {  // fp32 partial: acc * oscale (unnormalised), m (log2 domain), l
      const uint64_t prow_g = static_cast<uint64_t>(q0 + (rvalid ? rtok : 0)) * Hq + h * G + rr % G;
      float* part = p.part + (prow_g * nsplit + z) * kPartStride;
#pragma unroll
      for (uint32_t c = 0; c < kD; c += 32) {
        float o[32];
        if (niter > 0) tmem_ld32(tO + c, o);
        if (rvalid) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(part + c + j) =
                niter > 0 ? make_float4(o[j] * oscale, o[j + 1] * oscale, o[j + 2] * oscale, o[j + 3] * oscale)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      if (rvalid) *reinterpret_cast<float2*>(part + kD) = make_float2(niter > 0 ? m : -INFINITY, l);
    } else {
    const float inv = oscale / l;
    __half* orow = p.out + (static_cast<uint64_t>(q0 + (rvalid ? rtok : 0)) * Hq + h * G + rr % G) * kD;
#pragma unroll
    for (uint32_t c = 0; c < kD; c += 32) {
      float o[32];
      tmem_ld32(tO + c, o);
      if (rvalid) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 w;
          w.x = pack_h2(o[j] * inv, o[j + 1] * inv);
          w.y = pack_h2(o[j + 2] * inv, o[j + 3] * inv);
          w.z = pack_h2(o[j + 4] * inv, o[j + 5] * inv);
          w.w = pack_h2(o[j + 6] * inv, o[j + 7] * inv);
          *reinterpret_cast<uint4*>(orow + c + j) = w;
        }
      }
    }
    if (rvalid && p.lse)
      p.lse[static_cast<uint64_t>(q0 + rtok) * Hq + h * G + rr % G] = (m + __log2f(l)) * 0.69314718055994531f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(k2TmemCols));
}

// ------------------------------------------------------------ split-KV merge
// One warp per (query token, query head) row: O = sum_z 2^(m_z - M) acc_z /
// sum_z 2^(m_z - M) l_z over the row's nsplit partials (4 dims per lane).
__global__ void __launch_bounds__(256) prefill_merge_kernel(const PrefillParams p, uint32_t rows, uint32_t nsplit) {
  // rows of this launch's sequences: [cu_q[0], cu_q[batch]) x Hq (a sequence group may start past 0)
  const uint32_t Hq = p.H * p.G, r0 = static_cast<uint32_t>(p.cu_q[0]) * Hq;
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const uint32_t row = r0 + i;
  if (i >= rows || row >= static_cast<uint32_t>(p.cu_q[p.batch]) * Hq) return;
  const float* part = p.part + static_cast<uint64_t>(row) * nsplit * kPartStride;
  float M = -INFINITY;
  for (uint32_t z = 0; z < nsplit; ++z) M = fmaxf(M, part[z * kPartStride + kD]);
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t z = 0; z < nsplit; ++z) {
    const float* pz = part + z * kPartStride;
    const float mz = pz[kD];
    if (mz == -INFINITY) continue;  // empty split
    const float w = ex2(mz - M);
    L += w * pz[kD + 1];
    const float4 a = *reinterpret_cast<const float4*>(pz + 4 * lane);
    acc.x += w * a.x;
    acc.y += w * a.y;
    acc.z += w * a.z;
    acc.w += w * a.w;
  }
  const float inv = 1.f / L;
  __half* orow = p.out + static_cast<uint64_t>(row) * kD + 4 * lane;
  *reinterpret_cast<uint2*>(orow) = make_uint2(pack_h2(acc.x * inv, acc.y * inv), pack_h2(acc.z * inv, acc.w * inv));
  if (lane == 0 && p.lse) p.lse[row] = (M + __log2f(L)) * 0.69314718055994531f;
}

// ------------------------------------------------------------ K4 expand
// Quantised prefill, expand-once form: every context block of the batch is
// dequantised ONCE per call into fp16 chunks laid out exactly like an FP16
// slab block (half-major, 128B-swizzled, section 3) in the scratch block
// s * bt_stride + b, and the FP16 tcgen05 kernel then attends over the
// scratch (identity block table).  The direct quantised kernel instead
// re-dequantises each KV tile in every query-tile CTA of the head (up to
// max_q_len*G/256 times).  HBM-bound: one warp per (sequence, block, K|V,
// head) chunk reads 1-2 KB and writes 4 KB.  FP8 converts exactly (its
// per-head scales are applied in the FP16 kernel, as in the direct path);
// INT8 / INT4 apply the token's scale (and zero) in one fp16 rounding.
template <int FMT>
__global__ void __launch_bounds__(256) expand_kernel(const PrefillParams p, uint8_t* __restrict__ scratch,
                                                     float* __restrict__ sz_out) {
  constexpr uint32_t kChunk = kTPB * kD * Fmt<FMT>::kBits / 8;
  constexpr uint32_t kParam = FMT == kINT8 ? kTPB * 2 : (FMT == kINT4 ? kTPB * 4 : 0);
  pdl_launch_dependents();  // the attention kernel's prologue (TMEM, barriers, Q) overlaps this grid
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t twoH = 2 * p.H;
  const uint64_t per_seq = static_cast<uint64_t>(p.bt_stride) * twoH;
  const uint32_t s = static_cast<uint32_t>(gw / per_seq);
  if (s >= p.batch) return;
  const uint32_t rem = static_cast<uint32_t>(gw % per_seq), b = rem / twoH, c = rem % twoH;
  const int ctx = p.ctx_lens[s];
  if (ctx <= 0 || b * kTPB >= static_cast<uint32_t>(ctx)) return;
  const uint32_t kv = c / p.H;
  const uint8_t* blk = p.pool + block_offset(p.geom, static_cast<uint32_t>(
                                    __ldg(p.block_table + static_cast<uint64_t>(s) * p.bt_stride + b))) + p.layer_off;
  const uint8_t* __restrict__ chunk = blk + static_cast<uint64_t>(c) * kChunk;
  const uint8_t* __restrict__ prm = blk + static_cast<uint64_t>(twoH) * kChunk + static_cast<uint64_t>(c) * kParam;
  uint8_t* out = scratch + (static_cast<uint64_t>(s) * p.bt_stride + b) * (twoH * kTPB * kD * 2) +
                 static_cast<uint64_t>(c) * (kTPB * kD * 2);
  // INT8/INT4 K: exact integers (scale 1, zero 0); its per-token scale and
  // zero go to sz_out as fp32 x sm_scale_log2, applied to S by the kernel
  const bool exact = (FMT == kINT8 || FMT == kINT4) && kv == 0;
  if ((FMT == kINT8 || FMT == kINT4) && kv == 0) {
    float v = 0.f;
    if constexpr (FMT == kINT8) {
      if (lane < kTPB) v = __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short*>(prm) + lane)));
    } else {
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(prm) + (lane & 15));
      v = __half2float(__ushort_as_half(static_cast<uint16_t>(lane < kTPB ? w & 0xffffu : w >> 16)));
    }
    sz_out[((static_cast<uint64_t>(s) * p.bt_stride + b) * p.H + c) * 32 + lane] = v * p.sm_scale_log2;
  }
  // lane's outputs q = lane + 32 j: token t = q / 16 = 2j + lane / 16, dims 8 * (lane % 16) ..
  const uint32_t gi = lane & 15;
  // phase 1: every raw word and token parameter of the lane in flight at once
  uint2 w8[8];
  uint32_t pm[8];
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j) {
    const uint32_t t = 2 * j + (lane >> 4);
    if constexpr (FMT == kFP8 || FMT == kINT8) {
      w8[j] = __ldg(reinterpret_cast<const uint2*>(chunk + swz(t * 128 + 8 * gi)));
    } else if (kv == 0) {
      w8[j].x = __ldg(reinterpret_cast<const uint32_t*>(chunk + swz(t * 64 + 4 * gi)));
    } else {  // V token-pair line: bytes 4gi .. 4gi+3 of token t
      const uint32_t t8 = t & 7, tp = (t8 & 1) | ((t8 >> 2) << 1), side = (t8 >> 1) & 1;
      const uint32_t line = (2 * tp + (t >> 3)) * 128;
      const uint32_t lo = __ldg(reinterpret_cast<const unsigned short*>(chunk + swz(line + 8 * gi + 2 * side)));
      const uint32_t hi = __ldg(reinterpret_cast<const unsigned short*>(chunk + swz(line + 8 * gi + 4 + 2 * side)));
      w8[j].x = lo | (hi << 16);
    }
    if constexpr (FMT == kINT8) pm[j] = __ldg(reinterpret_cast<const unsigned short*>(prm) + t);
    else if constexpr (FMT == kINT4) pm[j] = __ldg(reinterpret_cast<const uint32_t*>(prm) + t);
    else pm[j] = 0;
  }
  // phase 2: convert and store 16-byte granules of the fp16 half-major chunk
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j) {
    const uint32_t t = 2 * j + (lane >> 4);
    uint32_t o[4];
    if constexpr (FMT == kFP8) {
      o[0] = e4m3x2_to_f16x2(static_cast<uint16_t>(w8[j].x & 0xffff));
      o[1] = e4m3x2_to_f16x2(static_cast<uint16_t>(w8[j].x >> 16));
      o[2] = e4m3x2_to_f16x2(static_cast<uint16_t>(w8[j].y & 0xffff));
      o[3] = e4m3x2_to_f16x2(static_cast<uint16_t>(w8[j].y >> 16));
    } else if constexpr (FMT == kINT8) {
      const uint32_t sc = exact ? 0x3C00u : pm[j];
      const uint32_t s2 = sc | (sc << 16);
      const uint32_t x = w8[j].x ^ 0x80808080u, y = w8[j].y ^ 0x80808080u;  // exact 1152 + b, minus 1152, times s
      o[0] = hmul2_u32(hsub2_u32(__byte_perm(x, 0x64646464u, 0x4140), 0x64806480u), s2);
      o[1] = hmul2_u32(hsub2_u32(__byte_perm(x, 0x64646464u, 0x4342), 0x64806480u), s2);
      o[2] = hmul2_u32(hsub2_u32(__byte_perm(y, 0x64646464u, 0x4140), 0x64806480u), s2);
      o[3] = hmul2_u32(hsub2_u32(__byte_perm(y, 0x64646464u, 0x4342), 0x64806480u), s2);
    } else {
      const uint32_t sz = exact ? 0x3C00u : pm[j];
      const uint32_t sc = sz & 0xffffu, z = sz >> 16;
      const uint32_t s2 = sc | (hmul2_u32(sc, 0x2C00u) << 16);  // (s, s/16): the high nibble enters as 16 n
      const uint32_t z2 = z | (z << 16);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t y = __byte_perm(w8[j].x, 0, k | (k << 8) | (k << 16) | (k << 24));
        const uint32_t n = hsub2_u32(lop3_and_or(y, 0x00F0000Fu, 0x64006400u), 0x64006400u);
        o[k] = hfma2_u32(n, s2, z2);
      }
    }
    *reinterpret_cast<uint4*>(out + swz((gi >> 3) * (kTPB * 128) + t * 128 + (gi & 7) * 16)) =
        make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace tc
}  // namespace dev

template <int FMT, bool EXP = false>
static cudaError_t launch_tc(const PrefillParams& p0, cudaStream_t stream, bool pdl = false) {
  using namespace dev::tc;
  PrefillParams p = p0;
  const uint32_t tpc = 2 * kRows / p.G;  // tokens per CTA (two 128-row query tiles)
  p.tiles = (p.max_q_len + tpc - 1) / tpc;
  if (p.tiles == 0) return cudaSuccess;
  const size_t smem = TcCfg<FMT, EXP>::kSmem + 1024;  // + alignment slack
  const uint32_t nsplit = p.kv_splits > 1 ? p.kv_splits : 1;
  auto kern = nsplit > 1 ? prefill_tc2_kernel<FMT, EXP, true> : prefill_tc2_kernel<FMT, EXP, false>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.batch * p.H, p.tiles, nsplit);
  cfg.blockDim = dim3(kThreadsOf<FMT, EXP>);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e2 = cudaLaunchKernelEx(&cfg, kern, p);
  if (e2 != cudaSuccess || nsplit == 1) return e2;
  const uint64_t rows = static_cast<uint64_t>(p.batch) * p.max_q_len * p.H * p.G;  // bound; exact count on device
  prefill_merge_kernel<<<static_cast<uint32_t>((rows + 7) / 8), 256, 0, stream>>>(p, static_cast<uint32_t>(rows),
                                                                                  nsplit);
  return cudaGetLastError();
}

// scratch: fp16 blocks [batch * bt_stride][2H chunks], then the K scale/zero
// arrays [batch * bt_stride][H][16 scales | 16 zeros] fp32
uint32_t prefill_kv_splits(uint32_t batch, uint32_t H, uint32_t G, uint32_t max_q_len, int num_sms) {
  const uint32_t tpc = 2 * dev::tc::kRows / G;
  const uint64_t ctas = static_cast<uint64_t>(batch) * H * ((max_q_len + tpc - 1) / tpc);
  if (ctas == 0) return 1;
  const uint64_t s = static_cast<uint64_t>(num_sms) / ctas;
  return static_cast<uint32_t>(s < 2 ? 1 : (s > 8 ? 8 : s));
}

size_t prefill_partial_bytes(uint32_t batch, uint32_t H, uint32_t G, uint32_t max_q_len, uint32_t splits) {
  return splits > 1 ? static_cast<size_t>(batch) * max_q_len * H * G * splits * dev::tc::kPartStride * 4 : 0;
}

size_t prefill_expand_bytes(uint32_t H, uint32_t batch, uint32_t bt_stride) {
  return static_cast<size_t>(batch) * bt_stride * (2ull * H * dev::kTPB * dev::kD * 2 + H * 128ull);
}

cudaError_t launch_paged_prefill_expand(const PrefillParams& p, int kv_dtype, uint8_t* scratch,
                                        cudaStream_t stream) {
  using namespace dev;
  const uint64_t warps = static_cast<uint64_t>(p.batch) * p.bt_stride * 2 * p.H;
  const uint64_t blocks = (warps + 7) / 8;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffULL) return cudaErrorInvalidValue;
  float* sz = reinterpret_cast<float*>(scratch + static_cast<size_t>(p.batch) * p.bt_stride *
                                                       (2ull * p.H * kTPB * kD * 2));
  const uint32_t nb = static_cast<uint32_t>(blocks);
  switch (kv_dtype) {
    case kFP8: tc::expand_kernel<kFP8><<<nb, 256, 0, stream>>>(p, scratch, sz); break;
    case kINT8: tc::expand_kernel<kINT8><<<nb, 256, 0, stream>>>(p, scratch, sz); break;
    case kINT4: tc::expand_kernel<kINT4><<<nb, 256, 0, stream>>>(p, scratch, sz); break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the scratch as a one-layer FP16 pool: block g at g * key, identity table
  PrefillParams q = p;
  q.pool = scratch;
  q.geom.key = 2ull * p.H * kTPB * kD * 2;
  q.geom.slab_size = q.geom.key;
  q.geom.bps = make_fastdiv(1);
  q.layer_off = 0;
  q.block_table = nullptr;
  q.kv_scales = kv_dtype == kFP8 ? p.kv_scales : nullptr;
  q.exp_sz = sz;
  if (kv_dtype == kINT8) return launch_tc<kINT8, true>(q, stream, true);
  if (kv_dtype == kINT4) return launch_tc<kINT4, true>(q, stream, true);
  return launch_tc<kFP16>(q, stream, true);  // FP8: exact in fp16, per-head scales in the kernel
}

cudaError_t launch_paged_prefill_tc(const PrefillParams& p, int kv_dtype, cudaStream_t stream) {
  using namespace dev;
  switch (kv_dtype) {
    case kFP16: return launch_tc<kFP16>(p, stream);
    case kFP8: return launch_tc<kFP8>(p, stream);
    case kINT8: return launch_tc<kINT8>(p, stream);
    case kINT4: return launch_tc<kINT4>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace kvslab
