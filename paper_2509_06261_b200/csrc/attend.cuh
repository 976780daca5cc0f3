// attend.cuh -- the tensor-core attention step shared by K2 (decode.cu) and
// the chunked-prefill kernel (prefill.cu): fragment loaders for the swizzled
// slab chunk layout, and one warp's online-softmax step
// over staged blocks (S^T = K.Q^T, O^T += V^T.P^T on mma.sync m16n8k16).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kvslab_device.cuh"
#include "launch.hpp"

namespace kvslab {
namespace dev {

constexpr int kD = 128;   // head dim
constexpr int kTPB = 16;  // tokens per block
constexpr float kLog2e = 1.4426950408889634f;

template <int FMT>
struct Geo {
  static constexpr int kRow = kD * Fmt<FMT>::kBits / 8;  // bytes per token row
  static constexpr int kChunk = kTPB * kRow;              // bytes per (K|V, head) chunk
  static constexpr int kParam = FMT == kINT8 ? kTPB * 2 : (FMT == kINT4 ? kTPB * 4 : 0);
  // integer formats enter the MMA as exact fp16 (q + kBias); the bias is
  // removed from the 16x8 score tile (kBias * sum(q)) and from O (kBias * sum(p'))
  static constexpr float kBias = FMT == kINT8 ? 1152.f : (FMT == kINT4 ? 1024.f : 0.f);
  static constexpr bool kBiased = FMT == kINT8 || FMT == kINT4;
};

// ------------------------------------------------------ fragment loaders
// Per-thread byte offsets (inside a K or V chunk) of the fragment loads; they
// only depend on (g, t) so they are computed once per kernel.
struct FragOff {
  uint32_t k[4];
  uint32_t v[4];
};

// token held in PV k-slot: slot 2t -> ta(t), 2t+1 -> tb(t), +8 for 2t+8/2t+9
// (FP16 pairs tokens (2t, 2t+1) like the 8-bit formats: with the half-major
// chunk a row is one 128-byte line, and even/odd rows keep the two lanes of a
// quarter-warp on different banks)
template <int FMT>
__device__ __forceinline__ int tok_a(int t) {
  if constexpr (FMT == kINT4) return (t & 1) + ((t >> 1) << 2);  // {0,1,4,5}
  else return 2 * t;
}
template <int FMT>
__device__ __forceinline__ int tok_b(int t) {
  if constexpr (FMT == kINT4) return 2 + (t & 1) + ((t >> 1) << 2);  // {2,3,6,7}
  else return 2 * t + 1;
}

template <int FMT>
__device__ __forceinline__ FragOff make_offsets(int g, int t) {
  FragOff o;
  const int ta = tok_a<FMT>(t), tb = tok_b<FMT>(t);
  if constexpr (FMT == kFP16) {
#pragma unroll
    // half-major chunk: dims 64h.. of token t at h*2048 + t*128 (16 tokens);
    // granule 2t + (c&1) of the half: rows g and g^1 of a quarter-warp then
    // hit disjoint banks under the row-keyed swizzle
    for (int c = 0; c < 4; ++c) o.k[c] = swz((c >> 1) * 2048 + g * 128 + 16 * (2 * t + (c & 1)));
    o.v[0] = swz(ta * 128 + 16 * g);
    o.v[1] = swz(2048 + ta * 128 + 16 * g);
    o.v[2] = swz(tb * 128 + 16 * g);
    o.v[3] = swz(2048 + tb * 128 + 16 * g);
  } else if constexpr (FMT == kFP8 || FMT == kINT8) {
    o.k[0] = swz(g * 128 + 16 * (2 * t));
    o.k[1] = swz(g * 128 + 16 * (2 * t + 1));
    o.k[2] = o.k[3] = 0;
    o.v[0] = swz(ta * 128 + 16 * g);
    o.v[1] = swz(tb * 128 + 16 * g);
    o.v[2] = o.v[3] = 0;
  } else {
    o.k[0] = swz(g * 64 + 16 * t);
    o.k[1] = swz((g + 8) * 64 + 16 * t);
    o.k[2] = o.k[3] = 0;
    // V token-pair lines: 2t holds (ta, tb), 2t+1 holds (ta+8, tb+8); with
    // the line-keyed swizzle a quarter-warp's 16-byte loads are conflict-free
    o.v[0] = swz(2 * t * 128 + 16 * g);
    o.v[1] = swz((2 * t + 1) * 128 + 16 * g);
    o.v[2] = o.v[3] = 0;
  }
  return o;
}

// K tile as the MMA A operand (rows = tokens g, g+8; k = dims permuted per
// format).  a[kk][0..3] for k-step kk.  Row g+8 sits 8 rows further, which is
// a constant (swizzle-preserving) offset for 256- and 128-byte rows.
template <int FMT>
__device__ __forceinline__ void load_k_frags(uint32_t sK, const FragOff& o, uint32_t (&a)[8][4]) {
  if constexpr (FMT == kFP16) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 lo = lds128(sK + o.k[c]);
      const uint4 hi = lds128(sK + o.k[c] + 1024);  // token g+8: 8 rows on
      a[2 * c][0] = lo.x; a[2 * c][1] = hi.x; a[2 * c][2] = lo.y; a[2 * c][3] = hi.y;
      a[2 * c + 1][0] = lo.z; a[2 * c + 1][1] = hi.z; a[2 * c + 1][2] = lo.w; a[2 * c + 1][3] = hi.w;
    }
  } else if constexpr (FMT == kFP8 || FMT == kINT8) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint4 lo = lds128(sK + o.k[c]);
      const uint4 hi = lds128(sK + o.k[c] + 1024);
      const uint32_t wl[4] = {lo.x, lo.y, lo.z, lo.w};
      const uint32_t wh[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t* r = a[4 * c + e];
        if constexpr (FMT == kFP8) {
          r[0] = e4m3x2_to_f16x2(static_cast<uint16_t>(wl[e] & 0xffff));
          r[2] = e4m3x2_to_f16x2(static_cast<uint16_t>(wl[e] >> 16));
          r[1] = e4m3x2_to_f16x2(static_cast<uint16_t>(wh[e] & 0xffff));
          r[3] = e4m3x2_to_f16x2(static_cast<uint16_t>(wh[e] >> 16));
        } else {
          const uint32_t xl = wl[e] ^ 0x80808080u, xh = wh[e] ^ 0x80808080u;
          // exact fp16 b + 1152 (the bias is removed after the MMA)
          r[0] = __byte_perm(xl, 0x64646464u, 0x4140);
          r[2] = __byte_perm(xl, 0x64646464u, 0x4342);
          r[1] = __byte_perm(xh, 0x64646464u, 0x4140);
          r[3] = __byte_perm(xh, 0x64646464u, 0x4342);
        }
      }
    }
  } else {  // INT4: one granule (32 dims) per row per thread
    const uint4 lo = lds128(sK + o.k[0]);
    const uint4 hi = lds128(sK + o.k[1]);
    const uint32_t wl[4] = {lo.x, lo.y, lo.z, lo.w};
    const uint32_t wh[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        uint32_t* r = a[2 * i + e];
        const uint32_t xl = e ? wl[i] >> 8 : wl[i], xh = e ? wh[i] >> 8 : wh[i];
        // exact fp16 1024 + n (low nibble, k-slots 2t, 2t+1) and 1024 + 16 n
        // (high nibble in place, k-slots 2t+8, 2t+9: their Q entries carry
        // the 1/16); the 1024 bias is removed after the MMA
        r[0] = lop3_and_or(xl, 0x000F000Fu, 0x64006400u);
        r[2] = lop3_and_or(xl, 0x00F000F0u, 0x64006400u);
        r[1] = lop3_and_or(xh, 0x000F000Fu, 0x64006400u);
        r[3] = lop3_and_or(xh, 0x00F000F0u, 0x64006400u);
      }
    }
  }
}

// Q rows of the unit -> MMA B fragments for query g of each n-tile, with the
// K dims permuted exactly like load_k_frags (the reduction order is free).
// PK (packed decode, G <= 4): column g carries query g & 3 (see attend_pk).
template <int FMT, int NT, bool PK = false>
__device__ __forceinline__ void load_q_frags(uint32_t sQ, int g, int t, uint32_t G,
                                             uint32_t (&qf)[NT][8][2]) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int qrow = PK ? (g & 3) : nt * 8 + g;
    const bool ok = qrow < static_cast<int>(G);
    const uint32_t row = sQ + qrow * kD * 2;
    if constexpr (FMT == kFP16) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int gr = 8 * (c >> 1) + 2 * t + (c & 1);  // the K fragments' dim order
        const uint4 v = ok ? lds128(row + 16 * gr) : make_uint4(0, 0, 0, 0);
        qf[nt][2 * c][0] = v.x; qf[nt][2 * c][1] = v.y;
        qf[nt][2 * c + 1][0] = v.z; qf[nt][2 * c + 1][1] = v.w;
      }
    } else if constexpr (FMT == kFP8 || FMT == kINT8) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // dims 32t + 8c .. +7 -> k-steps 2c, 2c+1
        const uint4 v = ok ? lds128(row + 64 * t + 16 * c) : make_uint4(0, 0, 0, 0);
        qf[nt][2 * c][0] = v.x; qf[nt][2 * c][1] = v.y;
        qf[nt][2 * c + 1][0] = v.z; qf[nt][2 * c + 1][1] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // dims 32t + 8i .. +7: pairs (0,4),(1,5) | (2,6),(3,7)
        const uint4 v = ok ? lds128(row + 64 * t + 16 * i) : make_uint4(0, 0, 0, 0);
        // high-nibble k-slots see K as 1024 + 16 n: their Q entries carry 1/16
        // (a power of two: exact for normal fp16)
        qf[nt][2 * i][0] = __byte_perm(v.x, v.z, 0x5410);
        qf[nt][2 * i][1] = hmul2_u32(__byte_perm(v.x, v.z, 0x7632), 0x2C002C00u);
        qf[nt][2 * i + 1][0] = __byte_perm(v.y, v.w, 0x5410);
        qf[nt][2 * i + 1][1] = hmul2_u32(__byte_perm(v.y, v.w, 0x7632), 0x2C002C00u);
      }
    }
  }
}

// V tile as the MMA A operand of O^T = V^T P^T (rows = dims, k = tokens).
template <int FMT>
__device__ __forceinline__ void load_v_frags(uint32_t sV, const FragOff& o, uint32_t (&a)[8][4]) {
  if constexpr (FMT == kFP16) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 va = lds128(sV + o.v[h]);
      const uint4 vb = lds128(sV + o.v[2 + h]);
      const uint4 vc = lds128(sV + o.v[h] + 1024);  // tokens +8: 8 rows on
      const uint4 vd = lds128(sV + o.v[2 + h] + 1024);
      const uint32_t A[4] = {va.x, va.y, va.z, va.w}, B[4] = {vb.x, vb.y, vb.z, vb.w};
      const uint32_t C[4] = {vc.x, vc.y, vc.z, vc.w}, Dd[4] = {vd.x, vd.y, vd.z, vd.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t* r = a[4 * h + i];
        r[0] = __byte_perm(A[i], B[i], 0x5410);
        r[1] = __byte_perm(A[i], B[i], 0x7632);
        r[2] = __byte_perm(C[i], Dd[i], 0x5410);
        r[3] = __byte_perm(C[i], Dd[i], 0x7632);
      }
    }
  } else if constexpr (FMT == kFP8 || FMT == kINT8) {
    const uint4 va = lds128(sV + o.v[0]);
    const uint4 vb = lds128(sV + o.v[1]);
    const uint4 vc = lds128(sV + o.v[0] + 1024);
    const uint4 vd = lds128(sV + o.v[1] + 1024);
    const uint32_t A[4] = {va.x, va.y, va.z, va.w}, B[4] = {vb.x, vb.y, vb.z, vb.w};
    const uint32_t C[4] = {vc.x, vc.y, vc.z, vc.w}, Dd[4] = {vd.x, vd.y, vd.z, vd.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t sel = e == 0 ? 0x5140u : 0x7362u;
        uint32_t* r = a[2 * j + e];
        if constexpr (FMT == kFP8) {
          const uint32_t ab = __byte_perm(A[j], B[j], sel), cd = __byte_perm(C[j], Dd[j], sel);
          r[0] = e4m3x2_to_f16x2(static_cast<uint16_t>(ab & 0xffff));
          r[1] = e4m3x2_to_f16x2(static_cast<uint16_t>(ab >> 16));
          r[2] = e4m3x2_to_f16x2(static_cast<uint16_t>(cd & 0xffff));
          r[3] = e4m3x2_to_f16x2(static_cast<uint16_t>(cd >> 16));
        } else {
          const uint32_t ab = __byte_perm(A[j] ^ 0x80808080u, B[j] ^ 0x80808080u, sel);
          const uint32_t cd = __byte_perm(C[j] ^ 0x80808080u, Dd[j] ^ 0x80808080u, sel);
          r[0] = __byte_perm(ab, 0x64646464u, 0x4140);
          r[1] = __byte_perm(ab, 0x64646464u, 0x4342);
          r[2] = __byte_perm(cd, 0x64646464u, 0x4140);
          r[3] = __byte_perm(cd, 0x64646464u, 0x4342);
        }
      }
    }
  } else {  // INT4: one 16-byte load per token pair, [A.j A.j+1 B.j B.j+1] per word
    const uint4 va = lds128(sV + o.v[0]);  // tokens ta, tb: bytes 8g .. 8g+7
    const uint4 vc = lds128(sV + o.v[1]);  // tokens ta+8, tb+8
    const uint32_t A[4] = {va.x, va.y, va.z, va.w}, C[4] = {vc.x, vc.y, vc.z, vc.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // m-tile i: byte 8g + i (dims 16g + 2i, +1)
      const uint32_t x = (i & 1) ? A[i >> 1] >> 8 : A[i >> 1];
      const uint32_t y = (i & 1) ? C[i >> 1] >> 8 : C[i >> 1];
      uint32_t* r = a[i];
      // rows g+8 (high nibbles, in place) enter as 1024 + 16 n: the epilogue
      // divides those output dims by 16
      r[0] = lop3_and_or(x, 0x000F000Fu, 0x64006400u);
      r[1] = lop3_and_or(x, 0x00F000F0u, 0x64006400u);
      r[2] = lop3_and_or(y, 0x000F000Fu, 0x64006400u);
      r[3] = lop3_and_or(y, 0x00F000F0u, 0x64006400u);
    }
  }
}
// output dim of V m-tile mt, row half r8 (0: row g, 1: row g+8)
template <int FMT>
__device__ __forceinline__ int vdim(int mt, int g, int r8) {
  if constexpr (FMT == kFP16) return 64 * (mt >> 2) + 8 * g + 2 * (mt & 3) + r8;
  else return 16 * g + 2 * mt + r8;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Online-softmax state of one warp's (unit segment, head): O^T accumulator
// tiles, reference max, row sums and the additive terms of biased formats
// (zb: -bias * sum(P'), zz: sum(p * z_v) for INT4).
template <int NT>
struct UnitState {
  float acc[8][NT][4];
  float m[NT][2], l[NT][2], zb[NT][2], zz[NT][2];
};

constexpr float kRescaleSlack = 8.0f;  // log2 units: P <= 2^8 before a rescale

// One consumer step: BPI staged blocks (shared-memory stage addresses sbs,
// valid token counts) of one head attended by one warp -- S^T = K.Q^T on
// tensor cores, lazy online softmax, O^T += V^T.P^T.
// Integer formats feed V to the MMA as biased exact fp16 (kBias + code), so
// the O accumulator also collects kBias * sum(P'), removed through u.zb.  Left
// to grow over a long context that bias costs the fp32 accumulator the low
// bits of the signal (INT4: bias/signal ~ 1024/8).  Folding the column sums of
// u.zb into the accumulator every kBiasFlush blocks bounds the bias to a few
// blocks' worth (measured: INT4 prefill at ctx 700, 1.5e-2 -> see DESIGN.md).
constexpr uint32_t kBiasFlush = 8;
template <int FMT, int NT>
__device__ __forceinline__ void flush_bias(UnitState<NT>& u) {
  if constexpr (Geo<FMT>::kBiased) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float z = u.zb[nt][c];
        z += __shfl_xor_sync(0xffffffffu, z, 4);
        z += __shfl_xor_sync(0xffffffffu, z, 8);
        z += __shfl_xor_sync(0xffffffffu, z, 16);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          u.acc[mt][nt][c] += z;
          u.acc[mt][nt][2 + c] += z;
        }
        u.zb[nt][c] = 0.f;
      }
  }
}

// CAUSAL (prefill): additionally, query column (nt, 2t+c) sees only the
// block's tokens below qlim[nt][c] (its position - block start + 1).
template <int FMT, int NT, int BPI, bool MASK = true, bool CAUSAL = false>
__device__ __forceinline__ void attend(UnitState<NT>& u, const uint32_t (&sbs)[BPI],
                                       const int (&valid)[BPI], uint32_t wK, uint32_t wP,
                                       uint32_t kvq, uint32_t pq, const FragOff& fo,
                                       const uint32_t (&qf)[NT][8][2], const float (&qsb)[NT][2],
                                       const float (&qst)[NT][2], float kscale, float sml2, int g,
                                       int t, const int (*qlim)[2] = nullptr) {
  using Gm = Geo<FMT>;
  // ---- S^T = K . Q^T per block (two accumulators halve the MMA chain) ----
  float sc[BPI][NT][4], svv[BPI][2], zvv[BPI][2];
#pragma unroll
  for (int bi = 0; bi < BPI; ++bi) {
    uint32_t ka[8][4];
    load_k_frags<FMT>(sbs[bi] + wK, fo, ka);
    float sk[2] = {kscale * sml2, kscale * sml2}, zk[2] = {0.f, 0.f};  // softmax scale folded in
    svv[bi][0] = svv[bi][1] = 1.f;
    zvv[bi][0] = zvv[bi][1] = 0.f;
    const uint32_t sKp = sbs[bi] + wP, sVp = sKp + pq;
    if constexpr (FMT == kINT8) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        sk[r] = __half2float(__ushort_as_half(lds16(sKp + 2 * (g + 8 * r)))) * sml2;
        svv[bi][r] = __half2float(__ushort_as_half(lds16(sVp + 2 * (g + 8 * r))));
      }
    } else if constexpr (FMT == kINT4) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t kp = lds32(sKp + 4 * (g + 8 * r)), vp = lds32(sVp + 4 * (g + 8 * r));
        sk[r] = __half2float(__ushort_as_half(static_cast<uint16_t>(kp & 0xffff))) * sml2;
        zk[r] = __half2float(__ushort_as_half(static_cast<uint16_t>(kp >> 16))) * sml2;
        svv[bi][r] = __half2float(__ushort_as_half(static_cast<uint16_t>(vp & 0xffff)));
        zvv[bi][r] = __half2float(__ushort_as_half(static_cast<uint16_t>(vp >> 16)));
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        mma16816(s1, ka[kk][0], ka[kk][1], ka[kk][2], ka[kk][3], qf[nt][kk][0], qf[nt][kk][1]);
        mma16816(s2, ka[kk + 1][0], ka[kk + 1][1], ka[kk + 1][2], ka[kk + 1][3],
                 qf[nt][kk + 1][0], qf[nt][kk + 1][1]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float dot = s1[e] + s2[e];
        float x;
        if constexpr (Gm::kBiased)  // s' * (dot' - bias*sum(q')) + z' * sum(q)
          x = sk[r] * (dot - Gm::kBias * qsb[nt][e & 1]) + zk[r] * qst[nt][e & 1];
        else
          x = dot * sk[r];
        bool ok = g + 8 * r < valid[bi];
        if constexpr (CAUSAL) ok = ok && g + 8 * r < qlim[nt][e & 1];
        sc[bi][nt][e] = ok ? x : -INFINITY;
      }
    }
  }

  // ---- online softmax over the BPI tiles ----
  // Lazy rescaling: the reference max u.m moves (and O is rescaled) only
  // when a score exceeds it by kRescaleSlack; the common case costs one vote.
  uint32_t pb[BPI][NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    bool grow = false;
#pragma unroll
    for (int bi = 0; bi < BPI; ++bi)
#pragma unroll
      for (int e = 0; e < 4; ++e) grow |= sc[bi][nt][e] > u.m[nt][e & 1] + kRescaleSlack;
    if (__any_sync(0xffffffffu, grow)) {
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int bi = 0; bi < BPI; ++bi) {
        mx[0] = fmaxf(mx[0], fmaxf(sc[bi][nt][0], sc[bi][nt][2]));
        mx[1] = fmaxf(mx[1], fmaxf(sc[bi][nt][1], sc[bi][nt][3]));
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 4));
        mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 8));
        mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 16));
        const float mn = fmaxf(u.m[nt][c], mx[c]);
        const float alpha = ex2(u.m[nt][c] - mn);
        u.m[nt][c] = mn;
        u.l[nt][c] *= alpha;
        u.zb[nt][c] *= alpha;
        u.zz[nt][c] *= alpha;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          u.acc[mt][nt][c] *= alpha;
          u.acc[mt][nt][2 + c] *= alpha;
        }
      }
    }
#pragma unroll
    for (int bi = 0; bi < BPI; ++bi) {
      float pr[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) pr[e] = ex2(sc[bi][nt][e] - u.m[nt][e & 1]);
      const uint32_t plo = pack_h2(pr[0] * svv[bi][0], pr[1] * svv[bi][0]);
      const uint32_t phi = pack_h2(pr[2] * svv[bi][1], pr[3] * svv[bi][1]);
#pragma unroll
      for (int c = 0; c < 2; ++c) u.l[nt][c] += pr[c] + pr[c + 2];
      if constexpr (Gm::kBiased) {
        // the bias term uses the exact fp16 P' that the MMA consumes
        const float2 flo = __half22float2(*reinterpret_cast<const __half2*>(&plo));
        const float2 fhi = __half22float2(*reinterpret_cast<const __half2*>(&phi));
        u.zb[nt][0] -= Gm::kBias * (flo.x + fhi.x);
        u.zb[nt][1] -= Gm::kBias * (flo.y + fhi.y);
        if constexpr (FMT == kINT4) {
          u.zz[nt][0] += pr[0] * zvv[bi][0] + pr[2] * zvv[bi][1];
          u.zz[nt][1] += pr[1] * zvv[bi][0] + pr[3] * zvv[bi][1];
        }
      }
      const int la = tok_a<FMT>(t) * 4 + (g >> 1), lb = tok_b<FMT>(t) * 4 + (g >> 1);
      const uint32_t xa = __shfl_sync(0xffffffffu, plo, la), xb = __shfl_sync(0xffffffffu, plo, lb);
      const uint32_t ya = __shfl_sync(0xffffffffu, phi, la), yb = __shfl_sync(0xffffffffu, phi, lb);
      const uint32_t sel = (g & 1) ? 0x7632u : 0x5410u;
      pb[bi][nt][0] = __byte_perm(xa, xb, sel);
      pb[bi][nt][1] = __byte_perm(ya, yb, sel);
    }
  }
  // ---- O^T += V^T . P^T ----
#pragma unroll
  for (int bi = 0; bi < BPI; ++bi) {
    uint32_t va[8][4];
    load_v_frags<FMT>(sbs[bi] + kvq + wK, fo, va);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        mma16816(u.acc[mt][nt], va[mt][0], va[mt][1], va[mt][2], va[mt][3], pb[bi][nt][0], pb[bi][nt][1]);
  }
}

// ------------------------------------------------- packed step (G <= 4)
// With a query group of at most 4 the m16n8k16 score tile (N = 8 query
// columns) would be half empty.  The packed step gives each tile column n the
// query n & 3 and lets columns 0-3 attend block sbs[0] and columns 4-7 block
// sbs[1]: two independent online-softmax streams of the same queries, folded
// at the end of the unit segment (fold_halves).  The MMA count is unchanged
// (both blocks' S^T and O^T tiles are computed in full); the per-element
// score epilogue, the softmax, the scale loads and the P shuffles -- most of
// a step's non-MMA instructions -- now serve two blocks.  Thread (g, t) owns
// columns 2t, 2t+1, i.e. block t >> 1.  NB = 1: one block in columns 0-3,
// columns 4-7 are masked (their P' is exactly 0).
// Split in two so K2 can software-pipeline it: pk_scores (QK^T of the next
// pair) is issued before pk_update (softmax + PV of the current pair), and the
// two independent dependency chains interleave.
template <int FMT, int NB>
__device__ __forceinline__ void pk_scores(const uint32_t (&sbs)[2], uint32_t wK, const FragOff& fo,
                                          const uint32_t (&qf)[1][8][2], int t, float (&dsel)[4]) {
  const bool hb = t >= 2;  // this thread's columns attend block 1
  float dot[NB][4];
#pragma unroll
  for (int bi = 0; bi < NB; ++bi) {
    uint32_t ka[8][4];
    load_k_frags<FMT>(sbs[bi] + wK, fo, ka);
    float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 8; kk += 2) {
      mma16816(s1, ka[kk][0], ka[kk][1], ka[kk][2], ka[kk][3], qf[0][kk][0], qf[0][kk][1]);
      mma16816(s2, ka[kk + 1][0], ka[kk + 1][1], ka[kk + 1][2], ka[kk + 1][3], qf[0][kk + 1][0],
               qf[0][kk + 1][1]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) dot[bi][e] = s1[e] + s2[e];
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) dsel[e] = (NB == 2 && hb) ? dot[NB - 1][e] : dot[0][e];
}

template <int FMT, int NB, bool MASK>
__device__ __forceinline__ void pk_update(UnitState<1>& u, const float (&dsel)[4],
                                          const uint32_t (&sbs)[2], const int (&valid)[2],
                                          uint32_t wK, uint32_t wP, uint32_t kvq, uint32_t pq,
                                          const FragOff& fo, const float (&qsb)[1][2],
                                          const float (&qst)[1][2], float kscale, float sml2, int g,
                                          int t) {
  using Gm = Geo<FMT>;
  const bool hb = t >= 2;
  // ---- this thread's block: token scales and the score epilogue ----
  const uint32_t sbh = (NB == 2 && hb) ? sbs[1] : sbs[0];
  const int vh = NB == 2 ? (hb ? valid[1] : valid[0]) : (hb ? 0 : valid[0]);
  float sk[2] = {kscale, kscale}, zk[2] = {0.f, 0.f}, svv[2] = {1.f, 1.f}, zvv[2] = {0.f, 0.f};
  const uint32_t sKp = sbh + wP, sVp = sKp + pq;
  if constexpr (FMT == kINT8) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      sk[r] = __half2float(__ushort_as_half(lds16(sKp + 2 * (g + 8 * r))));
      svv[r] = __half2float(__ushort_as_half(lds16(sVp + 2 * (g + 8 * r))));
    }
  } else if constexpr (FMT == kINT4) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t kp = lds32(sKp + 4 * (g + 8 * r)), vp = lds32(sVp + 4 * (g + 8 * r));
      sk[r] = __half2float(__ushort_as_half(static_cast<uint16_t>(kp & 0xffff)));
      zk[r] = __half2float(__ushort_as_half(static_cast<uint16_t>(kp >> 16)));
      svv[r] = __half2float(__ushort_as_half(static_cast<uint16_t>(vp & 0xffff)));
      zvv[r] = __half2float(__ushort_as_half(static_cast<uint16_t>(vp >> 16)));
    }
  }
  float sc[4];
#pragma unroll
  for (int r = 0; r < 2; ++r) {  // the softmax scale rides in the row scales
    sk[r] *= sml2;
    zk[r] *= sml2;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = e >> 1;
    float x;
    if constexpr (Gm::kBiased)  // s' * (dot' - bias*sum(q')) + z' * sum(q)
      x = sk[r] * (dsel[e] - Gm::kBias * qsb[0][e & 1]) + zk[r] * qst[0][e & 1];
    else
      x = dsel[e] * sk[r];
    sc[e] = (MASK || NB == 1) && !(g + 8 * r < vh) ? -INFINITY : x;
  }
  // ---- online softmax (lazy rescale, as in attend) ----
  bool grow = false;
#pragma unroll
  for (int e = 0; e < 4; ++e) grow |= sc[e] > u.m[0][e & 1] + kRescaleSlack;
  if (__any_sync(0xffffffffu, grow)) {
    float mx[2] = {fmaxf(sc[0], sc[2]), fmaxf(sc[1], sc[3])};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 4));
      mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 8));
      mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 16));
      const float mn = fmaxf(u.m[0][c], mx[c]);
      const float alpha = ex2(u.m[0][c] - mn);
      u.m[0][c] = mn;
      u.l[0][c] *= alpha;
      u.zb[0][c] *= alpha;
      u.zz[0][c] *= alpha;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        u.acc[mt][0][c] *= alpha;
        u.acc[mt][0][2 + c] *= alpha;
      }
    }
  }
  float pr[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) pr[e] = ex2(sc[e] - u.m[0][e & 1]);
  const uint32_t plo = pack_h2(pr[0] * svv[0], pr[1] * svv[0]);
  const uint32_t phi = pack_h2(pr[2] * svv[1], pr[3] * svv[1]);
#pragma unroll
  for (int c = 0; c < 2; ++c) u.l[0][c] += pr[c] + pr[c + 2];
  if constexpr (Gm::kBiased) {
    const float2 flo = __half22float2(*reinterpret_cast<const __half2*>(&plo));
    const float2 fhi = __half22float2(*reinterpret_cast<const __half2*>(&phi));
    u.zb[0][0] -= Gm::kBias * (flo.x + fhi.x);
    u.zb[0][1] -= Gm::kBias * (flo.y + fhi.y);
    if constexpr (FMT == kINT4) {
      u.zz[0][0] += pr[0] * zvv[0] + pr[2] * zvv[1];
      u.zz[0][1] += pr[1] * zvv[0] + pr[3] * zvv[1];
    }
  }
  const int la = tok_a<FMT>(t) * 4 + (g >> 1), lb = tok_b<FMT>(t) * 4 + (g >> 1);
  const uint32_t xa = __shfl_sync(0xffffffffu, plo, la), xb = __shfl_sync(0xffffffffu, plo, lb);
  const uint32_t ya = __shfl_sync(0xffffffffu, phi, la), yb = __shfl_sync(0xffffffffu, phi, lb);
  const uint32_t sel = (g & 1) ? 0x7632u : 0x5410u;
  const uint32_t pb0 = __byte_perm(xa, xb, sel), pb1 = __byte_perm(ya, yb, sel);
  // ---- O^T += V^T . P^T: block bi feeds only its own columns (B column = g) ----
#pragma unroll
  for (int bi = 0; bi < NB; ++bi) {
    const bool mine = NB == 1 || ((g >> 2) == bi);
    const uint32_t b0 = mine ? pb0 : 0u, b1 = mine ? pb1 : 0u;
    uint32_t va[8][4];
    load_v_frags<FMT>(sbs[bi] + kvq + wK, fo, va);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) mma16816(u.acc[mt][0], va[mt][0], va[mt][1], va[mt][2], va[mt][3], b0, b1);
  }
}

template <int FMT, int NB, bool MASK>
__device__ __forceinline__ void attend_pk(UnitState<1>& u, const uint32_t (&sbs)[2],
                                          const int (&valid)[2], uint32_t wK, uint32_t wP,
                                          uint32_t kvq, uint32_t pq, const FragOff& fo,
                                          const uint32_t (&qf)[1][8][2], const float (&qsb)[1][2],
                                          const float (&qst)[1][2], float kscale, float sml2, int g,
                                          int t) {
  float d[4];
  pk_scores<FMT, NB>(sbs, wK, fo, qf, t, d);
  pk_update<FMT, NB, MASK>(u, d, sbs, valid, wK, wP, kvq, pq, fo, qsb, qst, kscale, sml2, g, t);
}

// ------------------------------------- integer QK step (INT8/INT4, G <= 4)
// S^T = K.Q^T on IMMA (mma.sync m16n8k32, 8-bit A and B, s32 accumulate):
// the codes enter the MMA as stored -- INT8 s8 directly, INT4 as two u8
// registers per 32-bit word (w & 0x0F0F0F0F: even dims, (w >> 4) & 0x0F0F0F0F:
// odd dims) -- so K costs 0 (INT8) or 3 instructions per 8 values instead of
// the fp16 unpack's 5.  Q becomes 16-bit fixed point per query row,
// v = rint(q / s_q) with s_q = max|q| / QM, split v = 256 hi + lo with hi, lo
// in [-128, 127], and tile column n of the B operand is (query n >> 1, hi | lo):
// thread (g, t) receives rows g, g+8 of query t as (hi, lo) in (c0, c1) and
// (c2, c3), so S = 256 c0 + c1 needs no shuffle, and one 4-MMA chain per block
// replaces 8 HMMAs; the INT4 score is s_k s_q S + z_k sum(q).  Q is rounded
// to 1/32639 of its row maximum: with INT4's unsigned codes (mean 7.5) that
// error is not centred, and the first form -- odd dims kept in place as 16 n
// with 16 v on the even dims, QM = 2039 -- measured 1.6e-2 relative at ctx 16k
// with 8-sigma outliers (the tolerance is 1e-2); one SHF per word buys the
// 4 bits back (tests/test_gpu_kernels.py, scripts/acc_report.py).
// PV stays on fp16 HMMA exactly as attend_pk (the per-token V scale must ride
// in P).  The two packed column streams are kept in "score layout" during
// the loop -- thread t holds (m, l, zb, zz) of query t for block parities 0
// and 1 -- and moved to the accumulator's column layout (thread t owns
// columns 2t, 2t+1 = query (2t)&3 (+1), parity t >> 1) by to_acc_cols.
template <int FMT>
__device__ __forceinline__ void imma16832(int* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  if constexpr (FMT == kINT4)
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int FMT>
struct IqQ {
  static constexpr float kQM = 32639.f;  // |v| <= 32639: hi = (v + 128) >> 8 fits s8
};

// Q of the unit (rows of the group's head, G <= 4) -> IMMA B fragments of
// column g: query g >> 1, byte half g & 1.  qsc / qz of query t for the score
// epilogue: s_q * sml2 and sml2 * sum(q).
template <int FMT>
__device__ __forceinline__ void load_q_iq(uint32_t sQ, int g, int t, uint32_t G, float sml2,
                                          uint32_t (&qi)[4][2], float& qsc, float& qz) {
  const int qq = g >> 1;
  const bool ok = qq < static_cast<int>(G);
  const uint32_t row = sQ + qq * kD * 2;
  uint4 v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = ok ? lds128(row + 64 * t + 16 * c) : make_uint4(0, 0, 0, 0);
  float x[4][8];
  float amax = 0.f, sum = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
      x[c][2 * e] = f.x;
      x[c][2 * e + 1] = f.y;
      amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
      sum += f.x + f.y;
    }
  }
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
  sum += __shfl_xor_sync(0xffffffffu, sum, 1);
  sum += __shfl_xor_sync(0xffffffffu, sum, 2);
  const float inv = amax > 0.f ? IqQ<FMT>::kQM / amax : 0.f;
  const bool lo_half = g & 1;
  // byte of value v for this column's half: hi = (v + 128) >> 8, lo = v - 256 hi
  auto half_byte = [&](float xf) -> uint32_t {
    const int vv = __float2int_rn(xf * inv);
    const int hi = (vv + 128) >> 8;
    return static_cast<uint32_t>(lo_half ? vv - 256 * hi : hi) & 0xffu;
  };
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // k-step c: dims 32t + 8c .. +7
    uint32_t b0 = 0, b1 = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if constexpr (FMT == kINT4) {  // b0: even dims, b1: odd dims
        b0 |= half_byte(x[c][2 * j]) << (8 * j);
        b1 |= half_byte(x[c][2 * j + 1]) << (8 * j);
      } else {  // b0: dims 0..3, b1: dims 4..7
        b0 |= half_byte(x[c][j]) << (8 * j);
        b1 |= half_byte(x[c][4 + j]) << (8 * j);
      }
    }
    qi[c][0] = b0;
    qi[c][1] = b1;
  }
  const float sq = amax / IqQ<FMT>::kQM;
  // query t's values live in lanes g = 2t (any t'): broadcast to thread t
  qsc = __shfl_sync(0xffffffffu, sq, (2 * t) * 4) * sml2;
  qz = __shfl_sync(0xffffffffu, sum, (2 * t) * 4) * sml2;
}

// score layout (thread t: query t, parities 0/1, equal over g) -> the values
// of this thread's accumulator columns 2t, 2t+1 (query (2t)&3 (+1), parity t >> 1)
__device__ __forceinline__ void to_acc_cols(const float (&v)[2], int g, int t, float (&o)[2]) {
  const int q0 = (2 * t) & 3;
  const bool b = t >> 1;
  const float a0 = __shfl_sync(0xffffffffu, v[0], g * 4 + q0);
  const float a1 = __shfl_sync(0xffffffffu, v[1], g * 4 + q0);
  const float c0 = __shfl_sync(0xffffffffu, v[0], g * 4 + q0 + 1);
  const float c1 = __shfl_sync(0xffffffffu, v[1], g * 4 + q0 + 1);
  o[0] = b ? a1 : a0;
  o[1] = b ? c1 : c0;
}

// bias flush of the integer step: zb (score layout) summed over the 16 token
// rows and added to the accumulator columns
template <int FMT>
__device__ __forceinline__ void flush_bias_iq(UnitState<1>& u, int g, int t) {
  float z[2];
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    float s = u.zb[0][b];
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    z[b] = s;
    u.zb[0][b] = 0.f;
  }
  float zc[2];
  to_acc_cols(z, g, t, zc);
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      u.acc[mt][0][c] += zc[c];
      u.acc[mt][0][2 + c] += zc[c];
    }
}

// segment end: (m, l, zb, zz) from score layout to accumulator columns (the
// layout fold_halves and the epilogue expect); l/zb/zz stay per-row partials
__device__ __forceinline__ void iq_state_to_acc(UnitState<1>& u, int g, int t) {
  float o[2];
  to_acc_cols(u.m[0], g, t, o);
  u.m[0][0] = o[0]; u.m[0][1] = o[1];
  to_acc_cols(u.l[0], g, t, o);
  u.l[0][0] = o[0]; u.l[0][1] = o[1];
  to_acc_cols(u.zb[0], g, t, o);
  u.zb[0][0] = o[0]; u.zb[0][1] = o[1];
  to_acc_cols(u.zz[0], g, t, o);
  u.zz[0][0] = o[0]; u.zz[0][1] = o[1];
}

// INT4 V for the integer step: row g (low-nibble dim) is fed the whole byte,
// 1024 + 16 h + l (one PRMT per two values, no shift), row g+8 the high
// nibble in place, 1024 + 16 h (LOP3); the epilogue recovers the low dim as
// acc(g) - acc(g+8) (K2's o_lo for kIQ), so a word costs 4 instructions
// instead of 5.  The other formats load as load_v_frags.
template <int FMT>
__device__ __forceinline__ void load_v_frags_iq(uint32_t sV, const FragOff& o, uint32_t (&a)[8][4]) {
  if constexpr (FMT == kINT4) {
    const uint4 va = lds128(sV + o.v[0]);  // tokens ta, tb
    const uint4 vc = lds128(sV + o.v[1]);  // tokens ta+8, tb+8
    const uint32_t A[4] = {va.x, va.y, va.z, va.w}, C[4] = {vc.x, vc.y, vc.z, vc.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t x0 = __byte_perm(A[j], 0x64646464u, 0x4240);  // [b0 64 b2 64]: m-tile 2j
      const uint32_t x1 = __byte_perm(A[j], 0x64646464u, 0x4341);  // [b1 64 b3 64]: m-tile 2j+1
      const uint32_t y0 = __byte_perm(C[j], 0x64646464u, 0x4240);
      const uint32_t y1 = __byte_perm(C[j], 0x64646464u, 0x4341);
      a[2 * j][0] = x0;
      a[2 * j][1] = x0 & 0xFFF0FFF0u;
      a[2 * j][2] = y0;
      a[2 * j][3] = y0 & 0xFFF0FFF0u;
      a[2 * j + 1][0] = x1;
      a[2 * j + 1][1] = x1 & 0xFFF0FFF0u;
      a[2 * j + 1][2] = y1;
      a[2 * j + 1][3] = y1 & 0xFFF0FFF0u;
    }
  } else {
    load_v_frags<FMT>(sV, o, a);
  }
}

template <int FMT, int NB, bool MASK>
__device__ __forceinline__ void attend_iq(UnitState<1>& u, const uint32_t (&sbs)[2], const int (&valid)[2],
                                          uint32_t wK, uint32_t wP, uint32_t kvq, uint32_t pq,
                                          const FragOff& fo, const uint32_t (&qi)[4][2], float qsc,
                                          float qz, int g, int t) {
  using Gm = Geo<FMT>;
  // ---- scores of query t, rows g, g+8, both blocks ----
  float x[2][2], sv[2][2], zv[2][2];
#pragma unroll
  for (int bi = 0; bi < 2; ++bi) {
    if (bi >= NB) {
      x[bi][0] = x[bi][1] = -INFINITY;
      sv[bi][0] = sv[bi][1] = zv[bi][0] = zv[bi][1] = 0.f;
      continue;
    }
    const uint32_t sK = sbs[bi] + wK;
    int c[4] = {0, 0, 0, 0};
    if constexpr (FMT == kINT4) {
      const uint4 lo = lds128(sK + fo.k[0]);  // row g: dims 32t .. 32t+31
      const uint4 hi = lds128(sK + fo.k[1]);  // row g+8
      const uint32_t wl[4] = {lo.x, lo.y, lo.z, lo.w}, wh[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        imma16832<FMT>(c, wl[i] & 0x0F0F0F0Fu, wh[i] & 0x0F0F0F0Fu, (wl[i] >> 4) & 0x0F0F0F0Fu,
                       (wh[i] >> 4) & 0x0F0F0F0Fu, qi[i][0], qi[i][1]);
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 lo = lds128(sK + fo.k[h]);
        const uint4 hi = lds128(sK + fo.k[h] + 1024);
        imma16832<FMT>(c, lo.x, hi.x, lo.y, hi.y, qi[2 * h][0], qi[2 * h][1]);
        imma16832<FMT>(c, lo.z, hi.z, lo.w, hi.w, qi[2 * h + 1][0], qi[2 * h + 1][1]);
      }
    }
    const uint32_t sKp = sbs[bi] + wP, sVp = sKp + pq;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float sk, zk = 0.f;
      if constexpr (FMT == kINT4) {
        const uint32_t kp = lds32(sKp + 4 * (g + 8 * r)), vp = lds32(sVp + 4 * (g + 8 * r));
        const float2 kf = __half22float2(*reinterpret_cast<const __half2*>(&kp));
        const float2 vf = __half22float2(*reinterpret_cast<const __half2*>(&vp));
        sk = kf.x;
        zk = kf.y;
        sv[bi][r] = vf.x;
        zv[bi][r] = vf.y;
      } else {
        sk = __half2float(__ushort_as_half(lds16(sKp + 2 * (g + 8 * r))));
        sv[bi][r] = __half2float(__ushort_as_half(lds16(sVp + 2 * (g + 8 * r))));
        zv[bi][r] = 0.f;
      }
      const float s = static_cast<float>(c[2 * r] * 256 + c[2 * r + 1]);
      float xv = s * (sk * qsc);
      if constexpr (FMT == kINT4) xv = fmaf(zk, qz, xv);
      x[bi][r] = (MASK && !(g + 8 * r < valid[bi])) ? -INFINITY : xv;
    }
  }
  // ---- online softmax per parity stream (lazy rescale, as in attend) ----
  bool grow = false;
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int r = 0; r < 2; ++r) grow |= x[b][r] > u.m[0][b] + kRescaleSlack;
  if (__any_sync(0xffffffffu, grow)) {
    float al[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      float mx = fmaxf(x[b][0], x[b][1]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float mn = fmaxf(u.m[0][b], mx);
      al[b] = ex2(u.m[0][b] - mn);
      u.m[0][b] = mn;
      u.l[0][b] *= al[b];
      u.zb[0][b] *= al[b];
      u.zz[0][b] *= al[b];
    }
    float ac[2];
    to_acc_cols(al, g, t, ac);
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        u.acc[mt][0][c] *= ac[c];
        u.acc[mt][0][2 + c] *= ac[c];
      }
  }
  float pr[2][2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int r = 0; r < 2; ++r) pr[b][r] = ex2(x[b][r] - u.m[0][b]);
  // P' = p * s_v per token, one half2 per row holding both parities
  const uint32_t hr0 = pack_h2(pr[0][0] * sv[0][0], pr[1][0] * sv[1][0]);  // row g
  const uint32_t hr1 = pack_h2(pr[0][1] * sv[0][1], pr[1][1] * sv[1][1]);  // row g+8
  {
    const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&hr0));
    const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&hr1));
    u.zb[0][0] -= Gm::kBias * (f0.x + f1.x);  // the bias term of the exact fp16 P' the MMA sees
    u.zb[0][1] -= Gm::kBias * (f0.y + f1.y);
  }
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    u.l[0][b] += pr[b][0] + pr[b][1];
    if constexpr (FMT == kINT4) u.zz[0][b] = fmaf(pr[b][0], zv[b][0], fmaf(pr[b][1], zv[b][1], u.zz[0][b]));
  }
  // ---- P'^T B fragments: column g = (query g & 3, parity g >> 2) ----
  const int q = g & 3;
  const int sa = tok_a<FMT>(t) * 4 + q, sb = tok_b<FMT>(t) * 4 + q;
  const uint32_t ya0 = __shfl_sync(0xffffffffu, hr0, sa), yb0 = __shfl_sync(0xffffffffu, hr0, sb);
  const uint32_t ya1 = __shfl_sync(0xffffffffu, hr1, sa), yb1 = __shfl_sync(0xffffffffu, hr1, sb);
  const uint32_t sel = (g >> 2) ? 0x7632u : 0x5410u;
  const uint32_t pb0 = __byte_perm(ya0, yb0, sel), pb1 = __byte_perm(ya1, yb1, sel);
  // ---- O^T += V^T . P^T: block bi feeds only its own columns ----
#pragma unroll
  for (int bi = 0; bi < NB; ++bi) {
    const bool mine = (g >> 2) == bi;
    const uint32_t b0 = mine ? pb0 : 0u, b1 = mine ? pb1 : 0u;
    uint32_t va[8][4];
    load_v_frags_iq<FMT>(sbs[bi] + kvq + wK, fo, va);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) mma16816(u.acc[mt][0], va[mt][0], va[mt][1], va[mt][2], va[mt][3], b0, b1);
  }
}

// Folds the two packed streams (columns c and c + 4 = lanes t and t ^ 2) of
// every query into one online-softmax state, as the merge kernel does.
// Afterwards threads t < 2 hold the unit segment's state of queries 2t, 2t+1.
__device__ __forceinline__ void fold_halves(UnitState<1>& u) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float mo = __shfl_xor_sync(0xffffffffu, u.m[0][c], 2);
    const float mn = fmaxf(u.m[0][c], mo);
    const float a = ex2(u.m[0][c] - mn);
    u.m[0][c] = mn;
    auto f = [&](float x) {
      x *= a;
      return x + __shfl_xor_sync(0xffffffffu, x, 2);
    };
    u.l[0][c] = f(u.l[0][c]);
    u.zb[0][c] = f(u.zb[0][c]);
    u.zz[0][c] = f(u.zz[0][c]);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      u.acc[mt][0][c] = f(u.acc[mt][0][c]);
      u.acc[mt][0][2 + c] = f(u.acc[mt][0][2 + c]);
    }
  }
}

}  // namespace dev
}  // namespace kvslab
