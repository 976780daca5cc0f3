/* kvslab_oracle.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY (see kvslab_oracle.h).
 *
 * Plain C, compiled with -ffp-contract=off so every float operation is a
 * single IEEE-754 round-to-nearest-even step, which is what the CUDA append
 * kernel does with explicit __fdiv_rn/__fsub_rn intrinsics.  Deliberately
 * naive: O(num_slabs) scans, scalar loops, fp64 attention.
 */
#include "kvslab_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ======================= RNG =========================================
 * Restates slabsim::Rng (workload.hpp:32-48): std::mt19937_64 seeded with
 * the 64-bit seed, uniform01 = (word >> 11) * 2^-53. */
#define MT_N 312
#define MT_M 156
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}
static void mt_twist(orc_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}
uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}
double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
void orc_rng_fill_uniform(orc_rng* r, double* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_rng_uniform01(r);
}

/* ======================= geometry (precision.cpp:76-99) ================ */
int orc_token_size(uint32_t num_kv_heads, uint32_t head_dim, uint32_t tp_degree, int kv_bits,
                   uint64_t* out) {
  if (tp_degree == 0 || num_kv_heads % tp_degree != 0) return -1;
  uint64_t bits = (uint64_t)(num_kv_heads / tp_degree) * head_dim * 2ULL * (uint64_t)kv_bits;
  if (bits % 8 != 0) return -1;
  *out = bits / 8;
  return 0;
}
int orc_kv_block_size(uint32_t num_kv_heads, uint32_t head_dim, uint32_t tp_degree, int kv_bits,
                      uint64_t tpb, uint64_t qparams, uint32_t num_layers, uint64_t* out) {
  uint64_t ts;
  if (tpb < 1) return -1;
  if (orc_token_size(num_kv_heads, head_dim, tp_degree, kv_bits, &ts) != 0) return -1;
  *out = (uint64_t)num_layers * (tpb * ts + qparams);
  return 0;
}

/* ======================= slab allocator (slab_pool.cpp:51-272) ========= */
typedef struct {
  uint64_t key; /* 0 = FREE / unformatted */
  uint32_t total, used;
  uint8_t* bits; /* one byte per block, naive on purpose */
} orc_slab;
struct orc_pool {
  uint64_t slab_size;
  uint32_t nslabs, nkeys;
  uint64_t keys[64];
  orc_slab* slabs;
  uint64_t st[4]; /* allocated, free_block, residue, free_slab */
};

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int orc_pool_create(uint64_t capacity, uint64_t slab_size, const uint64_t* keys, uint32_t nkeys,
                    int require_lcm, orc_pool** out) {
  if (slab_size == 0 || nkeys == 0 || nkeys > 64) return ORC_INVALID_CONFIG;
  uint64_t k[64];
  memcpy(k, keys, nkeys * sizeof(uint64_t));
  qsort(k, nkeys, sizeof(uint64_t), cmp_u64);
  uint32_t n = 0;
  for (uint32_t i = 0; i < nkeys; ++i)
    if (n == 0 || k[n - 1] != k[i]) k[n++] = k[i];
  for (uint32_t i = 0; i < n; ++i)
    if (k[i] == 0 || k[i] > slab_size) return ORC_INVALID_CONFIG;
  if (require_lcm) {
    uint64_t l = 1;
    for (uint32_t i = 0; i < n; ++i) {
      l = l / gcd_u64(l, k[i]) * k[i];
      if (l > slab_size) return ORC_INVALID_CONFIG;
    }
    if (slab_size % l != 0) return ORC_INVALID_CONFIG;
  }
  uint64_t nslabs = capacity / slab_size;
  if (nslabs == 0) return ORC_INVALID_CONFIG;
  orc_pool* p = (orc_pool*)calloc(1, sizeof(orc_pool));
  p->slab_size = slab_size;
  p->nslabs = (uint32_t)nslabs;
  p->nkeys = n;
  memcpy(p->keys, k, n * sizeof(uint64_t));
  p->slabs = (orc_slab*)calloc(nslabs, sizeof(orc_slab));
  p->st[3] = nslabs * slab_size;
  *out = p;
  return ORC_OK;
}
void orc_pool_destroy(orc_pool* p) {
  if (!p) return;
  for (uint32_t i = 0; i < p->nslabs; ++i) free(p->slabs[i].bits);
  free(p->slabs);
  free(p);
}
static int key_known(const orc_pool* p, uint64_t key) {
  for (uint32_t i = 0; i < p->nkeys; ++i)
    if (p->keys[i] == key) return 1;
  return 0;
}
static void slab_format(orc_pool* p, uint32_t s, uint64_t key) {
  orc_slab* sl = &p->slabs[s];
  sl->key = key;
  sl->total = (uint32_t)(p->slab_size / key);
  sl->used = 0;
  sl->bits = (uint8_t*)calloc(sl->total ? sl->total : 1, 1);
  uint64_t blk = (uint64_t)sl->total * key;
  p->st[3] -= p->slab_size;
  p->st[1] += blk;
  p->st[2] += p->slab_size - blk;
}
static void slab_unformat(orc_pool* p, uint32_t s) {
  orc_slab* sl = &p->slabs[s];
  uint64_t blk = (uint64_t)sl->total * sl->key;
  p->st[1] -= blk;
  p->st[2] -= p->slab_size - blk;
  p->st[3] += p->slab_size;
  free(sl->bits);
  memset(sl, 0, sizeof(*sl));
}
static uint32_t slab_take_lowest(orc_pool* p, uint32_t s) {
  orc_slab* sl = &p->slabs[s];
  for (uint32_t l = 0; l < sl->total; ++l)
    if (!sl->bits[l]) {
      sl->bits[l] = 1;
      sl->used++;
      p->st[0] += sl->key;
      p->st[1] -= sl->key;
      return l;
    }
  abort();
}
int orc_pool_alloc(orc_pool* p, uint64_t key, orc_handle* out) {
  if (!key_known(p, key)) return ORC_INVALID_KEY;
  int64_t pick = -1;
  for (uint32_t s = 0; s < p->nslabs && pick < 0; ++s)
    if (p->slabs[s].key == key && p->slabs[s].used < p->slabs[s].total) pick = s;
  if (pick < 0) {
    for (uint32_t s = 0; s < p->nslabs && pick < 0; ++s)
      if (p->slabs[s].key == 0) pick = s;
    if (pick < 0) return ORC_EXHAUSTED;
    slab_format(p, (uint32_t)pick, key);
  }
  uint32_t l = slab_take_lowest(p, (uint32_t)pick);
  out->slab_id = (uint32_t)pick;
  out->local_block_id = l;
  out->global_block_id = (uint64_t)pick * p->slabs[pick].total + l;
  out->key = key;
  return ORC_OK;
}
int orc_pool_free(orc_pool* p, const orc_handle* h) {
  if (h->slab_id >= p->nslabs) return ORC_INVALID_FREE;
  orc_slab* sl = &p->slabs[h->slab_id];
  if (sl->key == 0 || sl->key != h->key || h->local_block_id >= sl->total ||
      h->global_block_id != (uint64_t)h->slab_id * sl->total + h->local_block_id)
    return ORC_INVALID_FREE;
  if (!sl->bits[h->local_block_id]) return ORC_INVALID_FREE;
  sl->bits[h->local_block_id] = 0;
  sl->used--;
  p->st[0] -= h->key;
  p->st[1] += h->key;
  if (sl->used == 0) slab_unformat(p, h->slab_id);
  return ORC_OK;
}
void orc_pool_stats(const orc_pool* p, uint64_t out[4]) { memcpy(out, p->st, sizeof(p->st)); }
uint32_t orc_pool_slab_count(const orc_pool* p) { return p->nslabs; }
void orc_pool_slab(const orc_pool* p, uint32_t s, int* state, uint64_t* key, uint32_t* used,
                   uint32_t* total) {
  const orc_slab* sl = &p->slabs[s];
  *state = sl->key == 0 ? 0 : (sl->used == sl->total ? 2 : 1);
  *key = sl->key;
  *used = sl->used;
  *total = sl->total;
}
int orc_pool_bit(const orc_pool* p, uint32_t s, uint32_t l) {
  if (s >= p->nslabs || p->slabs[s].key == 0 || l >= p->slabs[s].total) return -1;
  return p->slabs[s].bits[l];
}

/* ======================= compaction plan (new) ===== */
uint32_t orc_compact_plan(orc_pool* p, uint64_t key, uint32_t max_moves, uint64_t* src_gid,
                          uint64_t* dst_gid, uint32_t* slabs_freed) {
  uint32_t n = p->nslabs, nc = 0, moves = 0, freed = 0;
  uint32_t* cand = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint8_t* evac = (uint8_t*)calloc(n, 1);
  uint8_t* recv = (uint8_t*)calloc(n, 1);
  for (uint32_t s = 0; s < n; ++s)
    if (p->slabs[s].key == key && p->slabs[s].used < p->slabs[s].total) cand[nc++] = s;
  /* sources: (used asc, slab desc) -- insertion sort, naive on purpose */
  for (uint32_t i = 1; i < nc; ++i)
    for (uint32_t j = i; j > 0; --j) {
      uint32_t a = cand[j - 1], b = cand[j];
      int swap = p->slabs[b].used < p->slabs[a].used ||
                 (p->slabs[b].used == p->slabs[a].used && b > a);
      if (!swap) break;
      cand[j - 1] = b;
      cand[j] = a;
    }
  for (uint32_t ci = 0; ci < nc; ++ci) {
    uint32_t S = cand[ci];
    if (recv[S] || p->slabs[S].key != key) continue;
    uint32_t need = p->slabs[S].used;
    /* destination capacity: partial slabs of the key, not S, not evacuated */
    uint64_t cap = 0;
    for (uint32_t d = 0; d < n; ++d)
      if (d != S && !evac[d] && p->slabs[d].key == key)
        cap += p->slabs[d].total - p->slabs[d].used;
    if (cap < need || moves + need > max_moves) break;
    for (uint32_t l = 0; l < p->slabs[S].total; ++l) {
      if (!p->slabs[S].bits[l]) continue;
      /* pick destination: (used desc, slab asc) among slabs with room */
      int64_t D = -1;
      for (uint32_t d = 0; d < n; ++d) {
        if (d == S || evac[d] || p->slabs[d].key != key) continue;
        if (p->slabs[d].used >= p->slabs[d].total) continue;
        if (D < 0 || p->slabs[d].used > p->slabs[D].used) D = d;
      }
      uint32_t dl = slab_take_lowest(p, (uint32_t)D);
      recv[D] = 1;
      src_gid[moves] = (uint64_t)S * p->slabs[S].total + l;
      dst_gid[moves] = (uint64_t)D * p->slabs[D].total + dl;
      moves++;
      orc_handle h = {S, l, (uint64_t)S * p->slabs[S].total + l, key};
      int slab_will_empty = p->slabs[S].used == 1;
      orc_pool_free(p, &h);
      if (slab_will_empty) break;
    }
    evac[S] = 1;
    freed++;
  }
  free(cand);
  free(evac);
  free(recv);
  if (slabs_freed) *slabs_freed = freed;
  return moves;
}

/* ======================= number formats ================================ */
uint16_t orc_f32_to_f16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) return (uint16_t)(sign | (ax > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* >= 65520 -> inf */
  if (ax <= 0x33000000u) return (uint16_t)sign;             /* <= 2^-25 -> 0 (ties to even) */
  int e = (int)(ax >> 23) - 127;
  uint32_t mant = ax & 0x7fffffu;
  if (e < -14) { /* half subnormal: q = m * 2^(e+1), round to nearest even */
    uint32_t m = mant | 0x800000u;
    int s = -(e + 1);
    uint32_t q = m >> s, rem = m & ((1u << s) - 1u), half = 1u << (s - 1);
    if (rem > half || (rem == half && (q & 1u))) q++;
    return (uint16_t)(sign | q);
  }
  uint32_t h = ((uint32_t)(e + 15) << 10) | (mant >> 13);
  uint32_t rem = mant & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  return (uint16_t)(sign | h);
}
float orc_f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1f, m = h & 0x3ff;
  float v;
  if (e == 0)
    v = ldexpf((float)m, -24);
  else if (e == 31)
    v = m ? NAN : INFINITY;
  else
    v = ldexpf((float)(m | 0x400u), (int)e - 25);
  uint32_t x;
  memcpy(&x, &v, 4);
  x |= sign;
  memcpy(&v, &x, 4);
  return v;
}
/* OCP E4M3 (fn): bias 7, no inf, max 448, NaN = S.1111.111.  Round to
 * nearest even, saturate finite overflow to +-448 (the __NV_SATFINITE
 * behaviour of __nv_cvt_float_to_fp8). */
uint8_t orc_f32_to_e4m3(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint8_t sign = (uint8_t)((x >> 24) & 0x80u);
  if ((x & 0x7fffffffu) > 0x7f800000u) return 0x7f;
  float a = fabsf(f);
  if (a >= 448.0f) return (uint8_t)(sign | 0x7e);
  if (a < 0.015625f) { /* < 2^-6: subnormal grid of 2^-9 */
    float q = rintf(a * 512.0f);
    return (uint8_t)(sign | (uint8_t)q);
  }
  int e;
  float fr = frexpf(a, &e); /* a = fr * 2^e, fr in [0.5,1) */
  int E = e - 1;
  float m = rintf((fr * 2.0f - 1.0f) * 8.0f);
  int q = (int)m;
  if (q == 8) {
    E++;
    q = 0;
  }
  int code = ((E + 7) << 3) | q;
  if (code > 0x7e) code = 0x7e;
  return (uint8_t)(sign | code);
}
float orc_e4m3_to_f32(uint8_t c) {
  float s = (c & 0x80) ? -1.0f : 1.0f;
  if ((c & 0x7f) == 0x7f) return NAN;
  int E = (c >> 3) & 15, m = c & 7;
  if (E == 0) return s * ldexpf((float)m, -9);
  return s * ldexpf((float)(8 + m), E - 10);
}

/* ======================= layout ==================== */
static uint32_t fmt_bits(const orc_fmt* f) {
  return f->kv_dtype == ORC_FP16 ? 16 : (f->kv_dtype == ORC_INT4 ? 4 : 8);
}
uint64_t orc_fmt_token_size(const orc_fmt* f) {
  return (uint64_t)f->num_kv_heads * f->head_dim * 2 * fmt_bits(f) / 8;
}
uint64_t orc_fmt_chunk_bytes(const orc_fmt* f) {
  return (uint64_t)f->tokens_per_block * f->head_dim * fmt_bits(f) / 8;
}
uint64_t orc_fmt_layer_bytes(const orc_fmt* f) {
  return (uint64_t)f->tokens_per_block * orc_fmt_token_size(f) + f->qparams;
}
uint64_t orc_fmt_key(const orc_fmt* f) { return (uint64_t)f->num_layers * orc_fmt_layer_bytes(f); }
uint64_t orc_fmt_natural_qparams(const orc_fmt* f) {
  uint64_t H = f->num_kv_heads, T = f->tokens_per_block;
  switch (f->kv_dtype) {
    case ORC_FP8: return 2 * H * 4;     /* fp32 scale per (K|V, head) */
    case ORC_INT8: return 2 * H * T * 2; /* fp16 scale per (K|V, head, token) */
    case ORC_INT4: return 2 * H * T * 4; /* fp16 (scale, zero) per (K|V, head, token) */
    default: return 0;
  }
}
uint64_t orc_swz(uint64_t o) { return o ^ (((o >> 7) & 7ULL) << 4); }
uint64_t orc_block_offset(uint64_t slab_size, uint64_t key, uint64_t bps, uint64_t gid) {
  return (gid / bps) * slab_size + (gid % bps) * key;
}
/* byte offset of chunk (kv, head) of layer inside a block */
static uint64_t chunk_off(const orc_fmt* f, uint32_t layer, uint32_t kv, uint32_t head) {
  return (uint64_t)layer * orc_fmt_layer_bytes(f) +
         ((uint64_t)kv * f->num_kv_heads + head) * orc_fmt_chunk_bytes(f);
}
static uint64_t params_off(const orc_fmt* f, uint32_t layer) {
  return (uint64_t)layer * orc_fmt_layer_bytes(f) + 2ULL * f->num_kv_heads * orc_fmt_chunk_bytes(f);
}

/* FP16 element i of token slot: 64-element halves are stored half-major
 * ([dims 0-63 of all T tokens][dims 64-127 of all T tokens], 128-byte rows),
 * so each half of a chunk is a 128B-swizzled UMMA operand as it lies
 * (DESIGN.md section 3); head dims that are not a multiple of 64 keep plain
 * token rows. */
static uint64_t fp16_off(const orc_fmt* f, uint32_t slot, uint32_t i) {
  const uint32_t d = f->head_dim, T = f->tokens_per_block;
  if (d % 64 != 0) return orc_swz((uint64_t)slot * d * 2 + 2ULL * i);
  return orc_swz((uint64_t)(i / 64) * T * 128 + (uint64_t)slot * 128 + 2ULL * (i % 64));
}

/* INT4 byte j (dims 2j, 2j+1) of token slot.  K: 64-byte token rows.  V (with
 * T = 16, d = 128, as the kernels require): the PV fragment's token pair
 * (tok_a, tok_b) = ({0,1,4,5}, {2,3,6,7}) (+8) shares one 128-byte line,
 * interleaved in 2-byte units; other geometries keep
 * token rows. */
static uint64_t int4_off(const orc_fmt* f, uint32_t kv, uint32_t slot, uint32_t j) {
  const uint32_t d = f->head_dim, T = f->tokens_per_block;
  if (kv == 0 || d != 128 || T != 16) return orc_swz((uint64_t)slot * (d / 2) + j);
  const uint32_t t8 = slot & 7, tp = (t8 & 1) | ((t8 >> 2) << 1), side = (t8 >> 1) & 1;
  const uint32_t line = 2 * tp + (slot >> 3);
  return orc_swz((uint64_t)line * 128 + 4 * (j >> 1) + 2 * side + (j & 1));
}

/* ======================= quantised append (K1 restated) ================== */
static void quant_row(const orc_fmt* f, const uint16_t* x16, float fp8_scale, uint8_t* chunk,
                      uint32_t slot, uint8_t* params, uint32_t kv, uint32_t head) {
  uint32_t d = f->head_dim, T = f->tokens_per_block, H = f->num_kv_heads;
  uint64_t rowb = (uint64_t)d * fmt_bits(f) / 8, base = (uint64_t)slot * rowb;
  float x[1024] = {0};
  if (d == 0 || d > 1024) return;
  for (uint32_t i = 0; i < d; ++i) x[i] = orc_f16_to_f32(x16[i]);
  if (f->kv_dtype == ORC_FP16) {
    for (uint32_t i = 0; i < d; ++i) {
      uint64_t o = fp16_off(f, slot, i);
      chunk[o] = (uint8_t)(x16[i] & 0xff);
      chunk[o + 1] = (uint8_t)(x16[i] >> 8);
    }
  } else if (f->kv_dtype == ORC_FP8) {
    for (uint32_t i = 0; i < d; ++i) chunk[orc_swz(base + i)] = orc_f32_to_e4m3(x[i] / fp8_scale);
    if (f->qparams >= orc_fmt_natural_qparams(f)) {
      uint8_t* ps = params + ((uint64_t)kv * H + head) * 4;
      memcpy(ps, &fp8_scale, 4);
    }
  } else if (f->kv_dtype == ORC_INT8) {
    float amax = 0.0f;
    for (uint32_t i = 0; i < d; ++i) amax = fmaxf(amax, fabsf(x[i]));
    uint16_t sh = orc_f32_to_f16(amax / 127.0f);
    float sf = orc_f16_to_f32(sh);
    for (uint32_t i = 0; i < d; ++i) {
      int q = 0;
      if (sf != 0.0f) {
        float t = rintf(x[i] / sf);
        q = t > 127.0f ? 127 : (t < -127.0f ? -127 : (int)t);
      }
      chunk[orc_swz(base + i)] = (uint8_t)(int8_t)q;
    }
    uint8_t* ps = params + (((uint64_t)kv * H + head) * T + slot) * 2;
    ps[0] = (uint8_t)(sh & 0xff);
    ps[1] = (uint8_t)(sh >> 8);
  } else { /* INT4, asymmetric per (token, head) group of d */
    float mn = x[0], mx = x[0];
    for (uint32_t i = 1; i < d; ++i) {
      mn = fminf(mn, x[i]);
      mx = fmaxf(mx, x[i]);
    }
    uint16_t sh = orc_f32_to_f16((mx - mn) / 15.0f);
    uint16_t zh = orc_f32_to_f16(mn);
    /* a NaN parameter (an all-NaN row, or inf - inf) is stored as the one
       encoding 0x7e00: the sign of a generated NaN is platform-defined */
    if ((sh & 0x7fffu) > 0x7c00u) sh = 0x7e00u;
    if ((zh & 0x7fffu) > 0x7c00u) zh = 0x7e00u;
    float sf = orc_f16_to_f32(sh), zf = orc_f16_to_f32(zh);
    for (uint32_t i = 0; i < d; i += 2) {
      int q[2];
      for (int j = 0; j < 2; ++j) {
        q[j] = 0;
        if (sf != 0.0f) {
          float t = rintf((x[i + j] - zf) / sf);
          q[j] = t > 15.0f ? 15 : (t < 0.0f ? 0 : (int)t);
        }
      }
      chunk[int4_off(f, kv, slot, i / 2)] = (uint8_t)(q[0] | (q[1] << 4));
    }
    uint8_t* ps = params + (((uint64_t)kv * H + head) * T + slot) * 4;
    ps[0] = (uint8_t)(sh & 0xff);
    ps[1] = (uint8_t)(sh >> 8);
    ps[2] = (uint8_t)(zh & 0xff);
    ps[3] = (uint8_t)(zh >> 8);
  }
}

void orc_append(uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f, uint32_t layer,
                const uint16_t* k, const uint16_t* v, uint32_t n_tok, const int32_t* tok_seq,
                const int32_t* tok_pos, const int32_t* block_table, uint32_t bt_stride,
                const float* kv_scales) {
  uint32_t H = f->num_kv_heads, d = f->head_dim, T = f->tokens_per_block;
  uint64_t key = orc_fmt_key(f);
  for (uint32_t i = 0; i < n_tok; ++i) {
    int32_t s = tok_seq[i], pos = tok_pos[i];
    int32_t gid = block_table[(uint64_t)s * bt_stride + (uint32_t)pos / T];
    uint8_t* blk = pool + orc_block_offset(slab_size, key, bps, (uint64_t)gid);
    for (uint32_t h = 0; h < H; ++h)
      for (uint32_t kv = 0; kv < 2; ++kv) {
        const uint16_t* x = (kv == 0 ? k : v) + ((uint64_t)i * H + h) * d;
        float sc = kv_scales ? kv_scales[kv * H + h] : 1.0f;
        quant_row(f, x, sc, blk + chunk_off(f, layer, kv, h), (uint32_t)pos % T,
                  blk + params_off(f, layer), kv, h);
      }
  }
}

void orc_dequant(const uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                 uint32_t layer, uint64_t gid, uint32_t kv, uint32_t head, uint32_t slot,
                 const float* kv_scales, double* out) {
  uint32_t d = f->head_dim, T = f->tokens_per_block, H = f->num_kv_heads;
  const uint8_t* blk = pool + orc_block_offset(slab_size, orc_fmt_key(f), bps, gid);
  const uint8_t* chunk = blk + chunk_off(f, layer, kv, head);
  const uint8_t* params = blk + params_off(f, layer);
  uint64_t rowb = (uint64_t)d * fmt_bits(f) / 8, base = (uint64_t)slot * rowb;
  if (f->kv_dtype == ORC_FP16) {
    for (uint32_t i = 0; i < d; ++i) {
      uint64_t o = fp16_off(f, slot, i);
      out[i] = orc_f16_to_f32((uint16_t)(chunk[o] | (chunk[o + 1] << 8)));
    }
  } else if (f->kv_dtype == ORC_FP8) {
    double sc = kv_scales ? kv_scales[kv * H + head] : 1.0;
    for (uint32_t i = 0; i < d; ++i) out[i] = (double)orc_e4m3_to_f32(chunk[orc_swz(base + i)]) * sc;
  } else if (f->kv_dtype == ORC_INT8) {
    const uint8_t* ps = params + (((uint64_t)kv * H + head) * T + slot) * 2;
    double sf = orc_f16_to_f32((uint16_t)(ps[0] | (ps[1] << 8)));
    for (uint32_t i = 0; i < d; ++i) out[i] = (double)(int8_t)chunk[orc_swz(base + i)] * sf;
  } else {
    const uint8_t* ps = params + (((uint64_t)kv * H + head) * T + slot) * 4;
    double sf = orc_f16_to_f32((uint16_t)(ps[0] | (ps[1] << 8)));
    double zf = orc_f16_to_f32((uint16_t)(ps[2] | (ps[3] << 8)));
    for (uint32_t i = 0; i < d; ++i) {
      uint8_t b = chunk[int4_off(f, kv, slot, i / 2)];
      int q = (i & 1) ? (b >> 4) : (b & 15);
      out[i] = (double)q * sf + zf;
    }
  }
}

/* ======================= fp64 paged decode (K2 restated) ================= */
void orc_paged_decode(const uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                      uint32_t layer, const uint16_t* q, const int32_t* block_table,
                      uint32_t bt_stride, const int32_t* ctx_lens, uint32_t batch,
                      double sm_scale, const float* kv_scales, double* out, double* lse,
                      int nthreads) {
  const uint32_t H = f->num_kv_heads, Hq = f->num_q_heads, d = f->head_dim,
                 T = f->tokens_per_block, G = Hq / H;
  const int64_t units = (int64_t)batch * H;
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t u = 0; u < units; ++u) {
    uint32_t s = (uint32_t)(u / H), h = (uint32_t)(u % H);
    int32_t n = ctx_lens[s];
    double* qd = (double*)malloc(sizeof(double) * G * d);
    double* sc = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * G);
    double* acc = (double*)calloc((size_t)G * d, sizeof(double));
    double* kk = (double*)malloc(sizeof(double) * d);
    for (uint32_t g = 0; g < G; ++g)
      for (uint32_t i = 0; i < d; ++i)
        qd[g * d + i] = orc_f16_to_f32(q[((uint64_t)s * Hq + h * G + g) * d + i]);
    for (int32_t t = 0; t < n; ++t) {
      uint64_t gid = (uint64_t)block_table[(uint64_t)s * bt_stride + (uint32_t)t / T];
      orc_dequant(pool, slab_size, bps, f, layer, gid, 0, h, (uint32_t)t % T, kv_scales, kk);
      for (uint32_t g = 0; g < G; ++g) {
        double dot = 0.0;
        for (uint32_t i = 0; i < d; ++i) dot += qd[g * d + i] * kk[i];
        sc[(size_t)t * G + g] = dot * sm_scale;
      }
    }
    for (uint32_t g = 0; g < G; ++g) {
      double m = -INFINITY, l = 0.0;
      for (int32_t t = 0; t < n; ++t) m = fmax(m, sc[(size_t)t * G + g]);
      for (int32_t t = 0; t < n; ++t) {
        double p = exp(sc[(size_t)t * G + g] - m);
        sc[(size_t)t * G + g] = p;
        l += p;
      }
      if (lse) lse[(uint64_t)s * Hq + h * G + g] = n > 0 ? m + log(l) : -INFINITY;
      for (int32_t t = 0; t < n; ++t) sc[(size_t)t * G + g] /= l;
    }
    for (int32_t t = 0; t < n; ++t) {
      uint64_t gid = (uint64_t)block_table[(uint64_t)s * bt_stride + (uint32_t)t / T];
      orc_dequant(pool, slab_size, bps, f, layer, gid, 1, h, (uint32_t)t % T, kv_scales, kk);
      for (uint32_t g = 0; g < G; ++g) {
        double p = sc[(size_t)t * G + g];
        for (uint32_t i = 0; i < d; ++i) acc[g * d + i] += p * kk[i];
      }
    }
    for (uint32_t g = 0; g < G; ++g)
      for (uint32_t i = 0; i < d; ++i)
        out[((uint64_t)s * Hq + h * G + g) * d + i] = acc[g * d + i];
    free(qd);
    free(sc);
    free(acc);
    free(kk);
  }
}

/* Chunked-prefill attention over slab blocks (the
 * prefill claim of simulator.cpp:500-526 reserves the blocks, K1 writes the
 * chunk's K/V).  Sequence s contributes n_s = cu_q[s+1]-cu_q[s] query tokens
 * at positions ctx_lens[s]-n_s .. ctx_lens[s]-1; the query at position p
 * attends keys 0..p (causal).  fp64 softmax over the dequantised bytes. */
void orc_paged_prefill(const uint8_t* pool, uint64_t slab_size, uint64_t bps, const orc_fmt* f,
                       uint32_t layer, const uint16_t* q, const int32_t* block_table,
                       uint32_t bt_stride, const int32_t* cu_q, const int32_t* ctx_lens,
                       uint32_t batch, double sm_scale, const float* kv_scales, double* out,
                       double* lse, int nthreads) {
  const uint32_t H = f->num_kv_heads, Hq = f->num_q_heads, d = f->head_dim,
                 T = f->tokens_per_block, G = Hq / H;
  const int64_t units = (int64_t)batch * H;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t u = 0; u < units; ++u) {
    uint32_t s = (uint32_t)(u / H), h = (uint32_t)(u % H);
    int32_t n = ctx_lens[s], nq = cu_q[s + 1] - cu_q[s];
    if (nq <= 0) continue;
    double* kk = (double*)malloc(sizeof(double) * (size_t)n * d);
    double* vv = (double*)malloc(sizeof(double) * (size_t)n * d);
    double* sc = (double*)malloc(sizeof(double) * (size_t)n);
    double* qd = (double*)malloc(sizeof(double) * d);
    for (int32_t t = 0; t < n; ++t) {
      uint64_t gid = (uint64_t)block_table[(uint64_t)s * bt_stride + (uint32_t)t / T];
      orc_dequant(pool, slab_size, bps, f, layer, gid, 0, h, (uint32_t)t % T, kv_scales, kk + (size_t)t * d);
      orc_dequant(pool, slab_size, bps, f, layer, gid, 1, h, (uint32_t)t % T, kv_scales, vv + (size_t)t * d);
    }
    for (int32_t i = 0; i < nq; ++i) {
      const int32_t pos = n - nq + i;
      const uint64_t row0 = (uint64_t)(cu_q[s] + i) * Hq + h * G;
      for (uint32_t g = 0; g < G; ++g) {
        for (uint32_t e = 0; e < d; ++e) qd[e] = orc_f16_to_f32(q[(row0 + g) * d + e]);
        double m = -INFINITY, l = 0.0;
        for (int32_t t = 0; t <= pos; ++t) {
          double dot = 0.0;
          for (uint32_t e = 0; e < d; ++e) dot += qd[e] * kk[(size_t)t * d + e];
          sc[t] = dot * sm_scale;
          m = fmax(m, sc[t]);
        }
        for (int32_t t = 0; t <= pos; ++t) {
          sc[t] = exp(sc[t] - m);
          l += sc[t];
        }
        if (lse) lse[row0 + g] = m + log(l);
        double* o = out + (row0 + g) * d;
        for (uint32_t e = 0; e < d; ++e) o[e] = 0.0;
        for (int32_t t = 0; t <= pos; ++t) {
          const double p = sc[t] / l;
          for (uint32_t e = 0; e < d; ++e) o[e] += p * vv[(size_t)t * d + e];
        }
      }
    }
    free(kk);
    free(vv);
    free(sc);
    free(qd);
  }
}

uint64_t orc_decode_bytes(const orc_fmt* f, const int32_t* ctx_lens, uint32_t batch) {
  uint64_t ts = orc_fmt_token_size(f), T = f->tokens_per_block, total = 0;
  for (uint32_t s = 0; s < batch; ++s) {
    uint64_t n = (uint64_t)(ctx_lens[s] > 0 ? ctx_lens[s] : 0), nb = (n + T - 1) / T;
    total += n * ts + nb * f->qparams + nb * 4;
  }
  total += 2ULL * batch * f->num_q_heads * f->head_dim * 2;
  return total;
}
