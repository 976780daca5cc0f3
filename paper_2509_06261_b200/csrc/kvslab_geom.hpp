// kvslab_geom.hpp -- host/device-shared slab geometry (fast divide by
// blocks-per-slab, block byte offsets).  Safe to include from plain C++.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define KS_HD __host__ __device__ __forceinline__
#else
#define KS_HD inline
#endif

namespace kvslab {
namespace dev {

KS_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}

// Unsigned 32-bit division by a runtime-constant divisor (Granlund-Montgomery,
// round-up variant): q = (umulhi(n, m) + n) >> s, exact for all n < 2^32.
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  uint32_t l = 0;
  while ((uint64_t{1} << l) < d) ++l;
  f.s = l;
  f.m = static_cast<uint32_t>(((uint64_t{1} << 32) * ((uint64_t{1} << l) - d)) / d + 1);
  return f;
}
KS_HD uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return static_cast<uint32_t>((static_cast<uint64_t>(umulhi32(n, f.m)) + n) >> f.s);
}

// Where a model's blocks live: byte offset of global block id g is
// (g / bps) * slab_size + (g % bps) * key.
struct SlabGeom {
  uint64_t slab_size;
  uint64_t key;
  FastDiv bps;
};
KS_HD uint64_t block_offset(const SlabGeom& g, uint32_t gid) {
  const uint32_t slab = fdiv(gid, g.bps);
  const uint32_t local = gid - slab * g.bps.d;
  return static_cast<uint64_t>(slab) * g.slab_size + static_cast<uint64_t>(local) * g.key;
}

}  // namespace dev
}  // namespace kvslab
