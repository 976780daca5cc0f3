// func_cache.cpp -- see func_cache.hpp.
#include "func_cache.hpp"

#include <map>
#include <mutex>
#include <tuple>

namespace kvslab {
namespace {
std::mutex g_mu;
std::map<std::pair<const void*, int>, size_t> g_smem;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

cudaError_t ensure_dynamic_smem(const void* fn, size_t smem) {
  const auto k = std::make_pair(fn, current_device());
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_smem.find(k);
  if (it != g_smem.end() && it->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e == cudaSuccess) g_smem[k] = smem;
  return e;
}

cudaError_t cached_occupancy(const void* fn, int threads, size_t smem, int* per_sm) {
  const auto k = std::make_tuple(fn, current_device(), threads, smem);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(k);
    if (it != g_occ.end()) {
      *per_sm = it->second;
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fn, threads, smem);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_occ[k] = *per_sm;
  }
  return e;
}

}  // namespace kvslab
