// func_cache.hpp -- per-(kernel, device) launch attributes, set once.
//
// cudaFuncSetAttribute and the occupancy query cost a few microseconds of
// host time each; the launchers call them on every launch, so they are
// memoised here: the dynamic shared memory opted into so far per (kernel,
// device), and the resident CTAs per SM per (kernel, device, threads, smem).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace kvslab {

// Raises the kernel's dynamic shared memory limit to at least `smem` bytes.
cudaError_t ensure_dynamic_smem(const void* fn, size_t smem);
// cudaOccupancyMaxActiveBlocksPerMultiprocessor, memoised.
cudaError_t cached_occupancy(const void* fn, int threads, size_t smem, int* per_sm);

}  // namespace kvslab
