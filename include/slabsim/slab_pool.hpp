// slabsim/slab_pool.hpp -- drop-in shim: code written against the reference
// allocator (proj/core/include/slabsim/slab_pool.hpp) compiles unchanged
// against libkvslab.so by putting this repo's include/ first on the path.
// slabsim::SlabPool, SlabPoolConfig, BlockHandle, FragmentationStats,
// OpLogRecord, SlabState, write_op_log_line and the exception classes resolve
// to the kvslab implementations (same signatures and semantics).
#pragma once

#include "kvslab/slab_pool.hpp"

namespace slabsim {
using namespace kvslab;  // NOLINT: deliberate alias of the whole API
}  // namespace slabsim
