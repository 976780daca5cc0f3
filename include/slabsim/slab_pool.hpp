// slabsim/slab_pool.hpp -- drop-in replacement for the reference allocator
// header (proj/core/include/slabsim/slab_pool.hpp:26-202).
//
// With this repository's include/ first on the include path, code written
// against slabsim::SlabPool compiles unchanged and links against
// libkvslab.so: the names below resolve to the kvslab implementations, which
// keep the reference's signatures and observable semantics (pinned by
// tests/test_slab_pool_parity.py and, for the reference's own acceptance
// suite, tests/test_dropin.py).
#pragma once

#include "kvslab/slab_pool.hpp"
#include "slabsim/common.hpp"

namespace slabsim {
using kvslab::BlockHandle;
using kvslab::FragmentationStats;
using kvslab::OpLogRecord;
using kvslab::SlabPool;
using kvslab::SlabPoolConfig;
using kvslab::SlabState;
using kvslab::write_op_log_line;
}  // namespace slabsim
