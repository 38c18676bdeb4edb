// Redirect shim (see coding.hpp here): the reference's suites that include
// "ghostserve/kv_layout.hpp" get the drop-in facade include/ghostserve_gpu/kv_layout.hpp.
// Test infrastructure only.
#pragma once

#include "ghostserve/coding.hpp"
#include "ghostserve_gpu/kv_layout.hpp"

// the reference's other headers (trace.hpp) call these unqualified from
// inside ghostserve::detail
namespace ghostserve::detail {
using ghostserve_gpu::detail::mix_key;
using ghostserve_gpu::detail::splitmix64;
}
