// Redirect shim (see coding.hpp here): the reference's suites that include
// "ghostserve/kv_layout.hpp" get the drop-in facade include/ghostserve_gpu/kv_layout.hpp.
// Test infrastructure only.
#pragma once

#include "ghostserve/coding.hpp"
#include "ghostserve_gpu/kv_layout.hpp"
