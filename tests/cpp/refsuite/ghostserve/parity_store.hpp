// Redirect shim (see coding.hpp here): the reference's suites that include
// "ghostserve/parity_store.hpp" get the drop-in facade include/ghostserve_gpu/parity_store.hpp.
// Test infrastructure only.
#pragma once

#include "ghostserve/coding.hpp"
#include "ghostserve_gpu/parity_store.hpp"
