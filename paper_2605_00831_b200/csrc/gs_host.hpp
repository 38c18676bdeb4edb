// gs_host.hpp -- host-side helpers shared by gs_capi.cu and gs_store.cu:
// NUMA placement of pinned host memory next to a GPU's host link.
#pragma once

#include <cstddef>
#include <string>

namespace gsb {
int numa_node_of(int device);             // -1 if unknown
std::string local_cpulist_of(int device);  // sysfs local_cpulist, "" if unknown
// Pinned allocation on the GPU's NUMA node (cudaHostAlloc on single-node hosts).
int pinned_alloc_near(int device, size_t bytes, void** out);
// true if p came from pinned_alloc_near's mmap path (and is now freed)
bool pinned_free_near(void* p);
}  // namespace gsb
