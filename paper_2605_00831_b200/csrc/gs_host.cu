// gs_host.cu -- host-side placement of pinned memory (NUMA) and the C-ABI
// entry points that expose it (include/gs_capi.h: gs_host_alloc_near,
// gs_device_numa_node, gs_device_local_cpus).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/gs_capi.h"
#include "gs_host.hpp"

namespace gsb {
void set_last_error(const char* msg);  // gs_capi.cu: shared gs_last_error() slot
}

namespace {
int hfail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  gsb::set_last_error(buf);
  return status;
}
}  // namespace

// ---- NUMA placement of pinned host memory -----------------------------------
// On multi-socket hosts a GPU's host link hangs off one socket; parity D2H'd
// into memory on the other socket crosses the inter-socket link (shared by
// every GPU there). Pinned buffers are therefore placed on the GPU's NUMA node:
// mmap + mbind(MPOL_BIND) + first touch + cudaHostRegister. Single-node hosts
// (numa_node -1 or one node) fall back to cudaHostAlloc.
namespace {
std::string pci_sysfs(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return {};
  std::string id(bus);
  for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  // cudaDeviceGetPCIBusId gives "0000:40:00.0" (domain may be 8 hex digits)
  const auto colon = id.find(':');
  if (colon != std::string::npos && colon > 4) id = id.substr(colon - 4);
  return "/sys/bus/pci/devices/" + id;
}
std::string read_line(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) return {};
  char buf[4096] = {0};
  const char* r = std::fgets(buf, sizeof buf, f);
  std::fclose(f);
  std::string s = r ? r : "";
  while (!s.empty() && (s.back() == '\n' || s.back() == ' ')) s.pop_back();
  return s;
}
int numa_nodes_online() {
  const std::string s = read_line("/sys/devices/system/node/online");  // e.g. "0-1" or "0"
  if (s.empty()) return 1;
  const auto dash = s.find('-');
  return dash == std::string::npos ? 1 : std::atoi(s.c_str() + dash + 1) + 1;
}
std::mutex g_near_mu;
std::map<void*, size_t> g_near;  // mmap'ed + registered allocations
}  // namespace

int gsb::numa_node_of(int device) {
  const std::string dir = pci_sysfs(device);
  if (dir.empty()) return -1;
  const std::string s = read_line(dir + "/numa_node");
  return s.empty() ? -1 : std::atoi(s.c_str());
}

std::string gsb::local_cpulist_of(int device) {
  const std::string dir = pci_sysfs(device);
  return dir.empty() ? std::string() : read_line(dir + "/local_cpulist");
}

int gsb::pinned_alloc_near(int device, size_t bytes, void** out) {
  // GS_FORCE_NUMA_BIND=1 takes the mmap/mbind/register path even on
  // single-node hosts (node 0), so tests exercise it anywhere.
  static const bool force = [] {
    const char* e = std::getenv("GS_FORCE_NUMA_BIND");
    return e && std::atoi(e) != 0;
  }();
  int node = numa_node_of(device);
  if (force && node < 0) node = 0;
  if (!force && (node < 0 || numa_nodes_online() < 2 || bytes == 0)) {
    const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
    return e == cudaSuccess ? GS_OK : hfail(GS_CUDA_ERROR, "host_alloc_near: cudaHostAlloc: %s", cudaGetErrorString(e));
  }
  const size_t len = (bytes + 4095) / 4096 * 4096;
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return hfail(GS_RUNTIME_ERROR, "host_alloc_near: mmap of %zu B failed", len);
  unsigned long mask[16] = {0};
  if (node < 16 * 64) mask[node / 64] = 1ul << (node % 64);
  // MPOL_BIND = 2; best effort (a failed bind still yields usable memory)
  syscall(SYS_mbind, p, len, 2, mask, 16 * 64 + 1, 0);
  std::memset(p, 0, len);  // first touch on the bound node
  cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, len);
    return hfail(GS_CUDA_ERROR, "host_alloc_near: cudaHostRegister: %s", cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lk(g_near_mu);
  g_near[p] = len;
  *out = p;
  return GS_OK;
}

bool gsb::pinned_free_near(void* p) {
  size_t len = 0;
  {
    std::lock_guard<std::mutex> lk(g_near_mu);
    auto it = g_near.find(p);
    if (it == g_near.end()) return false;
    len = it->second;
    g_near.erase(it);
  }
  cudaHostUnregister(p);
  munmap(p, len);
  return true;
}


extern "C" {

int gs_device_numa_node(int device, int* node) {
  if (!node) return hfail(GS_INVALID_ARGUMENT, "device_numa_node: NULL out");
  *node = gsb::numa_node_of(device);
  return GS_OK;
}

int gs_device_local_cpus(int device, char* buf, size_t cap) {
  if (!buf || cap == 0) return hfail(GS_INVALID_ARGUMENT, "device_local_cpus: bad buffer");
  const std::string s = gsb::local_cpulist_of(device);
  std::snprintf(buf, cap, "%s", s.c_str());
  return GS_OK;
}

int gs_host_alloc_near(int device, size_t bytes, void** out) {
  if (!out) return hfail(GS_INVALID_ARGUMENT, "host_alloc_near: out is NULL");
  return gsb::pinned_alloc_near(device, bytes, out);
}

}  // extern "C"
