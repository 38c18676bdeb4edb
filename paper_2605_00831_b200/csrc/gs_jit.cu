// gs_jit.cu -- runtime-specialised kernels (see gs_jit.hpp).
//
// NVRTC runs in a helper process (gs_jit_helper, see compile()) and the
// driver's module/launch entry points come from cudaGetDriverEntryPoint, so
// the library has no link-time dependency on either: without them JIT is
// simply off and the generic kernel serves.
#include "gs_jit.hpp"

#include <cuda.h>
#include <dlfcn.h>
#include <spawn.h>
#include <sys/wait.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "gs_special.cuh"

extern char** environ;

namespace gsb {

// bumped whenever the kernel template or TileGeom layout changes, so stale
// on-disk cubins are never reused
constexpr const char* kJitVersion = "gsjit-4";
constexpr int kJitMaxRows = 8;
constexpr int kJitMaxUsed = 24;

struct JitKernel {
  std::string key;
  int n_out = 0, n_slots = 0;
  std::vector<uint8_t> coef;
  std::string arch;
  std::atomic<int> state{0};  // 0 pending, 1 ready, -1 failed
  std::vector<char> cubin;
  std::string lowered, log;
  std::mutex mu;
  std::condition_variable cv;
  std::map<int, std::pair<CUmodule, CUfunction>> loaded;
  std::map<int, int> occ;
};

namespace {

std::atomic<bool> g_jit_on{[] {
  const char* e = std::getenv("GS_JIT");
  return !(e && std::atoi(e) == 0);
}()};

struct Driver {
  bool ok = false;
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*get_fn)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  CUresult (*occ)(int*, CUfunction, int, size_t) = nullptr;
};

Driver& driver() {
  static Driver d = [] {
    Driver r;
    auto get = [](const char* sym) -> void* {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(sym, &fn, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
      return q == cudaDriverEntryPointSuccess ? fn : nullptr;
    };
    r.load = reinterpret_cast<decltype(r.load)>(get("cuModuleLoadData"));
    r.get_fn = reinterpret_cast<decltype(r.get_fn)>(get("cuModuleGetFunction"));
    r.launch = reinterpret_cast<decltype(r.launch)>(get("cuLaunchKernel"));
    r.occ = reinterpret_cast<decltype(r.occ)>(get("cuOccupancyMaxActiveBlocksPerMultiprocessor"));
    r.ok = r.load && r.get_fn && r.launch && r.occ;
    return r;
  }();
  return d;
}

// Directory of this shared library (…/paper_2605_00831_b200/_lib).
std::string lib_dir() {
  Dl_info info{};
  if (!dladdr(reinterpret_cast<void*>(&jit_request), &info) || !info.dli_fname) return {};
  std::string p(info.dli_fname);
  const auto slash = p.rfind('/');
  return slash == std::string::npos ? std::string(".") : p.substr(0, slash);
}

std::string csrc_dir() {
  const std::string d = lib_dir() + "/../csrc";
  struct stat st {};
  return stat((d + "/gs_kernels.cuh").c_str(), &st) == 0 ? d : std::string();
}

std::string cache_dir() {
  const char* e = std::getenv("GS_JIT_CACHE");
  std::string d = e && *e ? std::string(e) : lib_dir() + "/jit";
  mkdir(d.c_str(), 0755);
  return d;
}

uint64_t fnv(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char ch : s) h = (h ^ ch) * 0x100000001b3ull;
  return h;
}

std::string source_for(const JitKernel& k) {
  std::ostringstream o;
  o << "#include \"gs_kernels.cuh\"\n"
    << "struct GsJitSpec {\n"
    << "  static constexpr int NS = " << k.n_slots << ", NO = " << k.n_out << ";\n"
    << "  __host__ __device__ static constexpr gsb::CoefMatrix matrix() {\n"
    << "    gsb::CoefMatrix m{};\n"
    << "    m.rows = NO;\n    m.cols = NS;\n";
  for (int i = 0; i < k.n_out; ++i)
    for (int j = 0; j < k.n_slots; ++j)
      if (int v = k.coef[static_cast<size_t>(i) * k.n_slots + j]) o << "    m.c[" << i << "][" << j << "] = " << v << ";\n";
  o << "    return m;\n  }\n};\n";
  return o.str();
}

const char* kKernelExpr = "gsb::k_apply_special<GsJitSpec, 488, 1, false>";
static_assert(kPtrCap == 488, "JIT name expression hard-codes the pointer-table capacity");

bool load_cached(JitKernel& k, const std::string& base) {
  std::ifstream f(base + ".cubin", std::ios::binary), nf(base + ".name");
  if (!f || !nf) return false;
  k.cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  std::getline(nf, k.lowered);
  return !k.cubin.empty() && !k.lowered.empty();
}

// The compile runs in a helper process (gs_jit_helper next to this library):
// NVRTC is never loaded into the host process, so nothing of it can be torn
// down under an in-flight build when the process exits (the worker thread
// here only spawns, waits and reads files). The helper writes the cubin into
// the disk cache, which this process then loads.
void compile(JitKernel& k) {
  const std::string base = cache_dir() + "/" + [&] {
    char b[32];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(fnv(k.key)));
    return std::string(b);
  }();
  if (load_cached(k, base)) {
    k.log = "disk cache: " + base + ".cubin";
    return;
  }
  const std::string inc = csrc_dir(), helper = lib_dir() + "/gs_jit_helper";
  struct stat hs {};
  if (inc.empty() || stat(helper.c_str(), &hs) != 0) {
    k.log = inc.empty() ? "kernel headers (csrc/) not found next to the library" : "gs_jit_helper not built";
    throw 0;
  }
  const std::string src = base + ".src" + std::to_string(::getpid()) + ".cu";
  {
    std::ofstream f(src);
    f << source_for(k);
    if (!f) {
      k.log = "cannot write " + src;
      throw 0;
    }
  }
  std::string a_arch = k.arch, a_expr = kKernelExpr;
  char* argv[] = {const_cast<char*>(helper.c_str()), a_arch.data(), const_cast<char*>(inc.c_str()),
                  const_cast<char*>(src.c_str()), const_cast<char*>(base.c_str()), a_expr.data(), nullptr};
  pid_t pid = 0;
  int status = 0;
  const int sp = posix_spawn(&pid, helper.c_str(), nullptr, nullptr, argv, environ);
  if (sp == 0) {
    while (waitpid(pid, &status, 0) < 0 && errno == EINTR) {
    }
  }
  std::remove(src.c_str());
  if (sp != 0 || !WIFEXITED(status) || WEXITSTATUS(status) != 0 || !load_cached(k, base)) {
    std::ifstream lf(base + ".log");
    k.log = std::string("gs_jit_helper failed: ") +
            std::string(std::istreambuf_iterator<char>(lf), std::istreambuf_iterator<char>());
    throw 0;
  }
  k.log = "compiled by gs_jit_helper: " + base + ".cubin";
}

// one background compile worker
struct Worker {
  std::mutex mu;
  std::condition_variable cv, idle_cv;
  std::deque<JitKernel*> q;
  bool started = false, busy = false;
  void push(JitKernel* k) {
    std::lock_guard<std::mutex> lk(mu);
    q.push_back(k);
    if (!started) {
      started = true;
      std::thread([this] { run(); }).detach();
    }
    cv.notify_one();
  }
  void run() {
    for (;;) {
      JitKernel* k;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return !q.empty(); });
        k = q.front();
        q.pop_front();
        busy = true;
      }
      int st = 1;
      try {
        compile(*k);
        if (k->cubin.empty() || k->lowered.empty()) st = -1;
      } catch (...) {
        st = -1;
      }
      {
        std::lock_guard<std::mutex> lk(k->mu);
        k->state.store(st);
      }
      k->cv.notify_all();
      {
        std::lock_guard<std::mutex> lk(mu);
        busy = false;
      }
      idle_cv.notify_all();
    }
  }
  // drop queued builds (they stay pending: callers keep the generic kernel)
  // and wait for the one in flight; the worker keeps serving later requests
  void quiesce() {
    std::unique_lock<std::mutex> lk(mu);
    q.clear();
    idle_cv.wait(lk, [&] { return !busy; });
  }
};

Worker& worker() {
  static Worker* w = new Worker;  // intentionally leaked: the detached thread outlives statics
  return *w;
}

}  // namespace

void jit_quiesce() { worker().quiesce(); }

namespace {

std::mutex g_reg_mu;
std::map<std::string, std::unique_ptr<JitKernel>>& registry() {
  static auto* r = new std::map<std::string, std::unique_ptr<JitKernel>>;
  return *r;
}

std::string device_arch() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return {};
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return {};
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  char b[32];
  std::snprintf(b, sizeof b, "sm_%d%da", major, minor);
  return b;
}

}  // namespace

void jit_set_enabled(bool on) { g_jit_on.store(on); }

bool jit_eligible(int n_out, int n_slots, const uint8_t* coef) {
  if (n_out < 1 || n_out > kJitMaxRows || n_slots < 1 || n_slots > 2 * kMaxSpecial || !coef) return false;
  int used = 0;
  for (int j = 0; j < n_slots; ++j) {
    bool any = false;
    for (int i = 0; i < n_out; ++i) any |= coef[static_cast<size_t>(i) * n_slots + j] != 0;
    used += any;
  }
  return used >= 1 && used <= kJitMaxUsed;
}

// Content hash of the kernel headers the JIT source includes: a changed
// kernel never reuses a stale on-disk cubin.
const std::string& headers_hash() {
  static const std::string h = [] {
    std::string all;
    const std::string d = csrc_dir();
    for (const char* f : {"/gs_kernels.cuh", "/gs_field.hpp"}) {
      std::ifstream in(d + f, std::ios::binary);
      all.append(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    }
    char b[32];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(fnv(all)));
    return std::string(b);
  }();
  return h;
}

JitKernel* jit_request(int n_out, int n_slots, const uint8_t* coef) {
  if (!g_jit_on.load() || !jit_eligible(n_out, n_slots, coef)) return nullptr;
  const std::string arch = device_arch();
  if (arch.empty()) return nullptr;
  std::string key = std::string(kJitVersion) + "|" + headers_hash() + "|" + arch + "|" + std::to_string(n_out) + "x" +
                    std::to_string(n_slots) + "|";
  for (int i = 0; i < n_out * n_slots; ++i) {
    char b[4];
    std::snprintf(b, sizeof b, "%02x", coef[i]);
    key += b;
  }
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto& reg = registry();
  auto it = reg.find(key);
  if (it != reg.end()) return it->second.get();
  auto k = std::make_unique<JitKernel>();
  k->key = key;
  k->n_out = n_out;
  k->n_slots = n_slots;
  k->coef.assign(coef, coef + n_out * n_slots);
  k->arch = arch;
  JitKernel* raw = k.get();
  reg.emplace(key, std::move(k));
  worker().push(raw);
  return raw;
}

int jit_status(JitKernel* k, bool wait) {
  if (!k) return -1;
  if (wait) {
    std::unique_lock<std::mutex> lk(k->mu);
    k->cv.wait(lk, [&] { return k->state.load() != 0; });
  }
  return k->state.load();
}

const char* jit_last_log(JitKernel* k) { return k ? k->log.c_str() : ""; }

namespace {
// Load the module on the current device (once); false if unusable.
bool ensure_loaded(JitKernel* k, int dev, CUfunction* fn, int* occ) {
  std::lock_guard<std::mutex> lk(k->mu);
  auto it = k->loaded.find(dev);
  if (it == k->loaded.end()) {
    Driver& d = driver();
    CUmodule m = nullptr;
    CUfunction f = nullptr;
    if (!d.ok || d.load(&m, k->cubin.data()) != CUDA_SUCCESS || d.get_fn(&f, m, k->lowered.c_str()) != CUDA_SUCCESS) {
      k->state.store(-1);
      k->log += "\nmodule load failed";
      return false;
    }
    int b = 0;
    if (d.occ(&b, f, kThreads, 0) != CUDA_SUCCESS || b < 1) b = 1;
    it = k->loaded.emplace(dev, std::make_pair(m, f)).first;
    k->occ[dev] = b;
  }
  *fn = it->second.second;
  *occ = k->occ[dev];
  return true;
}
}  // namespace

int jit_occupancy(JitKernel* k) {
  if (!k || k->state.load() != 1) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  CUfunction f;
  int occ = 0;
  return ensure_loaded(k, dev, &f, &occ) ? occ : 0;
}

cudaError_t jit_launch(JitKernel* k, const void* const* ptrs, int count, const TileGeom& g, int sms,
                       cudaStream_t st) {
  if (!k || k->state.load() != 1) return cudaErrorNotReady;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorNotReady;
  CUfunction fn;
  int occ = 0;
  if (!ensure_loaded(k, dev, &fn, &occ)) return cudaErrorNotReady;
  PtrTable<kPtrCap> tab;
  for (int i = 0; i < count; ++i) tab.p[i] = static_cast<const uint8_t*>(ptrs[i]);
  TileGeom geom = g;
  void* params[] = {&tab, &geom};
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(g.total, static_cast<uint64_t>(occ) * sms));
  const CUresult r = driver().launch(fn, grid, 1, 1, kThreads, 1, 1, 0, reinterpret_cast<CUstream>(st), params,
                                     nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

}  // namespace gsb
