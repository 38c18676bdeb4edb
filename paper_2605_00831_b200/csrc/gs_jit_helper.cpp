// gs_jit_helper -- the NVRTC compile of a runtime-specialised kernel, in its
// own process (gs_jit.cu spawns it). Keeping NVRTC out of the host process
// means no NVRTC state exists there to be torn down while a compile is in
// flight: a process may exit at any moment with a build pending.
//
//   gs_jit_helper <arch> <include dir> <source file> <out base> <name expression>
//
// On success writes <out base>.cubin and <out base>.name (the lowered kernel
// name) via temp files + rename and exits 0; on failure writes the compile
// log to <out base>.log and exits 1.
#include <dlfcn.h>
#include <nvrtc.h>
#include <unistd.h>

#include <cstdio>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

namespace {

template <class F>
F sym(void* h, const char* name) {
  return reinterpret_cast<F>(dlsym(h, name));
}

int fail(const std::string& base, const std::string& log) {
  std::ofstream(base + ".log") << log;
  return 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 6) {
    std::fprintf(stderr, "usage: gs_jit_helper <arch> <include dir> <source> <out base> <name expr>\n");
    return 2;
  }
  const std::string arch = argv[1], inc = argv[2], src_path = argv[3], base = argv[4], expr = argv[5];
  void* h = nullptr;
  for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
    if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return fail(base, "libnvrtc not available");
  auto create = sym<decltype(&nvrtcCreateProgram)>(h, "nvrtcCreateProgram");
  auto compile = sym<decltype(&nvrtcCompileProgram)>(h, "nvrtcCompileProgram");
  auto log_size = sym<decltype(&nvrtcGetProgramLogSize)>(h, "nvrtcGetProgramLogSize");
  auto get_log = sym<decltype(&nvrtcGetProgramLog)>(h, "nvrtcGetProgramLog");
  auto cubin_size = sym<decltype(&nvrtcGetCUBINSize)>(h, "nvrtcGetCUBINSize");
  auto get_cubin = sym<decltype(&nvrtcGetCUBIN)>(h, "nvrtcGetCUBIN");
  auto add_name = sym<decltype(&nvrtcAddNameExpression)>(h, "nvrtcAddNameExpression");
  auto lowered = sym<decltype(&nvrtcGetLoweredName)>(h, "nvrtcGetLoweredName");
  auto destroy = sym<decltype(&nvrtcDestroyProgram)>(h, "nvrtcDestroyProgram");
  if (!create || !compile || !log_size || !get_log || !cubin_size || !get_cubin || !add_name || !lowered || !destroy)
    return fail(base, "libnvrtc lacks a required entry point");
  std::ifstream in(src_path, std::ios::binary);
  const std::string src((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (src.empty()) return fail(base, "empty source " + src_path);
  nvrtcProgram prog;
  if (create(&prog, src.c_str(), "gs_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(base, "nvrtcCreateProgram failed");
  add_name(prog, expr.c_str());
  const std::string a = "--gpu-architecture=" + arch, i = "-I" + inc;
  const char* opts[] = {a.c_str(), "-std=c++20", i.c_str(), "-lineinfo"};
  const nvrtcResult r = compile(prog, 4, opts);
  size_t ls = 0;
  log_size(prog, &ls);
  std::string log(ls, '\0');
  if (ls) get_log(prog, log.data());
  if (r != NVRTC_SUCCESS) return fail(base, log);
  size_t n = 0;
  cubin_size(prog, &n);
  std::vector<char> cubin(n);
  get_cubin(prog, cubin.data());
  const char* low = nullptr;
  lowered(prog, expr.c_str(), &low);
  const std::string name = low ? low : "";
  destroy(&prog);
  if (cubin.empty() || name.empty()) return fail(base, "no cubin / lowered name produced\n" + log);
  const std::string tmp = base + ".tmp" + std::to_string(::getpid());
  {
    std::ofstream f(tmp + ".cubin", std::ios::binary), nf(tmp + ".name");
    f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
    nf << name << "\n";
    if (!f || !nf) return fail(base, "cannot write " + tmp);
  }
  // name first: a reader that sees the cubin always finds its name
  if (std::rename((tmp + ".name").c_str(), (base + ".name").c_str()) ||
      std::rename((tmp + ".cubin").c_str(), (base + ".cubin").c_str()))
    return fail(base, "rename into the cache failed");
  return 0;
}
