// Host FNV-1a throughput probe (not product): T threads, each hashing two 80 MiB
// chains, with the bit-sliced SIMD chain (gs_fnv_simd.cpp) and the scalar
// lockstep pair. Build: g++ -O3 -std=c++20 -pthread -Ipaper_2605_00831_b200/csrc
//   tools/fnv_host_mt.cpp paper_2605_00831_b200/csrc/gs_fnv_simd.cpp -o tools/fnv_host_mt.bin
// aggregate throughput: T threads, each hashing its own 80 MiB chain (simd vs scalar x2 interleaved)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <thread>
#include <algorithm>
#include <cstdint>
#include "gs_fnv.hpp"
namespace gsb { uint64_t fnv1a64_fast(const uint8_t*, size_t, uint64_t); bool fnv_simd_available(); }
int main(int argc, char** argv) {
  const size_t L = 80u << 20;
  int maxT = argc > 1 ? atoi(argv[1]) : 16;
  std::vector<std::vector<uint8_t>> bufs(maxT * 2);
  for (auto& b : bufs) { b.resize(L); uint64_t s = (uint64_t)&b; for (auto& x : b) { s = s * 6364136223846793005ull + 1; x = s >> 56; } }
  for (int T : {1, 2, 4, 8, 14, 16}) {
    if (T > maxT) break;
    for (int mode = 0; mode < 2; ++mode) {
      std::vector<std::thread> th; std::vector<uint64_t> out(2 * T);
      auto t0 = std::chrono::steady_clock::now();
      for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
        if (mode == 0) { out[2*t] = gsb::fnv1a64_fast(bufs[2*t].data(), L, gsb::kFnvOffset); out[2*t+1] = gsb::fnv1a64_fast(bufs[2*t+1].data(), L, gsb::kFnvOffset); }
        else { const uint8_t* ps[2] = {bufs[2*t].data(), bufs[2*t+1].data()}; uint64_t h[2] = {gsb::kFnvOffset, gsb::kFnvOffset}; gsb::fnv1a64_x8(ps, 2, L, h); out[2*t] = h[0]; out[2*t+1] = h[1]; }
      });
      for (auto& x : th) x.join();
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("{\"threads\": %d, \"impl\": \"%s\", \"chains\": %d, \"ms\": %.1f, \"aggregate_gbs\": %.2f, \"per_chain_gbs\": %.2f}\n", T, mode ? "scalar_x2" : "simd", 2*T, s*1e3, 2.0*T*L/s/1e9, L/(s/(mode?1:2))/1e9);
      std::fflush(stdout);
    }
  }
}
