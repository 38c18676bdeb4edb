// Host FNV-1a bit-exactness + single-chain speed probe (not product). Build:
//   g++ -O3 -std=c++20 -Ipaper_2605_00831_b200/csrc tools/fnv_host_test.cpp paper_2605_00831_b200/csrc/gs_fnv_simd.cpp -o tools/fnv_host_test.bin
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstdint>
#include <thread>
#include "gs_fnv.hpp"

int main() {
  std::printf("simd %d\n", gsb::fnv_simd_available());
  std::vector<uint8_t> buf(80u << 20);
  uint64_t s = 12345;
  for (auto& b : buf) { s = s * 6364136223846793005ull + 1442695040888963407ull; b = s >> 56; }
  int bad = 0;
  for (int t = 0; t < 200; ++t) {
    size_t len = (t < 100) ? (rand() % 5000) : (rand() % 200000);
    size_t off = rand() % 1000;
    uint64_t h0 = (t % 3 == 0) ? gsb::kFnvOffset : ((uint64_t)rand() << 32 | rand());
    uint64_t a = gsb::fnv1a64_one(buf.data() + off, len, h0), b = gsb::fnv1a64_fast(buf.data() + off, len, h0);
    if (a != b) { if (bad < 5) std::printf("mismatch len %zu off %zu: %016lx %016lx\n", len, off, a, b); ++bad; }
  }
  // split form: h_end = h_mid * P^len1 + S1 with S1 from the low byte alone
  for (int t = 0; t < 50; ++t) {
    size_t l0 = rand() % 300000, l1 = rand() % 300000;
    const uint8_t* p0 = buf.data() + 7; const uint8_t* p1 = buf.data() + 500000 + (rand() % 100);
    uint64_t h0 = gsb::kFnvOffset;
    uint64_t mid = gsb::fnv1a64_one(p0, l0, h0), want = gsb::fnv1a64_one(p1, l1, mid);
    uint32_t lm = 0, le = 0; (void)gsb::fnv_partial(p0, l0, h0 & 0xFF, &lm);
    uint64_t S = gsb::fnv_partial(p1, l1, lm, &le);
    uint64_t got = mid * gsb::fnv_pow(l1) + S;
    if (lm != (mid & 0xFF) || got != want || le != (want & 0xFF)) { if (bad < 5) std::printf("split mismatch %zu %zu\n", l0, l1); ++bad; }
  }
  std::printf("bad %d\n", bad);
  double best1 = 1e9, best2 = 1e9; uint64_t a = 0, b = 0;
  for (int r = 0; r < 5; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    a = gsb::fnv1a64_one(buf.data(), buf.size(), gsb::kFnvOffset);
    auto t1 = std::chrono::steady_clock::now();
    b = gsb::fnv1a64_fast(buf.data(), buf.size(), gsb::kFnvOffset);
    auto t2 = std::chrono::steady_clock::now();

    best1 = std::min(best1, std::chrono::duration<double>(t1 - t0).count());
    best2 = std::min(best2, std::chrono::duration<double>(t2 - t1).count());
  }
  std::printf("80 MiB best of 5: scalar %.1f ms (%.2f GB/s)  simd %.1f ms (%.2f GB/s)  equal %d\n", best1 * 1e3, buf.size() / best1 / 1e9, best2 * 1e3, buf.size() / best2 / 1e9, a == b);
}
