// facade_test.cpp -- drives the drop-in C++ facade (include/ghostserve_gpu/
// coding.hpp) exactly the way the reference's own suites drive
// ghostserve::encode / reconstruct (coding_test.cpp:53-70, acceptance.cpp:
// 100-137), and checks every byte against the CPU oracle (test
// infrastructure). Exit code = number of failed checks. Needs a GPU.
#include <atomic>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <stdexcept>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "ghostserve_gpu/coding.hpp"
#include "../../oracle/gs_oracle.h"

namespace gs = ghostserve_gpu;

static std::atomic<int> failures{0};
#define CHECK(cond, ...)                \
  do {                                  \
    if (!(cond)) {                      \
      ++failures;                       \
      std::fprintf(stderr, __VA_ARGS__); \
      std::fprintf(stderr, "\n");       \
    }                                   \
  } while (0)

static std::vector<std::vector<uint8_t>> shards(int n, size_t len, uint64_t seed) {
  std::vector<std::vector<uint8_t>> out(static_cast<size_t>(n));
  uint64_t s = seed;
  for (auto& v : out) {
    v.resize(len);
    for (auto& b : v) {
      s += 0x9E3779B97F4A7C15ull;
      uint64_t z = s;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      b = static_cast<uint8_t>(z ^ (z >> 31));
    }
  }
  return out;
}

int main() {
  const std::vector<gs::CodingScheme> schemes = {
      gs::CodingScheme::xor_code(2), gs::CodingScheme::xor_code(8), gs::CodingScheme::rdp(4), gs::CodingScheme::rdp(6),
      gs::CodingScheme::reed_solomon(4, 1),
      gs::CodingScheme::reed_solomon(4, 2), gs::CodingScheme::reed_solomon(8, 2),
      gs::CodingScheme::reed_solomon(8, 3), gs::CodingScheme::reed_solomon(6, 2)};
  uint64_t seed = 1;
  for (const auto& sc : schemes) {
    for (size_t len : {size_t{1}, size_t{17}, size_t{4096}, size_t{1} << 20}) {
      const auto data = shards(sc.n, len, seed++);
      const auto parity = gs::encode(sc, data);
      // oracle parity
      std::vector<const uint8_t*> dp;
      for (auto& d : data) dp.push_back(d.data());
      std::vector<std::vector<uint8_t>> want(static_cast<size_t>(sc.k), std::vector<uint8_t>(len));
      std::vector<uint8_t*> wp;
      for (auto& w : want) wp.push_back(w.data());
      gso_encode(static_cast<int>(sc.kind), sc.n, sc.k, dp.data(), len, wp.data());
      CHECK(parity == want, "%s(%d,%d) len=%zu parity mismatch", gs::to_string(sc.kind), sc.n, sc.k, len);
      // every erasure pattern within tolerance (coding_test.cpp:36-70)
      const int total = sc.n + sc.k, tol = gs::max_tolerance(sc);
      for (unsigned mask = 1; mask < (1u << total); ++mask) {
        if (__builtin_popcount(mask) > tol) continue;
        std::vector<int> lost;
        for (int i = 0; i < total; ++i)
          if (mask & (1u << i)) lost.push_back(i);
        gs::ErasurePattern pat(lost);
        std::map<int, gs::ConstShardSpan> surv;
        for (int i = 0; i < sc.n; ++i)
          if (!pat.contains(i)) surv[i] = gs::ConstShardSpan(data[static_cast<size_t>(i)]);
        for (int i = 0; i < sc.k; ++i)
          if (!pat.contains(sc.n + i)) surv[sc.n + i] = gs::ConstShardSpan(parity[static_cast<size_t>(i)]);
        auto rebuilt = gs::reconstruct(sc, surv, pat);
        for (int idx : pat.lost) {
          if (idx >= sc.n) continue;
          CHECK(rebuilt.count(idx) && rebuilt.at(idx) == data[static_cast<size_t>(idx)],
                "%s(%d,%d) len=%zu lost mask %x: shard %d not rebuilt", gs::to_string(sc.kind), sc.n, sc.k,
                len, mask, idx);
        }
      }
    }
  }
  // error classes (coding_test.cpp:161-197)
  const auto rs = gs::CodingScheme::reed_solomon(8, 2);
  const auto d8 = shards(8, 16, 99);
  const auto p8 = gs::encode(rs, d8);
  try {
    gs::ErasurePattern lost({0, 1, 2});
    std::map<int, gs::ConstShardSpan> s;
    gs::reconstruct(rs, s, lost);
    CHECK(false, "over-tolerance did not throw");
  } catch (const gs::UnrecoverableError&) {
  }
  try {
    gs::ErasurePattern lost({0});
    std::map<int, gs::ConstShardSpan> s;
    for (int i = 1; i < 8; ++i) s[i] = gs::ConstShardSpan(d8[static_cast<size_t>(i)]);
    s[8] = gs::ConstShardSpan(p8[0]);  // parity 9 missing
    gs::reconstruct(rs, s, lost);
    CHECK(false, "missing survivor did not throw");
  } catch (const std::invalid_argument&) {
  }
  try {
    std::vector<std::vector<uint8_t>> ragged{{1, 2}, {3}};
    gs::encode(gs::CodingScheme::xor_code(2), ragged);
    CHECK(false, "ragged did not throw");
  } catch (const std::invalid_argument&) {
  }
  try {
    gs::CodingScheme{gs::CodeKind::kReedSolomon, 4, 5}.validate();
    CHECK(false, "k>n did not throw");
  } catch (const std::invalid_argument&) {
  }
  // device-pointer overloads: KV in HBM -> pinned host parity -> rebuilt in HBM
  {
    const size_t len = (size_t{1} << 20) + 48;
    const auto host = shards(8, len, 4242);
    std::vector<void*> dptr(8);
    for (int j = 0; j < 8; ++j) {
      cudaMalloc(&dptr[static_cast<size_t>(j)], len);
      cudaMemcpy(dptr[static_cast<size_t>(j)], host[static_cast<size_t>(j)].data(), len, cudaMemcpyHostToDevice);
    }
    std::vector<void*> hpar(2);
    for (auto& h : hpar) cudaMallocHost(&h, len);
    cudaStream_t st;
    cudaStreamCreate(&st);
    std::vector<const void*> din(dptr.begin(), dptr.end());
    gs::encode_device(rs, din, len, hpar, st, st);
    gs::sync(st);
    const auto want = gs::encode(rs, host);
    for (int i = 0; i < 2; ++i)
      CHECK(std::memcmp(hpar[static_cast<size_t>(i)], want[static_cast<size_t>(i)].data(), len) == 0,
            "encode_device parity %d mismatch", i);
    for (const std::vector<int>& lv : {std::vector<int>{3}, std::vector<int>{2, 7}, std::vector<int>{5, 8}}) {
      gs::ErasurePattern pat(lv);
      std::vector<const void*> surv(din);
      std::vector<const void*> par(hpar.begin(), hpar.end());
      std::vector<void*> outs;
      for (int idx : pat.lost) {
        if (idx < 8) {
          surv[static_cast<size_t>(idx)] = nullptr;
          void* o;
          cudaMalloc(&o, len);
          outs.push_back(o);
        } else {
          par[static_cast<size_t>(idx - 8)] = nullptr;
        }
      }
      gs::reconstruct_device(rs, pat, surv, par, outs, len, st);
      gs::sync(st);
      size_t b = 0;
      std::vector<uint8_t> got(len);
      for (int idx : pat.lost) {
        if (idx >= 8) continue;
        cudaMemcpy(got.data(), outs[b++], len, cudaMemcpyDeviceToHost);
        CHECK(got == host[static_cast<size_t>(idx)], "reconstruct_device shard %d mismatch", idx);
      }
      for (void* o : outs) cudaFree(o);
    }
    try {
      gs::ErasurePattern pat({0, 1, 2});
      std::vector<void*> outs(3, nullptr);
      gs::reconstruct_device(rs, pat, din, std::vector<const void*>(hpar.begin(), hpar.end()), outs, len, st);
      CHECK(false, "device over-tolerance did not throw");
    } catch (const gs::UnrecoverableError&) {
    }
    for (void* d : dptr) cudaFree(d);
    for (void* h : hpar) cudaFreeHost(h);
    cudaStreamDestroy(st);
  }
  // concurrency (the reference codec is safe to call from
  // many threads): 4 threads, thread t on device t % ndev, each driving
  // encode / reconstruct through its own per-(thread, device) pipeline with
  // no facade-wide lock; every byte checked against the oracle.
  {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    std::vector<std::thread> pool;
    std::atomic<int> calls{0};
    for (int t = 0; t < 4; ++t) {
      pool.emplace_back([t, ndev, &calls] {
        const int dev = t % std::max(ndev, 1);
        cudaSetDevice(dev);
        gs_pipeline* p = nullptr;
        int pdev = -1;
        CHECK(gs_thread_pipeline(&p) == GS_OK && gs_pipeline_device(p, &pdev) == GS_OK && pdev == dev,
              "thread %d: pipeline on device %d, expected %d", t, pdev, dev);
        const gs::CodingScheme mix[] = {gs::CodingScheme::reed_solomon(8, 2), gs::CodingScheme::reed_solomon(6, 2),
                                        gs::CodingScheme::xor_code(8), gs::CodingScheme::reed_solomon(4, 2)};
        for (int it = 0; it < 12; ++it) {
          const auto& sc = mix[(t + it) % 4];
          const size_t len = (size_t{1} << 18) + 16 * static_cast<size_t>(it * 7 + t);
          const auto data = shards(sc.n, len, 1000 + 100 * static_cast<uint64_t>(t) + it);
          const auto parity = gs::encode(sc, data);
          std::vector<const uint8_t*> dp;
          for (auto& d : data) dp.push_back(d.data());
          std::vector<std::vector<uint8_t>> want(static_cast<size_t>(sc.k), std::vector<uint8_t>(len));
          std::vector<uint8_t*> wp;
          for (auto& w : want) wp.push_back(w.data());
          gso_encode(static_cast<int>(sc.kind), sc.n, sc.k, dp.data(), len, wp.data());
          CHECK(parity == want, "thread %d it %d: parity mismatch", t, it);
          gs::ErasurePattern pat({(t + it) % sc.n});
          std::map<int, gs::ConstShardSpan> surv;
          for (int i = 0; i < sc.n; ++i)
            if (!pat.contains(i)) surv[i] = gs::ConstShardSpan(data[static_cast<size_t>(i)]);
          for (int i = 0; i < sc.k; ++i) surv[sc.n + i] = gs::ConstShardSpan(parity[static_cast<size_t>(i)]);
          auto rebuilt = gs::reconstruct(sc, surv, pat);
          const int lost = pat.lost[0];
          CHECK(rebuilt.count(lost) && rebuilt.at(lost) == data[static_cast<size_t>(lost)],
                "thread %d it %d: shard %d not rebuilt", t, it, lost);
          calls += 2;
        }
      });
    }
    for (auto& th : pool) th.join();
    std::printf("facade_test: concurrent: 4 threads on %d device(s), %d calls\n", std::max(ndev, 1), calls.load());
  }
  // a codec outside the compiled registry: its first launch requests a
  // runtime-specialised build (out-of-process NVRTC) and the process exits
  // right after, possibly mid-compile -- which must not crash
  if (!std::getenv("GS_FACADE_NO_JIT_EXIT")) {
    const auto odd = gs::CodingScheme::reed_solomon(7, 3);
    const auto d7 = shards(7, 4096, 77);
    const auto p7 = gs::encode(odd, d7);
    std::printf("facade_test: RS(7,3) encoded (%zu parity rows); exiting with its build in flight\n", p7.size());
  }
  std::printf("facade_test: %d failure(s), %llu kernels launched\n", failures.load(),
              static_cast<unsigned long long>(gs_kernel_launches()));
  return failures.load();
}
