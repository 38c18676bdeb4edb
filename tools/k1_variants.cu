// k1_variants.cu -- standalone A/B probe for K1 (RS(8,2) encode) work
// distribution at the C2 launch (32 stripes x 8 x 256 KiB) and a C3 piece
// (1 stripe x 8 x 32 MiB) / chunk (8 x 80 MiB). Not part of the product:
// it includes the product's kernel header to compare the shipped
// grid-stride walk with balanced-range variants before changing gs_capi.cu.
//
//   nvcc -std=c++20 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
//        -I paper_2605_00831_b200/csrc tools/k1_variants.cu -o /tmp/k1_variants
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gs_special.cuh"

using namespace gsb;
using Spec = EncSpec<kReedSolomon, 8, 2>;

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)

// Balanced contiguous ranges: the launch's 16-byte columns (stripe-major)
// are split into gridDim.x equal runs rounded to 8 columns (128 B); thread t
// of a CTA takes columns q0 + t, q0 + t + 256, ...
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_bal(const PtrTable<kPtrCap> tab, const TileGeom g) {
  stamp_start(g);
  const uint64_t cols = g.len / kVec;
  const uint64_t Q = cols * (g.total / g.tps);  // total / tps = stripes
  const uint64_t per = ((Q + gridDim.x - 1) / gridDim.x + 7) & ~7ull;
  const uint64_t q0 = per * blockIdx.x;
  const uint64_t q1 = q0 + per < Q ? q0 + per : Q;
  for (uint64_t q = q0 + threadIdx.x; q < q1; q += kThreads) {
    const uint32_t s = static_cast<uint32_t>(q / cols);
    const uint64_t off = (q - s * cols) * kVec;
    const int base = static_cast<int>(s) * g.stride;
    uint4 src[8], out[2];
#pragma unroll
    for (int j = 0; j < 8; ++j) src[j] = ld_stream(tab.p[base + j] + off);
    horner_apply<Spec>(src, out);
#pragma unroll
    for (int i = 0; i < 2; ++i) st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + off, out[i]);
  }
  stamp_end(g);
}

// Same balanced split, two columns per thread per iteration (loads of both
// issued before any arithmetic).
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_bal2(const PtrTable<kPtrCap> tab, const TileGeom g) {
  stamp_start(g);
  const uint64_t cols = g.len / kVec;
  const uint64_t Q = cols * (g.total / g.tps);
  const uint64_t per = ((Q + gridDim.x - 1) / gridDim.x + 511) & ~511ull;
  const uint64_t q0 = per * blockIdx.x;
  const uint64_t q1 = q0 + per < Q ? q0 + per : Q;
  for (uint64_t q = q0 + threadIdx.x; q < q1; q += 2 * kThreads) {
    uint4 src[2][8], out[2];
    uint64_t offs[2];
    int bases[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t qq = q + u * kThreads;
      ok[u] = qq < q1;
      const uint32_t s = static_cast<uint32_t>(qq / cols);
      offs[u] = (qq - s * cols) * kVec;
      bases[u] = static_cast<int>(s) * g.stride;
      if (ok[u]) {
#pragma unroll
        for (int j = 0; j < 8; ++j) src[u][j] = ld_stream(tab.p[bases[u] + j] + offs[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (ok[u]) {
        horner_apply<Spec>(src[u], out);
#pragma unroll
        for (int i = 0; i < 2; ++i) st_stream(const_cast<uint8_t*>(tab.p[bases[u] + g.out0 + i]) + offs[u], out[i]);
      }
    }
  }
  stamp_end(g);
}

// Plain copy of one stream (read + write), for the same-size ceiling.
__global__ void __launch_bounds__(kThreads) k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * kThreads)
    st_stream(reinterpret_cast<uint8_t*>(b + i), ld_stream(reinterpret_cast<const uint8_t*>(a + i)));
}

struct Geo {
  const char* name;
  int stripes;
  uint64_t len;
};

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const Geo geos[] = {{"C2 32x8x256KiB", 32, 256ull << 10},
                      {"C3 piece 1x8x32MiB", 1, 32ull << 20},
                      {"C3 chunk 1x8x80MiB", 1, 80ull << 20}};
  const int sets = 8;
  unsigned long long* ts;
  CK(cudaMalloc(&ts, 2 * sizeof(unsigned long long)));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (const Geo& G : geos) {
    const uint64_t alg = static_cast<uint64_t>(G.stripes) * 10 * G.len;  // 8 read + 2 written
    std::vector<PtrTable<kPtrCap>> tabs(sets);
    std::vector<uint8_t*> bufs;
    for (int s = 0; s < sets; ++s) {
      uint8_t* b;
      CK(cudaMalloc(&b, alg));
      CK(cudaMemset(b, s + 1, alg));
      bufs.push_back(b);
      for (int r = 0; r < G.stripes; ++r)
        for (int j = 0; j < 10; ++j) tabs[s].p[r * 10 + j] = b + (static_cast<uint64_t>(r) * 10 + j) * G.len;
    }
    TileGeom g{};
    g.len = G.len;
    g.tps = static_cast<uint32_t>(G.len / kTile);
    g.total = g.tps * G.stripes;
    g.stride = 10;
    g.out0 = 8;
    g.aligned = 1;
    g.tps_m = fastdiv_magic(g.tps);
    auto run = [&](const char* label, auto launch) {
      // warm
      for (int s = 0; s < sets; ++s) launch(tabs[s], g);
      CK(cudaStreamSynchronize(st));
      const int reps = 4;
      CK(cudaEventRecord(e0, st));
      for (int r = 0; r < reps; ++r)
        for (int s = 0; s < sets; ++s) launch(tabs[s], g);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us_ev = ms * 1e3 / (reps * sets);
      // kernel-internal span, one launch at a time (median-ish: mean of 8)
      double span = 0;
      for (int s = 0; s < sets; ++s) {
        unsigned long long init[2] = {~0ull, 0ull};
        CK(cudaMemcpyAsync(ts, init, sizeof(init), cudaMemcpyHostToDevice, st));
        TileGeom gg = g;
        gg.tstamp = ts;
        launch(tabs[s], gg);
        unsigned long long out[2];
        CK(cudaMemcpyAsync(out, ts, sizeof(out), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        span += (out[1] - out[0]) * 1e-3;
      }
      span /= sets;
      std::printf("{\"geo\": \"%s\", \"variant\": \"%s\", \"us_event\": %.2f, \"tbs_event\": %.3f, "
                  "\"us_span\": %.2f, \"tbs_span\": %.3f}\n",
                  G.name, label, us_ev, alg / us_ev * 1e-6, span, alg / span * 1e-6);
      std::fflush(stdout);
    };
    auto occ = [&](const void* k) {
      int b = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kThreads, 0));
      return b;
    };
    const int o0 = occ(reinterpret_cast<const void*>(&k_apply_special<Spec, kPtrCap, 1, false>));
    run("shipped persistent grid-stride", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
      k_apply_special<Spec, kPtrCap, 1, false><<<std::min<uint32_t>(g.total, o0 * sms), kThreads, 0, st>>>(t, gg);
    });
    run("one CTA per tile", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
      k_apply_special<Spec, kPtrCap, 1, false><<<g.total, kThreads, 0, st>>>(t, gg);
    });
    const int o4 = occ(reinterpret_cast<const void*>(&k_bal<4>));
    const int o6 = occ(reinterpret_cast<const void*>(&k_bal<6>));
    const int o8 = occ(reinterpret_cast<const void*>(&k_bal<8>));
    const int ob2 = occ(reinterpret_cast<const void*>(&k_bal2<2>));
    const int ob3 = occ(reinterpret_cast<const void*>(&k_bal2<3>));
    std::printf("# occupancy: shipped %d, bal4 %d, bal6 %d, bal8 %d, bal2x2 %d, bal2x3 %d\n", o0, o4, o6, o8, ob2,
                ob3);
    for (int m : {1, 2}) {
      char l[64];
      std::snprintf(l, sizeof l, "balanced minb4 grid %dx", m);
      run(l, [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bal<4><<<m * o4 * sms, kThreads, 0, st>>>(t, gg); });
    }
    run("balanced minb6", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bal<6><<<o6 * sms, kThreads, 0, st>>>(t, gg); });
    run("balanced minb8", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bal<8><<<o8 * sms, kThreads, 0, st>>>(t, gg); });
    run("balanced 2col minb2", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bal2<2><<<ob2 * sms, kThreads, 0, st>>>(t, gg); });
    run("balanced 2col minb3", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bal2<3><<<ob3 * sms, kThreads, 0, st>>>(t, gg); });
    // same-size copy (alg/2 read + alg/2 written) for the size ceiling
    {
      const uint64_t n16 = alg / 2 / 16;
      std::vector<PtrTable<kPtrCap>> dummy;
      auto cp = [&](const PtrTable<kPtrCap>& t, const TileGeom&) {
        const uint8_t* a = t.p[0];
        k_copy<<<4 * sms, kThreads, 0, st>>>(reinterpret_cast<const uint4*>(a),
                                            reinterpret_cast<uint4*>(const_cast<uint8_t*>(a) + alg / 2), n16);
      };
      run("copy kernel same bytes (no span)", cp);
    }
    for (auto b : bufs) CK(cudaFree(b));
  }
  return 0;
}
