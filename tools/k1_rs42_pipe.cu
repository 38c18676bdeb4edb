// k1_rs42_pipe.cu -- standalone A/B probe for K1 RS(4,2) (C1 geometry:
// 4 x 128 MiB -> 2 x 128 MiB) and RS(8,2) (C3 chunk): the shipped register
// kernel vs a software-pipelined walk that issues the NEXT tile's loads into
// a second register set before the Horner arithmetic of the current tile
// (RS(4,2) is twice the arithmetic per input byte of RS(8,2), so a warp
// computing has no loads in flight unless it prefetched). Not the product.
//
//   nvcc -std=c++20 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
//        -I paper_2605_00831_b200/csrc tools/k1_rs42_pipe.cu -o tools/k1_rs42_pipe.bin
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gs_special.cuh"

using namespace gsb;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

template <class Spec, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_pipe(const PtrTable<kPtrCap> tab, const TileGeom g) {
  stamp_start(g);
  uint4 cur[Spec::NS], nxt[Spec::NS];
  auto coords = [&](uint32_t t, uint64_t& off, int& base) {
    const uint32_t s = tile_stripe(t, g);
    off = static_cast<uint64_t>(t - s * g.tps) * kTile + threadIdx.x * kVec;
    base = static_cast<int>(s) * g.stride;
  };
  uint32_t t = blockIdx.x;
  uint64_t off = 0;
  int base = 0;
  if (t < g.total) {
    coords(t, off, base);
#pragma unroll
    for (int j = 0; j < Spec::NS; ++j) cur[j] = ld_stream(tab.p[base + j] + off);
  }
  for (; t < g.total; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
    uint64_t offn = 0;
    int basen = 0;
    if (tn < g.total) {
      coords(tn, offn, basen);
#pragma unroll
      for (int j = 0; j < Spec::NS; ++j) nxt[j] = ld_stream(tab.p[basen + j] + offn);
    }
    uint4 out[Spec::NO];
    horner_apply<Spec>(cur, out);
#pragma unroll
    for (int i = 0; i < Spec::NO; ++i) st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + off, out[i]);
#pragma unroll
    for (int j = 0; j < Spec::NS; ++j) cur[j] = nxt[j];
    off = offn;
    base = basen;
  }
  stamp_end(g);
}

template <class Spec>
void geo(const char* name, int n, uint64_t len, int stripes, int sms, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1,
         unsigned long long* ts) {
  const int k = 2, w = n + k, sets = 4;
  const uint64_t alg = static_cast<uint64_t>(stripes) * w * len;
  std::vector<PtrTable<kPtrCap>> tabs(sets);
  std::vector<uint8_t*> bufs;
  for (int s = 0; s < sets; ++s) {
    uint8_t* b;
    CK(cudaMalloc(&b, alg));
    CK(cudaMemset(b, s + 1, alg));
    bufs.push_back(b);
    for (int r = 0; r < stripes; ++r)
      for (int j = 0; j < w; ++j) tabs[s].p[r * w + j] = b + (static_cast<uint64_t>(r) * w + j) * len;
  }
  TileGeom g{};
  g.len = len;
  g.tps = static_cast<uint32_t>(len / kTile);
  g.total = g.tps * stripes;
  g.stride = w;
  g.out0 = n;
  g.aligned = 1;
  g.tps_m = fastdiv_magic(g.tps);
  auto occ = [&](const void* kf) {
    int b = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kf, kThreads, 0));
    return b;
  };
  auto run = [&](const char* label, auto launch) {
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
    std::printf("{\"geo\": \"%s\", \"variant\": \"%s\", \"us_event\": %.2f, \"tbs_event\": %.3f, \"us_span\": %.2f, "
                "\"tbs_span\": %.3f}\n",
                name, label, us_ev, alg / us_ev * 1e-6, span, alg / span * 1e-6);
    std::fflush(stdout);
  };
  const int o0 = occ(reinterpret_cast<const void*>(&k_apply_special<Spec, kPtrCap, 1, false>));
  run("shipped register kernel", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_apply_special<Spec, kPtrCap, 1, false><<<std::min<uint32_t>(g.total, o0 * sms), kThreads, 0, st>>>(t, gg);
  });
  const int o1 = occ(reinterpret_cast<const void*>(&k_pipe<Spec, 1>));
  const int o4 = occ(reinterpret_cast<const void*>(&k_pipe<Spec, 4>));
  const int o5 = occ(reinterpret_cast<const void*>(&k_pipe<Spec, 5>));
  std::printf("# %s occupancy: shipped %d, pipe %d / minb4 %d / minb5 %d\n", name, o0, o1, o4, o5);
  run("pipelined next-tile loads", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_pipe<Spec, 1><<<std::min<uint32_t>(g.total, o1 * sms), kThreads, 0, st>>>(t, gg);
  });
  run("pipelined, minBlocks 4", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_pipe<Spec, 4><<<std::min<uint32_t>(g.total, o4 * sms), kThreads, 0, st>>>(t, gg);
  });
  run("pipelined, minBlocks 5", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_pipe<Spec, 5><<<std::min<uint32_t>(g.total, o5 * sms), kThreads, 0, st>>>(t, gg);
  });
  for (auto b : bufs) CK(cudaFree(b));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* ts;
  CK(cudaMalloc(&ts, 2 * sizeof(unsigned long long)));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  geo<EncSpec<kReedSolomon, 4, 2>>("C1 RS(4,2) 4x128MiB", 4, 128ull << 20, 1, sms, st, e0, e1, ts);
  geo<EncSpec<kReedSolomon, 8, 2>>("C3 RS(8,2) 8x40MiB piece", 8, 40ull << 20, 1, sms, st, e0, e1, ts);
  geo<EncSpec<kReedSolomon, 8, 2>>("C2 RS(8,2) 32x8x256KiB", 8, 256ull << 10, 32, sms, st, e0, e1, ts);
  return 0;
}
