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

// Shipped walk with load hints: HINT bit0 = L2::256B sector promotion on the
// streaming loads; bit1 = L2 prefetch of the CTA's next tile (one 128-B line
// per thread: 8 sources x 4 KiB = 256 lines) before this tile's loads.
__device__ __forceinline__ uint4 ld_stream256(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void prefetch_l2(const uint8_t* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
template <int HINT>
__global__ void __launch_bounds__(kThreads) k_hint(const PtrTable<kPtrCap> tab, const TileGeom g) {
  stamp_start(g);
  for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
    if (HINT & 2) {
      const uint32_t tn = t + gridDim.x;
      if (tn < g.total) {
        const uint32_t sn = tile_stripe(tn, g);
        const uint64_t offn = static_cast<uint64_t>(tn - sn * g.tps) * kTile + (threadIdx.x & 31) * 128;
        prefetch_l2(tab.p[sn * g.stride + (threadIdx.x >> 5)] + offn);
      }
    }
    const uint32_t s = tile_stripe(t, g);
    const uint32_t tin = t - s * g.tps;
    const uint64_t off = static_cast<uint64_t>(tin) * kTile + threadIdx.x * kVec;
    const int base = static_cast<int>(s) * g.stride;
    uint4 src[8], out[2];
#pragma unroll
    for (int j = 0; j < 8; ++j) src[j] = (HINT & 1) ? ld_stream256(tab.p[base + j] + off) : ld_stream(tab.p[base + j] + off);
    horner_apply<Spec>(src, out);
#pragma unroll
    for (int i = 0; i < 2; ++i) st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + off, out[i]);
  }
  stamp_end(g);
}

// Bulk (TMA) prefetch of the CTA's next tile into L2 by one thread per source.
__global__ void __launch_bounds__(kThreads) k_bulkpf(const PtrTable<kPtrCap> tab, const TileGeom g) {
  stamp_start(g);
  for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
    if (tn < g.total && threadIdx.x < 8) {
      const uint32_t sn = tile_stripe(tn, g);
      const uint64_t offn = static_cast<uint64_t>(tn - sn * g.tps) * kTile;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tab.p[sn * g.stride + threadIdx.x] + offn),
                   "r"(kTile));
    }
    const uint32_t s = tile_stripe(t, g);
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * kTile + threadIdx.x * kVec;
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

// Paged C2 (one 16-token block per slice, tile == page): the page's cache
// offset from the tile index alone -- s = t % S (page-major), q = t / S,
// kv = q / layers, l = q % layers -- with no per-thread page arithmetic.
__global__ void __launch_bounds__(kThreads) k_paged_page(const PtrTable<kPtrCap> tab, const TileGeom g) {
  stamp_start(g);
  for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
    const uint32_t q = fdiv(t, g.nstripes, g.nstripes_m);
    const uint32_t s = t - q * g.nstripes;
    const uint32_t kv = fdiv(q, g.src.layers, g.src.layers_m);
    const uint32_t l = q - kv * g.src.layers;
    const uint64_t soff = kv * g.src.kv_stride + l * g.src.layer_stride + threadIdx.x * kVec;
    const uint64_t doff = static_cast<uint64_t>(q) * kTile + threadIdx.x * kVec;
    const int base = static_cast<int>(s) * g.stride;
    uint4 src[8], out[2];
#pragma unroll
    for (int j = 0; j < 8; ++j) src[j] = ld_stream(tab.p[base + j] + soff);
    horner_apply<Spec>(src, out);
#pragma unroll
    for (int i = 0; i < 2; ++i) st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + doff, out[i]);
  }
  stamp_end(g);
}

static void paged_section(int sms, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1, unsigned long long* ts) {
  // 8 worker caches [layers=32][2][blocks][16 tok][256 B]; ring of 8 steps x 32 stripes = 256 blocks
  const int layers = 32, S = 32, sets = 8, blocks = S * sets;
  const uint64_t page = 16 * 256, plane = blocks * page, cache = 2ull * layers * plane;
  const uint64_t slice = 2ull * layers * page;  // 256 KiB
  std::vector<uint8_t*> caches(8);
  for (auto& c : caches) {
    CK(cudaMalloc(&c, cache));
    CK(cudaMemset(c, 7, cache));
  }
  uint8_t* par;
  CK(cudaMalloc(&par, static_cast<uint64_t>(sets) * S * 2 * slice));
  PageMap pm{};
  pm.page_bytes = page;
  pm.layers = layers;
  pm.token_bytes = 256;
  pm.valid_tokens = 16;
  pm.layer_stride = 2 * plane;
  pm.kv_stride = plane;
  pm.table = nullptr;
  pm.block_bytes = page;
  pm.page_m = fastdiv_magic(pm.page_bytes);
  pm.layers_m = fastdiv_magic(pm.layers);
  pm.block_m = fastdiv_magic(pm.block_bytes);
  std::vector<PtrTable<kPtrCap>> tabs(sets);
  for (int b = 0; b < sets; ++b)
    for (int s = 0; s < S; ++s) {
      for (int j = 0; j < 8; ++j) tabs[b].p[s * 10 + j] = caches[j] + static_cast<uint64_t>(b * S + s) * page;
      for (int i = 0; i < 2; ++i) tabs[b].p[s * 10 + 8 + i] = par + (static_cast<uint64_t>(b * S + s) * 2 + i) * slice;
    }
  TileGeom g{};
  g.len = slice;
  g.tps = static_cast<uint32_t>(slice / kTile);
  g.total = g.tps * S;
  g.stride = 10;
  g.out0 = 8;
  g.aligned = 1;
  g.tps_m = fastdiv_magic(g.tps);
  g.paged_slots = 0xFF;
  g.src = pm;
  g.nstripes = S;
  g.nstripes_m = fastdiv_magic(S);
  const uint64_t alg = static_cast<uint64_t>(S) * 10 * slice;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, &k_apply_special<Spec, kPtrCap, 1, true>, kThreads, 0));
  auto run = [&](const char* label, auto launch, TileGeom gv) {
    for (int b = 0; b < sets; ++b) launch(tabs[b], gv);
    CK(cudaStreamSynchronize(st));
    const int reps = 4;
    CK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r)
      for (int b = 0; b < sets; ++b) launch(tabs[b], gv);
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us_ev = ms * 1e3 / (reps * sets);
    double span = 0;
    for (int b = 0; b < sets; ++b) {
      unsigned long long init[2] = {~0ull, 0ull};
      CK(cudaMemcpyAsync(ts, init, sizeof(init), cudaMemcpyHostToDevice, st));
      TileGeom gg = gv;
      gg.tstamp = ts;
      launch(tabs[b], gg);
      unsigned long long out[2];
      CK(cudaMemcpyAsync(out, ts, sizeof(out), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      span += (out[1] - out[0]) * 1e-3;
    }
    span /= sets;
    std::printf("{\"geo\": \"C2 paged 16-tok blocks\", \"variant\": \"%s\", \"us_event\": %.2f, \"tbs_event\": %.3f, "
                "\"us_span\": %.2f, \"tbs_span\": %.3f}\n",
                label, us_ev, alg / us_ev * 1e-6, span, alg / span * 1e-6);
    std::fflush(stdout);
  };
  const int grid = std::min<int>(g.total, occ * sms);
  run("shipped paged page-major", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_apply_special<Spec, kPtrCap, 1, true><<<grid, kThreads, 0, st>>>(t, gg); }, g);
  TileGeom gs = g;
  gs.nstripes = 0;
  run("shipped paged stripe-major", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_apply_special<Spec, kPtrCap, 1, true><<<grid, kThreads, 0, st>>>(t, gg); }, gs);
  run("page-per-tile kernel", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_paged_page<<<grid, kThreads, 0, st>>>(t, gg); }, g);
  run("shipped paged page-major full grid", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
    k_apply_special<Spec, kPtrCap, 1, true><<<g.total, kThreads, 0, st>>>(t, gg); }, g);
  for (auto c : caches) CK(cudaFree(c));
  CK(cudaFree(par));
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
  if (getenv("PAGED_ONLY")) {
    paged_section(sms, st, e0, e1, ts);
    return 0;
  }
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
    {  // every CTA the same number of tiles: grid = ceil(total / ceil(total / (occ * sms)))
      const uint32_t full = std::min<uint32_t>(g.total, o0 * sms);
      const uint32_t per = (g.total + full - 1) / full;
      const uint32_t eq = (g.total + per - 1) / per;
      char l[96];
      std::snprintf(l, sizeof l, "shipped grid-stride, equal tiles per CTA (grid %u x %u tiles)", eq, per);
      run(l, [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
        k_apply_special<Spec, kPtrCap, 1, false><<<eq, kThreads, 0, st>>>(t, gg);
      });
      for (int m : {2, 3}) {  // more CTAs than resident slots: the tail is finer-grained
        std::snprintf(l, sizeof l, "shipped grid-stride, grid %u (%dx resident)", std::min<uint32_t>(g.total, m * full), m);
        run(l, [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
          k_apply_special<Spec, kPtrCap, 1, false><<<std::min<uint32_t>(g.total, m * full), kThreads, 0, st>>>(t, gg);
        });
      }
    }
    run("one CTA per tile", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) {
      k_apply_special<Spec, kPtrCap, 1, false><<<g.total, kThreads, 0, st>>>(t, gg);
    });
    const int oh = occ(reinterpret_cast<const void*>(&k_hint<3>));
    run("hint L2::256B", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_hint<1><<<std::min<uint32_t>(g.total, oh * sms), kThreads, 0, st>>>(t, gg); });
    run("hint prefetch next tile", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_hint<2><<<std::min<uint32_t>(g.total, oh * sms), kThreads, 0, st>>>(t, gg); });
    run("hint both", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_hint<3><<<std::min<uint32_t>(g.total, oh * sms), kThreads, 0, st>>>(t, gg); });
    run("hint both grid/2", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_hint<3><<<std::min<uint32_t>(g.total, oh * sms / 2), kThreads, 0, st>>>(t, gg); });
    run("bulk L2 prefetch next tile", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bulkpf<<<std::min<uint32_t>(g.total, oh * sms), kThreads, 0, st>>>(t, gg); });
    run("bulk L2 prefetch grid/2", [&](const PtrTable<kPtrCap>& t, const TileGeom& gg) { k_bulkpf<<<std::min<uint32_t>(g.total, oh * sms / 2), kThreads, 0, st>>>(t, gg); });
    if (getenv("SKIP_BAL")) { for (auto b : bufs) CK(cudaFree(b)); continue; }
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
