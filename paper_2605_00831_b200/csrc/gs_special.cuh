// gs_special.cuh -- compile-time specialised kernels (Horner back end) and
// the registry the host dispatcher consults.
//
// A specialisation is keyed by (decoder?, kind, n, k, canonical lost mask).
// Encoders: the scheme's Cauchy / all-ones matrix. Decoders: the folded
// decode matrix of coding.hpp:535-566 for one erasure pattern, evaluated by
// the compiler. Patterns that pick the same parity rows for the same lost
// data shards share one canonical mask (see canonical_mask()).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "gs_kernels.cuh"

namespace gsb {

using LaunchFn = cudaError_t (*)(const void* const* ptrs, int count, const TileGeom& g, int grid,
                                 cudaStream_t st);
using KernelAddr = const void*;
using BulkLaunchFn = cudaError_t (*)(const void* const* ptrs, int count, const TileGeom& g, int grid,
                                     cudaStream_t st, int stages, size_t smem);

// Pointer-table capacity of one launch (pointers + TileGeom fit the classic
// 4 KiB kernel-parameter space).
constexpr int kPtrCap = 488;
// 16-byte groups per thread per source per tile of the specialised kernels.
constexpr int kSpecialU = 1;
// Consumer warps and 16-byte groups per consumer thread of the bulk variant.
constexpr int kBulkCW = 16;
constexpr int kBulkU = 1;
constexpr int kBulkThreads = (kBulkCW + 1) * 32;
constexpr int kBulkTile = kBulkCW * 32 * kVec * kBulkU;
constexpr size_t kBulkSmemHeader = 2 * bulk::kMaxStages * sizeof(uint64_t) + 112;
constexpr size_t kBulkSmemMax = 224 * 1024;

struct SpecialEntry {
  bool decoder;
  int kind, n, k;
  uint64_t mask;
  LaunchFn launch;
  KernelAddr kernel;
  LaunchFn launch_paged;    // same arithmetic, paged-KV address mapping
  KernelAddr kernel_paged;
  int tile;  // bytes of every shard per CTA tile
  // bulk-copy pipelined variant (k_apply_special_bulk)
  BulkLaunchFn launch_bulk;
  KernelAddr kernel_bulk;
  int tile_bulk;
  int used_cols;  // sources streamed per tile
};

constexpr int popcount64(uint64_t x) {
  int c = 0;
  while (x) {
    c += static_cast<int>(x & 1u);
    x >>= 1;
  }
  return c;
}

// The decode depends only on the lost data shards and on which parity rows
// the first-e-surviving rule picks. Canonical mask = lost data bits + the
// lost parity rows that were skipped before the last chosen row.
GS_HD constexpr uint64_t canonical_mask(int kind, int n, int k, uint64_t mask) {
  const uint64_t data_bits = mask & ((n >= 64 ? ~0ull : (1ull << n) - 1));
  if (kind != kReedSolomon) return data_bits;
  const int e = popcount64(data_bits);
  uint64_t out = data_bits;
  int chosen = 0;
  for (int i = 0; i < k && chosen < e; ++i) {
    if ((mask >> (n + i)) & 1u)
      out |= 1ull << (n + i);
    else
      ++chosen;
  }
  return out;
}

template <int KIND, int N, int K>
struct EncSpec {
  static constexpr int NS = N, NO = K;
  GS_HD static constexpr CoefMatrix matrix() { return encode_matrix(KIND, N, K); }
};

template <int KIND, int N, int K, uint64_t MASK>
struct DecSpec {
  static constexpr int NS = N + K;
  static constexpr int NO = popcount64(MASK & ((1ull << N) - 1));
  GS_HD static constexpr CoefMatrix matrix() { return decode_plan_mask(KIND, N, K, MASK).m; }
};

template <class Spec, int CAP, bool PAGED>
cudaError_t launch_special(const void* const* ptrs, int count, const TileGeom& g, int grid,
                           cudaStream_t st) {
  PtrTable<CAP> tab;
  for (int i = 0; i < count; ++i) tab.p[i] = static_cast<const uint8_t*>(ptrs[i]);
  k_apply_special<Spec, CAP, kSpecialU, PAGED><<<grid, kThreads, 0, st>>>(tab, g);
  return cudaGetLastError();
}

template <class Spec, int CAP>
cudaError_t launch_special_bulk(const void* const* ptrs, int count, const TileGeom& g, int grid,
                                cudaStream_t st, int stages, size_t smem) {
  PtrTable<CAP> tab;
  for (int i = 0; i < count; ++i) tab.p[i] = static_cast<const uint8_t*>(ptrs[i]);
  k_apply_special_bulk<Spec, CAP, kBulkCW, kBulkU><<<grid, kBulkThreads, smem, st>>>(tab, g, stages);
  return cudaGetLastError();
}

template <class Spec>
SpecialEntry make_entry(bool decoder, int kind, int n, int k, uint64_t mask) {
  SpecialEntry e;
  e.decoder = decoder;
  e.kind = kind;
  e.n = n;
  e.k = k;
  e.mask = mask;
  e.launch = &launch_special<Spec, kPtrCap, false>;
  e.kernel = reinterpret_cast<KernelAddr>(&k_apply_special<Spec, kPtrCap, kSpecialU, false>);
  e.launch_paged = &launch_special<Spec, kPtrCap, true>;
  e.kernel_paged = reinterpret_cast<KernelAddr>(&k_apply_special<Spec, kPtrCap, kSpecialU, true>);
  e.tile = kThreads * kVec * kSpecialU;
  e.launch_bulk = &launch_special_bulk<Spec, kPtrCap>;
  e.kernel_bulk = reinterpret_cast<KernelAddr>(&k_apply_special_bulk<Spec, kPtrCap, kBulkCW, kBulkU>);
  e.tile_bulk = kBulkTile;
  e.used_cols = bulk::used_cols<Spec>().n;
  return e;
}

template <int KIND, int N, int K>
void add_encoder(SpecialEntry* out, int& cnt) {
  out[cnt++] = make_entry<EncSpec<KIND, N, K>>(false, KIND, N, K, 0);
}

template <int KIND, int N, int K, int E, uint64_t MASK>
void add_decoder_if_canonical(SpecialEntry* out, int& cnt) {
  constexpr int tol = KIND == kReedSolomon ? K : 1;
  constexpr uint64_t data_bits = MASK & ((1ull << N) - 1);
  if constexpr (popcount64(MASK) <= tol && data_bits != 0 && (E == 0 || popcount64(data_bits) == E) &&
                canonical_mask(KIND, N, K, MASK) == MASK &&
                decode_plan_mask(KIND, N, K, MASK).ok) {
    out[cnt++] = make_entry<DecSpec<KIND, N, K, MASK>>(true, KIND, N, K, MASK);
  }
}

template <int KIND, int N, int K, int E, uint64_t... M>
void add_decoders_impl(SpecialEntry* out, int& cnt, std::integer_sequence<uint64_t, M...>) {
  (add_decoder_if_canonical<KIND, N, K, E, M>(out, cnt), ...);
}

// All canonical patterns of the scheme (E = 0) or only those losing exactly
// E data shards (lets one scheme's decoders spread over several TUs).
template <int KIND, int N, int K, int E = 0>
void add_decoders(SpecialEntry* out, int& cnt) {
  add_decoders_impl<KIND, N, K, E>(out, cnt, std::make_integer_sequence<uint64_t, (1ull << (N + K))>{});
}

// Filled by gs_special.cu.
int special_registry(const SpecialEntry** out);

}  // namespace gsb
