// gs_kv.cuh -- device generators for the KV data model (kv_layout.hpp).
// Included by gs_capi.cu only (non-template kernels: one definition).
#pragma once

#include <cstdint>

namespace gsb {

// ---- synthetic KV (kv_layout.hpp:88-134) ----------------------------------
//
// Word i of a slice is splitmix64 evaluated at state0 + (i+1)*gamma, so the
// stream is embarrassingly parallel. Bytes of tokens >= valid in each
// (tensor, layer) block are zeroed in the same pass (pad_partial, :73-84).

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) k_ground_truth(uint8_t* __restrict__ out, uint64_t len,
                                                      uint64_t state0, uint64_t block,
                                                      uint64_t keep) {
  const uint64_t words = (len + 7) / 8;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < words;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t w = splitmix_mix(state0 + (i + 1) * 0x9E3779B97F4A7C15ull);
    const uint64_t pos = i * 8;
    if (keep < block) {
      for (int b = 0; b < 8; ++b)
        if ((pos + b) % block >= keep) w &= ~(0xFFull << (8 * b));
    }
    if (pos + 8 <= len && (reinterpret_cast<uintptr_t>(out) & 7) == 0) {
      *reinterpret_cast<uint64_t*>(out + pos) = w;
    } else {
      for (int b = 0; b < 8 && pos + b < len; ++b) out[pos + b] = static_cast<uint8_t>(w >> (8 * b));
    }
  }
}

// pad_partial on an existing slice: zero tokens [valid, m) of each block.
__global__ void __launch_bounds__(256) k_pad_partial(uint8_t* __restrict__ out, uint64_t len,
                                                     uint64_t block, uint64_t keep) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (i % block >= keep) out[i] = 0;
}

}  // namespace gsb
